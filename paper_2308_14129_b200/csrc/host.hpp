// Host-side core of the SPEED hot path (C++20, no device code).
//
// These are the reference's L0-L4 host algorithms re-designed for feeding a
// B200: flat arrays instead of vector-of-vectors, per-node partition bitsets
// instead of A-set vectors, one pass over the stream for all partitions'
// induction, and local-id compaction + per-node time-sorted CSR for the
// device. Results are bit-identical to the reference (see tests/).
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "speed_c.h"

namespace spd {

using NodeId = std::uint32_t;
using PartId = std::int32_t;
inline constexpr PartId kDiscarded = -1;  // types.hpp:12

// Error types carrying the reference's code strings (errors.hpp:10-32).
struct Error : std::runtime_error {
    int status;
    std::string code;
    Error(int st, std::string c, const std::string& d)
        : std::runtime_error(d), status(st), code(std::move(c)) {}
};
[[noreturn]] inline void data_error(const std::string& code, const std::string& d) {
    throw Error(SPD_DATA, code, d);
}
[[noreturn]] inline void internal_error(const std::string& code, const std::string& d) {
    throw Error(SPD_INTERNAL, code, d);
}
[[noreturn]] inline void usage_error(const std::string& d) { throw Error(SPD_USAGE, "Usage", d); }

// ---------------------------------------------------------------- stream
struct Stream {
    const spd_edge* e = nullptr;
    std::uint64_t n = 0;
    NodeId node_count = 0;
    double t_max = 0.0;
};

void gen_powerlaw(NodeId nodes, std::uint64_t edges, double alpha, std::uint64_t seed,
                  spd_edge* out);
void chrono_split_sizes(std::uint64_t n, double f_train, double f_val, std::uint64_t* n_train,
                        std::uint64_t* n_val, std::uint64_t* n_test);

// ------------------------------------------------------------ centrality
void compute_centrality(const Stream& s, double beta, bool normalize, double* cent,
                        double* t_max_out);
void compute_degree_centrality(const Stream& s, double* cent);
std::vector<NodeId> select_hubs(const double* cent, NodeId node_count, double k, bool base_all);

// ----------------------------------------------------------- partitioner
struct PartitionerConfig {
    int num_parts = 1;
    double lambda = 1.0;
    double epsilon = 1.0;
    std::vector<double> cent;          // CentralityTable::cent
    std::vector<std::uint8_t> is_hub;  // dense over node_count
    double k = 0.0;
    double cent_of(NodeId i) const { return i < cent.size() ? cent[i] : 0.0; }
    bool hub(NodeId i) const { return i < is_hub.size() && is_hub[i]; }
};

struct Assignment {
    int num_parts = 1;
    NodeId node_count = 0;
    std::vector<PartId> edge_part;       // kDiscarded for dropped edges
    std::vector<std::uint64_t> np_off;   // node_parts CSR (node_count + 1)
    std::vector<PartId> np_parts;
    std::vector<NodeId> shared;          // ascending
    std::uint64_t discards = 0;
    double k_eff = 0.0;
};

Assignment partition_stream(const Stream& s, const PartitionerConfig& cfg, bool unrestricted);

// --------------------------------------------------------- eval routing
struct EvalRouting {
    std::vector<std::vector<std::uint64_t>> lists[2];  // [val/test][part]
    std::uint64_t unroutable[2] = {0, 0};
};
EvalRouting assign_eval_edges(const Stream& val, const Stream& test, const Assignment& a);

// ------------------------------------------------------------- subgraphs
struct SubGraph {
    std::vector<NodeId> nodes;           // ascending global ids
    std::vector<spd_edge> edges;         // time-ordered, global ids
    std::vector<std::uint64_t> eids;     // stream position of each edge
};
struct SubGraphs {
    std::vector<SubGraph> g;
};

// node membership given as per-partition node lists or per-node part lists
SubGraphs induce_from_node_parts(const Stream& s, const std::uint64_t* np_off,
                                 const PartId* np_parts, NodeId np_count, int num_parts);
SubGraphs induce_from_groups(const Stream& s, const std::uint64_t* off, const NodeId* nodes,
                             int n_groups, std::vector<std::uint8_t>* in_any);

std::vector<std::vector<NodeId>> shuffle_combine(const std::vector<std::vector<NodeId>>& small,
                                                 int num_workers, std::uint64_t epoch_seed);

// ------------------------------------------------------------- helpers
// mt19937_64 draw helpers with the reference's portable semantics
// (rng.hpp:13-41): results do not depend on std::*_distribution.
struct Rng {
    std::mt19937_64 g;  // the engine itself is fully specified by the standard
    explicit Rng(std::uint64_t seed) : g(seed) {}
    std::uint64_t next() { return g(); }
    double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    std::uint64_t below(std::uint64_t n) { return g() % n; }
    template <class T>
    void shuffle(T* v, std::uint64_t n) {  // Fisher-Yates, rng.hpp:36-41 draw order
        for (std::uint64_t i = n; i > 1; --i) std::swap(v[i - 1], v[below(i)]);
    }
};

std::string fnv1a64_hex(const double* state, std::uint64_t rows, int d, const double* last_ts);

}  // namespace spd
