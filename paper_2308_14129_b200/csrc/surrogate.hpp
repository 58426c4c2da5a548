// Parity mode: the reference's fixed surrogate MSG/UPD model and its PAC
// lockstep trainer on the device (pac_sim.cpp:13-338).
#pragma once

#include <string>
#include <vector>

#include "cuda_util.hpp"
#include "host.hpp"

namespace spd {

// Device-resident MemoryStore (pac_sim.hpp:19-39): f64 state rows + f64 clock.
struct MemStore {
    int device = 0;
    NodeId node_count = 0;
    int d = 0;
    DevBuf<double> state;   // node_count * d
    DevBuf<double> last_ts; // node_count
    MemStore(NodeId n, int d_, int dev);
    void reset(cudaStream_t s = 0);
    void copy_from(const MemStore& o, cudaStream_t s = 0);
    std::string digest() const;
};

// ModelParams (pac_sim.hpp:47-55) on the host.
struct SurrogateModel {
    int d = 8;
    double gamma = 0.5;
    std::vector<double> w_m;   // d x 3d row-major
    std::vector<double> omega; // d
    static SurrogateModel seeded(int d, std::uint64_t seed);
};

struct EpochOut {
    std::vector<std::uint64_t> batches, loops;
    std::uint64_t sync_events = 0;
    std::vector<std::string> digests;
    std::vector<std::uint64_t> log_steps;  // 4 per record
    std::vector<std::pair<int, std::string>> snaps;
    bool want_log = false;
};

void surrogate_model_update(MemStore& m, const spd_edge* e, std::uint64_t n,
                            const SurrogateModel& model);
void surrogate_sync_shared(const std::vector<MemStore*>& mems, const std::vector<NodeId>& shared,
                           bool average);
void surrogate_run_epoch(const std::vector<const std::vector<spd_edge>*>& edges,
                         const std::vector<MemStore*>& mems, const SurrogateModel& model,
                         const std::vector<NodeId>& shared, bool average,
                         std::uint64_t batch_size, EpochOut& out);

}  // namespace spd
