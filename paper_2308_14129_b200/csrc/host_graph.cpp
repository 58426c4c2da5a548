// Stream synthesis, chronological split, time-decay centrality and hub
// selection. Host C++; every result is bit-identical to the reference
// (tests/test_host_parity.py checks against oracle/_ref and golden vectors).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "host.hpp"

namespace spd {

// Preferential-attachment TIG with the shifted-linear kernel deg + a
// (graph_io.cpp:175-250). Same draw sequence as the reference so the stream is
// identical edge for edge; the working set is kept flat (u32 degrees and pool)
// so the 191M-edge GDELT shape stays cache-friendlier than vector<size_t>.
void gen_powerlaw(NodeId nodes, std::uint64_t edges, double alpha, std::uint64_t seed,
                  spd_edge* out) {
    if (nodes < 2 || edges < 1 || !(alpha > 1.0))
        data_error("InvalidParams", "need nodes >= 2, edges >= 1, alpha > 1");
    const std::uint64_t m_per = std::max<std::uint64_t>(1, edges / nodes);
    double a = (alpha - 3.0) * static_cast<double>(m_per);
    const double a_min = -0.95 * static_cast<double>(m_per);
    if (a < a_min) a = a_min;
    const double accept_ceil = a > 0.0 ? 1.0 + a / static_cast<double>(m_per) : 1.0;

    Rng rng(seed);
    std::vector<std::uint32_t> deg(nodes, 0);
    std::vector<NodeId> pool;
    pool.reserve(2 * edges);
    std::uint64_t count = 0;
    auto push = [&](NodeId u, NodeId v) {
        out[count] = spd_edge{u, v, static_cast<double>(count + 1)};
        ++count;
        ++deg[u];
        ++deg[v];
        pool.push_back(u);
        pool.push_back(v);
    };
    auto draw_pref = [&]() -> NodeId {
        for (int tries = 0; tries < 64; ++tries) {
            const NodeId u = pool[rng.below(pool.size())];
            const double ratio = (1.0 + a / static_cast<double>(deg[u])) / accept_ceil;
            if (rng.unit() < ratio) return u;
        }
        return pool[rng.below(pool.size())];
    };

    for (std::uint64_t r = 0; r < m_per && count < edges; ++r) push(0, 1);
    for (NodeId v = 2; v < nodes && count < edges; ++v) {
        for (std::uint64_t r = 0; r < m_per && count < edges; ++r) {
            NodeId u = draw_pref();
            for (int tries = 0; u == v && tries < 64; ++tries) u = draw_pref();
            if (u == v) u = (v + 1) % 2;
            push(v, u);
        }
    }
    while (count < edges) {
        const NodeId u = draw_pref();
        NodeId v = draw_pref();
        for (int tries = 0; v == u && tries < 64; ++tries) v = draw_pref();
        if (v == u) v = (u + 1) % nodes;
        push(u, v);
    }
    rng.shuffle(out, edges);
    for (std::uint64_t t = 0; t < edges; ++t) out[t].ts = static_cast<double>(t + 1);
}

// graph_io.cpp:156-173: floor(f * n) positional cut points.
void chrono_split_sizes(std::uint64_t n, double f_train, double f_val, std::uint64_t* n_train,
                        std::uint64_t* n_val, std::uint64_t* n_test) {
    if (!(f_train > 0.0 && f_train < 1.0) || f_val < 0.0 || f_train + f_val > 1.0)
        data_error("InvalidFractions", "need 0 < train < 1, val >= 0, train + val <= 1");
    const auto tr = static_cast<std::uint64_t>(std::floor(f_train * static_cast<double>(n)));
    const auto va = static_cast<std::uint64_t>(std::floor(f_val * static_cast<double>(n)));
    *n_train = tr;
    *n_val = va;
    *n_test = n - tr - va;
}

// Eq. 1 (centrality.cpp:27-52): per-role weight exp(beta*(t_norm - top)),
// accumulated in stream order — the f64 sum is order dependent, so the loop
// keeps the reference's order exactly (src role, then dst role, per edge).
void compute_centrality(const Stream& s, double beta, bool normalize, double* cent,
                        double* t_max_out) {
    if (!(beta > 0.0 && beta < 1.0)) data_error("BetaOutOfRange", "beta must lie in (0,1)");
    std::fill(cent, cent + s.node_count, 0.0);
    *t_max_out = 0.0;
    if (s.n == 0) return;
    const double t_min = s.e[0].ts;
    const double span = s.t_max - t_min;
    const bool scale = normalize && span > 0.0;
    const double top = scale ? (s.t_max - t_min) / span : s.t_max;
    *t_max_out = top;
    for (std::uint64_t k = 0; k < s.n; ++k) {
        const double t = scale ? (s.e[k].ts - t_min) / span : s.e[k].ts;
        const double w = std::exp(beta * (t - top));
        cent[s.e[k].src] += w;
        cent[s.e[k].dst] += w;
    }
}

void compute_degree_centrality(const Stream& s, double* cent) {  // centrality.cpp:54-64
    std::fill(cent, cent + s.node_count, 0.0);
    for (std::uint64_t k = 0; k < s.n; ++k) {
        cent[s.e[k].src] += 1.0;
        cent[s.e[k].dst] += 1.0;
    }
}

// Top floor(k * base) active nodes by (centrality desc, id asc), returned
// ascending (centrality.cpp:66-88). The comparator is a strict total order,
// so nth_element + sort selects exactly the reference's set.
std::vector<NodeId> select_hubs(const double* cent, NodeId node_count, double k, bool base_all) {
    if (!(k >= 0.0 && k <= 1.0)) data_error("InvalidParams", "k must lie in [0,1]");
    std::vector<NodeId> active;
    active.reserve(node_count);
    for (NodeId i = 0; i < node_count; ++i)
        if (cent[i] > 0.0) active.push_back(i);
    const std::uint64_t base = base_all ? node_count : active.size();
    const auto want = static_cast<std::uint64_t>(std::floor(k * static_cast<double>(base)));
    const std::uint64_t take = std::min<std::uint64_t>(want, active.size());
    auto before = [&](NodeId a, NodeId b) {
        if (cent[a] != cent[b]) return cent[a] > cent[b];
        return a < b;
    };
    if (take < active.size())
        std::nth_element(active.begin(), active.begin() + take, active.end(), before);
    active.resize(take);
    std::sort(active.begin(), active.end());
    return active;
}

// 64-bit FNV-1a over the little-endian image of each row followed by its
// timestamp (digest.hpp:12-37, pac_sim.cpp:18-26).
std::string fnv1a64_hex(const double* state, std::uint64_t rows, int d, const double* last_ts) {
    std::uint64_t h = 14695981039346656037ULL;
    auto absorb = [&](double v) {
        std::uint64_t bits;
        std::memcpy(&bits, &v, 8);
        for (int i = 0; i < 8; ++i) {
            h ^= static_cast<std::uint8_t>(bits >> (8 * i));
            h *= 1099511628211ULL;
        }
    };
    for (std::uint64_t i = 0; i < rows; ++i) {
        for (int r = 0; r < d; ++r) absorb(state[i * d + r]);
        absorb(last_ts[i]);
    }
    static const char* digits = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i, h >>= 4) out[i] = digits[h & 0xF];
    return out;
}

}  // namespace spd
