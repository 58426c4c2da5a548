// SEP streaming edge partitioner (Alg. 1; partitioner.cpp:11-163)
// and eval-edge routing (partitioner.cpp:212-242).
//
// Same five-case dispatch, same greedy score arithmetic (operation order kept
// so the f64 score is bit-identical) and same lowest-index tie break as the
// reference. What differs is the state layout: A(i) is a per-node partition
// bitset plus the first-assigned partition (A(i).front() in the reference),
// and max/min partition sizes are maintained incrementally instead of an
// O(P) scan per edge.
#include <algorithm>
#include <string>

#include "host.hpp"

namespace spd {

namespace {

struct State {
    int P;
    int words;
    std::vector<std::uint64_t> bits;  // node_count * words
    std::vector<PartId> first;        // A(i).front(), -1 when empty
    std::vector<std::uint16_t> count; // |A(i)| (capped, only >1 matters)
    std::vector<std::uint64_t> sizes;
    std::uint64_t maxsize = 0, minsize = 0;
    int n_at_min;

    State(NodeId n, int parts)
        : P(parts), words((parts + 63) / 64), bits(std::size_t(n) * ((parts + 63) / 64), 0),
          first(n, -1), count(n, 0), sizes(parts, 0), n_at_min(parts) {}

    bool in_a(NodeId i, PartId p) const {
        return (bits[std::size_t(i) * words + (p >> 6)] >> (p & 63)) & 1ULL;
    }
    void add_to_a(NodeId i, PartId p) {
        std::uint64_t& w = bits[std::size_t(i) * words + (p >> 6)];
        const std::uint64_t m = 1ULL << (p & 63);
        if (w & m) return;
        w |= m;
        if (first[i] < 0) first[i] = p;
        if (count[i] < 0xFFFF) ++count[i];
    }
    void add_edge_to(PartId p) {
        const std::uint64_t old = sizes[p]++;
        if (sizes[p] > maxsize) maxsize = sizes[p];
        if (old == minsize && --n_at_min == 0) {
            minsize = *std::min_element(sizes.begin(), sizes.end());
            n_at_min = static_cast<int>(std::count(sizes.begin(), sizes.end(), minsize));
        }
    }
};

// h(x,p) terms and the balance term in the reference's evaluation order
// (partitioner.cpp:27-42).
struct PairScore {
    double hi, hj;
    PairScore(const PartitionerConfig& cfg, NodeId i, NodeId j) {
        const double ci = cfg.cent_of(i);
        const double cj = cfg.cent_of(j);
        const double sum = ci + cj;
        const double theta_i = sum > 0.0 ? ci / sum : 0.5;
        const double theta_j = sum > 0.0 ? cj / sum : 0.5;
        hi = 1.0 + (1.0 - theta_i);
        hj = 1.0 + (1.0 - theta_j);
    }
};

inline double score_of(const PairScore& ps, NodeId i, NodeId j, PartId p, const State& st,
                       const PartitionerConfig& cfg) {
    double h = 0.0;
    if (st.in_a(i, p)) h += ps.hi;
    if (st.in_a(j, p)) h += ps.hj;
    const double spread = static_cast<double>(st.maxsize - st.minsize);
    const double slack = static_cast<double>(st.maxsize - st.sizes[p]);
    return h + cfg.lambda * slack / (cfg.epsilon + spread);
}

PartId argmax_all(NodeId i, NodeId j, const State& st, const PartitionerConfig& cfg) {
    const PairScore ps(cfg, i, j);
    PartId best = 0;
    double best_score = score_of(ps, i, j, 0, st, cfg);
    for (PartId p = 1; p < cfg.num_parts; ++p) {
        const double sc = score_of(ps, i, j, p, st, cfg);
        if (sc > best_score) {  // strict: ties keep the lowest index
            best = p;
            best_score = sc;
        }
    }
    return best;
}

}  // namespace

Assignment partition_stream(const Stream& s, const PartitionerConfig& cfg_in, bool unrestricted) {
    if (cfg_in.num_parts < 1 || !(cfg_in.lambda > 0.0) || !(cfg_in.epsilon > 0.0))
        data_error("InvalidParams", "need num_parts >= 1, lambda > 0, epsilon > 0");
    for (std::uint64_t e = 1; e < s.n; ++e)
        if (s.e[e].ts < s.e[e - 1].ts)
            data_error("UnsortedStream", "edge " + std::to_string(e) + " is out of order");

    const PartitionerConfig* cfgp = &cfg_in;
    PartitionerConfig open;
    if (unrestricted) {  // partitioner.cpp:156-163: every node is a hub
        open = cfg_in;
        open.is_hub.assign(s.node_count, 1);
        open.k = 1.0;
        cfgp = &open;
    }
    const PartitionerConfig& cfg = *cfgp;
    for (std::uint64_t e = 0; e < s.n; ++e)
        if (s.e[e].src >= s.node_count || s.e[e].dst >= s.node_count)
            data_error("InvalidParams", "edge " + std::to_string(e) + " names a node >= node_count");

    State st(s.node_count, cfg.num_parts);
    Assignment a;
    a.num_parts = cfg.num_parts;
    a.node_count = s.node_count;
    a.k_eff = cfg.k;
    a.edge_part.assign(s.n, kDiscarded);

    for (std::uint64_t e = 0; e < s.n; ++e) {
        const NodeId i = s.e[e].src;
        const NodeId j = s.e[e].dst;
        const bool ai = st.first[i] >= 0;
        const bool aj = st.first[j] >= 0;
        const bool hi = cfg.hub(i);
        const bool hj = cfg.hub(j);
        PartId target;
        if (!ai || !aj) {                       // Cases 4/5
            if (ai && !hi) target = st.first[i];
            else if (aj && !hj) target = st.first[j];
            else target = argmax_all(i, j, st, cfg);
        } else if (hi != hj) {                  // Case 1: follow the non-hub
            target = hi ? st.first[j] : st.first[i];
        } else if (hi) {                        // Case 2: two hubs
            target = argmax_all(i, j, st, cfg);
        } else {                                // Case 3: two resident non-hubs
            if (st.first[i] != st.first[j]) {
                ++a.discards;
                continue;
            }
            target = st.first[i];
        }
        a.edge_part[e] = target;
        st.add_to_a(i, target);
        st.add_to_a(j, target);
        if (!hi && st.count[i] > 1)
            internal_error("ResidencyViolation", "non-hub " + std::to_string(i) + " replicated");
        if (!hj && st.count[j] > 1)
            internal_error("ResidencyViolation", "non-hub " + std::to_string(j) + " replicated");
        st.add_edge_to(target);
    }

    // finish (partitioner.cpp:70-89): multi-resident nodes are shared and
    // join every partition; the rest keep their single home.
    a.np_off.assign(std::size_t(s.node_count) + 1, 0);
    a.np_parts.reserve(s.node_count);
    for (NodeId i = 0; i < s.node_count; ++i) {
        if (st.count[i] > 1) {
            a.shared.push_back(i);
            for (PartId p = 0; p < cfg.num_parts; ++p) a.np_parts.push_back(p);
        } else if (st.count[i] == 1) {
            a.np_parts.push_back(st.first[i]);
        }
        a.np_off[i + 1] = a.np_parts.size();
    }
    return a;
}

// Val/test edge -> every partition holding both endpoints
// (partitioner.cpp:212-242), via per-node partition bitsets.
EvalRouting assign_eval_edges(const Stream& val, const Stream& test, const Assignment& a) {
    const int P = a.num_parts;
    const int words = (P + 63) / 64;
    const NodeId N = a.node_count;
    std::vector<std::uint64_t> bits(std::size_t(N) * words, 0);
    for (NodeId i = 0; i < N; ++i)
        for (std::uint64_t k = a.np_off[i]; k < a.np_off[i + 1]; ++k) {
            const PartId p = a.np_parts[k];
            if (p >= 0 && p < P) bits[std::size_t(i) * words + (p >> 6)] |= 1ULL << (p & 63);
        }
    EvalRouting r;
    const Stream* ss[2] = {&val, &test};
    for (int w = 0; w < 2; ++w) {
        r.lists[w].assign(P, {});
        for (std::uint64_t e = 0; e < ss[w]->n; ++e) {
            const NodeId i = ss[w]->e[e].src;
            const NodeId j = ss[w]->e[e].dst;
            bool routed = false;
            if (i < N && j < N) {
                for (int wd = 0; wd < words; ++wd) {
                    std::uint64_t m = bits[std::size_t(i) * words + wd] &
                                      bits[std::size_t(j) * words + wd];
                    while (m) {
                        const int b = __builtin_ctzll(m);
                        m &= m - 1;
                        r.lists[w][wd * 64 + b].push_back(e);
                        routed = true;
                    }
                }
            }
            if (!routed) ++r.unroutable[w];
        }
    }
    return r;
}

}  // namespace spd
