// Per-partition induced event streams (pac_sim.cpp:106-132), the
// shuffle-combine regrouping (pac_sim.cpp:134-160) and simulate's shuffle
// re-induction with the `recovered` count (pac_sim.cpp:280-329).
//
// One pass over the stream serves every partition: each node carries a
// partition bitset, an edge belongs to partition p iff bit p is set in both
// endpoint sets. Each induced edge keeps its stream position (global edge id)
// so the device can index edge features without a second copy of the stream.
#include <algorithm>
#include <string>

#include "host.hpp"

namespace spd {

namespace {

SubGraphs induce_from_bits(const Stream& s, const std::vector<std::uint64_t>& bits, int words,
                           int P, std::vector<std::uint8_t>* in_any) {
    SubGraphs out;
    out.g.resize(P);
    std::vector<std::uint64_t> cnt(P, 0);
    for (NodeId i = 0; i < s.node_count; ++i)
        for (int w = 0; w < words; ++w) {
            std::uint64_t m = bits[std::size_t(i) * words + w];
            while (m) {
                const int b = __builtin_ctzll(m);
                m &= m - 1;
                out.g[w * 64 + b].nodes.push_back(i);
            }
        }
    // size pass, then fill (keeps memory tight at GDELT scale)
    auto visit = [&](auto&& fn) {
        for (std::uint64_t e = 0; e < s.n; ++e) {
            const NodeId u = s.e[e].src, v = s.e[e].dst;
            if (u >= s.node_count || v >= s.node_count) continue;
            for (int w = 0; w < words; ++w) {
                std::uint64_t m = bits[std::size_t(u) * words + w] & bits[std::size_t(v) * words + w];
                while (m) {
                    const int b = __builtin_ctzll(m);
                    m &= m - 1;
                    fn(e, w * 64 + b);
                }
            }
        }
    };
    visit([&](std::uint64_t, int p) { ++cnt[p]; });
    for (int p = 0; p < P; ++p) {
        out.g[p].edges.reserve(cnt[p]);
        out.g[p].eids.reserve(cnt[p]);
    }
    if (in_any) in_any->assign(s.n, 0);
    visit([&](std::uint64_t e, int p) {
        out.g[p].edges.push_back(s.e[e]);
        out.g[p].eids.push_back(e);
        if (in_any) (*in_any)[e] = 1;
    });
    return out;
}

}  // namespace

SubGraphs induce_from_node_parts(const Stream& s, const std::uint64_t* np_off,
                                 const PartId* np_parts, NodeId np_count, int num_parts) {
    if (num_parts < 1) data_error("InvalidParams", "need num_parts >= 1");
    const int words = (num_parts + 63) / 64;
    std::vector<std::uint64_t> bits(std::size_t(s.node_count) * words, 0);
    for (NodeId i = 0; i < np_count && i < s.node_count; ++i)
        for (std::uint64_t k = np_off[i]; k < np_off[i + 1]; ++k) {
            const PartId p = np_parts[k];
            if (p < 0 || p >= num_parts)
                data_error("InvalidPartition", "node " + std::to_string(i) + " lists partition " +
                                                   std::to_string(p));
            bits[std::size_t(i) * words + (p >> 6)] |= 1ULL << (p & 63);
        }
    return induce_from_bits(s, bits, words, num_parts, nullptr);
}

SubGraphs induce_from_groups(const Stream& s, const std::uint64_t* off, const NodeId* nodes,
                             int n_groups, std::vector<std::uint8_t>* in_any) {
    if (n_groups < 1) data_error("InvalidParams", "need at least one group");
    const int words = (n_groups + 63) / 64;
    std::vector<std::uint64_t> bits(std::size_t(s.node_count) * words, 0);
    for (int g = 0; g < n_groups; ++g)
        for (std::uint64_t k = off[g]; k < off[g + 1]; ++k)
            if (nodes[k] < s.node_count)
                bits[std::size_t(nodes[k]) * words + (g >> 6)] |= 1ULL << (g & 63);
    SubGraphs out = induce_from_bits(s, bits, words, n_groups, in_any);
    for (int g = 0; g < n_groups; ++g)  // simulate keeps the group list as given (pac_sim.cpp:318)
        out.g[g].nodes.assign(nodes + off[g], nodes + off[g + 1]);
    return out;
}

// pac_sim.cpp:134-160: seeded Fisher-Yates over part indices, consecutive
// groups of |small|/W parts, union sorted and deduplicated.
std::vector<std::vector<NodeId>> shuffle_combine(const std::vector<std::vector<NodeId>>& small,
                                                 int num_workers, std::uint64_t epoch_seed) {
    if (num_workers < 1 || small.empty() || small.size() % std::size_t(num_workers) != 0)
        data_error("IndivisibleParts", std::to_string(small.size()) +
                                           " parts cannot combine into " +
                                           std::to_string(num_workers) + " groups");
    std::vector<std::uint64_t> perm(small.size());
    for (std::size_t i = 0; i < perm.size(); ++i) perm[i] = i;
    Rng rng(epoch_seed);
    rng.shuffle(perm.data(), perm.size());
    const std::size_t gs = small.size() / std::size_t(num_workers);
    std::vector<std::vector<NodeId>> out(num_workers);
    for (std::size_t g = 0; g < out.size(); ++g) {
        auto& v = out[g];
        for (std::size_t r = 0; r < gs; ++r) {
            const auto& part = small[perm[g * gs + r]];
            v.insert(v.end(), part.begin(), part.end());
        }
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    return out;
}

}  // namespace spd
