// Shuffle-combine on the device: the training stream
// stays resident in HBM and every epoch's regrouped worker subgraphs
// (pac_sim.cpp:134-160, :280-329) are induced there — node membership as
// per-node group bitmasks, the induced event list by a stable compaction of
// the stream, local ids, the per-node time-sorted neighbour CSR by a stable
// radix sort of the (node, event, role) entries, the negative pool and the
// synthetic feature rows — instead of P passes of host re-induction plus an
// upload per epoch. The result is bit-identical to spd_induce_groups +
// spd_tgn_rebind (tests/test_tgn_gpu.py), and so is the `recovered` count
// (edges some combined group induces that no small part does).
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>

#include "tgn.hpp"
#include "tgn_common.cuh"

namespace spd {

namespace {

unsigned grid_for(std::uint64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// ng[n] = bitmask of the groups whose small parts contain node n
__global__ void k_node_groups(const std::uint64_t* bits, int words, std::uint32_t N,
                              const int* part_group, std::uint64_t* ng) {
    const std::uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    std::uint64_t m = 0;
    for (int w = 0; w < words; ++w) {
        std::uint64_t b = bits[(std::size_t)n * words + w];
        while (b) {
            const int p = w * 64 + __ffsll(static_cast<long long>(b)) - 1;
            b &= b - 1;
            m |= 1ull << part_group[p];
        }
    }
    ng[n] = m;
}

// in_small[e]: some small part induces edge e (both endpoints in it)
__global__ void k_in_small(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t E,
                           const std::uint64_t* bits, int words, std::uint8_t* in_small) {
    const std::uint64_t e = (std::uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    std::uint8_t any = 0;
    for (int w = 0; w < words; ++w)
        any |= (bits[(std::size_t)src[e] * words + w] & bits[(std::size_t)dst[e] * words + w]) != 0;
    in_small[e] = any;
}

// counts[g] = edges group g induces; counts[G] = recovered (induced by some
// group, by no small part). Block-level integer sums (order-free).
__global__ void k_group_counts(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t E,
                               const std::uint64_t* ng, const std::uint8_t* in_small, int G,
                               unsigned long long* counts) {
    __shared__ unsigned long long c[65];
    for (int i = threadIdx.x; i <= G; i += blockDim.x) c[i] = 0;
    __syncthreads();
    for (std::uint64_t e = (std::uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (std::uint64_t)gridDim.x * blockDim.x) {
        std::uint64_t m = ng[src[e]] & ng[dst[e]];
        if (m && !in_small[e]) atomicAdd(&c[G], 1ull);
        while (m) {
            atomicAdd(&c[__ffsll(static_cast<long long>(m)) - 1], 1ull);
            m &= m - 1;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= G; i += blockDim.x)
        if (c[i]) atomicAdd(&counts[i], c[i]);
}

struct EdgeInGroup {
    const std::uint32_t* src;
    const std::uint32_t* dst;
    const std::uint64_t* ng;
    std::uint64_t bit;
    __device__ bool operator()(std::uint64_t e) const { return (ng[src[e]] & ng[dst[e]] & bit) != 0; }
};
struct NodeInGroup {
    const std::uint64_t* ng;
    std::uint64_t bit;
    __device__ bool operator()(std::uint32_t n) const { return (ng[n] & bit) != 0; }
};

__global__ void k_scatter_loc(const std::uint32_t* nodes, std::uint32_t n, std::uint32_t* loc) {
    const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) loc[nodes[i]] = i;
}

// induced events in local ids + CSR sort entries (node, 2k + role) + degrees
__global__ void k_gather_events(const std::uint64_t* eidx, std::uint64_t E, const std::uint32_t* gsrc,
                                const std::uint32_t* gdst, const double* gts, const std::uint32_t* loc,
                                std::uint32_t* src, std::uint32_t* dst, double* ts, std::uint32_t* keys,
                                std::uint32_t* vals, unsigned long long* deg, std::uint8_t* is_dst) {
    const std::uint64_t k = (std::uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= E) return;
    const std::uint64_t e = eidx[k];
    const std::uint32_t s = loc[gsrc[e]], d = loc[gdst[e]];
    src[k] = s;
    dst[k] = d;
    ts[k] = gts[e];
    keys[2 * k] = s;
    keys[2 * k + 1] = d;
    vals[2 * k] = static_cast<std::uint32_t>(2 * k);
    vals[2 * k + 1] = static_cast<std::uint32_t>(2 * k + 1);
    atomicAdd(&deg[s], 1ull);
    atomicAdd(&deg[d], 1ull);
    is_dst[d] = 1;
}

// CSR entry i (sorted by node, stable: event order, src side first) -> (neighbour, event, ts)
__global__ void k_fill_adj(const std::uint32_t* order, std::uint64_t n2, const std::uint32_t* src,
                           const std::uint32_t* dst, const double* ts, std::uint32_t* anbr,
                           std::uint32_t* aev, double* ats) {
    const std::uint64_t i = (std::uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2) return;
    const std::uint32_t v = order[i], k = v >> 1;
    anbr[i] = (v & 1) ? src[k] : dst[k];
    aev[i] = k;
    ats[i] = ts[k];
}

// reusable CUB temporary storage
struct Temp {
    DevBuf<unsigned char> buf;
    void* get(std::size_t bytes) {
        if (buf.n < bytes) buf.alloc(bytes);
        return buf.p;
    }
};

}  // namespace

void TGNTrainer::attach_stream(const spd_edge* e, std::uint64_t n, NodeId node_count,
                               const std::uint64_t* off, const NodeId* nodes, int n_small) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        for (auto& l : lanes_) l->attach_stream(e, n, node_count, off, nodes, n_small);
        return;
    }
    if (n_small < 1 || n_small > 64 * 64) data_error("InvalidParams", "need 1 <= small parts <= 4096");
    if (total_workers_ > 64) data_error("InvalidParams", "device re-induction supports <= 64 workers");
    if (n_small % total_workers_)
        data_error("IndivisibleParts", std::to_string(n_small) + " parts cannot combine into " +
                                           std::to_string(total_workers_) + " groups");
    if (n > 0xFFFFFFFFull) data_error("InvalidParams", "stream exceeds 2^32 events");
    auto& S = dstream_;
    S = std::make_unique<DevStream>();
    S->E = n;
    S->N = node_count;
    S->n_small = n_small;
    S->words = (n_small + 63) / 64;
    std::vector<std::uint32_t> src(n), dst(n);
    std::vector<double> ts(n);
    for (std::uint64_t k = 0; k < n; ++k) {
        if (e[k].src >= node_count || e[k].dst >= node_count)
            data_error("InvalidParams", "edge endpoint outside [0, node_count)");
        if (k && e[k].ts < e[k - 1].ts) data_error("NonChronological", "stream must be time-ordered");
        src[k] = e[k].src;
        dst[k] = e[k].dst;
        ts[k] = e[k].ts;
    }
    std::vector<std::uint64_t> bits(std::size_t(node_count) * S->words, 0);
    for (int p = 0; p < n_small; ++p)
        for (std::uint64_t k = off[p]; k < off[p + 1]; ++k) {
            if (nodes[k] >= node_count) data_error("InvalidPartition", "small part lists a node out of range");
            bits[std::size_t(nodes[k]) * S->words + (p >> 6)] |= 1ull << (p & 63);
        }
    S->src.alloc(std::max<std::uint64_t>(1, n)); S->src.upload(src.data(), n, stream_);
    S->dst.alloc(std::max<std::uint64_t>(1, n)); S->dst.upload(dst.data(), n, stream_);
    S->ts.alloc(std::max<std::uint64_t>(1, n)); S->ts.upload(ts.data(), n, stream_);
    S->bits.alloc(std::max<std::size_t>(1, bits.size())); S->bits.upload(bits.data(), bits.size(), stream_);
    S->in_small.alloc(std::max<std::uint64_t>(1, n));
    if (n) k_in_small<<<grid_for(n), 256, 0, stream_>>>(S->src.p, S->dst.p, n, S->bits.p, S->words, S->in_small.p);
    SPD_CUDA(cudaGetLastError());
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::shuffle_epoch(std::uint64_t seed, std::uint64_t* recovered) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_wait();
        for (auto& l : lanes_) l->shuffle_epoch(seed, recovered);
        epoch_steps_ = lanes_[0]->epoch_steps_;
        return;
    }
    if (!dstream_) usage_error("shuffle_epoch needs spd_tgn_attach_stream first");
    auto& S = *dstream_;
    const int G = total_workers_;
    const int Fp = lay_.F ? (lay_.F + 7) / 8 * 8 : 0;
    // the groups: shuffle_combine's seeded Fisher-Yates over part indices
    // (pac_sim.cpp:134-160), consecutive runs of n_small / G parts
    std::vector<std::uint64_t> perm(S.n_small);
    std::iota(perm.begin(), perm.end(), std::uint64_t(0));
    Rng rng(seed);
    rng.shuffle(perm.data(), perm.size());
    const int gs = S.n_small / G;
    std::vector<int> part_group(S.n_small);
    for (int i = 0; i < S.n_small; ++i) part_group[perm[i]] = i / gs;
    DevBuf<int> pg(S.n_small);
    pg.upload(part_group.data(), S.n_small, stream_);
    DevBuf<std::uint64_t> ng(std::max<NodeId>(1, S.N));
    k_node_groups<<<grid_for(S.N), 256, 0, stream_>>>(S.bits.p, S.words, S.N, pg.p, ng.p);
    DevBuf<unsigned long long> counts(G + 1);
    counts.zero(stream_);
    if (S.E) k_group_counts<<<1184, 256, 0, stream_>>>(S.src.p, S.dst.p, S.E, ng.p, S.in_small.p, G, counts.p);
    SPD_CUDA(cudaGetLastError());
    std::vector<unsigned long long> cnt(G + 1);
    counts.download(cnt.data(), G + 1, stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
    if (recovered) *recovered = cnt[G];

    SPD_CUDA(cudaDeviceSynchronize());
    for (auto& ge : graph_exec_)
        if (ge) {
            SPD_CUDA(cudaGraphExecDestroy(ge));
            ge = nullptr;
        }
    eager_full_steps_ = 0;
    std::vector<int> ids;
    for (const auto& w : workers_) ids.push_back(w->gid);
    workers_.clear();
    syncbuf_.rows.clear();
    all_batches_.assign(G, 0);
    for (int k = 0; k < G; ++k) all_batches_[k] = (cnt[k] + cfg_.batch_size - 1) / cfg_.batch_size;
    epoch_steps_ = G ? *std::max_element(all_batches_.begin(), all_batches_.end()) : 0;

    Temp tmp;
    DevBuf<int> nsel(1);
    DevBuf<std::uint32_t> loc(std::max<NodeId>(1, S.N));
    for (int wid : ids) {
        auto W = std::make_unique<Worker>();
        Worker& w = *W;
        w.gid = wid;
        w.batches = all_batches_[wid];
        const std::uint64_t bit = 1ull << wid;
        // local nodes: every node of the group's small parts, ascending
        DevBuf<std::uint32_t> dnodes(std::max<NodeId>(1, S.N));
        {
            cub::CountingInputIterator<std::uint32_t> it(0);
            std::size_t bytes = 0;
            SPD_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, dnodes.p, nsel.p, int(S.N), NodeInGroup{ng.p, bit}, stream_));
            SPD_CUDA(cub::DeviceSelect::If(tmp.get(bytes), bytes, it, dnodes.p, nsel.p, int(S.N),
                                           NodeInGroup{ng.p, bit}, stream_));
        }
        int nn = 0;
        nsel.download(&nn, 1, stream_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
        w.N = static_cast<NodeId>(nn);
        w.nodes.resize(nn);
        dnodes.download(w.nodes.data(), nn, stream_);
        if (nn) k_scatter_loc<<<grid_for(nn), 256, 0, stream_>>>(dnodes.p, nn, loc.p);
        // induced events: stable compaction of the stream positions
        w.E = cnt[wid];
        DevBuf<std::uint64_t> eidx(std::max<std::uint64_t>(1, w.E));
        if (w.E) {
            cub::CountingInputIterator<std::uint64_t> it(0);
            std::size_t bytes = 0;
            DevBuf<std::uint64_t> ne(1);
            EdgeInGroup pred{S.src.p, S.dst.p, ng.p, bit};
            SPD_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, eidx.p, ne.p, S.E, pred, stream_));
            SPD_CUDA(cub::DeviceSelect::If(tmp.get(bytes), bytes, it, eidx.p, ne.p, S.E, pred, stream_));
        }
        const std::uint64_t E = w.E, N = std::max<std::uint64_t>(1, w.N);
        w.ev_src.alloc(std::max<std::uint64_t>(1, E));
        w.ev_dst.alloc(std::max<std::uint64_t>(1, E));
        w.ev_ts.alloc(std::max<std::uint64_t>(1, E));
        DevBuf<std::uint32_t> keys(std::max<std::uint64_t>(1, 2 * E)), vals(std::max<std::uint64_t>(1, 2 * E));
        DevBuf<unsigned long long> deg(N + 1);
        deg.zero(stream_);
        DevBuf<std::uint8_t> is_dst(N);
        is_dst.zero(stream_);
        if (E)
            k_gather_events<<<grid_for(E), 256, 0, stream_>>>(eidx.p, E, S.src.p, S.dst.p, S.ts.p, loc.p,
                                                               w.ev_src.p, w.ev_dst.p, w.ev_ts.p, keys.p,
                                                               vals.p, deg.p, is_dst.p);
        // CSR offsets (exclusive sum of the degrees) and the stable sort by node
        w.adj_off.alloc(N + 1);
        {
            std::size_t bytes = 0;
            SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg.p, reinterpret_cast<unsigned long long*>(w.adj_off.p),
                                                   int(N + 1), stream_));
            SPD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, deg.p,
                                                   reinterpret_cast<unsigned long long*>(w.adj_off.p), int(N + 1), stream_));
        }
        w.adj_nbr.alloc(std::max<std::uint64_t>(1, 2 * E));
        w.adj_ev.alloc(std::max<std::uint64_t>(1, 2 * E));
        w.adj_ts.alloc(std::max<std::uint64_t>(1, 2 * E));
        if (E) {
            DevBuf<std::uint32_t> keys2(2 * E), vals2(2 * E);
            int end_bit = 1;
            while ((1ull << end_bit) < N) ++end_bit;
            std::size_t bytes = 0;
            SPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p,
                                                     2 * E, 0, end_bit, stream_));
            SPD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, keys.p, keys2.p, vals.p, vals2.p,
                                                     2 * E, 0, end_bit, stream_));
            k_fill_adj<<<grid_for(2 * E), 256, 0, stream_>>>(vals2.p, 2 * E, w.ev_src.p, w.ev_dst.p, w.ev_ts.p,
                                                               w.adj_nbr.p, w.adj_ev.p, w.adj_ts.p);
        }
        // negative pool: the destination nodes, ascending
        DevBuf<std::uint32_t> pool(N);
        {
            cub::CountingInputIterator<std::uint32_t> it(0);
            std::size_t bytes = 0;
            SPD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, is_dst.p, pool.p, nsel.p, int(N), stream_));
            SPD_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, it, is_dst.p, pool.p, nsel.p, int(N), stream_));
        }
        int np = 0;
        nsel.download(&np, 1, stream_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
        if (np == 0) {  // (as the host path: an empty pool holds node 0)
            pool.zero(stream_);
            np = 1;
        }
        w.n_pool = static_cast<std::uint32_t>(np);
        w.pool = std::move(pool);
        // synthetic features from the global edge ids (the stream positions)
        w.feat.alloc(std::max<std::uint64_t>(1, E) * std::max(1, Fp));
        if (Fp && E) {
            tgnk::k_gen_features<<<grid_for(E * Fp), 256, 0, stream_>>>(w.feat.p, eidx.p, E, lay_.F, Fp,
                                                                        feat_seed_mixed_);
            SPD_CUDA(cudaGetLastError());
        }
        // host copy of the events (validates host-fed batches, spd_tgn_worker_events)
        {
            std::vector<std::uint32_t> hs(E), hd(E);
            std::vector<double> ht(E);
            w.ev_src.download(hs.data(), E, stream_);
            w.ev_dst.download(hd.data(), E, stream_);
            w.ev_ts.download(ht.data(), E, stream_);
            SPD_CUDA(cudaStreamSynchronize(stream_));
            w.ev_host.resize(E);
            for (std::uint64_t k = 0; k < E; ++k) w.ev_host[k] = spd_edge{hs[k], hd[k], ht[k]};
        }
        init_worker_state(w);
        workers_.push_back(std::move(W));
    }
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        workers_[k]->ctl = ctl_dev_.p + 2 * k;
        workers_[k]->ctl_index = static_cast<int>(k);
    }
    step_in_epoch_ = 0;
    SPD_CUDA(cudaGetLastError());
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

}  // namespace spd
