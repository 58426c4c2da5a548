// Parity mode on sm_100a: the reference's surrogate model_update
// (pac_sim.cpp:50-104), the lockstep run_epoch (pac_sim.cpp:205-264) and
// sync_shared (pac_sim.cpp:162-203) with memory stores resident in HBM.
//
// Semantics are the reference's sequential per-edge updates: one CTA owns one
// worker's batch and walks its edges in order; within an edge the d output
// rows of both messages run on 2d threads. Every product and sum uses
// explicitly rounded f64 intrinsics (__dmul_rn/__dadd_rn: no FMA contraction)
// in the reference's accumulation order, so the only deviation from the CPU
// reference is libm's cos/tanh vs CUDA's (<= 2 ulp per call).
#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>

#include "surrogate.hpp"

namespace spd {

void require_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        internal_error("CudaError", "no CUDA device visible (the B200 path has no CPU fallback)");
    if (device < 0 || device >= n)
        internal_error("CudaError", "device " + std::to_string(device) + " out of range");
    cudaDeviceProp prop{};
    SPD_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        internal_error("CudaError", std::string("device is sm_") + std::to_string(prop.major) +
                                        std::to_string(prop.minor) + ", built for sm_100a");
}

MemStore::MemStore(NodeId n, int d_, int dev) : device(dev), node_count(n), d(d_) {
    require_device(dev);
    DeviceGuard g(dev);
    state.alloc(std::size_t(n) * d_);
    last_ts.alloc(n);
    reset();
    SPD_CUDA(cudaStreamSynchronize(0));
}

void MemStore::reset(cudaStream_t s) {
    DeviceGuard g(device);
    state.zero(s);
    last_ts.zero(s);
}

void MemStore::copy_from(const MemStore& o, cudaStream_t s) {
    if (o.node_count != node_count || o.d != d)
        data_error("ConfigMismatch", "memory stores differ in shape");
    DeviceGuard g(device);
    if (state.n)
        SPD_CUDA(cudaMemcpyAsync(state.p, o.state.p, state.bytes(), cudaMemcpyDeviceToDevice, s));
    if (last_ts.n)
        SPD_CUDA(cudaMemcpyAsync(last_ts.p, o.last_ts.p, last_ts.bytes(), cudaMemcpyDeviceToDevice, s));
}

std::string MemStore::digest() const {
    DeviceGuard g(device);
    std::vector<double> st(state.n), ts(last_ts.n);
    SPD_CUDA(cudaDeviceSynchronize());
    state.download(st.data(), st.size());
    last_ts.download(ts.data(), ts.size());
    SPD_CUDA(cudaDeviceSynchronize());
    return fnv1a64_hex(st.data(), node_count, d, ts.data());
}

// ModelParams::seeded (pac_sim.cpp:28-46): Box-Muller normals (rng.hpp:28-34)
// scaled by 1/sqrt(3d); omega log-spaced over three decades times U(0.5,1.5).
SurrogateModel SurrogateModel::seeded(int d, std::uint64_t seed) {
    if (d < 1) data_error("InvalidParams", "need memory dimension >= 1");
    SurrogateModel m;
    m.d = d;
    Rng rng(seed);
    const std::size_t cols = 3 * std::size_t(d);
    m.w_m.resize(std::size_t(d) * cols);
    const double scale = 1.0 / std::sqrt(static_cast<double>(cols));
    for (double& w : m.w_m) {
        double u1 = rng.unit();
        const double u2 = rng.unit();
        while (u1 <= 0.0) u1 = rng.unit();
        w = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2) * scale;
    }
    const double f = 0.5 + (1.5 - 0.5) * rng.unit();
    m.omega.resize(d);
    const double steps = d > 1 ? static_cast<double>(d - 1) : 1.0;
    for (int r = 0; r < d; ++r)
        m.omega[r] = f * std::pow(10.0, -3.0 * static_cast<double>(r) / steps);
    return m;
}

namespace {

struct WorkerRun {
    const spd_edge* edges;  // device
    std::uint64_t lo, hi;
    double* state;
    double* last_ts;
};

struct DevModel {
    const double* w_t;    // 3d x d (transposed: coalesced per-row reads)
    const double* omega;  // d
    double gamma;
    int d;
};

// Sequential replay of a batch per CTA. Threads [0,d) build the message of
// the src endpoint, [d,2d) the dst endpoint (a self-loop uses only the first
// half, pac_sim.cpp:80-87).
__global__ void __launch_bounds__(256) surrogate_batch_kernel(const WorkerRun* runs,
                                                              DevModel m, int* err,
                                                              unsigned long long* err_edge) {
    extern __shared__ double sm[];
    const int d = m.d;
    double* s_old = sm;            // 2d: [si | sj]
    double* cosv = sm + 2 * d;     // 2d: [cos_i | cos_j]
    double* msg = sm + 4 * d;      // 2d
    const WorkerRun run = runs[blockIdx.x];
    const double g = m.gamma;
    const double one_minus_g = 1.0 - g;
    for (std::uint64_t k = run.lo; k < run.hi; ++k) {
        const spd_edge e = run.edges[k];
        const std::uint32_t i = e.src, j = e.dst;
        const double lti = run.last_ts[i], ltj = run.last_ts[j];
        if (e.ts < lti || e.ts < ltj) {  // pac_sim.cpp:73-76
            if (threadIdx.x == 0 && atomicCAS(err, 0, 1) == 0) *err_edge = k;
            return;
        }
        const bool self = (i == j);
        const double dti = __dadd_rn(e.ts, -lti);
        const double dtj = __dadd_rn(e.ts, -ltj);
        for (int c = threadIdx.x; c < 2 * d; c += blockDim.x) {
            const bool first = c < d;
            const int cc = first ? c : c - d;
            s_old[c] = first ? run.state[std::size_t(i) * d + cc] : run.state[std::size_t(j) * d + cc];
            cosv[c] = cos(__dmul_rn(m.omega[cc], first ? dti : dtj));
        }
        __syncthreads();
        const int n_out = self ? d : 2 * d;
        for (int t = threadIdx.x; t < n_out; t += blockDim.x) {
            const bool first = t < d;
            const int r = first ? t : t - d;
            const double* sx = first ? s_old : s_old + d;
            const double* sy = self ? s_old : (first ? s_old + d : s_old);
            const double* cs = first ? cosv : cosv + d;
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(m.w_t[std::size_t(c) * d + r], sx[c]));
            for (int c = 0; c < d; ++c)
                acc = __dadd_rn(acc, __dmul_rn(m.w_t[std::size_t(d + c) * d + r], sy[c]));
            for (int c = 0; c < d; ++c)
                acc = __dadd_rn(acc, __dmul_rn(m.w_t[std::size_t(2 * d + c) * d + r], cs[c]));
            msg[t] = tanh(acc);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < n_out; t += blockDim.x) {
            const bool first = t < d;
            const int r = first ? t : t - d;
            const double nv = __dadd_rn(__dmul_rn(one_minus_g, s_old[t]), __dmul_rn(g, msg[t]));
            run.state[std::size_t(first ? i : j) * d + r] = nv;
        }
        if (threadIdx.x == 0) {
            run.last_ts[i] = e.ts;
            run.last_ts[j] = e.ts;
        }
        __syncthreads();
    }
}

// sync_shared (pac_sim.cpp:162-203): one warp per shared node.
__global__ void sync_shared_kernel(double* const* states, double* const* clocks, int W, int d,
                                   const std::uint32_t* shared, std::uint64_t n_shared, int average) {
    const std::uint64_t sidx = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (sidx >= n_shared) return;
    const std::uint32_t n = shared[sidx];
    if (!average) {
        int best = 0;
        for (int w = 1; w < W; ++w)
            if (clocks[w][n] > clocks[best][n]) best = w;  // ties -> lowest worker
        const double ts = clocks[best][n];
        for (int c = lane; c < d; c += 32) {
            const double v = states[best][std::size_t(n) * d + c];
            for (int w = 0; w < W; ++w) states[w][std::size_t(n) * d + c] = v;
        }
        __syncwarp();
        if (lane == 0)
            for (int w = 0; w < W; ++w) clocks[w][n] = ts;
        return;
    }
    // Average: skip nodes whose copies already agree bit for bit (keeps a
    // second application idempotent for any W, pac_sim.cpp:178-188).
    bool agree = true;
    for (int w = 1; w < W; ++w) agree = agree && clocks[w][n] == clocks[0][n];
    for (int c = lane; c < d; c += 32)
        for (int w = 1; w < W; ++w)
            agree = agree && states[w][std::size_t(n) * d + c] == states[0][std::size_t(n) * d + c];
    agree = __all_sync(0xffffffffu, agree);
    if (agree) return;
    double ts = 0.0;
    for (int w = 0; w < W; ++w) ts = fmax(ts, clocks[w][n]);
    for (int c = lane; c < d; c += 32) {
        double s = 0.0;
        for (int w = 0; w < W; ++w) s = __dadd_rn(s, states[w][std::size_t(n) * d + c]);
        s = __ddiv_rn(s, static_cast<double>(W));
        for (int w = 0; w < W; ++w) states[w][std::size_t(n) * d + c] = s;
    }
    __syncwarp();
    if (lane == 0)
        for (int w = 0; w < W; ++w) clocks[w][n] = ts;
}

struct DevModelHolder {
    DevBuf<double> w_t, omega;
    DevModel dm;
    DevModelHolder(const SurrogateModel& m) {
        const int d = m.d;
        std::vector<double> wt(std::size_t(3) * d * d);
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < 3 * d; ++c) wt[std::size_t(c) * d + r] = m.w_m[std::size_t(r) * 3 * d + c];
        w_t.alloc(wt.size());
        w_t.upload(wt.data(), wt.size());
        omega.alloc(d);
        omega.upload(m.omega.data(), d);
        dm = DevModel{w_t.p, omega.p, m.gamma, d};
    }
};

void launch_runs(const std::vector<WorkerRun>& runs, const DevModel& dm, DevBuf<WorkerRun>& druns,
                 DevBuf<int>& err, DevBuf<unsigned long long>& err_edge, cudaStream_t s) {
    if (runs.empty()) return;
    if (druns.n < runs.size()) druns.alloc(runs.size());
    druns.upload(runs.data(), runs.size(), s);
    const int threads = std::min(256, std::max(32, ((2 * dm.d + 31) / 32) * 32));
    const std::size_t smem = sizeof(double) * 6 * dm.d;
    if (smem > 48 * 1024)
        SPD_CUDA(cudaFuncSetAttribute(surrogate_batch_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    surrogate_batch_kernel<<<unsigned(runs.size()), threads, smem, s>>>(druns.p, dm, err.p, err_edge.p);
    SPD_CUDA(cudaGetLastError());
}

void check_err(DevBuf<int>& err, DevBuf<unsigned long long>& err_edge) {
    int h = 0;
    unsigned long long k = 0;
    SPD_CUDA(cudaDeviceSynchronize());
    err.download(&h, 1);
    err_edge.download(&k, 1);
    SPD_CUDA(cudaDeviceSynchronize());
    if (h)
        data_error("NonChronological",
                   "edge " + std::to_string(k) + " is older than an endpoint's last update");
}

}  // namespace

void surrogate_model_update(MemStore& m, const spd_edge* e, std::uint64_t n,
                            const SurrogateModel& model) {
    if (m.d != model.d) internal_error("DimMismatch", "memory and model dimensions differ");
    for (std::uint64_t k = 0; k < n; ++k)
        if (e[k].src >= m.node_count || e[k].dst >= m.node_count)
            data_error("InvalidParams", "edge names a node outside the memory store");
    DeviceGuard g(m.device);
    DevModelHolder dmh(model);
    DevBuf<spd_edge> de(n);
    de.upload(e, n);
    DevBuf<WorkerRun> druns;
    DevBuf<int> err(1);
    DevBuf<unsigned long long> err_edge(1);
    err.zero();
    std::vector<WorkerRun> runs{{de.p, 0, n, m.state.p, m.last_ts.p}};
    launch_runs(runs, dmh.dm, druns, err, err_edge, 0);
    check_err(err, err_edge);
}

void surrogate_sync_shared(const std::vector<MemStore*>& mems, const std::vector<NodeId>& shared,
                           bool average) {
    if (mems.size() < 2 || shared.empty()) return;  // pac_sim.cpp:164
    const int W = static_cast<int>(mems.size());
    const int d = mems[0]->d;
    for (auto* m : mems) {
        if (m->d != d || m->node_count != mems[0]->node_count || m->device != mems[0]->device)
            data_error("ConfigMismatch", "memory stores differ in shape or device");
    }
    for (NodeId n : shared)
        if (n >= mems[0]->node_count) data_error("InvalidParams", "shared node out of range");
    DeviceGuard g(mems[0]->device);
    std::vector<double*> hs(W), hc(W);
    for (int w = 0; w < W; ++w) {
        hs[w] = mems[w]->state.p;
        hc[w] = mems[w]->last_ts.p;
    }
    DevBuf<double*> ds(W), dc(W);
    ds.upload(hs.data(), W);
    dc.upload(hc.data(), W);
    DevBuf<std::uint32_t> dsh(shared.size());
    dsh.upload(shared.data(), shared.size());
    const unsigned blocks = unsigned((shared.size() * 32 + 255) / 256);
    sync_shared_kernel<<<blocks, 256>>>(ds.p, dc.p, W, d, dsh.p, shared.size(), average ? 1 : 0);
    SPD_CUDA(cudaGetLastError());
    SPD_CUDA(cudaDeviceSynchronize());
}

// Lockstep loop-within-epoch (Alg. 2; pac_sim.cpp:205-264). Each
// global step launches ONE kernel holding every worker's batch (one CTA per
// worker); loop starts reset, loop ends snapshot device-to-device.
void surrogate_run_epoch(const std::vector<const std::vector<spd_edge>*>& edges,
                         const std::vector<MemStore*>& mems, const SurrogateModel& model,
                         const std::vector<NodeId>& shared, bool average,
                         std::uint64_t batch_size, EpochOut& out) {
    const std::size_t W = edges.size();
    if (mems.size() != W) data_error("ConfigMismatch", "one memory store per worker required");
    if (batch_size < 1) data_error("InvalidParams", "need batch_size >= 1");
    for (auto* m : mems)
        if (m->d != model.d) internal_error("DimMismatch", "memory and model dimensions differ");
    const int dev = W ? mems[0]->device : 0;
    DeviceGuard g(dev);
    DevModelHolder dmh(model);
    out.batches.assign(W, 0);
    out.loops.assign(W, 0);
    std::vector<DevBuf<spd_edge>> de(W);
    std::vector<std::unique_ptr<MemStore>> snap(W);
    std::vector<std::uint64_t> pos(W, 0);
    std::vector<std::uint8_t> done(W, 0);
    for (std::size_t w = 0; w < W; ++w) {
        const auto& ev = *edges[w];
        for (const auto& e : ev)
            if (e.src >= mems[w]->node_count || e.dst >= mems[w]->node_count)
                data_error("InvalidParams", "edge names a node outside the memory store");
        de[w].alloc(ev.size());
        de[w].upload(ev.data(), ev.size());
        snap[w] = std::make_unique<MemStore>(mems[w]->node_count, mems[w]->d, mems[w]->device);
        out.batches[w] = (ev.size() + batch_size - 1) / batch_size;
        if (out.batches[w] == 0) {  // vacuous worker (pac_sim.cpp:224-230)
            out.loops[w] = 1;
            snap[w]->copy_from(*mems[w]);
            done[w] = 1;
            if (out.want_log) out.snaps.emplace_back(int(w), mems[w]->digest());
        }
    }
    DevBuf<WorkerRun> druns;
    DevBuf<int> err(1);
    DevBuf<unsigned long long> err_edge(1);
    err.zero();
    std::uint64_t step = 0;
    std::vector<WorkerRun> runs;
    while (!std::all_of(done.begin(), done.end(), [](std::uint8_t f) { return f != 0; })) {
        ++step;
        runs.clear();
        for (std::size_t w = 0; w < W; ++w) {
            if (out.batches[w] == 0) continue;
            if (pos[w] == 0) mems[w]->reset();  // loop_start
            const std::uint64_t lo = pos[w] * batch_size;
            const std::uint64_t hi = std::min<std::uint64_t>(edges[w]->size(), (pos[w] + 1) * batch_size);
            runs.push_back({de[w].p, lo, hi, mems[w]->state.p, mems[w]->last_ts.p});
        }
        launch_runs(runs, dmh.dm, druns, err, err_edge, 0);
        for (std::size_t w = 0; w < W; ++w) {
            if (out.batches[w] == 0) continue;
            if (out.want_log) {
                out.log_steps.insert(out.log_steps.end(),
                                     {step, std::uint64_t(w), out.loops[w] + 1, pos[w] + 1});
            }
            ++pos[w];
            if (pos[w] == out.batches[w]) {  // loop_end: snapshot
                ++out.loops[w];
                snap[w]->copy_from(*mems[w]);
                done[w] = 1;
                pos[w] = 0;
                if (out.want_log) out.snaps.emplace_back(int(w), mems[w]->digest());
            }
        }
    }
    check_err(err, err_edge);
    for (std::size_t w = 0; w < W; ++w) mems[w]->copy_from(*snap[w]);  // drop partial loops
    SPD_CUDA(cudaDeviceSynchronize());
    surrogate_sync_shared(mems, shared, average);
    out.sync_events = W >= 2 ? shared.size() : 0;
    out.digests.clear();
    for (auto* m : mems) out.digests.push_back(m->digest());
}

}  // namespace spd
