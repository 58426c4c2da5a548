// Deterministic memory-row gradient of the GRU outputs (dH), without atomics.
//
// The GRU output row of pending node u (mem_new[u]) is read by the step in two
// places: as the memory part of a root's query / merge input (root entries)
// and as the memory part of a neighbour's key/value input (occurrence
// entries, one per (root, neighbour slot)). dH[u] is the sum of those
// entries' gradients. Summed with float atomics the order — and so the last
// bits — changes run to run; here every contribution is summed in a fixed
// order:
//
//   1. index (side stream, during the forward; needs only the neighbour lists
//      and the slot map): a stable counting sort of the entries by slot, in
//      four kernels — per-block slot histograms, a per-slot prefix over the
//      blocks, exclusive scans over the slots, and a scatter whose per-block
//      ranks are assigned warp by warp in entry order. Lists: occurrence
//      entries (r * K + j) and root entries (r), each grouped by slot in
//      ascending entry order, each slot's lists cut into chunks of 16.
//   2. k_dh_pull (backward, beside the dQ GEMMs): one warp per occurrence
//      chunk sums its entries' memory-column gradients
//        dx_j = sum_h a_hj dxbar_h + ds_hj q'_h          (tgn_attn.cu)
//      in list order into a chunk partial row; k_dh_pull_root (after the
//      query data-gradient GEMM) does the same for the root chunks' query /
//      merge memory columns (dq_in, dm_in).
//   3. k_gru_bwd_dh: one warp per pending row sums the row's chunk partials
//      in chunk order (occurrence chunks, then root chunks) and runs the
//      GRUCell backward on the result.
// Chunks bound every serial chain (a hub row read by thousands of entries is
// summed 16 entries per warp, then ~entries/16 partials).
// Semantics: oracle/tgn_oracle.py (autograd); only the summation order is the
// kernel's own — and it is the same every run.
#include "pdl.cuh"
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"

namespace spd {
namespace tgnk {

namespace {
__device__ __forceinline__ int occ_slot(const WorkerDev& w, const DhIndex& x, int e) {
    if (e < x.nb_occ * kDhBlock) {  // occurrence entry (r, j)
        if (e >= x.RK) return -1;
        const int r = e / x.K, j = e - r * x.K;
        if (j >= x.cnt[r]) return -1;
        return w.slot[x.nbr_node[e]];
    }
    const int r = e - x.nb_occ * kDhBlock;  // root entry
    if (r >= x.R) return -1;
    return w.slot[x.roots[r]];
}
__device__ __forceinline__ float4 f4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void fma4(float4& a, float s, const float4& x) {
    a.x = fmaf(s, x.x, a.x); a.y = fmaf(s, x.y, a.y); a.z = fmaf(s, x.z, a.z); a.w = fmaf(s, x.w, a.w);
}
__device__ __forceinline__ void add4(float4& a, const float4& x) {
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
}
}  // namespace

// Per-block slot histograms: hist[b][u] for u < U_cap.
__global__ void __launch_bounds__(kDhBlock) k_dh_hist(WorkerDev w, DhIndex x) {
    pdl_entry();
    extern __shared__ int h_s[];
    for (int u = threadIdx.x; u < x.U_cap; u += blockDim.x) h_s[u] = 0;
    __syncthreads();
    const int e = blockIdx.x * kDhBlock + threadIdx.x;
    const int s = occ_slot(w, x, e);
    if (s >= 0) atomicAdd(h_s + s, 1);  // a count: order-free
    __syncthreads();
    int* out = x.hist + (std::size_t)blockIdx.x * x.U_cap;
    for (int u = threadIdx.x; u < x.U_cap; u += blockDim.x) out[u] = h_s[u];
}

// Per slot u (one thread each): hist[b][u] -> exclusive prefix over the
// blocks of its list (occurrence blocks, then root blocks), in place; the
// two totals go to off_occ[u] / off_root[u] for k_dh_scan.
__global__ void __launch_bounds__(128) k_dh_colscan(DhIndex x) {
    pdl_entry();
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= x.U_cap) return;
    constexpr int G = 16;  // loads in flight per thread
    int tot[2];
#pragma unroll
    for (int list = 0; list < 2; ++list) {
        const int b0 = list ? x.nb_occ : 0, b1 = list ? x.nb_occ + x.nb_root : x.nb_occ;
        int run = 0;
        for (int g = b0; g < b1; g += G) {
            int v[G];
#pragma unroll
            for (int t = 0; t < G; ++t) v[t] = g + t < b1 ? x.hist[(std::size_t)(g + t) * x.U_cap + u] : 0;
#pragma unroll
            for (int t = 0; t < G; ++t) {
                if (g + t < b1) x.hist[(std::size_t)(g + t) * x.U_cap + u] = run;
                run += v[t];
            }
        }
        tot[list] = run;
    }
    x.off_occ[u] = tot[0];
    x.off_root[u] = tot[1];
}

// One block: per-slot totals -> exclusive scans off_occ / off_root and the
// chunk offsets of both lists (chunks of kDhChunk per slot), plus the
// chunk -> (slot, first list position) maps. Thread t owns the consecutive
// slots [t * per, (t + 1) * per).
__global__ void __launch_bounds__(1024) k_dh_scan(DhIndex x) {
    pdl_entry();
    __shared__ int warp_sums[4][32];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int per = (x.U_cap + blockDim.x - 1) / blockDim.x;
    const int u0 = min(x.U_cap, t * per), u1 = min(x.U_cap, u0 + per);
    int v[4] = {0, 0, 0, 0};  // occurrences, roots, occurrence chunks, root chunks
    for (int u = u0; u < u1; ++u) {
        const int to = x.off_occ[u], tr = x.off_root[u];
        v[0] += to;
        v[1] += tr;
        v[2] += (to + kDhChunk - 1) / kDhChunk;
        v[3] += (tr + kDhChunk - 1) / kDhChunk;
    }
    int ex[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int incl = v[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sums[q][wid] = incl;
        ex[q] = incl - v[q];  // exclusive within the warp
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int a = lane < (int)(blockDim.x >> 5) ? warp_sums[q][lane] : 0;
            int incl = a;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            warp_sums[q][lane] = incl - a;
        }
    }
    __syncthreads();
    int po = ex[0] + warp_sums[0][wid], pr = ex[1] + warp_sums[1][wid];
    int pc = ex[2] + warp_sums[2][wid], prc = ex[3] + warp_sums[3][wid];
    for (int u = u0; u < u1; ++u) {
        const int to = x.off_occ[u], tr = x.off_root[u];
        const int co = (to + kDhChunk - 1) / kDhChunk, cr = (tr + kDhChunk - 1) / kDhChunk;
        x.off_occ[u] = po;
        x.off_root[u] = pr;
        x.chunk_off[u] = pc;
        x.rchunk_off[u] = prc;
        for (int c = 0; c < co; ++c) {
            x.chunk_slot[pc + c] = u;
            x.chunk_start[pc + c] = po + c * kDhChunk;
        }
        for (int c = 0; c < cr; ++c) {
            x.rchunk_slot[prc + c] = u;
            x.rchunk_start[prc + c] = pr + c * kDhChunk;
        }
        po += to;
        pr += tr;
        pc += co;
        prc += cr;
    }
    if (t == (int)blockDim.x - 1) {
        x.off_occ[x.U_cap] = po;
        x.off_root[x.U_cap] = pr;
        x.chunk_off[x.U_cap] = pc;
        x.rchunk_off[x.U_cap] = prc;
    }
}

// Stable scatter: block b's running positions start at off[u] + prefix[b][u];
// warps take their turn in entry order, lanes of a warp with the same slot
// ranked by lane (match_any), so each slot's list is in ascending entry order.
__global__ void __launch_bounds__(kDhBlock) k_dh_scatter(WorkerDev w, DhIndex x) {
    pdl_entry();
    extern __shared__ int c_s[];
    const bool root_blk = blockIdx.x >= (unsigned)x.nb_occ;
    const int* off = root_blk ? x.off_root : x.off_occ;
    const int* pre = x.hist + (std::size_t)blockIdx.x * x.U_cap;
    for (int u = threadIdx.x; u < x.U_cap; u += blockDim.x) c_s[u] = off[u] + pre[u];
    const int e = blockIdx.x * kDhBlock + threadIdx.x;
    const int s = occ_slot(w, x, e);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned grp = __match_any_sync(0xffffffffu, s);
    const int rank = __popc(grp & ((1u << lane) - 1u));
    const bool leader = rank == 0;
    int* list = root_blk ? x.list_root : x.list_occ;
    const int val = root_blk ? e - x.nb_occ * kDhBlock : e;
    __syncthreads();
    for (int turn = 0; turn < kDhBlock / 32; ++turn) {
        if (wid == turn && s >= 0) {
            list[c_s[s] + rank] = val;
            __syncwarp(grp);
            if (leader) c_s[s] += __popc(grp);
        }
        __syncthreads();
    }
}

// One warp per occurrence chunk: the chunk's memory-column gradients summed in
// list order into partial[c] (D floats). NM = ceil(D / 128) float4 per lane;
// entries in groups of G whose loads are all issued before the first FMA.
template <int NM, int HMAX>
__global__ void __launch_bounds__(256) k_dh_pull(DhIndex x, Dims d, const float* alpha,
                                                 const float* dsc, const float* dxbar,
                                                 const float* Qp, float* partial) {
    pdl_entry();
    const int lane = threadIdx.x & 31, nchunks = x.chunk_off[x.U_cap];
    // grid-stride over the chunks (a capped grid leaves SMs to the query
    // backward running beside it)
    for (int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); c < nchunks;
         c += (int)((gridDim.x * blockDim.x) >> 5)) {
    const int u = x.chunk_slot[c], p0 = x.chunk_start[c];
    const int n = min(kDhChunk, x.off_occ[u + 1] - p0);
    float4 acc[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int ldr = d.H * d.ld_p;
    const int my_e = lane < n ? x.list_occ[p0 + lane] : 0;  // entry ids, broadcast in order
    constexpr int G = 8 / HMAX;
    for (int g = 0; g < n; g += G) {
        float a[G][HMAX], s[G][HMAX];
        float4 gx[G][HMAX][NM], qx[G][HMAX][NM];
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const int e = __shfl_sync(0xffffffffu, my_e, min(g + t, 31));
            const bool ok = g + t < n;
            const int r = e / d.K, j = e - r * d.K;
#pragma unroll
            for (int h = 0; h < HMAX; ++h) {
                const bool okh = ok && h < d.H;
                a[t][h] = okh ? alpha[((std::size_t)r * d.H + h) * d.K + j] : 0.f;
                s[t][h] = okh ? dsc[((std::size_t)r * d.H + h) * d.K + j] : 0.f;
#pragma unroll
                for (int i = 0; i < NM; ++i) {
                    const int col = 4 * (lane + 32 * i);
                    const bool okc = okh && col < d.D;
                    const std::size_t o = (std::size_t)r * ldr + (std::size_t)h * d.ld_p + col;
                    gx[t][h][i] = okc ? f4(dxbar + o) : make_float4(0.f, 0.f, 0.f, 0.f);
                    qx[t][h][i] = okc ? f4(Qp + o) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
            if (g + t >= n) break;
#pragma unroll
            for (int h = 0; h < HMAX; ++h) {
                if (h >= d.H) break;
#pragma unroll
                for (int i = 0; i < NM; ++i) {
                    fma4(acc[i], a[t][h], gx[t][h][i]);
                    fma4(acc[i], s[t][h], qx[t][h][i]);
                }
            }
        }
    }
    float* o = partial + (std::size_t)c * d.D;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col < d.D) *reinterpret_cast<float4*>(o + col) = acc[i];
    }
    }
}

// One warp per root chunk: the roots' query [s_root | phi(0)] and merge
// [attn | s_root] memory-column gradients summed in list order into
// rpartial[c].
template <int NM>
__global__ void __launch_bounds__(256) k_dh_pull_root(DhIndex x, Dims d, const float* dq_in,
                                                      const float* dm_in, float* rpartial) {
    pdl_entry();
    const int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (c >= x.rchunk_off[x.U_cap]) return;
    const int u = x.rchunk_slot[c], p0 = x.rchunk_start[c];
    const int n = min(kDhChunk, x.off_root[u + 1] - p0);
    float4 acc[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int my_r = lane < n ? x.list_root[p0 + lane] : 0;
    constexpr int G = 4;
    for (int g = 0; g < n; g += G) {
        float4 qa[G][NM], ma[G][NM];
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const int r = __shfl_sync(0xffffffffu, my_r, min(g + t, 31));
#pragma unroll
            for (int i = 0; i < NM; ++i) {
                const int col = 4 * (lane + 32 * i);
                const bool ok = g + t < n && col < d.D;
                qa[t][i] = ok ? f4(dq_in + (std::size_t)r * d.ld_q + col) : make_float4(0.f, 0.f, 0.f, 0.f);
                ma[t][i] = ok ? f4(dm_in + (std::size_t)r * d.ld_m + d.DQ + col) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
            if (g + t >= n) break;
#pragma unroll
            for (int i = 0; i < NM; ++i)
                add4(acc[i], make_float4(qa[t][i].x + ma[t][i].x, qa[t][i].y + ma[t][i].y,
                                         qa[t][i].z + ma[t][i].z, qa[t][i].w + ma[t][i].w));
        }
    }
    float* o = rpartial + (std::size_t)c * d.D;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col < d.D) *reinterpret_cast<float4*>(o + col) = acc[i];
    }
}

// Sum of the chunk partials [c0, c1) in chunk order, 4 loads in flight.
template <int NM>
__device__ __forceinline__ void sum_chunks(float4 (&g)[NM], const float* part, int c0, int c1,
                                           int D, int lane) {
    for (int c = c0; c < c1; c += 4) {
        float4 v[4][NM];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < NM; ++i) {
                const int col = 4 * (lane + 32 * i);
                v[t][i] = c + t < c1 && col < D ? f4(part + (std::size_t)(c + t) * D + col)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (c + t < c1)
#pragma unroll
                for (int i = 0; i < NM; ++i) add4(g[i], v[t][i]);
    }
}

// One warp per pending row u: dH = occurrence chunk partials then root chunk
// partials (chunk order), then the GRUCell backward (gate order r, z, n) to
// the gate pre-activation gradients dGi (input side) and dGh (hidden side).
template <int NM>
__global__ void __launch_bounds__(256) k_gru_bwd_dh(WorkerDev w, Dims d, DhIndex x,
                                                    const float* partial, const float* rpartial,
                                                    const float* save, float* dGi, float* dGh) {
    pdl_entry();
    const int u = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (u >= *w.nU) return;
    float4 g[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    sum_chunks<NM>(g, partial, x.chunk_off[u], x.chunk_off[u + 1], d.D, lane);
    sum_chunks<NM>(g, rpartial, x.rchunk_off[u], x.rchunk_off[u + 1], d.D, lane);
    const float* sv = save + (std::size_t)u * 4 * d.D;
    const float* hrow = w.mem + (std::size_t)w.pU[u] * d.D;  // exact h (h_gru may be tf32-rounded)
    float* gi = dGi + (std::size_t)u * d.ld_g;
    float* gh = dGh + (std::size_t)u * d.ld_g;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col >= d.D) continue;
        const float gv[4] = {g[i].x, g[i].y, g[i].z, g[i].w};
        const float4 r4 = f4(sv + col), z4 = f4(sv + d.D + col), n4 = f4(sv + 2 * d.D + col),
                     gn4 = f4(sv + 3 * d.D + col), h4 = f4(hrow + col);
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, zz[4] = {z4.x, z4.y, z4.z, z4.w};
        const float nn[4] = {n4.x, n4.y, n4.z, n4.w}, gg[4] = {gn4.x, gn4.y, gn4.z, gn4.w};
        const float hh[4] = {h4.x, h4.y, h4.z, h4.w};
        float o_r[4], o_z[4], o_n[4], o_hn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dn = gv[k] * (1.f - zz[k]);
            const float dz = gv[k] * (hh[k] - nn[k]);
            const float dpn = dn * (1.f - nn[k] * nn[k]);
            o_r[k] = rnd_if(dpn * gg[k] * rr[k] * (1.f - rr[k]), d.rnd);
            o_z[k] = rnd_if(dz * zz[k] * (1.f - zz[k]), d.rnd);
            o_n[k] = rnd_if(dpn, d.rnd);
            o_hn[k] = rnd_if(dpn * rr[k], d.rnd);
        }
        *reinterpret_cast<float4*>(gi + col) = make_float4(o_r[0], o_r[1], o_r[2], o_r[3]);
        *reinterpret_cast<float4*>(gi + d.D + col) = make_float4(o_z[0], o_z[1], o_z[2], o_z[3]);
        *reinterpret_cast<float4*>(gi + 2 * d.D + col) = make_float4(o_n[0], o_n[1], o_n[2], o_n[3]);
        *reinterpret_cast<float4*>(gh + col) = make_float4(o_r[0], o_r[1], o_r[2], o_r[3]);
        *reinterpret_cast<float4*>(gh + d.D + col) = make_float4(o_z[0], o_z[1], o_z[2], o_z[3]);
        *reinterpret_cast<float4*>(gh + 2 * d.D + col) = make_float4(o_hn[0], o_hn[1], o_hn[2], o_hn[3]);
    }
}

// JODIE: RNN cell backward on the summed memory-row gradients,
// dGi = dGh = dH (1 - h'^2), h' saved by k_rnn_fwd in save[u][0:D]
template <int NM>
__global__ void __launch_bounds__(256) k_rnn_bwd_dh(WorkerDev w, Dims d, DhIndex x,
                                                    const float* partial, const float* rpartial,
                                                    const float* save, float* dGi, float* dGh) {
    pdl_entry();
    const int u = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (u >= *w.nU) return;
    float4 g[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    sum_chunks<NM>(g, partial, x.chunk_off[u], x.chunk_off[u + 1], d.D, lane);
    sum_chunks<NM>(g, rpartial, x.rchunk_off[u], x.rchunk_off[u + 1], d.D, lane);
    const float* sv = save + (std::size_t)u * 4 * d.D;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col >= d.D) continue;
        const float4 h = f4(sv + col);
        const float4 o = make_float4(rnd_if(g[i].x * (1.f - h.x * h.x), d.rnd), rnd_if(g[i].y * (1.f - h.y * h.y), d.rnd),
                                     rnd_if(g[i].z * (1.f - h.z * h.z), d.rnd), rnd_if(g[i].w * (1.f - h.w * h.w), d.rnd));
        *reinterpret_cast<float4*>(dGi + (std::size_t)u * d.ld_g + col) = o;
        *reinterpret_cast<float4*>(dGh + (std::size_t)u * d.ld_g + col) = o;
    }
}
template __global__ void k_rnn_bwd_dh<1>(WorkerDev, Dims, DhIndex, const float*, const float*,
                                         const float*, float*, float*);
template __global__ void k_rnn_bwd_dh<2>(WorkerDev, Dims, DhIndex, const float*, const float*,
                                         const float*, float*, float*);

template __global__ void k_dh_pull<1, 2>(DhIndex, Dims, const float*, const float*, const float*,
                                         const float*, float*);
template __global__ void k_dh_pull<1, 4>(DhIndex, Dims, const float*, const float*, const float*,
                                         const float*, float*);
template __global__ void k_dh_pull<2, 2>(DhIndex, Dims, const float*, const float*, const float*,
                                         const float*, float*);
template __global__ void k_dh_pull<2, 4>(DhIndex, Dims, const float*, const float*, const float*,
                                         const float*, float*);
template __global__ void k_dh_pull_root<1>(DhIndex, Dims, const float*, const float*, float*);
template __global__ void k_dh_pull_root<2>(DhIndex, Dims, const float*, const float*, float*);
template __global__ void k_gru_bwd_dh<1>(WorkerDev, Dims, DhIndex, const float*, const float*,
                                         const float*, float*, float*);
template __global__ void k_gru_bwd_dh<2>(WorkerDev, Dims, DhIndex, const float*, const float*,
                                         const float*, float*, float*);

}  // namespace tgnk
}  // namespace spd
