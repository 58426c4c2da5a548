// Non-GEMM kernels of the TGN training step; see tgn_kernels.cuh. Semantics
// follow oracle/tgn_oracle.py line for line (which states the model choices).
#include "pdl.cuh"
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"

namespace spd {
namespace tgnk {

namespace {
__device__ __forceinline__ int warp_id_global() {
    return (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// memory row of local node n as seen by this step: the GRU-updated row when
// n had a pending message (slot >= 0), else the stored row.
__device__ __forceinline__ const float* memx_row(const WorkerDev& w, const float* mem_new, int D,
                                                 std::uint32_t n) {
    const int s = w.slot[n];
    return s >= 0 ? mem_new + (std::size_t)s * D : w.mem + (std::size_t)n * D;
}

__device__ __forceinline__ float softplusf(float x) { return x > 20.f ? x : log1pf(expf(x)); }
}  // namespace

__global__ void k_init_aug(float* buf, int rows, int cols, int ld) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)rows * ld) return;
    const int c = i % ld;
    if (c >= cols) buf[i] = c == cols ? 1.f : 0.f;
    else buf[i] = 0.f;
}

// Step-start zeroing of the gradient buffers and the backward's accumulation
// scratch (dH, and the GRU gate gradients whose unused rows the tensor-core
// weight-gradient GEMM reads), one launch beside the forward.
// Grid-stride over a small grid: a full-size grid would fill every SM for
// its few microseconds and hold the step's first critical-path kernels back.
__global__ void k_zero_list(ZeroList z) {
    pdl_entry();
    std::size_t mx = z.nd;
#pragma unroll
    for (int k = 0; k < ZeroList::kMax; ++k) mx = z.n[k] > mx ? z.n[k] : mx;
    for (std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x; i < mx;
         i += (std::size_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < ZeroList::kMax; ++k)
            if (i < z.n[k]) z.p[k][i] = 0.f;
        if (i < z.nd) z.d[i] = 0.0;
    }
}

__global__ void k_zero2(float* a, std::size_t na, double* b, std::size_t nb) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) a[i] = 0.f;
    if (i < nb) b[i] = 0.0;
}

// K5 + K8: roots (src | dst | neg) and the recent-k neighbours strictly
// before t: lower_bound of t in the node's time-sorted adjacency, last K
// entries. One warp per root: a 33-ary search (32 lanes probe, a ballot
// narrows the range 33x per round: 4 dependent rounds for a 10^6-entry hub
// instead of 20 for a binary search), then lanes copy the K neighbours.
__global__ void k_roots_nbrs(WorkerDev w, int B, int K,
                             std::uint32_t* roots, double* root_t, std::uint32_t* nbr_node,
                             std::uint32_t* nbr_ev, double* nbr_dt, int* cnt) {
    pdl_entry();
    const int r = warp_id_global(), lane = lane_id();
    if (r >= 3 * B) return;
    const std::uint64_t lo = w.ctl[0], neg_base = w.ctl[1];
    const int which = r / B, i = r % B;
    const std::uint64_t e = lo + i;
    const double t = w.ev_ts[e];
    std::uint32_t node;
    if (which == 0) node = w.ev_src[e];
    else if (which == 1) node = w.ev_dst[e];
    else node = w.pool[mix64(neg_base ^ (std::uint64_t)i) % w.n_pool];
    const std::uint64_t a = w.adj_off[node], b = w.adj_off[node + 1];
    std::uint64_t l = a, h = b;  // answer (first index with ts >= t) lies in [l, h]
    while (h - l > 32) {
        const std::uint64_t step = (h - l + 32) / 33;
        const std::uint64_t p = l + (std::uint64_t)(lane + 1) * step;
        const bool below = p < h && w.adj_ts[p] < t;
        const int c = __popc(__ballot_sync(0xffffffffu, below));  // probes below t: a prefix
        const std::uint64_t nl = l + (std::uint64_t)c * step + (c > 0 ? 1 : 0);
        h = min(h, l + (std::uint64_t)(c + 1) * step);
        l = nl;
    }
    const std::uint64_t p = l + lane;
    const bool below = p < h && w.adj_ts[p] < t;
    const std::uint64_t pos = l + __popc(__ballot_sync(0xffffffffu, below));
    const std::uint64_t avail = pos - a;
    const int c = avail < (std::uint64_t)K ? (int)avail : K;
    const std::uint64_t start = pos - c;
    if (lane == 0) {
        roots[r] = node;
        root_t[r] = t;
        cnt[r] = c;
    }
    if (lane < K) {
        const std::size_t o = (std::size_t)r * K + lane;
        if (lane < c) {
            const std::uint64_t idx = start + lane;
            nbr_node[o] = w.adj_nbr[idx];
            nbr_ev[o] = w.adj_ev[idx];
            nbr_dt[o] = t - w.adj_ts[idx];
        } else {
            nbr_node[o] = kPad;
            nbr_ev[o] = 0;
            nbr_dt[o] = 0.0;
        }
    }
}

// K1 + K2 for the memory updater: message [s_i | s_j | e | phi(t - t_i^-)]
// and hidden s_i for every pending node (one warp per node). 128-bit access:
// lane l moves memory columns 4l..4l+3 of both endpoint rows and 8 bf16
// feature columns (one 16-B load), and evaluates 4 time columns.
__global__ void k_gru_gather(WorkerDev w, Dims d, const float* time_w, const float* time_b,
                             float* x, float* h, int set_slot) {
    pdl_entry();
    const int u = warp_id_global(), lane = lane_id();
    if (u >= *w.nU) return;
    const std::uint32_t node = w.pU[u], other = w.pOther[u], ev = w.pEv[u];
    const double dt = w.pTs[u] - w.lu[node];
    if (set_slot && lane == 0) w.slot[node] = u;
    float* xr = x + (std::size_t)u * d.ld_x;
    float* hr = h + (std::size_t)u * d.ld_h;
    const float4* mn = reinterpret_cast<const float4*>(w.mem + (std::size_t)node * d.D);
    // (DyRep: the other endpoint's attention embedding stored with the message)
    const float4* mo = reinterpret_cast<const float4*>(w.pZ ? w.pZ + (std::size_t)u * d.D
                                                            : w.mem + (std::size_t)other * d.D);
    for (int c4 = lane; c4 < d.D / 4; c4 += 32) {
        const float4 v = rnd4_if(__ldg(mn + c4), d.rnd);
        reinterpret_cast<float4*>(xr)[c4] = v;
        reinterpret_cast<float4*>(hr)[c4] = v;
        reinterpret_cast<float4*>(xr + d.D)[c4] = rnd4_if(__ldg(mo + c4), d.rnd);
    }
    const uint4* fr = reinterpret_cast<const uint4*>(w.feat + (std::size_t)ev * d.Fp);
    float* xf = xr + 2 * d.D;
    for (int c8 = lane; 8 * c8 < d.F; c8 += 32) {  // bf16 -> f32 is exact
        const uint4 raw = __ldg(fr + c8);
        const float f[8] = {__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                            __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u),
                            __uint_as_float(raw.z << 16), __uint_as_float(raw.z & 0xFFFF0000u),
                            __uint_as_float(raw.w << 16), __uint_as_float(raw.w & 0xFFFF0000u)};
        if (8 * c8 + 8 <= d.F) {
            reinterpret_cast<float4*>(xf)[2 * c8] = make_float4(f[0], f[1], f[2], f[3]);
            reinterpret_cast<float4*>(xf)[2 * c8 + 1] = make_float4(f[4], f[5], f[6], f[7]);
        } else {
            for (int q = 0; q < 8 && 8 * c8 + q < d.F; ++q) xf[8 * c8 + q] = f[q];
        }
    }
    // time columns start at 2D + F: 16-, 8- or 4-B aligned by F mod 4
    float* xt = xr + 2 * d.D + d.F;
    for (int c4 = lane; c4 < d.T / 4; c4 += 32) {
        const float4 tw = __ldg(reinterpret_cast<const float4*>(time_w) + c4);
        const float4 tb = __ldg(reinterpret_cast<const float4*>(time_b) + c4);
        const float2 a = make_float2(rnd_if(time_cos(tw.x, tb.x, dt), d.rnd), rnd_if(time_cos(tw.y, tb.y, dt), d.rnd));
        const float2 b = make_float2(rnd_if(time_cos(tw.z, tb.z, dt), d.rnd), rnd_if(time_cos(tw.w, tb.w, dt), d.rnd));
        if (d.F % 4 == 0) {
            reinterpret_cast<float4*>(xt)[c4] = make_float4(a.x, a.y, b.x, b.y);
        } else if (d.F % 2 == 0) {
            reinterpret_cast<float2*>(xt)[2 * c4] = a;
            reinterpret_cast<float2*>(xt)[2 * c4 + 1] = b;
        } else {
            xt[4 * c4] = a.x; xt[4 * c4 + 1] = a.y; xt[4 * c4 + 2] = b.x; xt[4 * c4 + 3] = b.y;
        }
    }
}

// GRUCell (PyTorch gate order r, z, n) on G_i = W_ih x + b_ih, G_h = W_hh h + b_hh.
__global__ void k_gru_fwd(WorkerDev w, Dims d, const float* Gi, const float* Gh, const float* h,
                          float* save, float* mem_new) {
    pdl_entry();
    const int nU = *w.nU;
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)nU * d.D) return;
    const int u = i / d.D, c = i % d.D;
    const float* gi = Gi + (std::size_t)u * d.ld_g;
    const float* gh = Gh + (std::size_t)u * d.ld_g;
    const float r = sigmoidf_(gi[c] + gh[c]);
    const float z = sigmoidf_(gi[d.D + c] + gh[d.D + c]);
    const float ghn = gh[2 * d.D + c];
    const float n = tanhf(gi[2 * d.D + c] + r * ghn);
    const float hv = w.mem[(std::size_t)w.pU[u] * d.D + c];  // exact h (h_gru may be tf32-rounded)
    mem_new[(std::size_t)u * d.D + c] = (1.f - z) * n + z * hv;
    if (save) {
        float* s = save + (std::size_t)u * 4 * d.D;
        s[c] = r;
        s[d.D + c] = z;
        s[2 * d.D + c] = n;
        s[3 * d.D + c] = ghn;
    }
}

// ---- JODIE backbone (oracle/tgn_oracle.py states the model):
// RNN memory updater h' = tanh(Gi + Gh), Gi = [x | 1] W_ih^T, Gh = [h | 1] W_hh^T
// (TGN's "rnn" memory updater), and the time-projection embedding
// emb = s' (1 + log1p(t - t_last) w_tp + b_tp) of the root's (updated) memory.
__global__ void k_rnn_fwd(WorkerDev w, Dims d, const float* Gi, const float* Gh, float* save,
                          float* mem_new) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)(*w.nU) * d.D) return;
    const int u = static_cast<int>(i / d.D), c = static_cast<int>(i % d.D);
    const float v = tanhf(Gi[(std::size_t)u * d.ld_g + c] + Gh[(std::size_t)u * d.ld_g + c]);
    mem_new[(std::size_t)u * d.D + c] = v;
    if (save) save[(std::size_t)u * 4 * d.D + c] = v;
}

// one warp per root: s_r = log1p(max(0, t_r - t_last)) in f64 (t_last = the
// pending message's ts for a node just updated, else its clock), then the
// projected row; s_r kept for the backward
__global__ void k_jodie_embed(WorkerDev w, Dims d, int R, const std::uint32_t* roots,
                              const double* root_t, const float* mem_new, const float* tp, int ldtp,
                              float* emb, float* s_out) {
    pdl_entry();
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R) return;
    const std::uint32_t n = roots[r];
    const int sl = w.slot[n];
    const float* m = sl >= 0 ? mem_new + (std::size_t)sl * d.D : w.mem + (std::size_t)n * d.D;
    const double last = sl >= 0 ? w.pTs[sl] : w.lu[n];
    if (!tp) {  // DyRep: identity embedding (128-bit rows, D % 4 == 0)
        for (int c4 = lane; c4 < d.D / 4; c4 += 32)
            reinterpret_cast<float4*>(emb + (std::size_t)r * d.D)[c4] = reinterpret_cast<const float4*>(m)[c4];
        return;
    }
    const float s = static_cast<float>(log1p(fmax(0.0, root_t[r] - last)));
    for (int c = lane; c < d.D; c += 32)
        emb[(std::size_t)r * d.D + c] = m[c] * (1.f + s * tp[(std::size_t)c * ldtp] + tp[(std::size_t)c * ldtp + 1]);
    if (lane == 0) s_out[r] = s;
}

// Per-head A_h^T B_h (A_h, B_h: rows h dh .. (h+1) dh of A and B): out[i][h
// hstride + k] = sum_c A[h dh + c][i] B[h dh + c][k], i < rows, k < cols, in c
// order (tgn_trainer.cu build_wqk); tf32-rounded when it feeds tensor cores.
__global__ void k_wprod_t(float* out, int ldo, int hstride, const float* A, int lda, const float* B, int ldb,
                          int rows, int cols, int dh, int H, int rnd) {
    pdl_entry();
    const std::size_t t = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (std::size_t)H * rows * cols) return;
    const int k = static_cast<int>(t % cols), i = static_cast<int>((t / cols) % rows);
    const int h = static_cast<int>(t / ((std::size_t)rows * cols));
    const float* a = A + (std::size_t)h * dh * lda + i;
    const float* b = B + (std::size_t)h * dh * ldb + k;
    float acc = 0.f;
    for (int c = 0; c < dh; ++c) acc = fmaf(a[(std::size_t)c * lda], b[(std::size_t)c * ldb], acc);
    out[(std::size_t)i * ldo + (std::size_t)h * hstride + k] = rnd ? tf32r(acc) : acc;
}

// Folded output x value projection (tgn_trainer.cu build_wc): add b_o to head
// 0's bias column and round the product to tf32 when it feeds tensor cores.
__global__ void k_wc_fix(float* wc, int rows, int ld, int DK, const float* b_o, int ld_o, int rnd) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)rows * ld) return;
    const int n = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
    float v = wc[i];
    if (c == DK) v += b_o[(std::size_t)n * ld_o];
    wc[i] = rnd ? tf32r(v) : v;
}

// DyRep message payload: after k_pending filled the other pending set with
// this batch's last messages, copy each record's other-endpoint attention
// embedding (z = [z_src rows | z_dst rows] of the batch) beside it. Record of
// node u from event e = lo + k: u is the source (other = destination, row
// B + k) unless it is only the destination (other = source, row k); a
// self-loop's two rows are the same node at the same time, hence equal.
__global__ void k_dyrep_stash(WorkerDev w, int D, int B, const float* z) {
    pdl_entry();
    const int i = warp_id_global(), lane = lane_id();
    if (i >= *w.nxN) return;
    const std::uint64_t e = w.nxEv[i];
    const int k = static_cast<int>(e - w.ctl[0]);
    const int row = w.ev_src[e] == w.nxU[i] ? B + k : k;
    const float4* zr = reinterpret_cast<const float4*>(z + (std::size_t)row * D);
    float4* o = reinterpret_cast<float4*>(w.nxZ + (std::size_t)i * D);
    for (int c4 = lane; c4 < D / 4; c4 += 32) o[c4] = zr[c4];
}

// backward of the time projection: the roots' memory-row gradients go to
// dq_in[:, :D] (dm_in[:, DQ:DQ+D] = 0), where k_dh_pull_root sums them per
// pending row as for TGN's query / merge inputs; (w_tp, b_tp) gradients as
// per-block f64 partials over a fixed row range (k_jodie_tp_final sums them)
__global__ void k_jodie_bwd(WorkerDev w, Dims d, int R, const std::uint32_t* roots, const float* mem_new,
                            const float* tp, int ldtp, const float* s_in, const float* d_emb, float* dq_in,
                            float* dm_in, int rows_per_block, double* part) {
    pdl_entry();
    const int c = threadIdx.x;
    if (c >= d.D) return;
    if (!tp) {  // DyRep: identity embedding, d(memory row) = d_emb
        const int r0 = blockIdx.x * rows_per_block, r1 = min(R, r0 + rows_per_block);
        for (int r = r0; r < r1; ++r) {
            dq_in[(std::size_t)r * d.ld_q + c] = d_emb[(std::size_t)r * d.D + c];
            dm_in[(std::size_t)r * d.ld_m + d.DQ + c] = 0.f;
        }
        return;
    }
    const float wc = tp[(std::size_t)c * ldtp], bc = tp[(std::size_t)c * ldtp + 1];
    double aw = 0.0, ab = 0.0;
    const int r0 = blockIdx.x * rows_per_block, r1 = min(R, r0 + rows_per_block);
    for (int r = r0; r < r1; ++r) {
        const std::uint32_t n = roots[r];
        const int sl = w.slot[n];
        const float m = sl >= 0 ? mem_new[(std::size_t)sl * d.D + c] : w.mem[(std::size_t)n * d.D + c];
        const float g = d_emb[(std::size_t)r * d.D + c], s = s_in[r];
        dq_in[(std::size_t)r * d.ld_q + c] = g * (1.f + s * wc + bc);
        dm_in[(std::size_t)r * d.ld_m + d.DQ + c] = 0.f;
        aw += (double)(g * m * s);
        ab += (double)(g * m);
    }
    part[(std::size_t)blockIdx.x * 2 * d.D + c] = aw;
    part[(std::size_t)blockIdx.x * 2 * d.D + d.D + c] = ab;
}

__global__ void k_jodie_tp_final(int D, int nblk, const double* part, float* g, int ldtp) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * D) return;
    double a = 0.0;
    for (int b = 0; b < nblk; ++b) a += part[(std::size_t)b * 2 * D + i];
    g[(std::size_t)(i % D) * ldtp + i / D] += static_cast<float>(a);
}

// K1 + K2 for the attention query: q_in = [s_root | phi(0)] (one warp per
// root). The key/value rows are gathered inside the attention kernels
// (tgn_attn.cu) and never stored.
// The roots' memory rows go to both of their readers: the query input
// [s_root | phi(0)] and the MergeLayer input's s_root columns (m_in[:, DQ:];
// its attention columns come from the output-projection GEMM's row-masked
// epilogue), so m_in needs no gather of its own.
__global__ void k_query_gather(WorkerDev w, Dims d, int R, const float* time_w,
                               const float* time_b, const std::uint32_t* roots,
                               const float* mem_new, float* q_in, float* m_in) {
    pdl_entry();
    const int row = warp_id_global(), lane = lane_id();
    if (row >= R) return;
    const float4* m = reinterpret_cast<const float4*>(memx_row(w, mem_new, d.D, roots[row]));
    float* q = q_in + (std::size_t)row * d.ld_q;
    float* mi = m_in ? m_in + (std::size_t)row * d.ld_m + d.DQ : nullptr;
    for (int c4 = lane; c4 < d.D / 4; c4 += 32) {
        const float4 v = rnd4_if(m[c4], d.rnd);
        reinterpret_cast<float4*>(q)[c4] = v;
        if (mi) reinterpret_cast<float4*>(mi)[c4] = v;
    }
    for (int c4 = lane; c4 < d.T / 4; c4 += 32) {
        const float4 tw = __ldg(reinterpret_cast<const float4*>(time_w) + c4);
        const float4 tb = __ldg(reinterpret_cast<const float4*>(time_b) + c4);
        reinterpret_cast<float4*>(q + d.D)[c4] =
            make_float4(rnd_if(time_cos(tw.x, tb.x, 0.0), d.rnd), rnd_if(time_cos(tw.y, tb.y, 0.0), d.rnd),
                        rnd_if(time_cos(tw.z, tb.z, 0.0), d.rnd), rnd_if(time_cos(tw.w, tb.w, 0.0), d.rnd));
    }
}

// Decoder input rows: p < B -> [z_src | z_dst], p >= B -> [z_src | z_neg].
__global__ void k_dec_gather(Dims d, int B, const float* emb, float* d_in) {
    pdl_entry();
    const int p = warp_id_global(), lane = lane_id();
    if (p >= 2 * B) return;
    const int i = p < B ? p : p - B;
    const int other = p < B ? B + i : 2 * B + i;
    float4* o = reinterpret_cast<float4*>(d_in + (std::size_t)p * d.ld_din);
    const float4* a = reinterpret_cast<const float4*>(emb + (std::size_t)i * d.D);
    const float4* b = reinterpret_cast<const float4*>(emb + (std::size_t)other * d.D);
    for (int c4 = lane; c4 < d.D / 4; c4 += 32) {
        o[c4] = a[c4];
        o[d.D / 4 + c4] = b[c4];
    }
}

// K7 head: logit = D1 . w2 + b2, BCE-with-logits terms and their gradients.
// w2 = augmented [w | b] row of dec2.
__global__ void k_dec_head(Dims d, int B, const float* D1, const float* w2, float* dlogit,
                           float* lossv, float* dD1, float* logits) {
    pdl_entry();
    const int p = warp_id_global(), lane = lane_id();
    if (p >= 2 * B) return;
    const float* x = D1 + (std::size_t)p * d.ld_d1;
    float acc = 0.f;
    for (int c = lane; c < d.D; c += 32) acc += x[c] * w2[c];
    acc = warp_sum(acc) + w2[d.D];
    const bool pos = p < B;
    const float sig = sigmoidf_(acc);
    const float g = (sig - (pos ? 1.f : 0.f)) / (float)B;
    if (lane == 0) {
        dlogit[(std::size_t)p * 4] = g;
        lossv[p] = (pos ? softplusf(-acc) : softplusf(acc)) / (float)B;
        if (logits) logits[p] = acc;
    }
    float* dx = dD1 + (std::size_t)p * d.D;
    for (int c = lane; c < d.D; c += 32) dx[c] = x[c] > 0.f ? g * w2[c] : 0.f;
}

// Decoder layer 1 without the gathered [z_u | z_v] rows: the src half of the
// weight is applied once per event (Ya = z_src W_a^T), the other half to the
// dst and negative embeddings (Yb = z_{dst|neg} W_b^T), so
//   D1_pos[i] = relu(Ya[i] + Yb[i] + b1),  D1_neg[i] = relu(Ya[i] + Yb[B+i] + b1)
// (the MergeLayer's W [z_u | z_v] + b split by columns), then the head as
// k_dec_head. W1 = augmented dec1 rows [w(2D) | b], row stride ld1.
__global__ void k_dec_head2(Dims d, int B, const float* Ya, const float* Yb, const float* W1,
                            int ld1, const float* w2, float* D1, float* dlogit, float* lossv,
                            float* dD1, float* logits) {
    pdl_entry();
    const int p = warp_id_global(), lane = lane_id();
    if (p >= 2 * B) return;
    const int i = p < B ? p : p - B;
    const float* a = Ya + (std::size_t)i * d.D;
    const float* b = Yb + (std::size_t)p * d.D;  // dst rows [0, B), negative rows [B, 2B)
    float* x = D1 + (std::size_t)p * d.ld_d1;
    float acc = 0.f;
    for (int c = lane; c < d.D; c += 32) {
        const float z = fmaxf(a[c] + b[c] + W1[(std::size_t)c * ld1 + 2 * d.D], 0.f);
        x[c] = z;
        acc += z * w2[c];
    }
    acc = warp_sum(acc) + w2[d.D];
    const bool pos = p < B;
    const float sig = sigmoidf_(acc);
    const float g = (sig - (pos ? 1.f : 0.f)) / (float)B;
    if (lane == 0) {
        dlogit[(std::size_t)p * 4] = g;
        lossv[p] = (pos ? softplusf(-acc) : softplusf(acc)) / (float)B;
        if (logits) logits[p] = acc;
    }
    __syncwarp();
    float* dx = dD1 + (std::size_t)p * d.D;
    for (int c = lane; c < d.D; c += 32) dx[c] = x[c] > 0.f ? g * w2[c] : 0.f;
}

// K7 fused decoder (FP32 FFMA, the north star's rule for the decoder): per
// block of EV events (kDecEv, or kDecEvSmall for small batches), from the embeddings of their src / dst / negative
// roots to the data gradient of those embeddings, in one launch —
//   Y_src = W_a z_src, Y_dst = W_b z_dst, Y_neg = W_b z_neg
//   D1 = relu(Y_src + Y_{dst|neg} + b1); logit = D1 . w2 + b2; BCE terms
//   dlogit = (sigmoid - y) / B; dD1 = [D1 > 0] dlogit w2
//   d_src = dD1_pos W_a + dD1_neg W_a, d_dst = dD1_pos W_b, d_neg = dD1_neg W_b
// (the MergeLayer of oracle/tgn_oracle.py _decode applied to [z_u | z_v] by
// input halves). W1 = [W_a | W_b | b1] rows (row stride ld1) are staged in
// shared memory once per block; thread (kind, n) owns output column n of the
// block's EV rows of one kind (src, dst, neg) and reads its weight row /
// column with 16-B loads while the activations broadcast. Writes D1, dlogit,
// dD1 (the weight gradients' inputs), loss terms, logits and d_emb. bwd = 0
// (evaluation): forward and logits only.
template <int MAXT, int MINB, int EV>
__global__ void __launch_bounds__(MAXT, MINB)
    k_decoder(Dims d, int B, const float* emb, const float* W1, int ld1, const float* w2, float* D1,
              float* dlogit, float* lossv, float* dD1, float* logits, float* d_emb, int bwd, int pre) {
    // pre: the weight staging (parameters only) is issued before the wait for
    // the producer of emb (PDL), overlapping that kernel's tail
    pdl_launch();
    if (!pre) pdl_wait();
    extern __shared__ __align__(16) float dsm[];
    const int D = d.D, ldw = 2 * D + 4, ldz = D + 4;
    float* sW = dsm;                                  // [D][ldw]: W_a | W_b | b1
    float* sZ = sW + (std::size_t)D * ldw;            // [3 EV][ldz]: z rows; later dD1 [2 EV]
    float* sY = sZ + 3 * EV * ldz;                // [3 EV][ldz]
    float* sD1 = sY + 3 * EV * ldz;               // [2 EV][ldz]
    float* sw2 = sD1 + 2 * EV * ldz;              // [ldz]
    float* sg = sw2 + ldz;                            // [2 EV]
    float* sdD1 = sZ;
    __shared__ __align__(8) std::uint64_t bar;
    const int i0 = blockIdx.x * EV;
    const int nev = min(EV, B - i0);
    const int tid = threadIdx.x, nt = blockDim.x;
    // stage the weight rows (cols 0 .. 2D+3: W_a | W_b | b1 | pad) and the
    // block's embedding rows with TMA bulk copies issued by warp 0 on one mbarrier
    if (tid < 32) {
        if (tid == 0) {
            bar_init(&bar);
            bar_expect(&bar, unsigned(D * ldw * 4 + 3 * nev * D * 4));
        }
        __syncwarp();
        for (int n = tid; n < D; n += 32)
            bulk_g2s(sW + (std::size_t)n * ldw, W1 + (std::size_t)n * ld1, unsigned(ldw * 4), &bar);
        if (pre) pdl_wait();
        for (int r = tid; r < 3 * nev; r += 32) {
            const int kind = r / nev, e = r % nev;
            bulk_g2s(sZ + (std::size_t)(kind * EV + e) * ldz, emb + ((std::size_t)kind * B + i0 + e) * D,
                     unsigned(D * 4), &bar);
        }
    }
    for (int i = tid; i < 3 * (EV - nev) * D; i += nt) {  // rows past the batch: zero
        const int r = i / D, kind = r / (EV - nev), e = nev + r % (EV - nev);
        sZ[(std::size_t)(kind * EV + e) * ldz + i % D] = 0.f;
    }
    for (int i = tid; i <= D; i += nt) sw2[i] = w2[i];
    if (pre && tid >= 32) pdl_wait();  // (warp 0 waited before its embedding-row copies)
    __syncthreads();  // (barrier initialised before anyone waits)
    bar_wait(&bar, 0);
    // forward projections: thread (kind, n); for even D each thread owns the
    // output pair (n, n + D/2), sharing its activation loads (half the shared-
    // memory traffic; each output's summation order unchanged)
    const bool blk = (D & 1) == 0;
    const int Dh = D >> 1;
    if (blk) {
        if (tid < 3 * Dh) {
            const int kind = tid / Dh, n = tid % Dh;
            const float* wr0 = sW + (std::size_t)n * ldw + (kind ? D : 0);
            const float* wr1 = wr0 + (std::size_t)Dh * ldw;
            const float* z = sZ + (std::size_t)kind * EV * ldz;
            float a0[EV], a1[EV];
#pragma unroll
            for (int e = 0; e < EV; ++e) a0[e] = a1[e] = 0.f;
#pragma unroll 1
            for (int k = 0; k < D; k += 4) {
                const float4 w = *reinterpret_cast<const float4*>(wr0 + k);
                const float4 u = *reinterpret_cast<const float4*>(wr1 + k);
#pragma unroll
                for (int e = 0; e < EV; ++e) {
                    const float4 x = *reinterpret_cast<const float4*>(z + (std::size_t)e * ldz + k);
                    a0[e] = fmaf(x.x, w.x, a0[e]);
                    a0[e] = fmaf(x.y, w.y, a0[e]);
                    a0[e] = fmaf(x.z, w.z, a0[e]);
                    a0[e] = fmaf(x.w, w.w, a0[e]);
                    a1[e] = fmaf(x.x, u.x, a1[e]);
                    a1[e] = fmaf(x.y, u.y, a1[e]);
                    a1[e] = fmaf(x.z, u.z, a1[e]);
                    a1[e] = fmaf(x.w, u.w, a1[e]);
                }
            }
#pragma unroll
            for (int e = 0; e < EV; ++e) {
                sY[(std::size_t)(kind * EV + e) * ldz + n] = a0[e];
                sY[(std::size_t)(kind * EV + e) * ldz + n + Dh] = a1[e];
            }
        }
    } else if (tid < 3 * D) {
        const int kind = tid / D, n = tid % D;
        const float* wr = sW + (std::size_t)n * ldw + (kind ? D : 0);
        const float* z = sZ + (std::size_t)kind * EV * ldz;
        float acc[EV];
#pragma unroll
        for (int e = 0; e < EV; ++e) acc[e] = 0.f;
#pragma unroll 2
        for (int k = 0; k < D; k += 4) {
            const float4 w = *reinterpret_cast<const float4*>(wr + k);
#pragma unroll
            for (int e = 0; e < EV; ++e) {
                const float4 x = *reinterpret_cast<const float4*>(z + (std::size_t)e * ldz + k);
                acc[e] = fmaf(x.x, w.x, acc[e]);
                acc[e] = fmaf(x.y, w.y, acc[e]);
                acc[e] = fmaf(x.z, w.z, acc[e]);
                acc[e] = fmaf(x.w, w.w, acc[e]);
            }
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) sY[(std::size_t)(kind * EV + e) * ldz + n] = acc[e];
    }
    __syncthreads();
    // D1 rows: p < EV positive (src, dst), p >= EV negative (src, neg)
    for (int i = tid; i < 2 * EV * D; i += nt) {
        const int p = i / D, n = i % D, e = p % EV;
        const float v = sY[(std::size_t)e * ldz + n] + sY[(std::size_t)((p < EV ? 1 : 2) * EV + e) * ldz + n] +
                        sW[(std::size_t)n * ldw + 2 * D];
        const float x = fmaxf(v, 0.f);
        sD1[(std::size_t)p * ldz + n] = x;
        if (bwd && e < nev) D1[(std::size_t)((p < EV ? 0 : B) + i0 + e) * d.ld_d1 + n] = x;
    }
    __syncthreads();
    // logits and BCE terms: one warp per pair row
    {
        const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
        for (int p = warp; p < 2 * EV; p += nw) {
            const int e = p % EV;
            const float* x = sD1 + (std::size_t)p * ldz;
            float acc = 0.f;
            for (int c = lane; c < D; c += 32) acc += x[c] * sw2[c];
            acc = warp_sum(acc) + sw2[D];
            const bool pos = p < EV;
            const float g = (sigmoidf_(acc) - (pos ? 1.f : 0.f)) / (float)B;
            if (lane == 0) {
                sg[p] = g;
                if (e < nev) {
                    const std::size_t gp = (pos ? 0 : B) + i0 + e;
                    if (bwd) dlogit[gp * 4] = g;
                    lossv[gp] = (pos ? softplusf(-acc) : softplusf(acc)) / (float)B;
                    if (logits) logits[gp] = acc;
                }
            }
        }
    }
    if (!bwd) return;
    __syncthreads();
    for (int i = tid; i < 2 * EV * D; i += nt) {  // dD1 -> global (the weight gradients' input)
        const int p = i / D, n = i % D, e = p % EV;
        const float v = sD1[(std::size_t)p * ldz + n] > 0.f ? sg[p] * sw2[n] : 0.f;
        sD1[(std::size_t)p * ldz + n] = v;  // (D1 itself is no longer read)
        if (e < nev) dD1[(std::size_t)((p < EV ? 0 : B) + i0 + e) * D + n] = v;
    }
    __syncthreads();
    // data gradients, as the oracle's autograd forms them (two decoder calls,
    // pos and neg): thread (q, k), q = 0 dD1_pos W_a, 1 dD1_neg W_a, 2 dD1_pos W_b,
    // 3 dD1_neg W_b; d_src = q0 + q1 (summed through shared memory over the
    // z rows, no longer read), d_dst = q2, d_neg = q3
    float acc[EV];
    const int q = tid / D, k = tid % D;
    if (tid < 4 * D) {
        const float* wc = sW + (q >= 2 ? D : 0) + k;  // column k of W_a / W_b
        const float* g = sD1 + (std::size_t)(q & 1) * EV * ldz;
#pragma unroll
        for (int e = 0; e < EV; ++e) acc[e] = 0.f;
#pragma unroll 2
        for (int n = 0; n < D; n += 4) {
            const float w0 = wc[(std::size_t)n * ldw], w1 = wc[(std::size_t)(n + 1) * ldw],
                        w2_ = wc[(std::size_t)(n + 2) * ldw], w3 = wc[(std::size_t)(n + 3) * ldw];
#pragma unroll
            for (int e = 0; e < EV; ++e) {
                const float4 x = *reinterpret_cast<const float4*>(g + (std::size_t)e * ldz + n);
                acc[e] = fmaf(x.x, w0, acc[e]);
                acc[e] = fmaf(x.y, w1, acc[e]);
                acc[e] = fmaf(x.z, w2_, acc[e]);
                acc[e] = fmaf(x.w, w3, acc[e]);
            }
        }
        if (q == 1)
#pragma unroll
            for (int e = 0; e < EV; ++e) sdD1[(std::size_t)e * ldz + k] = acc[e];
    }
    __syncthreads();
    if (tid < 4 * D && q != 1) {
        const int kind = q == 0 ? 0 : q - 1;
#pragma unroll
        for (int e = 0; e < EV; ++e) {
            const float v = q == 0 ? acc[e] + sdD1[(std::size_t)e * ldz + k] : acc[e];
            if (e < nev) d_emb[((std::size_t)kind * B + i0 + e) * D + k] = rnd_if(v, d.rnd);
        }
    }
}

// Decoder weight gradients (FP32 FFMA), deterministic two-pass: block b sums
// its chunk of kDecWgEv events into part[b] = [dW1 (D x (2D+1)) | dW2 (D+1)]:
//   dW_a += dD1_pos^T z_src + dD1_neg^T z_src,  dW_b += dD1_pos^T z_dst + dD1_neg^T z_neg,
//   db1 += sum dD1_pos + sum dD1_neg,            dw2 += dlogit^T [D1 | 1]
// (the MergeLayer weight gradient of oracle/tgn_oracle.py by input halves);
// k_dec_wgrad_reduce adds the partials in block order to the gradients.
// blockIdx.y = (row half rs, input half): the block's 16 x 16 threads own
// rows tn + 16 (4 rs + i), columns half * D + tk + 16 j of dW1 (the same
// per-element summation order as one block per chunk, with 4x the blocks:
// a B = 200 batch has only 7 chunks).
__global__ void __launch_bounds__(256) k_dec_wgrad_part(Dims d, int B, const float* emb,
                                                        const float* dD1, const float* dlogit,
                                                        const float* D1, float* part) {
    pdl_entry();
    extern __shared__ __align__(16) float wsm[];
    const int D = d.D, ld = D + 4;
    float* sgp = wsm;                      // [TILE][ld] dD1 of positive pairs
    float* sgn = sgp + kDecWgTile * ld;    // [TILE][ld] dD1 of negative pairs
    float* sz = sgn + kDecWgTile * ld;     // [3][TILE][ld] z_src | z_dst | z_neg
    const int c0 = blockIdx.x * kDecWgEv, c1 = min(B, c0 + kDecWgEv);
    const int tid = threadIdx.x, D4 = D / 4;
    float* out = part + (std::size_t)blockIdx.x * (D * (2 * D + 1) + D + 1);
    const int tn = tid >> 4, tk = tid & 15;
    constexpr int TI = 4, TJ = 7;  // rows / columns per thread (D <= 112)
    const int half = blockIdx.y & 1, rb = 16 * TI * (blockIdx.y >> 1);  // input half, first row
    // the positive and the negative decoder call accumulate separately and
    // are added at the end (the oracle's autograd sums the two calls' grads);
    // the block's events stream through shared memory kDecWgTile at a time
    if (rb < D) {
        float ap[TI][TJ], an[TI][TJ];
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TJ; ++j) ap[i][j] = an[i][j] = 0.f;
        for (int e0 = c0; e0 < c1; e0 += kDecWgTile) {
            const int ne = min(kDecWgTile, c1 - e0);
            __syncthreads();  // the previous tile's readers are done
            for (int i = tid; i < 5 * kDecWgTile * D4; i += blockDim.x) {
                const int r = i / D4, c = 4 * (i % D4), which = r / kDecWgTile, e = r % kDecWgTile;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (e < ne) {
                    const float* src = which == 0 ? dD1 + (std::size_t)(e0 + e) * D
                                     : which == 1 ? dD1 + (std::size_t)(B + e0 + e) * D
                                                  : emb + ((std::size_t)(which - 2) * B + e0 + e) * D;
                    v = *reinterpret_cast<const float4*>(src + c);
                }
                *reinterpret_cast<float4*>(wsm + (std::size_t)r * ld + c) = v;
            }
            __syncthreads();
            for (int e = 0; e < ne; ++e) {
                float gp[TI], gn[TI], zp[TJ], zn[TJ];
#pragma unroll
                for (int i = 0; i < TI; ++i) {
                    const int n = min(rb + tn + 16 * i, D - 1);
                    gp[i] = sgp[e * ld + n];
                    gn[i] = sgn[e * ld + n];
                }
#pragma unroll
                for (int j = 0; j < TJ; ++j) {
                    const int k = min(tk + 16 * j, D - 1);
                    zp[j] = sz[((half == 0 ? 0 : 1) * kDecWgTile + e) * ld + k];  // z_src | z_dst
                    zn[j] = sz[((half == 0 ? 0 : 2) * kDecWgTile + e) * ld + k];  // z_src | z_neg
                }
#pragma unroll
                for (int i = 0; i < TI; ++i)
#pragma unroll
                    for (int j = 0; j < TJ; ++j) {
                        ap[i][j] = fmaf(gp[i], zp[j], ap[i][j]);
                        an[i][j] = fmaf(gn[i], zn[j], an[i][j]);
                    }
            }
        }
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TJ; ++j) {
                const int n = rb + tn + 16 * i, k = tk + 16 * j;
                if (n < D && k < D) out[(std::size_t)n * (2 * D + 1) + half * D + k] = ap[i][j] + an[i][j];
            }
    }
    if (blockIdx.y > 1) return;
    // bias columns: db1 (column 2D of dW1; y = 0) and dw2 (incl. db2; y = 1), straight from global
    if (blockIdx.y == 0)
    for (int n = tid; n < D; n += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int e = c0; e < c1; ++e) {
            a += dD1[(std::size_t)e * D + n];
            b += dD1[(std::size_t)(B + e) * D + n];
        }
        out[(std::size_t)n * (2 * D + 1) + 2 * D] = a + b;
    }
    if (blockIdx.y == 1)
    for (int c = tid; c <= D; c += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int e = c0; e < c1; ++e) {
            const std::size_t pp = e, pn = B + e;
            a += dlogit[pp * 4] * (c < D ? D1[pp * d.ld_d1 + c] : 1.f);
            b += dlogit[pn * 4] * (c < D ? D1[pn * d.ld_d1 + c] : 1.f);
        }
        out[(std::size_t)D * (2 * D + 1) + c] = a + b;
    }
}

__global__ void k_dec_wgrad_reduce(Dims d, int nblk, const float* part, float* g1, int ld1, float* g2) {
    pdl_entry();
    const int D = d.D, n1 = D * (2 * D + 1), per = n1 + D + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= per) return;
    float a = 0.f;
    for (int b = 0; b < nblk; ++b) a += part[(std::size_t)b * per + i];
    if (i < n1) g1[(std::size_t)(i / (2 * D + 1)) * ld1 + i % (2 * D + 1)] += a;
    else g2[i - n1] += a;
}

std::size_t dec_wgrad_smem_bytes(const Dims& d) { return 4 * std::size_t(5) * kDecWgTile * (d.D + 4); }

// 416 threads (d_mem <= 104) at two blocks per SM (<= 72 registers), else one;
// 8 events per block, 4 for small batches
#define SPD_DEC_INST(T, M, E)                                                                          \
    template __global__ void k_decoder<T, M, E>(Dims, int, const float*, const float*, int, const float*, \
                                                float*, float*, float*, float*, float*, float*, int, int);
SPD_DEC_INST(416, 2, kDecEv)
SPD_DEC_INST(416, 2, kDecEvSmall)
SPD_DEC_INST(768, 1, kDecEv)
SPD_DEC_INST(768, 1, kDecEvSmall)
#undef SPD_DEC_INST

std::size_t decoder_smem_bytes(const Dims& d, int ev) {
    const std::size_t D = d.D, ldw = 2 * D + 4, ldz = D + 4;
    return 4 * (D * ldw + 8 * ev * ldz + ldz + 2 * ev);
}

// Fixed-order single-block sum (deterministic loss).
__global__ void k_sum_loss(const float* lossv, int n, float* out) {
    pdl_entry();
    __shared__ float sh[32];
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += lossv[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) *out = v;
    }
}

__global__ void k_dec_scatter(Dims d, int B, const float* dd_in, float* d_emb) {
    pdl_entry();
    const int i = warp_id_global(), lane = lane_id();
    if (i >= B) return;
    const float* a = dd_in + (std::size_t)i * d.ld_din;
    const float* b = dd_in + (std::size_t)(B + i) * d.ld_din;
    for (int c = lane; c < d.D; c += 32) {
        d_emb[(std::size_t)i * d.D + c] = rnd_if(a[c] + b[c], d.rnd);
        d_emb[(std::size_t)(B + i) * d.D + c] = rnd_if(a[d.D + c], d.rnd);
        d_emb[(std::size_t)(2 * B + i) * d.D + c] = rnd_if(b[d.D + c], d.rnd);
    }
}

__global__ void k_mask_rows(float* buf, int R, int cols, int ld, const int* cnt) {
    pdl_entry();
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R || cnt[r] > 0) return;
    for (int c = lane; c < cols; c += 32) buf[(std::size_t)r * ld + c] = 0.f;
}

// Root-side time-encoder gradient: d/db of the query's phi(0) = cos(b)
// columns (f64 per-block fixed-order partials; d/dw is 0 at dt = 0). The
// roots' memory-column gradients are summed per pending row by tgn_dh.cu.
// block (32, 8); rows_per_block roots; part[block][2T].
__global__ void k_root_grad(Dims d, int R, const float* dq_in, const float* time_b,
                            int rows_per_block, double* part) {
    pdl_entry();
    __shared__ double red[8][32];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(R, r0 + rows_per_block);
    for (int c0 = 0; c0 < d.T; c0 += 32) {
        const int c = c0 + tx;
        double gb = 0.0;
        if (c < d.T) {
            const double sinb = sin((double)time_b[c]);
            for (int row = r0 + ty; row < r1; row += blockDim.y)
                gb -= sinb * (double)dq_in[(std::size_t)row * d.ld_q + d.D + c];
        }
        red[ty][tx] = gb;
        __syncthreads();
        if (ty == 0 && c < d.T) {
            double sb = 0.0;
            for (int y = 0; y < (int)blockDim.y; ++y) sb += red[y][tx];
            part[(std::size_t)blockIdx.x * 2 * d.T + c] = 0.0;
            part[(std::size_t)blockIdx.x * 2 * d.T + d.T + c] = sb;
        }
        __syncthreads();
    }
}

// one block per output (2T): fixed-order strided sums + tree -> deterministic.
__global__ void k_time_grad_final(int T, int nblocks, const double* part, double* acc) {
    pdl_entry();
    __shared__ double red[256];
    const int c = blockIdx.x;
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += part[(std::size_t)b * 2 * T + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) acc[c] += red[0];
}

__global__ void k_time_grad_apply(int T, const double* acc, float* gw, float* gb) {
    pdl_entry();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= T) return;
    gw[c] += (float)acc[c];
    gb[c] += (float)acc[T + c];
}

// Adam over the flat buffer, 4 parameters per thread (128-bit loads and
// stores; the flat layout is a multiple of 4 floats, a scalar tail otherwise)
__device__ __forceinline__ float adam_one(float& p, float g, float& m, float& v, float scale, float lr,
                                          float b1, float one_m_b1, float b2, float one_m_b2, float bc1,
                                          float bc2, float eps) {
    const float gi = g / scale;
    const float mi = b1 * m + one_m_b1 * gi;
    const float vi = b2 * v + one_m_b2 * gi * gi;
    m = mi;
    v = vi;
    const float mh = mi / bc1;
    const float vh = vi / bc2;
    p = p - lr * mh / (sqrtf(vh) + eps);
    return p;
}
// the flat gradient of parameter k with the deferred terms added as the
// kernels they replace would have (k_time_grad_apply: g + (float)acc;
// k_splitk_reduce: g + (((0 + w_0) + w_1) + ...))
__device__ __forceinline__ float fin_grad(float g, std::size_t k, const AdamFin& f) {
    if (f.tacc) {
        if (k >= f.tw && k < f.tw + f.T) return g + (float)f.tacc[k - f.tw];
        if (k >= f.tb && k < f.tb + f.T) return g + (float)f.tacc[f.T + (k - f.tb)];
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (q >= f.nsk) break;
        const AdamFin::SK& s = f.sk[q];
        if (k < s.off || k >= s.off + (std::size_t)s.M * s.ldc) continue;
        const int m = static_cast<int>((k - s.off) / s.ldc), c = static_cast<int>((k - s.off) % s.ldc);
        if (c >= s.N) return g;
        const float* w = s.ws + (std::size_t)m * s.ldws + c;
        float acc = 0.f;
        for (int z = 0; z < s.split; ++z) acc += w[(std::size_t)z * s.M * s.ldws];
        return g + acc;
    }
    return g;
}

__global__ void k_adam(float* p, float* g, float* m, float* v, std::size_t n, float scale,
                       float lr, float b1, float one_m_b1, float b2, float one_m_b2, const float* bc,
                       float eps, float* p_tc, AdamFin fin) {
    pdl_entry();
    const std::size_t i4 = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const std::size_t i = 4 * i4;
    if (i >= n) return;
    const float bc1 = bc[0], bc2 = bc[1];  // bias corrections of this step (host-written)
    if (i + 4 <= n) {
        float4 pp = *reinterpret_cast<float4*>(p + i), mm = *reinterpret_cast<float4*>(m + i);
        float4 vv = *reinterpret_cast<float4*>(v + i);
        float4 gg = *reinterpret_cast<float4*>(g + i);
        if (fin.tacc || fin.nsk) {  // (finalized gradients written back: introspection reads them)
            bool hit = false;
#pragma unroll
            for (int q = 0; q < 2; ++q) {  // split-K rows: 4 columns of one row per float4
                if (q >= fin.nsk) break;
                const AdamFin::SK& sk = fin.sk[q];
                if (i < sk.off || i >= sk.off + (std::size_t)sk.M * sk.ldc) continue;
                const int mr = static_cast<int>((i - sk.off) / sk.ldc), c = static_cast<int>((i - sk.off) % sk.ldc);
                if (c + 4 <= sk.N && sk.ldws % 4 == 0 && sk.ldc % 4 == 0) {
                    const float* w = sk.ws + (std::size_t)mr * sk.ldws + c;
                    float4 acc = *reinterpret_cast<const float4*>(w);
#pragma unroll 8
                    for (int z = 1; z < sk.split; ++z) {
                        const float4 t = *reinterpret_cast<const float4*>(w + (std::size_t)z * sk.M * sk.ldws);
                        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
                    }
                    gg.x += acc.x; gg.y += acc.y; gg.z += acc.z; gg.w += acc.w;
                    hit = true;
                }
            }
            if (!hit) {
                const float4 g0 = gg;
                gg.x = fin_grad(gg.x, i, fin);
                gg.y = fin_grad(gg.y, i + 1, fin);
                gg.z = fin_grad(gg.z, i + 2, fin);
                gg.w = fin_grad(gg.w, i + 3, fin);
                hit = g0.x != gg.x || g0.y != gg.y || g0.z != gg.z || g0.w != gg.w;
            }
            if (hit) *reinterpret_cast<float4*>(g + i) = gg;
        }
        adam_one(pp.x, gg.x, mm.x, vv.x, scale, lr, b1, one_m_b1, b2, one_m_b2, bc1, bc2, eps);
        adam_one(pp.y, gg.y, mm.y, vv.y, scale, lr, b1, one_m_b1, b2, one_m_b2, bc1, bc2, eps);
        adam_one(pp.z, gg.z, mm.z, vv.z, scale, lr, b1, one_m_b1, b2, one_m_b2, bc1, bc2, eps);
        adam_one(pp.w, gg.w, mm.w, vv.w, scale, lr, b1, one_m_b1, b2, one_m_b2, bc1, bc2, eps);
        *reinterpret_cast<float4*>(p + i) = pp;
        *reinterpret_cast<float4*>(m + i) = mm;
        *reinterpret_cast<float4*>(v + i) = vv;
        if (p_tc) *reinterpret_cast<float4*>(p_tc + i) = make_float4(tf32r(pp.x), tf32r(pp.y), tf32r(pp.z), tf32r(pp.w));
        return;
    }
    for (std::size_t k = i; k < n; ++k) {
        g[k] = fin_grad(g[k], k, fin);
        adam_one(p[k], g[k], m[k], v[k], scale, lr, b1, one_m_b1, b2, one_m_b2, bc1, bc2, eps);
        if (p_tc) p_tc[k] = tf32r(p[k]);
    }
}

// Adam on the sum of several gradient buffers (concurrent local workers,
// tgn_lanes.cu), summed in list order — the order the peer transport uses.
__global__ void k_adam_multi(float* p, GradList gl, float* m, float* v, std::size_t n, float scale,
                             float lr, float b1, float one_m_b1, float b2, float one_m_b2, const float* bc,
                             float eps, float* p_tc) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float g = gl.g[0][i];
    for (int r = 1; r < gl.n; ++r) g += gl.g[r][i];
    adam_one(p[i], g, m[i], v[i], scale, lr, b1, one_m_b1, b2, one_m_b2, bc[0], bc[1], eps);
    if (p_tc) p_tc[i] = tf32r(p[i]);
}

__global__ void k_round_tf32(const float* src, float* dst, std::size_t n) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = tf32r(src[i]);
}

// Persist the GRU rows of pending nodes (K11) and clear their slots.
__global__ void k_persist(WorkerDev w, int D, const float* mem_new) {
    pdl_entry();
    const int u = warp_id_global(), lane = lane_id();
    if (u >= *w.nU) return;
    const std::uint32_t node = w.pU[u];
    for (int c4 = lane; c4 < D / 4; c4 += 32)  // 128-bit rows (D % 4 == 0)
        reinterpret_cast<float4*>(w.mem + (std::size_t)node * D)[c4] =
            reinterpret_cast<const float4*>(mem_new + (std::size_t)u * D)[c4];
    if (lane == 0) {
        w.lu[node] = w.pTs[u];
        w.slot[node] = -1;
    }
}

// Bridge backbone: the reference's surrogate MSG/UPD
// (pac_sim.cpp:50-64 message, :68-104 model_update) in place of the GRU, applied
// to the pending last messages — every record reads the PRE-states of its node
// and of the other endpoint (as model_update reads both endpoints before
// writing either), m = tanh(W_m [s_u | s_other | cos(omega * (ts - lu_u))]),
// s_u <- (1 - gamma) s_u + gamma m. One thread per (record, output row); f64
// with explicitly rounded products and sums in the reference's column order
// (no FMA contraction); states are stored in the trainer's f32 memory.
__global__ void k_surrogate_update(WorkerDev w, int D, const double* w_m, const double* omega,
                                   double gamma, float* mem_new) {
    pdl_entry();
    const std::size_t t = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = *w.nU;
    if (t >= (std::size_t)n * D) return;
    const int i = static_cast<int>(t / D), r = static_cast<int>(t % D);
    const std::uint32_t u = w.pU[i], o = w.pOther[i];
    const double dt = __dadd_rn(w.pTs[i], -w.lu[u]);
    const float* su = w.mem + (std::size_t)u * D;
    const float* so = w.mem + (std::size_t)o * D;
    const double* wr = w_m + (std::size_t)r * 3 * D;
    double acc = 0.0;
    for (int c = 0; c < D; ++c) acc = __dadd_rn(acc, __dmul_rn(wr[c], double(su[c])));
    for (int c = 0; c < D; ++c) acc = __dadd_rn(acc, __dmul_rn(wr[D + c], double(so[c])));
    for (int c = 0; c < D; ++c) acc = __dadd_rn(acc, __dmul_rn(wr[2 * D + c], cos(__dmul_rn(omega[c], dt))));
    const double m = tanh(acc);
    mem_new[t] = float(__dadd_rn(__dmul_rn(1.0 - gamma, double(su[r])), __dmul_rn(gamma, m)));
}

// K3 last-message selection: endpoint slots q = 2k (src), 2k+1 (dst) of the
// batch's events; per node the max slot wins (max (ts, stream index)),
// compacted in slot order into the worker's other pending set (nx*).
// Single block; lastpos starts and ends at -1.
__global__ void k_pending(WorkerDev w, int B) {
    pdl_entry();
    const std::uint64_t lo = w.ctl[0];
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int nslots = 2 * B;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int q0 = 0; q0 < nslots; q0 += nt) {
        const int q = q0 + tid;
        std::uint32_t node = 0xFFFFFFFFu;
        if (q < nslots) {
            const std::uint64_t e = lo + (q >> 1);
            node = (q & 1) ? w.ev_dst[e] : w.ev_src[e];
        }
        // hubs repeat within a warp's 16 events: only the highest lane of each
        // equal-node group touches the contended counter
        const unsigned grp = __match_any_sync(0xffffffffu, node);
        if (q < nslots && (tid & 31) == 31 - __clz(grp)) atomicMax(w.lastpos + node, q);
    }
    if (tid == 0) base = 0;
    __syncthreads();
    for (int q0 = 0; q0 < nslots; q0 += nt) {
        const int q = q0 + tid;
        int win = 0;
        std::uint32_t node = 0, other = 0;
        std::uint64_t e = 0;
        if (q < nslots) {
            e = lo + (q >> 1);
            const std::uint32_t s = w.ev_src[e], t = w.ev_dst[e];
            node = (q & 1) ? t : s;
            other = (q & 1) ? s : t;
            win = w.lastpos[node] == q;
        }
        // block exclusive scan of win
        const int lane = tid & 31, wid = tid >> 5;
        const unsigned bal = __ballot_sync(0xffffffffu, win);
        const int pre = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        if (wid == 0) {
            int v = lane < (nt >> 5) ? warp_tot[lane] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane < (nt >> 5)) warp_tot[lane] = incl - v;  // exclusive
        }
        __syncthreads();
        const int pos = base + warp_tot[wid] + pre;
        if (win) {
            w.nxU[pos] = node;
            w.nxOther[pos] = other;
            w.nxEv[pos] = (std::uint32_t)e;
            w.nxTs[pos] = w.ev_ts[e];
        }
        __syncthreads();
        if (tid == nt - 1) base = pos + win;
        __syncthreads();
    }
    if (tid == 0) *w.nxN = base;
    for (int q = tid; q < nslots; q += nt) {
        const std::uint64_t e = lo + (q >> 1);
        const std::uint32_t node = (q & 1) ? w.ev_dst[e] : w.ev_src[e];
        w.lastpos[node] = -1;
    }
}

// Synthetic BF16-exact edge features for the partition's events (E x Fp, pad 0).
__global__ void k_gen_features(__nv_bfloat16* feat, const std::uint64_t* eids, std::uint64_t E,
                               int F, int Fp, std::uint64_t seed_mixed) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E * (std::size_t)Fp) return;
    const std::uint64_t e = i / Fp;
    const int c = i % Fp;
    const float v = c < F ? edge_feature_value(seed_mixed, eids[e], (std::uint32_t)c) : 0.f;
    feat[i] = __float2bfloat16_rn(v);
}

__global__ void k_gather_rows(const float* src, int ld, const std::uint32_t* idx, std::uint32_t n,
                              int cols, float* out) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)n * cols) return;
    const std::uint32_t r = i / cols, c = i % cols;
    out[i] = src[(std::size_t)idx[r] * ld + c];
}

}  // namespace tgnk
}  // namespace spd
