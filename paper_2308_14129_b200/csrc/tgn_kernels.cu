// Non-GEMM kernels of the TGN training step; see tgn_kernels.cuh. Semantics
// follow oracle/tgn_oracle.py line for line (which states the model choices).
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
__device__ __forceinline__ float4 r4(float4 v, int rnd) {
    return rnd ? make_float4(tf32r(v.x), tf32r(v.y), tf32r(v.z), tf32r(v.w)) : v;
}
}  // namespace

__global__ void k_init_aug(float* buf, int rows, int cols, int ld) {
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)rows * ld) return;
    const int c = i % ld;
    if (c >= cols) buf[i] = c == cols ? 1.f : 0.f;
    else buf[i] = 0.f;
}

// K5 + K8: roots (src | dst | neg) and the recent-k neighbours strictly
// before t: lower_bound on the node's time-sorted adjacency, last K entries.
__global__ void k_roots_nbrs(WorkerDev w, std::uint64_t lo, int B, std::uint64_t neg_base, int K,
                             std::uint32_t* roots, double* root_t, std::uint32_t* nbr_node,
                             std::uint32_t* nbr_ev, double* nbr_dt, int* cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= 3 * B) return;
    const int which = r / B, i = r % B;
    const std::uint64_t e = lo + i;
    const double t = w.ev_ts[e];
    std::uint32_t node;
    if (which == 0) node = w.ev_src[e];
    else if (which == 1) node = w.ev_dst[e];
    else node = w.pool[mix64(neg_base ^ (std::uint64_t)i) % w.n_pool];
    roots[r] = node;
    root_t[r] = t;
    const std::uint64_t a = w.adj_off[node], b = w.adj_off[node + 1];
    std::uint64_t l = a, h = b;
    while (l < h) {
        const std::uint64_t mid = (l + h) >> 1;
        if (w.adj_ts[mid] < t) l = mid + 1;
        else h = mid;
    }
    const std::uint64_t avail = l - a;
    const int c = avail < (std::uint64_t)K ? (int)avail : K;
    const std::uint64_t start = l - c;
    cnt[r] = c;
    for (int j = 0; j < K; ++j) {
        const std::size_t o = (std::size_t)r * K + j;
        if (j < c) {
            const std::uint64_t idx = start + j;
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
// and hidden s_i for every pending node (one warp per node).
__global__ void k_gru_gather(WorkerDev w, Dims d, const float* time_w, const float* time_b,
                             float* x, float* h, int set_slot) {
    const int u = warp_id_global(), lane = lane_id();
    if (u >= *w.nU) return;
    const std::uint32_t node = w.pU[u], other = w.pOther[u], ev = w.pEv[u];
    const double dt = w.pTs[u] - w.lu[node];
    if (set_slot && lane == 0) w.slot[node] = u;
    float* xr = x + (std::size_t)u * d.ld_x;
    float* hr = h + (std::size_t)u * d.ld_h;
    const float* mn = w.mem + (std::size_t)node * d.D;
    const float* mo = w.mem + (std::size_t)other * d.D;
    for (int c = lane; c < d.D; c += 32) {
        const float v = rnd_if(mn[c], d.rnd);
        xr[c] = v;
        hr[c] = v;
        xr[d.D + c] = rnd_if(mo[c], d.rnd);
    }
    const __nv_bfloat16* fr = w.feat + (std::size_t)ev * d.Fp;
    for (int c = lane; c < d.F; c += 32) xr[2 * d.D + c] = __bfloat162float(fr[c]);
    for (int c = lane; c < d.T; c += 32)
        xr[2 * d.D + d.F + c] = rnd_if(time_cos(time_w[c], time_b[c], dt), d.rnd);
}

// GRUCell (PyTorch gate order r, z, n) on G_i = W_ih x + b_ih, G_h = W_hh h + b_hh.
__global__ void k_gru_fwd(WorkerDev w, Dims d, const float* Gi, const float* Gh, const float* h,
                          float* save, float* mem_new) {
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

// K1 + K2 for attention: q_in = [s_root | phi(0)], kv_in = [s_nbr | e | phi(dt)]
// (one warp per row; padded neighbour rows are zero).
__global__ void k_embed_gather(WorkerDev w, Dims d, int R, const float* time_w,
                               const float* time_b, const std::uint32_t* roots,
                               const std::uint32_t* nbr_node, const std::uint32_t* nbr_ev,
                               const double* nbr_dt, const int* cnt, const float* mem_new,
                               float* q_in, float* kv_in) {
    const int row = warp_id_global(), lane = lane_id();
    if (row >= R * (1 + d.K)) return;
    if (row < R) {
        const float* m = memx_row(w, mem_new, d.D, roots[row]);
        float* q = q_in + (std::size_t)row * d.ld_q;
        for (int c = lane; c < d.D; c += 32) q[c] = rnd_if(m[c], d.rnd);
        for (int c = lane; c < d.T; c += 32) q[d.D + c] = rnd_if(time_cos(time_w[c], time_b[c], 0.0), d.rnd);
        return;
    }
    const int kr = row - R;  // r * K + j
    const int r = kr / d.K, j = kr % d.K;
    float* o = kv_in + (std::size_t)kr * d.ld_kv;
    if (j >= cnt[r]) {
        for (int c = lane; c < d.DK; c += 32) o[c] = 0.f;
        return;
    }
    const float* m = memx_row(w, mem_new, d.D, nbr_node[kr]);
    for (int c = lane; c < d.D; c += 32) o[c] = rnd_if(m[c], d.rnd);
    // column order [s_nbr | phi(dt) | e]: the gradient-carrying columns are a
    // contiguous prefix, so the data-gradient GEMM computes only D + T columns
    const double dt = nbr_dt[kr];
    for (int c = lane; c < d.T; c += 32) o[d.D + c] = rnd_if(time_cos(time_w[c], time_b[c], dt), d.rnd);
    const __nv_bfloat16* fr = w.feat + (std::size_t)nbr_ev[kr] * d.Fp;
    for (int c = lane; c < d.F; c += 32) o[d.D + d.T + c] = __bfloat162float(fr[c]);
}

// Multi-head attention core over <= K neighbours (one warp per root).
// KV rows: [K (DQ) | V (DQ)], row stride 2DQ. alpha: [R][H][K].
__global__ void k_attn_fwd(Dims d, int R, const int* cnt, const float* Q, const float* KV,
                           float* alpha, float* ctx) {
    extern __shared__ float sm[];
    const int warp_in_block = threadIdx.x >> 5, lane = lane_id();
    const int r = warp_id_global();
    if (r >= R) return;
    float* s = sm + warp_in_block * d.H * d.K;
    const int c_n = cnt[r];
    float* cr = ctx + (std::size_t)r * d.ld_ctx;
    if (c_n == 0) {
        for (int c = lane; c < d.DQ; c += 32) cr[c] = 0.f;
        return;
    }
    const int dh = d.DQ / d.H;
    const float* q = Q + (std::size_t)r * d.ld_Q;
    for (int h = 0; h < d.H; ++h) {
        for (int j = 0; j < c_n; ++j) {
            const float* k = KV + ((std::size_t)r * d.K + j) * d.ld_KV + h * dh;
            float p = 0.f;
            for (int c = lane; c < dh; c += 32) p += q[h * dh + c] * k[c];
            p = warp_sum(p);
            if (lane == 0) s[h * d.K + j] = p / sqrtf((float)dh);
        }
    }
    __syncwarp();
    // softmax per head over valid j (lane = j, K <= 32)
    for (int h = 0; h < d.H; ++h) {
        float v = lane < c_n ? s[h * d.K + lane] : -INFINITY;
        float mx = v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e = lane < c_n ? expf(v - mx) : 0.f;
        const float sum = warp_sum(e);
        const float a = e / sum;
        __syncwarp();
        if (lane < d.K) {
            const float av = lane < c_n ? a : 0.f;
            s[h * d.K + lane] = av;
            alpha[((std::size_t)r * d.H + h) * d.K + lane] = av;
        }
    }
    __syncwarp();
    for (int c = lane; c < d.DQ; c += 32) {
        const int h = c / dh;
        float acc = 0.f;
        for (int j = 0; j < c_n; ++j)
            acc += s[h * d.K + j] * KV[((std::size_t)r * d.K + j) * d.ld_KV + d.DQ + c];
        cr[c] = rnd_if(acc, d.rnd);
    }
}

// ---------------------------------------------------------------------------
// Register-tiled attention core (DQ <= 256, K <= KMAX, head dim % 4 == 0,
// H <= 4): one warp per root, lane l owns float4 chunks l and l+32 of every
// row. All K (then V) rows of the root are loaded up front — 2*K independent
// 128-bit loads in flight per lane — and each (key, head) dot product is an
// xor-shuffle all-reduce, so every lane holds all scores and computes the
// softmax redundantly without further communication.
template <int KMAX, int HMAX>
__global__ void __launch_bounds__(256) k_attn_fwd_reg(Dims d, int R, const int* cnt,
                                                      const float* Q, const float* KV,
                                                      float* alpha, float* ctx) {
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R) return;
    const int c_n = cnt[r];
    const int nc = d.DQ / 4;  // chunks per row
    const int dh4 = d.DQ / d.H / 4;
    float4* cr = reinterpret_cast<float4*>(ctx + (std::size_t)r * d.ld_ctx);
    const bool has0 = lane < nc, has1 = lane + 32 < nc;
    const int h0 = lane / dh4, h1 = (lane + 32) / dh4;
    if (c_n == 0) {
        if (has0) cr[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (has1) cr[lane + 32] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    const float4* q4 = reinterpret_cast<const float4*>(Q + (std::size_t)r * d.ld_Q);
    const float4 qa = has0 ? q4[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 qb = has1 ? q4[lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* base = reinterpret_cast<const float4*>(KV + (std::size_t)r * d.K * d.ld_KV);
    const int ld4 = d.ld_KV / 4;
    float4 ka[KMAX], kb[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j < c_n) {
            ka[j] = has0 ? base[j * ld4 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
            kb[j] = has1 ? base[j * ld4 + lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    float s[HMAX][KMAX];
    const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j >= c_n) break;
        float p[HMAX];
        const float da = qa.x * ka[j].x + qa.y * ka[j].y + qa.z * ka[j].z + qa.w * ka[j].w;
        const float db = qb.x * kb[j].x + qb.y * kb[j].y + qb.z * kb[j].z + qb.w * kb[j].w;
#pragma unroll
        for (int h = 0; h < HMAX; ++h) p[h] = (h0 == h ? da : 0.f) + (h1 == h ? db : 0.f);
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h >= d.H) break;
            s[h][j] = warp_sum(p[h]) * inv;
        }
    }
    // softmax per head (redundantly in every lane)
#pragma unroll
    for (int h = 0; h < HMAX; ++h) {
        if (h >= d.H) break;
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) mx = fmaxf(mx, s[h][j]);
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) {
                s[h][j] = expf(s[h][j] - mx);
                sum += s[h][j];
            }
        const float is = 1.f / sum;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) s[h][j] *= is;
    }
    if (lane < d.K) {
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h >= d.H) break;
            float v = 0.f;
#pragma unroll
            for (int j = 0; j < KMAX; ++j)
                if (j == lane && j < c_n) v = s[h][j];
            alpha[((std::size_t)r * d.H + h) * d.K + lane] = v;
        }
    }
    // context = sum_j alpha_hj V_j  (V chunks follow the K chunks in the row)
    const int voff = nc;  // V starts at column DQ = chunk nc
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j < c_n) {
            ka[j] = has0 ? base[j * ld4 + voff + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
            kb[j] = has1 ? base[j * ld4 + voff + lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    float4 oa = make_float4(0.f, 0.f, 0.f, 0.f), ob = oa;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j >= c_n) break;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h0 == h) a0 = s[h][j];
            if (h1 == h) a1 = s[h][j];
        }
        oa.x += a0 * ka[j].x; oa.y += a0 * ka[j].y; oa.z += a0 * ka[j].z; oa.w += a0 * ka[j].w;
        ob.x += a1 * kb[j].x; ob.y += a1 * kb[j].y; ob.z += a1 * kb[j].z; ob.w += a1 * kb[j].w;
    }
    if (d.rnd) {
        oa = make_float4(tf32r(oa.x), tf32r(oa.y), tf32r(oa.z), tf32r(oa.w));
        ob = make_float4(tf32r(ob.x), tf32r(ob.y), tf32r(ob.z), tf32r(ob.w));
    }
    if (has0) cr[lane] = oa;
    if (has1) cr[lane + 32] = ob;
}

template <int KMAX, int HMAX>
__global__ void __launch_bounds__(256) k_attn_bwd_reg(Dims d, int R, const int* cnt,
                                                      const float* Q, const float* KV,
                                                      const float* alpha, const float* dctx,
                                                      int ld_dctx, float* dQ, float* dKV) {
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R) return;
    const int c_n = cnt[r];
    const int nc = d.DQ / 4;
    const int dh4 = d.DQ / d.H / 4;
    const bool has0 = lane < nc, has1 = lane + 32 < nc;
    const int h0 = lane / dh4, h1 = (lane + 32) / dh4;
    const int ld4 = d.ld_KV / 4;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* base = reinterpret_cast<const float4*>(KV + (std::size_t)r * d.K * d.ld_KV);
    float4* obase = reinterpret_cast<float4*>(dKV + (std::size_t)r * d.K * d.ld_KV);
    float4* dq4 = reinterpret_cast<float4*>(dQ + (std::size_t)r * d.ld_Q);
    // padded key rows get zero gradients
    for (int j = c_n; j < d.K; ++j) {
        if (has0) { obase[j * ld4 + lane] = z4; obase[j * ld4 + nc + lane] = z4; }
        if (has1) { obase[j * ld4 + lane + 32] = z4; obase[j * ld4 + nc + lane + 32] = z4; }
    }
    if (c_n == 0) {
        if (has0) dq4[lane] = z4;
        if (has1) dq4[lane + 32] = z4;
        return;
    }
    const float4* dc4 = reinterpret_cast<const float4*>(dctx + (std::size_t)r * ld_dctx);
    const float4 ga = has0 ? dc4[lane] : z4, gb = has1 ? dc4[lane + 32] : z4;
    float4 va[KMAX], vb[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
        if (j < c_n) {
            va[j] = has0 ? base[j * ld4 + nc + lane] : z4;
            vb[j] = has1 ? base[j * ld4 + nc + lane + 32] : z4;
        }
    float a[HMAX][KMAX], ds[HMAX][KMAX];
    const float* al = alpha + (std::size_t)r * d.H * d.K;
#pragma unroll
    for (int h = 0; h < HMAX; ++h) {
        if (h >= d.H) break;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) a[h][j] = al[h * d.K + j];
    }
    // d alpha_hj = <dctx_h, V_jh>; dV_j = alpha_hj dctx
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j >= c_n) break;
        const float pa = ga.x * va[j].x + ga.y * va[j].y + ga.z * va[j].z + ga.w * va[j].w;
        const float pb = gb.x * vb[j].x + gb.y * vb[j].y + gb.z * vb[j].z + gb.w * vb[j].w;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h >= d.H) break;
            ds[h][j] = warp_sum((h0 == h ? pa : 0.f) + (h1 == h ? pb : 0.f));
            if (h0 == h) a0 = a[h][j];
            if (h1 == h) a1 = a[h][j];
        }
        if (has0) obase[j * ld4 + nc + lane] = r4(make_float4(a0 * ga.x, a0 * ga.y, a0 * ga.z, a0 * ga.w), d.rnd);
        if (has1)
            obase[j * ld4 + nc + lane + 32] = r4(make_float4(a1 * gb.x, a1 * gb.y, a1 * gb.z, a1 * gb.w), d.rnd);
    }
    // d score_hj = alpha_hj (dalpha_hj - sum_k alpha_hk dalpha_hk)
#pragma unroll
    for (int h = 0; h < HMAX; ++h) {
        if (h >= d.H) break;
        float dot = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) dot += a[h][j] * ds[h][j];
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < c_n) ds[h][j] = a[h][j] * (ds[h][j] - dot);
    }
    const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
    const float4* q4 = reinterpret_cast<const float4*>(Q + (std::size_t)r * d.ld_Q);
    const float4 qa = has0 ? q4[lane] : z4, qb = has1 ? q4[lane + 32] : z4;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
        if (j < c_n) {
            va[j] = has0 ? base[j * ld4 + lane] : z4;  // reuse registers for K rows
            vb[j] = has1 ? base[j * ld4 + lane + 32] : z4;
        }
    float4 oa = z4, ob = z4;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j >= c_n) break;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h0 == h) s0 = ds[h][j] * inv;
            if (h1 == h) s1 = ds[h][j] * inv;
        }
        oa.x += s0 * va[j].x; oa.y += s0 * va[j].y; oa.z += s0 * va[j].z; oa.w += s0 * va[j].w;
        ob.x += s1 * vb[j].x; ob.y += s1 * vb[j].y; ob.z += s1 * vb[j].z; ob.w += s1 * vb[j].w;
        if (has0) obase[j * ld4 + lane] = r4(make_float4(s0 * qa.x, s0 * qa.y, s0 * qa.z, s0 * qa.w), d.rnd);
        if (has1) obase[j * ld4 + lane + 32] = r4(make_float4(s1 * qb.x, s1 * qb.y, s1 * qb.z, s1 * qb.w), d.rnd);
    }
    if (has0) dq4[lane] = r4(oa, d.rnd);
    if (has1) dq4[lane + 32] = r4(ob, d.rnd);
}

#define SPD_ATTN_INST(KM, HM)                                                                  \
    template __global__ void k_attn_fwd_reg<KM, HM>(Dims, int, const int*, const float*,         \
                                                    const float*, float*, float*);              \
    template __global__ void k_attn_bwd_reg<KM, HM>(Dims, int, const int*, const float*,         \
                                                    const float*, const float*, const float*, int, \
                                                    float*, float*);
SPD_ATTN_INST(10, 2)
SPD_ATTN_INST(16, 4)
#undef SPD_ATTN_INST

// MergeLayer input [attn | s_root]; attn = 0 for a root without neighbours.
__global__ void k_merge_gather(WorkerDev w, Dims d, int R, const std::uint32_t* roots,
                               const int* cnt, const float* O, const float* mem_new, float* m_in) {
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R) return;
    float* o = m_in + (std::size_t)r * d.ld_m;
    const bool has = cnt[r] > 0;
    for (int c = lane; c < d.DQ; c += 32) o[c] = has ? rnd_if(O[(std::size_t)r * d.DQ + c], d.rnd) : 0.f;
    const float* m = memx_row(w, mem_new, d.D, roots[r]);
    for (int c = lane; c < d.D; c += 32) o[d.DQ + c] = rnd_if(m[c], d.rnd);
}

// Decoder input rows: p < B -> [z_src | z_dst], p >= B -> [z_src | z_neg].
__global__ void k_dec_gather(Dims d, int B, const float* emb, float* d_in) {
    const int p = warp_id_global(), lane = lane_id();
    if (p >= 2 * B) return;
    const int i = p < B ? p : p - B;
    const int other = p < B ? B + i : 2 * B + i;
    float* o = d_in + (std::size_t)p * d.ld_din;
    for (int c = lane; c < d.D; c += 32) {
        o[c] = emb[(std::size_t)i * d.D + c];
        o[d.D + c] = emb[(std::size_t)other * d.D + c];
    }
}

// K7 head: logit = D1 . w2 + b2, BCE-with-logits terms and their gradients.
// w2 = augmented [w | b] row of dec2.
__global__ void k_dec_head(Dims d, int B, const float* D1, const float* w2, float* dlogit,
                           float* lossv, float* dD1, float* logits) {
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

// Fixed-order single-block sum (deterministic loss).
__global__ void k_sum_loss(const float* lossv, int n, float* out) {
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
    const int r = warp_id_global(), lane = lane_id();
    if (r >= R || cnt[r] > 0) return;
    for (int c = lane; c < cols; c += 32) buf[(std::size_t)r * ld + c] = 0.f;
}

// Attention core backward (one warp per root).
__global__ void k_attn_bwd(Dims d, int R, const int* cnt, const float* Q, const float* KV,
                           const float* alpha, const float* dctx, int ld_dctx, float* dQ,
                           float* dKV) {
    extern __shared__ float sm[];
    const int warp_in_block = threadIdx.x >> 5, lane = lane_id();
    const int r = warp_id_global();
    if (r >= R) return;
    float* ds = sm + warp_in_block * d.H * d.K;
    const int c_n = cnt[r];
    const int dh = d.DQ / d.H;
    const float inv = 1.f / sqrtf((float)dh);
    const float* dc = dctx + (std::size_t)r * ld_dctx;
    const float* a = alpha + (std::size_t)r * d.H * d.K;
    if (c_n > 0) {
        for (int h = 0; h < d.H; ++h) {
            for (int j = 0; j < c_n; ++j) {
                const float* v = KV + ((std::size_t)r * d.K + j) * d.ld_KV + d.DQ + h * dh;
                float p = 0.f;
                for (int c = lane; c < dh; c += 32) p += dc[h * dh + c] * v[c];
                p = warp_sum(p);
                if (lane == 0) ds[h * d.K + j] = p;  // d alpha_j
            }
            __syncwarp();
            float da = lane < c_n ? ds[h * d.K + lane] : 0.f;
            const float aj = lane < c_n ? a[h * d.K + lane] : 0.f;
            const float dot = warp_sum(aj * da);
            __syncwarp();
            if (lane < c_n) ds[h * d.K + lane] = aj * (da - dot);  // d score_j
            __syncwarp();
        }
    }
    float* dq = dQ + (std::size_t)r * d.ld_Q;
    for (int c = lane; c < d.DQ; c += 32) {
        const int h = c / dh;
        float acc = 0.f;
        for (int j = 0; j < c_n; ++j)
            acc += ds[h * d.K + j] * KV[((std::size_t)r * d.K + j) * d.ld_KV + c];
        dq[c] = rnd_if(acc * inv, d.rnd);
    }
    const float* q = Q + (std::size_t)r * d.ld_Q;
    for (int j = 0; j < d.K; ++j) {
        float* o = dKV + ((std::size_t)r * d.K + j) * d.ld_KV;
        if (j >= c_n) {
            for (int c = lane; c < 2 * d.DQ; c += 32) o[c] = 0.f;
            continue;
        }
        for (int c = lane; c < d.DQ; c += 32) {
            const int h = c / dh;
            o[c] = rnd_if(ds[h * d.K + j] * q[c] * inv, d.rnd);
            o[d.DQ + c] = rnd_if(a[h * d.K + j] * dc[c], d.rnd);
        }
    }
}

// Memory-row gradients into the GRU output rows of pending nodes: roots
// (query + merge inputs) and neighbours (key/value inputs).
__global__ void k_mem_grad(WorkerDev w, Dims d, int R, const std::uint32_t* roots,
                           const std::uint32_t* nbr_node, const int* cnt, const float* dq_in,
                           const float* dm_in, const float* dkv_in, float* dH) {
    const int row = warp_id_global(), lane = lane_id();
    if (row >= R * (1 + d.K)) return;
    if (row < R) {
        const int s = w.slot[roots[row]];
        if (s < 0) return;
        const float* a = dq_in + (std::size_t)row * d.ld_q;
        const float* b = dm_in + (std::size_t)row * d.ld_m + d.DQ;
        for (int c = lane; c < d.D; c += 32) atomicAdd(dH + (std::size_t)s * d.D + c, a[c] + b[c]);
        return;
    }
    const int kr = row - R;
    const int r = kr / d.K, j = kr % d.K;
    if (j >= cnt[r]) return;
    const int s = w.slot[nbr_node[kr]];
    if (s < 0) return;
    const float* a = dkv_in + (std::size_t)kr * d.ld_kv;
    for (int c = lane; c < d.D; c += 32) atomicAdd(dH + (std::size_t)s * d.D + c, a[c]);
}

// Time-encoder gradients: per block, f64 column partials over a chunk of rows
// (kv rows: d/dw = -sin(ph) dt g, d/db = -sin(ph) g; query rows: phi(0)=cos(b)).
// part: [nblocks][2T] (w then b).
// blockDim = (32 columns, 8 row lanes); block covers 32 columns x rows_per_block
// rows; f64 accumulation, fixed-order in-block reduction -> part[block][2T].
__global__ void k_time_grad_partial(Dims d, int R, const int* cnt, const double* nbr_dt,
                                    const float* dkv_in, const float* dq_in, const float* time_w,
                                    const float* time_b, int rows_per_block, double* part) {
    __shared__ double red[2][8][33];
    const int total = R * (1 + d.K);
    const int c = blockIdx.y * 32 + threadIdx.x;
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(total, r0 + rows_per_block);
    double gw = 0.0, gb = 0.0;
    if (c < d.T) {
        const float wc = time_w[c], bc = time_b[c];
        const double sin_b = sin((double)bc);
        for (int row = r0 + threadIdx.y; row < r1; row += blockDim.y) {
            if (row < R) {
                gb -= sin_b * (double)dq_in[(std::size_t)row * d.ld_q + d.D + c];
            } else {
                const int kr = row - R;
                const int r = kr / d.K, j = kr % d.K;
                if (j >= cnt[r]) continue;
                const double dt = nbr_dt[kr];
                const double g = dkv_in[(std::size_t)kr * d.ld_kv + d.D + c];
                const double sn = (double)time_sin(wc, bc, dt);
                gw -= sn * dt * g;
                gb -= sn * g;
            }
        }
    }
    red[0][threadIdx.y][threadIdx.x] = gw;
    red[1][threadIdx.y][threadIdx.x] = gb;
    __syncthreads();
    if (threadIdx.y == 0 && c < d.T) {
        double sw = 0.0, sb = 0.0;
        for (int y = 0; y < (int)blockDim.y; ++y) {
            sw += red[0][y][threadIdx.x];
            sb += red[1][y][threadIdx.x];
        }
        part[(std::size_t)blockIdx.x * 2 * d.T + c] = sw;
        part[(std::size_t)blockIdx.x * 2 * d.T + d.T + c] = sb;
    }
}

// Fused single pass over the gradient-carrying input columns of every query
// and key/value row: memory-row gradients (atomics into the GRU outputs of
// pending nodes) and time-encoder gradients (f64, per-block fixed-order
// partials). block (32, 8); rows_per_block rows; part[block][2T].
__global__ void k_memtime_grad(WorkerDev w, Dims d, int R, const std::uint32_t* roots,
                               const std::uint32_t* nbr_node, const int* cnt, const double* nbr_dt,
                               const float* dq_in, const float* dm_in, const float* dkv_in,
                               const float* time_w, const float* time_b, int rows_per_block,
                               float* dH, double* part) {
    constexpr int TC = 4;  // time columns per thread: T <= 128
    __shared__ double red[2][8][32 * TC];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int total = R * (1 + d.K);
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(total, r0 + rows_per_block);
    double gw[TC], gb[TC], sinb[TC];
    float wc[TC], bc[TC];
#pragma unroll
    for (int i = 0; i < TC; ++i) {
        gw[i] = gb[i] = 0.0;
        const int c = tx + 32 * i;
        wc[i] = c < d.T ? time_w[c] : 0.f;
        bc[i] = c < d.T ? time_b[c] : 0.f;
        sinb[i] = sin((double)bc[i]);
    }
    for (int row = r0 + ty; row < r1; row += blockDim.y) {
        if (row < R) {
            const float* q = dq_in + (std::size_t)row * d.ld_q;
            const int s = w.slot[roots[row]];
            if (s >= 0) {
                const float* m = dm_in + (std::size_t)row * d.ld_m + d.DQ;
                for (int c = tx; c < d.D; c += 32) atomicAdd(dH + (std::size_t)s * d.D + c, q[c] + m[c]);
            }
#pragma unroll
            for (int i = 0; i < TC; ++i) {
                const int c = tx + 32 * i;
                if (c < d.T) gb[i] -= sinb[i] * (double)q[d.D + c];
            }
        } else {
            const int kr = row - R;
            const int r = kr / d.K, j = kr % d.K;
            if (j >= cnt[r]) continue;
            const float* g = dkv_in + (std::size_t)kr * d.ld_kv;
            const int s = w.slot[nbr_node[kr]];
            if (s >= 0)
                for (int c = tx; c < d.D; c += 32) atomicAdd(dH + (std::size_t)s * d.D + c, g[c]);
            const double dt = nbr_dt[kr];
#pragma unroll
            for (int i = 0; i < TC; ++i) {
                const int c = tx + 32 * i;
                if (c < d.T) {
                    const double sn = (double)time_sin(wc[i], bc[i], dt);
                    const double gv = g[d.D + c];
                    gw[i] -= sn * dt * gv;
                    gb[i] -= sn * gv;
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < TC; ++i) {
        red[0][ty][tx + 32 * i] = gw[i];
        red[1][ty][tx + 32 * i] = gb[i];
    }
    __syncthreads();
    if (ty == 0) {
#pragma unroll
        for (int i = 0; i < TC; ++i) {
            const int c = tx + 32 * i;
            if (c >= d.T) continue;
            double sw = 0.0, sb = 0.0;
            for (int y = 0; y < (int)blockDim.y; ++y) {
                sw += red[0][y][c];
                sb += red[1][y][c];
            }
            part[(std::size_t)blockIdx.x * 2 * d.T + c] = sw;
            part[(std::size_t)blockIdx.x * 2 * d.T + d.T + c] = sb;
        }
    }
}

// one block per output (2T): fixed-order strided sums + tree -> deterministic.
__global__ void k_time_grad_final(int T, int nblocks, const double* part, double* acc) {
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
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= T) return;
    gw[c] += (float)acc[c];
    gb[c] += (float)acc[T + c];
}

// GRUCell backward to the gate pre-activations (inputs x, h are constants).
__global__ void k_gru_bwd(WorkerDev w, Dims d, const float* dH, const float* save, const float* h,
                          float* dGi, float* dGh) {
    const int nU = *w.nU;
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)nU * d.D) return;
    const int u = i / d.D, c = i % d.D;
    const float* s = save + (std::size_t)u * 4 * d.D;
    const float r = s[c], z = s[d.D + c], n = s[2 * d.D + c], ghn = s[3 * d.D + c];
    const float g = dH[(std::size_t)u * d.D + c];
    const float hv = w.mem[(std::size_t)w.pU[u] * d.D + c];  // exact h
    const float dn = g * (1.f - z);
    const float dz = g * (hv - n);
    const float dpn = dn * (1.f - n * n);
    const float dpr = dpn * ghn * r * (1.f - r);
    const float dpz = dz * z * (1.f - z);
    float* gi = dGi + (std::size_t)u * d.ld_g;
    float* gh = dGh + (std::size_t)u * d.ld_g;
    gi[c] = rnd_if(dpr, d.rnd);
    gi[d.D + c] = rnd_if(dpz, d.rnd);
    gi[2 * d.D + c] = rnd_if(dpn, d.rnd);
    gh[c] = rnd_if(dpr, d.rnd);
    gh[d.D + c] = rnd_if(dpz, d.rnd);
    gh[2 * d.D + c] = rnd_if(dpn * r, d.rnd);
}

__global__ void k_adam(float* p, const float* g, float* m, float* v, std::size_t n, float scale,
                       float lr, float b1, float one_m_b1, float b2, float one_m_b2, float bc1,
                       float bc2, float eps, float* p_tc) {
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float gi = g[i] / scale;
    const float mi = b1 * m[i] + one_m_b1 * gi;
    const float vi = b2 * v[i] + one_m_b2 * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / bc1;
    const float vh = vi / bc2;
    const float pn = p[i] - lr * mh / (sqrtf(vh) + eps);
    p[i] = pn;
    if (p_tc) p_tc[i] = tf32r(pn);
}

__global__ void k_round_tf32(const float* src, float* dst, std::size_t n) {
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = tf32r(src[i]);
}

// Persist the GRU rows of pending nodes (K11) and clear their slots.
__global__ void k_persist(WorkerDev w, int D, const float* mem_new) {
    const int u = warp_id_global(), lane = lane_id();
    if (u >= *w.nU) return;
    const std::uint32_t node = w.pU[u];
    for (int c = lane; c < D; c += 32) w.mem[(std::size_t)node * D + c] = mem_new[(std::size_t)u * D + c];
    if (lane == 0) {
        w.lu[node] = w.pTs[u];
        w.slot[node] = -1;
    }
}

// K3 last-message selection: endpoint slots q = 2k (src), 2k+1 (dst) of the
// batch's events; per node the max slot wins (max (ts, stream index)),
// compacted in slot order. Single block; lastpos starts and ends at -1.
__global__ void k_pending(WorkerDev w, std::uint64_t lo, int B) {
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int nslots = 2 * B;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int q = tid; q < nslots; q += nt) {
        const std::uint64_t e = lo + (q >> 1);
        const std::uint32_t node = (q & 1) ? w.ev_dst[e] : w.ev_src[e];
        atomicMax(w.lastpos + node, q);
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
            w.pU[pos] = node;
            w.pOther[pos] = other;
            w.pEv[pos] = (std::uint32_t)e;
            w.pTs[pos] = w.ev_ts[e];
        }
        __syncthreads();
        if (tid == nt - 1) base = pos + win;
        __syncthreads();
    }
    if (tid == 0) *w.nU = base;
    for (int q = tid; q < nslots; q += nt) {
        const std::uint64_t e = lo + (q >> 1);
        const std::uint32_t node = (q & 1) ? w.ev_dst[e] : w.ev_src[e];
        w.lastpos[node] = -1;
    }
}

// Synthetic BF16-exact edge features for the partition's events (E x Fp, pad 0).
__global__ void k_gen_features(__nv_bfloat16* feat, const std::uint64_t* eids, std::uint64_t E,
                               int F, int Fp, std::uint64_t seed_mixed) {
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E * (std::size_t)Fp) return;
    const std::uint64_t e = i / Fp;
    const int c = i % Fp;
    const float v = c < F ? edge_feature_value(seed_mixed, eids[e], (std::uint32_t)c) : 0.f;
    feat[i] = __float2bfloat16_rn(v);
}

__global__ void k_gather_rows(const float* src, int ld, const std::uint32_t* idx, std::uint32_t n,
                              int cols, float* out) {
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)n * cols) return;
    const std::uint32_t r = i / cols, c = i % cols;
    out[i] = src[(std::size_t)idx[r] * ld + c];
}

}  // namespace tgnk
}  // namespace spd
