// Temporal graph attention with the key/value projections absorbed into the
// query side ("algorithmic FLOP reduction"). For one root with
// neighbour inputs x~_j = [s_nbr | phi(dt) | e | 1] (the augmented key/value
// input row of oracle/tgn_oracle.py TGNOracle._embed) and per-head weights
// [W_K,h | b_K,h], [W_V,h | b_V,h]:
//
//   score_hj = <q_h, W_K,h x~_j>        = <q'_h, x~_j>,  q'_h = [W_K,h|b_K,h]^T q_h
//   ctx_h    = sum_j a_hj W_V,h x~_j    = [W_V,h|b_V,h] xbar_h,  xbar_h = sum_j a_hj x~_j
//
// q'_h and ctx_h are GEMMs over R roots (R x dh x (DK+1) each) instead of the
// R*k x (DK+1) x 2DQ key/value projection; the k neighbour rows are gathered
// here and never written to HBM. Same algebra as the oracle; only the FP32
// summation order differs.
//
// Execution: 4 warps per block, one root per warp. Each warp first stages its
// root's k neighbour rows in shared memory with cp.async — memory row (f32,
// from the GRU output when the neighbour was just updated), raw bf16 feature
// row — and evaluates phi(dt) (f64 phase) into the same row, so every gather
// of the root is in flight at once; both passes then read shared memory.
// Lane l owns the float4 column chunks l, l+32, .. of the ld_p-wide augmented
// row (D, T multiples of 4: a chunk lies wholly in the memory, time or
// feature|1|pad region).
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"

namespace spd {
namespace tgnk {

namespace {

constexpr int kRootsPerBlock = 4;

__device__ __forceinline__ float dot4(const float4& a, const float4& b) {
    return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}
__device__ __forceinline__ void axpy4(float4& acc, float s, const float4& x) {
    acc.x += s * x.x; acc.y += s * x.y; acc.z += s * x.z; acc.w += s * x.w;
}
__device__ __forceinline__ float4 z4() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float4 rnd4(float4 v, int rnd) {
    return rnd ? make_float4(tf32r(v.x), tf32r(v.y), tf32r(v.z), tf32r(v.w)) : v;
}

__device__ __forceinline__ void cp_async16_ca(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// bytes of one staged neighbour row: [mem f32 D | phi f32 T | feat bf16 Fp]
__host__ __device__ __forceinline__ int row_bytes(const Dims& d) {
    return 4 * (d.D + d.T) + 2 * d.Fp;
}

// Stage root r's neighbour rows (warp-cooperative). Lane j < c_n holds
// neighbour j's (node, dt, slot) on return, for the caller's scatters.
__device__ __forceinline__ void stage_rows(const WorkerDev& w, const Dims& d, int r, int c_n,
                                           int lane, const float* time_w, const float* time_b,
                                           const std::uint32_t* nbr_node,
                                           const std::uint32_t* nbr_ev, const double* nbr_dt,
                                           const float* mem_new, unsigned char* xs,
                                           std::uint32_t& m_node, double& m_dt, int& m_slot) {
    std::uint32_t ev = 0;
    m_node = 0; m_dt = 0.0; m_slot = -1;
    if (lane < c_n) {
        const std::size_t o = (std::size_t)r * d.K + lane;
        m_node = nbr_node[o];
        ev = nbr_ev[o];
        m_dt = nbr_dt[o];
        m_slot = w.slot[m_node];
    }
    const int RB = row_bytes(d);
    const int mch = d.D / 4, fch = d.Fp / 8;  // 16-B chunks of the memory / feature rows
    for (int j = 0; j < c_n; ++j) {
        const std::uint32_t node = __shfl_sync(0xffffffffu, m_node, j);
        const std::uint32_t e = __shfl_sync(0xffffffffu, ev, j);
        const int slot = __shfl_sync(0xffffffffu, m_slot, j);
        const float* mrow = slot >= 0 ? mem_new + (std::size_t)slot * d.D : w.mem + (std::size_t)node * d.D;
        const __nv_bfloat16* frow = w.feat + (std::size_t)e * d.Fp;
        unsigned char* dst = xs + (std::size_t)j * RB;
        for (int c = lane; c < mch + fch; c += 32) {
            if (c < mch) cp_async16_ca(dst + 16 * c, mrow + 4 * c);
            else cp_async16_cg(dst + 4 * (d.D + d.T) + 16 * (c - mch), frow + 8 * (c - mch));
        }
    }
    // phi(dt) = cos(w dt + b), phase in f64
    for (int j = 0; j < c_n; ++j) {
        const double dt = __shfl_sync(0xffffffffu, m_dt, j);
        float* ph = reinterpret_cast<float*>(xs + (std::size_t)j * RB) + d.D;
        for (int t = lane; t < d.T; t += 32) ph[t] = time_cos(time_w[t], time_b[t], dt);
    }
    cp_async_wait_all();
    __syncwarp();
}

// Chunk ch (columns 4ch..4ch+3) of the staged augmented row.
__device__ __forceinline__ float4 x_chunk(const Dims& d, int ch, const unsigned char* row) {
    const int c = 4 * ch;
    if (c < d.D + d.T) return *reinterpret_cast<const float4*>(row + 4 * c);
    const int f = c - d.D - d.T;
    float4 v = z4();
    if (f < d.Fp) {  // Fp % 8 == 0: 4 bf16 never straddle the row end; pad columns are 0
        const uint2 raw = *reinterpret_cast<const uint2*>(row + 4 * (d.D + d.T) + 2 * f);
        const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
        const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
        v = make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
    }
    // augmented constant-1 column (bias) at feature index F
    const int b = d.F - f;
    if (b == 0) v.x = 1.f;
    else if (b == 1) v.y = 1.f;
    else if (b == 2) v.z = 1.f;
    else if (b == 3) v.w = 1.f;
    return v;
}

template <int NCH, int HMAX>
__device__ __forceinline__ void load_rows(float4 (&v)[HMAX][NCH], const float* base, const Dims& d,
                                          int lane, int nch) {
#pragma unroll
    for (int h = 0; h < HMAX; ++h)
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            const int ch = lane + 32 * i;
            v[h][i] = (h < d.H && ch < nch)
                          ? reinterpret_cast<const float4*>(base + (std::size_t)h * d.ld_p)[ch]
                          : z4();
        }
}

}  // namespace

__host__ __device__ std::size_t attn_smem_bytes(const Dims& d) {
    const std::size_t stage = std::size_t(kRootsPerBlock) * d.K * row_bytes(d);
    const std::size_t tpart = std::size_t(kRootsPerBlock) * 2 * d.T * sizeof(float);
    return (stage > tpart ? stage : tpart) + kRootsPerBlock * 2 * sizeof(float) * d.H * d.K;
}
int attn_roots_per_block() { return kRootsPerBlock; }

// Forward: scores from q'_h (Qp), softmax, alpha [R][H][K], xbar_h [R][H][ld_p]
// (tf32-rounded when it feeds a tensor-core GEMM). Roots without neighbours
// get xbar = 0 (bias slot 0 too: ctx = 0; the oracle masks them).
template <int NCH, int HMAX>
__global__ void __launch_bounds__(128) k_attn_abs_fwd(WorkerDev w, Dims d, int R,
                                                      const float* time_w, const float* time_b,
                                                      const std::uint32_t* nbr_node,
                                                      const std::uint32_t* nbr_ev,
                                                      const double* nbr_dt, const int* cnt,
                                                      const float* mem_new, const float* Qp,
                                                      float* alpha, float* xbar) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * kRootsPerBlock + warp;
    if (r >= R) return;
    const int RB = row_bytes(d);
    unsigned char* xs = smem + (std::size_t)warp * d.K * RB;
    float* sc = reinterpret_cast<float*>(smem + attn_smem_bytes(d)) - kRootsPerBlock * 2 * d.H * d.K +
                warp * 2 * d.H * d.K;
    const int c_n = cnt[r];
    const int nch = d.ld_p / 4;
    const std::size_t row0 = (std::size_t)r * d.H * d.ld_p;
    if (c_n == 0) {
        for (int h = 0; h < d.H; ++h)
            for (int ch = lane; ch < nch; ch += 32)
                reinterpret_cast<float4*>(xbar + row0 + (std::size_t)h * d.ld_p)[ch] = z4();
        if (lane < d.K)
            for (int h = 0; h < d.H; ++h) alpha[((std::size_t)r * d.H + h) * d.K + lane] = 0.f;
        return;
    }
    std::uint32_t m_node;
    double m_dt;
    int m_slot;
    stage_rows(w, d, r, c_n, lane, time_w, time_b, nbr_node, nbr_ev, nbr_dt, mem_new, xs, m_node,
               m_dt, m_slot);
    float4 v[HMAX][NCH];  // q'_h, then the xbar accumulators
    load_rows<NCH, HMAX>(v, Qp + row0, d, lane, nch);
    const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
#pragma unroll 1
    for (int j = 0; j < c_n; ++j) {
        const unsigned char* row = xs + (std::size_t)j * RB;
        float p[HMAX];
#pragma unroll
        for (int h = 0; h < HMAX; ++h) p[h] = 0.f;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            const int ch = lane + 32 * i;
            if (ch < nch) {
                const float4 x = x_chunk(d, ch, row);
#pragma unroll
                for (int h = 0; h < HMAX; ++h) p[h] += dot4(v[h][i], x);
            }
        }
#pragma unroll
        for (int h = 0; h < HMAX; ++h)
            if (h < d.H) {
                const float s = warp_sum(p[h]);
                if (lane == 0) sc[h * d.K + j] = s * inv;
            }
    }
    __syncwarp();
    // softmax per head over the c_n valid neighbours (lane = neighbour)
    for (int h = 0; h < d.H; ++h) {
        const float s = lane < c_n ? sc[h * d.K + lane] : -INFINITY;
        float mx = s;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e = lane < c_n ? expf(s - mx) : 0.f;
        const float a = e / warp_sum(e);
        __syncwarp();
        if (lane < d.K) {
            sc[h * d.K + lane] = a;
            alpha[((std::size_t)r * d.H + h) * d.K + lane] = a;
        }
    }
    __syncwarp();
    // xbar_h = sum_j a_hj x~_j
#pragma unroll
    for (int h = 0; h < HMAX; ++h)
#pragma unroll
        for (int i = 0; i < NCH; ++i) v[h][i] = z4();
#pragma unroll 1
    for (int j = 0; j < c_n; ++j) {
        const unsigned char* row = xs + (std::size_t)j * RB;
        float a[HMAX];
#pragma unroll
        for (int h = 0; h < HMAX; ++h) a[h] = h < d.H ? sc[h * d.K + j] : 0.f;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            const int ch = lane + 32 * i;
            if (ch < nch) {
                const float4 x = x_chunk(d, ch, row);
#pragma unroll
                for (int h = 0; h < HMAX; ++h) axpy4(v[h][i], a[h], x);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < HMAX; ++h) {
        if (h >= d.H) break;
        float4* o = reinterpret_cast<float4*>(xbar + row0 + (std::size_t)h * d.ld_p);
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            const int ch = lane + 32 * i;
            if (ch < nch) o[ch] = rnd4(v[h][i], d.rnd);
        }
    }
}

// Backward, given dxbar_h = [W_V,h|b_V,h]^T dctx_h (GEMM) per root:
//   da_hj = <dxbar_h, x~_j>;  ds_hj = a_hj (da_hj - sum_k a_hk da_hk) / sqrt(dh)
//   dq'_h = sum_j ds_hj x~_j                         -> dQp (GEMMs give dQ, dW_K)
//   dx_j  = sum_h a_hj dxbar_h + ds_hj q'_h  on the gradient-carrying columns:
//           memory part -> dH rows of pending nodes (float4 atomics), time part
//           -> d/dw, d/db of cos(w dt + b) (per-block partials, fixed order).
// part: [gridDim.x][2T] (w then b), f64; every block writes its row.
template <int NCH, int NCX, int HMAX>
__global__ void __launch_bounds__(128) k_attn_abs_bwd(WorkerDev w, Dims d, int R,
                                                      const float* time_w, const float* time_b,
                                                      const std::uint32_t* nbr_node,
                                                      const std::uint32_t* nbr_ev,
                                                      const double* nbr_dt, const int* cnt,
                                                      const float* mem_new, const float* Qp,
                                                      const float* alpha, const float* dxbar,
                                                      float* dQp, float* dH, double* part) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * kRootsPerBlock + warp;
    const int RB = row_bytes(d);
    unsigned char* xs = smem + (std::size_t)warp * d.K * RB;
    float* sc = reinterpret_cast<float*>(smem + attn_smem_bytes(d)) - kRootsPerBlock * 2 * d.H * d.K +
                warp * 2 * d.H * d.K;
    float* aa = sc + d.H * d.K;  // alpha of this root
    // time-encoder partials of this warp's root reuse the staging area at the end
    const int nch = d.ld_p / 4;
    const int nchx = (d.D + d.T) / 4;
    const int c_n = r < R ? cnt[r] : 0;
    const std::size_t row0 = (std::size_t)r * d.H * d.ld_p;
    float4 gw[NCX], gb[NCX];
#pragma unroll
    for (int i = 0; i < NCX; ++i) gw[i] = gb[i] = z4();
    if (r < R && c_n == 0) {
        for (int h = 0; h < d.H; ++h)
            for (int ch = lane; ch < nch; ch += 32)
                reinterpret_cast<float4*>(dQp + row0 + (std::size_t)h * d.ld_p)[ch] = z4();
    }
    if (c_n > 0) {
        std::uint32_t m_node;
        double m_dt;
        int m_slot;
        stage_rows(w, d, r, c_n, lane, time_w, time_b, nbr_node, nbr_ev, nbr_dt, mem_new, xs,
                   m_node, m_dt, m_slot);
        if (lane < d.K)
            for (int h = 0; h < d.H; ++h)
                aa[h * d.K + lane] = lane < c_n ? alpha[((std::size_t)r * d.H + h) * d.K + lane] : 0.f;
        float4 v[HMAX][NCH];  // dxbar_h, then the dq'_h accumulators
        load_rows<NCH, HMAX>(v, dxbar + row0, d, lane, nch);
        // pass 1: da_hj
#pragma unroll 1
        for (int j = 0; j < c_n; ++j) {
            const unsigned char* row = xs + (std::size_t)j * RB;
            float p[HMAX];
#pragma unroll
            for (int h = 0; h < HMAX; ++h) p[h] = 0.f;
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const int ch = lane + 32 * i;
                if (ch < nch) {
                    const float4 x = x_chunk(d, ch, row);
#pragma unroll
                    for (int h = 0; h < HMAX; ++h) p[h] += dot4(v[h][i], x);
                }
            }
#pragma unroll
            for (int h = 0; h < HMAX; ++h)
                if (h < d.H) {
                    const float s = warp_sum(p[h]);
                    if (lane == 0) sc[h * d.K + j] = s;
                }
        }
        __syncwarp();
        // softmax backward (lane = neighbour): ds = a (da - <a, da>) / sqrt(dh)
        const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
        for (int h = 0; h < d.H; ++h) {
            const float a = lane < c_n ? aa[h * d.K + lane] : 0.f;
            const float da = lane < c_n ? sc[h * d.K + lane] : 0.f;
            const float dot = warp_sum(a * da);
            __syncwarp();
            if (lane < d.K) sc[h * d.K + lane] = lane < c_n ? a * (da - dot) * inv : 0.f;
        }
        __syncwarp();
        // pass 2a: dq'_h = sum_j ds_hj x~_j
#pragma unroll
        for (int h = 0; h < HMAX; ++h)
#pragma unroll
            for (int i = 0; i < NCH; ++i) v[h][i] = z4();
#pragma unroll 1
        for (int j = 0; j < c_n; ++j) {
            const unsigned char* row = xs + (std::size_t)j * RB;
            float s[HMAX];
#pragma unroll
            for (int h = 0; h < HMAX; ++h) s[h] = h < d.H ? sc[h * d.K + j] : 0.f;
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const int ch = lane + 32 * i;
                if (ch < nch) {
                    const float4 x = x_chunk(d, ch, row);
#pragma unroll
                    for (int h = 0; h < HMAX; ++h) axpy4(v[h][i], s[h], x);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (h >= d.H) break;
            float4* o = reinterpret_cast<float4*>(dQp + row0 + (std::size_t)h * d.ld_p);
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const int ch = lane + 32 * i;
                if (ch < nch) o[ch] = rnd4(v[h][i], d.rnd);
            }
        }
        // pass 2b: input gradients on [s_nbr | phi] (no gather needed)
        float4 g[HMAX][NCX], q[HMAX][NCX];
#pragma unroll
        for (int h = 0; h < HMAX; ++h)
#pragma unroll
            for (int i = 0; i < NCX; ++i) {
                const int ch = lane + 32 * i;
                const bool ok = h < d.H && ch < nchx;
                g[h][i] = ok ? reinterpret_cast<const float4*>(dxbar + row0 + (std::size_t)h * d.ld_p)[ch] : z4();
                q[h][i] = ok ? reinterpret_cast<const float4*>(Qp + row0 + (std::size_t)h * d.ld_p)[ch] : z4();
            }
#pragma unroll 1
        for (int j = 0; j < c_n; ++j) {
            const int slot = __shfl_sync(0xffffffffu, m_slot, j);
            const double dt = __shfl_sync(0xffffffffu, m_dt, j);
            float a[HMAX], s[HMAX];
#pragma unroll
            for (int h = 0; h < HMAX; ++h) {
                a[h] = h < d.H ? aa[h * d.K + j] : 0.f;
                s[h] = h < d.H ? sc[h * d.K + j] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < NCX; ++i) {
                const int ch = lane + 32 * i;
                if (ch >= nchx) continue;
                float4 gx = z4();
#pragma unroll
                for (int h = 0; h < HMAX; ++h) {
                    axpy4(gx, a[h], g[h][i]);
                    axpy4(gx, s[h], q[h][i]);
                }
                const int c = 4 * ch;
                if (c < d.D) {
                    if (slot >= 0) atomicAdd(reinterpret_cast<float4*>(dH + (std::size_t)slot * d.D + c), gx);
                } else {
                    const int t = c - d.D;
                    const float4 wv = *reinterpret_cast<const float4*>(time_w + t);
                    const float4 bv = *reinterpret_cast<const float4*>(time_b + t);
                    const float s0 = time_sin(wv.x, bv.x, dt), s1 = time_sin(wv.y, bv.y, dt);
                    const float s2 = time_sin(wv.z, bv.z, dt), s3 = time_sin(wv.w, bv.w, dt);
                    const float fdt = (float)dt;
                    gb[i].x -= s0 * gx.x; gb[i].y -= s1 * gx.y; gb[i].z -= s2 * gx.z; gb[i].w -= s3 * gx.w;
                    gw[i].x -= s0 * gx.x * fdt; gw[i].y -= s1 * gx.y * fdt;
                    gw[i].z -= s2 * gx.z * fdt; gw[i].w -= s3 * gx.w * fdt;
                }
            }
        }
    }
    // fixed-order per-block reduction of the roots' time-encoder partials
    // (the staging area is reused: [kRootsPerBlock][2T] f32)
    __syncthreads();
    float* tw = reinterpret_cast<float*>(smem) + warp * 2 * d.T;
    for (int c = lane; c < 2 * d.T; c += 32) tw[c] = 0.f;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NCX; ++i) {
        const int ch = lane + 32 * i;
        const int c = 4 * ch;
        if (ch < nchx && c >= d.D) {
            const int t = c - d.D;
            tw[t] = gw[i].x; tw[t + 1] = gw[i].y; tw[t + 2] = gw[i].z; tw[t + 3] = gw[i].w;
            tw[d.T + t] = gb[i].x; tw[d.T + t + 1] = gb[i].y;
            tw[d.T + t + 2] = gb[i].z; tw[d.T + t + 3] = gb[i].w;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 2 * d.T; c += blockDim.x) {
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < kRootsPerBlock; ++k) sacc += (double)reinterpret_cast<float*>(smem)[k * 2 * d.T + c];
        part[(std::size_t)blockIdx.x * 2 * d.T + c] = sacc;
    }
}

#define SPD_ABS_FWD_INST(NCH, HM)                                                               \
    template __global__ void k_attn_abs_fwd<NCH, HM>(                                            \
        WorkerDev, Dims, int, const float*, const float*, const std::uint32_t*,                  \
        const std::uint32_t*, const double*, const int*, const float*, const float*, float*,     \
        float*);
#define SPD_ABS_BWD_INST(NCH, NCX, HM)                                                          \
    template __global__ void k_attn_abs_bwd<NCH, NCX, HM>(                                       \
        WorkerDev, Dims, int, const float*, const float*, const std::uint32_t*,                  \
        const std::uint32_t*, const double*, const int*, const float*, const float*,             \
        const float*, const float*, float*, float*, double*);
#define SPD_ABS_ALL(HM)                                                                         \
    SPD_ABS_FWD_INST(1, HM) SPD_ABS_FWD_INST(2, HM) SPD_ABS_FWD_INST(3, HM)                      \
    SPD_ABS_FWD_INST(4, HM)                                                                     \
    SPD_ABS_BWD_INST(1, 1, HM) SPD_ABS_BWD_INST(2, 1, HM) SPD_ABS_BWD_INST(2, 2, HM)             \
    SPD_ABS_BWD_INST(3, 1, HM) SPD_ABS_BWD_INST(3, 2, HM) SPD_ABS_BWD_INST(4, 1, HM)             \
    SPD_ABS_BWD_INST(4, 2, HM)
SPD_ABS_ALL(2)
SPD_ABS_ALL(4)
#undef SPD_ABS_ALL
#undef SPD_ABS_BWD_INST
#undef SPD_ABS_FWD_INST

}  // namespace tgnk
}  // namespace spd
