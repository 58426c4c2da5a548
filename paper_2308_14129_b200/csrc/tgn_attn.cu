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
// Execution: 3 warps per block, one root per warp. Each warp first stages its
// root's k neighbour rows in shared memory — memory row (f32, the GRU output
// when the neighbour was just updated) and raw bf16 feature row by TMA bulk
// copies, so every gather of the root is in flight at once — and, while those
// copies fly, each lane evaluates the time encoding cos(w dt + b) of its own
// time columns for every neighbour (f64 phase, tgn_common.cuh phase_sincos)
// into the same staged rows; both passes then read shared memory. Nothing of
// the time encoding is materialised in HBM.
//
// Lane slots are region-uniform: slot i < NM covers memory columns
// 4(lane + 32i), the next NT slots time columns, the last NF slots feature
// columns including the constant-1 bias column at F. Every slot of a warp is
// in one region, so the inner loops are branch-free (compile-time region).
#include "pdl.cuh"
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"

namespace spd {
namespace tgnk {

namespace {

// roots (warps) per block of the staging kernels: the staged rows (~11.8 KB
// per root at GDELT dims) bound residency, and 3-root blocks pack 18 warps
// per SM where 4-root blocks fit 16
#ifndef SPD_ATTN_ROOTS
#define SPD_ATTN_ROOTS 3
#endif
constexpr int kRootsPerBlock = SPD_ATTN_ROOTS;
constexpr int kRootsX = 4;  // roots per 128-thread block of the scatter kernel
// blocks per SM the staged rows allow at GDELT dims (6 x ~36.5 KB): registers
// capped to match for up to 4 slots and 2 heads, so shared memory stays the
// only residency limit (wider rows / more heads keep the compiler's choice)
template <int NM, int NT, int NF, int HMAX>
constexpr int attn_min_blocks() { return HMAX <= 2 && NM + NT + NF <= 4 ? 6 : 1; }

__device__ __forceinline__ float dot4acc(const float4& a, const float4& b, float acc) {
    return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, fmaf(a.x, b.x, acc))));
}
__device__ __forceinline__ void axpy4(float4& acc, float s, const float4& x) {
    acc.x += s * x.x; acc.y += s * x.y; acc.z += s * x.z; acc.w += s * x.w;
}
__device__ __forceinline__ float4 z4() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float4 rnd4(float4 v, int rnd) {
    return rnd ? make_float4(tf32r(v.x), tf32r(v.y), tf32r(v.z), tf32r(v.w)) : v;
}

// One staged neighbour row: [mem f32 D | cos f32 T | sin f32 T (bwd) | feat bf16 Fp]
// (each part one bulk copy: the memory row, the phi row, the feature row)
__host__ __device__ __forceinline__ int row_bytes(const Dims& d, bool with_sin) {
    return 4 * (d.D + d.T) + (with_sin ? 4 * d.T : 0) + 2 * d.Fp + 16;  // + 16 zero bytes (slot_offsets)
}
__host__ __device__ __forceinline__ int feat_off(const Dims& d, bool with_sin) {
    return 4 * (d.D + d.T) + (with_sin ? 4 * d.T : 0);
}

// Slot geometry (compile-time region per slot).
template <int NM, int NT, int NF>
struct Slots {
    static constexpr int N = NM + NT + NF;
    // region of slot i: 0 memory, 1 time, 2 feature|bias
    static constexpr __host__ __device__ int region(int i) { return i < NM ? 0 : (i < NM + NT ? 1 : 2); }
    static constexpr __host__ __device__ int local(int i) {
        return i < NM ? i : (i < NM + NT ? i - NM : i - NM - NT);
    }
    // first column of slot i for this lane, and whether it holds data
    static __device__ __forceinline__ int col(const Dims& d, int i, int lane) {
        const int o = 4 * (lane + 32 * local(i));
        return region(i) == 0 ? o : (region(i) == 1 ? d.D + o : d.D + d.T + o);
    }
    static __device__ __forceinline__ bool valid(const Dims& d, int i, int lane) {
        const int o = 4 * (lane + 32 * local(i));
        return region(i) == 0 ? o < d.D : (region(i) == 1 ? o < d.T : o <= d.F);
    }
};

// Slot i of a staged row: columns col(i)..+3 of [s_nbr | phi | e], the
// constant-1 bias column excluded (it reads as 0). Its terms drop out of the
// kernels exactly: <q'_h, e_bias> = <q_h, b_K,h> is the same for every
// neighbour, so softmax (shift invariant) ignores it and its gradient
// sum_j ds_hj is 0; in xbar it is sum_j a_hj = 1, set directly (set_bias).
// Byte offset of each slot's columns within a staged row, once per lane: a
// lane whose slot lies past its region reads the row's 16 zero tail bytes
// (zeroed at kernel start, after the feature row), so the inner loops are
// branch-free loads.
template <class S>
__device__ __forceinline__ void slot_offsets(int (&o)[S::N], const Dims& d, int lane, int foff) {
    const int tail = foff + 2 * d.Fp;
#pragma unroll
    for (int i = 0; i < S::N; ++i) {
        const int c = 4 * (lane + 32 * S::local(i));
        if (S::region(i) == 0) o[i] = c < d.D ? 4 * c : tail;
        else if (S::region(i) == 1) o[i] = c < d.T ? 4 * (d.D + c) : tail;
        else o[i] = c < d.Fp ? foff + 2 * c : tail;
    }
}
template <class S>
__device__ __forceinline__ float4 x_at(int i, const unsigned char* p) {
    if (S::region(i) != 2) return *reinterpret_cast<const float4*>(p);
    const uint2 raw = *reinterpret_cast<const uint2*>(p);
    return make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                       __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u));
}
__device__ __forceinline__ void zero_tails(const Dims& d, int lane, unsigned char* xs, int RB, int foff) {
    if (lane < d.K) *reinterpret_cast<float4*>(xs + (std::size_t)lane * RB + foff + 2 * d.Fp) = z4();
}

// Put value c into the bias column (feature index F) of every head's slots.
template <class S, int HMAX>
__device__ __forceinline__ void set_bias(float4 (&v)[HMAX][S::N], const Dims& d, int lane, float c) {
#pragma unroll
    for (int i = 0; i < S::N; ++i) {
        if (S::region(i) != 2) continue;
        const int b = d.F - 4 * (lane + 32 * S::local(i));
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            if (b == 0) v[h][i].x = c;
            else if (b == 1) v[h][i].y = c;
            else if (b == 2) v[h][i].z = c;
            else if (b == 3) v[h][i].w = c;
        }
    }
}

// Sum each of V values over the warp (V a power of two <= 32) with V - 1 +
// (5 - log2 V) shuffles instead of 5 V: every stage halves the values a lane
// carries. On return the lane holds the total of value index vidx<V>(lane).
template <int V>
__device__ __forceinline__ float warp_reduce_multi(float (&v)[V], int lane) {
    constexpr int LOG = V == 1 ? 0 : V == 2 ? 1 : V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;
#pragma unroll
    for (int st = 0; st < LOG; ++st) {
        const int o = 16 >> st;
        const bool up = lane & o;
#pragma unroll
        for (int k = 0; k < (V >> (st + 1)); ++k) {
            const int half = V >> (st + 1);
            const float send = up ? v[k] : v[k + half];
            const float keep = up ? v[k + half] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    float r = v[0];
#pragma unroll
    for (int o = 16 >> LOG; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}
template <int V>
__device__ __forceinline__ int vidx(int lane) {
    constexpr int LOG = V == 1 ? 0 : V == 2 ? 1 : V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;
    int idx = 0;
#pragma unroll
    for (int st = 0; st < LOG; ++st)
        if (lane & (16 >> st)) idx += V >> (st + 1);
    return idx;
}

// Stage root r's neighbour rows (warp-cooperative): lane j < c_n issues the
// two bulk copies of neighbour j's row — memory row (GRU output when just
// updated) and bf16 feature row — both completing on the warp's mbarrier, so
// every gather of the root is in flight at once for ~2 instructions per
// neighbour; the caller fills the time columns (fill_cos) and issues its
// per-root loads meanwhile, then waits. Lane j < c_n holds neighbour j's
// (dt, slot) on return.
__device__ __forceinline__ void stage_rows(const WorkerDev& w, const Dims& d, int r, int c_n,
                                           int lane, const std::uint32_t* nbr_node,
                                           const std::uint32_t* nbr_ev, const double* nbr_dt,
                                           const float* mem_new, unsigned char* xs,
                                           std::uint64_t* bar, double& m_dt, int& m_slot) {
    m_dt = 0.0;
    m_slot = -1;
    const unsigned per = 4u * d.D + 2u * d.Fp;
    if (lane == 0) bar_expect(bar, per * c_n);
    __syncwarp();
    if (lane < c_n) {
        const std::size_t o = (std::size_t)r * d.K + lane;
        const std::uint32_t node = nbr_node[o], ev = nbr_ev[o];
        m_dt = nbr_dt[o];
        m_slot = w.slot[node];
        const float* mrow = m_slot >= 0 ? mem_new + (std::size_t)m_slot * d.D : w.mem + (std::size_t)node * d.D;
        unsigned char* dst = xs + (std::size_t)lane * row_bytes(d, false);
        bulk_g2s(dst, mrow, 4u * d.D, bar);
        if (d.Fp) bulk_g2s(dst + feat_off(d, false), w.feat + (std::size_t)ev * d.Fp, 2u * d.Fp, bar);
    }
    // the caller fills the time columns, issues its own per-root loads, then
    // waits (bar_wait(bar, 0))
}

// Time columns of the staged rows: each lane writes cos(w dt_j + b) of its own
// time slots (the columns its x_at reads) for every neighbour j < c_n.
template <class S>
__device__ __forceinline__ void fill_cos(const Dims& d, int lane, int c_n, double m_dt,
                                         const float* time_w, const float* time_b,
                                         unsigned char* xs, int RB) {
    float4 tw[S::N], tb[S::N];
#pragma unroll
    for (int i = 0; i < S::N; ++i) {
        const int o = 4 * (lane + 32 * S::local(i));
        const bool ok = S::region(i) == 1 && o < d.T;
        tw[i] = ok ? *reinterpret_cast<const float4*>(time_w + o) : z4();
        tb[i] = ok ? *reinterpret_cast<const float4*>(time_b + o) : z4();
    }
    // two neighbours per pass: 8 independent phase chains per lane
#pragma unroll 1
    for (int j0 = 0; j0 < c_n; j0 += 2) {
        const int j1 = j0 + 1 < c_n ? j0 + 1 : j0;
        const double dt0 = __shfl_sync(0xffffffffu, m_dt, j0);
        const double dt1 = __shfl_sync(0xffffffffu, m_dt, j1);
        unsigned char* row0 = xs + (std::size_t)j0 * RB;
        unsigned char* row1 = xs + (std::size_t)j1 * RB;
#pragma unroll
        for (int i = 0; i < S::N; ++i) {
            if (S::region(i) != 1) continue;
            const int o = 4 * (lane + 32 * S::local(i));
            if (o >= d.T) continue;
            const float a0 = time_cos(tw[i].x, tb[i].x, dt0), a1 = time_cos(tw[i].y, tb[i].y, dt0);
            const float a2 = time_cos(tw[i].z, tb[i].z, dt0), a3 = time_cos(tw[i].w, tb[i].w, dt0);
            const float b0 = time_cos(tw[i].x, tb[i].x, dt1), b1 = time_cos(tw[i].y, tb[i].y, dt1);
            const float b2 = time_cos(tw[i].z, tb[i].z, dt1), b3 = time_cos(tw[i].w, tb[i].w, dt1);
            *reinterpret_cast<float4*>(row0 + 4 * (d.D + o)) = make_float4(a0, a1, a2, a3);
            *reinterpret_cast<float4*>(row1 + 4 * (d.D + o)) = make_float4(b0, b1, b2, b3);
        }
    }
}

template <class S, int HMAX>
__device__ __forceinline__ void load_slots(float4 (&v)[HMAX][S::N], const float* base, const Dims& d,
                                           int lane) {
#pragma unroll
    for (int h = 0; h < HMAX; ++h)
#pragma unroll
        for (int i = 0; i < S::N; ++i)
            v[h][i] = (h < d.H && S::valid(d, i, lane))
                          ? *reinterpret_cast<const float4*>(base + (std::size_t)h * d.ld_p + S::col(d, i, lane))
                          : z4();
}

template <class S, int HMAX>
__device__ __forceinline__ void store_slots(const float4 (&v)[HMAX][S::N], float* base, const Dims& d,
                                            int lane, int rnd) {
#pragma unroll
    for (int h = 0; h < HMAX; ++h) {
        if (h >= d.H) break;
#pragma unroll
        for (int i = 0; i < S::N; ++i)
            if (S::valid(d, i, lane))
                *reinterpret_cast<float4*>(base + (std::size_t)h * d.ld_p + S::col(d, i, lane)) = rnd4(v[h][i], rnd);
    }
}

// One group of G neighbours j0 .. j0+G-1 (all valid): their G*HMAX partial dot
// products share one multi-value warp reduction.
template <class S, int HMAX, int G>
__device__ __forceinline__ void dots_group(const float4 (&v)[HMAX][S::N], const Dims& d, int lane,
                                           const unsigned char* xs, int RB, const int (&off)[S::N],
                                           int j0, float* sc, float scale) {
    constexpr int V = G * HMAX;
    float p[V];
#pragma unroll
    for (int k = 0; k < V; ++k) p[k] = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const unsigned char* row = xs + (std::size_t)(j0 + g) * RB;
#pragma unroll
        for (int i = 0; i < S::N; ++i) {
            const float4 x = x_at<S>(i, row + off[i]);
#pragma unroll
            for (int h = 0; h < HMAX; ++h) p[h * G + g] = dot4acc(v[h][i], x, p[h * G + g]);
        }
    }
    const float r = warp_reduce_multi<V>(p, lane);
    const int vi = vidx<V>(lane);
    const int hv = vi / G, gv = vi % G;
    if ((lane & ((32 / V) - 1)) == 0 && hv < d.H) sc[hv * d.K + j0 + gv] = r * scale;
}

// sc[h*K + j] = scale * <v[h], x~_j> for every valid neighbour j: full groups
// of 8, then groups of 4, 2, 1 for the rest (no per-neighbour guards; every
// reduction carries only valid neighbours).
template <class S, int HMAX>
__device__ __forceinline__ void dots(const float4 (&v)[HMAX][S::N], const Dims& d, int lane,
                                     const unsigned char* xs, int RB, int foff, int c_n, float* sc,
                                     float scale) {
    int off[S::N];
    slot_offsets<S>(off, d, lane, foff);
    int j0 = 0;
#pragma unroll 1
    for (; j0 + 8 <= c_n; j0 += 8) dots_group<S, HMAX, 8>(v, d, lane, xs, RB, off, j0, sc, scale);
    if (j0 + 4 <= c_n) {
        dots_group<S, HMAX, 4>(v, d, lane, xs, RB, off, j0, sc, scale);
        j0 += 4;
    }
    if (j0 + 2 <= c_n) {
        dots_group<S, HMAX, 2>(v, d, lane, xs, RB, off, j0, sc, scale);
        j0 += 2;
    }
    if (j0 < c_n) dots_group<S, HMAX, 1>(v, d, lane, xs, RB, off, j0, sc, scale);
}

template <class S, int HMAX>
__device__ __forceinline__ void axpys(float4 (&v)[HMAX][S::N], const Dims& d, int lane,
                                      const unsigned char* xs, int RB, int foff, int c_n,
                                      const float* coef) {
    int off[S::N];
    slot_offsets<S>(off, d, lane, foff);
#pragma unroll 2
    for (int j = 0; j < c_n; ++j) {
        const unsigned char* row = xs + (std::size_t)j * RB;
        float a[HMAX];
#pragma unroll
        for (int h = 0; h < HMAX; ++h) a[h] = h < d.H ? coef[h * d.K + j] : 0.f;
#pragma unroll
        for (int i = 0; i < S::N; ++i) {
            const float4 x = x_at<S>(i, row + off[i]);
#pragma unroll
            for (int h = 0; h < HMAX; ++h) axpy4(v[h][i], a[h], x);
        }
    }
}

}  // namespace

__host__ __device__ std::size_t attn_smem_bytes(const Dims& d, bool bwd) {
    // forward and backward stage the same rows (memory | cos | features)
    const std::size_t stage = std::size_t(kRootsPerBlock) * d.K * row_bytes(d, false);
    return stage + kRootsPerBlock * 2 * sizeof(float) * d.H * d.K +
           kRootsPerBlock * sizeof(std::uint64_t);
}
int attn_roots_per_block() { return kRootsPerBlock; }
int attn_x_roots_per_block() { return kRootsX; }

// Forward: scores from q'_h (Qp), softmax, alpha [R][H][K], xbar_h [R][H][ld_p]
// (tf32-rounded when it feeds a tensor-core GEMM). Roots without neighbours
// get xbar = 0 (bias slot 0 too: ctx = 0; the oracle masks them).
template <int NM, int NT, int NF, int HMAX>
__global__ void __launch_bounds__(32 * kRootsPerBlock, (attn_min_blocks<NM, NT, NF, HMAX>())) k_attn_abs_fwd(WorkerDev w, Dims d, int R,
                                                      const float* time_w, const float* time_b,
                                                      const std::uint32_t* nbr_node,
                                                      const std::uint32_t* nbr_ev,
                                                      const double* nbr_dt, const int* cnt,
                                                      const float* mem_new, const float* Qp,
                                                      float* alpha, float* xbar) {
    pdl_entry();
    using S = Slots<NM, NT, NF>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * kRootsPerBlock + warp;
    if (r >= R) return;
    constexpr bool BWD = false;
    const int RB = row_bytes(d, BWD);
    unsigned char* xs = smem + (std::size_t)warp * d.K * RB;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(smem + attn_smem_bytes(d, BWD)) - kRootsPerBlock + warp;
    float* sc = reinterpret_cast<float*>(bar - warp) - kRootsPerBlock * 2 * d.H * d.K + warp * 2 * d.H * d.K;
    if (lane == 0) bar_init(bar);
    zero_tails(d, lane, xs, RB, feat_off(d, BWD));
    __syncwarp();
    const int c_n = cnt[r];
    const std::size_t row0 = (std::size_t)r * d.H * d.ld_p;
    float4 v[HMAX][S::N];  // q'_h, then the xbar accumulators
    if (c_n == 0) {
#pragma unroll
        for (int h = 0; h < HMAX; ++h)
#pragma unroll
            for (int i = 0; i < S::N; ++i) v[h][i] = z4();
        store_slots<S, HMAX>(v, xbar + row0, d, lane, 0);
        if (lane < d.K)
            for (int h = 0; h < d.H; ++h) alpha[((std::size_t)r * d.H + h) * d.K + lane] = 0.f;
        return;
    }
    double m_dt;
    int m_slot;
    stage_rows(w, d, r, c_n, lane, nbr_node, nbr_ev, nbr_dt, mem_new, xs, bar, m_dt, m_slot);
    fill_cos<S>(d, lane, c_n, m_dt, time_w, time_b, xs, RB);
    load_slots<S, HMAX>(v, Qp + row0, d, lane);
    bar_wait(bar, 0);
    const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
    dots<S, HMAX>(v, d, lane, xs, RB, feat_off(d, BWD), c_n, sc, inv);
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
        for (int i = 0; i < S::N; ++i) v[h][i] = z4();
    axpys<S, HMAX>(v, d, lane, xs, RB, feat_off(d, BWD), c_n, sc);
    set_bias<S, HMAX>(v, d, lane, 1.f);  // sum_j a_hj
    store_slots<S, HMAX>(v, xbar + row0, d, lane, d.rnd);
}

// Backward, given dxbar_h = [W_V,h|b_V,h]^T dctx_h (GEMM) per root, in three
// kernels so the critical path (dq'_h -> dQ GEMM -> query backward) does not
// wait for the input-gradient work:
//   k_attn_abs_bwd (critical path):
//     da_hj = <dxbar_h, x~_j>;  ds_hj = a_hj (da_hj - sum_k a_hk da_hk) / sqrt(dh)
//     dq'_h = sum_j ds_hj x~_j                       -> dQp (GEMMs give dQ, dW_K)
//     ds    -> dsc [R][H][K]
//   then, beside the dQ GEMMs, the input gradient of x~_j
//     dx_j  = sum_h a_hj dxbar_h + ds_hj q'_h
//   on its gradient-carrying columns: the memory part is summed per pending
//   row in a fixed order by tgn_dh.cu (k_dh_pull, no atomics), the time part
//   gives d/dw, d/db of cos(w dt + b) in k_attn_time_grad (per-block partials,
//   fixed order). Neither needs staged rows: only per-root vectors, alpha,
//   ds and the neighbours' dt.
template <int NM, int NT, int NF, int HMAX>
__global__ void __launch_bounds__(32 * kRootsPerBlock, (attn_min_blocks<NM, NT, NF, HMAX>())) k_attn_abs_bwd(WorkerDev w, Dims d, int R,
                                                      const float* time_w, const float* time_b,
                                                      const std::uint32_t* nbr_node,
                                                      const std::uint32_t* nbr_ev,
                                                      const double* nbr_dt, const int* cnt,
                                                      const float* mem_new, const float* Qp,
                                                      const float* alpha, const float* dxbar,
                                                      float* dQp, float* dsc) {
    pdl_entry();
    using S = Slots<NM, NT, NF>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * kRootsPerBlock + warp;
    if (r >= R) return;
    constexpr bool BWD = false;  // staged rows: memory | cos | features (as the forward)
    const int RB = row_bytes(d, BWD);
    unsigned char* xs = smem + (std::size_t)warp * d.K * RB;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(smem + attn_smem_bytes(d, true)) - kRootsPerBlock + warp;
    float* sc = reinterpret_cast<float*>(bar - warp) - kRootsPerBlock * 2 * d.H * d.K + warp * 2 * d.H * d.K;
    if (lane == 0) bar_init(bar);
    zero_tails(d, lane, xs, RB, feat_off(d, BWD));
    __syncwarp();
    float* aa = sc + d.H * d.K;  // alpha of this root
    const int c_n = cnt[r];
    const std::size_t row0 = (std::size_t)r * d.H * d.ld_p;
    float4 v[HMAX][S::N];  // dxbar_h, then the dq'_h accumulators
    if (c_n == 0) {
#pragma unroll
        for (int h = 0; h < HMAX; ++h)
#pragma unroll
            for (int i = 0; i < S::N; ++i) v[h][i] = z4();
        store_slots<S, HMAX>(v, dQp + row0, d, lane, 0);
        return;
    }
    double m_dt;
    int m_slot;
    stage_rows(w, d, r, c_n, lane, nbr_node, nbr_ev, nbr_dt, mem_new, xs, bar, m_dt, m_slot);
    fill_cos<S>(d, lane, c_n, m_dt, time_w, time_b, xs, RB);
    if (lane < d.K)
        for (int h = 0; h < d.H; ++h)
            aa[h * d.K + lane] = lane < c_n ? alpha[((std::size_t)r * d.H + h) * d.K + lane] : 0.f;
    load_slots<S, HMAX>(v, dxbar + row0, d, lane);
    bar_wait(bar, 0);
    __syncwarp();
    // pass 1: da_hj
    dots<S, HMAX>(v, d, lane, xs, RB, feat_off(d, BWD), c_n, sc, 1.f);
    __syncwarp();
    // softmax backward (lane = neighbour): ds = a (da - <a, da>) / sqrt(dh)
    const float inv = 1.f / sqrtf((float)(d.DQ / d.H));
    for (int h = 0; h < d.H; ++h) {
        const float a = lane < c_n ? aa[h * d.K + lane] : 0.f;
        const float da = lane < c_n ? sc[h * d.K + lane] : 0.f;
        const float dot = warp_sum(a * da);
        __syncwarp();
        const float ds = lane < c_n ? a * (da - dot) * inv : 0.f;
        if (lane < d.K) {
            sc[h * d.K + lane] = ds;
            dsc[((std::size_t)r * d.H + h) * d.K + lane] = ds;
        }
    }
    __syncwarp();
    // pass 2a: dq'_h = sum_j ds_hj x~_j
#pragma unroll
    for (int h = 0; h < HMAX; ++h)
#pragma unroll
        for (int i = 0; i < S::N; ++i) v[h][i] = z4();
    axpys<S, HMAX>(v, d, lane, xs, RB, feat_off(d, BWD), c_n, sc);
    store_slots<S, HMAX>(v, dQp + row0, d, lane, d.rnd);
}

// Time-encoder gradient of the attention backward (see above): one warp per
// root, kRootsX roots per block; part: [gridDim.x][2T] (w then b), f64, every
// block writes its row. Lane slot i covers time columns 4(lane + 32 i); the
// sin of the phase is evaluated inline (f64 phase, phase_sincos).
template <int NT, int HMAX>
__global__ void __launch_bounds__(128) k_attn_time_grad(Dims d, int R, const float* time_w,
                                                        const float* time_b, const double* nbr_dt,
                                                        const int* cnt, const float* Qp,
                                                        const float* alpha, const float* dsc,
                                                        const float* dxbar, double* part) {
    pdl_entry();
    __shared__ double red[kRootsX][2 * 4 * 32 * NT];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grid-stride over root groups (a capped grid leaves SMs to the critical
    // path beside it): per-root float partials, accumulated per lane in f64
    double aw[NT][4], ab[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) aw[i][k] = ab[i][k] = 0.0;
    for (int r = blockIdx.x * kRootsX + warp; r - warp < R; r += gridDim.x * kRootsX) {
    const int c_n = r < R ? cnt[r] : 0;
    float4 gw[NT], gb[NT];  // time-encoder gradient partials of this lane's time slots
#pragma unroll
    for (int i = 0; i < NT; ++i) gw[i] = gb[i] = z4();
    if (c_n > 0) {
        const std::size_t row0 = (std::size_t)r * d.H * d.ld_p;
        // neighbour j's dt on lane j; alpha and ds of lane j per head
        double m_dt = 0.0;
        float la[HMAX], ls[HMAX];
        if (lane < c_n) m_dt = nbr_dt[(std::size_t)r * d.K + lane];
#pragma unroll
        for (int h = 0; h < HMAX; ++h) {
            const bool ok = h < d.H && lane < c_n;
            la[h] = ok ? alpha[((std::size_t)r * d.H + h) * d.K + lane] : 0.f;
            ls[h] = ok ? dsc[((std::size_t)r * d.H + h) * d.K + lane] : 0.f;
        }
        float4 g[HMAX][NT], q[HMAX][NT], tw[NT], tb[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            const int o = 4 * (lane + 32 * i);
            const bool okc = o < d.T;
            tw[i] = okc ? *reinterpret_cast<const float4*>(time_w + o) : z4();
            tb[i] = okc ? *reinterpret_cast<const float4*>(time_b + o) : z4();
#pragma unroll
            for (int h = 0; h < HMAX; ++h) {
                const bool ok = h < d.H && okc;
                const std::size_t c = row0 + (std::size_t)h * d.ld_p + d.D + o;
                g[h][i] = ok ? *reinterpret_cast<const float4*>(dxbar + c) : z4();
                q[h][i] = ok ? *reinterpret_cast<const float4*>(Qp + c) : z4();
            }
        }
#pragma unroll 1
        for (int j = 0; j < c_n; ++j) {
            const double dt = __shfl_sync(0xffffffffu, m_dt, j);
            const float fdt = (float)dt;
            float a[HMAX], sv_[HMAX];
#pragma unroll
            for (int h = 0; h < HMAX; ++h) {
                a[h] = __shfl_sync(0xffffffffu, la[h], j);
                sv_[h] = __shfl_sync(0xffffffffu, ls[h], j);
            }
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                if (4 * (lane + 32 * i) >= d.T) continue;
                float4 gx = z4();
#pragma unroll
                for (int h = 0; h < HMAX; ++h) {
                    axpy4(gx, a[h], g[h][i]);
                    axpy4(gx, sv_[h], q[h][i]);
                }
                const float4 sv = make_float4(time_sin(tw[i].x, tb[i].x, dt), time_sin(tw[i].y, tb[i].y, dt),
                                              time_sin(tw[i].z, tb[i].z, dt), time_sin(tw[i].w, tb[i].w, dt));
                float4& bw = gw[i];
                float4& bb = gb[i];
                bb.x -= sv.x * gx.x; bb.y -= sv.y * gx.y; bb.z -= sv.z * gx.z; bb.w -= sv.w * gx.w;
                bw.x -= sv.x * gx.x * fdt; bw.y -= sv.y * gx.y * fdt;
                bw.z -= sv.z * gx.z * fdt; bw.w -= sv.w * gx.w * fdt;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        aw[i][0] += gw[i].x; aw[i][1] += gw[i].y; aw[i][2] += gw[i].z; aw[i][3] += gw[i].w;
        ab[i][0] += gb[i].x; ab[i][1] += gb[i].y; ab[i][2] += gb[i].z; ab[i][3] += gb[i].w;
    }
    }
    // fixed-order per-block reduction of the warps' time-encoder partials
    double* tws = red[warp];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int t = 4 * (lane + 32 * i) + k;
            tws[t] = aw[i][k];
            tws[4 * 32 * NT + t] = ab[i][k];
        }
    __syncthreads();
    for (int c = threadIdx.x; c < 2 * d.T; c += blockDim.x) {
        const int cc = c < d.T ? c : 4 * 32 * NT + (c - d.T);
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < kRootsX; ++k) sacc += red[k][cc];
        part[(std::size_t)blockIdx.x * 2 * d.T + c] = sacc;
    }
}

#define SPD_ABS_INST(NM, NT, NF, HM)                                                            \
    template __global__ void k_attn_abs_fwd<NM, NT, NF, HM>(                                     \
        WorkerDev, Dims, int, const float*, const float*, const std::uint32_t*,                  \
        const std::uint32_t*, const double*, const int*, const float*, const float*, float*,     \
        float*);                                                                                \
    template __global__ void k_attn_abs_bwd<NM, NT, NF, HM>(                                     \
        WorkerDev, Dims, int, const float*, const float*, const std::uint32_t*,                  \
        const std::uint32_t*, const double*, const int*, const float*, const float*,             \
        const float*, const float*, float*, float*);
#define SPD_ABS_NF(NM, NT, HM) \
    SPD_ABS_INST(NM, NT, 1, HM) SPD_ABS_INST(NM, NT, 2, HM) SPD_ABS_INST(NM, NT, 3, HM)
#define SPD_ABS_H(HM) SPD_ABS_NF(1, 1, HM) SPD_ABS_NF(1, 2, HM) SPD_ABS_NF(2, 1, HM)
SPD_ABS_H(2)
SPD_ABS_H(4)
#undef SPD_ABS_H
#undef SPD_ABS_NF
#undef SPD_ABS_INST
template __global__ void k_attn_time_grad<1, 2>(Dims, int, const float*, const float*, const double*,
                                                const int*, const float*, const float*, const float*,
                                                const float*, double*);
template __global__ void k_attn_time_grad<1, 4>(Dims, int, const float*, const float*, const double*,
                                                const int*, const float*, const float*, const float*,
                                                const float*, double*);
template __global__ void k_attn_time_grad<2, 2>(Dims, int, const float*, const float*, const double*,
                                                const int*, const float*, const float*, const float*,
                                                const float*, double*);
template __global__ void k_attn_time_grad<2, 4>(Dims, int, const float*, const float*, const double*,
                                                const int*, const float*, const float*, const float*,
                                                const float*, double*);

}  // namespace tgnk
}  // namespace spd
