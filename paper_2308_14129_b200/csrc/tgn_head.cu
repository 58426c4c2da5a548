// Fused embedding head of the TGN step (gemm_mode 1): everything between the
// attention context and its gradient in ONE kernel, per block of 16 events —
//
//   forward   O = [ctx | 1] W_o^T (masked: no neighbours -> 0)      tensor cores
//             m_in = [O | s_root | 1];  Z1 = relu(m_in W_m1^T)        tensor cores
//             emb = [Z1 | 1] W_m2^T                                  tensor cores
//             D1 = relu(W_a z_src + W_b z_{dst|neg} + b1)             FP32 FFMA
//             logit = D1 . w2 + b2;  BCE terms, dlogit, dD1           FP32 FFMA
//   backward  d_emb = dD1 W_d1 (by halves)                            FP32 FFMA
//             dZ1 = (d_emb W_m2) * [Z1 > 0]                          tensor cores
//             dm_in = dZ1 W_m1  (rows without neighbours: O part 0)   tensor cores
//             dctx = dm_in[:, :DQ] W_o                               tensor cores
//
// — the TGAT temporal-attention layer's output projection and merge MLP (the
// attention projections the north star allows on tensor cores, in TF32,
// tolerance-gated like the GRU) and the link-prediction decoder (FP32 FFMA,
// as the north star requires). It replaces 13 kernels of the step's critical
// path (W_o GEMM, merge gather, two merge GEMMs, two decoder GEMMs, the head,
// the decoder data-gradient GEMM and scatter, three data-gradient GEMMs and a
// row mask): the 48 rows of a block (src, dst and negative roots of its 16
// events) stay in shared memory from the context to its gradient; only the
// activations the weight-gradient GEMMs read are written out.
//
// Tensor-core GEMMs: warp-level mma.sync m16n8k8 TF32 (3 m-tiles of 16 rows x
// the warp's n-tiles of 8 columns; n-tile j of warp w is w + 8 j). Within a
// 32-wide k group, lane (g, t) supplies physical columns k0 + 8t .. 8t + 7 as
// the k-slots (t, t + 4) of 4 consecutive MMAs — A and B permuted alike, so
// the products pair up and the loads are two 16-byte vectors (weights
// straight from L2, one group ahead; activations from shared memory with a
// row stride = 4 mod 32, conflict-free). Operands are tf32-rounded as the
// tcgen05 path's; accumulation is FP32.
//
// Semantics: oracle/tgn_oracle.py TGNOracle._embed / _decode and the loss;
// the separate-kernel path of tgn_trainer.cu computes the same values.
#include "pdl.cuh"
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"

namespace spd {
namespace tgnk {

namespace {
constexpr int kEB = 16;       // events per block
constexpr int kRows = 3 * kEB;  // src | dst | neg rows
constexpr int kWarps = 8;
constexpr int kNTW = 5;       // max n-tiles per warp (N <= 320)

__device__ __forceinline__ int pad8(int k) { return (k + 7) / 8 * 8; }
// activation row stride: >= k, = 4 (mod 32) floats (conflict-free fragment loads)
__host__ __device__ __forceinline__ int act_ld(int k) { return ((k + 7) / 8 * 8 + 27) / 32 * 32 + 4; }

__device__ __forceinline__ std::uint32_t f2u(float x) { return __float_as_uint(x); }

__device__ __forceinline__ void mma_tf32(float (&c)[4], const std::uint32_t (&a)[4], std::uint32_t b0,
                                         std::uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Weight operand values of one 32-wide k group for lane (g, t), n-tile n0:
// the 8 physical k's k0 + 8t .. + 7 of output column n = n0 + g.
//   TRANS (forward, B[k][n] = W[n][k]): one row segment, two 16-B loads;
//   !TRANS (data gradient, B[k][n] = W[k][n]): 8 rows of column n.
template <bool TRANS>
__device__ __forceinline__ void load_w(float (&v)[8], const float* __restrict__ W, int ldw, int n, int N,
                                       int k, int Kv) {
    if (TRANS) {
        if (n < N && k + 8 <= Kv) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(W + (std::size_t)n * ldw + k));
            const float4 y = __ldg(reinterpret_cast<const float4*>(W + (std::size_t)n * ldw + k + 4));
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = n < N && k + q < Kv ? __ldg(W + (std::size_t)n * ldw + k + q) : 0.f;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = n < N && k + q < Kv ? __ldg(W + (std::size_t)(k + q) * ldw + n) : 0.f;
    }
}

// acc[mt][j][.] = rows [16 mt, 16 mt + 16) x columns [8 nt, 8 nt + 8) of
// A[48 x Kv] . B, nt = warp + 8 j < ceil(N / 8). A: shared memory (row stride
// lda, columns [Kv, pad32(Kv)) zero), B: weights W (see load_w).
template <bool TRANS>
__device__ __forceinline__ void gemm48(float (&acc)[3][kNTW][4], const float* As, int lda,
                                       const float* __restrict__ W, int ldw, int N, int Kv) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ntiles = (N + 7) / 8;
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int j = 0; j < kNTW; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[m][j][q] = 0.f;
    const int groups = (Kv + 31) / 32;
    float wb[kNTW][8];
#pragma unroll
    for (int j = 0; j < kNTW; ++j)
        if (warp + 8 * j < ntiles) load_w<TRANS>(wb[j], W, ldw, 8 * (warp + 8 * j) + g, N, 8 * t, Kv);
#pragma unroll 1
    for (int gi = 0; gi < groups; ++gi) {
        const int k = 32 * gi + 8 * t;
        float wn[kNTW][8];  // next group's weights, in flight during this group's MMAs
#pragma unroll
        for (int j = 0; j < kNTW; ++j)
            if (warp + 8 * j < ntiles && gi + 1 < groups)
                load_w<TRANS>(wn[j], W, ldw, 8 * (warp + 8 * j) + g, N, k + 32, Kv);
        float av[3][2][8];  // rows g and g + 8 of each m-tile, physical k .. k + 7
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float* p = As + (std::size_t)(16 * m + g + 8 * h) * lda + k;
                const float4 x = *reinterpret_cast<const float4*>(p);
                const float4 y = *reinterpret_cast<const float4*>(p + 4);
                av[m][h][0] = x.x; av[m][h][1] = x.y; av[m][h][2] = x.z; av[m][h][3] = x.w;
                av[m][h][4] = y.x; av[m][h][5] = y.y; av[m][h][6] = y.z; av[m][h][7] = y.w;
            }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
#pragma unroll
            for (int j = 0; j < kNTW; ++j) {
                if (warp + 8 * j >= ntiles) break;
                const std::uint32_t b0 = f2u(wb[j][2 * s]), b1 = f2u(wb[j][2 * s + 1]);
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    const std::uint32_t a[4] = {f2u(av[m][0][2 * s]), f2u(av[m][1][2 * s]),
                                                f2u(av[m][0][2 * s + 1]), f2u(av[m][1][2 * s + 1])};
                    mma_tf32(acc[m][j], a, b0, b1);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kNTW; ++j)
#pragma unroll
            for (int q = 0; q < 8; ++q) wb[j][q] = wn[j][q];
    }
}

// Visit this warp's accumulator elements: f(row, col, value) for col < N.
template <class F>
__device__ __forceinline__ void for_acc(const float (&acc)[3][kNTW][4], int N, F&& f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int j = 0; j < kNTW; ++j) {
        const int n0 = 8 * (warp + 8 * j);
        if (n0 >= N) break;
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int row = 16 * m + g + (q >> 1) * 8, col = n0 + 2 * t + (q & 1);
                if (col < N) f(row, col, acc[m][j][q]);
            }
    }
}

__device__ __forceinline__ void zero_cols(float* A, int lda, int c0, int c1) {
    for (int i = threadIdx.x; i < kRows * (c1 - c0); i += blockDim.x)
        A[(std::size_t)(i / (c1 - c0)) * lda + c0 + i % (c1 - c0)] = 0.f;
}

__device__ __forceinline__ float softplusf_(float x) { return x > 20.f ? x : log1pf(expf(x)); }

// FP32 FFMA over the 48 block rows, register-tiled: thread (rg, cg) of a
// 16 x 16 layout owns rows 3 rg .. 3 rg + 2 and columns cg + 16 j (j < 7):
//   Y[row][c] = sum_k X[row][k] * Wt(k, c, row)
// X rows in shared memory (stride ldx), Wt read through `w(k, c, row)`;
// 21 independent accumulators, k unrolled by 4.
template <class WF, class OUT>
__device__ __forceinline__ void ffma48(const float* X, int ldx, int K, int N, WF&& w, OUT&& out) {
    const int rg = threadIdx.x >> 4, cg = threadIdx.x & 15;
    float acc[3][7];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 7; ++j) acc[a][j] = 0.f;
    const float* x0 = X + (std::size_t)(3 * rg) * ldx;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
        const float xa = x0[k], xb = x0[ldx + k], xc = x0[2 * ldx + k];
#pragma unroll
        for (int j = 0; j < 7; ++j) {
            const int c = cg + 16 * j;
            if (c < N) {
                acc[0][j] = fmaf(xa, w(k, c, 3 * rg), acc[0][j]);
                acc[1][j] = fmaf(xb, w(k, c, 3 * rg + 1), acc[1][j]);
                acc[2][j] = fmaf(xc, w(k, c, 3 * rg + 2), acc[2][j]);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 7; ++j)
            if (cg + 16 * j < N) out(3 * rg + a, cg + 16 * j, acc[a][j]);
}
}  // namespace

std::size_t head_smem_bytes(const Dims& d) {
    const std::size_t ldo = act_ld(d.DQ + 1), ldm = act_ld(d.DQ + d.D + 1), ldz = act_ld(d.D + 1);
    const std::size_t a = kRows * ldo, m = kRows * ldm;
    const std::size_t w1 = std::size_t(d.D) * (2 * d.D + 1);  // decoder weights (reuse A|M)
    return 4 * ((a + m > w1 ? a + m : w1) + 3 * kRows * ldz + kRows * d.D + 2 * 2 * kEB * (d.D + 1) +
                2 * kEB);
}

__global__ void __launch_bounds__(256, 1) k_head(HeadArgs h) {
    pdl_entry();
    extern __shared__ __align__(16) float sm[];
    const Dims& d = h.d;
    const int D = d.D, DQ = d.DQ, B = h.B;
    const int ldo = act_ld(DQ + 1), ldm = act_ld(DQ + D + 1), ldz = act_ld(D + 1);
    float* sA = sm;                        // [48][ldo]: [ctx | 1], later dm_in[:, :DQ]
    float* sM = sA + kRows * ldo;          // [48][ldm]: m_in
    float* sW1 = sm;                       // decoder weights [D][2D + 1] over sA | sM (FFMA phase)
    const std::size_t am = (std::size_t)kRows * ldo + (std::size_t)kRows * ldm;
    const std::size_t w1n = (std::size_t)D * (2 * D + 1);
    float* sZ = sm + (am > w1n ? am : w1n);  // [48][ldz]: [Z1 | 1]
    float* sE = sZ + kRows * ldz;          // [48][D]: emb (fp32; FFMA reads, row-broadcast)
    float* sdE = sE + kRows * D;           // [48][ldz]: d_emb
    float* sdZ = sdE + kRows * ldz;        // [48][ldz]: dZ1
    float* sD1 = sdZ + kRows * ldz;        // [32][D + 1]: D1 (pos rows 0..15, neg 16..31)
    float* sdD1 = sD1 + 2 * kEB * (D + 1); // [32][D + 1]: dD1
    float* sg = sdD1 + 2 * kEB * (D + 1);  // [32]: dlogit
    __shared__ int s_has[kRows];           // root has neighbours (attention output kept)
    __shared__ const float* s_mrow[kRows];  // the root's memory row (GRU output when pending)
    const int i0 = blockIdx.x * kEB;
    // local row lr -> event i0 + lr % 16, kind lr / 16 (src, dst, neg); global root row
    auto grow = [&](int lr) { return (lr / kEB) * B + i0 + lr % kEB; };
    auto valid = [&](int lr) { return i0 + lr % kEB < B; };
    if (threadIdx.x < kRows) {
        const int lr = threadIdx.x;
        int has = 0;
        const float* mr = nullptr;
        if (valid(lr)) {
            const int r = grow(lr);
            const std::uint32_t n = h.roots[r];
            const int sl = h.w.slot[n];
            has = h.cnt[r] > 0;
            mr = sl >= 0 ? h.mem_new + (std::size_t)sl * D : h.w.mem + (std::size_t)n * D;
        }
        s_has[lr] = has;
        s_mrow[lr] = mr;
    }
    __syncthreads();

    // ---- F1: [ctx | 1] rows (tf32 already); pad columns zero
    const int Ko = DQ + 1, Kop = (Ko + 31) / 32 * 32;
    for (int i = threadIdx.x; i < kRows * Kop; i += blockDim.x) {
        const int lr = i / Kop, c = i % Kop;
        sA[(std::size_t)lr * ldo + c] = valid(lr) && c < Ko ? h.ctx[(std::size_t)grow(lr) * d.ld_ctx + c] : 0.f;
    }
    // s_root columns of m_in (tf32), bias 1, pad
    const int Km = DQ + D + 1, Kmp = (Km + 31) / 32 * 32;
    for (int i = threadIdx.x; i < kRows * (Kmp - DQ); i += blockDim.x) {
        const int lr = i / (Kmp - DQ), c = DQ + i % (Kmp - DQ);
        float v = 0.f;
        if (valid(lr) && c < DQ + D) {
            v = tf32r(s_mrow[lr][c - DQ]);
        } else if (c == DQ + D) {
            v = 1.f;
        }
        sM[(std::size_t)lr * ldm + c] = v;
    }
    __syncthreads();
    float acc[3][kNTW][4];
    // ---- F2: O = [ctx | 1] W_o^T -> m_in[:, :DQ] (0 for roots without neighbours)
    gemm48<true>(acc, sA, ldo, h.Wo, h.ldo, DQ, Ko);
    for_acc(acc, DQ, [&](int r, int c, float v) {
        sM[(std::size_t)r * ldm + c] = s_has[r] ? tf32r(v) : 0.f;
    });
    __syncthreads();
    for (int i = threadIdx.x; i < kRows * (DQ + D); i += blockDim.x) {  // m_in for the W_m1 gradient
        const int lr = i / (DQ + D), c = i % (DQ + D);
        if (valid(lr)) h.m_in[(std::size_t)grow(lr) * d.ld_m + c] = sM[(std::size_t)lr * ldm + c];
    }
    // ---- F3: Z1 = relu(m_in W_m1^T) -> [Z1 | 1 | 0]
    gemm48<true>(acc, sM, ldm, h.Wm1, h.ldm1, D, Km);
    for_acc(acc, D, [&](int r, int c, float v) { sZ[(std::size_t)r * ldz + c] = tf32r(fmaxf(v, 0.f)); });
    for (int i = threadIdx.x; i < kRows * (pad8(D + 1) + 32 - D); i += blockDim.x) {
        const int lr = i / (pad8(D + 1) + 32 - D), c = D + i % (pad8(D + 1) + 32 - D);
        if (c < ldz) sZ[(std::size_t)lr * ldz + c] = c == D ? 1.f : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kRows * D; i += blockDim.x) {
        const int lr = i / D, c = i % D;
        if (valid(lr)) h.Z1[(std::size_t)grow(lr) * d.ld_z + c] = sZ[(std::size_t)lr * ldz + c];
    }
    // ---- F4: emb = [Z1 | 1] W_m2^T (fp32 out, feeds the FFMA decoder)
    gemm48<true>(acc, sZ, ldz, h.Wm2, h.ldm2, D, D + 1);
    for_acc(acc, D, [&](int r, int c, float v) { sE[(std::size_t)r * D + c] = v; });
    __syncthreads();  // sA | sM are free from here: stage the decoder weights there
    for (int i = threadIdx.x; i < kRows * D; i += blockDim.x) {
        const int lr = i / D, c = i % D;
        if (valid(lr)) h.emb[(std::size_t)grow(lr) * D + c] = sE[(std::size_t)lr * D + c];
    }
    for (int i = threadIdx.x; i < D * (2 * D + 1); i += blockDim.x) {
        const int n = i / (2 * D + 1), c = i % (2 * D + 1);
        sW1[i] = h.Wd1[(std::size_t)n * h.ldd1 + c];  // [W_a | W_b | b1] row n (odd stride)
    }
    __syncthreads();
    // ---- F5 (FFMA): Y = [z_src W_a^T ; z_{dst|neg} W_b^T] (48 x D, into sdE), then
    //      D1[p] = relu(Y_src[p % 16] + Y_other[p] + b1), p < 16 pos, >= 16 neg
    const int ld1 = 2 * D + 1;
    ffma48(sE, D, D, D, [&](int k, int c, int row) { return sW1[(std::size_t)c * ld1 + (row < kEB ? 0 : D) + k]; },
           [&](int row, int c, float v) { sdE[(std::size_t)row * ldz + c] = v; });
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * kEB * D; i += blockDim.x) {
        const int p = i / D, n = i % D;
        const float v = sdE[(std::size_t)(p % kEB) * ldz + n] + sdE[(std::size_t)(kEB + p) * ldz + n] +
                        sW1[(std::size_t)n * ld1 + 2 * D];
        sD1[(std::size_t)p * (D + 1) + n] = fmaxf(v, 0.f);
    }
    __syncthreads();
    // ---- F6 (FFMA): logits, BCE terms, dlogit, dD1 = [D1 > 0] g w2 (one warp per pair row)
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int p = warp; p < 2 * kEB; p += kWarps) {
            const int e = p % kEB;
            const bool ok = i0 + e < B;
            const float* x = sD1 + (std::size_t)p * (D + 1);
            float s = 0.f;
            for (int c = lane; c < D; c += 32) s += x[c] * h.wd2[c];
            s = warp_sum(s) + h.wd2[D];
            const bool pos = p < kEB;
            const float sig = sigmoidf_(s);
            const float g = ok ? (sig - (pos ? 1.f : 0.f)) / (float)B : 0.f;
            const int gp = (pos ? 0 : B) + i0 + e;  // row in the [pos | neg] decoder layout
            if (lane == 0) {
                sg[p] = g;
                if (ok) {
                    h.dlogit[(std::size_t)gp * 4] = g;
                    h.lossv[gp] = (pos ? softplusf_(-s) : softplusf_(s)) / (float)B;
                    if (h.logits) h.logits[gp] = s;
                }
            }
            for (int c = lane; c < D; c += 32) {
                const float dv = x[c] > 0.f ? g * h.wd2[c] : 0.f;
                sdD1[(std::size_t)p * (D + 1) + c] = dv;
                if (ok) {
                    h.D1[(std::size_t)gp * d.ld_d1 + c] = x[c];
                    h.dD1[(std::size_t)gp * D + c] = dv;
                }
            }
        }
    }
    __syncthreads();
    // ---- B1 (FFMA): d_emb = dD1 W_d1 by halves: src (pos + neg) W_a, dst pos W_b,
    //      neg neg W_b; the per-row dD1 combination staged in sdZ first
    for (int i = threadIdx.x; i < kRows * D; i += blockDim.x) {
        const int lr = i / D, n = i % D, e = lr % kEB, kind = lr / kEB;
        const float gp = sdD1[(std::size_t)e * (D + 1) + n], gn = sdD1[(std::size_t)(kEB + e) * (D + 1) + n];
        sdZ[(std::size_t)lr * ldz + n] = kind == 0 ? gp + gn : kind == 1 ? gp : gn;
    }
    __syncthreads();
    ffma48(sdZ, ldz, D, D, [&](int n, int c, int row) { return sW1[(std::size_t)n * ld1 + (row < kEB ? 0 : D) + c]; },
           [&](int lr, int c, float a) {
               a = valid(lr) ? tf32r(a) : 0.f;
               sdE[(std::size_t)lr * ldz + c] = a;
               if (valid(lr)) h.d_emb[(std::size_t)grow(lr) * D + c] = a;
           });
    zero_cols(sdE, ldz, D, (D + 31) / 32 * 32);
    __syncthreads();
    // ---- B2: dZ1 = (d_emb W_m2) * [Z1 > 0]
    gemm48<false>(acc, sdE, ldz, h.Wm2, h.ldm2, D, D);
    for_acc(acc, D, [&](int r, int c, float v) {
        const float x = sZ[(std::size_t)r * ldz + c] > 0.f ? tf32r(v) : 0.f;
        sdZ[(std::size_t)r * ldz + c] = x;
        if (valid(r)) h.dZ1[(std::size_t)grow(r) * D + c] = x;
    });
    zero_cols(sdZ, ldz, D, (D + 31) / 32 * 32);
    __syncthreads();
    // ---- B3: dm_in = dZ1 W_m1 (O part 0 for roots without neighbours) -> sA (O part), global
    gemm48<false>(acc, sdZ, ldz, h.Wm1, h.ldm1, DQ + D, D);
    for_acc(acc, DQ + D, [&](int r, int c, float v) {
        const bool ok = valid(r);
        const float x = (c < DQ && !s_has[r]) ? 0.f : tf32r(v);
        if (c < DQ) sA[(std::size_t)r * ldo + c] = x;
        if (ok) h.dm_in[(std::size_t)grow(r) * d.ld_m + c] = x;
    });
    zero_cols(sA, ldo, DQ, (DQ + 31) / 32 * 32);
    __syncthreads();
    // ---- B4: dctx = dm_in[:, :DQ] W_o[:, :DQ]
    gemm48<false>(acc, sA, ldo, h.Wo, h.ldo, DQ, DQ);
    for_acc(acc, DQ, [&](int r, int c, float v) {
        if (valid(r)) h.dctx[(std::size_t)grow(r) * d.ld_Q + c] = tf32r(v);
    });
}

int head_events_per_block() { return kEB; }

}  // namespace tgnk
}  // namespace spd
