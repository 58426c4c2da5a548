// FP32 FFMA tiled GEMM for sm_100a (the tolerance-safe path; SURVEY K4/K6
// "otherwise use FP32 FFMA"; the merge and decoder layers always use it).
// One kernel template covers the three orientations a hand-written backward
// needs:
//
//   fwd         C[M,N]  = A[M,K]   . B[N,K]^T      (A row-major, B row-major)
//   data grad   C[M,N]  = A[M,K]   . B[K,N]        (B row-major)
//   weight grad C[M,N] += A[K,M]^T . B[K,N]        (reduction over K = rows, split-K)
//
// Every linear layer stores its bias as an extra weight column (augmented
// [W | b]) and every activation matrix carries a constant-1 column, so the
// bias gradient falls out of the weight-gradient GEMM. Leading dimensions are
// multiples of 4 floats and allocations are padded to them, so 128-bit loads
// along the contiguous dimension are always in bounds; only the reduction
// index is predicated (rows past a device-resident count read 0).
//
// Tile BM x 64 x BK (BK = 32 for BM = 64, 16 for BM = 128; BM = 128 or 64: the launcher picks 64 when 128-row tiles
// would leave SMs idle), 256 threads, (BM/16) x 4 outputs per thread,
// register-staged double buffering through shared memory. BK = 32 halves the
// k-tile count (one L2 round trip each) against 16: these GEMMs have K ~ 200
// and too few CTAs to hide a round trip per 16 k-steps.
#pragma once

#include "pdl.cuh"
#include <cuda_runtime.h>

#include <cstdint>

namespace spd {
namespace gemm {

constexpr int BN = 64, NT = 256, TN = 4;

enum Epi : int {
    EPI_NONE = 0,
    EPI_RELU = 1,
    EPI_MASK = 2,    // C *= (mask > 0)
    EPI_ROWMASK = 3  // C = 0 in columns < ldmask of rows with ((const int*) mask)[row] == 0
};

struct Args {
    const float* A;
    const float* B;
    float* C;
    int M, N, K;
    int lda, ldb, ldc;
    const int* M_dev;  // optional device-resident row count (min with M)
    const int* K_dev;  // optional device-resident reduction count (TN mode)
    float beta;        // 0: overwrite, 1: accumulate
    int epi;
    const float* mask;  // EPI_MASK: same shape/ld as C
    int ldmask;
    // split-K for the weight-gradient orientation
    int k_split;        // number of K slices (gridDim.z)
    float* workspace;   // [k_split][M][N] partials (ld = ldw)
    int ldw;
};

// A_KMAJOR: A stored [K x M] (weight-grad orientation). B_KN: B stored [K x N].
// BNT: tile width (64, or 32 for small problems: twice the CTAs, so a
// 4000 x 100 decoder GEMM fills the 148 SMs). Thread (tx, ty) owns rows
// ty*TM.. and columns tx*4..; every output still sums k in order.
template <bool A_KMAJOR, bool B_KN, int BM, int BNT = BN>
__global__ void __launch_bounds__(NT) gemm_kernel(Args a) {
    pdl_entry();
    constexpr int BK = BM >= 128 ? 16 : 32;  // static shared memory <= 48 KB
    constexpr int TX = BNT / 4, TY = NT / TX;
    constexpr int TM = BM / TY;       // rows per thread
    constexpr int AV = BM * BK / 4 / NT;  // float4 A loads per thread (2 or 1)
    constexpr int BV = BK * BNT / 4;      // float4 B loads per tile (threads < BV)
    static_assert(TM == 2 || TM % 4 == 0, "rows per thread");
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Bs[2][BK][BNT + 4];
    int M = a.M;
    if (a.M_dev) M = min(M, *a.M_dev);
    int K = a.K;
    if (a.K_dev) K = min(K, *a.K_dev);
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BNT;
    if (!A_KMAJOR && m0 >= M) return;
    if (n0 >= a.N) return;
    if (A_KMAJOR && m0 >= a.M) return;
    int k_begin = 0, k_end = K;
    if (a.k_split > 1) {
        const int per = ((K + a.k_split - 1) / a.k_split + BK - 1) / BK * BK;
        k_begin = blockIdx.z * per;
        k_end = min(K, k_begin + per);
    }
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;  // outputs (ty*TM.., tx*4..)

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    constexpr int BVT = (BV + NT - 1) / NT;  // float4 B loads per thread
    float4 ra[AV], rb[BVT];
    auto zero_tail = [&](float4& v, int gk) {
        if (gk + 3 >= k_end) {
            if (gk + 0 >= k_end) v.x = 0.f;
            if (gk + 1 >= k_end) v.y = 0.f;
            if (gk + 2 >= k_end) v.z = 0.f;
            if (gk + 3 >= k_end) v.w = 0.f;
        }
    };
    constexpr int KQ = BK / 4;  // float4 per BK-long row segment
    auto load_tiles = [&](int k0) {
#pragma unroll
        for (int r = 0; r < AV; ++r) {
            const int idx = tid + r * NT;
            if (!A_KMAJOR) {  // BM rows x BK k
                const int row = idx / KQ, kq = (idx % KQ) * 4;
                const int gm = m0 + row, gk = k0 + kq;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (gm < a.M && gk < k_end) v = *reinterpret_cast<const float4*>(a.A + (size_t)gm * a.lda + gk);
                zero_tail(v, gk);
                ra[r] = v;
            } else {  // BK k-rows x BM m
                const int kr = idx / (BM / 4), mq = (idx % (BM / 4)) * 4;
                const int gk = k0 + kr, gm = m0 + mq;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (gk < k_end && gm < a.M) v = *reinterpret_cast<const float4*>(a.A + (size_t)gk * a.lda + gm);
                ra[r] = v;
            }
        }
#pragma unroll
        for (int r = 0; r < BVT; ++r) {
            const int idx = tid + r * NT;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (idx < BV) {
                if (B_KN) {  // BK k-rows x BNT n
                    const int kr = idx / TX, nq = (idx % TX) * 4;
                    const int gk = k0 + kr, gn = n0 + nq;
                    if (gk < k_end && gn < a.N) v = *reinterpret_cast<const float4*>(a.B + (size_t)gk * a.ldb + gn);
                } else {  // BNT n-rows x BK k
                    const int row = idx / KQ, kq = (idx % KQ) * 4;
                    const int gn = n0 + row, gk = k0 + kq;
                    if (gn < a.N && gk < k_end) v = *reinterpret_cast<const float4*>(a.B + (size_t)gn * a.ldb + gk);
                    zero_tail(v, gk);
                }
            }
            rb[r] = v;
        }
    };
    auto store_tiles = [&](int buf) {
#pragma unroll
        for (int r = 0; r < AV; ++r) {
            const int idx = tid + r * NT;
            if (!A_KMAJOR) {
                const int row = idx / KQ, kq = (idx % KQ) * 4;
                As[buf][kq + 0][row] = ra[r].x;
                As[buf][kq + 1][row] = ra[r].y;
                As[buf][kq + 2][row] = ra[r].z;
                As[buf][kq + 3][row] = ra[r].w;
            } else {
                const int kr = idx / (BM / 4), mq = (idx % (BM / 4)) * 4;
                *reinterpret_cast<float4*>(&As[buf][kr][mq]) = ra[r];
            }
        }
#pragma unroll
        for (int r = 0; r < BVT; ++r) {
            const int idx = tid + r * NT;
            if (idx >= BV) continue;
            if (B_KN) {
                const int kr = idx / TX, nq = (idx % TX) * 4;
                *reinterpret_cast<float4*>(&Bs[buf][kr][nq]) = rb[r];
            } else {
                const int row = idx / KQ, kq = (idx % KQ) * 4;
                Bs[buf][kq + 0][row] = rb[r].x;
                Bs[buf][kq + 1][row] = rb[r].y;
                Bs[buf][kq + 2][row] = rb[r].z;
                Bs[buf][kq + 3][row] = rb[r].w;
            }
        }
    };

    if (k_begin < k_end) {
        load_tiles(k_begin);
        store_tiles(0);
        __syncthreads();
        int buf = 0;
        for (int k0 = k_begin; k0 < k_end; k0 += BK) {
            const bool more = k0 + BK < k_end;
            if (more) load_tiles(k0 + BK);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float av[TM];
                if constexpr (TM == 2) {
                    const float2 t = *reinterpret_cast<const float2*>(&As[buf][kk][ty * TM]);
                    av[0] = t.x; av[1] = t.y;
                } else {
#pragma unroll
                    for (int q = 0; q < TM; q += 4) {
                        const float4 t = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + q]);
                        av[q] = t.x; av[q + 1] = t.y; av[q + 2] = t.z; av[q + 3] = t.w;
                    }
                }
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
                const float bv[4] = {b0.x, b0.y, b0.z, b0.w};
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            if (more) {
                store_tiles(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }

    const int Mlim = A_KMAJOR ? a.M : M;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int gm = m0 + ty * TM + i;
        if (gm >= Mlim) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= a.N) continue;
            float v = acc[i][j];
            if (a.k_split > 1) {
                a.workspace[((size_t)blockIdx.z * a.M + gm) * a.ldw + gn] = v;
                continue;
            }
            if (a.epi == EPI_RELU) v = fmaxf(v, 0.f);
            if (a.epi == EPI_MASK) v = a.mask[(size_t)gm * a.ldmask + gn] > 0.f ? v : 0.f;
            if (a.epi == EPI_ROWMASK && gn < a.ldmask && reinterpret_cast<const int*>(a.mask)[gm] == 0) v = 0.f;
            float* c = a.C + (size_t)gm * a.ldc + gn;
            if (a.beta != 0.f) v += *c;
            *c = v;
        }
    }
}

// Fixed-order reduction of split-K partials into C (deterministic).
static __global__ void splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, int ldw,
                                     float* __restrict__ C, int ldc, float beta) {
    pdl_entry();
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)M * N) return;
    const int m = idx / N, n = idx % N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[((size_t)z * M + m) * ldw + n];
    float* c = C + (size_t)m * ldc + n;
    *c = beta != 0.f ? *c + s : s;
}

}  // namespace gemm
}  // namespace spd
