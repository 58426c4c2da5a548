// tcgen05 (5th-gen tensor core) TF32 GEMM for sm_100a, used for the GRU and
// attention projection GEMMs (the tensor-core-eligible ones).
//
//   C[M,N] (=|+=) A . B,  fp32 operands in global memory, fp32 accumulate in TMEM
//
// Operand majorness is a template parameter so one kernel serves
//   forward     A = X [M,K] K-major,   B = W [N,K] K-major
//   data grad   A = dY [M,K] K-major,  B = W [K,N] MN-major
//   weight grad A = dY^T (dY [K,M])    MN-major, B = X [K,N] MN-major
// without materialising transposes.
//
// Structure (one 128 x BN output tile per CTA, 6 warps):
//   warp 0  one lane issues TMA loads (SWIZZLE_128B boxes) into a 4-stage ring
//   warp 1  one lane issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) and
//           commits each stage back to the producer through an mbarrier
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> registers -> global (store,
//           accumulate, relu, mask, or split-K partial)
// Shared-memory canonical layouts (16-byte units, cute/arch/mma_sm100_desc.hpp):
//   K-major SW128 : rows of 128 B, 8-row atoms of 1024 B  (SBO = 1024 B)
//   MN-major SW128: K-rows of 128 B (32 fp32 along M/N), 8-row atoms of 1024 B
//                   (SBO = 1024 B), 32-column blocks LBO = BK*128 B apart.
#pragma once

#include "pdl.cuh"
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spd {
namespace umma {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 per 128-B swizzle row / K rows per stage
constexpr int STAGES = 4;
constexpr int THREADS = 192;

enum Mode : int { STORE = 0, ACCUM = 1, PARTIAL = 2 };
enum Epi : int { EPI_NONE = 0, EPI_RELU = 1, EPI_MASK = 2, EPI_ROWMASK = 3 /* gemm_simt.cuh */ };

struct Args {
    float* C;
    int ldc;
    int M, N, K;
    const int* M_dev;  // optional device row count (forward / data grad)
    const int* K_dev;  // optional device reduction count (weight grad)
    int k_split;
    int mode;
    int epi;
    const float* mask;
    int ldmask;
    float* ws;  // PARTIAL: [batch][k_split][M][ldws]
    int ldws;
    int rnd;    // STORE: round outputs to tf32 (they feed another tensor-core GEMM)
    // batched GEMMs (blockIdx.z = batch * k_split + split): C of batch b at
    // C + b * c_bstride; operands through maps.a[b] / maps.b[b]
    int batch;
    long long c_bstride;
    // B is a parameter tensor (forward / data-gradient GEMMs): its first
    // stages are loaded before the PDL wait, overlapping the producer of A
    int b_static;
};

constexpr int kMaxBatch = 4;
struct Maps {
    CUtensorMap a[kMaxBatch];
    CUtensorMap b[kMaxBatch];
};

__device__ __forceinline__ float tf32_rn(float x) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// Shared-memory matrix descriptor (version 1 for sm_100). layout: 2 =
// SWIZZLE_128B (K-major operands), 1 = SWIZZLE_128B_BASE32B (the only layout
// MN-major tf32 operands support: 32-B swizzle atoms, 4-row K groups).
__device__ __forceinline__ std::uint64_t make_desc(std::uint32_t saddr, std::uint32_t lbo,
                                                   std::uint32_t sbo, std::uint64_t layout) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ULL << 46;  // descriptor version (sm_100)
    d |= layout << 61;
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M=128, N=bn.
__host__ __device__ constexpr std::uint32_t make_idesc(bool a_mn, bool b_mn, int bn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | (static_cast<std::uint32_t>(bn >> 3) << 17) |
           (static_cast<std::uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ std::uint32_t cluster_rank() {
    std::uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// TMA 2D load delivered to the same smem offset of every CTA in `mask`; each
// destination's mbarrier (same offset) receives the complete_tx.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, std::uint64_t* bar,
                                               int c0, int c1, std::uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

// BN: N of one MMA (tile sub-width); NSUB sub-tiles side by side in TMEM, so a
// CTA owns a 128 x (NSUB*BN) output tile and reads its A tile once. CL CTAs
// along M form a cluster and split the B tile's TMA boxes between them, each
// box multicast to all CL CTAs (B streamed from L2 once per cluster).
// DEEP: one CTA per SM with the ring as deep as shared memory allows (up to 8
// stages), so every k-block of a short-K GEMM is in flight at once — for
// grids of at most one wave.
template <bool A_MN, bool B_MN, int BN, int NSUB, int CL, bool DEEP = false>
struct Cfg {
    static constexpr int NT = BN * NSUB;
    static constexpr int A_BYTES = BM * BK * 4;  // 16 KB
    static constexpr int B_BYTES = NT * BK * 4;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // narrow tiles: 3 CTAs per SM (3 stages, <= 113 registers), so a CTA's
    // epilogue and its neighbours' TMA round trips overlap; wider: 2 per SM
    static constexpr int CTAS_PER_SM = DEEP ? 1 : NT <= 64 ? 3 : 2;
    static constexpr int BUDGET = (DEEP ? 227 * 1024 : NT <= 64 ? 75 * 1024 : 227 * 1024) - 1024 - 256;
    static constexpr int MAXST = DEEP ? 8 : STAGES;
    static constexpr int STAGES_ = BUDGET / STAGE_BYTES >= MAXST ? MAXST : BUDGET / STAGE_BYTES;
    static constexpr int SMEM = STAGES_ * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int TMEM_COLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : NT <= 256 ? 256 : 512;
    // TMA boxes per stage for B: 32-column blocks (MN-major) or row slabs of
    // KROWS rows (K-major; at least one per cluster CTA so the multicast load
    // is spread evenly)
    static constexpr int KBOXES = NSUB >= CL ? NSUB : CL;
    static constexpr int KROWS = NT / KBOXES;
    static constexpr int B_BOXES = B_MN ? NT / 32 : KBOXES;
    static_assert(B_MN || (NT % KBOXES == 0 && KROWS % 8 == 0), "K-major B slabs of 8-row atoms");
    static_assert(STAGES_ >= 2, "tile too large for the smem budget");
    static_assert(!B_MN || BN % 32 == 0, "MN-major B needs whole 32-column boxes");
    static_assert(NT <= 512, "accumulator exceeds TMEM");
};

template <bool A_MN, bool B_MN, int BN, int NSUB, int CL, bool DEEP = false>
__global__ void __launch_bounds__(THREADS, (DEEP ? 1 : BN * NSUB <= 64 ? 3 : 2))
    umma_gemm_kernel(const __grid_constant__ Maps maps, Args args) {
    pdl_launch();
    if (!args.b_static) pdl_wait();  // (else below, after the set-up and the weight prefetch)
    using C_ = Cfg<A_MN, B_MN, BN, NSUB, CL, DEEP>;
    constexpr int NST = C_::STAGES_;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B alignment (SWIZZLE_128B atoms) by offset, keeping shared-space provenance
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + NST * C_::STAGE_BYTES);
    std::uint64_t* empty = full + NST;
    std::uint64_t* tmem_full = empty + NST;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int M = args.M;
    if (args.M_dev) M = min(M, *args.M_dev);
    int K = args.K;
    if (args.K_dev) K = min(K, *args.K_dev);
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * C_::NT;
    const int bz = args.k_split > 1 ? blockIdx.z / args.k_split : blockIdx.z;  // batch index
    const int sz = args.k_split > 1 ? blockIdx.z % args.k_split : 0;          // split index
    const CUtensorMap* tmA = &maps.a[bz];
    const CUtensorMap* tmB = &maps.b[bz];
    // a lone CTA past the rows can leave; cluster members must stay to serve
    // their share of the multicast B tiles
    if (CL == 1 && m0 >= M) return;
    const std::uint32_t crank = CL > 1 ? cluster_rank() : 0;
    int k_begin = 0, k_end = K;
    if (args.k_split > 1) {
        const int per = ((K + args.k_split - 1) / args.k_split + BK - 1) / BK * BK;
        k_begin = sz * per;
        k_end = min(K, k_begin + per);
    }
    const int n_k = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, CL);  // every cluster CTA's MMA releases the stage
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (CL > 1) cluster_sync_all();  // peers' barriers exist before any multicast lands
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *tmem_slot;

    if (!(warp == 0 && lane == 0)) pdl_wait();
    if (warp == 0) {
        if (lane == 0) {
            // stage s: expect its bytes once, then the B boxes (this CTA's
            // share when multicast) and the A tile
            auto load_b = [&](int kb) {
                const int s = kb % NST;
                unsigned char* b_s = smem + s * C_::STAGE_BYTES + C_::A_BYTES;
                const int kc = k_begin + kb * BK;
                mbar_expect_tx(full + s, C_::STAGE_BYTES);
#pragma unroll
                for (int j = 0; j < C_::B_BOXES; ++j) {
                    if (CL > 1 && (j % CL) != (int)crank) continue;
                    unsigned char* dst = B_MN ? b_s + j * 32 * 128 : b_s + j * C_::KROWS * 128;
                    const int c0 = B_MN ? n0 + 32 * j : kc;
                    const int c1 = B_MN ? kc : n0 + j * C_::KROWS;
                    if (CL > 1) tma_load_2d_mc(dst, tmB, full + s, c0, c1, (1u << CL) - 1);
                    else tma_load_2d(dst, tmB, full + s, c0, c1);
                }
            };
            const int pre = args.b_static ? (n_k < NST ? n_k : NST) : 0;
            for (int kb = 0; kb < pre; ++kb) load_b(kb);
            pdl_wait();
            for (int kb = 0; kb < n_k; ++kb) {
                const int s = kb % NST;
                if (kb >= NST) mbar_wait(empty + s, ((kb / NST) - 1) & 1);
                if (kb >= pre) load_b(kb);
                unsigned char* a_s = smem + s * C_::STAGE_BYTES;
                const int kc = k_begin + kb * BK;
                if (!A_MN) {
                    tma_load_2d(a_s, tmA, full + s, kc, m0);
                } else {
#pragma unroll
                    for (int j = 0; j < BM / 32; ++j) tma_load_2d(a_s + j * 32 * 128, tmA, full + s, m0 + 32 * j, kc);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr std::uint32_t idesc = make_idesc(A_MN, B_MN, BN);
            for (int kb = 0; kb < n_k; ++kb) {
                const int s = kb % NST;
                mbar_wait(full + s, (kb / NST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const std::uint32_t a_base = smem_u32(smem + s * C_::STAGE_BYTES);
                const std::uint32_t b_base = a_base + C_::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    // K-major: 128-B rows, 8-row atoms (SBO 1024), K=8 step = 32 B in-row.
                    // MN-major: 128-B K-rows, 4-row groups (SBO 512), 32-column blocks
                    // BK*128 B apart (LBO), K=8 step = 8 rows = 1024 B.
                    const std::uint64_t ad = A_MN ? make_desc(a_base + kk * 1024, BK * 128, 512, 1)
                                                  : make_desc(a_base + kk * 32, 16, 1024, 2);
                    const std::uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
                    for (int t = 0; t < NSUB; ++t) {
                        const std::uint32_t bt = B_MN ? b_base + t * (BN / 32) * (BK * 128)
                                                      : b_base + t * BN * 128;
                        const std::uint64_t bd = B_MN ? make_desc(bt + kk * 1024, BK * 128, 512, 1)
                                                      : make_desc(bt + kk * 32, 16, 1024, 2);
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "setp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                                tmem + t * BN),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                }
                if (CL > 1)
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster"
                        ".multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(empty + s)),
                        "h"(static_cast<std::uint16_t>((1u << CL) - 1))
                        : "memory");
                else
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(empty + s))
                        : "memory");
            }
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(tmem_full))
                : "memory");
        }
    } else {
        // epilogue warps 2..5 -> TMEM lanes 32*(warp%4) ..
        // TMEM -> registers (32 columns of this lane's row) -> smem transpose ->
        // coalesced 128-B row segments to global. The stage ring is idle once
        // tmem_full fires, so warp q stages through stage memory [q*32][33].
        const int quad = warp & 3;
        const int row0 = m0 + quad * 32;
        float* stage = reinterpret_cast<float*>(smem) + quad * 32 * 33;
        if (n_k > 0) {
            mbar_wait(tmem_full, 0);
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const bool partial = args.mode == PARTIAL;
        float* const C = args.C + bz * args.c_bstride;
        float* const ws_b = partial ? args.ws + (std::size_t)bz * args.k_split * args.M * args.ldws : nullptr;
        float* out_base = partial ? ws_b + (std::size_t)sz * args.M * args.ldws : C;
        const int ldo = partial ? args.ldws : args.ldc;
#pragma unroll 1
        for (int c0 = 0; c0 < C_::NT; c0 += 32) {
            if (n0 + c0 >= args.N) break;
            std::uint32_t v[32];
            if (n_k > 0) {
                const std::uint32_t taddr = tmem + (static_cast<std::uint32_t>(quad * 32) << 16) + c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                    "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31},"
                    " [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                      "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                      "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                      "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                      "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                      "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0u;
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) stage[lane * 33 + j] = __uint_as_float(v[j]);
            __syncwarp();
            const int col = n0 + c0 + lane;
            const int rows = min(32, M - row0);
            unsigned zero_rows = 0;  // EPI_ROWMASK: rows of this warp's slab with count 0
            if (args.epi == EPI_ROWMASK)
                zero_rows = __ballot_sync(0xffffffffu, lane < rows &&
                                                           reinterpret_cast<const int*>(args.mask)[row0 + lane] == 0);
            if (col < args.N && rows > 0) {
                float* c = out_base + (std::size_t)row0 * ldo + col;
                // mode/epilogue are CTA-uniform: branch once, keep the plain
                // store path free of loads
                if (partial || (args.mode == STORE && args.epi == EPI_NONE && !args.rnd)) {
#pragma unroll 8
                    for (int r = 0; r < rows; ++r) c[(std::size_t)r * ldo] = stage[r * 33 + lane];
                } else if (args.mode == STORE && args.epi == EPI_NONE) {
#pragma unroll 8
                    for (int r = 0; r < rows; ++r) c[(std::size_t)r * ldo] = tf32_rn(stage[r * 33 + lane]);
                } else if (args.mode == ACCUM) {
                    // all 32 read-modify-write loads in flight before any use
                    float cv[32];
#pragma unroll
                    for (int r = 0; r < 32; ++r) cv[r] = r < rows ? c[(std::size_t)r * ldo] : 0.f;
#pragma unroll
                    for (int r = 0; r < 32; ++r)
                        if (r < rows) c[(std::size_t)r * ldo] = cv[r] + stage[r * 33 + lane];
                } else if (args.epi == EPI_ROWMASK) {
                    // rows whose count is 0 are zero in the columns < ldmask
                    const bool masked_col = col < args.ldmask;
#pragma unroll 8
                    for (int r = 0; r < rows; ++r) {
                        const bool z = masked_col && ((zero_rows >> r) & 1u);
                        const float x = z ? 0.f : stage[r * 33 + lane];
                        c[(std::size_t)r * ldo] = args.rnd ? tf32_rn(x) : x;
                    }
                } else if (args.epi == EPI_RELU) {
#pragma unroll 8
                    for (int r = 0; r < rows; ++r) {
                        const float x = fmaxf(stage[r * 33 + lane], 0.f);
                        c[(std::size_t)r * ldo] = args.rnd ? tf32_rn(x) : x;
                    }
                } else {  // EPI_MASK: prefetch the 32 mask values, then store
                    const float* mk = args.mask + (std::size_t)row0 * args.ldmask + col;
                    float mv[32];
#pragma unroll
                    for (int r = 0; r < 32; ++r) mv[r] = r < rows ? mk[(std::size_t)r * args.ldmask] : 0.f;
#pragma unroll
                    for (int r = 0; r < 32; ++r)
                        if (r < rows) {
                            const float x = mv[r] > 0.f ? stage[r * 33 + lane] : 0.f;
                            c[(std::size_t)r * ldo] = args.rnd ? tf32_rn(x) : x;
                        }
                }
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (CL > 1) cluster_sync_all();  // no CTA leaves while peers may still signal it
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(C_::TMEM_COLS));
}

}  // namespace umma
}  // namespace spd
