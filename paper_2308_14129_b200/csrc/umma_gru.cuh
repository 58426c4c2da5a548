// Fused GRU memory updater on the 5th-gen tensor cores (gemm_mode 1): both
// gate GEMMs of a GRUCell and the cell itself in one kernel —
//
//   Gi = [x | 1] [W_ih | b_ih]^T,  Gh = [h | 1] [W_hh | b_hh]^T      tcgen05 TF32, TMEM
//   r = sigmoid(Gi_r + Gh_r), z = sigmoid(Gi_z + Gh_z)
//   n = tanh(Gi_n + r Gh_n),  h' = (1 - z) n + z h                    epilogue (FP32)
//
// (PyTorch GRUCell gate order, oracle/tgn_oracle.py TGNOracle._gru). A CTA owns
// 128 pending rows x UB memory units: its B tile stacks the UB rows of each
// gate block of W (r, z, n: three TMA boxes per k-block), so ONE
// M=128 x N=3UB MMA per k-step yields all three gates of its units, and the
// two accumulators (input side, hidden side) sit side by side in TMEM. The
// epilogue warps read both from TMEM (tcgen05.ld) and write h' and the gate
// values the backward needs (r, z, n, Gh_n) — Gi and Gh never reach HBM, and
// the separate cell kernel (k_gru_fwd) and its launch disappear.
//
// Same pipeline as umma_gemm.cuh (warp 0 TMA producer over a STAGES ring,
// warp 1 single-thread MMA issuer, warps 2-5 epilogue); the K loop runs the
// x blocks into accumulator 0, then the h blocks into accumulator 1.
#pragma once

#include "umma_gemm.cuh"

namespace spd {
namespace umma {

constexpr int kGruUB = 32;  // memory units per CTA (SPD_GRU_UB=16: twice the CTAs, two per SM)

struct GruArgs {
    int M;             // row capacity (pending slots); live rows from *M_dev
    const int* M_dev;  // *w.nU
    int K1, K2;        // augmented input widths of x and h (bias column included)
    int D;
    const float* mem;            // exact h rows (w.mem), indexed by node id
    const std::uint32_t* nodes;  // pending node id per row (w.pU)
    float* mem_new;              // [M][D]
    float* save;                 // [M][4D]: r | z | n | Gh_n, or null (no backward)
    int prefetch;                // issue the first stages' weight tiles before the PDL wait
};
struct GruMaps {
    CUtensorMap x, h, wih, whh;
};

template <int UB>
struct GruCfg {
    static constexpr int N = 3 * UB;  // one MMA covers the three gates of UB units
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = N * BK * 4;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // UB 32: a 7-stage (196 KB) ring, one CTA per SM (<= 128 CTAs at the
    // step's sizes, all in flight); UB 16: 4 stages, two CTAs per SM
    static constexpr int CTAS = UB >= 32 ? 1 : 2;
    static constexpr int STAGES = UB >= 32 ? 7 : 4;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int ACC_H = N <= 128 ? 128 : 256;  // TMEM column of the hidden-side accumulator
    static constexpr int TMEM_COLS = 2 * ACC_H;
    static_assert(N % 16 == 0 && N <= 256, "MMA N");
};

__device__ __forceinline__ void tmem_ld8(std::uint32_t taddr, float (&v)[8]) {
    std::uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}

template <int UB>
__global__ void __launch_bounds__(THREADS, GruCfg<UB>::CTAS) umma_gru_kernel(const __grid_constant__ GruMaps maps, GruArgs args) {
    // PDL: the set-up (barriers, TMEM) and the first stages' weight tiles
    // (parameters and the pending count, both final before this step's graph
    // began) overlap the gather kernel's tail; the gathered rows wait
    pdl_launch();
    if (!args.prefetch) pdl_wait();
    using C_ = GruCfg<UB>;
    constexpr int NST = C_::STAGES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + NST * C_::STAGE_BYTES);
    std::uint64_t* empty = full + NST;
    std::uint64_t* tmem_full = empty + NST;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int M = args.M;
    if (args.M_dev) M = min(M, *args.M_dev);
    const int m0 = blockIdx.y * BM, u0 = blockIdx.x * UB;
    if (m0 >= M) return;
    const int nk1 = (args.K1 + BK - 1) / BK, nk2 = (args.K2 + BK - 1) / BK, n_k = nk1 + nk2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
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
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *tmem_slot;

    if (!(warp == 0 && lane == 0)) pdl_wait();
    if (warp == 0) {
        if (lane == 0) {
            auto weights = [&](int kb) {
                const int s = kb % NST;
                unsigned char* b_s = smem + s * C_::STAGE_BYTES + C_::A_BYTES;
                mbar_expect_tx(full + s, C_::STAGE_BYTES);
                const bool hid = kb >= nk1;
                const int kc = (hid ? kb - nk1 : kb) * BK;
#pragma unroll
                for (int g = 0; g < 3; ++g)  // gate blocks r, z, n of W: rows g*D + u0 ..
                    tma_load_2d(b_s + g * UB * 128, hid ? &maps.whh : &maps.wih, full + s, kc,
                                g * args.D + u0);
            };
            const int pre = args.prefetch ? (n_k < NST ? n_k : NST) : 0;
            for (int kb = 0; kb < pre; ++kb) weights(kb);
            pdl_wait();
            for (int kb = 0; kb < n_k; ++kb) {
                const int s = kb % NST;
                if (kb >= NST) mbar_wait(empty + s, ((kb / NST) - 1) & 1);
                if (kb >= pre) weights(kb);
                unsigned char* a_s = smem + s * C_::STAGE_BYTES;
                const bool hid = kb >= nk1;
                const int kc = (hid ? kb - nk1 : kb) * BK;
                tma_load_2d(a_s, hid ? &maps.h : &maps.x, full + s, kc, m0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr std::uint32_t idesc = make_idesc(false, false, C_::N);
            for (int kb = 0; kb < n_k; ++kb) {
                const int s = kb % NST;
                mbar_wait(full + s, (kb / NST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const std::uint32_t a_base = smem_u32(smem + s * C_::STAGE_BYTES);
                const std::uint32_t b_base = a_base + C_::A_BYTES;
                const bool hid = kb >= nk1;
                const std::uint32_t acc_col = hid ? C_::ACC_H : 0;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const std::uint64_t ad = make_desc(a_base + kk * 32, 16, 1024, 2);
                    const std::uint64_t bd = make_desc(b_base + kk * 32, 16, 1024, 2);
                    const std::uint32_t acc = ((hid ? kb > nk1 : kb > 0) || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + acc_col),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
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
        // epilogue: warp q reads TMEM lanes 32 (q % 4) .. (its 32 rows); each
        // thread one row, 8 units at a time: 6 x 8 accumulator values
        const int quad = warp & 3;
        const int row = m0 + quad * 32 + lane;
        const bool live = row < M;
        const int D = args.D;
        // the row's exact h values (a gather from the memory store) are loaded
        // while the MMAs run, not after
        float hall[UB];
        {
            const float* hrow = live ? args.mem + (std::size_t)args.nodes[row] * D : nullptr;
#pragma unroll
            for (int j = 0; j < UB; j += 4) {
                if (live && u0 + j + 4 <= D) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(hrow + u0 + j));
                    hall[j] = v.x; hall[j + 1] = v.y; hall[j + 2] = v.z; hall[j + 3] = v.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) hall[j + q] = live && u0 + j + q < D ? hrow[u0 + j + q] : 0.f;
                }
            }
        }
        mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c0 = 0; c0 < UB; c0 += 8) {
            if (u0 + c0 >= D) break;
            const std::uint32_t base = tmem + (static_cast<std::uint32_t>(quad * 32) << 16) + c0;
            float ir[8], iz[8], in_[8], hr[8], hz[8], hn[8];
            tmem_ld8(base, ir);
            tmem_ld8(base + UB, iz);
            tmem_ld8(base + 2 * UB, in_);
            tmem_ld8(base + C_::ACC_H, hr);
            tmem_ld8(base + C_::ACC_H + UB, hz);
            tmem_ld8(base + C_::ACC_H + 2 * UB, hn);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (!live) continue;
            float o[8], rr[8], zz[8], nn[8];
            const float* hv = hall + c0;
            const int u = u0 + c0;
            const bool full8 = u + 8 <= D;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                rr[j] = 1.f / (1.f + expf(-(ir[j] + hr[j])));
                zz[j] = 1.f / (1.f + expf(-(iz[j] + hz[j])));
                nn[j] = tanhf(in_[j] + rr[j] * hn[j]);
                o[j] = (1.f - zz[j]) * nn[j] + zz[j] * hv[j];
            }
            float* mo = args.mem_new + (std::size_t)row * D + u;
            float* sv = args.save ? args.save + (std::size_t)row * 4 * D + u : nullptr;
            if (full8) {
                reinterpret_cast<float4*>(mo)[0] = make_float4(o[0], o[1], o[2], o[3]);
                reinterpret_cast<float4*>(mo)[1] = make_float4(o[4], o[5], o[6], o[7]);
                if (sv) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        reinterpret_cast<float4*>(sv)[h] = make_float4(rr[4 * h], rr[4 * h + 1], rr[4 * h + 2], rr[4 * h + 3]);
                        reinterpret_cast<float4*>(sv + D)[h] = make_float4(zz[4 * h], zz[4 * h + 1], zz[4 * h + 2], zz[4 * h + 3]);
                        reinterpret_cast<float4*>(sv + 2 * D)[h] = make_float4(nn[4 * h], nn[4 * h + 1], nn[4 * h + 2], nn[4 * h + 3]);
                        reinterpret_cast<float4*>(sv + 3 * D)[h] = make_float4(hn[4 * h], hn[4 * h + 1], hn[4 * h + 2], hn[4 * h + 3]);
                    }
                }
            } else {
                for (int j = 0; j < 8 && u + j < D; ++j) {
                    mo[j] = o[j];
                    if (sv) {
                        sv[j] = rr[j];
                        sv[D + j] = zz[j];
                        sv[2 * D + j] = nn[j];
                        sv[3 * D + j] = hn[j];
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(C_::TMEM_COLS));
}

}  // namespace umma
}  // namespace spd
