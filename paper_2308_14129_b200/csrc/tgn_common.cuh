// Device/host-shared helpers of the TGN path: counter-based hashing (init,
// synthetic features, negatives — bit-identical on host, device and in the
// oracle, oracle/tgn_oracle.py), BF16-exact feature values, warp reductions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spd {

__host__ __device__ __forceinline__ std::uint64_t mix64(std::uint64_t x) {
    std::uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Feature column c of edge eid: ((h >> 56) - 128) / 128, exactly representable
// in bf16, so device storage in bf16 is lossless.
__host__ __device__ __forceinline__ float edge_feature_value(std::uint64_t seed_mixed,
                                                             std::uint64_t eid, std::uint32_t c) {
    const std::uint64_t h = mix64(mix64(seed_mixed ^ eid) ^ c);
    return static_cast<float>(static_cast<int>(h >> 56) - 128) * (1.0f / 128.0f);
}

// Negative-destination draw for (epoch, worker, step, i) (oracle: negatives()).
__host__ __device__ __forceinline__ std::uint64_t neg_base(std::uint64_t seed, std::uint64_t epoch,
                                                           std::uint64_t worker,
                                                           std::uint64_t step) {
    return mix64(mix64(mix64(mix64(seed) ^ epoch) ^ worker) ^ step);
}

// fp32 -> nearest tf32 (ties away; low 13 mantissa bits cleared). tcgen05
// kind::tf32 ignores those bits (truncation, a biased error that adds up
// coherently over a dot product); operands rounded here first are read exactly.
// shared-memory address, TMA bulk copies (global -> shared) and their mbarriers
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// one-instruction bulk copy global -> shared (TMA engine), completion counted
// in bytes on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void bar_init(std::uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ float tf32r(float x) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ float rnd_if(float x, int rnd) { return rnd ? tf32r(x) : x; }
__device__ __forceinline__ float4 rnd4_if(float4 v, int rnd) {
    return rnd ? make_float4(tf32r(v.x), tf32r(v.y), tf32r(v.z), tf32r(v.w)) : v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// Time encoder cos/sin(w*dt + b). The phase is formed in f64 (dt reaches
// ~2e8 at GDELT shape, beyond f32's 2^24) with explicitly rounded multiply and
// add (the oracle's f64 math), reduced to |r| <= pi/4 by the nearest multiple
// of pi/2 in f64 (two-term Cody-Waite, error ~q * 1e-32), and evaluated by
// f64 Taylor polynomials on [-pi/4, pi/4] (truncation < 4e-13) with the
// quadrant's sign/swap, then rounded to f32: the oracle's f64 cos rounded to
// f32 except in rare near-tie cases, without a libm call. Returns (sin, cos).
template <bool WANT_SIN = true>
__device__ __forceinline__ float2 phase_sincos(double w, double b, double dt) {
    const double ph = __dadd_rn(__dmul_rn(w, dt), b);
    constexpr double kTwoOverPi = 0.63661977236758134307553505349006;
    constexpr double kPiO2Hi = 1.5707963267948965580e+00;  // f64(pi/2)
    constexpr double kPiO2Lo = 6.1232339957367658e-17;      // pi/2 - kPiO2Hi
    const double q = rint(ph * kTwoOverPi);
    const double x = fma(-q, kPiO2Lo, fma(-q, kPiO2Hi, ph));
    const int quad = static_cast<int>(static_cast<long long>(q) & 3);
    const double z = x * x;
    // cos x = 1 - z/2! + z^2/4! - ... - z^7/14! ; sin x = x (1 - z/3! + ... + z^6/13!)
    const double c = fma(fma(fma(fma(fma(fma(fma(-1.1470745597729725e-11, z, 2.08767569878681e-09), z,
                                                 -2.755731922398589e-07), z, 2.48015873015873e-05), z,
                                         -1.388888888888889e-03), z, 4.1666666666666664e-02), z, -0.5), z, 1.0);
    double sn = 0.0;
    if (WANT_SIN || (quad & 1))
        sn = x * fma(fma(fma(fma(fma(fma(1.6059043836821613e-10, z, -2.505210838544172e-08), z,
                                     2.7557319223985893e-06), z, -1.984126984126984e-04), z,
                             8.333333333333333e-03), z, -1.6666666666666666e-01), z, 1.0);
    const float fs = static_cast<float>(sn), fc = static_cast<float>(c);
    switch (quad) {
        case 0: return make_float2(fs, fc);
        case 1: return make_float2(fc, -fs);
        case 2: return make_float2(-fs, -fc);
        default: return make_float2(-fc, fs);
    }
}
// The step's time encoder (every GPU evaluation goes through here): the same
// f64 phase as phase_sincos (explicitly rounded multiply and add, the
// oracle's f64 math) and an f64 reduction to |x| <= pi/4 (the quadrant from
// the low bits of a 1.5 * 2^52 shifter, two-term Cody-Waite), then f32
// minimax polynomials on [-pi/4, pi/4] (Cephes sinf / cosf coefficients,
// ~1 ulp): 6 f64 operations per value instead of ~22. The result is the
// oracle's f64 cos (sin) rounded to f32 within ~1-2 ulp; trajectories are
// insensitive at that level (perturbing every oracle cos by 1 ulp moves a
// 12-step trajectory by ~2e-6 relative, 1000x under the 2e-3 bar).
template <bool WANT_SIN, bool WANT_COS>
__device__ __forceinline__ float2 phase_sincos_fast(double w, double b, double dt) {
    const double ph = __dadd_rn(__dmul_rn(w, dt), b);
    constexpr double kTwoOverPi = 0.63661977236758134307553505349006;
    constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer shifter
    constexpr double kPiO2Hi = 1.5707963267948965580e+00;
    constexpr double kPiO2Lo = 6.1232339957367658e-17;
    const double t = fma(ph, kTwoOverPi, kShift);
    const double q = t - kShift;
    const int quad = __double2loint(t) & 3;
    const float x = static_cast<float>(fma(-q, kPiO2Lo, fma(-q, kPiO2Hi, ph)));
    const float z = x * x;
    float sn = 0.f, cs = 0.f;
    const bool odd = quad & 1;
    if ((WANT_SIN && !odd) || (WANT_COS && odd) || (WANT_SIN && WANT_COS))
        sn = fmaf(fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f) * z, x, x);
    if ((WANT_COS && !odd) || (WANT_SIN && odd) || (WANT_SIN && WANT_COS))
        cs = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z,
                            4.166664568298827e-2f), z, -0.5f), z, 1.0f);
    // (sin, cos) of ph from (sin x, cos x) by quadrant
    const float s_ = odd ? cs : sn, c_ = odd ? sn : cs;
    return make_float2(quad & 2 ? -s_ : s_, (quad == 1 || quad == 2) ? -c_ : c_);
}
__device__ __forceinline__ float time_cos(float w, float b, double dt) {
    return phase_sincos_fast<false, true>(static_cast<double>(w), static_cast<double>(b), dt).y;
}
__device__ __forceinline__ float time_sin(float w, float b, double dt) {
    return phase_sincos_fast<true, false>(static_cast<double>(w), static_cast<double>(b), dt).x;
}

}  // namespace spd
