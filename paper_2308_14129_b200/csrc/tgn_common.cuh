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
__device__ __forceinline__ float tf32r(float x) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ float rnd_if(float x, int rnd) { return rnd ? tf32r(x) : x; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// Time-encoder phase w*dt + b formed in f64 (dt reaches ~2e8 at GDELT shape,
// beyond f32's 2^24) with explicitly rounded multiply-add (the oracle's f64
// math), reduced modulo 2*pi in f64 (k*2pi error ~k*2.4e-16 <= 1e-8 rad), then
// evaluated with f32 cos/sin on |r| <= pi: within ~2e-7 of the oracle's
// f64 cos rounded to f32.
__device__ __forceinline__ float reduced_phase(float w, float b, double dt) {
    const double ph = __dadd_rn(__dmul_rn(static_cast<double>(w), dt), static_cast<double>(b));
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    constexpr double kInvTwoPi = 0.15915494309189533576888376337251;
    const double k = rint(ph * kInvTwoPi);
    return static_cast<float>(fma(-k, kTwoPi, ph));
}
__device__ __forceinline__ float time_cos(float w, float b, double dt) {
    return cosf(reduced_phase(w, b, dt));
}
__device__ __forceinline__ float time_sin(float w, float b, double dt) {
    return sinf(reduced_phase(w, b, dt));
}

}  // namespace spd
