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

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// cos(w*dt + b) with the phase formed in f64 (dt up to ~2e8 at GDELT shape):
// explicitly rounded multiply-add (no FMA) to match the oracle's f64 math,
// f64 cosine, one rounding to f32.
__device__ __forceinline__ float time_cos(float w, float b, double dt) {
    const double ph = __dadd_rn(__dmul_rn(static_cast<double>(w), dt), static_cast<double>(b));
    return static_cast<float>(cos(ph));
}
__device__ __forceinline__ float time_sin(float w, float b, double dt) {
    const double ph = __dadd_rn(__dmul_rn(static_cast<double>(w), dt), static_cast<double>(b));
    return static_cast<float>(sin(ph));
}

}  // namespace spd
