// tcgen05 TF32 GEMM launchers (umma_host.cu). Same contracts as the FP32
// FFMA launchers in tgn_trainer.cu: fwd C = A.W^T, dgrad C = A.W,
// wgrad dW += dY^T.X (split-K with a deterministic reduction).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace spd {
namespace umma {

void fwd(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N, int K,
         const int* M_dev, cudaStream_t s, int epi = 0, const float* mask = nullptr,
         int ldmask = 0, int rnd = 0);
void dgrad(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N,
           int K, const int* M_dev, cudaStream_t s, int epi = 0, const float* mask = nullptr,
           int ldmask = 0, int rnd = 0);
void wgrad(const float* dY, int ldy, const float* X, int ldx, float* dW, int ldw, int N_out,
           int K_in, int rows, const int* rows_dev, float* ws, std::size_t ws_cap, cudaStream_t s);
std::uint64_t launches();

}  // namespace umma
}  // namespace spd
