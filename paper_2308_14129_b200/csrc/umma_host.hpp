// tcgen05 TF32 GEMM launchers (umma_host.cu). Same contracts as the FP32
// FFMA launchers in tgn_trainer.cu: fwd C = A.W^T, dgrad C = A.W,
// wgrad dW += dY^T.X (split-K with a deterministic reduction).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace spd {
namespace umma {

// Batched launch over heads: operand z at A + z*a, W + z*b, output at C + z*c
// (elements); n <= 4. Weight-gradient batches offset dY, X and dW the same way.
struct Batch {
    int n = 1;
    std::ptrdiff_t a = 0, b = 0, c = 0;
};

void fwd(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N, int K,
         const int* M_dev, cudaStream_t s, int epi = 0, const float* mask = nullptr,
         int ldmask = 0, int rnd = 0, const Batch& bt = {});
void dgrad(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N,
           int K, const int* M_dev, cudaStream_t s, int epi = 0, const float* mask = nullptr,
           int ldmask = 0, int rnd = 0, const Batch& bt = {});
// A split-K weight gradient whose fixed-order partial sum is left to a later
// kernel (the optimizer, k_adam): dW[m][n] += sum_z ws[z][m][n] for n < N.
struct SplitK {
    const float* ws = nullptr;
    int split = 0, M = 0, N = 0, ldws = 0;
    float* C = nullptr;
    int ldc = 0;
};
// target_ctas: the split-K grid aimed at (64: side-stream weight gradients;
// more for one on the step's critical tail). defer != null: a split-K result
// is described there instead of reduced (defer->split = 0 when none).
void wgrad(const float* dY, int ldy, const float* X, int ldx, float* dW, int ldw, int N_out,
           int K_in, int rows, const int* rows_dev, float* ws, std::size_t ws_cap, cudaStream_t s,
           const Batch& bt = {}, int target_ctas = 64, SplitK* defer = nullptr);
// Fused GRUCell on tensor cores (umma_gru.cuh): both gate GEMMs (x: [M x K1],
// h: [M x K2], augmented weights [3D x K]) and the cell; writes mem_new [M x D]
// and, when save != null, the backward's gate values [M x 4D] (r | z | n | Gh_n).
void gru_fused(const float* x, int ldx, int K1, const float* h, int ldh, int K2, const float* Wih,
               int ldwih, const float* Whh, int ldwhh, int D, int M, const int* M_dev,
               const float* mem, const std::uint32_t* nodes, float* mem_new, float* save,
               cudaStream_t s);
std::uint64_t launches();
int prefetch_knob(int bit);  // SPD_PREFETCH bit (umma_host.cu)

}  // namespace umma
}  // namespace spd
