// Host side of the tcgen05 TF32 GEMM: TMA tensor-map encoding (driver entry
// point, no libcuda link), tile-width selection, split-K and the three
// orientations used by the TGN step.
#include "pdl.cuh"
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>

#include "cuda_util.hpp"
#include "gemm_simt.cuh"
#include "umma_gemm.cuh"
#include "umma_gru.cuh"
#include "umma_host.hpp"

namespace spd {
namespace umma {

// Parameter prefetch before the PDL wait (umma_gemm.cuh Args::b_static,
// GruArgs::prefetch): SPD_PREFETCH = bitmask, bit 0 the forward / data-gradient
// GEMMs' weight operand, bit 1 the fused GRU's gate weights, bit 2 the
// decoder's W1 rows (tgn_trainer.cu). GDELT step (ms): none 0.3346 / 0.3350,
// GEMMs 0.3537 (their early CTAs hold shared memory and TMEM while waiting),
// GRU 0.3330, decoder 0.3316, GRU + decoder 0.3306 — the default (6).
int prefetch_knob(int bit) {
    static const int m = [] {
        const char* e = std::getenv("SPD_PREFETCH");
        return e ? std::atoi(e) : 6;
    }();
    return (m >> bit) & 1;
}

extern std::atomic<std::uint64_t> g_launch_counter;
std::atomic<std::uint64_t> g_launch_counter{0};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) internal_error("CudaError", "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// Row-major fp32 matrix [rows x inner] (row stride ld floats), 128-B swizzled
// boxes of {32 x box_rows}. Out-of-range elements load as zero.
CUtensorMap make_map(const float* base, std::uint64_t inner, std::uint64_t rows, int ld,
                     std::uint32_t box_rows, bool mn_major = false) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                          : CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) internal_error("CudaError", "cuTensorMapEncodeTiled failed");
    return m;
}

// Fixed-order sum of the split-K partials [batch][split][M][ldws] into the
// batch's dW (accumulate): deterministic, one launch for every batch.
__global__ void k_splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, int ldws,
                                float* __restrict__ C, int ldc, long long c_bstride, int batch) {
    pdl_entry();
    const std::size_t idx = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (std::size_t)batch * M * N) return;
    const int b = static_cast<int>(idx / ((std::size_t)M * N));
    const int e = static_cast<int>(idx % ((std::size_t)M * N));
    const int m = e / N, n = e % N;
    const float* w = ws + (std::size_t)b * splits * M * ldws + (std::size_t)m * ldws + n;
    float acc = 0.f;
#pragma unroll 8
    for (int z = 0; z < splits; ++z) acc += w[(std::size_t)z * M * ldws];
    float* c = C + b * c_bstride + (std::size_t)m * ldc + n;
    *c = *c + acc;
}

void reduce(const float* ws, int split, int M, int N, int ldws, float* C, int ldc, const Batch& bt,
            cudaStream_t s) {
    const std::size_t n = std::size_t(bt.n) * M * N;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((n + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int prio = 0;
    SPD_CUDA(cudaStreamGetPriority(s, &prio));
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // pdl.cuh
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_for(prio) ? 2 : 1;
    SPD_CUDA(cudaLaunchKernelEx(&cfg, k_splitk_reduce, ws, split, M, N, ldws, C, ldc,
                                static_cast<long long>(bt.c), bt.n));
    g_launch_counter.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}

template <bool A_MN, bool B_MN, int BN, int NSUB = 1, int CL = 1, bool DEEP = false>
void run(const Maps& maps, const Args& args, dim3 grid, cudaStream_t s) {
    using C_ = Cfg<A_MN, B_MN, BN, NSUB, CL, DEEP>;
    auto kern = umma_gemm_kernel<A_MN, B_MN, BN, NSUB, CL, DEEP>;
    ensure_smem(kern, C_::SMEM);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[3];
    int prio = 0;  // the stream's priority, explicit so graph kernel nodes keep it
    SPD_CUDA(cudaStreamGetPriority(s, &prio));
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = CL;
    attr[1].val.clusterDim.z = 1;
    attr[2].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // pdl.cuh
    attr[2].val.programmaticStreamSerializationAllowed = 1;
    int na = 1;
    if (CL > 1) attr[na++] = attr[1];
    if (pdl_for(prio)) attr[na++] = attr[2];
    cfg.attrs = attr;
    cfg.numAttrs = na;
    SPD_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, args));
    g_launch_counter.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}

// Deep one-wave tiles for the forward / data-gradient GEMMs (SPD_UMMA_DEEP=1):
// 128-wide tiles, one CTA per SM, every k-block in flight (experiment knob)
bool deep_tiles() {
    static const bool v = [] {
        const char* e = std::getenv("SPD_UMMA_DEEP");
        return e && *e == '1';
    }();
    return v;
}

template <bool A_MN, bool B_MN>
void dispatch(int bn, const Maps& maps, const Args& args, dim3 grid, cudaStream_t s) {
    if (bn == -128) {
        run<A_MN, B_MN, 128, 1, 1, true>(maps, args, grid, s);
        return;
    }
    switch (bn) {
        case 64: run<A_MN, B_MN, 64>(maps, args, grid, s); break;
        case 128: run<A_MN, B_MN, 128>(maps, args, grid, s); break;
        case 224: run<A_MN, B_MN, 224>(maps, args, grid, s); break;
        case 256: run<A_MN, B_MN, 256>(maps, args, grid, s); break;
        default: internal_error("InvalidParams", "unsupported tile width");
    }
}

// Tile-width cap for the forward / data-gradient GEMMs. Default 64: at the
// step's sizes (R = 6,000 rows) 128 x 64 tiles give ~190-380 CTAs at 3 per SM
// (3 stages, <= 113 registers), so each CTA's epilogue overlaps its
// neighbours' TMA round trips; measured 0.409 vs 0.432 ms per GDELT step
// against the widest-tile choice. SPD_UMMA_MAXBN overrides (experiments).
int max_bn() {
    static const int v = [] {
        const char* e = std::getenv("SPD_UMMA_MAXBN");
        return e ? std::atoi(e) : 64;
    }();
    return v;
}

// widest tile with the least padding of N (ties -> wider)
int pick_bn(int N, int cap = 0) {
    const int cands[] = {256, 224, 128, 64};
    int best = 64;
    long best_pad = 1L << 40;
    if (cap <= 0) cap = max_bn();
    for (int c : cands) {
        if (c > cap && c != 64) continue;
        const long tiles = (N + c - 1) / c;
        const long pad = tiles * c - N + tiles * 8;  // small per-tile overhead term
        if (pad < best_pad) {
            best_pad = pad;
            best = c;
        }
    }
    return best;
}

// SPD_UMMA_WIDE_BIG=1: GEMMs whose 64-wide tiles take more than one wave at
// 3 CTAs per SM (the per-head Qp / dxbar launches: 658 CTAs) use tiles up to
// 224 wide (experiment knob: measured 0.363 vs 0.358 ms per GDELT step)
int bn_for(int N, long mt, int nb) {
    static const bool wide = [] {
        const char* e = std::getenv("SPD_UMMA_WIDE_BIG");
        return e && *e == '1';
    }();
    const long ctas64 = long((N + 63) / 64) * mt * nb;
    return wide && ctas64 > 3L * 148 ? pick_bn(N, 224) : pick_bn(N);
}

void check_batch(const Batch& b) {
    if (b.n < 1 || b.n > kMaxBatch) internal_error("InvalidParams", "GEMM batch outside [1, 4]");
}

}  // namespace

std::uint64_t launches() { return g_launch_counter.load(); }

void fwd(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N, int K,
         const int* M_dev, cudaStream_t s, int epi, const float* mask, int ldmask, int rnd,
         const Batch& bt) {
    if (!M || !N) return;
    check_batch(bt);
    Args a{};
    a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.K = K; a.M_dev = M_dev; a.k_split = 1;
    a.mode = STORE; a.epi = epi; a.mask = mask; a.ldmask = ldmask; a.rnd = rnd;
    a.batch = bt.n; a.c_bstride = bt.c;
    a.b_static = prefetch_knob(0);  // W: a parameter tensor (umma_gemm.cuh Args)
    const int mt = (M + BM - 1) / BM;
    Maps maps{};
    if (mt >= 64 && N > 256 && N <= 416 && !M_dev && bt.n == 1) {
        // one CTA covers all N (2 x 208 in TMEM): A streamed once; W multicast
        // to CTA pairs: W streamed from L2 once per 256 rows
        maps.a[0] = make_map(A, K, M, lda, BM);
        maps.b[0] = make_map(W, K, N, ldw, 104);
        run<false, false, 208, 2, 4>(maps, a, dim3(1, (mt + 3) / 4 * 4, 1), s);
        return;
    }
    int bn = bn_for(N, mt, bt.n);
    const bool deep = deep_tiles() && long((N + 127) / 128) * mt * bt.n <= 148;
    if (deep) bn = 128;
    for (int z = 0; z < bt.n; ++z) {
        maps.a[z] = make_map(A + z * bt.a, K, M, lda, BM);
        maps.b[z] = make_map(W + z * bt.b, K, N, ldw, bn);
    }
    dispatch<false, false>(deep ? -128 : bn, maps, a, dim3((N + bn - 1) / bn, mt, bt.n), s);
}

void dgrad(const float* A, int lda, const float* W, int ldw, float* C, int ldc, int M, int N,
           int K, const int* M_dev, cudaStream_t s, int epi, const float* mask, int ldmask, int rnd,
           const Batch& bt) {
    if (!M || !N) return;
    check_batch(bt);
    Maps maps{};
    Args a{};
    a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.K = K; a.M_dev = M_dev; a.k_split = 1;
    a.mode = STORE; a.epi = epi; a.mask = mask; a.ldmask = ldmask; a.rnd = rnd;
    a.batch = bt.n; a.c_bstride = bt.c;
    a.b_static = prefetch_knob(0);  // W: a parameter tensor (umma_gemm.cuh Args)
    const int mt = (M + BM - 1) / BM;
    if (mt >= 64 && N <= 224 && !M_dev && bt.n == 1) {  // big: W multicast to CTA pairs
        maps.a[0] = make_map(A, K, M, lda, BM);
        maps.b[0] = make_map(W, N, K, ldw, BK, true);
        run<false, true, 224, 1, 4>(maps, a, dim3(1, (mt + 3) / 4 * 4, 1), s);
        return;
    }
    int bn = bn_for(N, mt, bt.n);  // multiple of 32: whole MN-major column blocks
    const bool deep = deep_tiles() && long((N + 127) / 128) * mt * bt.n <= 148;
    if (deep) bn = 128;
    for (int z = 0; z < bt.n; ++z) {
        maps.a[z] = make_map(A + z * bt.a, K, M, lda, BM);
        maps.b[z] = make_map(W + z * bt.b, N, K, ldw, BK, true);  // W [K x N], N contiguous
    }
    dispatch<false, true>(deep ? -128 : bn, maps, a, dim3((N + bn - 1) / bn, mt, bt.n), s);
}

void wgrad(const float* dY, int ldy, const float* X, int ldx, float* dW, int ldw, int N_out,
           int K_in, int rows, const int* rows_dev, float* ws, std::size_t ws_cap,
           cudaStream_t s, const Batch& bt, int target_ctas, SplitK* defer) {
    if (defer) defer->split = 0;
    if (!rows || !N_out || !K_in) return;
    auto finish = [&](int split, int ldws) {
        if (split <= 1) return;
        if (defer && bt.n == 1) {
            *defer = SplitK{ws, split, N_out, K_in, ldws, dW, ldw};
            return;
        }
        reduce(ws, split, N_out, K_in, ldws, dW, ldw, bt, s);
    };
    check_batch(bt);
    const int mt = (N_out + BM - 1) / BM;
    const int ldws = (K_in + 3) / 4 * 4;
    Maps maps{};
    Args a{};
    a.C = dW; a.ldc = ldw; a.M = N_out; a.N = K_in; a.K = rows; a.K_dev = rows_dev;
    a.epi = EPI_NONE; a.ws = ws; a.ldws = ldws; a.batch = bt.n; a.c_bstride = bt.c;
    if (rows >= 16384 && K_in > 224 && K_in <= 448 && mt >= 2 && mt <= 4 && !rows_dev && bt.n == 1) {
        // all M tiles of dW in one cluster: X (the B operand) streamed once,
        // each 128-row slice of dY^T once; K_in covered by 2 x 224 in TMEM
        int split = std::max(1, std::min(rows / (8 * BK), 148 / 4));
        while (split > 1 && std::size_t(split) * N_out * ldws > ws_cap) --split;
        maps.a[0] = make_map(dY, N_out, rows, ldy, BK, true);
        maps.b[0] = make_map(X, K_in, rows, ldx, BK, true);
        a.k_split = split; a.mode = split > 1 ? PARTIAL : ACCUM;
        const int cl = mt <= 2 ? 2 : 4;
        if (cl == 2) run<true, true, 224, 2, 2>(maps, a, dim3(1, 2, split), s);
        else run<true, true, 224, 2, 4>(maps, a, dim3(1, 4, split), s);
        finish(split, ldws);
        return;
    }
    const int bn = K_in <= 64 ? 64 : (K_in <= 128 ? 128 : 224);
    const int tiles = ((N_out + BM - 1) / BM) * ((K_in + bn - 1) / bn) * bt.n;
    // ~64 CTAs: enough K-parallelism for these small outputs without a split-K
    // partial traffic (split x |dW|) that the reduce then has to stream back
    int split = std::max(1, std::min(rows / (4 * BK), (target_ctas + tiles - 1) / tiles));
    while (split > 1 && std::size_t(split) * bt.n * N_out * ldws > ws_cap) --split;
    for (int z = 0; z < bt.n; ++z) {
        maps.a[z] = make_map(dY + z * bt.a, N_out, rows, ldy, BK, true);  // dY [rows x N_out]
        maps.b[z] = make_map(X + z * bt.b, K_in, rows, ldx, BK, true);    // X  [rows x K_in]
    }
    a.k_split = split; a.mode = split > 1 ? PARTIAL : ACCUM;
    dispatch<true, true>(bn, maps, a,
                         dim3((K_in + bn - 1) / bn, (N_out + BM - 1) / BM, split * bt.n), s);
    finish(split, ldws);
}

template <int UB>
void gru_fused_t(const float* x, int ldx, int K1, const float* h, int ldh, int K2, const float* Wih,
               int ldwih, const float* Whh, int ldwhh, int D, int M, const int* M_dev,
               const float* mem, const std::uint32_t* nodes, float* mem_new, float* save,
               cudaStream_t s) {
    if (!M || !D) return;
    using C_ = GruCfg<UB>;
    GruMaps maps{};
    maps.x = make_map(x, K1, M, ldx, BM);
    maps.h = make_map(h, K2, M, ldh, BM);
    maps.wih = make_map(Wih, K1, 3 * D, ldwih, UB);
    maps.whh = make_map(Whh, K2, 3 * D, ldwhh, UB);
    GruArgs a{};
    a.M = M; a.M_dev = M_dev; a.K1 = K1; a.K2 = K2; a.D = D;
    a.prefetch = prefetch_knob(1);
    a.mem = mem; a.nodes = nodes; a.mem_new = mem_new; a.save = save;
    auto kern = umma_gru_kernel<UB>;
    ensure_smem(kern, C_::SMEM);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((D + UB - 1) / UB), unsigned((M + BM - 1) / BM), 1);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int prio = 0;
    SPD_CUDA(cudaStreamGetPriority(s, &prio));
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // pdl.cuh
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_for(prio) ? 2 : 1;
    SPD_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, a));
    g_launch_counter.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}

// UB (memory units per CTA): 16 for small pending sets (<= 1,024 rows: twice
// the CTAs of a latency-bound launch; Reddit / LastFM B = 200 GRU 27.6 -> 24
// us), else kGruUB (GDELT: 32 measured faster); SPD_GRU_UB = 16 | 32 overrides
void gru_fused(const float* x, int ldx, int K1, const float* h, int ldh, int K2, const float* Wih,
               int ldwih, const float* Whh, int ldwhh, int D, int M, const int* M_dev,
               const float* mem, const std::uint32_t* nodes, float* mem_new, float* save,
               cudaStream_t s) {
    static const int forced = [] {
        const char* e = std::getenv("SPD_GRU_UB");
        return e ? std::atoi(e) : 0;
    }();
    const int ub = forced == 16 || forced == 32 ? forced : M <= 1024 ? 16 : kGruUB;
    if (ub == 16)
        gru_fused_t<16>(x, ldx, K1, h, ldh, K2, Wih, ldwih, Whh, ldwhh, D, M, M_dev, mem, nodes, mem_new, save, s);
    else
        gru_fused_t<kGruUB>(x, ldx, K1, h, ldh, K2, Wih, ldwih, Whh, ldwhh, D, M, M_dev, mem, nodes, mem_new, save, s);
}

}  // namespace umma
}  // namespace spd
