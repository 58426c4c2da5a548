// TGN trainer: the PAC lockstep schedule (Alg. 2; pac_sim.cpp:205-264)
// driving the per-partition TGN step on one B200, NCCL all-reduce of the flat
// gradient buffer every global step and the epoch-end shared-hub sync.
//
// Step anatomy (one worker; oracle/tgn_oracle.py TGNOracle.step):
//   roots+nbrs -> GRU gather -> G_i,G_h GEMMs -> GRU cell -> embed gather ->
//   Q, [K;V] GEMMs -> attention -> W_o GEMM -> merge gather -> W_m1, W_m2 ->
//   decoder gather -> W_d1 -> head/loss ; backward mirrors it with
//   weight-gradient GEMMs accumulating straight into the flat gradient.
#include "pdl.cuh"
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <type_traits>

#include "gemm_simt.cuh"
#include "nccl_dyn.hpp"
#include "surrogate.hpp"
#include "tgn.hpp"
#include "tgn_common.cuh"
#include "tgn_kernels.cuh"
#include "umma_host.hpp"

namespace spd {

std::atomic<std::uint64_t> g_kernel_launches{0};

// Every kernel of the TGN path goes through here: counted (bench.py reports
// the launches inside the timed region) and checked.
// Optionally launched with programmatic stream serialization (pdl.cuh).
template <class... KArgs, class... Args>
void launch(void (*k)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
            Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    // the stream's priority, explicit on the launch so graph kernel nodes keep
    // it: side-stream work yields SMs to the critical path
    int prio = 0;
    SPD_CUDA(cudaStreamGetPriority(s, &prio));
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_for(prio) ? 2 : 1;
    SPD_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(std::forward<Args>(args))...));
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

#define ncclCommInitRank NcclApi::get().CommInitRank
#define ncclCommDestroy NcclApi::get().CommDestroy
#define ncclAllReduce NcclApi::get().AllReduce
#define ncclGroupStart NcclApi::get().GroupStart
#define ncclGroupEnd NcclApi::get().GroupEnd

void ParamLayout::build(int d_mem, int d_time, int d_edge, int heads, int k, int bb) {
    backbone = bb;
    D = d_mem;
    T = d_time;
    F = d_edge;
    H = heads;
    Kn = k;
    DQ = D + T;
    DK = D + F + T;
    DM = 2 * D + F + T;
    std::size_t off = 0;
    time_w = off;
    off += ld4(T);
    time_b = off;
    off += ld4(T);
    auto lin = [&](Lin& l, int N, int K) {
        l.N = N;
        l.K = K;
        l.ld = ld_aug(K);
        l.off = off;
        off += std::size_t(N) * l.ld;
    };
    // order == oracle/tgn_oracle.py linear_specs. JODIE: one RNN gate block,
    // no attention / merge layers (zero rows), a time projection (1 -> D) last;
    // DyRep: one RNN gate block, the attention + merge layers (its message
    // embedding), no time projection
    const bool gru = backbone == 0, att = backbone != 1, tp = backbone == 1;
    lin(gru_ih, gru ? 3 * D : D, DM);
    lin(gru_hh, gru ? 3 * D : D, D);
    lin(att_q, att ? DQ : 0, DQ);
    lin(att_kv, att ? 2 * DQ : 0, DK);
    lin(att_o, att ? DQ : 0, DQ);
    lin(mrg1, att ? D : 0, DQ + D);
    lin(mrg2, att ? D : 0, D);
    lin(dec1, D, 2 * D);
    lin(dec2, 1, D);
    lin(tproj, tp ? D : 0, 1);
    total = off;
}

constexpr int kJodieRows = 64;  // roots per k_jodie_bwd block (fixed: the partials' order)

// ------------------------------------------------------------ scratch
struct Scratch {
    int B = 0, R = 0, RK = 0, U = 0;
    tgnk::Dims d{};
    DevBuf<std::uint32_t> roots, nbr_node, nbr_ev;
    DevBuf<double> root_t, nbr_dt;
    DevBuf<int> cnt;
    DevBuf<float> x_gru, h_gru, Gi, Gh, gsave, mem_new, dGi, dGh;
    DevBuf<float> Ya, Yb;  // decoder layer-1 halves (k_dec_head2)
    DevBuf<float> q_in, Q, Qp, xbar, alpha, dsc, ctx, O, m_in, Z1, emb, d_in, D1, logits, lossv, dlogit;
    DevBuf<float> dD1, dd_in, d_emb, dZ1, dm_in, dctx, dxbar, dQp, dQ, dq_in;
    DevBuf<float> ws;
    DevBuf<float> decw;  // decoder weight-gradient chunk partials (k_dec_wgrad_part)
    DevBuf<float> s_root;  // JODIE: log1p(dt) of each root
    DevBuf<float> zmsg;    // DyRep: attention embeddings of the batch's sources, destinations
    DevBuf<double> tp_part;  // JODIE: time-projection gradient partials [blocks][2D]
    DevBuf<double> tpart;
    // deterministic dH reduction (tgn_dh.cu): reader index + chunk partials
    DevBuf<int> dh_hist, dh_off_occ, dh_off_root, dh_chunk_off, dh_rchunk_off, dh_chunk_slot,
        dh_chunk_start, dh_rchunk_slot, dh_rchunk_start, dh_list_occ, dh_list_root;
    DevBuf<float> dh_partial, dh_rpartial;
    tgnk::DhIndex dh{};
    int dh_max_chunks = 0, dh_max_rchunks = 0;
    DevBuf<float> loss;  // per local worker
    int trows = 0, troot_blocks = 0, tattn_blocks = 0;  // time-grad partial blocks
};

namespace {

void init_aug(DevBuf<float>& b, int rows, int cols, int ld, cudaStream_t s) {
    const std::size_t n = std::size_t(rows) * ld;
    if (!n) return;
    launch(tgnk::k_init_aug, unsigned((n + 255) / 256), 256, 0, s, b.p, rows, cols, ld);
    SPD_CUDA(cudaGetLastError());
}

unsigned blocks_for(std::size_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// 64-row tiles when 128-row tiles would leave SMs idle (merge/decoder shapes).
bool use_bm64(int M, int N) {
    return long((M + 127) / 128) * ((N + gemm::BN - 1) / gemm::BN) < 2L * 148;
}
// 64 x 32 tiles when 64 x 64 ones would leave SMs idle
bool use_bn32(int M, int N) {
    return long((M + 63) / 64) * ((N + gemm::BN - 1) / gemm::BN) < 148L;
}

// C[M,N] (ldc) = A[M,K](lda) . B[N,K]^T(ldb), optional relu / mask epilogue.
void gemm_fwd(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N,
              int K, const int* M_dev, cudaStream_t s, int epi = gemm::EPI_NONE,
              const float* mask = nullptr, int ldmask = 0) {
    gemm::Args a{};
    a.A = A; a.B = B; a.C = C; a.M = M; a.N = N; a.K = K;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc; a.M_dev = M_dev; a.beta = 0.f; a.epi = epi;
    a.mask = mask; a.ldmask = ldmask; a.k_split = 1;
    if (!M || !N) return;
    if (use_bn32(M, N)) {
        dim3 grid((N + 31) / 32, (M + 63) / 64, 1);
        launch(gemm::gemm_kernel<false, false, 64, 32>, grid, gemm::NT, 0, s, a);
    } else if (use_bm64(M, N)) {
        dim3 grid((N + gemm::BN - 1) / gemm::BN, (M + 63) / 64, 1);
        launch(gemm::gemm_kernel<false, false, 64>, grid, gemm::NT, 0, s, a);
    } else {
        dim3 grid((N + gemm::BN - 1) / gemm::BN, (M + 127) / 128, 1);
        launch(gemm::gemm_kernel<false, false, 128>, grid, gemm::NT, 0, s, a);
    }
    SPD_CUDA(cudaGetLastError());
}

// C[M,N] = A[M,K] . B[K,N] (data gradient through a weight), optional mask.
void gemm_dgrad(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N,
                int K, const int* M_dev, cudaStream_t s, int epi = gemm::EPI_NONE,
                const float* mask = nullptr, int ldmask = 0) {
    gemm::Args a{};
    a.A = A; a.B = B; a.C = C; a.M = M; a.N = N; a.K = K;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc; a.M_dev = M_dev; a.beta = 0.f; a.epi = epi;
    a.mask = mask; a.ldmask = ldmask; a.k_split = 1;
    if (!M || !N) return;
    if (use_bn32(M, N)) {
        dim3 grid((N + 31) / 32, (M + 63) / 64, 1);
        launch(gemm::gemm_kernel<false, true, 64, 32>, grid, gemm::NT, 0, s, a);
    } else if (use_bm64(M, N)) {
        dim3 grid((N + gemm::BN - 1) / gemm::BN, (M + 63) / 64, 1);
        launch(gemm::gemm_kernel<false, true, 64>, grid, gemm::NT, 0, s, a);
    } else {
        dim3 grid((N + gemm::BN - 1) / gemm::BN, (M + 127) / 128, 1);
        launch(gemm::gemm_kernel<false, true, 128>, grid, gemm::NT, 0, s, a);
    }
    SPD_CUDA(cudaGetLastError());
}

// dW[N_out, K_in] += dY[rows, N_out]^T . X[rows, K_in]  (rows reduced, split-K,
// deterministic fixed-order reduction of the slices).
void gemm_wgrad(const float* dY, int ldy, const float* X, int ldx, float* dW, int ldw, int N_out,
                int K_in, int rows, const int* rows_dev, float* ws, std::size_t ws_cap,
                cudaStream_t s) {
    if (!rows || !N_out || !K_in) return;
    const int tiles = ((N_out + 63) / 64) * ((K_in + gemm::BN - 1) / gemm::BN);
    int split = std::max(1, std::min(64, (2 * 148 + tiles - 1) / tiles));
    split = std::min(split, std::max(1, rows / 256));
    const int ldws = ld4(K_in);
    while (split > 1 && std::size_t(split) * N_out * ldws > ws_cap) --split;
    gemm::Args a{};
    a.A = dY; a.B = X; a.C = dW; a.M = N_out; a.N = K_in; a.K = rows;
    a.lda = ldy; a.ldb = ldx; a.ldc = ldw; a.K_dev = rows_dev; a.beta = 1.f; a.epi = 0;
    a.k_split = split; a.workspace = ws; a.ldw = ldws;
    dim3 grid((K_in + gemm::BN - 1) / gemm::BN, (N_out + 63) / 64, split);
    launch(gemm::gemm_kernel<true, true, 64>, grid, gemm::NT, 0, s, a);
    SPD_CUDA(cudaGetLastError());
    if (split > 1) {
        const std::size_t n = std::size_t(N_out) * K_in;
        launch(gemm::splitk_reduce, blocks_for(n), 256, 0, s, ws, split, N_out, K_in, ldws, dW, ldw, 1.f);
        SPD_CUDA(cudaGetLastError());
    }
}

// Tensor-core-eligible layers (GRU, attention projections) dispatch on
// spd_tgn_config::gemm_mode: 0 = FP32 FFMA, 1 = tcgen05 TF32. A Batch runs
// per-head GEMMs as one launch on the tensor-core path (FFMA: one per head).
void proj_fwd(bool tc, const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M,
              int N, int K, const int* M_dev, cudaStream_t s, int epi = 0,
              const float* mask = nullptr, int ldmask = 0, int rnd = 0, const umma::Batch& bt = {}) {
    if (tc) return umma::fwd(A, lda, B, ldb, C, ldc, M, N, K, M_dev, s, epi, mask, ldmask, rnd, bt);
    for (int z = 0; z < bt.n; ++z)
        gemm_fwd(A + z * bt.a, lda, B + z * bt.b, ldb, C + z * bt.c, ldc, M, N, K, M_dev, s, epi, mask,
                 ldmask);
}
void proj_dgrad(bool tc, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
                int M, int N, int K, const int* M_dev, cudaStream_t s, int epi = 0,
                const float* mask = nullptr, int ldmask = 0, int rnd = 0, const umma::Batch& bt = {}) {
    if (tc) return umma::dgrad(A, lda, B, ldb, C, ldc, M, N, K, M_dev, s, epi, mask, ldmask, rnd, bt);
    for (int z = 0; z < bt.n; ++z)
        gemm_dgrad(A + z * bt.a, lda, B + z * bt.b, ldb, C + z * bt.c, ldc, M, N, K, M_dev, s, epi,
                   mask, ldmask);
}
// split-K target grid of the step's last (GRU) weight gradients
// (SPD_GRU_WGRAD_CTAS): 32 — fewer split-K partials for the optimizer to sum
// (AdamFin) — measured 0.3183 / 0.3185 / 0.3188 vs 0.3227 / 0.3231 / 0.3231
// ms per GDELT step at 64 (16: 0.3263, 48: 0.3208)
long tgru_ctas() {
    static const long v = [] {
        const char* e = std::getenv("SPD_GRU_WGRAD_CTAS");
        return e ? std::atol(e) : 32L;
    }();
    return v;
}

void proj_wgrad(bool tc, const float* dY, int ldy, const float* X, int ldx, float* dW, int ldw,
                int N_out, int K_in, int rows, const int* rows_dev, float* ws, std::size_t ws_cap,
                cudaStream_t s, const umma::Batch& bt = {}, int target_ctas = 64,
                umma::SplitK* defer = nullptr) {
    if (defer) defer->split = 0;
    if (tc)
        return umma::wgrad(dY, ldy, X, ldx, dW, ldw, N_out, K_in, rows, rows_dev, ws, ws_cap, s, bt,
                           target_ctas, defer);
    for (int z = 0; z < bt.n; ++z)
        gemm_wgrad(dY + z * bt.a, ldy, X + z * bt.b, ldx, dW + z * bt.c, ldw, N_out, K_in, rows,
                   rows_dev, ws, ws_cap, s);
}

// Absorbed-projection attention kernels (tgn_attn.cu), instantiated for lane
// slots NM, NT in {1, 2} (NM + NT <= 3), NF in {1, 2, 3} and H <= 2 or 4.
template <class Kern, class... Args>
void attn_launch(Kern k, unsigned grid, std::size_t smem, cudaStream_t st, Args&&... args) {
    ensure_smem(k, smem, true);  // > 48 KB shared memory
    launch(k, grid, 32 * tgnk::attn_roots_per_block(), smem, st, std::forward<Args>(args)...);
}

template <int NM, int NT, int NF, int HM>
void attn_pick(bool bwd, unsigned grid, cudaStream_t st, const tgnk::WorkerDev& wd,
               const tgnk::Dims& d, int R, const float* tw, const float* tb, const Scratch& s,
               double* part) {
    if (!bwd)
        attn_launch(&tgnk::k_attn_abs_fwd<NM, NT, NF, HM>, grid, tgnk::attn_smem_bytes(d, false), st,
                    wd, d, R, tw, tb, s.nbr_node.p, s.nbr_ev.p, s.nbr_dt.p, s.cnt.p, s.mem_new.p,
                    s.Qp.p, s.alpha.p, s.xbar.p);
    else
        attn_launch(&tgnk::k_attn_abs_bwd<NM, NT, NF, HM>, grid, tgnk::attn_smem_bytes(d, true), st,
                    wd, d, R, tw, tb, s.nbr_node.p, s.nbr_ev.p, s.nbr_dt.p, s.cnt.p, s.mem_new.p,
                    s.Qp.p, s.alpha.p, s.dxbar.p, s.dQp.p, s.dsc.p);
}

void attn_dispatch(bool bwd, unsigned grid, cudaStream_t st, const tgnk::WorkerDev& wd,
                   const tgnk::Dims& d, int R, const float* tw, const float* tb, const Scratch& s,
                   double* part) {
    const int nm = (d.D + 127) / 128, nt = (d.T + 127) / 128, nf = (d.F + 1 + 127) / 128;
    const int key = (nm * 3 + nt) * 4 + nf;
#define SPD_A(NM, NT, NF)                                                                       \
    case (NM * 3 + NT) * 4 + NF:                                                                \
        if (d.H <= 2) attn_pick<NM, NT, NF, 2>(bwd, grid, st, wd, d, R, tw, tb, s, part);        \
        else attn_pick<NM, NT, NF, 4>(bwd, grid, st, wd, d, R, tw, tb, s, part);                 \
        break;
    switch (key) {
        SPD_A(1, 1, 1) SPD_A(1, 1, 2) SPD_A(1, 1, 3)
        SPD_A(1, 2, 1) SPD_A(1, 2, 2) SPD_A(1, 2, 3)
        SPD_A(2, 1, 1) SPD_A(2, 1, 2) SPD_A(2, 1, 3)
        default: internal_error("InvalidParams", "attention row outside the instantiated shapes");
    }
#undef SPD_A
}

void attn_abs_fwd(const tgnk::WorkerDev& wd, const tgnk::Dims& d, int R, const float* tw,
                  const float* tb, const Scratch& s, cudaStream_t st) {
    const int rpb = tgnk::attn_roots_per_block();
    attn_dispatch(false, unsigned((R + rpb - 1) / rpb), st, wd, d, R, tw, tb, s, nullptr);
}

// time-encoder gradient of the attention backward (tgn_attn.cu k_attn_time_grad)
void attn_time_grad(const tgnk::Dims& d, int R, const float* tw, const float* tb, const Scratch& s,
                    double* part, cudaStream_t st) {
    const int nt = (d.T + 127) / 128;
    const unsigned grid = unsigned(s.tattn_blocks);  // every block writes its partial row
    auto go = [&](auto k) {
        launch(k, grid, 128, 0, st, d, R, tw, tb, static_cast<const double*>(s.nbr_dt.p),
               static_cast<const int*>(s.cnt.p), static_cast<const float*>(s.Qp.p),
               static_cast<const float*>(s.alpha.p), static_cast<const float*>(s.dsc.p),
               static_cast<const float*>(s.dxbar.p), part);
    };
    if (nt == 1) d.H <= 2 ? go(tgnk::k_attn_time_grad<1, 2>) : go(tgnk::k_attn_time_grad<1, 4>);
    else if (nt == 2) d.H <= 2 ? go(tgnk::k_attn_time_grad<2, 2>) : go(tgnk::k_attn_time_grad<2, 4>);
    else internal_error("InvalidParams", "time encoder wider than the instantiated shapes");
}

// memory-row gradients of the GRU outputs, deterministic (tgn_dh.cu)
void dh_index(const tgnk::WorkerDev& wd, const Scratch& s, cudaStream_t st) {
    const std::size_t sm = std::size_t(s.dh.U_cap) * sizeof(int);
    if (sm > 48 * 1024) {
        ensure_smem(tgnk::k_dh_hist, sm);
        ensure_smem(tgnk::k_dh_scatter, sm);
    }
    const unsigned nb = unsigned(s.dh.nb_occ + s.dh.nb_root);
    launch(tgnk::k_dh_hist, nb, tgnk::kDhBlock, sm, st, wd, s.dh);
    launch(tgnk::k_dh_colscan, unsigned((s.dh.U_cap + 127) / 128), 128, 0, st, s.dh);
    launch(tgnk::k_dh_scan, 1, 1024, 0, st, s.dh);
    launch(tgnk::k_dh_scatter, nb, tgnk::kDhBlock, sm, st, wd, s.dh);
}
// grid cap of k_dh_pull (grid-stride; SPD_DHPULL_CTAS, default 148: one
// 8-warp block per SM; 296 / 592 run it faster but slow the dQ GEMMs beside
// it: 0.351 / 0.350 vs 0.337 ms per GDELT step)
std::size_t dhpull_ctas() {
    static const std::size_t v = [] {
        const char* e = std::getenv("SPD_DHPULL_CTAS");
        return e ? std::size_t(std::atol(e)) : std::size_t(148);
    }();
    return v;
}
void dh_pull(const tgnk::Dims& d, const Scratch& s, cudaStream_t st) {
    const unsigned grid = unsigned(std::min<std::size_t>((std::size_t(s.dh_max_chunks) * 32 + 255) / 256, dhpull_ctas()));
    auto go = [&](auto k) {
        launch(k, grid, 256, 0, st, s.dh, d, static_cast<const float*>(s.alpha.p),
               static_cast<const float*>(s.dsc.p), static_cast<const float*>(s.dxbar.p),
               static_cast<const float*>(s.Qp.p), s.dh_partial.p);
    };
    const int nm = (d.D + 127) / 128;
    if (nm == 1) d.H <= 2 ? go(tgnk::k_dh_pull<1, 2>) : go(tgnk::k_dh_pull<1, 4>);
    else d.H <= 2 ? go(tgnk::k_dh_pull<2, 2>) : go(tgnk::k_dh_pull<2, 4>);
}
void dh_pull_root(const tgnk::Dims& d, const Scratch& s, cudaStream_t st) {
    const unsigned grid = unsigned((std::size_t(s.dh_max_rchunks) * 32 + 255) / 256);
    auto go = [&](auto k) {
        launch(k, grid, 256, 0, st, s.dh, d, static_cast<const float*>(s.dq_in.p),
               static_cast<const float*>(s.dm_in.p), s.dh_rpartial.p);
    };
    if ((d.D + 127) / 128 == 1) go(tgnk::k_dh_pull_root<1>);
    else go(tgnk::k_dh_pull_root<2>);
}
void gru_bwd_dh(const tgnk::WorkerDev& wd, const tgnk::Dims& d, const Scratch& s, cudaStream_t st,
                bool rnn = false) {
    const unsigned grid = unsigned((std::size_t(s.U) * 32 + 255) / 256);
    auto go = [&](auto k) {
        launch(k, grid, 256, 0, st, wd, d, s.dh, static_cast<const float*>(s.dh_partial.p),
               static_cast<const float*>(s.dh_rpartial.p), static_cast<const float*>(s.gsave.p),
               s.dGi.p, s.dGh.p);
    };
    const bool one = (d.D + 127) / 128 == 1;
    if (rnn) one ? go(tgnk::k_rnn_bwd_dh<1>) : go(tgnk::k_rnn_bwd_dh<2>);
    else one ? go(tgnk::k_gru_bwd_dh<1>) : go(tgnk::k_gru_bwd_dh<2>);
}

void attn_abs_bwd(const tgnk::WorkerDev& wd, const tgnk::Dims& d, int R, const float* tw,
                  const float* tb, const Scratch& s, double* part, cudaStream_t st) {
    const int rpb = tgnk::attn_roots_per_block();
    attn_dispatch(true, unsigned((R + rpb - 1) / rpb), st, wd, d, R, tw, tb, s, part);
}

tgnk::WorkerDev devview(Worker& w) {
    tgnk::WorkerDev v{};
    v.ev_src = w.ev_src.p; v.ev_dst = w.ev_dst.p; v.ev_ts = w.ev_ts.p; v.feat = w.feat.p;
    v.adj_off = w.adj_off.p; v.adj_nbr = w.adj_nbr.p; v.adj_ev = w.adj_ev.p; v.adj_ts = w.adj_ts.p;
    v.pool = w.pool.p; v.n_pool = w.n_pool; v.mem = w.mem.p; v.lu = w.lu.p; v.slot = w.slot.p;
    const Worker::PendingSet& c = w.pend[w.cur];
    const Worker::PendingSet& n = w.pend[w.cur ^ 1];
    v.lastpos = w.lastpos.p; v.pU = c.pU.p; v.pOther = c.pOther.p; v.pEv = c.pEv.p; v.pTs = c.pTs.p;
    v.nU = c.nU.p;
    v.nxU = n.pU.p; v.nxOther = n.pOther.p; v.nxEv = n.pEv.p; v.nxTs = n.pTs.p; v.nxN = n.nU.p;
    v.pZ = c.pZ.p; v.nxZ = n.pZ.p;  // (null unless DyRep)
    v.ctl = w.ctl;
    return v;
}

void init_params_host(const ParamLayout& L, std::uint64_t seed, std::vector<float>& flat) {
    flat.assign(L.total, 0.f);
    for (int i = 0; i < L.T; ++i)
        flat[L.time_w + i] = static_cast<float>(
            L.T > 1 ? std::pow(10.0, -9.0 * double(i) / double(L.T - 1)) : 1.0);
    const std::uint64_t s = mix64(seed);
    const ParamLayout::Lin* lins[] = {&L.gru_ih, &L.gru_hh, &L.att_q, &L.att_kv, &L.att_o,
                                      &L.mrg1,   &L.mrg2,   &L.dec1,  &L.dec2, &L.tproj};
    const int fans[] = {L.D, L.D, L.DQ, L.DK, L.DQ, L.DQ + L.D, L.D, 2 * L.D, L.D, L.D};
    for (int t = 0; t < 10; ++t) {
        const auto& l = *lins[t];
        const double a = 1.0 / std::sqrt(double(fans[t]));
        auto draw = [&](std::uint64_t tag, std::uint64_t i) {
            const std::uint64_t h = mix64(mix64(s ^ tag) ^ i);
            const double u = double(h >> 40) * 0x1.0p-24;
            return static_cast<float>((2.0 * u - 1.0) * a);
        };
        for (int n = 0; n < l.N; ++n) {
            for (int k = 0; k < l.K; ++k)
                flat[l.off + std::size_t(n) * l.ld + k] = draw(t, std::uint64_t(n) * l.K + k);
            flat[l.off + std::size_t(n) * l.ld + l.K] = draw(t + 100, n);
        }
    }
}

}  // namespace

// --------------------------------------------------------------- setup
TGNTrainer::TGNTrainer(const spd_tgn_config& cfg, const SubGraphs& subs,
                       const std::vector<int>& workers, const std::vector<NodeId>& shared,
                       NodeId node_count, int rank, int world, const void* nccl_id, int device)
    : cfg_(cfg), device_(device), rank_(rank), world_(world), shared_(shared) {
    if (cfg.d_mem < 4 || cfg.d_mem % 4 || cfg.d_time < 4 || cfg.d_time % 4 || cfg.d_edge < 0)
        data_error("InvalidParams", "d_mem and d_time must be positive multiples of 4, d_edge >= 0");
    if (cfg.n_heads < 1 || (cfg.d_mem + cfg.d_time) % cfg.n_heads)
        data_error("InvalidParams", "n_heads must divide d_mem + d_time");
    if (cfg.n_neighbors < 1 || cfg.n_neighbors > 16)
        data_error("InvalidParams", "n_neighbors must lie in [1, 16]");
    if (cfg.n_heads > 4 || ((cfg.d_mem + cfg.d_time) / cfg.n_heads) % 4)
        data_error("InvalidParams", "n_heads must be <= 4 with a head width that is a multiple of 4");
    if (cfg.d_mem + cfg.d_time > 256 || cfg.d_edge + 1 > 384 || cfg.d_mem > 192)
        data_error("InvalidParams", "need d_mem + d_time <= 256, d_mem <= 192 and d_edge < 384");
    if (cfg.batch_size < 1) data_error("InvalidParams", "need batch_size >= 1");
    if (world < 1 || rank < 0 || rank >= world) data_error("InvalidParams", "bad rank/world");
    require_device(device);
    DeviceGuard g(device);
    pdl_auto() = cfg.batch_size <= 512;  // launch-latency-bound steps (pdl.cuh)
    // the main stream carries the step's critical path: highest priority, so
    // its CTAs are scheduled ahead of the side streams' (weight gradients,
    // neighbour search, time encoding) whenever both have work queued
    int prio_lo = 0, prio_hi = 0;
    SPD_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SPD_CUDA(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, prio_hi));
    for (int k = 0; k < kSide; ++k) {
        SPD_CUDA(cudaStreamCreateWithPriority(&sides_[k], cudaStreamNonBlocking, prio_lo));
        SPD_CUDA(cudaEventCreateWithFlags(&ev_join_[k], cudaEventDisableTiming));
    }
    side_ = sides_[0];
    SPD_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    for (auto& e : marks_) SPD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

    SPD_CUDA(cudaStreamCreateWithPriority(&aux_, cudaStreamNonBlocking, prio_hi));
    SPD_CUDA(cudaStreamCreateWithPriority(&zs_, cudaStreamNonBlocking, prio_lo));
    for (cudaEvent_t* e : {&ev_aux_fork_, &ev_aux_join_, &ev_roots_, &ev_dhidx_, &ev_zfork_, &ev_zero_, &ev_bwdx_, &ev_pull_, &ev_pend_, &ev_wc_, &ev_ctx_, &ev_q_})
        SPD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    if (cfg.backbone < 0 || cfg.backbone > 2)
        data_error("InvalidParams", "backbone must be 0 (TGN), 1 (JODIE) or 2 (DyRep)");
    lay_.build(cfg.d_mem, cfg.d_time, cfg.d_edge, cfg.n_heads, cfg.n_neighbors, cfg.backbone);
    feat_seed_mixed_ = mix64(cfg.seed_feat);
    const int D = lay_.D, F = lay_.F;
    const int Fp = F ? (F + 7) / 8 * 8 : 0;
    const int B = static_cast<int>(cfg.batch_size);
    if (cfg.concurrent && world == 1 && workers.size() > 1) {  // concurrent lanes (tgn_lanes.cu)
        build_lanes(subs, workers, node_count);
        return;
    }
    build_workers(subs, workers);

    // parameters + optimiser state
    std::vector<float> flat;
    init_params_host(lay_, cfg.seed_init, flat);
    params_.alloc(lay_.total); params_.upload(flat.data(), lay_.total, stream_);
    params_tc_.alloc(lay_.total);
    // per-step control block (see commit_ctl)
    {
        const std::size_t words = 2 * workers_.size() + 2;  // + Adam bias corrections, step seq
        ctl_dev_.alloc(words);
        ctl_dev_.zero(stream_);
        ctl_stage_.assign(words, 0);
        for (std::size_t k = 0; k < workers_.size(); ++k) {
            workers_[k]->ctl = ctl_dev_.p + 2 * k;
            workers_[k]->ctl_index = static_cast<int>(k);
        }
        adam_bc_ = reinterpret_cast<const float*>(ctl_dev_.p + 2 * workers_.size());
        SPD_CUDA(cudaHostAlloc(&ctl_ring_, std::size_t(kCtlSlots) * words * sizeof(std::uint64_t),
                               cudaHostAllocDefault));
        for (auto& e : ctl_ev_) SPD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    refresh_tc_weights();
    grads_.alloc(lay_.total); grads_.zero(stream_);
    adam_m_.alloc(lay_.total); adam_m_.zero(stream_);
    adam_v_.alloc(lay_.total); adam_v_.zero(stream_);
    tgrad_.alloc(2 * ld4(lay_.T)); tgrad_.zero(stream_);

    // scratch for one batch
    s_ = std::make_unique<Scratch>();
    Scratch& s = *s_;
    s.B = B; s.R = 3 * B; s.RK = s.R * cfg.n_neighbors; s.U = 2 * B;
    auto& d = s.d;
    d.D = D; d.T = lay_.T; d.F = F; d.Fp = Fp; d.DQ = lay_.DQ; d.DK = lay_.DK; d.DM = lay_.DM;
    d.H = lay_.H; d.K = lay_.Kn;
    d.ld_x = ld_aug(d.DM); d.ld_h = ld_aug(D); d.ld_q = ld_aug(d.DQ);
    d.ld_ctx = ld_aug(d.DQ); d.ld_m = ld_aug(d.DQ + D); d.ld_z = ld_aug(D); d.ld_din = ld_aug(2 * D);
    d.ld_d1 = ld_aug(D); d.ld_g = ld32(3 * D);
    d.ld_Q = ld32(d.DQ); d.ld_p = ld_aug(d.DK);
    d.rnd = cfg.gemm_mode == 1 ? 1 : 0;
    const int R = s.R, RK = s.RK, U = s.U;
    s.roots.alloc(R); s.root_t.alloc(R); s.cnt.alloc(R);
    s.nbr_node.alloc(RK); s.nbr_ev.alloc(RK); s.nbr_dt.alloc(RK);
    {  // dH reader index (tgn_dh.cu)
        auto& x = s.dh;
        x.RK = RK; x.K = d.K; x.R = R; x.U_cap = U;
        x.nb_occ = (RK + tgnk::kDhBlock - 1) / tgnk::kDhBlock;
        x.nb_root = (R + tgnk::kDhBlock - 1) / tgnk::kDhBlock;
        // every slot adds at most one partly filled chunk per list
        s.dh_max_chunks = RK / tgnk::kDhChunk + U + 1;
        s.dh_max_rchunks = R / tgnk::kDhChunk + U + 1;
        s.dh_hist.alloc(std::size_t(x.nb_occ + x.nb_root) * U);
        s.dh_off_occ.alloc(U + 1); s.dh_off_root.alloc(U + 1);
        s.dh_chunk_off.alloc(U + 1); s.dh_rchunk_off.alloc(U + 1);
        s.dh_chunk_slot.alloc(s.dh_max_chunks); s.dh_chunk_start.alloc(s.dh_max_chunks);
        s.dh_rchunk_slot.alloc(s.dh_max_rchunks); s.dh_rchunk_start.alloc(s.dh_max_rchunks);
        s.dh_list_occ.alloc(RK); s.dh_list_root.alloc(R);
        s.dh_partial.alloc(std::size_t(s.dh_max_chunks) * D);
        s.dh_rpartial.alloc(std::size_t(s.dh_max_rchunks) * D);
        x.hist = s.dh_hist.p; x.off_occ = s.dh_off_occ.p; x.off_root = s.dh_off_root.p;
        x.chunk_off = s.dh_chunk_off.p; x.rchunk_off = s.dh_rchunk_off.p;
        x.chunk_slot = s.dh_chunk_slot.p; x.chunk_start = s.dh_chunk_start.p;
        x.rchunk_slot = s.dh_rchunk_slot.p; x.rchunk_start = s.dh_rchunk_start.p;
        x.list_occ = s.dh_list_occ.p; x.list_root = s.dh_list_root.p;
    }
    s.x_gru.alloc(std::size_t(U) * d.ld_x); init_aug(s.x_gru, U, d.DM, d.ld_x, stream_);
    s.h_gru.alloc(std::size_t(U) * d.ld_h); init_aug(s.h_gru, U, D, d.ld_h, stream_);
    s.Gi.alloc(std::size_t(U) * d.ld_g); s.Gh.alloc(std::size_t(U) * d.ld_g);
    s.gsave.alloc(std::size_t(U) * 4 * D); s.mem_new.alloc(std::size_t(U) * D);
    s.dGi.alloc(std::size_t(U) * d.ld_g); s.dGh.alloc(std::size_t(U) * d.ld_g);
    s.dGi.zero(stream_); s.dGh.zero(stream_); s.Gi.zero(stream_); s.Gh.zero(stream_);
    s.q_in.alloc(std::size_t(R) * d.ld_q); init_aug(s.q_in, R, d.DQ, d.ld_q, stream_);
    s.Q.alloc(std::size_t(R) * d.ld_Q);
    const std::size_t hp = std::size_t(R) * d.H * d.ld_p;  // per-root, per-head rows
    s.Qp.alloc(hp); s.xbar.alloc(hp); s.dxbar.alloc(hp); s.dQp.alloc(hp);
    s.Qp.zero(stream_); s.xbar.zero(stream_); s.dxbar.zero(stream_); s.dQp.zero(stream_);
    s.alpha.alloc(std::size_t(R) * d.H * d.K);
    s.dsc.alloc(std::size_t(R) * d.H * d.K);
    s.ctx.alloc(std::size_t(R) * d.ld_ctx); init_aug(s.ctx, R, d.DQ, d.ld_ctx, stream_);
    s.O.alloc(std::size_t(R) * d.DQ);
    s.m_in.alloc(std::size_t(R) * d.ld_m); init_aug(s.m_in, R, d.DQ + D, d.ld_m, stream_);
    s.Z1.alloc(std::size_t(R) * d.ld_z); init_aug(s.Z1, R, D, d.ld_z, stream_);
    s.emb.alloc(std::size_t(R) * D);
    s.Ya.alloc(std::size_t(B) * D); s.Yb.alloc(std::size_t(2 * B) * D);
    s.d_in.alloc(std::size_t(2 * B) * d.ld_din); init_aug(s.d_in, 2 * B, 2 * D, d.ld_din, stream_);
    s.D1.alloc(std::size_t(2 * B) * d.ld_d1); init_aug(s.D1, 2 * B, D, d.ld_d1, stream_);
    s.logits.alloc(2 * B); s.lossv.alloc(2 * B);
    s.dlogit.alloc(std::size_t(2 * B) * 4); s.dlogit.zero(stream_);
    s.dD1.alloc(std::size_t(2 * B) * D); s.dd_in.alloc(std::size_t(2 * B) * d.ld_din);
    s.d_emb.alloc(std::size_t(R) * D); s.dZ1.alloc(std::size_t(R) * D);
    s.dm_in.alloc(std::size_t(R) * d.ld_m); s.dctx.alloc(std::size_t(R) * d.ld_Q);
    s.dQ.alloc(std::size_t(R) * d.ld_Q); s.dq_in.alloc(std::size_t(R) * d.ld_q);
    s.ws.alloc(std::size_t(64) * 1024 * 1024 / 4 * 4);  // 64 MiB split-K workspace
    s.decw.alloc(std::size_t((B + tgnk::kDecWgEv - 1) / tgnk::kDecWgEv) *
                 (std::size_t(D) * (2 * D + 1) + D + 1));
    if (cfg.backbone == 2) s.zmsg.alloc(std::size_t(2) * B * D);  // DyRep message embeddings
    if (cfg.backbone != 0) {
        s.s_root.alloc(R);
        s.tp_part.alloc(std::size_t((R + kJodieRows - 1) / kJodieRows) * 2 * D);
    }
    s.trows = 16;
    s.troot_blocks = (R + s.trows - 1) / s.trows;
    // k_attn_time_grad: grid-stride over the roots on one block per SM (a
    // side kernel; full grids crowded the query backward's GEMMs off the SMs)
    // (grid cap of the attention time-encoder partials, SPD_TATTN_CTAS: 296
    // measured 0.3346 vs 0.3366 ms per GDELT step against 148)
    static const int tattn_cap = [] {
        const char* e = std::getenv("SPD_TATTN_CTAS");
        return e ? std::atoi(e) : 296;
    }();
    s.tattn_blocks = std::min((R + tgnk::attn_x_roots_per_block() - 1) / tgnk::attn_x_roots_per_block(), tattn_cap);
    s.tpart.alloc(std::size_t(s.troot_blocks + s.tattn_blocks) * 2 * d.T);
    s.dh.nbr_node = s.nbr_node.p; s.dh.cnt = s.cnt.p; s.dh.roots = s.roots.p;
    {
        const char* e = std::getenv("SPD_GRU_FUSED");
        gru_fused_ = !(e && *e == '0') && cfg.backbone == 0;
    }
    {  // folded output x value projection (build_wc); SPD_FOLD_O=0: separate ctx and O GEMMs
        const char* e = std::getenv("SPD_FOLD_O");
        // (TGN only: DyRep's forward-only message embedding measured 0.2148 folded
        // vs 0.2120 ms — the per-step build is not repaid by one forward GEMM)
        fold_o_ = !(e && *e == '0') && cfg.backbone == 0;
        if (fold_o_) {
            wc_.alloc(std::size_t(d.DQ) * d.H * d.ld_p);
            wc_.zero(stream_);  // the per-head pad columns stay 0
        }
        // (the query x key fold measured slower: GDELT 0.361 vs 0.326 ms — its
        // long-K data-gradient GEMM and the side Q / dQ GEMMs; SPD_FOLD_Q=1)
        const char* q = std::getenv("SPD_FOLD_Q");
        fold_q_ = (q && *q == '1') && cfg.backbone == 0;
        if (fold_q_) {
            wqk_.alloc(std::size_t(d.DQ + 1) * d.H * d.ld_p);
            wqk_.zero(stream_);
        }
    }
    s.loss.alloc(std::max<std::size_t>(1, workers_.size()));
    SPD_CUDA(cudaStreamSynchronize(stream_));

    if (world_ > 1 && !nccl_id) {  // peer-memory transport (peer_comm.hpp): connect before stepping
        const std::size_t S = shared_.size();
        const std::size_t sb = std::max<std::size_t>({256, S * lay_.D * sizeof(float), S * sizeof(double)});
        peer_ = std::make_unique<PeerComm>(rank_, world_, device_, grads_.p, sb);
    } else if (world_ > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclComm_t comm;
        SPD_NCCL(ncclCommInitRank(&comm, world_, id, rank_));
        nccl_ = comm;
    }
}

int TGNTrainer::feat_stride() const { return lanes_.empty() ? s_->d.Fp : lanes_[0]->feat_stride(); }
float* TGNTrainer::loss_dev() const { return s_->loss.p; }

// Fork f onto a side stream (round-robin unless `which` pins one) at the
// current point of the main stream; f's split-K GEMMs use ws_cur_/wsn_cur_.
void TGNTrainer::side(const std::function<void(cudaStream_t)>& f, int which) {
    const int k = which >= 0 ? which : (side_next_++ % kSide);
    SPD_CUDA(cudaEventRecord(ev_fork_, stream_));
    SPD_CUDA(cudaStreamWaitEvent(sides_[k], ev_fork_, 0));
    const std::size_t slice = s_->ws.n / kSide;
    ws_cur_ = s_->ws.p + slice * k;
    wsn_cur_ = slice;
    side_used_[k] = true;
    f(sides_[k]);
}

cudaEvent_t TGNTrainer::mark() {
    cudaEvent_t e = marks_[mark_next_++ % kMarks];
    SPD_CUDA(cudaEventRecord(e, stream_));
    return e;
}

void TGNTrainer::side_from(cudaEvent_t at, const std::function<void(cudaStream_t)>& f) {
    const int k = side_next_++ % kSide;
    SPD_CUDA(cudaStreamWaitEvent(sides_[k], at, 0));
    const std::size_t slice = s_->ws.n / kSide;
    ws_cur_ = s_->ws.p + slice * k;
    wsn_cur_ = slice;
    side_used_[k] = true;
    f(sides_[k]);
}

void TGNTrainer::join_side() {
    for (int k = 0; k < kSide; ++k) {
        if (!side_used_[k]) continue;
        SPD_CUDA(cudaEventRecord(ev_join_[k], sides_[k]));
        SPD_CUDA(cudaStreamWaitEvent(stream_, ev_join_[k], 0));
        side_used_[k] = false;
    }
}

TGNTrainer::~TGNTrainer() {
    if (!lanes_.empty()) {
        for (auto& l : lanes_) cudaStreamSynchronize(l->stream_);
        for (auto e : lane_end_)
            if (e) cudaEventDestroy(e);
        if (lanes_adam_) cudaEventDestroy(lanes_adam_);
    }
    for (auto g : graph_exec_)
        if (g) cudaGraphExecDestroy(g);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto e : ctl_ev_)
        if (e) cudaEventDestroy(e);
    if (ctl_ring_) cudaFreeHost(ctl_ring_);
    if (stage_) cudaFreeHost(stage_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    for (auto e : marks_)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < kSide; ++k) {
        if (ev_join_[k]) cudaEventDestroy(ev_join_[k]);
        if (sides_[k]) cudaStreamDestroy(sides_[k]);
    }
    for (cudaEvent_t e : {ev_aux_fork_, ev_aux_join_, ev_roots_, ev_dhidx_, ev_zfork_, ev_zero_, ev_bwdx_, ev_pull_, ev_pend_, ev_wc_, ev_ctx_, ev_q_})
        if (e) cudaEventDestroy(e);
    if (aux_) cudaStreamDestroy(aux_);
    for (auto& p : aring_)
        if (p) cudaFreeHost(p);
    for (auto& e : aring_ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : astep_ev_)
        if (e) cudaEventDestroy(e);
    if (copy_) cudaStreamDestroy(copy_);
    if (zs_) cudaStreamDestroy(zs_);
    if (nccl_) ncclCommDestroy(static_cast<ncclComm_t>(nccl_));
    if (stream_) cudaStreamDestroy(stream_);
}

// Per-worker device state from the subgraphs: local ids, time-sorted CSR,
// destination pool, features (generated on device), memory and pending sets.
void TGNTrainer::build_workers(const SubGraphs& subs, const std::vector<int>& ids) {
    syncbuf_.rows.clear();  // (shared-row maps of the previous workers)
    const int D = lay_.D, F = lay_.F;
    const int Fp = F ? (F + 7) / 8 * 8 : 0;
    const int B = static_cast<int>(cfg_.batch_size);
    const spd_tgn_config& cfg = cfg_;
    total_workers_ = static_cast<int>(subs.g.size());
    all_batches_.clear();
    for (const auto& sg : subs.g)
        all_batches_.push_back((sg.edges.size() + cfg.batch_size - 1) / cfg.batch_size);
    epoch_steps_ = all_batches_.empty() ? 0 : *std::max_element(all_batches_.begin(), all_batches_.end());

    for (int wid : ids) {
        if (wid < 0 || wid >= total_workers_) data_error("InvalidParams", "worker id out of range");
        const SubGraph& sg = subs.g[wid];
        auto W = std::make_unique<Worker>();
        Worker& w = *W;
        w.gid = wid;
        w.nodes = sg.nodes;
        w.N = static_cast<NodeId>(sg.nodes.size());
        w.E = sg.edges.size();
        w.batches = all_batches_[wid];
        // local ids
        std::vector<std::uint32_t> src(w.E), dst(w.E);
        std::vector<double> ts(w.E);
        auto loc = [&](NodeId gid) -> std::uint32_t {
            auto it = std::lower_bound(w.nodes.begin(), w.nodes.end(), gid);
            if (it == w.nodes.end() || *it != gid)
                data_error("InvalidPartition", "edge endpoint outside the subgraph's node set");
            return static_cast<std::uint32_t>(it - w.nodes.begin());
        };
        for (std::uint64_t k = 0; k < w.E; ++k) {
            src[k] = loc(sg.edges[k].src);
            dst[k] = loc(sg.edges[k].dst);
            ts[k] = sg.edges[k].ts;
            if (k && ts[k] < ts[k - 1])
                data_error("NonChronological", "subgraph edges must be time-ordered");
        }
        // per-node time-sorted adjacency (both directions; ties keep event
        // order, src side first — the oracle's (ts, event, role) order)
        std::vector<std::uint64_t> off(std::size_t(w.N) + 1, 0);
        for (std::uint64_t k = 0; k < w.E; ++k) {
            ++off[src[k] + 1];
            ++off[dst[k] + 1];
        }
        for (NodeId i = 0; i < w.N; ++i) off[i + 1] += off[i];
        std::vector<std::uint64_t> fill(off.begin(), off.end() - 1);
        std::vector<std::uint32_t> anbr(2 * w.E), aev(2 * w.E);
        std::vector<double> ats(2 * w.E);
        for (std::uint64_t k = 0; k < w.E; ++k) {  // events are time-ordered: append keeps order
            std::uint64_t p = fill[src[k]]++;
            anbr[p] = dst[k]; aev[p] = static_cast<std::uint32_t>(k); ats[p] = ts[k];
            p = fill[dst[k]]++;
            anbr[p] = src[k]; aev[p] = static_cast<std::uint32_t>(k); ats[p] = ts[k];
        }
        std::vector<std::uint32_t> pool(dst);
        std::sort(pool.begin(), pool.end());
        pool.erase(std::unique(pool.begin(), pool.end()), pool.end());
        if (pool.empty()) pool.push_back(0);
        w.n_pool = static_cast<std::uint32_t>(pool.size());
        if (w.E > 0xFFFFFFFFull) data_error("InvalidParams", "partition exceeds 2^32 events");

        w.ev_src.alloc(w.E); w.ev_src.upload(src.data(), w.E, stream_);
        w.ev_dst.alloc(w.E); w.ev_dst.upload(dst.data(), w.E, stream_);
        w.ev_ts.alloc(w.E); w.ev_ts.upload(ts.data(), w.E, stream_);
        w.adj_off.alloc(off.size()); w.adj_off.upload(off.data(), off.size(), stream_);
        w.adj_nbr.alloc(2 * w.E); w.adj_nbr.upload(anbr.data(), 2 * w.E, stream_);
        w.adj_ev.alloc(2 * w.E); w.adj_ev.upload(aev.data(), 2 * w.E, stream_);
        w.adj_ts.alloc(2 * w.E); w.adj_ts.upload(ats.data(), 2 * w.E, stream_);
        w.pool.alloc(pool.size()); w.pool.upload(pool.data(), pool.size(), stream_);
        // synthetic features, generated on the device from the global edge ids
        w.feat.alloc(std::max<std::uint64_t>(1, w.E) * std::max(1, Fp));
        if (Fp && w.E) {
            DevBuf<std::uint64_t> eids(w.E);
            eids.upload(sg.eids.data(), w.E, stream_);
            launch(tgnk::k_gen_features, blocks_for(w.E * Fp), 256, 0, stream_, 
                w.feat.p, eids.p, w.E, F, Fp, feat_seed_mixed_);
            SPD_CUDA(cudaGetLastError());
            SPD_CUDA(cudaStreamSynchronize(stream_));
        }
        init_worker_state(w);
        w.ev_host.resize(w.E);
        for (std::uint64_t k = 0; k < w.E; ++k) w.ev_host[k] = spd_edge{src[k], dst[k], ts[k]};
        workers_.push_back(std::move(W));
    }
}

void TGNTrainer::init_worker_state(Worker& w) {
    const int D = lay_.D;
    const int B = static_cast<int>(cfg_.batch_size);
    const std::size_t N = std::max<std::size_t>(1, w.N);
    w.mem.alloc(N * D); w.mem.zero(stream_);
    w.mem_snap.alloc(N * D); w.mem_snap.zero(stream_);
    w.lu.alloc(N); w.lu.zero(stream_);
    w.lu_snap.alloc(N); w.lu_snap.zero(stream_);
    w.slot.alloc(N);
    SPD_CUDA(cudaMemsetAsync(w.slot.p, 0xFF, w.slot.bytes(), stream_));
    w.lastpos.alloc(N);
    SPD_CUDA(cudaMemsetAsync(w.lastpos.p, 0xFF, w.lastpos.bytes(), stream_));
    for (auto& ps : w.pend) {
        ps.pU.alloc(2 * B); ps.pOther.alloc(2 * B); ps.pEv.alloc(2 * B); ps.pTs.alloc(2 * B);
        if (lay_.backbone == 2) ps.pZ.alloc(std::size_t(2) * B * D);
        ps.nU.alloc(1); ps.nU.zero(stream_);
    }
    w.shared_local.clear();
    for (NodeId sidx : shared_) {
        auto it = std::lower_bound(w.nodes.begin(), w.nodes.end(), sidx);
        w.shared_local.push_back(it != w.nodes.end() && *it == sidx
                                     ? static_cast<std::uint32_t>(it - w.nodes.begin())
                                     : 0xFFFFFFFFu);
    }
}

// Shuffle-combine (pac_sim.cpp:280-329): the next epoch trains on regrouped
// subgraphs. Parameters and optimiser state carry over; memory starts from
// zero (every loop start resets it, pac_sim.cpp:238), captured graphs and
// evaluation views are rebuilt.
void TGNTrainer::rebind(const SubGraphs& subs) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_wait();
        for (auto& l : lanes_) l->rebind(subs);
        epoch_steps_ = lanes_[0]->epoch_steps_;
        return;
    }
    if (static_cast<int>(subs.g.size()) != total_workers_)
        data_error("ConfigMismatch", "rebind needs one subgraph per worker (" +
                                         std::to_string(total_workers_) + ")");
    SPD_CUDA(cudaDeviceSynchronize());
    std::vector<int> ids;
    for (const auto& w : workers_) ids.push_back(w->gid);
    for (auto& ge : graph_exec_)
        if (ge) {
            SPD_CUDA(cudaGraphExecDestroy(ge));
            ge = nullptr;
        }
    eager_full_steps_ = 0;
    workers_.clear();
    build_workers(subs, ids);
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        workers_[k]->ctl = ctl_dev_.p + 2 * k;
        workers_[k]->ctl_index = static_cast<int>(k);
    }
    step_in_epoch_ = 0;
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

Worker& TGNTrainer::worker(int w) {
    if (!lanes_.empty()) return lane_of(w)->worker(w);
    for (auto& p : workers_)
        if (p->gid == w) return *p;
    usage_error("worker " + std::to_string(w) + " is not owned by this trainer");
}

void TGNTrainer::timed(const char* name, const std::function<void()>& f) {
    if (!profile_) {
        f();
        return;
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, stream_);
    f();
    cudaEventRecord(b, stream_);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    times_.ms.emplace_back(name, ms);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

// -------------------------------------------------------------- schedule
void TGNTrainer::begin_epoch(int epoch) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        for (auto& l : lanes_) l->begin_epoch(epoch);
        return;
    }
    epoch_ = epoch;
    step_in_epoch_ = 0;
    for (auto& wp : workers_) {
        Worker& w = *wp;
        w.pos = 0;
        w.loops = 0;
        w.done = w.batches == 0;
        if (w.batches == 0) {  // vacuous: snapshot of the untouched state (pac_sim.cpp:224-230)
            SPD_CUDA(cudaMemcpyAsync(w.mem_snap.p, w.mem.p, w.mem.bytes(), cudaMemcpyDeviceToDevice, stream_));
            SPD_CUDA(cudaMemcpyAsync(w.lu_snap.p, w.lu.p, w.lu.bytes(), cudaMemcpyDeviceToDevice, stream_));
            w.loops = 1;
        }
    }
}

void TGNTrainer::seek(std::uint64_t step) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        for (auto& l : lanes_) l->seek(step);
        return;
    }
    if (step >= epoch_steps_) usage_error("seek past the end of the epoch");
    step_in_epoch_ = step;
    for (auto& wp : workers_) {
        Worker& w = *wp;
        if (w.batches == 0) continue;
        w.pos = step % w.batches;
        w.loops = step / w.batches;
        w.done = w.loops > 0;
        w.mem.zero(stream_);
        w.lu.zero(stream_);
        for (auto& ps : w.pend) ps.nU.zero(stream_);
    }
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::set_surrogate(int d, const double* w_m, const double* omega, double gamma) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_wait();
        for (auto& l : lanes_) l->set_surrogate(d, w_m, omega, gamma);
        return;
    }
    if (d != lay_.D) data_error("ConfigMismatch", "surrogate dimension must equal d_mem");
    sur_w_.alloc(std::size_t(3) * d * d);
    sur_w_.upload(w_m, sur_w_.n, stream_);
    sur_om_.alloc(d);
    sur_om_.upload(omega, d, stream_);
    sur_gamma_ = gamma;
    surrogate_ = true;
    for (auto& ge : graph_exec_)
        if (ge) {
            SPD_CUDA(cudaGraphExecDestroy(ge));
            ge = nullptr;
        }
    eager_full_steps_ = 0;
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::surrogate_update(Worker& w, const tgnk::WorkerDev& wd) {
    Scratch& s = *s_;
    launch(tgnk::k_surrogate_update, blocks_for(std::size_t(s.U) * lay_.D), 256, 0, stream_, wd, lay_.D,
           static_cast<const double*>(sur_w_.p), static_cast<const double*>(sur_om_.p), sur_gamma_,
           s.mem_new.p);
}

void TGNTrainer::gru_forward(Worker& w, const tgnk::WorkerDev& wd, bool train,
                             const std::function<void()>& after_gather) {
    Scratch& s = *s_;
    if (surrogate_) {
        surrogate_update(w, wd);
        return;
    }
    const auto& d = s.d;
    const float* P = params_.p;
    const bool tc = cfg_.gemm_mode == 1;
    const float* PW = tc ? params_tc_.p : params_.p;  // tf32-rounded weights for tensor cores
    launch(tgnk::k_gru_gather, blocks_for(std::size_t(s.U) * 32), 256, 0, stream_, 
        wd, d, P + lay_.time_w, P + lay_.time_b, s.x_gru.p, s.h_gru.p, 1);
    if (after_gather) after_gather();
    if (lay_.backbone != 0) {  // JODIE, DyRep: RNN memory updater (one gate block)
        SPD_CUDA(cudaEventRecord(ev_aux_fork_, stream_));
        SPD_CUDA(cudaStreamWaitEvent(aux_, ev_aux_fork_, 0));
        proj_fwd(tc, s.h_gru.p, d.ld_h, PW + lay_.gru_hh.off, lay_.gru_hh.ld, s.Gh.p, d.ld_g, s.U, d.D,
                 d.D + 1, w.nU(), aux_);
        proj_fwd(tc, s.x_gru.p, d.ld_x, PW + lay_.gru_ih.off, lay_.gru_ih.ld, s.Gi.p, d.ld_g, s.U, d.D,
                 d.DM + 1, w.nU(), stream_);
        SPD_CUDA(cudaEventRecord(ev_aux_join_, aux_));
        SPD_CUDA(cudaStreamWaitEvent(stream_, ev_aux_join_, 0));
        launch(tgnk::k_rnn_fwd, blocks_for(std::size_t(s.U) * d.D), 256, 0, stream_, wd, d, s.Gi.p, s.Gh.p,
               train ? s.gsave.p : nullptr, s.mem_new.p);
        return;
    }
    if (tc && gru_fused_) {  // both gate GEMMs and the cell in one tcgen05 kernel (umma_gru.cuh)
        umma::gru_fused(s.x_gru.p, d.ld_x, d.DM + 1, s.h_gru.p, d.ld_h, d.D + 1, PW + lay_.gru_ih.off,
                        lay_.gru_ih.ld, PW + lay_.gru_hh.off, lay_.gru_hh.ld, d.D, s.U, w.nU(), w.mem.p,
                        w.pend[w.cur].pU.p, s.mem_new.p, train ? s.gsave.p : nullptr, stream_);
        return;
    }
    // the two gate GEMMs are independent: the hidden-side one on the aux stream
    SPD_CUDA(cudaEventRecord(ev_aux_fork_, stream_));
    SPD_CUDA(cudaStreamWaitEvent(aux_, ev_aux_fork_, 0));
    proj_fwd(tc, s.h_gru.p, d.ld_h, PW + lay_.gru_hh.off, lay_.gru_hh.ld, s.Gh.p, d.ld_g, s.U, 3 * d.D,
             d.D + 1, w.nU(), aux_);
    proj_fwd(tc, s.x_gru.p, d.ld_x, PW + lay_.gru_ih.off, lay_.gru_ih.ld, s.Gi.p, d.ld_g, s.U, 3 * d.D,
             d.DM + 1, w.nU(), stream_);
    SPD_CUDA(cudaEventRecord(ev_aux_join_, aux_));
    SPD_CUDA(cudaStreamWaitEvent(stream_, ev_aux_join_, 0));
    launch(tgnk::k_gru_fwd, blocks_for(std::size_t(s.U) * d.D), 256, 0, stream_, 
        wd, d, s.Gi.p, s.Gh.p, s.h_gru.p, train ? s.gsave.p : nullptr, s.mem_new.p);
    SPD_CUDA(cudaGetLastError());
}

// Wc = [W_o,0 [W_V,0 | b_V,0] | W_o,1 [W_V,1 | b_V,1] | ...] (DQ x H ld_p,
// per-head pads 0) + b_o in head 0's bias column: O = [xbar_0 | xbar_1 ...] Wc^T
// (xbar_h's bias slot is sum_j a_hj = 1, or 0 with xbar = 0 for a root without
// neighbours) and dxbar = dO Wc. Built from the FP32 parameters each step
// (FFMA, ~8 MFLOP), rounded to tf32 for the tensor cores.
void TGNTrainer::build_wc(cudaStream_t sx) {
    const auto& d = s_->d;
    const int dh = d.DQ / d.H, ldhp = d.H * d.ld_p;
    const float* P = params_.p;
    const float* WV = P + lay_.att_kv.off + std::size_t(d.DQ) * lay_.att_kv.ld;
    for (int h = 0; h < d.H; ++h)
        gemm_dgrad(P + lay_.att_o.off + h * dh, lay_.att_o.ld, WV + std::size_t(h) * dh * lay_.att_kv.ld,
                   lay_.att_kv.ld, wc_.p + std::size_t(h) * d.ld_p, ldhp, d.DQ, d.DK + 1, dh, nullptr, sx);
    launch(tgnk::k_wc_fix, blocks_for(std::size_t(d.DQ) * ldhp), 256, 0, sx, wc_.p, d.DQ, ldhp, d.DK,
           static_cast<const float*>(P + lay_.att_o.off + d.DQ), lay_.att_o.ld, cfg_.gemm_mode == 1 ? 1 : 0);
}

// Wqk_h = [W_q,h | b_q,h]^T [W_K,h | b_K,h] ((DQ + 1) x (DK + 1) per head, at
// column h ld_p of a (DQ + 1) x H ld_p matrix, pads 0): Qp = [q_in | 1] Wqk and
// dq_in = dQp Wqk^T (rows < DQ).
void TGNTrainer::build_wqk(cudaStream_t sx) {
    const auto& d = s_->d;
    const int dh = d.DQ / d.H, ldhp = d.H * d.ld_p;
    const float* P = params_.p;
    launch(tgnk::k_wprod_t, blocks_for(std::size_t(d.H) * (d.DQ + 1) * (d.DK + 1)), 256, 0, sx, wqk_.p,
           ldhp, d.ld_p, static_cast<const float*>(P + lay_.att_q.off), lay_.att_q.ld,
           static_cast<const float*>(P + lay_.att_kv.off), lay_.att_kv.ld, d.DQ + 1, d.DK + 1, dh, d.H,
           cfg_.gemm_mode == 1 ? 1 : 0);
}

// One batch of one worker: events [lo, lo+B) of the view's event list.
// train: forward + backward (weight grads accumulate into grads_) + post;
// eval (train = false): forward + post (scores in s.logits), no gradients.
void TGNTrainer::worker_post_kernels(Worker& w) {
    Scratch& s = *s_;
    const tgnk::WorkerDev wd = devview(w);
    timed("post", [&] {
        launch(tgnk::k_persist, blocks_for(std::size_t(s.U) * 32), 256, 0, stream_, wd, s.d.D,
               s.mem_new.p);
    });
}

void TGNTrainer::worker_step(Worker& w, const tgnk::WorkerDev& wd, int B, bool train,
                             int slot_idx, bool post) {
    Scratch& s = *s_;
    const auto& d = s.d;
    w.last_b = B;
    const int R = 3 * B;
    float* P = params_.p;
    float* G = grads_.p;
    cudaStream_t st = stream_;
    const bool tc = cfg_.gemm_mode == 1;  // tensor cores for GRU + attention projections only
    const float* PW = tc ? params_tc_.p : params_.p;
    // The recent-k search depends only on the batch and the static CSR, the
    // dH reader index (tgn_dh.cu) on the neighbour lists and the pending
    // slots: both run on the side stream beside the GRU update and the query
    // GEMMs; the main stream waits for the neighbours where they are first
    // read, the backward for the index. Profiled runs keep them on the main
    // stream so their phase times are their own.
    auto roots = [&](cudaStream_t sx) {
        launch(tgnk::k_roots_nbrs, blocks_for(std::size_t(R) * 32), 256, 0, sx, wd, B, d.K, s.roots.p,
               s.root_t.p, s.nbr_node.p, s.nbr_ev.p, s.nbr_dt.p, s.cnt.p);
    };
    if (profile_) timed("roots_nbrs", [&] { roots(st); });
    s.dh.R = R;  // this batch's roots and occurrences (a loop's last batch may be short)
    s.dh.RK = lay_.backbone != 0 ? 0 : R * d.K;  // JODIE, DyRep: no neighbour readers with gradient
    // this batch's last messages into the other pending set (K3): depends only
    // on the batch's events, off the critical path (the GRU below reads the
    // current set); eval steps run it in their post phase
    if (train)
        side([&](cudaStream_t sd) {
            launch(tgnk::k_pending, 1, 1024, 0, sd, wd, B);
            if (lay_.backbone == 2) SPD_CUDA(cudaEventRecord(ev_pend_, sd));  // DyRep's stash waits
        });
    // (the side-stream branch is forked after the GRU's first kernel is
    // enqueued: graph replays submit independent branches in creation order)
    cudaEvent_t at_gather = nullptr;
    auto fork_roots = [&] {
        side_from(at_gather, [&](cudaStream_t sd) {
            roots(sd);
            SPD_CUDA(cudaEventRecord(ev_roots_, sd));
            if (train) {
                dh_index(wd, s, sd);
                SPD_CUDA(cudaEventRecord(ev_dhidx_, sd));  // the dH index is ready
            }
        });
    };
    timed("gru_fwd", [&] {
        gru_forward(w, wd, train, [&] {
            if (profile_) return;  // (the index reads the slots the gather sets)
            at_gather = mark();
        });
    });
    // forked from the gather's end, but created after the GRU's GEMMs and cell
    // so replays hand those their SMs first
    if (!profile_) fork_roots();
    if (profile_ && train) timed("dh_index", [&] { dh_index(wd, s, st); });
    if (!profile_) SPD_CUDA(cudaStreamWaitEvent(st, ev_roots_, 0));
    if (lay_.backbone == 2) dyrep_messages(wd, B, train);  // DyRep: attention embeddings -> messages
    if (lay_.backbone != 0) {  // JODIE / DyRep: time projection or identity + decoder
        jodie_rest(w, wd, B, train, slot_idx, post);
        return;
    }
    timed("query_gather", [&] {
        launch(tgnk::k_query_gather, blocks_for(std::size_t(R) * 32), 256, 0, st, wd, d, R,
               P + lay_.time_w, P + lay_.time_b, s.roots.p, s.mem_new.p, s.q_in.p,
               s.m_in.p);
    });
    // attention with absorbed key/value projections (tgn_attn.cu):
    //   Qp_h = Q_h [W_K,h | b_K,h]; kernel -> alpha, xbar_h; ctx_h = xbar_h [W_V,h | b_V,h]^T
    const int dh = d.DQ / d.H, ldhp = d.H * d.ld_p;
    const float* WK = PW + lay_.att_kv.off;
    const float* WV = WK + std::size_t(d.DQ) * lay_.att_kv.ld;
    const int ldw = lay_.att_kv.ld;
    const std::ptrdiff_t wst = std::ptrdiff_t(dh) * ldw;  // per-head weight slab
    auto q_gemm = [&](cudaStream_t sx) {
        proj_fwd(tc, s.q_in.p, d.ld_q, PW + lay_.att_q.off, lay_.att_q.ld, s.Q.p, d.ld_Q, R, d.DQ,
                 d.DQ + 1, nullptr, sx, 0, nullptr, 0, tc);
    };
    if (fold_q_) {
        // Qp = [q_in | 1] Wqk in one GEMM (Wqk: the step's query x key
        // projection product, build_wc); Q itself is only read by dW_K:
        // computed beside it when training
        if (train) {
            cudaEvent_t at_q = mark();
            side_from(at_q, [&](cudaStream_t sd) {
                q_gemm(sd);
                SPD_CUDA(cudaEventRecord(ev_q_, sd));
            });
        }
        SPD_CUDA(cudaStreamWaitEvent(st, ev_wc_, 0));
        timed("gemm_qp", [&] {
            proj_dgrad(tc, s.q_in.p, d.ld_q, wqk_.p, ldhp, s.Qp.p, ldhp, R, ldhp, d.DQ + 1, nullptr, st, 0,
                       nullptr, 0, 0);
        });
    } else {
        timed("gemm_q", [&] { q_gemm(st); });
        timed("gemm_qp", [&] {
            proj_dgrad(tc, s.Q.p, d.ld_Q, WK, ldw, s.Qp.p, ldhp, R, d.DK + 1, dh, nullptr, st, 0, nullptr,
                       0, 0, umma::Batch{d.H, dh, wst, d.ld_p});
        });
    }
    timed("k_attn_abs_fwd", [&] { attn_abs_fwd(wd, d, R, P + lay_.time_w, P + lay_.time_b, s, st); });
    auto ctx_gemm = [&](cudaStream_t sx) {
        proj_fwd(tc, s.xbar.p, ldhp, WV, ldw, s.ctx.p, d.ld_ctx, R, dh, d.DK + 1, nullptr, sx, 0,
                 nullptr, 0, tc, umma::Batch{d.H, d.ld_p, wst, dh});
    };
    if (fold_o_) {
        // O = [xbar_0 | xbar_1] Wc^T in one GEMM (Wc: the step's value x output
        // projection product, build_wc); roots without neighbours have xbar = 0
        // (bias slot too), hence O = 0 without a row mask. ctx itself is only
        // read by dW_o: computed beside it when training.
        if (train) {
            cudaEvent_t at_x = mark();
            side_from(at_x, [&](cudaStream_t sd) {
                ctx_gemm(sd);
                SPD_CUDA(cudaEventRecord(ev_ctx_, sd));
            });
        }
        SPD_CUDA(cudaStreamWaitEvent(st, ev_wc_, 0));
    } else {
        timed("gemm_ctx", [&] { ctx_gemm(st); });
    }
    timed("head_fwd", [&] {
        // O = [ctx | 1] W_o^T straight into the MergeLayer input's attention
        // columns, 0 for roots without neighbours (the s_root columns came
        // with the query gather)
        if (fold_o_)
            proj_fwd(tc, s.xbar.p, ldhp, wc_.p, ldhp, s.m_in.p, d.ld_m, R, d.DQ, ldhp, nullptr, st, 0,
                     nullptr, 0, tc);
        else
            proj_fwd(tc, s.ctx.p, d.ld_ctx, PW + lay_.att_o.off, lay_.att_o.ld, s.m_in.p, d.ld_m, R, d.DQ,
                     d.DQ + 1, nullptr, st, gemm::EPI_ROWMASK, reinterpret_cast<const float*>(s.cnt.p), d.DQ, tc);
        proj_fwd(tc, s.m_in.p, d.ld_m, PW + lay_.mrg1.off, lay_.mrg1.ld, s.Z1.p, d.ld_z, R, d.D,
                 d.DQ + d.D + 1, nullptr, st, gemm::EPI_RELU, nullptr, 0, tc);
        proj_fwd(tc, s.Z1.p, d.ld_z, PW + lay_.mrg2.off, lay_.mrg2.ld, s.emb.p, d.D, R, d.D, d.D + 1,
                 nullptr, st);
        decode(B, train);
    });
    // the batch loss is only read by the host after the step: off the critical path
    auto sum_loss = [&](cudaStream_t sx) {
        launch(tgnk::k_sum_loss, 1, 1024, 0, sx, s.lossv.p, 2 * B, s.loss.p + slot_idx);
    };
    if (train) side(sum_loss);
    else sum_loss(st);
    if (train) backward(w, wd, B);
    // persist this batch's memory update and store its last messages now,
    // while the scratch still holds this worker's rows (K11, K3); the last
    // worker of a training step defers it to step_body (beside the optimizer)
    if (!post) return;
    timed("post", [&] {
        launch(tgnk::k_persist, blocks_for(std::size_t(s.U) * 32), 256, 0, st, wd, d.D, s.mem_new.p);
        if (!train) launch(tgnk::k_pending, 1, 1024, 0, st, wd, B);
    });
}

// Decoder weight gradients on side streams forked from `at` (both backbones).
void TGNTrainer::decoder_wgrads(cudaEvent_t at, int B) {
    Scratch& s = *s_;
    const auto& d = s.d;
    float* G = grads_.p;
    if (d.D <= 112) {  // decoder weight gradients: chunk partials + fixed-order sum (FFMA)
        side_from(at, [&](cudaStream_t sd) {
            const std::size_t sm = tgnk::dec_wgrad_smem_bytes(d);
            ensure_smem(tgnk::k_dec_wgrad_part, sm);
            const int nblk = (B + tgnk::kDecWgEv - 1) / tgnk::kDecWgEv;
            launch(tgnk::k_dec_wgrad_part, dim3(unsigned(nblk), 4), 256, sm, sd, d, B,
                   static_cast<const float*>(s.emb.p), static_cast<const float*>(s.dD1.p),
                   static_cast<const float*>(s.dlogit.p), static_cast<const float*>(s.D1.p), s.decw.p);
            const int per = d.D * (2 * d.D + 1) + d.D + 1;
            launch(tgnk::k_dec_wgrad_reduce, unsigned((per + 255) / 256), 256, 0, sd, d, nblk,
                   static_cast<const float*>(s.decw.p), G + lay_.dec1.off, lay_.dec1.ld, G + lay_.dec2.off);
        });
    } else {
        side_from(at, [&](cudaStream_t sd) { gemm_wgrad(s.dlogit.p, 4, s.D1.p, d.ld_d1, G + lay_.dec2.off,
                                                        lay_.dec2.ld, 1, d.D + 1, 2 * B, nullptr, ws_cur_,
                                                        wsn_cur_, sd); });
        side_from(at, [&](cudaStream_t sd) {
            // the gathered decoder input [z_u | z_v | 1] is only needed here
            launch(tgnk::k_dec_gather, blocks_for(std::size_t(2 * B) * 32), 256, 0, sd, d, B,
                   s.emb.p, s.d_in.p);
            gemm_wgrad(s.dD1.p, d.D, s.d_in.p, d.ld_din, G + lay_.dec1.off, lay_.dec1.ld, d.D,
                   2 * d.D + 1, 2 * B, nullptr, ws_cur_, wsn_cur_, sd); });
    }
}

// The decoder, its loss and its data gradient: one FFMA kernel (k_decoder)
// on the trainer stream (both backbones).
void TGNTrainer::decode(int B, bool train) {
    Scratch& s = *s_;
    const auto& d = s.d;
    const float* P = params_.p;
    cudaStream_t st = stream_;
    // (its TMA row copies need 16-B aligned weight rows)
    if (lay_.dec1.off % 4 || lay_.dec1.ld % 4) internal_error("InvalidParams", "decoder rows unaligned");
    // 8 events per block; 4 for small batches (GDELT B = 2000: 8 measured
    // 0.346 vs 0.354 ms; Reddit B = 200: 4 measured 0.187 vs 0.194 ms)
    const bool small = B <= tgnk::kDecSmallB;
    const int ev = small ? tgnk::kDecEvSmall : tgnk::kDecEv;
    const std::size_t dsm = tgnk::decoder_smem_bytes(d, ev);
    const bool narrow = 4 * d.D <= 416;
    auto kdec = narrow ? (small ? tgnk::k_decoder<416, 2, tgnk::kDecEvSmall> : tgnk::k_decoder<416, 2, tgnk::kDecEv>)
                       : (small ? tgnk::k_decoder<768, 1, tgnk::kDecEvSmall> : tgnk::k_decoder<768, 1, tgnk::kDecEv>);
    ensure_smem(kdec, dsm);
    launch(kdec, unsigned((B + ev - 1) / ev),
           unsigned((4 * d.D + 31) / 32 * 32), dsm, st, d, B, static_cast<const float*>(s.emb.p),
           static_cast<const float*>(P + lay_.dec1.off), lay_.dec1.ld,
           static_cast<const float*>(P + lay_.dec2.off), s.D1.p, s.dlogit.p, s.lossv.p, s.dD1.p,
           s.logits.p, s.d_emb.p, train ? 1 : 0, umma::prefetch_knob(2));
}

// JODIE after the memory update: time-projection embedding, decoder, loss and
// (training) the backward — decoder weight gradients, time projection, the
// roots' memory-row gradients summed per pending row (tgn_dh.cu), RNN cell
// backward and its weight gradients; then the post phase.
void TGNTrainer::jodie_rest(Worker& w, const tgnk::WorkerDev& wd, int B, bool train, int slot_idx,
                            bool post) {
    Scratch& s = *s_;
    const auto& d = s.d;
    const int R = 3 * B;
    float* P = params_.p;
    float* G = grads_.p;
    cudaStream_t st = stream_;
    const bool tc = cfg_.gemm_mode == 1;
    const float* TP = lay_.backbone == 1 ? P + lay_.tproj.off : nullptr;  // null: identity (DyRep)
    const int ldtp = lay_.tproj.ld;
    timed("jodie_embed", [&] {
        launch(tgnk::k_jodie_embed, blocks_for(std::size_t(R) * 32), 256, 0, st, wd, d, R, s.roots.p,
               static_cast<const double*>(s.root_t.p), static_cast<const float*>(s.mem_new.p), TP, ldtp,
               s.emb.p, s.s_root.p);
    });
    timed("head_fwd", [&] { decode(B, train); });
    auto sum_loss = [&](cudaStream_t sx) {
        launch(tgnk::k_sum_loss, 1, 1024, 0, sx, s.lossv.p, 2 * B, s.loss.p + slot_idx);
    };
    if (train) side(sum_loss);
    else sum_loss(st);
    if (train) {
        SPD_CUDA(cudaStreamWaitEvent(st, ev_zero_, 0));  // gradients cleared (step_body)
        const bool fresh = scratch_zeroed_;
        scratch_zeroed_ = false;
        timed("head_bwd", [&] {
            cudaEvent_t at = mark();
            const int nblk = (R + kJodieRows - 1) / kJodieRows;
            launch(tgnk::k_jodie_bwd, unsigned(nblk), unsigned((d.D + 31) / 32 * 32), 0, st, wd, d, R,
                   s.roots.p, static_cast<const float*>(s.mem_new.p), TP, ldtp,
                   static_cast<const float*>(s.s_root.p), static_cast<const float*>(s.d_emb.p), s.dq_in.p,
                   s.dm_in.p, kJodieRows, s.tp_part.p);
            if (TP) {
                cudaEvent_t at_tp = mark();
                side_from(at_tp, [&](cudaStream_t sd) {
                    launch(tgnk::k_jodie_tp_final, blocks_for(std::size_t(2) * d.D), 256, 0, sd, d.D, nblk,
                           static_cast<const double*>(s.tp_part.p), G + lay_.tproj.off, ldtp);
                });
            }
            decoder_wgrads(at, B);
        });
        timed("gru_bwd", [&] {
            if (tc && !fresh) {
                s.dGi.zero(st);
                s.dGh.zero(st);
            }
            if (!profile_) SPD_CUDA(cudaStreamWaitEvent(st, ev_dhidx_, 0));  // the dH reader index
            dh_pull_root(d, s, st);
            gru_bwd_dh(wd, d, s, st, true);
            side([&](cudaStream_t sd) { proj_wgrad(tc, s.dGi.p, d.ld_g, s.x_gru.p, d.ld_x, G + lay_.gru_ih.off,
                                                   lay_.gru_ih.ld, d.D, d.DM + 1, s.U, w.nU(), ws_cur_, wsn_cur_, sd,
                                                   {}, 64, fin_defer_ ? &fin_sk_[0] : nullptr); });
            side([&](cudaStream_t sd) { proj_wgrad(tc, s.dGh.p, d.ld_g, s.h_gru.p, d.ld_h, G + lay_.gru_hh.off,
                                                   lay_.gru_hh.ld, d.D, d.D + 1, s.U, w.nU(), ws_cur_, wsn_cur_, sd,
                                                   {}, 64, fin_defer_ ? &fin_sk_[1] : nullptr); });
        });
        join_side();
    }
    if (!post) return;
    timed("post", [&] {
        launch(tgnk::k_persist, blocks_for(std::size_t(s.U) * 32), 256, 0, st, wd, d.D, s.mem_new.p);
        if (!train) {
            launch(tgnk::k_pending, 1, 1024, 0, st, wd, B);
            if (lay_.backbone == 2)
                launch(tgnk::k_dyrep_stash, blocks_for(std::size_t(2) * B * 32), 256, 0, st, wd, d.D, B,
                       static_cast<const float*>(s.zmsg.p));
        }
    });
}

// DyRep's message function: the temporal-attention embedding (the TGN layer,
// forward only — message inputs carry no gradient) of the batch's sources and
// destinations over the updated memory, into s.zmsg; in training the
// records k_pending selected (side stream) get their payload rows here.
void TGNTrainer::dyrep_messages(const tgnk::WorkerDev& wd, int B, bool train) {
    Scratch& s = *s_;
    const auto& d = s.d;
    const int R = 2 * B;  // sources then destinations (the first 2B roots)
    const float* P = params_.p;
    cudaStream_t st = stream_;
    const bool tc = cfg_.gemm_mode == 1;
    const float* PW = tc ? params_tc_.p : params_.p;
    timed("dyrep_attn", [&] {
        launch(tgnk::k_query_gather, blocks_for(std::size_t(R) * 32), 256, 0, st, wd, d, R,
               P + lay_.time_w, P + lay_.time_b, s.roots.p, s.mem_new.p, s.q_in.p, s.m_in.p);
        proj_fwd(tc, s.q_in.p, d.ld_q, PW + lay_.att_q.off, lay_.att_q.ld, s.Q.p, d.ld_Q, R, d.DQ,
                 d.DQ + 1, nullptr, st, 0, nullptr, 0, tc);
        const int dh = d.DQ / d.H, ldhp = d.H * d.ld_p;
        const float* WK = PW + lay_.att_kv.off;
        const float* WV = WK + std::size_t(d.DQ) * lay_.att_kv.ld;
        const int ldw = lay_.att_kv.ld;
        const std::ptrdiff_t wst = std::ptrdiff_t(dh) * ldw;
        proj_dgrad(tc, s.Q.p, d.ld_Q, WK, ldw, s.Qp.p, ldhp, R, d.DK + 1, dh, nullptr, st, 0, nullptr,
                   0, 0, umma::Batch{d.H, dh, wst, d.ld_p});
        attn_abs_fwd(wd, d, R, P + lay_.time_w, P + lay_.time_b, s, st);
        if (fold_o_) {  // O = [xbar_0 | xbar_1] Wc^T (build_wc; no backward reads ctx here)
            SPD_CUDA(cudaStreamWaitEvent(st, ev_wc_, 0));
            proj_fwd(tc, s.xbar.p, ldhp, wc_.p, ldhp, s.m_in.p, d.ld_m, R, d.DQ, ldhp, nullptr, st, 0,
                     nullptr, 0, tc);
        } else {
            proj_fwd(tc, s.xbar.p, ldhp, WV, ldw, s.ctx.p, d.ld_ctx, R, dh, d.DK + 1, nullptr, st, 0,
                     nullptr, 0, tc, umma::Batch{d.H, d.ld_p, wst, dh});
            proj_fwd(tc, s.ctx.p, d.ld_ctx, PW + lay_.att_o.off, lay_.att_o.ld, s.m_in.p, d.ld_m, R, d.DQ,
                     d.DQ + 1, nullptr, st, gemm::EPI_ROWMASK, reinterpret_cast<const float*>(s.cnt.p), d.DQ, tc);
        }
        proj_fwd(tc, s.m_in.p, d.ld_m, PW + lay_.mrg1.off, lay_.mrg1.ld, s.Z1.p, d.ld_z, R, d.D,
                 d.DQ + d.D + 1, nullptr, st, gemm::EPI_RELU, nullptr, 0, tc);
        proj_fwd(tc, s.Z1.p, d.ld_z, PW + lay_.mrg2.off, lay_.mrg2.ld, s.zmsg.p, d.D, R, d.D, d.D + 1,
                 nullptr, st);
        if (train) {
            if (!profile_) SPD_CUDA(cudaStreamWaitEvent(st, ev_pend_, 0));  // k_pending's records
            launch(tgnk::k_dyrep_stash, blocks_for(std::size_t(R) * 32), 256, 0, st, wd, d.D, B,
                   static_cast<const float*>(s.zmsg.p));
        }
    });
}

// Hand-written backward of one worker's batch; weight-gradient GEMMs go to the
// side stream and are joined before the post phase rewrites their inputs.
void TGNTrainer::backward(Worker& w, const tgnk::WorkerDev& wd, int B) {
    Scratch& s = *s_;
    const auto& d = s.d;
    const int R = 3 * B;
    float* P = params_.p;
    float* G = grads_.p;
    cudaStream_t st = stream_;
    const bool tc = cfg_.gemm_mode == 1;
    const float* PW = tc ? params_tc_.p : params_.p;
    SPD_CUDA(cudaStreamWaitEvent(st, ev_zero_, 0));  // gradients cleared (step_body)
    // dGi / dGh rows past |pending|: cleared at step start for the step's
    // first backward; later local workers reuse the scratch and clear them
    const bool fresh = scratch_zeroed_;
    scratch_zeroed_ = false;
    timed("head_bwd", [&] {
        // (d_emb came with the forward: k_decoder). Each data-gradient GEMM is
        // created before the weight-gradient side work forked from the same
        // point, so replays hand the critical path its SMs first.
        // merge layer 2 (relu mask from Z1)
        cudaEvent_t at = mark();
        proj_dgrad(tc, s.d_emb.p, d.D, PW + lay_.mrg2.off, lay_.mrg2.ld, s.dZ1.p, d.D, R, d.D, d.D,
                   nullptr, st, gemm::EPI_MASK, s.Z1.p, d.ld_z, tc);
        side_from(at, [&](cudaStream_t sd) { proj_wgrad(tc, s.d_emb.p, d.D, s.Z1.p, d.ld_z, G + lay_.mrg2.off,
                                                        lay_.mrg2.ld, d.D, d.D + 1, R, nullptr, ws_cur_,
                                                        wsn_cur_, sd); });
        // merge layer 1
        at = mark();
        // (attention columns of roots without neighbours: 0)
        proj_dgrad(tc, s.dZ1.p, d.D, PW + lay_.mrg1.off, lay_.mrg1.ld, s.dm_in.p, d.ld_m, R,
                   d.DQ + d.D, d.D, nullptr, st, gemm::EPI_ROWMASK, reinterpret_cast<const float*>(s.cnt.p),
                   d.DQ, tc);
        side_from(at, [&](cudaStream_t sd) { proj_wgrad(tc, s.dZ1.p, d.D, s.m_in.p, d.ld_m, G + lay_.mrg1.off,
                                                        lay_.mrg1.ld, d.D, d.DQ + d.D + 1, R, nullptr,
                                                        ws_cur_, wsn_cur_, sd); });
        // output projection
        if (!fold_o_) {
            at = mark();
            proj_dgrad(tc, s.dm_in.p, d.ld_m, PW + lay_.att_o.off, lay_.att_o.ld, s.dctx.p, d.ld_Q, R, d.DQ,
                       d.DQ, nullptr, st, 0, nullptr, 0, tc);
            side_from(at, [&](cudaStream_t sd) { proj_wgrad(tc, s.dm_in.p, d.ld_m, s.ctx.p, d.ld_ctx,
                                                            G + lay_.att_o.off, lay_.att_o.ld, d.DQ, d.DQ + 1,
                                                            R, nullptr, ws_cur_, wsn_cur_, sd); });
        }
    });
    const int dh = d.DQ / d.H, ldhp = d.H * d.ld_p;
    const float* WK = PW + lay_.att_kv.off;
    const float* WV = WK + std::size_t(d.DQ) * lay_.att_kv.ld;
    const int ldw = lay_.att_kv.ld;
    float* GK = G + lay_.att_kv.off;
    float* GV = GK + std::size_t(d.DQ) * ldw;
    const std::ptrdiff_t wst = std::ptrdiff_t(dh) * ldw;  // per-head weight slab
    timed("gemm_dxbar", [&] {
        if (fold_o_) {
            // dxbar = dO Wc (one GEMM for the output and value projections);
            // beside it dctx = dO W_o for dW_o and dW_V,h += dctx_h^T xbar_h
            cudaEvent_t at = mark();
            proj_dgrad(tc, s.dm_in.p, d.ld_m, wc_.p, ldhp, s.dxbar.p, ldhp, R, ldhp, d.DQ, nullptr, st, 0,
                       nullptr, 0, 0);
            side_from(at, [&](cudaStream_t sd) {
                SPD_CUDA(cudaStreamWaitEvent(sd, ev_ctx_, 0));
                proj_wgrad(tc, s.dm_in.p, d.ld_m, s.ctx.p, d.ld_ctx, G + lay_.att_o.off, lay_.att_o.ld,
                           d.DQ, d.DQ + 1, R, nullptr, ws_cur_, wsn_cur_, sd);
            });
            side_from(at, [&](cudaStream_t sd) {
                proj_dgrad(tc, s.dm_in.p, d.ld_m, PW + lay_.att_o.off, lay_.att_o.ld, s.dctx.p, d.ld_Q, R,
                           d.DQ, d.DQ, nullptr, sd, 0, nullptr, 0, tc);
                proj_wgrad(tc, s.dctx.p, d.ld_Q, s.xbar.p, ldhp, GV, ldw, dh, d.DK + 1, R, nullptr, ws_cur_,
                           wsn_cur_, sd, umma::Batch{d.H, dh, d.ld_p, wst});
            });
            return;
        }
        // dW_V,h += dctx_h^T xbar_h ; dxbar_h = dctx_h [W_V,h | b_V,h]
        cudaEvent_t at = mark();
        proj_dgrad(tc, s.dctx.p, d.ld_Q, WV, ldw, s.dxbar.p, ldhp, R, d.DK + 1, dh, nullptr, st, 0,
                   nullptr, 0, 0, umma::Batch{d.H, dh, wst, d.ld_p});
        side_from(at, [&](cudaStream_t sd) {
            proj_wgrad(tc, s.dctx.p, d.ld_Q, s.xbar.p, ldhp, GV, ldw, dh, d.DK + 1, R, nullptr, ws_cur_,
                       wsn_cur_, sd, umma::Batch{d.H, dh, d.ld_p, wst});
        });
    });
    double* attn_part = s.tpart.p + std::size_t(s.troot_blocks) * 2 * d.T;
    // the decoder's weight gradients have ~200 us of slack before Adam: forked
    // once the attention backward is created, so the merge-layer data
    // gradients above run without them
    cudaEvent_t at_dec = mark();
    timed("k_attn_abs_bwd", [&] {
        attn_abs_bwd(wd, d, R, P + lay_.time_w, P + lay_.time_b, s, nullptr, st);
    });
    // ... forked after the dQ GEMM is created (their shared-memory-heavy blocks
    // held SMs the dQ GEMM then waited for: 0.3228 / 0.3232 vs 0.3236 / 0.3235
    // ms per GDELT step); SPD_DECWG_LATE=0 forks them here
    static const bool decwg_late = [] {
        const char* e = std::getenv("SPD_DECWG_LATE");
        return !(e && *e == '0');
    }();
    if (!decwg_late) decoder_wgrads(at_dec, B);
    // the attention input gradients — memory columns summed per pending row
    // (k_dh_pull, deterministic, tgn_dh.cu) and the time-encoder partials —
    // run beside the dQ GEMMs; the GRU backward and the time-grad reduction
    // wait for them
    if (profile_) {
        timed("dh_pull", [&] { dh_pull(d, s, st); });
        timed("attn_time_grad", [&] { attn_time_grad(d, R, P + lay_.time_w, P + lay_.time_b, s, attn_part, st); });
    }
    cudaEvent_t at_bwd = mark();  // the attention backward is done
    auto dq_gemm = [&](cudaStream_t sx) {
        // dQ_h = dQp_h [W_K,h | b_K,h]^T
        proj_fwd(tc, s.dQp.p, ldhp, WK, ldw, s.dQ.p, d.ld_Q, R, dh, d.DK + 1, nullptr, sx, 0, nullptr,
                 0, tc, umma::Batch{d.H, d.ld_p, wst, dh});
    };
    if (!fold_q_) timed("gemm_dq", [&] { dq_gemm(st); });
    if (decwg_late) decoder_wgrads(mark(), B);
    if (!profile_) {
        // the attention input gradients (dH pull, time-encoder partials) and
        // dW_K beside the query backward: created after the dQ GEMM
        side_from(at_bwd, [&](cudaStream_t sd) {
            SPD_CUDA(cudaStreamWaitEvent(sd, ev_dhidx_, 0));  // the dH reader index
            dh_pull(d, s, sd);
            SPD_CUDA(cudaEventRecord(ev_pull_, sd));
        });
        side_from(at_bwd, [&](cudaStream_t sd) {
            attn_time_grad(d, R, P + lay_.time_w, P + lay_.time_b, s, attn_part, sd);
            SPD_CUDA(cudaEventRecord(ev_bwdx_, sd));
        });
    }
    if (fold_q_) {
        // dq_in = dQp Wqk^T (one GEMM for the key and query projections);
        // beside it dQ for dW_q, and dW_K,h += Q_h^T dQp_h
        timed("q_bwd", [&] {
            proj_fwd(tc, s.dQp.p, ldhp, wqk_.p, ldhp, s.dq_in.p, d.ld_q, R, d.DQ, ldhp, nullptr, st, 0,
                     nullptr, 0, 0);
        });
        side_from(at_bwd, [&](cudaStream_t sd) {
            dq_gemm(sd);
            proj_wgrad(tc, s.dQ.p, d.ld_Q, s.q_in.p, d.ld_q, G + lay_.att_q.off, lay_.att_q.ld, d.DQ,
                       d.DQ + 1, R, nullptr, ws_cur_, wsn_cur_, sd);
        });
        side_from(at_bwd, [&](cudaStream_t sd) {
            SPD_CUDA(cudaStreamWaitEvent(sd, ev_q_, 0));
            proj_wgrad(tc, s.Q.p, d.ld_Q, s.dQp.p, ldhp, GK, ldw, dh, d.DK + 1, R, nullptr, ws_cur_,
                       wsn_cur_, sd, umma::Batch{d.H, dh, d.ld_p, wst});
        });
    } else {
    // dW_K,h += Q_h^T dQp_h
    side_from(at_bwd, [&](cudaStream_t sd) {
        proj_wgrad(tc, s.Q.p, d.ld_Q, s.dQp.p, ldhp, GK, ldw, dh, d.DK + 1, R, nullptr, ws_cur_,
                   wsn_cur_, sd, umma::Batch{d.H, dh, d.ld_p, wst});
    });
    timed("q_bwd", [&] {
        cudaEvent_t at = mark();
        proj_dgrad(tc, s.dQ.p, d.ld_Q, PW + lay_.att_q.off, lay_.att_q.ld, s.dq_in.p, d.ld_q, R, d.DQ,
                   d.DQ, nullptr, st);
        side_from(at, [&](cudaStream_t sd) { proj_wgrad(tc, s.dQ.p, d.ld_Q, s.q_in.p, d.ld_q, G + lay_.att_q.off,
                                                        lay_.att_q.ld, d.DQ, d.DQ + 1, R, nullptr, ws_cur_,
                                                        wsn_cur_, sd); });
    });
    }
    // root-side time-encoder partials and their reduction with the attention
    // partials: only the all-reduce reads the result, so off the critical path
    side([&](cudaStream_t sd) {
        launch(tgnk::k_root_grad, s.troot_blocks, dim3(32, 8), 0, sd, d, R,
               static_cast<const float*>(s.dq_in.p), P + lay_.time_b, s.trows, s.tpart.p);
        if (!profile_) SPD_CUDA(cudaStreamWaitEvent(sd, ev_bwdx_, 0));
        launch(tgnk::k_time_grad_final, 2 * d.T, 256, 0, sd, d.T, s.troot_blocks + s.tattn_blocks,
               s.tpart.p, tgrad_.p);
    });
    timed("gru_bwd", [&] {
        if (tc && !fresh) {  // the TC weight-grad reads whole K blocks: rows >= |pending| must be 0
            s.dGi.zero(st);
            s.dGh.zero(st);
        }
        if (!profile_) SPD_CUDA(cudaStreamWaitEvent(st, ev_dhidx_, 0));  // the dH reader index
        dh_pull_root(d, s, st);
        if (!profile_) SPD_CUDA(cudaStreamWaitEvent(st, ev_pull_, 0));  // occurrence chunk partials
        gru_bwd_dh(wd, d, s, st);
        // the step's last weight gradients (Adam waits for them): a grid of
        // about one wave each instead of the side streams' 64 CTAs
        const int gru_ctas = int(tgru_ctas());
        // (the step's last worker leaves their split-K sums to Adam: fin_defer_)
        side([&](cudaStream_t sd) { proj_wgrad(tc, s.dGi.p, d.ld_g, s.x_gru.p, d.ld_x, G + lay_.gru_ih.off, lay_.gru_ih.ld,
                   3 * d.D, d.DM + 1, s.U, w.nU(), ws_cur_, wsn_cur_, sd, {}, gru_ctas,
                   fin_defer_ ? &fin_sk_[0] : nullptr); });
        side([&](cudaStream_t sd) { proj_wgrad(tc, s.dGh.p, d.ld_g, s.h_gru.p, d.ld_h, G + lay_.gru_hh.off, lay_.gru_hh.ld,
                   3 * d.D, d.D + 1, s.U, w.nU(), ws_cur_, wsn_cur_, sd, {}, gru_ctas,
                   fin_defer_ ? &fin_sk_[1] : nullptr); });
    });
    // side-stream weight grads read the pending set (nU, GRU inputs) that the
    // post phase rewrites: join first
    join_side();
}

void TGNTrainer::flush_pending(Worker& w) {
    // loop end: apply the pending messages without gradient, persist
    const auto wd = devview(w);
    gru_forward(w, wd, false);
    launch(tgnk::k_persist, blocks_for(std::size_t(s_->U) * 32), 256, 0, stream_, wd, lay_.D,
           s_->mem_new.p);
    w.pend[w.cur].nU.zero(stream_);
}

// GEMM kernels on caller-owned device buffers, for numerics tests against a
// plain fp32 reference. impl: 0 FFMA, 1 tcgen05 TF32; which: 0 fwd (C=A.B^T),
// 1 dgrad (C=A.B), 2 wgrad (C += A^T.B, reduction over K rows).
int debug_gemm(int impl, int which, const float* A, int lda, const float* B, int ldb, float* C,
               int ldc, int M, int N, int K, float* ws, std::size_t ws_cap) {
    cudaStream_t s = 0;
    if (which == 0) proj_fwd(impl == 1, A, lda, B, ldb, C, ldc, M, N, K, nullptr, s);
    else if (which == 1) proj_dgrad(impl == 1, A, lda, B, ldb, C, ldc, M, N, K, nullptr, s);
    else proj_wgrad(impl == 1, A, lda, B, ldb, C, ldc, M, N, K, nullptr, ws, ws_cap, s);
    SPD_CUDA(cudaDeviceSynchronize());
    return 0;
}

std::uint64_t kernel_launches() { return g_kernel_launches.load() + umma::launches(); }

// n lockstep global steps (wrapping into the next epoch when one ends),
// bracketed by CUDA events on the trainer's stream: device time in ms.
float TGNTrainer::run_steps(std::uint64_t n) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) return lanes_run_steps(n);
    cudaEvent_t a, b;
    SPD_CUDA(cudaEventCreate(&a));
    SPD_CUDA(cudaEventCreate(&b));
    SPD_CUDA(cudaEventRecord(a, stream_));
    for (std::uint64_t k = 0; k < n; ++k) {
        if (step_in_epoch_ >= epoch_steps_) {
            end_epoch();
            begin_epoch(epoch_ + 1);
        }
        step(nullptr);
    }
    SPD_CUDA(cudaEventRecord(b, stream_));
    SPD_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    SPD_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

// End-to-end step: each local worker's next batch (events in local ids and
// bf16 feature rows) is copied from (pinned) host memory into its device
// stream window, the step runs, and the per-worker losses come back.
void TGNTrainer::step_host(const spd_edge* const* events, const std::uint16_t* const* feats,
                           float* loss_out) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {  // lane k feeds local worker k; losses once every lane is enqueued
        if (lanes_adam_valid_) lanes_after(lanes_adam_);
        for (std::size_t k = 0; k < lanes_.size(); ++k)
            lanes_[k]->step_host(events + k, feats ? feats + k : nullptr, nullptr);
        lanes_adam_step();
        if (loss_out) lanes_losses(loss_out);
        return;
    }
    if (step_in_epoch_ >= epoch_steps_) {
        end_epoch();
        begin_epoch(epoch_ + 1);
    }
    const int Fp = s_->d.Fp;
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        Worker& w = *workers_[k];
        if (w.batches == 0) continue;
        const std::uint64_t lo = w.pos * cfg_.batch_size;
        const std::uint64_t B = std::min<std::uint64_t>(w.E, lo + cfg_.batch_size) - lo;
        // events arrive as {src, dst, ts}; scatter into pinned SoA staging
        if (stage_bytes_ < B * 16) {
            if (stage_) cudaFreeHost(stage_);
            SPD_CUDA(cudaHostAlloc(&stage_, B * 16, cudaHostAllocDefault));
            stage_bytes_ = B * 16;
        }
        SPD_CUDA(cudaStreamSynchronize(stream_));  // staging reuse across workers/steps
        const spd_edge* e = events[k];
        check_host_events(w, lo, B, e);
        std::uint32_t* hs = reinterpret_cast<std::uint32_t*>(stage_);
        std::uint32_t* hd = hs + B;
        double* ht = reinterpret_cast<double*>(hd + B);
        for (std::uint64_t i = 0; i < B; ++i) {
            hs[i] = e[i].src;
            hd[i] = e[i].dst;
            ht[i] = e[i].ts;
        }
        SPD_CUDA(cudaMemcpyAsync(w.ev_src.p + lo, hs, B * 4, cudaMemcpyHostToDevice, stream_));
        SPD_CUDA(cudaMemcpyAsync(w.ev_dst.p + lo, hd, B * 4, cudaMemcpyHostToDevice, stream_));
        SPD_CUDA(cudaMemcpyAsync(w.ev_ts.p + lo, ht, B * 8, cudaMemcpyHostToDevice, stream_));
        if (Fp && feats && feats[k])
            SPD_CUDA(cudaMemcpyAsync(w.feat.p + lo * Fp, feats[k], B * Fp * 2,
                                     cudaMemcpyHostToDevice, stream_));
        h2d_bytes_ += B * 16 + (Fp ? B * Fp * 2 : 0);
    }
    step(loss_out);
    d2h_bytes_ += workers_.size() * sizeof(float);
}

// Pipelined end-to-end step: the same inputs and outputs as step_host, but
// host staging of this batch overlaps the device's previous step. Events are
// scattered into a ring of pinned SoA slots (the host waits only for the copy
// issued kStageSlots steps ago), copied on the copy stream together with the
// caller's pinned feature rows; the step's graph waits on that copy. The
// per-worker losses are copied into the caller's pinned loss_pinned without a
// host wait (NaN for idle workers is the caller's to apply); sync() waits.
void TGNTrainer::step_host_async(const spd_edge* const* events, const std::uint16_t* const* feats,
                                 float* loss_pinned) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        if (lanes_adam_valid_) lanes_after(lanes_adam_);
        for (std::size_t k = 0; k < lanes_.size(); ++k)
            lanes_[k]->step_host_async(events + k, feats ? feats + k : nullptr,
                                       loss_pinned ? loss_pinned + k : nullptr);
        lanes_adam_step();
        return;
    }
    if (step_in_epoch_ >= epoch_steps_) {
        end_epoch();
        begin_epoch(epoch_ + 1);
    }
    if (!copy_) {
        SPD_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
        for (auto& e : aring_ev_) SPD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : astep_ev_) SPD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const std::size_t need = workers_.size() * cfg_.batch_size * 16;
    if (aring_bytes_ < need) {
        SPD_CUDA(cudaDeviceSynchronize());
        for (auto& p : aring_) {
            if (p) cudaFreeHost(p);
            SPD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), need, cudaHostAllocDefault));
        }
        aring_bytes_ = need;
        for (auto& u : aring_used_) u = false;
    }
    const int slot = aring_next_;
    aring_next_ = (aring_next_ + 1) % kStageSlots;
    if (aring_used_[slot]) SPD_CUDA(cudaEventSynchronize(aring_ev_[slot]));
    const int Fp = s_->d.Fp;
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        Worker& w = *workers_[k];
        if (w.batches == 0) continue;
        const std::uint64_t lo = w.pos * cfg_.batch_size;
        const std::uint64_t B = std::min<std::uint64_t>(w.E, lo + cfg_.batch_size) - lo;
        std::uint32_t* hs = reinterpret_cast<std::uint32_t*>(aring_[slot] + k * cfg_.batch_size * 16);
        std::uint32_t* hd = hs + B;
        double* ht = reinterpret_cast<double*>(hd + B);
        const spd_edge* e = events[k];
        check_host_events(w, lo, B, e);
        for (std::uint64_t i = 0; i < B; ++i) {
            hs[i] = e[i].src;
            hd[i] = e[i].dst;
            ht[i] = e[i].ts;
        }
        // an earlier step still in flight may read this very window (a worker
        // with one or two batches per loop): the copy waits for that step
        for (int j = 0; j < kStageSlots; ++j)
            if (j != slot && k < astep_lo_[j].size() && astep_lo_[j][k] == lo)
                SPD_CUDA(cudaStreamWaitEvent(copy_, astep_ev_[j], 0));
        SPD_CUDA(cudaMemcpyAsync(w.ev_src.p + lo, hs, B * 4, cudaMemcpyHostToDevice, copy_));
        SPD_CUDA(cudaMemcpyAsync(w.ev_dst.p + lo, hd, B * 4, cudaMemcpyHostToDevice, copy_));
        SPD_CUDA(cudaMemcpyAsync(w.ev_ts.p + lo, ht, B * 8, cudaMemcpyHostToDevice, copy_));
        if (Fp && feats && feats[k])
            SPD_CUDA(cudaMemcpyAsync(w.feat.p + lo * Fp, feats[k], B * Fp * 2,
                                     cudaMemcpyHostToDevice, copy_));
        h2d_bytes_ += B * 16 + (Fp ? B * Fp * 2 : 0);
    }
    SPD_CUDA(cudaEventRecord(aring_ev_[slot], copy_));
    aring_used_[slot] = true;
    SPD_CUDA(cudaStreamWaitEvent(stream_, aring_ev_[slot], 0));
    astep_lo_[slot].assign(workers_.size(), ~std::uint64_t(0));
    for (std::size_t k = 0; k < workers_.size(); ++k)
        if (workers_[k]->batches) astep_lo_[slot][k] = workers_[k]->pos * cfg_.batch_size;
    step(nullptr);
    SPD_CUDA(cudaEventRecord(astep_ev_[slot], stream_));
    if (loss_pinned)
        SPD_CUDA(cudaMemcpyAsync(loss_pinned, s_->loss.p, workers_.size() * sizeof(float),
                                 cudaMemcpyDeviceToHost, stream_));
    d2h_bytes_ += workers_.size() * sizeof(float);
}

// Host-fed events must be the partition's own stream: the neighbour CSR, the
// negative pool and the feature rows of the resident stream are built from it
// at construction, so different events would train on inconsistent state.
void TGNTrainer::check_host_events(const Worker& w, std::uint64_t lo, std::uint64_t B,
                                   const spd_edge* e) const {
    if (!e) usage_error("step_host: missing event batch for worker " + std::to_string(w.gid));
    if (std::memcmp(e, w.ev_host.data() + lo, B * sizeof(spd_edge)) != 0)
        data_error("InvalidParams", "host-fed events of worker " + std::to_string(w.gid) +
                                        " differ from its resident stream at batch start " +
                                        std::to_string(lo));
}

void TGNTrainer::sync() {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        for (auto& l : lanes_) l->sync();
        return;
    }
    SPD_CUDA(cudaStreamSynchronize(stream_));
    if (copy_) SPD_CUDA(cudaStreamSynchronize(copy_));
}

void TGNTrainer::worker_post(Worker& w) {
    w.cur ^= 1;  // the set k_pending just filled holds the messages to apply next
    ++w.pos;
    if (w.pos == w.batches) {  // loop_end: flush (new params) + snapshot (pac_sim.cpp:248-255)
        // (a lane's step has no Adam yet: its parent flushes after the group Adam)
        if (lane_) w.flush_due = true;
        else loop_end_flush(w);
        ++w.loops;
        w.done = true;
        w.pos = 0;
    }
}

void TGNTrainer::loop_end_flush(Worker& w) {
    flush_pending(w);
    SPD_CUDA(cudaMemcpyAsync(w.mem_snap.p, w.mem.p, w.mem.bytes(), cudaMemcpyDeviceToDevice, stream_));
    SPD_CUDA(cudaMemcpyAsync(w.lu_snap.p, w.lu.p, w.lu.bytes(), cudaMemcpyDeviceToDevice, stream_));
    w.flush_due = false;
}

// One process, no lanes: the optimizer itself folds the time-encoder
// accumulators and the step's last split-K sums into the gradients (k_adam's
// AdamFin) — two or three fewer launches on the step's critical tail.
bool TGNTrainer::fused_finalize() const { return world_ == 1 && !peer_ && !lane_ && !profile_; }

void TGNTrainer::allreduce_grads(cudaStream_t st) {
    // time-encoder grads (f64 accumulators) into the flat buffer first
    if (!fused_finalize())
        launch(tgnk::k_time_grad_apply, blocks_for(lay_.T), 256, 0, st,
               lay_.T, tgrad_.p, grads_.p + lay_.time_w, grads_.p + lay_.time_b);
    SPD_CUDA(cudaGetLastError());
    if (world_ > 1 && !peer_) {  // (the peer transport sums inside its Adam kernel)
        SPD_NCCL(ncclAllReduce(grads_.p, grads_.p, lay_.total, ncclFloat, ncclSum,
                               static_cast<ncclComm_t>(nccl_), st));
    }
}

void TGNTrainer::adam_prepare() {
    ++adam_t_;
    const float bc[2] = {static_cast<float>(1.0 - std::pow(double(cfg_.beta1), double(adam_t_))),
                         static_cast<float>(1.0 - std::pow(double(cfg_.beta2), double(adam_t_)))};
    std::memcpy(&ctl_stage_[ctl_stage_.size() - 2], bc, sizeof(bc));
    ctl_stage_.back() = ++peer_seq_;  // the peer transport's step sequence
}

void TGNTrainer::commit_ctl() {
    const int slot = static_cast<int>(ctl_next_++ % kCtlSlots);
    if (ctl_used_[slot]) SPD_CUDA(cudaEventSynchronize(ctl_ev_[slot]));  // its copy ran ~64 steps ago
    std::uint64_t* h = ctl_ring_ + std::size_t(slot) * ctl_stage_.size();
    std::memcpy(h, ctl_stage_.data(), ctl_stage_.size() * sizeof(std::uint64_t));
    SPD_CUDA(cudaMemcpyAsync(ctl_dev_.p, h, ctl_stage_.size() * sizeof(std::uint64_t),
                             cudaMemcpyHostToDevice, stream_));
    SPD_CUDA(cudaEventRecord(ctl_ev_[slot], stream_));
    ctl_used_[slot] = true;
}

void TGNTrainer::adam(cudaStream_t st) {
    const double b1 = cfg_.beta1, b2 = cfg_.beta2;
    if (peer_) {  // all-reduce fused with the update: every rank's gradients read from its HBM
        peer_->adam_step(ctl_dev_.p + ctl_stage_.size() - 1, params_.p, adam_m_.p, adam_v_.p, lay_.total,
                         float(total_workers_), cfg_.lr, cfg_.beta1, static_cast<float>(1.0 - b1),
                         cfg_.beta2, static_cast<float>(1.0 - b2), adam_bc_, cfg_.adam_eps,
                         cfg_.gemm_mode == 1 ? params_tc_.p : nullptr, st);
        return;
    }
    tgnk::AdamFin fin{};
    if (fused_finalize()) {
        fin.tacc = tgrad_.p;
        fin.T = lay_.T;
        fin.tw = lay_.time_w;
        fin.tb = lay_.time_b;
        for (const umma::SplitK& k : fin_sk_) {
            if (k.split <= 1) continue;
            auto& o = fin.sk[fin.nsk++];
            o.ws = k.ws; o.split = k.split; o.M = k.M; o.N = k.N; o.ldws = k.ldws; o.ldc = k.ldc;
            o.off = static_cast<std::size_t>(k.C - grads_.p);
        }
    }
    for (auto& k : fin_sk_) k.split = 0;
    launch(tgnk::k_adam, blocks_for((lay_.total + 3) / 4), 256, 0, st,
        params_.p, grads_.p, adam_m_.p, adam_v_.p, lay_.total, float(total_workers_), cfg_.lr,
        cfg_.beta1, static_cast<float>(1.0 - b1), cfg_.beta2, static_cast<float>(1.0 - b2),
        adam_bc_, cfg_.adam_eps,
        cfg_.gemm_mode == 1 ? params_tc_.p : nullptr, fin);
    SPD_CUDA(cudaGetLastError());
}

void TGNTrainer::set_ctl(Worker& w, std::uint64_t lo, std::uint64_t nb) {
    ctl_stage_[2 * w.ctl_index] = lo;
    ctl_stage_[2 * w.ctl_index + 1] = nb;
}

// Everything a global step launches once the per-step control words are on
// the device: the local workers' batches, the gradient all-reduce and Adam.
// Bs[k] = batch size of local worker k (0: idle). Capturable as a CUDA graph.
void TGNTrainer::step_body(const std::vector<int>& Bs) {
    if (surrogate_) {  // bridge backbone: apply, persist and collect the last messages only
        s_->loss.zero(stream_);
        for (std::size_t k = 0; k < workers_.size(); ++k) {
            if (Bs[k] == 0) continue;
            Worker& w = *workers_[k];
            const tgnk::WorkerDev wd = devview(w);
            w.last_b = Bs[k];
            surrogate_update(w, wd);
            launch(tgnk::k_persist, blocks_for(std::size_t(s_->U) * 32), 256, 0, stream_, wd, lay_.D,
                   s_->mem_new.p);
            launch(tgnk::k_pending, 1, 1024, 0, stream_, wd, Bs[k]);
        }
        return;
    }
    // gradient buffers cleared by a kernel, not memset nodes: in a graph
    // replay a memset node costs a copy-engine hand-off before the first
    // kernel. It runs on its own stream beside the forward (nothing reads or
    // writes the gradients before the backward, which joins it).
    SPD_CUDA(cudaEventRecord(ev_zfork_, stream_));
    SPD_CUDA(cudaStreamWaitEvent(zs_, ev_zfork_, 0));
    {
        Scratch& s = *s_;
        tgnk::ZeroList z{};
        z.p[0] = grads_.p; z.n[0] = lay_.total;
        if (cfg_.gemm_mode == 1) {  // TC weight grads read whole K blocks of dGi/dGh
            z.p[1] = s.dGi.p; z.n[1] = s.dGi.n;
            z.p[2] = s.dGh.p; z.n[2] = s.dGh.n;
        }
        z.d = tgrad_.p; z.nd = std::size_t(2) * ld4(lay_.T);
        std::size_t mx = z.nd;
        for (int k = 0; k < tgnk::ZeroList::kMax; ++k) mx = std::max(mx, z.n[k]);
        // peers read these gradients until they signal DONE for the previous step
        if (peer_) peer_->wait(kDone, ctl_dev_.p + ctl_stage_.size() - 1, -1, zs_);
        launch(tgnk::k_zero_list, std::min<unsigned>(blocks_for(mx), 148), 256, 0, zs_, z);
        scratch_zeroed_ = true;  // the first backward of this step skips its own zeroing
    }
    SPD_CUDA(cudaEventRecord(ev_zero_, zs_));
    if (fold_o_ || fold_q_) side([&](cudaStream_t sd) {  // the step's Wc / Wqk, beside the memory update
        if (fold_o_) build_wc(sd);
        if (fold_q_) build_wqk(sd);
        SPD_CUDA(cudaEventRecord(ev_wc_, sd));
    });
    std::size_t last = workers_.size();
    for (std::size_t k = 0; k < workers_.size(); ++k)
        if (Bs[k] > 0) last = k;
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        Worker& w = *workers_[k];
        if (Bs[k] == 0) continue;
        fin_defer_ = k == last && fused_finalize();
        worker_step(w, devview(w), Bs[k], true, static_cast<int>(k), k != last);
        fin_defer_ = false;
        if (debug_) {  // taps before the next worker reuses the scratch
            const std::uint64_t B = w.last_b;
            const int D = lay_.D, K = lay_.Kn;
            w.tap_emb.resize(3 * B * D);
            w.tap_roots.resize(3 * B);
            w.tap_nbr.resize(3 * B * K);
            s_->emb.download(w.tap_emb.data(), w.tap_emb.size(), stream_);
            s_->roots.download(w.tap_roots.data(), w.tap_roots.size(), stream_);
            s_->nbr_node.download(w.tap_nbr.data(), w.tap_nbr.size(), stream_);
            SPD_CUDA(cudaMemcpyAsync(&w.tap_loss, s_->loss.p + k, sizeof(float),
                                     cudaMemcpyDeviceToHost, stream_));
            SPD_CUDA(cudaStreamSynchronize(stream_));
        }
    }
    // the last worker's post phase (memory persist, last messages) and the
    // gradient all-reduce + Adam touch disjoint state: run them side by side
    if (profile_ || last == workers_.size()) {
        if (last != workers_.size()) worker_post_kernels(*workers_[last]);
        if (peer_ || lane_) {  // (peer waits must not block the host: untimed)
            allreduce_grads(stream_);
            if (!lane_) adam(stream_);  // (a lane's Adam is its parent's, tgn_lanes.cu)
            return;
        }
        timed("allreduce", [&] { allreduce_grads(stream_); });
        timed("adam", [&] { adam(stream_); });
        return;
    }
    side([&](cudaStream_t sd) {
        allreduce_grads(sd);
        if (!lane_) adam(sd);
    });
    worker_post_kernels(*workers_[last]);
    join_side();
}

void TGNTrainer::peer_export(unsigned char* out) const {
    if (!lanes_.empty()) usage_error("peer transport: concurrent local workers use an in-process group");
    if (!peer_) usage_error("peer transport: trainer was created with an NCCL id or world 1");
    peer_->export_blob(out);
}

void TGNTrainer::peer_connect(const unsigned char* blobs) {
    if (!lanes_.empty()) usage_error("peer transport: concurrent local workers use an in-process group");
    if (!peer_) usage_error("peer transport: trainer was created with an NCCL id or world 1");
    peer_->connect(blobs);
}

void TGNTrainer::coll(void* data, std::size_t count, int type, int op, cudaStream_t st) {
    if (world_ < 2 || count == 0) return;
    if (peer_) {
        peer_->allreduce(data, count, type, op, st);
        return;
    }
    const ncclDataType_t t = type == kF64 ? ncclDouble : type == kI32 ? ncclInt32 : ncclFloat;
    const ncclRedOp_t o = op == kOpMin ? ncclMin : op == kOpMax ? ncclMax : ncclSum;
    SPD_NCCL(ncclAllReduce(data, data, count, t, o, static_cast<ncclComm_t>(nccl_), st));
}

void TGNTrainer::step(float* loss_out) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_step(loss_out);
        return;
    }
    if (peer_ && !peer_->connected())
        usage_error("peer transport not connected (spd_tgn_peer_export / spd_tgn_peer_connect)");
    ++step_in_epoch_;
    times_.ms.clear();
    std::vector<int> Bs(workers_.size(), 0);
    bool full = true;
    for (std::size_t k = 0; k < workers_.size(); ++k) {
        Worker& w = *workers_[k];
        if (w.batches == 0) continue;
        const std::uint64_t lo = w.pos * cfg_.batch_size;
        Bs[k] = static_cast<int>(std::min<std::uint64_t>(w.E, lo + cfg_.batch_size) - lo);
        full = full && Bs[k] == static_cast<int>(cfg_.batch_size);
        if (w.pos == 0) {  // loop_start: reset (pac_sim.cpp:238)
            w.mem.zero(stream_);
            w.lu.zero(stream_);
            for (auto& ps : w.pend) ps.nU.zero(stream_);
        }
        set_ctl(w, lo, neg_base(cfg_.seed_neg, std::uint64_t(epoch_), std::uint64_t(w.gid),
                                step_in_epoch_));
    }
    adam_prepare();
    commit_ctl();
    // one graph per pending-set parity (the sets' pointers are baked in); all
    // active workers flip together on full-batch steps
    int par = -1;
    bool same_par = true;
    for (std::size_t k = 0; k < workers_.size(); ++k)
        if (Bs[k] > 0) {
            if (par < 0) par = workers_[k]->cur;
            same_par = same_par && workers_[k]->cur == par;
        }
    // capture only after one eager full step (lazy attribute setup done)
    const bool graph_ok = use_graph_ && full && same_par && par >= 0 && !profile_ && !debug_ &&
                          eager_full_steps_ > 0;
    if (!graph_ok && full) ++eager_full_steps_;
    if (graph_ok) {
        // regular step: replay the captured graph (launch-free, fork/join of
        // the side stream preserved); capture it on first use
        cudaGraphExec_t& graph_exec = graph_exec_[par];
        if (!graph_exec) {
            const std::uint64_t k0 = kernel_launches();
            cudaGraph_t graph;
            SPD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            step_body(Bs);
            SPD_CUDA(cudaStreamEndCapture(stream_, &graph));
            SPD_CUDA(cudaGraphInstantiate(&graph_exec, graph, 0));
            SPD_CUDA(cudaGraphDestroy(graph));
            graph_kernels_ = kernel_launches() - k0;
            g_kernel_launches.fetch_sub(graph_kernels_, std::memory_order_relaxed);
        }
        SPD_CUDA(cudaGraphLaunch(graph_exec, stream_));
        g_kernel_launches.fetch_add(graph_kernels_, std::memory_order_relaxed);
    } else {
        step_body(Bs);
    }
    for (auto& wp : workers_)
        if (wp->batches > 0) worker_post(*wp);
    if (loss_out) {
        std::vector<float> l(workers_.size());
        s_->loss.download(l.data(), l.size(), stream_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
        for (std::size_t k = 0; k < l.size(); ++k)
            loss_out[k] = workers_[k]->batches > 0 ? l[k] : std::nanf("");
    }
}

void TGNTrainer::end_epoch(bool wait) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_end_epoch(wait);
        return;
    }
    for (auto& wp : workers_) {  // drop partial loops (pac_sim.cpp:259)
        Worker& w = *wp;
        SPD_CUDA(cudaMemcpyAsync(w.mem.p, w.mem_snap.p, w.mem.bytes(), cudaMemcpyDeviceToDevice, stream_));
        SPD_CUDA(cudaMemcpyAsync(w.lu.p, w.lu_snap.p, w.lu.bytes(), cudaMemcpyDeviceToDevice, stream_));
        for (auto& ps : w.pend) ps.nU.zero(stream_);
    }
    sync_shared(wait);
    if (wait) SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::run_epoch(int epoch, double* mean_loss) {
    begin_epoch(epoch);
    std::vector<float> l(lanes_.empty() ? workers_.size() : lanes_.size());
    double sum = 0.0;
    std::uint64_t n = 0;
    for (std::uint64_t k = 0; k < epoch_steps_; ++k) {
        step(mean_loss ? l.data() : nullptr);
        if (mean_loss)
            for (float v : l)
                if (!std::isnan(v)) {
                    sum += v;
                    ++n;
                }
    }
    end_epoch();
    if (mean_loss) *mean_loss = n ? sum / double(n) : 0.0;
}

// ---------------------------------------------------------- introspection
void TGNTrainer::get_params(float* out) const {
    DeviceGuard g(device_);
    if (!lanes_.empty()) return lanes_[0]->get_params(out);  // replicas are bit-identical
    SPD_CUDA(cudaStreamSynchronize(stream_));
    params_.download(out, lay_.total, stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
}
void TGNTrainer::refresh_tc_weights() {
    launch(tgnk::k_round_tf32, blocks_for(lay_.total), 256, 0, stream_, params_.p, params_tc_.p,
           lay_.total);
}

void TGNTrainer::set_gemm_mode(int mode) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_wait();
        for (auto& l : lanes_) l->set_gemm_mode(mode);
        cfg_.gemm_mode = mode;
        return;
    }
    SPD_CUDA(cudaStreamSynchronize(stream_));
    for (auto& ge : graph_exec_)
        if (ge) {
            SPD_CUDA(cudaGraphExecDestroy(ge));
            ge = nullptr;
        }
    eager_full_steps_ = 0;
    cfg_.gemm_mode = mode;
    s_->d.rnd = mode == 1 ? 1 : 0;
    refresh_tc_weights();
    // the TC weight-gradient GEMMs read whole K blocks of the gate gradients
    s_->dGi.zero(stream_);
    s_->dGh.zero(stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::set_params(const float* in) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {
        lanes_wait();
        for (auto& l : lanes_) l->set_params(in);
        return;
    }
    params_.upload(in, lay_.total, stream_);
    refresh_tc_weights();
    SPD_CUDA(cudaStreamSynchronize(stream_));
}
void TGNTrainer::get_grads(float* out) const {
    DeviceGuard g(device_);
    if (!lanes_.empty()) {  // each lane holds its own worker's gradient: mean in lane order
        std::vector<float> sum(lay_.total, 0.f), one(lay_.total);
        for (auto& l : lanes_) {
            SPD_CUDA(cudaStreamSynchronize(l->stream_));
            l->grads_.download(one.data(), lay_.total, l->stream_);
            SPD_CUDA(cudaStreamSynchronize(l->stream_));
            for (std::size_t i = 0; i < lay_.total; ++i) sum[i] += one[i];
        }
        for (std::size_t i = 0; i < lay_.total; ++i) out[i] = sum[i] / float(total_workers_);
        return;
    }
    SPD_CUDA(cudaStreamSynchronize(stream_));
    grads_.download(out, lay_.total, stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
    // the buffer holds the all-reduced SUM; report the applied mean
    for (std::size_t i = 0; i < lay_.total; ++i) out[i] /= float(total_workers_);
}
void TGNTrainer::get_memory(int wid, float* mem, double* lu) {
    if (!lanes_.empty()) return lane_of(wid)->get_memory(wid, mem, lu);
    Worker& w = worker(wid);
    DeviceGuard g(device_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
    if (mem) w.mem.download(mem, std::size_t(w.N) * lay_.D, stream_);
    if (lu) w.lu.download(lu, w.N, stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
}
void TGNTrainer::set_memory(int wid, const float* mem, const double* lu) {
    if (!lanes_.empty()) return lane_of(wid)->set_memory(wid, mem, lu);
    Worker& w = worker(wid);
    DeviceGuard g(device_);
    if (mem) w.mem.upload(mem, std::size_t(w.N) * lay_.D, stream_);
    if (lu) w.lu.upload(lu, w.N, stream_);
    SPD_CUDA(cudaStreamSynchronize(stream_));
}
std::size_t TGNTrainer::debug_scratch(const char* name, float* out, std::size_t cap) {
    DeviceGuard g(device_);
    if (!lanes_.empty()) return lanes_[0]->debug_scratch(name, out, cap);
    Scratch& s = *s_;
    const std::string n(name ? name : "");
    const DevBuf<float>* b = n == "x_gru" ? &s.x_gru : n == "h_gru" ? &s.h_gru : n == "Gi" ? &s.Gi
                             : n == "Gh" ? &s.Gh : n == "mem_new" ? &s.mem_new : n == "gsave" ? &s.gsave
                             : nullptr;
    if (!b) usage_error("unknown scratch buffer '" + n + "'");
    if (out) {
        SPD_CUDA(cudaDeviceSynchronize());
        b->download(out, std::min(cap, b->n), stream_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
    }
    return b->n;
}

void TGNTrainer::last_step(int wid, std::uint64_t* b, float* emb, std::uint32_t* negs,
                           std::uint32_t* nbr, float* loss) {
    if (!lanes_.empty()) return lane_of(wid)->last_step(wid, b, emb, negs, nbr, loss);
    Worker& w = worker(wid);
    if (!debug_) usage_error("debug taps are off (spd_tgn_set_debug)");
    const std::uint64_t B = w.last_b;
    if (b) *b = B;
    if (emb) std::copy(w.tap_emb.begin(), w.tap_emb.end(), emb);
    if (loss) *loss = w.tap_loss;
    if (negs)
        for (std::uint64_t i = 0; i < B; ++i) negs[i] = w.nodes[w.tap_roots[2 * B + i]];
    if (nbr)
        for (std::size_t k = 0; k < w.tap_nbr.size(); ++k)
            nbr[k] = w.tap_nbr[k] == tgnk::kPad ? 0xFFFFFFFFu : w.nodes[w.tap_nbr[k]];
}

// ----------------------------------------------------- shared-node sync
// Epoch-end sync of SEP's shared hubs (pac_sim.cpp:162-203) across every
// worker — local workers in order, then NCCL across processes. Average:
// mean row + max clock, skipped where all copies agree bit for bit; max-ts:
// the freshest copy, ties to the lowest worker id.
namespace {
__global__ void k_sync_pack(const float* mem, const double* lu, const std::uint32_t* rows, int S,
                            int D, int first, float* sum, float* mn, float* mx, double* ts_max) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)S * (D + 1)) return;
    const int sidx = i / (D + 1), c = i % (D + 1);
    const std::uint32_t r = rows[sidx];
    if (c == D) {
        const double t = r == 0xFFFFFFFFu ? 0.0 : lu[r];
        ts_max[sidx] = first ? t : fmax(ts_max[sidx], t);
        // clock agreement travels as min/max of the f64 clock in mn/mx tail
        return;
    }
    const float v = r == 0xFFFFFFFFu ? 0.f : mem[(std::size_t)r * D + c];
    const std::size_t o = (std::size_t)sidx * D + c;
    if (first) {
        sum[o] = v;
        mn[o] = v;
        mx[o] = v;
    } else {
        sum[o] = sum[o] + v;
        mn[o] = fminf(mn[o], v);
        mx[o] = fmaxf(mx[o], v);
    }
}
__global__ void k_sync_fill(float* mn, float* mx, std::size_t n, double* tmin, double* tmax,
                            int S) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        mn[i] = FLT_MAX;
        mx[i] = -FLT_MAX;
    }
    if (i < (std::size_t)S) {
        tmin[i] = INFINITY;
        tmax[i] = -INFINITY;
    }
}
__global__ void k_sync_ts_minmax(const double* lu, const std::uint32_t* rows, int S, int first,
                                 double* tmin, double* tmax) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const double t = rows[i] == 0xFFFFFFFFu ? 0.0 : lu[rows[i]];
    tmin[i] = first ? t : fmin(tmin[i], t);
    tmax[i] = first ? t : fmax(tmax[i], t);
}
__global__ void k_sync_apply_avg(float* mem, double* lu, const std::uint32_t* rows, int S, int D,
                                 const float* sum, const float* mn, const float* mx,
                                 const double* tmin, const double* tmax, float inv_w) {
    pdl_entry();
    const int sidx = blockIdx.x;
    if (sidx >= S) return;
    const std::uint32_t r = rows[sidx];
    if (r == 0xFFFFFFFFu) return;
    __shared__ int disagree;
    if (threadIdx.x == 0) disagree = tmin[sidx] != tmax[sidx];
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += blockDim.x)
        if (mn[(std::size_t)sidx * D + c] != mx[(std::size_t)sidx * D + c]) disagree = 1;
    __syncthreads();
    if (!disagree) return;
    for (int c = threadIdx.x; c < D; c += blockDim.x)
        mem[(std::size_t)r * D + c] = sum[(std::size_t)sidx * D + c] * inv_w;
    if (threadIdx.x == 0) lu[r] = tmax[sidx];
}
__global__ void k_sync_owner(const double* lu, const std::uint32_t* rows, int S, const double* tmax,
                             int gid, int* owner) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const double t = rows[i] == 0xFFFFFFFFu ? 0.0 : lu[rows[i]];
    if (t == tmax[i] && gid < owner[i]) owner[i] = gid;
}
__global__ void k_sync_owner_pack(const float* mem, const std::uint32_t* rows, int S, int D,
                                  const int* owner, int gid, float* sum) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)S * D) return;
    const int sidx = i / D, c = i % D;
    if (owner[sidx] != gid) return;
    const std::uint32_t r = rows[sidx];
    sum[i] = r == 0xFFFFFFFFu ? 0.f : mem[(std::size_t)r * D + c];
}
__global__ void k_sync_apply_max(float* mem, double* lu, const std::uint32_t* rows, int S, int D,
                                 const float* rowv, const double* tmax) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (std::size_t)S * D) return;
    const int sidx = i / D, c = i % D;
    const std::uint32_t r = rows[sidx];
    if (r == 0xFFFFFFFFu) return;
    mem[(std::size_t)r * D + c] = rowv[i];
    if (c == 0) lu[r] = tmax[sidx];
}
}  // namespace

void TGNTrainer::sync_shared(bool wait) {
    if (lane_) return;  // (the parent syncs every lane's worker, tgn_lanes.cu)
    std::vector<Worker*> ws;
    for (auto& w : workers_) ws.push_back(w.get());
    sync_workers(ws, stream_);
    if (wait) SPD_CUDA(cudaStreamSynchronize(stream_));
}

// The shared-hub sync over `wlist` (this process's workers, in worker order),
// then across ranks (coll), on stream st.
void TGNTrainer::sync_workers(const std::vector<Worker*>& wlist, cudaStream_t st) {
    const int S = static_cast<int>(shared_.size());
    if (total_workers_ < 2 || S == 0) return;
    const int D = lay_.D;
    // persistent buffers: no allocation (and no cudaFree's device-wide sync)
    // while the collectives' peer waits are in flight
    auto& SB = syncbuf_;
    if (SB.sum.n != std::size_t(S) * D) {
        SB.sum.alloc(std::size_t(S) * D); SB.mn.alloc(std::size_t(S) * D); SB.mx.alloc(std::size_t(S) * D);
        SB.tmin.alloc(S); SB.tmax.alloc(S); SB.owner.alloc(S);
    }
    if (SB.rows.size() != wlist.size()) {
        SB.rows.clear();
        SB.rows.resize(wlist.size());
        for (std::size_t k = 0; k < wlist.size(); ++k) {
            SB.rows[k].alloc(S);
            SB.rows[k].upload(wlist[k]->shared_local.data(), S, st);
        }
    }
    auto& sum = SB.sum; auto& mn = SB.mn; auto& mx = SB.mx; auto& tmin = SB.tmin; auto& tmax = SB.tmax;
    auto& rows = SB.rows;
    // local reduction in worker order (the reference's summation order)
    const bool have_local = !wlist.empty();
    if (!have_local) {  // identities of sum / min / max, so the collectives see only the peers
        sum.zero(st);
        launch(k_sync_fill, blocks_for(mn.n), 256, 0, st, mn.p, mx.p, mn.n, tmin.p, tmax.p, S);
    }
    for (std::size_t k = 0; k < wlist.size(); ++k) {
        Worker& w = *wlist[k];
        launch(k_sync_pack, blocks_for(std::size_t(S) * (D + 1)), 256, 0, st, 
            w.mem.p, w.lu.p, rows[k].p, S, D, k == 0, sum.p, mn.p, mx.p, tmax.p);
        launch(k_sync_ts_minmax, blocks_for(S), 256, 0, st, w.lu.p, rows[k].p, S, k == 0, tmin.p, tmax.p);
    }
    SPD_CUDA(cudaGetLastError());
    if (cfg_.sync_average) {
        if (world_ > 1 && !peer_) SPD_NCCL(ncclGroupStart());
        coll(sum.p, sum.n, kF32, kOpSum, st);
        coll(mn.p, mn.n, kF32, kOpMin, st);
        coll(mx.p, mx.n, kF32, kOpMax, st);
        coll(tmin.p, S, kF64, kOpMin, st);
        coll(tmax.p, S, kF64, kOpMax, st);
        if (world_ > 1 && !peer_) SPD_NCCL(ncclGroupEnd());
        for (std::size_t k = 0; k < wlist.size(); ++k) {
            Worker& w = *wlist[k];
            launch(k_sync_apply_avg, S, 128, 0, st, w.mem.p, w.lu.p, rows[k].p, S, D, sum.p, mn.p, mx.p,
                                                tmin.p, tmax.p, 1.f / float(total_workers_));
        }
    } else {
        coll(tmax.p, S, kF64, kOpMax, st);
        auto& owner = SB.owner;
        SPD_CUDA(cudaMemsetAsync(owner.p, 0x7F, owner.bytes(), st));
        for (std::size_t k = 0; k < wlist.size(); ++k)
            launch(k_sync_owner, blocks_for(S), 256, 0, st, wlist[k]->lu.p, rows[k].p, S, tmax.p,
                                                        wlist[k]->gid, owner.p);
        coll(owner.p, S, kI32, kOpMin, st);
        sum.zero(st);
        for (std::size_t k = 0; k < wlist.size(); ++k)
            launch(k_sync_owner_pack, blocks_for(std::size_t(S) * D), 256, 0, st, 
                wlist[k]->mem.p, rows[k].p, S, D, owner.p, wlist[k]->gid, sum.p);
        coll(sum.p, sum.n, kF32, kOpSum, st);
        for (std::size_t k = 0; k < wlist.size(); ++k)
            launch(k_sync_apply_max, blocks_for(std::size_t(S) * D), 256, 0, st, 
                wlist[k]->mem.p, wlist[k]->lu.p, rows[k].p, S, D, sum.p, tmax.p);
    }
    SPD_CUDA(cudaGetLastError());
}

namespace {
// per-node time-sorted CSR over both directions of a time-ordered event list
// (ties keep event order, src side first: the oracle's (ts, event, role) order)
void build_adj(const std::vector<std::uint32_t>& src, const std::vector<std::uint32_t>& dst,
               const std::vector<double>& ts, NodeId N, std::vector<std::uint64_t>& off,
               std::vector<std::uint32_t>& nbr, std::vector<std::uint32_t>& ev,
               std::vector<double>& ats) {
    const std::uint64_t E = src.size();
    off.assign(std::size_t(N) + 1, 0);
    for (std::uint64_t k = 0; k < E; ++k) {
        ++off[src[k] + 1];
        ++off[dst[k] + 1];
    }
    for (NodeId i = 0; i < N; ++i) off[i + 1] += off[i];
    std::vector<std::uint64_t> fill(off.begin(), off.end() - 1);
    nbr.resize(2 * E);
    ev.resize(2 * E);
    ats.resize(2 * E);
    for (std::uint64_t k = 0; k < E; ++k) {
        std::uint64_t q = fill[src[k]]++;
        nbr[q] = dst[k]; ev[q] = static_cast<std::uint32_t>(k); ats[q] = ts[k];
        q = fill[dst[k]]++;
        nbr[q] = src[k]; ev[q] = static_cast<std::uint32_t>(k); ats[q] = ts[k];
    }
}
}  // namespace

void TGNTrainer::set_eval_events(int wid, const spd_edge* e, const std::uint64_t* eids,
                                 std::uint64_t n) {
    if (!lanes_.empty()) {
        lanes_wait();
        return lane_of(wid)->set_eval_events(wid, e, eids, n);
    }
    Worker& w = worker(wid);
    DeviceGuard g(device_);
    const std::uint64_t E = w.E, Et = E + n;
    if (Et > 0xFFFFFFFFull) data_error("InvalidParams", "partition exceeds 2^32 events");
    std::vector<std::uint32_t> src(Et), dst(Et);
    std::vector<double> ts(Et);
    for (std::uint64_t k = 0; k < E; ++k) {
        src[k] = w.ev_host[k].src;
        dst[k] = w.ev_host[k].dst;
        ts[k] = w.ev_host[k].ts;
    }
    auto loc = [&](NodeId gid) -> std::uint32_t {
        auto it = std::lower_bound(w.nodes.begin(), w.nodes.end(), gid);
        if (it == w.nodes.end() || *it != gid)
            data_error("InvalidPartition", "eval edge endpoint outside the partition (route with "
                                           "assign_eval_edges)");
        return static_cast<std::uint32_t>(it - w.nodes.begin());
    };
    for (std::uint64_t k = 0; k < n; ++k) {
        src[E + k] = loc(e[k].src);
        dst[E + k] = loc(e[k].dst);
        ts[E + k] = e[k].ts;
        if (ts[E + k] < ts[E + k - (E + k > 0 ? 1 : 0)])
            data_error("NonChronological", "eval edges must follow the training events in time");
    }
    std::vector<std::uint64_t> off;
    std::vector<std::uint32_t> nbr, ev;
    std::vector<double> ats;
    build_adj(src, dst, ts, w.N, off, nbr, ev, ats);
    std::vector<std::uint32_t> pool(dst);
    std::sort(pool.begin(), pool.end());
    pool.erase(std::unique(pool.begin(), pool.end()), pool.end());
    if (pool.empty()) pool.push_back(0);
    w.x_n_pool = static_cast<std::uint32_t>(pool.size());
    w.x_src.alloc(Et); w.x_src.upload(src.data(), Et, stream_);
    w.x_dst.alloc(Et); w.x_dst.upload(dst.data(), Et, stream_);
    w.x_ts.alloc(Et); w.x_ts.upload(ts.data(), Et, stream_);
    w.x_adj_off.alloc(off.size()); w.x_adj_off.upload(off.data(), off.size(), stream_);
    w.x_adj_nbr.alloc(2 * Et); w.x_adj_nbr.upload(nbr.data(), 2 * Et, stream_);
    w.x_adj_ev.alloc(2 * Et); w.x_adj_ev.upload(ev.data(), 2 * Et, stream_);
    w.x_adj_ts.alloc(2 * Et); w.x_adj_ts.upload(ats.data(), 2 * Et, stream_);
    w.x_pool.alloc(pool.size()); w.x_pool.upload(pool.data(), pool.size(), stream_);
    const int Fp = s_->d.Fp, F = lay_.F;
    w.x_feat.alloc(std::max<std::uint64_t>(1, Et) * std::max(1, Fp));
    if (Fp && E)
        SPD_CUDA(cudaMemcpyAsync(w.x_feat.p, w.feat.p, E * Fp * sizeof(__nv_bfloat16),
                                 cudaMemcpyDeviceToDevice, stream_));
    if (Fp && n) {
        DevBuf<std::uint64_t> de(n);
        de.upload(eids, n, stream_);
        launch(tgnk::k_gen_features, blocks_for(n * Fp), 256, 0, stream_, w.x_feat.p + E * Fp, de.p,
               n, F, Fp, feat_seed_mixed_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
    }
    w.E_eval = n;
    SPD_CUDA(cudaStreamSynchronize(stream_));
}

void TGNTrainer::evaluate(int wid, std::uint64_t lo, std::uint64_t hi, std::uint64_t neg_seed,
                          float* pos, float* neg) {
    if (!lanes_.empty()) {
        lanes_wait();
        return lane_of(wid)->evaluate(wid, lo, hi, neg_seed, pos, neg);
    }
    Worker& w = worker(wid);
    if (hi > w.E_eval || lo > hi) usage_error("eval range outside the eval events");
    DeviceGuard g(device_);
    auto eval_view = [&] {
        tgnk::WorkerDev v = devview(w);
        v.ev_src = w.x_src.p; v.ev_dst = w.x_dst.p; v.ev_ts = w.x_ts.p; v.feat = w.x_feat.p;
        v.adj_off = w.x_adj_off.p; v.adj_nbr = w.x_adj_nbr.p; v.adj_ev = w.x_adj_ev.p;
        v.adj_ts = w.x_adj_ts.p; v.pool = w.x_pool.p; v.n_pool = w.x_n_pool;
        return v;
    };
    int slot_idx = 0;
    for (std::size_t k = 0; k < workers_.size(); ++k)
        if (workers_[k].get() == &w) slot_idx = static_cast<int>(k);
    if (fold_o_ || fold_q_) {
        if (fold_o_) build_wc(stream_);
        if (fold_q_) build_wqk(stream_);
        SPD_CUDA(cudaEventRecord(ev_wc_, stream_));
    }
    std::vector<float> lg;
    for (std::uint64_t b0 = lo; b0 < hi; b0 += cfg_.batch_size) {
        const int B = static_cast<int>(std::min<std::uint64_t>(hi, b0 + cfg_.batch_size) - b0);
        set_ctl(w, w.E + b0, neg_base(neg_seed, 0xE7A1ull, std::uint64_t(w.gid), b0));
        commit_ctl();
        worker_step(w, eval_view(), B, false, slot_idx);
        w.cur ^= 1;
        lg.resize(2 * B);
        s_->logits.download(lg.data(), 2 * B, stream_);
        SPD_CUDA(cudaStreamSynchronize(stream_));
        std::copy(lg.begin(), lg.begin() + B, pos + (b0 - lo));
        std::copy(lg.begin() + B, lg.end(), neg + (b0 - lo));
    }
}

}  // namespace spd
