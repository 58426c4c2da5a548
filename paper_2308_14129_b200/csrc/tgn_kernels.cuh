// Non-GEMM kernels of the TGN step. Each
// is memory/latency bound: warp-per-row gathers with the row's columns
// spread over lanes (coalesced 4-byte lanes, 16-byte for bf16x8 features),
// f64 time phases, deterministic fixed-order reductions where a parameter
// gradient is summed.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spd {
namespace tgnk {

constexpr std::uint32_t kPad = 0xFFFFFFFFu;

struct Dims {
    int D, T, F, Fp, DQ, DK, DM, H, K;
    int ld_x, ld_h, ld_q, ld_kv, ld_ctx, ld_m, ld_z, ld_din, ld_d1;  // aug strides
    int ld_g;  // 3D rounded
    int ld_Q;   // row stride of Q/dQ/dctx (DQ), a 128-B multiple
    int ld_p;   // per-head row width of Qp/xbar/dxbar/dQp: ld_aug(DK) (tgn_attn.cu)
    int rnd;          // round tensor-core operands to tf32 (round-to-nearest) at production
};

struct WorkerDev {
    const std::uint32_t* ev_src;
    const std::uint32_t* ev_dst;
    const double* ev_ts;
    const __nv_bfloat16* feat;
    const std::uint64_t* adj_off;
    const std::uint32_t* adj_nbr;
    const std::uint32_t* adj_ev;
    const double* adj_ts;
    const std::uint32_t* pool;
    std::uint32_t n_pool;
    float* mem;
    double* lu;
    std::int32_t* slot;
    std::int32_t* lastpos;
    std::uint32_t* pU;
    std::uint32_t* pOther;
    std::uint32_t* pEv;
    double* pTs;
    std::int32_t* nU;
    // the other pending set, written by k_pending with this batch's messages
    std::uint32_t* nxU;
    std::uint32_t* nxOther;
    std::uint32_t* nxEv;
    double* nxTs;
    std::int32_t* nxN;
    // DyRep: the other endpoint's attention embedding of each pending message
    // (current set, read by the gather) and of the set k_pending fills
    const float* pZ;
    float* nxZ;
    // per-step control written by the host before each step (stream-ordered,
    // so a captured CUDA graph replays with fresh values): [0] first event of
    // the batch, [1] negative-sampling base (oracle: negatives())
    const std::uint64_t* ctl;
};

// Index of the step's memory-row readers for the deterministic dH reduction
// (tgn_dh.cu). Entries: occurrence e = r * K + j for e < RK, then (from block
// nb_occ on) root r = e - nb_occ * kDhBlock.
constexpr int kDhBlock = 1024;  // entries per histogram / scatter block
constexpr int kDhChunk = 16;    // entries per pull warp
struct DhIndex {
    int RK, K, R, nb_occ, nb_root, U_cap;
    const std::uint32_t* nbr_node;
    const int* cnt;
    const std::uint32_t* roots;
    int* hist;          // [nb_occ + nb_root][U_cap] -> per-block exclusive prefixes
    int* off_occ;       // [U_cap + 1] occurrence list offsets per slot
    int* off_root;      // [U_cap + 1] root list offsets per slot
    int* chunk_off;     // [U_cap + 1] first occurrence chunk per slot
    int* rchunk_off;    // [U_cap + 1] first root chunk per slot
    int* chunk_slot;    // [max occurrence chunks] slot of the chunk
    int* chunk_start;   //                         first list position
    int* rchunk_slot;   // [max root chunks]
    int* rchunk_start;
    int* list_occ;      // [RK]
    int* list_root;     // [R]
};
__global__ void k_dh_hist(WorkerDev w, DhIndex x);
__global__ void k_dh_colscan(DhIndex x);
__global__ void k_dh_scan(DhIndex x);
__global__ void k_dh_scatter(WorkerDev w, DhIndex x);
template <int NM, int HMAX>
__global__ void k_dh_pull(DhIndex x, Dims d, const float* alpha, const float* dsc,
                          const float* dxbar, const float* Qp, float* partial);
template <int NM>
__global__ void k_dh_pull_root(DhIndex x, Dims d, const float* dq_in, const float* dm_in,
                               float* rpartial);
template <int NM>
__global__ void k_gru_bwd_dh(WorkerDev w, Dims d, DhIndex x, const float* partial,
                             const float* rpartial, const float* save, float* dGi, float* dGh);
template <int NM>
__global__ void k_rnn_bwd_dh(WorkerDev w, Dims d, DhIndex x, const float* partial,
                             const float* rpartial, const float* save, float* dGi, float* dGh);


// --- kernels (definitions in tgn_kernels.cu) -------------------------------
__global__ void k_init_aug(float* buf, int rows, int cols, int ld);
__global__ void k_zero2(float* a, std::size_t na, double* b, std::size_t nb);
struct ZeroList {
    static constexpr int kMax = 4;
    float* p[kMax];
    std::size_t n[kMax];
    double* d;
    std::size_t nd;
};
__global__ void k_zero_list(ZeroList z);
__global__ void k_roots_nbrs(WorkerDev w, int B, int K,
                             std::uint32_t* roots, double* root_t, std::uint32_t* nbr_node,
                             std::uint32_t* nbr_ev, double* nbr_dt, int* cnt);
__global__ void k_gru_gather(WorkerDev w, Dims d, const float* time_w, const float* time_b,
                             float* x, float* h, int set_slot);
__global__ void k_gru_fwd(WorkerDev w, Dims d, const float* Gi, const float* Gh, const float* h,
                          float* save, float* mem_new);
__global__ void k_query_gather(WorkerDev w, Dims d, int R, const float* time_w,
                               const float* time_b, const std::uint32_t* roots,
                               const float* mem_new, float* q_in, float* m_in);
// absorbed-projection attention (tgn_attn.cu): 4 roots per 128-thread block,
// dynamic shared memory attn_smem_bytes(d, bwd); lane slots per region
// NM = ceil(D / 128), NT = ceil(T / 128), NF = ceil((F + 1) / 128); HMAX >= H
__host__ __device__ std::size_t attn_smem_bytes(const Dims& d, bool bwd);
int attn_roots_per_block();
int attn_x_roots_per_block();
template <int NM, int NT, int NF, int HMAX>
__global__ void k_attn_abs_fwd(WorkerDev w, Dims d, int R, const float* time_w,
                               const float* time_b, const std::uint32_t* nbr_node,
                               const std::uint32_t* nbr_ev, const double* nbr_dt, const int* cnt,
                               const float* mem_new, const float* Qp, float* alpha, float* xbar);
template <int NM, int NT, int NF, int HMAX>
__global__ void k_attn_abs_bwd(WorkerDev w, Dims d, int R, const float* time_w,
                               const float* time_b, const std::uint32_t* nbr_node,
                               const std::uint32_t* nbr_ev, const double* nbr_dt, const int* cnt,
                               const float* mem_new, const float* Qp, const float* alpha,
                               const float* dxbar, float* dQp, float* dsc);
template <int NT, int HMAX>
__global__ void k_attn_time_grad(Dims d, int R, const float* time_w, const float* time_b,
                                 const double* nbr_dt, const int* cnt, const float* Qp,
                                 const float* alpha, const float* dsc, const float* dxbar,
                                 double* part);
__global__ void k_merge_gather(WorkerDev w, Dims d, int R, const std::uint32_t* roots,
                               const int* cnt, const float* O, const float* mem_new, float* m_in);
__global__ void k_dec_gather(Dims d, int B, const float* emb, float* d_in);
__global__ void k_dec_head(Dims d, int B, const float* D1, const float* w2, float* dlogit,
                           float* lossv, float* dD1, float* logits);
__global__ void k_dec_head2(Dims d, int B, const float* Ya, const float* Yb, const float* W1,
                            int ld1, const float* w2, float* D1, float* dlogit, float* lossv,
                            float* dD1, float* logits);
constexpr int kDecEv = 8;       // events per k_decoder block
constexpr int kDecEvSmall = 4;  // ... for batches of <= kDecSmallB events (twice the blocks)
constexpr int kDecSmallB = 1024;
// k_decoder launches roundup(4 d_mem, 32) threads (<= 768: d_mem <= 192)
template <int MAXT, int MINB, int EV>
__global__ void k_decoder(Dims d, int B, const float* emb, const float* W1, int ld1, const float* w2,
                          float* D1, float* dlogit, float* lossv, float* dD1, float* logits,
                          float* d_emb, int bwd, int pre);
std::size_t decoder_smem_bytes(const Dims& d, int ev);
// k_dec_wgrad_part: events per block and per shared-memory tile (128-event
// blocks — 16 long-running blocks — took 176 us on the side stream and moved
// the Wiki test AUC from 0.0028 to 0.0050 off the oracle: the chunk order
// is part of the numerics)
constexpr int kDecWgEv = 32;
constexpr int kDecWgTile = 32;
__global__ void k_dec_wgrad_part(Dims d, int B, const float* emb, const float* dD1, const float* dlogit,
                                 const float* D1, float* part);
__global__ void k_dec_wgrad_reduce(Dims d, int nblk, const float* part, float* g1, int ld1, float* g2);
std::size_t dec_wgrad_smem_bytes(const Dims& d);
__global__ void k_sum_loss(const float* lossv, int n, float* out);
__global__ void k_dec_scatter(Dims d, int B, const float* dd_in, float* d_emb);
__global__ void k_mask_rows(float* buf, int R, int cols, int ld, const int* cnt);
__global__ void k_root_grad(Dims d, int R, const float* dq_in, const float* time_b,
                            int rows_per_block, double* part);
__global__ void k_time_grad_final(int T, int nblocks, const double* part, double* acc);
__global__ void k_time_grad_apply(int T, const double* acc, float* gw, float* gb);
// Gradient terms not yet in the flat buffer when the optimizer runs on one
// process (tgn_trainer.cu adam): the time-encoder f64 accumulators and up to
// two deferred split-K weight gradients (fixed-order partial sums).
struct AdamFin {
    const double* tacc = nullptr;  // [2T]: d time_w then d time_b (null: none)
    int T = 0;
    std::size_t tw = 0, tb = 0;    // their flat offsets
    int nsk = 0;
    struct SK {
        const float* ws;
        int split, M, N, ldws, ldc;
        std::size_t off;           // flat offset of dW
    } sk[2];
};
__global__ void k_adam(float* p, float* g, float* m, float* v, std::size_t n, float scale,
                       float lr, float b1, float one_m_b1, float b2, float one_m_b2, const float* bc,
                       float eps, float* p_tc, AdamFin fin);
__global__ void k_round_tf32(const float* src, float* dst, std::size_t n);
struct GradList {
    const float* g[8];
    int n;
};
__global__ void k_adam_multi(float* p, GradList gl, float* m, float* v, std::size_t n, float scale,
                             float lr, float b1, float one_m_b1, float b2, float one_m_b2, const float* bc,
                             float eps, float* p_tc);
__global__ void k_persist(WorkerDev w, int D, const float* mem_new);
__global__ void k_pending(WorkerDev w, int B);
__global__ void k_rnn_fwd(WorkerDev w, Dims d, const float* Gi, const float* Gh, float* save, float* mem_new);
__global__ void k_jodie_embed(WorkerDev w, Dims d, int R, const std::uint32_t* roots, const double* root_t,
                              const float* mem_new, const float* tp, int ldtp, float* emb, float* s_out);
__global__ void k_dyrep_stash(WorkerDev w, int D, int B, const float* z);
__global__ void k_wprod_t(float* out, int ldo, int hstride, const float* A, int lda, const float* B, int ldb,
                          int rows, int cols, int dh, int H, int rnd);
__global__ void k_wc_fix(float* wc, int rows, int ld, int DK, const float* b_o, int ld_o, int rnd);
__global__ void k_jodie_bwd(WorkerDev w, Dims d, int R, const std::uint32_t* roots, const float* mem_new,
                            const float* tp, int ldtp, const float* s_in, const float* d_emb, float* dq_in,
                            float* dm_in, int rows_per_block, double* part);
__global__ void k_jodie_tp_final(int D, int nblk, const double* part, float* g, int ldtp);
__global__ void k_surrogate_update(WorkerDev w, int D, const double* w_m, const double* omega,
                                   double gamma, float* mem_new);
__global__ void k_gen_features(__nv_bfloat16* feat, const std::uint64_t* eids, std::uint64_t E,
                               int F, int Fp, std::uint64_t seed_mixed);
__global__ void k_gather_rows(const float* src, int ld, const std::uint32_t* idx,
                              std::uint32_t n, int cols, float* out);

}  // namespace tgnk
}  // namespace spd
