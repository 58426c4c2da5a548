// TGN training hot path on sm_100a: the per-partition memory-based TIG
// training step of SPEED, one or more SEP partitions
// (workers) per process/device, gradients all-reduced over NCCL every global
// step, shared hubs synced at epoch end. Semantics: oracle/tgn_oracle.py.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "cuda_util.hpp"
#include "host.hpp"
#include "peer_comm.hpp"
#include "tgn_kernels.cuh"
#include "umma_host.hpp"

namespace spd {

inline int ld4(int cols) { return (cols + 3) / 4 * 4; }
// Row strides of every matrix a GEMM streams are whole 128-B lines (32 f32):
// TMA boxes and FFMA tiles then touch each L2 line once.
inline int ld32(int cols) { return (cols + 31) / 32 * 32; }
inline int ld_aug(int cols) { return ld32(cols + 1); }  // [x | 1 | pad]

// Flat parameter buffer: every linear layer is an augmented [W | b] matrix
// (row stride ld_aug(K)); tensors start at 4-float boundaries.
struct ParamLayout {
    struct Lin { int N, K, ld; std::size_t off; };
    Lin gru_ih, gru_hh, att_q, att_kv, att_o, mrg1, mrg2, dec1, dec2, tproj;
    std::size_t time_w, time_b;
    std::size_t total;
    int D, T, F, DQ, DK, DM, H, Kn;
    int backbone = 0;  // 0 TGN, 1 JODIE (RNN rows, no attention/merge, time projection)
    void build(int d_mem, int d_time, int d_edge, int heads, int k, int backbone);
};

struct StepTimes {
    std::vector<std::pair<std::string, float>> ms;
};

class TGNTrainer;

// One SEP partition's static data + dynamic state on the device.
struct Worker {
    int gid = 0;                     // global worker / partition id
    NodeId N = 0;                    // local nodes
    std::uint64_t E = 0;             // training events
    std::vector<NodeId> nodes;       // local -> global (ascending)
    std::vector<spd_edge> ev_host;   // local ids
    // static device data
    DevBuf<std::uint32_t> ev_src, ev_dst;
    DevBuf<double> ev_ts;
    DevBuf<__nv_bfloat16> feat;      // E x Fp
    DevBuf<std::uint64_t> adj_off;   // N + 1
    DevBuf<std::uint32_t> adj_nbr, adj_ev;
    DevBuf<double> adj_ts;
    DevBuf<std::uint32_t> pool;      // destination nodes (negatives)
    std::uint32_t n_pool = 0;
    // dynamic state
    DevBuf<float> mem, mem_snap;     // N x D
    DevBuf<double> lu, lu_snap;      // N
    DevBuf<std::int32_t> slot;       // N: node -> row of the pending set, -1
    DevBuf<std::int32_t> lastpos;    // N: scratch for last-message selection
    // pending last-message sets (<= 2B each), double-buffered: a step's GRU
    // reads pend[cur] (the previous batch's messages) while k_pending writes
    // this batch's into pend[cur ^ 1]; cur flips after the step
    struct PendingSet {
        DevBuf<std::uint32_t> pU, pOther, pEv;
        DevBuf<double> pTs;
        DevBuf<float> pZ;         // DyRep: the other endpoint's attention embedding (<= 2B x D)
        DevBuf<std::int32_t> nU;  // device-resident |pending|
    } pend[2];
    int cur = 0;
    std::int32_t* nU() { return pend[cur].nU.p; }
    const std::uint64_t* ctl = nullptr;  // per-step control words in the trainer's block
    int ctl_index = 0;                   // its position in that block
    std::vector<std::uint32_t> shared_local;  // local row of each shared node (or UINT32_MAX)
    // schedule
    std::uint64_t batches = 0, pos = 0, loops = 0;
    bool done = false;
    bool flush_due = false;  // (lanes) loop ended: flush + snapshot after the group Adam
    double last_loss = 0.0;
    std::uint64_t last_b = 0;
    // evaluation view: train + eval events, their features and full-graph CSR
    std::uint64_t E_eval = 0;
    DevBuf<std::uint32_t> x_src, x_dst, x_adj_nbr, x_adj_ev, x_pool;
    DevBuf<double> x_ts, x_adj_ts;
    DevBuf<__nv_bfloat16> x_feat;
    DevBuf<std::uint64_t> x_adj_off;
    std::uint32_t x_n_pool = 0;
    // debug taps of the last step (filled only when TGNTrainer::debug_ is set)
    std::vector<float> tap_emb;
    std::vector<std::uint32_t> tap_roots, tap_nbr;
    float tap_loss = 0.f;
};

struct Scratch;  // per-step activations (sized for one batch)

// The training stream resident on the device for shuffle-combine
// re-induction (tgn_induce.cu): SoA events, per-node small-part bitmasks and
// the per-edge "induced by some small part" flags (for `recovered`).
struct DevStream {
    std::uint64_t E = 0;
    NodeId N = 0;
    int n_small = 0, words = 0;
    DevBuf<std::uint32_t> src, dst;
    DevBuf<double> ts;
    DevBuf<std::uint64_t> bits;  // N x words
    DevBuf<std::uint8_t> in_small;
};

std::uint64_t kernel_launches();  // process-wide count of TGN-path kernel launches
int debug_gemm(int impl, int which, const float* A, int lda, const float* B, int ldb, float* C,
               int ldc, int M, int N, int K, float* ws, std::size_t ws_cap);

class TGNTrainer {
public:
    TGNTrainer(const spd_tgn_config& cfg, const SubGraphs& subs, const std::vector<int>& workers,
               const std::vector<NodeId>& shared, NodeId node_count, int rank, int world,
               const void* nccl_id, int device);
    ~TGNTrainer();

    std::uint64_t epoch_steps() const { return epoch_steps_; }
    bool concurrent() const { return !lanes_.empty(); }
    std::uint64_t batch_size() const { return cfg_.batch_size; }
    void begin_epoch(int epoch);
    void seek(std::uint64_t step);
    void rebind(const SubGraphs& subs);
    void step_host_async(const spd_edge* const* events, const std::uint16_t* const* feats,
                         float* loss_pinned);
    void sync();  // shuffle-combine: next epoch's regrouped subgraphs
    void step(float* loss_out);
    void end_epoch(bool wait = true);
    void run_epoch(int epoch, double* mean_loss);
    // Evaluation events (routed val then test edges, global ids, time-ordered)
    // appended after the worker's training events: the full-graph neighbour
    // finder and feature rows cover train + eval events.
    void set_eval_events(int worker, const spd_edge* e, const std::uint64_t* eids,
                         std::uint64_t n);
    // Score eval events [lo, hi) in batches (positives + one sampled negative
    // each) and advance the memory through them; no gradients.
    void evaluate(int worker, std::uint64_t lo, std::uint64_t hi, std::uint64_t neg_seed,
                  float* pos, float* neg);

    std::size_t param_count() const { return lay_.total; }
    void get_params(float* out) const;
    void set_params(const float* in);
    void get_grads(float* out) const;
    Worker& worker(int w);
    void get_memory(int w, float* mem, double* lu);
    void set_memory(int w, const float* mem, const double* lu);
    // copy of a per-step scratch buffer (debugging / tests): names x_gru,
    // h_gru, Gi, Gh, mem_new, gsave; returns the element count
    std::size_t debug_scratch(const char* name, float* out, std::size_t cap);
    void last_step(int w, std::uint64_t* b, float* emb, std::uint32_t* negs, std::uint32_t* nbr,
                   float* loss);
    const StepTimes& times() const { return lanes_.empty() ? times_ : lanes_[0]->times_; }
    float run_steps(std::uint64_t n);
    // peer-memory transport (world > 1 without an NCCL id, peer_comm.hpp):
    // every rank exports its blob, the caller exchanges them, every rank connects
    bool peer_mode() const { return peer_ != nullptr; }
    // Bridge backbone: the reference's surrogate MSG/UPD
    // (pac_sim.cpp:50-104) replaces the GRU in this trainer's schedule; steps
    // apply the pending messages only (no embedding, loss, gradients)
    void set_surrogate(int d, const double* w_m, const double* omega, double gamma);
    // Shuffle-combine on the device (tgn_induce.cu): keep the training stream
    // and the small SEP parts in HBM, then re-induce every epoch's regrouped
    // worker subgraphs there (pac_sim.cpp:134-160, :280-329)
    void attach_stream(const spd_edge* e, std::uint64_t n, NodeId node_count, const std::uint64_t* off,
                       const NodeId* nodes, int n_small);
    void shuffle_epoch(std::uint64_t seed, std::uint64_t* recovered);
    void peer_export(unsigned char* out) const;
    void peer_connect(const unsigned char* blobs);
    void step_host(const spd_edge* const* events, const std::uint16_t* const* feats,
                   float* loss_out);
    std::uint64_t h2d_bytes() const {
        std::uint64_t n = h2d_bytes_;
        for (auto& l : lanes_) n += l->h2d_bytes_;
        return n;
    }
    std::uint64_t d2h_bytes() const {
        std::uint64_t n = d2h_bytes_;
        for (auto& l : lanes_) n += l->d2h_bytes_;
        return n;
    }
    std::uint64_t step_in_epoch() const { return lanes_.empty() ? step_in_epoch_ : lanes_[0]->step_in_epoch_; }
    int epoch() const { return lanes_.empty() ? epoch_ : lanes_[0]->epoch_; }
    int feat_stride() const;
    void set_debug(bool on) {
        debug_ = on;
        for (auto& l : lanes_) l->set_debug(on);
    }
    void set_profile(bool on) {
        profile_ = on;
        for (auto& l : lanes_) l->set_profile(on);
    }
    void set_graph(bool on) {
        use_graph_ = on;
        for (auto& l : lanes_) l->set_graph(on);
    }
    void set_gemm_mode(int mode);
    int device() const { return device_; }
    cudaStream_t stream() const { return lanes_.empty() ? stream_ : lanes_[0]->stream_; }
    float* loss_dev() const;  // device per-local-worker loss slots

private:
    void build_workers(const SubGraphs& subs, const std::vector<int>& ids);
    // concurrent local workers (tgn_lanes.cu): one child trainer per worker
    std::vector<std::unique_ptr<TGNTrainer>> lanes_;
    void build_lanes(const SubGraphs& subs, const std::vector<int>& workers, NodeId node_count);
    TGNTrainer* lane_of(int gid);
    void lanes_wait();
    void lanes_after(cudaEvent_t ev);
    void lanes_join();
    void lanes_losses(float* loss_out);
    void lanes_step(float* loss_out);
    void lanes_adam_step();
    void lanes_end_epoch(bool wait);
    float lanes_run_steps(std::uint64_t n);
    std::vector<cudaEvent_t> lane_end_;
    cudaEvent_t lanes_adam_ = nullptr;  // lane 0's point after the parent's Adam (or sync)
    bool lanes_adam_valid_ = false;
    void init_worker_state(Worker& w);  // memory, clocks, pending sets, shared-row map
    std::unique_ptr<DevStream> dstream_;
    void worker_step(Worker& w, const tgnk::WorkerDev& wd, int B, bool train, int slot_idx,
                     bool post = true);
    void worker_post_kernels(Worker& w);
    // Per-step control words (every worker's batch start and negative base,
    // Adam's bias corrections) are staged host-side by set_ctl / adam_prepare
    // and shipped as one block by commit_ctl from a ring of pinned slots
    // (asynchronous, stream-ordered: graph replays see fresh values and the
    // host never waits for the device).
    void set_ctl(Worker& w, std::uint64_t lo, std::uint64_t nb);
    void commit_ctl();
    void step_body(const std::vector<int>& Bs);  // worker steps + all-reduce + Adam (capturable)
    void adam_prepare();
    void backward(Worker& w, const tgnk::WorkerDev& wd, int B);
    void decode(int B, bool train);                // k_decoder (fwd, loss, data gradient)
    void decoder_wgrads(cudaEvent_t at, int B);    // decoder weight gradients (side streams)
    void jodie_rest(Worker& w, const tgnk::WorkerDev& wd, int B, bool train, int slot_idx, bool post);
    void dyrep_messages(const tgnk::WorkerDev& wd, int B, bool train);
    void worker_post(Worker& w);
    void loop_end_flush(Worker& w);
    void flush_pending(Worker& w);
    void gru_forward(Worker& w, const tgnk::WorkerDev& wd, bool train,
                     const std::function<void()>& after_gather = {});
    void allreduce_grads(cudaStream_t st);
    void adam(cudaStream_t st);
    void sync_shared(bool wait = true);
    void sync_workers(const std::vector<Worker*>& wlist, cudaStream_t st);
    bool lane_ = false;  // a lane of a concurrent parent: no Adam, no shared sync of its own
    void timed(const char* name, const std::function<void()>& f);
    // weight-gradient GEMMs run on a side stream forked from the main stream at
    // the point their inputs exist, and joined back once per worker step
    void side(const std::function<void(cudaStream_t)>& f, int which = -1);
    // Critical-path-first issue order: mark() records a point of the main
    // stream; side_from(mark, f) forks side work from that point AFTER the
    // main stream's next kernels were created, so graph replays submit the
    // critical-path kernel first and it claims SMs before the side work.
    cudaEvent_t mark();
    void side_from(cudaEvent_t at, const std::function<void(cudaStream_t)>& f);
    static constexpr int kMarks = 32;
    cudaEvent_t marks_[kMarks] = {};
    int mark_next_ = 0;
    void join_side();
    // Side streams: independent off-critical-path work (weight gradients, the
    // neighbour search, Adam) is spread round-robin over kSide streams, each
    // with its own slice of the split-K workspace, and joined where needed.
    static constexpr int kSide = 4;
    cudaStream_t sides_[kSide] = {};
    cudaEvent_t ev_join_[kSide] = {};
    bool side_used_[kSide] = {};
    int side_next_ = 0;
    cudaStream_t side_ = nullptr;  // == sides_[0]: the neighbour-search / time-encoding stream
    cudaEvent_t ev_fork_ = nullptr;
    float* ws_cur_ = nullptr;      // workspace slice of the side task being issued
    std::size_t wsn_cur_ = 0;
    // a second fork for the GRU's hidden-side gate GEMM, and the points of the
    // side stream the main stream waits for (neighbours found, dH index built)
    cudaStream_t aux_ = nullptr;
    cudaEvent_t ev_aux_fork_ = nullptr, ev_aux_join_ = nullptr, ev_roots_ = nullptr,
                ev_dhidx_ = nullptr;
    // gradient zeroing forked at step start beside the forward; the backward
    // (first gradient writer) joins it
    cudaStream_t zs_ = nullptr;
    cudaEvent_t ev_zfork_ = nullptr, ev_zero_ = nullptr;
    cudaEvent_t ev_bwdx_ = nullptr;  // attention time-encoder partials done
    cudaEvent_t ev_pull_ = nullptr;  // dH chunk partials done (tgn_dh.cu)
    cudaEvent_t ev_pend_ = nullptr;  // (DyRep) this batch's last messages selected
    cudaEvent_t ev_wc_ = nullptr;    // the step's folded output x value projection built
    cudaEvent_t ev_ctx_ = nullptr;   // ctx (dW_o's input) computed beside the folded O GEMM
    bool fold_o_ = false;
    DevBuf<float> wc_;               // DQ x H ld_p (build_wc)
    void build_wc(cudaStream_t sx);
    cudaEvent_t ev_q_ = nullptr;     // Q (dW_K's input) computed beside the folded Qp GEMM
    bool fold_q_ = false;
    DevBuf<float> wqk_;              // (DQ + 1) x H ld_p (build_wqk)
    void build_wqk(cudaStream_t sx);
    // deferred split-K sums of the step's last GRU weight gradients (fused_finalize)
    umma::SplitK fin_sk_[2];
    bool fin_defer_ = false;
    bool fused_finalize() const;
    bool scratch_zeroed_ = false;    // dGi/dGh cleared by this step's k_zero_list
    bool gru_fused_ = true;          // gemm_mode 1: fused tcgen05 GRU (SPD_GRU_FUSED=0: two GEMMs + cell)

    spd_tgn_config cfg_;
    ParamLayout lay_;
    int device_ = 0, rank_ = 0, world_ = 1;
    int total_workers_ = 1;
    cudaStream_t stream_ = nullptr;
    void* nccl_ = nullptr;  // ncclComm_t
    std::unique_ptr<PeerComm> peer_;  // peer-memory transport instead of NCCL
    struct SyncBufs {  // epoch-end shared-hub sync scratch (persistent)
        DevBuf<float> sum, mn, mx;
        DevBuf<double> tmin, tmax;
        DevBuf<int> owner;
        std::vector<DevBuf<std::uint32_t>> rows;  // per local worker; cleared when workers change
    } syncbuf_;
    bool surrogate_ = false;          // bridge backbone (set_surrogate)
    DevBuf<double> sur_w_, sur_om_;
    double sur_gamma_ = 0.0;
    void surrogate_update(Worker& w, const tgnk::WorkerDev& wd);
    // world > 1 collective over ranks (NCCL or the peer transport), in place
    void coll(void* data, std::size_t count, int type, int op, cudaStream_t st);
    std::uint64_t peer_seq_ = 0;  // global steps issued (the step protocol's sequence)
    std::vector<std::unique_ptr<Worker>> workers_;
    std::vector<std::uint64_t> all_batches_;  // per global worker
    std::uint64_t epoch_steps_ = 0, step_in_epoch_ = 0, adam_t_ = 0;
    int epoch_ = 0;
    std::vector<NodeId> shared_;
    DevBuf<float> params_, grads_, adam_m_, adam_v_;
    DevBuf<float> params_tc_;  // tf32-rounded copy read by the tensor-core GEMMs
    DevBuf<std::uint64_t> ctl_dev_;  // [2 per worker | Adam bias corrections (2 x f32) | step seq]
    std::vector<std::uint64_t> ctl_stage_;
    static constexpr int kCtlSlots = 64;
    std::uint64_t* ctl_ring_ = nullptr;  // pinned [kCtlSlots][ctl words]
    cudaEvent_t ctl_ev_[kCtlSlots] = {};
    bool ctl_used_[kCtlSlots] = {};
    std::uint64_t ctl_next_ = 0;
    const float* adam_bc_ = nullptr;
    // CUDA graph of the regular step (every local worker on a full batch)
    cudaGraphExec_t graph_exec_[2] = {};  // one per pending-set parity
    std::uint64_t graph_kernels_ = 0;
    bool use_graph_ = true;
    std::uint64_t eager_full_steps_ = 0;
    void refresh_tc_weights();
    DevBuf<double> tgrad_;  // f64 accumulators for the time encoder grads (2T)
    std::unique_ptr<Scratch> s_;
    StepTimes times_;
    bool profile_ = false;
    bool debug_ = false;
    unsigned char* stage_ = nullptr;  // pinned
    std::size_t stage_bytes_ = 0;
    // pipelined end-to-end steps (step_host_async): a ring of pinned SoA
    // staging slots, their copies on their own stream, one event per slot
    static constexpr int kStageSlots = 3;
    unsigned char* aring_[kStageSlots] = {};
    std::size_t aring_bytes_ = 0;
    cudaEvent_t aring_ev_[kStageSlots] = {};
    bool aring_used_[kStageSlots] = {};
    int aring_next_ = 0;
    cudaStream_t copy_ = nullptr;
    // the steps those copies fed: end-of-step event and each worker's window,
    // so a copy never overwrites a window an in-flight step still reads
    cudaEvent_t astep_ev_[kStageSlots] = {};
    std::vector<std::uint64_t> astep_lo_[kStageSlots];
    void check_host_events(const Worker& w, std::uint64_t lo, std::uint64_t B,
                           const spd_edge* e) const;
    std::uint64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
    std::uint64_t feat_seed_mixed_ = 0;
};

}  // namespace spd
