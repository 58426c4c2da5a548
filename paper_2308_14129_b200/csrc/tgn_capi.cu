// extern "C" entry points of the TGN training hot path (include/speed_c.h).
#include <cstring>
#include <vector>

#include "capi_types.hpp"
#include "nccl_dyn.hpp"
#include "tgn.hpp"
#include "tgn_common.cuh"

using namespace spd;

struct spd_tgn_trainer {
    std::unique_ptr<TGNTrainer> t;
};

extern "C" {

spd_status spd_nccl_unique_id(void* out128) {
    GUARD({
        ncclUniqueId id;
        SPD_NCCL(NcclApi::get().GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out128, &id, sizeof(id));
    });
}

spd_status spd_tgn_create(const spd_tgn_config* cfg, const spd_subgraphs* subs,
                          const int32_t* workers, int32_t n_workers, const uint32_t* shared,
                          uint64_t n_shared, uint32_t node_count, int32_t rank, int32_t world,
                          const void* nccl_id, int32_t device, spd_tgn_trainer** out) {
    GUARD({
        if (!cfg || !subs || !out) usage_error("null argument");
        std::vector<int> ws(workers, workers + n_workers);
        std::vector<NodeId> sh(shared, shared + n_shared);
        auto h = std::make_unique<spd_tgn_trainer>();
        h->t = std::make_unique<TGNTrainer>(*cfg, subs->s, ws, sh, node_count, rank, world,
                                            nccl_id, device);
        *out = h.release();
    });
}

void spd_tgn_destroy(spd_tgn_trainer* t) { delete t; }

spd_status spd_tgn_set_surrogate(spd_tgn_trainer* t, int32_t d, const double* w_m,
                                 const double* omega, double gamma) {
    GUARD({
        if (!t || !w_m || !omega) usage_error("null argument");
        t->t->set_surrogate(d, w_m, omega, gamma);
    });
}

spd_status spd_tgn_attach_stream(spd_tgn_trainer* t, const spd_edge* e, uint64_t n, uint32_t node_count,
                                 const uint64_t* small_off, const uint32_t* small_nodes, int32_t n_small) {
    GUARD({
        if (!t || (n && !e) || !small_off || !small_nodes) usage_error("null argument");
        t->t->attach_stream(e, n, node_count, small_off, small_nodes, n_small);
    });
}
spd_status spd_tgn_shuffle_epoch(spd_tgn_trainer* t, uint64_t epoch_seed, uint64_t* recovered) {
    GUARD({
        if (!t) usage_error("null argument");
        t->t->shuffle_epoch(epoch_seed, recovered);
    });
}

uint64_t spd_tgn_peer_blob_bytes(void) { return PeerComm::kBlobBytes; }
spd_status spd_tgn_peer_export(const spd_tgn_trainer* t, void* out) {
    GUARD({
        if (!t || !out) usage_error("null argument");
        t->t->peer_export(static_cast<unsigned char*>(out));
    });
}
spd_status spd_tgn_peer_connect(spd_tgn_trainer* t, const void* blobs) {
    GUARD({
        if (!t || !blobs) usage_error("null argument");
        t->t->peer_connect(static_cast<const unsigned char*>(blobs));
    });
}

spd_status spd_tgn_epoch_steps(const spd_tgn_trainer* t, uint64_t* steps) {
    GUARD({ *steps = t->t->epoch_steps(); });
}
spd_status spd_tgn_begin_epoch(spd_tgn_trainer* t, int32_t epoch) {
    GUARD({ t->t->begin_epoch(epoch); });
}
spd_status spd_tgn_seek(spd_tgn_trainer* t, uint64_t step) { GUARD({ t->t->seek(step); }); }
spd_status spd_tgn_rebind(spd_tgn_trainer* t, const spd_subgraphs* subs) {
    GUARD({
        if (!t || !subs) usage_error("null argument");
        t->t->rebind(subs->s);
    });
}
spd_status spd_tgn_step(spd_tgn_trainer* t, float* loss_out) { GUARD({ t->t->step(loss_out); }); }
spd_status spd_tgn_end_epoch(spd_tgn_trainer* t) { GUARD({ t->t->end_epoch(); }); }
spd_status spd_tgn_run_epoch(spd_tgn_trainer* t, int32_t epoch, double* mean_loss) {
    GUARD({ t->t->run_epoch(epoch, mean_loss); });
}
spd_status spd_tgn_set_eval_events(spd_tgn_trainer* t, int32_t worker, const spd_edge* e,
                                   const uint64_t* eids, uint64_t n) {
    GUARD({ t->t->set_eval_events(worker, e, eids, n); });
}
spd_status spd_tgn_evaluate(spd_tgn_trainer* t, int32_t worker, uint64_t lo, uint64_t hi,
                            uint64_t neg_seed, float* pos_scores, float* neg_scores) {
    GUARD({ t->t->evaluate(worker, lo, hi, neg_seed, pos_scores, neg_scores); });
}
spd_status spd_tgn_param_count(const spd_tgn_trainer* t, uint64_t* n) {
    GUARD({ *n = t->t->param_count(); });
}
spd_status spd_tgn_get_params(const spd_tgn_trainer* t, float* out) {
    GUARD({ t->t->get_params(out); });
}
spd_status spd_tgn_set_params(spd_tgn_trainer* t, const float* in) {
    GUARD({ t->t->set_params(in); });
}
spd_status spd_tgn_get_grads(const spd_tgn_trainer* t, float* out) {
    GUARD({ t->t->get_grads(out); });
}
spd_status spd_tgn_local_nodes(const spd_tgn_trainer* t, int32_t worker, uint64_t* n,
                               uint32_t* global_ids) {
    GUARD({
        Worker& w = t->t->worker(worker);
        if (n) *n = w.N;
        if (global_ids) std::copy(w.nodes.begin(), w.nodes.end(), global_ids);
    });
}
spd_status spd_tgn_get_memory(const spd_tgn_trainer* t, int32_t worker, float* mem,
                              double* last_update) {
    GUARD({ t->t->get_memory(worker, mem, last_update); });
}
spd_status spd_tgn_set_memory(spd_tgn_trainer* t, int32_t worker, const float* mem,
                              const double* last_update) {
    GUARD({ t->t->set_memory(worker, mem, last_update); });
}
spd_status spd_tgn_set_debug(spd_tgn_trainer* t, int32_t on) { GUARD({ t->t->set_debug(on != 0); }); }
spd_status spd_tgn_set_graph(spd_tgn_trainer* t, int32_t on) { GUARD({ t->t->set_graph(on != 0); }); }
spd_status spd_tgn_debug_scratch(spd_tgn_trainer* t, const char* name, float* out, uint64_t cap,
                                 uint64_t* n) {
    GUARD({
        const std::size_t m = t->t->debug_scratch(name, out, cap);
        if (n) *n = m;
    });
}
spd_status spd_tgn_set_gemm_mode(spd_tgn_trainer* t, int32_t mode) {
    GUARD({
        if (mode != 0 && mode != 1) usage_error("gemm_mode must be 0 or 1");
        t->t->set_gemm_mode(mode);
    });
}
spd_status spd_tgn_set_profile(spd_tgn_trainer* t, int32_t on) {
    GUARD({ t->t->set_profile(on != 0); });
}
spd_status spd_tgn_last_step(const spd_tgn_trainer* t, int32_t worker, uint64_t* b, float* emb,
                             uint32_t* negs, uint32_t* nbr_ids, float* loss) {
    GUARD({ t->t->last_step(worker, b, emb, negs, nbr_ids, loss); });
}
spd_status spd_tgn_kernel_times(const spd_tgn_trainer* t, float* ms, int32_t* n_kernels,
                                char* names, int32_t name_stride, int32_t cap) {
    GUARD({
        const auto& v = t->t->times().ms;
        const int n = std::min<int>(cap, static_cast<int>(v.size()));
        for (int k = 0; k < n; ++k) {
            ms[k] = v[k].second;
            if (names && name_stride > 0) {
                std::strncpy(names + std::size_t(k) * name_stride, v[k].first.c_str(),
                             std::size_t(name_stride - 1));
                names[std::size_t(k) * name_stride + name_stride - 1] = 0;
            }
        }
        *n_kernels = n;
    });
}

spd_status spd_tgn_run_steps(spd_tgn_trainer* t, uint64_t n, float* device_ms) {
    GUARD({
        const float ms = t->t->run_steps(n);
        if (device_ms) *device_ms = ms;
    });
}
spd_status spd_tgn_step_host(spd_tgn_trainer* t, const spd_edge* const* events,
                             const uint16_t* const* feats, float* loss_out) {
    GUARD({ t->t->step_host(events, feats, loss_out); });
}
spd_status spd_tgn_step_host_async(spd_tgn_trainer* t, const spd_edge* const* events,
                                   const uint16_t* const* feats, float* loss_pinned) {
    GUARD({ t->t->step_host_async(events, feats, loss_pinned); });
}
spd_status spd_tgn_sync(spd_tgn_trainer* t) { GUARD({ t->t->sync(); }); }
spd_status spd_tgn_next_batch(const spd_tgn_trainer* t, int32_t worker, uint64_t* lo,
                              uint64_t* hi, int32_t* feat_stride) {
    GUARD({
        Worker& w = t->t->worker(worker);
        TGNTrainer& tr = *t->t;
        std::uint64_t pos = w.pos;
        if (tr.step_in_epoch() >= tr.epoch_steps()) pos = 0;  // next call wraps the epoch
        const std::uint64_t B = tr.batch_size();
        *lo = pos * B;
        *hi = std::min<std::uint64_t>(w.E, *lo + B);
        if (feat_stride) *feat_stride = tr.feat_stride();
    });
}
spd_status spd_tgn_worker_events(const spd_tgn_trainer* t, int32_t worker, spd_edge* out) {
    GUARD({
        Worker& w = t->t->worker(worker);
        std::copy(w.ev_host.begin(), w.ev_host.end(), out);
    });
}
spd_status spd_tgn_worker_event_count(const spd_tgn_trainer* t, int32_t worker, uint64_t* n) {
    GUARD({
        if (!t || !n) usage_error("null argument");
        *n = t->t->worker(worker).E;
    });
}
spd_status spd_tgn_io_bytes(const spd_tgn_trainer* t, uint64_t* h2d, uint64_t* d2h) {
    GUARD({
        *h2d = t->t->h2d_bytes();
        *d2h = t->t->d2h_bytes();
    });
}
uint64_t spd_kernel_launches(void) { return kernel_launches(); }

spd_status spd_debug_gemm(int32_t impl, int32_t which, const float* A, int32_t lda, const float* B,
                          int32_t ldb, float* C, int32_t ldc, int32_t M, int32_t N, int32_t K,
                          float* ws, uint64_t ws_floats) {
    GUARD({ debug_gemm(impl, which, A, lda, B, ldb, C, ldc, M, N, K, ws, ws_floats); });
}

spd_status spd_edge_features_bf16(uint64_t seed, const uint64_t* eids, uint64_t n, int32_t F,
                                  int32_t stride, uint16_t* out) {
    GUARD({
        if (F < 0 || stride < F) usage_error("need 0 <= F <= stride");
        const std::uint64_t sm = mix64(seed);
        for (std::uint64_t e = 0; e < n; ++e)
            for (int32_t c = 0; c < stride; ++c) {
                const float v = c < F ? edge_feature_value(sm, eids[e], std::uint32_t(c)) : 0.f;
                std::uint32_t bits;
                std::memcpy(&bits, &v, 4);
                out[e * stride + c] = static_cast<std::uint16_t>(bits >> 16);  // exact in bf16
            }
    });
}

float spd_edge_feature(uint64_t seed, uint64_t eid, uint32_t c) {
    return edge_feature_value(mix64(seed), eid, c);
}

}  // extern "C"
