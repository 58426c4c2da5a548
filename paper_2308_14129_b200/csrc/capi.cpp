// extern "C" boundary (include/speed_c.h): host partitioner / subgraph API and
// the surrogate parity path. Exceptions never cross; they become spd_status +
// a thread-local (code, detail) pair, mirroring DataError/InternalError.
#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "capi_types.hpp"
#include "host.hpp"
#include "surrogate.hpp"

using namespace spd;

namespace {
thread_local std::string g_code;
thread_local std::string g_detail;
}  // namespace

int spd::guarded_call(const std::function<void()>& f) {
    try {
        f();
        g_code.clear();
        g_detail.clear();
        return SPD_OK;
    } catch (const Error& e) {
        g_code = e.code;
        g_detail = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_code = "OutOfMemory";
        g_detail = "host allocation failed";
        return SPD_INTERNAL;
    } catch (const std::exception& e) {
        g_code = "Exception";
        g_detail = e.what();
        return SPD_INTERNAL;
    }
}

struct spd_memstore {
    std::unique_ptr<MemStore> m;
};

namespace {
Stream stream_of(const spd_edge* e, std::uint64_t n, std::uint32_t node_count, double t_max) {
    if (n && !e) usage_error("null edge pointer");
    Stream s;
    s.e = e;
    s.n = n;
    s.node_count = node_count;
    s.t_max = t_max;
    return s;
}
PartitionerConfig config_of(const spd_partitioner_config* c, std::uint32_t node_count) {
    if (!c) usage_error("null config");
    PartitionerConfig cfg;
    cfg.num_parts = c->num_parts;
    cfg.lambda = c->lambda;
    cfg.epsilon = c->epsilon;
    if (c->cent_count) cfg.cent.assign(c->cent, c->cent + c->cent_count);
    cfg.is_hub.assign(node_count, 0);
    for (std::uint64_t k = 0; k < c->n_hubs; ++k) {
        if (c->hubs[k] >= node_count) data_error("InvalidParams", "hub id out of range");
        cfg.is_hub[c->hubs[k]] = 1;
    }
    cfg.k = c->k;
    return cfg;
}
}  // namespace

extern "C" {

const char* spd_last_error_code(void) { return g_code.c_str(); }
const char* spd_last_error_detail(void) { return g_detail.c_str(); }
const char* spd_version(void) { return "speed-b200 0.1 (sm_100a)"; }

spd_status spd_gen_powerlaw(uint32_t nodes, uint64_t edges, double alpha, uint64_t seed,
                            spd_edge* out, uint32_t* node_count, double* t_max) {
    GUARD({
        gen_powerlaw(nodes, edges, alpha, seed, out);
        if (node_count) *node_count = nodes;
        if (t_max) *t_max = static_cast<double>(edges);
    });
}

spd_status spd_chrono_split(uint64_t n, double f_train, double f_val, uint64_t* n_train,
                            uint64_t* n_val, uint64_t* n_test) {
    GUARD({ chrono_split_sizes(n, f_train, f_val, n_train, n_val, n_test); });
}

spd_status spd_compute_centrality(const spd_edge* e, uint64_t n, uint32_t node_count,
                                  double t_max, double beta, int32_t normalize_ts, double* cent,
                                  double* t_max_out) {
    GUARD({
        double tm = 0.0;
        compute_centrality(stream_of(e, n, node_count, t_max), beta, normalize_ts != 0, cent, &tm);
        if (t_max_out) *t_max_out = tm;
    });
}

spd_status spd_compute_degree_centrality(const spd_edge* e, uint64_t n, uint32_t node_count,
                                         double* cent) {
    GUARD({ compute_degree_centrality(stream_of(e, n, node_count, 0.0), cent); });
}

spd_status spd_select_hubs(const double* cent, uint32_t node_count, double k, int32_t base_all,
                           uint32_t* hubs, uint64_t* n_hubs) {
    GUARD({
        auto h = select_hubs(cent, node_count, k, base_all != 0);
        std::copy(h.begin(), h.end(), hubs);
        *n_hubs = h.size();
    });
}

spd_status spd_partition_stream(const spd_edge* e, uint64_t n, uint32_t node_count,
                                const spd_partitioner_config* cfg, spd_assignment** out) {
    GUARD({
        auto a = std::make_unique<spd_assignment>();
        a->a = partition_stream(stream_of(e, n, node_count, 0.0), config_of(cfg, node_count), false);
        *out = a.release();
    });
}

spd_status spd_partition_unrestricted(const spd_edge* e, uint64_t n, uint32_t node_count,
                                      const spd_partitioner_config* cfg, spd_assignment** out) {
    GUARD({
        auto a = std::make_unique<spd_assignment>();
        a->a = partition_stream(stream_of(e, n, node_count, 0.0), config_of(cfg, node_count), true);
        *out = a.release();
    });
}

spd_status spd_score(uint32_t i, uint32_t j, int32_t p, const spd_partitioner_config* c,
                     const uint64_t* sizes, uint64_t maxsize, uint64_t minsize,
                     uint32_t node_count, const uint64_t* a_off, const int32_t* a_parts,
                     double* out) {
    GUARD({
        PartitionerConfig cfg = config_of(c, node_count);
        if (p < 0 || p >= cfg.num_parts || i >= node_count || j >= node_count)
            data_error("InvalidParams", "score arguments out of range");
        auto has = [&](std::uint32_t x) {
            for (std::uint64_t k = a_off[x]; k < a_off[x + 1]; ++k)
                if (a_parts[k] == p) return true;
            return false;
        };
        // partitioner.cpp:27-42, same operation order as the streaming path
        const double ci = cfg.cent_of(i), cj = cfg.cent_of(j);
        const double sum = ci + cj;
        const double ti = sum > 0.0 ? ci / sum : 0.5;
        const double tj = sum > 0.0 ? cj / sum : 0.5;
        double h = 0.0;
        if (has(i)) h += 1.0 + (1.0 - ti);
        if (has(j)) h += 1.0 + (1.0 - tj);
        const double spread = static_cast<double>(maxsize - minsize);
        const double slack = static_cast<double>(maxsize - sizes[p]);
        *out = h + cfg.lambda * slack / (cfg.epsilon + spread);
    });
}

spd_status spd_assignment_from_parts(uint32_t node_count, int32_t num_parts, const uint64_t* np_off,
                                     const int32_t* np_parts, const int32_t* edge_part,
                                     uint64_t n_edges, uint64_t discards, spd_assignment** out) {
    GUARD({
        if (num_parts < 1) data_error("InvalidParams", "need num_parts >= 1");
        auto a = std::make_unique<spd_assignment>();
        a->a.num_parts = num_parts;
        a->a.node_count = node_count;
        a->a.np_off.assign(np_off, np_off + node_count + 1);
        a->a.np_parts.assign(np_parts, np_parts + np_off[node_count]);
        for (std::uint32_t i = 0; i < node_count; ++i)
            if (np_off[i + 1] - np_off[i] > 1) a->a.shared.push_back(i);
        if (edge_part) a->a.edge_part.assign(edge_part, edge_part + n_edges);
        a->a.discards = discards;
        *out = a.release();
    });
}

void spd_assignment_destroy(spd_assignment* a) { delete a; }

spd_status spd_assignment_info(const spd_assignment* a, int32_t* num_parts, uint32_t* node_count,
                               uint64_t* n_edges, uint64_t* n_shared, uint64_t* discards,
                               uint64_t* np_total, double* k_eff) {
    GUARD({
        if (!a) usage_error("null assignment");
        if (num_parts) *num_parts = a->a.num_parts;
        if (node_count) *node_count = a->a.node_count;
        if (n_edges) *n_edges = a->a.edge_part.size();
        if (n_shared) *n_shared = a->a.shared.size();
        if (discards) *discards = a->a.discards;
        if (np_total) *np_total = a->a.np_parts.size();
        if (k_eff) *k_eff = a->a.k_eff;
    });
}

spd_status spd_assignment_edge_part(const spd_assignment* a, int32_t* out) {
    GUARD({ std::copy(a->a.edge_part.begin(), a->a.edge_part.end(), out); });
}
spd_status spd_assignment_node_parts(const spd_assignment* a, uint64_t* off, int32_t* parts) {
    GUARD({
        std::copy(a->a.np_off.begin(), a->a.np_off.end(), off);
        std::copy(a->a.np_parts.begin(), a->a.np_parts.end(), parts);
    });
}
spd_status spd_assignment_shared(const spd_assignment* a, uint32_t* out) {
    GUARD({ std::copy(a->a.shared.begin(), a->a.shared.end(), out); });
}

spd_status spd_assign_eval_edges(const spd_edge* val, uint64_t n_val, const spd_edge* test,
                                 uint64_t n_test, const spd_assignment* a, spd_eval_routing** out) {
    GUARD({
        auto r = std::make_unique<spd_eval_routing>();
        r->r = assign_eval_edges(stream_of(val, n_val, a->a.node_count, 0.0),
                                 stream_of(test, n_test, a->a.node_count, 0.0), a->a);
        *out = r.release();
    });
}
spd_status spd_eval_routing_counts(const spd_eval_routing* r, int32_t which, uint64_t* counts,
                                   uint64_t* unroutable) {
    GUARD({
        if (which < 0 || which > 1) usage_error("which must be 0 (val) or 1 (test)");
        for (std::size_t p = 0; p < r->r.lists[which].size(); ++p)
            counts[p] = r->r.lists[which][p].size();
        if (unroutable) *unroutable = r->r.unroutable[which];
    });
}
spd_status spd_eval_routing_edges(const spd_eval_routing* r, int32_t which, uint64_t* idx) {
    GUARD({
        if (which < 0 || which > 1) usage_error("which must be 0 (val) or 1 (test)");
        for (const auto& l : r->r.lists[which]) idx = std::copy(l.begin(), l.end(), idx);
    });
}
void spd_eval_routing_destroy(spd_eval_routing* r) { delete r; }

spd_status spd_induce_subgraphs(const spd_edge* e, uint64_t n, uint32_t node_count,
                                const uint64_t* np_off, const int32_t* np_parts, uint32_t np_count,
                                int32_t num_parts, spd_subgraphs** out) {
    GUARD({
        auto s = std::make_unique<spd_subgraphs>();
        s->s = induce_from_node_parts(stream_of(e, n, node_count, 0.0), np_off, np_parts, np_count,
                                      num_parts);
        *out = s.release();
    });
}

spd_status spd_induce_groups(const spd_edge* e, uint64_t n, uint32_t node_count,
                             const uint64_t* group_off, const uint32_t* group_nodes,
                             int32_t n_groups, const uint64_t* small_off,
                             const uint32_t* small_nodes, int32_t n_small, spd_subgraphs** out,
                             uint64_t* recovered) {
    GUARD({
        const Stream s = stream_of(e, n, node_count, 0.0);
        auto sg = std::make_unique<spd_subgraphs>();
        std::vector<std::uint8_t> in_group;
        sg->s = induce_from_groups(s, group_off, group_nodes, n_groups, &in_group);
        if (recovered) {
            *recovered = 0;
            if (small_off && n_small > 0) {
                std::vector<std::uint8_t> in_small;
                induce_from_groups(s, small_off, small_nodes, n_small, &in_small);
                for (std::uint64_t k = 0; k < n; ++k) *recovered += in_group[k] && !in_small[k];
            }
        }
        *out = sg.release();
    });
}

spd_status spd_subgraphs_from_lists(int32_t n, const uint64_t* node_off, const uint32_t* nodes,
                                    const uint64_t* edge_off, const spd_edge* edges,
                                    const uint64_t* eids, spd_subgraphs** out) {
    GUARD({
        if (n < 0) usage_error("negative subgraph count");
        auto sg = std::make_unique<spd_subgraphs>();
        sg->s.g.resize(n);
        for (int32_t p = 0; p < n; ++p) {
            auto& g = sg->s.g[p];
            g.nodes.assign(nodes + node_off[p], nodes + node_off[p + 1]);
            g.edges.assign(edges + edge_off[p], edges + edge_off[p + 1]);
            if (eids) {
                g.eids.assign(eids + edge_off[p], eids + edge_off[p + 1]);
            } else {
                g.eids.resize(g.edges.size());
                for (std::size_t k = 0; k < g.eids.size(); ++k) g.eids[k] = k;
            }
        }
        *out = sg.release();
    });
}

spd_status spd_subgraphs_count(const spd_subgraphs* s, int32_t* count) {
    GUARD({ *count = static_cast<int32_t>(s->s.g.size()); });
}
spd_status spd_subgraph_sizes(const spd_subgraphs* s, int32_t p, uint64_t* n_nodes,
                              uint64_t* n_edges) {
    GUARD({
        if (p < 0 || p >= int32_t(s->s.g.size())) usage_error("subgraph index out of range");
        if (n_nodes) *n_nodes = s->s.g[p].nodes.size();
        if (n_edges) *n_edges = s->s.g[p].edges.size();
    });
}
spd_status spd_subgraph_nodes(const spd_subgraphs* s, int32_t p, uint32_t* out) {
    GUARD({
        if (p < 0 || p >= int32_t(s->s.g.size())) usage_error("subgraph index out of range");
        std::copy(s->s.g[p].nodes.begin(), s->s.g[p].nodes.end(), out);
    });
}
spd_status spd_subgraph_edges(const spd_subgraphs* s, int32_t p, spd_edge* out, uint64_t* eids) {
    GUARD({
        if (p < 0 || p >= int32_t(s->s.g.size())) usage_error("subgraph index out of range");
        if (out) std::copy(s->s.g[p].edges.begin(), s->s.g[p].edges.end(), out);
        if (eids) std::copy(s->s.g[p].eids.begin(), s->s.g[p].eids.end(), eids);
    });
}
void spd_subgraphs_destroy(spd_subgraphs* s) { delete s; }

spd_status spd_shuffle_combine(const uint64_t* small_off, const uint32_t* small_nodes,
                               uint64_t n_small, int32_t num_workers, uint64_t epoch_seed,
                               uint64_t* out_off, uint32_t* out_nodes) {
    GUARD({
        std::vector<std::vector<NodeId>> small(n_small);
        for (std::uint64_t p = 0; p < n_small; ++p)
            small[p].assign(small_nodes + small_off[p], small_nodes + small_off[p + 1]);
        auto g = shuffle_combine(small, num_workers, epoch_seed);
        out_off[0] = 0;
        for (std::size_t k = 0; k < g.size(); ++k) {
            out_nodes = std::copy(g[k].begin(), g[k].end(), out_nodes);
            out_off[k + 1] = out_off[k] + g[k].size();
        }
    });
}

// Alg. 2 lockstep schedule on the host (pac_sim.cpp:215-257 without the model):
// global steps = max_w ceil(|E_w|/B); per step every non-vacuous worker takes one
// batch, looping workers restart. Every rank of a multi-GPU run evaluates this
// identically from the same SEP assignment, so no collective is needed for it.
spd_status spd_lockstep_schedule(const spd_subgraphs* s, uint64_t batch_size, uint64_t* n_steps,
                                 uint64_t* log, uint64_t cap, uint64_t* n_log, uint64_t* batches,
                                 uint64_t* loops) {
    GUARD({
        if (batch_size < 1) data_error("InvalidParams", "need batch_size >= 1");
        const std::size_t W = s->s.g.size();
        std::vector<std::uint64_t> nb(W), lp(W, 0), pos(W, 0);
        std::vector<std::uint8_t> done(W, 0);
        for (std::size_t w = 0; w < W; ++w) {
            nb[w] = (s->s.g[w].edges.size() + batch_size - 1) / batch_size;
            if (nb[w] == 0) {
                lp[w] = 1;
                done[w] = 1;
            }
        }
        std::uint64_t step = 0, k = 0;
        while (!std::all_of(done.begin(), done.end(), [](std::uint8_t f) { return f != 0; })) {
            ++step;
            for (std::size_t w = 0; w < W; ++w) {
                if (nb[w] == 0) continue;
                if (log && k < cap) {
                    log[4 * k + 0] = step;
                    log[4 * k + 1] = w;
                    log[4 * k + 2] = lp[w] + 1;
                    log[4 * k + 3] = pos[w] + 1;
                }
                ++k;
                if (++pos[w] == nb[w]) {
                    ++lp[w];
                    done[w] = 1;
                    pos[w] = 0;
                }
            }
        }
        if (n_steps) *n_steps = step;
        if (n_log) *n_log = std::min(k, cap);
        for (std::size_t w = 0; w < W; ++w) {
            if (batches) batches[w] = nb[w];
            if (loops) loops[w] = lp[w];
        }
    });
}

// ------------------------------------------------------------ surrogate

spd_status spd_model_seeded(int32_t d, uint64_t seed, double* w_m, double* omega, double* gamma) {
    GUARD({
        SurrogateModel m = SurrogateModel::seeded(d, seed);
        std::copy(m.w_m.begin(), m.w_m.end(), w_m);
        std::copy(m.omega.begin(), m.omega.end(), omega);
        if (gamma) *gamma = m.gamma;
    });
}

spd_status spd_memstore_create(uint32_t node_count, int32_t d, int32_t device, spd_memstore** out) {
    GUARD({
        if (d < 1) data_error("InvalidParams", "need memory dimension >= 1");
        auto m = std::make_unique<spd_memstore>();
        m->m = std::make_unique<MemStore>(node_count, d, device);
        *out = m.release();
    });
}
void spd_memstore_destroy(spd_memstore* m) { delete m; }
spd_status spd_memstore_upload(spd_memstore* m, const double* state, const double* last_ts) {
    GUARD({
        DeviceGuard g(m->m->device);
        m->m->state.upload(state, m->m->state.n);
        m->m->last_ts.upload(last_ts, m->m->last_ts.n);
        SPD_CUDA(cudaDeviceSynchronize());
    });
}
spd_status spd_memstore_download(const spd_memstore* m, double* state, double* last_ts) {
    GUARD({
        DeviceGuard g(m->m->device);
        SPD_CUDA(cudaDeviceSynchronize());
        if (state) m->m->state.download(state, m->m->state.n);
        if (last_ts) m->m->last_ts.download(last_ts, m->m->last_ts.n);
        SPD_CUDA(cudaDeviceSynchronize());
    });
}
spd_status spd_memstore_reset(spd_memstore* m) {
    GUARD({
        m->m->reset();
        SPD_CUDA(cudaDeviceSynchronize());
    });
}
spd_status spd_memstore_copy(spd_memstore* dst, const spd_memstore* src) {
    GUARD({
        dst->m->copy_from(*src->m);
        SPD_CUDA(cudaDeviceSynchronize());
    });
}
spd_status spd_memstore_digest(const spd_memstore* m, char* out17) {
    GUARD({
        std::string h = m->m->digest();
        std::memcpy(out17, h.c_str(), 17);
    });
}

static SurrogateModel model_of(int d, const double* w_m, const double* omega, double gamma) {
    SurrogateModel m;
    m.d = d;
    m.gamma = gamma;
    m.w_m.assign(w_m, w_m + std::size_t(d) * 3 * d);
    m.omega.assign(omega, omega + d);
    return m;
}

spd_status spd_model_update(spd_memstore* m, const spd_edge* e, uint64_t n, const double* w_m,
                            const double* omega, double gamma) {
    GUARD({ surrogate_model_update(*m->m, e, n, model_of(m->m->d, w_m, omega, gamma)); });
}

spd_status spd_sync_shared(spd_memstore* const* mems, int32_t W, const uint32_t* shared,
                           uint64_t n_shared, int32_t average) {
    GUARD({
        std::vector<MemStore*> ms(W);
        for (int w = 0; w < W; ++w) ms[w] = mems[w]->m.get();
        surrogate_sync_shared(ms, std::vector<NodeId>(shared, shared + n_shared), average != 0);
    });
}

static void fill_report(const EpochOut& eo, int W, spd_epoch_report* rep) {
    for (int w = 0; w < W; ++w) {
        if (rep->batches) rep->batches[w] = eo.batches[w];
        if (rep->loops) rep->loops[w] = eo.loops[w];
        if (rep->digests) std::memcpy(rep->digests + 17 * w, eo.digests[w].c_str(), 17);
    }
    rep->sync_events = eo.sync_events;
    if (rep->log_cap) {
        const std::uint64_t nl = std::min<std::uint64_t>(rep->log_cap, eo.log_steps.size() / 4);
        std::copy(eo.log_steps.begin(), eo.log_steps.begin() + 4 * nl, rep->log_steps);
        rep->n_log = nl;
        const std::uint64_t ns = std::min<std::uint64_t>(rep->log_cap, eo.snaps.size());
        for (std::uint64_t s = 0; s < ns; ++s) {
            rep->snap_worker[s] = eo.snaps[s].first;
            std::memcpy(rep->snap_digests + 17 * s, eo.snaps[s].second.c_str(), 17);
        }
        rep->n_snap = ns;
    }
}

spd_status spd_run_epoch(const spd_subgraphs* subs, spd_memstore* const* mems, int32_t W,
                         const double* w_m, const double* omega, double gamma,
                         const uint32_t* shared, uint64_t n_shared, int32_t average,
                         uint64_t batch_size, spd_epoch_report* rep) {
    GUARD({
        if (!subs || W != int32_t(subs->s.g.size()))
            data_error("ConfigMismatch", "one memory store per worker required");
        std::vector<const std::vector<spd_edge>*> ev(W);
        std::vector<MemStore*> ms(W);
        for (int w = 0; w < W; ++w) {
            ev[w] = &subs->s.g[w].edges;
            ms[w] = mems[w]->m.get();
        }
        const int d = W ? ms[0]->d : 1;
        EpochOut eo;
        eo.want_log = rep && rep->log_cap > 0;
        surrogate_run_epoch(ev, ms, model_of(d, w_m, omega, gamma),
                            std::vector<NodeId>(shared, shared + n_shared), average != 0,
                            batch_size, eo);
        if (rep) fill_report(eo, W, rep);
    });
}

// simulate (pac_sim.cpp:266-338) over device memory stores.
spd_status spd_simulate(const spd_edge* e, uint64_t n, uint32_t node_count,
                        const spd_assignment* a, const spd_sim_config* cfg, int32_t device,
                        uint64_t* recovered, uint64_t* sync_events, uint64_t* loops,
                        char* digests, uint64_t* total_sync) {
    GUARD({
        const int needed = cfg->shuffle ? cfg->num_small_parts : cfg->num_workers;
        if (a->a.num_parts != needed)
            data_error("ConfigMismatch", "assignment has " + std::to_string(a->a.num_parts) +
                                             " partitions, run needs " + std::to_string(needed));
        if (cfg->num_workers < 1 || cfg->epochs < 0)
            data_error("InvalidParams", "need workers >= 1 and epochs >= 0");
        if (cfg->shuffle && cfg->num_small_parts % cfg->num_workers != 0)
            data_error("IndivisibleParts", "small parts must divide evenly across workers");
        const SurrogateModel model = SurrogateModel::seeded(cfg->d, cfg->model_seed);
        const Stream s = stream_of(e, n, node_count, 0.0);
        const SubGraphs small = induce_from_node_parts(s, a->a.np_off.data(), a->a.np_parts.data(),
                                                       a->a.node_count, a->a.num_parts);
        std::vector<std::uint64_t> small_off(1, 0);
        std::vector<NodeId> small_nodes;
        std::vector<std::vector<NodeId>> small_lists;
        for (const auto& g : small.g) {
            small_nodes.insert(small_nodes.end(), g.nodes.begin(), g.nodes.end());
            small_off.push_back(small_nodes.size());
            small_lists.push_back(g.nodes);
        }
        std::vector<std::uint8_t> in_small;
        if (cfg->shuffle)
            induce_from_groups(s, small_off.data(), small_nodes.data(), int(small.g.size()), &in_small);
        const int W = cfg->num_workers;
        std::vector<std::unique_ptr<MemStore>> mem_owned;
        std::vector<MemStore*> mems;
        for (int w = 0; w < W; ++w) {
            mem_owned.push_back(std::make_unique<MemStore>(node_count, cfg->d, device));
            mems.push_back(mem_owned.back().get());
        }
        std::uint64_t total = 0;
        for (int ep = 0; ep < cfg->epochs; ++ep) {
            SubGraphs grouped;
            const SubGraphs* subs = &small;
            std::uint64_t rec = 0;
            if (cfg->shuffle) {
                auto groups = shuffle_combine(small_lists, W, cfg->shuffle_seed + std::uint64_t(ep));
                std::vector<std::uint64_t> go(1, 0);
                std::vector<NodeId> gn;
                for (const auto& g : groups) {
                    gn.insert(gn.end(), g.begin(), g.end());
                    go.push_back(gn.size());
                }
                std::vector<std::uint8_t> in_group;
                grouped = induce_from_groups(s, go.data(), gn.data(), W, &in_group);
                for (std::uint64_t k = 0; k < n; ++k) rec += in_group[k] && !in_small[k];
                subs = &grouped;
            }
            std::vector<const std::vector<spd_edge>*> ev;
            for (const auto& g : subs->g) ev.push_back(&g.edges);
            EpochOut eo;
            surrogate_run_epoch(ev, mems, model, a->a.shared, cfg->average != 0, cfg->batch_size, eo);
            recovered[ep] = rec;
            sync_events[ep] = eo.sync_events;
            for (int w = 0; w < W; ++w) {
                loops[std::size_t(ep) * W + w] = eo.loops[w];
                std::memcpy(digests + 17 * (std::size_t(ep) * W + w), eo.digests[w].c_str(), 17);
            }
            total += eo.sync_events;
        }
        if (total_sync) *total_sync = total;
    });
}

}  // extern "C"
