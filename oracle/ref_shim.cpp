// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" veneer over the UNMODIFIED reference library (speedpart), so
// pytest (ctypes), bench.py's cpu_baseline leg and `bench.py --impl
// reference` can drive the reference's own code on the same inputs as the
// B200 path. The reference sources are compiled where they lie under
// /root/reference/proj/src by oracle/Makefile; nothing is copied. The
// output lands in oracle/_ref/ (git-ignored, travels to the GPU box).
//
// Every function mirrors one reference entry point (file:line under
// /root/reference/proj) and returns 0 ok / 2 DataError / 3 InternalError,
// the reference CLI's exit-code convention (tools/speedpart_main.cpp:436-447).
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "speedpart/centrality.hpp"
#include "speedpart/errors.hpp"
#include "speedpart/graph_io.hpp"
#include "speedpart/metrics.hpp"
#include "speedpart/pac_sim.hpp"
#include "speedpart/partitioner.hpp"

using namespace speedpart;

namespace {

thread_local std::string g_code;
thread_local std::string g_detail;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_code.clear();
        g_detail.clear();
        return 0;
    } catch (const DataError& e) {
        g_code = e.code();
        g_detail = e.what();
        return 2;
    } catch (const InternalError& e) {
        g_code = e.code();
        g_detail = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_code = "Exception";
        g_detail = e.what();
        return 3;
    }
}

EdgeStream make_stream(const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count,
                       double t_max) {
    EdgeStream s;
    s.edges.assign(e, e + n);
    s.node_count = node_count;
    s.t_max = t_max;
    return s;
}

// node_parts arrive as CSR (offsets[node_count+1], parts[]).
std::vector<std::vector<PartId>> parts_from_csr(std::uint32_t node_count,
                                                const std::uint64_t* off,
                                                const std::int32_t* parts) {
    std::vector<std::vector<PartId>> np(node_count);
    for (std::uint32_t i = 0; i < node_count; ++i)
        np[i].assign(parts + off[i], parts + off[i + 1]);
    return np;
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

PartitionerConfig make_cfg(int num_parts, double lambda, double eps, const double* cent,
                           std::uint32_t cent_n, const std::uint32_t* hubs,
                           std::uint64_t n_hubs, std::uint32_t node_count, double k) {
    PartitionerConfig cfg;
    cfg.num_parts = num_parts;
    cfg.lambda = lambda;
    cfg.epsilon = eps;
    cfg.centrality.cent.assign(cent, cent + cent_n);
    cfg.centrality.beta = 0.5;
    cfg.hub_set = HubSet::from_ids(std::vector<NodeId>(hubs, hubs + n_hubs), node_count, k);
    return cfg;
}

} // namespace

extern "C" {

const char* ref_last_error_code() { return g_code.c_str(); }
const char* ref_last_error_detail() { return g_detail.c_str(); }
void ref_free(void* p) { std::free(p); }

// graph_io.cpp:175-250
int ref_gen_powerlaw(std::uint32_t nodes, std::uint64_t edges, double alpha, std::uint64_t seed,
                     TemporalEdge* out, std::uint32_t* node_count, double* t_max) {
    return guarded([&] {
        EdgeStream s = gen_powerlaw(nodes, edges, alpha, seed);
        std::memcpy(out, s.edges.data(), sizeof(TemporalEdge) * s.edges.size());
        *node_count = s.node_count;
        *t_max = s.t_max;
    });
}

// graph_io.cpp:156-173
int ref_chrono_split_sizes(std::uint64_t n, double f_train, double f_val, std::uint64_t* n_train,
                           std::uint64_t* n_val, std::uint64_t* n_test) {
    return guarded([&] {
        EdgeStream s;
        s.edges.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) s.edges[i].ts = double(i + 1);
        ChronoSplit c = chrono_split(s, f_train, f_val);
        *n_train = c.train.size();
        *n_val = c.val.size();
        *n_test = c.test.size();
    });
}

// centrality.cpp:27-64
int ref_compute_centrality(const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count,
                           double t_max, double beta, int normalize, int degree_mode,
                           double* cent, double* t_max_out) {
    return guarded([&] {
        EdgeStream s = make_stream(e, n, node_count, t_max);
        CentralityTable t = degree_mode ? compute_degree_centrality(s)
                                        : compute_centrality(s, beta, normalize != 0);
        std::memcpy(cent, t.cent.data(), sizeof(double) * t.cent.size());
        *t_max_out = t.t_max;
    });
}

// centrality.cpp:66-88
int ref_select_hubs(const double* cent, std::uint32_t node_count, double k, int base_all,
                    std::uint32_t* hubs, std::uint64_t* n_hubs) {
    return guarded([&] {
        CentralityTable t;
        t.cent.assign(cent, cent + node_count);
        HubSet h = select_hubs(t, k, base_all ? HubBase::All : HubBase::Active);
        std::memcpy(hubs, h.hubs.data(), sizeof(NodeId) * h.hubs.size());
        *n_hubs = h.hubs.size();
    });
}

// partitioner.cpp:27-42 (score on an explicit state)
int ref_score(std::uint32_t i, std::uint32_t j, std::int32_t p, int num_parts,
              const std::uint64_t* sizes, std::uint64_t maxsize, std::uint64_t minsize,
              std::uint32_t node_count, const std::uint64_t* a_off, const std::int32_t* a_parts,
              const double* cent, std::uint32_t cent_n, double lambda, double eps, double* out) {
    return guarded([&] {
        PartitionerConfig cfg = make_cfg(num_parts, lambda, eps, cent, cent_n, nullptr, 0,
                                         node_count, 0.0);
        PartitionState st(node_count, num_parts);
        st.sizes.assign(sizes, sizes + num_parts);
        st.maxsize = maxsize;
        st.minsize = minsize;
        st.assigned = parts_from_csr(node_count, a_off, a_parts);
        *out = score(i, j, p, st, cfg);
    });
}

// partitioner.cpp:152-210. mode 0 = partition_stream, 1 = partition_unrestricted,
// 2 = partition_random. node_parts returned as malloc'd CSR.
int ref_partition(int mode, const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count,
                  double t_max, int num_parts, double lambda, double eps, const double* cent,
                  std::uint32_t cent_n, const std::uint32_t* hubs, std::uint64_t n_hubs,
                  double k, std::uint64_t seed, std::int32_t* edge_part,
                  std::uint64_t** np_off, std::int32_t** np_parts, std::uint32_t** shared,
                  std::uint64_t* n_shared, std::uint64_t* discards, double* k_eff) {
    return guarded([&] {
        EdgeStream s = make_stream(e, n, node_count, t_max);
        PartitionAssignment pa;
        if (mode == 2) {
            pa = partition_random(s, num_parts, seed);
        } else {
            PartitionerConfig cfg =
                make_cfg(num_parts, lambda, eps, cent, cent_n, hubs, n_hubs, node_count, k);
            pa = mode == 0 ? partition_stream(s, cfg) : partition_unrestricted(s, cfg);
        }
        std::memcpy(edge_part, pa.edge_part.data(), sizeof(PartId) * pa.edge_part.size());
        std::vector<std::uint64_t> off(1, 0);
        std::vector<PartId> flat;
        for (const auto& v : pa.node_parts) {
            flat.insert(flat.end(), v.begin(), v.end());
            off.push_back(flat.size());
        }
        *np_off = dup(off);
        *np_parts = dup(flat);
        *shared = dup(pa.shared);
        *n_shared = pa.shared.size();
        *discards = pa.discard_count;
        *k_eff = pa.k_eff;
    });
}

// partitioner.cpp:212-242. Outputs: per-partition CSR of indices.
int ref_assign_eval_edges(const TemporalEdge* val, std::uint64_t n_val, const TemporalEdge* test,
                          std::uint64_t n_test, std::uint32_t node_count, int num_parts,
                          const std::uint64_t* np_off, const std::int32_t* np_parts,
                          std::uint64_t** val_off, std::uint64_t** val_idx,
                          std::uint64_t** test_off, std::uint64_t** test_idx,
                          std::uint64_t* val_unroutable, std::uint64_t* test_unroutable) {
    return guarded([&] {
        ChronoSplit split;
        split.val = make_stream(val, n_val, node_count, 0.0);
        split.test = make_stream(test, n_test, node_count, 0.0);
        PartitionAssignment pa;
        pa.num_parts = num_parts;
        pa.node_parts = parts_from_csr(node_count, np_off, np_parts);
        EvalRouting r = assign_eval_edges(split, pa);
        auto pack = [](const std::vector<std::vector<std::size_t>>& lists,
                       std::uint64_t** off, std::uint64_t** idx) {
            std::vector<std::uint64_t> o(1, 0), f;
            for (const auto& l : lists) {
                f.insert(f.end(), l.begin(), l.end());
                o.push_back(f.size());
            }
            *off = dup(o);
            *idx = dup(f);
        };
        pack(r.val_edges, val_off, val_idx);
        pack(r.test_edges, test_off, test_idx);
        *val_unroutable = r.val_unroutable;
        *test_unroutable = r.test_unroutable;
    });
}

// pac_sim.cpp:106-132. Per-partition nodes and edges (as positions into the
// input stream, recovered by the unique timestamp-free trick of walking the
// stream in order) returned as malloc'd CSR.
int ref_induce_subgraphs(const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count,
                         const std::uint64_t* np_off, const std::int32_t* np_parts,
                         std::uint32_t np_n, int num_parts, std::uint64_t** node_off,
                         std::uint32_t** nodes, std::uint64_t** edge_off, TemporalEdge** edges) {
    return guarded([&] {
        EdgeStream s = make_stream(e, n, node_count, 0.0);
        std::vector<std::vector<PartId>> np = parts_from_csr(np_n, np_off, np_parts);
        std::vector<SubGraph> subs = induce_subgraphs(s, np, num_parts);
        std::vector<std::uint64_t> no(1, 0), eo(1, 0);
        std::vector<NodeId> nf;
        std::vector<TemporalEdge> ef;
        for (const auto& sg : subs) {
            nf.insert(nf.end(), sg.nodes.begin(), sg.nodes.end());
            no.push_back(nf.size());
            ef.insert(ef.end(), sg.edges.begin(), sg.edges.end());
            eo.push_back(ef.size());
        }
        *node_off = dup(no);
        *nodes = dup(nf);
        *edge_off = dup(eo);
        *edges = dup(ef);
    });
}

// pac_sim.cpp:134-160
int ref_shuffle_combine(const std::uint64_t* off, const std::uint32_t* nodes, std::uint64_t n_small,
                        int num_workers, std::uint64_t seed, std::uint64_t** out_off,
                        std::uint32_t** out_nodes) {
    return guarded([&] {
        std::vector<std::vector<NodeId>> small(n_small);
        for (std::uint64_t p = 0; p < n_small; ++p) small[p].assign(nodes + off[p], nodes + off[p + 1]);
        auto groups = shuffle_combine(small, num_workers, seed);
        std::vector<std::uint64_t> o(1, 0);
        std::vector<NodeId> f;
        for (const auto& g : groups) {
            f.insert(f.end(), g.begin(), g.end());
            o.push_back(f.size());
        }
        *out_off = dup(o);
        *out_nodes = dup(f);
    });
}

// pac_sim.cpp:28-46
int ref_model_seeded(int d, std::uint64_t seed, double* w_m, double* omega, double* gamma) {
    return guarded([&] {
        ModelParams m = ModelParams::seeded(d, seed);
        std::memcpy(w_m, m.w_m.data(), sizeof(double) * m.w_m.size());
        std::memcpy(omega, m.omega.data(), sizeof(double) * m.omega.size());
        *gamma = m.gamma;
    });
}

static ModelParams params_of(int d, const double* w_m, const double* omega, double gamma) {
    ModelParams m;
    m.d = d;
    m.gamma = gamma;
    m.w_m.assign(w_m, w_m + std::size_t(d) * 3 * d);
    m.omega.assign(omega, omega + d);
    return m;
}

// pac_sim.cpp:68-104, applied over a run of edges (state/last_ts in-out).
int ref_model_update_run(std::uint32_t node_count, int d, double* state, double* last_ts,
                         const TemporalEdge* e, std::uint64_t n, const double* w_m,
                         const double* omega, double gamma) {
    return guarded([&] {
        ModelParams m = params_of(d, w_m, omega, gamma);
        MemoryStore mem(node_count, d);
        std::memcpy(mem.state.data(), state, sizeof(double) * mem.state.size());
        std::memcpy(mem.last_ts.data(), last_ts, sizeof(double) * node_count);
        for (std::uint64_t k = 0; k < n; ++k) model_update(mem, e[k], m);
        std::memcpy(state, mem.state.data(), sizeof(double) * mem.state.size());
        std::memcpy(last_ts, mem.last_ts.data(), sizeof(double) * node_count);
    });
}

// Thread-parallel timing harness for the reference CPU arm: T independent
// MemoryStores each replay their own slice of edges through model_update
// (pac_sim.cpp:68-104) concurrently. Returns wall seconds in *secs.
int ref_model_update_threads(std::uint32_t node_count, int d, const TemporalEdge* e,
                             const std::uint64_t* slice_off, int threads, const double* w_m,
                             const double* omega, double gamma, double* secs) {
    return guarded([&] {
        ModelParams m = params_of(d, w_m, omega, gamma);
        std::vector<std::thread> pool;
        std::vector<std::string> errs(threads);
        auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    MemoryStore mem(node_count, d);
                    for (std::uint64_t k = slice_off[t]; k < slice_off[t + 1]; ++k)
                        model_update(mem, e[k], m);
                } catch (const std::exception& ex) {
                    errs[t] = ex.what();
                }
            });
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        *secs = std::chrono::duration<double>(t1 - t0).count();
        for (auto& s : errs)
            if (!s.empty()) throw InternalError("ThreadFailure", s);
    });
}

// pac_sim.cpp:162-203. states: W * node_count * d, last_ts: W * node_count.
int ref_sync_shared(int W, std::uint32_t node_count, int d, double* states, double* last_ts,
                    const std::uint32_t* shared, std::uint64_t n_shared, int average) {
    return guarded([&] {
        std::vector<MemoryStore> mems(W, MemoryStore(node_count, d));
        const std::size_t S = std::size_t(node_count) * d;
        for (int w = 0; w < W; ++w) {
            std::memcpy(mems[w].state.data(), states + w * S, sizeof(double) * S);
            std::memcpy(mems[w].last_ts.data(), last_ts + std::size_t(w) * node_count,
                        sizeof(double) * node_count);
        }
        sync_shared(mems, std::vector<NodeId>(shared, shared + n_shared),
                    average ? SyncStrategy::Average : SyncStrategy::MaxTimestamp);
        for (int w = 0; w < W; ++w) {
            std::memcpy(states + w * S, mems[w].state.data(), sizeof(double) * S);
            std::memcpy(last_ts + std::size_t(w) * node_count, mems[w].last_ts.data(),
                        sizeof(double) * node_count);
        }
    });
}

// pac_sim.cpp:18-26
int ref_digest(std::uint32_t node_count, int d, const double* state, const double* last_ts,
               char* out17) {
    return guarded([&] {
        MemoryStore mem(node_count, d);
        std::memcpy(mem.state.data(), state, sizeof(double) * mem.state.size());
        std::memcpy(mem.last_ts.data(), last_ts, sizeof(double) * node_count);
        std::string h = mem.digest();
        std::memcpy(out17, h.c_str(), 17);
    });
}

// pac_sim.cpp:205-264. Subgraph edges as CSR over W workers; states in-out.
// Step log (optional, pass log_cap = 0 to skip): 4 u64 per record
// (global_step, worker, loop, batch_in_loop); snapshot log: worker id + 17-char digest.
int ref_run_epoch(int W, std::uint32_t node_count, int d, const std::uint64_t* e_off,
                  const TemporalEdge* edges, double* states, double* last_ts, const double* w_m,
                  const double* omega, double gamma, const std::uint32_t* shared,
                  std::uint64_t n_shared, int average, std::uint64_t batch_size,
                  std::uint64_t* batches, std::uint64_t* loops, std::uint64_t* sync_events,
                  char* digests, std::uint64_t log_cap, std::uint64_t* log_steps,
                  std::uint64_t* n_log, std::int32_t* snap_worker, char* snap_digests,
                  std::uint64_t* n_snap) {
    return guarded([&] {
        ModelParams m = params_of(d, w_m, omega, gamma);
        std::vector<SubGraph> subs(W);
        for (int w = 0; w < W; ++w) subs[w].edges.assign(edges + e_off[w], edges + e_off[w + 1]);
        std::vector<MemoryStore> mems(W, MemoryStore(node_count, d));
        const std::size_t S = std::size_t(node_count) * d;
        for (int w = 0; w < W; ++w) {
            std::memcpy(mems[w].state.data(), states + w * S, sizeof(double) * S);
            std::memcpy(mems[w].last_ts.data(), last_ts + std::size_t(w) * node_count,
                        sizeof(double) * node_count);
        }
        StepLog log;
        EpochReport er = run_epoch(subs, mems, m, std::vector<NodeId>(shared, shared + n_shared),
                                   average ? SyncStrategy::Average : SyncStrategy::MaxTimestamp,
                                   batch_size, log_cap ? &log : nullptr);
        for (int w = 0; w < W; ++w) {
            std::memcpy(states + w * S, mems[w].state.data(), sizeof(double) * S);
            std::memcpy(last_ts + std::size_t(w) * node_count, mems[w].last_ts.data(),
                        sizeof(double) * node_count);
            batches[w] = er.batches[w];
            loops[w] = er.loops[w];
            std::memcpy(digests + 17 * w, er.digests[w].c_str(), 17);
        }
        *sync_events = er.sync_events;
        if (log_cap) {
            std::uint64_t k = 0;
            for (const auto& r : log.steps) {
                if (k >= log_cap) break;
                log_steps[4 * k + 0] = r.global_step;
                log_steps[4 * k + 1] = std::uint64_t(r.worker);
                log_steps[4 * k + 2] = r.loop;
                log_steps[4 * k + 3] = r.batch_in_loop;
                ++k;
            }
            *n_log = k;
            std::uint64_t s = 0;
            for (const auto& [w, dg] : log.snapshots) {
                if (s >= log_cap) break;
                snap_worker[s] = w;
                std::memcpy(snap_digests + 17 * s, dg.c_str(), 17);
                ++s;
            }
            *n_snap = s;
        }
    });
}

// pac_sim.cpp:266-338. Per-epoch outputs: recovered, sync_events, and W
// digests (17 chars each) per epoch; loops per worker per epoch.
int ref_simulate(const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count, double t_max,
                 int num_parts, const std::uint64_t* np_off, const std::int32_t* np_parts,
                 const std::uint32_t* shared, std::uint64_t n_shared, int num_workers,
                 int num_small_parts, int shuffle, int average, std::uint64_t batch_size,
                 int epochs, int d, std::uint64_t model_seed, std::uint64_t shuffle_seed,
                 std::uint64_t* recovered, std::uint64_t* sync_events, std::uint64_t* loops,
                 char* digests, std::uint64_t* total_sync) {
    return guarded([&] {
        EdgeStream s = make_stream(e, n, node_count, t_max);
        PartitionAssignment pa;
        pa.num_parts = num_parts;
        pa.node_parts = parts_from_csr(node_count, np_off, np_parts);
        pa.shared.assign(shared, shared + n_shared);
        SimConfig cfg;
        cfg.num_workers = num_workers;
        cfg.num_small_parts = num_small_parts;
        cfg.shuffle = shuffle != 0;
        cfg.sync = average ? SyncStrategy::Average : SyncStrategy::MaxTimestamp;
        cfg.batch_size = batch_size;
        cfg.epochs = epochs;
        cfg.d = d;
        cfg.model_seed = model_seed;
        cfg.shuffle_seed = shuffle_seed;
        SimReport rep = simulate(s, pa, cfg);
        for (std::size_t ep = 0; ep < rep.epochs.size(); ++ep) {
            const auto& er = rep.epochs[ep];
            recovered[ep] = er.recovered;
            sync_events[ep] = er.sync_events;
            for (int w = 0; w < num_workers; ++w) {
                loops[ep * num_workers + w] = er.loops[w];
                std::memcpy(digests + 17 * (ep * num_workers + w), er.digests[w].c_str(), 17);
            }
        }
        *total_sync = rep.sync_events;
    });
}

// graph_io.cpp:106-140 load_edges(path, assume_sorted); *out malloc'ed (ref_free)
int ref_load_edges(const char* path, int assume_sorted, TemporalEdge** out, std::uint64_t* n,
                   std::uint32_t* node_count, double* t_max) {
    return guarded([&] {
        EdgeStream s = load_edges(std::string(path), assume_sorted != 0);
        *out = dup(s.edges);
        *n = s.edges.size();
        *node_count = s.node_count;
        *t_max = s.t_max;
    });
}

// graph_io.cpp:142-154 write_edges(stream, path)
int ref_write_edges(const char* path, const TemporalEdge* e, std::uint64_t n) {
    return guarded([&] { write_edges(make_stream(e, n, 0, 0.0), std::string(path)); });
}

// metrics.cpp:33-68 (reporting only)
int ref_quality(const TemporalEdge* e, std::uint64_t n, std::uint32_t node_count, int num_parts,
                const std::int32_t* edge_part, const std::uint64_t* np_off,
                const std::int32_t* np_parts, std::uint64_t discards, double* rf, double* ec) {
    return guarded([&] {
        EdgeStream s = make_stream(e, n, node_count, 0.0);
        PartitionAssignment pa;
        pa.num_parts = num_parts;
        pa.edge_part.assign(edge_part, edge_part + n);
        pa.node_parts = parts_from_csr(node_count, np_off, np_parts);
        pa.discard_count = discards;
        QualityReport q = quality(pa, s);
        *rf = q.rf;
        *ec = q.ec;
    });
}

} // extern "C"
