/*
 * speed_c.h — C-ABI of the B200-native SPEED (arXiv 2308.14129) parallel-training
 * hot path: SEP partitioning, subgraph induction, the PAC lockstep trainer and the
 * per-partition TGN training step on sm_100a.
 *
 * The reference (speedpart, /root/reference/proj) exposes a C++ value-type API
 * and no FFI; every entry point below names the reference declaration it
 * replaces (file:line under /root/reference/proj/include/speedpart/). Bindings
 * (ctypes / cgo / JNI) for these are shown in INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers + sizes, caller-owned buffers; opaque handles own library
 *    memory and are released with their *_destroy function.
 *  - Every call returns spd_status with the reference CLI's exit-code numbering
 *    (tools/speedpart_main.cpp:436-447): 0 ok, 1 usage, 2 data (DataError,
 *    errors.hpp:10-20), 3 internal (InternalError, errors.hpp:23-32; also
 *    CUDA / NCCL failures). The reference's error code string ("UnsortedStream",
 *    "NonChronological", ...) and detail are readable per thread through
 *    spd_last_error_code()/spd_last_error_detail(). No exception crosses the ABI.
 *  - There is no CPU fallback: device entry points fail with status 3 and code
 *    "CudaError" when no sm_100 device is present.
 */
#ifndef SPEED_C_H
#define SPEED_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t spd_status;
enum { SPD_OK = 0, SPD_USAGE = 1, SPD_DATA = 2, SPD_INTERNAL = 3 };

const char* spd_last_error_code(void);
const char* spd_last_error_detail(void);
const char* spd_version(void);

/* One timestamped interaction event; byte-identical to speedpart::TemporalEdge
 * (types.hpp:15-21): {u32 src, u32 dst, f64 ts}, 16 bytes. */
typedef struct spd_edge {
    uint32_t src;
    uint32_t dst;
    double ts;
} spd_edge;

/* ---------------------------------------------------------------- L1 stream */

/* gen_powerlaw (graph_io.hpp:34). out: `edges` records. Bit-identical stream. */
spd_status spd_gen_powerlaw(uint32_t nodes, uint64_t edges, double alpha, uint64_t seed,
                            spd_edge* out, uint32_t* node_count, double* t_max);

/* chrono_split (graph_io.hpp:27): positional 3-way split sizes. */
spd_status spd_chrono_split(uint64_t n, double f_train, double f_val, uint64_t* n_train,
                            uint64_t* n_val, uint64_t* n_test);

/* -------------------------------------------------------- L2 partitioning */

/* compute_centrality (centrality.hpp:41). cent: node_count doubles. */
spd_status spd_compute_centrality(const spd_edge* e, uint64_t n, uint32_t node_count,
                                  double t_max, double beta, int32_t normalize_ts,
                                  double* cent, double* t_max_out);
/* compute_degree_centrality (centrality.hpp:44). */
spd_status spd_compute_degree_centrality(const spd_edge* e, uint64_t n, uint32_t node_count,
                                         double* cent);
/* select_hubs (centrality.hpp:48). base_all: HubBase::All if nonzero. hubs: capacity
 * node_count, ascending on return. */
spd_status spd_select_hubs(const double* cent, uint32_t node_count, double k, int32_t base_all,
                           uint32_t* hubs, uint64_t* n_hubs);

/* PartitionerConfig (partitioner.hpp:11-17). cent may be shorter than node_count
 * (CentralityTable::of returns 0 past its end, centrality.hpp:17). */
typedef struct spd_partitioner_config {
    int32_t num_parts;
    double lambda;
    double epsilon;
    const double* cent;
    uint32_t cent_count;
    const uint32_t* hubs;
    uint64_t n_hubs;
    double k;
} spd_partitioner_config;

/* PartitionAssignment (partitioner.hpp:40-47). */
typedef struct spd_assignment spd_assignment;

/* partition_stream (partitioner.hpp:62) — bit-identical edge_part / node_parts / shared. */
spd_status spd_partition_stream(const spd_edge* e, uint64_t n, uint32_t node_count,
                                const spd_partitioner_config* cfg, spd_assignment** out);
/* partition_unrestricted (partitioner.hpp:66). */
spd_status spd_partition_unrestricted(const spd_edge* e, uint64_t n, uint32_t node_count,
                                      const spd_partitioner_config* cfg, spd_assignment** out);
/* score (partitioner.hpp:50-51) on an explicit PartitionState
 * (sizes[num_parts], maxsize, minsize, A-sets as CSR over node_count). */
spd_status spd_score(uint32_t i, uint32_t j, int32_t p, const spd_partitioner_config* cfg,
                     const uint64_t* sizes, uint64_t maxsize, uint64_t minsize,
                     uint32_t node_count, const uint64_t* a_off, const int32_t* a_parts,
                     double* out);
/* Build an assignment from external node_parts (the CLI's load_assignment,
 * speedpart_main.cpp:135-179). edge_part may be NULL. */
spd_status spd_assignment_from_parts(uint32_t node_count, int32_t num_parts, const uint64_t* np_off,
                                     const int32_t* np_parts, const int32_t* edge_part,
                                     uint64_t n_edges, uint64_t discards,
                                     spd_assignment** out);
void spd_assignment_destroy(spd_assignment* a);
spd_status spd_assignment_info(const spd_assignment* a, int32_t* num_parts, uint32_t* node_count,
                               uint64_t* n_edges, uint64_t* n_shared, uint64_t* discards,
                               uint64_t* np_total, double* k_eff);
spd_status spd_assignment_edge_part(const spd_assignment* a, int32_t* out);
spd_status spd_assignment_node_parts(const spd_assignment* a, uint64_t* off, int32_t* parts);
spd_status spd_assignment_shared(const spd_assignment* a, uint32_t* out);

/* ------------------------------------------------------ on-disk formats (f3)
 * load_edges / write_edges (graph_io.hpp; graph_io.cpp:106-154): CSV
 * "src,dst,ts", same acceptance rules, error codes and texts (ParseError
 * "row N: ...", FileNotFound); rows stable-sorted by ts unless assume_sorted.
 * *out is malloc'ed: release with spd_free. */
void spd_free(void* p);
spd_status spd_load_edges_csv(const char* path, int32_t assume_sorted, spd_edge** out, uint64_t* n,
                              uint32_t* node_count, double* t_max);
spd_status spd_write_edges_csv(const char* path, const spd_edge* e, uint64_t n);
/* Binary event file: 32-B header {"SPDEDGE1", u64 n, u32 node_count, u32 0,
 * f64 t_max} + n TemporalEdge records (types.hpp:15-20) verbatim. The reader
 * fills caller memory (e.g. pinned buffers) and validates ids < node_count
 * (ParseError) and time order (UnsortedStream). */
spd_status spd_write_edges_bin(const char* path, const spd_edge* e, uint64_t n,
                               uint32_t node_count, double t_max);
spd_status spd_edges_bin_info(const char* path, uint64_t* n, uint32_t* node_count, double* t_max);
spd_status spd_load_edges_bin(const char* path, spd_edge* out, uint64_t cap);
/* Assignment JSON of the CLI's partition subcommand (speedpart_main.cpp:110-119)
 * — {"config":<config_json>,"edge_part":[..],"node_parts":{"0":[..],..},
 * "shared":[..],"discards":n}, compact — and its reader (load_assignment,
 * speedpart_main.cpp:129-166: missing keys -> ParseError "assignment is
 * missing '<key>'"; num_parts / k_eff from config.parts / config.topk).
 * config_out (optional) receives the raw config object text (spd_free). */
spd_status spd_assignment_write_json(const spd_assignment* a, const char* config_json,
                                     const char* path);
spd_status spd_assignment_read_json(const char* path, spd_assignment** out, char** config_out);

/* assign_eval_edges (partitioner.hpp:74-81). */
typedef struct spd_eval_routing spd_eval_routing;
spd_status spd_assign_eval_edges(const spd_edge* val, uint64_t n_val, const spd_edge* test,
                                 uint64_t n_test, const spd_assignment* a,
                                 spd_eval_routing** out);
/* which: 0 = val, 1 = test. count[num_parts]; idx: per-partition lists back to back. */
spd_status spd_eval_routing_counts(const spd_eval_routing* r, int32_t which, uint64_t* counts,
                                   uint64_t* unroutable);
spd_status spd_eval_routing_edges(const spd_eval_routing* r, int32_t which, uint64_t* idx);
void spd_eval_routing_destroy(spd_eval_routing* r);

/* ------------------------------------------------- L4 subgraphs and shuffle */

/* induce_subgraphs (pac_sim.hpp:102-104). Each subgraph keeps, next to its
 * time-ordered edges, the stream position (global edge id) of every edge. */
typedef struct spd_subgraphs spd_subgraphs;
spd_status spd_induce_subgraphs(const spd_edge* e, uint64_t n, uint32_t node_count,
                                const uint64_t* np_off, const int32_t* np_parts, uint32_t np_count,
                                int32_t num_parts, spd_subgraphs** out);
/* simulate's shuffle branch (pac_sim.cpp:313-324): induce on explicit node groups;
 * also returns how many edges the groups induce that no small part does
 * (`recovered`, pac_sim.cpp:325-326) when small_off/small_nodes are given. */
spd_status spd_induce_groups(const spd_edge* e, uint64_t n, uint32_t node_count,
                             const uint64_t* group_off, const uint32_t* group_nodes,
                             int32_t n_groups, const uint64_t* small_off,
                             const uint32_t* small_nodes, int32_t n_small,
                             spd_subgraphs** out, uint64_t* recovered);
/* Build a subgraph set from explicit per-subgraph node lists and time-ordered
 * edge lists (CSR over n; eids may be NULL = position in each list). */
spd_status spd_subgraphs_from_lists(int32_t n, const uint64_t* node_off, const uint32_t* nodes,
                                    const uint64_t* edge_off, const spd_edge* edges,
                                    const uint64_t* eids, spd_subgraphs** out);
spd_status spd_subgraphs_count(const spd_subgraphs* s, int32_t* count);
spd_status spd_subgraph_sizes(const spd_subgraphs* s, int32_t p, uint64_t* n_nodes,
                              uint64_t* n_edges);
spd_status spd_subgraph_nodes(const spd_subgraphs* s, int32_t p, uint32_t* out);
spd_status spd_subgraph_edges(const spd_subgraphs* s, int32_t p, spd_edge* out, uint64_t* eids);
void spd_subgraphs_destroy(spd_subgraphs* s);

/* shuffle_combine (pac_sim.hpp:108-110). out_off: num_workers+1; out_nodes:
 * capacity small_off[n_small]. */
spd_status spd_shuffle_combine(const uint64_t* small_off, const uint32_t* small_nodes,
                               uint64_t n_small, int32_t num_workers, uint64_t epoch_seed,
                               uint64_t* out_off, uint32_t* out_nodes);

/* The PAC lockstep schedule of run_epoch (pac_sim.cpp:215-257) on the host:
 * n_steps global steps; log (optional, 4*cap u64) = StepRecord rows
 * (global_step, worker, loop, batch_in_loop); batches/loops per worker (W each). */
spd_status spd_lockstep_schedule(const spd_subgraphs* s, uint64_t batch_size, uint64_t* n_steps,
                                 uint64_t* log, uint64_t cap, uint64_t* n_log, uint64_t* batches,
                                 uint64_t* loops);

/* ------------------------------------------- L4 surrogate model (parity mode) */

/* ModelParams::seeded (pac_sim.hpp:54). w_m: d*3d row-major, omega: d. */
spd_status spd_model_seeded(int32_t d, uint64_t seed, double* w_m, double* omega, double* gamma);

/* MemoryStore (pac_sim.hpp:19-39), resident in device HBM (f64 state + f64 last_ts). */
typedef struct spd_memstore spd_memstore;
spd_status spd_memstore_create(uint32_t node_count, int32_t d, int32_t device,
                               spd_memstore** out);
void spd_memstore_destroy(spd_memstore* m);
spd_status spd_memstore_upload(spd_memstore* m, const double* state, const double* last_ts);
spd_status spd_memstore_download(const spd_memstore* m, double* state, double* last_ts);
spd_status spd_memstore_reset(spd_memstore* m);
spd_status spd_memstore_copy(spd_memstore* dst, const spd_memstore* src);
/* MemoryStore::digest (pac_sim.cpp:18-26): 16 hex chars + NUL. */
spd_status spd_memstore_digest(const spd_memstore* m, char* out17);

/* model_update (pac_sim.hpp:59) over a run of edges, applied in order on the GPU. */
spd_status spd_model_update(spd_memstore* m, const spd_edge* e, uint64_t n, const double* w_m,
                            const double* omega, double gamma);

/* sync_shared (pac_sim.hpp:125-126). average: SyncStrategy::Average if nonzero. */
spd_status spd_sync_shared(spd_memstore* const* mems, int32_t W, const uint32_t* shared,
                           uint64_t n_shared, int32_t average);

/* EpochReport (pac_sim.hpp:75-81) + StepLog (pac_sim.hpp:88-100). Arrays are caller
 * owned and sized W (digests 17*W). Log arrays optional (log_cap 0 = no log):
 * log_steps 4*log_cap u64 (global_step, worker, loop, batch_in_loop), snapshot
 * worker ids + 17-char digests, log_cap entries each. */
typedef struct spd_epoch_report {
    uint64_t* batches;
    uint64_t* loops;
    uint64_t sync_events;
    char* digests;
    uint64_t log_cap;
    uint64_t* log_steps;
    uint64_t n_log;
    int32_t* snap_worker;
    char* snap_digests;
    uint64_t n_snap;
} spd_epoch_report;

/* run_epoch (pac_sim.hpp:117-120) on device memory stores. */
spd_status spd_run_epoch(const spd_subgraphs* subs, spd_memstore* const* mems, int32_t W,
                         const double* w_m, const double* omega, double gamma,
                         const uint32_t* shared, uint64_t n_shared, int32_t average,
                         uint64_t batch_size, spd_epoch_report* rep);

/* SimConfig (pac_sim.hpp:63-73). */
typedef struct spd_sim_config {
    int32_t num_workers;
    int32_t num_small_parts;
    int32_t shuffle;
    int32_t average;
    uint64_t batch_size;
    int32_t epochs;
    int32_t d;
    uint64_t model_seed;
    uint64_t shuffle_seed;
} spd_sim_config;

/* simulate (pac_sim.hpp:132-133). Per-epoch outputs (caller owned):
 * recovered[epochs], sync_events[epochs], loops[epochs*W], digests[17*epochs*W]. */
spd_status spd_simulate(const spd_edge* e, uint64_t n, uint32_t node_count,
                        const spd_assignment* a, const spd_sim_config* cfg, int32_t device,
                        uint64_t* recovered, uint64_t* sync_events, uint64_t* loops,
                        char* digests, uint64_t* total_sync);

/* ---------------------------------------------------- TGN training hot path */

/* Builder-defined TGN step: identity
 * message, last-message aggregation, GRU memory, 1-layer multi-head temporal
 * attention over the k most recent neighbours, MergeLayer decoder, BCE, Adam. */
typedef struct spd_tgn_config {
    int32_t d_mem;       /* memory / embedding dim (TGN default 100; multiple of 4) */
    int32_t d_time;      /* time-encoding dim (multiple of 4) */
    int32_t d_edge;      /* edge-feature dim (0 = no features) */
    int32_t n_neighbors; /* recent-k */
    int32_t n_heads;
    uint64_t batch_size;
    float lr;
    float beta1, beta2, adam_eps;
    uint64_t seed_init;  /* parameter init */
    uint64_t seed_feat;  /* synthetic edge features */
    uint64_t seed_neg;   /* negative sampling */
    int32_t sync_average;/* epoch-end shared-node sync: 1 average (default), 0 max-ts */
    int32_t gemm_mode;   /* 0 = FP32 FFMA, 1 = tcgen05 TF32 for the GRU and attention projections (tolerance-gated) */
    int32_t backbone;    /* 0 = TGN (GRU memory, temporal attention); 1 = JODIE (RNN memory,
                          * time-projection embedding); 2 = DyRep (RNN memory, identity
                          * embedding, attention-embedding messages): PAPER.md:373's
                          * other backbones */
    int32_t concurrent;  /* 1: a process's local workers (several SEP partitions on one GPU,
                          * world 1) train concurrently, each on its own streams with its own
                          * scratch and parameter replica; gradients meet in the fused
                          * all-reduce + Adam of the peer transport (in-process). 0: one after
                          * another in one scratch (default). */
} spd_tgn_config;

typedef struct spd_tgn_trainer spd_tgn_trainer;

/* One trainer owns the workers (partitions) this process trains, one device.
 * `workers` lists which subgraphs of `subs` it owns; across processes the
 * lists partition [0, count). world>1 joins an NCCL communicator from
 * nccl_id (128 bytes from spd_nccl_unique_id) for the per-step gradient
 * all-reduce and the epoch-end shared-node sync; with nccl_id == NULL it uses
 * the peer-memory transport below instead. shared: global ids of SEP's
 * shared hubs (PartitionAssignment::shared). edge ids in `subs` index the
 * synthetic feature generator. */
spd_status spd_tgn_create(const spd_tgn_config* cfg, const spd_subgraphs* subs,
                          const int32_t* workers, int32_t n_workers, const uint32_t* shared,
                          uint64_t n_shared, uint32_t node_count, int32_t rank, int32_t world,
                          const void* nccl_id, int32_t device, spd_tgn_trainer** out);
void spd_tgn_destroy(spd_tgn_trainer* t);
spd_status spd_nccl_unique_id(void* out128);
/* Peer-memory transport (world > 1 created with nccl_id == NULL): the
 * per-step gradient all-reduce is fused into Adam, reading every rank's
 * gradient buffer from its HBM (CUDA IPC: NVLink P2P across GPUs, shared HBM
 * for ranks on one GPU), in rank order — replicated parameters stay
 * bit-identical; the epoch-end shared-hub sync (pac_sim.cpp:162-203) reduces
 * over the same mappings. Replaces the Alg. 2 barrier + all-reduce of
 * PAPER.md:340-358 / pac_sim.cpp:233-260. Every rank exports a blob of
 * spd_tgn_peer_blob_bytes() bytes, the caller gathers them in rank order
 * (any host channel) and every rank connects before its first step. */
uint64_t spd_tgn_peer_blob_bytes(void);
spd_status spd_tgn_peer_export(const spd_tgn_trainer* t, void* out);
spd_status spd_tgn_peer_connect(spd_tgn_trainer* t, const void* blobs);

/* Number of lockstep global steps in one epoch = max_w ceil(|E_w| / B) over ALL
 * workers (run_epoch, pac_sim.cpp:221-234). */
spd_status spd_tgn_epoch_steps(const spd_tgn_trainer* t, uint64_t* steps);
/* Begin an epoch: positions to loop start (memory reset, pac_sim.cpp:238). */
spd_status spd_tgn_begin_epoch(spd_tgn_trainer* t, int32_t epoch);
/* Position the lockstep schedule at global step `step` of the current epoch:
 * each worker at batch (step mod its batch count), memory, clocks and pending
 * messages cleared. Benchmarks use it to time steady-state steps mid-epoch
 * (full recent-k neighbour lists) instead of an epoch's sparse first batches. */
spd_status spd_tgn_seek(spd_tgn_trainer* t, uint64_t step);
/* Shuffle-combine (simulate with SimConfig::shuffle, pac_sim.cpp:280-329):
 * before an epoch, rebind the trainer to that epoch's regrouped subgraphs
 * (spd_shuffle_combine + spd_induce_groups; one per worker, same count).
 * Parameters and Adam state carry over; memory, clocks and pending messages
 * start from zero (reset at every loop start, pac_sim.cpp:238); evaluation
 * views must be set again. ConfigMismatch if the worker count differs. */
spd_status spd_tgn_rebind(spd_tgn_trainer* t, const spd_subgraphs* subs);
/* Shuffle-combine on the device (K13; pac_sim.cpp:134-160, :280-329): attach
 * the time-ordered training stream (global ids) and the small SEP parts'
 * node lists (CSR small_off[n_small + 1] / small_nodes, as spd_shuffle_combine
 * takes them; n_small a multiple of the worker count, workers <= 64) once;
 * then spd_tgn_shuffle_epoch regroups the parts with shuffle_combine's seeded
 * permutation (epoch_seed = shuffle_seed + epoch, as simulate) and induces
 * every worker's subgraph in HBM — events, neighbour CSR, negative pool,
 * feature rows — with the same result as spd_shuffle_combine +
 * spd_induce_groups + spd_tgn_rebind, and the same `recovered` count.
 * Parameters and Adam state carry over; memory starts from zero. */
spd_status spd_tgn_attach_stream(spd_tgn_trainer* t, const spd_edge* e, uint64_t n, uint32_t node_count,
                                 const uint64_t* small_off, const uint32_t* small_nodes, int32_t n_small);
spd_status spd_tgn_shuffle_epoch(spd_tgn_trainer* t, uint64_t epoch_seed, uint64_t* recovered);
/* One global step: every local worker trains one batch, gradients are
 * all-reduced (mean over all workers), Adam updates. loss_out: per local
 * worker mean BCE of the batch (device->host read), may be NULL. */
spd_status spd_tgn_step(spd_tgn_trainer* t, float* loss_out);
/* Epoch end: restore loop-end snapshots + shared sync (pac_sim.cpp:259-260). */
spd_status spd_tgn_end_epoch(spd_tgn_trainer* t);
/* Whole epoch (begin + steps + end). */
spd_status spd_tgn_run_epoch(spd_tgn_trainer* t, int32_t epoch, double* mean_loss);

/* Evaluation (TGN protocol; routing = spd_assign_eval_edges, partitioner.hpp:74-81).
 * set: the worker's routed val edges followed by its routed test edges (GLOBAL
 * ids, time-ordered, eids for features) are appended after its training events;
 * the full-graph recent-k finder and the negative pool cover train + eval events.
 * evaluate: eval events [lo, hi) are scored in batches against the current
 * memory (logits of each positive and of one sampled negative, counter hash of
 * (neg_seed, worker, position)); memory then advances through them. No gradients. */
spd_status spd_tgn_set_eval_events(spd_tgn_trainer* t, int32_t worker, const spd_edge* e,
                                   const uint64_t* eids, uint64_t n);
spd_status spd_tgn_evaluate(spd_tgn_trainer* t, int32_t worker, uint64_t lo, uint64_t hi,
                            uint64_t neg_seed, float* pos_scores, float* neg_scores);

/* Global link-prediction metrics over the scores of every partition / rank
 * (SURVEY §8e(3)): the caller concatenates the routed edges' positive and
 * negative scores of all partitions (spd_tgn_evaluate on each rank, then an
 * all-gather); AP = sum_g (R_g - R_{g-1}) P_g over descending score groups,
 * AUC = trapezoidal ROC area (ties one half) — sklearn's
 * average_precision_score / roc_auc_score. Data error on empty lists or NaN.
 * Routing reference: assign_eval_edges, partitioner.cpp:212-242. */
spd_status spd_link_metrics(const float* pos, uint64_t n_pos, const float* neg, uint64_t n_neg,
                            double* ap, double* auc);

/* Introspection for parity tests. */
spd_status spd_tgn_param_count(const spd_tgn_trainer* t, uint64_t* n);
spd_status spd_tgn_get_params(const spd_tgn_trainer* t, float* out);
spd_status spd_tgn_set_params(spd_tgn_trainer* t, const float* in);
spd_status spd_tgn_get_grads(const spd_tgn_trainer* t, float* out);
/* worker-local memory (n_local_nodes x d_mem f32, last_update f64) */
spd_status spd_tgn_local_nodes(const spd_tgn_trainer* t, int32_t worker, uint64_t* n,
                               uint32_t* global_ids);
spd_status spd_tgn_get_memory(const spd_tgn_trainer* t, int32_t worker, float* mem,
                              double* last_update);
spd_status spd_tgn_set_memory(spd_tgn_trainer* t, int32_t worker, const float* mem,
                              const double* last_update);
/* Debug taps of the last step for worker: embeddings [3B x d_mem] (src,dst,neg),
 * negatives [B] (global ids), neighbour ids [3B x k] (global, UINT32_MAX = pad). */
spd_status spd_tgn_last_step(const spd_tgn_trainer* t, int32_t worker, uint64_t* b,
                             float* emb, uint32_t* negs, uint32_t* nbr_ids, float* loss);
/* Debug taps (spd_tgn_last_step) and per-phase CUDA-event timing of each step
 * (spd_tgn_kernel_times); both add synchronisation, off by default. */
spd_status spd_tgn_set_debug(spd_tgn_trainer* t, int32_t on);
spd_status spd_tgn_set_profile(spd_tgn_trainer* t, int32_t on);
/* Regular steps (every local worker on a full batch) replay a captured CUDA
 * graph of the step; on by default, off = launch every kernel eagerly. */
spd_status spd_tgn_set_graph(spd_tgn_trainer* t, int32_t on);
/* Switch spd_tgn_config::gemm_mode between steps (0 FP32 FFMA, 1 tcgen05 TF32
 * projections): parameters, optimiser state and memory carry over; captured
 * step graphs are rebuilt. */
spd_status spd_tgn_set_gemm_mode(spd_tgn_trainer* t, int32_t mode);
/* Debug: copy of the per-step scratch buffer `name` (x_gru, h_gru, Gi, Gh,
 * mem_new, gsave) into out[0, cap); *n = its element count. */
spd_status spd_tgn_debug_scratch(spd_tgn_trainer* t, const char* name, float* out, uint64_t cap,
                                 uint64_t* n);
/* Bridge backbone: replace the TGN model inside this
 * trainer's schedule (loop-start reset, pending last messages, loop-end flush
 * + snapshot, epoch-end restore + shared sync) by the reference's surrogate
 * MSG/UPD, ModelParams {d x 3d w_m row-major, omega[d], gamma}
 * (pac_sim.hpp:47-59, pac_sim.cpp:50-104). Steps then apply the pending
 * messages only: no embedding, loss or gradients. At batch_size 1 an epoch
 * reproduces run_epoch (pac_sim.cpp:205-264). d must equal d_mem. */
spd_status spd_tgn_set_surrogate(spd_tgn_trainer* t, int32_t d, const double* w_m,
                                 const double* omega, double gamma);
/* Per-phase times (ms, CUDA events on the trainer's stream) of the last step. */
spd_status spd_tgn_kernel_times(const spd_tgn_trainer* t, float* ms, int32_t* n_kernels,
                                char* names, int32_t name_stride, int32_t cap);

/* n global steps (wrapping epochs) timed with CUDA events on the trainer's
 * stream; device_ms = elapsed device time. */
spd_status spd_tgn_run_steps(spd_tgn_trainer* t, uint64_t n, float* device_ms);
/* End-to-end step from host memory: events[k] / feats[k] hold local worker k's
 * NEXT batch (events in that worker's local ids, spd_tgn_worker_events; bf16
 * feature rows of stride feat_stride) — copied H2D, trained, losses copied back. */
spd_status spd_tgn_step_host(spd_tgn_trainer* t, const spd_edge* const* events,
                             const uint16_t* const* feats, float* loss_out);
/* Pipelined form of spd_tgn_step_host: same inputs (pin them), but host
 * staging of this batch overlaps the device's previous step (pinned staging
 * ring, copies on a copy stream the step waits on) and the per-worker losses
 * land in the caller's pinned loss_pinned asynchronously. spd_tgn_sync waits
 * for all queued steps; read loss_pinned after it. */
spd_status spd_tgn_step_host_async(spd_tgn_trainer* t, const spd_edge* const* events,
                                   const uint16_t* const* feats, float* loss_pinned);
spd_status spd_tgn_sync(spd_tgn_trainer* t);
/* Event range [lo, hi) of worker's next batch in its local stream. */
spd_status spd_tgn_next_batch(const spd_tgn_trainer* t, int32_t worker, uint64_t* lo,
                              uint64_t* hi, int32_t* feat_stride);
spd_status spd_tgn_worker_events(const spd_tgn_trainer* t, int32_t worker, spd_edge* out);
/* Number of training events of worker (the length spd_tgn_worker_events fills). */
spd_status spd_tgn_worker_event_count(const spd_tgn_trainer* t, int32_t worker, uint64_t* n);
/* Host<->device bytes moved by spd_tgn_step_host so far. */
spd_status spd_tgn_io_bytes(const spd_tgn_trainer* t, uint64_t* h2d, uint64_t* d2h);
/* Host copy of the synthetic bf16 feature rows (row stride `stride`, pad 0) of
 * edges eids[0..n): the bytes spd_tgn_step_host expects. */
spd_status spd_edge_features_bf16(uint64_t seed, const uint64_t* eids, uint64_t n, int32_t F,
                                  int32_t stride, uint16_t* out);
/* Test hook: one projection GEMM on caller-owned DEVICE buffers (row-major fp32).
 * impl 0 = FP32 FFMA, 1 = tcgen05 TF32; which 0: C = A.B^T, 1: C = A.B,
 * 2: C += A^T.B (reduction over the K rows; ws = split-K workspace). */
spd_status spd_debug_gemm(int32_t impl, int32_t which, const float* A, int32_t lda, const float* B,
                          int32_t ldb, float* C, int32_t ldc, int32_t M, int32_t N, int32_t K,
                          float* ws, uint64_t ws_floats);
/* Process-wide count of kernel launches issued by the TGN path. */
uint64_t spd_kernel_launches(void);

/* Synthetic edge feature generator (identical on host and device): value of
 * feature column c of edge eid, BF16-exact. */
float spd_edge_feature(uint64_t seed, uint64_t eid, uint32_t c);

#ifdef __cplusplus
}
#endif
#endif /* SPEED_C_H */
