"""B200-native SPEED (arXiv 2308.14129) parallel-training hot path.

Python mirror of the reference's C++ API surface (speedpart; names, argument
meaning and error behaviour follow /root/reference/proj/include/speedpart/*.hpp)
over the product C-ABI (include/speed_c.h, libspeed_b200.so). Host
partitioning runs in the library's C++; memory stores, the surrogate parity
trainer and the TGN training step run on the B200. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from ._lib import (EDGE_DTYPE, EpochReportC, PartitionerConfigC, SimConfigC, lib, ptr,
                   u32, u64, i32, f64, f32)

__all__ = [
    "EDGE_DTYPE", "DataError", "InternalError", "UsageError", "EdgeStream", "ChronoSplit",
    "gen_powerlaw", "chrono_split", "make_stream", "CentralityTable", "HubSet", "HubBase",
    "compute_centrality", "compute_degree_centrality", "select_hubs", "PartitionerConfig",
    "PartitionState", "PartitionAssignment", "score", "partition_stream",
    "partition_unrestricted", "EvalRouting", "assign_eval_edges", "SubGraph",
    "induce_subgraphs", "induce_groups", "shuffle_combine", "ModelParams", "MemoryStore", "model_update",
    "SyncStrategy", "sync_shared", "StepLog", "EpochReport", "run_epoch", "SimConfig",
    "SimReport", "simulate", "kDiscarded",
]

kDiscarded = -1  # types.hpp:12


# --------------------------------------------------------------- errors
class SpeedError(RuntimeError):
    def __init__(self, code: str, detail: str):
        super().__init__(f"{code}: {detail}")
        self.code = code
        self.detail = detail


class UsageError(SpeedError):
    pass


class DataError(SpeedError):  # errors.hpp:10-20 (CLI exit 2)
    pass


class InternalError(SpeedError):  # errors.hpp:23-32 (CLI exit 3)
    pass


def _check(status: int) -> None:
    if status == 0:
        return
    code = (lib.spd_last_error_code() or b"").decode()
    detail = (lib.spd_last_error_detail() or b"").decode()
    cls = {1: UsageError, 2: DataError}.get(status, InternalError)
    raise cls(code, detail)


# --------------------------------------------------------------- streams
@dataclass
class EdgeStream:
    """types.hpp:25-32. ``edges`` is a structured array of EDGE_DTYPE."""
    edges: np.ndarray = field(default_factory=lambda: np.zeros(0, EDGE_DTYPE))
    node_count: int = 0
    t_max: float = 0.0

    def empty(self) -> bool:
        return len(self.edges) == 0

    def size(self) -> int:
        return len(self.edges)

    def __len__(self) -> int:
        return len(self.edges)


def make_stream(edges: Iterable[tuple], node_count: int) -> EdgeStream:
    """Test helper (test_pac_sim.cpp:20-26): t_max = max ts."""
    arr = np.array([tuple(e) for e in edges], dtype=EDGE_DTYPE)
    t_max = float(arr["ts"].max()) if len(arr) else 0.0
    return EdgeStream(arr, int(node_count), t_max)


def _edges(a) -> np.ndarray:
    if isinstance(a, EdgeStream):
        a = a.edges
    a = np.ascontiguousarray(a, dtype=EDGE_DTYPE)
    return a


def gen_powerlaw(nodes: int, edges: int, alpha: float, seed: int) -> EdgeStream:
    """graph_io.hpp:34 — bit-identical synthetic power-law TIG."""
    out = np.empty(int(edges), dtype=EDGE_DTYPE)
    nc = u32()
    tm = f64()
    _check(lib.spd_gen_powerlaw(nodes, edges, alpha, seed, ptr(out), C.byref(nc), C.byref(tm)))
    return EdgeStream(out, nc.value, tm.value)


@dataclass
class ChronoSplit:  # types.hpp:35-43
    train: EdgeStream
    val: EdgeStream
    test: EdgeStream
    f_train: float
    f_val: float
    f_test: float


def _sub(s: EdgeStream, lo: int, hi: int) -> EdgeStream:
    e = s.edges[lo:hi].copy()
    return EdgeStream(e, s.node_count, float(e["ts"].max()) if len(e) else 0.0)


def chrono_split(s: EdgeStream, f_train: float, f_val: float) -> ChronoSplit:
    """graph_io.hpp:27."""
    a, b, c = u64(), u64(), u64()
    _check(lib.spd_chrono_split(len(s.edges), f_train, f_val, C.byref(a), C.byref(b), C.byref(c)))
    n_tr, n_va = a.value, b.value
    return ChronoSplit(_sub(s, 0, n_tr), _sub(s, n_tr, n_tr + n_va), _sub(s, n_tr + n_va, len(s)),
                       f_train, f_val, 1.0 - f_train - f_val)


# ------------------------------------------------------------ centrality
@dataclass
class CentralityTable:  # centrality.hpp:13-20
    cent: np.ndarray
    beta: float = 0.0
    t_max: float = 0.0

    def of(self, i: int) -> float:
        return float(self.cent[i]) if i < len(self.cent) else 0.0

    def active_count(self) -> int:
        return int((self.cent > 0).sum())


class HubBase(enum.IntEnum):  # centrality.hpp:32-35
    Active = 0
    All = 1


@dataclass
class HubSet:  # centrality.hpp:22-30
    hubs: np.ndarray
    is_hub: np.ndarray
    k: float = 0.0

    def contains(self, i: int) -> bool:
        return i < len(self.is_hub) and bool(self.is_hub[i])

    @staticmethod
    def from_ids(ids: Sequence[int], node_count: int, k: float) -> "HubSet":
        h = np.array(sorted(int(x) for x in ids), dtype=np.uint32)
        is_hub = np.zeros(node_count, dtype=np.uint8)
        is_hub[h] = 1
        return HubSet(h, is_hub, k)


def compute_centrality(s: EdgeStream, beta: float, normalize_ts: bool = True) -> CentralityTable:
    """centrality.hpp:41 (Eq. 1, order-exact f64 accumulation)."""
    e = _edges(s)
    cent = np.zeros(s.node_count, dtype=np.float64)
    tm = f64()
    _check(lib.spd_compute_centrality(ptr(e), len(e), s.node_count, s.t_max, beta,
                                      1 if normalize_ts else 0, ptr(cent, f64), C.byref(tm)))
    return CentralityTable(cent, beta, tm.value)


def compute_degree_centrality(s: EdgeStream) -> CentralityTable:
    e = _edges(s)
    cent = np.zeros(s.node_count, dtype=np.float64)
    _check(lib.spd_compute_degree_centrality(ptr(e), len(e), s.node_count, ptr(cent, f64)))
    return CentralityTable(cent, 0.0, s.t_max)


def select_hubs(c: CentralityTable, k: float, base: HubBase = HubBase.Active) -> HubSet:
    """centrality.hpp:48."""
    cent = np.ascontiguousarray(c.cent, dtype=np.float64)
    hubs = np.zeros(max(1, len(cent)), dtype=np.uint32)
    n = u64()
    _check(lib.spd_select_hubs(ptr(cent, f64), len(cent), k, int(base), ptr(hubs, u32), C.byref(n)))
    return HubSet.from_ids(hubs[: n.value], len(cent), k)


# ----------------------------------------------------------- partitioner
@dataclass
class PartitionerConfig:  # partitioner.hpp:11-17
    num_parts: int = 1
    lambda_: float = 1.0
    epsilon: float = 1.0
    hub_set: HubSet | None = None
    centrality: CentralityTable | None = None


@dataclass
class PartitionState:  # partitioner.hpp:21-36
    sizes: list
    assigned: list
    maxsize: int = 0
    minsize: int = 0


@dataclass
class PartitionAssignment:  # partitioner.hpp:40-47
    edge_part: np.ndarray
    node_parts: list
    shared: np.ndarray
    discard_count: int = 0
    num_parts: int = 1
    k_eff: float = 0.0
    np_off: np.ndarray | None = None
    np_parts: np.ndarray | None = None

    def csr(self):
        if self.np_off is None:
            off = np.zeros(len(self.node_parts) + 1, dtype=np.uint64)
            off[1:] = np.cumsum([len(v) for v in self.node_parts])
            flat = [p for v in self.node_parts for p in v]
            self.np_off = off
            self.np_parts = np.array(flat if flat else [0], dtype=np.int32)
        return self.np_off, self.np_parts


class _CfgHolder:
    """Keeps numpy buffers alive while a PartitionerConfigC points at them."""

    def __init__(self, cfg: PartitionerConfig, node_count: int):
        cent = cfg.centrality.cent if cfg.centrality is not None else np.zeros(0)
        self.cent = np.ascontiguousarray(cent, dtype=np.float64)
        hubs = cfg.hub_set.hubs if cfg.hub_set is not None else np.zeros(0)
        self.hubs = np.ascontiguousarray(hubs, dtype=np.uint32)
        k = cfg.hub_set.k if cfg.hub_set is not None else 0.0
        self.c = PartitionerConfigC(cfg.num_parts, cfg.lambda_, cfg.epsilon,
                                    ptr(self.cent, f64) if len(self.cent) else None,
                                    len(self.cent), ptr(self.hubs, u32) if len(self.hubs) else None,
                                    len(self.hubs), k)


def _assignment_from_handle(h) -> PartitionAssignment:
    npart, nc, ne, ns, dis, npt = i32(), u32(), u64(), u64(), u64(), u64()
    keff = f64()
    _check(lib.spd_assignment_info(h, C.byref(npart), C.byref(nc), C.byref(ne), C.byref(ns),
                                   C.byref(dis), C.byref(npt), C.byref(keff)))
    ep = np.empty(ne.value, dtype=np.int32)
    off = np.empty(nc.value + 1, dtype=np.uint64)
    parts = np.empty(max(1, npt.value), dtype=np.int32)
    shared = np.empty(max(1, ns.value), dtype=np.uint32)
    _check(lib.spd_assignment_edge_part(h, ptr(ep, i32)))
    _check(lib.spd_assignment_node_parts(h, ptr(off, u64), ptr(parts, i32)))
    _check(lib.spd_assignment_shared(h, ptr(shared, u32)))
    lib.spd_assignment_destroy(h)
    node_parts = [parts[off[i]:off[i + 1]].tolist() for i in range(nc.value)]
    return PartitionAssignment(ep, node_parts, shared[: ns.value], dis.value, npart.value,
                               keff.value, off, parts[: npt.value] if npt.value else parts[:0])


def _partition(fn, s: EdgeStream, cfg: PartitionerConfig) -> PartitionAssignment:
    e = _edges(s)
    holder = _CfgHolder(cfg, s.node_count)
    h = C.c_void_p()
    _check(fn(ptr(e), len(e), s.node_count, C.byref(holder.c), C.byref(h)))
    return _assignment_from_handle(h)


def partition_stream(s: EdgeStream, cfg: PartitionerConfig) -> PartitionAssignment:
    """partitioner.hpp:62 — SEP (Alg. 1), bit-identical assignment."""
    return _partition(lib.spd_partition_stream, s, cfg)


def partition_unrestricted(s: EdgeStream, cfg: PartitionerConfig) -> PartitionAssignment:
    """partitioner.hpp:66."""
    return _partition(lib.spd_partition_unrestricted, s, cfg)


def score(i: int, j: int, p: int, st: PartitionState, cfg: PartitionerConfig) -> float:
    """partitioner.hpp:50-51."""
    n = len(st.assigned)
    holder = _CfgHolder(cfg, n)
    sizes = np.array(st.sizes, dtype=np.uint64)
    off = np.zeros(n + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(v) for v in st.assigned])
    flat = np.array([q for v in st.assigned for q in v] or [0], dtype=np.int32)
    out = f64()
    _check(lib.spd_score(i, j, p, C.byref(holder.c), ptr(sizes, u64), st.maxsize, st.minsize, n,
                         ptr(off, u64), ptr(flat, i32), C.byref(out)))
    return out.value


def assignment_handle(pa: PartitionAssignment, n_edges: int | None = None):
    off, parts = pa.csr()
    off = np.ascontiguousarray(off, dtype=np.uint64)
    parts = np.ascontiguousarray(parts if len(parts) else np.zeros(1, np.int32), dtype=np.int32)
    ep = np.ascontiguousarray(pa.edge_part, dtype=np.int32) if pa.edge_part is not None else None
    h = C.c_void_p()
    _check(lib.spd_assignment_from_parts(len(off) - 1, pa.num_parts, ptr(off, u64), ptr(parts, i32),
                                         ptr(ep, i32) if ep is not None and len(ep) else None,
                                         len(ep) if ep is not None else 0, pa.discard_count,
                                         C.byref(h)))
    return h


# ------------------------------------------------------- on-disk formats
def load_edges(path: str, assume_sorted: bool = False) -> EdgeStream:
    """graph_io.hpp load_edges (graph_io.cpp:106-140): CSV src,dst,ts."""
    out = C.c_void_p()
    n, nc, tm = u64(), u32(), f64()
    _check(lib.spd_load_edges_csv(str(path).encode(), int(assume_sorted), C.byref(out), C.byref(n),
                                  C.byref(nc), C.byref(tm)))
    try:
        arr = np.empty(n.value, dtype=EDGE_DTYPE)
        if n.value:
            C.memmove(arr.ctypes.data, out.value, n.value * EDGE_DTYPE.itemsize)
    finally:
        lib.spd_free(out)
    return EdgeStream(arr, nc.value, tm.value)


def write_edges(s: EdgeStream, path: str) -> None:
    """graph_io.hpp write_edges (graph_io.cpp:142-154): %.17g timestamps."""
    e = _edges(s)
    _check(lib.spd_write_edges_csv(str(path).encode(), ptr(e) if len(e) else None, len(e)))


def write_edges_bin(s: EdgeStream, path: str) -> None:
    """Binary event file (header + TemporalEdge records); see speed_c.h."""
    e = _edges(s)
    _check(lib.spd_write_edges_bin(str(path).encode(), ptr(e) if len(e) else None, len(e),
                                   s.node_count, s.t_max))


def load_edges_bin(path: str, out: np.ndarray | None = None) -> EdgeStream:
    """Reads a binary event file into ``out`` (e.g. a pinned buffer) or a new array."""
    n, nc, tm = u64(), u32(), f64()
    _check(lib.spd_edges_bin_info(str(path).encode(), C.byref(n), C.byref(nc), C.byref(tm)))
    arr = np.empty(n.value, dtype=EDGE_DTYPE) if out is None else out[: n.value]
    if arr.dtype != EDGE_DTYPE or len(arr) < n.value or not arr.flags.c_contiguous:
        raise UsageError("Usage", "output buffer must be a contiguous EDGE_DTYPE array of n records")
    _check(lib.spd_load_edges_bin(str(path).encode(), ptr(arr) if n.value else None, n.value))
    return EdgeStream(arr, nc.value, tm.value)


def write_assignment_json(pa: PartitionAssignment, path: str, config: dict | None = None) -> None:
    """The CLI partition subcommand's output document (speedpart_main.cpp:110-119)."""
    import json
    h = assignment_handle(pa)
    try:
        cfg = json.dumps(config if config is not None else {}, separators=(",", ":"))
        _check(lib.spd_assignment_write_json(h, cfg.encode(), str(path).encode()))
    finally:
        lib.spd_assignment_destroy(h)


def load_assignment_json(path: str):
    """load_assignment (speedpart_main.cpp:129-166) -> (PartitionAssignment, config dict)."""
    import json
    h, cfg = C.c_void_p(), C.c_void_p()
    _check(lib.spd_assignment_read_json(str(path).encode(), C.byref(h), C.byref(cfg)))
    try:
        text = C.string_at(cfg.value).decode()
    finally:
        lib.spd_free(cfg)
    return _assignment_from_handle(h), json.loads(text)


@dataclass
class EvalRouting:  # partitioner.hpp:74-79
    val_edges: list
    test_edges: list
    val_unroutable: int = 0
    test_unroutable: int = 0


def assign_eval_edges(split: ChronoSplit, pa: PartitionAssignment) -> EvalRouting:
    """partitioner.hpp:81."""
    ah = assignment_handle(pa)
    v, t = _edges(split.val), _edges(split.test)
    h = C.c_void_p()
    try:
        _check(lib.spd_assign_eval_edges(ptr(v), len(v), ptr(t), len(t), ah, C.byref(h)))
    finally:
        lib.spd_assignment_destroy(ah)
    out = []
    unr = []
    for which in (0, 1):
        counts = np.zeros(pa.num_parts, dtype=np.uint64)
        un = u64()
        _check(lib.spd_eval_routing_counts(h, which, ptr(counts, u64), C.byref(un)))
        idx = np.zeros(max(1, int(counts.sum())), dtype=np.uint64)
        _check(lib.spd_eval_routing_edges(h, which, ptr(idx, u64)))
        lists, o = [], 0
        for c in counts:
            lists.append(idx[o:o + int(c)].tolist())
            o += int(c)
        out.append(lists)
        unr.append(un.value)
    lib.spd_eval_routing_destroy(h)
    return EvalRouting(out[0], out[1], unr[0], unr[1])


# ------------------------------------------------------------- subgraphs

def link_metrics(pos, neg) -> tuple[float, float]:
    """Global (AP, AUC) of link-prediction scores (spd_link_metrics): positive
    and negative scores of the routed val / test edges, concatenated over
    every partition."""
    p = np.ascontiguousarray(pos, dtype=np.float32).ravel()
    n = np.ascontiguousarray(neg, dtype=np.float32).ravel()
    ap, auc = C.c_double(), C.c_double()
    _check(lib.spd_link_metrics(ptr(p, C.c_float), len(p), ptr(n, C.c_float), len(n),
                                C.byref(ap), C.byref(auc)))
    return ap.value, auc.value


def gather_link_metrics(pos, neg, allgather=None) -> tuple[float, float]:
    """Multi-rank evaluation: every rank scores the eval edges
    routed to its partitions (TGNTrainer.evaluate); the score lists of all
    ranks are gathered in rank order and the global AP / AUC computed once.

    ``allgather(obj) -> list`` collects one object per rank; by default
    torch.distributed's all_gather_object when a process group is initialised
    (the launcher's plumbing), else the local lists alone (one rank)."""
    mine = (np.asarray(pos, np.float32).ravel(), np.asarray(neg, np.float32).ravel())
    if allgather is None:
        try:
            import torch.distributed as dist
            ready = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        except ImportError:
            ready = False
        if ready:
            def allgather(obj):
                out = [None] * dist.get_world_size()
                dist.all_gather_object(out, obj)
                return out
    parts = allgather(mine) if allgather is not None else [mine]
    return link_metrics(np.concatenate([p for p, _ in parts]), np.concatenate([n for _, n in parts]))

@dataclass
class SubGraph:  # pac_sim.hpp:12-15 (+ stream positions for feature lookup)
    nodes: np.ndarray
    edges: np.ndarray
    eids: np.ndarray


def _subgraphs_from_handle(h) -> list:
    cnt = i32()
    _check(lib.spd_subgraphs_count(h, C.byref(cnt)))
    subs = []
    for p in range(cnt.value):
        nn, ne = u64(), u64()
        _check(lib.spd_subgraph_sizes(h, p, C.byref(nn), C.byref(ne)))
        nodes = np.empty(nn.value, dtype=np.uint32)
        edges = np.empty(ne.value, dtype=EDGE_DTYPE)
        eids = np.empty(ne.value, dtype=np.uint64)
        if nn.value:
            _check(lib.spd_subgraph_nodes(h, p, ptr(nodes, u32)))
        if ne.value:
            _check(lib.spd_subgraph_edges(h, p, ptr(edges), ptr(eids, u64)))
        subs.append(SubGraph(nodes, edges, eids))
    return subs


def induce_subgraphs(s: EdgeStream, node_parts, num_parts: int) -> list:
    """pac_sim.hpp:102-104."""
    e = _edges(s)
    off = np.zeros(len(node_parts) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(v) for v in node_parts])
    flat = np.array([p for v in node_parts for p in v] or [0], dtype=np.int32)
    h = C.c_void_p()
    _check(lib.spd_induce_subgraphs(ptr(e), len(e), s.node_count, ptr(off, u64), ptr(flat, i32),
                                    len(node_parts), num_parts, C.byref(h)))
    try:
        return _subgraphs_from_handle(h)
    finally:
        lib.spd_subgraphs_destroy(h)


def induce_groups(s: EdgeStream, groups: Sequence[Sequence[int]],
                  small: Sequence[Sequence[int]]):
    """One epoch of simulate's shuffle branch (pac_sim.cpp:306-326): the
    subgraph induced by each combined group, and the `recovered` count (edges
    some group induces that no small part does)."""
    e = _edges(s)

    def csr(lists):
        off = np.zeros(len(lists) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(v) for v in lists])
        flat = np.array([x for v in lists for x in v] or [0], dtype=np.uint32)
        return off, flat
    go, gn = csr(groups)
    so, sn = csr(small)
    h = C.c_void_p()
    rec = u64()
    _check(lib.spd_induce_groups(ptr(e), len(e), s.node_count, ptr(go, u64), ptr(gn, u32),
                                 len(groups), ptr(so, u64), ptr(sn, u32), len(small), C.byref(h),
                                 C.byref(rec)))
    try:
        return _subgraphs_from_handle(h), rec.value
    finally:
        lib.spd_subgraphs_destroy(h)


def subgraphs_handle(subs: Sequence[SubGraph]):
    """Opaque spd_subgraphs* for a list of SubGraph (caller destroys)."""
    n = len(subs)
    no = np.zeros(n + 1, dtype=np.uint64)
    eo = np.zeros(n + 1, dtype=np.uint64)
    no[1:] = np.cumsum([len(g.nodes) for g in subs])
    eo[1:] = np.cumsum([len(g.edges) for g in subs])
    nodes = np.concatenate([np.asarray(g.nodes, np.uint32) for g in subs] + [np.zeros(1, np.uint32)])
    edges = np.concatenate([_edges(g.edges) for g in subs] + [np.zeros(1, EDGE_DTYPE)])
    eids = np.concatenate([np.asarray(g.eids if g.eids is not None else np.arange(len(g.edges)),
                                      np.uint64) for g in subs] + [np.zeros(1, np.uint64)])
    h = C.c_void_p()
    _check(lib.spd_subgraphs_from_lists(n, ptr(no, u64), ptr(nodes, u32), ptr(eo, u64), ptr(edges),
                                        ptr(eids, u64), C.byref(h)))
    return h


def shuffle_combine(small: Sequence[Sequence[int]], num_workers: int, epoch_seed: int) -> list:
    """pac_sim.hpp:108-110."""
    off = np.zeros(len(small) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(v) for v in small])
    flat = np.array([x for v in small for x in v] or [0], dtype=np.uint32)
    out_off = np.zeros(max(1, num_workers) + 1, dtype=np.uint64)
    out = np.zeros(max(1, len(flat)), dtype=np.uint32)
    _check(lib.spd_shuffle_combine(ptr(off, u64), ptr(flat, u32), len(small), num_workers,
                                   epoch_seed, ptr(out_off, u64), ptr(out, u32)))
    return [out[out_off[g]:out_off[g + 1]].tolist() for g in range(num_workers)]


def lockstep_schedule(subgraphs: Sequence[SubGraph], batch_size: int):
    """Host evaluation of run_epoch's Alg. 2 schedule: (n_steps, StepLog rows,
    batches, loops) — identical on every rank of a multi-GPU run."""
    h = subgraphs_handle(subgraphs)
    W = len(subgraphs)
    try:
        n = u64()
        cap = 1 << 20
        log = np.zeros(4 * cap, np.uint64)
        nl = u64()
        b = np.zeros(max(1, W), np.uint64)
        lp = np.zeros(max(1, W), np.uint64)
        _check(lib.spd_lockstep_schedule(h, batch_size, C.byref(n), ptr(log, u64), cap, C.byref(nl),
                                         ptr(b, u64), ptr(lp, u64)))
    finally:
        lib.spd_subgraphs_destroy(h)
    rows = [tuple(int(x) for x in log[4 * k:4 * k + 4]) for k in range(nl.value)]
    return n.value, rows, b[:W].tolist(), lp[:W].tolist()


# ------------------------------------------------- surrogate (parity mode)
@dataclass
class ModelParams:  # pac_sim.hpp:47-55
    d: int = 8
    gamma: float = 0.5
    w_m: np.ndarray = field(default_factory=lambda: np.zeros(0))
    omega: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @staticmethod
    def seeded(d: int, seed: int) -> "ModelParams":
        w = np.zeros(max(1, d * 3 * d), dtype=np.float64)
        om = np.zeros(max(1, d), dtype=np.float64)
        g = f64()
        _check(lib.spd_model_seeded(d, seed, ptr(w, f64), ptr(om, f64), C.byref(g)))
        return ModelParams(d, g.value, w, om)


class MemoryStore:
    """pac_sim.hpp:19-39, resident in HBM of `device` (f64 rows + f64 clock)."""

    def __init__(self, node_count: int, d: int, device: int = 0):
        self.node_count = int(node_count)
        self.d = int(d)
        self.device = device
        self._h = C.c_void_p()
        _check(lib.spd_memstore_create(self.node_count, self.d, device, C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.spd_memstore_destroy(h)
            self._h = None

    def download(self):
        st = np.zeros(self.node_count * self.d, dtype=np.float64)
        ts = np.zeros(self.node_count, dtype=np.float64)
        _check(lib.spd_memstore_download(self._h, ptr(st, f64), ptr(ts, f64)))
        return st.reshape(self.node_count, self.d), ts

    def upload(self, state, last_ts):
        st = np.ascontiguousarray(state, dtype=np.float64).reshape(-1)
        ts = np.ascontiguousarray(last_ts, dtype=np.float64)
        _check(lib.spd_memstore_upload(self._h, ptr(st, f64), ptr(ts, f64)))

    @property
    def state(self) -> np.ndarray:
        return self.download()[0]

    @property
    def last_ts(self) -> np.ndarray:
        return self.download()[1]

    def row(self, i: int) -> np.ndarray:
        return self.state[i]

    def reset(self):
        _check(lib.spd_memstore_reset(self._h))

    def copy_from(self, other: "MemoryStore"):
        _check(lib.spd_memstore_copy(self._h, other._h))

    def digest(self) -> str:
        buf = C.create_string_buffer(17)
        _check(lib.spd_memstore_digest(self._h, buf))
        return buf.value.decode()


def model_update(mem: MemoryStore, edges, model: ModelParams) -> None:
    """pac_sim.hpp:59, for one edge or a run of edges (applied in order)."""
    if isinstance(edges, tuple):
        edges = [edges]
    e = np.array([tuple(x) for x in edges], dtype=EDGE_DTYPE) if isinstance(edges, list) else _edges(edges)
    w = np.ascontiguousarray(model.w_m, dtype=np.float64)
    om = np.ascontiguousarray(model.omega, dtype=np.float64)
    _check(lib.spd_model_update(mem._h, ptr(e), len(e), ptr(w, f64), ptr(om, f64), model.gamma))


class SyncStrategy(enum.IntEnum):  # pac_sim.hpp:61
    MaxTimestamp = 0
    Average = 1


def sync_shared(mems: Sequence[MemoryStore], shared, strategy: SyncStrategy) -> None:
    """pac_sim.hpp:125-126."""
    arr = (C.c_void_p * max(1, len(mems)))(*[m._h for m in mems])
    sh = np.ascontiguousarray(np.asarray(list(shared), dtype=np.uint32))
    _check(lib.spd_sync_shared(arr, len(mems), ptr(sh, u32) if len(sh) else None, len(sh),
                               int(strategy)))


@dataclass
class StepLog:  # pac_sim.hpp:88-100
    steps: list = field(default_factory=list)      # (global_step, worker, loop, batch_in_loop)
    snapshots: list = field(default_factory=list)  # (worker, digest)


@dataclass
class EpochReport:  # pac_sim.hpp:75-81
    batches: list
    loops: list
    recovered: int = 0
    sync_events: int = 0
    digests: list = field(default_factory=list)


def run_epoch(subgraphs: Sequence[SubGraph], mems: Sequence[MemoryStore], model: ModelParams,
              shared, sync: SyncStrategy, batch_size: int, log: StepLog | None = None) -> EpochReport:
    """pac_sim.hpp:117-120 — lockstep loop-within-epoch on device memory stores."""
    W = len(subgraphs)
    if len(mems) != W:
        raise DataError("ConfigMismatch", "one memory store per worker required")
    h = subgraphs_handle(subgraphs)
    try:
        arr = (C.c_void_p * max(1, W))(*[m._h for m in mems])
        sh = np.ascontiguousarray(np.asarray(list(shared), dtype=np.uint32))
        batches = np.zeros(max(1, W), dtype=np.uint64)
        loops = np.zeros(max(1, W), dtype=np.uint64)
        digests = C.create_string_buffer(17 * max(1, W))
        rep = EpochReportC()
        rep.batches = ptr(batches, u64)
        rep.loops = ptr(loops, u64)
        rep.digests = C.cast(digests, C.c_void_p)
        if log is not None:
            cap = 1 << 16
            steps = np.zeros(4 * cap, dtype=np.uint64)
            snap_w = np.zeros(cap, dtype=np.int32)
            snap_d = C.create_string_buffer(17 * cap)
            rep.log_cap = cap
            rep.log_steps = ptr(steps, u64)
            rep.snap_worker = ptr(snap_w, i32)
            rep.snap_digests = C.cast(snap_d, C.c_void_p)
        w = np.ascontiguousarray(model.w_m, dtype=np.float64)
        om = np.ascontiguousarray(model.omega, dtype=np.float64)
        _check(lib.spd_run_epoch(h, arr, W, ptr(w, f64), ptr(om, f64), model.gamma,
                                 ptr(sh, u32) if len(sh) else None, len(sh), int(sync), batch_size,
                                 C.byref(rep)))
    finally:
        lib.spd_subgraphs_destroy(h)
    if log is not None:
        for k in range(rep.n_log):
            log.steps.append(tuple(int(x) for x in steps[4 * k:4 * k + 4]))
        for k in range(rep.n_snap):
            log.snapshots.append((int(snap_w[k]), snap_d.raw[17 * k:17 * k + 16].decode()))
    dg = [digests.raw[17 * w:17 * w + 16].decode() for w in range(W)]
    return EpochReport(batches[:W].tolist(), loops[:W].tolist(), 0, rep.sync_events, dg)


@dataclass
class SimConfig:  # pac_sim.hpp:63-73
    num_workers: int = 1
    num_small_parts: int = 1
    shuffle: bool = False
    sync: SyncStrategy = SyncStrategy.MaxTimestamp
    batch_size: int = 1
    epochs: int = 1
    d: int = 8
    model_seed: int = 0
    shuffle_seed: int = 0


@dataclass
class SimReport:  # pac_sim.hpp:83-86
    epochs: list
    sync_events: int = 0


def simulate(s: EdgeStream, pa: PartitionAssignment, cfg: SimConfig, device: int = 0) -> SimReport:
    """pac_sim.hpp:132-133."""
    e = _edges(s)
    ah = assignment_handle(pa)
    E = max(1, cfg.epochs)
    W = max(1, cfg.num_workers)
    rec = np.zeros(E, np.uint64)
    syn = np.zeros(E, np.uint64)
    loops = np.zeros(E * W, np.uint64)
    dg = C.create_string_buffer(17 * E * W)
    tot = u64()
    c = SimConfigC(cfg.num_workers, cfg.num_small_parts, int(cfg.shuffle), int(cfg.sync),
                   cfg.batch_size, cfg.epochs, cfg.d, cfg.model_seed, cfg.shuffle_seed)
    try:
        _check(lib.spd_simulate(ptr(e), len(e), s.node_count, ah, C.byref(c), device, ptr(rec, u64),
                                ptr(syn, u64), ptr(loops, u64), C.cast(dg, C.c_void_p), C.byref(tot)))
    finally:
        lib.spd_assignment_destroy(ah)
    eps = []
    for ep in range(cfg.epochs):
        digs = [dg.raw[17 * (ep * W + w):17 * (ep * W + w) + 16].decode() for w in range(W)]
        eps.append(EpochReport([], loops[ep * W:(ep + 1) * W].tolist(), int(rec[ep]), int(syn[ep]), digs))
    return SimReport(eps, tot.value)


# ------------------------------------------------------ TGN training path
from ._lib import TGNConfigC  # noqa: E402


@dataclass
class TGNConfig:
    """spd_tgn_config (include/speed_c.h). Defaults: TGN paper dims."""
    d_mem: int = 100
    d_time: int = 100
    d_edge: int = 172
    n_neighbors: int = 10
    n_heads: int = 2
    batch_size: int = 200
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    seed_init: int = 3
    seed_feat: int = 2
    seed_neg: int = 4
    sync_average: int = 1
    gemm_mode: int = 0
    backbone: int = 0  # 0 TGN, 1 JODIE, 2 DyRep
    concurrent: int = 0  # 1: local workers train concurrently (world 1)

    def c(self) -> TGNConfigC:
        return TGNConfigC(self.d_mem, self.d_time, self.d_edge, self.n_neighbors, self.n_heads,
                          self.batch_size, self.lr, self.beta1, self.beta2, self.adam_eps,
                          self.seed_init, self.seed_feat, self.seed_neg, self.sync_average,
                          self.gemm_mode, self.backbone, self.concurrent)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId of the libnccl the library binds at run time (one
    already loaded into the process, else $SPD_NCCL_LIB, else the system's)."""
    buf = C.create_string_buffer(128)
    _check(lib.spd_nccl_unique_id(buf))
    return buf.raw


class TGNTrainer:
    """Per-process TGN trainer over the SEP partitions `workers` (default: all)
    of `subgraphs`, on `device`; world>1 joins an NCCL communicator (nccl_id)
    or, without an id, the peer-memory transport (peer_export / peer_connect)."""

    def __init__(self, cfg: TGNConfig, subgraphs: Sequence[SubGraph], workers=None, shared=(),
                 node_count: int | None = None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, device: int = 0):
        self.cfg = cfg
        self.workers = list(range(len(subgraphs))) if workers is None else list(workers)
        if node_count is None:
            node_count = int(max([int(g.nodes.max()) + 1 for g in subgraphs if len(g.nodes)] + [0]))
        self._events_per_worker = {w: len(subgraphs[w].edges) for w in self.workers}
        sh = subgraphs_handle(subgraphs)
        try:
            ws = np.array(self.workers or [0], np.int32)
            shared = np.ascontiguousarray(np.asarray(list(shared), np.uint32))
            self._c = cfg.c()
            self._h = C.c_void_p()
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            _check(lib.spd_tgn_create(C.byref(self._c), sh, ptr(ws, i32), len(self.workers),
                                      ptr(shared, u32) if len(shared) else None, len(shared),
                                      node_count, rank, world, idbuf, device, C.byref(self._h)))
        finally:
            lib.spd_subgraphs_destroy(sh)
        n = u64()
        _check(lib.spd_tgn_param_count(self._h, C.byref(n)))
        self.n_params = n.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.spd_tgn_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def attach_stream(self, stream: "EdgeStream", small: Sequence[Sequence[int]]):
        """Keep the training stream and the small SEP parts (node lists) in HBM
        for device-side shuffle-combine (spd_tgn_attach_stream)."""
        e = _edges(stream)
        off = np.zeros(len(small) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(v) for v in small])
        flat = np.array([x for v in small for x in v] or [0], dtype=np.uint32)
        _check(lib.spd_tgn_attach_stream(self._h, e.ctypes.data if len(e) else None, len(e),
                                         stream.node_count, ptr(off, u64), ptr(flat, u32), len(small)))

    def shuffle_epoch(self, epoch_seed: int) -> int:
        """Regroup the attached small parts (shuffle_combine's permutation for
        epoch_seed) and re-induce every worker on the device; returns the
        `recovered` count (spd_tgn_shuffle_epoch)."""
        r = u64()
        _check(lib.spd_tgn_shuffle_epoch(self._h, epoch_seed, C.byref(r)))
        return r.value

    def set_surrogate(self, model: "ModelParams"):
        """Bridge backbone: the reference's surrogate MSG/UPD replaces the GRU
        in this trainer's schedule (spd_tgn_set_surrogate)."""
        w = np.ascontiguousarray(model.w_m, np.float64)
        om = np.ascontiguousarray(model.omega, np.float64)
        _check(lib.spd_tgn_set_surrogate(self._h, model.d, ptr(w, f64), ptr(om, f64), model.gamma))

    def peer_export(self) -> bytes:
        """This rank's peer-transport blob (world > 1 without an NCCL id):
        gather every rank's blob in rank order, then peer_connect."""
        buf = C.create_string_buffer(int(lib.spd_tgn_peer_blob_bytes()))
        _check(lib.spd_tgn_peer_export(self._h, buf))
        return buf.raw

    def peer_connect(self, blobs: Sequence[bytes]):
        raw = b"".join(blobs)
        _check(lib.spd_tgn_peer_connect(self._h, C.create_string_buffer(raw, len(raw))))

    def epoch_steps(self) -> int:
        n = u64()
        _check(lib.spd_tgn_epoch_steps(self._h, C.byref(n)))
        return n.value

    def begin_epoch(self, epoch: int):
        _check(lib.spd_tgn_begin_epoch(self._h, epoch))

    def rebind(self, subgraphs: Sequence[SubGraph]):
        """Shuffle-combine: train the next epoch on regrouped subgraphs
        (spd_tgn_rebind; parameters and Adam state carry over)."""
        sh = subgraphs_handle(subgraphs)
        try:
            _check(lib.spd_tgn_rebind(self._h, sh))
        finally:
            lib.spd_subgraphs_destroy(sh)
        self._events_per_worker = {w: len(subgraphs[w].edges) for w in self.workers}

    def seek(self, step: int):
        """Position the schedule at global step `step` of this epoch (spd_tgn_seek)."""
        _check(lib.spd_tgn_seek(self._h, step))

    def step(self, want_loss: bool = True):
        if not want_loss:
            _check(lib.spd_tgn_step(self._h, None))
            return None
        out = np.zeros(max(1, len(self.workers)), np.float32)
        _check(lib.spd_tgn_step(self._h, ptr(out, f32)))
        return out[: len(self.workers)]

    def end_epoch(self):
        _check(lib.spd_tgn_end_epoch(self._h))

    def run_epoch(self, epoch: int) -> float:
        m = f64()
        _check(lib.spd_tgn_run_epoch(self._h, epoch, C.byref(m)))
        return m.value

    def params(self) -> np.ndarray:
        out = np.zeros(self.n_params, np.float32)
        _check(lib.spd_tgn_get_params(self._h, ptr(out, f32)))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, np.float32)
        _check(lib.spd_tgn_set_params(self._h, ptr(p, f32)))

    def grads(self) -> np.ndarray:
        out = np.zeros(self.n_params, np.float32)
        _check(lib.spd_tgn_get_grads(self._h, ptr(out, f32)))
        return out

    def local_nodes(self, w: int) -> np.ndarray:
        n = u64()
        _check(lib.spd_tgn_local_nodes(self._h, w, C.byref(n), None))
        out = np.zeros(max(1, n.value), np.uint32)
        _check(lib.spd_tgn_local_nodes(self._h, w, C.byref(n), ptr(out, u32)))
        return out[: n.value]

    def memory(self, w: int):
        n = len(self.local_nodes(w))
        mem = np.zeros(max(1, n * self.cfg.d_mem), np.float32)
        lu = np.zeros(max(1, n), np.float64)
        _check(lib.spd_tgn_get_memory(self._h, w, ptr(mem, f32), ptr(lu, f64)))
        return mem[: n * self.cfg.d_mem].reshape(n, self.cfg.d_mem), lu[:n]

    def set_memory(self, w: int, mem, lu):
        mem = np.ascontiguousarray(mem, np.float32)
        lu = np.ascontiguousarray(lu, np.float64)
        _check(lib.spd_tgn_set_memory(self._h, w, ptr(mem, f32), ptr(lu, f64)))

    def set_debug(self, on: bool = True):
        _check(lib.spd_tgn_set_debug(self._h, int(on)))

    def debug_scratch(self, name: str) -> np.ndarray:
        """Copy of a per-step scratch buffer (x_gru, h_gru, Gi, Gh, mem_new, gsave)."""
        n = u64()
        _check(lib.spd_tgn_debug_scratch(self._h, name.encode(), None, 0, C.byref(n)))
        out = np.zeros(n.value, np.float32)
        _check(lib.spd_tgn_debug_scratch(self._h, name.encode(), ptr(out, f32), n.value, C.byref(n)))
        return out

    def set_gemm_mode(self, mode: int):
        """0 = FP32 FFMA everywhere, 1 = tcgen05 TF32 GRU/attention projections."""
        _check(lib.spd_tgn_set_gemm_mode(self._h, int(mode)))
        self.cfg.gemm_mode = int(mode)

    def set_graph(self, on: bool):
        """Replay regular steps as a captured CUDA graph (default on)."""
        _check(lib.spd_tgn_set_graph(self._h, int(on)))

    def set_profile(self, on: bool = True):
        _check(lib.spd_tgn_set_profile(self._h, int(on)))

    def last_step(self, w: int):
        b = u64()
        cfg = self.cfg
        B = cfg.batch_size
        emb = np.zeros(3 * B * cfg.d_mem, np.float32)
        negs = np.zeros(B, np.uint32)
        nbr = np.zeros(3 * B * cfg.n_neighbors, np.uint32)
        loss = f32()
        _check(lib.spd_tgn_last_step(self._h, w, C.byref(b), ptr(emb, f32), ptr(negs, u32),
                                     ptr(nbr, u32), C.byref(loss)))
        n = b.value
        return dict(b=n, emb=emb[: 3 * n * cfg.d_mem].reshape(3 * n, cfg.d_mem), neg=negs[:n],
                    nbr=nbr[: 3 * n * cfg.n_neighbors].reshape(3 * n, cfg.n_neighbors),
                    loss=loss.value)

    def set_eval_events(self, w: int, edges, eids):
        """Routed val then test edges of worker w (global ids, time order)."""
        e = _edges(edges)
        ids = np.ascontiguousarray(eids, np.uint64)
        _check(lib.spd_tgn_set_eval_events(self._h, w, ptr(e), ptr(ids, u64), len(e)))

    def evaluate(self, w: int, lo: int, hi: int, neg_seed: int = 5):
        """Logits of eval events [lo, hi) and of one sampled negative each."""
        pos = np.zeros(max(1, hi - lo), np.float32)
        neg = np.zeros(max(1, hi - lo), np.float32)
        _check(lib.spd_tgn_evaluate(self._h, w, lo, hi, neg_seed, ptr(pos, f32), ptr(neg, f32)))
        return pos[: hi - lo], neg[: hi - lo]

    def run_steps(self, n: int) -> float:
        """n lockstep steps timed on the trainer's stream (device ms)."""
        ms = f32()
        _check(lib.spd_tgn_run_steps(self._h, n, C.byref(ms)))
        return ms.value

    def next_batch(self, w: int):
        lo, hi = u64(), u64()
        fs = i32()
        _check(lib.spd_tgn_next_batch(self._h, w, C.byref(lo), C.byref(hi), C.byref(fs)))
        return lo.value, hi.value, fs.value

    def worker_events(self, w: int) -> np.ndarray:
        n = len(self.local_nodes(w))  # noqa: F841 (validates the worker id)
        lo, hi, _ = self.next_batch(w)
        cnt = u64()
        # size from the subgraph: total events = epoch batches * B upper bound; ask C side
        out = np.zeros(self._n_events(w), EDGE_DTYPE)
        _check(lib.spd_tgn_worker_events(self._h, w, ptr(out)))
        return out

    def _n_events(self, w: int) -> int:
        n = u64()
        _check(lib.spd_tgn_worker_event_count(self._h, w, C.byref(n)))
        return n.value

    def step_host(self, events: list, feats: list | None) -> np.ndarray:
        """End-to-end step: per local worker, its next batch's events (local ids)
        and bf16 feature rows (uint16) in host memory (pin them for async H2D)."""
        ev = (C.c_void_p * len(events))(*[e.ctypes.data for e in events])
        ft = (C.c_void_p * len(events))(*[f.ctypes.data for f in feats]) if feats else None
        out = np.zeros(max(1, len(self.workers)), np.float32)
        _check(lib.spd_tgn_step_host(self._h, ev, ft, ptr(out, f32)))
        return out[: len(self.workers)]

    def step_host_async(self, events: list, feats: list | None, loss_pinned: np.ndarray):
        """Pipelined end-to-end step (spd_tgn_step_host_async): inputs as
        step_host (pinned), losses land in `loss_pinned` (float32[workers],
        pinned) once `sync()` returns. Keep the inputs alive until then."""
        ev = (C.c_void_p * len(events))(*[e.ctypes.data for e in events])
        ft = (C.c_void_p * len(events))(*[f.ctypes.data for f in feats]) if feats else None
        if loss_pinned.dtype != np.float32 or len(loss_pinned) < len(self.workers):
            raise UsageError("Usage", "loss_pinned must be float32[n_workers]")
        _check(lib.spd_tgn_step_host_async(self._h, ev, ft, loss_pinned.ctypes.data))

    def sync(self):
        _check(lib.spd_tgn_sync(self._h))

    def io_bytes(self):
        a, b = u64(), u64()
        _check(lib.spd_tgn_io_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def kernel_times(self):
        cap, stride = 256, 48
        ms = np.zeros(cap, np.float32)
        n = i32()
        names = C.create_string_buffer(cap * stride)
        _check(lib.spd_tgn_kernel_times(self._h, ptr(ms, f32), C.byref(n), names, stride, cap))
        return [(names.raw[k * stride:(k + 1) * stride].split(b"\0")[0].decode(), float(ms[k]))
                for k in range(n.value)]


def kernel_launches() -> int:
    """Process-wide count of kernels the TGN path has launched."""
    return int(lib.spd_kernel_launches())


def edge_features_bf16(seed: int, eids: np.ndarray, F: int, stride: int, out=None) -> np.ndarray:
    """Host bf16 bits (uint16) of the synthetic feature rows of `eids`."""
    eids = np.ascontiguousarray(eids, np.uint64)
    if out is None:
        out = np.zeros((len(eids), stride), np.uint16)
    _check(lib.spd_edge_features_bf16(seed, ptr(eids, u64), len(eids), F, stride, ptr(out)))
    return out


def edge_feature(seed: int, eid: int, c: int) -> float:
    return float(lib.spd_edge_feature(seed, eid, c))
