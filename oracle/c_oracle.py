"""TEST INFRASTRUCTURE ONLY: ctypes access to oracle/_build/liboracle.so, our
plain-C restatement of the reference algorithms (oracle/speed_oracle.c)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "liboracle.so")
EDGE_DTYPE = np.dtype([("src", "<u4"), ("dst", "<u4"), ("ts", "<f8")])
_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(SO)
        _lib.oracle_mt_first.restype = C.c_uint64
        _lib.oracle_digest.restype = C.c_uint64
        _lib.oracle_induce_one.restype = C.c_uint64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


u64, u32, i32, f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_double


def mt_first(seed):
    return lib().oracle_mt_first(u64(seed))


def gen_powerlaw(nodes, edges, alpha, seed):
    out = np.zeros(edges, EDGE_DTYPE)
    rc = lib().oracle_gen_powerlaw(u32(nodes), u64(edges), f64(alpha), u64(seed), _p(out))
    if rc:
        raise ValueError("InvalidParams")
    return out


def compute_centrality(edges, node_count, t_max, beta=0.5, normalize=True):
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    cent = np.zeros(node_count, np.float64)
    rc = lib().oracle_compute_centrality(_p(e), u64(len(e)), u32(node_count), f64(t_max), f64(beta),
                                         i32(int(normalize)), _p(cent))
    if rc:
        raise ValueError("BetaOutOfRange")
    return cent


def select_hubs(cent, k, base_all=False):
    cent = np.ascontiguousarray(cent, np.float64)
    hubs = np.zeros(max(1, len(cent)), np.uint32)
    n = u64()
    rc = lib().oracle_select_hubs(_p(cent), u32(len(cent)), f64(k), i32(int(base_all)), _p(hubs),
                                  C.byref(n))
    if rc:
        raise ValueError("InvalidParams")
    return hubs[: n.value]


def partition_stream(edges, node_count, P, cent, hubs, lam=1.0, eps=1.0):
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    cent = np.ascontiguousarray(cent, np.float64)
    is_hub = np.zeros(max(1, node_count), np.uint8)
    is_hub[np.asarray(hubs, np.int64)] = 1
    ep = np.zeros(max(1, len(e)), np.int32)
    flat = np.zeros(max(1, node_count * P), np.int32)
    counts = np.zeros(max(1, node_count), np.uint32)
    shared = np.zeros(max(1, node_count), np.uint32)
    ns, dis = u64(), u64()
    rc = lib().oracle_partition_stream(_p(e), u64(len(e)), u32(node_count), i32(P), f64(lam),
                                       f64(eps), _p(cent), u32(len(cent)), _p(is_hub), _p(ep),
                                       _p(flat), _p(counts), _p(shared), C.byref(ns), C.byref(dis))
    if rc:
        raise ValueError(f"oracle partition status {rc}")
    node_parts = [flat[i * P:i * P + counts[i]].tolist() for i in range(node_count)]
    return dict(edge_part=ep[: len(e)], node_parts=node_parts, shared=shared[: ns.value],
                discards=dis.value)


def induce(edges, node_count, node_parts, P):
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    out = []
    for p in range(P):
        member = np.zeros(max(1, node_count), np.uint8)
        for i, parts in enumerate(node_parts):
            if p in parts:
                member[i] = 1
        idx = np.zeros(max(1, len(e)), np.uint64)
        c = lib().oracle_induce_one(_p(e), u64(len(e)), _p(member), _p(idx))
        out.append((np.nonzero(member[:node_count])[0].astype(np.uint32), idx[:c]))
    return out


def model_seeded(d, seed):
    w = np.zeros(d * 3 * d, np.float64)
    om = np.zeros(d, np.float64)
    lib().oracle_model_seeded(i32(d), u64(seed), _p(w), _p(om))
    return w, om


def model_update_run(state, last_ts, edges, w, om, gamma):
    st = np.ascontiguousarray(state, np.float64).copy()
    ts = np.ascontiguousarray(last_ts, np.float64).copy()
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    d = st.shape[1]
    for k in range(len(e)):
        rc = lib().oracle_model_update(_p(st), _p(ts), i32(d), _p(e[k:k + 1]), _p(w), _p(om),
                                       f64(gamma))
        if rc:
            raise ValueError("NonChronological")
    return st, ts


def run_epoch(sub_edges, N, d, w, om, gamma, shared, average, B):
    W = len(sub_edges)
    off = np.zeros(W + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in sub_edges])
    eds = np.concatenate([np.ascontiguousarray(x, EDGE_DTYPE) for x in sub_edges] + [np.zeros(1, EDGE_DTYPE)])
    st = np.zeros((W, N, d))
    ts = np.zeros((W, N))
    sh = np.ascontiguousarray(shared, np.uint32) if len(shared) else np.zeros(1, np.uint32)
    b = np.zeros(W, np.uint64)
    lp = np.zeros(W, np.uint64)
    rc = lib().oracle_run_epoch(i32(W), u32(N), i32(d), _p(off), _p(eds), _p(st), _p(ts), _p(w),
                                _p(om), f64(gamma), _p(sh), u64(len(shared)), i32(int(average)),
                                u64(B), _p(b), _p(lp))
    if rc:
        raise ValueError("NonChronological")
    return st, ts, b.tolist(), lp.tolist()


def sync_shared(states, clocks, shared, average):
    st = np.ascontiguousarray(states, np.float64).copy()
    ts = np.ascontiguousarray(clocks, np.float64).copy()
    W, N, d = st.shape
    sh = np.ascontiguousarray(shared, np.uint32)
    lib().oracle_sync_shared(i32(W), u32(N), i32(d), _p(st), _p(ts), _p(sh), u64(len(sh)),
                             i32(int(average)))
    return st, ts


def digest(state, clocks):
    st = np.ascontiguousarray(state, np.float64)
    ts = np.ascontiguousarray(clocks, np.float64)
    h = lib().oracle_digest(_p(st), _p(ts), u32(st.shape[0]), i32(st.shape[1]))
    return f"{h:016x}"
