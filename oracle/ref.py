"""TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline / --impl reference).

ctypes access to oracle/_ref/libspeedpart_ref.so — the UNMODIFIED reference
library (speedpart, /root/reference/proj/src/*.cpp) compiled by oracle/Makefile
plus our extern "C" veneer oracle/ref_shim.cpp. Each wrapper names the
reference function it drives.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libspeedpart_ref.so")
EDGE_DTYPE = np.dtype([("src", "<u4"), ("dst", "<u4"), ("ts", "<f8")])

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        _lib = C.CDLL(REF_SO)
        _lib.ref_last_error_code.restype = C.c_char_p
        _lib.ref_last_error_detail.restype = C.c_char_p
        for n in ("ref_gen_powerlaw", "ref_chrono_split_sizes", "ref_compute_centrality",
                  "ref_select_hubs", "ref_score", "ref_partition", "ref_assign_eval_edges",
                  "ref_induce_subgraphs", "ref_shuffle_combine", "ref_model_seeded",
                  "ref_model_update_run", "ref_model_update_threads", "ref_sync_shared",
                  "ref_digest", "ref_run_epoch", "ref_simulate", "ref_quality",
                  "ref_load_edges", "ref_write_edges"):
            getattr(_lib, n).restype = C.c_int
    return _lib


class RefError(RuntimeError):
    def __init__(self, status, code, detail):
        super().__init__(f"[{status}] {code}: {detail}")
        self.status, self.code, self.detail = status, code, detail


def _chk(st):
    if st:
        L = lib()
        raise RefError(st, L.ref_last_error_code().decode(), L.ref_last_error_detail().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


u64, u32, i32, f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_double


def _take(ptr, n, dtype):
    if n == 0:
        lib().ref_free(ptr)
        return np.zeros(0, dtype)
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))), (n,)).copy()
    lib().ref_free(ptr)
    return arr


def gen_powerlaw(nodes, edges, alpha, seed):
    """graph_io.cpp:175-250."""
    out = np.empty(edges, EDGE_DTYPE)
    nc, tm = u32(), f64()
    _chk(lib().ref_gen_powerlaw(u32(nodes), u64(edges), f64(alpha), u64(seed), _p(out),
                                C.byref(nc), C.byref(tm)))
    return out, nc.value, tm.value


def chrono_split_sizes(n, f_train, f_val):
    a, b, c = u64(), u64(), u64()
    _chk(lib().ref_chrono_split_sizes(u64(n), f64(f_train), f64(f_val), C.byref(a), C.byref(b),
                                      C.byref(c)))
    return a.value, b.value, c.value


def compute_centrality(edges, node_count, t_max, beta=0.5, normalize=True, degree=False):
    """centrality.cpp:27-64."""
    cent = np.zeros(node_count, np.float64)
    tm = f64()
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    _chk(lib().ref_compute_centrality(_p(e), u64(len(e)), u32(node_count), f64(t_max), f64(beta),
                                      i32(int(normalize)), i32(int(degree)), _p(cent), C.byref(tm)))
    return cent, tm.value


def select_hubs(cent, k, base_all=False):
    cent = np.ascontiguousarray(cent, np.float64)
    hubs = np.zeros(max(1, len(cent)), np.uint32)
    n = u64()
    _chk(lib().ref_select_hubs(_p(cent), u32(len(cent)), f64(k), i32(int(base_all)), _p(hubs),
                               C.byref(n)))
    return hubs[: n.value]


def partition(edges, node_count, t_max, num_parts, cent, hubs, k, lam=1.0, eps=1.0, mode=0, seed=0):
    """mode 0 partition_stream (partitioner.cpp:152), 1 unrestricted (:156), 2 random (:165)."""
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    cent = np.ascontiguousarray(cent, np.float64)
    hubs = np.ascontiguousarray(hubs, np.uint32)
    ep = np.zeros(max(1, len(e)), np.int32)
    npo, npp, sh = C.c_void_p(), C.c_void_p(), C.c_void_p()
    nsh, dis, keff = u64(), u64(), f64()
    _chk(lib().ref_partition(i32(mode), _p(e), u64(len(e)), u32(node_count), f64(t_max),
                             i32(num_parts), f64(lam), f64(eps), _p(cent), u32(len(cent)),
                             _p(hubs), u64(len(hubs)), f64(k), u64(seed), _p(ep),
                             C.byref(npo), C.byref(npp), C.byref(sh), C.byref(nsh), C.byref(dis),
                             C.byref(keff)))
    off = _take(npo, node_count + 1, np.uint64)
    parts = _take(npp, int(off[-1]), np.int32)
    shared = _take(sh, nsh.value, np.uint32)
    node_parts = [parts[off[i]:off[i + 1]].tolist() for i in range(node_count)]
    return dict(edge_part=ep[: len(e)], node_parts=node_parts, np_off=off, np_parts=parts,
                shared=shared, discards=dis.value, k_eff=keff.value)


def induce_subgraphs(edges, node_count, node_parts, num_parts):
    """pac_sim.cpp:106-132 -> list of (nodes, edges)."""
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    off = np.zeros(len(node_parts) + 1, np.uint64)
    off[1:] = np.cumsum([len(v) for v in node_parts])
    flat = np.array([p for v in node_parts for p in v] or [0], np.int32)
    no, nn, eo, ee = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    _chk(lib().ref_induce_subgraphs(_p(e), u64(len(e)), u32(node_count), _p(off), _p(flat),
                                    u32(len(node_parts)), i32(num_parts), C.byref(no), C.byref(nn),
                                    C.byref(eo), C.byref(ee)))
    noff = _take(no, num_parts + 1, np.uint64)
    nodes = _take(nn, int(noff[-1]), np.uint32)
    eoff = _take(eo, num_parts + 1, np.uint64)
    eds = _take(ee, int(eoff[-1]), EDGE_DTYPE)
    return [(nodes[noff[p]:noff[p + 1]], eds[eoff[p]:eoff[p + 1]]) for p in range(num_parts)]


def shuffle_combine(small, num_workers, seed):
    off = np.zeros(len(small) + 1, np.uint64)
    off[1:] = np.cumsum([len(v) for v in small])
    flat = np.array([x for v in small for x in v] or [0], np.uint32)
    oo, on = C.c_void_p(), C.c_void_p()
    _chk(lib().ref_shuffle_combine(_p(off), _p(flat), u64(len(small)), i32(num_workers), u64(seed),
                                   C.byref(oo), C.byref(on)))
    o = _take(oo, num_workers + 1, np.uint64)
    n = _take(on, int(o[-1]), np.uint32)
    return [n[o[g]:o[g + 1]].tolist() for g in range(num_workers)]


def model_seeded(d, seed):
    """pac_sim.cpp:28-46."""
    w = np.zeros(d * 3 * d, np.float64)
    om = np.zeros(d, np.float64)
    g = f64()
    _chk(lib().ref_model_seeded(i32(d), u64(seed), _p(w), _p(om), C.byref(g)))
    return w, om, g.value


def model_update_run(state, last_ts, edges, w, om, gamma):
    """pac_sim.cpp:68-104 over a run of edges (in-place on copies)."""
    st = np.ascontiguousarray(state, np.float64).copy()
    ts = np.ascontiguousarray(last_ts, np.float64).copy()
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    n, d = st.shape
    _chk(lib().ref_model_update_run(u32(n), i32(d), _p(st), _p(ts), _p(e), u64(len(e)), _p(w),
                                    _p(om), f64(gamma)))
    return st, ts


def model_update_threads(node_count, d, edges, slice_off, w, om, gamma):
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    so = np.ascontiguousarray(slice_off, np.uint64)
    secs = f64()
    _chk(lib().ref_model_update_threads(u32(node_count), i32(d), _p(e), _p(so), i32(len(so) - 1),
                                        _p(w), _p(om), f64(gamma), C.byref(secs)))
    return secs.value


def sync_shared(states, last_ts, shared, average):
    """pac_sim.cpp:162-203. states [W, N, d], last_ts [W, N]."""
    st = np.ascontiguousarray(states, np.float64).copy()
    ts = np.ascontiguousarray(last_ts, np.float64).copy()
    W, N, d = st.shape
    sh = np.ascontiguousarray(shared, np.uint32)
    _chk(lib().ref_sync_shared(i32(W), u32(N), i32(d), _p(st), _p(ts), _p(sh), u64(len(sh)),
                               i32(int(average))))
    return st, ts


def digest(state, last_ts):
    st = np.ascontiguousarray(state, np.float64)
    ts = np.ascontiguousarray(last_ts, np.float64)
    buf = C.create_string_buffer(17)
    _chk(lib().ref_digest(u32(st.shape[0]), i32(st.shape[1]), _p(st), _p(ts), buf))
    return buf.value.decode()


def run_epoch(sub_edges, node_count, d, states, last_ts, w, om, gamma, shared, average, batch,
              log=False):
    """pac_sim.cpp:205-264."""
    W = len(sub_edges)
    off = np.zeros(W + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in sub_edges])
    eds = np.concatenate([np.ascontiguousarray(x, EDGE_DTYPE) for x in sub_edges] + [np.zeros(1, EDGE_DTYPE)])
    st = np.ascontiguousarray(states, np.float64).copy()
    ts = np.ascontiguousarray(last_ts, np.float64).copy()
    sh = np.ascontiguousarray(shared, np.uint32) if len(shared) else np.zeros(1, np.uint32)
    batches = np.zeros(W, np.uint64)
    loops = np.zeros(W, np.uint64)
    sev = u64()
    dg = C.create_string_buffer(17 * W)
    cap = (1 << 16) if log else 0
    steps = np.zeros(4 * max(1, cap), np.uint64)
    nlog = u64()
    sw = np.zeros(max(1, cap), np.int32)
    sd = C.create_string_buffer(17 * max(1, cap))
    nsnap = u64()
    _chk(lib().ref_run_epoch(i32(W), u32(node_count), i32(d), _p(off), _p(eds), _p(st), _p(ts),
                             _p(w), _p(om), f64(gamma), _p(sh), u64(len(shared)), i32(int(average)),
                             u64(batch), _p(batches), _p(loops), C.byref(sev), dg, u64(cap),
                             _p(steps), C.byref(nlog), _p(sw), sd, C.byref(nsnap)))
    digests = [dg.raw[17 * i:17 * i + 16].decode() for i in range(W)]
    out = dict(states=st, last_ts=ts, batches=batches.tolist(), loops=loops.tolist(),
               sync_events=sev.value, digests=digests)
    if log:
        out["steps"] = [tuple(int(x) for x in steps[4 * k:4 * k + 4]) for k in range(nlog.value)]
        out["snapshots"] = [(int(sw[k]), sd.raw[17 * k:17 * k + 16].decode()) for k in range(nsnap.value)]
    return out


def simulate(edges, node_count, t_max, num_parts, node_parts, shared, num_workers=1,
             num_small_parts=1, shuffle=False, average=False, batch=1, epochs=1, d=8, model_seed=0,
             shuffle_seed=0):
    """pac_sim.cpp:266-338."""
    e = np.ascontiguousarray(edges, EDGE_DTYPE)
    off = np.zeros(len(node_parts) + 1, np.uint64)
    off[1:] = np.cumsum([len(v) for v in node_parts])
    flat = np.array([p for v in node_parts for p in v] or [0], np.int32)
    sh = np.ascontiguousarray(shared, np.uint32) if len(shared) else np.zeros(1, np.uint32)
    E, W = max(1, epochs), max(1, num_workers)
    rec = np.zeros(E, np.uint64)
    sev = np.zeros(E, np.uint64)
    loops = np.zeros(E * W, np.uint64)
    dg = C.create_string_buffer(17 * E * W)
    tot = u64()
    _chk(lib().ref_simulate(_p(e), u64(len(e)), u32(node_count), f64(t_max), i32(num_parts),
                            _p(off), _p(flat), _p(sh), u64(len(shared)), i32(num_workers),
                            i32(num_small_parts), i32(int(shuffle)), i32(int(average)), u64(batch),
                            i32(epochs), i32(d), u64(model_seed), u64(shuffle_seed), _p(rec),
                            _p(sev), _p(loops), dg, C.byref(tot)))
    eps = []
    for ep in range(epochs):
        eps.append(dict(recovered=int(rec[ep]), sync_events=int(sev[ep]),
                        loops=loops[ep * W:(ep + 1) * W].tolist(),
                        digests=[dg.raw[17 * (ep * W + w):17 * (ep * W + w) + 16].decode()
                                 for w in range(W)]))
    return dict(epochs=eps, sync_events=tot.value)


def load_edges(path, assume_sorted=False):
    """graph_io.cpp:106-140 -> (edges EDGE_DTYPE array, node_count, t_max)."""
    L = lib()
    out = C.c_void_p()
    n, nc, tm = u64(), u32(), f64()
    _chk(L.ref_load_edges(str(path).encode(), int(assume_sorted), C.byref(out), C.byref(n),
                          C.byref(nc), C.byref(tm)))
    arr = np.empty(n.value, dtype=EDGE_DTYPE)
    if n.value:
        C.memmove(arr.ctypes.data, out.value, n.value * EDGE_DTYPE.itemsize)
    L.ref_free(out)
    return arr, nc.value, tm.value


_WRITE_SCRIPT = """
import ctypes as C, sys
L = C.CDLL(sys.argv[1])
raw = open(sys.argv[2], 'rb').read()
buf = C.create_string_buffer(raw, max(1, len(raw)))
L.ref_write_edges.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64]
L.ref_last_error_detail.restype = C.c_char_p
st = L.ref_write_edges(sys.argv[3].encode(), C.cast(buf, C.c_void_p), len(raw) // 16)
if st:
    sys.exit(f"ref_write_edges: {st} {L.ref_last_error_detail().decode()}")
"""


def write_edges(edges, path):
    """graph_io.cpp:142-154, run in a fresh interpreter: the reference's
    ostream number formatting (a libstdc++ linked into _ref) crashes once
    numpy's own C++ runtime is loaded in the same process."""
    import subprocess
    import sys
    import tempfile
    e = np.ascontiguousarray(edges, dtype=EDGE_DTYPE)
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        f.write(e.tobytes())
        f.flush()
        subprocess.run([sys.executable, "-c", _WRITE_SCRIPT, REF_SO, f.name, str(path)], check=True)
