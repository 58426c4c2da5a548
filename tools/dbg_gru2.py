"""Debug: TF32 vs FP32 trainers in lockstep; where do the GRU inputs/outputs differ?"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2308_14129_b200 as sp
s = sp.gen_powerlaw(16682, 400000, 2.5, 1)
split = sp.chrono_split(s, 0.70, 0.15)
tr_ = split.train
c = sp.compute_centrality(tr_, 0.5)
pa = sp.partition_stream(tr_, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
subs = sp.induce_subgraphs(tr_, pa.node_parts, 1)
T = {}
for mode in (1, 0):
    cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=186, n_neighbors=10, n_heads=2, batch_size=2000, lr=1e-4, gemm_mode=mode)
    t = sp.TGNTrainer(cfg, subs, shared=pa.shared); t.set_graph(False)
    t.begin_epoch(0); t.seek(t.epoch_steps() // 2); T[mode] = t
ev = T[1].worker_events(0)
sig = lambda v: 1 / (1 + np.exp(-v))
for k in range(3):
    lo = T[1].next_batch(0)[0]
    mem_before = {m: T[m].memory(0)[0] for m in T}
    for m in T: T[m].step()
    if k == 0: continue
    prev = ev[lo - 2000: lo]
    U = np.unique(np.r_[prev["src"], prev["dst"]]); nU = len(U)
    d = {}
    for m in T:
        d[m] = {n: T[m].debug_scratch(n) for n in ("x_gru", "h_gru", "Gi", "Gh", "mem_new")}
        d[m]["mem"] = T[m].memory(0)[0]
    x1, x0 = d[1]["x_gru"].reshape(4000, -1)[:nU], d[0]["x_gru"].reshape(4000, -1)[:nU]
    for name, a, b in (("mem_self", 0, 100), ("mem_other", 100, 200), ("feat", 200, 386), ("time", 386, 486), ("bias", 486, 487)):
        e = np.abs(x1[:, a:b] - x0[:, a:b]).max()
        print(f"step {k}: x {name} max abs diff tf32-fp32 {e:.3e}")
    for m in T:
        Gi = d[m]["Gi"].reshape(4000, -1)[:nU, :300]; Gh = d[m]["Gh"].reshape(4000, -1)[:nU, :300]
        h = mem_before[m]  # exact h of pending nodes; rows in pending order unknown -> use x mem_self (tf32-rounded in mode 1)
        hx = d[m]["x_gru"].reshape(4000, -1)[:nU, :100]
        r = sig(Gi[:, :100] + Gh[:, :100]); z = sig(Gi[:, 100:200] + Gh[:, 100:200])
        n = np.tanh(Gi[:, 200:] + r * Gh[:, 200:])
        mn = (1 - z) * n + z * hx
        got = d[m]["mem_new"].reshape(4000, -1)[:nU]
        print(f"  mode {m}: cell recompute vs mem_new max abs {np.abs(mn - got).max():.3e}")
    mn1 = d[1]["mem_new"].reshape(4000, -1)[:nU]; mn0 = d[0]["mem_new"].reshape(4000, -1)[:nU]
    re = np.linalg.norm(mn1 - mn0, axis=1) / np.maximum(np.linalg.norm(mn0, axis=1), 1e-30)
    print(f"  mem_new tf32 vs fp32: rows>5% {int((re > .05).sum())} max {re.max():.3e}")
    m1, m0 = d[1]["mem"], d[0]["mem"]
    rr = np.linalg.norm(m1 - m0, axis=1) / np.maximum(np.linalg.norm(m0, axis=1), 1e-30)
    bad = np.where(rr > .05)[0]
    print(f"  persisted mem tf32 vs fp32: rows>5% {len(bad)}; bad rows in U: {np.isin(bad, U).mean() if len(bad) else 0}")
    if len(bad):
        b = bad[0]
        # find b's mem_new row in each trainer by matching
        for m in T:
            mn = d[m]["mem_new"].reshape(4000, -1)[:nU]
            j = np.argmin(np.linalg.norm(mn - d[m]["mem"][b], axis=1))
            print(f"   mode {m}: mem row {b} equals mem_new row {j} (dist {np.linalg.norm(mn[j] - d[m]['mem'][b]):.2e}); "
                  f"sorted-U position of {b}: {np.searchsorted(U, b)}")
