"""Debug: recompute the TF32 GRU gate GEMMs of one GDELT-dims step on the host."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2308_14129_b200 as sp
from oracle.tgn_oracle import param_layout, TGNConfig as OC
s = sp.gen_powerlaw(16682, 400000, 2.5, 1)
split = sp.chrono_split(s, 0.70, 0.15)
tr_ = split.train
c = sp.compute_centrality(tr_, 0.5)
pa = sp.partition_stream(tr_, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
subs = sp.induce_subgraphs(tr_, pa.node_parts, 1)
def tf32(a):
    b = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x1000) & 0xFFFFE000).astype(np.uint32)  # round half away (approx of cvt.rna)
    return b.view(np.float32)
for mode in (1, 0):
    cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=186, n_neighbors=10, n_heads=2, batch_size=2000, lr=1e-4, gemm_mode=mode)
    t = sp.TGNTrainer(cfg, subs, shared=pa.shared); t.set_graph(False)
    t.begin_epoch(0); mid = t.epoch_steps() // 2; t.seek(mid)
    ev = t.worker_events(0)
    for k in range(3):
        P = t.params()
        lo = t.next_batch(0)[0]
        t.step()
        if k == 0: continue
        prev = ev[lo - 2000: lo]  # previous batch: its messages are this step's pending set
        nU = len(np.unique(np.r_[prev["src"], prev["dst"]]))
        lay, _ = param_layout(OC(d_mem=100, d_time=100, d_edge=186))
        off, N, K, ld = lay["gru_ih"]; Wih = P[off:off + N * ld].reshape(N, ld)
        off, N2, K2, ld2 = lay["gru_hh"]; Whh = P[off:off + N2 * ld2].reshape(N2, ld2)
        x = t.debug_scratch("x_gru").reshape(4000, -1)[:nU]
        h = t.debug_scratch("h_gru").reshape(4000, -1)[:nU]
        Gi = t.debug_scratch("Gi").reshape(4000, -1)[:nU, :300]
        Gh = t.debug_scratch("Gh").reshape(4000, -1)[:nU, :300]
        rw = (lambda a: tf32(a)) if mode == 1 else (lambda a: a)
        gi_ref = x[:, :K + 1].astype(np.float64) @ rw(Wih[:, :K + 1]).astype(np.float64).T
        gh_ref = h[:, :K2 + 1].astype(np.float64) @ rw(Whh[:, :K2 + 1]).astype(np.float64).T
        ei = np.abs(Gi - gi_ref).max(1) / np.maximum(np.abs(gi_ref).max(1), 1e-30)
        eh = np.abs(Gh - gh_ref).max(1) / np.maximum(np.abs(gh_ref).max(1), 1e-30)
        print(f"mode {mode} step {k}: nU {nU}, x ld {x.shape[1]}, Gi rel err max {ei.max():.2e} (rows>1e-2: {(ei>1e-2).sum()}), "
              f"Gh rel err max {eh.max():.2e} (rows>1e-2: {(eh>1e-2).sum()}); x cols nonzero {np.count_nonzero(np.abs(x).sum(0))}", flush=True)
        bad = np.where(ei > 1e-2)[0][:5]
        for r in bad:
            dcol = np.abs(Gi[r] - gi_ref[r])
            print(f"   row {r}: worst cols {np.argsort(-dcol)[:6]} gi {Gi[r][:3]} ref {gi_ref[r][:3]}; x nz cols {np.flatnonzero(x[r])[:5]}...")
    t.close()
