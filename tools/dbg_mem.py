"""Debug: which memory rows diverge in TF32 mode at GDELT dims, B=2000."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2308_14129_b200 as sp
from tests.tgn_cases import oracle_for, rel_err
N, E, B = int(os.environ.get("NN", 16682)), int(os.environ.get("EE", 400000)), int(os.environ.get("BB", 2000))
F = int(os.environ.get("FF", 186))
s = sp.gen_powerlaw(N, E, 2.5, 1)
split = sp.chrono_split(s, 0.70, 0.15)
tr_ = split.train
c = sp.compute_centrality(tr_, 0.5)
pa = sp.partition_stream(tr_, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
subs = sp.induce_subgraphs(tr_, pa.node_parts, 1)
trs = {}
for mode in (1, 0):
    cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=F, n_neighbors=10, n_heads=2, batch_size=B, lr=1e-4, gemm_mode=mode)
    t = sp.TGNTrainer(cfg, subs, shared=pa.shared); t.set_graph(False)
    t.begin_epoch(0); t.seek(t.epoch_steps() // 2); trs[mode] = t
o = oracle_for(cfg, subs, pa.shared); o.begin_epoch(0); o.seek(trs[1].epoch_steps() // 2)
prev = None
for k in range(3):
    for t in trs.values(): t.step()
    o.step()
    m1, lu1 = trs[1].memory(0); m0, lu0 = trs[0].memory(0); om = o.mem[0].numpy()
    re = lambda a, b: np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-30)
    r10, r0o = re(m1, m0), re(m0, om)
    bad = np.where(r10 > 0.05)[0]
    print(f"step {k}: TF32 vs FP32-GPU rows>5%: {len(bad)}; FP32-GPU vs oracle rows>5%: {int((r0o > 0.05).sum())}; "
          f"mem rel tf32/fp32 {rel_err(m1, m0):.2e} fp32/oracle {rel_err(m0, om):.2e}")
    if len(bad):
        upd = np.where(lu1 != (prev[1] if prev is not None else 0))[0]
        print("  bad rows:", bad[:12], "updated this step:", np.isin(bad[:12], upd))
        for r in bad[:4]:
            print(f"  row {r}: |tf32| {np.linalg.norm(m1[r]):.3f} |fp32| {np.linalg.norm(m0[r]):.3f} |oracle| {np.linalg.norm(om[r]):.3f} "
                  f"lu {lu1[r]} err {r10[r]:.3f}; tf32[:4] {m1[r][:4]} fp32[:4] {m0[r][:4]}")
            if prev is not None:
                print(f"     prev tf32 row [:4] {prev[0][r][:4]}")
    prev = (m1.copy(), lu1.copy())
