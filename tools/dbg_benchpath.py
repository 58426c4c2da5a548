"""Debug: bench-path scenario (GDELT dims, B=2000, seek, graph replay) vs the
oracle, per-step errors without asserting; PKG_ROOT selects the build."""
import os, sys
root = os.environ.get("PKG_ROOT", os.getcwd())
sys.path.insert(0, os.getcwd())
sys.path.insert(0, root)
import numpy as np
import paper_2308_14129_b200 as sp
print("package", sp.__file__)
from tests.tgn_cases import oracle_for, rel_err
s = sp.gen_powerlaw(16682, 400_000, 2.5, 1)
split = sp.chrono_split(s, 0.70, 0.15)
tr_ = split.train
c = sp.compute_centrality(tr_, 0.5)
pa = sp.partition_stream(tr_, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
subs = sp.induce_subgraphs(tr_, pa.node_parts, 1)
for mode in [int(x) for x in os.environ.get("MODES", "1,0").split(",")]:
    for graph in (True, False):
        cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=186, n_neighbors=10, n_heads=2,
                           batch_size=2000, lr=1e-4, gemm_mode=mode)
        tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
        tr.set_graph(graph)
        o = oracle_for(cfg, subs, pa.shared)
        tr.begin_epoch(0); o.begin_epoch(0)
        mid = tr.epoch_steps() // 2
        tr.seek(mid); o.seek(mid)
        for k in range(5):
            gl = float(tr.step()[0]); ol = float(o.step()[0])
            m, lu = tr.memory(0)
            om = o.mem[0].numpy()
            rowerr = np.linalg.norm(m - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-30)
            bad = np.where(rowerr > 0.05)[0]
            print(f"mode {mode} graph {graph} step {k}: loss {abs(gl-ol)/abs(ol):.2e} params {rel_err(tr.params(), o.flat.numpy()):.2e} "
                  f"mem {rel_err(m, om):.2e} lu_eq {np.array_equal(lu, o.lu[0])} bad_rows {len(bad)} {bad[:8]} "
                  f"gpu_zero_rows {int((np.abs(m[bad]).sum(1) == 0).sum())} ora_zero_rows {int((np.abs(om[bad]).sum(1) == 0).sum())}", flush=True)
        tr.close()
