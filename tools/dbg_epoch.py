"""Debug: test_epoch_end_restore_and_sync scenario step by step vs the oracle."""
import os, sys
root = os.environ.get("PKG_ROOT", os.getcwd())
sys.path.insert(0, os.getcwd()); sys.path.insert(0, root)
import numpy as np
import paper_2308_14129_b200 as sp
print("package", sp.__file__)
from tests.tgn_cases import oracle_for, partitioned, rel_err
_, _, pa, subs = partitioned(parts=2, nodes=200, edges=2500)
cfg = sp.TGNConfig(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=50, lr=1e-3)
tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
o = oracle_for(cfg, subs, pa.shared)
tr.begin_epoch(0); o.begin_epoch(0)
print("epoch steps", tr.epoch_steps(), "batches", [o.batches(w) for w in range(2)])
for k in range(tr.epoch_steps()):
    gl = tr.step(); ol = o.step()
    errs = [rel_err(tr.memory(w)[0], o.mem[w].numpy()) for w in range(2)]
    lue = [np.array_equal(tr.memory(w)[1], o.lu[w]) for w in range(2)]
    print(f"step {k}: loss {np.abs(np.array(gl) - np.array(ol)).max():.2e} params {rel_err(tr.params(), o.flat.numpy()):.2e} "
          f"grads {rel_err(tr.grads(), o.grad.numpy()):.2e} mem {errs[0]:.2e} {errs[1]:.2e} lu {lue}", flush=True)
tr.end_epoch(); o.end_epoch()
print("after end_epoch mem", [rel_err(tr.memory(w)[0], o.mem[w].numpy()) for w in range(2)])
