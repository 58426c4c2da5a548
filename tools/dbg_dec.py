import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2308_14129_b200 as sp
from tests.test_eval_gpu import build, scores
pa, subs, ev, r = build(400, 6000, 2)
cfg = sp.TGNConfig(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=64, lr=1e-3)
tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
losses = []
tr.begin_epoch(0)
for k in range(tr.epoch_steps()):
    losses.append(tr.step())
tr.end_epoch()
p = tr.params()
g = scores(tr, ev, False)
np.savez(os.environ["OUT"], p=p, l=np.array(losses), *g)
print(os.environ["OUT"], np.array(losses)[:3].ravel(), np.array(losses)[-3:].ravel())
