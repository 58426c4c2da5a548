"""Progress probe for concurrent local workers (lanes): prints each phase."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(int(os.environ.get("PROBE_TIMEOUT", "120")), exit=True)
import numpy as np  # noqa: E402
import paper_2308_14129_b200 as sp  # noqa: E402
from tests.tgn_cases import partitioned  # noqa: E402

graph = os.environ.get("PROBE_GRAPH", "1") == "1"
_, _, pa, subs = partitioned(parts=2)
cfg = sp.TGNConfig(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=64, lr=1e-3,
                   concurrent=1)
t0 = time.time()
tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
tr.set_graph(graph)
print("ctor ok", time.time() - t0, flush=True)
tr.begin_epoch(0)
print("begin ok", tr.epoch_steps(), flush=True)
for k in range(tr.epoch_steps()):
    l = tr.step()
    print("step", k, l, flush=True)
tr.end_epoch()
print("end_epoch ok", flush=True)
print("params", float(np.abs(tr.params()).sum()), flush=True)
