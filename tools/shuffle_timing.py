"""Shuffle-combine re-induction cost per epoch at a BASELINE shape:
the host path (spd_shuffle_combine + spd_induce_groups + spd_tgn_rebind: an
O(P·E) pass over the training stream and a re-upload) against the device path
(spd_tgn_shuffle_epoch on the stream kept in HBM). Prints one JSON line.

    python tools/shuffle_timing.py [config] [workers]   (default: gdelt 2)"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2308_14129_b200 as sp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gdelt"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
N, E, F, B = bench.CONFIGS[name]
log = lambda m: print(m, file=sys.stderr, flush=True)
wl = bench.build_workload(name, 2 * W, 0, log)  # 2W small SEP parts
split = wl["split"]
small = [g.nodes for g in wl["subs"]]
cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=F, n_neighbors=10, n_heads=2, batch_size=B,
                   lr=1e-4, gemm_mode=1)
out = {"config": name, "workers": W, "small_parts": 2 * W, "train_edges": len(split.train)}
for epoch in range(2):
    t0 = time.perf_counter()
    groups = sp.shuffle_combine(small, W, 11 + epoch)
    subs, rec_host = sp.induce_groups(split.train, groups, small)
    t_host_induce = time.perf_counter() - t0
    if epoch == 0:
        t0 = time.perf_counter()
        tr = sp.TGNTrainer(cfg, subs, shared=wl["shared"], node_count=N)
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        tr.attach_stream(split.train, small)
        t_attach = time.perf_counter() - t0
        out.update(trainer_build_s=t_build, attach_stream_s=t_attach)
    else:
        t0 = time.perf_counter()
        tr.rebind(subs)
        out["host_rebind_s"] = time.perf_counter() - t0
        out["host_induce_s"] = t_host_induce
    t0 = time.perf_counter()
    rec_dev = tr.shuffle_epoch(11 + epoch)
    t_dev = time.perf_counter() - t0
    assert rec_dev == rec_host, (rec_dev, rec_host)
    out[f"device_shuffle_epoch_s_{epoch}"] = t_dev
    out[f"recovered_{epoch}"] = rec_dev
    log(f"epoch {epoch}: host induce {t_host_induce:.2f}s, device shuffle_epoch {t_dev:.2f}s, "
        f"recovered {rec_dev}")
out["host_epoch_s"] = out["host_induce_s"] + out["host_rebind_s"]
print(json.dumps(out))
