"""Kernel timeline of a few graph-replayed GDELT steps via torch.profiler (CUPTI):
per-stream busy time, critical-path gaps and the kernels of one step in time order."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
import paper_2308_14129_b200 as sp

wl = bench.build_workload(os.environ.get("CFG", "gdelt"), 1, 0, lambda m: print(m, file=sys.stderr))
N, E, F, B = bench.CONFIGS[os.environ.get("CFG", "gdelt")]
cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=F, n_neighbors=10, n_heads=2, batch_size=B, lr=1e-4,
                   gemm_mode=1)
tr = sp.TGNTrainer(cfg, wl["subs"], workers=[0], shared=wl["shared"], node_count=N)
tr.begin_epoch(0)
tr.seek(tr.epoch_steps() // 2)
tr.run_steps(5)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.run_steps(3)
    torch.cuda.synchronize()
out = os.environ.get("OUT", "gpurun_out/trace.json")
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
print("kernels traced", len(ev))
t0 = ev[0]["ts"]
# one step = the span between consecutive k_adam ends
adam = [e for e in ev if "k_adam" in e["name"]]
if len(adam) >= 2:
    a, b = adam[-2]["ts"] + adam[-2]["dur"], adam[-1]["ts"] + adam[-1]["dur"]
    step = [e for e in ev if e["ts"] >= a and e["ts"] + e["dur"] <= b + 1]
    print(f"step span {b - a:.1f} us, kernels {len(step)}")
    streams = {}
    for e in step:
        streams.setdefault(e["args"].get("stream"), []).append(e)
    for sid, es in streams.items():
        busy = sum(x["dur"] for x in es)
        print(f"stream {sid}: {len(es)} kernels, busy {busy:.1f} us")
    # union of busy time across streams
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in step)
    tot, cs, ce = 0.0, None, None
    for s_, e_ in iv:
        if cs is None or s_ > ce:
            if cs is not None: tot += ce - cs
            cs, ce = s_, e_
        else:
            ce = max(ce, e_)
    tot += ce - cs
    print(f"GPU busy (any stream) {tot:.1f} us of {b - a:.1f}")
    for e in step:
        print(f"{e['ts'] - a:8.1f} {e['dur']:7.1f}  s{e['args'].get('stream')}  {e['name'][:80]}")
