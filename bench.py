#!/usr/bin/env python
"""Benchmark: SPEED's SEP-sharded TGN training step on B200 (one partition per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gdelt] [--impl ours|reference]

For N>1 launch under torchrun (one rank per GPU, 127.0.0.1 rendezvous); the
gradient all-reduce runs over NCCL inside the library, gloo only carries the
NCCL unique id and the max-over-ranks timing.

A "step" is one lockstep global step of PAC training (Alg. 2): every
rank trains one batch of its SEP partition (forward, backward, gradient
all-reduce, Adam, memory persist). value = training edges processed by all
ranks / max-over-ranks device time of the K timed steps. Inputs are
resident in HBM; the per-step working set (gathered neighbour feature rows of
a 50-100 GB feature table plus ~300 MB of activations) exceeds the 126 MB L2.

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: speedpart's model_update surrogate compiled from
/root/reference/proj/src) on the same workload, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (nodes, edges, d_edge, batch) — BASELINE.json configs; dims d_mem=d_time=100, k=10, 2 heads
CONFIGS = {
    "wiki": (9227, 157474, 172, 200),
    "reddit": (10984, 672447, 172, 200),
    "lastfm": (1980, 1293103, 0, 200),
    "ml25m": (221588, 25000095, 1, 2000),
    "gdelt": (16682, 191290882, 186, 2000),
    "tiny": (2000, 200000, 186, 2000),
}
BYTES_PER_EDGE = {"gdelt": 74316}  # SURVEY §8(d) algorithmic bytes per positive event


def bytes_per_edge(D, T, F, K):
    """SURVEY §8(d) formula (fwd + bwd re-gather), per positive training event."""
    fwd = 3 * (4 * D + 8) + 2 * (8 * D + 4 * F + 8) + 2 * (4 * D + 8) + 48 * K + 12 * K * D + 12 * K * F + 52
    return fwd + 12 * K * (D + F)


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes per launch) of `kernel`
    from the newest committed ncu --set full raw export under profiles/."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_k_attn_abs_raw.csv")))
    if not files:
        return None, None
    rows = list(csv.reader(open(files[-1])))
    h, units = rows[0], rows[1]
    row = next((r for r in rows[2:] if kernel + "<" in r[h.index("Kernel Name")]), None)
    if row is None:
        return None, None
    total = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
        total += float(row[i].replace(",", "")) * scale
    return total, os.path.relpath(files[-1], ROOT)


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    return rank, world, local, pg


def allreduce_max(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample so
            # the samples taken from here on fall inside the timed region
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        self.start_idx = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        during = self.lines[getattr(self, "start_idx", 0):] or self.lines
        for ln in during:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


def build_workload(name, P, rank, log, hub_k=0.05):
    import paper_2308_14129_b200 as sp
    N, E, F, B = CONFIGS[name]
    t0 = time.time()
    s = sp.gen_powerlaw(N, E, 2.5, 1)
    log(f"gen_powerlaw {N}x{E}: {time.time() - t0:.1f}s")
    split = sp.chrono_split(s, 0.70, 0.15)
    del s
    tr = split.train
    t0 = time.time()
    c = sp.compute_centrality(tr, 0.5)
    pa = sp.partition_stream(tr, sp.PartitionerConfig(P, 1.0, 1.0, sp.select_hubs(c, hub_k), c))
    log(f"SEP P={P}: {time.time() - t0:.1f}s, shared={len(pa.shared)}, discards={pa.discard_count}")
    t0 = time.time()
    subs = sp.induce_subgraphs(tr, pa.node_parts, P)
    log(f"induce: {time.time() - t0:.1f}s, edges/part={[len(g.edges) for g in subs]}")
    return dict(N=N, E=E, F=F, B=B, train_edges=len(tr), subs=subs, shared=pa.shared, split=split)


def build_workload_ref(name, P, log):
    """The same workload built by the REFERENCE library itself (oracle/_ref:
    gen_powerlaw graph_io.cpp:175-250, chrono_split :156-173, centrality +
    hubs centrality.cpp:27-88, partition_stream partitioner.cpp:152,
    induce_subgraphs pac_sim.cpp:106-132) — bit-identical to the product's
    (tests/test_host_parity.py), and the product library is never loaded."""
    from oracle import ref as R
    N, E, F, B = CONFIGS[name]
    t0 = time.time()
    edges, nc, _ = R.gen_powerlaw(N, E, 2.5, 1)
    log(f"reference gen_powerlaw {N}x{E}: {time.time() - t0:.1f}s")
    n_tr, _, _ = R.chrono_split_sizes(len(edges), 0.70, 0.15)
    tr = np.ascontiguousarray(edges[:n_tr])
    del edges
    t_max = float(tr["ts"].max()) if n_tr else 0.0
    t0 = time.time()
    cent, _ = R.compute_centrality(tr, nc, t_max, 0.5)
    hubs = R.select_hubs(cent, 0.05)
    t1 = time.time()
    pa = R.partition(tr, nc, t_max, P, cent, hubs, 0.05)
    t_part = time.time() - t1
    log(f"reference centrality+hubs {t1 - t0:.1f}s, partition_stream P={P}: {t_part:.1f}s "
        f"({n_tr / max(t_part, 1e-9) / 1e6:.1f} M edges/s), shared={len(pa['shared'])}")
    subs = R.induce_subgraphs(tr, nc, pa["node_parts"], P)
    return dict(N=N, E=E, F=F, B=B, train_edges=n_tr, subs=subs, shared=pa["shared"],
                partition_s=t_part, hubs_s=t1 - t0)


def cpu_partition_baseline(wl):
    """the reference partition_stream over the full train
    stream, single thread as written."""
    return {"what": "reference partition_stream (partitioner.cpp:152) over the full train stream",
            "value": wl["train_edges"] / wl["partition_s"], "unit": "edges/s", "cores": 1,
            "kind": "reference", "seconds": wl["partition_s"],
            "sample": f"{wl['train_edges']} train edges, P={len(wl['subs'])}, k=0.05"}


def cpu_tgn_oracle_rate(nodes, edges, eids, cfg, log, window=200_000, steps=3):
    """the CPU TGN oracle (oracle/tgn_oracle.py, torch fp32 on
    all host threads) — the same model as the GPU step — on a bounded window
    of the partition stream: history from the window's first half, `steps`
    batches timed from its middle (memory zero there, as the trainer's seek)."""
    import torch
    from oracle import tgn_oracle as T
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    E = len(edges)
    lo = max(0, E // 2 - window // 2)
    hi = min(E, lo + window)
    oc = T.TGNConfig(d_mem=cfg["D"], d_time=cfg["T"], d_edge=cfg["F"], n_neighbors=cfg["K"],
                     n_heads=cfg["H"], batch_size=cfg["B"], lr=1e-4)
    wd = T.WorkerData(nodes, edges[lo:hi], eids[lo:hi], oc.d_edge, oc.seed_feat)
    o = T.TGNOracle(oc, [wd])
    o.begin_epoch(0)
    o.seek((hi - lo) // 2 // oc.batch_size)
    o.step()  # warm-up (allocator, thread pool)
    t0 = time.perf_counter()
    for _ in range(steps):
        o.step()
    secs = time.perf_counter() - t0
    rate = steps * oc.batch_size / secs
    log(f"CPU TGN oracle: {steps} steps x B={oc.batch_size} in {secs:.1f}s on {threads} threads")
    return {"what": "CPU TGN oracle step (oracle/tgn_oracle.py: same model, torch fp32 + autograd)",
            "value": rate, "unit": "edges/s", "cores": threads, "kind": "port",
            "sample": f"{steps} steps of B={oc.batch_size} from the middle of a {hi - lo}-event "
                      f"window of partition 0"}


def cpu_reference_rate(sub_edges, node_count_local, d, seconds, log, threads=None):
    """The reference's own model_update (oracle/_ref) on host cores: T threads,
    each its own MemoryStore over a disjoint slice of the partition stream."""
    from oracle import ref as R
    threads = threads or os.cpu_count() or 1
    w, om, g = R.model_seeded(d, 0)
    # calibrate: one thread, 400 edges
    probe = np.ascontiguousarray(sub_edges[:400])
    secs = R.model_update_threads(node_count_local, d, probe, [0, len(probe)], w, om, g)
    rate1 = len(probe) / max(secs, 1e-9)
    per = int(min(len(sub_edges) // threads, max(200, rate1 * seconds)))
    off = np.arange(threads + 1, dtype=np.uint64) * per
    sample = np.ascontiguousarray(sub_edges[: per * threads])
    secs = R.model_update_threads(node_count_local, d, sample, off, w, om, g)
    log(f"reference CPU: {threads} threads x {per} edges in {secs:.1f}s")
    return per * threads / secs, threads, per


def localize(nodes, edges):
    """Partition events in local ids (the reference MemoryStore is dense over ids)."""
    from oracle.ref import EDGE_DTYPE
    loc = np.searchsorted(nodes, edges["src"]), np.searchsorted(nodes, edges["dst"])
    e = np.empty(len(edges), EDGE_DTYPE)
    e["src"], e["dst"], e["ts"] = loc[0], loc[1], edges["ts"]
    return e


def loaded_native_libs():
    """Shared objects of this repo mapped into the process (evidence of which
    implementation ran)."""
    try:
        maps = open("/proc/self/maps").read().split("\n")
    except OSError:
        return None
    libs = sorted({ln.split()[-1] for ln in maps if ln.endswith(".so") and ROOT in ln})
    return [os.path.relpath(x, ROOT) for x in libs]


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="gdelt", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--fp32-steps", type=int, default=100,
                    help="also time this many steps with gemm_mode 0 (FP32 FFMA) for comparison")
    ap.add_argument("--parts", type=int, default=0,
                    help="SEP partitions (default: one per GPU); more than --gpus trains several "
                         "partitions per GPU as local workers of one trainer")
    ap.add_argument("--hub-k", type=float, default=0.05, help="SEP shared-hub fraction k")
    ap.add_argument("--concurrent", action="store_true",
                    help="with --parts > --gpus: a GPU's partitions train concurrently (one "
                         "stream set and parameter replica each, in-process peer all-reduce)")
    ap.add_argument("--backbone", default="tgn", choices=["tgn", "jodie", "dyrep"],
                    help="memory-based TIG model: TGN (GRU + temporal attention), JODIE "
                         "(RNN + time projection) or DyRep (RNN + attention-embedding "
                         "messages), PAPER.md:373")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1 gradient all-reduce: peer = fused into Adam over CUDA-IPC-mapped "
                         "peer HBM (NVLink); nccl = ncclAllReduce then Adam")
    ap.add_argument("--gemm-mode", type=int, default=1,
                    help="0 = FP32 FFMA everywhere; 1 = tcgen05 TF32 for the GRU and attention "
                         "projection GEMMs (merge/decoder stay FP32 FFMA)")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    rank, world, local, pg = dist_init()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; on a box with fewer GPUs than ranks (a functional check
    # of the N>1 path, not a measurement) ranks share devices round-robin
    try:
        import torch
        ndev = max(1, torch.cuda.device_count())
    except Exception:
        ndev = 1
    local = local % ndev
    if world > 1 and args.impl == "ours" and args.transport == "peer" and ndev > 1:
        # the peer-memory transport maps every rank's HBM: needs P2P between the GPUs
        import torch
        others = {r % ndev for r in range(world)} - {local}
        if not all(torch.cuda.can_device_access_peer(local, o) for o in others):
            print(f"[bench] rank {rank}: no P2P access between GPUs, using NCCL", file=sys.stderr)
            args.transport = "nccl"
        flags = [None] * world  # every rank must agree on the transport
        pg.all_gather_object(flags, args.transport)
        if "nccl" in flags:
            args.transport = "nccl"
    verbose = rank == 0

    def log(msg):
        if verbose:
            print(f"[bench] {msg}", file=sys.stderr, flush=True)

    metric = "training edges/sec (TGN, SEP partitions = GPUs, processed events)"
    N, E, F, B = CONFIGS[args.config]
    P = args.parts or world
    if P % world:
        raise SystemExit(f"--parts {P} is not a multiple of the {world} ranks")
    mine = list(range(rank * (P // world), (rank + 1) * (P // world)))  # this rank's partitions
    D = T = 100
    K, H = 10, 2
    model = {"tgn": "TGN", "jodie": "JODIE", "dyrep": "DyRep"}[args.backbone]
    cfg_desc = {"workload": f"{args.config}-shape synthetic TIG ({N} nodes, {E} edges, d_e={F}), "
                            f"{model} d_mem=d_time=100 k={K} heads={H}, B={B}, SEP P={P}"
                            + (f" k_hub={args.hub_k}" if args.hub_k != 0.05 else ""),
                "nodes": N, "edges": E, "d_edge": F, "batch": B, "partitions": P,
                "partitions_per_gpu": P // world, "hub_k": args.hub_k,
                "parallelism": f"sep{P}" + (f" ({P // world} per GPU{', concurrent' if args.concurrent else ''})"
                                            if P > world else ""),
                "transport": (args.transport if world > 1 else None),
                "timed_from": "mid-epoch (spd_tgn_seek to epoch_steps/2)",
                "l2": "inputs larger than L2 (50-100 GB feature "
                "table gathers + >126 MB activations per step)"}

    if args.impl == "reference":
        if rank != 0:
            return
        # everything on this arm runs the reference library (oracle/_ref);
        # the product library is never imported or loaded
        wl = build_workload_ref(args.config, P, log)
        nodes, edges = wl["subs"][0]
        rate, cores, per = cpu_reference_rate(localize(nodes, edges), len(nodes), D,
                                              args.cpu_seconds, log)
        sample = f"{cores} threads x {per} consecutive partition-0 events, d={D}, surrogate model_update"
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": rate, "unit": "edges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic", "config": cfg_desc,
            "cpu_baseline": {"value": rate, "unit": "edges/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": rate, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "partition_baseline": cpu_partition_baseline(wl),
            "native_libs": loaded_native_libs(),
            "note": "speedpart has no TGN: its training path is the fixed surrogate model_update "
                    "(pac_sim.cpp:68-104), timed here via oracle/_ref on all host threads; the "
                    "workload (generator, split, SEP, induction) is built by oracle/_ref as well"}))
        return

    import paper_2308_14129_b200 as sp
    wl = build_workload(args.config, P, rank, log, args.hub_k)
    subs_mine = [wl["subs"][w] for w in mine]
    sub_mine = subs_mine[0]
    cfg = sp.TGNConfig(d_mem=D, d_time=T, d_edge=F, n_neighbors=K, n_heads=H, batch_size=B, lr=1e-4,
                       gemm_mode=args.gemm_mode, backbone={"tgn": 0, "jodie": 1, "dyrep": 2}[args.backbone],
                       concurrent=1 if args.concurrent else 0)
    nccl_id = None
    if world > 1 and args.transport == "nccl":
        import torch
        nid = sp.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(nid), dtype=torch.uint8)
        pg.broadcast(t, 0)
        nccl_id = bytes(t.tolist())
    t0 = time.time()
    tr = sp.TGNTrainer(cfg, wl["subs"], workers=mine, shared=wl["shared"], node_count=N,
                       rank=rank, world=world, nccl_id=nccl_id, device=local)
    if world > 1 and args.transport == "peer":  # exchange the peer-memory blobs over gloo
        blobs = [None] * world
        pg.all_gather_object(blobs, tr.peer_export())
        tr.peer_connect(blobs)
    log(f"trainer ready: {time.time() - t0:.1f}s, params={tr.n_params}, epoch_steps={tr.epoch_steps()}")
    # per-GPU device memory held after the trainer is built (events, CSR,
    # feature rows, memory, parameters, scratch): SURVEY §8 ML25M footprint
    mem_gb = None
    try:
        import torch
        free_b, total_b = torch.cuda.mem_get_info(local)
        mem_gb = {"used_gb": round((total_b - free_b) / 1e9, 2), "total_gb": round(total_b / 1e9, 2)}
    except Exception:
        pass
    tr.begin_epoch(0)
    # steady state: time steps from the middle of the epoch (full recent-k
    # neighbour lists), not the epoch's sparse first batches
    seek = tr.epoch_steps() // 2
    tr.seek(seek)
    tr.run_steps(args.warmup)
    barrier(pg)
    launches0 = sp.kernel_launches()
    with ClockSampler(local) as clk:
        barrier(pg)
        ms = tr.run_steps(args.steps)
        barrier(pg)
    launches = sp.kernel_launches() - launches0
    ms_max = allreduce_max(pg, ms)
    per_step = sum(min(B, len(g.edges)) for g in subs_mine)  # every worker steps (loop-within-epoch)
    edges_mine = per_step * args.steps
    edges_all = allreduce_sum(pg, float(edges_mine))
    value = edges_all / (ms_max / 1e3)
    ms_per_step = ms_max / args.steps

    # per-phase breakdown (one profiled step, outside the timed region)
    # (CUDA events around each phase on the trainer stream, eager launches,
    # averaged over 10 steps following the timed region)
    tr.set_profile(True)
    acc, n_prof = {}, 10
    for _ in range(n_prof):
        tr.run_steps(1)
        for n, t in tr.kernel_times():
            acc[n] = acc.get(n, 0.0) + t / n_prof
    phases = list(acc.items())
    tr.set_profile(False)
    # epoch-end work (pac_sim.cpp:259-260): restore the loop-end snapshots and
    # sync SEP's shared hubs across every worker (host wall clock around the
    # synchronous call; outside the timed steps)
    barrier(pg)
    t0 = time.perf_counter()
    tr.end_epoch()
    epoch_end_ms = allreduce_max(pg, (time.perf_counter() - t0) * 1e3)

    # end-to-end through the public API from pinned host buffers: every local
    # worker's next e2e_steps batches (wrapping within its partition stream,
    # loop-within-epoch) staged in pinned memory, fed through step_host_async
    import torch
    e2e_steps = args.e2e_steps
    e2e_warm = 3  # untimed: first use of the pinned staging ring and copy stream
    pin = torch.cuda.is_available()
    nw = len(mine)
    ev_batches = [[None] * nw for _ in range(e2e_warm + e2e_steps)]
    ft_batches = [[None] * nw for _ in range(e2e_warm + e2e_steps)]
    for j, w in enumerate(mine):
        ev_local = tr.worker_events(w)
        pos, _, Fp = tr.next_batch(w)
        nE = len(ev_local)
        for k in range(e2e_warm + e2e_steps):
            hi = min(nE, pos + B)
            idx = np.arange(pos, hi)
            eb = torch.empty(len(idx) * 16, dtype=torch.uint8, pin_memory=pin).numpy().view(sp.EDGE_DTYPE)
            eb[:] = ev_local[idx]
            fb = torch.empty(len(idx) * max(Fp, 1), dtype=torch.int16, pin_memory=pin).numpy().view(np.uint16)
            fb = fb.reshape(len(idx), max(Fp, 1))
            if Fp:
                sp.edge_features_bf16(cfg.seed_feat, subs_mine[j].eids[idx], F, Fp, out=fb)
            ev_batches[k][j] = eb
            ft_batches[k][j] = fb
            pos = hi if hi < nE else 0
    # one pinned loss slot per worker and step: every step's losses are read back (D2H)
    loss_pin = torch.empty((e2e_warm + e2e_steps) * nw, dtype=torch.float32, pin_memory=pin).numpy()
    for k in range(e2e_warm):
        tr.step_host_async(ev_batches[k], ft_batches[k] if F else None, loss_pin[k * nw:(k + 1) * nw])
    tr.sync()
    h0, d0 = tr.io_bytes()
    barrier(pg)
    t0 = time.perf_counter()
    for k in range(e2e_warm, e2e_warm + e2e_steps):
        tr.step_host_async(ev_batches[k], ft_batches[k] if F else None, loss_pin[k * nw:(k + 1) * nw])
    tr.sync()
    t_e2e = time.perf_counter() - t0
    if not np.all(np.isfinite(loss_pin)):
        raise RuntimeError(f"non-finite e2e losses {loss_pin}")
    h1, d1 = tr.io_bytes()
    t_e2e = allreduce_max(pg, t_e2e)
    e2e_edges = allreduce_sum(pg, float(sum(len(b) for bs in ev_batches[e2e_warm:] for b in bs)))
    e2e = {"value": e2e_edges / t_e2e, "unit": "edges/s",
           "h2d_bytes_per_step": (h1 - h0) // e2e_steps, "d2h_bytes_per_step": (d1 - d0) // e2e_steps,
           "steps": e2e_steps, "api": "TGNTrainer.step_host_async + sync (spd_tgn_step_host_async)"}

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    # dominant kernel: the larger of the two attention kernels on the critical
    # path; algorithmic bytes per launch, full recent-k lists (mid-epoch). Per
    # neighbour occurrence both read its memory row (4D), cos row of phi (4T),
    # bf16 feature row (2F) and (node, event, dt, slot) = 20 B. Per root the
    # forward reads q'_h and writes xbar_h (2 x H x 4(DK+1)) and alpha (4HK);
    # the backward reads dxbar_h and writes dq'_h (2 x H x 4(DK+1)), reads
    # alpha and writes ds (2 x 4HK).
    DK = D + T + F
    R_ = 3 * B
    occ_bytes = R_ * K * (4 * D + 4 * T + 2 * F + 20)
    alg = {"k_attn_abs_fwd": occ_bytes + R_ * (2 * H * 4 * (DK + 1) + 4 * H * K),
           "k_attn_abs_bwd": occ_bytes + R_ * (2 * H * 4 * (DK + 1) + 2 * 4 * H * K)}
    kern = dict(phases)
    name = max(alg, key=lambda k: kern.get(k, 0.0))
    dom = (name, kern.get(name, 0.0))
    roof = {"bound": "hbm", "kernel": dom[0], "achieved": None, "peak": hbm_peak, "unit": "GB/s",
            "frac": None, "traffic": None,
            "algorithmic_bytes_per_launch": alg[name],
            "launch_ms": dom[1], "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}
    if dom[1] > 0:
        roof["achieved"] = alg[name] / (dom[1] / 1e3) / 1e9
        roof["frac"] = roof["achieved"] / hbm_peak
    roof["other_kernels_ms"] = {k: kern.get(k) for k in ("k_attn_abs_fwd", "k_attn_abs_bwd", "attn_bwd_x")}
    # measured DRAM traffic of the same kernel: the committed ncu --set full capture
    roof["traffic"], roof["traffic_source"] = ncu_traffic(name)
    bpe = bytes_per_edge(D, T, F, K)
    step_roof = {"bytes_per_edge": bpe, "achieved_gbs_per_gpu": value / world * bpe / 1e9,
                 "frac_of_hbm": value / world * bpe / 1e9 / hbm_peak,
                 "roofline_edges_per_s_per_gpu": hbm_peak * 1e9 / bpe}
    # tensor-core roofline of one projection GEMM: the attention's per-head
    # key projection Qp_h = Q_h [W_K,h | b_K,h] (one batched tcgen05 launch,
    # 2 R x dh x (DK+1) x H FLOP) over its CUDA-event time; TF32 peak taken as
    # half the measured dense BF16 rate (tcgen05 kind::tf32 issues at half the
    # kind::f16 rate)
    gemm = None
    if args.gemm_mode == 1 and kern.get("gemm_qp"):
        flop = 2.0 * R_ * (D + T) / H * (DK + 1) * H
        bf16 = peaks.get("bf16_tflops") or 1590.0
        ach = flop / (kern["gemm_qp"] / 1e3) / 1e12
        gemm = {"bound": "tensor", "kernel": "umma_gemm_kernel (Qp: attention key projection, TF32)",
                "achieved": ach, "peak": bf16 / 2, "unit": "TFLOP/s", "frac": ach / (bf16 / 2),
                "flop_per_launch": flop, "launch_ms": kern["gemm_qp"],
                "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2" if peaks else "fallback 1590 / 2",
                "tensor_pipe_pct_ncu": "profiles/r2/kernel_table_final.txt (sm__pipe_tensor_cycles_active)"}

    # the same workload in FP32 FFMA (gemm_mode 0): the evidence behind the
    # TF32 tensor-core choice for the GRU / attention projections
    fp32 = None
    if args.gemm_mode == 1 and args.fp32_steps > 0:
        tr.set_gemm_mode(0)
        tr.seek(seek)
        tr.run_steps(args.warmup)
        barrier(pg)
        ms0 = allreduce_max(pg, tr.run_steps(args.fp32_steps))
        e0 = allreduce_sum(pg, float(per_step * args.fp32_steps))
        fp32 = {"gemm_mode": 0, "value": e0 / (ms0 / 1e3), "unit": "edges/s",
                "ms_per_step": ms0 / args.fp32_steps, "steps": args.fp32_steps,
                "what": "same trainer and workload with every GEMM in FP32 FFMA"}
        tr.set_gemm_mode(1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        extra = []
        try:
            rate, cores, per = cpu_reference_rate(localize(sub_mine.nodes, sub_mine.edges),
                                                  len(sub_mine.nodes), D, args.cpu_seconds, log)
            cpu = {"value": rate, "unit": "edges/s", "cores": cores, "kind": "reference",
                   "sample": f"{cores} threads x {per} consecutive partition events, d={D}, "
                             "speedpart model_update (surrogate: the reference has no TGN)"}
        except Exception as ex:  # the reference .so must travel; report, do not fail the bench
            cpu = {"value": None, "unit": "edges/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
        try:  # reference partition_stream on the full train stream
            from oracle import ref as R
            tre = wl["split"].train.edges
            t_max = float(tre["ts"].max()) if len(tre) else 0.0
            cent, _ = R.compute_centrality(tre, N, t_max, 0.5)
            hubs = R.select_hubs(cent, 0.05)
            t0 = time.time()
            R.partition(tre, N, t_max, P, cent, hubs, args.hub_k)
            extra.append(cpu_partition_baseline({"train_edges": len(tre), "partition_s": time.time() - t0,
                                                 "subs": [None] * P}))
        except Exception as ex:
            extra.append({"what": "reference partition_stream", "value": None, "sample": f"unavailable: {ex}"})
        try:  # the CPU TGN oracle (same model) on all host cores
            extra.append(cpu_tgn_oracle_rate(sub_mine.nodes, sub_mine.edges, sub_mine.eids,
                                             dict(D=D, T=T, F=F, K=K, H=H, B=B), log))
        except Exception as ex:
            extra.append({"what": "CPU TGN oracle", "value": None, "sample": f"unavailable: {ex}"})
        cpu["also"] = extra

    if rank == 0:
        out = {
            "metric": metric, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp32 (tf32 tensor-core GRU/attention projections)" if args.gemm_mode == 1 else "fp32",
            "data": "synthetic (gen_powerlaw topology seed 1, hashed bf16-exact edge features seed 2, "
                    "random-init TGN seed 3)",
            "config": cfg_desc, "e2e": e2e, "roofline": roof, "step_roofline": step_roof,
            "gemm_roofline": gemm,
            "cpu_baseline": cpu, "fp32_ffma": fp32, "gpu_launches": launches, "clocks": clk.summary(),
            "effective_edges_per_s": wl["train_edges"] / (tr.epoch_steps() * ms_per_step / 1e3),
            "device_memory_per_gpu": mem_gb,
            "epoch_steps": tr.epoch_steps(), "train_edges": wl["train_edges"],
            "shared_hubs": len(wl["shared"]), "epoch_end_sync_ms": epoch_end_ms,
            "phases_ms": {n: round(t, 4) for n, t in phases},
        }
        print(json.dumps(out))


if __name__ == "__main__":
    main()
