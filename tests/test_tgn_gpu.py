"""CUDA TGN step (through the C-ABI) vs the CPU oracle (oracle/tgn_oracle.py)
on identical inputs and seeds. Bit-exact: parameter init, negatives, sampled
neighbour ids, last-message sets. FP32 tolerances (stated per check) for
embeddings, loss, gradients, parameters and memory."""
import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from tests.tgn_cases import oracle_for, partitioned, rel_err

pytestmark = pytest.mark.gpu

# FP32 tolerances (relative L2): one step from identical state differs only by
# summation order (GEMM tiling, atomics) -> 1e-5; trajectories drift over steps.
TOL_STEP = 2e-5
TOL_GRAD = 2e-4
TOL_TRAJ = 2e-3
# tcgen05 TF32 projections (10-bit operand mantissas), stated tolerances:
# one step from identical state, and the drift of an 8-step trajectory.
TOL_TF32_STEP = 5e-3
TOL_TF32 = 3e-2
TOL_TF32_GRAD = 2e-2


def small_cfg(**kw):
    base = dict(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=64, lr=1e-3)
    base.update(kw)
    return sp.TGNConfig(**base)


def glob(o, w, local_ids):
    nodes = o.W[w].nodes
    out = np.where(np.asarray(local_ids) < 0, 0xFFFFFFFF, nodes[np.maximum(np.asarray(local_ids), 0)])
    return out.astype(np.uint32)


def test_param_init_bit_exact():
    _, _, pa, subs = partitioned()
    cfg = small_cfg()
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    assert tr.n_params == o.total
    assert np.array_equal(tr.params(), o.flat.numpy())


@pytest.mark.parametrize("parts", [1, 2])
def test_steps_match_oracle(parts):
    _, _, pa, subs = partitioned(parts=parts)
    cfg = small_cfg()
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.set_debug(True)
    o = oracle_for(cfg, subs, pa.shared)
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for step in range(12):
        gl = tr.step()
        ol = o.step()
        for w in range(parts):
            t = tr.last_step(w)
            ref = o.last[w]
            assert np.array_equal(t["neg"], glob(o, w, ref["neg"])), f"negatives differ step {step}"
            assert np.array_equal(t["nbr"], glob(o, w, ref["nbr_ids"])), f"neighbours differ step {step}"
            tol = TOL_STEP if step == 0 else TOL_TRAJ
            assert rel_err(t["emb"], ref["emb"]) < tol, (step, w, rel_err(t["emb"], ref["emb"]))
            assert abs(gl[w] - ol[w]) <= tol * max(1.0, abs(ol[w])), (step, gl[w], ol[w])
        if step == 0:
            assert rel_err(tr.grads(), o.grad.numpy()) < TOL_GRAD
        assert rel_err(tr.params(), o.flat.numpy()) < TOL_TRAJ
        for w in range(parts):
            m, lu = tr.memory(w)
            assert np.array_equal(lu, o.lu[w]), f"last_update differs step {step}"
            assert rel_err(m, o.mem[w].numpy()) < TOL_TRAJ


@pytest.mark.parametrize("parts", [1, 2])
def test_tensor_core_mode_within_tolerance(parts):
    """gemm_mode=1 (tcgen05 TF32 for the GRU and attention projections): bit-exact
    sampling as FP32, values within the stated TF32 tolerance of the FP32 oracle."""
    _, _, pa, subs = partitioned(parts=parts)
    cfg = small_cfg(gemm_mode=1)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.set_debug(True)
    o = oracle_for(cfg, subs, pa.shared)
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for step in range(8):
        gl = tr.step()
        ol = o.step()
        for w in range(parts):
            t = tr.last_step(w)
            ref = o.last[w]
            assert np.array_equal(t["neg"], glob(o, w, ref["neg"]))
            assert np.array_equal(t["nbr"], glob(o, w, ref["nbr_ids"]))
            tol = TOL_TF32_STEP if step == 0 else TOL_TF32
            assert rel_err(t["emb"], ref["emb"]) < tol, (step, rel_err(t["emb"], ref["emb"]))
            assert abs(gl[w] - ol[w]) <= tol * abs(ol[w])
        if step == 0:
            assert rel_err(tr.grads(), o.grad.numpy()) < TOL_TF32_GRAD
    assert rel_err(tr.params(), o.flat.numpy()) < TOL_TF32


def test_gradients_per_tensor_first_step():
    _, _, pa, subs = partitioned(parts=2)
    cfg = small_cfg()
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    # warm the memory so the GRU path carries gradient, then compare step 3's grads
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for _ in range(3):
        tr.step()
        o.step()
        # re-sync parameters and memory to the oracle so the next step starts identical
        tr.set_params(o.flat.numpy())
        for w in range(2):
            tr.set_memory(w, o.mem[w].numpy(), o.lu[w])
    g = tr.grads()
    og = o.grad.numpy()
    lay, _ = __import__("oracle.tgn_oracle", fromlist=["x"]).param_layout(o.c)
    for name, spec in lay.items():
        off, n = spec[0], (spec[1] * spec[3] if len(spec) == 4 else spec[1])
        e = rel_err(g[off:off + n], og[off:off + n])
        assert e < TOL_GRAD, (name, e)


def test_epoch_end_restore_and_sync():
    _, _, pa, subs = partitioned(parts=2, nodes=200, edges=2500)
    cfg = small_cfg(batch_size=50)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    assert tr.epoch_steps() == o.epoch_steps()
    tr.run_epoch(0)
    o.run_epoch(0)
    for w in range(2):
        m, lu = tr.memory(w)
        assert np.array_equal(lu, o.lu[w])
        assert rel_err(m, o.mem[w].numpy()) < TOL_TRAJ
    # shared hubs agree across workers after the average sync
    n0, n1 = tr.local_nodes(0), tr.local_nodes(1)
    m0, lu0 = tr.memory(0)
    m1, lu1 = tr.memory(1)
    for g in pa.shared:
        i0, i1 = np.searchsorted(n0, g), np.searchsorted(n1, g)
        assert np.array_equal(m0[i0], m1[i1]) and lu0[i0] == lu1[i1]


def test_two_epochs_loss_tracks_oracle():
    _, _, pa, subs = partitioned(parts=2, nodes=200, edges=3000)
    cfg = small_cfg(batch_size=100)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    for ep in range(2):
        lg = tr.run_epoch(ep)
        lo = np.nanmean([x for l in o.run_epoch(ep) for x in l])
        assert abs(lg - lo) < 5e-3 * abs(lo), (ep, lg, lo)


def test_no_cpu_fallback_without_device(monkeypatch):
    # the product path must fail loudly, not fall back, when no device is visible
    import subprocess, sys, os
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    code = ("import paper_2308_14129_b200 as sp\n"
            "from tests.tgn_cases import partitioned\n"
            "_,_,pa,subs = partitioned()\n"
            "try:\n    sp.TGNTrainer(sp.TGNConfig(d_mem=8,d_time=8,d_edge=4,batch_size=16), subs)\n"
            "except sp.InternalError as e:\n    print('LOUD', e.code)\n")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "LOUD CudaError" in out.stdout, out.stdout + out.stderr


# model shapes covering every attention-kernel instantiation class: GDELT dims
# (4 column chunks per lane, 2 gradient-carrying), no edge features (LastFM),
# one head, and the (K <= 16, H <= 4) variant
@pytest.mark.parametrize("dims", [
    dict(d_mem=100, d_time=100, d_edge=186, n_neighbors=10, n_heads=2, batch_size=48),
    dict(d_mem=32, d_time=16, d_edge=0, n_neighbors=5, n_heads=1),
    dict(d_mem=64, d_time=32, d_edge=60, n_neighbors=16, n_heads=4, batch_size=48),
    dict(d_mem=128, d_time=96, d_edge=20, n_neighbors=12, n_heads=2, batch_size=40),
])
def test_model_shapes_match_oracle(dims):
    _, _, pa, subs = partitioned(parts=1, nodes=150, edges=2000)
    cfg = small_cfg(**dims)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.set_debug(True)
    o = oracle_for(cfg, subs, pa.shared)
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for step in range(4):
        gl = tr.step()
        ol = o.step()
        t = tr.last_step(0)
        ref = o.last[0]
        assert np.array_equal(t["nbr"], glob(o, 0, ref["nbr_ids"]))
        tol = TOL_STEP if step == 0 else TOL_TRAJ
        assert rel_err(t["emb"], ref["emb"]) < tol, (step, rel_err(t["emb"], ref["emb"]))
        assert abs(gl[0] - ol[0]) <= tol * max(1.0, abs(ol[0]))
        if step == 0:
            assert rel_err(tr.grads(), o.grad.numpy()) < TOL_GRAD
    assert rel_err(tr.params(), o.flat.numpy()) < TOL_TRAJ


def test_seek_positions_schedule_mid_epoch():
    _, _, pa, subs = partitioned(parts=2)
    cfg = small_cfg()
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.begin_epoch(0)
    mid = tr.epoch_steps() // 2
    tr.seek(mid)
    for w in range(2):
        nb = -(-len(subs[w].edges) // cfg.batch_size)
        assert tr.next_batch(w)[0] == (mid % nb) * cfg.batch_size
    loss = tr.step()
    assert np.all(np.isfinite(loss))
    with pytest.raises(sp.UsageError):
        tr.seek(tr.epoch_steps())


@pytest.mark.parametrize("gemm_mode", [0, 1])
def test_graph_replay_matches_eager(gemm_mode):
    """Regular steps replay a captured CUDA graph; the per-step control words
    (batch start, negative base, Adam corrections) live on the device, so the
    replayed trajectory equals the eagerly launched one — bit for bit, since
    every reduction of the step has a fixed order."""
    _, _, pa, subs = partitioned(parts=2, nodes=200, edges=3000)
    cfg = small_cfg(batch_size=50, gemm_mode=gemm_mode)
    out = []
    for graph in (False, True):
        tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
        tr.set_graph(graph)
        losses = [tr.run_epoch(ep) for ep in range(2)]
        out.append((np.array(losses), tr.params(), tr.memory(0), tr.memory(1)))
    (l0, p0, m0, u0), (l1, p1, m1, u1) = out
    assert np.array_equal(l0, l1), (l0, l1)
    assert np.array_equal(p0, p1)
    for a, b in ((m0, m1), (u0, u1)):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("gemm_mode", [0, 1])
def test_training_is_deterministic(gemm_mode):
    """Two trainings from the same inputs and seeds are bit-identical (the
    memory-row gradient is a fixed-order reduction, tgn_dh.cu; every other
    sum already was): the per-step losses, parameters, Adam-updated weights
    and memory states. Hubs make many neighbour occurrences share a pending
    row, the case float atomics made order-dependent."""
    _, _, pa, subs = partitioned(parts=2, nodes=300, edges=12000)
    cfg = small_cfg(batch_size=400, d_mem=100, d_time=100, d_edge=20, n_neighbors=10,
                    gemm_mode=gemm_mode)
    runs = []
    for _ in range(2):
        tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
        tr.begin_epoch(0)
        losses = [tr.step() for _ in range(min(8, tr.epoch_steps()))]
        runs.append((np.array(losses), tr.params(), tr.grads(), tr.memory(0), tr.memory(1)))
        tr.close()
    (l0, p0, g0, a0, b0), (l1, p1, g1, a1, b1) = runs
    assert np.array_equal(l0, l1)
    assert np.array_equal(p0, p1) and np.array_equal(g0, g1)
    for x, y in ((a0, a1), (b0, b1)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


def test_shuffle_combine_rebind_matches_oracle():
    """simulate's shuffle branch (pac_sim.cpp:280-329) for the TGN trainer:
    4 small SEP parts regrouped into 2 workers per epoch (seeded), the trainer
    rebound each epoch; parameters and Adam state carry across epochs."""
    from oracle import tgn_oracle as T
    s, split, pa, small_subs = partitioned(nodes=200, edges=2400, parts=4)
    small = [g.nodes for g in small_subs]
    cfg = small_cfg()
    tr = o = None
    for epoch in range(2):
        groups = sp.shuffle_combine(small, 2, 11 + epoch)
        subs, recovered = sp.induce_groups(split.train, groups, small)
        assert recovered >= 0
        if tr is None:
            tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
            o = oracle_for(cfg, subs, pa.shared)
        else:
            tr.rebind(subs)
            o.rebind([T.WorkerData(g.nodes, g.edges, g.eids, o.c.d_edge, o.c.seed_feat) for g in subs])
        assert tr.epoch_steps() == o.epoch_steps()
        tr.begin_epoch(epoch)
        o.begin_epoch(epoch)
        for _ in range(o.epoch_steps()):
            gl = tr.step()
            ol = o.step()
            for w in range(2):
                if not np.isnan(ol[w]):
                    assert abs(gl[w] - ol[w]) <= TOL_TRAJ * max(1.0, abs(ol[w])), (epoch, gl, ol)
        tr.end_epoch()
        o.end_epoch()
        assert rel_err(tr.params(), o.flat.numpy()) < TOL_TRAJ, epoch
        for w in range(2):
            m, lu = tr.memory(w)
            assert np.array_equal(lu, o.lu[w]), (epoch, w)
            assert rel_err(m, o.mem[w].numpy()) < TOL_TRAJ, (epoch, w)
    with pytest.raises(sp.DataError) as ei:
        tr.rebind(subs[:1])
    assert ei.value.code == "ConfigMismatch"


def test_host_fed_steps_match_resident_steps():
    """End-to-end API (spd_tgn_step_host and its pipelined form
    spd_tgn_step_host_async + spd_tgn_sync): the same batches fed from host
    memory train like the device-resident stream (FP32 trajectory bar)."""
    import torch
    _, _, pa, subs = partitioned(parts=1)
    cfg = small_cfg()
    runs = {}
    for mode in ("resident", "host", "async"):
        tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
        tr.begin_epoch(0)
        ev_all = tr.worker_events(0)
        Fp = tr.next_batch(0)[2]
        n = min(8, tr.epoch_steps())
        losses = []
        loss_pin = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        keep = []
        for k in range(n):
            lo, hi, _ = tr.next_batch(0)
            if mode == "resident":
                losses.append(float(tr.step()[0]))
                continue
            ev = torch.empty((hi - lo) * 16, dtype=torch.uint8, pin_memory=True).numpy().view(sp.EDGE_DTYPE)
            ev[:] = ev_all[lo:hi]
            ft = torch.empty((hi - lo) * Fp, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
            ft = sp.edge_features_bf16(cfg.seed_feat, subs[0].eids[lo:hi], cfg.d_edge, Fp,
                                       out=ft.reshape(hi - lo, Fp))
            keep.append((ev, ft))
            if mode == "host":
                losses.append(float(tr.step_host([ev], [ft])[0]))
            else:
                tr.step_host_async([ev], [ft], loss_pin[k:k + 1])
        if mode == "async":
            tr.sync()
            losses = loss_pin.tolist()
        h2d, d2h = tr.io_bytes()
        if mode != "resident":
            assert h2d > 0 and d2h == 4 * n
        runs[mode] = (np.array(losses), tr.params())
        tr.close()
    ref_l, ref_p = runs["resident"]
    for mode in ("host", "async"):
        l, p = runs[mode]
        assert np.all(np.isfinite(l))
        assert np.max(np.abs(l - ref_l)) <= TOL_TRAJ * max(1.0, float(np.max(np.abs(ref_l)))), (mode, l, ref_l)
        assert rel_err(p, ref_p) < TOL_TRAJ, mode


def test_host_fed_events_must_match_resident_stream():
    """The neighbour CSR, negative pool and feature rows are built from the
    partition's resident stream: host-fed batches that differ are refused."""
    _, _, pa, subs = partitioned(parts=1)
    cfg = small_cfg()
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.begin_epoch(0)
    ev_all = tr.worker_events(0)
    lo, hi, Fp = tr.next_batch(0)
    ev = np.ascontiguousarray(ev_all[lo:hi]).copy()
    ev["ts"][3] += 0.25
    ft = sp.edge_features_bf16(cfg.seed_feat, subs[0].eids[lo:hi], cfg.d_edge, Fp)
    with pytest.raises(sp.DataError) as ei:
        tr.step_host([ev], [ft])
    assert ei.value.code == "InvalidParams"
    ok = np.ascontiguousarray(ev_all[lo:hi]).copy()
    assert np.all(np.isfinite(tr.step_host([ok], [ft])))
    tr.close()


@pytest.mark.parametrize("parts,workers", [(4, 2), (8, 4), (6, 3)])
def test_device_shuffle_combine_matches_host_rebind(parts, workers):
    """Shuffle-combine re-induction on the device (spd_tgn_attach_stream +
    spd_tgn_shuffle_epoch, K13) against the host path (spd_shuffle_combine +
    spd_induce_groups + spd_tgn_rebind): identical worker events, node sets
    and `recovered` counts every epoch, and bit-identical training (same
    parameters and memory after each epoch)."""
    s, split, pa, small_subs = partitioned(nodes=300, edges=4000, parts=parts, seed=3)
    small = [g.nodes for g in small_subs]
    cfg = small_cfg()
    host = dev = None
    for epoch in range(2):
        seed = 11 + epoch
        groups = sp.shuffle_combine(small, workers, seed)
        subs, rec_host = sp.induce_groups(split.train, groups, small)
        if host is None:
            host = sp.TGNTrainer(cfg, subs, shared=pa.shared)
            dev = sp.TGNTrainer(cfg, subs, shared=pa.shared)
            dev.attach_stream(split.train, small)
        else:
            host.rebind(subs)
        rec_dev = dev.shuffle_epoch(seed)
        assert rec_dev == rec_host, (epoch, rec_dev, rec_host)
        assert dev.epoch_steps() == host.epoch_steps()
        for w in range(workers):
            np.testing.assert_array_equal(dev.local_nodes(w), host.local_nodes(w))
            a, b = dev.worker_events(w), host.worker_events(w)
            assert a.tobytes() == b.tobytes(), (epoch, w)
        for t in (host, dev):
            t.begin_epoch(epoch)
            for _ in range(t.epoch_steps()):
                t.step(want_loss=False)
            t.end_epoch()
        assert np.array_equal(dev.params(), host.params()), epoch
        for w in range(workers):
            (m1, l1), (m2, l2) = dev.memory(w), host.memory(w)
            assert np.array_equal(m1, m2) and np.array_equal(l1, l2), (epoch, w)
    host.close()
    dev.close()


@pytest.mark.parametrize("backbone", [1, 2])
@pytest.mark.parametrize("gemm_mode", [0, 1])
@pytest.mark.parametrize("parts", [1, 2])
def test_jodie_backbone_matches_oracle(parts, gemm_mode, backbone):
    """JODIE and DyRep backbones (spd_tgn_config.backbone = 1 / 2):
    RNN memory updater + time-projection (JODIE) or identity (DyRep) embedding
    on the same message, last-message, decoder and PAC-schedule kernels;
    DyRep's messages carry the other endpoint's temporal-attention embedding
    (the TGN attention kernels, forward only). Per-step embeddings, losses,
    first-step gradients, parameters, memory and clocks against the oracle's
    JODIE / DyRep, a whole epoch with the epoch-end restore + shared-hub sync
    included."""
    _, _, pa, subs = partitioned(parts=parts)
    cfg = small_cfg(backbone=backbone, gemm_mode=gemm_mode)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    assert tr.n_params == o.total and np.array_equal(tr.params(), o.flat.numpy())
    tr.set_debug(True)
    step_tol = TOL_STEP if gemm_mode == 0 else TOL_TF32_STEP
    traj_tol = TOL_TRAJ if gemm_mode == 0 else TOL_TF32
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for step in range(o.epoch_steps()):
        gl = tr.step()
        ol = o.step()
        tol = step_tol if step == 0 else traj_tol
        for w in range(parts):
            if np.isnan(ol[w]):
                continue
            t = tr.last_step(w)
            assert np.array_equal(t["neg"], glob(o, w, o.last[w]["neg"]))
            assert rel_err(t["emb"], o.last[w]["emb"]) < tol, (step, w, rel_err(t["emb"], o.last[w]["emb"]))
            assert abs(gl[w] - ol[w]) <= tol * max(1.0, abs(ol[w])), (step, gl[w], ol[w])
        if step == 0:
            assert rel_err(tr.grads(), o.grad.numpy()) < (TOL_GRAD if gemm_mode == 0 else TOL_TF32_GRAD)
        assert rel_err(tr.params(), o.flat.numpy()) < traj_tol, step
    tr.end_epoch()
    o.end_epoch()
    # memory after a whole epoch: TF32 GEMM differences accumulate through
    # every RNN update of a row (parameters stay within the trajectory bar)
    mem_tol = traj_tol if gemm_mode == 0 else 6e-2
    for w in range(parts):
        m, lu = tr.memory(w)
        assert np.array_equal(lu, o.lu[w])
        assert rel_err(m, o.mem[w].numpy()) < mem_tol
    tr.close()


@pytest.mark.parametrize("concurrent", [1, 0])
@pytest.mark.parametrize("parts,sync_average,backbone", [(2, 1, 0), (3, 0, 0), (2, 1, 1), (2, 1, 2)])
def test_concurrent_workers_match_oracle(parts, sync_average, backbone, concurrent):
    """spd_tgn_config.concurrent = 1: a process's local workers train as
    concurrent lanes (own streams, scratch, graphs and parameter replica; an
    in-process peer group for the fused all-reduce + Adam and the epoch-end
    sync). Two epochs against the oracle at the FP32 trajectory bar, graph
    replay on, losses / parameters / memory / clocks, and the evaluation path."""
    _, _, pa, subs = partitioned(parts=parts)
    cfg = small_cfg(concurrent=concurrent, sync_average=sync_average, backbone=backbone)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    assert np.array_equal(tr.params(), o.flat.numpy())
    for epoch in range(2):
        tr.begin_epoch(epoch)
        o.begin_epoch(epoch)
        assert tr.epoch_steps() == o.epoch_steps()
        for _ in range(o.epoch_steps()):
            gl = tr.step()
            ol = o.step()
            for w in range(parts):
                if not np.isnan(ol[w]):
                    assert abs(gl[w] - ol[w]) <= TOL_TRAJ * max(1.0, abs(ol[w])), (epoch, gl, ol)
        tr.end_epoch()
        o.end_epoch()
        assert rel_err(tr.params(), o.flat.numpy()) < TOL_TRAJ, epoch
        for w in range(parts):
            m, lu = tr.memory(w)
            assert np.array_equal(lu, o.lu[w]), (epoch, w)
            print(f"epoch {epoch} worker {w} memory rel err {rel_err(m, o.mem[w].numpy()):.2e}")
            assert rel_err(m, o.mem[w].numpy()) < (TOL_TRAJ if epoch == 0 else 5e-3), (epoch, w)
    # timed steps across an epoch boundary run every lane
    ms = tr.run_steps(o.epoch_steps() + 3)
    assert ms > 0
    tr.close()


@pytest.mark.parametrize("gemm_mode", [0, 1])
@pytest.mark.parametrize("fold_o,fold_q", [("0", "0"), ("1", "1")])
def test_projection_fold_variants_match_oracle(gemm_mode, fold_o, fold_q, monkeypatch):
    """The per-step folded projections (O = [xbar] Wc^T, default on;
    Qp = [q_in | 1] Wqk, SPD_FOLD_Q=1) and the unfolded chains all meet the
    oracle's bars: embeddings, losses, first-step gradients and parameters."""
    monkeypatch.setenv("SPD_FOLD_O", fold_o)
    monkeypatch.setenv("SPD_FOLD_Q", fold_q)
    _, _, pa, subs = partitioned(parts=2)
    cfg = small_cfg(gemm_mode=gemm_mode)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    tr.set_debug(True)
    o = oracle_for(cfg, subs, pa.shared)
    step_tol, traj_tol = (TOL_STEP, TOL_TRAJ) if gemm_mode == 0 else (TOL_TF32_STEP, TOL_TF32)
    tr.begin_epoch(0)
    o.begin_epoch(0)
    for step in range(6):
        gl = tr.step()
        ol = o.step()
        tol = step_tol if step == 0 else traj_tol
        for w in range(2):
            e = rel_err(tr.last_step(w)["emb"], o.last[w]["emb"])
            assert e < tol, (step, w, e)
            assert abs(gl[w] - ol[w]) <= tol * max(1.0, abs(ol[w]))
        if step == 0:
            assert rel_err(tr.grads(), o.grad.numpy()) < (TOL_GRAD if gemm_mode == 0 else TOL_TF32_GRAD)
    assert rel_err(tr.params(), o.flat.numpy()) < traj_tol
    tr.close()
