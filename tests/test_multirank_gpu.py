"""World-2 and world-3 TGN training through the peer-memory transport
(spd_tgn_peer_*), one process per rank on cuda:0 (ranks sharing one GPU map each other's HBM through
CUDA IPC exactly as ranks on different GPUs do over NVLink): the per-step
gradient all-reduce fused into Adam and the epoch-end shared-hub sync must
reproduce one process training both partitions as local workers
(Alg. 2; run_epoch / sync_shared, pac_sim.cpp:162-264).

Bars: parameters of all ranks bit-identical to each other (same rank-order
sum on every rank); against the single-process run the FP32 trajectory bar
(2e-3; the only difference is where the per-worker gradient sum is rounded);
shared-hub rows identical across the ranks after end_epoch."""
import os
import socket

import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from tests.tgn_cases import partitioned, rel_err

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

EPOCHS = 2


def _cfg(sync_average, gemm_mode):
    return sp.TGNConfig(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=64,
                        lr=1e-3, sync_average=sync_average, gemm_mode=gemm_mode)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _train(tr, epochs):
    losses = []
    for e in range(epochs):
        tr.begin_epoch(e)
        for _ in range(tr.epoch_steps()):
            losses.append(tr.step())
        tr.end_epoch()
    return losses


def _rank(rank, world, port, sync_average, gemm_mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, _, pa, subs = partitioned(nodes=300, edges=4000, parts=world)
    tr = sp.TGNTrainer(_cfg(sync_average, gemm_mode), subs, workers=[rank], shared=pa.shared,
                       rank=rank, world=world, nccl_id=None, device=0)
    blobs = [None] * world
    dist.all_gather_object(blobs, tr.peer_export())
    tr.peer_connect(blobs)
    dist.barrier()
    losses = _train(tr, EPOCHS)
    nodes = tr.local_nodes(rank)
    mem, lu = tr.memory(rank)
    out.put((rank, tr.params(), [float(l[0]) for l in losses], nodes, mem, lu))
    dist.barrier()
    tr.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,sync_average", [(2, 1), (2, 0), (3, 1)])
def test_ranks_peer_transport_match_one_process(world, sync_average):
    gemm_mode = 0
    _, _, pa, subs = partitioned(nodes=300, edges=4000, parts=world)
    assert len(pa.shared) > 0
    one = sp.TGNTrainer(_cfg(sync_average, gemm_mode), subs, shared=pa.shared, device=0)
    ref_losses = _train(one, EPOCHS)
    ref_params = one.params()
    ref_mem = [one.memory(w) for w in range(world)]
    ref_nodes = [one.local_nodes(w) for w in range(world)]
    one.close()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, sync_average, gemm_mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    p0 = res[0][1]
    for r in range(1, world):
        assert np.array_equal(p0, res[r][1]), "replicated parameters diverged across ranks"
    assert rel_err(p0, ref_params) < 2e-3
    for w in range(world):
        _, _, losses, nodes, mem, lu = res[w]
        np.testing.assert_array_equal(nodes, ref_nodes[w])
        ref_loss_w = [float(l[w]) for l in ref_losses]
        assert rel_err(losses, ref_loss_w) < 2e-3
        assert rel_err(mem, ref_mem[w][0]) < 2e-3
        np.testing.assert_array_equal(lu, ref_mem[w][1])
    # shared-hub rows agree across the ranks after the epoch-end sync
    n0 = res[0][3]
    for r in range(1, world):
        n1 = res[r][3]
        common = np.intersect1d(np.intersect1d(n0, n1), np.asarray(pa.shared, np.uint32))
        assert len(common) > 0
        i0 = np.searchsorted(n0, common)
        i1 = np.searchsorted(n1, common)
        np.testing.assert_array_equal(res[0][4][i0], res[r][4][i1])
        np.testing.assert_array_equal(res[0][5][i0], res[r][5][i1])
