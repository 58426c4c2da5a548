"""Global link-prediction metrics (spd_link_metrics):
AP / AUC over the merged score lists of every partition, against sklearn's
average_precision_score / roc_auc_score (the TIG literature's evaluation),
and the multi-rank aggregation over a world-size-2 gloo group: each rank
scores the eval edges routed to its partition (assign_eval_edges,
partitioner.cpp:212-242), the global metric equals the one over the union."""
import os
import socket

import numpy as np
import pytest

import paper_2308_14129_b200 as sp

sk = pytest.importorskip("sklearn.metrics")


def _ref(pos, neg):
    y = np.r_[np.ones(len(pos)), np.zeros(len(neg))]
    s = np.r_[pos, neg].astype(np.float64)
    return sk.average_precision_score(y, s), sk.roc_auc_score(y, s)


@pytest.mark.parametrize("case", ["normal", "ties", "all_equal", "separable", "tiny", "one_each"])
def test_link_metrics_match_sklearn(case):
    rng = np.random.default_rng(7)
    if case == "normal":
        p, n = rng.normal(0.7, 1, 5000), rng.normal(0, 1, 4000)
    elif case == "ties":
        p, n = np.round(rng.normal(0.4, 1, 3000), 1), np.round(rng.normal(0, 1, 3000), 1)
    elif case == "all_equal":
        p, n = np.zeros(10), np.zeros(30)
    elif case == "separable":
        p, n = rng.uniform(2, 3, 100), rng.uniform(-1, 1, 50)
    elif case == "tiny":
        p, n = np.array([0.3, -2.0, 5.0]), np.array([0.3, 1.0])
    else:
        p, n = np.array([1.0]), np.array([2.0])
    p, n = p.astype(np.float32), n.astype(np.float32)
    ap, auc = sp.link_metrics(p, n)
    rap, rauc = _ref(p, n)
    assert abs(ap - rap) < 1e-12 and abs(auc - rauc) < 1e-12, (ap, rap, auc, rauc)


def test_link_metrics_errors():
    with pytest.raises(sp.DataError) as e:
        sp.link_metrics(np.zeros(0, np.float32), np.ones(3, np.float32))
    assert e.value.code == "InvalidParams"
    with pytest.raises(sp.DataError):
        sp.link_metrics(np.array([np.nan], np.float32), np.ones(3, np.float32))


def test_gather_single_rank_is_local():
    p, n = np.array([0.9, 0.1], np.float32), np.array([0.2], np.float32)
    assert sp.gather_link_metrics(p, n) == sp.link_metrics(p, n)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scores(rank):
    rng = np.random.default_rng(100 + rank)
    return rng.normal(0.5, 1, 700 + 300 * rank).astype(np.float32), rng.normal(0, 1, 650).astype(np.float32)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, n = _scores(rank)
    out.put((rank, sp.gather_link_metrics(p, n)))
    dist.destroy_process_group()


def test_two_ranks_gather_global_metrics():
    mp = pytest.importorskip("torch.multiprocessing")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = [_scores(r) for r in range(world)]
    want = _ref(np.concatenate([p for p, _ in parts]), np.concatenate([n for _, n in parts]))
    for r in range(world):  # every rank gets the global metric
        assert abs(res[r][0] - want[0]) < 1e-12 and abs(res[r][1] - want[1]) < 1e-12
