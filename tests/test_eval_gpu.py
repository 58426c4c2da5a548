"""Evaluation parity: routed val/test edges (assign_eval_edges, partitioner.cpp:212-242)
scored by the CUDA trainer vs the CPU oracle after one training epoch, and the
north-star bar: test AP / AUC within 0.005 of the CPU reference oracle."""
import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from tests.tgn_cases import oracle_for, rel_err

pytestmark = pytest.mark.gpu


def build(nodes, edges, parts, k=0.05, seed=1):
    s = sp.gen_powerlaw(nodes, edges, 2.5, seed)
    split = sp.chrono_split(s, 0.70, 0.15)
    tr = split.train
    c = sp.compute_centrality(tr, 0.5)
    pa = sp.partition_stream(tr, sp.PartitionerConfig(parts, 1.0, 1.0, sp.select_hubs(c, k), c))
    subs = sp.induce_subgraphs(tr, pa.node_parts, parts)
    r = sp.assign_eval_edges(split, pa)
    n_tr, n_va = len(split.train), len(split.val)
    ev = []
    for p in range(parts):
        vi = np.array(r.val_edges[p], np.int64)
        ti = np.array(r.test_edges[p], np.int64)
        edges_p = np.concatenate([split.val.edges[vi], split.test.edges[ti]])
        eids_p = np.concatenate([n_tr + vi, n_tr + n_va + ti]).astype(np.uint64)
        ev.append((edges_p, eids_p, len(vi), len(ti)))
    return pa, subs, ev, r


def scores(model, ev, is_oracle):
    val_p, val_n, test_p, test_n = [], [], [], []
    for w, (edges_p, eids_p, nv, nt) in enumerate(ev):
        if is_oracle:
            model.set_eval(w, edges_p, eids_p)
            a = model.evaluate(w, 0, nv)
            b = model.evaluate(w, nv, nv + nt)
        else:
            model.set_eval_events(w, edges_p, eids_p)
            a = model.evaluate(w, 0, nv)
            b = model.evaluate(w, nv, nv + nt)
        val_p.append(a[0]); val_n.append(a[1]); test_p.append(b[0]); test_n.append(b[1])
    return [np.concatenate(x) for x in (val_p, val_n, test_p, test_n)]


def ap_auc(pos, neg):
    from sklearn.metrics import average_precision_score, roc_auc_score
    y = np.r_[np.ones(len(pos)), np.zeros(len(neg))]
    s = np.r_[pos, neg]
    return average_precision_score(y, s), roc_auc_score(y, s)


@pytest.mark.parametrize("backbone", [0, 1, 2])
@pytest.mark.parametrize("gemm_mode", [0, 1])
def test_eval_scores_match_oracle(gemm_mode, backbone):
    pa, subs, ev, r = build(400, 6000, 2)
    cfg = sp.TGNConfig(d_mem=32, d_time=16, d_edge=12, n_neighbors=5, n_heads=2, batch_size=64,
                       lr=1e-3, gemm_mode=gemm_mode, backbone=backbone)
    tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
    o = oracle_for(cfg, subs, pa.shared)
    tr.run_epoch(0)
    o.run_epoch(0)
    # Evaluation from identical state: after a 94-step lr=1e-3 Adam epoch two
    # FP32 implementations that differ only in summation order drift apart by
    # a few % (Adam normalises gradient noise; e.g. the split decoder sums move
    # the scores 3% vs 0.1% for a single 201-long dot), which would test the
    # chaos of training rather than the eval path. The trajectories themselves
    # are pinned by test_tgn_gpu.py; the AP/AUC bar by the Wikipedia-shape run.
    tr.set_params(o.flat.numpy())
    for w in range(len(subs)):
        tr.set_memory(w, o.mem[w].numpy(), o.lu[w])
    g = scores(tr, ev, False)
    c = scores(o, ev, True)
    # FP32: summation order only; TF32 (10-bit operand mantissas) projections
    tol = 2e-4 if gemm_mode == 0 else 2e-2
    for a, b in zip(g, c):
        assert rel_err(a, b) < tol, rel_err(a, b)
    # (the AP/AUC bar is asserted on the Wikipedia-shaped run below: with ~900
    # test edges here, AP's own sampling noise is ~0.01)


@pytest.mark.slow
@pytest.mark.parametrize("gemm_mode", [0, 1])
def test_wiki_shape_test_ap_within_0005(gemm_mode):
    """BASELINE config 0: Wikipedia-shaped TIG (9,227 nodes, 157,474 edges, 172-d
    edge features), SEP into 2 partitions, 1 epoch, TGN d=100, k=10, B=200.

    Training is deterministic (every reduction has a fixed order, including
    the memory-gradient sum, tgn_dh.cu), so one GPU training is compared with
    the (deterministic) CPU oracle, and a repeated training must reproduce its
    scores bit for bit."""
    pa, subs, ev, r = build(9227, 157474, 2)
    cfg = sp.TGNConfig(d_mem=100, d_time=100, d_edge=172, n_neighbors=10, n_heads=2,
                       batch_size=200, lr=1e-4, gemm_mode=gemm_mode)
    o = oracle_for(cfg, subs, pa.shared)
    o.run_epoch(0)
    c = scores(o, ev, True)
    ca, cu = ap_auc(c[2], c[3])
    runs = []
    for _ in range(2):
        tr = sp.TGNTrainer(cfg, subs, shared=pa.shared)
        tr.run_epoch(0)
        runs.append(scores(tr, ev, False))
        tr.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b), "GPU training is not reproducible"
    ga, gu = ap_auc(runs[0][2], runs[0][3])
    print(f"test AP gpu {ga:.4f} oracle {ca:.4f}; AUC gpu {gu:.4f} oracle {cu:.4f}; "
          f"unroutable test edges {r.test_unroutable}")
    assert abs(ga - ca) <= 0.005 and abs(gu - cu) <= 0.005, (ga, ca, gu, cu)
