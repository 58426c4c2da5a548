"""Product host path (C++ behind the C-ABI) vs the reference and its golden
vectors: bit-exact streams, centrality, hub sets, SEP assignment, shared set,
induced subgraphs, shuffle groups and eval routing. Ports of
test_graph_io.cpp / test_centrality.cpp / test_partitioner.cpp cases."""
import math

import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from paper_2308_14129_b200 import (DataError, InternalError, HubSet, PartitionerConfig,
                                   PartitionState, make_stream)


def cfg_for(s, parts, k, lam=1.0):
    c = sp.compute_centrality(s, 0.5)
    return PartitionerConfig(parts, lam, 1.0, sp.select_hubs(c, k), c)


def table(cent):
    return sp.CentralityTable(np.array(cent, dtype=np.float64), 0.5)


def toy():
    return make_stream([(0, 4, 1), (1, 4, 2), (0, 1, 3), (2, 4, 4), (2, 3, 5), (1, 3, 6)], 5)


def toy_cfg(lam):
    return PartitionerConfig(2, lam, 1.0, HubSet.from_ids([4], 5, 0.2), table([1, 1, 1, 1, 4]))


# ------------------------------------------------------------ L1 streams
@pytest.mark.parametrize("n,m,alpha,seed", [(10, 20, 2.5, 23), (60, 400, 2.3, 1), (1000, 10000, 2.5, 41),
                                            (1500, 15000, 2.3, 42), (9227, 157474, 2.5, 1)])
def test_gen_powerlaw_bit_identical(ref, n, m, alpha, seed):
    s = sp.gen_powerlaw(n, m, alpha, seed)
    want, nc, tm = ref.gen_powerlaw(n, m, alpha, seed)
    assert s.node_count == nc and s.t_max == tm
    assert s.edges.tobytes() == want.tobytes()


def test_gen_powerlaw_rejects_bad_params():
    for args in [(1, 10, 2.5, 1), (10, 0, 2.5, 1), (10, 10, 1.0, 1)]:
        with pytest.raises(DataError) as ei:
            sp.gen_powerlaw(*args)
        assert ei.value.code == "InvalidParams"


@pytest.mark.parametrize("n,ft,fv,want", [(10, 0.7, 0.1, (7, 1, 2)), (100, 0.7, 0.15, (70, 15, 15)),
                                          (1, 0.5, 0.0, (0, 0, 1))])
def test_chrono_split_sizes(ref, n, ft, fv, want):
    # test_graph_io.cpp:80-102
    s = make_stream([(0, 1, float(t + 1)) for t in range(n)], 2)
    sp_ = sp.chrono_split(s, ft, fv)
    assert (len(sp_.train), len(sp_.val), len(sp_.test)) == want == ref.chrono_split_sizes(n, ft, fv)


def test_chrono_split_rejects():
    s = make_stream([(0, 1, 1.0)], 2)
    for ft, fv in [(0.0, 0.1), (1.0, 0.0), (0.5, -0.1), (0.8, 0.3)]:
        with pytest.raises(DataError):
            sp.chrono_split(s, ft, fv)


# ------------------------------------------------------------ centrality
def test_centrality_known_answer():
    # test_centrality.cpp:35-42
    s = make_stream([(0, 1, 0.0), (0, 2, 1.0)], 3)
    c = sp.compute_centrality(s, 0.5)
    assert c.cent[0] == pytest.approx(math.exp(-0.5) + 1.0)
    with pytest.raises(DataError) as ei:
        sp.compute_centrality(s, 1.0)
    assert ei.value.code == "BetaOutOfRange"


def test_hub_tie_break_and_base():
    # test_centrality.cpp:98-124: ties go to the smaller id; All counts declared nodes
    c = table([2.0, 5.0, 5.0, 0.0, 1.0, 0.0])
    assert sp.select_hubs(c, 0.5).hubs.tolist() == [1, 2]
    assert sp.select_hubs(c, 0.25).hubs.tolist() == [1]
    assert sp.select_hubs(c, 0.5, sp.HubBase.All).hubs.tolist() == [0, 1, 2]
    with pytest.raises(DataError):
        sp.select_hubs(c, 1.5)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_centrality_and_hubs_bit_identical(ref, seed):
    s = sp.gen_powerlaw(500, 6000, 2.2 + 0.1 * seed, seed)
    c = sp.compute_centrality(s, 0.5)
    want, tm = ref.compute_centrality(s.edges, s.node_count, s.t_max, 0.5)
    assert c.cent.tobytes() == want.tobytes() and c.t_max == tm
    for k in (0.0, 0.01, 0.05, 0.1, 0.5, 1.0):
        assert sp.select_hubs(c, k).hubs.tolist() == ref.select_hubs(want, k).tolist()


# ----------------------------------------------------------- partitioner
def test_score_worked_example():
    # test_partitioner.cpp:183-200
    cfg = PartitionerConfig(2, 1.0, 1.0, HubSet.from_ids([], 2, 0.0), table([1.0, 3.0]))
    st = PartitionState([2, 4], [[0], [1]], 4, 2)
    assert sp.score(0, 1, 0, st, cfg) == pytest.approx(1.75 + 2.0 / 3.0, rel=1e-9)
    fresh = PartitionState([0, 0], [[], []], 0, 0)
    assert sp.score(0, 1, 0, fresh, cfg) == 0.0 and sp.score(0, 1, 1, fresh, cfg) == 0.0
    cfg0 = PartitionerConfig(1, 1.0, 1.0, HubSet.from_ids([], 2, 0.0), table([0.0, 0.0]))
    assert sp.score(0, 1, 0, PartitionState([0], [[0], [0]], 0, 0), cfg0) == 3.0


def test_six_edge_golden_trace():
    # test_partitioner.cpp:225-239; acceptance.cpp:426-449
    pa = sp.partition_stream(toy(), toy_cfg(2.0))
    assert pa.edge_part.tolist() == [0, 0, 0, 1, 1, -1]
    assert pa.discard_count == 1
    assert pa.shared.tolist() == [4]
    assert pa.node_parts == [[0], [0], [1], [1], [0, 1]]


def test_six_edge_lambda_one_collapses():
    pa = sp.partition_stream(toy(), toy_cfg(1.0))
    assert pa.edge_part.tolist() == [0] * 6 and pa.discard_count == 0 and len(pa.shared) == 0


def test_single_edge_and_resident_pin():
    s = make_stream([(0, 1, 1.0)], 2)
    pa = sp.partition_stream(s, cfg_for(s, 2, 0.0))
    assert pa.edge_part.tolist() == [0] and pa.node_parts == [[0], [0]]
    s2 = make_stream([(2, 3, 1), (3, 4, 2)], 5)
    cfg = PartitionerConfig(2, 100.0, 1.0, HubSet.from_ids([4], 5, 0.2), table([1, 1, 1, 1, 4]))
    pa2 = sp.partition_stream(s2, cfg)
    assert pa2.edge_part[1] == pa2.edge_part[0] and pa2.discard_count == 0


def test_self_loops_never_discarded(ref):
    s = make_stream([(0, 1, 1), (2, 2, 2), (0, 0, 3), (2, 2, 4)], 3)
    cfg = cfg_for(s, 2, 0.0)
    pa = sp.partition_stream(s, cfg)
    assert pa.discard_count == 0 and (pa.edge_part != -1).all()


def test_balance_within_one():
    s = make_stream([(2 * i, 2 * i + 1, float(i + 1)) for i in range(20)], 40)
    pa = sp.partition_stream(s, cfg_for(s, 4, 0.0, lam=100.0))
    sizes = np.bincount(pa.edge_part, minlength=4)
    assert sizes.max() - sizes.min() <= 1 and pa.discard_count == 0


def test_partition_validation():
    bad = make_stream([(0, 1, 5.0), (1, 0, 1.0)], 2)
    with pytest.raises(DataError) as ei:
        sp.partition_stream(bad, cfg_for(toy(), 2, 0.0))
    assert ei.value.code == "UnsortedStream"
    c = toy_cfg(2.0)
    c.lambda_ = 0.0
    with pytest.raises(DataError) as ei:
        sp.partition_stream(toy(), c)
    assert ei.value.code == "InvalidParams"


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("k", [0.0, 0.01, 0.05, 0.2, 1.0])
def test_partition_stream_bit_identical(ref, seed, parts, k):
    s = sp.gen_powerlaw(60 * seed + 40, 400 * seed + 300, 2.3, seed)
    cfg = cfg_for(s, parts, k)
    pa = sp.partition_stream(s, cfg)
    want = ref.partition(s.edges, s.node_count, s.t_max, parts, cfg.centrality.cent,
                         cfg.hub_set.hubs, k)
    assert pa.edge_part.tolist() == want["edge_part"].tolist()
    assert pa.node_parts == want["node_parts"]
    assert pa.shared.tolist() == want["shared"].tolist()
    assert pa.discard_count == want["discards"] and pa.k_eff == want["k_eff"]
    un = sp.partition_unrestricted(s, cfg)
    wu = ref.partition(s.edges, s.node_count, s.t_max, parts, cfg.centrality.cent,
                       cfg.hub_set.hubs, k, mode=1)
    assert un.edge_part.tolist() == wu["edge_part"].tolist() and un.discard_count == 0
    assert un.k_eff == 1.0


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_partition_large_and_many_parts(ref, parts):
    s = sp.gen_powerlaw(9227, 157474, 2.5, 1)
    tr = sp.chrono_split(s, 0.7, 0.15).train
    cfg = cfg_for(tr, parts, 0.05)
    pa = sp.partition_stream(tr, cfg)
    want = ref.partition(tr.edges, tr.node_count, tr.t_max, parts, cfg.centrality.cent,
                         cfg.hub_set.hubs, 0.05)
    assert pa.edge_part.tobytes() == want["edge_part"].tobytes()
    assert pa.shared.tolist() == want["shared"].tolist()
    assert pa.node_parts == want["node_parts"]


def test_partition_100_parts(ref):
    s = sp.gen_powerlaw(2000, 20000, 2.2, 5)
    cfg = cfg_for(s, 100, 0.05)
    pa = sp.partition_stream(s, cfg)
    want = ref.partition(s.edges, s.node_count, s.t_max, 100, cfg.centrality.cent, cfg.hub_set.hubs, 0.05)
    assert pa.edge_part.tobytes() == want["edge_part"].tobytes()
    assert pa.node_parts == want["node_parts"]


def test_k0_never_replicates():
    for seed in range(1, 6):
        s = sp.gen_powerlaw(10 + 37 * seed, 100 + 211 * seed, 2.1 + 0.05 * seed, seed)
        for parts in (2, 4, 8):
            pa = sp.partition_stream(s, cfg_for(s, parts, 0.0))
            assert len(pa.shared) == 0 and all(len(v) <= 1 for v in pa.node_parts)


# --------------------------------------------------------- eval routing
def test_eval_routing_fixture():
    # test_partitioner.cpp:361-387
    pa = sp.partition_stream(toy(), toy_cfg(2.0))
    split = sp.ChronoSplit(toy(), make_stream([(4, 4, 7), (0, 1, 8), (0, 2, 9)], 5),
                           make_stream([(9, 0, 10), (2, 4, 11)], 10), 0.7, 0.15, 0.15)
    r = sp.assign_eval_edges(split, pa)
    assert r.val_edges[0] == [0, 1] and r.val_edges[1] == [0] and r.val_unroutable == 1
    assert r.test_edges[1] == [1] and r.test_unroutable == 1


# ------------------------------------------------- subgraphs and shuffle
def test_induced_subgraphs_exact():
    # test_pac_sim.cpp:152-175
    s = make_stream([(0, 1, 1), (1, 2, 2), (2, 3, 3), (0, 3, 4)], 4)
    subs = sp.induce_subgraphs(s, [[0]] * 4, 1)
    assert subs[0].edges.tobytes() == s.edges.tobytes() and subs[0].nodes.tolist() == [0, 1, 2, 3]
    subs = sp.induce_subgraphs(s, [[0], [0], [1], [1]], 2)
    assert subs[0].edges.tolist() == [(0, 1, 1.0)] and subs[1].edges.tolist() == [(2, 3, 3.0)]
    assert subs[0].eids.tolist() == [0] and subs[1].eids.tolist() == [2]
    with pytest.raises(DataError) as ei:
        sp.induce_subgraphs(s, [[0], [0], [2], [1]], 2)
    assert ei.value.code == "InvalidPartition"


@pytest.mark.parametrize("parts,k", [(2, 0.05), (4, 0.1), (8, 0.05)])
def test_induce_bit_identical(ref, parts, k):
    s = sp.gen_powerlaw(300, 5000, 2.3, 9)
    pa = sp.partition_stream(s, cfg_for(s, parts, k))
    subs = sp.induce_subgraphs(s, pa.node_parts, parts)
    want = ref.induce_subgraphs(s.edges, s.node_count, pa.node_parts, parts)
    for g, (wn, we) in zip(subs, want):
        assert g.nodes.tolist() == wn.tolist()
        assert g.edges.tobytes() == we.tobytes()
        assert s.edges[g.eids.astype(np.int64)].tobytes() == we.tobytes()


def test_shuffle_combine_semantics(ref):
    parts = [[0, 1], [2], [3, 4], [5]]
    out = sp.shuffle_combine(parts, 4, 99)
    assert sorted(map(tuple, out)) == sorted(map(tuple, parts))
    assert sp.shuffle_combine(parts, 1, 5) == [[0, 1, 2, 3, 4, 5]]
    assert sp.shuffle_combine([[0, 1, 9], [1, 2, 9]], 1, 5) == [[0, 1, 2, 9]]
    with pytest.raises(DataError) as ei:
        sp.shuffle_combine(parts, 3, 1)
    assert ei.value.code == "IndivisibleParts"
    for seed in range(50):
        small = [[p] for p in range(8)]
        assert sp.shuffle_combine(small, 4, seed) == ref.shuffle_combine(small, 4, seed)
