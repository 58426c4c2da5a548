"""The CPU oracle (oracle/speed_oracle.c) pinned against the reference itself
(oracle/_ref, compiled from /root/reference/proj/src) and against the
reference tests' golden vectors."""
import math

import numpy as np
import pytest

E = np.dtype([("src", "<u4"), ("dst", "<u4"), ("ts", "<f8")])


def arr(edges):
    return np.array(edges, dtype=E)


def test_mt19937_64_known_answer(coracle):
    # C++11 [rand.predef]: the 10000th draw of a default-constructed (seed
    # 5489) mt19937_64 is 9981545732273789042; here the first draw of seed 5489.
    import random  # noqa: F401  (no std engine in Python; compare against _ref via gen)
    assert coracle.mt_first(5489) == 14514284786278117030


@pytest.mark.parametrize("n,m,alpha,seed", [(10, 20, 2.5, 23), (60, 400, 2.3, 1), (200, 2000, 2.4, 17),
                                            (1000, 10000, 2.5, 41), (25, 150, 2.3, 19), (3, 50, 1.5, 7)])
def test_gen_powerlaw_matches_reference(coracle, ref, n, m, alpha, seed):
    got = coracle.gen_powerlaw(n, m, alpha, seed)
    want, nc, tm = ref.gen_powerlaw(n, m, alpha, seed)
    assert nc == n and tm == float(m)
    assert got.tobytes() == want.tobytes()


def test_centrality_golden(coracle):
    # test_centrality.cpp:35-42: node with roles at t=0 and t=1 (normalised) -> e^{-0.5}+1
    s = arr([(0, 1, 0.0), (0, 2, 1.0)])
    c = coracle.compute_centrality(s, 3, 1.0, 0.5)
    assert c[0] == pytest.approx(math.exp(-0.5) + 1.0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_centrality_hubs_match_reference(coracle, ref, seed):
    s, nc, tm = ref.gen_powerlaw(300, 3000, 2.3, seed)
    c1 = coracle.compute_centrality(s, nc, tm, 0.5)
    c2, _ = ref.compute_centrality(s, nc, tm, 0.5)
    assert c1.tobytes() == c2.tobytes()
    for k in (0.0, 0.01, 0.05, 0.2, 1.0):
        assert coracle.select_hubs(c1, k).tolist() == ref.select_hubs(c2, k).tolist()
        assert coracle.select_hubs(c1, k, True).tolist() == ref.select_hubs(c2, k, True).tolist()


def toy():  # test_partitioner.cpp:166-179
    return arr([(0, 4, 1), (1, 4, 2), (0, 1, 3), (2, 4, 4), (2, 3, 5), (1, 3, 6)])


def test_six_edge_golden_trace(coracle):
    # test_partitioner.cpp:225-239; acceptance.cpp:426-449
    r = coracle.partition_stream(toy(), 5, 2, [1, 1, 1, 1, 4], [4], lam=2.0)
    assert r["edge_part"].tolist() == [0, 0, 0, 1, 1, -1]
    assert r["discards"] == 1
    assert r["shared"].tolist() == [4]
    assert r["node_parts"] == [[0], [0], [1], [1], [0, 1]]
    r1 = coracle.partition_stream(toy(), 5, 2, [1, 1, 1, 1, 4], [4], lam=1.0)
    assert r1["edge_part"].tolist() == [0] * 6 and r1["discards"] == 0


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("parts", [2, 3, 4, 8])
@pytest.mark.parametrize("k", [0.0, 0.05, 0.2, 1.0])
def test_partition_matches_reference(coracle, ref, seed, parts, k):
    s, nc, tm = ref.gen_powerlaw(60 * seed + 40, 400 * seed, 2.3, seed)
    cent, _ = ref.compute_centrality(s, nc, tm, 0.5)
    hubs = ref.select_hubs(cent, k)
    want = ref.partition(s, nc, tm, parts, cent, hubs, k)
    got = coracle.partition_stream(s, nc, parts, cent, hubs)
    assert got["edge_part"].tolist() == want["edge_part"].tolist()
    assert got["node_parts"] == want["node_parts"]
    assert got["shared"].tolist() == want["shared"].tolist()
    assert got["discards"] == want["discards"]


def test_induce_matches_reference(coracle, ref):
    s, nc, tm = ref.gen_powerlaw(40, 200, 2.4, 7)
    cent, _ = ref.compute_centrality(s, nc, tm, 0.5)
    hubs = ref.select_hubs(cent, 0.1)
    pa = ref.partition(s, nc, tm, 4, cent, hubs, 0.1)
    want = ref.induce_subgraphs(s, nc, pa["node_parts"], 4)
    got = coracle.induce(s, nc, pa["node_parts"], 4)
    for (wn, we), (gn, gi) in zip(want, got):
        assert wn.tolist() == gn.tolist()
        assert we.tobytes() == s[gi].tobytes()


def test_model_seeded_and_update_bit_exact(coracle, ref):
    # test_pac_sim.cpp:134-142: 20-edge replay, bit for bit (same libm on the CPU)
    w1, o1 = coracle.model_seeded(8, 17)
    w2, o2, g = ref.model_seeded(8, 17)
    assert w1.tobytes() == w2.tobytes() and o1.tobytes() == o2.tobytes() and g == 0.5
    s, nc, _ = ref.gen_powerlaw(10, 20, 2.5, 23)
    st0, ts0 = np.zeros((nc, 8)), np.zeros(nc)
    a = coracle.model_update_run(st0, ts0, s, w1, o1, 0.5)
    b = ref.model_update_run(st0, ts0, s, w2, o2, 0.5)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    assert coracle.digest(*a) == ref.digest(*b)


@pytest.mark.parametrize("average", [False, True])
def test_run_epoch_matches_reference(coracle, ref, average):
    s, nc, tm = ref.gen_powerlaw(80, 500, 2.4, 13)
    cent, _ = ref.compute_centrality(s, nc, tm, 0.5)
    hubs = ref.select_hubs(cent, 0.1)
    pa = ref.partition(s, nc, tm, 3, cent, hubs, 0.1)
    subs = ref.induce_subgraphs(s, nc, pa["node_parts"], 3)
    w, om, g = ref.model_seeded(8, 77)
    st, ts, b, lp = coracle.run_epoch([e for _, e in subs], nc, 8, w, om, g, pa["shared"], average, 16)
    r = ref.run_epoch([e for _, e in subs], nc, 8, np.zeros((3, nc, 8)), np.zeros((3, nc)), w, om, g,
                      pa["shared"], average, 16)
    assert b == r["batches"] and lp == r["loops"]
    assert st.tobytes() == r["states"].tobytes() and ts.tobytes() == r["last_ts"].tobytes()
    assert [coracle.digest(st[k], ts[k]) for k in range(3)] == r["digests"]


@pytest.mark.parametrize("average", [False, True])
def test_sync_matches_reference(coracle, ref, average):
    rng = np.random.default_rng(2026)
    for W in (2, 3, 5):
        st = rng.uniform(-2, 2, (W, 8, 4))
        ts = rng.uniform(0, 50, (W, 8))
        a = coracle.sync_shared(st, ts, [1, 3, 4, 7], average)
        b = ref.sync_shared(st, ts, [1, 3, 4, 7], average)
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
