"""Parity mode on the B200: the reference's surrogate MSG/UPD, lockstep
run_epoch, sync_shared and simulate (pac_sim.cpp) with device memory stores,
against the reference library itself (oracle/_ref) and the ports of
test_pac_sim.cpp / acceptance.cpp criteria 5-8.

Tolerance: the device sums in the reference's order with explicitly rounded
f64 ops, so states differ from libm's only through cos/tanh (<= 2 ulp per
call): rel 1e-12 on states; clocks, schedules, digests of untouched/agreeing
stores and recovered counts are exact."""
import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from paper_2308_14129_b200 import (DataError, MemoryStore, ModelParams, SyncStrategy, make_stream)

pytestmark = pytest.mark.gpu
TOL = 1e-12


def close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    return np.allclose(a, b, rtol=tol, atol=tol)


def test_model_params_seeded_bit_exact(ref):
    for d, seed in [(8, 3), (4, 1), (100, 21)]:
        mp = ModelParams.seeded(d, seed)
        w, om, g = ref.model_seeded(d, seed)
        assert mp.w_m.tobytes() == w.tobytes() and mp.omega.tobytes() == om.tobytes()
    a, c = ModelParams.seeded(8, 3), ModelParams.seeded(8, 4)
    assert not np.array_equal(a.w_m, c.w_m)
    assert (np.diff(a.omega) < 0).all()


def test_gamma_zero_and_clock():
    mp = ModelParams.seeded(4, 1)
    mp.gamma = 0.0
    mem = MemoryStore(3, 4)
    sp.model_update(mem, (0, 1, 5.0), mp)
    st, ts = mem.download()
    assert (st == 0).all() and ts.tolist() == [5.0, 5.0, 0.0]


@pytest.mark.parametrize("d,n,m,seed", [(8, 10, 20, 23), (4, 2, 1, 9), (100, 60, 400, 5)])
def test_replay_matches_reference(ref, d, n, m, seed):
    mp = ModelParams.seeded(d, 17)
    s = sp.gen_powerlaw(max(n, 2), m, 2.5, seed) if m > 1 else make_stream([(1, 1, 2.0)], 2)
    mem = MemoryStore(s.node_count, d)
    sp.model_update(mem, s.edges, mp)
    st, ts = mem.download()
    wst, wts = ref.model_update_run(np.zeros((s.node_count, d)), np.zeros(s.node_count), s.edges,
                                    mp.w_m, mp.omega, mp.gamma)
    assert np.array_equal(ts, wts)
    assert close(st, wst)


def test_stale_edges_rejected():
    mp = ModelParams.seeded(4, 1)
    mem = MemoryStore(3, 4)
    sp.model_update(mem, (0, 1, 5.0), mp)
    with pytest.raises(DataError) as ei:
        sp.model_update(mem, (1, 2, 3.0), mp)
    assert ei.value.code == "NonChronological"
    sp.model_update(mem, (0, 1, 5.0), mp)  # equal timestamps are fine


def test_lockstep_three_and_five():
    # test_pac_sim.cpp:277-319; acceptance.cpp criterion 6
    s = make_stream([(0, 1, 1), (2, 3, 2), (0, 1, 3), (2, 3, 4), (0, 1, 5), (2, 3, 6), (2, 3, 7),
                     (2, 3, 8)], 4)
    subs = sp.induce_subgraphs(s, [[0], [0], [1], [1]], 2)
    mp = ModelParams.seeded(4, 2)
    mems = [MemoryStore(4, 4), MemoryStore(4, 4)]
    log = sp.StepLog()
    er = sp.run_epoch(subs, mems, mp, [], SyncStrategy.MaxTimestamp, 1, log)
    assert er.batches == [3, 5] and er.loops == [1, 1]
    assert max(r[0] for r in log.steps) == 5
    w0 = [r for r in log.steps if r[1] == 0]
    assert [r[3] for r in w0] == [1, 2, 3, 1, 2] and [r[2] for r in w0] == [1, 1, 1, 2, 2]
    assert log.snapshots[0][0] == 0 and mems[0].digest() == log.snapshots[0][1]


def test_run_epoch_matches_reference(ref):
    s = sp.gen_powerlaw(80, 500, 2.4, 13)
    c = sp.compute_centrality(s, 0.5)
    pa = sp.partition_stream(s, sp.PartitionerConfig(3, 1.0, 1.0, sp.select_hubs(c, 0.1), c))
    subs = sp.induce_subgraphs(s, pa.node_parts, 3)
    mp = ModelParams.seeded(8, 77)
    for sync in (SyncStrategy.MaxTimestamp, SyncStrategy.Average):
        mems = [MemoryStore(s.node_count, 8) for _ in range(3)]
        er = sp.run_epoch(subs, mems, mp, pa.shared, sync, 16)
        r = ref.run_epoch([g.edges for g in subs], s.node_count, 8, np.zeros((3, s.node_count, 8)),
                          np.zeros((3, s.node_count)), mp.w_m, mp.omega, mp.gamma, pa.shared,
                          int(sync), 16)
        assert er.batches == r["batches"] and er.loops == r["loops"]
        assert er.sync_events == r["sync_events"]
        for w in range(3):
            st, ts = mems[w].download()
            assert np.array_equal(ts, r["last_ts"][w]) and close(st, r["states"][w])


def test_vacuous_worker_and_identical_subgraphs():
    s = make_stream([(0, 1, 1), (0, 1, 2)], 3)
    subs = sp.induce_subgraphs(s, [[0], [0], [1]], 2)
    mems = [MemoryStore(3, 4), MemoryStore(3, 4)]
    er = sp.run_epoch(subs, mems, ModelParams.seeded(4, 4), [], SyncStrategy.MaxTimestamp, 1)
    assert er.batches == [2, 0] and er.loops == [1, 1]
    assert mems[1].digest() == MemoryStore(3, 4).digest()
    s2 = sp.gen_powerlaw(15, 60, 2.5, 9)
    subs2 = sp.induce_subgraphs(s2, [[0, 1, 2]] * s2.node_count, 3)
    mems2 = [MemoryStore(s2.node_count, 8) for _ in range(3)]
    er2 = sp.run_epoch(subs2, mems2, ModelParams.seeded(8, 7), [], SyncStrategy.MaxTimestamp, 4)
    assert er2.digests[0] == er2.digests[1] == er2.digests[2]


def test_sync_semantics_and_idempotence(ref):
    rng = np.random.default_rng(2026)
    for W in (2, 3, 5, 6):
        st = rng.uniform(-2, 2, (W, 8, 4))
        ts = rng.uniform(0, 50, (W, 8))
        for strat in (SyncStrategy.MaxTimestamp, SyncStrategy.Average):
            mems = []
            for w in range(W):
                m = MemoryStore(8, 4)
                m.upload(st[w], ts[w])
                mems.append(m)
            sp.sync_shared(mems, [1, 3, 4, 7], strat)
            want_s, want_t = ref.sync_shared(st, ts, [1, 3, 4, 7], int(strat))
            got = [m.download() for m in mems]
            for w in range(W):
                assert np.array_equal(got[w][1], want_t[w])
                assert got[w][0].tobytes() == want_s[w].tobytes()  # sequential f64 sum: exact
            once = [m.digest() for m in mems]
            sp.sync_shared(mems, [1, 3, 4, 7], strat)
            assert [m.digest() for m in mems] == once


def test_max_ts_ties_lowest_worker():
    a, b = MemoryStore(2, 1), MemoryStore(2, 1)
    a.upload(np.array([[1.0], [0.0]]), np.array([5.0, 0.0]))
    b.upload(np.array([[2.0], [0.0]]), np.array([5.0, 0.0]))
    sp.sync_shared([a, b], [0], SyncStrategy.MaxTimestamp)
    assert a.state[0, 0] == 1.0 and b.state[0, 0] == 1.0


def test_simulate_sequential_equivalence(ref):
    # acceptance.cpp criterion 5 / test_pac_sim.cpp:425-445
    for seed in range(1, 8):
        s = sp.gen_powerlaw(5 + 11 * seed, 40 + 23 * seed, 2.2 + 0.04 * seed, 1000 + seed)
        c = sp.compute_centrality(s, 0.5)
        pa = sp.partition_stream(s, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.0), c))
        rep = sp.simulate(s, pa, sp.SimConfig(num_workers=1, batch_size=13, epochs=1, d=8,
                                              model_seed=500 + seed))
        mp = ModelParams.seeded(8, 500 + seed)
        wst, wts = ref.model_update_run(np.zeros((s.node_count, 8)), np.zeros(s.node_count), s.edges,
                                        mp.w_m, mp.omega, mp.gamma)
        # digest equality needs bit-equal cos/tanh; compare states through a fresh store
        m = MemoryStore(s.node_count, 8)
        sp.model_update(m, s.edges, mp)
        st, ts = m.download()
        assert np.array_equal(ts, wts) and close(st, wst)
        assert len(rep.epochs) == 1 and rep.epochs[0].loops == [1]


def test_shuffle_recovery_matches_reference(ref):
    s = sp.gen_powerlaw(120, 900, 2.3, 37)
    c = sp.compute_centrality(s, 0.5)
    pa = sp.partition_stream(s, sp.PartitionerConfig(8, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
    cfg = sp.SimConfig(num_workers=4, num_small_parts=8, shuffle=True, batch_size=32, epochs=20,
                       model_seed=3, shuffle_seed=100)
    rep = sp.simulate(s, pa, cfg)
    r = ref.simulate(s.edges, s.node_count, s.t_max, 8, pa.node_parts, pa.shared, num_workers=4,
                     num_small_parts=8, shuffle=True, batch=32, epochs=20, model_seed=3,
                     shuffle_seed=100)
    assert [e.recovered for e in rep.epochs] == [e["recovered"] for e in r["epochs"]]
    assert any(e.recovered for e in rep.epochs)
    assert [e.loops for e in rep.epochs] == [e["loops"] for e in r["epochs"]]
    assert rep.sync_events == r["sync_events"]


def test_simulate_validation():
    s = sp.gen_powerlaw(20, 100, 2.5, 1)
    c = sp.compute_centrality(s, 0.5)
    pa = sp.partition_stream(s, sp.PartitionerConfig(1, 1.0, 1.0, sp.select_hubs(c, 0.0), c))
    assert sp.simulate(s, pa, sp.SimConfig(num_workers=1, epochs=0)).epochs == []
    with pytest.raises(DataError):
        sp.simulate(s, pa, sp.SimConfig(num_workers=2))
    with pytest.raises(DataError):
        sp.simulate(s, pa, sp.SimConfig(num_workers=3, num_small_parts=8, shuffle=True))
