"""Bridge between the reference oracle and the TGN trainer:
with the reference's surrogate MSG/UPD plugged into the TGN trainer's memory-
update slot (spd_tgn_set_surrogate) and batch size 1, one epoch of the TGN
trainer's own schedule — loop-start reset, pending last messages (K3),
loop-end flush + snapshot, epoch-end restore and shared-hub sync — must
reproduce the UNMODIFIED reference run_epoch (oracle/_ref,
pac_sim.cpp:205-264; sync_shared :162-203) on the same SEP subgraphs.

This pins the trainer's schedule machinery to the reference itself (the TGN
oracle is builder-authored). Bars: last-update clocks bit-exact; states to
1e-5 absolute (the trainer stores memory in f32, the reference in f64; the
surrogate's arithmetic is f64 with the reference's operation order)."""
import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from oracle import ref as R
from tests.tgn_cases import partitioned

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


def _run_bridge(subs, shared, parts, mp, average, epochs):
    cfg = sp.TGNConfig(d_mem=mp.d, d_time=4, d_edge=0, n_neighbors=1, n_heads=1, batch_size=1,
                       sync_average=average, gemm_mode=0)
    tr = sp.TGNTrainer(cfg, subs, shared=shared)
    tr.set_surrogate(mp)
    for e in range(epochs):
        tr.begin_epoch(e)
        steps = tr.epoch_steps()
        for _ in range(steps):
            tr.step(want_loss=False)
        tr.end_epoch()
    out = [(tr.local_nodes(w), *tr.memory(w)) for w in range(parts)]
    tr.close()
    return steps, out


@pytest.mark.parametrize("parts,average", [(2, 1), (2, 0), (3, 1), (3, 0)])
def test_surrogate_in_tgn_schedule_matches_reference_run_epoch(ref, parts, average):
    s, _, pa, subs = partitioned(nodes=200, edges=2400, parts=parts, k=0.1, seed=7)
    assert len(pa.shared) > 0
    n = int(s.node_count)
    mp = sp.ModelParams.seeded(8, 77)
    steps, got = _run_bridge(subs, pa.shared, parts, mp, average, epochs=1)
    r = ref.run_epoch([g.edges for g in subs], n, mp.d, np.zeros((parts, n, mp.d)),
                      np.zeros((parts, n)), mp.w_m, mp.omega, mp.gamma, pa.shared, average, 1)
    assert steps == max(r["batches"])
    for w in range(parts):
        nodes, mem, lu = got[w]
        np.testing.assert_array_equal(lu, r["last_ts"][w][nodes])
        err = np.abs(mem.astype(np.float64) - r["states"][w][nodes]).max()
        assert err <= 1e-5, (w, err)
        # rows the worker does not hold stay at the reference's reset state
        others = np.setdiff1d(np.arange(n), nodes)
        assert not np.any(r["states"][w][others]) and not np.any(r["last_ts"][w][others])
