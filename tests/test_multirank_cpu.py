"""N>1 host logic on CPU with a world_size-2 gloo group (127.0.0.1):
every rank derives the same SEP assignment, the same lockstep schedule
(so the per-step gradient all-reduce lines up without a collective), a disjoint
partition -> rank map, and the same NCCL unique id after the broadcast. The
schedule is also pinned to the reference's StepLog (oracle/_ref run_epoch)."""
import os
import socket

import numpy as np
import pytest

import paper_2308_14129_b200 as sp

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return int.from_bytes(h.digest()[:7], "little")


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = sp.gen_powerlaw(600, 12000, 2.4, 5)
    tr = sp.chrono_split(s, 0.7, 0.15).train
    c = sp.compute_centrality(tr, 0.5)
    pa = sp.partition_stream(tr, sp.PartitionerConfig(world, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
    subs = sp.induce_subgraphs(tr, pa.node_parts, world)
    steps, rows, batches, loops = sp.lockstep_schedule(subs, 100)
    mine = len(subs[rank].edges)
    local = torch.tensor([_digest(pa.edge_part, pa.shared, pa.np_parts), steps, mine,
                          _digest(np.array(rows, np.uint64))], dtype=torch.int64)
    gathered = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(gathered, local)
    nid = sp.nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(nid), dtype=torch.uint8)
    dist.broadcast(t, 0)
    ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(ids, t)
    if rank == 0:
        out.put(([g.tolist() for g in gathered], [bytes(i.tolist()) for i in ids],
                 sum(len(g.edges) for g in subs), batches))
    dist.destroy_process_group()


def test_two_ranks_agree_on_partition_schedule_and_nccl_id():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered, ids, total_edges, batches = res
    assert gathered[0][0] == gathered[1][0]          # identical SEP assignment
    assert gathered[0][1] == gathered[1][1]          # identical lockstep length
    assert gathered[0][3] == gathered[1][3]          # identical step log
    assert gathered[0][2] + gathered[1][2] == total_edges  # disjoint partition -> rank map
    assert gathered[0][1] == max(batches)
    assert ids[0] == ids[1] and any(ids[0])


def test_schedule_matches_reference_steplog(ref):
    s = sp.make_stream([(0, 1, 1), (2, 3, 2), (0, 1, 3), (2, 3, 4), (0, 1, 5), (2, 3, 6), (2, 3, 7),
                        (2, 3, 8)], 4)
    subs = sp.induce_subgraphs(s, [[0], [0], [1], [1]], 2)
    steps, rows, batches, loops = sp.lockstep_schedule(subs, 1)
    w, om, g = ref.model_seeded(4, 2)
    r = ref.run_epoch([x.edges for x in subs], 4, 4, np.zeros((2, 4, 4)), np.zeros((2, 4)), w, om, g,
                      [], 0, 1, log=True)
    assert rows == r["steps"] and batches == r["batches"] and loops == r["loops"] and steps == 5
    # random partitions, several batch sizes, a vacuous worker
    big = sp.gen_powerlaw(200, 3000, 2.3, 3)
    c = sp.compute_centrality(big, 0.5)
    pa = sp.partition_stream(big, sp.PartitionerConfig(5, 1.0, 1.0, sp.select_hubs(c, 0.05), c))
    subs = sp.induce_subgraphs(big, pa.node_parts, 5) + [sp.SubGraph(np.zeros(0, np.uint32),
                                                                      np.zeros(0, sp.EDGE_DTYPE),
                                                                      np.zeros(0, np.uint64))]
    for B in (7, 64, 500):
        steps, rows, batches, loops = sp.lockstep_schedule(subs, B)
        r = ref.run_epoch([x.edges for x in subs], big.node_count, 2,
                          np.zeros((6, big.node_count, 2)), np.zeros((6, big.node_count)),
                          *ref.model_seeded(2, 1), [], 0, B, log=True)
        assert rows == r["steps"] and batches == r["batches"] and loops == r["loops"]
