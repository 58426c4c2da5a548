"""Shared fixtures for TGN parity tests: a seeded synthetic TIG, SEP-partitioned
through the product host path, and the matching CPU oracle workers."""
from __future__ import annotations

import numpy as np

import paper_2308_14129_b200 as sp


def partitioned(nodes=300, edges=4000, parts=2, k=0.05, seed=1, f_train=0.7):
    s = sp.gen_powerlaw(nodes, edges, 2.5, seed)
    split = sp.chrono_split(s, f_train, 0.15)
    tr = split.train
    c = sp.compute_centrality(tr, 0.5)
    cfg = sp.PartitionerConfig(parts, 1.0, 1.0, sp.select_hubs(c, k), c)
    pa = sp.partition_stream(tr, cfg)
    subs = sp.induce_subgraphs(tr, pa.node_parts, parts)
    return s, split, pa, subs


def oracle_for(cfg: sp.TGNConfig, subs, shared):
    from oracle import tgn_oracle as T
    oc = T.TGNConfig(d_mem=cfg.d_mem, d_time=cfg.d_time, d_edge=cfg.d_edge,
                     n_neighbors=cfg.n_neighbors, n_heads=cfg.n_heads, batch_size=cfg.batch_size,
                     lr=cfg.lr, beta1=cfg.beta1, beta2=cfg.beta2, adam_eps=cfg.adam_eps,
                     seed_init=cfg.seed_init, seed_feat=cfg.seed_feat, seed_neg=cfg.seed_neg,
                     sync_average=cfg.sync_average, backbone=cfg.backbone)
    ws = [T.WorkerData(g.nodes, g.edges, g.eids, oc.d_edge, oc.seed_feat) for g in subs]
    return T.TGNOracle(oc, ws, list(shared))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
