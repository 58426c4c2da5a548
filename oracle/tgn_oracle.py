"""TEST INFRASTRUCTURE ONLY — CPU oracle for the TGN training step.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, as the checker; the product path never imports it.

PARITY UNPINNED BY THE REFERENCE: the reference (speedpart) contains no TGN —
its model is the fixed surrogate of pac_sim.cpp:50-104 and SPEC.md:13 puts
gradient-based learning out of scope. This module is the builder-authored
restatement of the TGN data flow the paper describes (PAPER.md:301-315,
SURVEY.md Appendix A), in plain torch fp32 with autograd supplying the
backward (an independent check of the hand-written CUDA backward). Choices
that the paper leaves open are fixed here once, and the CUDA path follows them:

  * time encoding (TGAT): phi(dt) = cos(w*dt + b), w_i =
    10^(-9 i/(T-1)), b = 0, both learnable; the phase w*dt + b is formed in
    f64 (dt reaches 1.9e8 > 2^24 at GDELT shape), cos in f64,
    result rounded to f32.
  * memory: identity message [s_i || s_j || e_ij || phi(t - t_i^-)],
    last-message aggregation (max (ts, stream index)), GRUCell
    updater. Pending messages of batch b-1 are applied at the start of batch b
    (with gradient into the GRU); message inputs are detached.
  * embedding: one temporal-attention layer over the k
    most recent neighbours strictly before t in the partition's training
    events (both directions, ties by (ts, event, src-side first)); query
    [s_root || phi(0)], keys/values [s_nbr || e || phi(t - t_nbr)], H heads,
    output projection; a root with no neighbour gets a zero attention output;
    MergeLayer [attn || s_root] -> relu -> d.
  * decoder: MergeLayer [z_u || z_v] -> relu -> 1; loss =
    mean BCE(pos) + mean BCE(neg), one negative per positive drawn uniformly
    from the partition's destination nodes with a counter-based hash.
  * optimiser: Adam, gradients averaged over all workers every global step.
  * PAC schedule (pac_sim.cpp:205-264): memory reset at
    every loop start, loop-end flush + snapshot, epoch-end restore + shared
    node sync (average default, max-ts optional).
  * backbone = 1, JODIE (one of the paper's other backbones; as
    TGN's reference implementation configures it): the same messages and
    last-message aggregation, an RNN memory updater h' = tanh(W_ih m + b_ih +
    W_hh h + b_hh), and the time-projection embedding
    emb = s'(t) * (1 + log1p(t - t_last) w_tp + b_tp) (t_last = the clock after
    this batch's memory update; log1p keeps raw timestamp gaps of up to 1e8 in
    range where JODIE normalises them by dataset statistics); no attention or
    merge layers; the same decoder and loss.
  * backbone = 2, DyRep (the TGN framework's DyRep row: RNN
    memory updater, identity embedding, attention message function): the
    same RNN updater as JODIE; the decoder reads the roots' (updated) memory
    rows directly (identity embedding); the message of endpoint i of event
    (i, j) is [s_i || z_j || e_ij || phi(t - t_i^-)] where z_j is j's
    temporal-attention embedding (the TGN attention layer + MergeLayer above,
    over the updated memory) at the event's batch, stored with the pending
    message. Message inputs are detached (as for every backbone), so the
    attention parameters carry no gradient; they shape the messages only.
"""
from __future__ import annotations

import bisect
import math
from dataclasses import dataclass

import numpy as np
import torch

M64 = (1 << 64) - 1

# The oracle must be reproducible bit for bit run to run (CPU index_put
# accumulation is otherwise thread-order dependent).
torch.use_deterministic_algorithms(True, warn_only=True)


# ------------------------------------------------------------- hashing
def mix(x: int) -> int:
    """SplitMix64 finalizer (shared bit-for-bit with csrc/tgn_common.cuh)."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def key3(seed, a, b):
    return mix(mix(mix(seed) ^ a) ^ b)


def edge_features(seed: int, eids: np.ndarray, F: int) -> np.ndarray:
    """BF16-exact U[-1,1) features: ((h >> 56) - 128) / 128."""
    if F == 0:
        return np.zeros((len(eids), 0), np.float32)
    e = np.asarray(eids, np.uint64)[:, None]
    c = np.arange(F, dtype=np.uint64)[None, :]
    s = np.uint64(mix(seed))
    h = mix_np(mix_np(s ^ e) ^ c)
    k = (h >> np.uint64(56)).astype(np.int64) - 128
    return (k.astype(np.float32) / np.float32(128.0))


def negatives(seed: int, epoch: int, worker: int, step: int, n: int, pool: np.ndarray) -> np.ndarray:
    """Counter-hash uniform draw from the destination pool (csrc: tgn_neg)."""
    base = mix(mix(mix(mix(seed) ^ epoch) ^ worker) ^ step)
    i = np.arange(n, dtype=np.uint64)
    h = mix_np(np.uint64(base) ^ i)
    return pool[(h % np.uint64(len(pool))).astype(np.int64)]


# ------------------------------------------------------------- params
@dataclass
class TGNConfig:
    d_mem: int = 100
    d_time: int = 100
    d_edge: int = 172
    n_neighbors: int = 10
    n_heads: int = 2
    batch_size: int = 200
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    seed_init: int = 3
    seed_feat: int = 2
    seed_neg: int = 4
    sync_average: int = 1
    backbone: int = 0  # 0 TGN, 1 JODIE, 2 DyRep


def ld_aug(k: int) -> int:
    """Row stride of an augmented [W | b | 0-pad] matrix: whole 128-B lines."""
    return (k + 1 + 31) // 32 * 32


def linear_specs(c: TGNConfig):
    """Linear layers (name, N out, K in, init fan_in) in flat-buffer order
    (csrc/tgn_trainer.cu ParamLayout::build). Each is stored as an augmented
    [W | b | 0-pad] matrix of row stride ld_aug(K)."""
    D, T, F = c.d_mem, c.d_time, c.d_edge
    DQ, DK, DM = D + T, D + F + T, 2 * D + F + T
    g = c.backbone == 0  # GRU (TGN) or one RNN gate block (JODIE, DyRep)
    t = c.backbone != 1  # attention + merge rows (TGN, DyRep's message embedding)
    j = c.backbone == 1  # JODIE's time projection
    return [("gru_ih", 3 * D if g else D, DM, D), ("gru_hh", 3 * D if g else D, D, D),
            ("att_q", DQ if t else 0, DQ, DQ), ("att_kv", 2 * DQ if t else 0, DK, DK),
            ("att_o", DQ if t else 0, DQ, DQ), ("mrg1", D if t else 0, DQ + D, DQ + D),
            ("mrg2", D if t else 0, D, D), ("dec1", D, 2 * D, 2 * D), ("dec2", 1, D, D),
            ("tproj", D if j else 0, 1, D)]


def param_layout(c: TGNConfig):
    """{name: (offset, N, K, ld)} for linears, time_w/time_b offsets, total floats."""
    off = 0
    lay = {}
    T = c.d_time
    lay["time_w"] = (off, T)
    off += (T + 3) // 4 * 4
    lay["time_b"] = (off, T)
    off += (T + 3) // 4 * 4
    for name, N, K, fan in linear_specs(c):
        ld = ld_aug(K)
        lay[name] = (off, N, K, ld)
        off += N * ld
    return lay, off


def init_params(c: TGNConfig) -> np.ndarray:
    lay, total = param_layout(c)
    flat = np.zeros(total, np.float32)
    T = c.d_time
    i = np.arange(T, dtype=np.float64)
    w = 10.0 ** (-9.0 * i / (T - 1)) if T > 1 else np.ones(1)
    o = lay["time_w"][0]
    flat[o:o + T] = w.astype(np.float32)
    s = np.uint64(mix(c.seed_init))
    for t, (name, N, K, fan) in enumerate(linear_specs(c)):
        off, _, _, ld = lay[name]
        a = 1.0 / math.sqrt(fan)

        def draw(tag, n):
            h = mix_np(mix_np(s ^ np.uint64(tag)) ^ np.arange(n, dtype=np.uint64))
            u = (h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)
            return ((2.0 * u - 1.0) * a).astype(np.float32)
        m = flat[off:off + N * ld].reshape(N, ld)
        m[:, :K] = draw(t, N * K).reshape(N, K)
        m[:, K] = draw(t + 100, N)
    return flat


# --------------------------------------------------------- partition data
class WorkerData:
    """One partition's training events in local ids (the device's layout)."""

    def __init__(self, nodes_global: np.ndarray, edges: np.ndarray, eids: np.ndarray, F: int,
                 seed_feat: int):
        self.nodes = np.asarray(nodes_global, np.uint32)
        self.loc = {int(g): i for i, g in enumerate(self.nodes)}
        self.N = len(self.nodes)
        self.src = np.array([self.loc[int(x)] for x in edges["src"]], np.int64)
        self.dst = np.array([self.loc[int(x)] for x in edges["dst"]], np.int64)
        self.ts = np.asarray(edges["ts"], np.float64)
        self.eids = np.asarray(eids, np.uint64)
        self.E = len(self.ts)
        self.feat = torch.from_numpy(edge_features(seed_feat, self.eids, F))
        self.pool = np.unique(self.dst).astype(np.int64) if self.E else np.zeros(1, np.int64)
        # adjacency: per node entries (ts, event, role, nbr) ascending
        adj = [[] for _ in range(self.N)]
        for k in range(self.E):
            adj[self.src[k]].append((self.ts[k], k, 0, int(self.dst[k])))
            adj[self.dst[k]].append((self.ts[k], k, 1, int(self.src[k])))
        for a in adj:
            a.sort()
        self.adj = adj
        self.adj_ts = [[x[0] for x in a] for a in adj]

    def neighbors(self, node: int, t: float, k: int):
        pos = bisect.bisect_left(self.adj_ts[node], t)
        return self.adj[node][max(0, pos - k):pos]


# ------------------------------------------------------------- model
def time_enc(w: torch.Tensor, b: torch.Tensor, dt: np.ndarray) -> torch.Tensor:
    """cos(w*dt + b): phase in f64, rounded to f32, differentiable in w, b."""
    dt64 = torch.from_numpy(np.asarray(dt, np.float64))[:, None]
    ph = w.double()[None, :] * dt64 + b.double()[None, :]
    return torch.cos(ph).float()


class TGNOracle:
    def __init__(self, cfg: TGNConfig, workers: list[WorkerData], shared_global=(), params=None):
        self.c = cfg
        self.W = workers
        self.lay, self.total = param_layout(cfg)
        flat = init_params(cfg) if params is None else np.asarray(params, np.float32).copy()
        self.flat = torch.from_numpy(flat)
        self.m = torch.zeros(self.total)
        self.v = torch.zeros(self.total)
        self.t = 0
        self.shared = list(shared_global)
        D = cfg.d_mem
        self.mem = [torch.zeros(w.N, D) for w in workers]
        self.lu = [np.zeros(w.N) for w in workers]
        self.pend = [dict() for _ in workers]
        self.pos = [0] * len(workers)
        self.snap = [None] * len(workers)
        self.last = {}

    def rebind(self, workers: list[WorkerData]):
        """Shuffle-combine (pac_sim.cpp:280-329): the next epoch's regrouped
        workers; parameters and Adam state carry over, per-worker state restarts."""
        if len(workers) != len(self.W):
            raise ValueError("rebind needs the same number of workers")
        D = self.c.d_mem
        self.W = workers
        self.mem = [torch.zeros(w.N, D) for w in workers]
        self.lu = [np.zeros(w.N) for w in workers]
        self.pend = [dict() for _ in workers]
        self.pos = [0] * len(workers)
        self.snap = [None] * len(workers)
        self.last = {}

    # views into a differentiable copy of the flat params
    def views(self, flat: torch.Tensor):
        c = self.c
        lay = self.lay
        P = {}
        o, T = lay["time_w"]
        P["time_w"] = flat[o:o + T]
        o, T = lay["time_b"]
        P["time_b"] = flat[o:o + T]

        def lin(name):
            off, N, K, ld = lay[name]
            m = flat[off:off + N * ld].view(N, ld)
            return m[:, :K], m[:, K]
        P["gru_w_ih"], P["gru_b_ih"] = lin("gru_ih")
        P["gru_w_hh"], P["gru_b_hh"] = lin("gru_hh")
        P["att_w_q"], P["att_b_q"] = lin("att_q")
        wkv, bkv = lin("att_kv")
        DQ = c.d_mem + c.d_time
        P["att_w_k"], P["att_w_v"] = wkv[:DQ], wkv[DQ:]
        P["att_b_k"], P["att_b_v"] = bkv[:DQ], bkv[DQ:]
        P["att_w_o"], P["att_b_o"] = lin("att_o")
        P["mrg_w1"], P["mrg_b1"] = lin("mrg1")
        P["mrg_w2"], P["mrg_b2"] = lin("mrg2")
        P["dec_w1"], P["dec_b1"] = lin("dec1")
        P["dec_w2"], P["dec_b2"] = lin("dec2")
        tw, tb = lin("tproj")
        P["tp_w"], P["tp_b"] = tw[:, 0], tb
        return P

    def _gru(self, P, x, h):
        gi = x @ P["gru_w_ih"].T + P["gru_b_ih"]
        gh = h @ P["gru_w_hh"].T + P["gru_b_hh"]
        if self.c.backbone != 0:  # JODIE, DyRep: RNN cell
            return torch.tanh(gi + gh)
        D = self.c.d_mem
        r = torch.sigmoid(gi[:, :D] + gh[:, :D])
        z = torch.sigmoid(gi[:, D:2 * D] + gh[:, D:2 * D])
        n = torch.tanh(gi[:, 2 * D:] + r * gh[:, 2 * D:])
        return (1 - z) * n + z * h

    def _messages(self, w, P, U, data=None):
        wd = self.W[w] if data is None else data
        mem = self.mem[w]
        pend = self.pend[w]
        other = [pend[u][0] for u in U]
        ev = [pend[u][1] for u in U]
        ts = np.array([pend[u][2] for u in U])
        with torch.no_grad():
            phi = time_enc(P["time_w"], P["time_b"], ts - self.lu[w][U])
        if self.c.backbone == 2:  # DyRep: the other endpoint's attention embedding
            zo = torch.stack([pend[u][3] for u in U]) if len(U) else torch.zeros(0, self.c.d_mem)
        else:
            zo = mem[other]
        x = torch.cat([mem[U], zo, wd.feat[ev], phi], 1).detach()
        return x, mem[U].detach(), ts

    def _embed_jodie(self, w, P, memx, roots, t_roots, upd):
        """JODIE time projection of the roots' (updated) memory."""
        lu = self.lu[w].copy()
        U, mts = upd
        if len(U):
            lu[U] = mts
        s = torch.from_numpy(np.log1p(np.maximum(0.0, np.asarray(t_roots, np.float64) - lu[roots]))).float()
        emb = memx[roots] * (1 + s[:, None] * P["tp_w"] + P["tp_b"])
        R = len(roots)
        return emb, np.full((R, self.c.n_neighbors), -1, np.int64), np.zeros(R, np.int64)

    def _embed(self, w, P, memx, roots, t_roots, data=None, upd=None):
        if self.c.backbone == 1:
            return self._embed_jodie(w, P, memx, roots, t_roots, upd)
        if self.c.backbone == 2:  # DyRep: identity embedding
            R = len(roots)
            return memx[roots], np.full((R, self.c.n_neighbors), -1, np.int64), np.zeros(R, np.int64)
        return self._embed_attn(w, P, memx, roots, t_roots, data)

    def _msg_embed(self, w, P, memx, src, dst, ts, data=None):
        """DyRep: attention embeddings of the batch's sources then destinations
        (no gradient), the payload of the messages stored after the batch."""
        if self.c.backbone != 2:
            return None
        with torch.no_grad():
            z, _, _ = self._embed_attn(w, P, memx.detach(), np.concatenate([src, dst]),
                                       np.concatenate([ts, ts]), data)
        return z

    def _embed_attn(self, w, P, memx, roots, t_roots, data=None):
        c, wd = self.c, (self.W[w] if data is None else data)
        D, T, K, H = c.d_mem, c.d_time, c.n_neighbors, c.n_heads
        R = len(roots)
        nb_node = np.zeros((R, K), np.int64)
        nb_ev = np.zeros((R, K), np.int64)
        nb_dt = np.zeros((R, K), np.float64)
        cnt = np.zeros(R, np.int64)
        ids = np.full((R, K), -1, np.int64)
        for i, (r, t) in enumerate(zip(roots, t_roots)):
            nb = wd.neighbors(int(r), float(t), K)
            cnt[i] = len(nb)
            for j, (ts_, ev, _role, n) in enumerate(nb):
                nb_node[i, j], nb_ev[i, j], nb_dt[i, j] = n, ev, t - ts_
                ids[i, j] = n
        phi0 = torch.cos(P["time_b"].double()).float()
        q_in = torch.cat([memx[roots], phi0.expand(R, T)], 1)
        Q = q_in @ P["att_w_q"].T + P["att_b_q"]
        # key/value input [s_nbr | phi(dt) | e]: the differentiable columns first
        kv_in = torch.cat([memx[nb_node.reshape(-1)],
                           time_enc(P["time_w"], P["time_b"], nb_dt.reshape(-1)),
                           wd.feat[nb_ev.reshape(-1)]], 1)
        Kt = (kv_in @ P["att_w_k"].T + P["att_b_k"]).view(R, K, -1)
        Vt = (kv_in @ P["att_w_v"].T + P["att_b_v"]).view(R, K, -1)
        DQ = D + T
        dh = DQ // H
        mask = torch.from_numpy(np.arange(K)[None, :] < cnt[:, None])
        outs = []
        for h in range(H):
            q = Q[:, h * dh:(h + 1) * dh]
            k = Kt[:, :, h * dh:(h + 1) * dh]
            v = Vt[:, :, h * dh:(h + 1) * dh]
            s = (k @ q[:, :, None]).squeeze(2) / math.sqrt(dh)
            s = s.masked_fill(~mask, float("-inf"))
            s = torch.where(mask.any(1, keepdim=True), s, torch.zeros_like(s))
            a = torch.softmax(s, 1)
            outs.append((a[:, :, None] * v).sum(1))
        ctx = torch.cat(outs, 1)
        attn = ctx @ P["att_w_o"].T + P["att_b_o"]
        attn = torch.where(torch.from_numpy(cnt > 0)[:, None], attn, torch.zeros_like(attn))
        z1 = torch.relu(torch.cat([attn, memx[roots]], 1) @ P["mrg_w1"].T + P["mrg_b1"])
        emb = z1 @ P["mrg_w2"].T + P["mrg_b2"]
        return emb, ids, cnt

    def _decode(self, P, a, b):
        d1 = torch.relu(torch.cat([a, b], 1) @ P["dec_w1"].T + P["dec_b1"])
        return (d1 @ P["dec_w2"].T + P["dec_b2"]).squeeze(1)

    def _flush(self, w, P):
        """Apply pending messages without gradient (loop end / eval)."""
        U = np.array(sorted(self.pend[w].keys()), np.int64)
        if len(U) == 0:
            return
        with torch.no_grad():
            x, h, ts = self._messages(w, P, U)
            self.mem[w][U] = self._gru(P, x, h)
        self.lu[w][U] = ts
        self.pend[w] = {}

    def _store_pending(self, w, src, dst, ts, ev, z=None):
        pend = {}
        B = len(src)
        for k in range(B):  # later events overwrite: last-message wins
            zs = None if z is None else z[B + k]  # the source's message carries z_dst
            zd = None if z is None else z[k]
            pend[int(src[k])] = (int(dst[k]), int(ev[k]), float(ts[k]), zs)
            pend[int(dst[k])] = (int(src[k]), int(ev[k]), float(ts[k]), zd)
        self.pend[w] = pend

    def batches(self, w):
        return (self.W[w].E + self.c.batch_size - 1) // self.c.batch_size

    def epoch_steps(self):
        return max([self.batches(w) for w in range(len(self.W))] + [0])

    def begin_epoch(self, epoch):
        self.epoch = epoch
        self.step_in_epoch = 0
        self.pos = [0] * len(self.W)
        self.done = [self.batches(w) == 0 for w in range(len(self.W))]
        for w in range(len(self.W)):
            if self.batches(w) == 0:
                self.snap[w] = (self.mem[w].clone(), self.lu[w].copy())

    def seek(self, step):
        """Position the schedule at global step `step` of the current epoch
        with memory, clocks and pending messages cleared (the trainer's
        spd_tgn_seek: a timed region starts mid-epoch from a reset state)."""
        if step >= self.epoch_steps():
            raise ValueError("seek past the end of the epoch")
        self.step_in_epoch = step
        for w in range(len(self.W)):
            nb = self.batches(w)
            if nb == 0:
                continue
            self.pos[w] = step % nb
            self.done[w] = step // nb > 0
            self.mem[w].zero_()
            self.lu[w][:] = 0
            self.pend[w] = {}

    def step(self):
        """One lockstep global step over all workers; returns per-worker loss."""
        c = self.c
        self.step_in_epoch += 1
        flat = self.flat.clone().requires_grad_(True)
        P = self.views(flat)
        grads = torch.zeros(self.total)
        losses = []
        n_active = 0
        for w, wd in enumerate(self.W):
            if self.batches(w) == 0:
                losses.append(float("nan"))
                continue
            if self.pos[w] == 0:  # loop_start reset
                self.mem[w].zero_()
                self.lu[w][:] = 0
                self.pend[w] = {}
            lo = self.pos[w] * c.batch_size
            hi = min(wd.E, lo + c.batch_size)
            src, dst, ts = wd.src[lo:hi], wd.dst[lo:hi], wd.ts[lo:hi]
            B = hi - lo
            neg = negatives(c.seed_neg, self.epoch, w, self.step_in_epoch, B, wd.pool)
            U = np.array(sorted(self.pend[w].keys()), np.int64)
            memx = self.mem[w].clone()
            if len(U):
                x, h, mts = self._messages(w, P, U)
                hn = self._gru(P, x, h)
                memx = memx.index_put((torch.from_numpy(U),), hn)
            roots = np.concatenate([src, dst, neg])
            emb, ids, cnt = self._embed(w, P, memx, roots, np.concatenate([ts, ts, ts]),
                                        upd=(U, mts if len(U) else None))
            zmsg = self._msg_embed(w, P, memx, src, dst, ts)
            pos_l = self._decode(P, emb[:B], emb[B:2 * B])
            neg_l = self._decode(P, emb[:B], emb[2 * B:])
            loss = torch.nn.functional.softplus(-pos_l).mean() + torch.nn.functional.softplus(neg_l).mean()
            g, = torch.autograd.grad(loss, flat, allow_unused=True)
            if g is None:
                g = torch.zeros(self.total)
            grads += g
            n_active += 1
            losses.append(float(loss.detach()))
            self.last[w] = dict(emb=emb.detach().numpy(), neg=neg, nbr_ids=ids, cnt=cnt,
                                loss=float(loss.detach()), U=U, memx=memx.detach().numpy(),
                                post=(U, hn.detach() if len(U) else None,
                                      mts if len(U) else None, src, dst, ts, lo, hi),
                                zmsg=zmsg)
        # gradient mean over ALL workers (an idle worker contributes zeros)
        self.grad = grads / len(self.W)
        self._adam(self.grad)
        P_new = self.views(self.flat)
        for w, wd in enumerate(self.W):
            if self.batches(w) == 0:
                continue
            U, hn, mts, src, dst, ts, lo, hi = self.last[w]["post"]
            with torch.no_grad():  # persist the memory update, store new messages
                if len(U):
                    self.mem[w][U] = hn
                    self.lu[w][U] = mts
            self._store_pending(w, src, dst, ts, np.arange(lo, hi), self.last[w]["zmsg"])
            self.pos[w] += 1
            if self.pos[w] == self.batches(w):  # loop_end: flush (new params), snapshot
                self._flush(w, P_new)
                self.snap[w] = (self.mem[w].clone(), self.lu[w].copy())
                self.done[w] = True
                self.pos[w] = 0
        return losses

    def _adam(self, g):
        c = self.c
        self.t += 1
        self.m = c.beta1 * self.m + (1 - c.beta1) * g
        self.v = c.beta2 * self.v + (1 - c.beta2) * g * g
        bc1 = 1 - c.beta1 ** self.t
        bc2 = 1 - c.beta2 ** self.t
        mh = self.m / bc1
        vh = self.v / bc2
        self.flat = self.flat - c.lr * mh / (torch.sqrt(vh) + c.adam_eps)

    def end_epoch(self):
        for w in range(len(self.W)):
            self.mem[w], self.lu[w] = self.snap[w][0].clone(), self.snap[w][1].copy()
            self.pend[w] = {}
        if len(self.W) >= 2 and self.shared:
            self._sync()

    def _sync(self):
        """pac_sim.cpp:162-203 on the local rows of each shared node."""
        for g in self.shared:
            rows = [wd.loc.get(int(g)) for wd in self.W]
            if any(r is None for r in rows):
                continue
            vals = [self.mem[w][r] for w, r in enumerate(rows)]
            tss = [self.lu[w][r] for w, r in enumerate(rows)]
            if self.c.sync_average:
                if all(torch.equal(v, vals[0]) for v in vals) and all(t == tss[0] for t in tss):
                    continue
                mean = torch.zeros_like(vals[0])
                for v in vals:
                    mean = mean + v
                mean = mean / len(vals)
                ts = max(tss)
            else:
                best = max(range(len(vals)), key=lambda w: (tss[w], -w))
                mean, ts = vals[best].clone(), tss[best]
            for w, r in enumerate(rows):
                self.mem[w][r] = mean
                self.lu[w][r] = ts

    def run_epoch(self, epoch):
        self.begin_epoch(epoch)
        losses = []
        for _ in range(self.epoch_steps()):
            losses.append(self.step())
        self.end_epoch()
        return losses

    # --------------------------------------------------------- evaluation
    def set_eval(self, w, edges_global, eids):
        """Routed val then test edges of worker w appended after its training
        events: the evaluation view (full-graph neighbours, features, pool)."""
        wd = self.W[w]
        tr = np.zeros(wd.E, dtype=edges_global.dtype)
        tr["src"], tr["dst"], tr["ts"] = wd.nodes[wd.src], wd.nodes[wd.dst], wd.ts
        comb = np.concatenate([tr, np.asarray(edges_global)])
        ids = np.concatenate([wd.eids, np.asarray(eids, np.uint64)])
        if not hasattr(self, "X"):
            self.X = {}
        self.X[w] = WorkerData(wd.nodes, comb, ids, self.c.d_edge, self.c.seed_feat)

    def evaluate(self, w, lo, hi, neg_seed=5):
        """TGN evaluation over eval events [lo, hi): per batch apply pending
        messages, embed src/dst/negative, score, persist, store messages."""
        X, E, B = self.X[w], self.W[w].E, self.c.batch_size
        P = self.views(self.flat)
        pos, neg = [], []
        with torch.no_grad():
            for b0 in range(lo, hi, B):
                b1 = min(hi, b0 + B)
                k0, n = E + b0, b1 - b0
                src, dst, ts = X.src[k0:k0 + n], X.dst[k0:k0 + n], X.ts[k0:k0 + n]
                ng = negatives(neg_seed, 0xE7A1, w, b0, n, X.pool)
                U = np.array(sorted(self.pend[w].keys()), np.int64)
                memx = self.mem[w].clone()
                if len(U):
                    x, h, mts = self._messages(w, P, U, X)
                    hn = self._gru(P, x, h)
                    memx[U] = hn
                emb, _, _ = self._embed(w, P, memx, np.concatenate([src, dst, ng]),
                                        np.concatenate([ts, ts, ts]), X, upd=(U, mts if len(U) else None))
                zmsg = self._msg_embed(w, P, memx, src, dst, ts, X)
                pos.append(self._decode(P, emb[:n], emb[n:2 * n]).numpy())
                neg.append(self._decode(P, emb[:n], emb[2 * n:]).numpy())
                if len(U):
                    self.mem[w][U] = hn
                    self.lu[w][U] = mts
                self._store_pending(w, src, dst, ts, np.arange(k0, k0 + n), zmsg)
        return np.concatenate(pos), np.concatenate(neg)
