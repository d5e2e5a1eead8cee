"""Data-parallel critic / policy updates (config 5) on CPU with
world_size 2 over gloo.

The GPU path (pqlg_vlearner_create_dp) computes, on every rank, the local
gradient of its B rows with dLoss/dQ scaled by 1/(B*world), all-reduces
(sum) the gradients and the loss, then clips per critic on the full-batch
norm and applies Adam + Polyak identically on every rank.  These tests run
that exact composition with the oracle restatement as the per-rank compute
and gloo as the exchange, and check it against the single-process oracle
update on the concatenated batch -- the parity statement of SURVEY 8(e) --
plus the NCCL unique-id exchange the benchmark uses to build the
communicator.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle_lib import orc, param_count, ptr, sizes_arr
from oracle_model import adam, f32


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_problem(D=13, A=4, H=32, nh=2, B=64, seed=0):
    rng = np.random.default_rng(seed)
    qs = [D + A] + [H] * nh + [1]
    ps = [D] + [H] * nh + [A]
    q1 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    q2 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    pol = f32(rng.standard_normal(param_count(ps)) * 0.2)
    Bg = 2 * B
    rows = dict(obs=f32(rng.standard_normal((Bg, D))), act=f32(rng.uniform(-1, 1, (Bg, A))),
                boot=f32(rng.standard_normal((Bg, D))), ret=f32(rng.standard_normal(Bg) * 0.1),
                eff=f32(np.full(Bg, 0.970299)))
    return dict(D=D, A=A, qs=qs, ps=ps, q1=q1, q2=q2, pol=pol, rows=rows, L=nh + 1)


def critic_grads(pb, lo, hi):
    """orc_ddpg_critic_loss on rows [lo, hi) (ddpg.hpp:24-76)."""
    r = {k: np.ascontiguousarray(v[lo:hi]) for k, v in pb["rows"].items()}
    n = hi - lo
    P = param_count(pb["qs"])
    dq = [np.zeros(P, np.float32), np.zeros(P, np.float32)]
    loss = np.zeros(1, np.float32)
    y = np.zeros(n, np.float32)
    rc = orc().orc_ddpg_critic_loss(
        ptr(pb["pol"]), ptr(sizes_arr(pb["ps"])), ptr(pb["q1"]), ptr(pb["q2"]), ptr(pb["q1"]),
        ptr(pb["q2"]), ptr(sizes_arr(pb["qs"])), pb["L"], ptr(r["obs"]), ptr(r["act"]),
        ptr(r["boot"]), ptr(r["ret"]), ptr(r["eff"]), n, pb["D"], pb["A"], np.float32(-1),
        np.float32(1), ptr(loss), ptr(y), ptr(dq[0]), ptr(dq[1]))
    assert rc == 0
    return float(loss[0]), dq


def apply_update(pb, dq, lr=5e-4, tau=0.05):
    """clip_global_norm per critic -> Adam -> soft_update (learners.cpp:182-187)."""
    P = param_count(pb["qs"])
    out = []
    for k, q in enumerate((pb["q1"], pb["q2"])):
        g = dq[k].copy()
        orc().orc_clip_global_norm(ptr(g), P, np.float32(0.5))
        p = q.copy()
        m = np.zeros(P, np.float32)
        v = np.zeros(P, np.float32)
        adam(p, g, m, v, 1, lr)
        t = q.copy()
        orc().orc_lerp_towards(ptr(t), ptr(p), P, np.float32(tau))
        out += [p, t]
    return out


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # (1) the NCCL unique-id exchange of the benchmark's communicator setup
        from paper_2307_12983_b200 import _lib
        ident = _lib.exchange_comm_id(rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, ident)
        # (2) the data-parallel critic update with the oracle as the per-rank compute
        pb = make_problem()
        B = pb["rows"]["ret"].shape[0] // world
        loss, dq = critic_grads(pb, rank * B, (rank + 1) * B)
        # local upstream 2e/B -> 2e/(B*world): scale by 1/world (exact for world 2)
        buf = torch.from_numpy(np.concatenate([dq[0], dq[1], [loss]]).astype(np.float32)
                               * np.float32(1.0 / world))
        dist.all_reduce(buf)
        P = param_count(pb["qs"])
        g = buf.numpy()
        upd = apply_update(pb, [g[:P].copy(), g[P:2 * P].copy()])
        q.put((rank, ids, float(g[-1]), g[:2 * P].copy(), [u.copy() for u in upd]))
    finally:
        dist.destroy_process_group()


def test_dp_critic_update_matches_single_process_on_concatenated_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the unique id reached every rank intact
    assert res[0][1][0] == res[0][1][1] and len(res[0][1][0]) == 128
    # every rank holds the same all-reduced gradient and applies the same update
    assert np.array_equal(res[0][3], res[1][3])
    for a, b in zip(res[0][4], res[1][4]):
        assert np.array_equal(a, b)
    # == the single-process update on the concatenated batch (reduction-order tolerance)
    pb = make_problem()
    Bg = pb["rows"]["ret"].shape[0]
    loss, dq = critic_grads(pb, 0, Bg)
    P = param_count(pb["qs"])
    full = np.concatenate([dq[0], dq[1]])
    assert abs(res[0][2] - loss) <= 1e-5 * abs(loss)
    assert np.linalg.norm(res[0][3] - full) <= 1e-5 * np.linalg.norm(full)
    want = apply_update(pb, dq)
    for got, w in zip(res[0][4], want):
        assert np.max(np.abs(got - w)) <= 1e-6 + 1e-5 * np.max(np.abs(w))


def _norm_worker(rank, world, port, q):
    """A sharded actor's normalizer step (pqlg_actor_create_sharded): the
    shard's batch (mean, M2, n), an all-gather, the rank-order combination
    and the merge into the running stats -- on every rank."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        D, n, steps = 17, 40, 3
        count = np.array([500.0])
        mean = rng.standard_normal(D) * 0.5
        m2 = np.abs(rng.standard_normal(D)) * 500.0
        for t in range(steps):
            rows = f32(rng.standard_normal((world * n, D)) * 2.0 + 3.0)  # same on every rank
            mine = np.ascontiguousarray(rows[rank * n:(rank + 1) * n])
            bm, b2 = np.zeros(D), np.zeros(D)
            orc().orc_norm_batch_stats(ptr(mine), n, D, ptr(bm), ptr(b2))
            rec = torch.from_numpy(np.concatenate([bm, b2, [float(n)]]))
            recs = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(recs, rec)
            g = [r.numpy() for r in recs]
            # combine shards in rank order, then merge into the running stats
            cn = np.array([g[0][2 * D]])
            cm, c2 = g[0][:D].copy(), g[0][D:2 * D].copy()
            for k in range(1, world):
                orc().orc_norm_merge(ptr(cn), ptr(cm), ptr(c2), D, g[k][2 * D],
                                     ptr(np.ascontiguousarray(g[k][:D])),
                                     ptr(np.ascontiguousarray(g[k][D:2 * D])))
            orc().orc_norm_merge(ptr(count), ptr(mean), ptr(m2), D, cn[0], ptr(cm), ptr(c2))
        q.put((rank, float(count[0]), mean.copy(), m2.copy()))
    finally:
        dist.destroy_process_group()


def test_sharded_normalizer_merge_matches_single_normalizer():
    """the shards' merged running stats equal RunningNormalizer
    on the concatenated batches (fp64 rounding, 1e-12 rel) and are
    identical on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_norm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][2], res[1][2]) and np.array_equal(res[0][3], res[1][3])
    rng = np.random.default_rng(3)
    D, n, steps = 17, 40, 3
    count = np.array([500], np.int64)
    mean = rng.standard_normal(D) * 0.5
    m2 = np.abs(rng.standard_normal(D)) * 500.0
    for t in range(steps):
        rows = f32(rng.standard_normal((world * n, D)) * 2.0 + 3.0)
        orc().orc_norm_update(ptr(count), ptr(mean), ptr(m2), ptr(rows), world * n, D)
    assert res[0][1] == float(count[0])
    np.testing.assert_allclose(res[0][2], mean, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(res[0][3], m2, rtol=1e-12)
