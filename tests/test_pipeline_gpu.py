"""run_parallel on one B200 (pqlg_pipeline): the Actor / V-learner /
P-learner threads with counter gating, device data channels and latest-wins
snapshots.  Checks the SPEC.md invariants (:481-484, :486-492): no data loss
(every batch consumed exactly once by each learner, no sequence gaps or
duplicates), pacing near beta_av = 1/8 and beta_pv = 1/2, policy staleness
within one publish interval, snapshots flowing both ways, finite losses."""
import ctypes as C

import pytest

from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu


def run_pipeline(cfg, dims, rc, steps, seconds=60.0, seed=3):
    h = C.c_void_p()
    _lib.call("pqlg_pipeline_create", C.byref(cfg), C.byref(dims), C.byref(rc), seed, C.byref(h))
    rep = _lib.RunReport()
    try:
        _lib.call("pqlg_pipeline_run", h, steps, seconds, C.byref(rep))
    finally:
        _lib.call("pqlg_pipeline_destroy", h)
    return rep


@pytest.mark.parametrize("algo", [_lib.ALGO_DDPG, _lib.ALGO_C51, _lib.ALGO_SAC])
def test_pipeline_invariants(algo):
    cfg = _lib.default_config(algo=algo, n_envs=256, batch_size=512, buffer_capacity=100_000,
                              hidden=64, hidden_layers=2, seed=1)
    dims = _lib.TaskDims(17, 6, -1.0, 1.0)
    rc = _lib.ratio_config()
    steps = 400
    r = run_pipeline(cfg, dims, rc, steps)
    print(f"\nc_a={r.c_a} c_v={r.c_v} c_p={r.c_p} ratios av={r.ratio_av:.4f} pv={r.ratio_pv:.4f} "
          f"sent={r.batches_sent} consumed v/p={r.batches_consumed_v}/{r.batches_consumed_p} "
          f"versions pol/crit={r.policy_version}/{r.critic_version} stale={r.max_policy_staleness} "
          f"losses {r.last_critic_loss:.4f} {r.last_actor_loss:.4f} wall {r.wall_s:.2f}s")
    assert r.ok == 1
    assert r.c_a >= steps and r.env_steps == r.c_a * 256
    # no data loss: every batch reached both learners exactly once, in order
    assert r.batches_sent * rc.horizon == r.c_a
    assert r.batches_consumed_v == r.batches_sent and r.batches_consumed_p == r.batches_sent
    assert r.seq_gaps == 0 and r.seq_duplicates == 0
    # pacing (gating after warm-up, slack of one horizon / one update)
    assert abs(r.ratio_av - 1 / 8) <= 0.2 / 8
    assert abs(r.ratio_pv - 1 / 2) <= 0.1
    # snapshots flowed both ways; staleness bound
    assert r.policy_version >= 1 and r.critic_version >= 1
    assert r.max_policy_staleness <= 1
    assert abs(r.last_critic_loss) < 1e6 and abs(r.last_actor_loss) < 1e6


def test_pipeline_free_running_actor_only_pacing_off():
    cfg = _lib.default_config(n_envs=1024, batch_size=512, buffer_capacity=200_000, hidden=64,
                              hidden_layers=2)
    dims = _lib.TaskDims(17, 6, -1.0, 1.0)
    rc = _lib.ratio_config(free_running=1)
    r = run_pipeline(cfg, dims, rc, 200)
    assert r.ok == 1 and r.c_a >= 200
    assert r.batches_consumed_v == r.batches_sent and r.seq_gaps == 0


def read_csv(path):
    lines = path.read_text().splitlines()
    assert lines[0] == _lib.lib().pqlg_metrics_header().decode()
    rows = [ln.split(",") for ln in lines[1:]]
    return [[float(x) for x in r] for r in rows]


def test_pipeline_metrics_csv(tmp_path):
    """a well-formed metrics CSV with a strictly increasing
    wall clock; env_steps = c_a * N; counters monotone; the last row is the
    run's final state."""
    N = 256
    cfg = _lib.default_config(n_envs=N, batch_size=512, buffer_capacity=100_000, hidden=64,
                              hidden_layers=2, seed=1, max_episode_len=50)
    dims = _lib.TaskDims(17, 6, -1.0, 1.0)
    rc = _lib.ratio_config()
    path = tmp_path / "metrics.csv"
    m = _lib.metrics_config(str(path), interval_s=0.25, eval_episodes=16)
    h = C.c_void_p()
    _lib.call("pqlg_pipeline_create", C.byref(cfg), C.byref(dims), C.byref(rc), 3, C.byref(h))
    _lib.call("pqlg_pipeline_set_metrics", h, C.byref(m))
    rep = _lib.RunReport()
    try:
        _lib.call("pqlg_pipeline_run", h, 100_000, 2.0, C.byref(rep))
    finally:
        _lib.call("pqlg_pipeline_destroy", h)
    rows = read_csv(path)
    print(f"\n{len(rows)} rows; last {rows[-1]}")
    assert len(rows) >= 3
    for a, b in zip(rows, rows[1:]):
        assert b[0] > a[0]                                   # wall clock strictly increasing
        assert all(b[k] >= a[k] for k in (1, 2, 3, 4))       # counters monotone
    for r in rows:
        assert r[1] == r[2] * N                               # env_steps = c_a * N
        assert r[5] == r[5] and r[6] >= 0.0                   # finite eval, stderr >= 0
    last = rows[-1]
    assert (last[2], last[3], last[4]) == (rep.c_a, rep.c_v, rep.c_p)
    assert last[7] != 0.0 and last[8] != 0.0                  # both loss EMAs sampled


@pytest.mark.parametrize("algo", [_lib.ALGO_DDPG, _lib.ALGO_SAC])
def test_run_synchronous_deterministic_and_paced(tmp_path, algo):
    """one sequential loop in Algorithm order; fixed seed ->
    identical metrics (all columns but the wall clock) and identical final
    losses; update counts follow the ratios exactly."""
    N = 128
    cfg = _lib.default_config(algo=algo, n_envs=N, batch_size=256, buffer_capacity=50_000,
                              hidden=64, hidden_layers=2, seed=5, max_episode_len=40)
    dims = _lib.TaskDims(11, 4, -1.0, 1.0)
    rc = _lib.ratio_config()
    outs = []
    for k in range(2):
        path = tmp_path / f"sync{k}.csv"
        m = _lib.metrics_config(str(path), every_actor_steps=40, eval_episodes=8)
        rep = _lib.RunReport()
        _lib.call("pqlg_run_synchronous", C.byref(cfg), C.byref(dims), C.byref(rc), 9, 200,
                  C.byref(m), C.byref(rep))
        outs.append((rep, read_csv(path)))
    (r0, m0), (r1, m1) = outs
    print(f"\nc_a={r0.c_a} c_v={r0.c_v} c_p={r0.c_p} losses {r0.last_critic_loss} "
          f"{r0.last_actor_loss} rows {len(m0)}")
    assert (r0.c_a, r0.c_v, r0.c_p) == (r1.c_a, r1.c_v, r1.c_p)
    assert r0.last_critic_loss == r1.last_critic_loss
    assert r0.last_actor_loss == r1.last_actor_loss
    assert [r[1:] for r in m0] == [r[1:] for r in m1]
    # pacing: every post-warm-up iteration runs H / beta_av critic updates
    # and policy updates up to beta_pv * c_v
    H = rc.horizon
    iters = r0.c_a // H
    assert r0.c_a == 200
    warm = max(-(-rc.warm_up // H), -(-cfg.batch_size // N)) - 1
    assert r0.c_v == (iters - warm) * round(H / rc.beta_av)
    assert r0.c_p == int(rc.beta_pv * r0.c_v)
    assert r0.policy_version == r0.c_p // rc.publish_every
    assert r0.critic_version == r0.c_v // rc.publish_every


def test_pipeline_nonfinite_update_aborts_the_run():
    """SPEC.md:461 (child fault -> propagate): a critic update that turns
    non-finite stops every thread and run() reports PQLG_ENONFINITE."""
    cfg = _lib.default_config(n_envs=128, batch_size=256, buffer_capacity=50_000, hidden=32,
                              hidden_layers=2, seed=2, lr_critic=1e30, lr_actor=1e30)
    dims = _lib.TaskDims(9, 3, -1.0, 1.0)
    rc = _lib.ratio_config()
    with pytest.raises(_lib.NonFinite):
        run_pipeline(cfg, dims, rc, 2000, seconds=30.0)


def test_run_synchronous_nonfinite_update_raises():
    cfg = _lib.default_config(n_envs=128, batch_size=256, buffer_capacity=50_000, hidden=32,
                              hidden_layers=2, seed=2, lr_critic=1e30, lr_actor=1e30)
    dims = _lib.TaskDims(9, 3, -1.0, 1.0)
    rc = _lib.ratio_config()
    rep = _lib.RunReport()
    with pytest.raises(_lib.NonFinite):
        _lib.call("pqlg_run_synchronous", C.byref(cfg), C.byref(dims), C.byref(rc), 1, 400, None,
                  C.byref(rep))


def test_pipeline_time_budget_shutdown_joins_promptly():
    """SPEC.md:464 (deterministic shutdown): a run stopped by its wall-clock
    budget joins all threads within 5 s and still consumed every batch."""
    import time
    cfg = _lib.default_config(n_envs=512, batch_size=512, buffer_capacity=200_000, hidden=64,
                              hidden_layers=2, seed=3)
    dims = _lib.TaskDims(17, 6, -1.0, 1.0)
    rc = _lib.ratio_config()
    t0 = time.perf_counter()
    r = run_pipeline(cfg, dims, rc, 10**9, seconds=1.0)
    dt = time.perf_counter() - t0
    print(f"\nstopped after {r.wall_s:.2f}s (call {dt:.2f}s), c_a={r.c_a}")
    assert r.ok == 1 and r.wall_s < 5.0
    assert r.batches_consumed_v == r.batches_sent == r.batches_consumed_p


@pytest.mark.parametrize("free_running,publish_every", [(1, 8), (0, 3), (0, 1)])
def test_pipeline_p_learner_critics_are_a_published_snapshot(free_running, publish_every):
    """The P-learner's critic replicas at the end of a run are exactly the
    snapshot the V-learner published under the version the P-learner holds
    (learners.cpp:222-227), also when actor iterations carry no new critic
    snapshot (free running, other publish intervals): a slot reused from an
    earlier iteration must not hand its stale buffer on as current."""
    cfg = _lib.default_config(n_envs=256, batch_size=256, buffer_capacity=100_000, hidden=32,
                              hidden_layers=2, seed=5)
    dims = _lib.TaskDims(9, 3, -1.0, 1.0)
    rc = _lib.ratio_config(free_running=free_running, publish_every=publish_every)
    h = C.c_void_p()
    _lib.call("pqlg_pipeline_create", C.byref(cfg), C.byref(dims), C.byref(rc), 7, C.byref(h))
    try:
        _lib.call("pqlg_pipeline_record_snapshots", h, 1)
        rep = _lib.RunReport()
        _lib.call("pqlg_pipeline_run", h, 600, 60.0, C.byref(rep))
        ver, diff = C.c_int64(), C.c_double()
        _lib.call("pqlg_pipeline_check_critics", h, C.byref(ver), C.byref(diff))
    finally:
        _lib.call("pqlg_pipeline_destroy", h)
    print(f"\nfree={free_running} K_pub={publish_every}: critic versions published "
          f"{rep.critic_version}, P-learner holds {ver.value}, max|diff| {diff.value}")
    assert rep.ok == 1 and rep.critic_version >= 1
    # every actor iteration after the first publish forwards a batch; most
    # of them carry no new snapshot (the stale-slot case) when free running
    if free_running:
        assert rep.batches_sent > rep.critic_version
    assert ver.value >= 1
    assert diff.value == 0.0
