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
