"""run_parallel pacing rule on CPU: pqlg_ratio_may_proceed (the library's
RatioGate::may_proceed) against the compiled reference's own
sched::RatioGate::may_proceed (ratio_gate.hpp:44-60, ref_ratio_may_proceed
in oracle/ref_harness.cpp) and a transcription of it, over a grid of
counters and ratio settings, plus the SPEC.md pacing examples.  Pure host
logic: no GPU needed."""
import itertools

import pytest

from oracle_lib import ref

from paper_2307_12983_b200 import _lib


def ref_may_proceed(p, ca, cv, cp, c):
    # ratio_gate.hpp:44-60
    if c.free_running:
        return True
    if ca < c.warm_up:
        return True
    if p == _lib.PROC_ACTOR:
        return ca + 1.0 <= c.beta_av * cv + c.slack_a
    if p == _lib.PROC_PLEARNER:
        return cp + 1.0 <= c.beta_pv * cv + c.slack_p
    return cv + 1.0 <= ca / c.beta_av + c.slack_v


def test_defaults_match_ratio_config_and_spec():
    rc = _lib.ratio_config()
    assert (rc.beta_av, rc.beta_pv) == (1 / 8, 1 / 2)
    assert (rc.slack_a, rc.slack_p, rc.slack_v, rc.warm_up) == (4.0, 1.0, 1.0, 32)
    assert (rc.horizon, rc.channel_capacity, rc.publish_every) == (4, 8, 8)


def test_may_proceed_matches_reference_rule_on_a_grid():
    for free in (0, 1):
        rc = _lib.ratio_config(free_running=free)
        for p, ca, cv, cp in itertools.product(range(3), (0, 31, 32, 33, 40, 64, 100),
                                               range(0, 600, 23), range(0, 300, 17)):
            got = _lib.lib().pqlg_ratio_may_proceed(p, ca, cv, cp, rc)
            assert got == int(ref_may_proceed(p, ca, cv, cp, rc)), (free, p, ca, cv, cp)


def test_may_proceed_matches_compiled_ratio_gate():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    n = 0
    for free, beta_av, beta_pv, slack_a, warm in itertools.product(
            (0, 1), (1 / 8, 1 / 4, 1.0, 3.0), (1 / 2, 1.0, 0.25), (4.0, 0.0, 2.5), (32, 0, 7)):
        rc = _lib.ratio_config(free_running=free, beta_av=beta_av, beta_pv=beta_pv,
                               slack_a=slack_a, warm_up=warm)
        for p, ca, cv, cp in itertools.product(range(3), (0, 6, 7, 31, 32, 33, 64, 101),
                                               range(0, 420, 37), range(0, 220, 29)):
            want = R.ref_ratio_may_proceed(p, ca, cv, cp, rc.beta_av, rc.beta_pv, rc.slack_a,
                                           rc.slack_p, rc.slack_v, rc.warm_up, rc.free_running)
            assert _lib.lib().pqlg_ratio_may_proceed(p, ca, cv, cp, rc) == want, \
                (free, beta_av, beta_pv, slack_a, warm, p, ca, cv, cp)
            n += 1
    assert n > 100_000


def test_pacing_examples():
    rc = _lib.ratio_config()
    f = _lib.lib().pqlg_ratio_may_proceed
    # warm-up: everything proceeds before 32 rollout steps
    assert f(_lib.PROC_ACTOR, 31, 0, 0, rc) == 1
    # after warm-up the actor waits for 8 critic updates per step (+ one horizon of slack)
    assert f(_lib.PROC_ACTOR, 40, 288, 0, rc) == 0
    assert f(_lib.PROC_ACTOR, 40, 296, 0, rc) == 1
    # the V-learner must not outrun the data: c_v + 1 <= 8 c_a + 1
    assert f(_lib.PROC_VLEARNER, 40, 320, 0, rc) == 1
    assert f(_lib.PROC_VLEARNER, 40, 321, 0, rc) == 0
    # the P-learner runs at half the critic rate
    assert f(_lib.PROC_PLEARNER, 40, 100, 50, rc) == 1
    assert f(_lib.PROC_PLEARNER, 40, 100, 51, rc) == 0
    assert f(5, 0, 0, 0, rc) == -1
