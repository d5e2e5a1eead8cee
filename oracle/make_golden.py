"""Generates tests/golden/*.npz from the compiled reference (oracle/_ref).

Run here (the build container, where /root/reference exists):
    make -C oracle ref && python oracle/make_golden.py
The fixtures pin the CPU restatement (tests/test_oracle_cpu.py) and, through
it, the GPU path; they travel with the repo because /root/reference does not
exist on the GPU box.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import acts_arr, param_count, ptr, ref, sizes_arr, traj_hash  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def episodes(rng, T, N, D, A, p_term=0.05, p_trunc=0.05):
    obs = f32(rng.standard_normal((T, N, D)))
    act = f32(rng.uniform(-1, 1, (T, N, A)))
    boot = f32(rng.standard_normal((T, N, D)))
    rew = f32(rng.standard_normal((T, N)))
    u = rng.uniform(size=(T, N))
    term = (u < p_term).astype(np.uint8)
    trunc = ((u >= p_term) & (u < p_term + p_trunc)).astype(np.uint8)
    return obs, act, boot, rew, term, trunc


def gen_indices(R, out):
    cases = [(0, 1, 100, 8, 1), (0, 1, 100, 64, 3), (7, 2, 5_000_000, 256, 2),
             (3, 1, 1, 16, 1), (11, 1, 3, 64, 2), (5, 1, (1 << 33) + 12345, 64, 1)]
    for k, (seed, learner, count, B, n) in enumerate(cases):
        if count > 20_000_000:
            continue  # ref_sample_indices materialises `count` rows
        idx = np.zeros(B * n, dtype=np.uint64)
        R.ref_sample_indices(seed, learner, count, B, n, ptr(idx))
        out[f"idx{k}"] = idx
        out[f"idx{k}_args"] = np.array([seed, learner, count, B, n], dtype=np.uint64)
    draws = np.zeros(1000, dtype=np.uint64)
    R.ref_mt64_draws(R.ref_derive_seed(0, 4, 1), 1000, ptr(draws))
    out["mt64_draws"] = draws


def gen_nstep(R, out):
    rng = np.random.default_rng(1)
    for k, (T, N, D, A, n, cap) in enumerate([(40, 6, 5, 3, 3, 50), (30, 9, 4, 2, 1, 1000),
                                              (25, 4, 3, 2, 4, 7)]):
        obs, act, boot, rew, term, trunc = episodes(rng, T, N, D, A, 0.08, 0.08)
        maxr = T * N * n
        counts = np.zeros(T, dtype=np.uint64)
        eo, ea, eb = (np.zeros((maxr, D), np.float32), np.zeros((maxr, A), np.float32),
                      np.zeros((maxr, D), np.float32))
        er, ee = np.zeros(maxr, np.float32), np.zeros(maxr, np.float32)
        ro, rr = np.zeros((cap, D), np.float32), np.zeros(cap, np.float32)
        cc = np.zeros(2, np.uint64)
        total = R.ref_nstep_replay(T, N, D, A, np.float32(0.99), n, cap, ptr(obs), ptr(act),
                                   ptr(boot), ptr(rew), ptr(term), ptr(trunc), ptr(counts),
                                   ptr(eo), ptr(ea), ptr(eb), ptr(er), ptr(ee), maxr, ptr(ro),
                                   ptr(rr), ptr(cc))
        for name, v in dict(obs=obs, act=act, boot=boot, rew=rew, term=term, trunc=trunc,
                            counts=counts, e_obs=eo[:total], e_act=ea[:total],
                            e_boot=eb[:total], e_ret=er[:total], e_eff=ee[:total],
                            ring_obs=ro, ring_ret=rr, cursor_count=cc,
                            args=np.array([T, N, D, A, n, cap])).items():
            out[f"c{k}_{name}"] = v


def gen_elementwise(R, out):
    rng = np.random.default_rng(2)
    n = 4099
    p = f32(rng.standard_normal(n)); g = f32(rng.standard_normal(n) * 0.1)
    m = f32(rng.standard_normal(n) * 0.01); v = f32(np.abs(rng.standard_normal(n)) * 1e-3)
    out.update(adam_p=p.copy(), adam_g=g.copy(), adam_m=m.copy(), adam_v=v.copy())
    for t in (0, 1, 9, 99):
        pp, mm, vv = p.copy(), m.copy(), v.copy()
        R.ref_adam_step(ptr(pp), ptr(g), ptr(mm), ptr(vv), n, t, np.float32(5e-4))
        out[f"adam_t{t}"] = np.stack([pp, mm, vv])
    for scale in (0.01, 1.0, 30.0):
        gg = f32(g * scale)
        R.ref_clip_global_norm(ptr(gg), n, np.float32(0.5))
        out[f"clip_{scale}"] = gg
    out["sumsq"] = np.array([R.ref_sum_squares(ptr(g), n)])
    t = f32(rng.standard_normal(n))
    tt = t.copy()
    R.ref_soft_update(ptr(tt), ptr(p), n, np.float32(0.05))
    out.update(lerp_t=t, lerp_out=tt)
    for N in (1, 2, 4, 7, 4096):
        s = np.zeros(N, np.float32)
        R.ref_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(s))
        out[f"sched_{N}"] = s


def gen_norm(R, out):
    rng = np.random.default_rng(3)
    D = 11
    rows = np.array([1, 7, 64, 3], dtype=np.uintp)
    data = f32(rng.standard_normal((int(rows.sum()), D)) * 3 + 1)
    x = f32(rng.standard_normal((50, D)) * 20)
    x[0, 0] = np.nan
    cnt = np.zeros(1, np.int64); mean = np.zeros(D); m2 = np.zeros(D)
    xn = np.zeros_like(x)
    R.ref_normalizer(D, len(rows), ptr(rows), ptr(data), ptr(cnt), ptr(mean), ptr(m2), ptr(x),
                     50, ptr(xn))
    out.update(norm_rows=rows, norm_data=data, norm_x=x, norm_count=cnt, norm_mean=mean,
               norm_m2=m2, norm_xn=xn)


def gen_noise(R, out):
    rng = np.random.default_rng(4)
    for N, A, steps in ((64, 8, 3), (33, 20, 2), (5, 1, 4)):
        a = f32(rng.uniform(-1, 1, (steps, N, A)))
        a0 = a.copy()
        R.ref_apply_noise(np.float32(0.05), np.float32(0.8), N, A, 0, steps, np.float32(-1),
                          np.float32(1), ptr(a))
        out[f"noise_{N}_{A}_in"] = a0
        out[f"noise_{N}_{A}_out"] = a


def gen_mlp(R, out):
    rng = np.random.default_rng(5)
    sizes = [13, 32, 24, 5]
    L = len(sizes) - 1
    sa = sizes_arr(sizes)
    P = param_count(sizes)
    flat = f32(rng.standard_normal(P) * 0.3)
    B = 17
    x = f32(rng.standard_normal((B, sizes[0])))
    y = np.zeros((B, sizes[-1]), np.float32)
    R.ref_mlp_forward(ptr(flat), ptr(sa), L, ptr(x), B, ptr(y))
    up = f32(rng.standard_normal((B, sizes[-1])))
    gr = np.zeros(P, np.float32)
    din = np.zeros((B, sizes[0]), np.float32)
    R.ref_mlp_backward(ptr(flat), ptr(sa), L, ptr(x), ptr(up), B, ptr(gr), ptr(din))
    out.update(mlp_sizes=np.array(sizes), mlp_flat=flat, mlp_x=x, mlp_y=y, mlp_up=up,
               mlp_grads=gr, mlp_din=din)
    # orthogonal init, policy (learners.cpp:17-33) and critic pair (critic.hpp:16-26)
    pol = np.zeros(param_count([6, 16, 16, 3]), np.float32)
    R.ref_policy_init(6, 3, 16, 0, ptr(pol))
    out["init_policy"] = pol
    qs = sizes_arr([9, 16, 16, 1])
    q = np.zeros(2 * param_count([9, 16, 16, 1]), np.float32)
    R.ref_init_mlp(ptr(qs), 3, 12345, np.float32(np.sqrt(2.0)), np.float32(1.0), 2, ptr(q))
    out["init_critics"] = q
    # same at a GEMM-friendly width (32) for the device learners' init check
    pol = np.zeros(param_count([6, 32, 32, 3]), np.float32)
    R.ref_policy_init(6, 3, 32, 0, ptr(pol))
    out["init_policy_h32"] = pol
    qs = sizes_arr([9, 32, 32, 1])
    q = np.zeros(2 * param_count([9, 32, 32, 1]), np.float32)
    R.ref_init_mlp(ptr(qs), 3, 12345, np.float32(np.sqrt(2.0)), np.float32(1.0), 2, ptr(q))
    out["init_critics_h32"] = q


def small_nets(rng, D, A, H, L, out_dim=1):
    ps = [D] + [H] * (L - 1) + [A]
    qs = [D + A] + [H] * (L - 1) + [out_dim]
    pol = f32(rng.standard_normal(param_count(ps)) * 0.3)
    qn = [f32(rng.standard_normal(param_count(qs)) * 0.3) for _ in range(4)]
    return ps, qs, pol, qn


def gen_agents(R, out):
    rng = np.random.default_rng(6)
    D, A, H, L, B = 7, 3, 16, 3, 24
    ps, qs, pol, (q1, q2, q1t, q2t) = small_nets(rng, D, A, H, L)
    obs = f32(rng.standard_normal((B, D))); act = f32(rng.uniform(-1, 1, (B, A)))
    boot = f32(rng.standard_normal((B, D))); ret = f32(rng.standard_normal(B))
    eff = f32(np.where(rng.uniform(size=B) < 0.2, 0, 0.970299))
    loss = np.zeros(1, np.float32); y = np.zeros(B, np.float32)
    P = param_count(qs)
    dq1 = np.zeros(P, np.float32); dq2 = np.zeros(P, np.float32)
    R.ref_ddpg_critic_loss(ptr(pol), ptr(sizes_arr(ps)), ptr(q1), ptr(q2), ptr(q1t), ptr(q2t),
                           ptr(sizes_arr(qs)), L, ptr(obs), ptr(act), ptr(boot), ptr(ret),
                           ptr(eff), B, D, A, np.float32(-1), np.float32(1), ptr(loss), ptr(y),
                           ptr(dq1), ptr(dq2))
    aloss = np.zeros(1, np.float32); dpol = np.zeros(param_count(ps), np.float32)
    R.ref_ddpg_actor_loss(ptr(pol), ptr(sizes_arr(ps)), ptr(q1), ptr(q2), ptr(sizes_arr(qs)), L,
                          ptr(obs), B, D, np.float32(-1), np.float32(1), ptr(aloss), ptr(dpol))
    out.update(ag_dims=np.array([D, A, H, L, B]), ag_pol=pol, ag_q1=q1, ag_q2=q2, ag_q1t=q1t,
               ag_q2t=q2t, ag_obs=obs, ag_act=act, ag_boot=boot, ag_ret=ret, ag_eff=eff,
               ag_loss=loss.copy(), ag_y=y, ag_dq1=dq1, ag_dq2=dq2, ag_aloss=aloss.copy(),
               ag_dpol=dpol.copy())
    # C51
    La = 11
    ps, qs, pol, (q1, q2, q1t, q2t) = small_nets(rng, D, A, H, L, La)
    ret2 = f32(rng.standard_normal(B) * 2)
    P = param_count(qs)
    dq1 = np.zeros(P, np.float32); dq2 = np.zeros(P, np.float32)
    R.ref_c51_critic_loss(ptr(pol), ptr(sizes_arr(ps)), ptr(q1), ptr(q2), ptr(q1t), ptr(q2t),
                          ptr(sizes_arr(qs)), L, ptr(obs), ptr(act), ptr(boot), ptr(ret2),
                          ptr(eff), B, D, A, np.float32(-1), np.float32(1), La, np.float32(-10),
                          np.float32(10), ptr(loss), ptr(dq1), ptr(dq2))
    dpol = np.zeros(param_count(ps), np.float32)
    R.ref_c51_actor_loss(ptr(pol), ptr(sizes_arr(ps)), ptr(q1), ptr(q2), ptr(sizes_arr(qs)), L,
                         ptr(obs), B, D, np.float32(-1), np.float32(1), La, np.float32(-10),
                         np.float32(10), ptr(aloss), ptr(dpol))
    out.update(c51_pol=pol, c51_q1=q1, c51_q2=q2, c51_q1t=q1t, c51_q2t=q2t, c51_ret=ret2,
               c51_loss=loss.copy(), c51_dq1=dq1, c51_dq2=dq2, c51_aloss=aloss.copy(),
               c51_dpol=dpol, c51_L=np.array([La]))
    probs = rng.uniform(size=(40, La)).astype(np.float64)
    probs = f32(probs / probs.sum(1, keepdims=True))
    pret = f32(rng.standard_normal(40) * 4)
    peff = f32(rng.choice([0.0, 0.970299, 1.0, 0.5], 40))
    pret[0], peff[0] = 0.0, 1.0  # identity projection
    proj = np.zeros_like(probs)
    R.ref_c51_project(ptr(probs), ptr(pret), ptr(peff), 40, La, np.float32(-10), np.float32(10),
                      ptr(proj))
    out.update(proj_probs=probs, proj_ret=pret, proj_eff=peff, proj_out=proj)


def gen_vupdate(R, out):
    """k=3 successive V-learner updates (agents-level composition) and 3
    P-learner updates on a small config; used for the k-step weight check."""
    rng = np.random.default_rng(7)
    D, A, H, nh, B, cap = 9, 4, 32, 2, 48, 500
    ps = [D] + [H] * nh + [A]
    qs = [D + A] + [H] * nh + [1]
    pol = f32(rng.standard_normal(param_count(ps)) * 0.2)
    q1 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    q2 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    n_rows = 300
    obs = f32(rng.standard_normal((n_rows, D))); act = f32(rng.uniform(-1, 1, (n_rows, A)))
    boot = f32(rng.standard_normal((n_rows, D))); ret = f32(rng.standard_normal(n_rows) * 0.1)
    eff = f32(np.where(rng.uniform(size=n_rows) < 0.05, 0.0, 0.970299))
    cnt = 1000; mean = rng.standard_normal(D) * 0.1; m2 = np.abs(rng.standard_normal(D)) * cnt
    h = R.ref_vupdate_create(D, A, H, nh, B, cap, 0, ptr(q1), ptr(q2), ptr(pol), 0, 51,
                             np.float32(-10), np.float32(10))
    R.ref_vupdate_insert(h, ptr(obs), ptr(act), ptr(boot), ptr(ret), ptr(eff), n_rows)
    R.ref_vupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    losses = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_vupdate_step(h, ptr(l)) == 0
        losses[k] = l[0]
    P = param_count(qs)
    res = np.zeros((4, P), np.float32)
    for w in range(4):
        R.ref_vupdate_params(h, w, ptr(res[w]))
    R.ref_vupdate_destroy(h)
    out.update(vu_dims=np.array([D, A, H, nh, B, cap]), vu_pol=pol, vu_q1=q1, vu_q2=q2,
               vu_obs=obs, vu_act=act, vu_boot=boot, vu_ret=ret, vu_eff=eff,
               vu_norm=np.array([cnt]), vu_mean=mean, vu_m2=m2, vu_losses=losses, vu_params=res)
    h = R.ref_pupdate_create(D, A, H, nh, B, cap, 0, ptr(pol), ptr(q1), ptr(q2), 0, 51,
                             np.float32(-10), np.float32(10))
    R.ref_pupdate_insert(h, ptr(obs), n_rows)
    R.ref_pupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    pl = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_pupdate_step(h, ptr(l)) == 0
        pl[k] = l[0]
    pp = np.zeros(param_count(ps), np.float32)
    R.ref_pupdate_params(h, ptr(pp))
    R.ref_pupdate_destroy(h)
    out.update(pu_losses=pl, pu_params=pp)


def gen_c51update(R, out):
    """k=3 successive PQL-D (C51) V-learner updates and 3 P-learner updates
    (c51_critic_loss / c51_actor_loss compositions, learners.cpp:157-188,
    :239-270) with 51 atoms on [-10, 10]."""
    rng = np.random.default_rng(8)
    D, A, H, nh, B, cap, L = 9, 4, 32, 2, 48, 500, 51
    ps = [D] + [H] * nh + [A]
    qs = [D + A] + [H] * nh + [L]
    pol = f32(rng.standard_normal(param_count(ps)) * 0.2)
    q1 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    q2 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    n_rows = 300
    obs = f32(rng.standard_normal((n_rows, D))); act = f32(rng.uniform(-1, 1, (n_rows, A)))
    boot = f32(rng.standard_normal((n_rows, D))); ret = f32(rng.standard_normal(n_rows) * 2.0)
    eff = f32(np.where(rng.uniform(size=n_rows) < 0.05, 0.0, 0.970299))
    cnt = 1000; mean = rng.standard_normal(D) * 0.1; m2 = np.abs(rng.standard_normal(D)) * cnt
    h = R.ref_vupdate_create(D, A, H, nh, B, cap, 0, ptr(q1), ptr(q2), ptr(pol), 1, L,
                             np.float32(-10), np.float32(10))
    R.ref_vupdate_insert(h, ptr(obs), ptr(act), ptr(boot), ptr(ret), ptr(eff), n_rows)
    R.ref_vupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    losses = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_vupdate_step(h, ptr(l)) == 0
        losses[k] = l[0]
    P = param_count(qs)
    res = np.zeros((4, P), np.float32)
    for w in range(4):
        R.ref_vupdate_params(h, w, ptr(res[w]))
    R.ref_vupdate_destroy(h)
    out.update(cu_dims=np.array([D, A, H, nh, B, cap, L]), cu_pol=pol, cu_q1=q1, cu_q2=q2,
               cu_obs=obs, cu_act=act, cu_boot=boot, cu_ret=ret, cu_eff=eff,
               cu_norm=np.array([cnt]), cu_mean=mean, cu_m2=m2, cu_losses=losses, cu_params=res)
    h = R.ref_pupdate_create(D, A, H, nh, B, cap, 0, ptr(pol), ptr(q1), ptr(q2), 1, L,
                             np.float32(-10), np.float32(10))
    R.ref_pupdate_insert(h, ptr(obs), n_rows)
    R.ref_pupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    pl = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_pupdate_step(h, ptr(l)) == 0
        pl[k] = l[0]
    pp = np.zeros(param_count(ps), np.float32)
    R.ref_pupdate_params(h, ptr(pp))
    R.ref_pupdate_destroy(h)
    out.update(cpu_losses=pl, cpu_params=pp)


def gen_sac(R, out):
    """pql_sac: the eps stream (normal_distribution<float> over
    make_rng(0, sac, 1)), GaussianPolicy::sample, k=3 V-learner and 3
    P-learner updates (sac_critic_loss / sac_actor_loss / sac_alpha_loss,
    learners.cpp:168-176, :246-258) and one stochastic actor step
    (learners.cpp:87-94)."""
    rng = np.random.default_rng(11)
    nrm = np.zeros(1001, np.float32)
    R.ref_normals(0, 6, 1, 1001, ptr(nrm))
    out.update(sac_normals=nrm)
    D, A, H, nh, B, cap = 9, 4, 32, 2, 48, 500
    ps = [D] + [H] * nh + [2 * A]
    qs = [D + A] + [H] * nh + [1]
    pol = f32(rng.standard_normal(param_count(ps)) * 0.2)
    q1 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    q2 = f32(rng.standard_normal(param_count(qs)) * 0.2)
    # sample(): act / logp for a batch with a few log_std values clamped
    obs = f32(rng.standard_normal((64, D)))
    eps = f32(rng.standard_normal((64, A)))
    act = np.zeros((64, A), np.float32)
    logp = np.zeros(64, np.float32)
    assert R.ref_gauss_sample(ptr(pol), ptr(sizes_arr(ps)), nh + 1, ptr(obs), ptr(eps), 64, None,
                              None, ptr(act), ptr(logp), None) == 0
    out.update(gs_obs=obs, gs_eps=eps, gs_act=act, gs_logp=logp)
    n_rows = 300
    obs = f32(rng.standard_normal((n_rows, D))); act = f32(rng.uniform(-1, 1, (n_rows, A)))
    boot = f32(rng.standard_normal((n_rows, D))); ret = f32(rng.standard_normal(n_rows) * 2.0)
    eff = f32(np.where(rng.uniform(size=n_rows) < 0.05, 0.0, 0.970299))
    cnt = 1000; mean = rng.standard_normal(D) * 0.1; m2 = np.abs(rng.standard_normal(D)) * cnt
    log_alpha = np.float32(-0.7)
    h = R.ref_vupdate_create(D, A, H, nh, B, cap, 0, ptr(q1), ptr(q2), ptr(pol), 2, 1,
                             np.float32(-10), np.float32(10))
    R.ref_vupdate_set_log_alpha(h, log_alpha)
    R.ref_vupdate_insert(h, ptr(obs), ptr(act), ptr(boot), ptr(ret), ptr(eff), n_rows)
    R.ref_vupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    losses = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_vupdate_step(h, ptr(l)) == 0
        losses[k] = l[0]
    P = param_count(qs)
    res = np.zeros((4, P), np.float32)
    for w in range(4):
        R.ref_vupdate_params(h, w, ptr(res[w]))
    R.ref_vupdate_destroy(h)
    out.update(su_dims=np.array([D, A, H, nh, B, cap]), su_pol=pol, su_q1=q1, su_q2=q2,
               su_obs=obs, su_act=act, su_boot=boot, su_ret=ret, su_eff=eff,
               su_norm=np.array([cnt]), su_mean=mean, su_m2=m2, su_log_alpha=np.array([log_alpha]),
               su_losses=losses, su_params=res)
    h = R.ref_pupdate_create(D, A, H, nh, B, cap, 0, ptr(pol), ptr(q1), ptr(q2), 2, 1,
                             np.float32(-10), np.float32(10))
    R.ref_pupdate_insert(h, ptr(obs), n_rows)
    R.ref_pupdate_adopt_norm(h, cnt, ptr(mean), ptr(m2))
    pl = np.zeros(3, np.float32)
    la = np.zeros(3, np.float32)
    for k in range(3):
        l = np.zeros(1, np.float32)
        assert R.ref_pupdate_step(h, ptr(l)) == 0
        pl[k] = l[0]
        la[k] = R.ref_pupdate_log_alpha(h)
    pp = np.zeros(param_count(ps), np.float32)
    R.ref_pupdate_params(h, ptr(pp))
    R.ref_pupdate_destroy(h)
    out.update(sp_losses=pl, sp_log_alpha=la, sp_params=pp)
    # one stochastic actor step on N envs (normalizer seeded by one observe)
    N = 40
    a = R.ref_actor_create_sac(N, D, A, H, nh, 0, ptr(pol))
    o0 = f32(rng.standard_normal((N, D)))
    R.ref_actor_observe(a, ptr(o0))
    o1 = f32(rng.standard_normal((N, D)))
    acts = np.zeros((N, A), np.float32)
    R.ref_actor_act(a, ptr(o1), ptr(acts))
    R.ref_actor_destroy(a)
    out.update(sa_obs0=o0, sa_obs1=o1, sa_act=acts)


METRICS_ROWS = [
    [0.0, 0, 0, 0, 0, 0.0, 0.0, 0.0, 0.0],
    [1.23456, 262144, 64, 256, 128, -1234.5678912, 12.3456789, 0.000123456789, -7.25],
    [59.9995, 1 << 40, 1 << 26, (1 << 29) + 3, 1 << 28, 1e-300, 3.5e12, 123456789.0, -0.0],
    [3600.0004, 16384 * 1000, 1000, 8000, 4000, -200.0, 0.5, 1.0 / 3.0, 2.0 / 3.0],
    [0.0005, 7, 7, 1, 0, float("inf"), float("nan"), -float("inf"), 1e-7],
]


def gen_metrics(R, out):
    """rt::MetricsWriter output for METRICS_ROWS (tests/golden/metrics_ref.csv)."""
    rows = np.ascontiguousarray(np.array(METRICS_ROWS, np.float64))
    path = str(GOLDEN / "metrics_ref.csv")
    assert R.ref_metrics_write(path.encode(), ptr(rows), rows.shape[0]) == 0
    out.update(mt_dummy=np.zeros(1))


def ckpt_content(seed=9):
    """A small checkpoint payload: three nets of the learners' shapes + stats."""
    rng = np.random.default_rng(seed)
    nets = [("q1", [9, 32, 32, 1]), ("q2", [9, 32, 32, 1]), ("policy", [5, 32, 32, 4])]
    flats = [f32(rng.standard_normal(param_count(sz))) for _, sz in nets]
    mean = rng.standard_normal(5)
    m2 = np.abs(rng.standard_normal(5)) * 100
    return nets, flats, 1234, mean, m2


def gen_checkpoint(R, out):
    """fa::save_checkpoint output for ckpt_content(), kept as raw bytes
    (tests/golden/ckpt_ref.bin) to pin the writer byte for byte."""
    import ctypes as C
    nets, flats, count, mean, m2 = ckpt_content()
    names = (C.c_char_p * len(nets))(*[n.encode() for n, _ in nets])
    nl = np.array([len(sz) - 1 for _, sz in nets], np.uint64)
    szs = [np.array(sz, np.uint64) for _, sz in nets]
    szp = (C.c_void_p * len(nets))(*[a.ctypes.data for a in szs])
    fp = (C.c_void_p * len(nets))(*[a.ctypes.data for a in flats])
    path = str(GOLDEN / "ckpt_ref.bin")
    assert R.ref_checkpoint_save(path.encode(), len(nets), names, nl.ctypes.data, szp, fp, count,
                                 ptr(mean), ptr(m2), 5) == 0
    out.update(ck_dummy=np.zeros(1))


def synth_coupling(seed, D, A):
    """The synthetic task's M (SyntheticEnv in ref_harness.cpp) -- used only to
    build actions that drive |s_0| past the terminal threshold."""
    R = ref()
    mseed = R.ref_derive_seed(seed, 1, 1 << 40)
    from oracle_lib import orc
    M = np.zeros((D, A))
    for d in range(D):
        for k in range(A):
            u = orc().orc_splitmix64((mseed + d * A + k) & ((1 << 64) - 1))
            M[d, k] = float(np.float32((u >> 11) * 2.0**-53 * 2.0 - 1.0))
    return M


ENV_CASES = [  # N, D, A, max_len, T, seed, full trajectories stored
    (64, 5, 2, 7, 60, 3, True),
    (40, 60, 8, 13, 30, 3, True),
    (32, 211, 20, 200, 80, 15, False),
]


def gen_env(R, out):
    """The reference's own EnvBatch::reset_all / step (vecenv.cpp:73-106) on the
    synthetic task (SyntheticEnv, ref_harness.cpp), staggered time limits:
    random (partly out-of-range) actions, and for the c3-dims case half the
    envs pushed along sign(M[0]) so |s_0| crosses 9 (terminal resets)."""
    for k, (N, D, A, max_len, T, seed, full) in enumerate(ENV_CASES):
        rng = np.random.default_rng(100 + k)
        obs0 = np.zeros((N, D), np.float32)
        h = R.ref_synth_env_create(N, D, A, seed, max_len, np.float32(-1), np.float32(1), 1,
                                   ptr(obs0))
        drive = np.sign(synth_coupling(seed, D, A)[0]).astype(np.float32)
        acts = np.zeros((T, N, A), np.float32)
        nxt = np.zeros((T, N, D), np.float32)
        term_obs = np.zeros((T, N, D), np.float32)
        rew = np.zeros((T, N), np.float32)
        done = np.zeros((T, N), np.uint8)
        trunc = np.zeros((T, N), np.uint8)
        hashes = np.zeros((T, 2), np.uint64)
        for t in range(T):
            a = f32(rng.uniform(-1.5, 1.5, (N, A)))
            a[: N // 2] = np.where(rng.uniform(size=(N // 2, 1)) < 0.9, drive, a[: N // 2])
            acts[t] = a
            assert R.ref_synth_env_step(h, ptr(acts[t]), ptr(nxt[t]), ptr(term_obs[t]),
                                        ptr(rew[t]), ptr(done[t]), ptr(trunc[t])) == 0
            term_obs[t][done[t] == 0] = 0.0
            hashes[t] = (traj_hash(nxt[t]), traj_hash(term_obs[t]))
        ep = np.zeros(N, np.int64)
        R.ref_synth_env_episode_steps(h, ptr(ep))
        last = nxt[T - 1].copy()
        bad = f32(np.full((N, A), np.nan))
        nan_rc = R.ref_synth_env_step(h, ptr(bad), ptr(nxt[0]), ptr(term_obs[0]), ptr(rew[0]),
                                      ptr(done[0]), ptr(trunc[0]))
        R.ref_synth_env_destroy(h)
        out[f"env{k}_args"] = np.array([N, D, A, max_len, T, seed], np.int64)
        out[f"env{k}_obs0"] = obs0
        out[f"env{k}_act"] = acts
        out[f"env{k}_rew"] = rew
        out[f"env{k}_done"] = done
        out[f"env{k}_trunc"] = trunc
        out[f"env{k}_hash"] = hashes
        out[f"env{k}_last"] = last
        out[f"env{k}_nan_rc"] = np.array([nan_rc], np.int64)
        out[f"env{k}_episode_step"] = ep
        if full:
            out[f"env{k}_next"] = nxt
            out[f"env{k}_term_obs"] = term_obs
        n_term = int(np.sum(done & (trunc == 0)))
        print(f"  env{k}: terminals {n_term}, truncations {int(trunc.sum())}, nan rc {nan_rc}")


ACTOR_CASES = [  # N, D, A, hidden, seed, max_len, T, sac
    (256, 32, 8, 256, 5, 50, 5, 0),
    (256, 211, 20, 512, 7, 1000, 3, 0),
    (128, 17, 6, 64, 9, 20, 6, 1),
]


def gen_actor_core(R, out):
    """The reference's own rt::ActorCore (learners.cpp:62-116: constructor,
    PolicyHandle::create, noise schedule / streams, rollout_step) on the
    synthetic task: the StepSlices of T steps and the final normalizer.
    Generated with the scalar kernel backend (kernels::set_backend), the
    op-order ground truth the restatement follows bit for bit (the AVX2
    backend's FMA-reassociated policy layers differ in the last ulp)."""
    R.ref_set_backend(0)
    for k, (N, D, A, H, seed, max_len, T, sac) in enumerate(ACTOR_CASES):
        h = R.ref_actor_core_create(N, D, A, H, seed, 0.05, 0.8, -1.0, max_len, sac)
        P = R.ref_actor_core_policy(h, None)
        pol = np.zeros(P, np.float32)
        R.ref_actor_core_policy(h, ptr(pol))
        obs = np.zeros((T, N, D), np.float32)
        act = np.zeros((T, N, A), np.float32)
        boot = np.zeros((T, N, D), np.float32)
        rew = np.zeros((T, N), np.float32)
        term = np.zeros((T, N), np.uint8)
        trunc = np.zeros((T, N), np.uint8)
        for t in range(T):
            assert R.ref_actor_core_step(h, ptr(obs[t]), ptr(act[t]), ptr(boot[t]), ptr(rew[t]),
                                         ptr(term[t]), ptr(trunc[t])) == 0
        cnt = np.zeros(1, np.int64)
        mean, m2 = np.zeros(D), np.zeros(D)
        R.ref_actor_core_norm(h, ptr(cnt), ptr(mean), ptr(m2))
        ep = np.zeros(N, np.int64)
        R.ref_actor_core_episode_steps(h, ptr(ep))
        R.ref_actor_core_destroy(h)
        out[f"ac{k}_args"] = np.array([N, D, A, H, seed, max_len, T, sac], np.int64)
        if pol.size > 100_000:  # re-derivable (PolicyHandle::create): keep only its digest
            out[f"ac{k}_policy_hash"] = np.array([traj_hash(pol)], np.uint64)
        else:
            out[f"ac{k}_policy"] = pol
        out[f"ac{k}_obs"] = obs
        out[f"ac{k}_act"] = act
        out[f"ac{k}_boot"] = boot
        out[f"ac{k}_rew"] = rew
        out[f"ac{k}_term"] = term
        out[f"ac{k}_trunc"] = trunc
        out[f"ac{k}_norm"] = np.concatenate([cnt.astype(np.float64), mean, m2])
        out[f"ac{k}_episode_step"] = ep
    R.ref_set_backend(1)


EVAL_CASES = [  # D, A, H, n_hidden, episodes, eval_seed, max_len, sac
    (19, 6, 64, 2, 96, 77, 40, 0),
    (19, 6, 64, 2, 96, 77, 200, 0),
    (31, 5, 64, 3, 64, 78, 60, 0),
    (23, 4, 64, 2, 48, 79, 50, 1),
]


def gen_evaluate(R, out):
    """The reference's own rt::evaluate_policy (learners.cpp:280-325) on the
    synthetic task: mean return and standard error (scalar kernel backend,
    as gen_actor_core)."""
    R.ref_set_backend(0)
    for k, (D, A, H, nh, M, seed, max_len, sac) in enumerate(EVAL_CASES):
        rng = np.random.default_rng(200 + k)
        ps = [D] + [H] * nh + [2 * A if sac else A]
        pol = f32(rng.standard_normal(param_count(ps)) * 0.1)
        mean = rng.standard_normal(D) * 0.1
        m2 = np.abs(rng.standard_normal(D)) * 50 + 10
        count = 100
        mu, se = np.zeros(1), np.zeros(1)
        assert R.ref_evaluate_synth(ptr(pol), ptr(sizes_arr(ps)), nh + 1, sac, count, ptr(mean),
                                    ptr(m2), M, seed, max_len, np.float32(-1), np.float32(1),
                                    ptr(mu), ptr(se)) == 0
        out[f"ev{k}_args"] = np.array([D, A, H, nh, M, seed, max_len, sac, count], np.int64)
        out[f"ev{k}_policy"] = pol
        out[f"ev{k}_mean"] = mean
        out[f"ev{k}_m2"] = m2
        out[f"ev{k}_result"] = np.array([mu[0], se[0]])
    R.ref_set_backend(1)


def main():
    R = ref()
    if R is None:
        raise SystemExit("oracle/_ref/libpqlref.so missing: run `make -C oracle ref` first")
    GOLDEN.mkdir(parents=True, exist_ok=True)
    for name, fn in [("indices", gen_indices), ("nstep", gen_nstep),
                     ("elementwise", gen_elementwise), ("norm", gen_norm), ("noise", gen_noise),
                     ("mlp", gen_mlp), ("agents", gen_agents), ("vupdate", gen_vupdate),
                     ("c51update", gen_c51update), ("sac", gen_sac),
                     ("checkpoint", gen_checkpoint), ("metrics", gen_metrics),
                     ("env", gen_env), ("actor_core", gen_actor_core),
                     ("evaluate", gen_evaluate)]:
        if len(sys.argv) > 1 and name not in sys.argv[1:]:
            continue
        out: dict = {}
        fn(R, out)
        if name in ("checkpoint", "metrics"):  # raw bytes only (ckpt_ref.bin, metrics_ref.csv)
            continue
        np.savez_compressed(GOLDEN / f"{name}.npz", **out)
        print(name, sum(v.nbytes for v in out.values()), "bytes")


if __name__ == "__main__":
    main()
