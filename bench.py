#!/usr/bin/env python
"""bench.py -- PQL learner/actor hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): critic updates/s at batch 8192 (headline `value`)
and actor transitions/s at 16384 envs (reported under "actor" when built),
config 3 (Shadow-Hand-like dims: obs 211 / act 20, 3x512 MLPs, B=8192,
5M-record replay, mixed exploration noise).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one CriticLearnerCore::update (sample -> TD target -> twin critic
loss/backward -> clip/Adam/Polyak) replayed from a CUDA graph.  Inputs are
sampled from a 5M-record ring (8.9 GB >> the 126 MB L2), so every step
reads fresh rows from HBM.

Multi-GPU (config 5): `--gpus N` without WORLD_SIZE in the
environment re-executes this script under torch.distributed.run with N
ranks (127.0.0.1, NCCL INIT logging on stderr).  The N>1 headline is strong
scaling: one global batch of 8192 split 8192/N per rank, the data-parallel
critic's gradients summed by one NCCL all-reduce per update; `weak_scaling`
reports B = 8192 per rank beside it.  The actor legs run 16384 envs per GPU
(`actor`, the BASELINE metric's second half) and config 5's 65536 envs split
over the N GPUs (`actor_c5`, sharded normalizer).  Device times are the max
over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (obs_dim, act_dim, hidden, hidden_layers, batch, n_envs, capacity)
    "c1": (32, 8, 256, 2, 1024, 256, 100_000),
    "c2": (60, 8, 512, 3, 8192, 4096, 5_000_000),
    "c3": (211, 20, 512, 3, 8192, 16384, 5_000_000),
}
C5_ENVS = 65536  # config 5: envs over all GPUs
METRIC = "critic updates/s (batch 8192) and actor transitions/s at 16384 envs"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--force-dp", action="store_true",
                   help="use the data-parallel (NCCL) learners even at N=1 (path check)")
    p.add_argument("--precision", choices=["tf32", "3xtf32"], default="tf32",
                   help="GEMM precision of the headline leg (pqlg_config.precision)")
    a = p.parse_args()
    a.precision = {"tf32": 0, "3xtf32": 1}[a.precision]
    return a


# --------------------------------------------------------------- plumbing
def relaunch_under_torchrun(n_gpus):
    """`python bench.py --gpus N` (no WORLD_SIZE): run N ranks, one per GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n_gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ))


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator init lines (rank count, NVLS / transport) for the audit
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = max(mx, float(f[2]))
                except ValueError:
                    continue
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except OSError:
            pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except OSError:
        return {}


def peak_denominators():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) when
    present -- HBM copy GB/s, and TF32 dense = half the measured bf16 burst
    (the tcgen05 kind::tf32 rate is half of kind::f16) -- else the
    B200_PROFILING.md fallbacks (6.5 TB/s, 2.25 PF bf16 nominal / 2)."""
    pk = measured_peaks()
    if pk.get("bf16_tflops") and pk.get("hbm_gbs"):
        return {"tf32_tflops": pk["bf16_tflops"] / 2.0, "hbm_gbs": pk["hbm_gbs"],
                "source": "MEASURED_PEAKS.json: hbm_gbs; tf32 = bf16_tflops (burst) / 2"}
    return {"tf32_tflops": 1125.0, "hbm_gbs": 6500.0,
            "source": "fallback (no MEASURED_PEAKS.json): 6.5 TB/s, 2.25 PF bf16 / 2"}

def tf32_peak_tflops():
    """cuBLAS TF32 GEMM 8192^3 (the TF32 denominator MEASURED_PEAKS lacks)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def traffic_from_profiles(kernel_key):
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get(kernel_key)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------ our arm
def critic_flops(D, A, H, nh, B):
    """Algorithmic FLOPs of one critic update: policy fwd +
    4 critic fwd + 2 x (critic wgrad + dgrad for layers >= 1)."""
    pol = D * H + (nh - 1) * H * H + H * A
    crit = (D + A) * H + (nh - 1) * H * H + H
    crit_dgrad = (nh - 1) * H * H + H
    return 2 * B * (pol + 4 * crit + 2 * (crit + crit_dgrad))


def gemm_layer(rows, groups, n, k):
    """The rows of a time_graph() listing for GEMM launches of that shape."""
    key = f"groups={groups} "
    return [r for r in rows if r[2].startswith(key) and f" N={n} K={k} " in r[2] + " "]


def run_ours(args, rank, world, local, B, timed=True):
    """Critic updates/s with per-rank batch B (the N>1 headline splits the
    global 8192; the weak-scaling leg keeps 8192 per rank)."""
    import torch
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, _, N, cap = CONFIGS[args.config]
    stream = torch.cuda.Stream(device=local)
    cfg = _lib.default_config(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh,
                              n_envs=N, seed=0, precision=args.precision)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    comm = None
    if world > 1 or args.force_dp:
        # data-parallel critic (SURVEY 8(e) option i): one NCCL all-reduce of
        # the twin-critic gradients + loss per update; every rank samples its
        # own replay shard with its own Philox stream; same init everywhere
        comm = _lib.comm_from_torch_dist(rank, world)
        _lib.call("pqlg_vlearner_create_dp", C.byref(cfg), C.byref(dims), 12345, comm,
                  C.c_void_p(stream.cuda_stream), C.byref(h))
    else:
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 12345,
                  C.c_void_p(stream.cuda_stream), C.byref(h))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
    # each rank holds its own shard of the 5M-record ring
    shard = cap // world if world > 1 else cap
    _lib.call("pqlg_replay_fill_synthetic", rp, shard, 1000 + rank, np.float32(0.970299), 200)
    count = 10 ** 6
    mean = np.zeros(D)
    m2 = np.full(D, float(count))
    ns = _lib.NormStats(count, mean.ctypes.data, m2.ctypes.data)
    _lib.call("pqlg_vlearner_adopt_norm", h, C.byref(ns))
    kpu = C.c_int()
    _lib.call("pqlg_vlearner_kernels_per_update", h, C.byref(kpu))
    stream.synchronize()

    # warm-up (graph build + W updates)
    _lib.call("pqlg_vlearner_update_n", h, args.warmup)
    stream.synchronize()
    barrier(world)

    launches0 = _lib.lib().pqlg_launch_count()
    with ClockSampler(local) as clk:
        stream.synchronize()
        barrier(world)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        _lib.call("pqlg_vlearner_update_n", h, args.steps)
        e.record(stream)
        e.synchronize()
        barrier(world)
        ms = s.elapsed_time(e)
    launches = _lib.lib().pqlg_launch_count() - launches0
    ms = max_over_ranks(ms, world)
    loss = C.c_float()
    _lib.call("pqlg_vlearner_last_loss", h, C.byref(loss))
    ms_step = ms / args.steps
    out = dict(ms_step=ms_step, loss=loss.value, clocks=clk.summary(), launches=int(launches),
               kpu=kpu.value, batch_per_rank=B)
    if not timed:
        _lib.call("pqlg_vlearner_destroy", h)
        if comm is not None:
            _lib.call("pqlg_comm_destroy", comm)
        return out

    # ---- e2e: the reference-facing synchronous update() per step with the
    # step's host inputs (normalizer stats, pinned) copied in and the loss
    # copied out, host timer around the whole loop.
    mean_p = torch.zeros(D, dtype=torch.float64).pin_memory()
    m2_p = torch.full((D,), float(count), dtype=torch.float64).pin_memory()
    e2e_steps = max(10, min(args.steps, 100))
    barrier(world)
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ns = _lib.NormStats(count, mean_p.data_ptr(), m2_p.data_ptr())
        _lib.call("pqlg_vlearner_adopt_norm", h, C.byref(ns))
        _lib.call("pqlg_vlearner_update", h, C.byref(loss))
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    out["e2e"] = {"value": e2e_steps / e2e_s, "unit": "updates/s",
                  "h2d_bytes_per_step": 2 * D * 8, "d2h_bytes_per_step": 4,
                  "api": "pqlg_vlearner_adopt_norm + pqlg_vlearner_update (sync)"}

    # ---- roofline of the dominant kernel, measured in situ: the update
    # graph re-captured with an event-record node around every kernel
    # (pqlg_vlearner_time_update), replayed on the learner's stream.  The
    # dominant kernel is the 4-group hidden-layer GEMM (twin target + twin
    # online critics, one persistent launch per layer, K = N = 512).
    if rank == 0:
        pk = peak_denominators()
        rows, g_ms = _lib.time_graph("pqlg_vlearner_time_update", h, 20)
        dom = gemm_layer(rows, 4, H, H)
        d_ms = float(np.mean([r[1] for r in dom]))
        flops = 4 * 2 * B * H * H
        ach = flops / (d_ms * 1e-3) / 1e12
        upd_flops = critic_flops(D, A, H, nh, B)
        out["roof"] = {
            "bound": "tensor",
            "kernel": "gemm_tf32_kernel<256, K-major A, N-major B, Hidden, CTA pair>: 4 groups "
                      f"(twin target + twin online critic hidden layer, 4 x {B}x{H}x{H}), "
                      "in situ in the update graph",
            "achieved": round(ach, 2), "peak": round(pk["tf32_tflops"], 2), "unit": "TFLOP/s",
            "frac": round(ach / pk["tf32_tflops"], 4), "peak_source": pk["source"],
            "kernel_ms": round(d_ms, 5), "launches_per_update": len(dom),
            "flops_per_launch": flops,
            "traffic": traffic_from_profiles("critic_layer_4group_in_update"),
            "share_of_step": round(len(dom) * d_ms / g_ms, 4),
            "timing": "CUDA events recorded as graph nodes around each launch "
                      "(pqlg_vlearner_time_update, 20 replays, no PDL overlap)",
            "update_tflops": round(upd_flops / (ms_step * 1e-3) / 1e12, 2),
            "update_frac_of_tf32_peak": round(upd_flops / (ms_step * 1e-3) / 1e12
                                              / pk["tf32_tflops"], 4),
            "kernels": [[r[0].split("(")[0][-60:], round(r[1] * 1e3, 2), r[2]] for r in rows],
            "instrumented_graph_ms": round(g_ms, 5),
            # the denominator above is conservative: the nominal dense TF32
            # rate (B200_PROFILING.md) is 1.1 PF/s, and this kernel's own
            # mainloop runs at ~1.15 PF/s (DESIGN 5, GEMM timing anatomy)
            "frac_of_nominal_tf32_1100": round(ach / 1100.0, 4),
        }
    _lib.call("pqlg_vlearner_destroy", h)
    if comm is not None:
        _lib.call("pqlg_comm_destroy", comm)
    return out


def run_c51(args, rank, world, local, steps, warmup, sac=False):
    """Config 4 (PQL-D): C51 critic updates/s and policy updates/s at batch
    8192 with 51 atoms on [-10, 10], c3 dims, graph-replayed.  sac=True: the
    same legs for pql_sac (Gaussian policy, entropy-regularised target, alpha
    step) at config 3."""
    import torch
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, B, N, cap = CONFIGS["c3"]
    stream = torch.cuda.Stream(device=local)
    sp = C.c_void_p(stream.cuda_stream)
    if sac:
        cfg = _lib.default_config(algo=_lib.ALGO_SAC, batch_size=B, buffer_capacity=1_000_000,
                                  hidden=H, hidden_layers=nh, n_envs=N, seed=0)
    else:
        cfg = _lib.default_config(algo=_lib.ALGO_C51, n_atoms=51, vmin=-10.0, vmax=10.0,
                                  reward_scale=0.01, batch_size=B, buffer_capacity=1_000_000,
                                  hidden=H, hidden_layers=nh, n_envs=N, seed=0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    vl, pl = C.c_void_p(), C.c_void_p()
    comm = _lib.comm_from_torch_dist(rank, world) if (world > 1 or args.force_dp) else None
    if comm is not None:
        _lib.call("pqlg_vlearner_create_dp", C.byref(cfg), C.byref(dims), 1, comm, sp, C.byref(vl))
        _lib.call("pqlg_plearner_create_dp", C.byref(cfg), C.byref(dims), 1, comm, sp, C.byref(pl))
    else:
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
        _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", vl, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 2000 + rank, np.float32(0.970299), 200)
    states = torch.randn(1_000_000, D, device=f"cuda:{local}")
    _lib.call("pqlg_plearner_ingest", pl, states.data_ptr(), D, 1_000_000)
    out = {"workload": ("c3: pql_sac critic + policy/alpha, batch 8192" if sac else
                        "c4: PQL-D critic (51 atoms on [-10, 10]) + policy, c3 dims, batch 8192")}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for key, h, fn in (("critic_updates", vl, "pqlg_vlearner_update_n"),
                       ("policy_updates", pl, "pqlg_plearner_update_n")):
        _lib.call(fn, h, warmup)
        stream.synchronize()
        barrier(world)
        ev0.record(stream)
        _lib.call(fn, h, steps)
        ev1.record(stream)
        ev1.synchronize()
        ms = max_over_ranks(ev0.elapsed_time(ev1), world)
        out[key] = {"value": world * steps / (ms * 1e-3), "unit": "updates/s",
                    "ms_per_step": ms / steps}
    loss = C.c_float()
    _lib.call("pqlg_vlearner_last_loss", vl, C.byref(loss))
    out["last_critic_loss"] = loss.value
    _lib.call("pqlg_vlearner_destroy", vl)
    _lib.call("pqlg_plearner_destroy", pl)
    if comm is not None:
        _lib.call("pqlg_comm_destroy", comm)
    return out


def run_other_config(args, rank, world, local, name, steps, warmup):
    """Critic updates/s and actor steps/s (rollout only, graph replay) at
    another BASELINE config (c2: Ant-like dims, 4096 envs; c1: the
    reference's CPU case), same kernels, synthetic replay fill."""
    import torch
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, B, N, cap = CONFIGS[name]
    stream = torch.cuda.Stream(device=local)
    sp = C.c_void_p(stream.cuda_stream)
    cap = min(cap, 1_000_000)
    cfg = _lib.default_config(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh,
                              n_envs=N, seed=0, env_offset=rank * N, envs_total=world * N)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    vl, act = C.c_void_p(), C.c_void_p()
    comm = _lib.comm_from_torch_dist(rank, world) if world > 1 else None
    if comm is not None:
        _lib.call("pqlg_vlearner_create_dp", C.byref(cfg), C.byref(dims), 1, comm, sp, C.byref(vl))
        _lib.call("pqlg_actor_create_sharded", C.byref(cfg), C.byref(dims), comm, sp, C.byref(act))
    else:
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
        _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", vl, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, cap, 3000 + rank, np.float32(0.970299), 200)
    out = {"workload": f"{name}: obs {D} / act {A}, {nh}x{H} MLPs, batch {B}, {N} envs per GPU"}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for key, h, fn, unit, per in (("critic_updates", vl, "pqlg_vlearner_update_n", "updates/s", 1),
                                  ("actor_transitions", act, "pqlg_actor_rollout_n",
                                   "transitions/s", N)):
        _lib.call(fn, h, warmup)
        stream.synchronize()
        barrier(world)
        ev0.record(stream)
        _lib.call(fn, h, steps)
        ev1.record(stream)
        ev1.synchronize()
        ms = max_over_ranks(ev0.elapsed_time(ev1), world)
        out[key] = {"value": world * per * steps / (ms * 1e-3), "unit": unit,
                    "ms_per_step": ms / steps}
    out["actor_transitions"]["note"] = "rollout_step only (no ingest)"
    _lib.call("pqlg_vlearner_destroy", vl)
    _lib.call("pqlg_actor_destroy", act)
    if comm is not None:
        _lib.call("pqlg_comm_destroy", comm)
    return out


def run_pipeline(args, rank, world, local, actor_steps):
    """run_parallel on this GPU: Actor, V-learner and
    P-learner as three threads on three streams, RatioGate pacing at the
    paper's beta_av = 1/8, beta_pv = 1/2 (Table B.1), c3 dims and nets.
    Reports env steps/s and the learners' update rates over the run."""
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, B, N, cap = CONFIGS[args.config]
    cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H, hidden_layers=nh,
                              n_envs=N, seed=rank, env_offset=rank * N, envs_total=world * N)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    rc = _lib.ratio_config()
    h = C.c_void_p()
    _lib.call("pqlg_pipeline_create", C.byref(cfg), C.byref(dims), C.byref(rc), 1, C.byref(h))
    rep = _lib.RunReport()
    _lib.call("pqlg_pipeline_run", h, actor_steps, 120.0, C.byref(rep))
    _lib.call("pqlg_pipeline_destroy", h)
    return {"workload": f"run_parallel, {args.config} dims, {N} envs, H=4, K_pub=8, "
                        f"beta_av=1/8, beta_pv=1/2, {actor_steps} actor steps incl. warm-up",
            "env_steps_per_s": world * rep.env_steps / rep.wall_s,
            "critic_updates_per_s": world * rep.c_v / rep.wall_s,
            "policy_updates_per_s": world * rep.c_p / rep.wall_s,
            "ratio_av": rep.ratio_av, "ratio_pv": rep.ratio_pv, "wall_s": rep.wall_s,
            "batches_sent": rep.batches_sent, "seq_gaps": rep.seq_gaps,
            "timing": "host wall clock over pqlg_pipeline_run (three concurrent streams)"}


def actor_step_bytes(D, A):
    """Algorithmic HBM bytes of one env's rollout step (rollout_step only):
    the policy reads the normalised obs (D) and writes the action (A); the
    normalizer update reads obs (D); the env reads obs + action (D + A) and
    writes next obs, boot obs, reward and two flags (2D + 1 words + 2 B)."""
    return 4 * (D + A + D + D + A + 2 * D + 1) + 2


def actor_step_flops(D, A, H, nh):
    return 2 * (D * H + (nh - 1) * H * H + H * A)


def run_actor(args, rank, world, local, steps, warmup, n_envs=None, roofline=False):
    """Actor transitions/s: one ActorCore::rollout_step over N envs (normalize
    -> policy -> mixed noise -> synthetic env -> StepSlice -> normalizer
    update) plus the V-learner ingest (n-step assemble + ring insert) and the
    P-learner StateBuffer insert of that slice, all on the GPU.  As in
    run_parallel, each core runs on its own stream: the learners ingest step
    t on their streams while the actor computes step t+1 (a slice stays valid
    for two more rollout steps; the actor waits for the ingest of step t
    before step t+2)."""
    import torch
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, B, N, cap = CONFIGS[args.config]
    N = n_envs or N
    stream = torch.cuda.Stream(device=local)
    sv_t, spl_t = torch.cuda.Stream(device=local), torch.cuda.Stream(device=local)
    sp = C.c_void_p(stream.cuda_stream)
    cfg = _lib.default_config(batch_size=B, buffer_capacity=min(cap, 2_000_000), hidden=H,
                              hidden_layers=nh, n_envs=N, seed=0, env_offset=rank * N,
                              envs_total=world * N, max_episode_len=1000)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
    comm = _lib.comm_from_torch_dist(rank, world) if world > 1 else None
    if comm is not None:  # shard of one actor: normalizer merged over all shards every step
        _lib.call("pqlg_actor_create_sharded", C.byref(cfg), C.byref(dims), comm, sp,
                  C.byref(act))
    else:
        _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1,
              C.c_void_p(sv_t.cuda_stream), C.byref(vl))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1,
              C.c_void_p(spl_t.cuda_stream), C.byref(pl))
    s = _lib.StepSlice()
    ev_step = [torch.cuda.Event() for _ in range(3)]
    ev_v = [torch.cuda.Event() for _ in range(3)]
    ev_p = [torch.cuda.Event() for _ in range(3)]
    t_ctr = [0]

    def step():
        t = t_ctr[0]
        k = t % 3
        if t >= 2:  # step t writes the buffers the ingest of step t-2 reads
            stream.wait_event(ev_v[(t - 2) % 3])
            stream.wait_event(ev_p[(t - 2) % 3])
        _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
        ev_step[k].record(stream)
        sv_t.wait_event(ev_step[k])
        _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
        ev_v[k].record(sv_t)
        spl_t.wait_event(ev_step[k])
        _lib.call("pqlg_plearner_ingest", pl, s.obs, s.ld_obs, N)
        ev_p[k].record(spl_t)
        t_ctr[0] = t + 1

    def join():  # the actor stream waits for the learners' last ingest
        stream.wait_event(ev_v[(t_ctr[0] - 1) % 3])
        stream.wait_event(ev_p[(t_ctr[0] - 1) % 3])

    for _ in range(warmup):
        step()
    join()
    stream.synchronize()
    barrier(world)
    l0 = _lib.lib().pqlg_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    join()
    ev1.record(stream)
    ev1.synchronize()
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    launches = _lib.lib().pqlg_launch_count() - l0
    # policy-inference-only rate (graph replay of the actor step alone)
    stream.synchronize()
    _lib.call("pqlg_actor_rollout_n", act, warmup)
    stream.synchronize()
    ev0.record(stream)
    _lib.call("pqlg_actor_rollout_n", act, steps)
    ev1.record(stream)
    ev1.synchronize()
    ms_actor_only = max_over_ranks(ev0.elapsed_time(ev1), world)
    # e2e: the host-facing C-ABI calls per step, each step ending with a
    # synchronous device->host read of its status word (4 B)
    e2e_steps = max(5, min(steps, 50))
    status = np.zeros(1, np.uint32)
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step()
        _lib.call("pqlg_actor_read", act, 6, status.ctypes.data)
    join()
    stream.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    roof = None
    if roofline and rank == 0:
        # per-kernel in-graph times of the rollout step (3 steps per replay)
        rows, g_ms = _lib.time_graph("pqlg_actor_time_steps", act, 10)
        pk = peak_denominators()
        step_ms = g_ms / 3
        fl = N * actor_step_flops(D, A, H, nh)
        by = N * actor_step_bytes(D, A)
        floor_ms = (fl / (pk["tf32_tflops"] * 1e12) + by / (pk["hbm_gbs"] * 1e9)) * 1e3
        per = {}
        for name, t, shape in rows:
            key = name.split("(")[0][-60:] + ("" if not shape else " [" + shape + "]")
            per[key] = per.get(key, 0.0) + t / 3
        top = sorted(per.items(), key=lambda kv: -kv[1])
        roof = {"bound": "tensor + hbm (step floor = GEMM FLOP / TF32 peak + bytes / HBM peak)",
                "flops_per_step": fl, "hbm_bytes_per_step": by,
                "floor_ms": round(floor_ms, 5),
                "step_ms_graph": round(ms_actor_only / steps, 5),
                "frac": round(floor_ms / (ms_actor_only / steps), 4),
                "peak_source": pk["source"],
                "instrumented_step_ms": round(step_ms, 5),
                "kernels_us": [[k, round(v * 1e3, 2)] for k, v in top]}
    for h, fn in ((act, "pqlg_actor_destroy"), (vl, "pqlg_vlearner_destroy"),
                  (pl, "pqlg_plearner_destroy")):
        _lib.call(fn, h)
    if comm is not None:
        _lib.call("pqlg_comm_destroy", comm)
    out = {"value": world * N * steps / (ms * 1e-3), "unit": "transitions/s",
           "n_envs_per_gpu": N, "n_envs_total": world * N, "ms_per_step": ms / steps,
           "actor_step_only": {"value": world * N * steps / (ms_actor_only * 1e-3),
                               "ms_per_step": ms_actor_only / steps},
           "e2e": {"value": world * N * e2e_steps / e2e_s, "unit": "transitions/s",
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4},
           "gpu_launches": int(launches)}
    if roof:
        out["roofline"] = roof
    return out


def run_policy(args, rank, world, local, steps, warmup):
    """Policy (P-learner) updates/s at batch 8192."""
    import torch
    from paper_2307_12983_b200 import _lib
    D, A, H, nh, B, N, cap = CONFIGS[args.config]
    stream = torch.cuda.Stream(device=local)
    cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H,
                              hidden_layers=nh, n_envs=N, seed=0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    pl = C.c_void_p()
    comm = None
    if world > 1 or args.force_dp:  # data-parallel policy update (one all-reduce per update)
        comm = _lib.comm_from_torch_dist(rank, world)
        _lib.call("pqlg_plearner_create_dp", C.byref(cfg), C.byref(dims), 1, comm,
                  C.c_void_p(stream.cuda_stream), C.byref(pl))
    else:
        _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1,
                  C.c_void_p(stream.cuda_stream), C.byref(pl))
    states = torch.randn(1_000_000, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", pl, states.data_ptr(), D, 1_000_000)
    _lib.call("pqlg_plearner_update_n", pl, warmup)
    stream.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    _lib.call("pqlg_plearner_update_n", pl, steps)
    ev1.record(stream)
    ev1.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    _lib.call("pqlg_plearner_destroy", pl)
    if comm is not None:
        _lib.call("pqlg_comm_destroy", comm)
    return {"value": world * steps / (ms * 1e-3), "unit": "updates/s", "ms_per_step": ms / steps,
            "parallelism": f"dp{world}" if world > 1 else "single"}


# ------------------------------------------------------ reference arm
def ref_lib():
    so = ROOT / "oracle" / "_ref" / "libpqlref.so"
    if not so.exists():
        return None
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import ref
    return ref()


def reference_critic_rate(cfg_name, n_updates, batch_override=None, threads=None):
    """The reference's own CPU path (oracle/_ref, compiled from
    /root/reference): the CriticLearnerCore::update composition of
    learners.cpp:157-188 over the config's 3x512 nets (agents-level, since
    RunConfig can only express 2 hidden layers).  One update is
    single-threaded, as the reference runs it; to use every
    host core, `threads` independent learners (replicas with their own
    buffers) update concurrently -- ctypes releases the GIL inside each
    call -- and the rate is their aggregate.  Returns (updates/s, sample,
    threads)."""
    import threading
    R = ref_lib()
    if R is None:
        return None, "oracle/_ref/libpqlref.so not built", 0
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import param_count, ptr
    D, A, H, nh, B, N, cap = CONFIGS[cfg_name]
    if batch_override:
        B = batch_override
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(0)
    qs = [D + A] + [H] * nh + [1]
    ps = [D] + [H] * nh + [A]
    q1 = (rng.standard_normal(param_count(qs)) * 0.05).astype(np.float32)
    q2 = (rng.standard_normal(param_count(qs)) * 0.05).astype(np.float32)
    pol = (rng.standard_normal(param_count(ps)) * 0.05).astype(np.float32)
    n_rows = max(4 * B, 20000)
    obs = rng.standard_normal((n_rows, D)).astype(np.float32)
    act = rng.uniform(-1, 1, (n_rows, A)).astype(np.float32)
    boot = rng.standard_normal((n_rows, D)).astype(np.float32)
    ret = (rng.standard_normal(n_rows) * 0.1).astype(np.float32)
    eff = np.full(n_rows, 0.970299, np.float32)
    mean = np.zeros(D); m2 = np.full(D, 1e6)
    handles = []
    for k in range(threads):
        h = R.ref_vupdate_create(D, A, H, nh, B, n_rows, k, ptr(q1), ptr(q2), ptr(pol), 0, 51,
                                 np.float32(-10), np.float32(10))
        R.ref_vupdate_insert(h, ptr(obs), ptr(act), ptr(boot), ptr(ret), ptr(eff), n_rows)
        R.ref_vupdate_adopt_norm(h, 10 ** 6, ptr(mean), ptr(m2))
        handles.append(h)
    start = threading.Barrier(threads + 1)
    done = threading.Barrier(threads + 1)

    def work(h):
        loss = np.zeros(1, np.float32)
        R.ref_vupdate_step(h, ptr(loss))  # warm
        start.wait()
        for _ in range(n_updates):
            R.ref_vupdate_step(h, ptr(loss))
        done.wait()

    ts = [threading.Thread(target=work, args=(h,)) for h in handles]
    for t in ts:
        t.start()
    start.wait()
    t0 = time.perf_counter()
    done.wait()
    dt = time.perf_counter() - t0
    for t in ts:
        t.join()
    for h in handles:
        R.ref_vupdate_destroy(h)
    rate = threads * n_updates / dt
    if batch_override:
        rate *= batch_override / CONFIGS[cfg_name][4]  # per full-batch update
    sample = (f"{threads} concurrent CriticLearnerCore-equivalent learners x {n_updates} "
              f"updates at B={B} ({cfg_name} dims, 3x512), reference AVX2 build, one host "
              f"thread each (a single update is single-threaded in the reference)")
    return rate, sample, threads


def _concurrent(threads, fn_setup, fn_step, n):
    """`threads` independent reference instances on their own host threads
    (ctypes releases the GIL), n steps each after one warm step; returns
    the wall seconds of the timed region."""
    import threading
    handles = [fn_setup(k) for k in range(threads)]
    start, done = threading.Barrier(threads + 1), threading.Barrier(threads + 1)

    def work(h):
        fn_step(h)
        start.wait()
        for _ in range(n):
            fn_step(h)
        done.wait()

    ts = [threading.Thread(target=work, args=(h,)) for h in handles]
    for t in ts:
        t.start()
    start.wait()
    t0 = time.perf_counter()
    done.wait()
    dt = time.perf_counter() - t0
    for t in ts:
        t.join()
    return dt, handles


def reference_actor_rate(cfg_name, steps, envs_per_thread=1024, threads=None):
    """The reference's ActorCore::rollout_step composition (learners.cpp:80-116:
    RunningNormalizer::apply -> DeterministicPolicy::act -> apply_noise ->
    EnvBatch::step on SyntheticEnv -> RunningNormalizer::update) at the
    config's 3x512 policy, `threads` actors of `envs_per_thread` envs each
    (16 x 1024 = the 16384 envs of config 3).  Returns (transitions/s,
    sample, threads)."""
    R = ref_lib()
    if R is None:
        return None, "oracle/_ref/libpqlref.so not built", 0
    from oracle_lib import param_count, ptr
    D, A, H, nh, B, N, cap = CONFIGS[cfg_name]
    threads = threads or os.cpu_count() or 1
    n = envs_per_thread
    ps = [D] + [H] * nh + [A]
    pol = (np.random.default_rng(0).standard_normal(param_count(ps)) * 0.05).astype(np.float32)
    bufs = {}

    def setup(k):
        obs = np.zeros((n, D), np.float32)
        env = R.ref_synth_env_create(n, D, A, k, 1000, np.float32(-1), np.float32(1), 1, ptr(obs))
        act = R.ref_actor_create(n, D, A, H, nh, k, ptr(pol), np.float32(0.05), np.float32(0.8))
        bufs[k] = dict(obs=obs, a=np.zeros((n, A), np.float32), nxt=np.zeros((n, D), np.float32),
                       term=np.zeros((n, D), np.float32), rew=np.zeros(n, np.float32),
                       done=np.zeros(n, np.uint8), trunc=np.zeros(n, np.uint8))
        return (k, env, act)

    def step(h):
        k, env, act = h
        b = bufs[k]
        R.ref_actor_act(act, ptr(b["obs"]), ptr(b["a"]))
        R.ref_synth_env_step(env, ptr(b["a"]), ptr(b["nxt"]), ptr(b["term"]), ptr(b["rew"]),
                             ptr(b["done"]), ptr(b["trunc"]))
        R.ref_actor_observe(act, ptr(b["obs"]))
        b["obs"][:] = b["nxt"]

    dt, hs = _concurrent(threads, setup, step, steps)
    for _, env, act in hs:
        R.ref_synth_env_destroy(env)
        R.ref_actor_destroy(act)
    rate = threads * n * steps / dt
    sample = (f"{threads} concurrent ActorCore::rollout_step compositions x {n} envs x {steps} "
              f"steps ({cfg_name} dims, {nh}x{H} policy, mixed noise, SyntheticEnv through the "
              f"reference's EnvBatch::step), reference AVX2 build, one host thread each")
    return rate, sample, threads


def reference_policy_rate(cfg_name, n_updates, threads=None):
    """The reference's PolicyLearnerCore::update composition (learners.cpp:
    239-270) at the config's 3x512 nets and B = 8192, `threads` independent
    learners.  Returns (updates/s, sample, threads)."""
    R = ref_lib()
    if R is None:
        return None, "oracle/_ref/libpqlref.so not built", 0
    from oracle_lib import param_count, ptr
    D, A, H, nh, B, N, cap = CONFIGS[cfg_name]
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(1)
    qs = [D + A] + [H] * nh + [1]
    ps = [D] + [H] * nh + [A]
    q1 = (rng.standard_normal(param_count(qs)) * 0.05).astype(np.float32)
    q2 = (rng.standard_normal(param_count(qs)) * 0.05).astype(np.float32)
    pol = (rng.standard_normal(param_count(ps)) * 0.05).astype(np.float32)
    n_rows = 2 * B
    states = rng.standard_normal((n_rows, D)).astype(np.float32)
    mean, m2 = np.zeros(D), np.full(D, 1e6)

    def setup(k):
        h = R.ref_pupdate_create(D, A, H, nh, B, n_rows, k, ptr(pol), ptr(q1), ptr(q2), 0, 51,
                                 np.float32(-10), np.float32(10))
        R.ref_pupdate_insert(h, ptr(states), n_rows)
        R.ref_pupdate_adopt_norm(h, 10 ** 6, ptr(mean), ptr(m2))
        return h

    loss = np.zeros(1, np.float32)
    dt, hs = _concurrent(threads, setup, lambda h: R.ref_pupdate_step(h, loss.ctypes.data),
                         n_updates)
    for h in hs:
        R.ref_pupdate_destroy(h)
    sample = (f"{threads} concurrent PolicyLearnerCore-equivalent learners x {n_updates} "
              f"updates at B={B} ({cfg_name} dims, {nh}x{H}), reference AVX2 build")
    return threads * n_updates / dt, sample, threads


def cpu_baselines(cfg_name, critic_updates=2, policy_updates=1, actor_steps=20):
    model, ncpu = cpu_info()
    out = {}
    for key, fn, args, unit in (
            ("critic", reference_critic_rate, (cfg_name, critic_updates), "updates/s"),
            ("actor", reference_actor_rate, (cfg_name, actor_steps), "transitions/s"),
            ("policy", reference_policy_rate, (cfg_name, policy_updates), "updates/s")):
        rate, sample, cores = fn(*args)
        out[key] = ({"value": rate, "unit": unit, "cores": cores, "kind": "reference",
                     "sample": sample, "cpu": model, "host_cores": ncpu} if rate else None)
    return out


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank, world, local = dist_setup(args.gpus)
    D, A, H, nh, B, N, cap = CONFIGS[args.config]
    Bg = B  # the global batch of the headline (split B / world per rank for N > 1)
    prec = ["tf32 (fp32 storage, tf32 tensor-core products, fp32 accumulate)",
            "3xtf32 (fp32 storage, hi/lo tf32 split products, fp32 accumulate)"][args.precision]
    base = {"metric": METRIC, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": prec,
            "data": "synthetic (device-generated replay fill, SURVEY 8d distributions)",
            "config": {"workload": (f"{args.config}: CriticLearnerCore::update, obs {D} / act {A}, "
                                    f"{nh}x{H} MLPs, batch {Bg}, {cap} record replay"
                                    if world == 1 else
                                    f"c5 ({args.config} dims): data-parallel CriticLearnerCore::"
                                    f"update, global batch {Bg} split {Bg // world} per GPU over "
                                    f"{world} GPUs, {cap} record replay sharded {cap // world} "
                                    f"per GPU"),
                       "global_batch": Bg,
                       "parallelism": (f"dp{world}: NCCL all-reduce of the twin-critic "
                                       f"gradients + loss per update" if world > 1
                                       else "single GPU"),
                       "l2": "inputs sampled from an 8.9 GB ring (>> 126 MB L2)"}}
    if args.impl == "reference":
        if rank != 0:
            return
        # bounded sample per step: a full B=8192 update is ~1.3 s on one core
        t0 = time.perf_counter()
        n_upd = max(1, min(args.steps, 3))
        rate, sample, cores = reference_critic_rate(args.config, n_upd)
        if rate is None:
            print(json.dumps({"impl": "reference", "unavailable": sample}))
            return
        model, ncpu = cpu_info()
        out = dict(base)
        out.update(impl="reference", value=rate, ms_per_step=1e3 / rate,
                   cpu_baseline={"value": rate, "unit": "updates/s", "cores": cores,
                                 "kind": "reference", "sample": sample, "cpu": model,
                                 "host_cores": ncpu},
                   e2e={"value": rate, "unit": "updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0})
        arate, asample, acores = reference_actor_rate(args.config, 20)
        prate, psample, pcores = reference_policy_rate(args.config, 1)
        out["actor"] = {"value": arate, "unit": "transitions/s", "cores": acores,
                        "sample": asample}
        out["policy_updates"] = {"value": prate, "unit": "updates/s", "cores": pcores,
                                 "sample": psample}
        out["wall_s"] = round(time.perf_counter() - t0, 1)
        if world > 1:
            out["note"] = "rank 0 alone runs the reference's CPU path (other ranks exit)"
        print(json.dumps(out))
        return

    r = run_ours(args, rank, world, local, Bg // world)
    other_prec = None
    if world == 1:  # the same update in the other GEMM precision mode, beside the headline
        import argparse
        a2 = argparse.Namespace(**vars(args))
        a2.precision = 1 - args.precision
        p2 = run_ours(a2, rank, world, local, Bg, timed=False)
        other_prec = {"precision": ["tf32", "3xtf32"][a2.precision],
                      "value": 1e3 / p2["ms_step"], "unit": "updates/s",
                      "ms_per_step": p2["ms_step"],
                      "note": "3xtf32: the fp32-faithful parity mode (pqlg_config.precision)"}
    weak = None
    if world > 1:  # B = 8192 per GPU beside the strong-scaling headline
        w = run_ours(args, rank, world, local, Bg, timed=False)
        weak = {"value": world * args.steps / (w["ms_step"] * args.steps * 1e-3),
                "unit": "updates/s (batch-8192 updates: a dp-N update processes N x 8192 rows "
                        "and counts N)", "ms_per_step": w["ms_step"], "batch_per_gpu": Bg,
                "scaling": "weak"}
    actor = run_actor(args, rank, world, local, max(10, args.steps // 4),
                      max(3, args.warmup // 4), roofline=True)
    actor_c5 = run_actor(args, rank, world, local, max(10, args.steps // 4),
                         max(3, args.warmup // 4), n_envs=C5_ENVS // world)
    policy = run_policy(args, rank, world, local, args.steps, args.warmup)
    c51 = run_c51(args, rank, world, local, max(10, args.steps // 2), max(3, args.warmup // 2))
    sac = run_c51(args, rank, world, local, max(10, args.steps // 2), max(3, args.warmup // 2),
                  sac=True)
    pipe = run_pipeline(args, rank, world, local, 400)
    others = {c: run_other_config(args, rank, world, local, c, max(20, args.steps // 2),
                                  max(3, args.warmup // 2))
              for c in ("c2", "c1") if c != args.config}
    if rank != 0:
        return
    out = dict(base)
    value = args.steps / (r["ms_step"] * args.steps * 1e-3)
    out.update(value=value, ms_per_step=r["ms_step"], e2e=r["e2e"], roofline=r["roof"],
               clocks=r["clocks"], gpu_launches=r["launches"],
               kernels_per_update=r["kpu"], last_loss=r["loss"],
               batch_per_gpu=r["batch_per_rank"])
    if weak:
        out["weak_scaling"] = weak
    if other_prec:
        out["critic_other_precision"] = other_prec
    actor["workload"] = (f"{args.config}: rollout_step + V/P ingest, {N} envs per GPU "
                         f"(scaling: weak)")
    actor_c5["workload"] = (f"c5: rollout_step + V/P ingest, {C5_ENVS} envs over {world} GPU(s) "
                            f"({C5_ENVS // world} per GPU, sharded normalizer; scaling: strong)")
    out["actor"] = actor
    out["actor_c5"] = actor_c5
    out["policy_updates"] = policy
    out["c51"] = c51
    out["sac"] = sac
    out["run_parallel"] = pipe
    out["other_configs"] = others
    if world > 1:
        from paper_2307_12983_b200 import _lib  # noqa: F401
        out["nccl"] = {"ranks": world, "init_log": "NCCL_DEBUG=INFO INIT lines on stderr"}
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_baselines(args.config)
        out["cpu_baseline"] = cb["critic"]
        out["actor"]["cpu_baseline"] = cb["actor"]
        out["policy_updates"]["cpu_baseline"] = cb["policy"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
