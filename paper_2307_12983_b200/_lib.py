"""ctypes binding of libpqlg.so (the C ABI in include/pqlg.h).

There is deliberately no fallback: if the library or a CUDA device is
missing, the first call raises.  Signatures are declared once here so the
Python mirror classes and the tests call through the exact C ABI.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# PQLG_LIB_VARIANT=name loads libpqlg_<name>.so (an in-tree A/B build of the
# same sources with extra nvcc flags, tools/build_variant.sh); default: the product
_VARIANT = os.environ.get("PQLG_LIB_VARIANT", "")
LIB_PATH = _PKG / (f"libpqlg_{_VARIANT}.so" if _VARIANT else "libpqlg.so")

PQLG_OK, PQLG_NOT_READY = 0, 1
PQLG_EINVAL, PQLG_ENONFINITE, PQLG_ECUDA, PQLG_ENCCL = -1, -2, -3, -4

vp, i32, i64, u64, f32, f64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_float, C.c_double


class StepSlice(C.Structure):
    """pqlg_step_slice (device views of a StepSlice)."""
    _fields_ = [("obs", vp), ("act", vp), ("boot_obs", vp), ("rew", vp), ("term", vp),
                ("trunc", vp), ("ld_obs", i64), ("ld_act", i64)]


class NStepBatch(C.Structure):
    """pqlg_nstep_batch (device views of an NStepBatch)."""
    _fields_ = [("obs", vp), ("act", vp), ("boot_obs", vp), ("ret", vp), ("eff_disc", vp),
                ("ld_obs", i64), ("ld_act", i64)]


class NormStats(C.Structure):
    """pqlg_norm_stats (host NormStats)."""
    _fields_ = [("count", i64), ("mean", vp), ("m2", vp)]


class Rng(C.Structure):
    """pqlg_rng: Philox (key, counter) or explicit host indices."""
    _fields_ = [("mode", i32), ("key", u64), ("counter", u64), ("host_indices", vp)]


RNG_PHILOX, RNG_INDICES = 0, 1
ALGO_DDPG, ALGO_C51, ALGO_SAC = 0, 1, 2
PREC_TF32, PREC_3XTF32 = 0, 1
P = C.POINTER


class Config(C.Structure):
    """pqlg_config: the RunConfig fields the cores consume (config.hpp:15-48)."""
    _fields_ = [("algo", i32), ("n_envs", i32), ("batch_size", i32), ("buffer_capacity", u64),
                ("gamma", f64), ("tau", f64), ("n_step", i32), ("lr_actor", f64),
                ("lr_critic", f64), ("warm_up", i64), ("sigma_min", f64), ("sigma_max", f64),
                ("sigma_fixed", f64), ("reward_scale", f64), ("seed", u64), ("hidden", i32),
                ("hidden_layers", i32), ("n_atoms", i32), ("vmin", f64), ("vmax", f64),
                ("max_episode_len", i32), ("env_offset", i32), ("envs_total", i32),
                ("precision", i32)]


class TaskDims(C.Structure):
    """pqlg_task_dims (learners.hpp:23-26)."""
    _fields_ = [("obs_dim", i32), ("act_dim", i32), ("low", f32), ("high", f32)]

class RatioConfig(C.Structure):
    """pqlg_ratio_config (RatioConfig, ratio_gate.hpp:17-25 + SPEC.md:486-492)."""
    _fields_ = [("beta_av", C.c_double), ("beta_pv", C.c_double), ("slack_a", C.c_double),
                ("slack_p", C.c_double), ("slack_v", C.c_double), ("warm_up", i64),
                ("free_running", i32), ("horizon", i32), ("channel_capacity", i32),
                ("publish_every", i32)]


class RunReport(C.Structure):
    """pqlg_run_report (RunReport, run.hpp:11-31)."""
    _fields_ = [("ok", i32), ("c_a", i64), ("c_v", i64), ("c_p", i64), ("env_steps", i64),
                ("wall_s", C.c_double), ("ratio_av", C.c_double), ("ratio_pv", C.c_double),
                ("batches_sent", i64), ("batches_consumed_v", i64), ("batches_consumed_p", i64),
                ("seq_duplicates", i64), ("seq_gaps", i64), ("max_policy_staleness", i64),
                ("policy_version", i64), ("critic_version", i64),
                ("last_critic_loss", f32), ("last_actor_loss", f32)]


class MetricsRow(C.Structure):
    """pqlg_metrics_row (MetricsRow, metrics.hpp:9-15)."""
    _fields_ = [("wall_clock_s", C.c_double), ("env_steps", i64), ("c_a", i64), ("c_v", i64),
                ("c_p", i64), ("eval_return_mean", C.c_double),
                ("eval_return_stderr", C.c_double), ("critic_loss_ema", C.c_double),
                ("actor_loss_ema", C.c_double)]


class MetricsConfig(C.Structure):
    """pqlg_metrics_config: the evaluator + metrics writer of a run."""
    _fields_ = [("path", C.c_char_p), ("interval_s", C.c_double), ("every_actor_steps", i64),
                ("eval_episodes", i32), ("eval_seed", u64), ("ema", C.c_double)]


PROC_ACTOR, PROC_VLEARNER, PROC_PLEARNER = 0, 1, 2

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "pqlg_last_error": (C.c_char_p, []),
    "pqlg_abi_version": (i32, []),
    "pqlg_launch_count": (u64, []),
    "pqlg_profile_begin": (i32, []),
    "pqlg_profile_end": (i32, [C.c_char_p, i32]),
    "pqlg_k_gemm_tf32": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                               i32, vp]),
    "pqlg_replay_create": (i32, [u64, i32, i32, vp, P(vp)]),
    "pqlg_replay_destroy": (i32, [vp]),
    "pqlg_replay_size": (i32, [vp, P(u64)]),
    "pqlg_replay_cursor": (i32, [vp, P(u64)]),
    "pqlg_replay_insert": (i32, [vp, P(NStepBatch), u64]),
    "pqlg_replay_sample": (i32, [vp, u64, P(Rng), u64, P(NormStats), P(NStepBatch)]),
    "pqlg_replay_read_rows": (i32, [vp, u64, u64, vp, vp, vp, vp, vp]),
    "pqlg_nstep_create": (i32, [i32, i32, i32, f32, i32, vp, P(vp)]),
    "pqlg_nstep_destroy": (i32, [vp]),
    "pqlg_nstep_push_step": (i32, [vp, P(StepSlice), f32, vp]),
    "pqlg_states_create": (i32, [u64, i32, vp, P(vp)]),
    "pqlg_states_destroy": (i32, [vp]),
    "pqlg_states_size": (i32, [vp, P(u64)]),
    "pqlg_states_insert": (i32, [vp, vp, i64, u64]),
    "pqlg_states_sample": (i32, [vp, u64, P(Rng), u64, P(NormStats), vp, i64]),
    "pqlg_config_default": (None, [P(Config)]),
    "pqlg_comm_unique_id": (i32, [vp]),
    "pqlg_comm_init": (i32, [i32, i32, vp, P(vp)]),
    "pqlg_comm_destroy": (i32, [vp]),
    "pqlg_comm_rank": (i32, [vp, P(i32), P(i32)]),
    "pqlg_comm_allreduce_f32": (i32, [vp, vp, u64, vp]),
    "pqlg_vlearner_create": (i32, [P(Config), P(TaskDims), u64, vp, P(vp)]),
    "pqlg_vlearner_create_dp": (i32, [P(Config), P(TaskDims), u64, vp, vp, P(vp)]),
    "pqlg_vlearner_destroy": (i32, [vp]),
    "pqlg_vlearner_adopt_policy": (i32, [vp, vp, i64]),
    "pqlg_vlearner_adopt_policy_sac": (i32, [vp, vp, f32, i64]),
    "pqlg_vlearner_log_alpha": (i32, [vp, P(f32)]),
    "pqlg_vlearner_adopt_norm": (i32, [vp, P(NormStats)]),
    "pqlg_vlearner_ingest": (i32, [vp, P(StepSlice)]),
    "pqlg_vlearner_ingest_host": (i32, [vp, P(StepSlice)]),
    "pqlg_vlearner_ready": (i32, [vp, i64, P(i32)]),
    "pqlg_vlearner_update": (i32, [vp, P(f32)]),
    "pqlg_vlearner_update_n": (i32, [vp, i32]),
    "pqlg_vlearner_last_loss": (i32, [vp, P(f32)]),
    "pqlg_vlearner_get_params": (i32, [vp, i32, vp]),
    "pqlg_vlearner_param_count": (i32, [vp, i32, P(i64)]),
    "pqlg_vlearner_snapshot": (i32, [vp, vp, vp]),
    "pqlg_vlearner_buffer_size": (i32, [vp, P(u64)]),
    "pqlg_vlearner_set_sampler": (i32, [vp, i32]),
    "pqlg_vlearner_replay": (i32, [vp, P(vp)]),
    "pqlg_vlearner_set_params": (i32, [vp, i32, vp]),
    "pqlg_vlearner_debug_read": (i32, [vp, i32, vp]),
    "pqlg_vlearner_kernels_per_update": (i32, [vp, P(i32)]),
    "pqlg_replay_fill_synthetic": (i32, [vp, u64, u64, f32, C.c_uint32]),
    "pqlg_k_gemm_tf32_repeat": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                      vp]),
    "pqlg_k_gemm_tf32_repeat_groups": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32,
                                             i32, vp]),
    "pqlg_plearner_create": (i32, [P(Config), P(TaskDims), u64, vp, P(vp)]),
    "pqlg_plearner_create_dp": (i32, [P(Config), P(TaskDims), u64, vp, vp, P(vp)]),
    "pqlg_plearner_destroy": (i32, [vp]),
    "pqlg_plearner_adopt_critics": (i32, [vp, vp, vp, i64]),
    "pqlg_plearner_adopt_norm": (i32, [vp, P(NormStats)]),
    "pqlg_plearner_ingest": (i32, [vp, vp, i64, u64]),
    "pqlg_plearner_ingest_host": (i32, [vp, vp, i64, u64]),
    "pqlg_plearner_ready": (i32, [vp, i64, P(i32)]),
    "pqlg_plearner_update": (i32, [vp, P(f32)]),
    "pqlg_plearner_update_n": (i32, [vp, i32]),
    "pqlg_plearner_last_loss": (i32, [vp, P(f32)]),
    "pqlg_plearner_snapshot": (i32, [vp, vp]),
    "pqlg_plearner_get_params": (i32, [vp, i32, vp]),
    "pqlg_plearner_set_params": (i32, [vp, i32, vp]),
    "pqlg_plearner_param_count": (i32, [vp, i32, P(i64)]),
    "pqlg_plearner_log_alpha": (i32, [vp, P(f32)]),
    "pqlg_plearner_buffer_size": (i32, [vp, P(u64)]),
    "pqlg_plearner_set_sampler": (i32, [vp, i32]),
    "pqlg_plearner_kernels_per_update": (i32, [vp, P(i32)]),
    "pqlg_actor_create": (i32, [P(Config), P(TaskDims), vp, P(vp)]),
    "pqlg_actor_create_sharded": (i32, [P(Config), P(TaskDims), vp, vp, P(vp)]),
    "pqlg_actor_step_event": (i32, [vp, P(vp)]),
    "pqlg_vlearner_wait_event": (i32, [vp, vp]),
    "pqlg_actor_wait_event": (i32, [vp, vp]),
    "pqlg_vlearner_record_event": (i32, [vp, P(vp)]),
    "pqlg_plearner_record_event": (i32, [vp, P(vp)]),
    "pqlg_plearner_wait_event": (i32, [vp, vp]),
    "pqlg_actor_destroy": (i32, [vp]),
    "pqlg_actor_adopt_policy": (i32, [vp, vp, i64]),
    "pqlg_actor_rollout_step": (i32, [vp, P(StepSlice)]),
    "pqlg_actor_rollout_n": (i32, [vp, i32]),
    "pqlg_actor_norm": (i32, [vp, P(i64), vp, vp]),
    "pqlg_actor_policy_version": (i32, [vp, P(i64)]),
    "pqlg_actor_read": (i32, [vp, i32, vp]),
    "pqlg_actor_kernels_per_step": (i32, [vp, P(i32)]),
    "pqlg_checkpoint_write": (i32, [C.c_char_p, i32, vp, vp, vp, vp, i64, vp, vp, i32]),
    "pqlg_checkpoint_read": (i32, [C.c_char_p, P(i32), P(i64), vp, P(i64), vp, vp, P(i32)]),
    "pqlg_vlearner_save": (i32, [vp, C.c_char_p]),
    "pqlg_vlearner_load": (i32, [vp, C.c_char_p]),
    "pqlg_plearner_save": (i32, [vp, C.c_char_p]),
    "pqlg_plearner_load": (i32, [vp, C.c_char_p]),
    "pqlg_actor_save": (i32, [vp, C.c_char_p]),
    "pqlg_actor_load": (i32, [vp, C.c_char_p]),
    "pqlg_evaluate": (i32, [P(Config), P(TaskDims), vp, P(NormStats), i32, u64, vp, P(f64),
                            P(f64)]),
    "pqlg_ratio_config_default": (None, [P(RatioConfig)]),
    "pqlg_ratio_may_proceed": (i32, [i32, i64, i64, i64, P(RatioConfig)]),
    "pqlg_pipeline_create": (i32, [P(Config), P(TaskDims), P(RatioConfig), u64, P(vp)]),
    "pqlg_pipeline_run": (i32, [vp, i64, C.c_double, P(RunReport)]),
    "pqlg_pipeline_destroy": (i32, [vp]),
    "pqlg_vlearner_time_update": (i32, [vp, i32, C.c_char_p, i32]),
    "pqlg_plearner_time_update": (i32, [vp, i32, C.c_char_p, i32]),
    "pqlg_actor_time_steps": (i32, [vp, i32, C.c_char_p, i32]),
    "pqlg_actor_read_slice": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "pqlg_k_sample_indices": (i32, [u64, P(u64), u64, u64, vp, P(C.c_uint32)]),
    "pqlg_pipeline_record_snapshots": (i32, [vp, i32]),
    "pqlg_pipeline_check_critics": (i32, [vp, P(i64), P(C.c_double)]),
    "pqlg_pipeline_set_metrics": (i32, [vp, P(MetricsConfig)]),
    "pqlg_run_synchronous": (i32, [P(Config), P(TaskDims), P(RatioConfig), u64, i64,
                                   P(MetricsConfig), P(RunReport)]),
    "pqlg_metrics_header": (C.c_char_p, []),
    "pqlg_metrics_open": (i32, [C.c_char_p, P(vp)]),
    "pqlg_metrics_append": (i32, [vp, P(MetricsRow)]),
    "pqlg_metrics_close": (i32, [vp]),
    "pqlg_metrics_config_default": (None, [P(MetricsConfig)]),
    "pqlg_env_create": (i32, [i32, i32, i32, u64, i32, i32, f32, f32, vp, P(vp)]),
    "pqlg_env_destroy": (i32, [vp]),
    "pqlg_env_reset_all": (i32, [vp, vp, i64]),
    "pqlg_env_step": (i32, [vp, vp, i64, vp, vp, vp, vp, vp, i64]),
    "pqlg_k_apply_noise": (i32, [vp, i64, i32, i32, vp, f32, f32, vp, vp]),
    "pqlg_k_evaluate_seq": (i32, [P(Config), P(TaskDims), vp, i32, P(NormStats), i32, u64, vp,
                                  vp, vp]),
    "pqlg_k_normalizer_update": (i32, [vp, vp, vp, vp, i64, i32, i32, vp, vp, vp]),
}


def default_config(**overrides) -> Config:
    cfg = Config()
    lib().pqlg_config_default(C.byref(cfg))
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


class PqlgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class NotReady(PqlgError):
    pass


class NonFinite(PqlgError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -m paper_2307_12983_b200.build` "
                "(there is no CPU fallback)")
        # libpqlg.so links NCCL by its SONAME (libnccl.so.2).  Load torch's
        # bundled NCCL first when torch is present: otherwise the system
        # libnccl.so.2 (older) would claim that SONAME and a later
        # `import torch` could not resolve its newer NCCL symbols.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().pqlg_last_error().decode()


def check(status: int) -> int:
    """Maps a PQLG status to the reference's exception convention."""
    if status == PQLG_OK:
        return status
    msg = last_error()
    if status == PQLG_NOT_READY:
        raise NotReady(status, msg)
    if status == PQLG_EINVAL:
        raise ValueError(msg)
    if status == PQLG_ENONFINITE:
        raise NonFinite(status, msg)
    raise PqlgError(status, msg)


def call(name: str, *args) -> int:
    return check(getattr(lib(), name)(*args))


COMM_ID_BYTES = 128


def exchange_comm_id(rank: int, world: int) -> bytes:
    """Rank 0 makes the NCCL unique id (pqlg_comm_unique_id); torch.distributed
    (any backend, gloo included) broadcasts the 128 bytes to every rank."""
    import torch
    import torch.distributed as dist
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    if rank == 0:
        call("pqlg_comm_unique_id", buf)
    t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    if world > 1:
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def comm_from_torch_dist(rank: int, world: int) -> C.c_void_p:
    """NCCL communicator for this process (one rank per GPU, its CUDA device
    current): the id exchange above, then pqlg_comm_init."""
    ident = (C.c_uint8 * COMM_ID_BYTES)(*exchange_comm_id(rank, world))
    comm = C.c_void_p()
    call("pqlg_comm_init", rank, world, ident, C.byref(comm))
    return comm


def metrics_config(path: str, **overrides) -> MetricsConfig:
    m = MetricsConfig()
    lib().pqlg_metrics_config_default(C.byref(m))
    m.path = path.encode()
    for k, v in overrides.items():
        setattr(m, k, v)
    return m


def ratio_config(**overrides) -> RatioConfig:
    rc = RatioConfig()
    lib().pqlg_ratio_config_default(C.byref(rc))
    for k, v in overrides.items():
        setattr(rc, k, v)
    return rc


def time_graph(fn: str, h, reps: int = 20):
    """In-graph per-kernel device times (pqlg_*_time_update / _time_steps):
    returns ([(kernel, ms, shape), ...] in launch order, graph_ms)."""
    buf = C.create_string_buffer(1 << 20)
    call(fn, h, reps, buf, len(buf))
    rows, graph_ms = [], None
    for line in buf.value.decode().splitlines():
        name, ms, shape = (line.split("\t") + ["", ""])[:3]
        if name == "__graph__":
            graph_ms = float(ms)
        else:
            rows.append((name, float(ms), shape))
    return rows, graph_ms
