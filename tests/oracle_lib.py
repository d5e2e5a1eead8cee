"""ctypes bindings of the CPU oracle (tests only).

- `orc()`  : oracle/_build/liboracle.so, the restatement (oracle/pql_oracle.c),
             built on demand with `make -C oracle`.
- `ref()`  : oracle/_ref/libpqlref.so, the reference itself compiled from
             /root/reference (present in the build container; travels to the
             GPU box as a built artefact).  None when unavailable.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE = ROOT / "oracle"
ORC_SO = ORACLE / "_build" / "liboracle.so"
REF_SO = ORACLE / "_ref" / "libpqlref.so"

vp, sz, i32, i64, u64, f32, f64 = (C.c_void_p, C.c_size_t, C.c_int, C.c_int64, C.c_uint64,
                                   C.c_float, C.c_double)

_ORC_SIGS = {
    "orc_splitmix64": (u64, [u64]),
    "orc_derive_seed": (u64, [u64, u64, u64]),
    "orc_mt64_seed": (None, [vp, u64]),
    "orc_mt64_next": (u64, [vp]),
    "orc_philox4x32_10": (None, [vp, vp, vp]),
    "orc_philox_draw": (u64, [u64, u64]),
    "orc_sample_indices_mt": (None, [vp, u64, sz, vp]),
    "orc_sample_indices_philox": (None, [u64, vp, u64, sz, vp]),
    "orc_nstep_create": (vp, [sz, sz, sz, f32, sz]),
    "orc_nstep_destroy": (None, [vp]),
    "orc_batch_create": (vp, [sz, sz]),
    "orc_batch_destroy": (None, [vp]),
    "orc_batch_clear": (None, [vp]),
    "orc_nstep_push_step": (None, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "orc_replay_create": (vp, [sz, sz, sz]),
    "orc_replay_destroy": (None, [vp]),
    "orc_replay_insert": (None, [vp, vp]),
    "orc_replay_gather": (None, [vp, vp, sz, vp, vp, vp, vp, vp]),
    "orc_states_create": (vp, [sz, sz]),
    "orc_states_destroy": (None, [vp]),
    "orc_states_insert": (None, [vp, vp, sz]),
    "orc_norm_stats_to_f32": (None, [i64, vp, vp, sz, vp, vp]),
    "orc_normalize_clip": (None, [vp, vp, vp, vp, sz, sz, f32]),
    "orc_normalize_apply": (None, [i64, vp, vp, vp, vp, sz, sz]),
    "orc_norm_update": (None, [vp, vp, vp, vp, sz, sz]),
    "orc_adam_bias_corrections": (None, [i64, vp, vp]),
    "orc_adam_update": (None, [vp, vp, vp, vp, sz, f32, f32, f32, f32, f32, f32]),
    "orc_sum_squares": (f64, [vp, sz]),
    "orc_clip_global_norm": (f32, [vp, sz, f32]),
    "orc_lerp_towards": (None, [vp, vp, sz, f32]),
    "orc_build_schedule": (None, [f32, f32, sz, vp]),
    "orc_apply_noise": (None, [vp, sz, sz, vp, f32, f32, vp]),
    "orc_glibc_logf": (f32, [f32]),
    "orc_mlp_param_count": (sz, [vp, sz]),
    "orc_mlp_forward": (None, [vp, vp, vp, sz, vp, sz, vp, vp]),
    "orc_mlp_backward": (None, [vp, vp, vp, sz, vp, vp, vp, sz, vp, vp]),
    "orc_policy_act": (None, [vp, vp, sz, vp, sz, f32, f32, vp]),
    "orc_ddpg_target": (i32, [vp, vp, vp, vp, vp, sz, vp, vp, vp, sz, sz, sz, f32, f32, vp]),
    "orc_ddpg_critic_loss": (i32, [vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, sz, sz,
                                   sz, f32, f32, vp, vp, vp, vp]),
    "orc_ddpg_actor_loss": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, sz, sz, f32, f32, vp, vp]),
    "orc_c51_atoms": (None, [sz, f32, f32, vp]),
    "orc_evaluate": (i32, [vp, vp, sz, i64, vp, vp, sz, u64, sz, sz, f32, f32, sz, vp, vp, vp]),
    "orc_c51_project": (i32, [vp, vp, vp, sz, sz, f32, f32, vp, vp]),
    "orc_c51_critic_loss": (i32, [vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, sz, sz,
                                  sz, f32, f32, sz, f32, f32, vp, vp, vp]),
    "orc_c51_actor_loss": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, sz, sz, f32, f32, sz, f32, f32,
                                 vp, vp]),
    "orc_normals": (None, [i32, vp, u64, vp, sz, vp]),
    "orc_norm_batch_stats": (None, [vp, sz, sz, vp, vp]),
    "orc_norm_merge": (None, [vp, vp, vp, sz, f64, vp, vp]),
    "orc_normals_rows": (None, [vp, sz, sz, vp]),
    "orc_gauss_sample": (i32, [vp, vp, sz, vp, vp, sz, f32, f32, vp, vp]),
    "orc_sac_critic_loss": (i32, [vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, sz, sz,
                                  sz, f32, f32, f32, vp, vp, vp, vp, vp]),
    "orc_sac_actor_loss": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, sz, sz, f32, f32, f32, vp, vp,
                                 vp, vp]),
    "orc_env_create": (vp, [sz, sz, sz, u64, sz]),
    "orc_env_destroy": (None, [vp]),
    "orc_env_observe": (None, [vp, vp]),
    "orc_env_step": (i32, [vp, vp, vp, vp, vp, vp, vp]),
}

_REF_SIGS = {
    "ref_derive_seed": (u64, [u64, u64, u64]),
    "ref_mt64_draws": (None, [u64, sz, vp]),
    "ref_sample_indices": (None, [u64, u64, u64, sz, sz, vp]),
    "ref_nstep_replay": (sz, [sz, sz, sz, sz, f32, sz, sz, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                              vp, vp, vp, sz, vp, vp, vp]),
    "ref_state_buffer": (None, [sz, sz, sz, sz, vp, u64, sz, sz, vp, vp]),
    "ref_normalizer": (None, [sz, sz, vp, vp, vp, vp, vp, vp, sz, vp]),
    "ref_normalize_apply": (None, [i64, vp, vp, sz, vp, sz, vp]),
    "ref_adam_step": (i32, [vp, vp, vp, vp, sz, i64, f32]),
    "ref_clip_global_norm": (None, [vp, sz, f32]),
    "ref_sum_squares": (f64, [vp, sz]),
    "ref_soft_update": (None, [vp, vp, sz, f32]),
    "ref_build_schedule": (None, [f32, f32, sz, vp]),
    "ref_apply_noise": (None, [f32, f32, sz, sz, u64, sz, f32, f32, vp]),
    "ref_mlp_forward": (None, [vp, vp, sz, vp, sz, vp]),
    "ref_mlp_backward": (None, [vp, vp, sz, vp, vp, sz, vp, vp]),
    "ref_init_mlp": (None, [vp, sz, u64, f32, f32, sz, vp]),
    "ref_policy_init": (None, [sz, sz, sz, u64, vp]),
    "ref_ddpg_critic_loss": (i32, [vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, sz, sz,
                                   sz, f32, f32, vp, vp, vp, vp]),
    "ref_ddpg_actor_loss": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, sz, f32, f32, vp, vp]),
    "ref_c51_project": (i32, [vp, vp, vp, sz, sz, f32, f32, vp]),
    "ref_c51_atoms": (None, [sz, f32, f32, vp]),
    "ref_c51_critic_loss": (i32, [vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, sz, sz,
                                  sz, f32, f32, sz, f32, f32, vp, vp, vp]),
    "ref_c51_actor_loss": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, sz, f32, f32, sz, f32, f32, vp,
                                 vp]),
    "ref_vcore_snapshot": (None, [vp, i64, vp, vp]),
    "ref_pcore_create": (vp, [sz, sz, sz, sz, sz, u64, u64, i32]),
    "ref_pcore_destroy": (None, [vp]),
    "ref_pcore_ingest": (None, [vp, vp, sz]),
    "ref_pcore_ready": (i32, [vp, i64]),
    "ref_pcore_buffer_size": (sz, [vp]),
    "ref_pcore_adopt_norm": (None, [vp, i64, vp, vp]),
    "ref_pcore_adopt_critics": (None, [vp, vp, vp, i64]),
    "ref_pcore_update": (i32, [vp, vp]),
    "ref_pcore_snapshot": (sz, [vp, i64, vp, vp]),
    "ref_sample_indices_philox": (u64, [u64, u64, u64, sz, vp]),
    "ref_ratio_may_proceed": (i32, [i32, i64, i64, i64, f64, f64, f64, f64, f64, i64, i32]),
    "ref_set_backend": (None, [i32]),
    "ref_active_backend": (i32, []),
    "ref_synth_env_create": (vp, [sz, sz, sz, u64, sz, f32, f32, i32, vp]),
    "ref_synth_env_destroy": (None, [vp]),
    "ref_synth_env_step": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "ref_synth_env_episode_steps": (None, [vp, vp]),
    "ref_actor_core_create": (vp, [sz, sz, sz, sz, u64, f64, f64, f64, sz, i32]),
    "ref_actor_core_destroy": (None, [vp]),
    "ref_actor_core_step": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "ref_actor_core_norm": (None, [vp, vp, vp, vp]),
    "ref_actor_core_policy": (sz, [vp, vp]),
    "ref_actor_core_episode_steps": (None, [vp, vp]),
    "ref_evaluate_synth": (i32, [vp, vp, sz, i32, i64, vp, vp, sz, u64, sz, f32, f32, vp, vp]),
    "ref_vupdate_create": (vp, [sz, sz, sz, sz, sz, sz, u64, vp, vp, vp, i32, sz, f32, f32]),
    "ref_vupdate_destroy": (None, [vp]),
    "ref_vupdate_insert": (None, [vp, vp, vp, vp, vp, vp, sz]),
    "ref_vupdate_adopt_norm": (None, [vp, i64, vp, vp]),
    "ref_vupdate_step": (i32, [vp, vp]),
    "ref_vupdate_params": (None, [vp, i32, vp]),
    "ref_vupdate_set_log_alpha": (None, [vp, f32]),
    "ref_pupdate_log_alpha": (f32, [vp]),
    "ref_actor_create_sac": (vp, [sz, sz, sz, sz, sz, u64, vp]),
    "ref_normals": (None, [u64, u64, u64, sz, vp]),
    "ref_gauss_sample": (i32, [vp, vp, sz, vp, vp, sz, vp, vp, vp, vp, vp]),
    "ref_pupdate_create": (vp, [sz, sz, sz, sz, sz, sz, u64, vp, vp, vp, i32, sz, f32, f32]),
    "ref_pupdate_destroy": (None, [vp]),
    "ref_pupdate_insert": (None, [vp, vp, sz]),
    "ref_pupdate_adopt_norm": (None, [vp, i64, vp, vp]),
    "ref_pupdate_step": (i32, [vp, vp]),
    "ref_pupdate_params": (None, [vp, vp]),
    "ref_actor_create": (vp, [sz, sz, sz, sz, sz, u64, vp, f32, f32]),
    "ref_actor_destroy": (None, [vp]),
    "ref_actor_act": (None, [vp, vp, vp]),
    "ref_actor_observe": (None, [vp, vp]),
    "ref_actor_stats": (None, [vp, vp, vp, vp]),
    "ref_vcore_create": (vp, [sz, sz, sz, sz, sz, sz, u64, u64, f32, i32]),
    "ref_vcore_destroy": (None, [vp]),
    "ref_vcore_ingest": (None, [vp, vp, vp, vp, vp, vp, vp]),
    "ref_vcore_ready": (i32, [vp, i64]),
    "ref_vcore_buffer_size": (sz, [vp]),
    "ref_vcore_adopt_norm": (None, [vp, i64, vp, vp]),
    "ref_vcore_adopt_policy": (None, [vp, vp, i64]),
    "ref_vcore_update": (i32, [vp, vp]),
    "ref_vcore_params": (None, [vp, i32, vp]),
    "ref_metrics_write": (i32, [C.c_char_p, vp, sz]),
    "ref_checkpoint_save": (i32, [C.c_char_p, i32, vp, vp, vp, vp, i64, vp, vp, sz]),
    "ref_checkpoint_load": (i32, [C.c_char_p, vp, C.POINTER(sz), C.POINTER(i64), vp, vp, C.POINTER(sz)]),
}

_orc = None
_ref = None
_ref_b200 = None
REF_B200_SO = ORACLE / "_ref" / "libpqlref_b200.so"


def _bind(path: Path, sigs: dict) -> C.CDLL:
    lib = C.CDLL(str(path))
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORC_SO.exists():
            subprocess.run(["make", "-C", str(ORACLE)], check=True, capture_output=True)
        _orc = _bind(ORC_SO, _ORC_SIGS)
    return _orc


def ref():
    """The compiled reference, or None if it was not built here."""
    global _ref
    if _ref is None and REF_SO.exists():
        _ref = _bind(REF_SO, _REF_SIGS)
    return _ref


def ref_b200():
    """The reference with its runtime cores bound to libpqlg.so (oracle/Makefile
    b200: learners.hpp/.cpp patched at build time under PQL_B200), driven by
    the same ref_* entry points; None if it was not built."""
    global _ref_b200
    if _ref_b200 is None and REF_B200_SO.exists():
        _ref_b200 = _bind(REF_B200_SO, _REF_SIGS)
    return _ref_b200


def ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the oracle must be contiguous"
    return a.ctypes.data_as(C.c_void_p)


def sizes_arr(sizes) -> np.ndarray:
    return np.asarray(sizes, dtype=np.uintp)


def acts_arr(n_layers: int) -> np.ndarray:
    a = np.ones(n_layers, dtype=np.uint8)
    a[-1] = 0
    return a


def param_count(sizes) -> int:
    return int(sum(sizes[i] * sizes[i + 1] + sizes[i + 1] for i in range(len(sizes) - 1)))


class MT64:
    """Restated std::mt19937_64 (oracle)."""

    def __init__(self, seed: int):
        self._state = C.create_string_buffer(312 * 8 + 8)
        orc().orc_mt64_seed(self._state, seed)

    @property
    def handle(self):
        return self._state

    def __call__(self) -> int:
        return orc().orc_mt64_next(self._state)


def traj_hash(x) -> np.uint64:
    """Order-sensitive 64-bit digest of a float32 array's bit patterns (the
    golden fixtures store it where a full trajectory would be megabytes)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64).ravel()
    w = np.arange(1, b.size + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    return np.bitwise_xor.reduce(b * w) if b.size else np.uint64(0)


def derive_seed(master: int, stream: int, index: int) -> int:
    return orc().orc_derive_seed(master, stream, index)


STREAM_ENV, STREAM_NOISE, STREAM_INIT, STREAM_SAMPLE = 1, 2, 3, 4
STREAM_SAC = 6
