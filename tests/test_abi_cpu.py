"""CPU-side checks of the drop-in boundary: the C-ABI library builds/loads,
exports every symbol include/pqlg.h declares, the Python binding declares a
signature for each, and the product never reaches into the oracle."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pqlg.h"
LIB = ROOT / "paper_2307_12983_b200" / "libpqlg.so"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"PQLG_API\s+[\w\s\*]+?\b(pqlg_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_2307_12983_b200 import build
        build.build()
    return C.CDLL(str(LIB))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["pqlg_replay_create", "pqlg_replay_sample", "pqlg_nstep_push_step",
                 "pqlg_states_insert", "pqlg_vlearner_create", "pqlg_vlearner_update",
                 "pqlg_vlearner_update_n", "pqlg_k_gemm_tf32"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (pqlg_\w+)", out))
    assert set(declared()) <= exported
    # nothing beyond the ABI leaks (hidden visibility)
    assert all(n.startswith("pqlg_") for n in exported)


def test_python_binding_covers_the_header():
    from paper_2307_12983_b200 import _lib
    assert set(declared()) <= set(_lib.SIGNATURES), set(declared()) - set(_lib.SIGNATURES)


def test_abi_without_gpu_fails_loudly_not_silently(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2307_12983_b200 import _lib
    h = C.c_void_p()
    with pytest.raises(_lib.PqlgError) as e:
        _lib.call("pqlg_replay_create", 16, 4, 2, None, C.byref(h))
    assert e.value.status == _lib.PQLG_ECUDA


def test_config_defaults_match_reference_runconfig(lib):
    from paper_2307_12983_b200 import _lib
    c = _lib.default_config()
    # config.hpp:15-48 (Table B.1)
    assert (c.batch_size, c.buffer_capacity, c.n_step, c.warm_up) == (8192, 5_000_000, 3, 32)
    assert (c.gamma, c.tau, c.lr_actor, c.lr_critic) == (0.99, 0.05, 5e-4, 5e-4)
    assert (c.sigma_min, c.sigma_max, c.n_atoms, c.vmin, c.vmax) == (0.05, 0.8, 51, -10.0, 10.0)


def test_product_does_not_touch_the_oracle():
    pkg = ROOT / "paper_2307_12983_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + \
            list(pkg.rglob("*.h")):
        text = p.read_text()
        assert "oracle" not in text.lower().replace("oracle (", ""), p
        assert "libpqlref" not in text and "/root/reference" not in text, p


def test_cpp_layer_compiles_and_maps_errors(tmp_path):
    """include/pqlg.hpp (the C++ layer a reference build would include, see
    INTEGRATION.md) compiles against the library and maps ABI statuses to the
    reference's exception types; without a GPU, construction must throw
    std::runtime_error (no CPU fallback)."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include "pqlg.hpp"
int main(int argc, char**) {
  if (pqlg_abi_version() <= 0) return 2;
  pqlg_config cfg; pqlg_config_default(&cfg);
  pqlg_task_dims dims{4, 2, -1.0f, 1.0f};
  cfg.batch_size = -1;
  try { pqlg::VLearner v(cfg, dims, 1); return 3; }
  catch (const std::invalid_argument&) { std::puts("einval"); }
  catch (const std::runtime_error&) { std::puts("runtime"); }
  return 0;
}
''')
    lib = ROOT / "paper_2307_12983_b200"
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(src),
                    f"-L{lib}", "-lpqlg", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out
    assert out.stdout.strip() in ("einval", "runtime")


def test_evaluate_rejects_zero_episodes_without_a_gpu():
    """evaluate_policy throws invalid_argument for episodes < 1
    (learners.cpp:282) before any device work."""
    import ctypes as C
    import numpy as np
    from paper_2307_12983_b200 import _lib
    cfg = _lib.default_config(hidden=32, hidden_layers=2)
    dims = _lib.TaskDims(4, 2, -1.0, 1.0)
    pol = np.zeros(1000, np.float32)
    m = np.zeros(4)
    ns = _lib.NormStats(0, m.ctypes.data, m.ctypes.data)
    mu, se = C.c_double(), C.c_double()
    rc = _lib.lib().pqlg_evaluate(C.byref(cfg), C.byref(dims), pol.ctypes.data, C.byref(ns), 0, 1,
                                  None, C.byref(mu), C.byref(se))
    assert rc == -1  # PQLG_EINVAL
