"""Checkpoints in the reference's format: the
library's writer (pqlg_checkpoint_write) produces byte-identical files to the
reference's fa::save_checkpoint (tests/golden/ckpt_ref.bin, made by
oracle/make_golden.py from the compiled reference), and each side reads the
other's files.  Host code only: no GPU needed."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import ptr
from paper_2307_12983_b200 import _lib

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
from make_golden import ckpt_content  # noqa: E402


def write_ours(path, nets, flats, count, mean, m2):
    names = (C.c_char_p * len(nets))(*[n.encode() for n, _ in nets])
    nl = np.array([len(sz) - 1 for _, sz in nets], np.int32)
    szs = [np.array(sz, np.int32) for _, sz in nets]
    szp = (C.c_void_p * len(nets))(*[a.ctypes.data for a in szs])
    fp = (C.c_void_p * len(nets))(*[a.ctypes.data for a in flats])
    _lib.call("pqlg_checkpoint_write", str(path).encode(), len(nets), names, nl.ctypes.data, szp,
              fp, count, ptr(mean), ptr(m2), len(mean))


def read_ours(path):
    n, npar, cnt, dim = C.c_int(), C.c_int64(), C.c_int64(), C.c_int()
    _lib.call("pqlg_checkpoint_read", str(path).encode(), C.byref(n), C.byref(npar), None,
              C.byref(cnt), None, None, C.byref(dim))
    flat = np.zeros(npar.value, np.float32)
    mean = np.zeros(dim.value)
    m2 = np.zeros(dim.value)
    _lib.call("pqlg_checkpoint_read", str(path).encode(), C.byref(n), C.byref(npar), ptr(flat),
              C.byref(cnt), ptr(mean), ptr(m2), C.byref(dim))
    return n.value, flat, cnt.value, mean, m2


def test_writer_is_byte_identical_to_reference(tmp_path):
    nets, flats, count, mean, m2 = ckpt_content()
    p = tmp_path / "ours.bin"
    write_ours(p, nets, flats, count, mean, m2)
    assert p.read_bytes() == (GOLDEN / "ckpt_ref.bin").read_bytes()


def test_reader_reads_reference_file():
    nets, flats, count, mean, m2 = ckpt_content()
    n, flat, cnt, mu, s2 = read_ours(GOLDEN / "ckpt_ref.bin")
    assert n == 3 and cnt == count
    assert np.array_equal(flat, np.concatenate(flats))
    assert np.array_equal(mu, mean) and np.array_equal(s2, m2)


def test_reference_reads_our_file(tmp_path):
    from oracle_lib import ref
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    nets, flats, count, mean, m2 = ckpt_content(seed=21)
    p = tmp_path / "ours.bin"
    write_ours(p, nets, flats, count, mean, m2)
    npar, cnt, dim = C.c_size_t(), C.c_int64(), C.c_size_t()
    assert R.ref_checkpoint_load(str(p).encode(), None, C.byref(npar), C.byref(cnt), None, None,
                                 C.byref(dim)) == 3
    flat = np.zeros(npar.value, np.float32)
    mu, s2 = np.zeros(dim.value), np.zeros(dim.value)
    assert R.ref_checkpoint_load(str(p).encode(), ptr(flat), C.byref(npar), C.byref(cnt), ptr(mu),
                                 ptr(s2), C.byref(dim)) == 3
    assert cnt.value == count and np.array_equal(flat, np.concatenate(flats))
    assert np.array_equal(mu, mean) and np.array_equal(s2, m2)


def test_bad_files_are_rejected(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTACKPT" + b"\0" * 32)
    with pytest.raises(ValueError):
        read_ours(p)
    good = (GOLDEN / "ckpt_ref.bin").read_bytes()
    (tmp_path / "trunc.bin").write_bytes(good[:100])
    with pytest.raises(ValueError):
        read_ours(tmp_path / "trunc.bin")
