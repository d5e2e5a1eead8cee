"""The Philox sampling contract on CPU: the restatement's
orc_sample_indices_philox against libstdc++'s own
std::uniform_int_distribution<size_t> -- the call ReplayBuffer::sample makes
(replay_buffer.hpp:58-60) -- driven by a Philox4x32-10 URBG inside the
compiled reference (ref_sample_indices_philox, oracle/ref_harness.cpp):
identical indices and counter advance, including live counts where most
draws fall in Lemire's rejection zone.  test_replay_gpu.py checks the
device sampler against the same function."""
import numpy as np
import pytest

from oracle_lib import orc, ptr, ref

CASES = [  # count, batch
    (1, 8), (100, 64), (5_000_000, 4096), (30_000, 8192),
    ((1 << 63) + 1, 512),          # ~half the draws rejected
    ((1 << 64) - 1, 256),          # threshold 1: essentially never rejected
    ((3 << 62) + 12345, 300),      # ~quarter rejected
]


@pytest.mark.parametrize("count,B", CASES)
def test_oracle_philox_indices_match_libstdcxx_distribution(count, B):
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    key = 0x1234_5678_9ABC_DEF0 ^ count
    for ctr0 in (0, 7, (1 << 40) + 3):
        want = np.zeros(B, np.uint64)
        ctr_ref = R.ref_sample_indices_philox(key, ctr0, count, B, ptr(want))
        got = np.zeros(B, np.uint64)
        ctr = np.array([ctr0], np.uint64)
        orc().orc_sample_indices_philox(key, ptr(ctr), count, B, ptr(got))
        assert np.array_equal(got, want)
        assert int(ctr[0]) == ctr_ref
        assert np.all(want < np.uint64(count))
        if count == (1 << 63) + 1:
            assert ctr_ref - ctr0 > B  # the redraw loop ran
