"""The device Omega generator is bit-identical to the reference's numpy
generator (default_rng(seed).standard_normal((n, k)), rangefinder.py:101,112)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2404_09459_b200 import device as dv  # noqa: E402

SEEDS = [0, 1, 2, 7, 12345, 2**32 + 5, 2**63 + 7, 2**64 - 1, -1]


@pytest.mark.parametrize("n,k", [(200, 30), (1000, 60), (64, 16), (7, 3), (4000, 120),
                                 (333, 13)])
def test_omega_bit_exact(n, k):
    seeds = SEEDS if n * k < 200000 else SEEDS[:3]
    om = dv.omega_device(n, k, seeds).cpu().numpy()
    for i, seed in enumerate(seeds):
        ref = np.random.default_rng(int(seed) & ((1 << 64) - 1)).standard_normal((n, k))
        got = om[i, :k, :n].T
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (seed, n, k)
        assert not om[i, k:, :].any() and not om[i, :, n:].any()  # zero padding


def test_omega_many_streams_including_tails():
    """4096 streams x 1024 normals (cfg3's per-pair Omega): every slow and
    tail path of the ziggurat is exercised thousands of times."""
    seeds = list(range(0, 8192, 2))
    om = dv.omega_device(64, 16, seeds).cpu().numpy()
    bad = 0
    for i, seed in enumerate(seeds):
        ref = np.random.default_rng(seed).standard_normal((64, 16))
        bad += int(np.count_nonzero(om[i, :16, :64].T != ref))
    assert bad == 0
