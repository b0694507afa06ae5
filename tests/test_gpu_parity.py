"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): max-abs <= 1e-3 on the [0,255] scale with fp32
accumulation.  Oracle = oracle/fbf_oracle.c, pinned bit-for-bit to the
reference (tests/test_oracle.py).  Full-size configs are checked on row strips
(the oracle's row-range evaluation is bit-identical to a whole-image run).
"""
import numpy as np
import pytest

from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

pytestmark = pytest.mark.gpu
TOL = 1e-3


def oracle_rows(oracle, img, spatial, approx, check_eps, row0, row1, nthreads=8):
    out, rc, _ = oracle.bilateral_fast(img, spatial.profile, spatial.radius, spatial.w0, approx.d, approx.omega,
                                       approx.max_pointwise_error, check_eps, row0, row1, nthreads)
    assert rc == 0
    return out


@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_c1_full_image(fb, oracle, variant):
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    gpu = fb.bilateral_fast(img, s, a, variant=variant)
    ref = oracle_rows(oracle, img, s, a, True, 0, c.height)
    err = np.abs(gpu.astype(np.float64) - ref).max()
    assert err <= TOL, err


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_configs_on_strips(fb, oracle, name):
    c = CONFIGS[name]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    gpu = fb.bilateral_fast(img, s, a, check_epsilon=c.check_epsilon)
    h = c.height
    for r0 in (0, h // 2 - 7, h - 24):
        ref = oracle_rows(oracle, img, s, a, c.check_epsilon, r0, r0 + 24)
        err = np.abs(gpu[r0:r0 + 24].astype(np.float64) - ref).max()
        assert err <= TOL, (name, r0, err)
