"""GPU: the library's real entry point, filter() (bilateral.hpp:173-196), end to
end on the device: integer rounding, local_dynamic_range on the GPU (fp64,
exact), the host recursive-QR fit, bilateral_fast on the GPU."""
import numpy as np
import pytest
from scipy.ndimage import maximum_filter, minimum_filter

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, image_of

pytestmark = pytest.mark.gpu


def ldr_scipy(img, W):
    """independent restatement: scipy 'reflect' == mirror_index (half-sample symmetric)"""
    size = 2 * W + 1
    return int(np.ceil((maximum_filter(img, size=size, mode="reflect") -
                        minimum_filter(img, size=size, mode="reflect")).max()))


def test_ldr_known_cases_and_oracle(oracle):
    # test_bilateral.cpp:133-162
    assert fb.local_dynamic_range(np.full((4, 5), 9.0), 2) == 0
    assert fb.local_dynamic_range(np.array([[0.0, 255.0], [0.0, 255.0]]), 1) == 255
    assert fb.local_dynamic_range(np.array([[0.0, 1.25, 0.0]]), 1) == 2
    rng = np.random.default_rng(0)
    for seed in range(6):
        img = rng.integers(0, 256, (5 if seed % 3 else 12, 7 if seed % 2 else 16)).astype(np.float64)
        for W in (1, 2, 5):
            assert fb.local_dynamic_range(img, W) == oracle.local_dynamic_range(img, W)
    with pytest.raises(ValueError):
        fb.local_dynamic_range(np.zeros((4, 4)), 0)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_ldr_full_size(name):
    c = CONFIGS[name]
    img = image_of(c).astype(np.float64)
    W = c.radius
    assert fb.local_dynamic_range(img, W) == ldr_scipy(img, W)
    # the BASELINE images span most of [0, 255] inside a window (241-255)
    assert 200 <= fb.local_dynamic_range(np.floor(img + 0.5), W) <= 255


def test_filter_end_to_end_matches_oracle_pipeline(oracle):
    rng = np.random.default_rng(200)
    img = rng.integers(0, 256, (24, 24)).astype(np.float64)
    s = fb.make_spatial_gaussian(2.0)
    out, rep = fb.filter(img, s, fb.RANGE_GAUSSIAN, 30.0, 1e-3)
    T = oracle.local_dynamic_range(img, s.radius)
    assert rep["T"] == T
    d, N, _, mx = oracle.progressive_fit(0, 30.0, T, 1e-3)
    assert rep["N"] == N and rep["epsilon_achieved"] == mx
    ref, rc, _ = oracle.bilateral_fast(img, s.profile, s.radius, s.w0, d, np.pi / T, mx)
    assert rc == 0 and np.abs(out - ref).max() <= 1e-3
    exact = oracle.bilateral_exact(img, s.profile, s.radius, 0, 30.0)
    assert np.abs(exact - out).max() <= rep["predicted_bound"]


def test_filter_short_circuits_and_rounds():
    flat = np.full((8, 8), 42.0)
    out, rep = fb.filter(flat, fb.make_spatial_gaussian(2.0), 0, 30.0)
    assert np.array_equal(out, flat) and rep["T"] == 0 and rep["N"] is None
    rng = np.random.default_rng(17)
    img = rng.integers(0, 256, (10, 10)).astype(np.float64)
    a, ra = fb.filter(img, fb.make_spatial_gaussian(1.0), 0, 20.0)
    b, rb = fb.filter(img + 0.25, fb.make_spatial_gaussian(1.0), 0, 20.0)
    assert ra["T"] == rb["T"] and np.array_equal(a, b)
    _, rw = fb.filter(img + 0.5, fb.make_spatial_gaussian(1.0), 0, 20.0, integer_intensities=False)
    assert rw["weaker_guarantee_flag"] and rw["T"] > 0
    with pytest.raises(ValueError):
        fb.filter(img, fb.make_spatial_gaussian(3.0), 0, 30.0, 0.02)
