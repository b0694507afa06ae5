"""GPU: randomized geometries against the fp64 oracle -- image sizes, batches,
Gaussian / box radii, harmonic counts, strip sub-geometries (device entry) and
the pipelined host entry (>= 1 Mpixel) -- to catch edge cases of the lane
mappings, rings and chunking that the fixed configs do not reach."""
import numpy as np
import pytest

import paper_1603_08081_b200 as fb

pytestmark = pytest.mark.gpu
TOL = 1e-3


def case(seed):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    b = int(rng.choice([1, 1, 2, 3]))
    box = bool(rng.random() < 0.3)
    if box:
        s = fb.make_spatial_box(int(rng.integers(1, 17)))
    else:
        s = fb.make_spatial_gaussian(float(rng.choice([0.4, 1.0, 1.7, 2.5, 3.3, 4.0, 5.0, 6.5, 8.0, 9.7])))
    N = int(rng.integers(0, 24))
    a = fb.fit_fixed(int(rng.integers(0, 2)), float(rng.uniform(10, 60)), 255, N)
    img = np.clip(rng.normal(128, 60, (b, h, w)), 0, 255)
    return img, s, a


def oracle_out(oracle, img, s, a):
    out = np.empty_like(img)
    for k in range(img.shape[0]):
        o, rc, _ = oracle.bilateral_fast(img[k], s.profile, s.radius, s.w0, a.d, a.omega, a.max_pointwise_error,
                                         False, 0, None, 8)
        assert rc == 0
        out[k] = o
    return out


@pytest.mark.parametrize("seed", range(24))
def test_random_geometries(oracle, seed):
    img, s, a = case(seed)
    ref = oracle_out(oracle, img, s, a)
    got = fb.bilateral_fast(img if img.shape[0] > 1 else img[0], s, a, check_epsilon=False)
    assert np.abs(got.reshape(ref.shape) - ref).max() <= TOL


@pytest.mark.parametrize("seed", range(4))
def test_random_large_pipelined(oracle, seed):
    """>= 1 Mpixel calls: the host entry's strip / image-chunk pipeline"""
    rng = np.random.default_rng(100 + seed)
    h, w = int(rng.integers(1100, 2100)), int(rng.integers(1100, 2100))
    s = fb.make_spatial_gaussian(float(rng.choice([1.0, 2.5, 5.0])))
    a = fb.fit_fixed(0, 25.0, 255, 10)
    img = np.clip(rng.normal(128, 60, (h, w)), 0, 255).astype(np.float32)
    got = fb.bilateral_fast(img, s, a)
    for r0 in (0, h // 3, h - 20):  # rows around strip cuts and both edges
        o, rc, _ = oracle.bilateral_fast(img.astype(np.float64), s.profile, s.radius, s.w0, a.d, a.omega,
                                         a.max_pointwise_error, True, r0, r0 + 20, 8)
        assert rc == 0
        assert np.abs(got[r0:r0 + 20] - o).max() <= TOL
