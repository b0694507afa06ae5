"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): max-abs <= 1e-3 on the [0,255] scale, fp32
accumulation.  Oracle = oracle/fbf_oracle.c, pinned bit-for-bit to the
reference (tests/test_oracle.py).  Full-size configs are checked on row strips
(the oracle's row-range evaluation is bit-identical to a whole-image run) and
through size-independent properties.  The reference fast-path tests
(test_bilateral.cpp:218-312) are restated with fp32 tolerances.
"""
import os

import numpy as np
import pytest

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, T_FIXED, approx_of, image_of, spatial_of

pytestmark = pytest.mark.gpu
TOL = 1e-3
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def oracle_rows(oracle, img, spatial, approx, check_eps=True, row0=0, row1=None, nthreads=8):
    out, rc, _ = oracle.bilateral_fast(img, spatial.profile, spatial.radius, spatial.w0, approx.d, approx.omega,
                                       approx.max_pointwise_error, check_eps, row0, row1, nthreads)
    assert rc == 0
    return out


def maxabs(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_c1_full_image(oracle, variant):
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    gpu = fb.bilateral_fast(img, s, a, variant=variant)
    assert maxabs(gpu, oracle_rows(oracle, img, s, a)) <= TOL


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_configs_on_strips(oracle, name):
    c = CONFIGS[name]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    gpu = fb.bilateral_fast(img, s, a, check_epsilon=c.check_epsilon)
    h = c.height
    for r0 in (0, h // 2 - 7, h - 24):
        ref = oracle_rows(oracle, img, s, a, c.check_epsilon, r0, r0 + 24)
        assert maxabs(gpu[r0:r0 + 24], ref) <= TOL, (name, r0)


def test_c5_batch_images(oracle):
    c = CONFIGS["c5"]
    s, a = spatial_of(c), approx_of(c)
    idx = [0, 7, 255]
    batch = np.stack([image_of(c, i) for i in idx])
    gpu = fb.bilateral_fast(batch, s, a)
    for k, i in enumerate(idx):
        ref = oracle_rows(oracle, batch[k], s, a, True, 500, 532)
        assert maxabs(gpu[k, 500:532], ref) <= TOL
        # batched result == the image filtered alone, bit for bit: the host
        # entry runs a lone 1 Mpixel image as two pipeline strips with their own
        # harmonic grouping, and the fixed-point (Q, P) sums make the result
        # independent of that partition
        alone = fb.bilateral_fast(batch[k], s, a)
        assert np.array_equal(alone, gpu[k])


@pytest.mark.parametrize("name", list(CONFIGS))
def test_reference_golden_vectors(name):
    """The reference's own outputs (tests/golden/filters.npz, made by oracle/_ref)."""
    f = np.load(os.path.join(GOLD, "filters.npz"))
    fits = np.load(os.path.join(GOLD, "fits.npz"))
    c = CONFIGS[name]
    a = fb.FourierKernelApprox(T_FIXED, np.pi / T_FIXED, c.N, fits[f"{name}_d"], 0.0, float(fits[f"{name}_eps"]))
    for variant in ("fused", "naive"):
        gpu = fb.bilateral_fast(f[f"{name}_img"], spatial_of(c), a, variant=variant, check_epsilon=c.check_epsilon)
        assert maxabs(gpu, f[f"{name}_out"]) <= TOL, (name, variant)


@pytest.mark.parametrize("i", range(5))
def test_reference_golden_small_and_ragged(i):
    f = np.load(os.path.join(GOLD, "filters.npz"))
    s = fb.make_spatial_gaussian(float(f[f"rand{i}_sigma"]))
    a = fb.FourierKernelApprox(255, np.pi / 255, 10, f["rand_d"], 0.0, float(f["rand_eps"]))
    for variant in ("fused", "naive"):
        assert maxabs(fb.bilateral_fast(f[f"rand{i}_img"], s, a, variant=variant), f[f"rand{i}_out"]) <= TOL


@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (9, 1), (3, 3), (5, 7), (17, 200), (130, 67), (64, 64)])
@pytest.mark.parametrize("sigma", [1.0, 1.5, 2.0, 3.0, 8.0])
def test_edge_shapes_all_radii(oracle, shape, sigma):
    """Tiny and ragged images (periodic mirror), fused radii (3,5,6,9,24) vs oracle."""
    rng = np.random.default_rng(hash((shape, sigma)) % 2**32)
    img = rng.integers(0, 256, shape).astype(np.float64)
    s = fb.make_spatial_gaussian(sigma)
    a = fb.fit_fixed(0, 30.0, 255, 14)
    if not a.max_pointwise_error < s.w0:
        pytest.skip("fit not admissible for this window")
    assert maxabs(fb.bilateral_fast(img, s, a), oracle_rows(oracle, img, s, a, nthreads=1)) <= TOL


@pytest.mark.parametrize("radius", [1, 2, 4, 7, 10, 16, 17, 24, 25])
def test_box_radii(oracle, radius):
    """Box windows: running-sum fused instances for radii 1..24, the naive chain beyond."""
    rng = np.random.default_rng(radius)
    img = rng.integers(0, 256, (37, 45)).astype(np.float64)
    s = fb.make_spatial_box(radius)
    a = fb.fit_fixed(1, 25.0, 255, 40)
    ref = oracle_rows(oracle, img, s, a, check_eps=False, nthreads=1)
    for variant in ("fused", "naive"):
        assert maxabs(fb.bilateral_fast(img, s, a, variant=variant, check_epsilon=False), ref) <= TOL


# ---- test_bilateral.cpp:218-312 fast-path properties, fp32 tolerances ----

def test_constant_image_passes_through():
    s = fb.make_spatial_gaussian(1.0)
    a = fb.progressive_fit(0, 30.0, 255, 1e-3)
    out = fb.bilateral_fast(np.full((8, 8), 120.0), s, a)
    assert maxabs(out, 120.0) <= 1e-4


def test_identity_approximation_reduces_to_convolve(oracle):
    rng = np.random.default_rng(77)
    img = rng.integers(0, 256, (9, 14)).astype(np.float64)
    s = fb.make_spatial_gaussian(2.0)
    ident = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([1.0]), 0.0, 0.0)
    conv = oracle.convolve(img, s.profile, s.radius)
    assert maxabs(fb.bilateral_fast(img, s, ident), conv) <= 1e-4
    assert maxabs(fb.convolve(img, s), conv) <= 1e-4


def test_shift_equivariance_at_full_size():
    c = CONFIGS["c2"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    base = fb.bilateral_fast(img, s, a)
    shifted = fb.bilateral_fast(img.astype(np.float64) + 10.0, s, a)
    assert maxabs(shifted, base.astype(np.float64) + 10.0) <= 2 * TOL


def test_commutes_with_mirroring():
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    out = fb.bilateral_fast(img, s, a)
    assert maxabs(fb.bilateral_fast(img[:, ::-1].copy(), s, a), out[:, ::-1]) <= 2 * TOL
    assert maxabs(fb.bilateral_fast(img[::-1].copy(), s, a), out[::-1]) <= 2 * TOL


def test_within_paper_bound_vs_brute_force(oracle):
    """|fast - exact| <= 2 T eps / (w0 - eps) (analysis.hpp:27-34) on full-width strips."""
    for name in ("c1", "c2", "c5"):
        c = CONFIGS[name]
        img, s, a = image_of(c), spatial_of(c), approx_of(c)
        gpu = fb.bilateral_fast(img, s, a)
        bound = fb.error_bound(T_FIXED, a.max_pointwise_error, s.w0)
        r0 = c.height // 3
        ex = oracle.bilateral_exact(img, s.profile, s.radius, c.range_family, c.sigma_r, r0, r0 + 8, 8)
        assert maxabs(gpu[r0:r0 + 8], ex) <= bound, name


def test_accuracy_improves_with_tighter_tolerance(oracle):
    rng = np.random.default_rng(123)
    img = rng.integers(0, 256, (32, 32)).astype(np.float64)
    s = fb.make_spatial_gaussian(1.0)
    T = oracle.local_dynamic_range(img, s.radius)
    ex = oracle.bilateral_exact(img, s.profile, s.radius, 0, 30.0)
    loose = fb.bilateral_fast(img, s, fb.progressive_fit(0, 30.0, T, 1e-2))
    tight = fb.bilateral_fast(img, s, fb.progressive_fit(0, 30.0, T, 1e-5))
    assert maxabs(tight, ex) <= maxabs(loose, ex)


def test_rejects_approximation_wider_than_center_weight():
    bad = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([1.0]), 0.0, 0.5)
    with pytest.raises(ValueError):
        fb.bilateral_fast(np.zeros((8, 8)), fb.make_spatial_gaussian(3.0), bad)


@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_collapsed_denominator_names_the_pixel(variant):
    rng = np.random.default_rng(8)
    img = rng.integers(0, 256, (6, 6)).astype(np.float64)
    lying = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([0.0]), 0.0, 0.0)
    with pytest.raises(fb.FilterError, match=r"pixel \(0, 0\)"):
        fb.bilateral_fast(img, fb.make_spatial_gaussian(1.0), lying, variant=variant)


def test_reruns_are_bit_identical():
    c = CONFIGS["c2"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    assert np.array_equal(fb.bilateral_fast(img, s, a), fb.bilateral_fast(img, s, a))


def test_fused_and_naive_agree():
    c = CONFIGS["c5"]
    img, s, a = image_of(c, 3), spatial_of(c), approx_of(c)
    assert maxabs(fb.bilateral_fast(img, s, a), fb.bilateral_fast(img, s, a, variant="naive")) <= TOL


def test_convolve_matches_oracle(oracle):
    rng = np.random.default_rng(5)
    for shape, sk in (((16, 16), fb.make_spatial_gaussian(1.0)), ((5, 7), fb.make_spatial_gaussian(2.0)),
                      ((9, 1), fb.make_spatial_box(4)), ((300, 257), fb.make_spatial_gaussian(8.0))):
        img = rng.random(shape) * 255
        assert maxabs(fb.convolve(img, sk), oracle.convolve(img, sk.profile, sk.radius)) <= 1e-3


@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_harmonic_count_beyond_one_launch(oracle, variant):
    """N up to T (progressive_fit's limit, kernel_approx.hpp:189-203): a dynamic
    range of 600 and N = 300 -> the fused path runs two chained launches of
    <= 256 harmonics (the second accumulating onto the first's (Q, P))."""
    rng = np.random.default_rng(600)
    img = np.clip(rng.normal(300, 120, (40, 72)), 0, 600)
    img[8:30, 20:50] += 150
    img = np.minimum(img, 600.0)
    s = fb.make_spatial_gaussian(1.5)
    a = fb.fit_fixed(fb.RANGE_GAUSSIAN, 40.0, 600, 300)
    assert a.N == 300
    gpu = fb.bilateral_fast(img, s, a, variant=variant)
    # fp32 over a range 600/255 times wider than 8-bit images
    assert maxabs(gpu, oracle_rows(oracle, img, s, a)) <= TOL * 600 / 255


def test_exponential_kernel_high_order(oracle):
    """the CLI's box / exponential case: progressive_fit picks N > 127"""
    rng = np.random.default_rng(25)
    img = np.floor(np.clip(rng.normal(120, 50, (40, 48)), 0, 255) + 0.5)
    s = fb.make_spatial_box(2)
    T = oracle.local_dynamic_range(img, s.radius)
    d, N, _, mx = oracle.progressive_fit(1, 25.0, T, 1e-3)
    assert N > 127
    a = fb.progressive_fit(fb.RANGE_EXPONENTIAL, 25.0, T, 1e-3)
    assert a.N == N
    gpu = fb.bilateral_fast(img, s, a)
    assert maxabs(gpu, oracle_rows(oracle, img, s, a)) <= TOL


@pytest.mark.parametrize("sigma", [0.3, 0.6, 1.3, 2.3, 3.3, 3.6, 4.3, 6.0, 7.0, 8.7, 10.0, 11.0, 12.0, 13.3])
def test_fused_radii_1_to_40(oracle, sigma):
    """Every Gaussian radius 1..40 (sigma <= 13.3, the reference CLI sweep's
    sigma <= 12 included) has a fused instance; radii above 25 run one
    128-thread CTA per SM (the 256-thread tiles exceed shared memory)."""
    rng = np.random.default_rng(int(sigma * 10))
    img = rng.integers(0, 256, (72, 130)).astype(np.float64)
    s = fb.make_spatial_gaussian(sigma)
    a = fb.fit_fixed(0, 30.0, 255, 14)
    ref = oracle_rows(oracle, img, s, a, check_eps=False, nthreads=4)
    assert maxabs(fb.bilateral_fast(img, s, a, check_epsilon=False), ref) <= TOL
    assert fb.launches_per_call(fb.whole_geometry(130, 72), s, a) <= 4  # prep, n=0 plane, fused (, group sum): no naive chain
