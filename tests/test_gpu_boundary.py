"""GPU: the C-ABI boundary beyond the fused hot path -- fp64 host entry,
multi-device entry, any-radius / asymmetric windows (naive chain with taps in
memory), tall images (no launch-dimension limit), the fp64 convolve() against
the reference build bit for bit."""
import numpy as np
import pytest

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

pytestmark = pytest.mark.gpu
TOL = 1e-3  # north_star: max-abs vs the fp64 oracle on the [0, 255] scale


def maxabs(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_f64_host_entry_equals_f32(name):
    """fbf_bilateral_fast_host_f64 (the reference Image's doubles, converted on the
    host thread pool, pipelined) == the fp32 entry on the same values, bit for bit."""
    c = CONFIGS[name]
    s, a = spatial_of(c), approx_of(c)
    img = np.stack([image_of(c, i) for i in range(3)]) if c.batch > 1 else image_of(c)
    out32 = fb.bilateral_fast(img, s, a)
    out64 = fb.bilateral_fast(img.astype(np.float64), s, a)
    assert out64.dtype == np.float64
    assert np.array_equal(out64, out32.astype(np.float64))


@pytest.mark.parametrize("shape,devices", [((2048, 2048), [0, 0]), ((600, 512), [0, 0, 0]), ((5, 256, 320), [0, 0])])
def test_multi_device_entry_equals_one_device(shape, devices):
    """fbf_bilateral_fast_host_multi with the strips / images all on device 0
    (the per-device worker threads run them one after another): == one call."""
    c = CONFIGS["c2"]
    s, a = spatial_of(c), approx_of(c)
    rng = np.random.default_rng(len(shape) * 7 + shape[-1])
    img = np.clip(rng.normal(128, 50, shape), 0, 255).astype(np.float32)
    one = fb.bilateral_fast(img, s, a)
    assert np.array_equal(fb.bilateral_fast_multi(img, s, a, devices), one)
    assert np.array_equal(fb.bilateral_fast_multi(img.astype(np.float64), s, a, devices), one.astype(np.float64))


def test_multi_device_entry_reports_the_first_collapse():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (3, 64, 80)).astype(np.float32)
    lying = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([0.0]), 0.0, 0.0)
    with pytest.raises(fb.FilterError, match=r"pixel \(0, 0\)"):
        fb.bilateral_fast_multi(img, fb.make_spatial_gaussian(2.0), lying, [0, 0])


@pytest.mark.parametrize("spatial", [("gaussian", 13.0), ("gaussian", 25.0), ("box", 40)])
def test_large_windows_match_the_oracle(oracle, spatial):
    """Radii beyond the fused kernels (W = 39, 75 Gaussian; box 40): the naive
    chain with its taps in device memory; no radius limit."""
    kind, p = spatial
    s = fb.make_spatial_gaussian(p) if kind == "gaussian" else fb.make_spatial_box(p)
    a = fb.fit_fixed(0, 30.0, 255, 10)
    img = image_of(CONFIGS["c1"])[:90, :130].copy()
    gpu = fb.bilateral_fast(img, s, a, check_epsilon=False)
    ref, rc, _ = oracle.bilateral_fast(img, s.profile, s.radius, s.w0, a.d, a.omega, a.max_pointwise_error,
                                       check_eps=False)
    assert rc == 0
    assert maxabs(gpu, ref) <= TOL


def test_asymmetric_window_matches_the_oracle(oracle):
    """A user SpatialKernel whose profile is not symmetric runs the naive chain
    with all 2W+1 taps, out(i) = sum_j profile[j+W] in(i-j) (spatial.hpp:74-89)."""
    prof = np.array([0.05, 0.1, 0.2, 0.3, 0.2, 0.1, 0.05, 0.0, 0.0])[::-1].copy()
    prof /= prof.sum()
    W = 4
    s = fb.SpatialKernel(fb.SPATIAL_GAUSSIAN, 0.0, W, prof, float(prof[W] ** 2))
    a = fb.fit_fixed(0, 30.0, 255, 12)
    img = image_of(CONFIGS["c1"])[:70, :90].copy()
    gpu = fb.bilateral_fast(img, s, a, check_epsilon=False)
    ref, rc, _ = oracle.bilateral_fast(img, prof, W, s.w0, a.d, a.omega, a.max_pointwise_error, check_eps=False)
    assert rc == 0
    assert maxabs(gpu, ref) <= TOL


@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_tall_image_beyond_the_launch_limit(oracle, variant):
    """70,000 rows: more than the 65,535 blocks of a grid's y dimension."""
    h, w = 70000, 8
    rng = np.random.default_rng(70000)
    img = rng.integers(0, 256, (h, w)).astype(np.float32)
    s, a = fb.make_spatial_gaussian(1.0), fb.fit_fixed(0, 30.0, 255, 8)
    gpu = fb.bilateral_fast(img, s, a, variant=variant)
    for r0 in (0, 35000, h - 20):
        ref, rc, _ = oracle.bilateral_fast(img, s.profile, s.radius, s.w0, a.d, a.omega, a.max_pointwise_error,
                                           row0=r0, row1=r0 + 20)
        assert rc == 0
        assert maxabs(gpu[r0:r0 + 20], ref) <= TOL


@pytest.mark.parametrize("kind,param", [(0, 1.0), (0, 2.0), (1, 1), (1, 4), (0, 12.0), (1, 70)])
def test_convolve_fp64_equals_the_reference(kind, param):
    """convolve() in fp64 on the device, separate multiply and add in ascending
    j: the reference build's bits (test_spatial.cpp:91-107 asks for 1e-11)."""
    from oracle.pyoracle import Reference
    ref = Reference()
    rng = np.random.default_rng(int(param * 10) + kind)
    img = rng.uniform(0.0, 255.0, (37, 53))
    s = fb.make_spatial_gaussian(param) if kind == 0 else fb.make_spatial_box(int(param))
    assert np.array_equal(fb.convolve(img, s), ref.convolve(img, kind, float(param)))


def test_cpp_bilateral_exact_runs_on_the_gpu(oracle):
    """The C++ API's bilateral_exact for Gaussian / exponential ranges is the fp64
    device brute force (fbf_bilateral_exact_host_f64) == the oracle to 1e-9."""
    import ctypes
    img = image_of(CONFIGS["c1"])[:40, :56].astype(np.float64)
    s = fb.make_spatial_gaussian(2.0)
    for fam, sr in ((0, 30.0), (1, 20.0)):
        out = np.empty_like(img)
        prof = np.ascontiguousarray(s.profile)
        rc = fb.lib.fbf_bilateral_exact_host_f64(56, 40, prof.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                 s.radius, fam, sr,
                                                 img.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        assert rc == 0
        ref = oracle.bilateral_exact(img, s.profile, s.radius, fam, sr)
        assert maxabs(out, ref) <= 1e-9
