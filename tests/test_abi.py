"""CPU: the C-ABI library loads, exports every symbol include/fourierbf_b200.h
declares, validates arguments like the reference (no GPU touched), and its
host-side pieces (spatial taps, range kernels, the recursive-QR fit, the
synthetic generator) agree with the reference / are deterministic."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, T_FIXED

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fourierbf_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fbf_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_are_exported_and_bound():
    names = declared_functions()
    assert len(names) >= 20
    so = ctypes.CDLL(fb.LIB_PATH)
    for n in names:
        assert hasattr(so, n), f"{n} declared in fourierbf_b200.h but not exported"
        assert n in fb.SIGNATURES, f"{n} has no ctypes binding in the Python mirror"


def test_argument_validation_without_gpu():
    g = fb.whole_geometry(0, 5)
    assert fb.lib.fbf_workspace_bytes(ctypes.byref(g), 3, fb.VARIANT_FUSED) == 0
    s, a = fb.make_spatial_gaussian(1.0), fb.fit_fixed(0, 30.0, 255, 8)
    f = fb._filter_struct(s, a)
    rc = fb.lib.fbf_bilateral_fast_device(ctypes.byref(g), ctypes.byref(f), None, None, None, 0, None, 0, None)
    assert rc == fb.FBF_EINVAL and "empty image" in fb.lib.fbf_last_error().decode()
    g = fb.whole_geometry(8, 8)
    bad = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([1.0]), 0.0, 0.5)  # eps >= w0
    f = fb._filter_struct(fb.make_spatial_gaussian(3.0), bad)
    rc = fb.lib.fbf_bilateral_fast_device(ctypes.byref(g), ctypes.byref(f), None, None, None, 0, None, 0, None)
    assert rc == fb.FBF_EINVAL
    assert "kernel approximation error must stay below the center spatial weight" in fb.lib.fbf_last_error().decode()
    with pytest.raises(ValueError):
        fb.bilateral_fast(np.zeros((8, 8)), fb.make_spatial_gaussian(3.0), bad)
    # a strip without its halo rows is rejected before any launch
    g = fb.strip_geometry(64, 64, 10, 20, 3)
    g.src_row0, g.src_rows = 10, 20
    f = fb._filter_struct(s, a)
    rc = fb.lib.fbf_bilateral_fast_device(ctypes.byref(g), ctypes.byref(f), None, None, None, 0, None, 0, None)
    assert rc == fb.FBF_EINVAL and "halo" in fb.lib.fbf_last_error().decode()


def test_host_spatial_and_fit_match_reference_golden():
    sp = np.load(os.path.join(GOLD, "spatial.npz"))
    for s in (1.0, 1.5, 2.0, 2.5, 3.0, 4.0, 5.0, 8.0):
        k = fb.make_spatial_gaussian(s)
        assert k.radius == int(sp[f"g{s}_radius"])
        assert np.array_equal(k.profile, sp[f"g{s}_profile"]) and k.w0 == float(sp[f"g{s}_w0"])
    for r in range(1, 6):
        k = fb.make_spatial_box(r)
        assert np.array_equal(k.profile, sp[f"b{r}_profile"]) and k.w0 == float(sp[f"b{r}_w0"])
    fits = np.load(os.path.join(GOLD, "fits.npz"))
    for name, c in CONFIGS.items():
        a = fb.fit_fixed(c.range_family, c.sigma_r, T_FIXED, c.N)
        assert np.array_equal(a.d, fits[f"{name}_d"]), name  # host C++ fit == reference, bit for bit
        assert a.max_pointwise_error == float(fits[f"{name}_eps"])
    p = fb.progressive_fit(0, 30.0, 217, 1e-3)
    assert p.N == 9 and np.array_equal(p.d, fits["prog_g30_T217_e1e-3_d"])
    with pytest.raises(ValueError):
        fb.make_spatial_gaussian(0.0)
    with pytest.raises(ValueError):
        fb.make_spatial_box(0)
    with pytest.raises(ValueError):
        fb.progressive_fit(0, 30.0, 255, 100.0)  # eps >= sqrt(T+1)


def test_error_bound_matches_analysis_hpp():
    # analysis.hpp:27-34 and SURVEY Appendix B (c1 bound 0.09713)
    c = CONFIGS["c1"]
    a = fb.fit_fixed(0, c.sigma_r, 255, c.N)
    w0 = fb.make_spatial_gaussian(c.sigma_s).w0
    assert fb.error_bound(255, a.max_pointwise_error, w0) == pytest.approx(0.09713, rel=1e-3)
    with pytest.raises(ValueError):
        fb.error_bound(255, 0.1, 0.05)


def test_range_kernels():
    assert fb.lib.fbf_range_eval(0, 30.0, 0.0) == 1.0
    assert fb.lib.fbf_range_eval(0, 30.0, -30.0) == pytest.approx(np.exp(-0.5))
    assert fb.lib.fbf_range_eval(1, 20.0, 40.0) == pytest.approx(np.exp(-2.0))


def test_synthetic_generator_is_deterministic_and_strip_local():
    c = CONFIGS["c2"]
    a = fb.synth_image(c.seeds[0], 300, 200, c.rects, c.noise)
    b = fb.synth_image(c.seeds[0], 300, 200, c.rects, c.noise, nthreads=1)
    assert a.dtype == np.float32 and a.shape == (200, 300)
    assert np.array_equal(a, b)
    strip = fb.synth_image(c.seeds[0], 300, 200, c.rects, c.noise, row0=57, rows=40)
    assert np.array_equal(strip, a[57:97])  # ranks can generate their own strips
    assert a.min() >= 0.0 and a.max() <= 255.0
    assert not np.array_equal(a, fb.synth_image(c.seeds[0] + 1, 300, 200, c.rects, c.noise))
    # gradient 0 -> 128 underneath: the noise-free image would be monotone in x
    col_means = fb.synth_image(5, 256, 512, 0, 10.0).mean(axis=0)
    assert col_means[0] < 10 and abs(col_means[-1] - 128) < 10


def test_config_op_counts_match_survey():
    # ops per pixel
    assert CONFIGS["c1"].ops_per_pixel() == 2008
    assert CONFIGS["c2"].ops_per_pixel() == 5264
    assert CONFIGS["c3"].ops_per_pixel() == 846
    assert CONFIGS["c4"].ops_per_pixel() == 13028
    assert CONFIGS["c5"].ops_per_pixel() == 3444
