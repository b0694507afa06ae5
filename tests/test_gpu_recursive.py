"""GPU: the recursive convolution backend (ConvolutionBackend::recursive,
recursive_gaussian.hpp -- third-order van Vliet/Young/Verbeek IIR with a
mirror-padded warm-up) against the reference build itself (oracle/_ref): the
IIR and Algorithm 1 on it run in fp64 on the device, in the reference's
evaluation order, so parity is near round-off.  The reference's dispatch rule
(spatial.hpp:102-104: Gaussian windows with sigma >= 2 only) is checked too."""
import numpy as np
import pytest

import paper_1603_08081_b200 as fb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import Reference
    try:
        return Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")


def image(seed, h, w):
    rng = np.random.default_rng(seed)
    img = np.clip(rng.normal(120, 45, (h, w)), 0, 255)
    img[h // 4:3 * h // 4, w // 3:2 * w // 3] += 70
    return np.floor(np.minimum(img, 255.0) + 0.5)


@pytest.mark.parametrize("shape,sigma", [((40, 48), 2.0), ((37, 91), 2.3), ((64, 33), 5.0), ((9, 7), 4.0)])
def test_convolve_recursive_matches_reference(ref, shape, sigma):
    img = image(sum(shape), *shape)
    gpu = fb.convolve(img, fb.make_spatial_gaussian(sigma), backend="recursive")
    assert np.abs(gpu - ref.convolve_recursive(img, sigma)).max() <= 1e-9 * 255


def test_convolve_recursive_dispatch_rule(oracle):
    img = image(3, 24, 30)
    for s in (fb.make_spatial_gaussian(1.5), fb.make_spatial_box(2)):  # sigma < 2 / box: the direct FIR
        direct = fb.convolve(img, s)
        assert np.array_equal(fb.convolve(img, s, backend="recursive"), direct)
    s = fb.make_spatial_gaussian(3.0)
    # an approximation of the Gaussian, not the FIR itself
    assert 1e-6 < np.abs(fb.convolve(img, s, backend="recursive") - fb.convolve(img, s)).max() < 5.0


@pytest.mark.parametrize("shape,sigma,sigma_r", [((48, 64), 2.0, 30.0), ((40, 72), 3.5, 20.0)])
def test_bilateral_recursive_matches_reference(ref, shape, sigma, sigma_r):
    img = image(7 + shape[0], *shape)
    s = fb.make_spatial_gaussian(sigma)
    a = fb.progressive_fit(fb.RANGE_GAUSSIAN, sigma_r, 255, 1e-3)
    gpu = fb.bilateral_fast(img, s, a, variant="recursive")  # fp64 host entry
    theirs = ref.bilateral_fast_recursive(img, sigma, a.d, 255, a.max_pointwise_error)
    assert np.abs(gpu - theirs).max() <= 1e-7
    gpu32 = fb.bilateral_fast(img.astype(np.float32), s, a, variant="recursive")  # fp32 host entry
    assert np.abs(gpu32 - theirs).max() <= 1e-3
    # the FIR path differs from the IIR by the IIR's approximation of the Gaussian
    # (a few grey levels at edges for small sigma)
    assert 1e-3 < np.abs(fb.bilateral_fast(img, s, a) - theirs).max() < 5.0


def test_bilateral_recursive_falls_back_to_direct_and_reports_collapse():
    img = image(11, 32, 40)
    s = fb.make_spatial_gaussian(1.0)  # sigma < 2: the reference keeps the FIR
    a = fb.progressive_fit(fb.RANGE_GAUSSIAN, 30.0, 255, 1e-3)
    assert np.array_equal(fb.bilateral_fast(img, s, a, variant="recursive"), fb.bilateral_fast(img, s, a))
    lying = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([0.0]), 0.0, 0.0)
    with pytest.raises(fb.FilterError, match=r"pixel \(0, 0\)"):
        fb.bilateral_fast(img, fb.make_spatial_gaussian(2.5), lying, variant="recursive")
