"""Small filter calls for compute-sanitizer (racecheck / synccheck / memcheck).

Covers every fused-kernel instance family on c1-size-or-smaller images:
  * 128-thread, G=16, two CTAs per SM (Gaussian W <= 9): c1's W=9
  * 256-thread, G=32, double-buffered M + deferred demodulation (10 <= W <= 25): W=15
  * 128-thread, one CTA per SM (W >= 26): W=30
  * box running sums (W=5, the c3 window)
  * harmonic groups > 1 (finish kernel) and chained launches (N > 256 harmonics)
  * the naive multi-kernel chain
Each result is checked against the fp64 oracle, so a race that corrupts the
output also fails here, not only in the sanitizer log.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1603_08081_b200 as fb  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402


def case(name, img, spatial, approx, variant="fused", check_epsilon=True):
    out = fb.bilateral_fast(img, spatial, approx, variant=variant, check_epsilon=check_epsilon)
    err = 0.0
    for o, im in zip(out.reshape((-1,) + out.shape[-2:]), img.reshape((-1,) + img.shape[-2:])):
        ref, rc, _ = Oracle().bilateral_fast(im, spatial.profile, spatial.radius, spatial.w0, approx.d,
                                             approx.omega, approx.max_pointwise_error, check_epsilon)
        assert rc == 0
        err = max(err, float(np.abs(o.astype(np.float64) - ref).max()))
    print(f"{name:28s} {variant:6s} max-abs {err:.3e}", flush=True)
    assert err <= 1e-3, name


def main():
    quick = "--quick" in sys.argv
    img = fb.synth_image(0, 160, 144, 6, 10.0)
    g = fb.make_spatial_gaussian
    case("W=9 (128 thr, 2/SM)", img, g(3.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 30.0, 255, 12))
    case("W=15 (256 thr, defer)", img, g(5.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 20.0, 255, 20))
    case("box W=5", img, fb.make_spatial_box(5), fb.fit_fixed(fb.RANGE_EXPONENTIAL, 20.0, 255, 30),
         check_epsilon=False)
    if quick:
        return
    case("W=30 (128 thr, 1/SM)", img, g(10.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 20.0, 255, 20),
         check_epsilon=False)
    # tall narrow: many units per CTA and harmonic groups
    tall = fb.synth_image(5, 64, 700, 3, 10.0)
    case("W=12 tall (groups)", tall, g(4.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 25.0, 255, 16))
    # more harmonics than one launch carries: chained launches accumulate
    small = fb.synth_image(7, 48, 40, 2, 10.0)
    case("N=300 chained", small, g(2.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 3.0, 600, 300), check_epsilon=False)
    case("W=9 naive", img, g(3.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 30.0, 255, 12), variant="naive")
    batch = np.stack([fb.synth_image(100 + i, 96, 80, 4, 10.0) for i in range(3)])
    case("batch of 3, W=12", batch, g(4.0), fb.fit_fixed(fb.RANGE_GAUSSIAN, 25.0, 255, 16))


if __name__ == "__main__":
    main()
