import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, paper_1603_08081_b200 as fb
from oracle.pyoracle import Oracle
O = Oracle()
img = fb.synth_image(0, 160, 144, 6, 10.0)
for name, sp, a, ce in [("g W3", fb.make_spatial_gaussian(1.0), fb.fit_fixed(0, 30.0, 255, 12), True),
                        ("g W5", fb.make_spatial_gaussian(1.5), fb.fit_fixed(0, 30.0, 255, 12), True),
                        ("g W8", fb.make_spatial_gaussian(2.5), fb.fit_fixed(0, 30.0, 255, 12), True),
                        ("box5", fb.make_spatial_box(5), fb.fit_fixed(1, 20.0, 255, 30), False),
                        ("box8", fb.make_spatial_box(8), fb.fit_fixed(1, 20.0, 255, 30), False),
                        ("box12", fb.make_spatial_box(12), fb.fit_fixed(1, 20.0, 255, 30), False),
                        ("g W15", fb.make_spatial_gaussian(5.0), fb.fit_fixed(0, 20.0, 255, 20), True)]:
    out = fb.bilateral_fast(img, sp, a, check_epsilon=ce)
    ref, rc, _ = O.bilateral_fast(img, sp.profile, sp.radius, sp.w0, a.d, a.omega, a.max_pointwise_error, ce)
    d = np.abs(out - ref); yy, xx = np.unravel_index(d.argmax(), d.shape)
    print(name, "max", d.max(), "at", yy, xx, "rows bad", np.unique(np.where(d > 1e-3)[0])[:20])
