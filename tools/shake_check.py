"""Race check without compute-sanitizer (closed on the GPU pool): the shake
build (make -C paper_1603_08081_b200/csrc shake) sleeps random 0-2 us per warp
at every phase boundary of the fused kernel.  Every case runs 3x on it and must
equal the product build bit for bit (the arithmetic does not depend on timing:
fixed-point (Q, P) sums, fixed tap orders); parity with the fp64 oracle is
the -m gpu tests' job.  Covers the 128-thread (two CTAs per SM, and one per SM for W > 25),
256-thread (double-buffered M, deferred demodulation, warp-pair barriers),
box, harmonic-group, chained-launch, batch and pipelined host paths.

    python tools/shake_check.py        (prints one line per case; exit 1 on any mismatch)
"""
import os
import time
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(ROOT, "paper_1603_08081_b200", "_lib")


def run_cases(libname):
    os.environ["FBF_LIBRARY"] = os.path.join(LIB, libname)
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_1603_08081_b200 as fb
    g = fb.make_spatial_gaussian
    img = fb.synth_image(0, 160, 144, 6, 10.0)
    tall = fb.synth_image(5, 64, 700, 3, 10.0)
    small = fb.synth_image(7, 48, 40, 2, 10.0)
    batch = np.stack([fb.synth_image(100 + i, 96, 80, 4, 10.0) for i in range(3)])
    big = fb.synth_image(1, 1024, 1100, 24, 15.0)  # pipelined host path (>= 1 Mpixel), 256-thread W = 15
    cases = [("W=9 small", img, g(3.0), fb.fit_fixed(0, 30.0, 255, 12), True),
             ("W=15 big defer", img, g(5.0), fb.fit_fixed(0, 20.0, 255, 20), True),
             ("box W=5", img, fb.make_spatial_box(5), fb.fit_fixed(1, 20.0, 255, 30), False),
             ("box W=12 big", img, fb.make_spatial_box(12), fb.fit_fixed(1, 20.0, 255, 30), False),
             ("W=30 small 1/SM", img, g(10.0), fb.fit_fixed(0, 20.0, 255, 20), False),
             ("W=40", img, g(13.3), fb.fit_fixed(0, 20.0, 255, 20), False),
             ("W=12 tall groups", tall, g(4.0), fb.fit_fixed(0, 25.0, 255, 16), True),
             ("N=300 chained", small, g(2.0), fb.fit_fixed(0, 3.0, 600, 300), False),
             ("batch W=12", batch, g(4.0), fb.fit_fixed(0, 25.0, 255, 16), True),
             ("1 Mpx pipeline W=15", big, g(5.0), fb.fit_fixed(0, 20.0, 255, 20), True)]
    out = {}
    t0 = time.perf_counter()
    for name, im, sp, ap, ce in cases:
        out[name] = [fb.bilateral_fast(im.astype(np.float32), sp, ap, check_epsilon=ce) for _ in range(3)]
    out["_seconds"] = time.perf_counter() - t0
    return out, cases


def main():
    import pickle
    if len(sys.argv) > 3 and sys.argv[1] == "--dump":
        out, _ = run_cases(sys.argv[2])
        pickle.dump(out, open(sys.argv[3], "wb"))
        return 0
    import numpy as np
    res = {}
    for lib in ("libfourierbf_b200.so", "libfourierbf_b200_shake.so"):
        f = f"/tmp/shake_{lib}.pkl"
        subprocess.run([sys.executable, __file__, "--dump", lib, f], check=True)
        res[lib] = pickle.load(open(f, "rb"))
    prod, shake = res["libfourierbf_b200.so"], res["libfourierbf_b200_shake.so"]
    print(f"wall time of all cases: product {prod.pop('_seconds'):.3f} s, shake {shake.pop('_seconds'):.3f} s")
    ok = True
    for name in prod:
        same = all(np.array_equal(prod[name][0], r) for r in prod[name][1:] + shake[name])
        ok &= same
        print(f"{name:24s} product x3 + shake x3 bit-identical: {same}", flush=True)
    print("shake check:", "PASS" if ok else "FAIL")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
