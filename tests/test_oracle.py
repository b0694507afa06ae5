"""CPU: pin the oracle (oracle/fbf_oracle.c) before trusting it.

1. against golden vectors produced by the reference itself (tests/golden, made by
   tests/golden/make_golden.py from oracle/_ref = the unmodified reference headers);
2. against the reference's own known-answer tests
   (test_spatial.cpp:48-61, test_kernel_approx.cpp:62-80,139-158);
3. bit-for-bit against the live reference build when oracle/_ref is present.
"""
import os

import numpy as np
import pytest

from paper_1603_08081_b200.configs import CONFIGS, T_FIXED

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return Reference()


def test_mirror_index_matches_reference_rule(oracle):
    # image.hpp:34-40: -1 -> 0, n -> n-1, period 2n for any offset
    assert oracle.mirror_index(-1, 5) == 0
    assert oracle.mirror_index(5, 5) == 4
    assert oracle.mirror_index(-6, 5) == 4
    assert oracle.mirror_index(10, 5) == 0
    assert oracle.mirror_index(-11, 5) == 0
    assert [oracle.mirror_index(i, 1) for i in range(-3, 4)] == [0] * 7
    for n in (1, 2, 3, 7):
        for i in range(-4 * n, 5 * n):
            m = oracle.mirror_index(i, n)
            assert 0 <= m < n
            j = i % (2 * n)
            assert m == (j if j < n else 2 * n - 1 - j)


def test_spatial_known_answers(oracle):
    # test_spatial.cpp:48-61
    r, p, w0 = oracle.spatial_gaussian(1.0)
    assert r == 3 and abs(w0 - 0.159241125690702) < 1e-14
    r, p, w0 = oracle.spatial_gaussian(2.0)
    assert r == 6 and abs(w0 - 0.039870356216689) < 1e-14
    r, p, w0 = oracle.spatial_gaussian(3.0)
    assert r == 9 and abs(w0 - 0.017735845914730) < 1e-14
    assert oracle.spatial_gaussian(2.5)[0] == 8
    r, p, w0 = oracle.spatial_box(2)
    assert np.all(p == 0.2) and w0 == pytest.approx(1.0 / 25.0, rel=1e-15)  # EXPECT_DOUBLE_EQ


def test_spatial_matches_golden(oracle):
    g = gold("spatial")
    for s in (1.0, 1.5, 2.0, 2.5, 3.0, 4.0, 5.0, 8.0):
        r, p, w0 = oracle.spatial_gaussian(s)
        assert r == int(g[f"g{s}_radius"])
        assert np.array_equal(p, g[f"g{s}_profile"]) and w0 == float(g[f"g{s}_w0"])
    for r in range(1, 6):
        _, p, w0 = oracle.spatial_box(r)
        assert np.array_equal(p, g[f"b{r}_profile"]) and w0 == float(g[f"b{r}_w0"])


def test_fit_matches_golden_and_survey(oracle):
    g = gold("fits")
    for name, c in CONFIGS.items():
        d, rn, mx = oracle.fit_fixed(c.range_family, c.sigma_r, T_FIXED, c.N)
        assert np.array_equal(d, g[f"{name}_d"]), name
        assert rn == float(g[f"{name}_residual"]) and mx == float(g[f"{name}_eps"])
    # c1 coefficients and the c3 precondition violation
    d, _, _ = oracle.fit_fixed(0, 30.0, 255, 12)
    assert np.allclose(d[:3], [0.147449, 0.275428, 0.224398], atol=1e-6)
    assert float(g["c3_eps"]) > 1.0 / 121.0


def test_qr_two_point_and_progressive_known_answers(oracle):
    # test_kernel_approx.cpp:139-158: N = 9 at (gaussian 30, T = 217, eps = 1e-3)
    d, n, rn, mx = oracle.progressive_fit(0, 30.0, 217, 1e-3)
    assert n == 9 and rn <= 1e-3 and mx <= rn
    g = gold("fits")
    assert np.array_equal(d, g["prog_g30_T217_e1e-3_d"])


def test_bilateral_fast_matches_reference_golden(oracle):
    g = gold("fits")
    f = gold("filters")
    for name, c in CONFIGS.items():
        img = f[f"{name}_img"].astype(np.float64)
        if c.spatial == "box":
            r, p, w0 = oracle.spatial_box(int(c.sigma_s))
        else:
            r, p, w0 = oracle.spatial_gaussian(c.sigma_s)
        out, rc, _ = oracle.bilateral_fast(img, p, r, w0, g[f"{name}_d"], np.pi / T_FIXED,
                                           float(g[f"{name}_eps"]), c.check_epsilon)
        assert rc == 0
        assert np.array_equal(out, f[f"{name}_out"]), name  # bit-identical to the reference
    for i in range(5):
        img = f[f"rand{i}_img"]
        r, p, w0 = oracle.spatial_gaussian(float(f[f"rand{i}_sigma"]))
        out, rc, _ = oracle.bilateral_fast(img, p, r, w0, f["rand_d"], np.pi / 255, float(f["rand_eps"]))
        assert rc == 0 and np.array_equal(out, f[f"rand{i}_out"])


def test_bilateral_exact_matches_reference_golden(oracle):
    e = gold("exact")
    for i in range(2):
        r, p, _ = oracle.spatial_gaussian(float(e[f"e{i}_sigma"]))
        out = oracle.bilateral_exact(e[f"e{i}_img"], p, r, 0, float(e[f"e{i}_sr"]))
        assert np.array_equal(out, e[f"e{i}_out"])


def test_row_ranges_and_threads_are_bit_identical(oracle):
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (41, 37)).astype(np.float64)
    r, p, w0 = oracle.spatial_gaussian(2.0)
    d, _, mx = oracle.fit_fixed(0, 25.0, 255, 9)
    whole, rc, _ = oracle.bilateral_fast(img, p, r, w0, d, np.pi / 255, mx)
    assert rc == 0
    for a, b in ((0, 5), (3, 20), (30, 41)):
        part, rc, _ = oracle.bilateral_fast(img, p, r, w0, d, np.pi / 255, mx, True, a, b, 3)
        assert rc == 0 and np.array_equal(part, whole[a:b])


def test_oracle_exceptions_mirror_reference(oracle):
    img = np.full((6, 6), 50.0)
    r, p, w0 = oracle.spatial_gaussian(1.0)
    _, rc, _ = oracle.bilateral_fast(img, p, r, w0, np.array([1.0]), np.pi / 255, 0.5)  # eps >= w0
    assert rc == 1
    _, rc, bad = oracle.bilateral_fast(img, p, r, w0, np.array([0.0]), np.pi / 255, 0.0)  # Q = 0
    assert rc == 2 and bad == 0


def test_oracle_bit_identical_to_live_reference(oracle, ref):
    rng = np.random.default_rng(11)
    for (w, h, s, kind) in ((29, 23, 2.0, 0), (17, 31, 3, 1), (5, 4, 1.5, 0), (1, 12, 1.0, 0)):
        img = rng.integers(0, 256, (h, w)).astype(np.float64) + rng.random((h, w))
        r, p, w0 = oracle.spatial_box(int(s)) if kind else oracle.spatial_gaussian(s)
        d, _, mx = ref.fit_fixed(0, 20.0, 255, 11)
        o1, rc1, _ = oracle.bilateral_fast(img, p, r, w0, d, np.pi / 255, mx)
        o2, rc2, _ = ref.bilateral_fast(img, kind, s, d, 255, mx)
        assert rc1 == rc2 == 0 and np.array_equal(o1, o2)
        assert np.array_equal(oracle.convolve(img, p, r), ref.convolve(img, kind, s))
        assert oracle.local_dynamic_range(img, r) == ref.local_dynamic_range(img, r)
