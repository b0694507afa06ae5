"""GPU: the command-line driver (include/fourierbf/cli.hpp run(), the
`fourierbf` tool = reference proj/tools/main.cpp) end to end -- PGM in,
filter() on the B200, PGM + key=value report out -- against the reference's
own run() (oracle/_ref) on the same files, plus the reference test suite's
behaviours (test_cli.cpp)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1603_08081_b200", "_lib", "fourierbf")


def write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode() + np.clip(np.floor(img + 0.5), 0, 255).astype(np.uint8).tobytes())


def read_pgm(path):
    data = open(path, "rb").read()
    head = data.split(b"\n", 3)
    w, h = map(int, head[1].split())
    return np.frombuffer(head[3], dtype=np.uint8).reshape(h, w).astype(np.float64)


def report_of(path):
    return dict(line.split("=", 1) for line in open(path).read().splitlines() if "=" in line)


def checkered(w, h):
    y, x = np.mgrid[0:h, 0:w]
    return np.where((x + y) % 2, 200.0, 40.0)


def cli(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import Reference
    try:
        return Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")


def test_matches_reference_run(tmp_path, ref):
    """same input file -> same output raster (up to rounding ties) and report"""
    rng = np.random.default_rng(33)
    img = np.clip(rng.normal(120, 50, (40, 48)), 0, 255)
    img[10:30, 12:36] += 60
    src = str(tmp_path / "in.pgm")
    write_pgm(src, img)
    for spatial, sigma_s, family, sigma_r in [("gaussian", 2.0, "gaussian", 30.0), ("box", 2.0, "exponential", 25.0)]:
        ours, theirs = str(tmp_path / "o.pgm"), str(tmp_path / "t.pgm")
        rep_o, rep_t = str(tmp_path / "o.txt"), str(tmp_path / "t.txt")
        rc, _, err = cli("--input", src, "--output", ours, "--sigma-s", sigma_s, "--sigma-r", sigma_r,
                         "--spatial", spatial, "--kernel", family, "--report", rep_o, "--compare-exact")
        assert rc == 0, err
        rc_t, _, err_t = ref.cli_run(src, theirs, sigma_s, sigma_r, 1e-3, 1 if family == "exponential" else 0,
                                     spatial=1 if spatial == "box" else 0, compare_exact=True, report=rep_t)
        assert rc_t == 0, err_t
        a, b = read_pgm(ours), read_pgm(theirs)
        assert a.shape == b.shape and np.abs(a - b).max() <= 1 and (a != b).mean() < 0.01
        ro, rt = report_of(rep_o), report_of(rep_t)
        assert ro.keys() == rt.keys()
        for k in ("T", "N", "weaker_guarantee_flag"):
            assert ro[k] == rt[k], k
        for k in ("epsilon_requested", "epsilon_achieved", "w0", "predicted_bound"):
            assert float(ro[k]) == pytest.approx(float(rt[k]), rel=1e-9, abs=1e-12), k
        assert float(ro["measured_linf"]) <= float(ro["predicted_bound"])


def test_constant_image_and_report(tmp_path):
    src, out, rep = (str(tmp_path / n) for n in ("c.pgm", "c_out.pgm", "c.txt"))
    write_pgm(src, np.full((8, 8), 93.0))
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 1, "--sigma-r", 30, "--report", rep)
    assert rc == 0, err
    assert np.all(read_pgm(out) == 93.0)
    text = open(rep).read()
    assert "T=0\n" in text and "N=" not in text


def test_deterministic_box_and_recursive(tmp_path):
    src, out, rep = (str(tmp_path / n) for n in ("d.pgm", "d_out.pgm", "d.txt"))
    write_pgm(src, checkered(20, 14))
    args = ("--input", src, "--output", out, "--sigma-s", 1, "--sigma-r", 30, "--report", rep)
    assert cli(*args)[0] == 0
    first = (open(out, "rb").read(), open(rep).read())
    assert cli(*args)[0] == 0
    assert (open(out, "rb").read(), open(rep).read()) == first
    assert cli("--input", src, "--output", out, "--sigma-s", 1.7, "--sigma-r", 30, "--spatial", "box")[0] == 0
    # the recursive (IIR) backend, as the reference test suite runs it (test_cli.cpp BoxSpatialAndRecursiveBackend)
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 2, "--sigma-r", 30, "--backend", "recursive")
    assert rc == 0, err


def test_recursive_backend_matches_reference_run(tmp_path, ref):
    rng = np.random.default_rng(44)
    src, ours, theirs = (str(tmp_path / n) for n in ("r.pgm", "r_o.pgm", "r_t.pgm"))
    write_pgm(src, np.clip(rng.normal(120, 50, (36, 44)), 0, 255))
    rc, _, err = cli("--input", src, "--output", ours, "--sigma-s", 2.5, "--sigma-r", 25, "--backend", "recursive")
    assert rc == 0, err
    # the reference driver with the recursive backend: build the same run through its run()
    rc_t, _, err_t = ref.cli_run(src, theirs, 2.5, 25.0, 1e-3, backend=1)
    assert rc_t == 0, err_t
    assert np.array_equal(read_pgm(ours), read_pgm(theirs))


def test_tabulated_ones_is_a_plain_blur(tmp_path, oracle):
    src, out, table = (str(tmp_path / n) for n in ("t.pgm", "t_out.pgm", "ones.txt"))
    img = checkered(10, 10)
    write_pgm(src, img)
    open(table, "w").write("1.0\n" * 256)
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 1, "--kernel", f"tabulated:{table}")
    assert rc == 0, err
    s = __import__("paper_1603_08081_b200").make_spatial_gaussian(1.0)
    blur = oracle.convolve(img, s.profile, s.radius)
    frac = blur - np.floor(blur)
    settled = np.abs(frac - 0.5) > 1e-3
    assert np.array_equal(read_pgm(out)[settled], np.floor(blur + 0.5)[settled])


def test_bench_sweeps(tmp_path):
    src = str(tmp_path / "b.pgm")
    write_pgm(src, checkered(16, 16))
    rc, out, err = cli("--input", src, "--sigma-s", 1, "--sigma-r", 30, "--bench")
    assert rc == 0, err
    rows = out.strip().split("\n")
    assert rows[0] == "param,value,millis" and len(rows) == 13
    want = [f"sigma_s,{v}," for v in (1, 2, 5, 8, 10, 12)] + [f"sigma_r,{v}," for v in (10, 15, 20, 30, 50, 100)]
    for row, prefix in zip(rows[1:], want):
        assert row.startswith(prefix) and float(row.split(",")[2]) >= 0
    open(str(tmp_path / "u.txt"), "w").write("1.0\n")
    rc, _, err = cli("--input", src, "--sigma-s", 1, "--bench", "--kernel", f"tabulated:{tmp_path}/u.txt")
    assert rc == 1 and "error:" in err


def test_diagnostics(tmp_path):
    src = str(tmp_path / "x.pgm")
    write_pgm(src, checkered(8, 8))
    out = str(tmp_path / "y.pgm")
    assert cli("--output", out, "--sigma-s", 1, "--sigma-r", 30)[0] != 0  # --input required
    rc, _, err = cli("--input", src, "--sigma-s", 1, "--sigma-r", 30)
    assert rc == 1 and "--output" in err
    rc, _, err = cli("--input", str(tmp_path / "none.pgm"), "--output", out, "--sigma-s", 1, "--sigma-r", 30)
    assert rc == 1 and "error:" in err
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 1, "--sigma-r", 0)
    assert rc == 1 and "--sigma-r" in err
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 3, "--sigma-r", 30, "--epsilon", 0.02)
    assert rc == 1 and "center spatial weight" in err
    open(src, "wb").write(b"P5\n4 4\n255\nxy")
    rc, _, err = cli("--input", src, "--output", out, "--sigma-s", 1, "--sigma-r", 30)
    assert rc == 1 and "at byte" in err
    assert cli("--no-such-flag")[0] != 0
