"""PGM codec of the drop-in C++ API (include/fourierbf/pgm.hpp) against the
reference codec (pgm.hpp:62-133, compiled unmodified into oracle/_ref): same
raster, same bytes, and the same error message -- including the byte offset --
on every malformed input of a handcrafted + mutated corpus.  CPU only."""
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIBDIR = os.path.join(ROOT, "paper_1603_08081_b200", "_lib")


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("pgm") / "pgm_probe")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(HERE, "cpp", "pgm_probe.cpp"), "-o", out, "-L", LIBDIR, "-lfourierbf_b200",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import Reference
    try:
        return Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built (needs /root/reference; __graft_entry__.build())")


def ours_decode(probe, data: bytes):
    r = subprocess.run([probe, "decode"], input=data, capture_output=True, check=True)
    text = r.stdout.decode()
    if text.startswith("error "):
        return "error", text[6:].rstrip("\n")
    lines = text.split("\n")
    _, w, h = lines[0].split()
    w, h = int(w), int(h)
    return "ok", np.array([float(v) for v in lines[1:1 + w * h]]).reshape(h, w)


def ours_encode(probe, img) -> bytes:
    h, w = img.shape
    text = "\n".join(repr(float(v)) for v in img.ravel())
    return subprocess.run([probe, "encode", str(w), str(h)], input=text.encode(), capture_output=True,
                          check=True).stdout


def same(a, b):
    if a[0] != b[0]:
        return False
    return a[1] == b[1] if a[0] == "error" else np.array_equal(a[1], b[1])


def p2_text(img, maxval=255, comment=False):
    h, w = img.shape
    s = "P2\n" + ("# ascii\n" if comment else "") + f"{w} {h}\n{maxval}\n"
    return (s + "\n".join(str(int(v)) for v in img.ravel()) + "\n").encode()


# handcrafted: the reference tests' cases (test_pgm.cpp) and more edges
HANDCRAFTED = [
    b"P5\n1 1\n255\n\x80",
    b"P5 # binary graymap\n# comment line\n  2 1 # dims\n255\n\x03\xfa",
    b"P5\n1 1\n15\n\x07",
    b"P6\n1 1\n255\nx", b"P5\n1 1\n", b"P5\n1 1\n300\nx", b"P5\n2 2\n255\nab", b"P5\n0 1\n255\n",
    b"P2\n2 1\n255\n12", b"P2\n1 1\n100\n101", b"", b"P", b"P5", b"P5\n", b"P5\n-1 1\n255\n",
    b"P5\n1 1\n255", b"P5\n1 1\n255x\x00", b"P5\n1 1\n0\n\x00", b"P5\n1 1\n256\n\x00",
    b"P5\n99999999999 1\n255\n", b"P5\n1048577 1\n255\n", b"P5\n1048576 0\n255\n",
    b"P5\n2 1\n7\n\x07\x08", b"P5\n2 1\n255\n\x01\x02trailing", b"P5\n1 1\n255\r\x05",
    b"P5\n1 1\n255\t\x05", b"P5\n1 1\n255\x0b\x05", b"P2\n2 2\n255\n1 2\n3 # c\n4",
    b"P2\n2 1\n255\n1 x", b"P2 1 1 255 0", b"P5#c\n1 1\n255\n\x00", b"P5\n1#c\n1\n255\n\x09",
    b"p5\n1 1\n255\n\x00", b"P3\n1 1\n255\n0",
]


def test_decode_matches_reference_handcrafted(probe, ref):
    for data in HANDCRAFTED:
        assert same(ours_decode(probe, data), ref.decode_pgm(data)), data


def test_decode_matches_reference_random_and_mutated(probe, ref):
    rng = np.random.default_rng(1603)
    cases = []
    for k in range(40):
        w, h = int(rng.integers(1, 13)), int(rng.integers(1, 9))
        maxval = int(rng.choice([1, 15, 200, 255]))
        img = rng.integers(0, maxval + 1, (h, w)).astype(np.float64)
        raw = ref.encode_pgm(img) if maxval == 255 else (f"P5\n{w} {h}\n{maxval}\n".encode() +
                                                        img.astype(np.uint8).tobytes())
        txt = p2_text(img, maxval, comment=bool(k % 2))
        cases += [raw, txt]
        for base in (raw, txt):  # truncations and byte flips
            cut = int(rng.integers(0, len(base)))
            cases.append(base[:cut])
            b = bytearray(base)
            for _ in range(2):
                b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
            cases.append(bytes(b))
    for data in cases:
        assert same(ours_decode(probe, data), ref.decode_pgm(data)), data


def test_encode_matches_reference(probe, ref):
    rng = np.random.default_rng(7)
    for k in range(20):
        w, h = int(rng.integers(1, 17)), int(rng.integers(1, 9))
        img = rng.uniform(-20, 280, (h, w))
        img.ravel()[: min(4, w * h)] = [0.5, 1.49, 254.5, -0.5][: min(4, w * h)]  # ties and edges
        assert ours_encode(probe, img) == ref.encode_pgm(img)
    ints = rng.integers(0, 256, (7, 16)).astype(np.float64)
    assert same(ours_decode(probe, ours_encode(probe, ints)), ("ok", ints))
