"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracles.

* ``Oracle``    : oracle/_build/libfbf_oracle.so, the plain-C fp64 restatement
                  (oracle/fbf_oracle.c) of the reference path.
* ``Reference`` : oracle/_ref/libfbf_ref.so, the UNMODIFIED reference headers
                  compiled in place (oracle/ref_shim.cpp + oracle/Makefile).
* ``synth_image``: oracle/_synth/libfbf_synth.so, the BASELINE input generator
                  built from the product's own generator source, so the
                  reference arm of bench.py never loads the product library.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfbf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfbf_ref.so")
SYNTH_SO = os.path.join(HERE, "_synth", "libfbf_synth.so")

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_LL = ctypes.POINTER(ctypes.c_longlong)


def build() -> None:
    """Compile the restatement (always) and the reference shim (when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def spatial_kind(spatial) -> int:
    return int(spatial.kind)


class Oracle:
    """fp64 restatement; bit-identical to the reference by construction (evaluation order)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.fbo_mirror_index.restype = ctypes.c_int
        L.fbo_mirror_index.argtypes = [ctypes.c_int, ctypes.c_int]
        L.fbo_spatial_gaussian.argtypes = [ctypes.c_double, _D, _I, _D]
        L.fbo_spatial_box.argtypes = [ctypes.c_int, _D, _D]
        L.fbo_range_eval.restype = ctypes.c_double
        L.fbo_range_eval.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.fbo_fit_fixed.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _D, _D]
        L.fbo_progressive_fit.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double, _D, _I,
                                          _D, _D]
        L.fbo_convolve.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_int]
        L.fbo_bilateral_fast.argtypes = [_D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, ctypes.c_double, _D,
                                         ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, _D, _LL]
        L.fbo_bilateral_exact.argtypes = [_D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.fbo_local_dynamic_range.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.fbo_partial_sums.argtypes = [_D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, _D, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, _D]
        L.fbo_error_bound.restype = ctypes.c_double
        L.fbo_error_bound.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        self.L = L

    def mirror_index(self, i, n):
        return self.L.fbo_mirror_index(i, n)

    def spatial_gaussian(self, sigma_s):
        r = ctypes.c_int()
        self.L.fbo_spatial_gaussian(sigma_s, None, ctypes.byref(r), None)
        p = np.zeros(2 * r.value + 1)
        w0 = ctypes.c_double()
        self.L.fbo_spatial_gaussian(sigma_s, _dp(p), ctypes.byref(r), ctypes.byref(w0))
        return r.value, p, w0.value

    def spatial_box(self, radius):
        p = np.zeros(2 * radius + 1)
        w0 = ctypes.c_double()
        self.L.fbo_spatial_box(radius, _dp(p), ctypes.byref(w0))
        return radius, p, w0.value

    def range_eval(self, family, sigma_r, t):
        return self.L.fbo_range_eval(family, sigma_r, t)

    def fit_fixed(self, family, sigma_r, T, N):
        d = np.zeros(N + 1)
        rn, mx = ctypes.c_double(), ctypes.c_double()
        rc = self.L.fbo_fit_fixed(family, sigma_r, T, N, _dp(d), ctypes.byref(rn), ctypes.byref(mx))
        if rc:
            raise ValueError("fit rejected a column")
        return d, rn.value, mx.value

    def progressive_fit(self, family, sigma_r, T, eps):
        d = np.zeros(T + 1)
        n = ctypes.c_int()
        rn, mx = ctypes.c_double(), ctypes.c_double()
        rc = self.L.fbo_progressive_fit(family, sigma_r, T, eps, _dp(d), ctypes.byref(n), ctypes.byref(rn),
                                        ctypes.byref(mx))
        if rc:
            raise ValueError("progressive_fit failed")
        return d[: n.value + 1].copy(), n.value, rn.value, mx.value

    def convolve(self, img, profile, radius):
        a = _f64(img)
        out = np.empty_like(a)
        self.L.fbo_convolve(_dp(a), _dp(out), a.shape[1], a.shape[0], _dp(_f64(profile)), radius)
        return out

    def bilateral_fast(self, img, profile, radius, w0, d, omega, max_err, check_eps=True, row0=0, row1=None,
                       nthreads=1):
        """Returns (out rows [row0,row1), rc, bad_index)."""
        a = _f64(img)
        h, w = a.shape
        row1 = h if row1 is None else row1
        out = np.zeros((row1 - row0, w))
        bad = ctypes.c_longlong(-1)
        dd = _f64(d)
        rc = self.L.fbo_bilateral_fast(_dp(a), w, h, _dp(_f64(profile)), radius, w0, _dp(dd), len(dd) - 1, omega,
                                       max_err, 1 if check_eps else 0, row0, row1, nthreads, _dp(out),
                                       ctypes.byref(bad))
        return out, rc, bad.value

    def bilateral_exact(self, img, profile, radius, family, sigma_r, row0=0, row1=None, nthreads=1):
        a = _f64(img)
        h, w = a.shape
        row1 = h if row1 is None else row1
        out = np.zeros((row1 - row0, w))
        self.L.fbo_bilateral_exact(_dp(a), w, h, _dp(_f64(profile)), radius, family, sigma_r, row0, row1,
                                   nthreads, _dp(out))
        return out

    def local_dynamic_range(self, img, W):
        a = _f64(img)
        return self.L.fbo_local_dynamic_range(_dp(a), a.shape[1], a.shape[0], W)

    def error_bound(self, T, eps, w0):
        return self.L.fbo_error_bound(T, eps, w0)

    def partial_sums(self, img, profile, radius, d, omega, n_lo, n_hi, row0=0, row1=None):
        """(P, Q) over harmonics [n_lo, n_hi)."""
        a = _f64(img)
        h, w = a.shape
        row1 = h if row1 is None else row1
        P = np.zeros((row1 - row0, w))
        Q = np.zeros((row1 - row0, w))
        dd = _f64(d)
        self.L.fbo_partial_sums(_dp(a), w, h, _dp(_f64(profile)), radius, _dp(dd), len(dd) - 1, omega, n_lo, n_hi,
                                row0, row1, _dp(P), _dp(Q))
        return P, Q


class Reference:
    """The reference library itself (oracle/_ref/libfbf_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_make_spatial.argtypes = [ctypes.c_int, ctypes.c_double, _D, _I, _D]
        L.ref_range_eval.restype = ctypes.c_double
        L.ref_range_eval.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.ref_fit_fixed.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _D, _D]
        L.ref_progressive_fit.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double, _D, _I,
                                          _D, _D]
        L.ref_convolve.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.ref_bilateral_fast_rows.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _D,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.ref_bilateral_exact_rows.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, _D]
        L.ref_local_dynamic_range.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ref_error_bound.restype = ctypes.c_double
        L.ref_error_bound.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.ref_decode_pgm.argtypes = [ctypes.c_char_p, ctypes.c_size_t, _D, ctypes.c_size_t, _I, _I]
        L.ref_cli_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                                  ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int]
        L.ref_convolve_recursive.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.ref_bilateral_fast_recursive.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_double, _D, ctypes.c_int,
                                                   ctypes.c_int, ctypes.c_double, _D]
        L.ref_encode_pgm.restype = ctypes.c_long
        L.ref_encode_pgm.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]
        self.L = L

    def last_error(self):
        return self.L.ref_last_error().decode()

    def make_spatial(self, kind, param):
        r = ctypes.c_int()
        self.L.ref_make_spatial(kind, param, None, ctypes.byref(r), None)
        p = np.zeros(2 * r.value + 1)
        w0 = ctypes.c_double()
        rc = self.L.ref_make_spatial(kind, param, _dp(p), ctypes.byref(r), ctypes.byref(w0))
        if rc:
            raise ValueError(self.last_error())
        return r.value, p, w0.value

    def range_eval(self, family, sigma_r, t):
        return self.L.ref_range_eval(family, sigma_r, t)

    def fit_fixed(self, family, sigma_r, T, N):
        d = np.zeros(N + 1)
        rn, mx = ctypes.c_double(), ctypes.c_double()
        if self.L.ref_fit_fixed(family, sigma_r, T, N, _dp(d), ctypes.byref(rn), ctypes.byref(mx)):
            raise ValueError(self.last_error())
        return d, rn.value, mx.value

    def progressive_fit(self, family, sigma_r, T, eps):
        d = np.zeros(T + 1)
        n = ctypes.c_int()
        rn, mx = ctypes.c_double(), ctypes.c_double()
        if self.L.ref_progressive_fit(family, sigma_r, T, eps, _dp(d), ctypes.byref(n), ctypes.byref(rn),
                                      ctypes.byref(mx)):
            raise ValueError(self.last_error())
        return d[: n.value + 1].copy(), n.value, rn.value, mx.value

    def convolve(self, img, kind, param):
        a = _f64(img)
        out = np.empty_like(a)
        if self.L.ref_convolve(_dp(a), _dp(out), a.shape[1], a.shape[0], kind, param):
            raise ValueError(self.last_error())
        return out

    def bilateral_fast(self, img, kind, param, d, T, max_err, check_eps=True, row0=0, row1=None, nthreads=1):
        a = _f64(img)
        h, w = a.shape
        row1 = h if row1 is None else row1
        out = np.zeros((row1 - row0, w))
        dd = _f64(d)
        rc = self.L.ref_bilateral_fast_rows(_dp(a), w, h, kind, param, _dp(dd), len(dd) - 1, T, max_err,
                                            1 if check_eps else 0, row0, row1, nthreads, _dp(out))
        return out, rc, (self.last_error() if rc else "")

    def bilateral_exact(self, img, kind, param, family, sigma_r, row0=0, row1=None, nthreads=1):
        a = _f64(img)
        h, w = a.shape
        row1 = h if row1 is None else row1
        out = np.zeros((row1 - row0, w))
        if self.L.ref_bilateral_exact_rows(_dp(a), w, h, kind, param, family, sigma_r, row0, row1, nthreads,
                                           _dp(out)):
            raise ValueError(self.last_error())
        return out

    def local_dynamic_range(self, img, W):
        a = _f64(img)
        return self.L.ref_local_dynamic_range(_dp(a), a.shape[1], a.shape[0], W)

    def error_bound(self, T, eps, w0):
        return self.L.ref_error_bound(T, eps, w0)

    def decode_pgm(self, data: bytes):
        """pgm.hpp decode_pgm -> ("ok", array HxW) or ("error", message)"""
        cap = 1 << 22
        v = np.zeros(cap)
        w, h = ctypes.c_int(), ctypes.c_int()
        if self.L.ref_decode_pgm(data, len(data), _dp(v), cap, ctypes.byref(w), ctypes.byref(h)):
            return "error", self.last_error()
        return "ok", v[: w.value * h.value].reshape(h.value, w.value).copy()

    def encode_pgm(self, img) -> bytes:
        a = _f64(img)
        h, w = a.shape
        buf = ctypes.create_string_buffer(w * h + 64)
        n = self.L.ref_encode_pgm(_dp(a), w, h, buf, len(buf))
        if n < 0:
            raise ValueError(self.last_error())
        return buf.raw[:n]

    def cli_run(self, input_path, output_path="", sigma_s=1.0, sigma_r=30.0, epsilon=1e-3, family=0, table="",
                spatial=0, compare_exact=False, report="", bench=False, backend=0):
        """cli.hpp run() -> (rc, stdout text, stderr text)"""
        out = ctypes.create_string_buffer(1 << 16)
        err = ctypes.create_string_buffer(1 << 12)
        enc = lambda v: v.encode() if v else None  # noqa: E731
        rc = self.L.ref_cli_run(enc(input_path), enc(output_path), sigma_s, sigma_r, epsilon, family, enc(table),
                                spatial, int(compare_exact), enc(report), int(bench), out, len(out), err, len(err),
                                backend)
        return rc, out.value.decode(), err.value.decode()

    def convolve_recursive(self, img, sigma):
        """convolve(..., ConvolutionBackend::recursive) on a whole image"""
        a = _f64(img)
        out = np.empty_like(a)
        if self.L.ref_convolve_recursive(_dp(a), _dp(out), a.shape[1], a.shape[0], sigma):
            raise ValueError(self.last_error())
        return out

    def bilateral_fast_recursive(self, img, sigma, d, T, max_err):
        """bilateral_fast(..., ConvolutionBackend::recursive) on a whole image, Gaussian window of sigma"""
        a = _f64(img)
        out = np.empty_like(a)
        dd = _f64(d)
        if self.L.ref_bilateral_fast_recursive(_dp(a), a.shape[1], a.shape[0], sigma, _dp(dd), len(dd) - 1, T, max_err,
                                               _dp(out)):
            raise ValueError(self.last_error())
        return out


_SYNTH = None


def synth_image(seed, width, height, rects, noise, row0=0, rows=None, nthreads=None):
    """fbf_synth_image from oracle/_synth/libfbf_synth.so -> float32 array (rows x width)."""
    global _SYNTH
    if _SYNTH is None:
        if not os.path.exists(SYNTH_SO):
            build()
        L = ctypes.CDLL(SYNTH_SO)
        L.fbf_synth_image.argtypes = [ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_float), ctypes.c_int]
        _SYNTH = L
    rows = height - row0 if rows is None else rows
    out = np.empty((rows, width), dtype=np.float32)
    rc = _SYNTH.fbf_synth_image(seed, width, height, rects, noise, row0, rows,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), nthreads or os.cpu_count() or 1)
    if rc:
        raise ValueError("fbf_synth_image: invalid arguments")
    return out
