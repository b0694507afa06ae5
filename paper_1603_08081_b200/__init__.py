"""paper_1603_08081_b200 -- B200-native shiftable Fourier-kernel bilateral filter.

Python mirror of the reference's operator interface for the hot path
(/root/reference/proj/include/fourierbf: ``make_spatial_gaussian``,
``make_spatial_box``, ``progressive_fit``, ``bilateral_fast``, ``convolve``,
``error_bound``), implemented as a thin ctypes layer over the C-ABI
``include/fourierbf_b200.h`` of ``_lib/libfourierbf_b200.so``.  The native
library is required: importing this package without it raises ImportError, and
no call ever falls back to a CPU implementation.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FBF_LIBRARY: diagnostics only (tools/phase_probe.py loads an instrumented build)
LIB_PATH = os.environ.get("FBF_LIBRARY") or os.path.join(_HERE, "_lib", "libfourierbf_b200.so")

FBF_OK, FBF_EINVAL, FBF_EANOMALY, FBF_ECUDA, FBF_EUNSUPPORTED = 0, 1, 2, 3, 4
SPATIAL_GAUSSIAN, SPATIAL_BOX = 0, 1
RANGE_GAUSSIAN, RANGE_EXPONENTIAL = 0, 1
VARIANT_FUSED, VARIANT_NAIVE, VARIANT_RECURSIVE = 0, 1, 2
# "recursive" = ConvolutionBackend::recursive (IIR Gaussian, fp64; Gaussian windows with sigma >= 2)
_VARIANTS = {"fused": VARIANT_FUSED, "naive": VARIANT_NAIVE, "recursive": VARIANT_RECURSIVE}


class Geometry(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int), ("height", ctypes.c_int), ("batch", ctypes.c_int),
        ("src_row0", ctypes.c_int), ("src_rows", ctypes.c_int),
        ("out_row0", ctypes.c_int), ("out_rows", ctypes.c_int),
        ("src_pitch", ctypes.c_longlong), ("dst_pitch", ctypes.c_longlong),
        ("src_bstride", ctypes.c_longlong), ("dst_bstride", ctypes.c_longlong),
    ]


class Filter(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int), ("radius", ctypes.c_int),
        ("profile", ctypes.POINTER(ctypes.c_double)), ("w0", ctypes.c_double),
        ("N", ctypes.c_int), ("d", ctypes.POINTER(ctypes.c_double)),
        ("omega", ctypes.c_double), ("max_pointwise_error", ctypes.c_double),
        ("check_epsilon", ctypes.c_int),
        ("sigma_s", ctypes.c_double),
    ]


# name -> (restype, argtypes): every symbol include/fourierbf_b200.h declares
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_I = ctypes.POINTER(ctypes.c_int)
_LL = ctypes.POINTER(ctypes.c_longlong)
SIGNATURES = {
    "fbf_last_error": (ctypes.c_char_p, []),
    "fbf_version": (ctypes.c_int, []),
    "fbf_geometry_whole": (None, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "fbf_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int]),
    "fbf_bilateral_fast_device": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _P, _P, _P,
                                                 ctypes.c_size_t, _P, ctypes.c_int, _P]),
    "fbf_prepare_device": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _P, _P,
                                          ctypes.c_size_t, ctypes.c_int, _P]),
    "fbf_filter_prepared_device": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _P, _P,
                                                  ctypes.c_size_t, _P, ctypes.c_int, _P]),
    "fbf_launches_per_call": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), ctypes.c_int]),
    "fbf_partial_sums_device": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), ctypes.c_int,
                                               ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_int, _P]),
    "fbf_finish_device": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _P, _P, _P, _P]),
    "fbf_bilateral_fast_host": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _F, _F,
                                               ctypes.c_int, _LL]),
    "fbf_bilateral_fast_host_f64": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _D, _D,
                                                   ctypes.c_int, _LL]),
    "fbf_convolve_device": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, _P, _P, _P,
                                           ctypes.c_size_t, _P]),
    "fbf_convolve_host_f64": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, _D, _D]),
    "fbf_convolve_device_f64": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, _P, _P, _P,
                                               ctypes.c_size_t, _P]),
    "fbf_convolve_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "fbf_bilateral_fast_host_multi": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _F, _F,
                                                     ctypes.c_int, _LL, _I, ctypes.c_int]),
    "fbf_bilateral_fast_host_multi_f64": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.POINTER(Filter), _D, _D,
                                                         ctypes.c_int, _LL, _I, ctypes.c_int]),
    "fbf_convolve_recursive_host_f64": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_double, _D, _D]),
    "fbf_harmonic_groups": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int]),
    "fbf_spatial_gaussian": (ctypes.c_int, [ctypes.c_double, _D, _I, _D]),
    "fbf_spatial_box": (ctypes.c_int, [ctypes.c_int, _D, _D]),
    "fbf_range_eval": (ctypes.c_double, [ctypes.c_int, ctypes.c_double, ctypes.c_double]),
    "fbf_fit_fixed": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _D, _D]),
    "fbf_progressive_fit": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double, _D,
                                           _I, _D, _D]),
    "fbf_error_bound": (ctypes.c_double, [ctypes.c_int, ctypes.c_double, ctypes.c_double]),
    "fbf_synth_image": (ctypes.c_int, [ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, _F, ctypes.c_int]),
    "fbf_probe_fma_peak": (ctypes.c_int, [_D, _D, _P]),
    "fbf_release_host_buffers": (None, []),
    "fbf_local_dynamic_range_host_f64": (ctypes.c_int, [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I]),
    "fbf_bilateral_exact_host_f64": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D, ctypes.c_int, ctypes.c_int,
                                                    ctypes.c_double, _D, _D]),
    "fbf_bilateral_exact_device": (ctypes.c_int, [ctypes.POINTER(Geometry), _D, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_double, _P, _P, _P]),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the filter)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class FilterError(RuntimeError):
    """std::runtime_error of the reference (numerical anomaly, CUDA failure)."""


def _check(rc: int) -> None:
    if rc == FBF_OK:
        return
    msg = lib.fbf_last_error().decode()
    if rc == FBF_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise FilterError(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


# --------------------------------------------------------------------- types

@dataclass
class SpatialKernel:
    """spatial.hpp:22-33"""
    kind: int
    sigma_s: float
    radius: int
    profile: np.ndarray
    w0: float

    def weight(self, dx: int, dy: int) -> float:
        return float(self.profile[dx + self.radius] * self.profile[dy + self.radius])


@dataclass
class FourierKernelApprox:
    """kernel_approx.hpp:19-44"""
    T: int
    omega: float
    N: int
    d: np.ndarray
    residual_norm: float = 0.0
    max_pointwise_error: float = 0.0

    def evaluate(self, t):
        n = np.arange(self.N + 1)
        return np.cos(np.multiply.outer(np.asarray(t, dtype=np.float64), n * self.omega)) @ self.d


def make_spatial_gaussian(sigma_s: float) -> SpatialKernel:
    r = ctypes.c_int()
    if lib.fbf_spatial_gaussian(float(sigma_s), None, ctypes.byref(r), None) != FBF_OK:
        raise ValueError("spatial sigma must be positive")
    prof = np.zeros(2 * r.value + 1)
    w0 = ctypes.c_double()
    lib.fbf_spatial_gaussian(float(sigma_s), _dp(prof), ctypes.byref(r), ctypes.byref(w0))
    return SpatialKernel(SPATIAL_GAUSSIAN, float(sigma_s), r.value, prof, w0.value)


def make_spatial_box(radius: int) -> SpatialKernel:
    if radius < 1:
        raise ValueError("box radius must be at least 1")
    prof = np.zeros(2 * radius + 1)
    w0 = ctypes.c_double()
    lib.fbf_spatial_box(int(radius), _dp(prof), ctypes.byref(w0))
    return SpatialKernel(SPATIAL_BOX, 0.0, int(radius), prof, w0.value)


def fit_fixed(family: int, sigma_r: float, T: int, N: int) -> FourierKernelApprox:
    """Fixed-order least-squares fit via the recursive QR (acceptance.cpp:247-263 pattern)."""
    d = np.zeros(N + 1)
    rn, mx = ctypes.c_double(), ctypes.c_double()
    _check(lib.fbf_fit_fixed(family, float(sigma_r), int(T), int(N), _dp(d), ctypes.byref(rn), ctypes.byref(mx)))
    return FourierKernelApprox(int(T), float(np.pi / T), int(N), d, rn.value, mx.value)


def progressive_fit(family: int, sigma_r: float, T: int, epsilon: float) -> FourierKernelApprox:
    """kernel_approx.hpp:169-219"""
    d = np.zeros(T + 1)
    n = ctypes.c_int()
    rn, mx = ctypes.c_double(), ctypes.c_double()
    _check(lib.fbf_progressive_fit(family, float(sigma_r), int(T), float(epsilon), _dp(d), ctypes.byref(n),
                                   ctypes.byref(rn), ctypes.byref(mx)))
    return FourierKernelApprox(int(T), float(np.pi / T), n.value, d[: n.value + 1].copy(), rn.value, mx.value)


def local_dynamic_range(image: np.ndarray, W: int) -> int:
    """bilateral.hpp:21-74 on the GPU (fp64, exact)."""
    a = np.ascontiguousarray(image, dtype=np.float64)
    if a.size == 0:
        raise ValueError("local_dynamic_range: empty image")
    if W < 1:
        raise ValueError("local_dynamic_range: window radius must be positive")
    T = ctypes.c_int()
    rc = lib.fbf_local_dynamic_range_host_f64(_dp(a), a.shape[1], a.shape[0], int(W), ctypes.byref(T))
    if rc != FBF_OK:
        raise FilterError("local_dynamic_range: CUDA failure")
    return T.value


def filter(image: np.ndarray, spatial: SpatialKernel, family: int, sigma_r: float, epsilon: float = 1e-3,
           integer_intensities: bool = True):
    """bilateral.hpp:173-196: round, T from the data (GPU), progressive fit (host), bilateral_fast (GPU).

    Returns (output, report dict) like the reference's (Image, AccuracyReport)."""
    if not epsilon > 0.0:
        raise ValueError("filter: tolerance must be positive")
    if not epsilon < spatial.w0:
        raise ValueError("filter: tolerance must stay below the center spatial weight w(0); lower "
                         "--epsilon or reduce the spatial radius")
    src = np.asarray(image, dtype=np.float64)
    working = np.floor(src + 0.5) if integer_intensities else src
    T = local_dynamic_range(working, spatial.radius)
    weaker = not integer_intensities
    if T == 0:
        return src.copy(), {"T": 0, "N": None, "epsilon_requested": epsilon, "epsilon_achieved": 0.0,
                            "w0": spatial.w0, "predicted_bound": 0.0, "weaker_guarantee_flag": weaker}
    approx = progressive_fit(family, sigma_r, T, epsilon)
    out = bilateral_fast(working, spatial, approx)
    bound = (lib.fbf_error_bound(T, approx.max_pointwise_error, spatial.w0)
             if approx.max_pointwise_error < spatial.w0 else float("inf"))
    return out, {"T": T, "N": approx.N, "epsilon_requested": epsilon,
                 "epsilon_achieved": approx.max_pointwise_error, "w0": spatial.w0, "predicted_bound": bound,
                 "weaker_guarantee_flag": weaker}


def error_bound(T: int, epsilon: float, w0: float) -> float:
    """analysis.hpp:27-34"""
    if T < 0 or not epsilon >= 0.0 or not epsilon < w0:
        raise ValueError("error_bound: tolerance must stay below the center spatial weight")
    return lib.fbf_error_bound(int(T), float(epsilon), float(w0))


def _filter_struct(spatial: SpatialKernel, approx: FourierKernelApprox, check_epsilon: bool = True):
    prof = np.ascontiguousarray(spatial.profile, dtype=np.float64)
    d = np.ascontiguousarray(approx.d, dtype=np.float64)
    f = Filter(spatial.kind, spatial.radius, _dp(prof), spatial.w0, approx.N, _dp(d), approx.omega,
               approx.max_pointwise_error, 1 if check_epsilon else 0, spatial.sigma_s)
    f._keep = (prof, d)  # keep the buffers alive with the struct
    return f


def harmonic_groups(geometry: Geometry, radius: int, N: int) -> int:
    """CTA groups the fused path splits the N+1 harmonics into for this geometry."""
    return lib.fbf_harmonic_groups(ctypes.byref(geometry), radius, N)


def whole_geometry(width: int, height: int, batch: int = 1) -> Geometry:
    g = Geometry()
    lib.fbf_geometry_whole(ctypes.byref(g), int(width), int(height), int(batch))
    return g


def strip_geometry(width: int, height: int, out_row0: int, out_rows: int, radius: int,
                   batch: int = 1) -> Geometry:
    """Row strip [out_row0, out_row0+out_rows) with its W halo rows (mirror only at global edges)."""
    lo = max(0, out_row0 - radius)
    hi = min(height, out_row0 + out_rows + radius)
    if height <= 2 * radius + 1:
        lo, hi = 0, height
    g = Geometry()
    g.width, g.height, g.batch = width, height, batch
    g.src_row0, g.src_rows = lo, hi - lo
    g.out_row0, g.out_rows = out_row0, out_rows
    g.src_pitch = g.dst_pitch = width
    g.src_bstride = (hi - lo) * width
    g.dst_bstride = out_rows * width
    return g


def bilateral_fast(image: np.ndarray, spatial: SpatialKernel, approx: FourierKernelApprox,
                   variant: str = "fused", check_epsilon: bool = True) -> np.ndarray:
    """bilateral.hpp:109-160 on the GPU: host array in, host array out (fp32 compute).

    ``image`` is (H, W) or (B, H, W); float64 or float32.  Raises ValueError
    (invalid_argument) / FilterError (runtime_error) like the reference.
    """
    a = np.asarray(image)
    if a.size == 0:
        raise ValueError("bilateral_fast: empty image")
    batch = 1 if a.ndim == 2 else a.shape[0]
    h, w = a.shape[-2], a.shape[-1]
    g = whole_geometry(w, h, batch)
    f = _filter_struct(spatial, approx, check_epsilon)
    bad = ctypes.c_longlong(-1)
    if a.dtype == np.float32:
        src = np.ascontiguousarray(a)
        out = np.empty_like(src)
        rc = lib.fbf_bilateral_fast_host(ctypes.byref(g), ctypes.byref(f), src.ctypes.data_as(_F),
                                         out.ctypes.data_as(_F), _VARIANTS[variant], ctypes.byref(bad))
    else:
        src = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty_like(src)
        rc = lib.fbf_bilateral_fast_host_f64(ctypes.byref(g), ctypes.byref(f), _dp(src), _dp(out),
                                             _VARIANTS[variant], ctypes.byref(bad))
    _check(rc)
    return out


def bilateral_fast_multi(image: np.ndarray, spatial: SpatialKernel, approx: FourierKernelApprox,
                         devices: Sequence[int], variant: str = "fused", check_epsilon: bool = True) -> np.ndarray:
    """One call over several GPUs (fbf_bilateral_fast_host_multi[_f64]): row strips of one image or
    images of a batch per device, one host worker thread per device; bit-identical to one device."""
    a = np.asarray(image)
    if a.size == 0:
        raise ValueError("bilateral_fast: empty image")
    batch = 1 if a.ndim == 2 else a.shape[0]
    h, w = a.shape[-2], a.shape[-1]
    g = whole_geometry(w, h, batch)
    f = _filter_struct(spatial, approx, check_epsilon)
    bad = ctypes.c_longlong(-1)
    devs = (ctypes.c_int * len(devices))(*devices)
    if a.dtype == np.float32:
        src = np.ascontiguousarray(a)
        out = np.empty_like(src)
        rc = lib.fbf_bilateral_fast_host_multi(ctypes.byref(g), ctypes.byref(f), src.ctypes.data_as(_F),
                                               out.ctypes.data_as(_F), _VARIANTS[variant], ctypes.byref(bad),
                                               devs, len(devices))
    else:
        src = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty_like(src)
        rc = lib.fbf_bilateral_fast_host_multi_f64(ctypes.byref(g), ctypes.byref(f), _dp(src), _dp(out),
                                                   _VARIANTS[variant], ctypes.byref(bad), devs, len(devices))
    _check(rc)
    return out


def bilateral_fast_device(src_ptr: int, dst_ptr: int, geometry: Geometry, spatial: SpatialKernel,
                          approx: FourierKernelApprox, workspace_ptr: int, workspace_bytes: int,
                          bad_ptr: int, stream: int = 0, variant: str = "fused",
                          check_epsilon: bool = True) -> None:
    """Asynchronous device-resident call (pointers from torch tensors, cudaStream_t as int)."""
    f = _filter_struct(spatial, approx, check_epsilon)
    _check(lib.fbf_bilateral_fast_device(ctypes.byref(geometry), ctypes.byref(f), src_ptr, dst_ptr,
                                         workspace_ptr, workspace_bytes, bad_ptr, _VARIANTS[variant], stream))


def prepare_device(src_ptr: int, geometry: Geometry, spatial: SpatialKernel, approx: FourierKernelApprox,
                   workspace_ptr: int, workspace_bytes: int, stream: int = 0, variant: str = "fused",
                   check_epsilon: bool = True) -> None:
    """Stage 1 of bilateral_fast_device: base phase + shifted intensity into the workspace."""
    f = _filter_struct(spatial, approx, check_epsilon)
    _check(lib.fbf_prepare_device(ctypes.byref(geometry), ctypes.byref(f), src_ptr, workspace_ptr,
                                  workspace_bytes, _VARIANTS[variant], stream))


def filter_prepared_device(dst_ptr: int, geometry: Geometry, spatial: SpatialKernel, approx: FourierKernelApprox,
                           workspace_ptr: int, workspace_bytes: int, bad_ptr: int, stream: int = 0,
                           variant: str = "fused", check_epsilon: bool = True) -> None:
    """Stage 2 of bilateral_fast_device: the filter proper (fused kernel or the naive chain)."""
    f = _filter_struct(spatial, approx, check_epsilon)
    _check(lib.fbf_filter_prepared_device(ctypes.byref(geometry), ctypes.byref(f), dst_ptr, workspace_ptr,
                                          workspace_bytes, bad_ptr, _VARIANTS[variant], stream))


def launches_per_call(geometry: Geometry, spatial: SpatialKernel, approx: FourierKernelApprox,
                      variant: str = "fused") -> int:
    f = _filter_struct(spatial, approx)
    return int(lib.fbf_launches_per_call(ctypes.byref(geometry), ctypes.byref(f), _VARIANTS[variant]))


def partial_sums_device(pq_ptr: int, geometry: Geometry, spatial: SpatialKernel, approx: FourierKernelApprox,
                        n_lo: int, n_hi: int, workspace_ptr: int, workspace_bytes: int, stream: int = 0,
                        variant: str = "fused", check_epsilon: bool = True) -> None:
    """(Q, P) partial sums over harmonics [n_lo, n_hi) into a dense fp64-pair device array (after
    prepare_device): exact multiples of the call's fixed-point grid, so partial planes of disjoint
    harmonic ranges sum exactly, in any order, to the single-call values."""
    f = _filter_struct(spatial, approx, check_epsilon)
    _check(lib.fbf_partial_sums_device(ctypes.byref(geometry), ctypes.byref(f), int(n_lo), int(n_hi), pq_ptr,
                                       workspace_ptr, workspace_bytes, _VARIANTS[variant], stream))


def finish_device(pq_ptr: int, dst_ptr: int, geometry: Geometry, spatial: SpatialKernel,
                  approx: FourierKernelApprox, bad_ptr: int, stream: int = 0, check_epsilon: bool = True) -> None:
    """Divide summed fp64 (Q, P) pairs into the output with the reference's denominator-collapse check."""
    f = _filter_struct(spatial, approx, check_epsilon)
    _check(lib.fbf_finish_device(ctypes.byref(geometry), ctypes.byref(f), pq_ptr, dst_ptr, bad_ptr, stream))


def workspace_bytes(geometry: Geometry, radius: int, variant: str = "fused") -> int:
    return int(lib.fbf_workspace_bytes(ctypes.byref(geometry), int(radius), _VARIANTS[variant]))


def bilateral_exact_gpu(image: np.ndarray, spatial: SpatialKernel, family: int, sigma_r: float,
                        row0: int = 0, rows: Optional[int] = None) -> np.ndarray:
    """bilateral.hpp:78-102 on the GPU (fp64 accumulation): output rows [row0, row0+rows)."""
    import torch
    img = np.ascontiguousarray(image, dtype=np.float32)
    h, w = img.shape
    rows = h - row0 if rows is None else rows
    from .shard import source_rows
    lo, hi = source_rows(row0, rows, h, spatial.radius)
    g = strip_geometry(w, h, row0, rows, spatial.radius)
    g.src_row0, g.src_rows = lo, hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    src = torch.from_numpy(img[lo:hi]).to(dev)
    dst = torch.empty((rows, w), dtype=torch.float64, device=dev)
    prof = np.ascontiguousarray(spatial.profile, dtype=np.float64)
    rc = lib.fbf_bilateral_exact_device(ctypes.byref(g), _dp(prof), spatial.radius, int(family), float(sigma_r),
                                        src.data_ptr(), dst.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _check(rc)
    return dst.cpu().numpy()


def convolve(plane: np.ndarray, spatial: SpatialKernel, backend: str = "direct") -> np.ndarray:
    """spatial.hpp:98-112 on the GPU; backend "recursive" runs the IIR Gaussian
    for Gaussian windows with sigma >= 2 and the direct path otherwise, like the reference."""
    p = np.ascontiguousarray(plane, dtype=np.float64)
    if p.size == 0:
        raise ValueError("convolve: empty plane")
    out = np.empty_like(p)
    if backend == "recursive" and spatial.kind == SPATIAL_GAUSSIAN and spatial.sigma_s >= 2.0:
        _check(lib.fbf_convolve_recursive_host_f64(p.shape[1], p.shape[0], spatial.sigma_s, _dp(p), _dp(out)))
        return out
    prof = np.ascontiguousarray(spatial.profile, dtype=np.float64)
    _check(lib.fbf_convolve_host_f64(p.shape[1], p.shape[0], _dp(prof), spatial.radius, _dp(p), _dp(out)))
    return out


def synth_image(seed: int, width: int, height: int, rects: int, noise_sigma: float,
                row0: int = 0, rows: Optional[int] = None, nthreads: int = 0) -> np.ndarray:
    """BASELINE.json's seeded synthetic image, rows [row0, row0+rows)."""
    rows = height - row0 if rows is None else rows
    out = np.empty((rows, width), dtype=np.float32)
    nt = nthreads or min(32, os.cpu_count() or 1)
    _check(lib.fbf_synth_image(int(seed), int(width), int(height), int(rects), float(noise_sigma),
                               int(row0), int(rows), out.ctypes.data_as(_F), nt))
    return out


def probe_fma_peak(stream: int = 0):
    ops, mhz = ctypes.c_double(), ctypes.c_double()
    _check(lib.fbf_probe_fma_peak(ctypes.byref(ops), ctypes.byref(mhz), stream))
    return ops.value, mhz.value


from . import configs  # noqa: E402,F401
