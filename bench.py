#!/usr/bin/env python
"""bench.py -- Mpixel/s of the shiftable Fourier-kernel bilateral filter on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One step = one pass of the hot path (phase prep + fused filter kernel) over the
workload's synthetic input, inputs resident in HBM.  Default workload: BASELINE
config c2 (2048x2048 fp32, Gaussian sigma_s=5 / W=15, Gaussian sigma_r=20,
N=20), the config BASELINE.json's metric is quoted on that fits one GPU.

N GPUs: one process per GPU.  Under torchrun (WORLD_SIZE set) the ranks are
the launcher's; `--gpus N` without WORLD_SIZE launches the N ranks itself
(127.0.0.1 rendezvous).  The headline line then runs STRONG scaling (the
default `--scaling auto`): the one c2 image is split into N row strips with W
halo rows each (mirror padding only at the global edges, 16-row aligned cuts,
bit-identical to one GPU), so N = 1 is the single-GPU line.  The same line
carries `sharded` records for c4 (8192^2 row strips with 24-row halos) and c5
(256 images split by image), each with its own 1-GPU time on rank 0 and the
speed-up.  `--scaling weak` instead gives every rank a whole copy of the
workload (its own seeds).  No collective is on the data path; NCCL carries the
barrier and the max-over-ranks timing.

Printed on rank 0: ONE JSON line (metric/value/unit/.../roofline/cpu_baseline/
e2e/e2e_f64/gpu_launches/clocks).  `--impl reference` times the reference's own
CPU implementation (oracle/_ref/libfbf_ref.so, the unmodified reference headers
compiled in place) with all host threads on the same workload, with inputs from
the standalone generator library and the reference's own fit (it never loads
the product library).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel/s of Fourier-kernel shiftable BF"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="c2")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--variant", default="fused", choices=["fused", "naive"])
    p.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                   help="N>1: strong (auto) = split the one workload, weak = one whole workload per rank")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sharded", action="store_true", help="N>1: skip the c4 / c5 sharded records")
    p.add_argument("--profile-once", action="store_true",
                   help="run exactly one prep+filter pass (for ncu) and exit")
    p.add_argument("--dry-run", action="store_true",
                   help="no GPU: plan the shards and exercise the launcher / rendezvous over gloo (CPU tests)")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` without a launcher: start the N ranks here (one process per GPU)."""
    port = str(free_port())
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.002):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_traffic(cfg_name: str, variant: str):
    """dram bytes per launch of the fused kernel from the committed ncu --set full summary (or None)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{variant}_{cfg_name}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def load_configs():
    """paper_1603_08081_b200/configs.py loaded by path: pure data, so the reference
    arm never imports the product package (whose import loads libfourierbf_b200.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("fbf_bench_configs",
                                                  os.path.join(ROOT, "paper_1603_08081_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


def loaded_native_libs():
    """In-tree shared objects mapped into this process (evidence of what each arm ran)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                parts = ln.split()
                p = parts[-1] if parts else ""
                if p.endswith(".so") and p.startswith(ROOT):
                    libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


# --------------------------------------------------------------- reference arm

def cpu_reference_rate(cfg, nthreads: int, rows: int | None = None, ref=None):
    """Reference bilateral_fast (oracle/_ref) on `rows` rows of image 0, all host threads.

    Everything on this leg comes from oracle/: the fit is the reference's own
    QrState fit (ref_fit_fixed), the image the standalone generator library
    (oracle/_synth, the product's generator source compiled on its own); the
    product library is never loaded.  Returns (Mpixel/s, seconds, sample)."""
    from oracle.pyoracle import Reference, synth_image
    ref = ref or Reference()
    T = load_configs().T_FIXED
    d, _, max_err = ref.fit_fixed(cfg.range_family, cfg.sigma_r, T, cfg.N)
    img = synth_image(cfg.seeds[0], cfg.width, cfg.height, cfg.rects, cfg.noise).astype(np.float64)
    kind = 1 if cfg.spatial == "box" else 0
    rows = cfg.height if rows is None else rows
    r0 = (cfg.height - rows) // 2
    t = time.perf_counter()
    _, rc, msg = ref.bilateral_fast(img, kind, float(cfg.sigma_s), d, T, max_err, cfg.check_epsilon,
                                    r0, r0 + rows, nthreads)
    dt = time.perf_counter() - t
    if rc:
        raise RuntimeError(msg)
    px = rows * cfg.width
    return px / dt / 1e6, dt, f"rows [{r0},{r0 + rows}) of image 0 ({px} px), {nthreads} threads, fp64"


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    nthreads = os.cpu_count() or 1
    # each step: a bounded sample of the workload (a centred row band) sized for ~1-4 s
    rows = cfg.height if cfg.pixels() // cfg.batch <= 2048 * 2048 else 512
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, nthreads, rows)
    times = []
    for _ in range(args.steps):
        _, dt, sample = cpu_reference_rate(cfg, nthreads, rows)
        times.append(dt)
    px = rows * cfg.width
    ms = 1e3 * statistics.mean(times)
    value = px / (ms / 1e3) / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling_of(args, world), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json generator, oracle/_synth/libfbf_synth.so = fbf_synth.cpp)",
        "config": config_dict(cfg, world, scaling_of(args, world)),
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": nthreads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs": loaded_native_libs(),
    }
    if any("libfourierbf_b200" in p for p in line["native_libs"]):
        raise RuntimeError("reference arm loaded the product library")
    print(json.dumps(line), flush=True)
    return 0


def scaling_of(args, world):
    if args.scaling != "auto":
        return args.scaling
    return "strong" if world > 1 else "weak"


def config_dict(cfg, world, scaling="weak"):
    return {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "batch": cfg.batch,
            "spatial": cfg.spatial, "sigma_s": cfg.sigma_s, "W": cfg.radius,
            "range": "exponential" if cfg.range_family else "gaussian", "sigma_r": cfg.sigma_r, "N": cfg.N,
            "T": 255,
            "parallelism": (f"workload-per-rank-x{world}" if scaling == "weak" or world == 1 else
                            f"row-strips-x{world}" if cfg.batch == 1 else f"images-x{world}"),
            "l2": "flushed between steps (512 MiB write)"}


# ------------------------------------------------------------------ B200 arm

class Workload:
    """One rank's share of a config on its GPU: device buffers + the two stages."""

    def __init__(self, fb, cfg, world, rank, dev, weak, variant, seed_off=0, need_host=True):
        import torch
        from paper_1603_08081_b200.configs import approx_of, spatial_of
        from paper_1603_08081_b200.shard import geometry as shard_geometry
        from paper_1603_08081_b200.shard import plan
        self.fb, self.cfg, self.variant = fb, cfg, variant
        self.spatial, self.approx = spatial_of(cfg), approx_of(cfg)
        W = self.spatial.radius
        self.part = plan(cfg.width, cfg.height, cfg.batch, W, 1 if weak else world, 0 if weak else rank)
        self.geo = shard_geometry(self.part, cfg.width, cfg.height)
        if cfg.batch > 1:
            host = np.stack([fb.synth_image(cfg.seeds[i] + seed_off, cfg.width, cfg.height, cfg.rects, cfg.noise)
                             for i in self.part.images])
        else:  # each rank generates only its own rows (with halo rows)
            host = fb.synth_image(cfg.seeds[0] + seed_off, cfg.width, cfg.height, cfg.rects, cfg.noise,
                                  self.part.src_row0, self.part.src_rows)[None]
        self.host = host if need_host else None
        self.nb = host.shape[0]
        self.px = self.nb * self.geo.out_rows * cfg.width
        self.src = torch.from_numpy(host).to(dev)
        self.dst = torch.empty((self.nb, self.geo.out_rows, cfg.width), dtype=torch.float32, device=dev)
        self.ws_bytes = fb.workspace_bytes(self.geo, W, variant)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.bad = torch.full((1,), -1, dtype=torch.int64, device=dev)

    def prep(self, sh):
        self.fb.prepare_device(self.src.data_ptr(), self.geo, self.spatial, self.approx, self.ws.data_ptr(),
                               self.ws_bytes, sh, self.variant, self.cfg.check_epsilon)

    def filt(self, sh):
        self.fb.filter_prepared_device(self.dst.data_ptr(), self.geo, self.spatial, self.approx, self.ws.data_ptr(),
                                       self.ws_bytes, self.bad.data_ptr(), sh, self.variant, self.cfg.check_epsilon)

    def launches(self):
        return self.fb.launches_per_call(self.geo, self.spatial, self.approx, self.variant)

    def check(self):
        if int(self.bad.item()) != -1:
            raise RuntimeError(f"denominator collapsed at linear index {int(self.bad.item())}")


def time_steps(wl, stream, steps, warmup, flush, world, dist, clocks=None):
    """Device time of `steps` prep+filter passes (CUDA events on the launching stream, L2 flushed before
    each step, outside the events); barrier + synchronize on both sides.  Returns (step, fused, prep) ms."""
    import torch
    sh = stream.cuda_stream
    for _ in range(max(warmup, 3)):
        wl.prep(sh)
        wl.filt(sh)
    torch.cuda.synchronize()
    wl.check()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        for k in range(steps):
            flush.zero_()  # evict L2 (126 MB) between steps; outside the events
            ev[k][0].record(stream)
            wl.prep(sh)
            ev[k][1].record(stream)
            wl.filt(sh)
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = statistics.mean(ev[k][0].elapsed_time(ev[k][2]) for k in range(steps))
    fused_ms = statistics.mean(ev[k][1].elapsed_time(ev[k][2]) for k in range(steps))
    prep_ms = statistics.mean(ev[k][0].elapsed_time(ev[k][1]) for k in range(steps))
    return step_ms, fused_ms, prep_ms


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def host_e2e(fb, wl, world, dist, calls, f64=False):
    """The public host entry (fbf_bilateral_fast_host / _f64 through the C-ABI), host buffers in and out,
    copies inside the timed region.  fp32: pinned buffers; fp64: plain (pageable) numpy doubles, the
    reference Image's storage.  Returns mean seconds per call and the bytes crossing PCIe."""
    import ctypes
    import torch
    cfg = wl.cfg
    gh = fb.Geometry.from_buffer_copy(wl.geo)
    gh.src_pitch = gh.dst_pitch = cfg.width
    gh.src_bstride = wl.geo.src_rows * cfg.width
    gh.dst_bstride = wl.geo.out_rows * cfg.width
    f = fb._filter_struct(wl.spatial, wl.approx, cfg.check_epsilon)
    badh = ctypes.c_longlong(-1)
    if f64:
        src = wl.host.astype(np.float64)
        dst = np.empty((wl.nb, wl.geo.out_rows, cfg.width), dtype=np.float64)
        ps, pd = src.ctypes.data_as(fb._D), dst.ctypes.data_as(fb._D)
        fn = fb.lib.fbf_bilateral_fast_host_f64
        h2d, d2h = src.size * 4, dst.size * 4  # converted to fp32 on the host before the copy
    else:
        src = torch.from_numpy(wl.host).pin_memory()
        dst = torch.empty((wl.nb, wl.geo.out_rows, cfg.width), dtype=torch.float32).pin_memory()
        ps, pd = ctypes.cast(src.data_ptr(), fb._F), ctypes.cast(dst.data_ptr(), fb._F)
        fn = fb.lib.fbf_bilateral_fast_host
        h2d, d2h = int(wl.host.nbytes), int(dst.numel() * 4)
    call = lambda: fb._check(fn(ctypes.byref(gh), ctypes.byref(f), ps, pd, fb._VARIANTS[wl.variant],  # noqa: E731
                                ctypes.byref(badh)))
    for _ in range(2):
        call()
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(calls):
        t = time.perf_counter()
        call()
        times.append(time.perf_counter() - t)
    return statistics.mean(times), statistics.median(times), h2d, d2h


def sharded_record(fb, cfg, world, rank, dev, stream, args, dist, flush):
    """A config split over the ranks (c4: row strips with W halo rows; c5: images), the max-over-ranks time,
    and the same config on rank 0 alone: the 1-GPU time and the speed-up."""
    import torch
    wl = Workload(fb, cfg, world, rank, dev, False, args.variant, need_host=False)
    steps = max(3, min(args.steps, 10))
    step_ms, fused_ms, _ = time_steps(wl, stream, steps, args.warmup, flush, world, dist)
    px = wl.px
    del wl
    torch.cuda.empty_cache()
    vals = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    sums = torch.tensor([px], dtype=torch.float64, device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    one = torch.zeros(1, dtype=torch.float64, device=dev)
    if rank == 0:  # the same workload on one GPU
        wl1 = Workload(fb, cfg, 1, 0, dev, True, args.variant, need_host=False)
        one[0] = time_steps(wl1, stream, steps, args.warmup, flush, 1, dist)[0]
        del wl1
        torch.cuda.empty_cache()
    dist.barrier()
    n_ms = float(vals[0])
    total_px = float(sums[0])
    return {"workload": cfg.name, "parallelism": ("row-strips" if cfg.batch == 1 else "images") + f"-x{world}",
            "ms_per_step": n_ms, "value": total_px / (n_ms / 1e3) / 1e6, "unit": "Mpixel/s",
            "ms_per_step_1gpu": float(one[0]), "speedup": float(one[0]) / n_ms if rank == 0 else None,
            "steps": steps}


def dry_run(args, cfg, world, rank):
    """No GPU: the launcher, the rendezvous and the shard plan over gloo (tests/test_bench_launcher.py)."""
    import torch
    import torch.distributed as dist
    mod = load_configs()
    W = mod.CONFIGS[args.config].radius
    sys.path.insert(0, os.path.join(ROOT, "paper_1603_08081_b200"))
    import importlib.util
    spec = importlib.util.spec_from_file_location("fbf_bench_shard", os.path.join(ROOT, "paper_1603_08081_b200",
                                                                                 "shard.py"))
    shard = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = shard
    spec.loader.exec_module(shard)
    if world > 1:
        dist.init_process_group("gloo")
    scaling = scaling_of(args, world)
    part = shard.plan(cfg.width, cfg.height, cfg.batch, W, 1 if scaling == "weak" else world,
                      0 if scaling == "weak" else rank)
    px = torch.tensor([float(len(part.images) * part.out_rows * cfg.width)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(px)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "scaling": scaling,
                          "config": config_dict(cfg, world, scaling), "pixels": float(px[0])}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    cfg = load_configs().CONFIGS[args.config]
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    world = max(world, 1)

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if args.dry_run:
        return dry_run(args, cfg, world, rank)

    import torch
    import torch.distributed as dist
    import paper_1603_08081_b200 as fb

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the init log shows the rank count and transports
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    scaling = scaling_of(args, world)
    weak = scaling == "weak"

    wl = Workload(fb, cfg, world, rank, dev, weak, args.variant, seed_off=1000 * rank if weak else 0)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    if args.profile_once:
        wl.prep(sh)
        wl.filt(sh)
        torch.cuda.synchronize()
        return 0

    peak_ops, peak_mhz = fb.probe_fma_peak(sh)
    with ClockSampler(local) as clk:
        step_ms, fused_ms, prep_ms = time_steps(wl, stream, args.steps, args.warmup, flush, world, dist)
    launches = wl.launches()

    # ---- end to end through the public host API (H2D + D2H inside the timed region each call)
    e2e = e2e64 = None
    if not args.no_e2e:
        calls = max(20, min(args.steps, 50))  # host-timed calls: enough of them to average out jitter
        e2e = host_e2e(fb, wl, world, dist, calls)
        e2e64 = host_e2e(fb, wl, world, dist, max(10, calls // 2), f64=True)

    # ---- aggregate over ranks (max time, summed bytes)
    vals = torch.tensor([step_ms, fused_ms, prep_ms, e2e[0] if e2e else 0.0, e2e64[0] if e2e64 else 0.0],
                        dtype=torch.float64, device=dev)
    sums = torch.tensor([wl.px, e2e[2] if e2e else 0, e2e[3] if e2e else 0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    step_ms, fused_ms, prep_ms, e2e_s, e2e64_s = vals.tolist()
    total_px, h2d, d2h = sums.tolist()
    px_rank = wl.px
    host_img = wl.host
    del wl

    sharded = None
    if world > 1 and not weak and not args.no_sharded:
        CONFIGS = load_configs().CONFIGS
        sharded = {name: sharded_record(fb, CONFIGS[name], world, rank, dev, stream, args, dist, flush)
                   for name in ("c4", "c5") if name != cfg.name}

    if rank == 0:
        value = total_px / (step_ms / 1e3) / 1e6
        ops = cfg.ops_per_pixel() * px_rank
        achieved = ops / (fused_ms / 1e3) / 1e12
        peak = peak_ops / 1e12
        if args.variant == "naive":  # the HBM-resident chain: bound by HBM traffic, not the FMA pipe
            # per harmonic: modulate writes M (16 B/px); row FIR reads M, writes T; column FIR reads T,
            # writes C; demod reads M, C and (Q, P), writes (Q, P): 128 B/px; prep 12 B, divide 12 B
            nbytes = ((cfg.N + 1) * 128 + 24) * px_rank
            hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            gbs = nbytes / (fused_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                    "traffic": load_traffic(cfg.name, args.variant), "kernel": "naive chain", "kernel_ms": fused_ms,
                    "prep_ms": prep_ms, "hbm_bytes_per_pixel_algorithmic": (cfg.N + 1) * 128 + 24,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth, burst)"}
        else:
            roof = {
                "bound": "fp32_fma", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                "frac": achieved / peak, "traffic": load_traffic(cfg.name, args.variant),
                "kernel": "fbf::n0_plane_kernel + fbf::fused_kernel (+ finish_groups)", "kernel_ms": fused_ms, "prep_ms": prep_ms,
                "ops_per_pixel": cfg.ops_per_pixel(),
                "peak_source": f"measured in this run: FFMA2 probe fbf_probe_fma_peak at {peak_mhz:.0f} MHz "
                               "(128 FP32 lanes x 148 SMs); ops = FP32 FMA-pipe lane ops (FFMA/FMUL/FADD = 1)",
                "hbm_bytes_per_pixel_algorithmic": 8,
            }
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (BASELINE.json generator, seeded; include/fourierbf_b200.h fbf_synth_image)",
            "config": config_dict(cfg, world, scaling),
            "variant": args.variant,
            "roofline": roof,
            "gpu_launches": args.steps * launches,
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = {"value": total_px / e2e_s / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": int(h2d),
                           "d2h_bytes_per_step": int(d2h),
                           "path": "fbf_bilateral_fast_host (C-ABI): pinned fp32 H2D + prep + filter + D2H + sync",
                           "statistic": f"mean of {max(20, min(args.steps, 50))} host-timed calls, max over ranks"}
            line["e2e_f64"] = {"value": total_px / e2e64_s / 1e6, "unit": "Mpixel/s",
                               "ratio_to_e2e": e2e_s / e2e64_s,
                               "path": "fbf_bilateral_fast_host_f64 (what bilateral_fast(const Image&) calls): "
                                       "pageable fp64 host buffers, pooled host conversion + the same pipeline"}
        if sharded:
            line["sharded"] = sharded
        if world == 1 and not args.no_cpu_baseline:
            try:
                rate, dt, sample = cpu_reference_rate(cfg, os.cpu_count() or 1,
                                                      None if cfg.pixels() <= 2048 * 2048 else 256)
                line["cpu_baseline"] = {"value": rate, "unit": "Mpixel/s", "cores": os.cpu_count(),
                                        "kind": "reference", "sample": sample, "seconds": dt}
            except Exception as exc:  # oracle/_ref not built on this box
                line["cpu_baseline"] = {"value": None, "unit": "Mpixel/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {exc}"}
        line["native_libs"] = loaded_native_libs()
        print(json.dumps(line), flush=True)
    del host_img
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
