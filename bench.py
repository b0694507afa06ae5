#!/usr/bin/env python
"""bench.py -- Mpixel/s of the shiftable Fourier-kernel bilateral filter on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One step = one pass of the hot path (phase prep + fused filter kernel) over the
workload's synthetic input, inputs resident in HBM.  Default workload: BASELINE
config c2 (2048x2048 fp32, Gaussian sigma_s=5 / W=15, Gaussian sigma_r=20,
N=20), the config BASELINE.json's metric is quoted on that fits one GPU.  With
N GPUs (torchrun, one process per GPU) and the default `--scaling weak`, every
rank filters its own copy of the workload (the same shapes, its own seeds:
seed + 1000 * rank), so the work per GPU is fixed and there is no collective
on the data path.  `--scaling strong` instead splits the one workload: a single
image into N row strips, each carrying W halo rows, a batch (c5) by image.

Printed on rank 0: ONE JSON line (metric/value/unit/.../roofline/cpu_baseline/
e2e/gpu_launches/clocks).  `--impl reference` times the reference's own CPU
implementation (oracle/_ref/libfbf_ref.so, the unmodified reference headers
compiled in place) with all host threads on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="N>1: weak = one whole workload per rank (own seeds), strong = split one workload")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-once", action="store_true",
                   help="run exactly one prep+filter pass (for ncu) and exit")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.005):
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


def cpu_reference_rate(cfg, nthreads: int, rows: int | None = None):
    """Reference bilateral_fast (oracle/_ref) on `rows` rows of image 0, all host threads.

    Returns (Mpixel/s, seconds, sample description)."""
    from oracle.pyoracle import Reference
    from paper_1603_08081_b200.configs import T_FIXED, approx_of, image_of
    ref = Reference()
    a = approx_of(cfg)
    img = image_of(cfg, 0).astype(np.float64)
    kind = 1 if cfg.spatial == "box" else 0
    rows = cfg.height if rows is None else rows
    r0 = (cfg.height - rows) // 2
    t = time.perf_counter()
    _, rc, msg = ref.bilateral_fast(img, kind, float(cfg.sigma_s), a.d, T_FIXED, a.max_pointwise_error,
                                    cfg.check_epsilon, r0, r0 + rows, nthreads)
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
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json generator, include/fourierbf_b200.h fbf_synth_image)",
        "config": config_dict(cfg, world, args.scaling),
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": nthreads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, world, scaling="weak"):
    return {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "batch": cfg.batch,
            "spatial": cfg.spatial, "sigma_s": cfg.sigma_s, "W": cfg.radius,
            "range": "exponential" if cfg.range_family else "gaussian", "sigma_r": cfg.sigma_r, "N": cfg.N,
            "T": 255,
            "parallelism": (f"workload-per-rank-x{world}" if scaling == "weak" or world == 1 else
                            f"row-strips-x{world}" if cfg.batch == 1 else f"images-x{world}"),
            "l2": "flushed between steps (512 MiB write)"}


def main():
    args = parse()
    from paper_1603_08081_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    world, rank, local = dist_env()
    world = max(world, 1)

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)

    import torch
    import torch.distributed as dist
    import paper_1603_08081_b200 as fb
    from paper_1603_08081_b200.configs import approx_of, image_of, spatial_of
    from paper_1603_08081_b200.shard import geometry as shard_geometry
    from paper_1603_08081_b200.shard import plan

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    spatial, approx = spatial_of(cfg), approx_of(cfg)
    W = spatial.radius
    weak = args.scaling == "weak"
    # weak: this rank's own whole workload; strong: its share of the one workload
    part = plan(cfg.width, cfg.height, cfg.batch, W, 1 if weak else world, 0 if weak else rank)
    geo = shard_geometry(part, cfg.width, cfg.height)
    seed_off = 1000 * rank if weak else 0
    if cfg.batch > 1:
        host = np.stack([fb.synth_image(cfg.seeds[i] + seed_off, cfg.width, cfg.height, cfg.rects, cfg.noise)
                         for i in part.images])
    else:  # each rank generates only its own rows (with halo rows)
        host = fb.synth_image(cfg.seeds[0] + seed_off, cfg.width, cfg.height, cfg.rects, cfg.noise,
                              part.src_row0, part.src_rows)[None]
    nb = host.shape[0]
    src = torch.from_numpy(host).to(dev)
    dst = torch.empty((nb, geo.out_rows, cfg.width), dtype=torch.float32, device=dev)
    ws_bytes = fb.workspace_bytes(geo, W, args.variant)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        fb.prepare_device(src.data_ptr(), geo, spatial, approx, ws.data_ptr(), ws_bytes, sh, args.variant,
                          cfg.check_epsilon)

    def filt():
        fb.filter_prepared_device(dst.data_ptr(), geo, spatial, approx, ws.data_ptr(), ws_bytes,
                                  bad.data_ptr(), sh, args.variant, cfg.check_epsilon)

    if args.profile_once:
        step(); filt()
        torch.cuda.synchronize()
        return 0

    peak_ops, peak_mhz = fb.probe_fma_peak(sh)
    for _ in range(max(args.warmup, 3)):
        step(); filt()
    torch.cuda.synchronize()
    if int(bad.item()) != -1:
        raise RuntimeError(f"denominator collapsed at linear index {int(bad.item())}")

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()  # evict L2 (126 MB) between steps; outside the events
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            filt()
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = statistics.mean(ev[k][0].elapsed_time(ev[k][2]) for k in range(args.steps))
    fused_ms = statistics.mean(ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps))
    prep_ms = statistics.mean(ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps))

    # ---- end to end through the public host API (H2D from pinned memory + D2H each step)
    e2e = None
    if not args.no_e2e:
        pin_src = torch.from_numpy(host).pin_memory()
        pin_dst = torch.empty((nb, geo.out_rows, cfg.width), dtype=torch.float32).pin_memory()
        gh = fb.Geometry.from_buffer_copy(geo)
        gh.src_pitch = gh.dst_pitch = cfg.width
        gh.src_bstride = geo.src_rows * cfg.width
        gh.dst_bstride = geo.out_rows * cfg.width
        f = fb._filter_struct(spatial, approx, cfg.check_epsilon)
        import ctypes
        badh = ctypes.c_longlong(-1)
        pfs, pfd = ctypes.cast(pin_src.data_ptr(), fb._F), ctypes.cast(pin_dst.data_ptr(), fb._F)
        call = lambda: fb._check(fb.lib.fbf_bilateral_fast_host(ctypes.byref(gh), ctypes.byref(f), pfs, pfd,
                                                                fb._VARIANTS[args.variant], ctypes.byref(badh)))
        for _ in range(2):
            call()
        if world > 1:
            dist.barrier()
        e2e_times = []
        for _ in range(max(20, min(args.steps, 50))):  # host-timed calls: enough of them to average out jitter
            t = time.perf_counter()
            call()
            e2e_times.append(time.perf_counter() - t)
        e2e_s = statistics.mean(e2e_times)
        e2e = {"s": e2e_s, "h2d": int(host.nbytes), "d2h": int(pin_dst.numel() * 4),
               "median_s": statistics.median(e2e_times), "calls": len(e2e_times)}

    # ---- aggregate over ranks (max time, summed bytes)
    px_rank = nb * geo.out_rows * cfg.width
    vals = torch.tensor([step_ms, fused_ms, prep_ms, e2e["s"] if e2e else 0.0], dtype=torch.float64, device=dev)
    sums = torch.tensor([px_rank, e2e["h2d"] if e2e else 0, e2e["d2h"] if e2e else 0], dtype=torch.float64,
                        device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    step_ms, fused_ms, prep_ms, e2e_s = vals.tolist()
    total_px, h2d, d2h = sums.tolist()

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
                "kernel": "fbf::fused_kernel", "kernel_ms": fused_ms, "prep_ms": prep_ms,
                "ops_per_pixel": cfg.ops_per_pixel(),
                "peak_source": f"measured in this run: FFMA2 probe fbf_probe_fma_peak at {peak_mhz:.0f} MHz "
                               "(128 FP32 lanes x 148 SMs); ops = FP32 FMA-pipe lane ops (FFMA/FMUL/FADD = 1)",
                "hbm_bytes_per_pixel_algorithmic": 8,
            }
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (BASELINE.json generator, seeded; include/fourierbf_b200.h fbf_synth_image)",
            "config": config_dict(cfg, world, args.scaling),
            "variant": args.variant,
            "roofline": roof,
            "gpu_launches": args.steps * fb.launches_per_call(geo, spatial, approx, args.variant),
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = {"value": total_px / e2e_s / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": int(h2d),
                           "d2h_bytes_per_step": int(d2h),
                           "path": "fbf_bilateral_fast_host (C-ABI): pinned H2D + prep + filter + D2H + sync",
                           "statistic": f"mean of {e2e['calls']} host-timed calls (rank 0); median "
                                        f"{total_px / e2e['median_s'] / 1e6 if world == 1 else float('nan'):.1f}"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                rate, dt, sample = cpu_reference_rate(cfg, os.cpu_count() or 1,
                                                      None if cfg.pixels() <= 2048 * 2048 else 256)
                line["cpu_baseline"] = {"value": rate, "unit": "Mpixel/s", "cores": os.cpu_count(),
                                        "kind": "reference", "sample": sample, "seconds": dt}
            except Exception as exc:  # oracle/_ref not built on this box
                line["cpu_baseline"] = {"value": None, "unit": "Mpixel/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {exc}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
