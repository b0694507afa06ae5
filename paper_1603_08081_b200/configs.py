"""The five BASELINE.json configurations (SURVEY.md §8 shorthand c1..c5).

T = 255 everywhere (omega = pi/255); the fit is the fixed-order recursive-QR
least-squares fit on t in {0..255} (kernel_approx.hpp:51-149, pattern
tests/acceptance.cpp:247-263).  c3's fit error (0.0743) exceeds its centre
weight w0 = 1/121, so the reference's precondition (bilateral.hpp:114-118) is
bypassed for it (check_epsilon=False, precedent test_bilateral.cpp:120-129) and
the paper's bound is undefined there.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

T_FIXED = 255


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    batch: int
    seeds: List[int]
    rects: int
    noise: float
    spatial: str        # "gaussian" | "box"
    sigma_s: float      # gaussian sigma, or the box radius
    range_family: int   # 0 gaussian, 1 exponential
    sigma_r: float
    N: int

    @property
    def radius(self) -> int:
        import math
        return int(self.sigma_s) if self.spatial == "box" else int(math.ceil(3.0 * self.sigma_s))

    @property
    def check_epsilon(self) -> bool:
        return self.name != "c3"

    def pixels(self) -> int:
        return self.width * self.height * self.batch

    def ops_per_pixel(self) -> int:
        """Algorithmic FP32 FMA-pipe ops per output pixel.

        Gaussian: (4N+1)*2*(2W+1) + 12N + 2   (4 planes x 2 passes x (2W+1) MACs
                  per harmonic n>=1, 1 plane for n=0, 6 modulation + 6 demod ops)
        Box (running sums, 2 ops per pass): (4N+1)*4 + 12N + 2
        """
        N, W = self.N, self.radius
        if self.spatial == "box":
            return (4 * N + 1) * 4 + 12 * N + 2
        return (4 * N + 1) * 2 * (2 * W + 1) + 12 * N + 2


CONFIGS = {
    "c1": Config("c1", 512, 512, 1, [0], 6, 10.0, "gaussian", 3.0, 0, 30.0, 12),
    "c2": Config("c2", 2048, 2048, 1, [1], 24, 15.0, "gaussian", 5.0, 0, 20.0, 20),
    "c3": Config("c3", 1024, 1024, 1, [2], 12, 10.0, "box", 5, 1, 20.0, 30),
    "c4": Config("c4", 8192, 8192, 1, [3], 400, 10.0, "gaussian", 8.0, 0, 15.0, 32),
    "c5": Config("c5", 1024, 1024, 256, list(range(100, 356)), 16, 10.0, "gaussian", 4.0, 0, 25.0, 16),
}


def spatial_of(cfg: Config):
    from . import make_spatial_box, make_spatial_gaussian
    return make_spatial_box(int(cfg.sigma_s)) if cfg.spatial == "box" else make_spatial_gaussian(cfg.sigma_s)


def approx_of(cfg: Config):
    from . import fit_fixed
    return fit_fixed(cfg.range_family, cfg.sigma_r, T_FIXED, cfg.N)


def image_of(cfg: Config, index: int = 0, row0: int = 0, rows: int | None = None):
    from . import synth_image
    return synth_image(cfg.seeds[index], cfg.width, cfg.height, cfg.rects, cfg.noise, row0, rows)
