"""Seeded synthetic blind-pansharpening scenes (BASELINE.json ``configs``).

The paper's datasets (Pavia, Cambria Fire, ...) are not available, so these seeded scenes
stand in for them, with the shapes, kernel supports and noise levels BASELINE.json names:

* PAN: 1/f^2 Gaussian random field (white noise shaped by 1/|f| amplitude, DC removed)
  plus 20 constant-intensity convex polygons, min-max normalised to [0, 1].
* HRMS_c = a_c(x) * PAN + b_c(x) + N(0, 0.01^2), a_c a smooth field in [0.5, 1.5],
  b_c a smooth field in [-0.1, 0.1].
* Blur: anisotropic Gaussian on an S x S support (sigma_x, sigma_y ~ U[1, 2.5], rotation
  theta ~ U[0, pi), sub-pixel centre shift ~ U[-m, m]), unit sum.
* LRMS = downsample_r(circular_convolve(HRMS, k)) + N(0, sigma^2), with the reference's
  centre-at-origin circular convention (reference ``proj/src/ops.cpp:9-22``).

PAN and LRMS are quantised to float32 so every consumer (the CPU oracle, the GPU path,
the reference-facing C++ API) reads identical values; they are returned as float64 arrays
holding float32-representable numbers.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 210309943


@dataclass(frozen=True)
class SceneConfig:
    """One BASELINE.json configuration (C1..C5)."""

    name: str
    hr: int            # PAN side H = W
    bands: int         # N
    ratio: int         # r = c (decimation factor)
    support: int       # blur support S (also the estimated kernel side n)
    shift: float       # max |sub-pixel shift| m in px
    scenes: int = 1
    per_band_noise: bool = False
    index: int = 1     # config index used in the seed

    @property
    def lr(self) -> int:
        return self.hr // self.ratio


CONFIGS = {
    "C1": SceneConfig("C1", 256, 4, 4, 15, 2.0, index=1),
    "C2": SceneConfig("C2", 1024, 4, 4, 17, 3.0, index=2),
    "C3": SceneConfig("C3", 2048, 8, 4, 15, 2.0, per_band_noise=True, index=3),
    "C4": SceneConfig("C4", 512, 4, 4, 15, 2.0, scenes=64, index=4),
    "C5": SceneConfig("C5", 8192, 8, 4, 21, 2.0, index=5),
}


@dataclass
class Scene:
    pan: np.ndarray          # (H, W) float64 holding float32 values
    lrms: np.ndarray         # (N, h, w) float64 holding float32 values
    hrms: np.ndarray         # (N, H, W) ground truth (float64)
    kernel: np.ndarray       # (S, S) true blur (float64, unit sum)
    seed: int
    meta: dict = field(default_factory=dict)


def _power_field(rng: np.random.Generator, h: int, w: int, amp) -> np.ndarray:
    noise = rng.standard_normal((h, w))
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.fftfreq(w)[None, :]
    f = np.sqrt(fy * fy + fx * fx)
    a = amp(f)
    a[0, 0] = 0.0
    return np.real(np.fft.ifft2(np.fft.fft2(noise) * a))


def _rescale(x: np.ndarray, lo: float, hi: float) -> np.ndarray:
    mn, mx = float(x.min()), float(x.max())
    if mx <= mn:
        return np.full_like(x, 0.5 * (lo + hi))
    return lo + (hi - lo) * (x - mn) / (mx - mn)


def _smooth_field(rng: np.random.Generator, h: int, w: int, lo: float, hi: float) -> np.ndarray:
    f0 = 4.0 / max(h, w)  # a few cycles across the scene
    return _rescale(_power_field(rng, h, w, lambda f: np.exp(-(f / f0) ** 2)), lo, hi)


def _polygons(rng: np.random.Generator, img: np.ndarray, count: int = 20) -> None:
    h, w = img.shape
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    for _ in range(count):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        rad = rng.uniform(0.03, 0.15) * min(h, w)
        nv = int(rng.integers(3, 9))
        ang = np.sort(rng.uniform(0, 2 * np.pi, nv))
        rr = rad * rng.uniform(0.5, 1.0, nv)
        vy, vx = cy + rr * np.sin(ang), cx + rr * np.cos(ang)
        val = rng.uniform(0.0, 1.0)
        y0, y1 = int(max(0, np.floor(vy.min()))), int(min(h, np.ceil(vy.max()) + 1))
        x0, x1 = int(max(0, np.floor(vx.min()))), int(min(w, np.ceil(vx.max()) + 1))
        if y1 <= y0 or x1 <= x0:
            continue
        py, px = yy[y0:y1, x0:x1], xx[y0:y1, x0:x1]
        inside = np.ones(py.shape, dtype=bool)
        for i in range(nv):  # convex, counter-clockwise in (x, y) with y down: same-sign test
            j = (i + 1) % nv
            cross = (vx[j] - vx[i]) * (py - vy[i]) - (vy[j] - vy[i]) * (px - vx[i])
            inside &= cross >= 0
        img[y0:y1, x0:x1][inside] = val


def make_pan(rng: np.random.Generator, h: int, w: int) -> np.ndarray:
    field_ = _rescale(_power_field(rng, h, w, lambda f: 1.0 / np.maximum(f, 1e-12)), 0.0, 1.0)
    _polygons(rng, field_, 20)
    return _rescale(field_, 0.0, 1.0)


def make_kernel(rng: np.random.Generator, support: int, max_shift: float) -> np.ndarray:
    sx, sy = rng.uniform(1.0, 2.5, 2)
    th = rng.uniform(0.0, np.pi)
    cx, cy = rng.uniform(-max_shift, max_shift, 2)
    c = (support - 1) / 2
    y, x = np.mgrid[0:support, 0:support].astype(np.float64)
    dx, dy = x - c - cx, y - c - cy
    u = np.cos(th) * dx + np.sin(th) * dy
    v = -np.sin(th) * dx + np.cos(th) * dy
    k = np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))
    return k / k.sum()


def embed_kernel(k: np.ndarray, h: int, w: int) -> np.ndarray:
    """Centre tap at the origin, other taps wrapped (reference ``ops.cpp:9-22``)."""
    n = k.shape[0]
    c = (n - 1) // 2
    out = np.zeros((h, w))
    for r in range(n):
        for q in range(n):
            out[(r - c) % h, (q - c) % w] += k[r, q]
    return out


def circular_convolve(img: np.ndarray, k: np.ndarray) -> np.ndarray:
    kh = np.fft.fft2(embed_kernel(k, *img.shape[-2:]))
    return np.real(np.fft.ifft2(np.fft.fft2(img) * kh))


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def scene_seed(cfg: SceneConfig, scene_index: int = 0) -> int:
    return SEED_BASE + 1000 * cfg.index + scene_index


def make_scene(cfg: SceneConfig | str, scene_index: int = 0, *, hr: int | None = None) -> Scene:
    """Build scene ``scene_index`` of ``cfg`` (``hr`` overrides the side for small tests)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    H = W = hr or cfg.hr
    r = cfg.ratio
    seed = scene_seed(cfg, scene_index)
    rng = np.random.default_rng(seed)
    pan = make_pan(rng, H, W).astype(np.float32).astype(np.float64)
    k = make_kernel(rng, cfg.support, cfg.shift)
    kh = np.fft.fft2(embed_kernel(k, H, W))
    hrms = np.empty((cfg.bands, H, W))
    lrms = np.empty((cfg.bands, H // r, W // r))
    sig = []
    for b in range(cfg.bands):
        brng = np.random.default_rng(_splitmix64(seed * 64 + b))
        a = _smooth_field(brng, H, W, 0.5, 1.5)
        off = _smooth_field(brng, H, W, -0.1, 0.1)
        hrms[b] = a * pan + off + brng.normal(0.0, 0.01, (H, W))
        sigma = brng.uniform(0.003, 0.01) if cfg.per_band_noise else 0.005
        sig.append(sigma)
        blurred = np.real(np.fft.ifft2(np.fft.fft2(hrms[b]) * kh))
        lrms[b] = blurred[::r, ::r] + brng.normal(0.0, sigma, (H // r, W // r))
    lrms = lrms.astype(np.float32).astype(np.float64)
    return Scene(pan=pan, lrms=lrms, hrms=hrms, kernel=k, seed=seed,
                 meta={"config": cfg.name, "H": H, "W": W, "bands": cfg.bands, "ratio": r,
                       "support": cfg.support, "noise_sigma": sig})
