"""Seeded synthetic input fields shaped like the paper's workloads.

This module is shared by the tests, ``bench.py`` and ``__graft_entry__``.  It
holds none of LOPC's arithmetic: it only draws random fields with the
structure of the inputs the paper evaluates on (Table II, §V,
P:364-383) and of the five configs in BASELINE.json.  Recipes (also in
DESIGN.md §"Input recipe"):

  cfg1  2D f32 64x64    12 Gaussians, clipped at the 10th/90th percentile
                         (plateaus = exact ties), snapped to a grid of eps/16
                         (near-ties), NOA 1e-2.               seed 1
  cfg2  3D f32 100x500x500 Isabel-like vortex:
                         -exp(-(r/0.12)^2)(1 - z/(2 nz)) + 0.2 z/nz
                         + 0.02 GRF(P~k^-3), NOA 1e-3.        seed 2
  cfg3  3D f32 512^3    NYX-like log-normal exp(1.5 g), g = unit GRF with
                         P~k^-2, NOA 1e-4.                    seed 3
  cfg4  2D f32 1800x3600 CESM-ATM-like 288 - 40 sin^2(lat)
                         + 5 cos(3 lon) cos(lat) + 2 GRF(k^-3), rounded to
                         0.01 (many exact ties), NOA 1e-3.    seed 4
  cfg5  3D f64 2048^3   turbulence (Kolmogorov, generated on the GPU, not
                         here).

The GRF is white noise filtered in Fourier space by k^(-a/2) and normalised
to zero mean / unit variance.  ``eps_noa`` is the caller-side step a0 of
SURVEY §8(a): R = max - min in double, eps = rel * R rounded to nearest.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


def _grf(shape, alpha: float, rng: np.random.Generator) -> np.ndarray:
    noise = rng.standard_normal(shape, dtype=np.float32)
    spec = np.fft.rfftn(noise)
    del noise
    k2 = None
    for ax, n in enumerate(shape):
        f = np.fft.rfftfreq(n) if ax == len(shape) - 1 else np.fft.fftfreq(n)
        f = f.astype(np.float32) ** 2
        sh = [1] * len(shape)
        sh[ax] = f.shape[0]
        f = f.reshape(sh)
        k2 = f if k2 is None else k2 + f
    with np.errstate(divide="ignore"):
        amp = np.where(k2 > 0, k2 ** np.float32(-alpha / 4.0), np.float32(0))
    del k2
    spec *= amp
    del amp
    g = np.fft.irfftn(spec, s=shape, axes=list(range(len(shape)))).astype(np.float32)
    del spec
    g -= g.mean(dtype=np.float64)
    sd = g.std(dtype=np.float64)
    if sd > 0:
        g /= np.float32(sd)
    return g


def eps_noa(x: np.ndarray, rel: float) -> float:
    """Step a0: eps = rel * (max - min), in double."""
    xf = x[np.isfinite(x)]
    if xf.size == 0:
        return float(rel)
    r = float(np.float64(xf.max()) - np.float64(xf.min()))
    return float(np.float64(rel) * np.float64(r)) if r > 0 else float(rel)


def gaussians2d(ny: int = 64, nx: int = 64, seed: int = 1, rel: float = 1e-2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    f = np.zeros((ny, nx))
    for _ in range(12):
        cy, cx = rng.uniform(0, ny), rng.uniform(0, nx)
        sg = rng.uniform(3, 12)
        a = rng.uniform(-1, 1)
        f += a * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sg * sg))
    lo, hi = np.percentile(f, [10, 90])
    f = np.clip(f, lo, hi)
    eps = rel * (f.max() - f.min())
    q = eps / 16.0
    f = np.round(f / q) * q
    return f.astype(np.float32)


def isabel3d(nz: int = 100, ny: int = 500, nx: int = 500, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = (np.arange(nz, dtype=np.float32) / nz).reshape(nz, 1, 1)
    y = (np.arange(ny, dtype=np.float32) / ny - 0.5).reshape(1, ny, 1)
    x = (np.arange(nx, dtype=np.float32) / nx - 0.5).reshape(1, 1, nx)
    r2 = y * y + x * x
    f = _grf((nz, ny, nx), 3.0, rng)
    f *= np.float32(0.02)
    f += -np.exp(-r2 / np.float32(0.12 ** 2)) * (1 - z / 2) + np.float32(0.2) * z
    return f.astype(np.float32)


def nyx3d(n0: int = 512, n1: int = 512, n2: int = 512, seed: int = 3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    g = _grf((n0, n1, n2), 2.0, rng)
    g *= np.float32(1.5)
    np.exp(g, out=g)
    return g


def cesm2d(ny: int = 1800, nx: int = 3600, seed: int = 4) -> np.ndarray:
    rng = np.random.default_rng(seed)
    lat = np.linspace(-np.pi / 2, np.pi / 2, ny, dtype=np.float64).reshape(ny, 1)
    lon = np.linspace(0, 2 * np.pi, nx, endpoint=False, dtype=np.float64).reshape(1, nx)
    f = 288.0 - 40.0 * np.sin(lat) ** 2 + 5.0 * np.cos(3 * lon) * np.cos(lat)
    f = f + 2.0 * _grf((ny, nx), 3.0, rng).astype(np.float64)
    f = np.round(f * 100.0) / 100.0
    return f.astype(np.float32)


@dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    dtype: str
    rel: float
    seed: int

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def raw_bytes(self) -> int:
        return self.n * (4 if self.dtype == "f32" else 8)

    def generate(self, dims=None) -> np.ndarray:
        d = tuple(dims) if dims is not None else self.dims
        if self.name == "cfg1":
            return gaussians2d(*d, seed=self.seed, rel=self.rel)
        if self.name == "cfg2":
            return isabel3d(*d, seed=self.seed)
        if self.name == "cfg3":
            return nyx3d(*d, seed=self.seed)
        if self.name == "cfg4":
            return cesm2d(*d, seed=self.seed)
        raise ValueError(f"{self.name} is generated on the GPU (see DESIGN.md)")


CONFIGS = {
    "cfg1": Config("cfg1", (64, 64), "f32", 1e-2, 1),
    "cfg2": Config("cfg2", (100, 500, 500), "f32", 1e-3, 2),
    "cfg3": Config("cfg3", (512, 512, 512), "f32", 1e-4, 3),
    "cfg4": Config("cfg4", (1800, 3600), "f32", 1e-3, 4),
    "cfg5": Config("cfg5", (2048, 2048, 2048), "f64", 1e-5, 5),
}


def random_field(dims, dtype="f32", kind="noise", seed=0) -> np.ndarray:
    """Small fuzz fields for property tests: noise, smooth, plateau/tie-heavy,
    decreasing ramps, and the eps/16 tie grid."""
    rng = np.random.default_rng(seed)
    dt = np.float32 if dtype == "f32" else np.float64
    dims = tuple(int(d) for d in dims)
    if kind == "noise":
        f = rng.standard_normal(dims)
    elif kind == "smooth":
        f = _grf(dims, 3.0, rng).astype(np.float64) if min(dims) > 1 else rng.standard_normal(dims)
    elif kind == "ties":
        f = rng.integers(0, 4, size=dims).astype(np.float64) * 0.25
    elif kind == "plateau":
        f = np.clip(rng.standard_normal(dims), -0.3, 0.3)
    elif kind == "ramp_down":
        f = -np.arange(int(np.prod(dims)), dtype=np.float64).reshape(dims) * 1e-3
    elif kind == "grid16":
        f = np.round(rng.standard_normal(dims) * 16.0) / 16.0
    elif kind == "signed_zero_subnormal":
        # bin 0 crowded with -0.0 beside +0.0 (equal values: ties by index,
        # G13), subnormals of both signs and tiny normals, inside a smooth
        # field of range ~1 (so NOA eps stays a normal number)
        f = _grf(dims, 3.0, rng).astype(np.float64) if min(dims) > 1 else rng.standard_normal(dims)
        f = (f / max(1e-30, float(np.abs(f).max()))).astype(dt)
        u = np.dtype(dt).itemsize * 8
        ut = np.uint32 if u == 32 else np.uint64
        mant = (1 << (23 if u == 32 else 52)) - 1
        sub = (rng.integers(1, mant, size=dims, dtype=np.uint64).astype(ut)).view(dt)  # positive subnormals
        tiny = np.finfo(dt).tiny
        pick = rng.integers(0, 8, size=dims)
        sign = np.where(rng.random(dims) < 0.5, -1.0, 1.0).astype(dt)
        choice = [np.zeros(dims, dt), -np.zeros(dims, dt), sub, -sub,
                  np.full(dims, np.finfo(dt).smallest_subnormal, dt) * sign, np.full(dims, tiny, dt) * sign,
                  sub * sign, f]
        g = np.choose(pick, choice)
        mask = rng.random(dims) < 0.6
        f = np.where(mask, g, f)
        return np.ascontiguousarray(f.astype(dt))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(f.astype(dt))


def sha256(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).view(np.uint8)).hexdigest()
