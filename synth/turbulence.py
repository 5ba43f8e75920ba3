"""cfg5 input: a seeded Kolmogorov-like turbulence scalar, generated pointwise
from global grid coordinates.

This module holds none of LOPC's arithmetic; it only draws the synthetic
input.  The field is a random-Fourier-mode sum

    f(z, y, x) = sum_m a_m sin(kz_m z + ky_m y + kx_m x + phi_m)

over M = 256 modes with log-spaced wavenumbers |k_m| in [2 pi / 2048, pi / 2],
directions uniform on the sphere and phases uniform in [0, 2 pi), drawn from a
Philox generator keyed by the seed.  With log spacing, a_m^2 ~ E(k) k dlnk and
E(k) ~ k^(-5/3) (P(k) ~ k^(-11/3), Kolmogorov), so a_m ~ k_m^(-1/3); the
amplitudes are scaled to unit variance.

Because the sum is pointwise in global coordinates, any z-range of the field
can be built on its own, so a slab is the same bytes whoever generates it
(the bench's weak-scaling field for N ranks is 2048 x 2048 x (256 N); at N = 8
it is cfg5).  sin(A + B) = sin A cos B + cos A sin B splits every mode into an
x factor Q[., x] and a (z, y) factor P[(z, y), .], so a block of planes is one
(planes * ny) x 2M x nx matrix product — on the GPU a cuBLAS DGEMM (input
generation is plumbing, not the product).  Blocks are always 16 planes with
the same shapes, so the product runs the same kernel for every block.
"""
from __future__ import annotations

import math

import numpy as np

N_MODES = 256
BLOCK = 16


def modes(seed: int = 5, n_modes: int = N_MODES, L: int = 2048):
    """(k[M, 3] as (kz, ky, kx), phase[M], amp[M]) — host float64."""
    rng = np.random.Generator(np.random.Philox(seed))
    kmin, kmax = 2.0 * math.pi / L, 0.5 * math.pi
    kmag = np.exp(np.linspace(math.log(kmin), math.log(kmax), n_modes))
    dlnk = math.log(kmax / kmin) / (n_modes - 1)
    amp = kmag ** (-1.0 / 3.0) * math.sqrt(dlnk)
    amp /= math.sqrt(0.5 * float(np.sum(amp * amp)))  # unit variance
    d = rng.standard_normal((n_modes, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    phase = rng.uniform(0.0, 2.0 * math.pi, n_modes)
    return kmag[:, None] * d, phase, amp


def planes_torch(z0: int, z1: int, ny: int, nx: int, device="cuda", seed: int = 5, out=None):
    """Planes [z0, z1) of the field as a float64 torch tensor (z1-z0, ny, nx),
    built in blocks of BLOCK planes (the last block may be shorter)."""
    import torch

    k, ph, a = modes(seed)
    kz = torch.tensor(k[:, 0], dtype=torch.float64, device=device)
    ky = torch.tensor(k[:, 1], dtype=torch.float64, device=device)
    kx = torch.tensor(k[:, 2], dtype=torch.float64, device=device)
    pht = torch.tensor(ph, dtype=torch.float64, device=device)
    at = torch.tensor(a, dtype=torch.float64, device=device)
    xs = torch.arange(nx, dtype=torch.float64, device=device)
    A = kx[:, None] * xs[None, :] + pht[:, None]
    Q = torch.cat([torch.sin(A), torch.cos(A)], 0)  # (2M, nx)
    del A
    if out is None:
        out = torch.empty((z1 - z0, ny, nx), dtype=torch.float64, device=device)
    ys = torch.arange(ny, dtype=torch.float64, device=device)
    for zb in range(z0, z1, BLOCK):
        ze = min(zb + BLOCK, z1)
        zz = torch.arange(zb, ze, dtype=torch.float64, device=device)
        B = ky[None, None, :] * ys[None, :, None] + kz[None, None, :] * zz[:, None, None]  # (bz, ny, M)
        P = torch.cat([at * torch.cos(B), at * torch.sin(B)], -1).reshape((ze - zb) * ny, -1)
        del B
        torch.matmul(P, Q, out=out[zb - z0:ze - z0].view((ze - zb) * ny, nx))
    return out


def planes_numpy(z0: int, z1: int, ny: int, nx: int, seed: int = 5) -> np.ndarray:
    """The same field on the host by the direct mode sum (small crops only;
    equal to planes_torch up to the rounding of the summation order)."""
    k, ph, a = modes(seed)
    z = np.arange(z0, z1, dtype=np.float64)[:, None, None, None]
    y = np.arange(ny, dtype=np.float64)[None, :, None, None]
    x = np.arange(nx, dtype=np.float64)[None, None, :, None]
    arg = k[:, 0] * z + k[:, 1] * y + k[:, 2] * x + ph
    return np.sum(a * np.sin(arg), axis=-1)


CFG5_DIMS = (2048, 2048, 2048)
CFG5_REL = 1e-5
_range_cache: dict = {}


def field_range(nz: int = 2048, ny: int = 2048, nx: int = 2048, device="cuda", seed: int = 5):
    """(min, max) of planes [0, nz) of the field, found block by block on the
    device without keeping the field (cfg5: 64 GiB)."""
    import torch

    key = (nz, ny, nx, seed, str(device))
    if key not in _range_cache:
        lo, hi = math.inf, -math.inf
        buf = torch.empty((BLOCK, ny, nx), dtype=torch.float64, device=device)
        for z0 in range(0, nz, BLOCK):
            z1 = min(z0 + BLOCK, nz)
            v = planes_torch(z0, z1, ny, nx, device, seed, out=buf[: z1 - z0])
            lo, hi = min(lo, float(v.min())), max(hi, float(v.max()))
        del buf
        _range_cache[key] = (lo, hi)
    return _range_cache[key]


def eps_noa_range(vmin: float, vmax: float, rel: float) -> float:
    """Step a0 from a known range: eps = rel * (max - min) in double."""
    r = float(np.float64(vmax) - np.float64(vmin))
    return float(np.float64(rel) * np.float64(r)) if r > 0 else float(rel)
