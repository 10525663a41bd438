"""Seeded synthetic scalar fields (input generators only).

This module holds none of the method's arithmetic: it only produces float32
grids.  It is the one module both the CUDA path's tests/bench and the oracle's
tests consume; each field is generated ONCE and the same float32 bits feed both
sides.

Shapes and structure follow the paper's workloads (3D
simulation/CT volumes of 128^3..1024^3 float32, split tree of -f,
PAPER.md:450-459) as fixed by BASELINE.json's five configs:

  c1  16^3   white noise  u24(seed, i)                    (6-conn)
  c2  4096^2 Gaussian mixture, K = 256 bumps              (4-conn, 2D)
  c3  256^3  sum of 6 sinusoids with integer wave vectors (6-conn)
  c4  512^3  white noise  u24(4, i)                       (6-conn)
  c5  1024^3 lognormal Gaussian random field, input = -rho (6-conn)

``u24(seed, i) = (splitmix64(seed * 0x9E3779B97F4A7C15 + i) >> 40) * 2^-24``
is exact in float32 and takes only 2^24 levels, so large grids have many exact
ties (exercising the id tie break).  All integer arithmetic is mod 2^64.
"""
from __future__ import annotations

import hashlib

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Steele/Lea/Flood splitmix64 finaliser on uint64 arrays (mod 2^64)."""
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def u24(seed: int, n: int, chunk: int = 1 << 24) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * _GOLDEN
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            i = np.arange(lo, hi, dtype=np.uint64)
            r = splitmix64(base + i) >> np.uint64(40)
            out[lo:hi] = r.astype(np.float32) * np.float32(2.0 ** -24)
    return out


def white_noise(dims, seed: int) -> np.ndarray:
    nx, ny, nz = dims
    return u24(seed, nx * ny * nz)


def gaussian_mixture_2d(nx: int, ny: int, seed: int, k: int = 256) -> np.ndarray:
    """f(x,y) = sum_k a_k exp(-((x-cx_k)^2 + (y-cy_k)^2) / (2 sigma_k^2)),
    centres U[0,n)^2, sigma_k = exp(U[ln 16, ln 256]), a_k ~ U[-1, 1];
    separable, summed in float64 (one matmul), rounded to float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cx = rng.uniform(0, nx, k)
    cy = rng.uniform(0, ny, k)
    sig = np.exp(rng.uniform(np.log(16.0), np.log(256.0), k))
    a = rng.uniform(-1.0, 1.0, k)
    xs = np.arange(nx, dtype=np.float64)
    ys = np.arange(ny, dtype=np.float64)
    gx = np.exp(-((xs[None, :] - cx[:, None]) ** 2) / (2 * sig[:, None] ** 2))  # k x nx
    gy = np.exp(-((ys[None, :] - cy[:, None]) ** 2) / (2 * sig[:, None] ** 2))  # k x ny
    f = (gy.T * a[None, :]) @ gx                                              # ny x nx
    return np.ascontiguousarray(f.astype(np.float32)).reshape(-1)


def sinusoids_3d(n: int, seed: int, k: int = 6) -> np.ndarray:
    """f = sum_k a_k sin(2 pi (k . x) / n + phi_k), integer wave vectors in
    [-4, 4]^3 \\ {0}, a_k ~ U[0.5, 1], phi_k ~ U[0, 2 pi); float64 -> float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    waves = []
    while len(waves) < k:
        w = rng.integers(-4, 5, 3)
        if np.any(w != 0):
            waves.append(w)
    amp = rng.uniform(0.5, 1.0, k)
    phi = rng.uniform(0.0, 2 * np.pi, k)
    t = 2 * np.pi * np.arange(n, dtype=np.float64) / n
    f = np.zeros((n, n, n), dtype=np.float64)  # [z, y, x]
    for (wx, wy, wz), a, p in zip(waves, amp, phi):
        # sin(A + B + C + p) accumulated plane by plane to bound memory
        ax = wx * t
        ay = wy * t
        for z in range(n):
            f[z] += a * np.sin(ax[None, :] + ay[:, None] + (wz * t[z] + p))
    return f.astype(np.float32).reshape(-1)


def lognormal_grf(n: int, seed: int, ns: float = -1.5, r: float = 0.5, device="cpu") -> np.ndarray:
    """Cosmology-like density: delta from white noise shaped by
    sqrt(P(k)), P(k) ~ k^ns exp(-k^2 r^2), rho = exp(delta / std(delta)),
    input = -rho (the split tree of rho).  ns = -1.5 and
    r = 0.5 cell give about 5% of the vertices as branches (NYX 512^3 has
    7-8e6 branches).  The field bits depend on the device
    torch generates on (the FFT); both sides always consume one buffer."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    kx = torch.fft.fftfreq(n, device=device, dtype=torch.float64) * 2 * np.pi
    kz = torch.fft.rfftfreq(n, device=device, dtype=torch.float64) * 2 * np.pi
    k2 = kx[:, None, None] ** 2 + kx[None, :, None] ** 2 + kz[None, None, :] ** 2
    k2[0, 0, 0] = 1.0
    amp = k2 ** (ns / 4.0) * torch.exp(-k2 * r * r / 2.0)
    amp[0, 0, 0] = 0.0
    noise = torch.complex(torch.randn(amp.shape, generator=g, device=device, dtype=torch.float64),
                          torch.randn(amp.shape, generator=g, device=device, dtype=torch.float64))
    delta = torch.fft.irfftn(noise * amp, s=(n, n, n))
    delta = delta / delta.std()
    rho = torch.exp(delta)
    return (-rho).to(torch.float32).cpu().numpy().reshape(-1)


CONFIGS = {
    "c1": dict(name="16^3 white noise, 6-conn", dims=(16, 16, 16), conn=6),
    "c2": dict(name="4096^2 Gaussian mixture, 4-conn", dims=(4096, 4096, 1), conn=4),
    "c3": dict(name="256^3 sum of sinusoids, 6-conn", dims=(256, 256, 256), conn=6),
    "c4": dict(name="512^3 white noise, 6-conn", dims=(512, 512, 512), conn=6),
    "c5": dict(name="1024^3 lognormal GRF (-rho), 6-conn", dims=(1024, 1024, 1024), conn=6),
}


def make(cfg: str, seed: int | None = None, scale: int | None = None, device="cpu") -> tuple[np.ndarray, tuple, int]:
    """Field of config ``cfg`` (c1..c5).  ``scale`` overrides the edge length
    (same recipe, smaller grid) for parity cases the oracle finishes quickly."""
    c = CONFIGS[cfg]
    dims = c["dims"]
    if scale is not None:
        dims = (scale, scale, 1) if cfg == "c2" else (scale, scale, scale)
    if cfg == "c1":
        f = white_noise(dims, 1 if seed is None else seed)
    elif cfg == "c2":
        f = gaussian_mixture_2d(dims[0], dims[1], 2 if seed is None else seed)
    elif cfg == "c3":
        f = sinusoids_3d(dims[0], 3 if seed is None else seed)
    elif cfg == "c4":
        f = white_noise(dims, 4 if seed is None else seed)
    elif cfg == "c5":
        f = lognormal_grf(dims[0], 5 if seed is None else seed, device=device)
    else:
        raise KeyError(cfg)
    return f, dims, c["conn"]


def field_hash(f: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(f).view(np.uint8)).hexdigest()[:16]
