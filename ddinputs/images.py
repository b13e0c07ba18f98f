"""Seeded Gaussian-mixture test images (SURVEY.md Sec. 8(d) "Generator").

Recipe (readings A20/A21 of DESIGN.md):
  * PRNG: splitmix64 seeded with ``(cfg << 32) ^ seed``; a uniform draw is
    ``(z >> 11) * 2**-53``.
  * Draw order per image: number of blobs K; then per blob
    cx, cy, sigma1, sigma2, theta, w; then (cfg 5 only) the noise field
    r ~ U[0,1) in row-major order.
  * Density evaluated at pixel centres ((i+1/2)h, (j+1/2)h), h = 1/N,
    g(x) = sum_k w_k exp(-1/2 (x-c_k)^T Sigma_k^-1 (x-c_k)),
    Sigma_k = R(theta) diag(sigma1^2, sigma2^2) R(theta)^T.
  * image = g / max g + floor (floor = 1e-3), normalised to mass 1.  The
    floor gives every basic cell positive mass, as P:299 requires.
  * cfg 5 ("plus seeded uniform noise 10%"): image = 0.9 * image + 0.1 * r / sum r.
  * Seeds: mu = 2k+1, nu = 2k+2 for image pair k.

Axis convention: array index [i, j] = (row, column) = (x1, x2).
"""
from __future__ import annotations

import math

import numpy as np

_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014); scalar draws in Python ints."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + _GAMMA) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def uniform_array(self, n: int) -> np.ndarray:
        """n consecutive draws, vectorised (identical to n calls of uniform())."""
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * np.uint64(_GAMMA)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * _GAMMA) & _MASK
        return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# Per-config generator parameters (BASELINE.json "configs").
CONFIGS = {
    1: dict(n=32, s=4, blobs=(3, 3), sigma=(0.05, 0.2), isotropic=True, noise=0.0,
            kappa_final=2.0, schedule="fixed"),
    2: dict(n=64, s=4, blobs=(3, 3), sigma=(0.05, 0.2), isotropic=True, noise=0.0,
            kappa_final=0.5, schedule="ladder", coarsest=16, eps_start=1.0),
    3: dict(n=256, s=4, blobs=(5, 10), sigma=(0.02, 0.15), isotropic=False, noise=0.0,
            kappa_final=0.5, schedule="ladder", coarsest=8, eps_start=0.0),
    4: dict(n=1024, s=8, blobs=(5, 10), sigma=(0.02, 0.15), isotropic=False, noise=0.0,
            kappa_final=0.5, schedule="ladder", coarsest=8, eps_start=0.0),
    5: dict(n=2048, s=8, blobs=(5, 10), sigma=(0.02, 0.15), isotropic=False, noise=0.1,
            kappa_final=0.5, schedule="ladder", coarsest=8, eps_start=0.0),
}

FLOOR = 1e-3


def _mixture_density(n: int, rng: SplitMix64, blobs, sigma, isotropic) -> np.ndarray:
    kmin, kmax = blobs
    nblobs = kmin + int(rng.uniform() * (kmax - kmin + 1)) if kmax > kmin else kmin
    nblobs = min(nblobs, kmax)
    h = 1.0 / n
    t = (np.arange(n, dtype=np.float64) + 0.5) * h
    x1 = t[:, None]
    x2 = t[None, :]
    g = np.zeros((n, n), dtype=np.float64)
    for _ in range(nblobs):
        cx = rng.uniform(0.1, 0.9)
        cy = rng.uniform(0.1, 0.9)
        s1 = rng.uniform(*sigma)
        s2 = rng.uniform(*sigma)
        th = rng.uniform(0.0, math.pi)
        w = rng.uniform(0.2, 1.0)
        if isotropic:
            s2, th = s1, 0.0
        c, s = math.cos(th), math.sin(th)
        # Sigma^-1 = R diag(1/s1^2, 1/s2^2) R^T
        a11 = c * c / s1**2 + s * s / s2**2
        a22 = s * s / s1**2 + c * c / s2**2
        a12 = c * s * (1.0 / s1**2 - 1.0 / s2**2)
        d1 = x1 - cx
        d2 = x2 - cy
        q = a11 * d1 * d1 + 2.0 * a12 * d1 * d2 + a22 * d2 * d2
        g += w * np.exp(-0.5 * q)
    return g


def gaussian_mixture_image(n: int, seed: int, cfg: int = 3, *, blobs=None, sigma=None,
                           isotropic=None, noise=None) -> np.ndarray:
    """One normalised n x n image (float64, C-contiguous, mass 1, all entries > 0)."""
    p = CONFIGS.get(cfg, CONFIGS[3])
    blobs = p["blobs"] if blobs is None else blobs
    sigma = p["sigma"] if sigma is None else sigma
    isotropic = p["isotropic"] if isotropic is None else isotropic
    noise = p["noise"] if noise is None else noise
    rng = SplitMix64((cfg << 32) ^ seed)
    g = _mixture_density(n, rng, blobs, sigma, isotropic)
    img = g / g.max() + FLOOR
    img /= img.sum()
    if noise > 0.0:
        r = rng.uniform_array(n * n).reshape(n, n)
        img = (1.0 - noise) * img + noise * r / r.sum()
        img /= img.sum()
    return np.ascontiguousarray(img)


def _mixture_1d(n: int, rng: SplitMix64, kmin=3, kmax=5) -> np.ndarray:
    nblobs = kmin + int(rng.uniform() * (kmax - kmin + 1))
    nblobs = min(nblobs, kmax)
    t = (np.arange(n, dtype=np.float64) + 0.5) / n
    g = np.zeros(n)
    for _ in range(nblobs):
        c = rng.uniform(0.1, 0.9)
        s = rng.uniform(0.05, 0.2)
        w = rng.uniform(0.2, 1.0)
        g += w * np.exp(-0.5 * ((t - c) / s) ** 2)
    g = g / g.max() + FLOOR
    return g / g.sum()


def product_image(n: int, seed: int, cfg: int = 0):
    """Product image m = m1 (x) m2 of two 1D mixtures (pin P2 of SURVEY 8(c)).

    Returns (image, m1, m2) with image[i, j] = m1[i] * m2[j]."""
    rng = SplitMix64((cfg << 32) ^ seed ^ 0x5A5A)
    m1 = _mixture_1d(n, rng)
    m2 = _mixture_1d(n, rng)
    return np.ascontiguousarray(np.outer(m1, m2)), m1, m2


def config_images(cfg: int, pair: int = 0, n: int | None = None):
    """(mu, nu) for BASELINE config ``cfg`` and image pair ``pair`` (seeds 2k+1, 2k+2)."""
    p = CONFIGS[cfg]
    n = p["n"] if n is None else n
    mu = gaussian_mixture_image(n, 2 * pair + 1, cfg)
    nu = gaussian_mixture_image(n, 2 * pair + 2, cfg)
    return mu, nu
