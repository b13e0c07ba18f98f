"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no Sinkhorn, no partitions, no
marginals).  It only draws the test images mu, nu the paper describes:
"mixtures of Gaussians with random variances and magnitudes" on 2^n x 2^n
grids (Sec. 7.1 "Test data"), with the recipe of
SURVEY.md Sec. 8(d) / BASELINE.json configs.  Both libraries receive the same
float64 arrays through their C-ABI, so they see bit-identical inputs.
"""
from .images import (  # noqa: F401
    SplitMix64,
    gaussian_mixture_image,
    product_image,
    config_images,
    CONFIGS,
)
