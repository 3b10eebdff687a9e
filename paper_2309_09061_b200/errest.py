"""GPU matvecs and the power-iteration error estimate of the product (reference h2.py:224-267,
bench.py:126-174), on device-resident matrices.

estimate_relative_spectral_error(x, y, g) = |X Y - G|_2 / |X Y|_2, both norms estimated by the
same `steps`-step power iteration on A^T A with the reference's seeding (one
np.random.default_rng(seed) stream: the first start vector for the denominator, the second for
the numerator).  Six H^2 matvecs per step run on the GPU; only the start vectors come from the
host.
"""

from __future__ import annotations

import math

import numpy as np

from .device import DeviceH2
from .errors import InvalidInputError

__all__ = ["h2_matvec", "h2_matvec_adjoint", "estimate_spectral_norm", "estimate_relative_spectral_error"]


def _torch():
    import torch
    return torch


def h2_matvec(g: DeviceH2, x, y=None, alpha: float = 1.0):
    """y <- y + alpha * G x (reference h2.py:224-244) with x, y CUDA tensors."""
    return g.matvec(x, alpha=alpha, out=y, accumulate=y is not None)


def h2_matvec_adjoint(g: DeviceH2, x, y=None, alpha: float = 1.0):
    """y <- y + alpha * G^T x (reference h2.py:247-267)."""
    return g.matvec(x, trans=True, alpha=alpha, out=y, accumulate=y is not None)


def estimate_spectral_norm(apply, apply_transposed, dim: int, steps: int, rng, device) -> float:
    """Power iteration on A^T A; sigma_1 estimate |A v| (reference bench.py:126-144)."""
    torch = _torch()
    v = rng.standard_normal(dim)
    nv = np.linalg.norm(v)
    if nv == 0 or dim == 0:
        return 0.0
    v = torch.as_tensor(v / nv, dtype=torch.float64, device=device)
    sigma = 0.0
    for _ in range(steps):
        w = apply(v)
        sigma = float(torch.linalg.vector_norm(w))
        if sigma == 0.0:
            return 0.0
        v = apply_transposed(w)
        nv = float(torch.linalg.vector_norm(v))
        if nv == 0.0:
            return sigma
        v = v / nv
    return sigma


def estimate_relative_spectral_error(x: DeviceH2, y: DeviceH2, g: DeviceH2, steps: int = 20,
                                     seed: int = 0) -> float:
    """|X Y - G|_2 / |X Y|_2 (reference bench.py:147-174), all matvecs on the GPU."""
    if steps < 1:
        raise InvalidInputError(f"steps must be >= 1, got {steps}")
    torch = _torch()
    n_k = y.shape[1]
    if x.shape[1] != y.shape[0] or g.shape != (x.shape[0], n_k):
        raise InvalidInputError("dimension mismatch between x, y and g")
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", g.ctx.device)

    def xy(v):
        return x.matvec(y.matvec(v))

    def xy_t(v):
        return y.matvec(x.matvec(v, trans=True), trans=True)

    def residual(v):
        return g.matvec(v, alpha=-1.0, out=xy(v), accumulate=True)

    def residual_t(v):
        return g.matvec(v, trans=True, alpha=-1.0, out=xy_t(v), accumulate=True)

    denom = estimate_spectral_norm(xy, xy_t, n_k, steps, rng, dev)
    numer = estimate_spectral_norm(residual, residual_t, n_k, steps, rng, dev)
    if denom == 0.0:
        return 0.0 if numer == 0.0 else math.inf
    return numer / denom
