"""TEST INFRASTRUCTURE — seeded Gaussian-mixture data for the golden fixtures.

make_golden.py generates fixtures from this data in the dev container and the
GPU tests regenerate the same arrays on the GPU box from the same seeds, so
only the reference's OUTPUTS are committed. Every step is elementwise or an
exactly rounded sum (math.fsum) — no BLAS/LAPACK kernels whose rounding could
differ between host CPUs — and each fixture stores a digest of the raw data
the tests compare against before using it.

Model (BASELINE.json configs): x = center_c + R diag(sqrt(lambda)) z,
z ~ N(0, I), component c uniform, lambda_i = i^-alpha normalised to trace D,
R Haar-orthogonal (modified Gram-Schmidt with positive norms, as
random_orthogonal in proj/src/transform.cpp:179-207), centers ~ N(0, s^2 I).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np


def spectrum(dim: int, alpha: float) -> np.ndarray:
    lam = np.array([(i + 1) ** -alpha for i in range(dim)], np.float64)
    return lam * (dim / math.fsum(lam))


def haar(dim: int, g: np.random.Generator) -> np.ndarray:
    """Columns of a Haar-random orthogonal matrix (MGS, two passes, exact dots)."""
    m = g.standard_normal((dim, dim))  # column k = m[:, k]
    q = np.zeros((dim, dim))
    for k in range(dim):
        v = m[:, k].copy()
        for _ in range(2):
            for j in range(k):
                v = v - math.fsum(q[:, j] * v) * q[:, j]
        q[:, k] = v / math.sqrt(math.fsum(v * v))
    return q


class Mixture:
    def __init__(self, dim: int, n_comp: int, alpha: float, center_std: float, seed: int, rotate: bool = True):
        g = np.random.default_rng(seed)
        self.dim, self.n_comp = dim, n_comp
        self.rot = haar(dim, g) if rotate else None
        self.sd = np.sqrt(spectrum(dim, alpha))
        self.centers = g.standard_normal((n_comp, dim)) * center_std

    def draw(self, n: int, seed: int) -> np.ndarray:
        g = np.random.default_rng(seed)
        comp = g.integers(0, self.n_comp, n)
        z = g.standard_normal((n, self.dim)) * self.sd
        if self.rot is None:
            y = z
        else:  # y = z @ R^T, accumulated over k in a fixed order with elementwise ops
            y = np.zeros((n, self.dim))
            for k in range(self.dim):
                y += np.multiply.outer(z[:, k], self.rot[:, k])
        return (self.centers[comp] + y).astype(np.float32)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# BASELINE.json config 0 (CPU-runnable oracle config)
CFG0 = dict(n=100_000, dim=128, nq=1_000, n_comp=64, alpha=1.0, center_std=4.0, seed=0, qseed=1,
            nlist=256, kmeans_iters=20, kmeans_seed=2, nprobe=16, k=10, delta_d=16, p_s=0.1,
            cal_pairs=100_000, cal_seed=1)

# long-vector cases (configs 2 and 4 shapes, scaled down): data already in its
# principal basis (R = I, spectrum decreasing), so the transform is the identity
# with the generating spectrum as eigenvalues
HD = {
    768: dict(n=8_000, dim=768, nq=48, n_comp=32, alpha=1.3, center_std=4.0, seed=40, qseed=41, nlist=16,
              nprobe=4, k=10, delta_d=64, p_s=0.1),
    960: dict(n=8_000, dim=960, nq=48, n_comp=32, alpha=1.5, center_std=2.0, seed=20, qseed=21, nlist=16,
              nprobe=4, k=20, delta_d=64, p_s=0.05),
}


def config0():
    c = CFG0
    mix = Mixture(c["dim"], c["n_comp"], c["alpha"], c["center_std"], c["seed"])
    return mix.draw(c["n"], c["seed"] + 1000), mix.draw(c["nq"], c["qseed"] + 1000)


def high_dim(dim: int):
    c = HD[dim]
    mix = Mixture(dim, c["n_comp"], c["alpha"], c["center_std"], c["seed"], rotate=False)
    return mix.draw(c["n"], c["seed"] + 1000), mix.draw(c["nq"], c["qseed"] + 1000), spectrum(dim, c["alpha"])
