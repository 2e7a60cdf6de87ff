"""BASELINE.json workloads and their GPU-built artifacts.

The artifacts the search path reads (rotated base in IVF posting lists, PCA
transform, calibration table) are produced here on the GPU, then handed both
to libdade_gpu.so and — through the reference file formats — to the reference
CPU library, so the two arms search identical lists.
This is offline index building, outside every timed region.

Data (BASELINE configs; paper datasets are not available here): each vector =
center_c + R diag(sqrt(lambda)) z with z ~ N(0, I), component c uniform,
lambda_i = i^-a normalised to trace D, R Haar-orthogonal, centers ~ N(0, s^2 I).
Seeded synthetic stand-ins for DEEP/GIST shapes; torch is used only as the
device-memory / GEMM plumbing of this offline build:
  * PCA: fp64 covariance (1/N, centred) + eigh, columns by descending variance,
    sign-oriented like proj/src/transform.cpp:40-56; base rotation with the
    bit-exact fp64 rotation kernel of libdade_gpu.so.
  * k-means: random-sample seeding (the reference seeds with k-means++,
    proj/src/ivf.cpp:38-68 — sequential over N per centroid, too slow at 1M-10M)
    then Lloyd iterations; posting lists ascending by id (ivf.cpp:163-191).
  * calibration: dade_gpu_calibrate (the reference algorithm, bit-exact).
  * ground truth: fp32 GEMM candidates re-ranked exactly in fp64 with
    (d^2, id) order (compute_ground_truth, proj/src/dataset_io.cpp:101-135).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .api import CalibrationTable, Device, OrthoTransform


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dim: int
    nq: int
    n_comp: int
    alpha: float
    center_std: float
    seed: int
    qseed: int
    nlist: int
    nprobe: int
    k: int
    delta_d: int
    p_s: float
    kmeans_iters: int = 20
    kmeans_seed: int = 2
    cal_pairs: int = 100_000
    cal_seed: int = 1
    flat: bool = False

    def describe(self) -> str:
        if self.flat:
            return (f"{self.name}: flat N={self.n} D={self.dim} nq={self.nq} K={self.k} "
                    f"dd={self.delta_d} p_s={self.p_s}")
        return (f"{self.name}: N={self.n} D={self.dim} nq={self.nq} nlist={self.nlist} "
                f"nprobe={self.nprobe} K={self.k} dd={self.delta_d} p_s={self.p_s}")


CONFIGS = {
    "config0": Config("config0", 100_000, 128, 1_000, 64, 1.0, 4.0, 0, 1, 256, 16, 10, 16, 0.1),
    "config1": Config("config1", 1_000_000, 256, 10_000, 1024, 1.2, 4.0, 10, 11, 1024, 32, 100, 32, 0.1),
    "config2": Config("config2", 1_000_000, 960, 1_000, 512, 1.5, 2.0, 20, 21, 1024, 64, 20, 64, 0.05),
    "config3": Config("config3", 10_000_000, 128, 100_000, 4096, 1.0, 4.0, 30, 31, 16384, 64, 100, 16, 0.1),
    "config4": Config("config4", 2_000_000, 768, 4_096, 256, 1.3, 4.0, 40, 41, 0, 0, 10, 64, 0.1, flat=True),
}


def _spectrum(dim: int, alpha: float) -> torch.Tensor:
    lam = torch.arange(1, dim + 1, dtype=torch.float64) ** (-alpha)
    return lam * (dim / lam.sum())


class Mixture:
    """Seeded Gaussian mixture model (shared by base and query draws)."""

    def __init__(self, cfg: Config, device: torch.device):
        self.cfg, self.device = cfg, device
        g = torch.Generator(device="cpu").manual_seed(cfg.seed)
        a = torch.randn(cfg.dim, cfg.dim, generator=g, dtype=torch.float64)
        q, r = torch.linalg.qr(a)
        q = q * torch.sign(torch.diagonal(r))[None, :]  # Haar: positive diag(R)
        self.rot = q.to(device)
        self.sd = _spectrum(cfg.dim, cfg.alpha).sqrt().to(device)
        self.centers = (torch.randn(cfg.n_comp, cfg.dim, generator=g, dtype=torch.float64)
                        * cfg.center_std).to(device)

    def draw(self, n: int, seed: int, chunk: int = 1 << 18) -> torch.Tensor:
        cfg = self.cfg
        g = torch.Generator(device=self.device).manual_seed(seed)
        out = torch.empty(n, cfg.dim, dtype=torch.float32, device=self.device)
        for s in range(0, n, chunk):
            m = min(chunk, n - s)
            comp = torch.randint(0, cfg.n_comp, (m,), generator=g, device=self.device)
            z = torch.randn(m, cfg.dim, generator=g, device=self.device, dtype=torch.float64) * self.sd
            out[s:s + m] = (self.centers[comp] + z @ self.rot.T).to(torch.float32)
        return out


def fit_pca(x: torch.Tensor, chunk: int = 1 << 18) -> OrthoTransform:
    n, d = x.shape
    mean = torch.zeros(d, dtype=torch.float64, device=x.device)
    for s in range(0, n, chunk):
        mean += x[s:s + chunk].double().sum(0)
    mean /= n
    cov = torch.zeros(d, d, dtype=torch.float64, device=x.device)
    for s in range(0, n, chunk):
        c = x[s:s + chunk].double() - mean
        cov += c.T @ c
    cov /= n
    evals, evecs = torch.linalg.eigh(cov.cpu())
    evals = evals.flip(0).numpy().copy()
    evecs = evecs.flip(1).numpy().copy()  # columns = directions, descending variance
    for k in range(d):  # orient_column: first nonzero component positive
        col = evecs[:, k]
        nz = np.nonzero(col)[0]
        if nz.size and col[nz[0]] < 0:
            evecs[:, k] = -col
    evals = np.where((evals < 0) & (evals > -1e-6), 0.0, evals)
    matrix = np.ascontiguousarray(evecs.T).reshape(-1)  # column-major: column k contiguous
    return OrthoTransform(d, 0, mean.cpu().numpy(), evals, matrix)


def rotate_device(dev: Device, t: OrthoTransform, x: torch.Tensor, chunk: int = 1 << 18) -> torch.Tensor:
    """apply_transform on the device with the bit-exact fp64 kernel."""
    t.upload(dev)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    dev.set_stream(stream)
    for s in range(0, x.shape[0], chunk):
        m = min(chunk, x.shape[0] - s)
        _capi.check(_capi.lib.dade_gpu_rotate(dev.h, _capi.ptr(x[s:s + m]), m, _capi.ptr(out[s:s + m]),
                                              _capi.DEVICE_PTRS))
    dev.synchronize()
    dev.set_stream(None)
    return out


@torch.no_grad()
def kmeans(x: torch.Tensor, c: int, iters: int, seed: int, chunk: int = 1 << 16):
    n, d = x.shape
    g = torch.Generator(device="cpu").manual_seed(seed)
    init = torch.randperm(n, generator=g)[:c].to(x.device)
    cen = x[init].clone()
    assign = torch.empty(n, dtype=torch.int64, device=x.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for it in range(iters + 1):
            cn = (cen.double() ** 2).sum(1).float()
            for s in range(0, n, chunk):
                xs = x[s:s + chunk]
                dist = cn[None, :] - 2.0 * (xs @ cen.T)
                assign[s:s + chunk] = dist.argmin(1)
            if it == iters:
                break
            sums = torch.zeros(c, d, dtype=torch.float64, device=x.device)
            sums.index_add_(0, assign, x.double())
            cnt = torch.bincount(assign, minlength=c)
            keep = cnt > 0
            cen[keep] = (sums[keep] / cnt[keep, None].double()).float()
            if (~keep).any():  # re-seed empties from random points
                empt = torch.nonzero(~keep).squeeze(1)
                pick = torch.randint(0, n, (empt.numel(),), generator=g).to(x.device)
                cen[empt] = x[pick]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return cen, assign


def build_lists(x: torch.Tensor, cen: torch.Tensor, assign: torch.Tensor):
    n = x.shape[0]
    key = assign * n + torch.arange(n, device=x.device)
    order = torch.argsort(key)
    counts = torch.bincount(assign, minlength=cen.shape[0])
    offsets = torch.zeros(cen.shape[0] + 1, dtype=torch.int64, device=x.device)
    offsets[1:] = torch.cumsum(counts, 0)
    return order, offsets


@torch.no_grad()
def ground_truth(base: torch.Tensor, q: torch.Tensor, k: int, extra: int = 64, qchunk: int = 1024,
                 bchunk: int = 1 << 18) -> np.ndarray:
    """Exact top-k by (fp64 d^2, id): fp32 GEMM shortlist, fp64 re-rank."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    kk = min(k + extra, base.shape[0])
    bn = (base.double() ** 2).sum(1).float()
    out = np.zeros((q.shape[0], k), np.uint32)
    try:
        for s in range(0, q.shape[0], qchunk):
            qs = q[s:s + qchunk]
            best_d = best_i = None
            for b in range(0, base.shape[0], bchunk):
                bs = base[b:b + bchunk]
                d = bn[None, b:b + bchunk] - 2.0 * (qs @ bs.T)
                dv, di = torch.topk(d, min(kk, d.shape[1]), dim=1, largest=False)
                di = di + b
                if best_d is None:
                    best_d, best_i = dv, di
                else:
                    cd = torch.cat([best_d, dv], 1)
                    ci = torch.cat([best_i, di], 1)
                    best_d, sel = torch.topk(cd, kk, dim=1, largest=False)
                    best_i = torch.gather(ci, 1, sel)
            cand = base[best_i]  # [m, kk, D]
            d2 = ((cand.double() - qs.double()[:, None, :]) ** 2).sum(2)
            # (d2, id) lexicographic
            ids = best_i
            order = torch.argsort(ids, dim=1)
            d2, ids = torch.gather(d2, 1, order), torch.gather(ids, 1, order)
            order = torch.argsort(d2, dim=1, stable=True)
            out[s:s + qs.shape[0]] = torch.gather(ids, 1, order)[:, :k].cpu().numpy().astype(np.uint32)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


@dataclass
class Artifacts:
    cfg: Config
    transform: OrthoTransform
    cal: CalibrationTable
    base_rot: torch.Tensor        # [N, D] rotated base (device), id order
    q_raw: torch.Tensor           # [nq, D] raw queries (device)
    q_rot: torch.Tensor           # [nq, D] rotated queries (device)
    centroids: np.ndarray | None = None
    offsets: np.ndarray | None = None
    ids: np.ndarray | None = None
    storage: np.ndarray | None = None
    gt: np.ndarray | None = None


def build(cfg: Config, dev: Device, device: torch.device, with_gt: bool = True, nq: int | None = None,
          log=print) -> Artifacts:
    import time
    t0 = time.time()
    mix = Mixture(cfg, device)
    base = mix.draw(cfg.n, cfg.seed + 1000)
    q_raw = mix.draw(nq or cfg.nq, cfg.qseed + 1000)
    t = fit_pca(base)
    base_rot = rotate_device(dev, t, base)
    q_rot = rotate_device(dev, t, q_raw)
    del base
    log(f"[build] data+pca+rotate {time.time() - t0:.1f}s")
    cal = CalibrationTable.calibrate(dev, t, base_rot, cfg.p_s, cfg.delta_d, cfg.cal_pairs, cfg.cal_seed,
                                     device_ptr=True, count=cfg.n)
    log(f"[build] calibration eps={['%.4f' % e for e in cal.epsilons]}")
    art = Artifacts(cfg, t, cal, base_rot, q_raw, q_rot)
    if not cfg.flat:
        cen, assign = kmeans(base_rot, cfg.nlist, cfg.kmeans_iters, cfg.kmeans_seed)
        order, offsets = build_lists(base_rot, cen, assign)
        art.centroids = cen.cpu().numpy()
        art.offsets = offsets.cpu().numpy().astype(np.uint32)
        art.ids = order.cpu().numpy().astype(np.uint32)
        art.storage = base_rot[order].cpu().numpy()
        sizes = np.diff(art.offsets)
        log(f"[build] kmeans {time.time() - t0:.1f}s lists min/mean/max {sizes.min()}/{sizes.mean():.0f}/{sizes.max()}")
    if with_gt:
        art.gt = ground_truth(base_rot, q_rot, cfg.k)
        log(f"[build] ground truth {time.time() - t0:.1f}s")
    torch.cuda.synchronize()
    return art
