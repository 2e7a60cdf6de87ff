"""BASELINE.json workloads and their GPU-built artifacts.

The artifacts the search path reads (rotated base in IVF posting lists, PCA
transform, calibration table) are produced here on the GPU, then handed both
to libdade_gpu.so and — through the reference file formats — to the reference
CPU library, so the two arms search identical lists.
This is offline index building, outside every timed region.

Data (BASELINE configs; paper datasets are not available here): each vector =
center_c + R diag(sqrt(lambda)) z with z ~ N(0, I), component c uniform,
lambda_i = i^-a normalised to trace D, R Haar-orthogonal, centers ~ N(0, s^2 I);
seeded synthetic stand-ins for DEEP/GIST shapes, drawn with torch's device RNG.
The build runs the reference's algorithms on the GPU (libdade_gpu.so):
  * PCA: compute_covariance bit-identical (dade_gpu_covariance), fp64 eigh,
    the reference's column order / orientation / clamp (api.fit_pca);
    rotation with the bit-exact fp64 kernel (dade_gpu_rotate);
  * calibration: calibrate, bit-exact (dade_gpu_calibrate);
  * IVF lists: IvfIndex::build with k-means++ seeding, early stop and
    empty-cluster re-seeding (dade_gpu_ivf_build): the reference's lists;
  * ground truth: compute_ground_truth, exact (dade_gpu_ground_truth).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from pathlib import Path

from . import _capi
from .api import CalibrationTable, Device, IvfIndex, OrthoTransform, compute_ground_truth
from .api import fit_pca as api_fit_pca
from .configs import ART_VERSION, CONFIGS, Config, artifact_dir  # noqa: F401


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
          log=print, gt_queries: int | None = None) -> Artifacts:
    """The workload's artifacts, built on the GPU with the reference's
    arithmetic (api.fit_pca, CalibrationTable.calibrate, IvfIndex.build,
    compute_ground_truth), so the reference CPU library given the same files
    holds the index it would build itself. gt_queries: ground truth for the
    first queries only (recall sample)."""
    import time
    t0 = time.time()
    mix = Mixture(cfg, device)
    base = mix.draw(cfg.n, cfg.seed + 1000)
    q_raw = mix.draw(nq or cfg.nq, cfg.qseed + 1000)
    t = api_fit_pca(dev, base)
    base_rot = rotate_device(dev, t, base)
    q_rot = rotate_device(dev, t, q_raw)
    del base
    log(f"[build] data+pca+rotate {time.time() - t0:.1f}s")
    cal = CalibrationTable.calibrate(dev, t, base_rot, cfg.p_s, cfg.delta_d, cfg.cal_pairs, cfg.cal_seed,
                                     device_ptr=True, count=cfg.n)
    log(f"[build] calibration eps={['%.4f' % e for e in cal.epsilons]}")
    art = Artifacts(cfg, t, cal, base_rot, q_raw, q_rot)
    if not cfg.flat:
        idx = IvfIndex.build(dev, base_rot, cfg.nlist, cfg.kmeans_iters, cfg.kmeans_seed)
        art.centroids, art.offsets, art.ids, art.storage = idx.centroids, idx.offsets, idx.ids, idx.storage
        sizes = np.diff(art.offsets.astype(np.int64))
        log(f"[build] k-means++ / Lloyd {time.time() - t0:.1f}s lists min/mean/max "
            f"{sizes.min()}/{sizes.mean():.0f}/{sizes.max()}")
    if with_gt:
        m = q_rot.shape[0] if gt_queries is None else min(gt_queries, q_rot.shape[0])
        art.gt = compute_ground_truth(dev, base_rot, q_rot[:m].contiguous(), cfg.k)
        log(f"[build] ground truth ({m} queries) {time.time() - t0:.1f}s")
    torch.cuda.synchronize()
    return art


# ---- on-disk artifacts in the reference's formats (shared by both bench arms) ------------
def save(art: Artifacts, out: Path) -> None:
    """t.dade, c.cal, index.ivf (or base.fvecs for the flat config), queries.fvecs
    (raw), gt.ivecs: the files the reference's loaders read."""
    from .io import Divf, write_cal, write_divf, write_fvecs, write_ivecs, write_transform
    cfg = art.cfg
    out.mkdir(parents=True, exist_ok=True)
    tmp = out.with_name(out.name + ".part")
    tmp.mkdir(parents=True, exist_ok=True)
    write_transform(tmp / "t.dade", art.transform)
    write_cal(tmp / "c.cal", art.cal)
    if cfg.flat:
        write_fvecs(tmp / "base.fvecs", art.base_rot.cpu().numpy())
    else:
        write_divf(tmp / "index.ivf", Divf(cfg.dim, cfg.n, cfg.nlist, 0, cfg.dim, art.centroids, art.offsets,
                                           art.ids, art.storage.reshape(-1)))
    write_fvecs(tmp / "queries.fvecs", art.q_raw.cpu().numpy())
    if art.gt is not None:
        write_ivecs(tmp / "gt.ivecs", art.gt.astype(np.int32))
    for f in tmp.iterdir():
        f.replace(out / f.name)
    tmp.rmdir()
    (out / "DONE").write_text(cfg.describe())


def ensure_artifacts(cfg: Config, nq: int | None = None, gt_queries: int | None = None, log=print) -> Path:
    """Build (in this process) and save the workload's artifacts once per box."""
    out = artifact_dir(cfg, nq=nq)
    if (out / "DONE").exists():
        return out
    dev = Device(0)
    art = build(cfg, dev, torch.device("cuda:0"), with_gt=True, nq=nq, log=log, gt_queries=gt_queries)
    save(art, out)
    return out


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(description="build a BASELINE workload's artifacts in the reference formats")
    ap.add_argument("--config", default="config1")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--gt-queries", type=int, default=None)
    a = ap.parse_args(argv)
    import sys
    print(ensure_artifacts(CONFIGS[a.config], a.nq, a.gt_queries, log=lambda *x: print(*x, file=sys.stderr)))


if __name__ == "__main__":
    main()
