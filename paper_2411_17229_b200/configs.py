"""BASELINE.json workload definitions (pure Python: importable by file path
without loading libdade_gpu.so, which the reference bench arm must not map)."""
from __future__ import annotations

import tempfile
from dataclasses import dataclass
from pathlib import Path

ART_VERSION = "v2"  # bump when the generator or the artifact build changes


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



def artifact_dir(cfg: Config, root=None, nq: int | None = None) -> Path:
    """Where a workload's artifacts (reference file formats) live on this box."""
    root = Path(root or Path(tempfile.gettempdir()) / "dade_artifacts")
    return root / f"{cfg.name}-{ART_VERSION}-nq{nq or cfg.nq}"
