"""GPU: the C++ mirror of the reference API (include/dade_gpu.hpp) driven end
to end from reference-format artifact files (DIVF, DADE transform, .cal,
fvecs), FD ids compared with the golden reference output."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "build" / "host_api_test"


def test_cpp_mirror_api(tmp_path, ivf_fix):
    from paper_2411_17229_b200 import CalibrationTable, OrthoTransform
    from paper_2411_17229_b200.io import Divf, read_ivecs, write_cal, write_divf, write_fvecs, write_transform
    if not EXE.exists():
        pytest.skip("build/host_api_test not built (python __graft_entry__.py build)")
    fx = ivf_fix
    n, d = fx["data"].shape
    write_divf(tmp_path / "i.divf", Divf(d, n, 12, 0, d, fx["centroids"], fx["offsets"], fx["ids"], fx["storage"]))
    write_transform(tmp_path / "t.dade", OrthoTransform(d, 0, np.zeros(d), fx["eig"], fx["matrix"]))
    write_cal(tmp_path / "c.cal", CalibrationTable(float(fx["cal_p_s"]), int(fx["cal_delta_d"]),
                                                   [int(x) for x in fx["cal_cps"]], [float(x) for x in fx["cal_eps"]]))
    write_fvecs(tmp_path / "q.fvecs", fx["queries"])
    out = tmp_path / "out.ivecs"
    res = subprocess.run([str(EXE), str(tmp_path / "i.divf"), str(tmp_path / "t.dade"), str(tmp_path / "c.cal"),
                          str(tmp_path / "q.fvecs"), str(out)], capture_output=True, text=True, timeout=120)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    ids = read_ivecs(out)
    assert np.array_equal(ids.astype(np.uint32), fx["fd_np3_ids"])
