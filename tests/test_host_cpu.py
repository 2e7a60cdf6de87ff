"""CPU: the product library loads and exports every symbol of include/dade_gpu.h,
fails loudly without a GPU, the C++ mirror header compiles, and the
reference-format artifact readers/writers round-trip (no GPU calls)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "dade_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(dade_gpu_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2411_17229_b200 import _capi
    lib = _capi.lib
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", nm), s
    assert set(declared_symbols()) <= set(_capi.EXPORTED)


def test_library_is_sm100a_native():
    from paper_2411_17229_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2411_17229_b200 as gp
    with pytest.raises(gp.CudaError):
        gp.Device(0)


def test_cpp_mirror_header_compiles(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "dade_gpu.hpp"\nint main(){ dade::gpu::CalibrationTable c = '
                   'dade::gpu::CalibrationTable::unbounded(32, 8); return c.checkpoints.size() == 3 ? 0 : 1; }\n')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    f"-L{ROOT / 'paper_2411_17229_b200'}", "-ldade_gpu",
                    f"-Wl,-rpath,{ROOT / 'paper_2411_17229_b200'}"], check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def test_expected_checkpoints_mirror():
    from paper_2411_17229_b200 import expected_checkpoints
    assert expected_checkpoints(32, 8) == [8, 16, 24]
    assert expected_checkpoints(33, 8) == [8, 16, 24, 32]
    assert expected_checkpoints(8, 3) == [3, 6]
    assert expected_checkpoints(32, 32) == []


def test_artifact_roundtrips_match_reference_files(tmp_path, ref_lib, ivf_fix):
    from paper_2411_17229_b200 import CalibrationTable, OrthoTransform
    from paper_2411_17229_b200.io import (Divf, read_cal, read_divf, read_transform, write_cal, write_divf,
                                          write_transform)
    fx = ivf_fix
    n, d = fx["data"].shape
    dv = Divf(d, n, 12, 0, d, fx["centroids"], fx["offsets"], fx["ids"], fx["storage"])
    write_divf(tmp_path / "a.ivf", dv)
    back = read_divf(tmp_path / "a.ivf")
    assert np.array_equal(back.storage, dv.storage) and np.array_equal(back.ids, dv.ids)
    # the reference library loads our DIVF and finds the same neighbours
    ivf = ref_lib.ivf_load(tmp_path / "a.ivf")
    ids, dist, cnt, st, _ = ivf.search(ref_lib.strategy_fd(d), fx["queries"], 10, 3)
    assert np.array_equal(ids, fx["fd_np3_ids"])
    t = OrthoTransform(d, 0, np.zeros(d), fx["eig"], fx["matrix"])
    write_transform(tmp_path / "t.dade", t)
    rt = ref_lib.load_transform(tmp_path / "t.dade")  # reference validates orthogonality on load
    assert rt.dim == d
    assert np.array_equal(read_transform(tmp_path / "t.dade").matrix, t.matrix)
    cal = CalibrationTable(0.1, 4, [int(x) for x in fx["cal_cps"]], [float(x) for x in fx["cal_eps"]])
    write_cal(tmp_path / "c.cal", cal)
    assert read_cal(tmp_path / "c.cal") == cal


def test_list_shard_plan_balances_and_partitions():
    from paper_2411_17229_b200.dist import plan_list_shards, plan_row_shards
    g = np.random.default_rng(3)
    sizes = g.integers(0, 5000, 1024)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    for world in (1, 2, 4, 8):
        owner = plan_list_shards(offsets, world, 256)
        assert owner.min() >= 0 and owner.max() < world
        load = np.bincount(owner, weights=sizes, minlength=world)
        assert load.max() - load.min() <= sizes.max()  # greedy LPT bound
        assert np.array_equal(owner, plan_list_shards(offsets, world, 256))  # deterministic
    shards = plan_row_shards(10, 4)
    assert shards == [(0, 3), (3, 6), (6, 8), (8, 10)]


def test_non_orthogonal_transform_rejected_like_reference(tmp_path, ref_lib, ivf_fix):
    """OrthoTransform::load's corruption check (proj/src/transform.cpp:344-356):
    the reference, the Python reader and the C++ mirror all refuse a DADE file
    whose columns are not orthonormal (max deviation > 1e-5), and accept it below."""
    from paper_2411_17229_b200 import OrthoTransform
    from paper_2411_17229_b200.io import read_transform, write_transform
    fx = ivf_fix
    d = fx["matrix"].size
    d = int(round(d ** 0.5))
    good = OrthoTransform(d, 0, np.zeros(d), fx["eig"], fx["matrix"])
    bad_m = np.array(fx["matrix"], np.float64).copy()
    bad_m[3] += 1e-3  # one entry of column 0 perturbed
    bad = OrthoTransform(d, 0, np.zeros(d), fx["eig"], bad_m)
    write_transform(tmp_path / "good.dade", good)
    write_transform(tmp_path / "bad.dade", bad)
    ref_lib.load_transform(tmp_path / "good.dade")
    read_transform(tmp_path / "good.dade")
    with pytest.raises(Exception, match="not orthogonal"):
        ref_lib.load_transform(tmp_path / "bad.dade")
    with pytest.raises(RuntimeError, match="not orthogonal"):
        read_transform(tmp_path / "bad.dade")
    src = tmp_path / "t.cpp"
    src.write_text('#include "dade_gpu.hpp"\n#include <iostream>\nint main(int, char** v){ try { '
                   'dade::gpu::OrthoTransform::load(v[1]); } catch (const std::runtime_error& e) { '
                   'std::cout << e.what(); return 3; } return 0; }\n')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    f"-L{ROOT / 'paper_2411_17229_b200'}", "-ldade_gpu",
                    f"-Wl,-rpath,{ROOT / 'paper_2411_17229_b200'}"], check=True)
    assert subprocess.run([str(exe), str(tmp_path / "good.dade")]).returncode == 0
    r = subprocess.run([str(exe), str(tmp_path / "bad.dade")], capture_output=True, text=True)
    assert r.returncode == 3 and "not orthogonal" in r.stdout
