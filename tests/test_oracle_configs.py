"""CPU: the oracle (oracle/dade_oracle.c) reproduces the reference's outputs
stored in the config-level fixtures (tests/golden/cfg0_fix.npz, hd_fix.npz),
and the fixtures' data regenerate bit-identically here from their seeds."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def cfg0_data(synth, cfg0_fix):
    base_raw, q_raw = synth.config0()
    assert synth.digest(base_raw) == str(cfg0_fix["base_raw_digest"])
    assert synth.digest(q_raw) == str(cfg0_fix["q_raw_digest"])
    return base_raw, q_raw


def test_cfg0_oracle_reproduces_reference(oracle_lib, synth, cfg0_fix, cfg0_data):
    fx = cfg0_fix
    base_raw, q_raw = cfg0_data
    base = oracle_lib.apply_transform(fx["matrix"], base_raw)
    assert synth.digest(base) == str(fx["base_digest"])  # transform_vector bits
    q = oracle_lib.apply_transform(fx["matrix"], q_raw)
    ids = fx["ids"].astype(np.int64)
    qs = q[:200]
    oi, od, oc, st = oracle_lib.ivf_search(fx["centroids"], fx["offsets"], fx["ids"], base[ids], qs, 10, 16)
    assert np.array_equal(oi, fx["fd_np16_ids"][:200]) and np.array_equal(od, fx["fd_np16_dists"][:200])
    assert np.array_equal(oc, fx["fd_np16_counts"][:200])
    coeff, scale = oracle_lib.dade_tables(fx["lambda_prefix"], 128, fx["cal_cps"], fx["cal_eps"])
    oi, od, oc, st = oracle_lib.ivf_search(fx["centroids"], fx["offsets"], fx["ids"], base[ids], qs, 10, 16,
                                           fx["cal_cps"], coeff, scale)
    assert np.array_equal(oi, fx["dade_np16_ids"][:200]) and np.array_equal(oc, fx["dade_np16_counts"][:200])
    assert np.array_equal(oracle_lib.ground_truth(base, q[:20], 10), fx["gt"][:20])


@pytest.mark.parametrize("dim", [768, 960])
def test_hd_oracle_reproduces_reference(oracle_lib, synth, hd_fix, dim):
    p = f"d{dim}_"
    base, q, lam = synth.high_dim(dim)
    assert synth.digest(base) == str(hd_fix[p + "base_digest"]) and synth.digest(q) == str(hd_fix[p + "q_digest"])
    c = synth.HD[dim]
    ids = hd_fix[p + "ids"].astype(np.int64)
    oi, od, oc, st = oracle_lib.ivf_search(hd_fix[p + "centroids"], hd_fix[p + "offsets"], hd_fix[p + "ids"],
                                           base[ids], q, c["k"], c["nprobe"])
    npb = c["nprobe"]
    assert np.array_equal(oi, hd_fix[p + f"fd_np{npb}_ids"]) and np.array_equal(od, hd_fix[p + f"fd_np{npb}_dists"])
    assert np.array_equal(st, hd_fix[p + f"fd_np{npb}_stats"])
