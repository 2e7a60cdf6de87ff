"""The C ABI's own NCCL layer (csrc/comm.cu; SURVEY.md §8b init_nccl /
sharded_*): a one-rank communicator runs every step of the sharded protocols
(all-gather, all-reduce MIN of the radius, send/recv to the owner, device
merge), so FD results must equal the unsharded search bit for bit, for host
and device buffers and raw (unrotated) queries. Multi-rank runs need one GPU
per rank (the pool has one); the protocol's host logic is covered on CPU by
tests/test_dist_gloo.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gp():
    import paper_2411_17229_b200 as gp
    return gp


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def data(seed, n, dim, comps=12):
    g = np.random.default_rng(seed)
    centers = g.standard_normal((comps, dim)) * 3
    lam = np.arange(1, dim + 1) ** -1.0
    x = centers[g.integers(0, comps, n)] + g.standard_normal((n, dim)) * np.sqrt(lam * dim / lam.sum())
    q = x[g.integers(0, n, 200)] + 0.2 * g.standard_normal((200, dim))
    return x.astype(np.float32), q.astype(np.float32)


def test_sharded_ivf_search_one_rank_nccl(gp):
    import torch

    from paper_2411_17229_b200.dist import NcclComm
    x, q = data(1, 30000, 64)
    dev = gp.Device(0)
    idx = gp.IvfIndex.build(dev, x, 40, 10, 3)
    fd = gp.FdScanningStrategy(64)
    ri, rd, rc = idx.search_batch(q, 20, 6, fd)
    comm = NcclComm(dev, 1, 0)
    dev.apply(fd)
    st = gp.DcoStats()
    ci, cd, cc = comm.ivf_search(q, q.shape[0], 20, 6, stats=st)
    assert np.array_equal(ci, ri) and np.array_equal(bits(cd), bits(rd)) and np.array_equal(cc, rc)
    assert st.total_dco > 0
    qd = torch.from_numpy(q).cuda()
    ci, cd, cc = comm.ivf_search(qd, q.shape[0], 20, 6)
    assert np.array_equal(ci.cpu().numpy().astype(np.uint32), ri)
    assert np.array_equal(bits(cd.cpu().numpy()), bits(rd))
    # raw queries: rotated on the device first (identity transform here), DADE unbounded == FD
    t = gp.OrthoTransform(64, 0, np.zeros(64), np.linspace(2, 0.1, 64), np.eye(64).reshape(-1))
    unb = gp.DadeStrategy(t, gp.CalibrationTable.unbounded(64, 16), 16, dev=dev)
    ci, cd, cc = comm.ivf_search(q, q.shape[0], 20, 6, raw=True)
    assert np.array_equal(ci, ri) and np.array_equal(bits(cd), bits(rd))
    comm.close()


def test_sharded_flat_search_one_rank_nccl(gp):
    from paper_2411_17229_b200.dist import NcclComm
    x, q = data(2, 20000, 96)
    dev = gp.Device(0)
    fi = gp.FlatIndex(dev, x)
    fd = gp.FdScanningStrategy(96)
    ri, rd, rc = fi.search_batch(q, 10, fd)
    comm = NcclComm(dev, 1, 0)
    ci, cd, cc = comm.flat_search(q, q.shape[0], 10)
    assert np.array_equal(ci, ri) and np.array_equal(bits(cd), bits(rd)) and np.array_equal(cc, rc)


def test_comm_errors(gp):
    import ctypes as C

    from paper_2411_17229_b200 import _capi
    dev = gp.Device(0)
    h = C.c_void_p()
    uid = (C.c_uint8 * 128)()
    with pytest.raises(gp.InvalidInput, match="bad rank"):
        _capi.check(_capi.lib.dade_gpu_comm_create(dev.h, 1, 3, uid, C.byref(h)))
