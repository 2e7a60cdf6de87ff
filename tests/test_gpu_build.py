"""GPU index build against the live reference library:
k-means (proj/src/ivf.cpp:24-143) incl. its all-zero-distance seeding branch
and empty-cluster re-seeding, IvfIndex::build's posting lists, ground truth
with distance ties (proj/src/dataset_io.cpp:101-135), the covariance of
fit_pca (proj/src/transform.cpp:68-95) and the fitted transform. Bar:
bit-identical, except fit_pca's eigenvectors (the reference's cyclic Jacobi vs
LAPACK; tolerance written in the test)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gp():
    import paper_2411_17229_b200 as gp
    return gp


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def mixture(seed, n, dim, comps, spread=3.0):
    g = np.random.default_rng(seed)
    centers = g.standard_normal((comps, dim)) * spread
    lam = np.arange(1, dim + 1) ** -1.0
    x = centers[g.integers(0, comps, n)] + g.standard_normal((n, dim)) * np.sqrt(lam * dim / lam.sum())
    return x.astype(np.float32)


@pytest.mark.parametrize("n,dim,c,iters,seed", [(3000, 24, 17, 15, 3), (5000, 64, 40, 25, 9), (4000, 130, 33, 8, 1),
                                                (20000, 128, 256, 20, 2)])
def test_kmeans_matches_reference(gp, ref_lib, n, dim, c, iters, seed):
    x = mixture(seed + dim, n, dim, max(4, c // 3))
    dev = gp.Device(0)
    cen, asg, it = gp.kmeans(dev, x, c, iters, seed)
    rc, ra, ri = ref_lib.kmeans(x, c, iters, seed)
    assert it == ri
    assert np.array_equal(asg, ra)
    assert np.array_equal(bits(cen), bits(rc))


def test_kmeans_zero_distance_seeding_and_empty_clusters(gp, ref_lib):
    """40 distinct rows x 40 copies, 50 clusters: once every distinct row is a
    centroid the k-means++ total is 0 (rng::bounded pick), duplicate centroids
    leave clusters empty and the Lloyd step re-seeds them from the largest
    cluster's farthest member."""
    g = np.random.default_rng(11)
    pts = (g.standard_normal((40, 16)) * 2).astype(np.float32)
    x = np.repeat(pts, 40, axis=0)
    g.shuffle(x)
    dev = gp.Device(0)
    for c in (50, 40, 7):
        cen, asg, it = gp.kmeans(dev, x, c, 10, 4)
        rc, ra, ri = ref_lib.kmeans(x, c, 10, 4)
        assert it == ri and np.array_equal(asg, ra) and np.array_equal(bits(cen), bits(rc)), c


def test_kmeans_errors(gp):
    dev = gp.Device(0)
    x = np.zeros((10, 8), np.float32)
    with pytest.raises(gp.InvalidInput, match="n_clusters must be in"):
        gp.kmeans(dev, x, 11, 5, 1)
    with pytest.raises(gp.InvalidInput, match="max_iters must be positive"):
        gp.kmeans(dev, x, 2, 0, 1)


def test_ivf_build_lists_match_reference(gp, ref_lib, tmp_path):
    from paper_2411_17229_b200.io import read_divf
    x = mixture(5, 12000, 96, 30)
    dev = gp.Device(0)
    idx = gp.IvfIndex.build(dev, x, 48, 12, 7)
    ref = ref_lib.ivf_build(x, 48, layout=0, split=0, iters=12, seed=7)
    ref.save(tmp_path / "r.ivf")
    dv = read_divf(tmp_path / "r.ivf")
    assert np.array_equal(idx.offsets, dv.offsets) and np.array_equal(idx.ids, dv.ids)
    assert np.array_equal(bits(idx.centroids), bits(dv.centroids))
    assert np.array_equal(bits(idx.storage), bits(dv.storage.reshape(idx.storage.shape)))
    # the built index is installed: FD search equals the reference's on its own index
    q = x[::97][:60] + 0.01
    gi, gd, gc = idx.search_batch(q, 10, 5, gp.FdScanningStrategy(96))
    ri, rd, rcnt, _, _ = ref.search(ref_lib.strategy_fd(96), q, 10, 5)
    assert np.array_equal(gi, ri) and np.array_equal(bits(gd), bits(rd))


@pytest.mark.parametrize("n,dim,nq,k", [(6000, 48, 120, 7), (5000, 33, 64, 300), (3000, 256, 50, 100),
                                        (1000, 16, 20, 1000)])
def test_ground_truth_matches_reference(gp, ref_lib, n, dim, nq, k):
    g = np.random.default_rng(n + k)
    x = mixture(dim, n, dim, 5)
    x[1::5] = x[::5][: len(x[1::5])]  # duplicated rows: exact distance ties, broken by id
    q = x[g.integers(0, n, nq)] + (g.standard_normal((nq, dim)) * 0.05).astype(np.float32)
    q[0] = x[3]
    dev = gp.Device(0)
    assert np.array_equal(gp.compute_ground_truth(dev, x, q, k), ref_lib.ground_truth(x, q, k))


def test_ground_truth_errors(gp):
    dev = gp.Device(0)
    x = np.zeros((10, 8), np.float32)
    with pytest.raises(gp.InvalidInput, match="k must be in"):
        gp.compute_ground_truth(dev, x, x[:2], 11)


@pytest.mark.parametrize("n,dim", [(5000, 40), (3001, 7), (20000, 96)])
def test_covariance_bit_exact(gp, ref_lib, n, dim):
    x = mixture(n, n, dim, 6) + 5.0
    dev = gp.Device(0)
    mean, cov = gp.compute_covariance(dev, x)
    rm, rcv = ref_lib.covariance(x)
    assert np.array_equal(mean.view(np.uint64), rm.view(np.uint64))
    assert np.array_equal(cov.view(np.uint64), rcv.view(np.uint64))


def test_fit_pca_matches_reference(gp, ref_lib):
    """Eigenvalues within 1e-9 x trace, columns within 1e-6 with the reference's
    order and orientation (the reference's Jacobi stops at off-diagonal norm
    1e-10 x trace, transform.cpp:118-119)."""
    x = mixture(64, 20000, 64, 8)
    dev = gp.Device(0)
    t = gp.fit_pca(dev, x)
    mean, eig, mat, _ = ref_lib.fit_pca(x).arrays()
    assert np.array_equal(t.mean, mean)
    tr = float(eig.sum())
    assert np.max(np.abs(t.eigenvalues - eig)) <= 1e-9 * tr
    assert np.max(np.abs(t.matrix - mat)) <= 1e-6
