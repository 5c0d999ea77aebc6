"""GPU parity of the cross product akm_kernel_cross_mvm (K_{*X} V for prediction)
against the dense oracle (oracle/cross.py), through the C ABI.

Gate: relative Frobenius error over the n_t x r block <= 1e-6 (Gaussian) / 1e-3 (Matern), as for
the square products (BASELINE.json north_star; reading R8), full rows at small sizes and
seeded row samples of the x4 workload at full size.
"""
import numpy as np
import pytest

import workloads
from oracle import dense_apply
from oracle.cross import dense_cross

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def akm():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as mod
    return mod


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def gpu_cross(akm, X, n_src, windows, family, theta, V, N=32, m=6, host=False):
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(np.ascontiguousarray(X)).to(dev), windows, family, N, 2.0, m, 1.0 / 16)
    plan.set_theta(*theta)
    V = np.ascontiguousarray(V if V.ndim == 2 else V[:, None])
    n_t = X.shape[0] - n_src
    if host:
        Yt = np.full((n_t, V.shape[1]), np.nan)
        plan.cross_mvm(n_src, V, Yt)
    else:
        Yt = torch.full((n_t, V.shape[1]), float("nan"), dtype=torch.float64, device=dev)
        plan.cross_mvm(n_src, torch.from_numpy(V).to(dev), Yt)
        torch.cuda.synchronize()
        Yt = Yt.cpu().numpy()
    plan.close()
    return Yt


@pytest.mark.parametrize("n_src,n_t,r", [(4000, 1000, 1), (3000, 2500, 3), (2500, 37, 11)])
def test_cross_gaussian_d3_matches_oracle(akm, n_src, n_t, r):
    wl = workloads.CONFIGS["c2"]
    X = workloads.make_X(wl, n=n_src + n_t)
    V = workloads.make_V(wl, n=n_src, r=r)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    got = gpu_cross(akm, X, n_src, wl.windows, wl.family, theta, V)
    want = dense_cross(X[:n_src], X[n_src:], wl.windows, wl.family, theta, V)
    assert rel(got, want) <= 1e-6


def test_cross_matern_d2_matches_oracle(akm):
    wl = workloads.CONFIGS["c3"]
    X = workloads.make_X(wl, n=3000)
    V = workloads.make_V(wl, n=2400, r=11)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    got = gpu_cross(akm, X, 2400, wl.windows, wl.family, theta, V, N=128, m=8)
    want = dense_cross(X[:2400], X[2400:], wl.windows, wl.family, theta, V)
    assert rel(got, want) <= 1e-3


def test_cross_host_buffers_and_edges(akm):
    wl = workloads.CONFIGS["c1"]
    X = workloads.make_X(wl, n=1500)
    V = workloads.make_V(wl, n=1000, r=2)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    dev_out = gpu_cross(akm, X, 1000, wl.windows, wl.family, theta, V)
    host_out = gpu_cross(akm, X, 1000, wl.windows, wl.family, theta, V, host=True)
    np.testing.assert_allclose(host_out, dev_out, rtol=1e-13, atol=1e-13)
    assert rel(dev_out, dense_cross(X[:1000], X[1000:], wl.windows, wl.family, theta, V)) <= 1e-6
    # no sources: the product is exactly zero
    z = gpu_cross(akm, X, 0, wl.windows, wl.family, theta, np.zeros((0, 2)))
    assert z.shape == (1500, 2) and np.all(z == 0.0)


def test_cross_argument_errors(akm):
    wl = workloads.CONFIGS["c1"]
    X = workloads.make_X(wl, n=200)
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    V = torch.zeros((100, 1), dtype=torch.float64, device=dev)
    Y = torch.zeros((100, 1), dtype=torch.float64, device=dev)
    with pytest.raises(akm.AkmError):   # before set_points / set_theta
        plan.cross_mvm(100, V, Y)
    plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, 2.0, wl.m, 1.0 / 16)
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    with pytest.raises(ValueError):     # V rows != n_src
        plan.cross_mvm(101, V, Y)
    st = akm._lib.akm_kernel_cross_mvm(plan.handle, 201, None, 1, 1, None, 1, None)
    assert st == akm.AKM_ERR_INVALID_ARG
    # n_src == n: nothing to compute, OK
    assert akm._lib.akm_kernel_cross_mvm(plan.handle, 200, V.data_ptr(), 1, 1, None, 1, None) == akm.AKM_OK
    plan.close()


def test_cross_full_size_x4_row_sample(akm):
    """x4 at full size (1e6 sources -> 1e5 targets, r = 11): seeded target rows vs the oracle."""
    wl = workloads.CONFIGS["x4"]
    n_src = wl.extra["n_src"]
    X = workloads.make_X(wl)
    V = workloads.make_V(wl, n=n_src)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    got = gpu_cross(akm, X, n_src, wl.windows, wl.family, theta, V)
    rows = workloads.make_rows(wl, 64, n=wl.n - n_src)
    # the C dense oracle on the union with zero-padded V (equal to dense_cross by
    # tests/test_oracle_cross.py), row-sampled at the targets
    Vu = np.vstack([V, np.zeros((wl.n - n_src, wl.r))])
    want = dense_apply(X, wl.windows, wl.family, theta, Vu, rows=n_src + rows, ops=("K",))["K"]
    assert rel(got[rows], want) <= 1e-6


def test_square_products_unchanged_after_a_cross_split(akm):
    """A cross call re-sorts the plan's points (sources, then targets, inside every bin); the square
    products on the same plan must stay within the same tolerance, before and after."""
    wl = workloads.CONFIGS["c2"]
    X = workloads.make_X(wl, n=4000)
    V = workloads.make_V(wl, n=4000, r=2)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, 2.0, wl.m, 1.0 / 16)
    plan.set_theta(*theta)
    Vd = torch.from_numpy(V).to(dev)
    Y0 = torch.empty_like(Vd)
    plan.mvm(Vd, Y0)
    Yt = torch.empty((1000, 2), dtype=torch.float64, device=dev)
    plan.cross_mvm(3000, Vd[:3000].contiguous(), Yt)
    Y1 = torch.empty_like(Vd)
    plan.mvm(Vd, Y1)
    torch.cuda.synchronize()
    want = dense_apply(X, wl.windows, wl.family, theta, V, ops=("K",))["K"]
    assert rel(Y0.cpu().numpy(), want) <= 1e-6 and rel(Y1.cpu().numpy(), want) <= 1e-6
    assert rel(Yt.cpu().numpy(), dense_cross(X[:3000], X[3000:], wl.windows, wl.family, theta, V[:3000])) <= 1e-6
    # a different split, then the first again
    plan.cross_mvm(2000, Vd[:2000].contiguous(), torch.empty((2000, 2), dtype=torch.float64, device=dev))
    plan.cross_mvm(3000, Vd[:3000].contiguous(), Yt)
    torch.cuda.synchronize()
    assert rel(Yt.cpu().numpy(), dense_cross(X[:3000], X[3000:], wl.windows, wl.family, theta, V[:3000])) <= 1e-6
    plan.close()


@pytest.mark.parametrize("family", [0, 1])
def test_cross_mixed_window_dims(akm, family):
    """windows of 1, 2 and 3 features in one plan (three groups, three kernel paths)."""
    rng = np.random.default_rng(41)
    X = rng.random((2600, 6))
    windows = [(0,), (1, 2), (3, 4, 5)]
    theta = (1.1, 0.7 if family == 1 else 0.25, 0.2)
    V = rng.standard_normal((2000, 3))
    N, m = (128, 8) if family == 1 else (32, 6)   # Matern: the method needs N = 128 for 1e-3 (cf. test_gpu_parity)
    got = gpu_cross(akm, X, 2000, windows, family, theta, V, N=N, m=m)
    want = dense_cross(X[:2000], X[2000:], windows, family, theta, V)
    assert rel(got, want) <= (1e-3 if family == 1 else 1e-6)


def test_cross_strided_blocks(akm):
    """V and Yt as column slices of wider row-major blocks (ld > r), device and host."""
    wl = workloads.CONFIGS["c2"]
    X = workloads.make_X(wl, n=3000)
    theta = (wl.sigma_f, wl.ell, wl.sigma_eps)
    Vw = workloads.make_V(wl, n=2200, r=5)
    want = dense_cross(X[:2200], X[2200:], wl.windows, wl.family, theta, Vw[:, 1:4])
    dev = torch.device("cuda:0")
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(X).to(dev), wl.windows, wl.family, wl.N, 2.0, wl.m, 1.0 / 16)
    plan.set_theta(*theta)
    Vd = torch.from_numpy(Vw).to(dev)
    Yw = torch.full((800, 7), float("nan"), dtype=torch.float64, device=dev)
    plan.cross_mvm(2200, Vd[:, 1:4], Yw[:, 2:5])
    torch.cuda.synchronize()
    Yh = Yw.cpu().numpy()
    assert rel(Yh[:, 2:5], want) <= 1e-6
    assert np.isnan(Yh[:, :2]).all() and np.isnan(Yh[:, 5:]).all()   # untouched columns
    Yhost = np.full((800, 6), np.nan)
    plan.cross_mvm(2200, Vw[:, 1:4], Yhost[:, 1:4])
    assert rel(Yhost[:, 1:4], want) <= 1e-6 and np.isnan(Yhost[:, 0]).all() and np.isnan(Yhost[:, 4:]).all()
    plan.close()


def test_cross_2d_windows_past_the_small_launch_threshold(akm):
    """2-D windows at sizes where the strip kernels run (spreading over the class-0 sources only,
    interpolation at the class-1 targets only; > 2 x 148 per-bin items, so not the per-point
    small-launch path), Gaussian windows (method error ~1e-15 here, so the 1e-6 gate tests the
    implementation), 11 RHS, two length scales: against the dense cross oracle on 512 sampled target
    rows."""
    rng = np.random.default_rng(77)
    n_src, n_t = 30000, 12000
    X = rng.random((n_src + n_t, 4))
    V = rng.standard_normal((n_src, 11))
    rows = np.sort(rng.choice(n_t, 512, replace=False))
    for ell in (0.3, 0.15):
        theta = (1.0, ell, 0.1)
        got = gpu_cross(akm, X, n_src, [(0, 1), (2, 3)], 0, theta, V, N=64, m=8)
        want = dense_cross(X[:n_src], X[n_src:][rows], [(0, 1), (2, 3)], 0, theta, V)
        assert rel(got[rows], want) <= 1e-6, (ell, rel(got[rows], want))
