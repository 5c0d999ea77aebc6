"""Streaming host batches (include/akm.h akm_kernel_mvm_pipelined / akm_pipeline_wait): a sequence
of independent products from pinned host blocks, the copies of neighbouring batches overlapping the
products, gives exactly what the synchronous call gives for each batch -- in deterministic mode
(akm_set_deterministic) bitwise -- and the outputs are complete after pipeline_wait + a sync.
Also the ragged cases: a change of r between calls (slots regrow), strided host blocks, n = 0, and
the argument checks (pageable buffers are rejected)."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def akm():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as mod
    return mod


def _plan(akm, name, n, det=True):
    wl = workloads.CONFIGS[name]
    X = workloads.make_X(wl, n=n)
    plan = akm.Plan(0)
    plan.set_points(torch.from_numpy(np.ascontiguousarray(X)).cuda(), wl.windows, wl.family, wl.N, wl.sigma_over,
                    wl.m, wl.eps_B)
    plan.set_theta(wl.sigma_f, wl.ell, wl.sigma_eps)
    if det:
        plan.set_deterministic(True)
    return wl, plan


def _sync_products(plan, V, ops):
    outs = {op: np.zeros_like(V) for op in ops}
    plan.mvm_multi(V, Y=outs.get("K"), dY_ell=outs.get("dell"), dY_sf=outs.get("dsf"))
    return outs


@pytest.mark.parametrize("split", ["0", "1000000000"])   # copy streams / the caller's stream
@pytest.mark.parametrize("name,n,r", [("c4", 20000, 11), ("c2", 6000, 1), ("c3", 8000, 3)])
def test_pipelined_batches_equal_synchronous_calls(akm, monkeypatch, split, name, n, r):
    monkeypatch.setenv("AKM_PIPE_SPLIT_MIN_BYTES", split)
    wl, plan = _plan(akm, name, n)
    ops = ("K", "dell", "dsf")
    rng = np.random.default_rng(7)
    batches = [rng.standard_normal((n, r)) for _ in range(5)]
    ref = [_sync_products(plan, V, ops) for V in batches]
    stream = torch.cuda.Stream()
    Vh = [torch.from_numpy(V).pin_memory() for V in batches]
    Oh = [{op: torch.full((n, r), np.nan, dtype=torch.float64).pin_memory() for op in ops} for _ in batches]
    with torch.cuda.stream(stream):
        for k in range(len(batches)):
            plan.mvm_pipelined(Vh[k], Y=Oh[k]["K"], dY_ell=Oh[k]["dell"], dY_sf=Oh[k]["dsf"],
                               stream=stream.cuda_stream)
        plan.pipeline_wait(stream=stream.cuda_stream)
    stream.synchronize()
    for k in range(len(batches)):
        for op in ops:
            assert np.array_equal(Oh[k][op].numpy(), ref[k][op]), (k, op)
    plan.close()


def test_pipelined_default_mode_rhs_change_and_strided_blocks(akm, monkeypatch):
    # 8 bytes x 6000 rows x r: r = 1, 2 stay on the caller's stream, r = 5 goes through the copy
    # streams, so the mixed sequence crosses both modes on the same slots
    monkeypatch.setenv("AKM_PIPE_SPLIT_MIN_BYTES", str(8 * 6000 * 3))
    n = 6000
    wl, plan = _plan(akm, "c1", n, det=False)
    rng = np.random.default_rng(11)
    stream = torch.cuda.Stream()
    Vs = [rng.standard_normal((n, r)) for r in (2, 5, 1, 5)]   # slots regrow when r grows
    refs = [_sync_products(plan, V, ("K",))["K"] for V in Vs]  # (all before the pipelined calls: one
    results = []                                               # plan is ordered on one stream at a time)
    for V, ref in zip(Vs, refs):
        r = V.shape[1]
        Vbig = torch.zeros(n, r + 3, dtype=torch.float64).pin_memory()
        Vbig[:, 1:1 + r] = torch.from_numpy(V)
        Ybig = torch.full((n, r + 2), 7.0, dtype=torch.float64).pin_memory()
        plan.mvm_pipelined(Vbig[:, 1:1 + r], Y=Ybig[:, :r], stream=stream.cuda_stream)
        results.append((ref, Ybig, r))
    plan.pipeline_wait(stream=stream.cuda_stream)
    stream.synchronize()
    for ref, Ybig, r in results:
        Y = Ybig.numpy()
        assert np.max(np.abs(Y[:, :r] - ref)) <= 1e-13 * np.max(np.abs(ref))
        assert np.all(Y[:, r:] == 7.0)
    plan.close()


def test_pipelined_argument_checks(akm):
    n = 500
    wl, plan = _plan(akm, "c1", n, det=False)
    V = np.ones((n, 2))
    with pytest.raises(akm.AkmError):   # pageable host memory
        plan.mvm_pipelined(V, Y=np.zeros_like(V))
    Vp = torch.ones(n, 2, dtype=torch.float64).pin_memory()
    with pytest.raises(akm.AkmError):   # device output
        plan.mvm_pipelined(Vp, Y=torch.zeros(n, 2, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):     # wrong row count
        plan.mvm_pipelined(torch.ones(n - 1, 2, dtype=torch.float64).pin_memory(),
                           Y=torch.zeros(n - 1, 2, dtype=torch.float64).pin_memory())
    plan.pipeline_wait()                # no pipelined call on a fresh plan stream: a no-op
    plan.close()
