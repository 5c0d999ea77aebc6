"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/akm.h declares,
the Python binding mirrors them, and calls fail cleanly without a GPU.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "akm.h")


def _declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(akm_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2504_00480_b200 as akm
    return ctypes.CDLL(akm.LIB_PATH), akm


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for s in ("akm_create", "akm_set_points", "akm_set_theta", "akm_kernel_mvm", "akm_kernel_deriv_mvm",
              "akm_kernel_mvm_multi", "akm_get_info", "akm_destroy", "akm_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    cdll, akm = lib
    for s in _declared_symbols():
        assert hasattr(cdll, s), s
        assert s in akm.ABI_SYMBOLS, s
        assert hasattr(akm, s), s


def test_info_struct_matches_header_fields(lib):
    _, akm = lib
    text = open(HEADER).read()
    body = text[text.index("typedef struct {"):text.index("} akm_info;")]
    names = re.findall(r"\b([a-z_0-9]+)(?:\[[A-Z_0-9]+\])*(?:\[3\])?;", body)
    fields = [f[0] for f in akm.akm_info._fields_]
    flat = []
    for line in body.splitlines():
        line = line.split("/*")[0]
        m = re.match(r"\s*(int64_t|int32_t|double)\s+(.*);", line)
        if m:
            flat += [v.strip().split("[")[0] for v in m.group(2).split(",")]
    assert flat == fields, (flat, fields)
    assert names  # parsed something


def test_version_and_no_gpu_errors(lib):
    _, akm = lib
    assert "sm_100a" in akm.akm_version()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present: the no-device error path is not observable")
    with pytest.raises(akm.AkmError) as ei:
        akm.akm_create(0)
    assert ei.value.status == akm.AKM_ERR_CUDA


def test_null_plan_is_rejected(lib):
    cdll, akm = lib
    assert akm._lib.akm_set_theta(None, 1.0, 1.0, 0.1, None) == akm.AKM_ERR_INVALID_ARG
    assert akm._lib.akm_kernel_mvm(None, None, 1, 1, None, 1, None) == akm.AKM_ERR_INVALID_ARG
    akm._lib.akm_destroy(None)  # no-op


def test_objective_struct_matches_header_fields(lib):
    _, akm = lib
    text = open(HEADER).read()
    end = text.index("} akm_objective_out;")
    body = text[text.rindex("typedef struct {", 0, end):end]
    flat = []
    for line in body.splitlines():
        line = line.split("/*")[0]
        m = re.match(r"\s*(int64_t|int32_t|double)\s+(.*);", line)
        if m:
            flat += [v.strip().split("[")[0] for v in m.group(2).split(",")]
    assert flat == [f[0] for f in akm.akm_objective_out._fields_]
    assert "#define AKM_MAX_PROBES %d" % akm.AKM_MAX_PROBES in text


def test_binding_rejects_mismatched_row_counts(lib):
    """The C side reads / writes exactly the plan's n rows (n - n_src for the cross product); the
    binding rejects blocks of another height before any pointer crosses the ABI."""
    import numpy as np
    _, akm = lib
    fake = ctypes.c_void_p(0xABC0)
    akm._ROWS[fake.value] = 10
    try:
        for call in (lambda: akm.akm_kernel_mvm(fake, np.zeros((9, 2)), np.zeros((9, 2))),
                     lambda: akm.akm_kernel_mvm(fake, np.zeros((10, 2)), np.zeros((9, 2))),
                     lambda: akm.akm_kernel_mvm_multi(fake, np.zeros((10, 2)), Y=np.zeros((10, 1))),
                     lambda: akm.akm_kernel_deriv_mvm(fake, 0, np.zeros((11, 1)), np.zeros((11, 1))),
                     lambda: akm.akm_kernel_cross_mvm(fake, 4, np.zeros((4, 1)), np.zeros((5, 1))),
                     lambda: akm.akm_objective_diag(fake, np.zeros(9), np.zeros((9, 2))),
                     lambda: akm.akm_gradient_diag(fake, np.zeros(10), np.zeros((8, 2)))):
            with pytest.raises(ValueError):
                call()
    finally:
        akm._ROWS.pop(fake.value, None)


def test_binding_makes_strided_vectors_contiguous(lib):
    """A strided column (e.g. V[:, 0]) passed as y is copied to contiguous memory: the C ABI reads n
    consecutive doubles."""
    import numpy as np
    _, akm = lib
    V = np.arange(30.0).reshape(10, 3)
    y = akm._vector(V[:, 1], "y")
    assert y.flags["C_CONTIGUOUS"] and np.array_equal(y, V[:, 1])
    torch = pytest.importorskip("torch")
    t = torch.arange(30.0, dtype=torch.float64).reshape(10, 3)
    yt = akm._vector(t[:, 2], "y")
    assert yt.is_contiguous() and torch.equal(yt, t[:, 2])
    with pytest.raises(ValueError):
        akm._vector(np.zeros((4, 2)), "y")
