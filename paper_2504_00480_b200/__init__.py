"""paper_2504_00480_b200 -- B200-native additive-kernel MVM by NFFT fast summation (arXiv 2504.00480).

Thin Python binding of the C ABI in ``include/akm.h`` (``libakm.so``, built in-tree for
sm_100a by ``_build.py`` / ``__graft_entry__.build()``).  This module only marshals arguments:
every step of the product runs in the library's CUDA kernels.  There is no CPU fallback -- if
the shared library is missing, importing the package raises ``ImportError``.

Module-level functions carry the C names (``akm_create``, ``akm_set_points``, ``akm_set_theta``,
``akm_kernel_mvm``, ``akm_kernel_deriv_mvm``, ``akm_kernel_mvm_multi``, ``akm_get_info``,
``akm_set_scale_override``, ``akm_last_error``, ``akm_destroy``); ``Plan`` wraps them with
tensor-friendly signatures.  Arrays may be CUDA torch tensors (device pointers, the caller's
current stream is used) or host numpy arrays / CPU tensors (the library stages them).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libakm.so")

AKM_OK, AKM_ERR_INVALID_ARG, AKM_ERR_NONFINITE, AKM_ERR_STATE, AKM_ERR_OOM, AKM_ERR_CUDA, AKM_ERR_UNSUPPORTED = range(7)
STATUS_NAMES = {0: "AKM_OK", 1: "AKM_ERR_INVALID_ARG", 2: "AKM_ERR_NONFINITE", 3: "AKM_ERR_STATE", 4: "AKM_ERR_OOM",
                5: "AKM_ERR_CUDA", 6: "AKM_ERR_UNSUPPORTED"}
AKM_GAUSSIAN, AKM_MATERN12 = 0, 1
AKM_D_ELL, AKM_D_SIGMA_F, AKM_D_SIGMA_EPS = 0, 1, 2
AKM_MAX_WINDOWS = 32

# names exported by include/akm.h (checked by tests/test_abi_cpu.py)
ABI_SYMBOLS = ("akm_create", "akm_set_points", "akm_set_theta", "akm_kernel_mvm", "akm_kernel_deriv_mvm",
               "akm_kernel_mvm_multi", "akm_get_info", "akm_set_scale_override", "akm_last_error", "akm_destroy",
               "akm_version", "akm_set_profiling", "akm_get_stage_times", "akm_objective_diag",
               "akm_kernel_cross_mvm", "akm_gradient_diag", "akm_get_window_poly",
               "akm_get_bounds", "akm_set_bounds", "akm_set_radius", "akm_set_bin_override", "akm_grid_size",
               "akm_spread_grid", "akm_mvm_from_grid", "akm_set_regularization", "akm_set_preconditioner",
               "akm_precond_apply", "akm_precond_landmarks", "akm_objective", "akm_gradient",
               "akm_gradient_columns", "akm_set_deterministic", "akm_kernel_mvm_pipelined", "akm_pipeline_wait")
AKM_MAX_PROBES = 31


class akm_info(ctypes.Structure):
    W = AKM_MAX_WINDOWS
    _fields_ = [
        ("n", ctypes.c_int64),
        ("p", ctypes.c_int32), ("P", ctypes.c_int32), ("N", ctypes.c_int32), ("m", ctypes.c_int32),
        ("n_g", ctypes.c_int32), ("family", ctypes.c_int32),
        ("sigma_f", ctypes.c_double), ("ell", ctypes.c_double), ("sigma_eps", ctypes.c_double),
        ("d", ctypes.c_int32 * W),
        ("c_w", ctypes.c_double * W),
        ("ell_eff", ctypes.c_double * W),
        ("radius", ctypes.c_double * W),
        ("box", (ctypes.c_int32 * 3) * W),
        ("bin", ctypes.c_int32 * W),
        ("occupied_bins", ctypes.c_int64 * W),
        ("max_bin_points", ctypes.c_int64 * W),
        ("work_items_spread", ctypes.c_int64),
        ("work_items_interp", ctypes.c_int64),
        ("workspace_bytes", ctypes.c_int64),
    ]


class akm_stage_times(ctypes.Structure):
    _fields_ = [("spread_ms", ctypes.c_double), ("fft_ms", ctypes.c_double), ("interp_ms", ctypes.c_double),
                ("epilogue_ms", ctypes.c_double), ("exchange_ms", ctypes.c_double), ("calls", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("spread_launches", ctypes.c_int64), ("interp_launches", ctypes.c_int64)]


class akm_objective_out(ctypes.Structure):
    _fields_ = [("Z", ctypes.c_double), ("quad", ctypes.c_double), ("logdet_M", ctypes.c_double),
                ("slq", ctypes.c_double), ("n_log_2pi", ctypes.c_double),
                ("samples", ctypes.c_double * AKM_MAX_PROBES), ("steps", ctypes.c_int32 * AKM_MAX_PROBES),
                ("n_z", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("lanczos_steps", ctypes.c_int32),
                ("products", ctypes.c_int32), ("cg_relres", ctypes.c_double), ("cg_relres_true", ctypes.c_double),
                ("landmarks", ctypes.c_int32), ("product_columns", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    st = ctypes.c_int
    lib.akm_create.argtypes = [ctypes.POINTER(P), ctypes.c_int]
    lib.akm_create.restype = st
    lib.akm_set_points.argtypes = [P, P, i64, i32, i64, P, P, i32, i32, i32, d, i32, d, P]
    lib.akm_set_points.restype = st
    lib.akm_set_theta.argtypes = [P, d, d, d, P]
    lib.akm_set_theta.restype = st
    lib.akm_kernel_mvm.argtypes = [P, P, i64, i32, P, i64, P]
    lib.akm_kernel_mvm.restype = st
    lib.akm_kernel_deriv_mvm.argtypes = [P, i32, P, i64, i32, P, i64, P]
    lib.akm_kernel_deriv_mvm.restype = st
    lib.akm_kernel_mvm_multi.argtypes = [P, P, i64, i32, P, P, P, i64, P]
    lib.akm_kernel_mvm_multi.restype = st
    lib.akm_kernel_mvm_pipelined.argtypes = [P, P, i64, i32, P, P, P, i64, P]
    lib.akm_kernel_mvm_pipelined.restype = st
    lib.akm_pipeline_wait.argtypes = [P, P]
    lib.akm_pipeline_wait.restype = st
    lib.akm_kernel_cross_mvm.argtypes = [P, i64, P, i64, i32, P, i64, P]
    lib.akm_kernel_cross_mvm.restype = st
    lib.akm_gradient_diag.argtypes = [P, P, P, i64, i32, i32, P, P, P]
    lib.akm_gradient_diag.restype = st
    lib.akm_get_info.argtypes = [P, ctypes.POINTER(akm_info)]
    lib.akm_get_info.restype = st
    lib.akm_set_scale_override.argtypes = [P, P]
    lib.akm_set_scale_override.restype = st
    lib.akm_last_error.argtypes = [P]
    lib.akm_last_error.restype = ctypes.c_char_p
    lib.akm_destroy.argtypes = [P]
    lib.akm_destroy.restype = None
    lib.akm_set_profiling.argtypes = [P, i32]
    lib.akm_set_profiling.restype = st
    lib.akm_get_stage_times.argtypes = [P, ctypes.POINTER(akm_stage_times), i32]
    lib.akm_get_stage_times.restype = st
    lib.akm_objective_diag.argtypes = [P, P, P, i64, i32, i32, i32, ctypes.POINTER(akm_objective_out), P, P]
    lib.akm_objective_diag.restype = st
    lib.akm_get_window_poly.argtypes = [P, P, P, P]
    lib.akm_get_window_poly.restype = st
    lib.akm_get_bounds.argtypes = [P, P, P]
    lib.akm_get_bounds.restype = st
    lib.akm_set_bounds.argtypes = [P, P, P, P, P]
    lib.akm_set_bounds.restype = st
    lib.akm_set_radius.argtypes = [P, P]
    lib.akm_set_radius.restype = st
    lib.akm_set_bin_override.argtypes = [P, P]
    lib.akm_set_bin_override.restype = st
    lib.akm_grid_size.argtypes = [P, i32, ctypes.POINTER(i64)]
    lib.akm_grid_size.restype = st
    lib.akm_spread_grid.argtypes = [P, P, i64, i32, P, P]
    lib.akm_spread_grid.restype = st
    lib.akm_mvm_from_grid.argtypes = [P, P, P, i64, i32, P, P, P, i64, P]
    lib.akm_mvm_from_grid.restype = st
    lib.akm_set_regularization.argtypes = [P, d, i32]
    lib.akm_set_regularization.restype = st
    lib.akm_set_deterministic.argtypes = [P, i32]
    lib.akm_set_deterministic.restype = st
    lib.akm_set_preconditioner.argtypes = [P, i32]
    lib.akm_set_preconditioner.restype = st
    lib.akm_precond_apply.argtypes = [P, i32, P, i32, P, P, P, P]
    lib.akm_precond_apply.restype = st
    lib.akm_precond_landmarks.argtypes = [P, P, P]
    lib.akm_precond_landmarks.restype = st
    lib.akm_objective.argtypes = [P, P, P, i64, i32, i32, i32, ctypes.POINTER(akm_objective_out), P, P]
    lib.akm_objective.restype = st
    lib.akm_gradient.argtypes = [P, P, P, i64, i32, i32, P, P, P]
    lib.akm_gradient.restype = st
    lib.akm_gradient_columns.argtypes = [P, P, P, i64, i32, i32, i32, P, P, P, P]
    lib.akm_gradient_columns.restype = st
    lib.akm_version.argtypes = []
    lib.akm_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


class AkmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# ---------------------------------------------------------------- argument marshalling
def _ptr_ld(a, name):
    """(pointer, leading dimension, rows, cols, is_cuda_tensor, keepalive) of a 2-D float64 array."""
    if a is None:
        return None, 0, 0, 0, False, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise TypeError(f"{name} must be float64")
            if a.dim() == 1:
                a = a.unsqueeze(1)
            if a.dim() == 2 and a.numel() == 0:  # empty blocks carry no strides (torch reports 0)
                return ctypes.c_void_p(a.data_ptr()), max(1, a.shape[1]), a.shape[0], a.shape[1], a.is_cuda, a
            if a.dim() != 2 or (a.stride(1) != 1 and a.shape[1] > 1):
                raise ValueError(f"{name} must be 2-D with unit column stride")
            ld = a.stride(0) if a.shape[0] > 1 else a.shape[1]
            return ctypes.c_void_p(a.data_ptr()), max(ld, a.shape[1]), a.shape[0], a.shape[1], a.is_cuda, a
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(a)
    if arr.dtype != np.float64:
        raise TypeError(f"{name} must be float64")
    if arr.ndim == 1:
        arr = arr[:, None]
    if arr.ndim == 2 and arr.size == 0:
        return ctypes.c_void_p(arr.ctypes.data), max(1, arr.shape[1]), arr.shape[0], arr.shape[1], False, arr
    if arr.ndim != 2 or (arr.strides[1] != 8 and arr.shape[1] > 1):
        raise ValueError(f"{name} must be 2-D row-major")
    ld = arr.strides[0] // 8 if arr.shape[0] > 1 else arr.shape[1]
    return ctypes.c_void_p(arr.ctypes.data), max(ld, arr.shape[1]), arr.shape[0], arr.shape[1], False, arr


def _stream(stream, *tensors):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    for t in tensors:
        if t is not None and getattr(t, "is_cuda", False):
            import torch
            return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    return ctypes.c_void_p(0)


# rows n of the last successful akm_set_points per plan handle: the C side reads and writes exactly
# n rows of every block (n - n_src target rows for the cross product), so mismatched tensors are
# rejected here before any pointer crosses the ABI
_ROWS = {}


def _expect_rows(plan, name, rows, want=None):
    if want is None:
        want = _ROWS.get(getattr(plan, "value", plan))
    if want is not None and rows != want:
        raise ValueError(f"{name} has {rows} rows; the plan expects {want}")


def _vector(a, name):
    """A 1-D float64 vector (or n x 1 block) made contiguous: the C ABI reads n consecutive doubles."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dim() == 2 and a.shape[1] == 1:
                a = a[:, 0]
            if a.dim() != 1:
                raise ValueError(f"{name} must be a vector")
            return a.contiguous()
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(a)
    if arr.ndim == 2 and arr.shape[1] == 1:
        arr = arr[:, 0]
    if arr.ndim != 1:
        raise ValueError(f"{name} must be a vector")
    return np.ascontiguousarray(arr)


def _check(plan, status):
    if status != AKM_OK:
        msg = _lib.akm_last_error(plan).decode() if plan else ""
        raise AkmError(status, msg)


# ---------------------------------------------------------------- C-named functions
def akm_version() -> str:
    return _lib.akm_version().decode()


def akm_create(device: int = 0):
    h = ctypes.c_void_p()
    st = _lib.akm_create(ctypes.byref(h), int(device))
    if st != AKM_OK:
        raise AkmError(st, f"akm_create(device={device}) failed")
    return h


def akm_destroy(plan) -> None:
    _ROWS.pop(getattr(plan, "value", plan), None)
    _lib.akm_destroy(plan)


def akm_last_error(plan) -> str:
    return _lib.akm_last_error(plan).decode()


def akm_set_points(plan, X, windows, family, N, sigma_over, m, eps_B, stream=None):
    px, ldx, n, p, _, keep = _ptr_ld(X, "X")
    feat = np.ascontiguousarray([f for w in windows for f in w], dtype=np.int32)
    lens = np.ascontiguousarray([len(w) for w in windows], dtype=np.int32)
    st = _lib.akm_set_points(plan, px, n, p, ldx, feat.ctypes.data_as(ctypes.c_void_p),
                             lens.ctypes.data_as(ctypes.c_void_p), len(windows), int(family), int(N),
                             float(sigma_over), int(m), float(eps_B), _stream(stream, keep))
    _ROWS.pop(getattr(plan, "value", plan), None)
    _check(plan, st)
    _ROWS[getattr(plan, "value", plan)] = n


def akm_set_theta(plan, sigma_f, ell, sigma_eps, stream=None):
    _check(plan, _lib.akm_set_theta(plan, float(sigma_f), float(ell), float(sigma_eps), _stream(stream)))


def _same_block(plan, V, outs):
    """Marshal V and the outputs of a square product: every block n x r with the plan's n."""
    pv, ldv, n, r, _, kv = _ptr_ld(V, "V")
    _expect_rows(plan, "V", n)
    res = []
    for name, o in outs:
        m = _ptr_ld(o, name)
        if o is not None and (m[2] != n or m[3] != r):
            raise ValueError(f"{name} must be {n} x {r} like V (got {m[2]} x {m[3]})")
        res.append(m)
    return (pv, ldv, n, r, kv), res


def akm_kernel_mvm(plan, V, Y, stream=None):
    (pv, ldv, n, r, kv), [(py, ldy, _, _, _, ky)] = _same_block(plan, V, [("Y", Y)])
    _check(plan, _lib.akm_kernel_mvm(plan, pv, ldv, r, py, ldy, _stream(stream, kv, ky)))


def akm_kernel_deriv_mvm(plan, which, V, dY, stream=None):
    (pv, ldv, n, r, kv), [(py, ldy, _, _, _, ky)] = _same_block(plan, V, [("dY", dY)])
    _check(plan, _lib.akm_kernel_deriv_mvm(plan, int(which), pv, ldv, r, py, ldy, _stream(stream, kv, ky)))


def akm_kernel_mvm_multi(plan, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
    (pv, ldv, n, r, kv), outs = _same_block(plan, V, [("Y", Y), ("dY_ell", dY_ell), ("dY_sf", dY_sf)])
    lds = {o[1] for o in outs if o[0] is not None}
    if len(lds) > 1:
        raise ValueError("all outputs of akm_kernel_mvm_multi must share one leading dimension")
    ldy = lds.pop() if lds else r
    _check(plan, _lib.akm_kernel_mvm_multi(plan, pv, ldv, r, outs[0][0], outs[1][0], outs[2][0], ldy,
                                           _stream(stream, kv, *[o[5] for o in outs])))


def akm_kernel_mvm_pipelined(plan, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
    """Streaming host batches (include/akm.h): V and the outputs are pinned host blocks; the call only
    enqueues, and the outputs are complete after akm_pipeline_wait(plan, stream) and a sync."""
    (pv, ldv, n, r, kv), outs = _same_block(plan, V, [("Y", Y), ("dY_ell", dY_ell), ("dY_sf", dY_sf)])
    lds = {o[1] for o in outs if o[0] is not None}
    if len(lds) > 1:
        raise ValueError("all outputs of akm_kernel_mvm_pipelined must share one leading dimension")
    ldy = lds.pop() if lds else r
    _check(plan, _lib.akm_kernel_mvm_pipelined(plan, pv, ldv, r, outs[0][0], outs[1][0], outs[2][0], ldy,
                                               _stream(stream, kv, *[o[5] for o in outs])))


def akm_pipeline_wait(plan, stream=None):
    _check(plan, _lib.akm_pipeline_wait(plan, _stream(stream)))


def akm_kernel_cross_mvm(plan, n_src, V, Yt, stream=None):
    """Yt = sigma_f^2 sum_w K_w(X_t, X_s) V; the plan's points are [X_s (n_src rows); X_t]."""
    pv, ldv, nv, r, _, kv = _ptr_ld(V, "V")
    py, ldy, _, ry, _, ky = _ptr_ld(Yt, "Yt")
    if nv != n_src or (Yt is not None and ry != r):
        raise ValueError(f"V must have n_src = {n_src} rows and Yt the same number of columns ({r})")
    n_all = _ROWS.get(getattr(plan, "value", plan))
    if n_all is not None and Yt is not None:
        _expect_rows(plan, "Yt", _ptr_ld(Yt, "Yt")[2], n_all - int(n_src))
    _check(plan, _lib.akm_kernel_cross_mvm(plan, int(n_src), pv, ldv, r, py, ldy, _stream(stream, kv, ky)))


def akm_get_info(plan) -> dict:
    info = akm_info()
    _check(plan, _lib.akm_get_info(plan, ctypes.byref(info)))
    P = info.P
    return {
        "n": info.n, "p": info.p, "P": P, "N": info.N, "m": info.m, "n_g": info.n_g, "family": info.family,
        "theta": (info.sigma_f, info.ell, info.sigma_eps),
        "d": list(info.d[:P]), "c_w": list(info.c_w[:P]), "ell_eff": list(info.ell_eff[:P]),
        "radius": list(info.radius[:P]), "box": [tuple(info.box[w]) for w in range(P)], "bin": list(info.bin[:P]),
        "occupied_bins": list(info.occupied_bins[:P]), "max_bin_points": list(info.max_bin_points[:P]),
        "work_items_spread": info.work_items_spread, "work_items_interp": info.work_items_interp,
        "workspace_bytes": info.workspace_bytes,
    }


def akm_set_scale_override(plan, c_w=None):
    if c_w is None:
        _check(plan, _lib.akm_set_scale_override(plan, None))
    else:
        arr = np.ascontiguousarray(c_w, dtype=np.float64)
        _check(plan, _lib.akm_set_scale_override(plan, arr.ctypes.data_as(ctypes.c_void_p)))


def akm_get_window_poly(plan):
    """(coefficients (2m, degree + 1), taps, degree) of the window polynomials the kernels evaluate."""
    coef = np.zeros(16 * 15, dtype=np.float64)
    taps, deg = ctypes.c_int32(), ctypes.c_int32()
    _check(plan, _lib.akm_get_window_poly(plan, coef.ctypes.data_as(ctypes.c_void_p), ctypes.byref(taps),
                                          ctypes.byref(deg)))
    return coef[:taps.value * (deg.value + 1)].reshape(taps.value, deg.value + 1), taps.value, deg.value


def akm_get_bounds(plan):
    """(lo, hi) of this plan's points per window and padded axis, arrays of shape (P, 3)."""
    P = akm_get_info(plan)["P"]
    lo, hi = np.zeros(3 * P), np.zeros(3 * P)
    _check(plan, _lib.akm_get_bounds(plan, lo.ctypes.data_as(ctypes.c_void_p), hi.ctypes.data_as(ctypes.c_void_p)))
    return lo.reshape(P, 3), hi.reshape(P, 3)


def akm_set_bounds(plan, lo, hi, stream=None):
    """Adopt the union's bounding box; returns this plan's radius per window about the new centers."""
    lo = np.ascontiguousarray(lo, dtype=np.float64).reshape(-1)
    hi = np.ascontiguousarray(hi, dtype=np.float64).reshape(-1)
    rad = np.zeros(lo.size // 3)
    _check(plan, _lib.akm_set_bounds(plan, lo.ctypes.data_as(ctypes.c_void_p), hi.ctypes.data_as(ctypes.c_void_p),
                                     rad.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
    return rad


def akm_set_radius(plan, radius):
    rad = np.ascontiguousarray(radius, dtype=np.float64)
    _check(plan, _lib.akm_set_radius(plan, rad.ctypes.data_as(ctypes.c_void_p)))


def akm_set_bin_override(plan, bins=None):
    if bins is None:
        _check(plan, _lib.akm_set_bin_override(plan, None))
    else:
        b = np.ascontiguousarray(bins, dtype=np.int32)
        _check(plan, _lib.akm_set_bin_override(plan, b.ctypes.data_as(ctypes.c_void_p)))


def akm_grid_size(plan, r) -> int:
    c = ctypes.c_int64()
    _check(plan, _lib.akm_grid_size(plan, int(r), ctypes.byref(c)))
    return c.value


def akm_spread_grid(plan, V, grid, stream=None):
    pv, ldv, n, r, _, kv = _ptr_ld(V, "V")
    _expect_rows(plan, "V", n)
    if grid.numel() < akm_grid_size(plan, r):
        raise ValueError("grid is smaller than akm_grid_size(r)")
    _check(plan, _lib.akm_spread_grid(plan, pv, ldv, r, ctypes.c_void_p(grid.data_ptr()), _stream(stream, kv, grid)))


def akm_mvm_from_grid(plan, grid, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
    (pv, ldv, n, r, kv), outs = _same_block(plan, V, [("Y", Y), ("dY_ell", dY_ell), ("dY_sf", dY_sf)])
    lds = {o[1] for o in outs if o[0] is not None}
    if len(lds) > 1:
        raise ValueError("all outputs must share one leading dimension")
    ldy = lds.pop() if lds else r
    if grid.numel() < akm_grid_size(plan, r):
        raise ValueError("grid is smaller than akm_grid_size(r)")
    _check(plan, _lib.akm_mvm_from_grid(plan, ctypes.c_void_p(grid.data_ptr()), pv, ldv, r, outs[0][0], outs[1][0],
                                        outs[2][0], ldy, _stream(stream, kv, grid)))


def akm_set_regularization(plan, eps_I=0.0, p=0):
    """kappa_R with inner (eps_I, near-field corrected) and outer (eps_B) smoothing of order p (include/akm.h)."""
    _check(plan, _lib.akm_set_regularization(plan, float(eps_I), int(p)))


def akm_set_deterministic(plan, on: bool):
    """Bitwise run-to-run reproducible products (integer-limb spreading flushes; include/akm.h)."""
    _check(plan, _lib.akm_set_deterministic(plan, 1 if on else 0))


def akm_set_profiling(plan, enable: bool):
    _check(plan, _lib.akm_set_profiling(plan, 1 if enable else 0))


def akm_get_stage_times(plan, reset: bool = False) -> dict:
    t = akm_stage_times()
    _check(plan, _lib.akm_get_stage_times(plan, ctypes.byref(t), 1 if reset else 0))
    return {f[0]: getattr(t, f[0]) for f in akm_stage_times._fields_}


def akm_objective_diag(plan, y, Z, cg_iters=50, lanczos_steps=30, stream=None) -> dict:
    """eq. (1.4) with M = diag(Khat): CG + SLQ, every Krylov step one block product (include/akm.h)."""
    return _objective(_lib.akm_objective_diag, plan, y, Z, cg_iters, lanczos_steps, stream)


def akm_objective(plan, y, Z, cg_iters=50, lanczos_steps=30, stream=None) -> dict:
    """eq. (1.4) with the plan's preconditioner (diagonal or AAFN, akm_set_preconditioner)."""
    return _objective(_lib.akm_objective, plan, y, Z, cg_iters, lanczos_steps, stream)


def _objective(fn, plan, y, Z, cg_iters, lanczos_steps, stream) -> dict:
    y = _vector(y, "y")
    py, _, n, _, _, ky = _ptr_ld(y, "y")
    pz, ldz, nz_rows, n_z, _, kz = _ptr_ld(Z, "Z")
    _expect_rows(plan, "y", n)
    _expect_rows(plan, "Z", nz_rows)
    out = akm_objective_out()
    hist = (ctypes.c_double * max(int(cg_iters), 1))()
    _check(plan, fn(plan, py, pz, ldz, n_z, int(cg_iters), int(lanczos_steps), ctypes.byref(out), hist,
                    _stream(stream, ky, kz)))
    return {"Z": out.Z, "quad": out.quad, "logdetM": out.logdet_M, "slq": out.slq, "n_log_2pi": out.n_log_2pi,
            "samples": list(out.samples[:n_z]), "steps": list(out.steps[:n_z]), "products": out.products,
            "cg_relres": out.cg_relres, "cg_relres_true": out.cg_relres_true, "landmarks": out.landmarks,
            "product_columns": out.product_columns,
            "cg_hist": [h for h in hist[:cg_iters]]}


def akm_set_preconditioner(plan, k_per_window=0):
    """AAFN with k_per_window FPS landmarks per window (0: the diagonal preconditioner)."""
    _check(plan, _lib.akm_set_preconditioner(plan, int(k_per_window)))


def akm_precond_landmarks(plan, stream=None) -> int:
    c = ctypes.c_int32()
    _check(plan, _lib.akm_precond_landmarks(plan, ctypes.byref(c), _stream(stream)))
    return c.value


def akm_precond_apply(plan, T, out, transpose=False, stream=None):
    """out = U^{-1} T (or U^{-T} T); returns (log det M, landmark indices)."""
    pt, ldt, n, r, _, kt = _ptr_ld(T, "T")
    po, ldo, _, _, _, ko = _ptr_ld(out, "out")
    if ldt != r or ldo != r:
        raise ValueError("T and out must be contiguous n x r blocks")
    _expect_rows(plan, "T", n)
    k = akm_precond_landmarks(plan, stream)
    lm = np.zeros(max(k, 1), dtype=np.int32)
    ld = ctypes.c_double()
    _check(plan, _lib.akm_precond_apply(plan, 1 if transpose else 0, pt, r, po, ctypes.byref(ld),
                                        lm.ctypes.data_as(ctypes.c_void_p), _stream(stream, kt, ko)))
    return ld.value, lm[:k]


def akm_gradient(plan, y, Z, cg_iters=50, stream=None) -> dict:
    """Gradient of Z~ with the plan's preconditioner (AAFN: plain Hutchinson form, include/akm.h)."""
    return _gradient(_lib.akm_gradient, plan, y, Z, cg_iters, stream)


def akm_gradient_diag(plan, y, Z, cg_iters=50, stream=None) -> dict:
    """eq. (div) with M = diag(Khat): block PCG on [y | Z], one fused derivative product (include/akm.h)."""
    return _gradient(_lib.akm_gradient_diag, plan, y, Z, cg_iters, stream)


def akm_gradient_columns(plan, y, Z, cg_iters=50, preconditioned=False, stream=None) -> dict:
    """Raw per-column gradient terms (include/akm.h): dots (3, 1 + n_z) and sqnorms (1 + n_z)."""
    y = _vector(y, "y")
    py, _, n, _, _, ky = _ptr_ld(y, "y")
    pz, ldz, nz_rows, n_z, _, kz = _ptr_ld(Z, "Z")
    _expect_rows(plan, "y", n)
    _expect_rows(plan, "Z", nz_rows)
    R = 1 + n_z
    dots = np.zeros(3 * R)
    sq = np.zeros(R)
    hist = (ctypes.c_double * max(int(cg_iters), 1))()
    _check(plan, _lib.akm_gradient_columns(plan, py, pz, ldz, n_z, int(cg_iters), 1 if preconditioned else 0,
                                           dots.ctypes.data_as(ctypes.c_void_p), sq.ctypes.data_as(ctypes.c_void_p),
                                           hist, _stream(stream, ky, kz)))
    return {"dots": dots.reshape(3, R), "sqnorms": sq, "cg_hist": [h for h in hist[:cg_iters]]}


def _gradient(fn, plan, y, Z, cg_iters, stream) -> dict:
    y = _vector(y, "y")
    py, _, n, _, _, ky = _ptr_ld(y, "y")
    pz, ldz, nz_rows, n_z, _, kz = _ptr_ld(Z, "Z")
    _expect_rows(plan, "y", n)
    _expect_rows(plan, "Z", nz_rows)
    grad = (ctypes.c_double * 3)()
    hist = (ctypes.c_double * max(int(cg_iters), 1))()
    _check(plan, fn(plan, py, pz, ldz, n_z, int(cg_iters), grad, hist, _stream(stream, ky, kz)))
    return {"grad": {"sf": grad[0], "ell": grad[1], "se": grad[2]}, "cg_hist": [h for h in hist[:cg_iters]],
            "products": int(cg_iters) + 1}


# ---------------------------------------------------------------- convenience wrapper
class Plan:
    """RAII wrapper: ``Plan(device).set_points(...).set_theta(...)`` then ``mvm`` / ``deriv_mvm`` / ``mvm_multi``."""

    def __init__(self, device: int = 0):
        self.handle = akm_create(device)
        self.device = device

    def close(self):
        if self.handle is not None:
            akm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def set_points(self, X, windows, family=AKM_GAUSSIAN, N=32, sigma_over=2.0, m=6, eps_B=1.0 / 16, stream=None):
        akm_set_points(self.handle, X, windows, family, N, sigma_over, m, eps_B, stream)
        return self

    def set_theta(self, sigma_f, ell, sigma_eps, stream=None):
        akm_set_theta(self.handle, sigma_f, ell, sigma_eps, stream)
        return self

    def set_regularization(self, eps_I=0.0, p=0):
        akm_set_regularization(self.handle, eps_I, p)
        return self

    def set_deterministic(self, on=True):
        akm_set_deterministic(self.handle, on)
        return self

    def set_scale_override(self, c_w=None):
        akm_set_scale_override(self.handle, c_w)
        return self

    def mvm(self, V, Y, stream=None):
        akm_kernel_mvm(self.handle, V, Y, stream)
        return Y

    def deriv_mvm(self, which, V, dY, stream=None):
        akm_kernel_deriv_mvm(self.handle, which, V, dY, stream)
        return dY

    def mvm_multi(self, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
        akm_kernel_mvm_multi(self.handle, V, Y, dY_ell, dY_sf, stream)
        return Y, dY_ell, dY_sf

    def mvm_pipelined(self, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
        akm_kernel_mvm_pipelined(self.handle, V, Y, dY_ell, dY_sf, stream)
        return Y, dY_ell, dY_sf

    def pipeline_wait(self, stream=None):
        akm_pipeline_wait(self.handle, stream)

    def cross_mvm(self, n_src, V, Yt, stream=None):
        akm_kernel_cross_mvm(self.handle, n_src, V, Yt, stream)
        return Yt

    def gradient_diag(self, y, Z, cg_iters=50, stream=None):
        return akm_gradient_diag(self.handle, y, Z, cg_iters, stream)

    def gradient(self, y, Z, cg_iters=50, stream=None):
        return akm_gradient(self.handle, y, Z, cg_iters, stream)

    def gradient_columns(self, y, Z, cg_iters=50, preconditioned=False, stream=None):
        return akm_gradient_columns(self.handle, y, Z, cg_iters, preconditioned, stream)

    def objective_diag(self, y, Z, cg_iters=50, lanczos_steps=30, stream=None):
        return akm_objective_diag(self.handle, y, Z, cg_iters, lanczos_steps, stream)

    def objective(self, y, Z, cg_iters=50, lanczos_steps=30, stream=None):
        return akm_objective(self.handle, y, Z, cg_iters, lanczos_steps, stream)

    def set_preconditioner(self, k_per_window=0):
        akm_set_preconditioner(self.handle, k_per_window)
        return self

    def precond_apply(self, T, out, transpose=False, stream=None):
        return akm_precond_apply(self.handle, T, out, transpose, stream)

    def info(self):
        return akm_get_info(self.handle)

    def window_poly(self):
        return akm_get_window_poly(self.handle)

    # point sharding (include/akm.h; paper_2504_00480_b200.dist.ShardedPlan drives these)
    def bounds(self):
        return akm_get_bounds(self.handle)

    def set_bounds(self, lo, hi, stream=None):
        return akm_set_bounds(self.handle, lo, hi, stream)

    def set_radius(self, radius):
        akm_set_radius(self.handle, radius)
        return self

    def set_bin_override(self, bins=None):
        akm_set_bin_override(self.handle, bins)
        return self

    def grid_size(self, r):
        return akm_grid_size(self.handle, r)

    def spread_grid(self, V, grid, stream=None):
        akm_spread_grid(self.handle, V, grid, stream)
        return grid

    def mvm_from_grid(self, grid, V, Y=None, dY_ell=None, dY_sf=None, stream=None):
        akm_mvm_from_grid(self.handle, grid, V, Y, dY_ell, dY_sf, stream)
        return Y, dY_ell, dY_sf

    def set_profiling(self, enable=True):
        akm_set_profiling(self.handle, enable)
        return self

    def stage_times(self, reset=False):
        return akm_get_stage_times(self.handle, reset)
