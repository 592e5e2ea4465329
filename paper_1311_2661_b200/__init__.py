"""Python binding of libthetis (include/thetis.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libthetis.so; PyTorch
only provides device memory (the workspace and the array arguments) and the
stream.  There is no CPU fallback: importing this package without the built
library raises.

Module-level functions carry the C names (thetis_build_graph_lp, thetis_solve,
...) and take raw pointers like the C ABI; the `LP` class is a convenience
wrapper that owns the workspace tensor and converts torch / numpy arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libthetis.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build it with __graft_entry__.build() "
                      "(there is no CPU fallback)")
_L = ctypes.CDLL(_LIB_PATH)

THETIS_OK = 0
THETIS_ERR_INVALID_ARG = -1
THETIS_ERR_WORKSPACE_TOO_SMALL = -2
THETIS_ERR_CUDA = -3
THETIS_ERR_NOT_SUPPORTED = -4
THETIS_ERR_DIVERGED = -5
THETIS_ERR_ROUND_PRECONDITION = -6
THETIS_EQ, THETIS_GE, THETIS_LE = 0, 1, 2
THETIS_MIN, THETIS_MAX = 0, 1
THETIS_PROB_GENERIC, THETIS_PROB_VC, THETIS_PROB_MIS, THETIS_PROB_MWC = 0, 1, 2, 3
THETIS_MODE_DETERMINISTIC, THETIS_MODE_ASYNC, THETIS_MODE_ASYNC_SERIAL = 0, 1, 2
THETIS_MODE_ASYNC_HUBLAG, THETIS_MODE_ASYNC_HUBLAG_SERIAL = 3, 4
THETIS_STEP_LMAX, THETIS_STEP_LJ = 0, 1
THETIS_ROUND_VC_HALF, THETIS_ROUND_VC_FIXUP, THETIS_ROUND_MIS_GREEDY, THETIS_ROUND_MWC_CKR = 1, 2, 3, 4
THETIS_ROUND_SC_THRESHOLD, THETIS_ROUND_SC_RANDOM, THETIS_ROUND_MIS_BANSAL = 5, 6, 7
THETIS_MAX_EPOCH_TIMES = 64

LIB_PATH = _LIB_PATH


class SolveStats(ctypes.Structure):
    _fields_ = [("epochs", ctypes.c_int64), ("coordinate_updates", ctypes.c_int64),
                ("nnz_processed", ctypes.c_int64), ("ms_total", ctypes.c_double),
                ("ms_per_epoch", ctypes.c_float * THETIS_MAX_EPOCH_TIMES), ("L_max", ctypes.c_double),
                ("n_colours", ctypes.c_int64), ("mode", ctypes.c_int32), ("step_rule", ctypes.c_int32),
                ("ms_row_pass", ctypes.c_double), ("ms_hub_update", ctypes.c_double),
                ("ms_tiles", ctypes.c_double), ("row_pass_launches", ctypes.c_int64)]


class Objective(ctypes.Structure):
    _fields_ = [("lp_obj", ctypes.c_double), ("f_beta", ctypes.c_double),
                ("resid_l2", ctypes.c_double), ("resid_inf", ctypes.c_double),
                ("max_violation_eps", ctypes.c_double), ("drift_inf", ctypes.c_double),
                ("nonfinite", ctypes.c_int64)]


class RoundResult(ctypes.Structure):
    _fields_ = [("cost", ctypes.c_double), ("feasible", ctypes.c_int64),
                ("n_selected", ctypes.c_int64), ("eps_or_alpha", ctypes.c_double),
                ("best_rep", ctypes.c_int64), ("fallback", ctypes.c_int64),
                ("rounds", ctypes.c_int64)]


THETIS_MAX_ALM_ROUNDS = 64


class AlmStats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("epochs_total", ctypes.c_int64), ("ms_total", ctypes.c_double),
                ("beta", ctypes.c_float * THETIS_MAX_ALM_ROUNDS), ("eps", ctypes.c_double * THETIS_MAX_ALM_ROUNDS),
                ("resid_inf", ctypes.c_double * THETIS_MAX_ALM_ROUNDS),
                ("lp_obj", ctypes.c_double * THETIS_MAX_ALM_ROUNDS)]


class Dims(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("m", "n_struct", "N", "U", "nnz_struct", "n_blocks", "block_k",
                                              "m_edges", "n_vertices", "n_ineq")] + \
               [("problem", ctypes.c_int32), ("obj_sense", ctypes.c_int32)]


_vp, _i64, _i32, _f32, _u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_uint64
_sz = ctypes.POINTER(ctypes.c_size_t)
_PROTOS = {
    "thetis_build_graph_lp_workspace": (_i32, [_i32, _i64, _i64, _i32, _sz]),
    "thetis_build_graph_lp": (_i32, [ctypes.POINTER(_vp), _vp, ctypes.c_size_t, _vp, _i32, _i64, _i64, _vp, _vp,
                                     _vp, _vp, _i32, _vp, _i32]),
    "thetis_build_lp_workspace": (_i32, [_i64, _i64, _i64, _sz]),
    "thetis_build_lp": (_i32, [ctypes.POINTER(_vp), _vp, ctypes.c_size_t, _vp, _i64, _i64, _i64, _vp, _vp, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i64]),
    "thetis_get_dims": (_i32, [_vp, ctypes.POINTER(Dims)]),
    "thetis_set_anchors": (_i32, [_vp, _vp, _vp]),
    "thetis_set_x": (_i32, [_vp, _vp]),
    "thetis_get_x": (_i32, [_vp, _vp, _i64]),
    "thetis_get_r": (_i32, [_vp, _vp, _i64]),
    "thetis_solve": (_i32, [_vp, _f32, _i32, _i32, _u64, _i32, ctypes.POINTER(SolveStats)]),
    "thetis_objective": (_i32, [_vp, _f32, ctypes.POINTER(Objective)]),
    "thetis_solve_alm": (_i32, [_vp, _vp, _vp, _f32, _f32, _i32, _i32, _i32, _u64, _i32, ctypes.c_double,
                                ctypes.POINTER(AlmStats)]),
    "thetis_round": (_i32, [_vp, _i32, _u64, _i32, _vp, ctypes.POINTER(RoundResult)]),
    "thetis_round_x": (_i32, [_vp, _vp, _i32, _u64, _i32, _vp, ctypes.POINTER(RoundResult)]),
    "thetis_get_csc": (_i32, [_vp, _vp, _vp, _vp]),
    "thetis_get_edges": (_i32, [_vp, _vp, _vp]),
    "thetis_get_colouring": (_i32, [_vp, _u64, _vp, ctypes.POINTER(_i64)]),
    "thetis_tile_perm": (_i32, [_i64, _u64, _i64, _vp, _vp]),
    "thetis_sync": (_i32, [_vp]),
    "thetis_free": (None, [_vp]),
    "thetis_error_string": (ctypes.c_char_p, [_i32]),
    "thetis_last_error": (ctypes.c_char_p, [_vp]),
    "thetis_version": (ctypes.c_char_p, []),
}
EXPORTED = tuple(_PROTOS)
for _name, (_res, _args) in _PROTOS.items():
    _fn = getattr(_L, _name)
    _fn.restype = _res
    _fn.argtypes = _args
    globals()[_name] = _fn


class ThetisError(RuntimeError):
    def __init__(self, code, what, detail=""):
        super().__init__(f"{what}: {thetis_error_string(code).decode()} {detail}".strip())
        self.code = code


def _check(rc, what, handle=None):
    if rc != THETIS_OK:
        detail = thetis_last_error(handle).decode(errors="replace") if handle is not None else \
            thetis_last_error(None).decode(errors="replace")
        raise ThetisError(rc, what, detail)


def _torch():
    import torch
    return torch


def _dev_array(a, dtype, device):
    """torch tensor on `device` (contiguous, dtype) or None; numpy arrays are uploaded."""
    if a is None:
        return None
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


def _ptr(t):
    return None if t is None else t.data_ptr()


class LP:
    """An LP held by libthetis in a workspace tensor owned by this object."""

    def __init__(self, handle, workspace, stream, keep=()):
        self._h = handle
        self.workspace = workspace
        self.stream = stream
        self._keep = list(keep)
        d = Dims()
        _check(thetis_get_dims(handle, ctypes.byref(d)), "thetis_get_dims", handle)
        for f, _ in Dims._fields_:
            setattr(self, f, int(getattr(d, f)))
        self.device = workspace.device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _L is not None:
            try:
                _L.thetis_free(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @staticmethod
    def _stream(stream, device):
        torch = _torch()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        return stream

    @classmethod
    def from_graph(cls, problem, n, src, dst, vertex_w=None, edge_w=None, k=0, terminals=None, t_per_label=0,
                   device="cuda", stream=None, host_inputs=False):
        """Build a VC / MIS / MWC LP.  Inputs may be numpy arrays or torch tensors;
        with host_inputs=True numpy / CPU arrays are passed to the C ABI as host
        pointers (the library copies them in), otherwise they are uploaded first."""
        torch = _torch()
        device = torch.device(device)
        stream = cls._stream(stream, device)
        n_edges = int(len(src))
        need = ctypes.c_size_t()
        _check(thetis_build_graph_lp_workspace(problem, n, n_edges, k, ctypes.byref(need)),
               "thetis_build_graph_lp_workspace")
        ws = torch.empty(int(need.value), dtype=torch.uint8, device=device)
        keep = []

        def arg(a, dtype):
            if a is None:
                return None
            if host_inputs and not (isinstance(a, torch.Tensor) and a.is_cuda):
                t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
                t = t.to(dtype).contiguous()
            else:
                t = _dev_array(a, dtype, device)
            keep.append(t)
            return t.data_ptr()

        h = ctypes.c_void_p()
        with torch.cuda.stream(stream):
            rc = thetis_build_graph_lp(ctypes.byref(h), ws.data_ptr(), ws.numel(), stream.cuda_stream, problem, n,
                                       n_edges, arg(src, torch.int32), arg(dst, torch.int32),
                                       arg(vertex_w, torch.float32), arg(edge_w, torch.float32), k,
                                       arg(terminals, torch.int32), t_per_label)
        _check(rc, "thetis_build_graph_lp")
        return cls(h, ws, stream)

    @classmethod
    def from_csc_csr(cls, m, n, colptr, rowidx, val, rowptr, colidx, rval, b, c, sense=None, lo=None, hi=None,
                     obj_sense=THETIS_MIN, block_k=0, n_blocks=0, device="cuda", stream=None):
        torch = _torch()
        device = torch.device(device)
        stream = cls._stream(stream, device)
        nnz = int(len(rowidx))
        need = ctypes.c_size_t()
        _check(thetis_build_lp_workspace(m, n, nnz, ctypes.byref(need)), "thetis_build_lp_workspace")
        ws = torch.empty(int(need.value), dtype=torch.uint8, device=device)
        t = [_dev_array(a, dt, device) for a, dt in (
            (colptr, torch.int64), (rowidx, torch.int32), (val, torch.float32), (rowptr, torch.int64),
            (colidx, torch.int32), (rval, torch.float32), (b, torch.float32), (c, torch.float32),
            (sense, torch.int8), (lo, torch.float32), (hi, torch.float32))]
        h = ctypes.c_void_p()
        rc = thetis_build_lp(ctypes.byref(h), ws.data_ptr(), ws.numel(), stream.cuda_stream, m, n, nnz,
                             *[_ptr(x) for x in t], obj_sense, block_k, n_blocks)
        _check(rc, "thetis_build_lp")
        return cls(h, ws, stream, keep=t)

    # ---- state
    def set_anchors(self, zbar=None, ubar=None):
        zb = _dev_array(zbar, _torch().float32, self.device)
        ub = _dev_array(ubar, _torch().float32, self.device)
        self._anchors = (zb, ub)
        _check(thetis_set_anchors(self._h, _ptr(zb), _ptr(ub)), "thetis_set_anchors", self._h)

    def set_x(self, z):
        zt = _dev_array(z, _torch().float32, self.device)
        assert zt.numel() == self.N
        _check(thetis_set_x(self._h, zt.data_ptr()), "thetis_set_x", self._h)
        self.sync()

    def get_x(self):
        out = _torch().empty(max(self.N, 1), dtype=_torch().float32, device=self.device)
        _check(thetis_get_x(self._h, out.data_ptr(), self.N), "thetis_get_x", self._h)
        return out[: self.N]

    def get_r(self):
        out = _torch().empty(max(self.m, 1), dtype=_torch().float32, device=self.device)
        _check(thetis_get_r(self._h, out.data_ptr(), self.m), "thetis_get_r", self._h)
        return out[: self.m]

    # ---- method
    def solve(self, beta, epochs, mode=THETIS_MODE_DETERMINISTIC, seed=0, step_rule=THETIS_STEP_LMAX,
              stats=True):
        st = SolveStats() if stats else None
        rc = thetis_solve(self._h, beta, epochs, mode, seed, step_rule, ctypes.byref(st) if stats else None)
        _check(rc, "thetis_solve", self._h)
        if not stats:
            return None
        out = {f: getattr(st, f) for f, _ in SolveStats._fields_ if f != "ms_per_epoch"}
        out["ms_per_epoch"] = list(st.ms_per_epoch)[: min(epochs, THETIS_MAX_EPOCH_TIMES)]
        return out

    def solve_alm(self, beta0, beta_growth=2.0, max_outer=10, inner_epochs=50, mode=THETIS_MODE_DETERMINISTIC,
                  seed=0, step_rule=THETIS_STEP_LMAX, target_eps=0.0, ubar=None, zbar=None):
        """thetis_solve_alm: the augmented-Lagrangian outer loop; returns (stats, ubar, zbar)
        with the final anchors (device tensors, also left registered on the LP)."""
        torch = _torch()
        ub = torch.zeros(max(self.m, 1), dtype=torch.float32, device=self.device)
        zb = torch.zeros(max(self.N, 1), dtype=torch.float32, device=self.device)
        if ubar is not None:
            ub[: self.m] = _dev_array(ubar, torch.float32, self.device)
        if zbar is not None:
            zb[: self.N] = _dev_array(zbar, torch.float32, self.device)
        self._anchors = (zb, ub)
        st = AlmStats()
        rc = thetis_solve_alm(self._h, ub.data_ptr(), zb.data_ptr(), beta0, beta_growth, max_outer, inner_epochs,
                              mode, seed, step_rule, target_eps, ctypes.byref(st))
        _check(rc, "thetis_solve_alm", self._h)
        n = int(st.rounds)
        out = dict(rounds=n, epochs_total=int(st.epochs_total), ms_total=float(st.ms_total),
                   beta=list(st.beta)[:n], eps=list(st.eps)[:n], resid_inf=list(st.resid_inf)[:n],
                   lp_obj=list(st.lp_obj)[:n])
        return out, ub[: self.m], zb[: self.N]

    def objective(self, beta):
        o = Objective()
        rc = thetis_objective(self._h, beta, ctypes.byref(o))
        if rc not in (THETIS_OK, THETIS_ERR_DIVERGED):
            _check(rc, "thetis_objective", self._h)
        return {f: getattr(o, f) for f, _ in Objective._fields_}

    def _round(self, x, rule, seed, reps, out):
        res = RoundResult()
        torch = _torch()
        n_out = self.n_struct if rule in (THETIS_ROUND_SC_THRESHOLD, THETIS_ROUND_SC_RANDOM) else self.n_vertices
        if out is None:
            out = torch.empty(max(n_out, 1), dtype=torch.uint8, device=self.device)
        if x is None:
            rc = thetis_round(self._h, rule, seed, reps, out.data_ptr(), ctypes.byref(res))
        else:
            xt = _dev_array(x, torch.float32, self.device)
            rc = thetis_round_x(self._h, xt.data_ptr(), rule, seed, reps, out.data_ptr(), ctypes.byref(res))
        _check(rc, "thetis_round", self._h)
        return out[:n_out], {f: getattr(res, f) for f, _ in RoundResult._fields_}

    def round(self, rule, seed=0, reps=10, out=None):
        return self._round(None, rule, seed, reps, out)

    def round_x(self, x, rule, seed=0, reps=10, out=None):
        return self._round(x, rule, seed, reps, out)

    # ---- inspection
    def csc(self):
        cp = np.zeros(self.n_struct + 1, np.int64)
        ri = np.zeros(max(self.nnz_struct, 1), np.int32)
        va = np.zeros(max(self.nnz_struct, 1), np.float32)
        _check(thetis_get_csc(self._h, cp.ctypes.data, ri.ctypes.data, va.ctypes.data), "thetis_get_csc", self._h)
        return cp, ri[: self.nnz_struct] & 0x7FFFFFFF, va[: self.nnz_struct]

    def edges(self):
        u = np.zeros(max(self.m_edges, 1), np.int32)
        v = np.zeros(max(self.m_edges, 1), np.int32)
        _check(thetis_get_edges(self._h, u.ctypes.data, v.ctypes.data), "thetis_get_edges", self._h)
        return u[: self.m_edges], v[: self.m_edges]

    def colouring(self, seed):
        col = np.zeros(max(self.U, 1), np.int32)
        K = ctypes.c_int64()
        _check(thetis_get_colouring(self._h, seed, col.ctypes.data, ctypes.byref(K)), "thetis_get_colouring",
               self._h)
        return int(K.value), col[: self.U]

    def sync(self):
        _check(thetis_sync(self._h), "thetis_sync", self._h)


def tile_perm(n_tiles, seed, epoch, device="cuda"):
    torch = _torch()
    out = torch.empty(max(n_tiles, 1), dtype=torch.int64, device=device)
    stream = torch.cuda.current_stream(device)
    _check(thetis_tile_perm(n_tiles, seed, epoch, out.data_ptr(), stream.cuda_stream), "thetis_tile_perm")
    stream.synchronize()
    return out[:n_tiles]
