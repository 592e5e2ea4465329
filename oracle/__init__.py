"""ctypes wrapper of the oracle libraries (libthetis_ref64.so / libthetis_ref32.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package
(paper_1311_2661_b200), which fails loudly when its CUDA library is missing.
See oracle/thetis_ref.h for what is implemented and the paper passages.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS: dict = {}

PROB_VC, PROB_MIS, PROB_MWC = 1, 2, 3
MODE_DET, MODE_ASYNC, MODE_CYCLIC, MODE_HUBLAG_REPLAY, MODE_PI_TILE_SYNC = 0, 1, 2, 3, 4
STEP_LMAX, STEP_LJ = 0, 1
ROUND_VC_HALF, ROUND_VC_FIXUP, ROUND_MIS_GREEDY, ROUND_MWC_CKR = 1, 2, 3, 4
ROUND_SC_THRESHOLD, ROUND_SC_RANDOM, ROUND_MIS_BANSAL = 5, 6, 7
SENSE_EQ, SENSE_GE, SENSE_LE = 0, 1, 2


class RefStats(ctypes.Structure):
    _fields_ = [("epochs", ctypes.c_int64), ("coordinate_updates", ctypes.c_int64),
                ("nnz_processed", ctypes.c_int64), ("L_max", ctypes.c_double),
                ("n_colours", ctypes.c_int64)]


class RefObjective(ctypes.Structure):
    _fields_ = [("lp_obj", ctypes.c_double), ("f_beta", ctypes.c_double),
                ("resid_l2", ctypes.c_double), ("resid_inf", ctypes.c_double),
                ("max_violation_eps", ctypes.c_double), ("drift_inf", ctypes.c_double),
                ("nonfinite", ctypes.c_int64)]


class RefAlm(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("beta", ctypes.c_float * 64), ("eps", ctypes.c_double * 64),
                ("resid_inf", ctypes.c_double * 64), ("lp_obj", ctypes.c_double * 64)]


class RefRound(ctypes.Structure):
    _fields_ = [("cost", ctypes.c_double), ("feasible", ctypes.c_int64),
                ("n_selected", ctypes.c_int64), ("eps_or_alpha", ctypes.c_double),
                ("best_rep", ctypes.c_int64), ("fallback", ctypes.c_int64),
                ("rounds", ctypes.c_int64)]


def _load(bits: int):
    if bits in _LIBS:
        return _LIBS[bits]
    path = os.path.join(_HERE, f"libthetis_ref{bits}.so")
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
    L = bind(ctypes.CDLL(path))
    assert L.ref_real_bytes() == bits // 8
    _LIBS[bits] = L
    return L


def bind(L):
    """argument / result types of the oracle's C entry points on a loaded library (also used
    by tests/experiments, whose library includes the oracle's source)"""
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    L.ref_real_bytes.restype = i32
    L.thetis_ref_build_lp.restype = i32
    L.thetis_ref_build_lp.argtypes = [ctypes.POINTER(vp), i64, i64, i64, vp, vp, vp, vp, vp, vp,
                                      vp, vp, i32, i32, i64]
    L.thetis_ref_build_graph_lp.restype = i32
    L.thetis_ref_build_graph_lp.argtypes = [ctypes.POINTER(vp), i32, i64, i64, vp, vp, vp, vp,
                                            i32, vp, i32]
    L.thetis_ref_free.argtypes = [vp]
    L.thetis_ref_free.restype = None
    L.thetis_ref_dims.argtypes = [vp, vp]
    L.thetis_ref_dims.restype = None
    for name in ("get_csc", "get_rows", "get_edges"):
        getattr(L, f"thetis_ref_{name}").restype = None
    L.thetis_ref_get_csc.argtypes = [vp, vp, vp, vp]
    L.thetis_ref_get_rows.argtypes = [vp, vp, vp, vp]
    L.thetis_ref_get_edges.argtypes = [vp, vp, vp]
    L.thetis_ref_set_anchors.restype = i32
    L.thetis_ref_set_anchors.argtypes = [vp, vp, vp]
    L.thetis_ref_set_x.restype = i32
    L.thetis_ref_set_x.argtypes = [vp, vp]
    for name in ("get_x", "get_r", "get_x_f32", "get_r_f32"):
        fn = getattr(L, f"thetis_ref_{name}")
        fn.restype = None
        fn.argtypes = [vp, vp]
    L.thetis_ref_step_unit.restype = i32
    L.thetis_ref_step_unit.argtypes = [vp, f32, i64, i32]
    L.thetis_ref_grad.restype = ctypes.c_double
    L.thetis_ref_grad.argtypes = [vp, f32, i64]
    L.thetis_ref_solve.restype = i32
    L.thetis_ref_solve.argtypes = [vp, f32, i32, i32, ctypes.c_uint64, i32, ctypes.POINTER(RefStats)]
    L.thetis_ref_objective.restype = i32
    L.thetis_ref_objective.argtypes = [vp, f32, ctypes.POINTER(RefObjective)]
    L.thetis_ref_solve_alm.restype = i32
    L.thetis_ref_solve_alm.argtypes = [vp, vp, vp, f32, f32, i32, i32, i32, ctypes.c_uint64, i32, ctypes.c_double,
                                       ctypes.POINTER(RefAlm)]
    L.thetis_ref_get_anchors.restype = None
    L.thetis_ref_get_anchors.argtypes = [vp, vp, vp]
    L.thetis_ref_colouring.restype = i64
    L.thetis_ref_colouring.argtypes = [vp, ctypes.c_uint64, vp]
    L.thetis_ref_tile_perm.restype = None
    L.thetis_ref_tile_perm.argtypes = [i64, ctypes.c_uint64, i64, vp]
    L.thetis_ref_project_simplex.restype = None
    L.thetis_ref_project_simplex.argtypes = [vp, i32, vp]
    L.thetis_ref_round_x.restype = i32
    L.thetis_ref_round_x.argtypes = [vp, vp, i32, ctypes.c_uint64, i32, vp, ctypes.POINTER(RefRound)]
    L.thetis_ref_round.restype = i32
    L.thetis_ref_round.argtypes = [vp, i32, ctypes.c_uint64, i32, vp, ctypes.POINTER(RefRound)]
    return L


def _p(a):
    return None if a is None else a.ctypes.data


def _arr(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what} failed with status {code}")
        self.code = code


class RefLP:
    """One LP held by the oracle (bits = 64: fp64 build; 32: fp32 build)."""

    def __init__(self, handle, lib, bits, keep):
        self._h = handle
        self._L = lib
        self.bits = bits
        self._keep = keep
        d = np.zeros(10, np.int64)
        lib.thetis_ref_dims(handle, d.ctypes.data)
        (self.m, self.n_struct, self.N, self.U, self.nnz_struct, self.n_blocks, self.block_k,
         self.m_edges, self.n_vertices, self.n_ineq) = (int(v) for v in d)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.thetis_ref_free(self._h)
            self._h = None

    @classmethod
    def graph(cls, problem, n, src, dst, vertex_w=None, edge_w=None, k=0, terminals=None,
              t_per_label=0, bits=64):
        L = _load(bits)
        src, dst = _arr(src, np.int32), _arr(dst, np.int32)
        vw, ew, te = _arr(vertex_w, np.float32), _arr(edge_w, np.float32), _arr(terminals, np.int32)
        h = ctypes.c_void_p()
        rc = L.thetis_ref_build_graph_lp(ctypes.byref(h), problem, n, len(src), _p(src), _p(dst),
                                         _p(vw), _p(ew), k, _p(te), t_per_label)
        if rc != 0:
            raise OracleError(rc, "thetis_ref_build_graph_lp")
        return cls(h, L, bits, None)

    @classmethod
    def generic(cls, m, n, colptr, rowidx, val, b, c, sense=None, lo=None, hi=None, obj_sense=0,
                block_k=0, n_blocks=0, bits=64):
        L = _load(bits)
        colptr, rowidx = _arr(colptr, np.int64), _arr(rowidx, np.int32)
        val, b, c = _arr(val, np.float32), _arr(b, np.float32), _arr(c, np.float32)
        sense, lo, hi = _arr(sense, np.int8), _arr(lo, np.float32), _arr(hi, np.float32)
        h = ctypes.c_void_p()
        rc = L.thetis_ref_build_lp(ctypes.byref(h), m, n, len(rowidx), _p(colptr), _p(rowidx),
                                   _p(val), _p(b), _p(c), _p(sense), _p(lo), _p(hi), obj_sense,
                                   block_k, n_blocks)
        if rc != 0:
            raise OracleError(rc, "thetis_ref_build_lp")
        return cls(h, L, bits, None)

    # -- accessors --------------------------------------------------------
    def csc(self):
        cp = np.zeros(self.n_struct + 1, np.int64)
        ri = np.zeros(max(self.nnz_struct, 1), np.int32)
        va = np.zeros(max(self.nnz_struct, 1), np.float64)
        self._L.thetis_ref_get_csc(self._h, cp.ctypes.data, ri.ctypes.data, va.ctypes.data)
        return cp, ri[: self.nnz_struct], va[: self.nnz_struct]

    def rows(self):
        b = np.zeros(max(self.m, 1), np.float64)
        s = np.zeros(max(self.m, 1), np.int8)
        c = np.zeros(max(self.n_struct, 1), np.float64)
        self._L.thetis_ref_get_rows(self._h, b.ctypes.data, s.ctypes.data, c.ctypes.data)
        return b[: self.m], s[: self.m], c[: self.n_struct]

    def edges(self):
        u = np.zeros(max(self.m_edges, 1), np.int32)
        v = np.zeros(max(self.m_edges, 1), np.int32)
        self._L.thetis_ref_get_edges(self._h, u.ctypes.data, v.ctypes.data)
        return u[: self.m_edges], v[: self.m_edges]

    def x(self):
        z = np.zeros(max(self.N, 1), np.float64)
        self._L.thetis_ref_get_x(self._h, z.ctypes.data)
        return z[: self.N]

    def r(self):
        r = np.zeros(max(self.m, 1), np.float64)
        self._L.thetis_ref_get_r(self._h, r.ctypes.data)
        return r[: self.m]

    def x32(self):
        z = np.zeros(max(self.N, 1), np.float32)
        self._L.thetis_ref_get_x_f32(self._h, z.ctypes.data)
        return z[: self.N]

    def r32(self):
        r = np.zeros(max(self.m, 1), np.float32)
        self._L.thetis_ref_get_r_f32(self._h, r.ctypes.data)
        return r[: self.m]

    def set_x(self, z):
        z = _arr(z, np.float64)
        assert len(z) == self.N
        self._L.thetis_ref_set_x(self._h, z.ctypes.data)

    def set_anchors(self, zbar=None, ubar=None):
        zb, ub = _arr(zbar, np.float64), _arr(ubar, np.float64)
        self._L.thetis_ref_set_anchors(self._h, _p(zb), _p(ub))

    # -- method -----------------------------------------------------------
    def step_unit(self, beta, u, step_rule=STEP_LMAX):
        rc = self._L.thetis_ref_step_unit(self._h, beta, u, step_rule)
        if rc != 0:
            raise OracleError(rc, "thetis_ref_step_unit")

    def grad(self, beta, j):
        return self._L.thetis_ref_grad(self._h, beta, j)

    def solve(self, beta, epochs, mode=MODE_DET, seed=0, step_rule=STEP_LMAX):
        st = RefStats()
        rc = self._L.thetis_ref_solve(self._h, beta, epochs, mode, seed, step_rule, ctypes.byref(st))
        if rc != 0:
            raise OracleError(rc, "thetis_ref_solve")
        return {f: getattr(st, f) for f, _ in RefStats._fields_}

    def solve_alm(self, beta0, beta_growth=2.0, max_outer=10, inner_epochs=50, mode=MODE_DET, seed=0,
                  step_rule=STEP_LMAX, target_eps=0.0, ubar=None, zbar=None):
        """the augmented-Lagrangian outer loop (thetis_ref_solve_alm); returns per-round stats"""
        ub, zb = _arr(ubar, np.float64), _arr(zbar, np.float64)
        st = RefAlm()
        rc = self._L.thetis_ref_solve_alm(self._h, _p(ub), _p(zb), beta0, beta_growth, max_outer, inner_epochs,
                                          mode, seed, step_rule, target_eps, ctypes.byref(st))
        if rc != 0:
            raise OracleError(rc, "thetis_ref_solve_alm")
        n = int(st.rounds)
        return dict(rounds=n, beta=list(st.beta)[:n], eps=list(st.eps)[:n], resid_inf=list(st.resid_inf)[:n],
                    lp_obj=list(st.lp_obj)[:n])

    def anchors(self):
        ub = np.zeros(max(self.m, 1))
        zb = np.zeros(max(self.N, 1))
        self._L.thetis_ref_get_anchors(self._h, ub.ctypes.data, zb.ctypes.data)
        return ub[: self.m], zb[: self.N]

    def objective(self, beta):
        o = RefObjective()
        self._L.thetis_ref_objective(self._h, beta, ctypes.byref(o))
        return {f: getattr(o, f) for f, _ in RefObjective._fields_}

    def colouring(self, seed):
        col = np.zeros(max(self.U, 1), np.int32)
        K = self._L.thetis_ref_colouring(self._h, seed, col.ctypes.data)
        return int(K), col[: self.U]

    def round_x(self, x, rule, seed=0, reps=10):
        x = _arr(x, np.float32)
        n_out = self.n_struct if rule in (ROUND_SC_THRESHOLD, ROUND_SC_RANDOM) else self.n_vertices
        out = np.zeros(max(n_out, 1), np.uint8)
        res = RefRound()
        rc = self._L.thetis_ref_round_x(self._h, x.ctypes.data, rule, seed, reps, out.ctypes.data,
                                        ctypes.byref(res))
        if rc != 0:
            raise OracleError(rc, "thetis_ref_round_x")
        return out[:n_out], {f: getattr(res, f) for f, _ in RefRound._fields_}

    def round(self, rule, seed=0, reps=10):
        n_out = self.n_struct if rule in (ROUND_SC_THRESHOLD, ROUND_SC_RANDOM) else self.n_vertices
        out = np.zeros(max(n_out, 1), np.uint8)
        res = RefRound()
        rc = self._L.thetis_ref_round(self._h, rule, seed, reps, out.ctypes.data, ctypes.byref(res))
        if rc != 0:
            raise OracleError(rc, "thetis_ref_round")
        return out[:n_out], {f: getattr(res, f) for f, _ in RefRound._fields_}


def tile_perm(n_tiles, seed, epoch, bits=64):
    out = np.zeros(max(n_tiles, 1), np.int64)
    _load(bits).thetis_ref_tile_perm(n_tiles, seed, epoch, out.ctypes.data)
    return out[:n_tiles]


def project_simplex(y, bits=64):
    y = np.ascontiguousarray(y, np.float64)
    out = np.zeros_like(y)
    _load(bits).thetis_ref_project_simplex(y.ctypes.data, len(y), out.ctypes.data)
    return out
