"""Seeded synthetic inputs shared by the CUDA path and the oracle.

Holds none of the method's arithmetic: raw edge lists (loops / duplicates kept,
orientation as drawn), weights and terminals only.  Recipes follow SURVEY.md
§8(d) and are restated in DESIGN.md §Inputs.  The five BASELINE.json configs
are in CONFIGS; `make_graph(name)` returns numpy arrays for any of them (the
host generator), `make_rmat_device` generates config 5 directly in HBM with
the device twin (inputs/gen_cuda.cu).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LIB_CUDA = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libthetis_inputs.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        i64, u64, i32p, f32p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p
        L.inputs_draw.restype = u64
        L.inputs_draw.argtypes = [u64, u64]
        L.inputs_er.restype = i64
        L.inputs_er.argtypes = [i64, i64, u64, i32p, i32p]
        L.inputs_chung_lu.restype = ctypes.c_int
        L.inputs_chung_lu.argtypes = [i64, ctypes.c_double, i64, u64, i32p, i32p]
        L.inputs_grid.restype = i64
        L.inputs_grid.argtypes = [i64, i32p, i32p]
        L.inputs_rmat.restype = ctypes.c_int
        L.inputs_rmat.argtypes = [ctypes.c_int, i64, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_uint32, u64, i32p, i32p]
        L.inputs_uniform_weights.restype = None
        L.inputs_uniform_weights.argtypes = [i64, u64, f32p]
        L.inputs_exp_weights.restype = None
        L.inputs_exp_weights.argtypes = [i64, u64, f32p]
        L.inputs_terminals.restype = ctypes.c_int
        L.inputs_terminals.argtypes = [i64, i64, u64, i32p]
        _LIB = L
    return _LIB


def _lib_cuda():
    global _LIB_CUDA
    if _LIB_CUDA is None:
        path = os.path.join(_HERE, "libthetis_inputs_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        L.inputs_rmat_device.restype = ctypes.c_int
        L.inputs_rmat_device.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.inputs_uniform_weights_device.restype = ctypes.c_int
        L.inputs_uniform_weights_device.argtypes = [ctypes.c_int64, ctypes.c_uint64,
                                                    ctypes.c_void_p, ctypes.c_void_p]
        _LIB_CUDA = L
    return _LIB_CUDA


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def draw(seed: int, i: int) -> int:
    return int(_lib().inputs_draw(seed, i))


def er(n: int, m: int, seed: int):
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    r = _lib().inputs_er(n, m, seed, _ptr(src), _ptr(dst))
    if r < 0:
        raise ValueError("inputs_er: bad arguments")
    return src, dst


def chung_lu(n: int, gamma: float, samples: int, seed: int):
    src = np.empty(samples, np.int32)
    dst = np.empty(samples, np.int32)
    if _lib().inputs_chung_lu(n, gamma, samples, seed, _ptr(src), _ptr(dst)) != 0:
        raise ValueError("inputs_chung_lu: bad arguments")
    return src, dst


def grid(side: int):
    m = 2 * side * (side - 1)
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    got = _lib().inputs_grid(side, _ptr(src), _ptr(dst))
    assert got == m
    return src, dst


def rmat_thresholds(a: float, b: float, c: float):
    t = lambda p: min(int(math.floor(p * 4294967296.0)), 0xFFFFFFFF)
    return t(a), t(a + b), t(a + b + c)


def rmat(scale: int, samples: int, a: float, b: float, c: float, seed: int):
    src = np.empty(samples, np.int32)
    dst = np.empty(samples, np.int32)
    ta, tab, tabc = rmat_thresholds(a, b, c)
    if _lib().inputs_rmat(scale, samples, ta, tab, tabc, seed, _ptr(src), _ptr(dst)) != 0:
        raise ValueError("inputs_rmat: bad arguments")
    return src, dst


def uniform_weights(n: int, seed: int) -> np.ndarray:
    w = np.empty(n, np.float32)
    _lib().inputs_uniform_weights(n, seed, _ptr(w))
    return w


def exp_weights(n: int, seed: int) -> np.ndarray:
    w = np.empty(n, np.float32)
    _lib().inputs_exp_weights(n, seed, _ptr(w))
    return w


def terminals(n: int, count: int, seed: int) -> np.ndarray:
    out = np.empty(count, np.int32)
    if _lib().inputs_terminals(n, count, seed, _ptr(out)) != 0:
        raise ValueError("inputs_terminals: count > n")
    return out


def rmat_device(scale, samples, a, b, c, seed, src_ptr, dst_ptr, stream_ptr):
    ta, tab, tabc = rmat_thresholds(a, b, c)
    if _lib_cuda().inputs_rmat_device(scale, samples, ta, tab, tabc, seed,
                                      src_ptr, dst_ptr, stream_ptr) != 0:
        raise RuntimeError("inputs_rmat_device failed")


def uniform_weights_device(n, seed, w_ptr, stream_ptr):
    if _lib_cuda().inputs_uniform_weights_device(n, seed, w_ptr, stream_ptr) != 0:
        raise RuntimeError("inputs_uniform_weights_device failed")


# --------------------------------------------------------------------------
# The five BASELINE.json configs (seeds [PROPOSED] there).
# --------------------------------------------------------------------------
PROB_VC, PROB_MIS, PROB_MWC = 1, 2, 3


@dataclass
class Config:
    index: int
    name: str
    problem: int
    generator: str
    params: dict
    beta: float
    epochs: int
    k: int = 0
    t_per_label: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def graph_seed(self):
        return 1311 * 10 + self.index

    @property
    def weight_seed(self):
        return 2661 * 10 + self.index

    @property
    def solve_seed(self):
        return 7 * 10 + self.index

    @property
    def round_seed(self):
        return 9 * 10 + self.index


CONFIGS = {
    "vc_er_1k": Config(1, "vc_er_1k", PROB_VC, "er", {"n": 1000, "m": 5000}, 10.0, 20),
    "mis_er_1m": Config(2, "mis_er_1m", PROB_MIS, "er", {"n": 1_000_000, "m": 5_000_000}, 10.0, 50),
    "vc_chunglu_10m": Config(3, "vc_chunglu_10m", PROB_VC, "chung_lu",
                             {"n": 10_000_000, "gamma": 2.1, "samples": 100_000_000}, 10.0, 50),
    "mwc_grid_2048": Config(4, "mwc_grid_2048", PROB_MWC, "grid", {"side": 2048}, 10.0, 30,
                            k=5, t_per_label=5),
    "vc_rmat_26": Config(5, "vc_rmat_26", PROB_VC, "rmat",
                         {"scale": 26, "samples": 16 << 26, "a": 0.57, "b": 0.19, "c": 0.19},
                         10.0, 20),
}


@dataclass
class GraphInput:
    n: int
    src: np.ndarray
    dst: np.ndarray
    vertex_w: np.ndarray | None
    edge_w: np.ndarray | None
    k: int = 0
    terminals: np.ndarray | None = None
    t_per_label: int = 0


def make_graph(cfg: Config, seed_offset: int = 0, **override) -> GraphInput:
    """Host generation of a config's raw input (override params for scaled samples)."""
    p = dict(cfg.params)
    p.update(override)
    gs = cfg.graph_seed + 1000 * seed_offset
    ws = cfg.weight_seed + 1000 * seed_offset
    if cfg.generator == "er":
        n = p["n"]
        src, dst = er(n, p["m"], gs)
    elif cfg.generator == "chung_lu":
        n = p["n"]
        src, dst = chung_lu(n, p["gamma"], p["samples"], gs)
    elif cfg.generator == "grid":
        n = p["side"] * p["side"]
        src, dst = grid(p["side"])
    elif cfg.generator == "rmat":
        n = 1 << p["scale"]
        src, dst = rmat(p["scale"], p["samples"], p["a"], p["b"], p["c"], gs)
    else:
        raise ValueError(cfg.generator)
    if cfg.problem == PROB_MWC:
        ew = exp_weights(len(src), ws)
        terms = terminals(n, cfg.k * cfg.t_per_label, gs ^ 0x5EED)
        return GraphInput(n, src, dst, None, ew, cfg.k, terms, cfg.t_per_label)
    vw = uniform_weights(n, ws)
    return GraphInput(n, src, dst, vw, None)
