"""The five BASELINE.json configs on the GPU (SURVEY §8(d) recipes).

Element-wise parity with the oracle where the oracle finishes in seconds (config 2 at full
size; configs 3 and 4 at reduced size, same recipe, spanning many tiles with ragged tails);
at full size (configs 3, 4, 5 in the launch configuration bench.py times) properties that
hold at any size: residual drift, bounds / simplex feasibility, monotone f_beta per epoch
in the deterministic mode (each class step is a descent step), rounding feasibility and the
Def. 1 / Lemma 1 cost bounds.
"""
import numpy as np
import pytest

import inputs
import oracle
from oracle import RefLP

pytestmark = pytest.mark.gpu

VC, MIS, MWC = 1, 2, 3


@pytest.fixture(scope="module")
def th():
    import paper_1311_2661_b200 as th
    return th


def gpu_lp(th, g, problem):
    if problem == MWC:
        return th.LP.from_graph(MWC, g.n, g.src, g.dst, edge_w=g.edge_w, k=g.k, terminals=g.terminals,
                                t_per_label=g.t_per_label)
    return th.LP.from_graph(problem, g.n, g.src, g.dst, vertex_w=g.vertex_w)


def ref_lp(g, problem, bits):
    if problem == MWC:
        return RefLP.graph(MWC, g.n, g.src, g.dst, edge_w=g.edge_w, k=g.k, terminals=g.terminals,
                           t_per_label=g.t_per_label, bits=bits)
    return RefLP.graph(problem, g.n, g.src, g.dst, vertex_w=g.vertex_w, bits=bits)


def rule_of(problem):
    return {VC: 1, MIS: 3, MWC: 4}[problem]


def det_parity(th, g, problem, cfg, epochs):
    lp = gpu_lp(th, g, problem)
    r32 = ref_lp(g, problem, 32)
    lp.solve(cfg.beta, epochs, mode=0, seed=cfg.solve_seed)
    r32.solve(cfg.beta, epochs, mode=0, seed=cfg.solve_seed)
    assert np.array_equal(lp.get_x().cpu().numpy(), r32.x32())
    assert np.array_equal(lp.get_r().cpu().numpy(), r32.r32())
    sel, res = lp.round(rule_of(problem), seed=cfg.round_seed, reps=10)
    rsel, rres = r32.round(rule_of(problem), seed=cfg.round_seed, reps=10)
    assert np.array_equal(sel.cpu().numpy(), rsel) and res["feasible"] == rres["feasible"] == 1
    assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12)
    return lp


def async_parity(th, g, problem, cfg, epochs):
    lp = gpu_lp(th, g, problem)
    r64 = ref_lp(g, problem, 64)
    lp.solve(cfg.beta, epochs, mode=1, seed=cfg.solve_seed)
    r64.solve(cfg.beta, epochs, mode=oracle.MODE_TILE_SYNC, seed=cfg.solve_seed)
    o, ro = lp.objective(cfg.beta), r64.objective(cfg.beta)
    assert o["f_beta"] == pytest.approx(ro["f_beta"], rel=1e-3)
    assert o["lp_obj"] == pytest.approx(ro["lp_obj"], rel=1e-3)
    _, res = lp.round(rule_of(problem), seed=cfg.round_seed, reps=10)
    _, rres = r64.round(rule_of(problem), seed=cfg.round_seed, reps=10)
    assert res["feasible"] == 1 and res["cost"] == pytest.approx(rres["cost"], rel=1e-2)


# ---------------------------------------------------------------- config 2 (full size)
def test_config2_mis_full_det_bit_exact(th):
    cfg = inputs.CONFIGS["mis_er_1m"]
    g = inputs.make_graph(cfg)
    det_parity(th, g, MIS, cfg, cfg.epochs)


def test_config2_mis_full_async(th):
    cfg = inputs.CONFIGS["mis_er_1m"]
    g = inputs.make_graph(cfg)
    async_parity(th, g, MIS, cfg, cfg.epochs)


# ---------------------------------------------------------------- config 3 (reduced + full)
def config3_reduced():
    cfg = inputs.CONFIGS["vc_chunglu_10m"]
    return cfg, inputs.make_graph(cfg, n=1_000_000, samples=10_000_000)


def test_config3_reduced_det_bit_exact(th):
    cfg, g = config3_reduced()
    det_parity(th, g, VC, cfg, 5)


def test_config3_reduced_async(th):
    cfg, g = config3_reduced()
    async_parity(th, g, VC, cfg, cfg.epochs)


# ---------------------------------------------------------------- config 4 (reduced + full)
def config4_reduced():
    cfg = inputs.CONFIGS["mwc_grid_2048"]
    return cfg, inputs.make_graph(cfg, side=256)


def test_config4_reduced_det_bit_exact(th):
    cfg, g = config4_reduced()
    lp = det_parity(th, g, MWC, cfg, cfg.epochs)
    x = lp.get_x().cpu().numpy()[: g.n * g.k].reshape(g.n, g.k)
    assert x.min() >= 0 and np.abs(x.sum(1) - 1).max() < 1e-5


def test_config4_reduced_async(th):
    cfg, g = config4_reduced()
    async_parity(th, g, MWC, cfg, cfg.epochs)


# ---------------------------------------------------------------- full size, properties
def full_size_properties(th, lp, problem, cfg, mode, epochs, vertex_w=None, check_monotone=True):
    beta = cfg.beta
    f_prev = lp.objective(beta)["f_beta"]
    for e in range(epochs):
        lp.solve(beta, 1, mode=mode, seed=cfg.solve_seed + 1000 * e)
        o = lp.objective(beta)
        assert o["nonfinite"] == 0
        assert o["drift_inf"] < 1e-3  # maintained r = A z - b up to fp32 rounding
        if check_monotone:
            assert o["f_beta"] <= f_prev * (1 + 1e-6) + 1e-6
        f_prev = o["f_beta"]
    z = lp.get_x()
    xs = z[: lp.n_struct]
    assert float(xs.min()) >= 0.0 and float(xs.max()) <= 1.0
    assert float(z[lp.n_struct:].min()) >= 0.0 if lp.N > lp.n_struct else True
    sel, res = lp.round(rule_of(problem), seed=cfg.round_seed, reps=10)
    assert res["feasible"] == 1
    return o, res, xs


@pytest.mark.parametrize("mode", [0, 1])
def test_config3_full_properties(th, mode):
    cfg = inputs.CONFIGS["vc_chunglu_10m"]
    g = inputs.make_graph(cfg)
    lp = gpu_lp(th, g, VC)
    o, res, xs = full_size_properties(th, lp, VC, cfg, mode, 3)
    eps = res["eps_or_alpha"]
    if eps < 1:  # Lemma 1 + P:139-146: cover cost <= 2 c^T x / (1 - eps)
        assert res["cost"] <= 2 * o["lp_obj"] / (1 - eps) * (1 + 1e-6)


def test_config4_full_properties(th):
    cfg = inputs.CONFIGS["mwc_grid_2048"]
    g = inputs.make_graph(cfg)
    lp = gpu_lp(th, g, MWC)
    full_size_properties(th, lp, MWC, cfg, 1, 3)
    x = lp.get_x()[: g.n * g.k].reshape(g.n, g.k)
    assert float(x.min()) >= 0 and float((x.sum(1) - 1).abs().max()) < 1e-5  # App. C.3
    lab, res = lp.round(4, seed=cfg.round_seed, reps=10)
    lab = lab.cpu().numpy()
    terms = g.terminals.reshape(g.k, g.t_per_label)
    for l in range(g.k):
        assert (lab[terms[l]] == l).all()


def test_config5_full_properties_bench_launch(th):
    # the bench workload in bench.py's launch configuration: async, STEP_LMAX, device inputs
    import torch
    cfg = inputs.CONFIGS["vc_rmat_26"]
    p = cfg.params
    n, E = 1 << p["scale"], p["samples"]
    src = torch.empty(E, dtype=torch.int32, device="cuda")
    dst = torch.empty(E, dtype=torch.int32, device="cuda")
    w = torch.empty(n, dtype=torch.float32, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    inputs.rmat_device(p["scale"], E, p["a"], p["b"], p["c"], cfg.graph_seed, src.data_ptr(), dst.data_ptr(), sp)
    inputs.uniform_weights_device(n, cfg.weight_seed, w.data_ptr(), sp)
    lp = th.LP.from_graph(VC, n, src, dst, vertex_w=w)
    del src, dst
    o, res, xs = full_size_properties(th, lp, VC, cfg, 1, 3)
    eps = res["eps_or_alpha"]
    assert res["cost"] <= float(w.double().sum())
    if eps < 1:
        assert res["cost"] <= 2 * o["lp_obj"] / (1 - eps) * (1 + 1e-6)


# ---------------------------------------------------------------- config 5 recipe, reduced
@pytest.mark.parametrize("rule", [0, 1])
def test_config5_reduced_async_matches_reference(th, rule):
    # R-MAT scale 18 with config 5's (a, b, c) and edge factor: hub tiles, the hub step, the
    # fused row pass and many concurrent light tiles (the bench's code path at reduced size)
    cfg = inputs.CONFIGS["vc_rmat_26"]
    g = inputs.make_graph(cfg, scale=18, samples=16 << 18)
    lp = gpu_lp(th, g, VC)
    r64 = ref_lp(g, VC, 64)
    lp.solve(cfg.beta, 8, mode=1, seed=cfg.solve_seed, step_rule=rule)
    r64.solve(cfg.beta, 8, mode=oracle.MODE_TILE_SYNC, seed=cfg.solve_seed, step_rule=rule)
    o, ro = lp.objective(cfg.beta), r64.objective(cfg.beta)
    assert o["f_beta"] == pytest.approx(ro["f_beta"], rel=1e-3)
    assert o["lp_obj"] == pytest.approx(ro["lp_obj"], rel=1e-3)
    assert o["drift_inf"] < 1e-4
    _, res = lp.round(1)
    _, rres = r64.round(1)
    assert res["feasible"] == 1 and res["cost"] == pytest.approx(rres["cost"], rel=1e-2)
