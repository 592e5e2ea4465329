"""Per-config epoch throughput on one B200 (GPU box only; writes one JSON line per run).

For each BASELINE.json config: build the LP through the C ABI from the seeded recipe
(configs 1-4 generated on the host, config 5 on the device), solve with the config's
beta and epochs, and report the median epoch time (CUDA events on the solve stream),
coordinate updates/s, nonzeros/s and the algorithmic bytes per epoch of SURVEY 8(d)
(20 n_s + 12 nnz_s + 16 m) over the measured HBM peak.  Deterministic mode runs a
bounded number of epochs where its per-class launches are slow (power-law colourings).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

RUNS = [  # (config, mode, step rule, epochs cap); modes: 0 det, 1 async (Alg. 1 order), 3 hub-lag
    ("vc_er_1k", 0, 0, None), ("vc_er_1k", 1, 0, None), ("vc_er_1k", 3, 0, None),
    ("mis_er_1m", 0, 0, None), ("mis_er_1m", 1, 0, None), ("mis_er_1m", 3, 0, None),
    ("vc_chunglu_10m", 0, 0, 3), ("vc_chunglu_10m", 1, 0, None), ("vc_chunglu_10m", 1, 1, None),
    ("vc_chunglu_10m", 3, 0, None),
    ("mwc_grid_2048", 0, 0, None), ("mwc_grid_2048", 1, 0, None), ("mwc_grid_2048", 3, 0, None),
    ("vc_rmat_26", 1, 0, None), ("vc_rmat_26", 1, 1, None), ("vc_rmat_26", 3, 0, None), ("vc_rmat_26", 3, 1, None),
    ("sc_1m", 0, 0, None), ("sc_1m", 1, 0, None),  # NEXT-3 set cover (not a BASELINE config)
]
MODE_NAME = {0: "det", 1: "async", 3: "hublag"}
PROBLEM = {"vc_er_1k": 1, "mis_er_1m": 2, "vc_chunglu_10m": 1, "mwc_grid_2048": 3, "vc_rmat_26": 1, "sc_1m": 0}


def set_cover_instance(n_elem=1_000_000, n_sets=200_000, mean_extra=4.0, seed=31):
    """synthetic set cover (NEXT-3): element a lies in 1 + Poisson(mean_extra) random sets
    (duplicates dropped); costs U[1, 10).  Returns the covering LP's CSC and CSR."""
    import numpy as np
    rng = np.random.default_rng(seed)
    k = 1 + rng.poisson(mean_extra, n_elem)
    elem = np.repeat(np.arange(n_elem, dtype=np.int64), k)
    sets = rng.integers(0, n_sets, len(elem))
    key = np.unique(elem * n_sets + sets)
    elem, sets = key // n_sets, key % n_sets
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(elem, minlength=n_elem))]).astype(np.int64)
    order = np.lexsort((elem, sets))
    colptr = np.concatenate([[0], np.cumsum(np.bincount(sets, minlength=n_sets))]).astype(np.int64)
    cost = (1.0 + 9.0 * rng.random(n_sets)).astype(np.float32)
    return (n_elem, n_sets, colptr, elem[order].astype(np.int32), rowptr, sets.astype(np.int32), cost)


def async_form(mode, prob, m):
    """the form THETIS_MODE_ASYNC takes (R-23; the library's rule, restated)"""
    if mode != 1:
        return None
    if prob not in (1, 2):
        return "residual"
    return "residual" if os.environ.get("THETIS_ASYNC_FORM") == "residual" else "colsum"


def main():
    import torch

    import inputs
    import paper_1311_2661_b200 as th

    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--modes", default=None, help="comma list of modes to run (0 det, 1 async, 3 hub-lag)")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = float(peaks["hbm_gbs"])
    dev = torch.device("cuda", 0)
    cache = {}
    for name, mode, rule, cap in RUNS:
        if a.only and a.only not in name:
            continue
        if a.modes and str(mode) not in a.modes.split(","):
            continue
        prob = PROBLEM[name]
        if name == "sc_1m":
            import numpy as np
            m_, n_, cp, ri, rp, ci, cost = cache.get(name) or set_cover_instance()
            cache = {name: (m_, n_, cp, ri, rp, ci, cost)}
            ones = np.ones(len(ri), np.float32)
            lp = th.LP.from_csc_csr(m_, n_, cp, ri, ones, rp, ci, ones, np.ones(m_, np.float32), cost,
                                    sense=np.full(m_, th.THETIS_GE, np.int8), device=dev)
            cfg = type("C", (), dict(beta=10.0, epochs=30, solve_seed=7))
        else:
            cfg = inputs.CONFIGS[name]
        if name == "sc_1m":
            pass
        elif name == "vc_rmat_26":
            p = cfg.params
            n, E = 1 << p["scale"], p["samples"]
            src = torch.empty(E, dtype=torch.int32, device=dev)
            dst = torch.empty(E, dtype=torch.int32, device=dev)
            w = torch.empty(n, dtype=torch.float32, device=dev)
            sp = torch.cuda.current_stream(dev).cuda_stream
            inputs.rmat_device(p["scale"], E, p["a"], p["b"], p["c"], cfg.graph_seed, src.data_ptr(), dst.data_ptr(), sp)
            inputs.uniform_weights_device(n, cfg.weight_seed, w.data_ptr(), sp)
            lp = th.LP.from_graph(prob, n, src, dst, vertex_w=w, device=dev)
            del src, dst
        else:
            g = cache.get(name) or inputs.make_graph(cfg)
            cache = {name: g}
            if prob == 3:
                lp = th.LP.from_graph(prob, g.n, g.src, g.dst, edge_w=g.edge_w, k=g.k, terminals=g.terminals,
                                      t_per_label=g.t_per_label, device=dev)
            else:
                lp = th.LP.from_graph(prob, g.n, g.src, g.dst, vertex_w=g.vertex_w, device=dev)
        epochs = cfg.epochs if cap is None else min(cap, cfg.epochs)
        st = lp.solve(cfg.beta, epochs, mode=mode, seed=cfg.solve_seed, step_rule=rule)
        ms = st["ms_per_epoch"]
        med = statistics.median(ms[1:] if len(ms) > 2 else ms)
        upd = st["coordinate_updates"] / max(st["epochs"], 1)
        nnz = st["nnz_processed"] / max(st["epochs"], 1)
        alg = 20 * lp.n_struct + 12 * lp.nnz_struct + 16 * lp.n_ineq
        ob = lp.objective(cfg.beta)
        extra = {}
        rules = {1: [("VC_HALF", th.THETIS_ROUND_VC_HALF)], 2: [("MIS_GREEDY", th.THETIS_ROUND_MIS_GREEDY),
                                                                 ("MIS_BANSAL", th.THETIS_ROUND_MIS_BANSAL)],
                 3: [("MWC_CKR", th.THETIS_ROUND_MWC_CKR)]}.get(prob, [])
        for rname, rrule in rules:  # device time of one rounding call (CUDA events, 10 repetitions)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            lp.round(rrule, seed=3, reps=10)  # warm-up
            e0.record(lp.stream)
            _, rr = lp.round(rrule, seed=3, reps=10)
            e1.record(lp.stream)
            e1.synchronize()
            extra["round_" + rname] = dict(ms=e0.elapsed_time(e1), cost=rr["cost"], feasible=rr["feasible"])
        if name == "sc_1m":
            for rname, rrule in (("SC_THRESHOLD", th.THETIS_ROUND_SC_THRESHOLD), ("SC_RANDOM", th.THETIS_ROUND_SC_RANDOM)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                lp.round(rrule, seed=3)
                e0.record(lp.stream)
                _, rr = lp.round(rrule, seed=3)
                e1.record(lp.stream)
                e1.synchronize()
                extra["round_" + rname] = dict(ms=e0.elapsed_time(e1), cost=rr["cost"], feasible=rr["feasible"])
            pass  # (lp_obj and eps are in every line)
        out = dict(config=name, form=async_form(mode, prob, lp.m), mode=MODE_NAME[mode], step_rule="LJ" if rule else "LMAX", epochs=epochs,
                   ms_epoch_median=med, eps=ob["max_violation_eps"], lp_obj=ob["lp_obj"],
                   ms_epoch_first=ms[0], updates_per_s=upd / med * 1e3, nnz_per_s=nnz / med * 1e3,
                   alg_bytes_per_epoch=alg, alg_GBps=alg / med / 1e6, frac_of_measured_hbm=alg / med / 1e6 / peak,
                   colours=st["n_colours"], n_struct=lp.n_struct, m=lp.m, nnz_struct=lp.nnz_struct,
                   f_beta=ob["f_beta"], drift_inf=ob["drift_inf"],
                   ms_row_pass=st["ms_row_pass"] / max(st["row_pass_launches"], 1),
                   ms_hub_update=st["ms_hub_update"] / epochs, ms_tiles=st["ms_tiles"] / epochs, **extra)
        print(json.dumps(out), flush=True)
        del lp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
