#!/usr/bin/env python
"""GPU async vs the oracle's Alg. 1 trajectory (MODE_ASYNC) on scaled config recipes.

  python tests/async_check.py CASE[,CASE...] [--modes 1,3] [--rules 0,1]

CASE = cfgname[:scale-or-size]: vc_rmat_26:20, vc_er_1k, mis_er_1m, vc_chunglu_10m:1000000,
mwc_grid_2048:256.  Prints per case / mode / rule the relative deviations of f_beta, c^T x and
the rounded cost from the fp64 oracle run with the same seed, and the GPU epoch time.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # (tests/ helper: it runs the oracle)
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1311_2661_b200 as th  # noqa: E402

CACHE = os.environ.get("ASYNC_CHECK_CACHE", os.path.join(ROOT, "gpurun_out", "oracle_cache.json"))


def graph_of(case):
    name, _, arg = case.partition(":")
    cfg = inputs.CONFIGS[name]
    if not arg:
        return cfg, inputs.make_graph(cfg)
    a = int(arg)
    if cfg.generator == "rmat":
        return cfg, inputs.make_graph(cfg, scale=a, samples=16 << a)
    if cfg.generator == "chung_lu":
        return cfg, inputs.make_graph(cfg, n=a, samples=10 * a)
    if cfg.generator == "grid":
        return cfg, inputs.make_graph(cfg, side=a)
    if cfg.generator == "er":
        return cfg, inputs.make_graph(cfg, n=a, m=5 * a)
    raise ValueError(case)


def rule_round(cfg):
    return {1: th.THETIS_ROUND_VC_HALF, 2: th.THETIS_ROUND_MIS_GREEDY, 3: th.THETIS_ROUND_MWC_CKR}[cfg.problem]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases")
    ap.add_argument("--modes", default="1")
    ap.add_argument("--rules", default="0,1")
    ap.add_argument("--epochs", type=int, default=0)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--forms", default="auto", help="THETIS_ASYNC_FORM values for mode 1 on VC / MIS: "
                                                    "auto (the library's rule), residual, colsum")
    a = ap.parse_args()
    cache = json.load(open(CACHE)) if os.path.exists(CACHE) else {}
    for case in a.cases.split(","):
        cfg, g = graph_of(case)
        ep = a.epochs or cfg.epochs
        kw = dict(vertex_w=g.vertex_w, edge_w=g.edge_w, k=g.k, terminals=g.terminals, t_per_label=g.t_per_label)
        for rule in [int(x) for x in a.rules.split(",")]:
            base = None
            key = f"{case}|{rule}|{ep}"
            if key in cache:
                base = tuple(cache[key])
            elif not a.no_oracle:
                t0 = time.time()
                ref = oracle.RefLP.graph(cfg.problem, g.n, g.src, g.dst, **kw)
                ref.solve(cfg.beta, ep, mode=oracle.MODE_ASYNC, seed=cfg.solve_seed, step_rule=rule)
                o = ref.objective(cfg.beta)
                _, rr = ref.round(rule_round(cfg), seed=cfg.round_seed)
                base = (o["f_beta"], o["lp_obj"], rr["cost"])
                cache[key] = base
                json.dump(cache, open(CACHE, "w"))
                print(f"{case} rule {rule} oracle f={base[0]:.9e} cx={base[1]:.9e} cost={base[2]:.9e} "
                      f"({time.time() - t0:.1f}s)", flush=True)
            runs = []
            for mode in [int(x) for x in a.modes.split(",")]:
                forms = a.forms.split(",") if mode == 1 and cfg.problem in (1, 2) else ["auto"]
                runs += [(mode, f) for f in forms]
            for mode, form in runs:
                if form == "auto":
                    os.environ.pop("THETIS_ASYNC_FORM", None)
                else:
                    os.environ["THETIS_ASYNC_FORM"] = form
                lp = th.LP.from_graph(cfg.problem, g.n, g.src, g.dst, device="cuda:0", **kw)
                st = lp.solve(cfg.beta, ep, mode=mode, seed=cfg.solve_seed, step_rule=rule)
                o = lp.objective(cfg.beta)
                _, rr = lp.round(rule_round(cfg), seed=cfg.round_seed)
                v = (o["f_beta"], o["lp_obj"], rr["cost"])
                ms = np.median(st["ms_per_epoch"]) if st["ms_per_epoch"] else 0.0
                msg = f"{case} rule {rule} mode {mode} form {form} f={v[0]:.9e} cx={v[1]:.9e} cost={v[2]:.9e} ms/epoch={ms:.3f}"
                if base:
                    d = [(v[i] - base[i]) / abs(base[i]) if base[i] else 0.0 for i in range(3)]
                    msg += f" | df={d[0]:+.2e} dcx={d[1]:+.2e} dcost={d[2]:+.2e} drift={o['drift_inf']:.1e}"
                print(msg, flush=True)
                del lp


if __name__ == "__main__":
    main()
