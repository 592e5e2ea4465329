#!/usr/bin/env python
"""How far other schedules of the same coordinate steps move the 20-epoch point from Alg. 1's
permuted sweep (oracle MODE_ASYNC, fp64), on the config-5 recipe at a reduced R-MAT scale.

TEST INFRASTRUCTURE (runs the oracle).  Prints relative deviations of f_beta, c^T x and the
rounded VC cost for: other seeds of Alg. 1 itself (the algorithm's own spread), the
deterministic coloured order, windows of W tiles stepping together, all slacks first, the
hub schedules of tests/experiments/sched_variants.c, and the two replays (modes 3, 4).

  python tests/experiments/schedule_sensitivity.py [scale]
"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402


def lib():
    out = os.path.join(HERE, "libsched_variants.so")
    src = os.path.join(HERE, "sched_variants.c")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-DREAL=double",
                        "-I", os.path.join(ROOT, "oracle"), src, "-o", out, "-lm"], check=True)
    L = oracle.bind(ctypes.CDLL(out))
    L.exp_window.argtypes = [ctypes.c_void_p, ctypes.c_float, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                             ctypes.c_int64, ctypes.c_int]
    L.exp_hubs.argtypes = [ctypes.c_void_p, ctypes.c_float, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int64]
    return L


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    cfg = inputs.CONFIGS["vc_rmat_26"]
    g = inputs.make_graph(cfg, scale=scale, samples=16 << scale)
    L = lib()
    beta, ep, seed = cfg.beta, cfg.epochs, cfg.solve_seed

    def fresh():
        # the experiment library holds the oracle's code: build the LP with it
        h = ctypes.c_void_p()
        src, dst = np.ascontiguousarray(g.src, np.int32), np.ascontiguousarray(g.dst, np.int32)
        vw = np.ascontiguousarray(g.vertex_w, np.float32)
        rc = L.thetis_ref_build_graph_lp(ctypes.byref(h), 1, g.n, len(src), src.ctypes.data, dst.ctypes.data,
                                         vw.ctypes.data, None, 0, None, 0)
        assert rc == 0
        return oracle.RefLP(h, L, 64, None)

    def res(lp):
        o = lp.objective(beta)
        _, rr = lp.round(oracle.ROUND_VC_HALF)
        return o["f_beta"], o["lp_obj"], rr["cost"]

    print(f"R-MAT scale {scale}, beta {beta}, {ep} epochs, deviations relative to Alg. 1 (MODE_ASYNC, seed {seed})")
    for rule, rname in ((oracle.STEP_LMAX, "1/L_max"), (oracle.STEP_LJ, "1/L_j")):
        lp = fresh()
        lp.solve(beta, ep, mode=oracle.MODE_ASYNC, seed=seed, step_rule=rule)
        base = res(lp)
        rows = []

        def add(name, v):
            rows.append((name, [(v[i] - base[i]) / abs(base[i]) for i in range(3)]))

        for s2 in (seed + 1, seed + 2):
            lp = fresh(); lp.solve(beta, ep, mode=oracle.MODE_ASYNC, seed=s2, step_rule=rule)
            add(f"Alg. 1, seed {s2}", res(lp))
        for mode, name in ((oracle.MODE_DET, "coloured order (mode 0)"), (oracle.MODE_PI_TILE_SYNC, "mode 4"),
                           (oracle.MODE_HUBLAG_REPLAY, "hub-lag replay (mode 3)")):
            lp = fresh(); lp.solve(beta, ep, mode=mode, seed=seed, step_rule=rule)
            add(name, res(lp))
        n_tiles = (lp.U + 31) // 32
        for W in (16, 128, 1024):
            lp = fresh(); L.exp_window(lp._h, beta, ep, seed, rule, W, 0)
            add(f"windows of {W} tiles ({100 * W / n_tiles:.2f}%)", res(lp))
        lp = fresh(); L.exp_window(lp._h, beta, ep, seed, rule, 1, 1)
        add("all slacks first", res(lp))
        for sched, name in ((0, "hubs sequential before light tiles"), (1, "hubs synchronous, at once"),
                            (2, "hubs synchronous, after light tiles")):
            lp = fresh(); L.exp_hubs(lp._h, beta, ep, seed, rule, sched, 512)
            add(f"slacks first + {name}", res(lp))
        print(f"\nstep rule {rname}: Alg. 1 f_beta {base[0]:.6e}, c^T x {base[1]:.6e}, cover {base[2]:.6e}")
        print(f"{'schedule':48s} {'f_beta':>10s} {'c^T x':>10s} {'cover':>10s}")
        for name, d in rows:
            print(f"{name:48s} {d[0]:+10.2e} {d[1]:+10.2e} {d[2]:+10.2e}")


if __name__ == "__main__":
    main()
