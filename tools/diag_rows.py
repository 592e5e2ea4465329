"""Row-pass diagnostics on the bench workload (GPU box only; not part of the product).

Builds the config-5 LP (or --scale S) through the C ABI, prints the hub structure
(hub tiles, hub rows, max-side runs) and the per-kernel times of a short async solve.
Run once per THETIS_EXP value (the library reads it at load) to split the row pass.
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import inputs
    import paper_1311_2661_b200 as th

    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--epochs", type=int, default=6)
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--mode", type=int, default=1, help="1 async (Alg. 1 order), 3 hub-lag")
    ap.add_argument("--rule", type=int, default=0, help="0 1/L_max, 1 1/L_j")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = inputs.CONFIGS["vc_rmat_26"]
    p = dict(cfg.params)
    n, E = 1 << a.scale, 16 << a.scale
    s = torch.cuda.Stream(dev)
    sp = s.cuda_stream
    src = torch.empty(E, dtype=torch.int32, device=dev)
    dst = torch.empty(E, dtype=torch.int32, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    with torch.cuda.stream(s):
        inputs.rmat_device(a.scale, E, p["a"], p["b"], p["c"], cfg.graph_seed, src.data_ptr(), dst.data_ptr(), sp)
        inputs.uniform_weights_device(n, cfg.weight_seed, w.data_ptr(), sp)
    s.synchronize()
    need = ctypes.c_size_t()
    th._check(th.thetis_build_graph_lp_workspace(th.THETIS_PROB_VC, n, E, 0, ctypes.byref(need)), "ws")
    ws = torch.empty(int(need.value), dtype=torch.uint8, device=dev)
    h = ctypes.c_void_p()
    tev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    tev[0].record(s)
    th._check(th.thetis_build_graph_lp(ctypes.byref(h), ws.data_ptr(), ws.numel(), sp, th.THETIS_PROB_VC, n, E,
                                       src.data_ptr(), dst.data_ptr(), w.data_ptr(), None, 0, None, 0), "build")
    tev[1].record(s)
    del src, dst
    d = th.Dims()
    th.thetis_get_dims(h, ctypes.byref(d))
    out = {"exp": os.environ.get("THETIS_EXP", "0"), "m": d.m, "n": d.n_vertices, "nnz": d.nnz_struct}
    if a.stats:
        eu = torch.empty(d.m, dtype=torch.int32, device=dev)
        ev = torch.empty(d.m, dtype=torch.int32, device=dev)
        th._check(th.thetis_get_edges(h, eu.data_ptr(), ev.data_ptr()), "edges")
        torch.cuda.synchronize()
        inc = torch.bincount((eu >> 5).long(), minlength=(n + 31) // 32) + \
            torch.bincount((ev >> 5).long(), minlength=(n + 31) // 32)
        hub = inc > 512
        out["hub_tiles"] = int(hub.sum())
        out["hub_tile_nnz_frac"] = float(inc[hub].sum()) / float(inc.sum())
        li = inc[~hub]
        out["light_tiles"] = int(li.numel())
        out["light_nnz"] = int(li.sum())
        out["light_tiles_empty"] = int((li == 0).sum())
        out["light_tile_nnz_pct"] = [int(x) for x in torch.quantile(li.float()[:1 << 24], torch.tensor([0.5, 0.9, 0.99], device=dev)).tolist()]
        hv = hub[(ev >> 5).long()]
        mh = int(hv.sum())
        out["hub_rows"] = mh
        hu = hub[(eu >> 5).long()]
        out["rows_min_hub"] = int(hu.sum())
        out["rows_both_hub"] = int((hu & hv).sum())
        u, v = eu[:mh].long(), ev[:mh].long()
        key = (u >> 14) * (1 << 32) + v
        out["max_runs_u_ranged"] = int((key[1:] != key[:-1]).sum()) + 1
        # alternative: v-ranged (v >> 14, u): distinct pairs among hub-min rows
        sel = hu[:mh]
        k2 = torch.unique((v[sel] >> 14) * (1 << 32) + u[sel])
        out["min_pairs_v_ranged"] = int(k2.numel())
        # distinct (range_u, v) pairs of all rows with hub v
        for lg in (18, 20, 22):  # rows with both endpoints below 2^lg (a dense corner for 2D tiling)
            out["rows_both_below_2^%d" % lg] = int(((u < (1 << lg)) & (v < (1 << lg))).sum())
        del u, v, key, k2, eu, ev
        torch.cuda.empty_cache()
    st = th.SolveStats()
    th._check(th.thetis_solve(h, 10.0, a.epochs, a.mode, cfg.solve_seed, a.rule,
                              ctypes.byref(st)), "solve", h)
    eps = list(st.ms_per_epoch[:a.epochs])
    out.update(epoch_ms=sorted(eps)[len(eps) // 2], row_pass_ms=st.ms_row_pass / max(1, st.row_pass_launches),
               hub_update_ms=st.ms_hub_update / a.epochs, tiles_ms=st.ms_tiles / a.epochs)
    tev[2].record(s)
    ob = th.Objective()
    th._check(th.thetis_objective(h, 10.0, ctypes.byref(ob)), "obj", h)
    tev[3].record(s)
    sel = torch.empty(n, dtype=torch.uint8, device=dev)
    rr = th.RoundResult()
    th._check(th.thetis_round(h, th.THETIS_ROUND_VC_HALF, cfg.round_seed, 1, sel.data_ptr(), ctypes.byref(rr)), "round", h)
    tev[4].record(s)
    s.synchronize()
    out["f_beta"] = ob.f_beta
    out["ms_build"] = tev[0].elapsed_time(tev[1])
    out["ms_solve_setup_and_epochs"] = tev[1].elapsed_time(tev[2])
    out["ms_objective"] = tev[2].elapsed_time(tev[3])
    out["ms_round"] = tev[3].elapsed_time(tev[4])
    th.thetis_free(h)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
