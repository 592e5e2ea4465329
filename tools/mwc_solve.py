"""Config 4 (MWC grid) async solve for profiling (GPU box only): build, 3 async epochs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import inputs
    import paper_1311_2661_b200 as th
    cfg = inputs.CONFIGS["mwc_grid_2048"]
    g = inputs.make_graph(cfg)
    lp = th.LP.from_graph(3, g.n, g.src, g.dst, edge_w=g.edge_w, k=g.k, terminals=g.terminals,
                          t_per_label=g.t_per_label)
    st = lp.solve(cfg.beta, 3, mode=th.THETIS_MODE_ASYNC, seed=cfg.solve_seed)
    print("epochs ms", st["ms_per_epoch"])


if __name__ == "__main__":
    main()
