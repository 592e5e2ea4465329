#!/usr/bin/env python
"""bench.py — the Thetis hot path on B200 (BASELINE.json metric).

A step is one pass of the whole hot path over one synthetic instance of the
workload: LP build from the edge list (K1-K3: canonicalise / dedup / CSC /
L_max / r0), the SCD epochs (THETIS_MODE_ASYNC: Alg. 1's per-epoch permuted sweep
run Hogwild-style, the mode whose trajectory is checked against the oracle's
Alg. 1 in tests/), the fused reductions (K9) and the rounding pass (K10).
The colouring (K4) belongs to the deterministic mode and is not on this
workload's path (BASELINE: config 5 runs in async mode).

Workload (N=1): BASELINE.json configs[4], the largest vertex-cover graph, on
which the north-star target (>= 60% of the HBM roofline per epoch) is stated:
R-MAT scale 26, 16*2^26 edge samples (a,b,c) = (0.57,0.19,0.19), weights
U[1,10), beta = 10, 20 async epochs, Lemma-1 rounding.  Inputs are generated
on the device (inputs/gen_cuda.cu) before timing; they exceed the 126 MB L2.
Beside the headline, `variants` times the same 20 epochs under the hub-lag
throughput schedule (THETIS_MODE_ASYNC_HUBLAG, R-22) and under the
1/L_j step rule.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun): replicas only — the path does not shard (DESIGN.md
§Multi-GPU); each rank solves its own instance (seed offset by rank),
value = all ranks' coordinate updates / max-over-ranks time, scaling "weak".
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "coordinate updates/sec & HBM GB/s (fraction of roofline) per SCD epoch, 1 B200"
CFG_NAME = "vc_rmat_26"
BETA = 10.0
EPOCHS = 20
REF_SAMPLE_SCALE = 18  # bounded CPU sample: R-MAT scale 18, same (a,b,c), edge factor 16


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="thetis", choices=["thetis", "reference"])
    p.add_argument("--scale", type=int, default=None, help="R-MAT scale override (testing only)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-variants", action="store_true", help="skip the hub-lag / STEP_LJ variant epochs")
    return p.parse_args()


def max_over_ranks(x: float, device=None) -> float:
    """max of a host scalar over all ranks (NCCL on the GPU, gloo on the CPU); the value
    itself when not distributed"""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_step_per_rank: float, steps: int, world: int, ms_max: float) -> float:
    """whole-job throughput: the units all ranks processed over the max-over-ranks time"""
    return units_per_step_per_rank * steps * world / (ms_max / 1e3)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def algorithmic_bytes(n_s, nnz_s, m):
    # SURVEY §8(d) / DESIGN.md: 20 B per structural coordinate, 12 B per structural
    # nonzero, 16 B per slack coordinate (r-resident design, +-1 coefficients)
    return 20 * n_s + 12 * nnz_s + 16 * m


def ncu_summary():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# random RED rate into an L2-resident array on this part (tools/microbench_l2_red.cu,
# profiles/r02_l2_red_microbench.txt: 220 G/s for fp32 and fp64, 22 MB and 48 MB arrays)
L2_RED_PEAK_GOPS = 220.0
# random ld.global.cg.f32 rate from an L2-resident array, same microbenchmark
L2_READ_PEAK_GOPS = 255.0


def ncu_traffic():
    """DRAM bytes of one SCD epoch (its kernels' dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed ncu summary (tools/profile_round.sh + tools/ncu_summary.py), or None"""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("epoch_dram_bytes")
    except Exception:
        return None


def l2_ops(ep_ms):
    sm = ncu_summary()
    red, rd = sm.get("l2_red_sectors"), sm.get("l2_read_sectors")
    if red is None or not rd:
        return None
    return {"bound": "l2 random 32-byte sector operations (reads of x; REDs when slacks move)",
            "read_sectors": rd, "red_sectors": red, "achieved_Gsectors_per_s": (red + rd) / ep_ms / 1e6,
            "peak_read_Gsectors_per_s": L2_READ_PEAK_GOPS, "peak_red_Gsectors_per_s": L2_RED_PEAK_GOPS,
            "frac_of_read_peak": (red + rd) / ep_ms / 1e6 / L2_READ_PEAK_GOPS,
            "source": "sector counts: profiles/ncu_summary.json (one k_async_pi launch under ncu --set full); peaks: "
                      "tools/microbench_l2_red.cu on this pool (profiles/r02_l2_red_microbench.txt); time: this run"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)"""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_thetis(args):
    import torch

    import inputs
    import paper_1311_2661_b200 as th

    ws_n, rank, local = dist_env()
    torch.cuda.set_device(local)  # before the process group: NCCL binds each rank to its own GPU
    if ws_n > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg = inputs.CONFIGS[CFG_NAME]
    p = dict(cfg.params)
    if args.scale:
        p["scale"], p["samples"] = args.scale, 16 << args.scale
    n, E = 1 << p["scale"], p["samples"]
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream
    # inputs resident in HBM (generated on the device; > L2)
    src = torch.empty(E, dtype=torch.int32, device=dev)
    dst = torch.empty(E, dtype=torch.int32, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    gseed = cfg.graph_seed + 1000 * rank
    with torch.cuda.stream(stream):
        inputs.rmat_device(p["scale"], E, p["a"], p["b"], p["c"], gseed, src.data_ptr(), dst.data_ptr(), sp)
        inputs.uniform_weights_device(n, cfg.weight_seed + 1000 * rank, w.data_ptr(), sp)
    stream.synchronize()
    need = ctypes.c_size_t()
    th._check(th.thetis_build_graph_lp_workspace(th.THETIS_PROB_VC, n, E, 0, ctypes.byref(need)), "workspace")
    ws = torch.empty(int(need.value), dtype=torch.uint8, device=dev)
    sel = torch.empty(n, dtype=torch.uint8, device=dev)
    info = {}

    def step(src_p, dst_p, w_p, out_p, record=None, mode=None, rule=None, start=False):
        h = ctypes.c_void_p()
        th._check(th.thetis_build_graph_lp(ctypes.byref(h), ws.data_ptr(), ws.numel(), sp, th.THETIS_PROB_VC, n, E,
                                           src_p, dst_p, w_p, None, 0, None, 0), "build")
        if start and record is not None:  # f_beta at z0 (progress measure; outside the timed region)
            ob0 = th.Objective()
            th._check(th.thetis_objective(h, BETA, ctypes.byref(ob0)), "objective", h)
            record["ob0"] = ob0
        st = th.SolveStats()
        th._check(th.thetis_solve(h, BETA, EPOCHS, th.THETIS_MODE_ASYNC if mode is None else mode, cfg.solve_seed,
                                  th.THETIS_STEP_LMAX if rule is None else rule, ctypes.byref(st)), "solve", h)
        ob = th.Objective()
        th._check(th.thetis_objective(h, BETA, ctypes.byref(ob)), "objective", h)
        rr = th.RoundResult()
        th._check(th.thetis_round(h, th.THETIS_ROUND_VC_HALF, cfg.round_seed, 1, out_p, ctypes.byref(rr)), "round", h)
        d = th.Dims()
        th.thetis_get_dims(h, ctypes.byref(d))
        th.thetis_free(h)
        if record is not None:
            record.update(dict(st=st, ob=ob, rr=rr, dims=d))

    def barrier():
        if ws_n > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up
    for i in range(args.warmup):
        step(src.data_ptr(), dst.data_ptr(), w.data_ptr(), sel.data_ptr(), info, start=i == 0)
    stream.synchronize()
    # timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    epoch_ms, recs = [], []
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            rec = {}
            step(src.data_ptr(), dst.data_ptr(), w.data_ptr(), sel.data_ptr(), rec)
            epoch_ms += list(rec["st"].ms_per_epoch)[:EPOCHS]
            recs.append(rec)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1), dev)
    clocks = clk.summary()
    last = recs[-1]
    dims = last["dims"]
    upd_step = last["st"].coordinate_updates
    nnz_step = last["st"].nnz_processed
    value = job_throughput(upd_step, args.steps, ws_n, ms)
    ep_med = statistics.median(epoch_ms)
    # live per-kernel device time of the epoch's launches (CUDA events on the solve stream)
    b_epoch = algorithmic_bytes(dims.n_struct, dims.nnz_struct, dims.m)
    peak, peak_src = load_peaks()
    achieved = b_epoch / (ep_med / 1e3) / 1e9

    # the same workload under the hub-lag throughput variant (R-22) and under STEP_LJ
    # (SURVEY A-4): 20 epochs each on the same LP, timed per epoch (not the headline)
    variants = {}
    if not args.no_variants:
        for name, mode, rule in (("hublag_lmax", th.THETIS_MODE_ASYNC_HUBLAG, th.THETIS_STEP_LMAX),
                                 ("async_lj", th.THETIS_MODE_ASYNC, th.THETIS_STEP_LJ)):
            rec = {}
            step(src.data_ptr(), dst.data_ptr(), w.data_ptr(), sel.data_ptr(), rec, mode=mode, rule=rule)
            x = rec["st"]
            med = statistics.median(list(x.ms_per_epoch)[:EPOCHS])
            v = {"mode": mode, "step_rule": rule, "epoch_ms_median": med,
                 "updates_per_s": x.coordinate_updates / EPOCHS / (med / 1e3),
                 "GBps": b_epoch / (med / 1e3) / 1e9, "frac": b_epoch / (med / 1e3) / 1e9 / peak,
                 "f_beta": rec["ob"].f_beta, "lp_obj": rec["ob"].lp_obj,
                 "max_violation_eps": rec["ob"].max_violation_eps, "cover_cost": rec["rr"].cost}
            if x.row_pass_launches:
                ne = min(int(x.epochs), 64)
                v["kernels_ms_per_launch"] = {"k_rows_pass": x.ms_row_pass / x.row_pass_launches,
                                              "k_hub_update": x.ms_hub_update / ne, "k_async": x.ms_tiles / ne}
            variants[name] = v

    # end to end through the C ABI with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        hsrc = torch.empty(E, dtype=torch.int32, pin_memory=True)
        hdst = torch.empty(E, dtype=torch.int32, pin_memory=True)
        hw = torch.empty(n, dtype=torch.float32, pin_memory=True)
        hsel = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        hsrc.copy_(src.cpu())
        hdst.copy_(dst.cpu())
        hw.copy_(w.cpu())
        step(hsrc.data_ptr(), hdst.data_ptr(), hw.data_ptr(), hsel.data_ptr())  # warm
        stream.synchronize()
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ke = max(1, min(args.steps, 3))
        for _ in range(ke):
            step(hsrc.data_ptr(), hdst.data_ptr(), hw.data_ptr(), hsel.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3), dev)
        e2e = {"value": job_throughput(upd_step, ke, ws_n, ms_e2e), "unit": "coordinate updates/s",
               "h2d_bytes_per_step": 8 * E + 4 * n, "d2h_bytes_per_step": n + ctypes.sizeof(th.RoundResult),
               "ms_per_step": ms_e2e / ke}

    # kernel launches of one step, counted by the CUDA profiler (CUPTI), not estimated
    launches = count_launches(lambda: step(src.data_ptr(), dst.data_ptr(), w.data_ptr(), sel.data_ptr()), stream)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and ws_n == 1:
        cpu = cpu_baseline()
    if ws_n > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    ob, rr = last["ob"], last["rr"]
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "coordinate updates/s",
        "n_gpus": ws_n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (R-MAT generated on device from seed; BASELINE configs[4])",
        "config": {"workload": f"{CFG_NAME}: VC LP of R-MAT scale {p['scale']} ({E} edge samples, a,b,c = "
                               f"{p['a']},{p['b']},{p['c']}), weights U[1,10), beta {BETA}, {EPOCHS} async "
                               "epochs (THETIS_MODE_ASYNC: Alg. 1's permuted sweep, Hogwild, column-sum form "
                               "R-23 (pull); STEP_LMAX), VC_HALF rounding",
                   "step": "build + 20 SCD epochs + reductions + rounding",
                   "vertices": n, "unique_edges_rows": int(dims.m), "coordinates": int(dims.N),
                   "nnz_struct": int(dims.nnz_struct), "l2": "inputs (8.6 GB edge list) and state exceed the L2",
                   "parallelism": "replicas" if ws_n > 1 else "single GPU"},
        "epoch": {"ms_median": ep_med, "ms_first": epoch_ms[0], "updates_per_s": upd_step / EPOCHS / (ep_med / 1e3),
                  "nnz_per_s": nnz_step / EPOCHS / (ep_med / 1e3), "alg_bytes": b_epoch,
                  "GBps": achieved, "frac_of_8TBps_nominal": achieved / 8000.0},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(),
                     "traffic_source": "profiles/ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum of "
                                       "one k_async_pi launch (ncu --set full on this command), not measured in "
                                       "this run",
                     "kernel": "k_async_pi<kGD>: one SCD epoch of THETIS_MODE_ASYNC in column-sum form (one launch per "
                               "epoch; CUDA events around each epoch on the launching stream; SURVEY 8(d) bytes "
                               "per epoch)",
                     "peak_source": peak_src,
                     # the kernel is not DRAM-bound: its epoch is set by random L2 sector reads (x, once per
                     # structural nonzero from its column's tile and once from its row's slack tile).
                     # Sector counts from the committed ncu capture, time live.
                     "l2_ops": l2_ops(ep_med)},
        "result": {"lp_obj": ob.lp_obj, "f_beta": ob.f_beta, "max_violation_eps": ob.max_violation_eps,
                   "drift_inf": ob.drift_inf, "cover_cost": rr.cost, "feasible": int(rr.feasible),
                   "selected": int(rr.n_selected)},
        "progress": {"f_beta_start": info["ob0"].f_beta if "ob0" in info else None, "f_beta_end": ob.f_beta,
                     "eps_start": info["ob0"].max_violation_eps if "ob0" in info else None,
                     "eps_end": ob.max_violation_eps,
                     "note": "20 epochs of Alg. 1 with 1/L_max (Eq. 7) on R-MAT: L_max ~ beta * max degree, so "
                             "steps are small; variants.async_lj shows the same epochs with 1/L_j"},
        "variants": variants or None,
        "e2e": e2e,
        "gpu_launches": launches * args.steps if launches is not None else None,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)


def count_launches(fn, stream):
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.cuda.stream(stream):
                fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [nm for nm in names if not nm.lower().startswith(("memset", "memcpy")) and "at::" not in nm]
        return len(ours)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# oracle: cpu_baseline and the reference arm
# ---------------------------------------------------------------------------
def oracle_step(sample):
    import oracle
    src, dst, w, n = sample
    t0 = time.perf_counter()
    lp = oracle.RefLP.graph(oracle.PROB_VC, n, src, dst, vertex_w=w)
    t1 = time.perf_counter()
    st = lp.solve(BETA, EPOCHS, mode=oracle.MODE_ASYNC, seed=75, step_rule=oracle.STEP_LMAX)
    t2 = time.perf_counter()
    lp.objective(BETA)
    lp.round(oracle.ROUND_VC_HALF)
    t3 = time.perf_counter()
    return st["coordinate_updates"], t3 - t0, t2 - t1


def ref_sample():
    import inputs
    cfg = inputs.CONFIGS[CFG_NAME]
    p = cfg.params
    s = REF_SAMPLE_SCALE
    src, dst = inputs.rmat(s, 16 << s, p["a"], p["b"], p["c"], cfg.graph_seed)
    w = inputs.uniform_weights(1 << s, cfg.weight_seed)
    return src, dst, w, 1 << s


SAMPLE_DESC = (f"the same recipe at R-MAT scale {REF_SAMPLE_SCALE} ({1 << REF_SAMPLE_SCALE} vertices, "
               f"{16 << REF_SAMPLE_SCALE} samples): build + {EPOCHS} epochs of Alg. 1 in the permuted order "
               "(oracle MODE_ASYNC, the async reference trajectory) + reductions + rounding, oracle fp64, "
               "one thread pinned to one core")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class PinnedCore:
    """Run the oracle on one host core (SURVEY §8(d) "Timing, oracle": taskset -c 0 equivalent)."""

    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = min(self.prev)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *a):
        if self.prev:
            os.sched_setaffinity(0, self.prev)


def host_info(core):
    return {"cpu_model": cpu_model(), "pinned_core": core, "host_cores": os.cpu_count(),
            "threads_used": "1 of %s cores" % os.cpu_count()}


def cpu_baseline():
    sample = ref_sample()
    with PinnedCore() as pc:
        upd, t, t_ep = oracle_step(sample)
    return {"value": upd / t, "unit": "coordinate updates/s", "cores": 1, "kind": "oracle",
            "sample": SAMPLE_DESC, "epoch_updates_per_s": upd / t_ep, "seconds": t, **host_info(pc.core)}


def run_reference(args):
    ws_n, rank, _ = dist_env()
    if rank != 0:
        return
    sample = ref_sample()
    tot_t, tot_u = 0.0, 0
    with PinnedCore() as pc:
        for _ in range(args.warmup):
            oracle_step(sample)
        for _ in range(args.steps):
            u, t, _ = oracle_step(sample)
            tot_t += t
            tot_u += u
    v = tot_u / tot_t
    out = {"metric": METRIC, "value": v, "unit": "coordinate updates/s", "n_gpus": ws_n, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{CFG_NAME} (bounded CPU sample)", "sample": SAMPLE_DESC},
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": "coordinate updates/s", "cores": 1, "kind": "oracle",
                            "sample": SAMPLE_DESC, **host_info(pc.core)},
           "e2e": {"value": v, "unit": "coordinate updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_thetis(a)
