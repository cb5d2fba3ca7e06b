"""Stage-1 benchmark: candidates evaluated/sec and stage-1 solve time on B200.

One step = one full stage-1 solve of BASELINE config 2 (catalog.extended_scenario:
6 models x 20 node configs x 3 regions, caps (6, 12)): T-hat tables -> enumeration
-> placement-DP evaluation of every (model, phase, combo) candidate -> per-region
frontier (+ NCCL all-gather and merge when N > 1). Spec tables are uploaded to HBM
before the timed region (`value`); `e2e` times the public API build_frontier() from
host spec objects to frontier ServingTemplate objects, H2D/D2H included.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Rank 0 prints ONE JSON line. Under torchrun each rank evaluates an interleaved
candidate shard; time = max over ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidates evaluated/sec"
UNIT = "candidates/s"
WORKLOAD = "c2"
RECORD_BYTES = 32          # coral_s1_record written per candidate
KEY_BYTES = 8              # packed combo key read per candidate
CPU_SAMPLE_STRIDE = 61     # every 61st candidate of each (model, phase) for the CPU leg


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--c5", action="store_true", help="(default) also time BASELINE config 5")
    ap.add_argument("--no-c5", action="store_true", help="skip the BASELINE config 5 solve (seconds)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def cpu_baseline(workload: str, stride: int = CPU_SAMPLE_STRIDE):
    """The CPU restatement of the reference (oracle/, a C port of the numba path) on a
    stride sample of the same candidates, all host threads. Returns (cand/s, n, s)."""
    from oracle.oracle import OracleProblem
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.library import GenContext, LibraryCaps
    w = catalog.WORKLOADS[workload]()
    op = OracleProblem.from_specs(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                                  GenContext(perf=w.perf, granularity=w.granularity),
                                  ("prefill", "decode"))
    work = []
    for mi in range(len(w.models)):
        keys = op.enumerate(mi)
        for code in (0, 1):
            work.append((mi, code, keys, op.tables(mi, code)))
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    n = 0
    for mi, code, keys, tabs in work:
        op.solve(mi, code, keys, 0, stride, tables=tabs, threads=threads)
        n += (len(keys) + stride - 1) // stride
    dt = time.perf_counter() - t0
    return n / dt, n, dt, threads


class ClockSampler:
    """`nvidia-smi -lms 20` streamed during the timed region: SM clocks + throttle reasons."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._t = None

    def _reader(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.3)  # first samples before the timed region starts
        except OSError:
            self._p = None
        return self

    def __exit__(self, *exc):
        if self._p is not None:
            time.sleep(0.05)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = sorted(v for v in (num(s[1]) for s in self.samples) if v is not None)
        mx = max((v for v in (num(s[2]) for s in self.samples) if v is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[5 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


BASELINE_CONFIG = {"c1": "BASELINE config 1: Llama-3-8B x {A100, L4} x {1,2,4,8}, small pool",
                   "extended": "BASELINE config 2: 6 models x 20 node configs x 3 regions",
                   "c2": "BASELINE config 2: 6 models x 20 node configs x 3 regions",
                   "c3": "BASELINE config 3: llama3-70b, 20 configs, granularity 1 (Lu = 80)",
                   "c5": "BASELINE config 5: 50 synthetic models x 40 node configs x 3 regions",
                   "core": "reference core scenario: 3 models x 12 configs x 2 regions"}


def workload_label(name: str) -> str:
    from paper_2605_04357_b200 import catalog
    w = catalog.WORKLOADS[name]()
    return f"{w.name} ({BASELINE_CONFIG.get(name, name)})"


def onchip_calibration():
    """Per-pair instruction / L1-wavefront costs of the two lattice search kernels from
    the committed ncu capture (tools/onchip_calib.py -> profiles/r02_onchip_calib.json),
    and the measured on-chip peaks (tools/onchip_peaks.cu -> profiles/r01_onchip_peaks.json)."""
    out = {}
    for name in ("r02_onchip_calib.json", "r01_onchip_peaks.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                out[name] = json.load(fh)
        except (OSError, ValueError):
            out[name] = {}
    return out["r02_onchip_calib.json"], out["r01_onchip_peaks.json"]


def lattice_states(K: int, n_max: int) -> int:
    """Multisets of 1..n_max-1 of K configs: the lattice table rows (csrc/lattice.cuh)."""
    from math import comb
    return sum(comb(K + s - 1, s) for s in range(1, n_max))


def top_kernel_bytes(counts, lsteps, smax, masks, K, n_max):
    """Algorithmic bytes of the lat_top_kernel launches of one solve: per candidate the
    8 B key read + 32 B record read + 32 B record write, plus one read of every
    value_S / f_S[S-1] table row it searches (S >= 2 of its mask)."""
    states = lattice_states(K, n_max)
    total = 0
    for mp, mask in enumerate(masks):
        m = mp // 2
        nS2 = sum(1 for S in range(2, min(smax[m], lsteps[m]) + 1) if (mask >> S) & 1)
        if not mask or not counts[m]:
            continue
        total += int(counts[m]) * 72 + nS2 * 2 * states * (int(lsteps[m]) + 1) * 8
    return total


def other_configs(args, h_main):
    """Device time of one stage-1 solve of BASELINE configs 3 and 5 (not with --no-c5), and of
    a config-4 epoch re-pricing from cached records (frontier only). Parity cases, not
    the headline."""
    import torch
    from paper_2605_04357_b200 import FrontierSession, catalog
    from paper_2605_04357_b200.frontier import _price_matrix
    from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem
    out = {}
    names = ["c3"] + (["c5"] if not args.no_c5 and args.workload not in ("c5",) else [])
    for name in names:
        w = catalog.WORKLOADS[name]()
        prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                             GenContext(perf=w.perf, granularity=w.granularity))
        _, pm = _price_matrix(prob.configs, w.prices, w.regions)
        times = []
        for i in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prob.run()
            n = prob.h.frontier(pm)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        out[name] = {"candidates": prob.num_candidates, "frontier_survivors": int(n),
                     "stage1_ms": times[-1], "candidates_per_s": prob.num_candidates / (times[-1] / 1e3)}
        # streaming-path roofline: the per-model window compaction of the
        # last solve, CUDA events around its launch, algorithmic bytes from the library
        ws_ms, ws_bytes = prob.h.window_select_stats()
        if ws_ms > 0:
            hbm = measured_peaks()[0].get("hbm_gbs", 6650.0)
            gbs = ws_bytes / (ws_ms / 1e3) / 1e9
            out[name]["roofline_window_select"] = {
                "bound": "hbm", "kernel": "window_select_kernel", "achieved": gbs, "peak": hbm,
                "unit": "GB/s", "frac": gbs / hbm, "launch_ms": ws_ms, "alg_bytes": ws_bytes}
    w = catalog.extended_workload()
    sess = FrontierSession(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf))
    ts = []
    for epoch in range(1, 6):
        prices = catalog.c4_epoch_prices(w, epoch)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = sess.frontier(prices, regions=w.regions)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out["c4_reprice"] = {"epochs": len(ts), "ms_per_epoch": 1e3 * sum(ts[1:]) / (len(ts) - 1),
                         "frontier_survivors_last": len(f), "note": "cached records, frontier only, host API"}
    del h_main
    return out


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port) on host cores."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_baseline(args.workload, stride=CPU_SAMPLE_STRIDE * 8)
    vals = []
    t_all = 0.0
    n_all = 0
    threads = os.cpu_count()
    for _ in range(args.steps):
        v, n, dt, threads = cpu_baseline(args.workload)
        vals.append(v)
        t_all += dt
        n_all += n
    value = n_all / t_all
    from paper_2605_04357_b200 import catalog
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic spec tables (reference catalog)",
        "config": {"workload": workload_label(args.workload),
                   "sample": f"every {CPU_SAMPLE_STRIDE}th candidate per (model, phase)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n_all // args.steps} candidates/step (stride {CPU_SAMPLE_STRIDE}), "
                                   f"C restatement of the numba path, {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)




def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import torch
    import torch.distributed as tdist
    torch.cuda.set_device(local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_04357_b200 import _native, build_frontier, catalog
    from paper_2605_04357_b200.frontier import _frontier_across_ranks, _price_matrix, rank_pieces
    from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem

    w = catalog.WORKLOADS[args.workload]()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
    prob = Stage1Problem(w.configs, w.models, w.slos, caps, ctx)   # spec tables -> HBM
    regions, pmat = _price_matrix(prob.configs, w.prices, w.regions)
    h = prob.h
    NP = len(prob.phases)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    masks = None

    def step():
        nonlocal masks
        h.tables()
        h.enumerate()
        if world > 1:
            pieces = rank_pieces(prob, tdist)  # memoised after the first (warm-up) step
            masks = [0] * (len(w.models) * NP)
            for mp, mk, lo, hi in pieces:
                masks[mp] |= mk
            h.evaluate_pieces(pieces)
            return _frontier_across_ranks(prob, pmat, tdist)
        h.evaluate(0, -1)
        return h.frontier(pmat)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ncand = h.num_candidates()
    total_ms = 0.0
    launches0 = h.launches
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            l2_flush.fill_(1)
            if world > 1:
                tdist.barrier()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            nf = step()
            ev1.record()
            torch.cuda.synchronize()
            total_ms += ev0.elapsed_time(ev1)
    launches = h.launches - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = ncand * args.steps / (total_ms / 1e3)
    stages = h.stage_ms()
    rank_eval = [stages["evaluate"]]
    if world > 1:  # per-rank evaluate time of the last step (load balance of the unit split)
        ev = torch.tensor([stages["evaluate"]], dtype=torch.float64, device="cuda")
        allv = torch.empty(world, dtype=torch.float64, device="cuda")
        tdist.all_gather_into_tensor(allv, ev)
        rank_eval = allv.tolist()

    # e2e: the public API, host spec objects in -> frontier ServingTemplates out
    e2e_times = []
    front, p2 = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx,
                               return_problem=True)
    h2d = sum(a.nbytes for a in p2.h._keep) + pmat.nbytes
    d2h = len(front) * _native.FRONTIER_DTYPE.itemsize + 8 * (len(w.models) + 2)
    del front, p2  # its handle returns to the pool: every timed call below reuses it warm
    for i in range(args.e2e_steps + 1):
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        front = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_times.append(dt)
        del front
    et = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(et, op=tdist.ReduceOp.MAX)
    e2e_s = float(et.item())

    # roofline of the dominant kernel (lat_layer_kernel) and of lat_top_kernel, from ONE
    # extra serialised pass (one chain stream: no launch overlaps another, so launches x
    # mean duration adds up within the pass, as in ncu's serialised launch list) after a
    # census pass that counts each kernel's algorithmic bytes and (u, l) / (u, S) pairs
    # (csrc/lattice.cuh: 10 B per f/choice cell written + one read of each computed
    # state's value_S and f_{sg-1} rows + its sub-table entries)
    peaks, peak_kind = measured_peaks()
    h.set_streams(1)
    h.set_timing(True)  # per-launch events for this pass only (off in the timed steps)
    h.set_census(True)
    step()
    census = h.census_all()
    h.set_census(False)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l2_flush.fill_(1)
    ev0.record()
    step()
    ev1.record()
    torch.cuda.synchronize()
    serial_ms = ev0.elapsed_time(ev1)
    layer_ms, layer_n = h.kernel_stats(1)
    top_ms, top_n = h.kernel_stats(0)
    sk = {k: h.kernel_stats(k) for k in (2, 3, 4)}
    h.set_streams(0)
    h.set_timing(False)
    layer_alg, layer_pairs, top_pairs = census[0], census[1], census[2]
    layer_launch_s = (layer_ms / max(layer_n, 1)) / 1e3
    alg_per_launch = layer_alg / max(layer_n, 1)
    achieved = alg_per_launch / layer_launch_s / 1e9 if layer_n else 0.0
    counts = h.num_combos()
    _, lsteps, smax = h.table_layout()
    if masks is None:
        masks = [sum(1 << S for S in range(1, _native.MAX_NODES + 1))] * (len(w.models) * NP)
    top_alg = top_kernel_bytes(counts, lsteps, smax, masks, len(w.configs), w.n_max)
    top_launch_s = (top_ms / max(top_n, 1)) / 1e3
    top_achieved = (top_alg / max(top_n, 1)) / top_launch_s / 1e9 if top_n else 0.0
    traffic, top_traffic = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        traffic = tj.get("lat_layer_kernel_dram_bytes_per_launch")
        top_traffic = tj.get("lat_top_kernel_dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    # on-chip roofline (the bound that actually applies): instruction issue
    # for the layer kernel, L1 wavefronts for the top kernel; per-pair costs from the
    # committed ncu capture x the live pair counts / the live serialised durations
    calib, onchip = onchip_calibration()
    clk_mhz = (clk.summary().get("sm_mhz") or onchip.get("sm_clock_mhz_nominal") or 1965.0)
    sms = onchip.get("sms", 148)
    roofline_onchip = {"sm_mhz": clk_mhz, "calibration": "profiles/r02_onchip_calib.json",
                       "peaks": "profiles/r01_onchip_peaks.json"}
    if calib.get("lat_layer_kernel", {}).get("inst_per_pair") and layer_n:
        ipp = calib["lat_layer_kernel"]["inst_per_pair"]
        rate = ipp * layer_pairs / (layer_ms / 1e3)
        peak = 4.0 * sms * clk_mhz * 1e6
        roofline_onchip["lat_layer_kernel"] = {
            "bound": "issue", "unit": "warp-instructions/s", "achieved": rate, "peak": peak,
            "frac": rate / peak, "inst_per_pair": ipp, "pairs": layer_pairs,
            "ncu_issue_slots_busy": calib["lat_layer_kernel"].get("issue_slots_busy")}
    if calib.get("lat_top_kernel", {}).get("wavefronts_per_pair") and top_n:
        wpp = calib["lat_top_kernel"]["wavefronts_per_pair"]
        rate = wpp * top_pairs / (top_ms / 1e3)
        peak = onchip.get("l1_gather_lanes_per_sm_clk", 0.985) * sms * clk_mhz * 1e6
        roofline_onchip["lat_top_kernel"] = {
            "bound": "l1_wavefronts", "unit": "wavefronts/s", "achieved": rate, "peak": peak,
            "frac": rate / peak, "wavefronts_per_pair": wpp, "pairs": top_pairs,
            "ncu_l1tex_throughput": calib["lat_top_kernel"].get("l1tex_throughput")}
    # (model, phase, combo, S) DP evaluations the reference performs: its per-combo S
    # loop runs S = 1..min(n, Lu) (templates.py:314-316: 8.125 M for c2)
    dp_evals = 0
    for m in range(len(w.models)):
        keys = h.get_combos(m)
        nodes = sum(((keys >> np.uint64(9 * t)) & np.uint64(7)).astype(np.int64) for t in range(_native.MAX_NODES))
        dp_evals += int(np.minimum(nodes, int(lsteps[m])).sum()) * NP
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic spec tables (reference catalog, BASELINE config 2)",
        "config": {"workload": workload_label(args.workload),
                   "candidates": ncand, "dp_evaluations": dp_evals,
                   "dp_evaluations_per_s": dp_evals * args.steps / (total_ms / 1e3),
                   "frontier_survivors": int(nf),
                   "parallelism": f"pieces over {world} GPUs: (model, phase, S) units, the largest split by candidate range (measured costs), + one NCCL all-gather of partial frontiers"
                                  if world > 1 else "single GPU",
                   "l2": "256 MB buffer written between timed steps",
                   "stage1_solve_s": total_ms / args.steps / 1e3},
        "stage_ms": stages,
        "rank_evaluate_ms": rank_eval,
        "e2e": {"value": ncand / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "stage1_solve_s": e2e_s},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "lat_layer_kernel", "achieved": achieved,
                     "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / peaks.get("hbm_gbs", 6650.0), "traffic": traffic,
                     "peak_kind": peak_kind, "launch_ms": 1e3 * layer_launch_s,
                     "launches_per_step": layer_n, "timing": "serialised pass (1 chain stream)",
                     "serial_step_ms": serial_ms,
                     "share_of_serial_step": layer_ms / max(serial_ms, 1e-9),
                     "alg_bytes_per_launch": alg_per_launch,
                     "note": "fp64 max-min crossing searches over L2-resident lattice tables: bound by "
                             "instruction issue (roofline_onchip), not HBM bandwidth; the north_star's "
                             ">=60% of HBM cannot apply to this DP (SURVEY.md 7 hard part 5, DESIGN.md 5)"},
        "roofline_top": {"kernel": "lat_top_kernel", "achieved": top_achieved, "unit": "GB/s",
                         "frac": top_achieved / peaks.get("hbm_gbs", 6650.0), "traffic": top_traffic,
                         "launch_ms": 1e3 * top_launch_s, "launches_per_step": top_n,
                         "share_of_serial_step": top_ms / max(serial_ms, 1e-9),
                         "alg_bytes_per_launch": top_alg / max(top_n, 1)},
        "roofline_onchip": roofline_onchip,
        "serial_kernel_ms": {"lat_layer_kernel": layer_ms, "lat_top_kernel": top_ms, "lat_value_kernel": sk[2][0],
                             "lat_decode_kernel": sk[3][0], "lat_ranks_kernel": sk[4][0]},
    }
    if world == 1:
        line["other_configs"] = other_configs(args, h)
    if rank == 0:
        line["clocks"] = clk.summary()
        if world == 1 and not args.no_cpu_baseline:
            v, n, dt, threads = cpu_baseline(args.workload)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"{n} candidates (every {CPU_SAMPLE_STRIDE}th per model/phase) "
                                              f"in {dt:.1f}s, {cpu_model()}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
