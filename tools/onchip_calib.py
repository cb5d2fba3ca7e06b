"""Per-pair on-chip costs of the lattice search kernels (bench.py roofline_onchip).

  # on the GPU box: census of one c2 solve -> gpurun_out/calib_census.json, then ncu over
  # the next solve's lat_layer/lat_top launches (the census solve is skipped by -s)
  python tools/onchip_calib.py run [workload]
  ncu --metrics smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,\
sm__inst_executed_pipe_lsu.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv \
    -k regex:"lat_layer|lat_top_kernel" -s $SKIP -c $COUNT \
    --log-file gpurun_out/calib_ncu.csv python tools/onchip_calib.py run
  # here: combine -> profiles/r02_onchip_calib.json
  python tools/onchip_calib.py reduce gpurun_out/calib_census.json gpurun_out/calib_ncu.csv

Solve 1 warms up, solve 2 runs with the census on (pair counts), solve 3 is the one ncu
measures (census off: the kernels run exactly as in the bench). One chain stream, so
every launch runs alone, as in ncu's serialised replay.
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(name):
    import torch
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.frontier import _price_matrix
    from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity))
    _, pm = _price_matrix(prob.configs, w.prices, w.regions)
    prob.h.set_streams(1)
    prob.h.set_timing(True)
    prob.run()
    prob.h.frontier(pm)
    per_solve = {k: prob.h.kernel_stats(k)[1] for k in (0, 1)}
    prob.h.set_census(True)
    prob.run()
    census = prob.h.census_all()
    prob.h.set_census(False)
    prob.run()
    torch.cuda.synchronize()
    out = {"workload": name, "layer_pairs": census[1], "top_pairs": census[2], "layer_alg_bytes": census[0],
           "launches_per_solve": {"lat_top_kernel": per_solve[0], "lat_layer_kernel": per_solve[1]},
           "stage_ms_serial": prob.h.stage_ms()}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/calib_census.json", "w") as fh:
        json.dump(out, fh)
    n = per_solve[0] + per_solve[1]
    with open("gpurun_out/calib_skip.txt", "w") as fh:
        fh.write(f"{2 * n} {n}\n")
    print(json.dumps(out))


def reduce(census_path, ncu_csv):
    census = json.load(open(census_path))
    sums = {}
    with open(ncu_csv) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 10]
    head = rows[0]
    ki, mi, vi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    for r in rows[1:]:
        kern = "lat_layer_kernel" if "lat_layer" in r[ki] else "lat_top_kernel"  # incl. lat_layer_run_kernel
        v = float(r[vi].replace(",", ""))
        d = sums.setdefault(kern, {})
        d.setdefault(r[mi], []).append(v)
    out = {"source": f"ncu over one serialised {census['workload']} solve + census of the same solve "
                     "(tools/onchip_calib.py)", "census": census}
    for kern, pairs in (("lat_layer_kernel", census["layer_pairs"]), ("lat_top_kernel", census["top_pairs"])):
        m = sums.get(kern, {})
        inst = sum(m.get("smsp__inst_executed.sum", []))
        wf = sum(m.get("l1tex__data_pipe_lsu_wavefronts.sum", []))
        dur = m.get("gpu__time_duration.sum", [])
        w = [x for x in dur]
        wavg = lambda key: (sum(a * b for a, b in zip(m.get(key, []), w)) / sum(w)) if w and m.get(key) else None  # noqa
        out[kern] = {"launches": len(dur), "inst": inst, "wavefronts": wf, "pairs": pairs,
                     "inst_per_pair": inst / pairs if pairs else None,
                     "wavefronts_per_pair": wf / pairs if pairs else None,
                     "ncu_ms": sum(dur) / 1e6,
                     "issue_slots_busy": wavg("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "l1tex_throughput": wavg("l1tex__throughput.avg.pct_of_peak_sustained_active")}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "r02_onchip_calib.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "c2")
    else:
        reduce(sys.argv[2], sys.argv[3])
