"""Golden vectors at n_max = 7 from the UNMODIFIED reference (numba path).

The reference's own acceptance sweep runs the (7, 14) caps point
(pkg/tests/test_acceptance.py:320-348, c09); these fixtures pin the GPU path there:

  n7.json.gz
    c09:      the c09 model (m120b on H100x2 + L40Sx1, prefill) at (4,8), (6,12), (7,14):
              sweep rows (n_max, rho, templates, best T / price) and the full (7,14) library
    core7:    the core scenario at caps (7, 14): per (model, phase) counts, sha256 of the
              canonical lines and every 41st line; its cmd_sweep row
    kernels7: placement_search (kernels.py:279-295) on cases with 7 nodes (up to 7
              configs, L up to 32; monotone, tolerance-monotone, non-monotone, ties)

Usage: python tests/golden/make_golden_n7.py   (build container only; ~2-4 min)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import digest, dump, lib_records, rec_line  # noqa: E402
from run_reference_library import scenario_inputs  # noqa: E402

import hetserve.kernels as RK  # noqa: E402
from hetserve import catalog as RC  # noqa: E402
from hetserve.domain import PREFILL, ModelSpec, NodeConfig, SloSpec  # noqa: E402
from hetserve.templates import GenContext, LibraryCaps, build_library  # noqa: E402

assert RK.USE_NUMBA


def c09():
    model = ModelSpec("m120b", num_layers=36, params_total_b=116.8, params_active_b=5.1,
                      hidden_size=2880, kv_bytes_per_token_per_layer=2048, is_moe=True,
                      is_hybrid_attn=True)
    cfgs = [NodeConfig(RC.GPU_CATALOG["H100"], 2, 64.0), NodeConfig(RC.GPU_CATALOG["L40S"], 1, 64.0)]
    rows, lib7 = [], None
    for n_max, rho in ((4, 8.0), (6, 12.0), (7, 14.0)):
        lib = build_library(cfgs, [model], {"m120b": SloSpec(1000, 40)}, LibraryCaps(n_max, rho),
                            GenContext(), phases=(PREFILL,))
        best = 0.0
        for t in lib.entries:
            price = sum(n * c.gpu.rel_cost * c.gpu_count for c, n in t.combo.items)
            best = max(best, t.throughput_tps / price)
        rows.append([n_max, rho, len(lib), best])
        lib7 = lib
    return {"rows": rows, "library": [rec_line(r) for r in lib_records(lib7)]}


def core7():
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs("core")
    lib = build_library(configs, models, slos, LibraryCaps(7, 14.0), ctx, workers=os.cpu_count())
    lines = [rec_line(r) for r in lib_records(lib)]
    best = 0.0
    for t in lib.entries:
        price = min(sum(n * prices[(r.name, cfg.name)] for cfg, n in t.combo.items) for r in regions)
        best = max(best, t.throughput_tps / price)
    return {"count": len(lines), "sha256": digest(lines), "sample_every": 41, "sample": lines[::41],
            "counts": {f"{k[0]}|{k[1]}": v for k, v in lib.counts_by_model_phase().items()},
            "sweep_row": [7, 14.0, len(lib), best]}


def kernels7():
    rng = np.random.default_rng(77)
    cases = []
    for k in range(160):
        C = int(rng.integers(1, 8))
        counts = np.ones(C, dtype=np.int64)
        for _ in range(7 - C):
            counts[int(rng.integers(0, C))] += 1
        L = int(rng.integers(7, 33))
        kind = k % 4
        if kind == 3:
            tput = rng.integers(0, 4, size=(C, L)).astype(np.float64)
            tput = np.sort(tput, axis=1)[:, ::-1].copy()
        else:
            tput = rng.uniform(0, 50, size=(C, L))
            if kind in (0, 1):
                tput = np.sort(tput, axis=1)[:, ::-1].copy()
            if kind == 1:
                tput[:, 1::3] += 1e-13  # monotone only within the 1e-12 tolerance
        for S in range(1, 9):
            best, sj, sc = RK.placement_search(counts, tput, S)
            cases.append({"counts": counts.tolist(), "tput": tput.tolist(), "S": S, "best": float(best),
                          "stage_j": [int(x) for x in sj], "stage_counts": [[int(y) for y in r] for r in sc]})
    return cases


if __name__ == "__main__":
    out = {"c09": c09()}
    print("c09 rows", out["c09"]["rows"], len(out["c09"]["library"]))
    out["kernels7"] = kernels7()
    print("kernels7", len(out["kernels7"]))
    out["core7"] = core7()
    print("core7", out["core7"]["count"], out["core7"]["counts"])
    dump("n7.json.gz", out)
