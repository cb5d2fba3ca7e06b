"""Randomised GPU-vs-oracle stress beyond the test suite's seeds: library records AND
per-(model, phase, region) frontier, with n_max up to 7, ProfileTable overrides
(non-monotone and 1e-12-tolerance rows on some configs), random regional prices with
unpriced configs, and a 3-rank pieces emulation merged through the device-slot path.
  python tools/stress_random.py [first_seed] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_04357_b200 import LibraryGenError, build_library  # noqa: E402
from paper_2605_04357_b200 import _native  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402
from paper_2605_04357_b200.shard import calibrate, pieces_to_ranges, plan_pieces  # noqa: E402
from paper_2605_04357_b200.specs import GpuSpec, ModelSpec, NodeConfig, PerfParams, ProfileTable, SloSpec  # noqa: E402
from tests.helpers import cfg_by_rank, key_str, oracle_library_lines, oracle_problem, template_line  # noqa: E402


def inputs(seed):
    rng = np.random.default_rng(1000 + seed)
    gpus = [GpuSpec(f"G{i}", float(rng.choice([16, 24, 40, 48, 80, 141])), float(rng.uniform(0.2, 4.0)),
                    float(rng.uniform(50, 1000)), float(rng.uniform(0.5, 8))) for i in range(int(rng.integers(2, 5)))]
    configs = [NodeConfig(g, int(n)) for g in gpus for n in rng.choice([1, 2, 4, 8], size=2, replace=False)]
    models, slos = [], {}
    for k in range(int(rng.integers(1, 4))):
        L = int(rng.choice([8, 12, 24, 32, 40, 61, 80]))
        tot = float(rng.uniform(1, 120))
        models.append(ModelSpec(f"m{k}", L, tot, tot * float(rng.uniform(0.1, 1.0)), int(rng.choice([1024, 4096, 8192])),
                                kv_bytes_per_token_per_layer=float(rng.choice([512, 2048, 4096]))))
        slos[f"m{k}"] = SloSpec(float(rng.uniform(300, 3000)), float(rng.uniform(10, 150)))
    perf = PerfParams(mfu=float(rng.uniform(0.3, 0.8)), mbu=float(rng.uniform(0.5, 0.95)),
                      avg_prompt_tokens=float(rng.uniform(100, 3000)), avg_ctx_tokens=float(rng.uniform(100, 3000)),
                      slo_budget_frac=0.6)
    prof = ProfileTable()
    kind = seed % 3  # 0: none, 1: zigzag (non-monotone), 2: +1e-13 bumps (tolerance-monotone)
    if kind:
        for c in rng.choice(len(configs), size=min(2, len(configs)), replace=False):
            cfg = configs[int(c)]
            for m in models:
                for ph in ("prefill", "decode"):
                    base = float(rng.uniform(1e3, 1e5))
                    for j in range(1, m.num_layers + 1):
                        v = base / j
                        v = v * (1.3 if j % 2 else 1.0) if kind == 1 else v + (1e-13 if j % 3 == 1 else 0.0)
                        prof.add(cfg.name, m.name, ph, j, -1, v)
    n_max = int(rng.integers(2, 8))
    caps = LibraryCaps(n_max, float(rng.uniform(4, 30)))
    gran = int(rng.choice([0, 1, 2]))
    if any(m.num_layers % max(gran, 1) for m in models):
        gran = 0
    ctx = GenContext(perf=perf, granularity=gran, profile=prof if kind else None)
    regions = [f"r{i}" for i in range(int(rng.integers(1, 4)))]
    prices = {}
    for r in regions:
        for c in configs:
            if rng.uniform() < 0.9:
                prices[(r, c.name)] = float(np.round(rng.uniform(0.3, 40) * c.gpu_count, 3))
    return configs, models, slos, caps, ctx, regions, prices


def frontier_rows(h, n, prob):
    items = h.get_frontier(n)
    cbr = prob.cfg_by_rank
    return sorted((int(it["mp"]), int(it["region"]), key_str(int(it["combo_key"]), cbr), float(it["price_usd_h"]),
                   float(it["throughput_tps"]), int(it["rec"]["num_stages"])) for it in items)


def check(seed) -> str:
    """'' when the GPU path equals the oracle on scenario `seed`, else what differed."""
    configs, models, slos, caps, ctx, regions, prices = inputs(seed)
    op = oracle_problem((configs, models, slos, caps, ctx))
    ref = oracle_library_lines(op)
    try:
        lib = build_library(configs, models, slos, caps, ctx)
        got = [template_line(t) for t in lib.entries]
    except LibraryGenError:
        got = None
    if got is not None and got != ref:
        return f"library mismatch (n_max {caps.n_max})"
    # frontier: device vs the oracle's skyline over its own records
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    from tests.helpers import price_matrix
    pm = price_matrix(configs, prices, regions)
    n = prob.h.frontier(pm)
    dev = frontier_rows(prob.h, n, prob)
    cbr = cfg_by_rank(op.configs)
    oref = []
    for mi in range(len(op.models)):
        for ph, code in (("prefill", 0), ("decode", 1)):
            keys = op.enumerate(mi)
            recs = op.solve(mi, code, keys)
            reg, idx = op.frontier(keys, recs, pm)
            for r, i in zip(reg, idx):
                oref.append((mi * 2 + code, int(r), key_str(keys[i], cbr), float(recs[i]["throughput_tps"])))
    d2 = sorted((a, b, c, e) for a, b, c, _, e, _ in dev)
    if d2 != sorted(oref):
        return f"frontier mismatch ({len(d2)} vs {len(oref)} items)"
    # three-rank pieces emulation through the device-slot merge
    NP = 2
    _, lsteps, smax = prob.h.table_layout()
    smax_mp = [min(int(smax[mp // NP]), int(lsteps[mp // NP])) if prob.counts[mp // NP] else 0
               for mp in range(len(models) * NP)]
    plan = plan_pieces(calibrate(prob.h, len(smax_mp), smax_mp, NP), 3)
    item = _native.FRONTIER_DTYPE.itemsize
    cap = 1 << 14
    stride = item + cap * item
    gath = torch.zeros(3 * stride, dtype=torch.uint8, device="cuda")
    for r in range(3):
        prob.h.evaluate_pieces(pieces_to_ranges(plan[r], prob.counts, NP))
        prob.h.frontier_candidates_into(pm, gath.data_ptr() + r * stride, item, cap)
    n3, mx = prob.h.frontier_merge_gathered(gath.data_ptr(), 3, stride, item, cap)
    if frontier_rows(prob.h, n3, prob) != dev:
        return "pieces merge mismatch"
    prob.close()
    return ""


def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    bad = 0
    for seed in range(first, first + count):
        err = check(seed)
        bad += bool(err)
        print(f"seed {seed}: {err or 'ok'}", flush=True)
    print(f"{count} seeds, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
