"""Generate golden vectors by running the UNMODIFIED reference (numba path) here.

Runs only in the build container (needs /root/reference). Writes small gzip'd JSON
fixtures into tests/golden/ that pin the CPU oracle and the CUDA path:

  kernels.json.gz     placement_search (kernels.py:279-295) on seeded random cases
                      (the test_kernels.py generators, seeds 7/8/3/11, plus wider
                      cases up to 6 configs / 6 nodes / 40 layer units), outputs
                      (best, stage_j, stage_counts) of the numba path.
  tables_<w>.json.gz  throughput_table + stage_budget_s for every (model, phase, S)
  enum_<w>.json.gz    enumerate_combos: full str(combo) lists (small workloads) or
                      count + sha256 (big ones)
  library_<w>.json.gz build_library records: full (c1, core, profile) or counts +
                      sha256 + every 97th record (extended)
  frontier_<w>.json.gz SURVEY.md 8c frontier computed on the reference library
  perf_grid.json.gz   node_max_throughput on a grid in the style of test_perf.py
  tolmono.json.gz     library on T-hat rows monotone only within the 1e-12 tolerance
                      (--tolmono)

Usage: python tests/golden/make_golden.py [--extended-pkl /tmp/ref_extended.pkl]
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import pickle
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import hetserve.kernels as RK  # noqa: E402
from hetserve import catalog as RC  # noqa: E402
from hetserve.domain import (DECODE, PREFILL, GpuSpec, ModelSpec, NodeConfig,  # noqa: E402
                             SloSpec)
from hetserve.perf import PerfParams, ProfileTable, node_max_throughput  # noqa: E402
from hetserve.templates import (GenContext, LibraryCaps, build_library,  # noqa: E402
                                enumerate_combos, stage_budget_s, throughput_table)

from run_reference_library import scenario_inputs  # noqa: E402

assert RK.USE_NUMBA, "golden vectors must come from the default numba path"


def dump(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {name} ({os.path.getsize(path)} B)")


def rec_line(t) -> str:
    return (f"{t[0]}|{t[1]}|{t[2]}|{t[3]}|{','.join(map(str, t[4]))}|"
            f"{','.join(map(str, t[5]))}|{t[6]!r}")


def lib_records(lib):
    return [(t.model, t.phase, str(t.combo), t.placement.num_stages,
             tuple(t.placement.layers_per_stage), tuple(t.placement.stage_of_node),
             t.throughput_tps) for t in lib.entries]


def digest(lines) -> str:
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def frontier_oracle(records, prices, regions):
    """SURVEY.md 8c on reference records: per (model, phase, region) sort by
    (price asc, T desc, str(combo) asc), keep iff T > running max. Price is
    allocation.py:91-98 _template_price (sequential in combo order)."""
    by_mp = {}
    for r in records:
        by_mp.setdefault((r[0], r[1]), []).append(r)
    out = []
    for (model, phase), recs in sorted(by_mp.items()):
        for region in regions:
            cands = []
            for r in recs:
                total = 0.0
                ok = True
                for tok in r[2].split("+"):
                    name, n = tok.rsplit("*", 1)
                    p = prices.get((region, name))
                    if p is None:
                        ok = False
                        break
                    total += int(n) * p
                if ok:
                    cands.append((total, -r[6], r[2], r))
            cands.sort()
            best = -float("inf")
            for total, negT, combo, r in cands:
                if -negT > best:
                    best = -negT
                    out.append([model, phase, region, combo, total, r[6]])
    return out


def kernel_cases():
    cases = []

    def test_kernels_case(rng, monotone):  # tests/test_kernels.py:35-42
        C = int(rng.integers(1, 3))
        counts = rng.integers(1, 3, size=C).astype(np.int64)
        L = int(rng.integers(2, 9))
        tput = rng.uniform(0, 10, size=(C, L))
        if monotone:
            tput = np.sort(tput, axis=1)[:, ::-1].copy()
        return counts, tput

    for seed, mono in ((7, True), (8, False), (3, True), (3, False), (11, True)):
        rng = np.random.default_rng(seed)
        for _ in range(40):
            counts, tput = test_kernels_case(rng, mono)
            for S in range(1, int(counts.sum()) + 2):
                cases.append((counts, tput, S))
    # wider cases: up to 6 configs, sum(counts) <= 6, L up to 40; monotone,
    # monotone within 1e-12 only, non-monotone, heavy ties, zeros
    rng = np.random.default_rng(2605)
    for k in range(400):
        C = int(rng.integers(1, 7))
        counts = np.zeros(C, dtype=np.int64)
        n = int(rng.integers(C, 7))
        for i in range(n):
            counts[i % C if i < C else int(rng.integers(0, C))] += 1
        L = int(rng.integers(1, 41))
        kind = k % 5
        if kind == 4:
            tput = rng.integers(0, 4, size=(C, L)).astype(np.float64)  # ties
        else:
            tput = rng.uniform(0, 1000, size=(C, L))
        if kind in (0, 2, 4):
            tput = np.sort(tput, axis=1)[:, ::-1].copy()
        if kind == 2:  # non-increasing up to +1e-13 bumps: monotone flag still set
            bumps = (rng.random(size=(C, L)) < 0.2) * 1e-13
            tput = tput + bumps
            tput[tput < 0] = 0
        if k % 17 == 0:
            tput[:, L // 2:] = 0.0  # memory-infeasible tail
        for S in sorted({1, 2, int(counts.sum()), int(rng.integers(1, counts.sum() + 1))}):
            cases.append((counts, tput, S))
    out = []
    for counts, tput, S in cases:
        best, sj, sc = RK.placement_search(counts, tput, S)
        out.append({"counts": counts.tolist(), "tput": [[float(x) for x in row] for row in tput],
                    "S": int(S), "best": float(best), "stage_j": sj.tolist(),
                    "stage_counts": sc.tolist()})
    return out


def tables_fixture(name):
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    configs = sorted(configs, key=lambda c: c.name)
    out = {"configs": [c.name for c in configs], "models": [m.name for m in models], "tables": {}}
    for m in models:
        for ph in (PREFILL, DECODE):
            for S in range(1, min(caps.n_max, m.num_layers) + 1):
                tab = throughput_table(configs, m, slos[m.name], ph, S, ctx)
                out["tables"][f"{m.name}|{ph}|{S}"] = {
                    "budget": stage_budget_s(m, slos[m.name], ph, S, ctx),
                    "rows": [[float(x) for x in row] for row in tab]}
    return out


def enum_fixture(name, full):
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    out = {}
    for m in models:
        strs = [str(k) for k in enumerate_combos(configs, m, caps)]
        ent = {"count": len(strs), "sha256": digest(strs)}
        if full:
            ent["combos"] = strs
        out[m.name] = ent
    return out


def library_fixture(name, records, full, wall=None):
    counts = {}
    for r in records:
        counts[f"{r[0]}|{r[1]}"] = counts.get(f"{r[0]}|{r[1]}", 0) + 1
    lines = [rec_line(r) for r in records]
    out = {"count": len(records), "counts": counts, "sha256": digest(lines), "wall_s": wall}
    if full:
        out["records"] = lines
    else:
        out["sample_every"] = 97
        out["sample"] = lines[::97]
    return out


def perf_grid():
    """node_max_throughput over nodes x models x phases x j x budgets (test_perf.py:106-124)."""
    nodes = [NodeConfig(g, n) for g in RC.GPU_CATALOG.values() for n in (1, 2, 8)]
    models = list(RC.MODEL_CATALOG.values()) + [
        ModelSpec("tiny", 4, 0.5, 0.5, 256, kv_bytes_per_token_per_layer=128.0)]
    params = [PerfParams(), PerfParams(mfu=0.3, mbu=0.9, fixed_overhead_ms=0.0,
                                       avg_prompt_tokens=333.3, avg_ctx_tokens=777.7)]
    out = []
    rng = np.random.default_rng(99)
    for pi, p in enumerate(params):
        for node in nodes:
            for m in models:
                for ph in (PREFILL, DECODE):
                    for _ in range(3):
                        j = int(rng.integers(1, m.num_layers + 1))
                        budget = float(rng.choice([0.003, 0.02, 0.05, 0.3, 1.0, 5.0]))
                        out.append({"p": pi, "gpu": node.gpu.name, "gc": node.gpu_count,
                                    "model": m.name, "phase": ph, "j": j, "budget": budget,
                                    "tput": node_max_throughput(node, m, ph, j, budget, p)})
    return out


def profile_case():
    """A ProfileTable-override library (perf.py:94-116 semantics inside stage 1)."""
    configs = [NodeConfig(RC.GPU_CATALOG["L40S"], 1, 64.0), NodeConfig(RC.GPU_CATALOG["L40S"], 2, 64.0),
               NodeConfig(RC.GPU_CATALOG["L4"], 1, 64.0), NodeConfig(RC.GPU_CATALOG["L4"], 4, 64.0)]
    model = ModelSpec("m7b", num_layers=32, params_total_b=7, params_active_b=7, hidden_size=4096)
    slo = SloSpec(1500, 80)
    prof = ProfileTable()
    prof.add("1xL40S", "m7b", DECODE, 32, -1, 123.0)
    prof.add("1xL40S", "m7b", DECODE, 16, -1, 77.5)
    prof.add("1xL4", "m7b", PREFILL, 8, -1, 4321.0)
    b2 = stage_budget_s(model, slo, DECODE, 2, GenContext(profile=prof))
    prof.add("4xL4", "m7b", DECODE, 16, int(round(b2 * 1e3)), 999.0)
    ctx = GenContext(profile=prof)
    lib = build_library(configs, [model], {"m7b": slo}, LibraryCaps(3, 10.0), ctx)
    entries = [[k[0], k[1], k[2], k[3], k[4], v] for k, v in prof.entries.items()]
    return {"profile": entries, "library": library_fixture("profile", lib_records(lib), True)}


def tolmono_case():
    """T-hat rows (ProfileTable overrides for every S) that rise by < 1e-12: monotone for
    kernels.py:291 but not exactly, so the reference's binary search runs on a
    predicate that is not monotone; includes an equal adjacent pair (ties)."""
    configs = [NodeConfig(RC.GPU_CATALOG["A100"], 1), NodeConfig(RC.GPU_CATALOG["A100"], 2),
               NodeConfig(RC.GPU_CATALOG["L40S"], 2)]
    model = ModelSpec("m8", num_layers=8, params_total_b=14, params_active_b=14, hidden_size=5120)
    slo = SloSpec(1500, 80)
    prof = ProfileTable()
    for k, cfg in enumerate(configs):
        for ph in (PREFILL, DECODE):
            base = 1000.0 * (k + 1) + (0.5 if ph == DECODE else 0.0)
            row = [base, base * 0.9, base * 0.8, base * 0.8 + 3e-13 * (k + 1), base * 0.65, base * 0.65,
                   base * 0.5 + 4e-13, base * 0.3]
            for j, v in enumerate(row, start=1):
                prof.add(cfg.name, "m8", ph, j, -1, v)
    lib = build_library(configs, [model], {"m8": slo}, LibraryCaps(4, 40.0), GenContext(profile=prof))
    entries = [[k[0], k[1], k[2], k[3], k[4], v] for k, v in prof.entries.items()]
    return {"profile": entries, "library": library_fixture("tolmono", lib_records(lib), True)}


def main():
    argv = sys.argv[1:]
    if "--tolmono" in argv:
        return dump("tolmono.json.gz", tolmono_case())
    ext_pkl = argv[argv.index("--extended-pkl") + 1] if "--extended-pkl" in argv else None
    if "--only-extended" in argv:
        return extended(ext_pkl)
    if "--c3-pkl" in argv:
        return big_library("c3", argv[argv.index("--c3-pkl") + 1])
    dump("kernels.json.gz", kernel_cases())
    dump("perf_grid.json.gz", perf_grid())
    dump("profile.json.gz", profile_case())
    for w in ("c1", "core", "extended"):
        dump(f"tables_{w}.json.gz", tables_fixture(w))
    dump("enum_c1.json.gz", enum_fixture("c1", True))
    dump("enum_core.json.gz", enum_fixture("core", True))
    dump("enum_extended.json.gz", enum_fixture("extended", False))
    for w in ("c1", "core"):
        configs, models, slos, caps, ctx, regions, prices = scenario_inputs(w)
        lib = build_library(configs, models, slos, caps, ctx, workers=os.cpu_count())
        recs = lib_records(lib)
        dump(f"library_{w}.json.gz", library_fixture(w, recs, True))
        dump(f"frontier_{w}.json.gz", frontier_oracle(recs, prices, [r.name for r in regions]))
    if ext_pkl:
        extended(ext_pkl)


def big_library(name, pkl):
    with open(pkl, "rb") as fh:
        data = pickle.load(fh)
    recs = data["records"]
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    dump(f"library_{name}.json.gz", library_fixture(name, recs, False, data["wall_s"]))
    dump(f"frontier_{name}.json.gz", frontier_oracle(recs, prices, [r.name for r in regions]))


def extended(ext_pkl):
    if ext_pkl:
        with open(ext_pkl, "rb") as fh:
            data = pickle.load(fh)
        recs = data["records"]
        configs, models, slos, caps, ctx, regions, prices = scenario_inputs("extended")
        dump("library_extended.json.gz", library_fixture("extended", recs, False, data["wall_s"]))
        dump("frontier_extended.json.gz", frontier_oracle(recs, prices, [r.name for r in regions]))


if __name__ == "__main__" and "--save-digests" not in sys.argv and "--sweep" not in sys.argv:
    main()


def saved_file_digest(name, records_or_lib):
    """sha256 of the reference's own TemplateLibrary.save (templates.py:364-377) output."""
    import tempfile
    from hetserve.domain import NodeComboKey, Placement, ServingTemplate
    from hetserve.templates import TemplateLibrary, _library_meta
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    if isinstance(records_or_lib, TemplateLibrary):
        lib = records_or_lib
    else:
        cfg = {c.name: c for c in configs}
        entries = []
        for (model, phase, combo, S, layers, son, T) in records_or_lib:
            items = tuple((cfg[tok.rsplit("*", 1)[0]], int(tok.rsplit("*", 1)[1])) for tok in combo.split("+"))
            entries.append(ServingTemplate(model, phase, slos[model], NodeComboKey(items),
                                           Placement(S, tuple(layers), tuple(son)), T))
        lib = TemplateLibrary(entries=entries,
                              meta=_library_meta(sorted(configs, key=lambda c: c.name), models, slos, caps, ctx))
    with tempfile.NamedTemporaryFile(suffix=".jsonl") as fh:
        lib.save(fh.name)
        data = open(fh.name, "rb").read()
    return {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
            "header": data.split(b"\n", 1)[0].decode()}


def save_digests(pkls):
    out = {}
    for name in ("c1", "core"):
        configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
        out[name] = saved_file_digest(name, build_library(configs, models, slos, caps, ctx,
                                                          workers=os.cpu_count()))
    for name, pkl in pkls.items():
        with open(pkl, "rb") as fh:
            out[name] = saved_file_digest(name, pickle.load(fh)["records"])
    dump("saved_libraries.json.gz", out)


if __name__ == "__main__" and "--save-digests" in sys.argv:
    save_digests({"extended": "/tmp/ref_extended.pkl", "c3": "/tmp/ref_c3.pkl"})


def sweep_rows():
    """Reference cmd_sweep semantics (cli.py:248-260): build_library per caps, best
    tokens/s per USD-h with price = min over regions; core scenario and the c09
    model (test_acceptance.py:320-348) on a single price list."""
    out = {}
    points = [(4, 8.0), (5, 10.0), (6, 12.0)]
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs("core")
    rows = []
    for n_max, rho in points:
        lib = build_library(configs, models, slos, LibraryCaps(n_max, rho), ctx, workers=os.cpu_count())
        best = 0.0
        for t in lib.entries:
            price = min(sum(n * prices[(r.name, cfg.name)] for cfg, n in t.combo.items) for r in regions)
            best = max(best, t.throughput_tps / price)
        rows.append([n_max, rho, len(lib), best])
    out["core"] = rows
    model = ModelSpec("m120b", num_layers=36, params_total_b=116.8, params_active_b=5.1,
                      hidden_size=2880, kv_bytes_per_token_per_layer=2048, is_moe=True,
                      is_hybrid_attn=True)
    cfgs = [NodeConfig(RC.GPU_CATALOG["H100"], 2, 64.0), NodeConfig(RC.GPU_CATALOG["L40S"], 1, 64.0)]
    rows = []
    for n_max, rho in points:
        lib = build_library(cfgs, [model], {"m120b": SloSpec(1000, 40)}, LibraryCaps(n_max, rho),
                            GenContext(), phases=(PREFILL,))
        best = 0.0
        for t in lib.entries:
            price = sum(n * c.gpu.rel_cost * c.gpu_count for c, n in t.combo.items)
            best = max(best, t.throughput_tps / price)
        rows.append([n_max, rho, len(lib), best])
    out["c09"] = rows
    dump("sweep.json.gz", out)


if __name__ == "__main__" and "--sweep" in sys.argv:
    sweep_rows()
