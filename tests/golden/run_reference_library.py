"""Run the UNMODIFIED reference stage-1 generator (hetserve.templates.build_library,
/root/reference/pkg/src/hetserve/templates.py:417-505) on a named scenario and dump
its templates as compact records (pickle) for make_golden.py.

Only runs in the build container (the reference is not present on GPU boxes).
Usage: python tests/golden/run_reference_library.py {c1,core,extended,c3} OUT.pkl [workers]
"""
import os
import pickle
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from hetserve import catalog  # noqa: E402
from hetserve.domain import ModelSpec, Region, SloSpec  # noqa: E402
from hetserve.templates import GenContext, LibraryCaps, build_library  # noqa: E402


def scenario_inputs(name):
    """(configs, models, slos, caps, ctx, regions, prices) for a BASELINE config."""
    if name == "core":
        sc = catalog.core_scenario()
    elif name in ("extended", "c3"):
        sc = catalog.extended_scenario()
    elif name == "c1":
        # llama3-8b x {A100, L4} x {1,2,4,8}, one region.
        model = ModelSpec("llama3-8b", num_layers=32, params_total_b=8.03,
                          params_active_b=8.03, hidden_size=4096,
                          kv_bytes_per_token_per_layer=4096)
        configs = catalog.make_configs(["A100", "L4"])
        regions = [Region("us-east")]
        perf = catalog.perf_for_workload(catalog._synth_spec(["llama3-8b"], 10.0))
        return (configs, [model], {"llama3-8b": SloSpec(1500, 80)}, LibraryCaps(6, 12.0),
                GenContext(perf=perf), regions, catalog.make_prices(configs, regions))
    else:
        raise SystemExit(f"unknown scenario {name}")
    models = sc.models
    ctx = GenContext(perf=sc.perf)
    if name == "c3":
        models = [catalog.MODEL_CATALOG["llama3-70b"]]
        ctx = GenContext(perf=sc.perf, granularity=1)
    slos = {m.name: sc.slos[m.name] for m in models}
    return sc.configs, models, slos, sc.caps, ctx, sc.regions, sc.prices


def main():
    name, out = sys.argv[1], sys.argv[2]
    workers = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    t0 = time.monotonic()
    lib = build_library(configs, models, slos, caps, ctx, workers=workers)
    wall = time.monotonic() - t0
    recs = [(t.model, t.phase, str(t.combo), t.placement.num_stages,
             tuple(t.placement.layers_per_stage), tuple(t.placement.stage_of_node),
             t.throughput_tps) for t in lib.entries]
    with open(out, "wb") as fh:
        pickle.dump({"name": name, "wall_s": wall, "workers": workers,
                     "records": recs}, fh)
    print(f"{name}: {len(recs)} templates in {wall:.1f}s ({workers} workers)")


if __name__ == "__main__":
    main()
