"""The unchanged reference stage 2 consumes this package's template objects
(SURVEY.md 8b "consumers must keep working unchanged"). Build-container only: the
reference is not shipped to GPU boxes, so these tests skip when it is absent."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
MODEL = "phi4-14b"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import hetserve.allocation as alloc
    import hetserve.catalog as cat
    import hetserve.domain as dom
    return alloc, cat, dom


def _market_demand(ref, scale=1.0):
    alloc, cat, dom = ref
    sc = cat.core_scenario()
    market = dom.MarketState(availability=sc.availability.for_epoch(0), prices=dict(sc.prices))
    demand = dom.DemandSpec({(MODEL, ph): scale * 20000.0 for ph in ("prefill", "decode")})
    return market, demand


def test_reference_allocation_runs_on_our_full_library(ref):
    alloc, cat, dom = ref
    from tests.helpers import golden
    from tests.test_persistence import library_from_lines
    lib = library_from_lines("core", [ln for ln in golden("library_core.json.gz")["records"]
                                      if ln.startswith(MODEL + "|")])
    market, demand = _market_demand(ref)
    prob = alloc.build_allocation_model(lib, demand, market, alloc.RunningState(), k_init=0.0,
                                        prune_ratio=1.25)
    plan = alloc.solve_allocation(prob, time_budget_s=120)
    assert plan.total_instances() > 0
    for (r, tid), n in plan.counts.items():
        assert lib.get(tid).template_id == tid


def test_reference_allocation_runs_on_frontier_library(ref):
    """The frontier as the MILP's library: far fewer variables; the
    plan is feasible and never cheaper than the full-library optimum."""
    alloc, cat, dom = ref
    from tests.helpers import golden
    from tests.test_persistence import library_from_lines
    records = [ln for ln in golden("library_core.json.gz")["records"] if ln.startswith(MODEL + "|")]
    full = library_from_lines("core", records)
    keep = {(m, ph, combo) for m, ph, r, combo, p, t in golden("frontier_core.json.gz")}
    lines = [ln for ln in records if tuple(ln.split("|")[:3]) in keep]
    front = library_from_lines("core", lines)
    market, demand = _market_demand(ref)
    pf = alloc.build_allocation_model(front, demand, market, alloc.RunningState(), k_init=0.0,
                                      prune_ratio=0)
    pl = alloc.build_allocation_model(full, demand, market, alloc.RunningState(), k_init=0.0,
                                      prune_ratio=0)
    assert pf.meta["num_vars"] * 10 < pl.meta["num_vars"]
    plan_f = alloc.solve_allocation(pf, time_budget_s=120)
    plan_l = alloc.solve_allocation(pl, time_budget_s=120)
    assert plan_f.objective_usd_per_h >= plan_l.objective_usd_per_h - 1e-6


def test_reference_stage2_on_gpu_produced_c1_frontier(ref):
    """BASELINE config 1: the frontier the CUDA path produced on a B200
    (tools/dump_c1_frontier.py -> tests/golden/c1_frontier_gpu.jsonl) is loaded by the
    reference's own TemplateLibrary.load and fed to its unchanged allocate_with_fallback
    (allocation.py:318-359) on the small node pool (4 nodes per config)."""
    alloc, cat, dom = ref
    from hetserve.templates import TemplateLibrary as RefLibrary
    from tests.helpers import GOLDEN, golden, workload
    path = os.path.join(GOLDEN, "c1_frontier_gpu.jsonl")
    lib = RefLibrary.load(path)
    want = {(m, ph, combo) for m, ph, r, combo, p, t in golden("frontier_c1.json.gz")}
    assert {(t.model, t.phase, str(t.combo)) for t in lib.entries} == want
    configs, models, slos, caps, ctx, regions, prices = workload("c1")
    avail = {(r.name, c.name): 4 for r in regions for c in configs}
    market = dom.MarketState(availability=avail, prices=dict(prices))
    demand = dom.DemandSpec({(models[0].name, "prefill"): 30000.0, (models[0].name, "decode"): 3000.0})
    plan = alloc.allocate_with_fallback(lib, demand, market, alloc.RunningState(), k_init=0.0)
    assert plan.status == "optimal" and plan.total_instances() > 0
    for (r, tid), n in plan.counts.items():
        assert lib.get(tid).template_id == tid
    # the full reference library never costs more (the frontier is lossy only when
    # capacity binds)
    from tests.test_persistence import library_from_lines
    full = library_from_lines("c1", golden("library_c1.json.gz")["records"])
    plan_full = alloc.allocate_with_fallback(full, demand, market, alloc.RunningState(), k_init=0.0)
    assert plan.objective_usd_per_h >= plan_full.objective_usd_per_h - 1e-6
    assert plan.demand_scale == plan_full.demand_scale
