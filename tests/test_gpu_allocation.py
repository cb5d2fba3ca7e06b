"""Stage-2 model construction on the device against the
unmodified reference's build_allocation_model (allocation.py:108-195): the same
variables, bounds, objective and constraints, in the same order, on the core library
(golden alloc_core.json.gz from tests/golden/make_alloc_golden.py)."""

import pytest

from paper_2605_04357_b200 import build_library
from paper_2605_04357_b200.allocation import (DemandSpec, InstanceInfo, MarketState, RunningState,
                                              build_allocation_model)
from tests.helpers import alloc_inputs, golden, milp_digest, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def core_lazy():
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    lib = build_library(configs, models, slos, caps, ctx, lazy=True)
    return lib, [c.name for c in configs], [r.name for r in regions]


@pytest.mark.parametrize("prune", [3.0, 1.25, 0.0])
def test_allocation_model_equals_reference(core_lazy, prune):
    lib, cfg_names, reg_names = core_lazy
    g = golden("alloc_core.json.gz")[repr(prune)]
    prices, avail, demand, running, k_init = alloc_inputs(cfg_names, reg_names, lib)
    market = MarketState(availability=avail, prices=prices)
    rs = RunningState([InstanceInfo(f"i{k}", r, tid) for k, (r, tid) in enumerate(running)])
    prob = build_allocation_model(lib, DemandSpec(demand), market, rs, k_init, prune_ratio=prune)
    assert {k: prob.meta[k] for k in ("pruned_vars", "num_vars", "num_constraints")} == g["meta"]
    assert [list(x) for x in prob.meta["uncovered_demands"]] == g["uncovered"]
    d = milp_digest(prob.milp)
    for k in ("n_vars", "n_cons", "sense", "first_vars", "first_cons", "vars_sha", "obj_sha", "cons_sha"):
        assert d[k] == g[k], k
    csr = prob.csr
    assert len(csr.ub) * (2 if k_init > 0 else 1) == prob.meta["num_vars"]
    assert csr.cap_ptr[-1] == len(csr.cap_idx)
