"""Golden stage-2 models from the UNMODIFIED reference's build_allocation_model
(/root/reference/pkg/src/hetserve/allocation.py:108-195) on the core library.

Runs only in the build container (needs /root/reference). The library is the
reference's own core library (tests/golden/library_core.json.gz, 30,739 templates);
the market varies availability per (region, config), leaves a few configs unpriced
in one region, and a few templates are already running, so every branch of the model
build (price None, prune, running exemption, availability cap, ceil(demand / T) bound,
init-penalty rows) is exercised. Writes tests/golden/alloc_core.json.gz:
per prune_ratio the meta counts and sha256 digests of the variables, objective and
constraints in the canonical text form of tests/helpers.milp_digest.

Usage: python tests/golden/make_alloc_golden.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from hetserve import allocation as RA  # noqa: E402
from hetserve import catalog as RC  # noqa: E402
from hetserve.domain import (DemandSpec, MarketState, NodeComboKey, Placement,  # noqa: E402
                             ServingTemplate)
from hetserve.templates import TemplateLibrary  # noqa: E402

from tests.helpers import alloc_inputs, golden, milp_digest  # noqa: E402


def reference_library():
    sc = RC.core_scenario()
    cfg = {c.name: c for c in sc.configs}
    entries = []
    for ln in golden("library_core.json.gz")["records"]:
        model, phase, combo, S, layers, son, T = ln.split("|")
        items = tuple((cfg[t.rsplit("*", 1)[0]], int(t.rsplit("*", 1)[1])) for t in combo.split("+"))
        entries.append(ServingTemplate(model, phase, sc.slos[model], NodeComboKey(items),
                                       Placement(int(S), tuple(int(x) for x in layers.split(",")),
                                                 tuple(int(x) for x in son.split(","))), float(T)))
    return TemplateLibrary(entries=entries), sc


def main():
    lib, sc = reference_library()
    out = {}
    for prune in (3.0, 1.25, 0.0):
        prices, avail, demand, running, k_init = alloc_inputs(
            [c.name for c in sc.configs], [r.name for r in sc.regions], lib)
        market = MarketState(availability=avail, prices=prices)
        rs = RA.RunningState([RA.InstanceInfo(f"i{k}", r, tid) for k, (r, tid) in enumerate(running)])
        prob = RA.build_allocation_model(lib, DemandSpec(demand), market, rs, k_init, prune_ratio=prune)
        out[repr(prune)] = {"meta": {k: prob.meta[k] for k in ("pruned_vars", "num_vars", "num_constraints")},
                            "uncovered": [list(x) for x in prob.meta["uncovered_demands"]],
                            **milp_digest(prob.milp)}
        print(prune, out[repr(prune)]["meta"])
    path = os.path.join(HERE, "alloc_core.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path}")


if __name__ == "__main__":
    np.seterr(all="ignore")
    main()
