"""Measure evaluate time per (model, phase, S) unit and per whole chain on one GPU
(inputs for the multi-GPU cost model in paper_2605_04357_b200/shard.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402

w = catalog.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                     GenContext(perf=w.perf, granularity=w.granularity))
h = prob.h
h.tables()
h.enumerate()
counts = h.num_combos()
_, lsteps, smax = h.table_layout()
NMP = len(w.models) * 2


def timed(mask, reps=3):
    best = 1e9
    for _ in range(reps):
        h.evaluate_units(mask)
        torch.cuda.synchronize()
        best = min(best, h.stage_ms()["evaluate"])
    return best


empty = timed([0] * NMP)
rows = []
for mp in range(NMP):
    m = mp // 2
    Smx = min(int(smax[m]), int(lsteps[m]))
    full = [0] * NMP
    full[mp] = sum(1 << S for S in range(1, Smx + 1))
    chain = timed(full) - empty
    per_S = {}
    for S in range(1, Smx + 1):
        mk = [0] * NMP
        mk[mp] = 1 << S
        per_S[S] = timed(mk) - empty
    rows.append({"mp": mp, "model": w.models[m].name, "ncombo": int(counts[m]), "lsteps": int(lsteps[m]),
                 "chain_ms": chain, "per_S_ms": per_S})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"empty_ms": empty}))
