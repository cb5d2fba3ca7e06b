"""Histogram of the winning stage count S per (model, phase) and combo size n (c2)."""
import sys, collections
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2605_04357_b200 import catalog
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem
w = catalog.extended_workload()
prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf)).run()
for mp in range(len(w.models) * 2):
    r = prob.records(mp)
    S = r["num_stages"]; n = r["num_nodes"]
    ok = S > 0
    h = collections.Counter(zip(n[ok].tolist(), S[ok].tolist()))
    tot = ok.sum()
    line = []
    for nn in range(1, 7):
        row = [h.get((nn, s), 0) for s in range(1, 7)]
        if sum(row): line.append(f"n{nn}:" + "/".join(str(x) for x in row))
    print(mp, w.models[mp // 2].name, "feasible", tot, " ".join(line))
