import sys; sys.path.insert(0, ".")
import torch
from paper_2605_04357_b200 import catalog
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem
w = catalog.WORKLOADS["extended"]()
prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf)).run()
h = prob.h
h.set_streams(1)
h.set_timing(True)
for S in (1, 2, 4):
    for rep in range(2):
        h.evaluate_pieces([(mp, 1 << S, 0, -1) for mp in range(12)])
        torch.cuda.synchronize()
    print("S", S, "evaluate ms", h.stage_ms()["evaluate"])
    for kind, mp, ms in h.kernel_launches():
        print("  ", kind, mp, round(ms, 4))
