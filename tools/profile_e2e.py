"""cProfile of the public build_frontier() call (host overhead of the e2e path)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import build_frontier, catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps  # noqa: E402

w = catalog.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
for _ in range(3):
    build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
torch.cuda.synchronize()
print("mean e2e s", (time.perf_counter() - t0) / 5)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
