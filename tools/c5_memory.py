"""Device memory a BASELINE config-5 solve holds (tables, keys, records, lattice
workspaces, frontier buffers): cudaMemGetInfo before and after one full solve + frontier.

  python tools/c5_memory.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402

torch.cuda.init()
free0, total = torch.cuda.mem_get_info()
w = catalog.c5_workload()
prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf))
_, pm = _price_matrix(prob.configs, w.prices, w.regions)
prob.run()
n = prob.h.frontier(pm)
torch.cuda.synchronize()
free1, _ = torch.cuda.mem_get_info()
print(f"c5: {prob.num_candidates} candidates, {n} survivors; device memory held by the solve "
      f"{(free0 - free1) / 2**30:.1f} GiB of {total / 2**30:.1f} GiB (stage ms {prob.h.stage_ms()})")
