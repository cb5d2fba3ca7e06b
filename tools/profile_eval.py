"""One stage-1 solve of a workload, for ncu captures (warm-up solve first).

  python tools/profile_eval.py [workload] [--solves N]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
    solves = int(sys.argv[sys.argv.index("--solves") + 1]) if "--solves" in sys.argv else 2
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity))
    _, pm = _price_matrix(prob.configs, w.prices, w.regions)
    for _ in range(solves):
        prob.run()
        n = prob.h.frontier(pm)
    torch.cuda.synchronize()
    print(name, prob.num_candidates, "candidates;", n, "survivors;", prob.h.stage_ms())


if __name__ == "__main__":
    main()
