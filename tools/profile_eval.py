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
    shard = None
    if "--rank" in sys.argv:  # emulate one rank of a multi-GPU solve on this device
        from paper_2605_04357_b200.shard import assign_units, table_posfrac
        shard = (int(sys.argv[sys.argv.index("--rank") + 1]), int(sys.argv[sys.argv.index("--world") + 1]))
    for _ in range(solves):
        if shard is None:
            prob.run()
        else:
            prob.h.tables()
            prob.h.enumerate()
            prob.counts = prob.h.num_combos()
            _, lsteps, smax = prob.h.table_layout()
            prob.cand_off = [0]
            prob.h.evaluate_units(assign_units(prob.counts, lsteps, smax, 2, shard[1],
                                               table_posfrac(prob.h, len(prob.configs)))[shard[0]])
        n = prob.h.frontier(pm)
    torch.cuda.synchronize()
    print(name, prob.h.num_candidates(), "candidates;", n, "survivors;", prob.h.stage_ms())


if __name__ == "__main__":
    main()
