"""Frontier stage timing (device, CUDA events on the handle's stream) over one solve's
records: python tools/frontier_time.py [workload]  (CORAL_S1_LIB selects a build)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity)).run()
    _, pm = _price_matrix(prob.configs, w.prices, w.regions)
    ms = []
    for _ in range(5):
        n = prob.h.frontier(pm)
        torch.cuda.synchronize()
        ms.append(prob.h.stage_ms()["frontier"])
    digest = hashlib.sha256(prob.h.get_frontier(n).tobytes()).hexdigest()[:16]
    print(f"{name} frontier ms: {' '.join(f'{x:.3f}' for x in ms)}  survivors {n} "
          f"candidates {prob.num_candidates} regions {pm.shape[0]} digest {digest}")


if __name__ == "__main__":
    main()
