"""Enumeration stage timing (device, CUDA events on the handle's stream) of one workload:
python tools/enum_time.py [workload]  (CORAL_S1_LIB selects a build for A/B runs)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity))
    ms, wall, wsm = [], [], []
    for _ in range(int(os.environ.get("ENUM_ITERS", "5"))):
        prob.h.tables()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob.h.enumerate()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ms.append(prob.h.stage_ms()["enumerate"])
        wsm.append(prob.h.window_select_stats()[0])
        wall.append(1e3 * (t1 - t0))
    prob.counts = prob.h.num_combos()
    sha = hashlib.sha256()
    for m in range(len(w.models)):
        sha.update(prob.keys(m).tobytes())
    print(f"{name} enumerate ms: {' '.join(f'{x:.3f}' for x in ms)}  host call ms: "
          f"{' '.join(f'{x:.3f}' for x in wall)}  window_select ms: {' '.join(f'{x:.3f}' for x in wsm)}  combos {sum(prob.h.num_combos())} digest {sha.hexdigest()[:16]}")


if __name__ == "__main__":
    main()
