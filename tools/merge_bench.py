"""The multi-GPU frontier merge emulated on one GPU: W ranks' pieces (shard.plan_pieces)
evaluated in turn, each rank's prefiltered candidates written into its slot of one
buffer (frontier_candidates_into), then the device-count merge (frontier_merge_gathered)
timed alone -- for ncu captures of the merge kernels.
  python tools/merge_bench.py [workload] [W]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import _native, catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402
from paper_2605_04357_b200.shard import calibrate, pieces_to_ranges, plan_pieces  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity)).run()
    _, pm = _price_matrix(prob.configs, w.prices, w.regions)
    NP = 2
    _, lsteps, smax = prob.h.table_layout()
    smax_mp = [min(int(smax[mp // NP]), int(lsteps[mp // NP])) if prob.counts[mp // NP] else 0
               for mp in range(len(prob.models) * NP)]
    plan = plan_pieces(calibrate(prob.h, len(smax_mp), smax_mp, NP), W)
    item = _native.FRONTIER_DTYPE.itemsize
    cap = 1 << 14
    stride = item + cap * item
    gath = torch.zeros(W * stride, dtype=torch.uint8, device="cuda")
    for r in range(W):
        prob.h.evaluate_pieces(pieces_to_ranges(plan[r], prob.counts, NP))
        prob.h.frontier_candidates_into(pm, gath.data_ptr() + r * stride, item, cap)
    torch.cuda.synchronize()
    counts = gath.view(W, stride)[:, :8].contiguous().view(torch.int64).view(-1).tolist()
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n, mx = prob.h.frontier_merge_gathered(gath.data_ptr(), W, stride, item, cap)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{name} W={W} parts {counts} survivors {n}: merge wall ms median {sorted(ts)[10]:.3f} min {min(ts):.3f}")


if __name__ == "__main__":
    main()
