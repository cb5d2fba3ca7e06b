"""Host timeline of the multi-GPU build_frontier path (frontier.py, dist) per rank:
wall time at each call's return (no extra syncs except where the path has them), so the
host share of the multi-GPU e2e number shows.
  torchrun --nproc-per-node N tools/e2e_timeline_dist.py [workload]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

from paper_2605_04357_b200 import build_frontier, catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _frontier_across_ranks, _price_matrix, materialise, rank_pieces  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem, library_meta  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = sys.argv[1] if len(sys.argv) > 1 else "extended"
    w = catalog.WORKLOADS[name]()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
    for _ in range(3):
        build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
    rows = []
    for it in range(6):
        tdist.barrier()
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        cs = sorted(w.configs, key=lambda c: c.name)
        meta = library_meta(cs, w.models, w.slos, caps, ctx)
        names, pm = _price_matrix(cs, w.prices, w.regions)
        prob = Stage1Problem(w.configs, w.models, w.slos, caps, ctx)
        t.append(time.perf_counter())
        prob.h.tables()
        prob.h.enumerate()
        t.append(time.perf_counter())
        pieces = rank_pieces(prob, tdist)
        t.append(time.perf_counter())
        prob.h.evaluate_pieces(pieces)
        t.append(time.perf_counter())
        n = _frontier_across_ranks(prob, pm, tdist)
        t.append(time.perf_counter())
        prob.counts = prob.h.num_combos()
        NP = len(prob.phases)
        prob.cand_off = np.zeros(len(prob.models) * NP + 1, dtype=np.int64)
        for mp in range(len(prob.models) * NP):
            prob.cand_off[mp + 1] = prob.cand_off[mp] + prob.counts[mp // NP]
        items = prob.h.get_frontier(n)
        t.append(time.perf_counter())
        front = materialise(prob, items, names, meta)
        t.append(time.perf_counter())
        rows.append(([1e3 * (b - a) for a, b in zip(t, t[1:])], 1e3 * (t[-1] - t[0]), prob.h.stage_ms()))
        del front, prob
    bf = []
    for _ in range(6):
        tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        front = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
        torch.cuda.synchronize()
        bf.append(1e3 * (time.perf_counter() - t0))
        del front
    labels = ["setup", "tables+enum", "rank_pieces", "evaluate()", "merge path", "counts+get", "materialise"]
    d, tot, st = rows[-1]
    print(f"rank {tdist.get_rank()}: total {tot:.3f} ms | " + " ".join(f"{k} {v:.3f}" for k, v in zip(labels, d)) +
          " | device " + " ".join(f"{k} {v:.3f}" for k, v in st.items()) +
          " | build_frontier " + " ".join(f"{x:.2f}" for x in bf), flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
