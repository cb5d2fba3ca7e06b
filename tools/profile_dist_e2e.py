"""Phase timing of the distributed build_frontier on each rank (torchrun)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _merge_across_ranks, _price_matrix, materialise  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem, library_meta  # noqa: E402
from paper_2605_04357_b200.shard import assign_units, table_posfrac  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = catalog.extended_workload()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf)
    for it in range(4):
        tdist.barrier()
        torch.cuda.synchronize()
        marks = [("start", time.perf_counter())]

        def mark(name):
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))

        configs_sorted = sorted(w.configs, key=lambda c: c.name)
        meta = library_meta(configs_sorted, w.models, w.slos, caps, ctx)
        names, pm = _price_matrix(configs_sorted, w.prices, w.regions)
        prob = Stage1Problem(w.configs, w.models, w.slos, caps, ctx)
        mark("setup")
        prob.h.tables()
        prob.h.enumerate()
        prob.counts = prob.h.num_combos()
        NP = 2
        prob.cand_off = np.zeros(len(prob.models) * NP + 1, dtype=np.int64)
        for mp in range(len(prob.models) * NP):
            prob.cand_off[mp + 1] = prob.cand_off[mp] + prob.counts[mp // NP]
        mark("tables+enum")
        _, lsteps, smax = prob.h.table_layout()
        prob.h.evaluate_units(assign_units(prob.counts, lsteps, smax, NP, tdist.get_world_size(),
                                            table_posfrac(prob.h, len(prob.configs)))[tdist.get_rank()])
        mark("evaluate")
        n_local = prob.h.frontier_candidates(pm)
        mark("local frontier")
        n = _merge_across_ranks(prob, n_local, tdist)
        mark("merge")
        items = prob.h.get_frontier(n)
        front = materialise(prob, items, names, meta)
        mark("materialise")
        if it == 3:
            phases = [(marks[i][0], 1e3 * (marks[i][1] - marks[i - 1][1])) for i in range(1, len(marks))]
            print(f"rank {tdist.get_rank()}: total {1e3 * (marks[-1][1] - marks[0][1]):.2f} ms "
                  + " ".join(f"{k}={v:.2f}" for k, v in phases), flush=True)
    tdist.destroy_process_group()
    del front


if __name__ == "__main__":
    main()
