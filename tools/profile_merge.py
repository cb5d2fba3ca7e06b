"""Per-phase wall time of the multi-GPU merge (torchrun): after a barrier (so waiting
for the slowest rank is excluded) time the candidates pass straight into the gather
slot, the all-gather and the device-count merge on every rank -- once with a sync
between the phases (breakdown) and once as the product runs them (one sync at the end).
python -m torch.distributed.run --nproc-per-node N tools/profile_merge.py [workload]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

from paper_2605_04357_b200 import _native, catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _frontier_across_ranks, _gather_merge, _price_matrix, rank_pieces  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402


def main():
    if os.environ.get("MERGE_CAP_ENV"):  # A/B of the all-gather slot capacity
        from paper_2605_04357_b200 import frontier as _fr
        _fr._MERGE_CAP[0] = int(os.environ["MERGE_CAP_ENV"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = catalog.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "extended"]()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
    prob = Stage1Problem(w.configs, w.models, w.slos, caps, ctx)
    _, pm = _price_matrix(prob.configs, w.prices, w.regions)
    dev = torch.device("cuda", local)
    item = _native.FRONTIER_DTYPE.itemsize
    for it in range(6):
        torch.cuda.synchronize()
        tdist.barrier()
        t0 = time.perf_counter()
        prob.h.tables()
        prob.h.enumerate()
        pieces = rank_pieces(prob, tdist)
        t1 = time.perf_counter()
        prob.h.evaluate_pieces(pieces)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ev = prob.h.stage_ms()["evaluate"]
        tdist.barrier()
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        world = tdist.get_world_size()
        gat = {}

        def fill(send, offset, cap):
            prob.h.frontier_candidates_into(pm, send.data_ptr(), offset, cap)
            torch.cuda.synchronize()
            t.append(time.perf_counter())

        def merge(recv, stride, offset, cap):
            torch.cuda.synchronize()
            t.append(time.perf_counter())
            gat["counts"] = recv.view(world, stride)[:, :8].contiguous().view(torch.int64).view(-1).tolist()
            return prob.h.frontier_merge_gathered(recv.data_ptr(), world, stride, offset, cap)

        n = _gather_merge(fill, merge, tdist, dev, item)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        tdist.barrier()
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        n2 = _frontier_across_ranks(prob, pm, tdist)
        torch.cuda.synchronize()
        t6 = time.perf_counter()
        assert n2 == n
        if it == 5:
            d = np.diff(t) * 1e3
            print(f"rank {tdist.get_rank()}: pieces {len(pieces)} | tables+enum+plan {1e3 * (t1 - t0):.3f} ms "
                  f"evaluate wall {1e3 * (t2 - t1):.3f} device {ev:.3f} ms | parts {gat['counts']} survivors {n} | "
                  f"candidates {d[0]:.3f} ms gather {d[1]:.3f} ms merge {d[2]:.3f} ms | "
                  f"unsynced total {1e3 * (t6 - t5):.3f} ms", flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
