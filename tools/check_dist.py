"""torchrun check: the multi-GPU frontier (unit shards + NCCL all-gather + merge) equals
the single-GPU frontier on every rank, for BASELINE configs 2 and 3.

  python -m torch.distributed.run --nproc-per-node N tools/check_dist.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

from paper_2605_04357_b200 import build_frontier, catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps  # noqa: E402


def rows(front):
    return sorted((k, str(e.template.combo), e.template.placement.num_stages,
                   e.template.placement.layers_per_stage, e.template.placement.stage_of_node,
                   e.template.throughput_tps, e.price_usd_h) for k, v in front.segments.items() for e in v)


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for name in ("extended", "c3", "core", "c1"):
        w = catalog.WORKLOADS[name]()
        caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
        dist = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
        single = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx,
                                dist=False)
        same = rows(dist) == rows(single)
        ok &= same
        print(f"rank {tdist.get_rank()}/{tdist.get_world_size()} {name}: {len(dist)} survivors, "
              f"identical to single-GPU: {same}", flush=True)
    tdist.barrier()
    tdist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
