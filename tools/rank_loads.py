"""Predicted (shard.py cost model) vs measured evaluate time of each rank's unit share,
each share emulated alone on one GPU.  python tools/rank_loads.py [world ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402
from paper_2605_04357_b200.shard import assign_units, chain_fixed, table_posfrac, unit_cost  # noqa: E402


def main():
    only = None
    if "--only" in sys.argv:  # python tools/rank_loads.py --only WORLD RANK (for ncu launch lists)
        i = sys.argv.index("--only")
        only = (int(sys.argv[i + 1]), int(sys.argv[i + 2]))
        del sys.argv[i:i + 3]
    worlds = [int(a) for a in sys.argv[1:]] or [2, 4]
    w = catalog.extended_workload()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf))
    prob.h.set_timing(True)
    prob.h.tables()
    prob.h.enumerate()
    counts = prob.h.num_combos()
    _, lsteps, smax = prob.h.table_layout()
    print("counts", list(counts), "lsteps", list(lsteps), "smax", list(smax))
    full = [sum(1 << S for S in range(1, 7))] * (len(counts) * 2)
    pf = table_posfrac(prob.h, len(prob.configs))
    if only is not None:
        mk = assign_units(counts, lsteps, smax, 2, only[0], pf)[only[1]] if only[0] > 1 else full
        for _ in range(3):
            prob.h.evaluate_units(mk)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        prob.h.evaluate_units(mk)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    for world in [1] + worlds:
        masks = [full] if world == 1 else assign_units(counts, lsteps, smax, 2, world, pf)
        for r, mk in enumerate(masks):
            pred = 0.0
            for mp, m in enumerate(mk):
                if not m:
                    continue
                nc = int(counts[mp // 2])
                pred += chain_fixed(nc) + sum(unit_cost(nc, int(lsteps[mp // 2]), S, dict(pf[mp]).get(S, 0.5))
                                              for S in range(1, 7) if m >> S & 1)
            ts = []
            for _ in range(6):
                prob.h.evaluate_units(mk)
                torch.cuda.synchronize()
                ts.append(prob.h.stage_ms()["evaluate"])
            ks = [prob.h.kernel_stats(k) for k in range(3)]
            print(f"world {world} rank {r}: measured {sorted(ts)[3]:.2f} ms predicted {pred:.2f} ms "
                  f"top/layer/value {[(round(k[0], 2), k[1]) for k in ks]} "
                  f"units {[(mp, [S for S in range(1, 7) if m >> S & 1]) for mp, m in enumerate(mk) if m]}",
                  flush=True)


if __name__ == "__main__":
    main()
