"""Predicted (shard._rank_load on the calibrated costs) vs measured evaluate time of each
rank's pieces, every rank's share emulated alone on one GPU (min of 3 warm runs).
  python tools/plan_check.py [workload] [world ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402
from paper_2605_04357_b200.shard import _rank_load, calibrate, pieces_to_ranges, plan_pieces  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    worlds = [int(a) for a in sys.argv[2:]] or [2, 4]
    w = catalog.WORKLOADS[name]()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
                         GenContext(perf=w.perf, granularity=w.granularity))
    prob.run()
    NP = len(prob.phases)
    _, lsteps, smax = prob.h.table_layout()
    smax_mp = [min(int(smax[mp // NP]), int(lsteps[mp // NP])) if prob.counts[mp // NP] else 0
               for mp in range(len(prob.models) * NP)]
    for rep in range(2):
        costs = calibrate(prob.h, len(smax_mp), smax_mp, NP)
        F, L, T = costs
        print(f"calibration {rep}: F", [round(x, 4) for x in F])
        for mp in range(len(F)):
            print(f"  mp {mp} L", {S: round(v, 4) for S, v in L[mp]}, "T", {S: round(v, 4) for S, v in T[mp]})
    Ld = [dict(x) for x in L]
    Td = [dict(x) for x in T]
    for world in worlds:
        plan = plan_pieces(costs, world)
        for r, ps in enumerate(plan):
            units = []
            for mp, mk, a, b in ps:
                units += [(mp, S, a, b) for S in range(1, 8) if mk >> S & 1]
            pred = _rank_load(units, F, Ld, Td)
            # the serial sum and the slot count (fit of the overlap model)
            groups = {}
            seen = set()
            for mp, S, a, b in units:
                g = groups.get(mp, 0.0)
                if (mp, a, b) not in seen:
                    seen.add((mp, a, b))
                    g += F[mp] * (b - a)
                groups[mp] = g + Ld[mp].get(S, 0.0) + Td[mp].get(S, 0.0) * (b - a)
            serial = sum(groups.values())
            top = max(groups.values()) if groups else 0.0
            pieces = pieces_to_ranges(ps, prob.counts, NP)
            ms = []
            for _ in range(4):
                prob.h.evaluate_pieces(pieces)
                torch.cuda.synchronize()
                ms.append(prob.h.stage_ms()["evaluate"])
            print(f"world {world} rank {r}: slots {len(groups)} serial {serial:.3f} top {top:.3f} "
                  f"predicted {pred:.3f} ms measured {min(ms[1:]):.3f} ms  pieces "
                  + " ".join(f"(mp{mp} S{[S for S in range(1, 8) if mk >> S & 1]} {a:.3f}-{b:.3f})" for mp, mk, a, b in ps))


if __name__ == "__main__":
    main()
