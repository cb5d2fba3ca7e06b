"""Per-stream timeline of one warm c2 evaluate (CUDA events around each lattice launch).

  python tools/timeline.py [workload] [--serial] [--zigzag]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import catalog  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem  # noqa: E402

KIND = {0: "top", 1: "layer", 2: "value", 3: "decode", 4: "ranks"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    serial = "--serial" in sys.argv
    w = catalog.WORKLOADS[name]()
    ctx = GenContext(perf=w.perf, granularity=w.granularity)
    if "--zigzag" in sys.argv:  # tests/helpers.zigzag_profile: non-monotone rows on two configs
        from paper_2605_04357_b200.specs import ProfileTable
        from tests.helpers import zigzag_profile
        ctx = GenContext(perf=w.perf, granularity=w.granularity,
                         profile=zigzag_profile(w.configs, w.models, ProfileTable))
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), ctx)
    prob.h.set_timing(True)
    if serial:
        prob.h.set_streams(1)
    for _ in range(3):
        prob.run()
    torch.cuda.synchronize()
    tl = prob.h.kernel_timeline()
    ev = prob.h.stage_ms()["evaluate"]
    print(f"evaluate {ev:.3f} ms, {len(tl)} timed launches; stages", {k: round(v, 3) for k, v in prob.h.stage_ms().items()})
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob.run()
    torch.cuda.synchronize()
    print(f"prob.run() wall {1e3 * (time.perf_counter() - t0):.3f} ms; stages",
          {k: round(v, 3) for k, v in prob.h.stage_ms().items()})
    for slot in sorted({s for _, s, _, _ in tl}):
        row = [(b, e, KIND[k]) for k, s, b, e in tl if s == slot]
        print(f"stream {slot}: " + " ".join(f"{KIND_ABBR(k)}[{b:.2f}-{e:.2f}]" for b, e, k in row))
    # concurrency profile: time with k streams busy
    pts = sorted([(b, 1) for _, _, b, _ in tl] + [(e, -1) for _, _, _, e in tl])
    busy = {}
    cur, last = 0, 0.0
    for t, d in pts:
        busy[cur] = busy.get(cur, 0.0) + (t - last)
        cur += d
        last = t
    busy[cur] = busy.get(cur, 0.0) + max(0.0, ev - last)
    print("ms with k kernels in flight:", {k: round(v, 3) for k, v in sorted(busy.items())})
    per = {}
    for k, _, b, e in tl:
        per[KIND[k]] = per.get(KIND[k], 0.0) + (e - b)
    print("summed event ms per kind:", {k: round(v, 3) for k, v in per.items()})
    if serial:  # per (model, phase) chain alone: ms per kind, candidates, layers
        per_mp = {}
        for k, mp, ms in prob.h.kernel_launches(4096):
            d = per_mp.setdefault(mp, {})
            d[KIND[k]] = d.get(KIND[k], 0.0) + ms
        NP = len(prob.phases)
        for mp in sorted(per_mp):
            m = prob.models[mp // NP]
            n = int(prob.cand_off[mp + 1] - prob.cand_off[mp]) if hasattr(prob, "cand_off") else -1
            d = per_mp[mp]
            print(f"mp {mp} {m.name:14s} L={m.num_layers:3d} cand={n:7d} total={sum(d.values()):.3f} " +
                  " ".join(f"{k}={v:.3f}" for k, v in sorted(d.items())))

def KIND_ABBR(k):
    return {"top": "T", "layer": "L", "value": "V", "decode": "D", "ranks": "R"}[k]


if __name__ == "__main__":
    main()
