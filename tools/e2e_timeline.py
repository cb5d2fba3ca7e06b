"""Host timeline of one single-GPU build_frontier (frontier.py) step by step: wall time at
each call's return next to the device stage times (CUDA events), so the host gaps in the
e2e number show.  python tools/e2e_timeline.py [workload]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import build_frontier, catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix, materialise  # noqa: E402
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem, library_meta  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = catalog.WORKLOADS[name]()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf, granularity=w.granularity)
    for _ in range(3):
        build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
    torch.cuda.synchronize()
    rows = []
    for it in range(6):
        t = [time.perf_counter()]
        cs = sorted(w.configs, key=lambda c: c.name)
        meta = library_meta(cs, w.models, w.slos, caps, ctx)
        names, pm = _price_matrix(cs, w.prices, w.regions)
        t.append(time.perf_counter())
        prob = Stage1Problem(w.configs, w.models, w.slos, caps, ctx)
        t.append(time.perf_counter())
        prob.h.tables()
        t.append(time.perf_counter())
        prob.h.enumerate()
        t.append(time.perf_counter())
        prob.counts = prob.h.num_combos()
        prob.h.evaluate(0, -1)
        t.append(time.perf_counter())
        n = prob.h.frontier(pm)
        t.append(time.perf_counter())
        items = prob.h.get_frontier(n)
        t.append(time.perf_counter())
        front = materialise(prob, items, names, meta)
        t.append(time.perf_counter())
        st = prob.h.stage_ms()
        rows.append(([1e3 * (b - a) for a, b in zip(t, t[1:])], 1e3 * (t[-1] - t[0]), st))
        del front, prob
    bf = []
    for it in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        front = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
        torch.cuda.synchronize()
        bf.append(1e3 * (time.perf_counter() - t0))
        del front
    print("build_frontier ms:", " ".join(f"{x:.3f}" for x in bf))
    labels = ["meta+prices", "Stage1Problem", "tables()", "enumerate()", "evaluate()", "frontier()",
              "get_frontier", "materialise"]
    for d, tot, st in rows[2:]:
        print(f"total {tot:.3f} ms | " + " ".join(f"{k} {v:.3f}" for k, v in zip(labels, d)) +
              " | device " + " ".join(f"{k} {v:.3f}" for k, v in st.items()))


if __name__ == "__main__":
    main()
