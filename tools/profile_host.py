"""Host-side cost breakdown of one single-GPU build_frontier (c2): cProfile + pieces."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_04357_b200 import build_frontier, catalog  # noqa: E402
from paper_2605_04357_b200.frontier import _price_matrix, materialise  # noqa: E402
from paper_2605_04357_b200.library import (GenContext, LibraryCaps, Stage1Problem, _pack_problem,  # noqa: E402
                                           library_meta)


def main():
    w = catalog.extended_workload()
    caps, ctx = LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf)
    for _ in range(3):
        front, prob = build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions,
                                     ctx=ctx, return_problem=True)
    torch.cuda.synchronize()
    t = []
    for _ in range(20):
        t0 = time.perf_counter()
        build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    print("e2e ms median", 1e3 * sorted(t)[10])
    cfgs = sorted(w.configs, key=lambda c: c.name)
    names, pm = _price_matrix(cfgs, w.prices, w.regions)
    meta = library_meta(cfgs, w.models, w.slos, caps, ctx)
    n = len(front)
    for label, fn in [
        ("library_meta", lambda: library_meta(cfgs, w.models, w.slos, caps, ctx)),

        ("price_matrix", lambda: _price_matrix(cfgs, w.prices, w.regions)),
        ("frontier()", lambda: prob.h.frontier(pm)),
        ("get_frontier", lambda: prob.h.get_frontier(n)),
        ("materialise", lambda: materialise(prob, prob.h.get_frontier(n), names, meta)),
        # last: a new problem re-targets the shared per-device handle
        ("_pack_problem", lambda: _pack_problem(sorted(w.configs, key=lambda c: c.name), w.models, w.slos,
                                                ("prefill", "decode"), caps, ctx)),
        ("Stage1Problem", lambda: Stage1Problem(w.configs, w.models, w.slos, caps, ctx)),
    ]:
        fn()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        print(f"{label:14s} {1e3 * (time.perf_counter() - t0) / 20:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        build_frontier(w.configs, w.models, w.slos, caps, w.prices, regions=w.regions, ctx=ctx)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
