"""Golden libraries with monotonicity-breaking ProfileTable overrides, from the
UNMODIFIED reference (numba path): tests/helpers.zigzag_profile on two node configs of
the core scenario and of BASELINE config 2 (extended). Combos containing those configs
run the reference's full-scan DP (kernels.py:240-249); the GPU must match bit for bit.

  python tests/golden/make_golden_profile.py core       (~1 min)
  python tests/golden/make_golden_profile.py extended   (~30-60 min, 8 workers)
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from make_golden import digest, dump, lib_records, rec_line  # noqa: E402
from run_reference_library import scenario_inputs  # noqa: E402

import hetserve.kernels as RK  # noqa: E402
from hetserve.perf import ProfileTable  # noqa: E402
from hetserve.templates import GenContext, build_library  # noqa: E402

from tests.helpers import zigzag_profile  # noqa: E402

assert RK.USE_NUMBA


def main(name):
    configs, models, slos, caps, ctx, regions, prices = scenario_inputs(name)
    prof = zigzag_profile(configs, models, ProfileTable)
    t0 = time.monotonic()
    lib = build_library(configs, models, slos, caps, GenContext(perf=ctx.perf, profile=prof),
                        workers=os.cpu_count())
    wall = time.monotonic() - t0
    lines = [rec_line(r) for r in lib_records(lib)]
    every = 7 if name == "core" else 97
    dump(f"profile_{name}.json.gz", {
        "count": len(lines), "sha256": digest(lines), "sample_every": every, "sample": lines[::every],
        "counts": {f"{k[0]}|{k[1]}": v for k, v in lib.counts_by_model_phase().items()},
        "reference_wall_s": wall, "workers": os.cpu_count(), "profile_entries": len(prof.entries)})
    print(name, len(lines), f"{wall:.1f}s")


if __name__ == "__main__":
    main(sys.argv[1])
