"""Write the GPU-produced BASELINE config-1 frontier (as a TemplateLibrary file) for the
reference-interop test (tests/test_reference_interop.py runs the unchanged reference
stage 2 on it in the build container).

  python tools/dump_c1_frontier.py OUT.jsonl
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_04357_b200 import build_frontier  # noqa: E402
from tests.helpers import workload  # noqa: E402

configs, models, slos, caps, ctx, regions, prices = workload("c1")
front = build_frontier(configs, models, slos, caps, prices, regions=regions, ctx=ctx)
lib = front.library()
lib.reindex()
lib.save(sys.argv[1])
print(f"wrote {sys.argv[1]}: {len(lib)} frontier templates")
