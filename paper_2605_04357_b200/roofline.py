"""T-hat roofline operators on the GPU (simulator reuse).

Mirrors of the reference's per-node model and its template-level users:
  node_max_throughput (perf.py:159-175), planned_batch (perf.py:178-183),
  planned_batch_and_tput (perf.py:186-230), recompute_throughput
  (templates.py:267-280) and stage_node_weights (templates.py:283-293).
Every value comes from the CUDA kernel (csrc/roofline.cuh via coral_s1_node_queries);
`*_batch` forms evaluate many queries in one launch.
"""

from __future__ import annotations

from . import _native
from .library import GenContext, LibraryCaps, _pack_problem, stage_budget_s
from .specs import PREFILL, SloSpec


def _problem(h, nodes, models, params, profile):
    """A throw-away problem (on a leased handle) holding exactly the configs and models
    being queried."""
    cfgs, seen = [], {}
    for n in nodes:
        if n.name not in seen:
            seen[n.name] = len(cfgs)
            cfgs.append(n)
    mdls, mseen = [], {}
    for m in models:
        if m.name not in mseen:
            mseen[m.name] = len(mdls)
            mdls.append(m)
    ctx = GenContext(perf=params, profile=profile)
    arrays, scalars = _pack_problem(cfgs, mdls, {m.name: SloSpec(1.0, 1.0) for m in mdls},
                                    (PREFILL,), LibraryCaps(1, 2.0), ctx)
    h.set_problem(arrays, scalars)
    return seen, mseen


def node_queries(queries, params, profile=None, use_profile=True):
    """queries: iterable of (node, model, phase, j, stage_budget_s) -> (tputs, batches)."""
    queries = list(queries)
    if not queries:
        return [], []
    for _, _, phase, j, budget in queries:
        if not (budget > 0 and j >= 1):  # perf.py:189 assert
            raise AssertionError("stage_budget_s > 0 and j >= 1 required")
    with _native.lease() as h:
        cidx, midx = _problem(h, [q[0] for q in queries], [q[1] for q in queries], params, profile)
        tput, batch = h.node_queries([cidx[q[0].name] for q in queries], [midx[q[1].name] for q in queries],
                                     [_native.PHASE_CODE[q[2]] for q in queries], [q[3] for q in queries],
                                     [q[4] for q in queries], use_profile and profile is not None)
    return tput.tolist(), batch.tolist()


def node_max_throughput(node, model, phase, j, stage_budget_s, params, profile=None) -> float:
    return node_queries([(node, model, phase, j, stage_budget_s)], params, profile)[0][0]


def planned_batch_and_tput(node, model, phase, j, stage_budget_s, params):
    t, b = node_queries([(node, model, phase, j, stage_budget_s)], params, None, use_profile=False)
    return int(b[0]), float(t[0])


def planned_batch(node, model, phase, j, stage_budget_s, params) -> int:
    return planned_batch_and_tput(node, model, phase, j, stage_budget_s, params)[0]


def stage_node_weights(template, model, ctx) -> list:
    """Per-stage per-node expected throughput (templates.py:283-293)."""
    budget = stage_budget_s(model, template.slo, template.phase, template.placement.num_stages, ctx)
    stages = template.placement.stage_nodes(template.combo)
    qs = [(n, model, template.phase, template.placement.layers_per_stage[s], budget)
          for s, nodes in enumerate(stages) for n in nodes]
    vals, _ = node_queries(qs, ctx.perf, ctx.profile)
    out, k = [], 0
    for nodes in stages:
        out.append(vals[k:k + len(nodes)])
        k += len(nodes)
    return out


def recompute_throughput(template, model, ctx) -> float:
    """Min-stage aggregate throughput re-derived from the placement (templates.py:267-280)."""
    budget = stage_budget_s(model, template.slo, template.phase, template.placement.num_stages, ctx)
    if budget <= 0:
        return 0.0
    per_stage = stage_node_weights(template, model, ctx)
    return min(sum(v) for v in per_stage)
