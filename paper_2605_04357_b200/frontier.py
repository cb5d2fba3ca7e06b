"""Per-(model, phase, region) throughput-vs-cost Pareto frontier of stage 1.

The reference has no frontier step; its nearest analogues are the
stage-2 cost-efficiency prune (allocation.py:131-153) and the sweep's best
tokens/s per USD-h (cli.py:253-260). This module is the new output the north star
asks for, defined exactly as the oracle in SURVEY.md 8c:

  for each (model, phase) and region r, over templates t whose price
  p = sum_(cfg, n) n * price[r, cfg] (allocation.py:91-98, sequential in combo order;
  unpriced configs drop the template) exists, sort by (p asc, T desc, str(combo) asc)
  and keep t iff T > the running max of T over the earlier ones.

Everything runs on the device (pricing, an exact bucketed prefilter, one stable sort,
segmented running max, compaction); with torch.distributed initialised the candidates are interleaved over
ranks and the per-rank frontiers are merged after ONE NCCL all-gather.
"""

from __future__ import annotations

from collections import namedtuple
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .library import GenContext, Stage1Problem, TemplateLibrary, library_meta
from .shard import calibrate, pieces_to_ranges, plan_pieces
from .specs import PHASES, NodeComboKey, Placement, ServingTemplate


class FrontierEntry(namedtuple("FrontierEntry", ("template", "price_usd_h"))):
    """One survivor: the template and its one-instance price (USD/h) in the segment's region."""

    __slots__ = ()

    @property
    def throughput_tps(self) -> float:
        return self.template.throughput_tps


@dataclass
class TemplateFrontier:
    """Frontier survivors per (model, phase, region), each list in ascending price."""

    segments: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)
    num_candidates: int = 0

    def templates_for(self, model: str, phase: str, region: str) -> list:
        return self.segments.get((model, phase, region), [])

    def __len__(self) -> int:
        return sum(len(v) for v in self.segments.values())

    def library(self) -> TemplateLibrary:
        """Union of the survivors over regions as a TemplateLibrary, the input the
        unchanged stage-2 MILP (allocation.build_allocation_model) consumes."""
        seen = {}
        for entries in self.segments.values():
            for e in entries:
                seen[id(e.template)] = e.template
        return TemplateLibrary(entries=list(seen.values()), meta=dict(self.meta))


def _price_matrix(configs, prices, regions):
    """prices: {(region, config name): USD/h} or an object with .prices -> [R, K]."""
    table = getattr(prices, "prices", prices)
    if regions is None:
        regions = sorted({r for r, _ in table})
    regions = [getattr(r, "name", r) for r in regions]
    mat = np.full((len(regions), len(configs)), np.nan)
    for i, r in enumerate(regions):
        for k, c in enumerate(configs):
            p = table.get((r, c.name))
            if p is not None:
                mat[i, k] = float(p)
    return regions, mat


def _dist_info(dist):
    if dist is False:
        return None
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()):
        return None
    if tdist.get_world_size() <= 1:
        return None
    return tdist


# Items per rank of the single all-gather. Grown (never shrunk) from the largest
# partial frontier seen; every rank derives it from the same gathered headers, so all
# ranks always agree on it without a separate exchange.
_MERGE_CAP = [4096]
_GATHER_BUFS: dict = {}


def _gather_merge(fill, merge, tdist, device, item_bytes: int):
    """ONE all-gather of fixed-capacity partial frontiers (north_star: "merged with a
    single NCCL all-gather"), with no host round trip before it: each rank's slot is
    [int64 count | cap items], written by fill(send, offset_bytes, cap) on the device
    (the count may exceed cap: overflow). merge(recv, stride, offset_bytes, cap) reads
    the counts on the device and returns (result, largest count). All ranks see the
    same headers, so if some part overflowed all grow cap to the next power of two and
    repeat once."""
    import torch
    world = tdist.get_world_size()
    hdr = item_bytes
    for _ in range(2):
        cap = _MERGE_CAP[0]
        stride = hdr + cap * item_bytes
        key = (str(device), world, stride)
        bufs = _GATHER_BUFS.get(key)
        if bufs is None:
            _GATHER_BUFS.clear()  # one live size
            bufs = (torch.empty(stride, dtype=torch.uint8, device=device),
                    torch.empty(world * stride, dtype=torch.uint8, device=device))
            _GATHER_BUFS[key] = bufs
        send, recv = bufs
        fill(send, hdr, cap)
        tdist.all_gather_into_tensor(recv, send)
        res, mx = merge(recv, stride, hdr, cap)
        if mx <= cap:
            return res
        grow = 1
        while grow < mx:
            grow <<= 1
        _MERGE_CAP[0] = max(cap, grow)
    raise RuntimeError("partial frontier capacity did not converge")


def _frontier_across_ranks(prob: Stage1Problem, pmat, tdist) -> int:
    """Each rank's exactly prefiltered candidates (items no strictly cheaper item of the
    shard dominates) go straight into its all-gather slot; after the single all-gather
    every rank takes the same skyline over the union (associative: all ranks end
    identical). The skyline of the union of prefiltered shards is the global skyline,
    because every dropped item's dominator is itself in the union or dominated by a
    kept, cheaper one. One host sync per step: the merge's survivor count."""
    import torch
    dev = torch.device("cuda", prob.h.device)
    item = _native.FRONTIER_DTYPE.itemsize
    world = tdist.get_world_size()

    def fill(send, offset, cap):
        prob.h.frontier_candidates_into(pmat, send.data_ptr(), offset, cap)

    def merge(recv, stride, offset, cap):
        return prob.h.frontier_merge_gathered(recv.data_ptr(), world, stride, offset, cap)

    return _gather_merge(fill, merge, tdist, dev, item)


_CALIBRATION: dict = {}
_PIECES: dict = {}
_MEMO_KEEP = 64  # distinct problems remembered (oldest dropped first)


def _remember(memo: dict, key, value) -> None:
    if len(memo) >= _MEMO_KEEP:
        memo.pop(next(iter(memo)))
    memo[key] = value


def rank_pieces(prob: Stage1Problem, tdist) -> list:
    """This rank's evaluation pieces (shard.plan_pieces): (model, phase, S)
    units, the largest split by candidate range, balanced on costs measured once per
    problem on rank 0 (shard.calibrate) and broadcast, so every rank derives the same
    plan. Needs the problem's tables and enumeration. Memoised on the problem's
    signature (its inputs fix the candidate counts): a repeat solve enqueues its
    evaluation without reading the counts back first."""
    world, rank = tdist.get_world_size(), tdist.get_rank()
    pkey = (prob.signature(), world, rank)
    hit = _PIECES.get(pkey)
    if hit is not None:
        return hit
    prob.counts = prob.h.num_combos()
    NP = len(prob.phases)
    _, lsteps, smax = prob.h.table_layout()
    smax_mp = [min(int(smax[mp // NP]), int(lsteps[mp // NP])) if prob.counts[mp // NP] else 0
               for mp in range(len(prob.models) * NP)]
    key = (tuple(int(c) for c in prob.counts), tuple(int(x) for x in lsteps), tuple(smax_mp), NP,
           prob.signature())
    costs = _CALIBRATION.get(key)
    if costs is None:
        world = tdist.get_world_size()
        costs = calibrate(prob.h, len(smax_mp), smax_mp, NP) if tdist.get_rank() == 0 else None
        if world > 1:
            box = [costs]
            tdist.broadcast_object_list(box, src=0)
            costs = box[0]
        _remember(_CALIBRATION, key, costs)
    plan = plan_pieces(costs, world)
    pieces = pieces_to_ranges(plan[rank], prob.counts, NP)
    _remember(_PIECES, pkey, pieces)
    return pieces


def build_frontier(configs, models, slos, caps, prices, regions=None, ctx=None,
                   phases=PHASES, dist=None, return_problem: bool = False):
    """Stage 1 end to end on the GPU: spec tables in, frontier templates out.

    `prices` is a MarketState-like object (`.prices`) or its dict
    {(region, config name): USD/h}; `regions` defaults to every region priced.
    """
    ctx = ctx or GenContext()
    configs_sorted = sorted(configs, key=lambda c: c.name)
    meta = library_meta(configs_sorted, models, slos, caps, ctx)
    region_names, pmat = _price_matrix(configs_sorted, prices, regions)
    if not models:
        return TemplateFrontier(meta=meta)
    prob = Stage1Problem(configs, models, slos, caps, ctx, phases)
    tdist = _dist_info(dist)
    if tdist is not None:
        prob.h.tables()
        prob.h.enumerate()
        prob.h.evaluate_pieces(rank_pieces(prob, tdist))
        n = _frontier_across_ranks(prob, pmat, tdist)
        prob.counts = prob.h.num_combos()  # ready by now: no wait
        NP = len(prob.phases)
        prob.cand_off = np.zeros(len(prob.models) * NP + 1, dtype=np.int64)
        for mp in range(len(prob.models) * NP):
            prob.cand_off[mp + 1] = prob.cand_off[mp] + prob.counts[mp // NP]
    else:
        prob.run()
        n = prob.h.frontier(pmat)
    items = prob.h.get_frontier(n)
    front = materialise(prob, items, region_names, meta)
    return (front, prob) if return_problem else front


def materialise(prob: Stage1Problem, items: np.ndarray, region_names, meta) -> TemplateFrontier:
    """Survivor records -> ServingTemplate objects (one per (mp, combo)), built by the
    CPython extension _lib/_materialize (csrc/materialize.c)."""
    from ._lib import _materialize
    from .library import _no_gc
    with _no_gc():
        segments = _materialise_native(_materialize, prob, items, region_names)
    return TemplateFrontier(segments=segments, meta=meta,
                            num_candidates=int(prob.cand_off[-1]) if prob.cand_off is not None else 0)


def _materialise_native(mod, prob, items, region_names):
    items = np.ascontiguousarray(items)
    return mod.materialise(items.view(np.uint8).tobytes() if len(items) else b"", list(prob.cfg_by_rank),
                           [m.name for m in prob.models], tuple(prob.phases),
                           [prob.slos[m.name] for m in prob.models], list(region_names),
                           len(prob.phases), ServingTemplate, Placement, NodeComboKey, FrontierEntry)


def materialise_py(prob: Stage1Problem, items: np.ndarray, region_names, meta) -> TemplateFrontier:
    """Pure-Python twin of materialise (used by the tests to check the extension)."""
    NP = len(prob.phases)
    cache = {}
    segments = {}
    mps = items["mp"].tolist()
    keys = items["combo_key"].tolist()
    first = {}
    for i, mk in enumerate(zip(mps, keys)):
        first.setdefault(mk, i)
    uniq = list(first.values())
    objs = prob.combo_objects(items["combo_key"][uniq]) if uniq else []
    combo_of = dict(zip(first.keys(), objs))
    regs = items["region"].tolist()
    prices = items["price_usd_h"].tolist()
    rec = items["rec"]
    tps = rec["throughput_tps"].tolist()
    nst = rec["num_stages"].tolist()
    nn = rec["num_nodes"].tolist()
    lps = rec["layers_per_stage"].tolist()
    son = rec["stage_of_node"].tolist()
    models, phases, slos = prob.models, prob.phases, prob.slos
    new = object.__new__
    for i in range(len(mps)):
        mp, key = mps[i], keys[i]
        t = cache.get((mp, key))
        if t is None:
            model = models[mp // NP]
            S = nst[i]
            pl = new(Placement)
            pl.__dict__.update(num_stages=S, layers_per_stage=tuple(lps[i][:S]),
                               stage_of_node=tuple(son[i][:nn[i]]))
            t = new(ServingTemplate)
            t.__dict__.update(model=model.name, phase=phases[mp % NP], slo=slos[model.name],
                              combo=combo_of[(mp, key)], placement=pl, throughput_tps=tps[i])
            cache[(mp, key)] = t
        seg = (t.model, t.phase, region_names[regs[i]])
        entries = segments.get(seg)
        if entries is None:
            entries = segments[seg] = []
        entries.append(FrontierEntry(t, prices[i]))
    return TemplateFrontier(segments=segments, meta=meta,
                            num_candidates=int(prob.cand_off[-1]) if prob.cand_off is not None else 0)


class FrontierSession:
    """Stage 1 solved once, frontiers re-priced many times (BASELINE config 4).

    Stage-1 records are price-invariant (T-hat and the DP never read prices), so an
    epoch whose prices or regions change only re-runs the device pricing + skyline
    over the cached records ("incremental re-solve").
    """

    def __init__(self, configs, models, slos, caps, ctx=None, phases=PHASES):
        self.ctx = ctx or GenContext()
        self.prob = Stage1Problem(configs, models, slos, caps, self.ctx, phases).run()
        self.meta = library_meta(self.prob.configs, models, slos, caps, self.ctx)

    def frontier(self, prices, regions=None) -> TemplateFrontier:
        region_names, pmat = _price_matrix(self.prob.configs, prices, regions)
        n = self.prob.h.frontier(pmat)
        return materialise(self.prob, self.prob.h.get_frontier(n), region_names, self.meta)


__all__ = ["FrontierEntry", "FrontierSession", "TemplateFrontier", "build_frontier", "materialise"]


def sweep(configs, models, slos, caps_list, prices, regions=None, ctx=None, phases=PHASES):
    """cmd_sweep (cli.py:233-272) for a list of LibraryCaps from ONE device solve.

    Stage-1 records do not depend on the caps (only the enumeration window does), so
    the problem is solved once at the widest caps and every entry is a device-side
    filter. Rows mirror the reference CSV:
    (n_max, rho, templates, gen_seconds, best_tokens_per_usd_h); gen_seconds is the
    shared solve + sweep wall time. Caps must stay within the GPU envelope (n_max <= 7).
    """
    import time

    from .library import LibraryCaps, LibraryGenError
    t0 = time.monotonic()
    widest = LibraryCaps(max(c.n_max for c in caps_list), max(c.rho for c in caps_list))
    prob = Stage1Problem(configs, models, slos, widest, ctx or GenContext(), phases).run()
    _, pmat = _price_matrix(prob.configs, prices, regions)
    counts, best, unpriced, mp_counts = prob.h.sweep([c.n_max for c in caps_list], [c.rho for c in caps_list],
                                                     pmat, (1 << len(prob.phases)) - 1)
    NP = len(prob.phases)
    for k, c in enumerate(caps_list):
        # build_library at these caps raises first (templates.py:499-502) ...
        missing = [(prob.models[mp // NP].name, prob.phases[mp % NP])
                   for mp in range(mp_counts.shape[1]) if mp_counts[k, mp] == 0]
        if missing:
            raise LibraryGenError(f"no feasible template for: {sorted(missing)}")
        # ... then cli.py:255 indexes scenario.prices[(region, config)] for every template
        if unpriced[k]:
            raise KeyError(f"{int(unpriced[k])} templates at caps ({c.n_max}, {c.rho}) use a config "
                           "without a price in some region")
    wall = time.monotonic() - t0
    return [(c.n_max, c.rho, int(n), wall, float(b)) for c, n, b in zip(caps_list, counts, best)]


__all__.append("sweep")
