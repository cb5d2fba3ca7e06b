"""Multi-GPU work split for stage 1.

Units are (model, phase, S) triples: each S has its own lattice layers and top
cells, and a candidate's best over S is combined with an order-independent rule
(ties -> fewer stages), so any rank may own any subset of S values of a (model,
phase). A rank that owns at least one S of a (model, phase) also pays that chain's
fixed part (its top-cell setup per candidate, memory-window table, decode, launches),
so assign_units places whole chains first and splits one only where moving an S unit
lowers the peak load by more than the repeated fixed part.

Cost model (milliseconds on one B200, fitted by tools/fit_shard.py to the unit and
chain timings of tools/calibrate_units.py on BASELINE config 2,
profiles/r01_calibration_v2.txt; relative rms error 0.18):
  fixed(chain)  = 0.045 + 9.0e-7 * candidates
  unit(chain,S) = 0.032 + 2.42e-8 * candidates * layer_units * W[S] * (1 + 2.2 * p[S])

p[S] is the fraction of positive entries of the chain's T-hat table at S (read from
the device tables before the split). Rows that fall to zero early let the capped
crossing searches stop early (csrc/placement_dp.cuh), so a chain's per-pair cost
tracks p: decode chains of the big models (p ~ 0.05-0.3) cost 1.2-1.6x less than their
prefill twins (p ~ 0.4-0.6). Without p the two phases tie in the greedy and land on
alternating ranks, so every prefill chain piles onto the same ranks.
"""

from __future__ import annotations

import functools

W = {1: 0.0, 2: 0.075, 3: 0.71, 4: 1.0, 5: 0.79, 6: 0.59}
OVERLAP = 0.8  # a rank with >= 3 chains runs them concurrently on 4 streams: ~0.8x their sum


def chain_fixed(ncombo: int) -> float:
    return 0.045 + 9.0e-7 * ncombo


def unit_cost(ncombo: int, lsteps: int, S: int, posfrac: float = 0.5) -> float:
    if S == 1:
        return 0.005
    return 0.032 + 2.42e-8 * ncombo * lsteps * W.get(S, 0.6) * (1.0 + 2.2 * posfrac)


def table_posfrac(handle, num_configs: int = 0) -> tuple:
    """Per (model, phase) chain, {S: fraction of positive T-hat entries}, counted by the
    device tables kernel (coral_s1_table_posfrac)."""
    pf = handle.table_posfrac()
    return tuple(tuple((S, float(pf[mp, S - 1])) for S in range(1, pf.shape[1] + 1))
                 for mp in range(pf.shape[0]))


def assign_units(counts, lsteps, smax, num_phases: int, world: int, posfrac=None) -> list:
    """-> per rank, a list of S bit-masks indexed by mp = model * num_phases + phase.
    posfrac: table_posfrac() of the problem (None: 0.5 everywhere). A pure function of
    its inputs, memoised (repeated solves of one problem reuse the split)."""
    key = (tuple(int(c) for c in counts), tuple(int(x) for x in lsteps), tuple(int(x) for x in smax),
           int(num_phases), int(world), posfrac if posfrac is None or isinstance(posfrac, tuple)
           else tuple(tuple(sorted(d.items())) for d in posfrac))
    return [list(r) for r in _assign_units(*key)]


@functools.lru_cache(maxsize=64)
def _assign_units(counts, lsteps, smax, num_phases, world, posfrac):
    """The split of assign_units (hashable arguments; posfrac as ((S, p), ...) per mp).

    Whole chains first (longest-processing-time order onto the least loaded rank),
    then single S units move from the most to the least loaded rank while that lowers
    the larger of the two loads; a rank receiving a piece of a chain pays the chain's
    fixed part again, so chains split only where the balance gains more than that."""
    nmp = len(counts) * num_phases
    unit = {}   # mp -> {S: cost}
    fixed = {}
    for m, (nc, lu, sm) in enumerate(zip(counts, lsteps, smax)):
        if not nc:
            continue
        for p in range(num_phases):
            mp = m * num_phases + p
            unit[mp] = {}
            for S in range(1, min(int(sm), int(lu)) + 1):
                pf = dict(posfrac[mp]).get(S, 0.5) if posfrac is not None else 0.5
                unit[mp][S] = unit_cost(int(nc), int(lu), S, pf)
            fixed[mp] = chain_fixed(int(nc))
    masks = [[0] * nmp for _ in range(world)]
    raw = [0.0] * world
    nch = [0] * world

    def eff(load, n):  # chains of one rank overlap on its streams (OVERLAP)
        return load * (1.0 if n <= 2 else OVERLAP)

    chains = sorted(unit, key=lambda mp: (-(fixed[mp] + sum(unit[mp].values())), mp))
    for mp in chains:
        c = fixed[mp] + sum(unit[mp].values())
        r = min(range(world), key=lambda i: (eff(raw[i] + c, nch[i] + 1), i))
        masks[r][mp] = sum(1 << S for S in unit[mp])
        raw[r] += c
        nch[r] += 1
    for _ in range(4 * len(unit) * 6):
        load = [eff(raw[i], nch[i]) for i in range(world)]
        hi = max(range(world), key=lambda i: (load[i], -i))
        best = None
        for lo in range(world):
            if lo == hi:
                continue
            for mp in range(nmp):
                mk = masks[hi][mp]
                if not mk:
                    continue
                for S, c in unit[mp].items():
                    if not (mk >> S) & 1:
                        continue
                    gone = mk == (1 << S)  # hi drops the chain entirely
                    new_hi = eff(raw[hi] - c - (fixed[mp] if gone else 0.0), nch[hi] - gone)
                    new_lo = eff(raw[lo] + c + (0.0 if masks[lo][mp] else fixed[mp]),
                                 nch[lo] + (0 if masks[lo][mp] else 1))
                    peak = max(new_hi, new_lo)
                    if peak < load[hi] - 1e-6 and (best is None or peak < best[0]):
                        best = (peak, lo, mp, S, gone)
        if best is None:
            break
        _, lo, mp, S, gone = best
        c = unit[mp][S]
        raw[hi] -= c + (fixed[mp] if gone else 0.0)
        nch[hi] -= int(gone)
        raw[lo] += c + (0.0 if masks[lo][mp] else fixed[mp])
        nch[lo] += 0 if masks[lo][mp] else 1
        masks[hi][mp] &= ~(1 << S)
        masks[lo][mp] |= 1 << S
    return tuple(tuple(r) for r in masks)


# ---------------------------------------------------------------------------------------
# Pieces: (model, phase, S) units whose top-cell candidates may be split by range
# ---------------------------------------------------------------------------------------
# A piece (mp, S-set, [a, b)) evaluates the stage counts S-set of slot mp for the
# candidates a..b (fractions of the model's candidate list, library order): the north
# star's (model, GPU-type combination) axis. Costs come from ONE measured calibration
# per problem (calibrate(): serial, S-isolated evaluations on the device, milliseconds):
#   L[mp][S]  value + layer kernels of S (the lattice: independent of the range)
#   T[mp][S]  marginal top-cell + decode work of S (proportional to the range)
#   F[mp]     per-candidate part every piece of mp pays once per range (rank table,
#             top-cell setup, decode, S = 1), proportional to the range
# A rank's load = sum over its pieces of L + T (b - a), plus F (b - a) once per distinct
# (mp, a, b); a rank runs its slots concurrently on its streams (CONCURRENT).


def calibrate(handle, nmp: int, smax_mp, num_phases: int = 2) -> tuple:
    """Measure (F, L, T) per (model, phase) slot on this device (see above): one serial
    evaluation per stage count S, each launch attributed to its slot."""
    handle.set_streams(1)
    handle.set_timing(True)
    try:
        maxS = max(smax_mp) if len(smax_mp) else 0
        F = [0.0] * nmp
        L = [dict() for _ in range(nmp)]
        T = [dict() for _ in range(nmp)]
        top1 = [0.0] * nmp
        handle.evaluate_pieces([(mp, (1 << (smax_mp[mp] + 1)) - 2, 0, -1) for mp in range(nmp) if smax_mp[mp]])
        for S in range(1, maxS + 1):
            pieces = [(mp, 1 << S, 0, -1) for mp in range(nmp) if smax_mp[mp] >= S]
            if not pieces:
                continue
            lay, top, rk = [float("inf")] * nmp, [float("inf")] * nmp, [float("inf")] * nmp
            for _ in range(2):  # warm, then the smaller of two serial runs per launch kind
                handle.evaluate_pieces(pieces)
                a, b, c = [0.0] * nmp, [0.0] * nmp, [0.0] * nmp
                for kind, mp, ms in handle.kernel_launches():
                    if mp < 0 or mp >= nmp:
                        continue
                    if kind in (1, 2):
                        a[mp] += ms
                    elif kind in (0, 3):
                        b[mp] += ms
                    elif kind == 4:
                        c[mp] += ms
                lay = [min(x, y) for x, y in zip(lay, a)]
                top = [min(x, y) for x, y in zip(top, b)]
                rk = [min(x, y) for x, y in zip(rk, c)]
            for mp in range(nmp):
                if smax_mp[mp] < S:
                    continue
                if S == 1:
                    # the rank table is launch-tagged with the model's first slot; every
                    # slot that runs on a stream of its own computes it
                    top1[mp] = top[mp]
                    F[mp] = top[mp] + rk[mp - mp % num_phases]
                else:
                    L[mp][S] = lay[mp]
                    T[mp][S] = max(0.0, top[mp] - top1[mp])
        return tuple(F), tuple(tuple(sorted(d.items())) for d in L), tuple(tuple(sorted(d.items())) for d in T)
    finally:
        handle.set_streams(0)
        handle.set_timing(False)


CONCURRENT = 0.92  # a rank runs its (model, phase) slots on up to 4 streams at once
#                   (tools/plan_check.py: two big slots overlap to ~0.90-0.93 of their sum)


def _rank_load(pieces, F, L, T):
    """Device time of a rank's pieces: the pieces of one (model, phase) slot run in order
    on one stream (a rank table + per-candidate setup F once per distinct range); slots
    run concurrently (the sum scaled by CONCURRENT, never below the longest slot)."""
    groups, ranges = {}, set()
    for mp, S, a, b in pieces:
        g = groups.get(mp, 0.0)
        if (mp, a, b) not in ranges:
            ranges.add((mp, a, b))
            g += F[mp] * (b - a)
        groups[mp] = g + L[mp].get(S, 0.0) + T[mp].get(S, 0.0) * (b - a)
    if not groups:
        return 0.0
    tot, top = sum(groups.values()), max(groups.values())
    return max(top, tot * (CONCURRENT if len(groups) > 1 else 1.0))


def plan_pieces(costs, world: int, max_depth: int = 3) -> list:
    """-> per rank a list of pieces (mp, smask, a, b) (fractions a < b of the model's
    candidates) that cover every (mp, S) unit and every candidate exactly once."""
    return [list(r) for r in _plan_pieces(costs, int(world), int(max_depth))]


@functools.lru_cache(maxsize=64)
def _plan_pieces(costs, world, max_depth):
    F, Lt, Tt = costs
    L = [dict(x) for x in Lt]
    T = [dict(x) for x in Tt]
    nmp = len(F)
    units = []  # (mp, S): S = 1 rides with S = 2 (or alone when it is the only S)
    for mp in range(nmp):
        Ss = sorted(set(L[mp]) | set(T[mp]))
        if not Ss and F[mp] > 0:
            units.append((mp, 1))
        units += [(mp, S) for S in Ss]
    ranks = [[] for _ in range(world)]

    def load(r, extra=(), drop=()):
        ps = [p for p in ranks[r] if p not in drop] + list(extra)
        return _rank_load(ps, F, L, T)

    # whole chains first (longest first onto the least loaded rank): a chain split over
    # ranks pays its per-candidate part F once per rank; the moves below split only
    # where that pays off
    chains = {}
    for mp, S in units:
        chains.setdefault(mp, []).append((mp, S, 0.0, 1.0))
    order = sorted(chains, key=lambda mp: (-_rank_load(chains[mp], F, L, T), mp))
    for mp in order:
        r = min(range(world), key=lambda i: (load(i, extra=chains[mp]), i))
        ranks[r] += chains[mp]
    for _ in range(64 * world):
        loads = [load(i) for i in range(world)]
        hi = max(range(world), key=lambda i: (loads[i], -i))
        best = None
        for p in ranks[hi]:
            mp, S, a, b = p
            for r in range(world):
                if r == hi:
                    continue
                # (a) move the piece
                nh, nr = load(hi, drop=(p,)), load(r, extra=(p,))
                peak = max(nh, nr)
                if peak < loads[hi] - 1e-6 and (best is None or peak < best[0]):
                    best = (peak, "move", p, r)
                # (b) split it: keep [a, m), give [m, b)
                if (b - a) > 1.0 / (1 << max_depth) + 1e-12:
                    m = (a + b) / 2
                    keep, give = (mp, S, a, m), (mp, S, m, b)
                    nh = load(hi, extra=(keep,), drop=(p,))
                    nr = load(r, extra=(give,))
                    peak = max(nh, nr)
                    if peak < loads[hi] - 1e-6 and (best is None or peak < best[0]):
                        best = (peak, "split", p, r)
            # (c) swap it with a piece of another rank
            for r in range(world):
                if r == hi:
                    continue
                for q in ranks[r]:
                    nh, nr = load(hi, extra=(q,), drop=(p,)), load(r, extra=(p,), drop=(q,))
                    peak = max(nh, nr)
                    if peak < loads[hi] - 1e-6 and (best is None or peak < best[0]):
                        best = (peak, "swap", p, (r, q))
        if best is None:
            break
        _, kind, p, r = best
        ranks[hi].remove(p)
        if kind == "swap":
            r, q = r
            ranks[r].remove(q)
            ranks[r].append(p)
            ranks[hi].append(q)
        elif kind == "move":
            ranks[r].append(p)
        else:
            mp, S, a, b = p
            m = (a + b) / 2
            ranks[hi].append((mp, S, a, m))
            ranks[r].append((mp, S, m, b))
    out = []
    for r in range(world):
        merged = {}
        for mp, S, a, b in ranks[r]:
            bits = (1 << S) | ((1 << 1) if S == 2 or (S == 1) else 0)
            merged[(mp, a, b)] = merged.get((mp, a, b), 0) | bits
        out.append(tuple(sorted((mp, mk, a, b) for (mp, a, b), mk in merged.items())))
    return tuple(out)


def pieces_to_ranges(pieces, counts, num_phases: int) -> list:
    """Fractional pieces -> (mp, smask, lo, hi) with candidate indices of the model."""
    out = []
    for mp, mk, a, b in pieces:
        n = int(counts[mp // num_phases])
        lo, hi = int(round(a * n)), int(round(b * n))
        if hi > lo:
            out.append((mp, mk, lo, hi))
    return out
