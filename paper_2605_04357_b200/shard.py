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
