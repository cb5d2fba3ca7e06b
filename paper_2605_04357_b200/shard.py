"""Multi-GPU work split for stage 1.

Units are (model, phase, S) triples: each S has its own lattice layers and top
cells, and a candidate's best over S is combined with an order-independent rule
(ties -> fewer stages), so any rank may own any subset of S values of a (model,
phase). A rank that owns at least one S of a (model, phase) also pays that chain's
fixed part (its top-cell setup per candidate, memory-window table, decode, launches),
so the greedy below charges the fixed part once per (rank, chain) and keeps the S
values of a chain together unless splitting balances better.

Cost model (milliseconds on one B200, calibrated with tools/calibrate_units.py on
BASELINE config 2, profiles/r01_calibration.txt):
  fixed(chain)  = 0.09 + 1.4e-6 * candidates
  unit(chain,S) = 6.8e-8 * candidates * layer_units * W[S] * PHASE_W[phase]

PHASE_W: prefill chains of the same model measure 1.01-1.37x their decode twins
(profiles/r01_calibration.txt: more crossing searches survive the dp_pair end-point
shortcuts). Without a weight the two phases tie in the greedy and land on
alternating ranks, so every prefill chain piles onto the same ranks; 1.1 balanced
best over 2, 4 and 8 ranks (tools/sweep_phase_w.sh).
"""

from __future__ import annotations

import os

W = {1: 0.01, 2: 0.22, 3: 0.8, 4: 1.0, 5: 0.7, 6: 0.45}
PHASE_W = (float(os.environ.get("CORAL_SHARD_PREFILL_W", "1.1")), 1.0)  # (prefill, decode)


def chain_fixed(ncombo: int) -> float:
    return 0.09 + 1.4e-6 * ncombo


def unit_cost(ncombo: int, lsteps: int, S: int, phase: int = 1) -> float:
    return 6.8e-8 * ncombo * lsteps * W.get(S, 0.5) * PHASE_W[phase if phase < len(PHASE_W) else 1] + 0.005


def assign_units(counts, lsteps, smax, num_phases: int, world: int) -> list:
    """-> per rank, a list of S bit-masks indexed by mp = model * num_phases + phase."""
    units = []
    for m, (nc, lu, sm) in enumerate(zip(counts, lsteps, smax)):
        if not nc:
            continue
        for p in range(num_phases):
            for S in range(1, min(int(sm), int(lu)) + 1):
                units.append((unit_cost(int(nc), int(lu), S, p if num_phases == 2 else 1), m * num_phases + p, S))
    units.sort(key=lambda u: -u[0])  # stable: ties keep (mp, S) order
    load = [0.0] * world
    nmp = len(counts) * num_phases
    masks = [[0] * nmp for _ in range(world)]
    for cost, mp, S in units:
        fixed = chain_fixed(int(counts[mp // num_phases]))

        def after(r):
            return load[r] + cost + (0.0 if masks[r][mp] else fixed)

        r = min(range(world), key=lambda i: (after(i), i))
        load[r] = after(r)
        masks[r][mp] |= 1 << S
    return masks
