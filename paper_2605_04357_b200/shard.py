"""Multi-GPU work split for stage 1.

Units are (model, phase, S) triples: each has its own lattice chain, and a candidate's
best over S is combined with an order-independent rule, so any rank may own any
subset of S values of a (model, phase). Units are assigned longest-processing-time
first on a deterministic cost estimate; every rank computes the same assignment.
"""

from __future__ import annotations


def unit_cost(ncombo: int, lsteps: int, S: int) -> float:
    """Relative cost of one (model, phase, S) unit: the top cells of every candidate
    plus S - 1 lattice layers over ~lsteps layer counts."""
    return ncombo * (1.0 + (S - 1) * lsteps / 8.0)


def assign_units(counts, lsteps, smax, num_phases: int, world: int) -> list:
    """-> per rank, a list of S bit-masks indexed by mp = model * num_phases + phase."""
    units = []
    for m, (nc, lu, sm) in enumerate(zip(counts, lsteps, smax)):
        for p in range(num_phases):
            for S in range(1, min(sm, lu) + 1):
                units.append((unit_cost(int(nc), int(lu), S), m * num_phases + p, S))
    units.sort(key=lambda u: -u[0])  # stable: ties keep (mp, S) order
    load = [0.0] * world
    masks = [[0] * (len(counts) * num_phases) for _ in range(world)]
    for cost, mp, S in units:
        r = min(range(world), key=lambda i: load[i])
        load[r] += cost
        masks[r][mp] |= 1 << S
    return masks
