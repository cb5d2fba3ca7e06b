"""Kernel-level operator mirror: `placement_search` (kernels.py:279-295 of the reference).

Same signature, argument meaning, return layout and errors as
/root/reference/pkg/src/hetserve/kernels.py:279-295, executed by the CUDA placement
DP (the numba `_placement_dp_nb`, kernels.py:143-276, defines the tie rules).
`placement_search_batch` runs many cases in one launch (one CTA per case).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .specs import DomainError

NEG_INF = _native.NEG_INF


def placement_search_batch(cases):
    """cases: iterable of (counts[C], tput[C, L], S). Returns a list of
    (objective, stage_layers[S], stage_counts[S, C]) exactly like placement_search."""
    cases = list(cases)
    if not cases:
        return []
    ncfg, counts, lsteps, offs, S_arr, flat = [], [], [], [], [], []
    off = 0
    for cnt, tput, S in cases:
        cnt = np.ascontiguousarray(cnt, dtype=np.int64)
        tput = np.ascontiguousarray(tput, dtype=np.float64)
        if tput.ndim != 2 or tput.shape[0] != cnt.shape[0]:
            raise ValueError("tput must be (C, L) with C = len(counts)")
        if np.any(tput < 0):
            raise ValueError("throughput table must be non-negative")
        C = cnt.shape[0]
        if C > _native.MAX_NODES or int(cnt.sum()) > _native.MAX_NODES:
            raise DomainError(f"placement_search on the GPU covers <= {_native.MAX_NODES} nodes "
                              f"(got {C} configs, {int(cnt.sum())} nodes)")
        row = np.zeros(_native.MAX_NODES, dtype=np.int64)
        row[:C] = cnt
        ncfg.append(C)
        counts.append(row)
        lsteps.append(tput.shape[1])
        offs.append(off)
        S_arr.append(int(S))
        flat.append(tput.ravel())
        off += tput.size
    with _native.lease() as h:
        best, sj, sc = h.placement_search(np.array(ncfg), np.stack(counts), np.array(lsteps), np.array(offs),
                                          np.concatenate(flat), np.array(S_arr))
    out = []
    for i, (cnt, _, S) in enumerate(cases):
        C = len(cnt)
        S = int(S)
        if S > _native.MAX_NODES:  # more stages than any multiset has nodes: all zeros
            out.append((float(best[i]), np.zeros(S, dtype=np.int64), np.zeros((S, C), dtype=np.int64)))
        else:
            out.append((float(best[i]), sj[i, :S].copy(), sc[i, :S, :C].copy()))
    return out


def placement_search(counts, tput, S: int):
    """Best max-min pipeline layout for one node combo at a fixed stage count.

    counts: per-config node counts (len C); tput: (C, L) per-node throughput by layer
    count. Returns (objective, stage_layers[S], stage_counts[S, C]); objective is
    NEG_INF when no assignment exists (more stages than nodes or layers).
    """
    return placement_search_batch([(counts, tput, S)])[0]
