"""TEST INFRASTRUCTURE: ctypes front end of the C oracle (coral_oracle.c).

Restates the reference's stage-1 algorithm on the CPU so tests can check the CUDA
path on identical inputs. Never imported by the product package.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
NEG_INF = -1e300
MAXC = 6


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "coral_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "build/liboracle.so"],
                       check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp, i64, f64p = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
        L.or_stage_budget.restype = C.c_double
        L.or_stage_budget.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.or_node_max_throughput.restype = C.c_double
        L.or_node_max_throughput.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
        L.or_throughput_table.restype = None
        L.or_throughput_table.argtypes = [vp, C.c_int, C.c_int, C.c_int, f64p]
        L.or_enumerate.restype = i64
        L.or_enumerate.argtypes = [vp, C.c_int, C.POINTER(C.c_uint64), i64]
        L.or_placement_search.restype = C.c_double
        L.or_placement_search.argtypes = [C.POINTER(C.c_int64), C.c_int, f64p, C.c_int, C.c_int,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_solve_many.restype = None
        L.or_solve_many.argtypes = [vp, C.c_int, f64p, C.POINTER(C.c_uint64), i64, i64, i64, vp, C.c_int,
                                    C.c_uint32]
        L.or_frontier.restype = i64
        L.or_frontier.argtypes = [vp, C.POINTER(C.c_uint64), vp, i64, C.c_int, f64p,
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        _lib = L
    return _lib


class OracleProblem:
    """The same coral_s1_problem struct the product's C ABI takes, for the oracle."""

    def __init__(self, arrays: dict, scalars: dict):
        from paper_2605_04357_b200._native import Problem
        p = Problem()
        self._keep = []
        for name, ctype in Problem._fields_:
            if name in arrays:
                base = ctype._type_
                dt = np.int32 if base is C.c_int32 else np.float64
                arr = np.ascontiguousarray(arrays[name], dtype=dt)
                if arr.size == 0:
                    arr = np.zeros(1, dtype=dt)
                self._keep.append(arr)
                setattr(p, name, arr.ctypes.data_as(ctype))
        for name, v in scalars.items():
            setattr(p, name, v)
        self.p = p
        self.arrays, self.scalars = arrays, scalars
        self.ref = C.byref(p)

    @classmethod
    def from_specs(cls, configs, models, slos, caps, ctx, phases):
        from paper_2605_04357_b200.library import _pack_problem
        configs = sorted(configs, key=lambda c: c.name)
        arrays, scalars = _pack_problem(configs, list(models), slos, tuple(phases), caps, ctx)
        op = cls(arrays, scalars)
        op.configs, op.models, op.phases = configs, list(models), tuple(phases)
        return op

    # -- restated reference functions ------------------------------------------
    def lsteps(self, m):
        return int(self.arrays["mdl_num_layers"][m]) // int(self.arrays["mdl_granularity"][m])

    def stage_budget(self, m, phase_code, S):
        return lib().or_stage_budget(self.ref, m, phase_code, S)

    def table(self, m, phase_code, S):
        K = self.scalars["num_configs"]
        out = np.zeros(K * self.lsteps(m))
        lib().or_throughput_table(self.ref, m, phase_code, S, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out.reshape(K, self.lsteps(m))

    def tables(self, m, phase_code):
        """S = 1..min(n_max, L) stacked, as templates.py:445-447 builds them."""
        smax = min(self.scalars["n_max"], int(self.arrays["mdl_num_layers"][m]))
        return np.stack([self.table(m, phase_code, S) for S in range(1, smax + 1)])

    def enumerate(self, m):
        n = lib().or_enumerate(self.ref, m, None, 0)
        keys = np.zeros(max(n, 1), dtype=np.uint64)
        lib().or_enumerate(self.ref, m, keys.ctypes.data_as(C.POINTER(C.c_uint64)), n)
        return keys[:n]

    def solve(self, m, phase_code, keys, first=0, stride=1, tables=None, threads=0, smask=0):
        from paper_2605_04357_b200._native import RECORD_DTYPE
        if tables is None:
            tables = self.tables(m, phase_code)
        tables = np.ascontiguousarray(tables, dtype=np.float64)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        recs = np.zeros(max(len(keys), 1), dtype=RECORD_DTYPE)
        lib().or_solve_many(self.ref, m, tables.ctypes.data_as(C.POINTER(C.c_double)),
                            keys.ctypes.data_as(C.POINTER(C.c_uint64)), len(keys), first, stride,
                            recs.ctypes.data_as(C.c_void_p), threads, smask)
        return recs[:len(keys)]

    def frontier(self, keys, recs, prices):
        prices = np.ascontiguousarray(prices, dtype=np.float64)
        R = prices.shape[0]
        n = len(keys)
        reg = np.zeros(max(n * R, 1), dtype=np.int32)
        idx = np.zeros(max(n * R, 1), dtype=np.int64)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        recs = np.ascontiguousarray(recs)
        ns = lib().or_frontier(self.ref, keys.ctypes.data_as(C.POINTER(C.c_uint64)),
                               recs.ctypes.data_as(C.c_void_p), n, R,
                               prices.ctypes.data_as(C.POINTER(C.c_double)),
                               reg.ctypes.data_as(C.POINTER(C.c_int32)),
                               idx.ctypes.data_as(C.POINTER(C.c_int64)))
        return reg[:ns], idx[:ns]


def placement_search(counts, tput, S):
    """kernels.py:279-295 restated (numba tie rules): (best, stage_j[S], stage_counts[S, C])."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    tput = np.ascontiguousarray(tput, dtype=np.float64)
    C_ = counts.shape[0]
    L = tput.shape[1]
    sj = np.zeros(max(S, 1), dtype=np.int64)
    sc = np.zeros((max(S, 1), max(C_, 1)), dtype=np.int64)
    best = lib().or_placement_search(counts.ctypes.data_as(C.POINTER(C.c_int64)), C_,
                                     tput.ctypes.data_as(C.POINTER(C.c_double)), L, S,
                                     sj.ctypes.data_as(C.POINTER(C.c_int64)),
                                     sc.ctypes.data_as(C.POINTER(C.c_int64)))
    return best, sj[:S], sc[:S, :C_]
