"""ctypes binding of the C ABI in include/coral_s1.h (libcoral_s1.so, built in-tree).

There is no fallback: if the shared library is missing or no CUDA device is usable,
every entry point raises. The product path is the CUDA path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .specs import DomainError

# CORAL_S1_LIB: alternative build of the same library (A/B timing runs only)
_LIB_PATH = os.environ.get("CORAL_S1_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                           "libcoral_s1.so")

OK, EINVAL, ENOTEMPLATE, ECUDA, EUNSUPPORTED = 0, 1, 2, 3, 4
PHASE_CODE = {"prefill": 0, "decode": 1}
MAX_NODES = 7
NEG_INF = -1e300

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class Problem(C.Structure):
    _fields_ = [
        ("num_configs", C.c_int32), ("cfg_gpu_count", _i32p), ("cfg_mem_gb", _f64p),
        ("cfg_bw_tbps", _f64p), ("cfg_tflops", _f64p), ("cfg_str_rank", _i32p),
        ("num_models", C.c_int32), ("mdl_num_layers", _i32p), ("mdl_granularity", _i32p),
        ("mdl_params_total_b", _f64p), ("mdl_params_active_b", _f64p),
        ("mdl_hidden_size", _f64p), ("mdl_bytes_per_param", _f64p), ("mdl_kv_bytes", _f64p),
        ("slo_prefill_ms", _f64p), ("slo_decode_ms", _f64p),
        ("num_phases", C.c_int32), ("phases", _i32p),
        ("mfu", C.c_double), ("mbu", C.c_double), ("net_eff", C.c_double),
        ("fixed_overhead_ms", C.c_double), ("avg_prompt_tokens", C.c_double),
        ("avg_ctx_tokens", C.c_double), ("slo_budget_frac", C.c_double),
        ("net_gbps", C.c_double), ("net_latency_ms", C.c_double),
        ("n_max", C.c_int32), ("rho", C.c_double),
        ("num_profile", C.c_int32), ("prof_model", _i32p), ("prof_phase", _i32p),
        ("prof_cfg", _i32p), ("prof_j", _i32p), ("prof_bucket", _i32p), ("prof_tps", _f64p),
    ]


RECORD_DTYPE = np.dtype([("throughput_tps", "<f8"), ("num_stages", "u1"), ("num_nodes", "u1"),
                         ("layers_per_stage", "<u2", (MAX_NODES,)),
                         ("stage_of_node", "u1", (MAX_NODES,)), ("_pad", "u1", (1,))], align=True)
FRONTIER_DTYPE = np.dtype([("price_usd_h", "<f8"), ("throughput_tps", "<f8"),
                           ("combo_key", "<u8"), ("mp", "<i4"), ("region", "<i4"),
                           ("rec", RECORD_DTYPE)], align=True)
ALLOC_VAR_DTYPE = np.dtype([("combo_key", "<u8"), ("mp", "<i4"), ("region", "<i4"), ("ub", "<i8"),
                            ("price_usd_h", "<f8"), ("throughput_tps", "<f8")], align=True)
assert RECORD_DTYPE.itemsize == 32 and FRONTIER_DTYPE.itemsize == 64 and ALLOC_VAR_DTYPE.itemsize == 40

_lib = None
_lib_lock = threading.Lock()


def _ptr(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load libcoral_s1.so (raises if it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `python __graft_entry__.py build` "
                              "(the CUDA extension is the only implementation)")
        lib = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        sig = {
            "coral_s1_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "coral_s1_destroy": (C.c_int, [vp]),
            "coral_s1_last_error": (C.c_char_p, []),
            "coral_s1_version": (C.c_int, []),
            "coral_s1_set_stream": (C.c_int, [vp, vp]),
            "coral_s1_launch_count": (C.c_int64, [vp]),
            "coral_s1_set_problem": (C.c_int, [vp, C.POINTER(Problem)]),
            "coral_s1_tables": (C.c_int, [vp]),
            "coral_s1_table_layout": (C.c_int, [vp, _i64p, _i32p, _i32p]),
            "coral_s1_get_tables": (C.c_int, [vp, _f64p, C.c_int64]),
            "coral_s1_get_budgets": (C.c_int, [vp, _f64p, C.c_int64]),
            "coral_s1_enumerate": (C.c_int, [vp]),
            "coral_s1_num_combos": (C.c_int, [vp, _i64p]),
            "coral_s1_get_combos": (C.c_int, [vp, C.c_int, C.c_int, _u64p, C.c_int64]),
            "coral_s1_evaluate": (C.c_int, [vp, C.c_int64, C.c_int64]),
            "coral_s1_evaluate_units": (C.c_int, [vp, C.POINTER(C.c_uint32)]),
            "coral_s1_evaluate_pieces": (C.c_int, [vp, C.c_int, _i32p, C.POINTER(C.c_uint32), _i64p, _i64p]),
            "coral_s1_kernel_launches": (C.c_int, [vp, C.c_int64, _i32p, _i32p, _f64p, _i64p]),
            "coral_s1_num_candidates": (C.c_int, [vp, _i64p]),
            "coral_s1_get_records": (C.c_int, [vp, C.c_int, vp, C.c_int64]),
            "coral_s1_frontier": (C.c_int, [vp, C.c_int, _f64p, _i64p]),
            "coral_s1_get_frontier": (C.c_int, [vp, vp, C.c_int64]),
            "coral_s1_frontier_export_device": (C.c_int, [vp, vp, C.c_int64, _i64p]),
            "coral_s1_frontier_merge_device": (C.c_int, [vp, vp, C.c_int64, _i64p]),
            "coral_s1_placement_search": (C.c_int, [vp, C.c_int64, _i32p, _i64p, _i32p, _i64p,
                                                    _f64p, C.c_int64, _i32p, _f64p, _i64p, _i64p]),
            "coral_s1_stage_ms": (C.c_int, [vp, _f64p, _f64p, _f64p, _f64p]),
            "coral_s1_kernel_stats": (C.c_int, [vp, C.c_int, _f64p, _i64p]),
            "coral_s1_window_select_stats": (C.c_int, [vp, _f64p, _i64p]),
            "coral_s1_set_census": (C.c_int, [vp, C.c_int]),
            "coral_s1_set_timing": (C.c_int, [vp, C.c_int]),
            "coral_s1_table_posfrac": (C.c_int, [vp, _f64p, C.c_int64]),
            "coral_s1_frontier_merge_parts": (C.c_int, [vp, vp, C.c_int, C.c_int64, C.c_int64, _i64p, _i64p]),
            "coral_s1_frontier_candidates": (C.c_int, [vp, C.c_int, _f64p, _i64p]),
            "coral_s1_frontier_candidates_into": (C.c_int, [vp, C.c_int, _f64p, vp, C.c_int64, C.c_int64]),
            "coral_s1_frontier_merge_gathered": (C.c_int, [vp, vp, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                                           _i64p, _i64p]),
            "coral_s1_kernel_timeline": (C.c_int, [vp, C.c_int64, _i32p, _i32p, _f64p, _f64p, _i64p]),
            "coral_s1_census": (C.c_int, [vp, _i64p]),
            "coral_s1_census_all": (C.c_int, [vp, _i64p, C.c_int]),
            "coral_s1_set_streams": (C.c_int, [vp, C.c_int]),
            "coral_s1_write_library": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_int, _i32p,
                                                 C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                                 C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), _i64p]),
            "coral_s1_format_double": (C.c_int, [C.c_double, C.c_char_p, C.c_int]),
            "coral_s1_node_queries": (C.c_int, [vp, C.c_int64, _i32p, _i32p, _i32p, _i32p, _f64p, C.c_int,
                                                _f64p, _i64p]),
            "coral_s1_sweep": (C.c_int, [vp, C.c_int, _i32p, _f64p, C.c_int, _f64p, C.c_uint32, _i64p,
                                         _f64p, _i64p, _i64p]),
            "coral_s1_feasible_counts": (C.c_int, [vp, _i64p, C.c_int64]),
            "coral_s1_allocation_model": (C.c_int, [vp, C.c_int, _f64p, _i64p, _f64p, C.c_int, _i32p, C.c_double,
                                                    C.c_int64, _i32p, _i32p, _u64p, _i64p, _i64p, _f64p]),
            "coral_s1_get_allocation_vars": (C.c_int, [vp, vp, C.c_int64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list:
    """Every coral_s1_* function declared in include/coral_s1.h."""
    import re
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "include", "coral_s1.h")
    with open(hdr) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(coral_s1_[a-z_0-9]+)\s*\(", text)))


def format_double(v: float) -> str:
    """CPython repr(float) computed by the native writer's formatter (host only)."""
    buf = C.create_string_buffer(64)
    _check(load().coral_s1_format_double(float(v), buf, 64))
    return buf.value.decode()


class NativeError(RuntimeError):
    pass


class LibraryGenErrorNative(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().coral_s1_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise DomainError(msg)
    if rc == EUNSUPPORTED:
        raise DomainError(f"outside the GPU path's envelope: {msg}")
    if rc == ENOTEMPLATE:
        raise LibraryGenErrorNative(msg)
    raise NativeError(msg)


class Handle:
    """One device context (coral_s1_create/destroy) bound to torch's current stream."""

    def __init__(self, device: int = 0):
        lib = load()
        self._lib = lib
        self.device = device
        h = C.c_void_p()
        _check(lib.coral_s1_create(device, C.byref(h)))
        self._h = h
        self._keep = []
        self.NM = self.NP = self.K = 0

    def close(self):
        if self._h:
            self._lib.coral_s1_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        _check(self._lib.coral_s1_set_stream(self._h, C.c_void_p(stream_ptr)))

    @property
    def launches(self) -> int:
        return int(self._lib.coral_s1_launch_count(self._h))

    def set_problem(self, arrays: dict, scalars: dict):
        p = Problem()
        keep = []
        for name, ctype in (("cfg_gpu_count", C.c_int32), ("cfg_mem_gb", C.c_double),
                            ("cfg_bw_tbps", C.c_double), ("cfg_tflops", C.c_double),
                            ("cfg_str_rank", C.c_int32), ("mdl_num_layers", C.c_int32),
                            ("mdl_granularity", C.c_int32), ("mdl_params_total_b", C.c_double),
                            ("mdl_params_active_b", C.c_double), ("mdl_hidden_size", C.c_double),
                            ("mdl_bytes_per_param", C.c_double), ("mdl_kv_bytes", C.c_double),
                            ("slo_prefill_ms", C.c_double), ("slo_decode_ms", C.c_double),
                            ("phases", C.c_int32), ("prof_model", C.c_int32),
                            ("prof_phase", C.c_int32), ("prof_cfg", C.c_int32),
                            ("prof_j", C.c_int32), ("prof_bucket", C.c_int32),
                            ("prof_tps", C.c_double)):
            dt = np.int32 if ctype is C.c_int32 else np.float64
            arr = np.ascontiguousarray(arrays[name], dtype=dt)
            if arr.size == 0:
                arr = np.zeros(1, dtype=dt)
            keep.append(arr)
            setattr(p, name, _ptr(arr, ctype))
        for name, value in scalars.items():
            setattr(p, name, value)
        self._keep = keep
        self.NM, self.NP, self.K = p.num_models, p.num_phases, p.num_configs
        self.n_max = p.n_max
        _check(self._lib.coral_s1_set_problem(self._h, C.byref(p)))

    def tables(self):
        _check(self._lib.coral_s1_tables(self._h))

    def table_layout(self):
        offs = np.zeros(self.NM * self.NP + 1, dtype=np.int64)
        ls = np.zeros(max(self.NM, 1), dtype=np.int32)
        sm = np.zeros(max(self.NM, 1), dtype=np.int32)
        _check(self._lib.coral_s1_table_layout(self._h, _ptr(offs, C.c_int64), _ptr(ls, C.c_int32),
                                               _ptr(sm, C.c_int32)))
        return offs, ls[:self.NM], sm[:self.NM]

    def get_tables(self):
        offs, ls, sm = self.table_layout()
        out = np.zeros(max(int(offs[-1]), 1))
        _check(self._lib.coral_s1_get_tables(self._h, _ptr(out, C.c_double), out.size))
        return out, offs, ls

    def table_posfrac(self):
        """[mp][n_max] fraction of positive T-hat entries (device-counted by the tables kernel)."""
        out = np.zeros(max(self.NM * self.NP * self.n_max, 1))
        _check(self._lib.coral_s1_table_posfrac(self._h, _ptr(out, C.c_double), out.size))
        return out[:self.NM * self.NP * self.n_max].reshape(self.NM * self.NP, self.n_max)

    def get_budgets(self):
        out = np.zeros(max(self.NM * self.NP * self.n_max, 1))
        _check(self._lib.coral_s1_get_budgets(self._h, _ptr(out, C.c_double), out.size))
        return out[:self.NM * self.NP * self.n_max].reshape(self.NM * self.NP, self.n_max)

    def enumerate(self):
        _check(self._lib.coral_s1_enumerate(self._h))

    def num_combos(self):
        out = np.zeros(max(self.NM, 1), dtype=np.int64)
        _check(self._lib.coral_s1_num_combos(self._h, _ptr(out, C.c_int64)))
        return out[:self.NM]

    def get_combos(self, model: int, enumeration_order: bool = False, count=None):
        if count is None:
            count = int(self.num_combos()[model])
        out = np.zeros(max(count, 1), dtype=np.uint64)
        _check(self._lib.coral_s1_get_combos(self._h, model, int(enumeration_order),
                                             _ptr(out, C.c_uint64), out.size))
        return out[:count]

    def evaluate(self, lo: int = 0, hi: int = -1):
        _check(self._lib.coral_s1_evaluate(self._h, lo, hi))

    def evaluate_units(self, smask):
        m = np.ascontiguousarray(smask, dtype=np.uint32)
        _check(self._lib.coral_s1_evaluate_units(self._h, m.ctypes.data_as(C.POINTER(C.c_uint32))))

    def evaluate_pieces(self, pieces):
        """pieces: [(mp, smask, lo, hi)] -- stage counts smask of slot mp for the model's
        candidates [lo, hi) (hi < 0: to the end)."""
        n = len(pieces)
        mp = np.ascontiguousarray([p[0] for p in pieces] or [0], dtype=np.int32)
        sm = np.ascontiguousarray([p[1] for p in pieces] or [0], dtype=np.uint32)
        lo = np.ascontiguousarray([p[2] for p in pieces] or [0], dtype=np.int64)
        hi = np.ascontiguousarray([p[3] for p in pieces] or [0], dtype=np.int64)
        _check(self._lib.coral_s1_evaluate_pieces(self._h, n, _ptr(mp, C.c_int32),
                                                  sm.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                  _ptr(lo, C.c_int64), _ptr(hi, C.c_int64)))

    def kernel_launches(self, cap: int = 2048):
        """[(kind, mp, ms)] of the last evaluate's timed lattice launches."""
        kind = np.zeros(cap, np.int32)
        mp = np.zeros(cap, np.int32)
        ms = np.zeros(cap)
        n = C.c_int64()
        _check(self._lib.coral_s1_kernel_launches(self._h, cap, _ptr(kind, C.c_int32), _ptr(mp, C.c_int32),
                                                  _ptr(ms, C.c_double), C.byref(n)))
        k = n.value
        return list(zip(kind[:k].tolist(), mp[:k].tolist(), ms[:k].tolist()))

    def num_candidates(self) -> int:
        n = C.c_int64()
        _check(self._lib.coral_s1_num_candidates(self._h, C.byref(n)))
        return n.value

    def get_records(self, mp: int, count: int):
        out = np.zeros(max(count, 1), dtype=RECORD_DTYPE)
        _check(self._lib.coral_s1_get_records(self._h, mp, out.ctypes.data_as(C.c_void_p), out.size))
        return out[:count]

    def frontier(self, prices: np.ndarray) -> int:
        prices = np.ascontiguousarray(prices, dtype=np.float64)
        n = C.c_int64()
        _check(self._lib.coral_s1_frontier(self._h, prices.shape[0], _ptr(prices, C.c_double),
                                           C.byref(n)))
        return n.value

    def frontier_candidates(self, prices) -> int:
        """Prefiltered frontier candidates of this shard (no skyline), for a multi-GPU merge."""
        pm = np.ascontiguousarray(prices, dtype=np.float64)
        n = C.c_int64()
        _check(self._lib.coral_s1_frontier_candidates(self._h, pm.shape[0], _ptr(pm, C.c_double), C.byref(n)))
        return n.value

    def frontier_candidates_into(self, prices, dev_part: int, item_offset_bytes: int, cap: int) -> None:
        """The prefilter's candidates straight into a device slot: int64 count at dev_part
        (may exceed cap), items after item_offset_bytes. No host sync."""
        pm = np.ascontiguousarray(prices, dtype=np.float64)
        _check(self._lib.coral_s1_frontier_candidates_into(self._h, pm.shape[0], _ptr(pm, C.c_double),
                                                           C.c_void_p(dev_part), item_offset_bytes, cap))

    def frontier_merge_gathered(self, dev_ptr: int, parts: int, stride_bytes: int, item_offset_bytes: int,
                                cap: int):
        """Merge of gathered candidates_into slots, counts read on the device.
        -> (survivors or -1 if some part overflowed cap, largest part count)."""
        n, mx = C.c_int64(), C.c_int64()
        _check(self._lib.coral_s1_frontier_merge_gathered(self._h, C.c_void_p(dev_ptr), parts, stride_bytes,
                                                          item_offset_bytes, cap, C.byref(n), C.byref(mx)))
        return n.value, mx.value

    def get_frontier(self, count: int):
        out = np.zeros(max(count, 1), dtype=FRONTIER_DTYPE)
        _check(self._lib.coral_s1_get_frontier(self._h, out.ctypes.data_as(C.c_void_p), out.size))
        return out[:count]

    def frontier_export_device(self, dev_ptr: int, cap: int) -> int:
        n = C.c_int64()
        _check(self._lib.coral_s1_frontier_export_device(self._h, C.c_void_p(dev_ptr), cap, C.byref(n)))
        return n.value

    def frontier_merge_parts(self, dev_ptr: int, stride_bytes: int, item_offset_bytes: int, counts) -> int:
        cnt = np.ascontiguousarray(counts, dtype=np.int64)
        n = C.c_int64()
        _check(self._lib.coral_s1_frontier_merge_parts(self._h, C.c_void_p(dev_ptr), len(cnt), stride_bytes,
                                                       item_offset_bytes, _ptr(cnt, C.c_int64), C.byref(n)))
        return n.value

    def frontier_merge_device(self, dev_ptr: int, n_items: int) -> int:
        n = C.c_int64()
        _check(self._lib.coral_s1_frontier_merge_device(self._h, C.c_void_p(dev_ptr), n_items,
                                                        C.byref(n)))
        return n.value

    def placement_search(self, ncfg, counts, lsteps, tput_off, tput, S):
        ncases = len(ncfg)
        ncfg = np.ascontiguousarray(ncfg, dtype=np.int32)
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        lsteps = np.ascontiguousarray(lsteps, dtype=np.int32)
        tput_off = np.ascontiguousarray(tput_off, dtype=np.int64)
        tput = np.ascontiguousarray(tput, dtype=np.float64)
        S = np.ascontiguousarray(S, dtype=np.int32)
        best = np.zeros(ncases)
        sj = np.zeros((ncases, MAX_NODES), dtype=np.int64)
        sc = np.zeros((ncases, MAX_NODES, MAX_NODES), dtype=np.int64)
        tp = tput if tput.size else np.zeros(1)
        _check(self._lib.coral_s1_placement_search(
            self._h, ncases, _ptr(ncfg, C.c_int32), _ptr(counts, C.c_int64), _ptr(lsteps, C.c_int32),
            _ptr(tput_off, C.c_int64), _ptr(tp, C.c_double), tput.size, _ptr(S, C.c_int32),
            _ptr(best, C.c_double), _ptr(sj, C.c_int64), _ptr(sc, C.c_int64)))
        return best, sj, sc

    def set_timing(self, on: bool) -> None:
        """Per-launch timing events of the lattice kernels (kernel_stats / _timeline /
        _launches); off by default (no event records in the evaluate)."""
        _check(self._lib.coral_s1_set_timing(self._h, 1 if on else 0))

    def set_census(self, on: bool) -> None:
        _check(self._lib.coral_s1_set_census(self._h, 1 if on else 0))

    def census(self) -> int:
        """Algorithmic bytes of the last evaluate's lat_layer_kernel launches (census on)."""
        v = C.c_int64()
        _check(self._lib.coral_s1_census(self._h, C.byref(v)))
        return v.value

    def census_all(self):
        """[layer alg bytes, layer (u, l) pairs, top (u, S) pairs, 0] of the last evaluate."""
        out = np.zeros(4, dtype=np.int64)
        _check(self._lib.coral_s1_census_all(self._h, _ptr(out, C.c_int64), 4))
        return out.tolist()

    def set_streams(self, n: int) -> None:
        _check(self._lib.coral_s1_set_streams(self._h, int(n)))

    def kernel_timeline(self, cap: int = 2048):
        """[(kind, stream slot, begin ms, end ms)] of the last evaluate's lattice launches."""
        kind = np.zeros(cap, np.int32)
        slot = np.zeros(cap, np.int32)
        b = np.zeros(cap)
        e = np.zeros(cap)
        n = C.c_int64()
        _check(self._lib.coral_s1_kernel_timeline(self._h, cap, _ptr(kind, C.c_int32), _ptr(slot, C.c_int32),
                                                  _ptr(b, C.c_double), _ptr(e, C.c_double), C.byref(n)))
        k = n.value
        return list(zip(kind[:k].tolist(), slot[:k].tolist(), b[:k].tolist(), e[:k].tolist()))

    def kernel_stats(self, kind: int):
        """(total ms, launches) of the last evaluate's lattice kernels: 0 top, 1 layer, 2 value."""
        t, n = C.c_double(), C.c_int64()
        _check(self._lib.coral_s1_kernel_stats(self._h, kind, C.byref(t), C.byref(n)))
        return t.value, n.value

    def window_select_stats(self):
        """(ms, algorithmic bytes) of the last enumerate's window_select_kernel."""
        t, b = C.c_double(), C.c_int64()
        _check(self._lib.coral_s1_window_select_stats(self._h, C.byref(t), C.byref(b)))
        return t.value, b.value

    def write_library(self, path: str, header: str, mp_order, model_json, phase_json, slo_json,
                      cfg_json) -> int:
        def strs(xs):
            arr = (C.c_char_p * max(len(xs), 1))()
            for i, x in enumerate(xs):
                arr[i] = x.encode()
            return arr
        order = np.ascontiguousarray(mp_order, dtype=np.int32)
        n = C.c_int64()
        _check(self._lib.coral_s1_write_library(
            self._h, path.encode(), header.encode(), len(order), _ptr(order, C.c_int32),
            strs(model_json), strs(phase_json), strs(slo_json), strs(cfg_json), C.byref(n)))
        return n.value

    def sweep(self, n_max, rho, prices, phase_mask: int):
        """-> (counts[k], best[k], unpriced[k], mp_counts[k, NM*NP])."""
        n_max = np.ascontiguousarray(n_max, dtype=np.int32)
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        prices = np.ascontiguousarray(prices, dtype=np.float64)
        k = max(len(n_max), 1)
        counts = np.zeros(k, dtype=np.int64)
        best = np.zeros(k)
        unpriced = np.zeros(k, dtype=np.int64)
        mpc = np.zeros(k * max(self.NM * self.NP, 1), dtype=np.int64)
        _check(self._lib.coral_s1_sweep(self._h, len(n_max), _ptr(n_max, C.c_int32), _ptr(rho, C.c_double),
                                        prices.shape[0], _ptr(prices, C.c_double), phase_mask,
                                        _ptr(counts, C.c_int64), _ptr(best, C.c_double),
                                        _ptr(unpriced, C.c_int64), _ptr(mpc, C.c_int64)))
        n = len(n_max)
        return (counts[:n], best[:n], unpriced[:n],
                mpc[:n * self.NM * self.NP].reshape(n, self.NM * self.NP))

    def allocation_model(self, prices, avail, demand, mp_order, prune_ratio, run_mp, run_region, run_key):
        """-> (vars ALLOC_VAR_DTYPE[n], pruned, best_eff[NM*NP]) of build_allocation_model."""
        pm = np.ascontiguousarray(prices, dtype=np.float64)
        av = np.ascontiguousarray(avail, dtype=np.int64)
        dm = np.ascontiguousarray(demand, dtype=np.float64)
        order = np.ascontiguousarray(mp_order, dtype=np.int32)
        rm = np.ascontiguousarray(run_mp if len(run_mp) else [0], dtype=np.int32)
        rr = np.ascontiguousarray(run_region if len(run_region) else [0], dtype=np.int32)
        rk = np.ascontiguousarray(run_key if len(run_key) else [0], dtype=np.uint64)
        best = np.zeros(max(self.NM * self.NP, 1))
        nv, npr = C.c_int64(), C.c_int64()
        _check(self._lib.coral_s1_allocation_model(
            self._h, pm.shape[0], _ptr(pm, C.c_double), _ptr(av, C.c_int64), _ptr(dm, C.c_double), len(order),
            _ptr(order, C.c_int32), float(prune_ratio), len(run_mp), _ptr(rm, C.c_int32), _ptr(rr, C.c_int32),
            _ptr(rk, C.c_uint64), C.byref(nv), C.byref(npr), _ptr(best, C.c_double)))
        out = np.zeros(max(nv.value, 1), dtype=ALLOC_VAR_DTYPE)
        _check(self._lib.coral_s1_get_allocation_vars(self._h, out.ctypes.data_as(C.c_void_p), out.size))
        return out[:nv.value], npr.value, best[:self.NM * self.NP]

    def feasible_counts(self):
        """Feasible templates per (model, phase) slot; raises LibraryGenErrorNative when an
        evaluated slot has none (templates.py:499-502)."""
        out = np.zeros(max(self.NM * self.NP, 1), dtype=np.int64)
        rc = self._lib.coral_s1_feasible_counts(self._h, _ptr(out, C.c_int64), out.size)
        if rc not in (OK, ENOTEMPLATE):
            _check(rc)
        return out[:self.NM * self.NP], rc == ENOTEMPLATE

    def node_queries(self, cfg, model, phase, j, budget, use_profile: bool):
        a = [np.ascontiguousarray(x, dtype=np.int32) for x in (cfg, model, phase, j)]
        bud = np.ascontiguousarray(budget, dtype=np.float64)
        n = len(bud)
        tput = np.zeros(max(n, 1))
        batch = np.zeros(max(n, 1), dtype=np.int64)
        _check(self._lib.coral_s1_node_queries(self._h, n, *[_ptr(x, C.c_int32) for x in a],
                                               _ptr(bud, C.c_double), int(use_profile),
                                               _ptr(tput, C.c_double), _ptr(batch, C.c_int64)))
        return tput[:n], batch[:n]

    def stage_ms(self) -> dict:
        vals = [C.c_double() for _ in range(4)]
        _check(self._lib.coral_s1_stage_ms(self._h, *[C.byref(v) for v in vals]))
        return dict(zip(("tables", "enumerate", "evaluate", "frontier"), [v.value for v in vals]))


# Free handles per device. A handle carries one problem's device state (spec blob,
# tables, keys, records, frontier), so every live Stage1Problem leases its OWN handle
# and gives it back when it is closed or collected; stateless users (placement_search,
# T-hat queries) lease one for the duration of the call. Released handles keep their
# device buffers (lattice workspaces, CUB scratch) warm for the next lease.
_pool: dict = {}
_POOL_KEEP = 2


def _cuda_device(device):
    import torch
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the stage-1 generator runs only on the GPU")
    return torch.cuda.current_device() if device is None else int(device)


def acquire(device: int | None = None) -> Handle:
    """Lease a handle on `device` (default: torch's current device), bound to torch's
    current stream. The caller owns it exclusively until release()."""
    import torch
    device = _cuda_device(device)
    free = _pool.setdefault(device, [])
    h = free.pop() if free else Handle(device)
    h.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return h


def release(h: Handle) -> None:
    """Return a leased handle; beyond _POOL_KEEP free handles per device it is destroyed."""
    if h is None or not h._h:
        return
    free = _pool.setdefault(h.device, [])
    if any(x is h for x in free):
        return
    if len(free) < _POOL_KEEP:
        h.set_timing(False)  # per-lease diagnostics settings do not carry over
        h.set_census(False)
        h.set_streams(0)
        free.append(h)
    else:
        h.close()


class lease:
    """Context manager over acquire/release for call-scoped (stateless) users."""

    def __init__(self, device: int | None = None):
        self.device = device
        self.h = None

    def __enter__(self) -> Handle:
        self.h = acquire(self.device)
        return self.h

    def __exit__(self, *exc):
        release(self.h)
        self.h = None
