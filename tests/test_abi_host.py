"""CPU-only checks of the C-ABI library and the host-side logic around it (no device
calls): every entry point include/coral_s1.h declares is exported by the built
library, the host-only repr(float) formatter the native writer uses, the packed
combo-key order, and the native materialiser against its pure-Python twin."""

import ctypes
import json
import os
import random
import re
import struct

import numpy as np

from paper_2605_04357_b200 import _native, catalog
from paper_2605_04357_b200.frontier import FrontierEntry, _materialise_native, materialise_py
from paper_2605_04357_b200.library import Stage1Problem, str_ranks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "coral_s1.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(coral_s1_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native._LIB_PATH)  # loading needs the CUDA runtime, not a GPU
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes binding declares a prototype for every one of them
    bound = set(re.findall(r'"(coral_s1_\w+)"', open(_native.__file__).read()))
    assert set(syms) <= bound, sorted(set(syms) - bound)


def test_version_and_error_text_without_device():
    lib = _native.load()
    assert lib.coral_s1_version() > 0
    assert lib.coral_s1_last_error() is not None
    # creating a handle without a device fails loudly (no CPU fallback)
    h = ctypes.c_void_p()
    if lib.coral_s1_create(0, ctypes.byref(h)) != 0:
        assert lib.coral_s1_last_error()


def test_format_double_is_json_dumps_of_float():
    """json.dumps(float) as TemplateLibrary.save writes it: repr for finite values."""
    rng = random.Random(5)
    vals = [0.0, -0.0, 1.0, 0.1, 1e16, 1e17, 1.5e-4, 1e-5, 123456789.123, 2.0 ** 60, 5e-324,
            1.7976931348623157e308, float("inf"), float("-inf")]
    vals += [rng.uniform(0, 1e6) for _ in range(2000)]
    vals += [struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0] for _ in range(3000)]
    for v in vals:
        if v != v:
            continue
        assert _native.format_double(v) == json.dumps(v), v


def _pack(tokens):
    """(rank, count) tokens, ascending rank -> the device's u64 combo key."""
    key = 0
    for i, (r, c) in enumerate(tokens):
        key |= ((r + 1) << 3 | c) << (9 * (_native.MAX_NODES - 1 - i))
    return key


def test_packed_key_order_equals_str_order():
    """str(NodeComboKey) order == u64 key order (templates.py:112, 340)."""
    names = ["1xA100", "1xA10", "2xA100", "10xL4", "1xL4", "8xH100", "1xH1", "4xB200", "1xB2"]
    rank = str_ranks(names)
    rng = random.Random(11)
    combos = set()
    while len(combos) < 3000:
        k = rng.randint(1, 4)
        picks = sorted(rng.sample(range(len(names)), k), key=lambda i: names[i])
        cnts = [rng.randint(1, 6 - (k - 1)) for _ in picks]
        if sum(cnts) <= _native.MAX_NODES:
            combos.add(tuple(zip(picks, cnts)))
    as_str = {c: "+".join(f"{names[i]}*{n}" for i, n in c) for c in combos}
    as_key = {c: _pack(sorted(((int(rank[i]), n) for i, n in c))) for c in combos}
    assert sorted(combos, key=as_str.get) == sorted(combos, key=as_key.get)


def _fake_problem(w):
    """A Stage1Problem without a device handle (host fields only)."""
    prob = object.__new__(Stage1Problem)
    prob.configs = sorted(w.configs, key=lambda c: c.name)
    prob.models = list(w.models)
    prob.slos = w.slos
    prob.phases = ("prefill", "decode")
    rank = str_ranks([c.name for c in prob.configs])
    prob.cfg_by_rank = [None] * len(prob.configs)
    for i, r in enumerate(rank):
        prob.cfg_by_rank[r] = prob.configs[i]
    prob.cand_off = np.array([0, 10])
    return prob


def test_native_materialise_matches_python_twin():
    w = catalog.extended_workload()
    prob = _fake_problem(w)
    rng = np.random.default_rng(3)
    n = 1500
    items = np.zeros(n, dtype=_native.FRONTIER_DTYPE)
    items["mp"] = rng.integers(0, 2 * len(prob.models), n)
    items["region"] = rng.integers(0, 3, n)
    K = len(prob.configs)
    keys = []
    for _ in range(n):
        k = int(rng.integers(1, 4))
        picks = sorted(rng.choice(K, k, replace=False).tolist())
        keys.append(_pack([(r, 2 if j == 0 and k < 3 else 1) for j, r in enumerate(picks)]))
    # repeat some (mp, combo) pairs across regions, as real frontiers do
    keys[n // 2:] = keys[: n - n // 2]
    items["combo_key"] = np.array(keys, dtype=np.uint64)
    items["mp"][n // 2:] = items["mp"][: n - n // 2]
    nn = np.array([sum(((k >> (9 * t)) & 7) for t in range(_native.MAX_NODES)) for k in keys])
    items["rec"]["num_nodes"] = nn
    items["rec"]["num_stages"] = np.minimum(nn, 2)
    items["rec"]["layers_per_stage"][:, 0] = 30
    items["rec"]["layers_per_stage"][:, 1] = np.where(nn >= 2, 34, 0)
    items["rec"]["stage_of_node"][:, 1] = 1
    items["rec"]["throughput_tps"] = rng.uniform(1, 1e4, n)
    items["price_usd_h"] = rng.uniform(0.5, 80, n)
    regions = ["us-east", "eu-west", "ap-south"]
    native = _materialise_native(__import__("paper_2605_04357_b200._lib._materialize",
                                            fromlist=["x"]), prob, items, regions)
    py = materialise_py(prob, items, regions, {}).segments
    assert list(native) == list(py)
    for seg in py:
        a, b = native[seg], py[seg]
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert type(x) is FrontierEntry and x.price_usd_h == y.price_usd_h
            tx, ty = x.template, y.template
            assert (tx.model, tx.phase, tx.slo, str(tx.combo), tx.combo.items, tx.placement,
                    tx.throughput_tps, tx.template_id) == \
                   (ty.model, ty.phase, ty.slo, str(ty.combo), ty.combo.items, ty.placement,
                    ty.throughput_tps, ty.template_id)
    # shared template objects: one per (model, phase, combo) across regions
    ids = {}
    for seg, lst in native.items():
        for e in lst:
            assert ids.setdefault(e.template.template_id, id(e.template)) == id(e.template)
