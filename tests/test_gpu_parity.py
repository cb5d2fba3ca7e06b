"""CUDA path (libcoral_s1.so through the C ABI) vs the reference's golden vectors
and the CPU oracle. Bit-exact for ids, enumeration, placements and fp64 values."""

import numpy as np
import pytest

from paper_2605_04357_b200 import (DomainError, LibraryGenError, build_frontier, build_library,
                                   enumerate_combos, placement_search_batch, throughput_table)
from paper_2605_04357_b200.library import GenContext, LibraryCaps, Stage1Problem
from tests.helpers import (cfg_by_rank, digest, golden, key_str, oracle_library_lines,
                           oracle_problem, record_line, template_line, workload)

pytestmark = pytest.mark.gpu


def test_native_library_is_loaded():
    import paper_2605_04357_b200._native as N
    with N.lease() as h:
        assert h.launches >= 0
    assert N._lib is not None


def test_placement_search_golden_bit_exact():
    cases = golden("kernels.json.gz")
    got = placement_search_batch([(c["counts"], np.array(c["tput"]), c["S"]) for c in cases])
    for c, (best, sj, sc) in zip(cases, got):
        assert best == c["best"], c
        assert sj.tolist() == c["stage_j"], c
        assert sc.tolist() == c["stage_counts"], c


def test_placement_search_rejects_negative():
    with pytest.raises(ValueError):
        placement_search_batch([(np.array([1]), np.array([[-1.0, 0.0]]), 1)])


@pytest.mark.parametrize("w", ["c1", "core", "extended"])
def test_tables_golden_bit_exact(w):
    g = golden(f"tables_{w}.json.gz")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    prob = Stage1Problem(configs, models, slos, caps, ctx)
    prob.h.tables()
    tab, offs, ls = prob.h.get_tables()
    budgets = prob.h.get_budgets()
    K = len(configs)
    for mi, m in enumerate(models):
        for pi, ph in enumerate(("prefill", "decode")):
            mp = mi * 2 + pi
            block = tab[offs[mp]:offs[mp + 1]].reshape(6, K, ls[mi])
            for S in range(1, min(6, m.num_layers) + 1):
                ref = g["tables"][f"{m.name}|{ph}|{S}"]
                assert budgets[mp, S - 1] == ref["budget"]
                np.testing.assert_array_equal(block[S - 1], np.array(ref["rows"]))


def test_throughput_table_operator():
    g = golden("tables_core.json.gz")
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    configs = sorted(configs, key=lambda c: c.name)
    m = models[0]
    tab = throughput_table(configs, m, slos[m.name], "decode", 3, ctx)
    np.testing.assert_array_equal(tab, np.array(g["tables"][f"{m.name}|decode|3"]["rows"]))


@pytest.mark.parametrize("w", ["c1", "core"])
def test_enumerate_combos_golden(w):
    g = golden(f"enum_{w}.json.gz")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    for m in models:
        assert [str(c) for c in enumerate_combos(configs, m, caps)] == g[m.name]["combos"]


def test_enumeration_extended_digest():
    g = golden("enum_extended.json.gz")
    configs, models, slos, caps, ctx, regions, prices = workload("extended")
    prob = Stage1Problem(configs, models, slos, caps, ctx)
    prob.h.enumerate()
    cbr = prob.cfg_by_rank
    for mi, m in enumerate(models):
        strs = [key_str(k, cbr) for k in prob.h.get_combos(mi, True)]
        assert len(strs) == g[m.name]["count"]
        assert digest(strs) == g[m.name]["sha256"]


@pytest.mark.parametrize("w", ["c1", "core"])
def test_build_library_golden_bit_exact(w):
    g = golden(f"library_{w}.json.gz")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    lib = build_library(configs, models, slos, caps, ctx)
    lines = [template_line(t) for t in lib.entries]
    assert len(lines) == g["count"]
    assert lines == g["records"]
    assert {f"{k[0]}|{k[1]}": v for k, v in lib.counts_by_model_phase().items()} == g["counts"]


@pytest.mark.parametrize("w", ["extended", "c3"])
def test_build_library_big_golden(w):
    """Full BASELINE config 2 (1,084,362 templates) and config 3 (llama3-70b at
    granularity 1, Lu = 80: 344,548 templates): every record bit-identical
    (sha256 over canonical lines incl. repr(throughput))."""
    try:
        g = golden(f"library_{w}.json.gz")
    except FileNotFoundError:
        pytest.skip(f"{w} golden not generated")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    cbr = prob.cfg_by_rank
    NP = 2
    lines = []
    order = sorted(range(len(models) * NP), key=lambda mp: (models[mp // NP].name, ("prefill", "decode")[mp % NP]))
    for mp in order:
        m = models[mp // NP]
        ph = ("prefill", "decode")[mp % NP]
        keys = prob.keys(mp // NP)
        recs = prob.records(mp)
        for k, r in zip(keys, recs):
            if r["num_stages"] > 0:
                lines.append(record_line(m.name, ph, k, r, cbr))
    assert len(lines) == g["count"]
    assert lines[::g["sample_every"]] == g["sample"]
    assert digest(lines) == g["sha256"]


def test_profile_override_library():
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, ProfileTable, SloSpec
    g = golden("profile.json.gz")
    configs = [NodeConfig(catalog.GPU_CATALOG["L40S"], 1, 64.0),
               NodeConfig(catalog.GPU_CATALOG["L40S"], 2, 64.0),
               NodeConfig(catalog.GPU_CATALOG["L4"], 1, 64.0),
               NodeConfig(catalog.GPU_CATALOG["L4"], 4, 64.0)]
    model = ModelSpec("m7b", num_layers=32, params_total_b=7, params_active_b=7, hidden_size=4096)
    prof = ProfileTable()
    for cfg, mdl, ph, j, b, v in g["profile"]:
        prof.add(cfg, mdl, ph, j, b, v)
    lib = build_library(configs, [model], {"m7b": SloSpec(1500, 80)}, LibraryCaps(3, 10.0),
                        GenContext(profile=prof))
    assert [template_line(t) for t in lib.entries] == g["library"]["records"]


@pytest.mark.parametrize("w", ["c1", "core", "extended", "c3"])
def test_frontier_golden(w):
    try:
        g = golden(f"frontier_{w}.json.gz")
    except FileNotFoundError:
        pytest.skip("golden not generated")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    front = build_frontier(configs, models, slos, caps, prices, regions=regions, ctx=ctx)
    got = []
    for (m, ph, r), entries in front.segments.items():
        for e in entries:
            got.append([m, ph, r, str(e.template.combo), e.price_usd_h, e.throughput_tps])
    key = lambda t: (t[0], t[1], t[2])  # noqa: E731
    assert sorted(got, key=key) == sorted(g, key=key)
    # the sweep's best tokens/s per USD-h (cli.py:253-260) is always on the frontier
    for (m, ph, r), entries in front.segments.items():
        assert entries == sorted(entries, key=lambda e: e.price_usd_h)


def _random_inputs(seed):
    from paper_2605_04357_b200.specs import GpuSpec, ModelSpec, NodeConfig, PerfParams, SloSpec
    rng = np.random.default_rng(seed)
    gpus = [GpuSpec(f"G{i}", float(rng.choice([16, 24, 40, 48, 80, 141])),
                    float(rng.uniform(0.2, 4.0)), float(rng.uniform(50, 1000)),
                    float(rng.uniform(0.5, 8))) for i in range(int(rng.integers(2, 5)))]
    configs = [NodeConfig(g, int(n)) for g in gpus for n in rng.choice([1, 2, 4, 8], size=2, replace=False)]
    models, slos = [], {}
    for k in range(3):
        L = int(rng.choice([8, 12, 24, 32, 40, 61, 80]))
        tot = float(rng.uniform(1, 120))
        models.append(ModelSpec(f"m{k}", L, tot, tot * float(rng.uniform(0.1, 1.0)),
                                int(rng.choice([1024, 4096, 8192])),
                                kv_bytes_per_token_per_layer=float(rng.choice([512, 2048, 4096]))))
        slos[f"m{k}"] = SloSpec(float(rng.uniform(300, 3000)), float(rng.uniform(10, 150)))
    perf = PerfParams(mfu=float(rng.uniform(0.3, 0.8)), mbu=float(rng.uniform(0.5, 0.95)),
                      avg_prompt_tokens=float(rng.uniform(100, 3000)),
                      avg_ctx_tokens=float(rng.uniform(100, 3000)), slo_budget_frac=0.6)
    caps = LibraryCaps(int(rng.integers(3, 7)), float(rng.uniform(4, 30)))
    return configs, models, slos, caps, GenContext(perf=perf, granularity=int(rng.choice([0, 1, 2])))


@pytest.mark.parametrize("seed", range(6))
def test_random_scenarios_match_oracle(seed):
    configs, models, slos, caps, ctx = _random_inputs(seed)
    if any(m.num_layers % ctx.layer_granularity(m) for m in models):
        ctx = GenContext(perf=ctx.perf)
    op = oracle_problem((configs, models, slos, caps, ctx))
    ref = oracle_library_lines(op)
    try:
        lib = build_library(configs, models, slos, caps, ctx)
    except LibraryGenError:
        # the reference raises when some (model, phase) has no template
        present = {tuple(ln.split("|")[:2]) for ln in ref}
        assert len(present) < len(models) * 2
        return
    assert [template_line(t) for t in lib.entries] == ref


@pytest.mark.parametrize("name,W", [("core", 3), ("core", 8), ("c1", 8)])
def test_sharded_evaluation_and_merge_equal_single_gpu(name, W):
    """(model, phase, S) unit shards + per-shard frontier + merge == full frontier
    (the multi-GPU protocol, emulated on one device). W=8 on c1 (2 chains of <= 6 S
    units) leaves some ranks with no units: their empty parts must merge cleanly."""
    from paper_2605_04357_b200 import _native
    configs, models, slos, caps, ctx, regions, prices = workload(name)
    from tests.helpers import price_matrix
    pm = price_matrix(configs, prices, regions)
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    n_full = prob.h.frontier(pm)
    full = prob.h.get_frontier(n_full)
    import torch
    from paper_2605_04357_b200.shard import assign_units
    parts = []
    _, lsteps, smax = prob.h.table_layout()
    from paper_2605_04357_b200.shard import table_posfrac
    masks = assign_units(prob.counts, lsteps, smax, 2, W, table_posfrac(prob.h))
    for r in range(W):
        prob.h.evaluate_units(masks[r])
        n = prob.h.frontier(pm)
        parts.append(prob.h.get_frontier(n))
    union = np.concatenate(parts)
    dev = torch.from_numpy(union.view(np.uint8).copy()).cuda()
    n = prob.h.frontier_merge_device(dev.data_ptr(), len(union))
    merged = prob.h.get_frontier(n)
    assert merged.tobytes() == full.tobytes()
    # the multi-GPU path's layout: one strided buffer [header | cap items] per part
    item = _native.FRONTIER_DTYPE.itemsize
    cap = max(len(p) for p in parts) + 3
    stride = item + cap * item
    buf = np.zeros(W * stride, dtype=np.uint8)
    for r, part in enumerate(parts):
        buf[r * stride + item: r * stride + item + len(part) * item] = part.view(np.uint8)
    dbuf = torch.from_numpy(buf).cuda()
    n = prob.h.frontier_merge_parts(dbuf.data_ptr(), stride, item, [len(p) for p in parts])
    assert prob.h.get_frontier(n).tobytes() == full.tobytes()
    # what the ranks actually exchange: prefiltered candidates, no local skyline
    cands = []
    for r in range(W):
        prob.h.evaluate_units(masks[r])
        n = prob.h.frontier_candidates(pm)
        cands.append(prob.h.get_frontier(n))
    assert sum(len(c) for c in cands) >= sum(len(p) for p in parts)
    cap = max(len(c) for c in cands) + 1
    stride = item + cap * item
    buf = np.zeros(W * stride, dtype=np.uint8)
    for r, part in enumerate(cands):
        buf[r * stride + item: r * stride + item + len(part) * item] = part.view(np.uint8)
    dbuf = torch.from_numpy(buf).cuda()
    n = prob.h.frontier_merge_parts(dbuf.data_ptr(), stride, item, [len(c) for c in cands])
    assert prob.h.get_frontier(n).tobytes() == full.tobytes()
    assert _native.FRONTIER_DTYPE.itemsize == 64


def test_errors():
    from paper_2605_04357_b200.specs import ModelSpec, SloSpec
    configs, models, slos, caps, ctx, regions, prices = workload("c1")
    with pytest.raises(DomainError):
        LibraryCaps(0, 2.0)
    with pytest.raises(DomainError):
        build_library(configs, models, slos, LibraryCaps(8, 12.0), ctx)
    huge = ModelSpec("huge", 32, 5000.0, 5000.0, 4096)
    with pytest.raises(LibraryGenError):
        build_library(configs, [huge], {"huge": SloSpec(1500, 80)}, caps, ctx)
    assert len(build_library(configs, [], {}, caps, ctx)) == 0


def test_lattice_path_equals_per_candidate_path():
    """The lattice evaluator (full range) and the per-candidate fallback kernel
    (sub-ranges) produce byte-identical records."""
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    full = [prob.records(mp).tobytes() for mp in range(len(models) * 2)]
    n = prob.num_candidates
    prob.h.evaluate(0, n - 1)  # sub-range -> per-candidate kernel
    part = [prob.records(mp) for mp in range(len(models) * 2)]
    for mp in range(len(models) * 2):
        recs = part[mp]
        if mp == len(models) * 2 - 1:
            recs = recs[:-1]
            assert recs.tobytes() == full[mp][:len(recs.tobytes())]
        else:
            assert recs.tobytes() == full[mp]


@pytest.mark.parametrize("w", ["c1", "core", "extended", "c3"])
def test_lazy_library_native_save_byte_identical(w, tmp_path):
    """the array-backed library streams a JSONL file
    byte-identical to the reference's TemplateLibrary.save (285.7 MB for config 2)."""
    import hashlib
    import time
    ref = golden("saved_libraries.json.gz")[w]
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    lib = build_library(configs, models, slos, caps, ctx, lazy=True)
    path = str(tmp_path / "lib.jsonl")
    t0 = time.perf_counter()
    n = lib.save(path)
    dt = time.perf_counter() - t0
    data = open(path, "rb").read()
    assert n == len(lib)
    assert len(data) == ref["bytes"]
    assert hashlib.sha256(data).hexdigest() == ref["sha256"]
    print(f"{w}: {n} templates, {len(data)} bytes saved in {dt:.3f}s")
    if w in ("c1", "core"):
        eager = build_library(configs, models, slos, caps, ctx)
        assert [template_line(t) for t in lib.entries] == [template_line(t) for t in eager.entries]
        assert lib.counts_by_model_phase() == eager.counts_by_model_phase()
        for t in eager.entries[::37]:
            assert template_line(lib.get(t.template_id)) == template_line(t)
        mp = lib.model_phases()[0]
        assert [template_line(t) for t in lib.templates_for(*mp)] == \
               [template_line(t) for t in eager.templates_for(*mp)]


def test_sweep_matches_reference_cmd_sweep():
    """cmd_sweep (cli.py:233-272) from one solve: template counts and best tokens/s per
    USD-h equal the reference's per-caps rebuilds (core scenario and the c09 model)."""
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.frontier import sweep
    from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, SloSpec
    g = golden("sweep.json.gz")
    caps_list = [LibraryCaps(n, r) for n, r, _, _ in g["core"]]
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    rows = sweep(configs, models, slos, caps_list, prices, regions=regions, ctx=ctx)
    assert [(n, r, c, b) for n, r, c, _, b in rows] == [tuple(x) for x in g["core"]]
    model = ModelSpec("m120b", num_layers=36, params_total_b=116.8, params_active_b=5.1,
                      hidden_size=2880, kv_bytes_per_token_per_layer=2048, is_moe=True,
                      is_hybrid_attn=True)
    cfgs = [NodeConfig(catalog.GPU_CATALOG["H100"], 2, 64.0), NodeConfig(catalog.GPU_CATALOG["L40S"], 1, 64.0)]
    p = {("r", c.name): c.gpu.rel_cost * c.gpu_count for c in cfgs}
    rows = sweep(cfgs, [model], {"m120b": SloSpec(1000, 40)}, [LibraryCaps(n, r) for n, r, _, _ in g["c09"]],
                 p, regions=["r"], ctx=GenContext(), phases=("prefill",))
    assert [(n, r, c, b) for n, r, c, _, b in rows] == [tuple(x) for x in g["c09"]]
    effs = [b for *_, b in rows]
    assert effs == sorted(effs)  # c09: best goodput/USD non-decreasing in the caps


def test_native_materialise_equals_python():
    """The CPython extension builds the same frontier objects as the Python twin."""
    from paper_2605_04357_b200.frontier import _price_matrix, materialise, materialise_py
    configs, models, slos, caps, ctx, regions, prices = workload("extended")
    front, prob = build_frontier(configs, models, slos, caps, prices, regions=regions, ctx=ctx,
                                 return_problem=True)
    names, pm = _price_matrix(prob.configs, prices, regions)
    items = prob.h.get_frontier(prob.h.frontier(pm))
    a = materialise(prob, items, names, {})
    b = materialise_py(prob, items, names, {})

    def rows(f):
        return [(k, e.template.template_id, e.template.placement, e.template.throughput_tps,
                 e.template.slo, e.template.combo, e.price_usd_h) for k, v in f.segments.items() for e in v]
    assert rows(a) == rows(b)
    assert len(a) == 2225


def test_roofline_operators_match_reference_grid():
    """node_max_throughput on the device == the reference's perf.py values on the
    golden grid (nodes x models x phases x j x budgets, two PerfParams), one batch."""
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.roofline import node_queries, planned_batch_and_tput
    from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, PerfParams
    params = [PerfParams(), PerfParams(mfu=0.3, mbu=0.9, fixed_overhead_ms=0.0,
                                       avg_prompt_tokens=333.3, avg_ctx_tokens=777.7)]
    models = dict(catalog.MODEL_CATALOG)
    models["tiny"] = ModelSpec("tiny", 4, 0.5, 0.5, 256, kv_bytes_per_token_per_layer=128.0)
    grid = golden("perf_grid.json.gz")
    for pi, p in enumerate(params):
        rows = [e for e in grid if e["p"] == pi]
        qs = [(NodeConfig(catalog.GPU_CATALOG[e["gpu"]], e["gc"]), models[e["model"]], e["phase"], e["j"],
               e["budget"]) for e in rows]
        got, _ = node_queries(qs, p)
        assert got == [e["tput"] for e in rows]
    b, t = planned_batch_and_tput(NodeConfig(catalog.GPU_CATALOG["H100"], 2), models["llama3-70b"],
                                  "decode", 40, 0.05, params[0])
    assert b > 0 and t > 0


def test_recompute_throughput_invariant():
    """templates.py:267-280 recomputed from the placement equals the template value
    (test_templates.py:151-155 invariant, exact here)."""
    from paper_2605_04357_b200.roofline import recompute_throughput
    configs, models, slos, caps, ctx, regions, prices = workload("c1")
    lib = build_library(configs, models, slos, caps, ctx)
    m = models[0]
    for t in lib.entries[::5]:
        assert recompute_throughput(t, m, ctx) == t.throughput_tps


def test_native_load_round_trip_extended(tmp_path):
    """TemplateLibrary.load of the full config-2 file (285.7 MB): the same objects as
    the reference-style Python loop on a sample, and a byte-identical re-save."""
    import hashlib
    import time
    from paper_2605_04357_b200 import TemplateLibrary
    ref = golden("saved_libraries.json.gz")["extended"]
    configs, models, slos, caps, ctx, regions, prices = workload("extended")
    path = str(tmp_path / "lib.jsonl")
    build_library(configs, models, slos, caps, ctx, lazy=True).save(path)
    t0 = time.perf_counter()
    lib = TemplateLibrary.load(path)
    dt = time.perf_counter() - t0
    assert len(lib) == 1084362
    lines = [template_line(t) for t in lib.entries]
    assert lines[::97] == golden("library_extended.json.gz")["sample"]
    out = str(tmp_path / "again.jsonl")
    lib.save(out)
    assert hashlib.sha256(open(out, "rb").read()).hexdigest() == ref["sha256"]
    print(f"native load of {len(lib)} templates: {dt:.2f}s")


def test_eager_library_build_time_extended():
    """build_library (eager objects) for config 2: 1,084,362 templates, sampled lines
    identical to the reference; reports the end-to-end time."""
    import time
    configs, models, slos, caps, ctx, regions, prices = workload("extended")
    t0 = time.perf_counter()
    lib = build_library(configs, models, slos, caps, ctx)
    dt = time.perf_counter() - t0
    assert len(lib) == 1084362
    g = golden("library_extended.json.gz")
    assert [template_line(t) for t in lib.entries[::97]] == g["sample"]
    print(f"eager build_library(c2): {dt:.2f}s")


def test_table_posfrac_counts_positive_entries():
    """The tables kernel's positive-entry counts (shard cost model input) equal a host
    count over the same T-hat tables."""
    from paper_2605_04357_b200 import catalog
    w = catalog.extended_workload()
    prob = Stage1Problem(w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho), GenContext(perf=w.perf))
    prob.h.tables()
    tabs, offs, lsteps = prob.h.get_tables()
    pf = prob.h.table_posfrac()
    K = len(w.configs)
    for mp in range(len(offs) - 1):
        blk = tabs[offs[mp]:offs[mp + 1]].reshape(-1, K * int(lsteps[mp // 2]))
        for S in range(1, blk.shape[0] + 1):
            assert pf[mp, S - 1] == np.count_nonzero(blk[S - 1] > 0) / blk.shape[1]


def test_rows_monotone_only_within_tolerance_take_the_literal_search():
    """T-hat rows that rise by < 1e-12 pass the reference's monotone test
    (kernels.py:291) but are not exactly monotone: the lattice must then run the
    literal [1, jmax] search without the cap bracket or the u <-> X-u symmetry, and
    match the unmodified reference (golden tolmono.json.gz) and the oracle exactly."""
    from tests.test_oracle_golden import tolmono_inputs
    g, inputs = tolmono_inputs()
    configs, models, slos, caps, ctx = inputs
    prob = Stage1Problem(configs, models, slos, caps, ctx)
    prob.h.tables()
    tabs, offs, lsteps = prob.h.get_tables()
    rows = tabs[offs[0]:offs[1]].reshape(-1, int(lsteps[0]))
    d = np.diff(rows, axis=1)
    assert (d <= 1e-12).all() and (d > 0).any()  # tolerance-monotone, not exactly
    lib = build_library(configs, models, slos, caps, ctx)
    lines = [template_line(t) for t in lib.entries]
    assert lines == g["library"]["records"]
    assert lines == oracle_library_lines(oracle_problem(inputs))


@pytest.mark.parametrize("streams", [0, 2])
def test_lattice_workspace_beyond_device_memory(streams, monkeypatch):
    """When the lattice tables of all four chain streams do not fit in device memory,
    fewer streams run them; when none fits, every unit takes the exact per-candidate
    kernel. Both give the reference's library (golden core, 30,739 templates).
    CORAL_S1_MEM_LIMIT caps the memory a fresh handle sees."""
    from math import comb
    from paper_2605_04357_b200 import _native
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    probe = Stage1Problem(configs, models, slos, caps, ctx)
    _, lsteps, _ = probe.h.table_layout()
    probe.h.enumerate()
    counts = probe.h.num_combos()
    probe.close()
    K, n_max = len(configs), caps.n_max
    ns = sum(comb(K + s - 1, s) for s in range(1, n_max))
    pitch = (int(max(lsteps)) + 2) & ~1  # lat_pitch
    per_stream = ns * pitch * (8 * 3 * (n_max - 1) + 2 * ((n_max - 2) * (n_max - 1) // 2)) + 2 * ((n_max - 1) * ns * 32 + 32)
    # lattice_prepare first sets aside the evaluate's own buffers: records, per-stream
    # rank tables + winners, and the bounded frontier item buffer
    reserve = (64 << 20) + 2 * int(counts.sum()) * 32 + 4 * int(counts.max()) * (256 + 16)
    limit = 1 if streams == 0 else int((per_stream * streams + reserve) / 0.9) + (1 << 20)
    monkeypatch.setenv("CORAL_S1_MEM_LIMIT", str(limit))
    fresh = _native.Handle(0)
    fresh.set_timing(True)  # per-launch events: which stream each layer launch ran on
    monkeypatch.setitem(_native._pool, 0, [fresh])
    lib = build_library(configs, models, slos, caps, ctx)
    assert [template_line(t) for t in lib.entries] == golden("library_core.json.gz")["records"]
    layers = [slot for kind, slot, _, _ in fresh.kernel_timeline() if kind == 1]
    if streams == 0:
        assert not layers  # no lattice: per-candidate kernel only
    else:
        assert layers and set(layers) <= set(range(streams))


@pytest.mark.parametrize("w", ["core", "extended"])
def test_non_monotone_profile_rows_stay_on_the_lattice(w):
    """ProfileTable overrides that break kernels.py:291's monotone test for two configs
    (tests/helpers.zigzag_profile): the candidates containing them take the reference's
    full-scan DP (kernels.py:240-249), the others the binary-search crossing, both on the
    lattice (scan variant + search variant; no per-candidate kernel). The whole library
    is identical to the unmodified reference's (golden profile_<w>.json.gz)."""
    import time
    from paper_2605_04357_b200.specs import ProfileTable
    from tests.helpers import zigzag_profile
    try:
        g = golden(f"profile_{w}.json.gz")
    except FileNotFoundError:
        pytest.skip(f"profile_{w} golden not generated")
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    ctxp = GenContext(perf=ctx.perf, profile=zigzag_profile(configs, models, ProfileTable))
    prob = Stage1Problem(configs, models, slos, caps, ctxp)
    prob.run()
    prob.h.set_timing(True)  # per-launch events: which kernels ran
    t0 = time.perf_counter()
    prob.run()
    import torch
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    kinds = {k for k, _, _, _ in prob.h.kernel_timeline()}
    assert 0 in kinds and 1 in kinds  # top cells and layers ran on the lattice
    cbr = prob.cfg_by_rank
    lines = []
    order = sorted(range(len(models) * 2), key=lambda mp: (models[mp // 2].name, ("prefill", "decode")[mp % 2]))
    for mp in order:
        keys, recs = prob.keys(mp // 2), prob.records(mp)
        for k, r in zip(keys, recs):
            if r["num_stages"] > 0:
                lines.append(record_line(models[mp // 2].name, ("prefill", "decode")[mp % 2], k, r, cbr))
    assert len(lines) == g["count"]
    assert lines[::g["sample_every"]] == g["sample"]
    assert digest(lines) == g["sha256"]
    print(f"{w} with non-monotone profile rows: {len(lines)} templates, solve {1e3 * dt:.2f} ms")


@pytest.mark.parametrize("name,W", [("c3", 2), ("c3", 8), ("core", 3), ("extended", 8)])
def test_pieces_split_by_candidate_range_merge_equal_single_gpu(name, W):
    """The multi-GPU pieces (shard.plan_pieces on costs measured by shard.calibrate):
    (model, phase, S) units whose top cells are split by candidate range over ranks --
    the north star's (model, GPU-type combination) axis -- evaluated rank by rank on one
    device, prefiltered, merged with the single all-gather layout: byte-identical to the
    single-GPU frontier. Also a hand-made plan that cuts every chain into 3 ranges."""
    from paper_2605_04357_b200 import _native
    from paper_2605_04357_b200.shard import calibrate, pieces_to_ranges, plan_pieces
    from tests.helpers import price_matrix
    configs, models, slos, caps, ctx, regions, prices = workload(name)
    pm = price_matrix(configs, prices, regions)
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    full = prob.h.get_frontier(prob.h.frontier(pm)).tobytes()
    _, lsteps, smax = prob.h.table_layout()
    NP = 2
    smax_mp = [min(int(smax[mp // NP]), int(lsteps[mp // NP])) if prob.counts[mp // NP] else 0
               for mp in range(len(models) * NP)]
    costs = calibrate(prob.h, len(smax_mp), smax_mp)
    plan = plan_pieces(costs, W)
    hand = [[(mp, sum(1 << S for S in range(1, smax_mp[mp] + 1)), r / 3, (r + 1) / 3)
             for mp in range(len(smax_mp)) if smax_mp[mp]] for r in range(3)]
    # overlapping ranges of one slot on one rank (S <= 3 over all candidates, S >= 4 over
    # the first half): their decodes update the same records, in stream order
    low = lambda mp: sum(1 << S for S in range(1, min(3, smax_mp[mp]) + 1))  # noqa: E731
    high = lambda mp: sum(1 << S for S in range(4, smax_mp[mp] + 1))  # noqa: E731
    overlap = [[(mp, low(mp), 0.0, 1.0) for mp in range(len(smax_mp)) if smax_mp[mp]] +
               [(mp, high(mp), 0.0, 0.5) for mp in range(len(smax_mp)) if high(mp)],
               [(mp, high(mp), 0.5, 1.0) for mp in range(len(smax_mp)) if high(mp)]]
    item = _native.FRONTIER_DTYPE.itemsize
    for rank_plans in (plan, hand, overlap):
        cands = []
        for r in range(len(rank_plans)):
            prob.h.evaluate_pieces(pieces_to_ranges(rank_plans[r], prob.counts, NP))
            n = prob.h.frontier_candidates(pm)
            cands.append(prob.h.get_frontier(n))
        cap = max(len(c) for c in cands) + 1
        stride = item + cap * item
        buf = np.zeros(len(cands) * stride, dtype=np.uint8)
        for r, part in enumerate(cands):
            buf[r * stride + item: r * stride + item + len(part) * item] = part.view(np.uint8)
        import torch
        dbuf = torch.from_numpy(buf).cuda()
        n = prob.h.frontier_merge_parts(dbuf.data_ptr(), stride, item, [len(c) for c in cands])
        assert prob.h.get_frontier(n).tobytes() == full
        # the product's path: each rank's candidates straight into its device slot
        # (count header written on the device), merged on device-read counts; a slot
        # too small reports the overflow instead of a frontier
        mx = max(len(c) for c in cands)
        for cap2, ok in ((max(mx - 1, 0), mx == 0), (mx, True), (mx + 37, True)):
            stride2 = item + cap2 * item
            gath = torch.zeros(len(cands) * stride2, dtype=torch.uint8, device="cuda")
            for r in range(len(rank_plans)):
                prob.h.evaluate_pieces(pieces_to_ranges(rank_plans[r], prob.counts, NP))
                prob.h.frontier_candidates_into(pm, gath.data_ptr() + r * stride2, item, cap2)
            n2, got_mx = prob.h.frontier_merge_gathered(gath.data_ptr(), len(cands), stride2, item, cap2)
            assert got_mx == mx
            if ok:
                assert prob.h.get_frontier(n2).tobytes() == full
            else:
                assert n2 == -1
        # more parts than the device-count path holds (32): headers read on the host
        stride2 = item + mx * item
        gath = torch.zeros(40 * stride2, dtype=torch.uint8, device="cuda")
        for r in range(len(rank_plans)):
            prob.h.evaluate_pieces(pieces_to_ranges(rank_plans[r], prob.counts, NP))
            prob.h.frontier_candidates_into(pm, gath.data_ptr() + (39 - r) * stride2, item, mx)
        n2, got_mx = prob.h.frontier_merge_gathered(gath.data_ptr(), 40, stride2, item, mx)
        assert got_mx == mx and prob.h.get_frontier(n2).tobytes() == full


def test_candidates_into_empty_price_matrix_writes_an_empty_slot():
    """The multi-GPU slot path with nothing to price (no regions): the count header is
    still written (0), so the all-gather never carries a stale count."""
    import torch
    from paper_2605_04357_b200 import _native
    configs, models, slos, caps, ctx, regions, prices = workload("c1")
    prob = Stage1Problem(configs, models, slos, caps, ctx).run()
    item = _native.FRONTIER_DTYPE.itemsize
    slot = torch.full((item + 4 * item,), 0xFF, dtype=torch.uint8, device="cuda")
    prob.h.frontier_candidates_into(np.zeros((0, len(configs))), slot.data_ptr(), item, 4)
    torch.cuda.synchronize()
    assert slot[:8].view(torch.int64).item() == 0


@pytest.mark.parametrize("seed", [1, 2, 4, 12, 16, 32])
def test_random_scenarios_library_frontier_and_pieces(seed):
    """tools/stress_random.py scenarios (n_max up to 7, non-monotone / 1e-12-tolerance
    ProfileTable rows, regional prices with unpriced configs): records, frontier and a
    three-rank pieces merge through the device slots all equal the oracle."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "stress_random.py")
    spec = importlib.util.spec_from_file_location("stress_random", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.check(seed) == ""
