"""Pin the CPU oracle (oracle/coral_oracle.c) against golden vectors produced by
running the unmodified reference (tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_04357_b200._native import MAX_NODES
from tests.helpers import (cfg_by_rank, digest, golden, key_str, oracle_library_lines,
                           oracle_problem, workload)


@pytest.fixture(scope="module", autouse=True)
def _built():
    O.build()


def test_placement_search_matches_reference_bit_exact():
    """kernels.py:279-295 on the test_kernels.py generators + wider cases:
    objective, stage layers and stage counts identical to the numba path."""
    cases = golden("kernels.json.gz")
    assert len(cases) > 1500
    for c in cases:
        best, sj, sc = O.placement_search(np.array(c["counts"]), np.array(c["tput"]), c["S"])
        assert best == c["best"]
        assert sj.tolist() == c["stage_j"]
        assert sc.tolist() == c["stage_counts"]


@pytest.mark.parametrize("w", ["c1", "core", "extended"])
def test_throughput_tables_and_budgets_bit_exact(w):
    g = golden(f"tables_{w}.json.gz")
    op = oracle_problem(w)
    assert [c.name for c in op.configs] == g["configs"]
    for mi, m in enumerate(op.models):
        for ph, code in (("prefill", 0), ("decode", 1)):
            for S in range(1, min(6, m.num_layers) + 1):
                ref = g["tables"][f"{m.name}|{ph}|{S}"]
                assert op.stage_budget(mi, code, S) == ref["budget"]
                np.testing.assert_array_equal(op.table(mi, code, S), np.array(ref["rows"]))


def test_perf_grid_bit_exact():
    """node_max_throughput (perf.py:159-230) on a nodes x models x phases x j x
    budget grid, two PerfParams; exact equality."""
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.library import GenContext, LibraryCaps
    from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, PerfParams, SloSpec
    from oracle.oracle import OracleProblem, lib
    params = [PerfParams(), PerfParams(mfu=0.3, mbu=0.9, fixed_overhead_ms=0.0,
                                       avg_prompt_tokens=333.3, avg_ctx_tokens=777.7)]
    models = {m.name: m for m in catalog.MODEL_CATALOG.values()}
    models["tiny"] = ModelSpec("tiny", 4, 0.5, 0.5, 256, kv_bytes_per_token_per_layer=128.0)
    grid = golden("perf_grid.json.gz")
    assert len(grid) >= 100
    cache = {}
    for e in grid:
        key = (e["p"], e["gpu"], e["gc"], e["model"])
        if key not in cache:
            node = NodeConfig(catalog.GPU_CATALOG[e["gpu"]], e["gc"])
            m = models[e["model"]]
            cache[key] = OracleProblem.from_specs([node], [m], {m.name: SloSpec(1, 1)},
                                                  LibraryCaps(1, 2.0),
                                                  GenContext(perf=params[e["p"]]), ("prefill",))
        op = cache[key]
        code = 0 if e["phase"] == "prefill" else 1
        got = lib().or_node_max_throughput(op.ref, 0, 0, code, e["j"], e["budget"])
        assert got == e["tput"], e


@pytest.mark.parametrize("w", ["c1", "core"])
def test_enumeration_full_lists(w):
    """enumerate_combos (templates.py:99-113): same set, and the packed-key sort
    reproduces (num_nodes, str(combo)) order exactly."""
    g = golden(f"enum_{w}.json.gz")
    op = oracle_problem(w)
    cbr = cfg_by_rank(op.configs)
    for mi, m in enumerate(op.models):
        keys = op.enumerate(mi)
        strs = [key_str(k, cbr) for k in keys]
        ref = g[m.name]["combos"]
        assert strs == sorted(ref)  # library (str) order
        by_nodes = sorted(strs, key=lambda s: sum(int(t.rsplit("*", 1)[1]) for t in s.split("+")))
        assert by_nodes == ref      # enumeration order (num_nodes, str), stable


def test_enumeration_extended_digest():
    g = golden("enum_extended.json.gz")
    op = oracle_problem("extended")
    cbr = cfg_by_rank(op.configs)
    for mi, m in enumerate(op.models):
        strs = [key_str(k, cbr) for k in op.enumerate(mi)]
        strs.sort(key=lambda s: sum(int(t.rsplit("*", 1)[1]) for t in s.split("+")))
        assert len(strs) == g[m.name]["count"]
        assert digest(strs) == g[m.name]["sha256"]


def test_library_c1_full():
    g = golden("library_c1.json.gz")
    lines = oracle_library_lines(oracle_problem("c1"))
    assert lines == g["records"]
    assert digest(lines) == g["sha256"]


def test_library_core_sampled():
    """Every 5th combo of the core library (templates.py:417-505) against the
    reference records: values, S and canonical placements bit-identical."""
    g = golden("library_core.json.gz")
    ref = {ln.rsplit("|", 4)[0]: ln for ln in g["records"]}
    lines = oracle_library_lines(oracle_problem("core"), stride=5)
    assert len(lines) > 5000
    for ln in lines:
        assert ref[ln.rsplit("|", 4)[0]] == ln


def test_profile_override_library():
    """ProfileTable overrides (perf.py:94-116) flow through stage 1 exactly."""
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.library import GenContext, LibraryCaps
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
    op = oracle_problem((configs, [model], {"m7b": SloSpec(1500, 80)}, LibraryCaps(3, 10.0),
                         GenContext(profile=prof)))
    assert oracle_library_lines(op) == g["library"]["records"]


def tolmono_inputs():
    """Inputs of tests/golden/tolmono.json.gz (make_golden.tolmono_case)."""
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.library import GenContext, LibraryCaps
    from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, ProfileTable, SloSpec
    g = golden("tolmono.json.gz")
    configs = [NodeConfig(catalog.GPU_CATALOG["A100"], 1), NodeConfig(catalog.GPU_CATALOG["A100"], 2),
               NodeConfig(catalog.GPU_CATALOG["L40S"], 2)]
    model = ModelSpec("m8", num_layers=8, params_total_b=14, params_active_b=14, hidden_size=5120)
    prof = ProfileTable()
    for cfg, mdl, ph, j, b, v in g["profile"]:
        prof.add(cfg, mdl, ph, j, b, v)
    return g, (configs, [model], {"m8": SloSpec(1500, 80)}, LibraryCaps(4, 40.0), GenContext(profile=prof))


def test_tolerance_monotone_rows_library():
    """Rows monotone only within kernels.py:291's 1e-12: the reference's binary search
    on a non-monotone predicate, reproduced literally."""
    g, inputs = tolmono_inputs()
    assert oracle_library_lines(oracle_problem(inputs)) == g["library"]["records"]


@pytest.mark.parametrize("w", ["c1", "core"])
def test_frontier_matches_reference_library_frontier(w):
    """SURVEY.md 8c frontier: the oracle's skyline over its own records equals the
    frontier computed in Python on the reference's library."""
    g = golden(f"frontier_{w}.json.gz")
    lib = {ln.rsplit("|", 4)[0] for ln in golden(f"library_{w}.json.gz")["records"]}
    configs, models, slos, caps, ctx, regions, prices = workload(w)
    op = oracle_problem(w)
    cbr = cfg_by_rank(op.configs)
    from tests.helpers import price_matrix
    pm = price_matrix(op.configs, prices, regions)
    got = []
    for mi, m in sorted(enumerate(op.models), key=lambda t: t[1].name):
        for ph in sorted(op.phases):
            keys = op.enumerate(mi)
            # frontier candidates are exactly the reference library's templates
            recs = op.solve(mi, 0 if ph == "prefill" else 1, keys)
            feas = [key_str(k, cbr) for k, r in zip(keys, recs) if r["num_stages"] > 0]
            assert {f"{m.name}|{ph}|{s}" for s in feas} <= lib
            reg, idx = op.frontier(keys, recs, pm)
            for r, i in zip(reg, idx):
                got.append([m.name, ph, regions[r].name, key_str(keys[i], cbr),
                            None, float(recs[i]["throughput_tps"])])
    ref = [[a, b, c, d, None, f] for a, b, c, d, e, f in g]
    key = lambda t: (t[0], t[1], t[2])  # noqa: E731
    assert sorted(got, key=key) == sorted(ref, key=key)


@pytest.mark.parametrize("w", ["extended", "c3"])
def test_library_big_sample(w):
    """Every 97th template of the reference libraries of BASELINE config 2
    (1,084,362 templates) and config 3 (344,548, Lu = 80): the oracle re-solves those
    combos and matches bit for bit."""
    g = golden(f"library_{w}.json.gz")
    op = oracle_problem(w)
    cbr = cfg_by_rank(op.configs)
    rank_of = {c.name: r for r, c in enumerate(cbr)}
    midx = {m.name: i for i, m in enumerate(op.models)}
    by_mp = {}
    for ln in g["sample"]:
        model, phase, combo = ln.split("|")[:3]
        key = 0
        toks = combo.split("+")
        for name, n in (t.rsplit("*", 1) for t in toks):
            key = (key << 9) | ((rank_of[name] + 1) << 3) | int(n)
        key <<= 9 * (MAX_NODES - len(toks))
        by_mp.setdefault((model, phase), []).append((key, ln))
    from tests.helpers import record_line
    checked = 0
    for (model, phase), items in by_mp.items():
        keys = np.array([k for k, _ in items], dtype=np.uint64)
        recs = op.solve(midx[model], 0 if phase == "prefill" else 1, keys)
        for (k, ln), r in zip(items, recs):
            assert record_line(model, phase, k, r, cbr) == ln
            checked += 1
    assert checked == len(g["sample"]) > 3000
