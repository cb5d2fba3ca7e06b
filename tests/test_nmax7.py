"""n_max = 7: the caps point (7, 14) of the reference's own acceptance sweep
(pkg/tests/test_acceptance.py:320-348, c09). Golden vectors from the unmodified
reference (tests/golden/make_golden_n7.py, n7.json.gz): placement_search on 7-node
multisets, the c09 model's library and sweep rows, and the core scenario at (7, 14)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_04357_b200 import catalog
from paper_2605_04357_b200.library import GenContext, LibraryCaps
from paper_2605_04357_b200.specs import ModelSpec, NodeConfig, SloSpec
from tests.helpers import digest, golden, oracle_library_lines, oracle_problem, template_line, workload

C09_MODEL = ModelSpec("m120b", num_layers=36, params_total_b=116.8, params_active_b=5.1, hidden_size=2880,
                      kv_bytes_per_token_per_layer=2048, is_moe=True, is_hybrid_attn=True)


def c09_inputs(n_max=7, rho=14.0):
    cfgs = [NodeConfig(catalog.GPU_CATALOG["H100"], 2, 64.0), NodeConfig(catalog.GPU_CATALOG["L40S"], 1, 64.0)]
    return cfgs, [C09_MODEL], {"m120b": SloSpec(1000, 40)}, LibraryCaps(n_max, rho), GenContext()


def test_oracle_placement_search_seven_nodes():
    cases = golden("n7.json.gz")["kernels7"]
    assert len(cases) >= 1000 and max(sum(c["counts"]) for c in cases) == 7
    for c in cases:
        best, sj, sc = O.placement_search(np.array(c["counts"]), np.array(c["tput"]), c["S"])
        assert best == c["best"] and sj.tolist() == c["stage_j"] and sc.tolist() == c["stage_counts"]


def test_oracle_c09_library_at_7_14():
    g = golden("n7.json.gz")["c09"]
    lines = oracle_library_lines(oracle_problem(c09_inputs(), phases=("prefill",)))
    assert lines == g["library"]


def test_oracle_core_at_7_14_sample():
    g = golden("n7.json.gz")["core7"]
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    op = oracle_problem((configs, models, slos, LibraryCaps(7, 14.0), ctx))
    # every 41st reference line re-solved by the oracle
    from tests.helpers import cfg_by_rank, record_line
    from paper_2605_04357_b200._native import MAX_NODES
    cbr = cfg_by_rank(op.configs)
    rank_of = {c.name: r for r, c in enumerate(cbr)}
    midx = {m.name: i for i, m in enumerate(op.models)}
    for ln in g["sample"][::3]:
        model, phase, combo = ln.split("|")[:3]
        toks = combo.split("+")
        key = 0
        for name, n in (t.rsplit("*", 1) for t in toks):
            key = (key << 9) | ((rank_of[name] + 1) << 3) | int(n)
        key <<= 9 * (MAX_NODES - len(toks))
        rec = op.solve(midx[model], 0 if phase == "prefill" else 1, np.array([key], dtype=np.uint64))[0]
        assert record_line(model, phase, key, rec, cbr) == ln


@pytest.mark.gpu
def test_gpu_placement_search_seven_nodes():
    from paper_2605_04357_b200 import placement_search_batch
    cases = golden("n7.json.gz")["kernels7"]
    got = placement_search_batch([(np.array(c["counts"]), np.array(c["tput"]), c["S"]) for c in cases])
    for c, (best, sj, sc) in zip(cases, got):
        assert best == c["best"] and sj.tolist() == c["stage_j"] and sc.tolist() == c["stage_counts"], c


@pytest.mark.gpu
def test_gpu_c09_library_and_sweep_at_7_14():
    """The c09 point (7, 14): the full library bit-identical, and the sweep rows
    (4,8), (6,12), (7,14) from ONE solve equal the reference's per-caps rebuilds,
    with the acceptance test's plateau shape (test_acceptance.py:340-346)."""
    from paper_2605_04357_b200 import build_library
    from paper_2605_04357_b200.frontier import sweep
    g = golden("n7.json.gz")["c09"]
    cfgs, models, slos, caps, ctx = c09_inputs()
    lib = build_library(cfgs, models, slos, caps, ctx, phases=("prefill",))
    assert [template_line(t) for t in lib.entries] == g["library"]
    prices = {("r", c.name): c.gpu.rel_cost * c.gpu_count for c in cfgs}
    rows = sweep(cfgs, models, slos, [LibraryCaps(n, r) for n, r, _, _ in g["rows"]], prices, regions=["r"],
                 ctx=ctx, phases=("prefill",))
    assert [(n, r, c, b) for n, r, c, _, b in rows] == [tuple(x) for x in g["rows"]]
    effs = [b for *_, b in rows]
    counts = [c for _, _, c, _, _ in rows]
    assert effs[0] <= effs[1] + 1e-9 and effs[1] <= effs[2] + 1e-9 and effs[1] - effs[0] > effs[2] - effs[1]
    assert counts[0] < counts[1] < counts[2]


@pytest.mark.gpu
def test_gpu_core_library_at_7_14():
    """The core scenario at (7, 14): 82,129 templates, sha256 of every line equal to the
    reference's, and its cmd_sweep row."""
    from paper_2605_04357_b200 import build_library
    from paper_2605_04357_b200.frontier import sweep
    g = golden("n7.json.gz")["core7"]
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    lib = build_library(configs, models, slos, LibraryCaps(7, 14.0), ctx)
    lines = [template_line(t) for t in lib.entries]
    assert len(lines) == g["count"]
    assert lines[::g["sample_every"]] == g["sample"]
    assert digest(lines) == g["sha256"]
    row = sweep(configs, models, slos, [LibraryCaps(7, 14.0)], prices, regions=regions, ctx=ctx)[0]
    assert (row[0], row[1], row[2], row[4]) == tuple(g["sweep_row"])
