"""Reference stage-1 semantics on the GPU path, ported from the reference's own tests
(/root/reference/pkg/tests/test_templates.py, test_kernels.py) to this package's API."""

import numpy as np
import pytest

from paper_2605_04357_b200 import catalog
from paper_2605_04357_b200 import (DomainError, LibraryGenError, build_library,
                                   enumerate_combos, placement_search, stage_budget_s)
from paper_2605_04357_b200.library import GenContext, LibraryCaps
from paper_2605_04357_b200.roofline import node_max_throughput
from paper_2605_04357_b200.specs import (DECODE, PREFILL, GpuSpec, ModelSpec, NodeConfig,
                                         SloSpec, combo_key)
from tests.helpers import oracle_library_lines, oracle_problem, template_line

pytestmark = pytest.mark.gpu

FAST = NodeConfig(GpuSpec("FastG", 80, 3.35, 989, 7.6), 2)
SLOW = NodeConfig(GpuSpec("SlowG", 24, 0.60, 70, 1.2), 1)
M8 = ModelSpec("m8", num_layers=8, params_total_b=14, params_active_b=14, hidden_size=5120)
SLO = SloSpec(1200, 60)
CTX = GenContext()


def test_enumeration_window_and_counts():  # test_templates.py:24-54
    cfg = NodeConfig(GpuSpec("g", 40, 1.0, 100, 1.0), 1)
    model = ModelSpec("m", num_layers=4, params_total_b=15, params_active_b=15, hidden_size=64)
    assert [str(c) for c in enumerate_combos([cfg], model, LibraryCaps(2, 2.0))] == ["1xg*1"]
    model32 = ModelSpec("m32", num_layers=4, params_total_b=32, params_active_b=32, hidden_size=64)
    big = NodeConfig(GpuSpec("g", 80, 1.0, 100, 1.0), 1)
    for c in enumerate_combos([big], model32, LibraryCaps(6, 12.0)):
        assert model32.weight_bytes <= c.total_mem_bytes < 12.0 * model32.weight_bytes
    gpus = [GpuSpec(f"g{i}", 1000, 1.0, 100, 1.0) for i in range(3)]
    tiny = ModelSpec("m", num_layers=2, params_total_b=0.001, params_active_b=0.001, hidden_size=8)
    assert len(enumerate_combos([NodeConfig(g, 1) for g in gpus], tiny, LibraryCaps(3, 1e9))) == 19
    a = enumerate_combos([FAST, SLOW], M8, LibraryCaps(3, 12.0))
    b = enumerate_combos([SLOW, FAST], M8, LibraryCaps(3, 12.0))
    assert [str(c) for c in a] == [str(c) for c in b]


def test_best_of_s1_s2_closed_form_and_tie_to_fewer_stages():  # test_templates.py:79-95
    combo = combo_key([FAST, FAST])
    lib = build_library([FAST], [M8], {"m8": SLO}, LibraryCaps(2, 13.0), CTX, phases=(DECODE,))
    t = next(t for t in lib.entries if str(t.combo) == str(combo))
    b1 = stage_budget_s(M8, SLO, DECODE, 1, CTX)
    s1 = 2 * node_max_throughput(FAST, M8, DECODE, 8, b1, CTX.perf)
    b2 = stage_budget_s(M8, SLO, DECODE, 2, CTX)
    s2 = max(min(node_max_throughput(FAST, M8, DECODE, j, b2, CTX.perf),
                 node_max_throughput(FAST, M8, DECODE, 8 - j, b2, CTX.perf)) for j in range(1, 8))
    assert t.throughput_tps == max(s1, s2)
    assert t.placement.num_stages == (1 if s1 >= s2 else 2)  # ties -> fewer stages


def test_memory_infeasible_node_never_gets_a_stage():  # test_templates.py:97-104
    tiny = NodeConfig(GpuSpec("tiny", 1, 0.60, 70, 1.2), 1)
    lib = build_library([FAST, tiny], [M8], {"m8": SLO}, LibraryCaps(2, 40.0), CTX, phases=(DECODE,))
    for t in lib.entries:
        for s, cfg in zip(t.placement.stage_of_node, t.combo.expand()):
            if cfg.name == "1xtiny":
                assert t.placement.num_stages == 1 and s == 0


def test_config_order_independence_and_caps_growth():  # test_templates.py:127-149
    a = build_library([FAST, SLOW], [M8], {"m8": SLO}, LibraryCaps(2, 8.0), CTX)
    b = build_library([SLOW, FAST], [M8], {"m8": SLO}, LibraryCaps(2, 8.0), CTX)
    assert [template_line(t) for t in a.entries] == [template_line(t) for t in b.entries]
    big = build_library([FAST, SLOW], [M8], {"m8": SLO}, LibraryCaps(3, 10.0), CTX)
    small_ids = {t.template_id for t in a.entries}
    big_ids = {t.template_id for t in big.entries}
    assert len(big) >= len(a) and small_ids <= big_ids
    assert len(big_ids) == len(big.entries)  # no duplicate ids


def test_superset_monotonicity():  # test_templates.py:203-221: adding configs never loses templates
    base = build_library([FAST, SLOW], [M8], {"m8": SLO}, LibraryCaps(3, 12.0), CTX)
    more = build_library([FAST, SLOW, NodeConfig(catalog.GPU_CATALOG["L4"], 2)], [M8], {"m8": SLO},
                         LibraryCaps(3, 12.0), CTX)
    got = {t.template_id: t.throughput_tps for t in more.entries}
    for t in base.entries:
        assert got[t.template_id] == t.throughput_tps


def test_granularity_two_for_long_models():  # test_templates.py:182-189
    m80 = ModelSpec("m80", num_layers=80, params_total_b=70, params_active_b=70, hidden_size=8192)
    cfgs = catalog.make_configs(["H100"])
    lib = build_library(cfgs, [m80], {"m80": SloSpec(1500, 80)}, LibraryCaps(3, 12.0), CTX)
    assert lib.meta["granularity"]["m80"] == 2
    assert all(j % 2 == 0 for t in lib.entries for j in t.placement.layers_per_stage)
    odd = ModelSpec("m81", num_layers=81, params_total_b=70, params_active_b=70, hidden_size=8192)
    with pytest.raises(DomainError):
        build_library(cfgs, [odd], {"m81": SloSpec(1500, 80)}, LibraryCaps(3, 12.0), GenContext(granularity=2))


def test_budget_formula():  # test_templates.py:192-200
    ctx = GenContext()
    b1 = stage_budget_s(M8, SLO, PREFILL, 1, ctx)
    b3 = stage_budget_s(M8, SLO, PREFILL, 3, ctx)
    act = ctx.perf.avg_prompt_tokens * M8.hidden_size * M8.bytes_per_param
    hop = ctx.net_latency_ms / 1e3 + act / (ctx.net_gbps * 1e9 * ctx.perf.net_eff)
    assert b1 == SLO.prefill_ms / 1e3 * ctx.perf.slo_budget_frac
    assert b3 == pytest.approx((b1 - 2 * hop) / 3, rel=1e-15)
    assert stage_budget_s(M8, SLO, DECODE, 4, ctx) == pytest.approx(b1 * SLO.decode_ms / SLO.prefill_ms / 4)


def test_hard_errors_and_edge_shapes():  # test_templates.py:165-170 + envelope
    tiny = NodeConfig(GpuSpec("tiny", 1, 0.60, 70, 1.2), 1)
    with pytest.raises(LibraryGenError):
        build_library([tiny], [M8], {"m8": SLO}, LibraryCaps(2, 12.0), CTX)
    with pytest.raises(DomainError):
        build_library([FAST], [M8], {"m8": SLO}, LibraryCaps(2, 12.0), CTX, method="ilp")
    with pytest.raises(ValueError):
        placement_search(np.array([1]), np.array([[-1.0, 0.0]]), 1)
    best, sj, sc = placement_search(np.array([1]), np.ones((1, 5)), 2)  # test_kernels.py:85-89
    assert best == -1e300
    # n_max = 1: only single-node combos, S = 1
    lib = build_library([FAST, SLOW], [M8], {"m8": SLO}, LibraryCaps(1, 12.0), CTX)
    assert all(t.combo.num_nodes == 1 and t.placement.num_stages == 1 for t in lib.entries)
    # one phase only; a model with fewer layers than n_max (S <= L)
    m2 = ModelSpec("m2", num_layers=2, params_total_b=1, params_active_b=1, hidden_size=64)
    lib = build_library([SLOW], [m2], {"m2": SloSpec(500, 50)}, LibraryCaps(4, 50.0), CTX, phases=(DECODE,))
    assert {t.phase for t in lib.entries} == {DECODE}
    assert all(t.placement.num_stages <= 2 for t in lib.entries)
    ref = oracle_library_lines(oracle_problem(([SLOW], [m2], {"m2": SloSpec(500, 50)},
                                               LibraryCaps(4, 50.0), CTX), phases=(DECODE,)))
    assert [template_line(t) for t in lib.entries] == ref


def test_reference_objects_are_accepted_duck_typed():
    """hetserve-style inputs: any objects with the reference's attributes work."""
    class G:  # noqa: D401 - minimal duck-typed GPU spec
        def __init__(self, **kw):
            self.__dict__.update(kw)

    class N:
        def __init__(self, gpu, n):
            self.gpu, self.gpu_count, self.intra_node_interconnect_gbps = gpu, n, 64.0

        @property
        def name(self):
            return f"{self.gpu_count}x{self.gpu.name}"

        @property
        def mem_bytes(self):
            return self.gpu_count * self.gpu.mem_gb * (1 << 30)

    gpu = G(name="FastG", mem_gb=80, bw_tbps=3.35, tflops=989, rel_cost=7.6)
    lib = build_library([N(gpu, 2)], [M8], {"m8": SLO}, LibraryCaps(2, 12.0), CTX)
    ref = build_library([FAST], [M8], {"m8": SLO}, LibraryCaps(2, 12.0), CTX)
    assert [template_line(t) for t in lib.entries] == [template_line(t) for t in ref.entries]


def test_live_problems_keep_their_own_device_state(tmp_path):
    """a FrontierSession and a lazy library keep reading their own device
    records while other solves and T-hat queries run in between."""
    import hashlib
    from paper_2605_04357_b200 import FrontierSession, build_frontier, node_max_throughput
    from tests.helpers import golden, workload
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    sess = FrontierSession(configs, models, slos, caps, ctx)
    first = sess.frontier(prices, regions=regions)
    lazy = build_library(configs, models, slos, caps, ctx, lazy=True)
    c1 = workload("c1")
    build_frontier(c1[0], c1[1], c1[2], c1[3], c1[6], regions=c1[5], ctx=c1[4])
    build_library(*c1[:5])
    node_max_throughput(c1[0][0], c1[1][0], "decode", 8, 0.05, c1[4].perf)
    again = sess.frontier(prices, regions=regions)

    def rows(f):
        return sorted((k, str(e.template.combo), e.price_usd_h, e.throughput_tps)
                      for k, v in f.segments.items() for e in v)
    assert rows(again) == rows(first)
    path = str(tmp_path / "core.jsonl")
    lazy.save(path)
    ref = golden("saved_libraries.json.gz")["core"]
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == ref["sha256"]


def test_placement_search_beyond_seven_nodes_is_rejected():
    """more nodes than the envelope (7) would overrun the DP's per-size
    tables; the GPU operator raises DomainError instead (the reference accepts them)."""
    with pytest.raises(DomainError):
        placement_search(np.array([8]), np.ones((1, 8)), 2)
    with pytest.raises(DomainError):
        placement_search(np.array([4, 4]), np.ones((2, 8)), 7)
    # S above the node count stays the reference's infeasible answer (kernels.py:174-175)
    best, sj, sc = placement_search(np.array([2, 1]), np.ones((2, 8)), 5)
    assert best == -1e300


def test_sweep_raises_like_build_library_and_cmd_sweep():
    """the one-solve sweep raises LibraryGenError when a caps entry leaves a
    (model, phase) without templates (templates.py:499-502), and KeyError when a
    template uses a config unpriced in some region (cli.py:255)."""
    from paper_2605_04357_b200.frontier import sweep
    big = ModelSpec("big", num_layers=8, params_total_b=60, params_active_b=60, hidden_size=5120)
    p = {("r", FAST.name): 2.0, ("r", SLOW.name): 1.0}
    rows = sweep([FAST, SLOW], [big], {"big": SLO}, [LibraryCaps(3, 12.0)], p, regions=["r"], ctx=CTX)
    assert rows[0][2] > 0
    with pytest.raises(LibraryGenError):  # one node of <= 160 GB cannot hold 120 GB x rho window... caps n_max=1
        sweep([SLOW], [big], {"big": SLO}, [LibraryCaps(1, 1.5), LibraryCaps(3, 12.0)],
              {("r", SLOW.name): 1.0}, regions=["r"], ctx=CTX)
    with pytest.raises(KeyError):
        sweep([FAST, SLOW], [big], {"big": SLO}, [LibraryCaps(3, 12.0)], {("r", FAST.name): 2.0},
              regions=["r"], ctx=CTX)


def test_per_launch_timing_is_opt_in_and_reset_on_release(monkeypatch):
    """coral_s1_set_timing: the evaluate records per-launch events only when asked (the
    default path records none); a handle returned to the pool forgets the diagnostics
    settings of its last lease (timing, census, streams)."""
    from paper_2605_04357_b200 import _native
    from paper_2605_04357_b200.library import Stage1Problem
    from tests.helpers import workload
    configs, models, slos, caps, ctx, regions, prices = workload("core")
    monkeypatch.setitem(_native._pool, 0, [])  # an empty pool: the released handle comes back
    prob = Stage1Problem(configs, models, slos, caps, ctx)
    prob.run()
    assert prob.h.kernel_timeline() == []
    prob.h.set_timing(True)
    prob.run()
    tl = prob.h.kernel_timeline()
    assert tl and {k for k, _, _, _ in tl} >= {0, 1, 2, 3}
    assert all(e >= b >= 0.0 for _, _, b, e in tl)
    h = prob.h
    prob.h.set_census(True)
    prob.h.set_streams(1)
    prob.close()
    again = _native.acquire(h.device)
    try:
        assert again is h
        from paper_2605_04357_b200.library import _pack_problem
        arrays, scalars = _pack_problem(sorted(configs, key=lambda c: c.name), models, slos,
                                        ("prefill", "decode"), caps, ctx)
        again.set_problem(arrays, scalars)
        again.tables()
        again.enumerate()
        again.evaluate(0, -1)
        assert again.kernel_timeline() == []
        assert again.census_all() == [0, 0, 0, 0]
    finally:
        _native.release(again)
