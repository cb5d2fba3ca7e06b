"""Shared test helpers: golden fixtures, canonical record lines, workload inputs."""

from __future__ import annotations

import gzip
import hashlib
import json
import os

import numpy as np

from paper_2605_04357_b200 import catalog
from paper_2605_04357_b200.library import GenContext, LibraryCaps, decode_key

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


def digest(lines) -> str:
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def line(model, phase, combo_str, S, layers, son, T) -> str:
    return (f"{model}|{phase}|{combo_str}|{S}|{','.join(map(str, layers))}|"
            f"{','.join(map(str, son))}|{float(T)!r}")


def template_line(t) -> str:
    return line(t.model, t.phase, str(t.combo), t.placement.num_stages,
                t.placement.layers_per_stage, t.placement.stage_of_node, t.throughput_tps)


def key_str(key, cfg_by_rank) -> str:
    return "+".join(f"{cfg_by_rank[r].name}*{n}" for r, n in decode_key(int(key)))


def record_line(model, phase, key, rec, cfg_by_rank) -> str:
    S = int(rec["num_stages"])
    n = int(rec["num_nodes"])
    return line(model, phase, key_str(key, cfg_by_rank), S,
                [int(x) for x in rec["layers_per_stage"][:S]],
                [int(x) for x in rec["stage_of_node"][:n]], rec["throughput_tps"])


def workload(name):
    """(configs, models, slos, caps, ctx, regions, prices) exactly as
    tests/golden/run_reference_library.py builds them from the reference."""
    w = catalog.WORKLOADS[name]()
    return (w.configs, w.models, w.slos, LibraryCaps(w.n_max, w.rho),
            GenContext(perf=w.perf, granularity=w.granularity), w.regions, w.prices)


def cfg_by_rank(configs):
    from paper_2605_04357_b200.library import str_ranks
    configs = sorted(configs, key=lambda c: c.name)
    ranks = str_ranks([c.name for c in configs])
    out = [None] * len(configs)
    for i, r in enumerate(ranks):
        out[r] = configs[i]
    return out


def oracle_problem(name_or_inputs, phases=("prefill", "decode")):
    from oracle.oracle import OracleProblem
    if isinstance(name_or_inputs, str):
        configs, models, slos, caps, ctx, regions, prices = workload(name_or_inputs)
    else:
        configs, models, slos, caps, ctx = name_or_inputs[:5]
    return OracleProblem.from_specs(configs, models, slos, caps, ctx, phases)


def oracle_library_lines(op, stride=1, threads=0):
    """Oracle records of every (model, phase) as canonical lines in library order,
    solving every `stride`-th combo only."""
    cbr = cfg_by_rank(op.configs)
    lines = []
    order = sorted(((m.name, ph, mi, pi) for mi, m in enumerate(op.models)
                    for pi, ph in enumerate(op.phases)))
    for mname, ph, mi, pi in order:
        keys = op.enumerate(mi)
        code = 0 if ph == "prefill" else 1
        recs = op.solve(mi, code, keys, 0, stride, threads=threads)
        for i in range(0, len(keys), stride):
            if recs[i]["num_stages"] > 0:
                lines.append(record_line(mname, ph, keys[i], recs[i], cbr))
    return lines


def price_matrix(configs, prices, regions):
    configs = sorted(configs, key=lambda c: c.name)
    mat = np.full((len(regions), len(configs)), np.nan)
    for i, r in enumerate(regions):
        for k, c in enumerate(configs):
            p = prices.get((getattr(r, "name", r), c.name))
            if p is not None:
                mat[i, k] = p
    return mat


def alloc_inputs(config_names, region_names, library):
    """Deterministic stage-2 inputs for the allocation-model parity tests
    (tests/golden/make_alloc_golden.py): prices of the core workload with two configs
    unpriced in the last region, seeded availability per (region, config), a demand per
    (model, phase) with one zero, three running templates and an init penalty."""
    w = catalog.WORKLOADS["core"]()
    cfgs = sorted(config_names)
    regs = sorted(region_names)
    prices = {k: v for k, v in w.prices.items() if k[0] in regs}
    for c in cfgs[:2]:
        prices.pop((regs[-1], c), None)
    rng = np.random.default_rng(7)
    avail = {(r, c): int(rng.integers(0, 40)) for r in regs for c in cfgs}
    mps = library.model_phases()
    demand = {(m, ph): (20000.0 if ph == "prefill" else 6000.0) for m, ph in mps}
    demand[mps[-1]] = 0.0
    running = []
    for m, ph in mps[:3]:
        ts = library.templates_for(m, ph)
        running.append((regs[0], ts[-1].template_id))
    return prices, avail, demand, running, 0.25


def milp_digest(milp) -> dict:
    """Canonical text digests of a MilpModel (milp/model.py:55-120): variables in
    insertion order, objective, constraints with their coefficient dicts in order."""
    def sha(lines):
        return digest(lines)
    return {
        "n_vars": len(milp.variables), "n_cons": len(milp.constraints), "sense": milp.sense,
        "vars_sha": sha(f"{v.vid}|{v.kind}|{v.ub!r}" for v in milp.variables.values()),
        "obj_sha": sha(f"{k}|{c!r}" for k, c in milp.objective.items()),
        "cons_sha": sha(f"{c.name}|{c.sense}|{c.rhs!r}|" + ";".join(f"{v}:{x!r}" for v, x in c.coeffs.items())
                        for c in milp.constraints),
        "first_vars": [f"{v.vid}|{v.kind}|{v.ub!r}" for v in list(milp.variables.values())[:40]],
        "first_cons": [f"{c.name}|{c.sense}|{c.rhs!r}|{len(c.coeffs)}" for c in milp.constraints[:40]],
    }


def zigzag_profile(configs, models, table_cls, names=("1xL4", "2xA10G")):
    """A ProfileTable (perf.py:94-141) that breaks the T-hat monotonicity test of
    kernels.py:291 for two node configs: for every model, phase and layer count j a
    zigzag throughput (odd layer units 30% faster than their even neighbours), any
    budget (bucket -1). Combos with these configs take the reference's full-scan DP
    (kernels.py:240-249); the rest keep the binary-search crossing."""
    prof = table_cls()
    for c in configs:
        if c.name not in names:
            continue
        for m in models:
            for ph in ("prefill", "decode"):
                base = (4.0e5 if ph == "prefill" else 6.0e4) * c.gpu_count * c.gpu.tflops / (312.0 * m.params_active_b)
                for j in range(1, m.num_layers + 1):
                    prof.add(c.name, m.name, ph, j, -1, base / j * (1.3 if j % 2 else 1.0))
    return prof
