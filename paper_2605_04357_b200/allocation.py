"""Stage-2 model construction from device records.

`build_allocation_model` has the signature, arguments and result of the reference's
hetserve.allocation.build_allocation_model (/root/reference/pkg/src/hetserve/
allocation.py:108-195) for a device-backed library (build_library(..., lazy=True) or a
Stage1Problem). The per-(template, region) work -- price (allocation.py:91-98),
cost-efficiency p/T, the per-(model, phase) best, the prune rule (:143-153), the
availability cap (:101-105) and ceil(demand / T) bound (:154-157) -- runs over the
device records in one pass per rule (csrc/coral_s1.cu alloc_*_kernel) and emits the
surviving variables in the reference's insertion order. The host then assembles the
same MilpModel (variables, capacity rows sorted by (region, config), demand rows
sorted by (model, phase), init-penalty rows) the unchanged stage-2 solver consumes,
or exposes it as CSR arrays (`AllocationCSR`) for a direct HiGHS call.

The model types mirror milp/model.py:30-120 field for field (MilpVar, Constraint,
MilpModel) so the reference's solver accepts them unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .specs import DomainError

BINARY, INTEGER, CONTINUOUS = "binary", "integer", "continuous"
LE, EQ, GE = "<=", "=", ">="


@dataclass(frozen=True)
class MilpVar:
    vid: str
    kind: str
    ub: float | None = None


@dataclass
class Constraint:
    name: str
    coeffs: dict
    sense: str
    rhs: float


@dataclass
class MilpModel:
    """milp/model.py:55-120: variables in insertion order, constraints, objective."""

    name: str = "model"
    variables: dict = field(default_factory=dict)
    constraints: list = field(default_factory=list)
    objective: dict = field(default_factory=dict)
    sense: str = "min"

    def add_var(self, vid: str, kind: str = CONTINUOUS, ub: float | None = None) -> str:
        if vid in self.variables:
            raise DomainError(f"duplicate variable {vid!r}")
        self.variables[vid] = MilpVar(vid, kind, ub)
        return vid

    def add_constraint(self, name: str, coeffs: dict, sense: str, rhs: float) -> None:
        self.constraints.append(Constraint(name, dict(coeffs), sense, rhs))

    def set_objective(self, coeffs: dict, sense: str = "min") -> None:
        self.objective = dict(coeffs)
        self.sense = sense

    @property
    def var_order(self) -> list:
        return list(self.variables)

    def int_var_ids(self) -> list:
        return [v.vid for v in self.variables.values() if v.kind in (BINARY, INTEGER)]


@dataclass
class DemandSpec:
    """Required throughput in tokens/s per (model, phase) (domain.py:205-221)."""

    rates: dict = field(default_factory=dict)

    def __post_init__(self):
        for key, rate in self.rates.items():
            if rate < 0:
                raise DomainError(f"negative demand for {key}")

    def get(self, model: str, phase: str) -> float:
        return self.rates.get((model, phase), 0.0)

    def scaled(self, factor: float) -> "DemandSpec":
        return DemandSpec({k: v * factor for k, v in self.rates.items()})


@dataclass
class MarketState:
    """Per (region, config): available node count and per-node price (domain.py:223-246)."""

    availability: dict = field(default_factory=dict)
    prices: dict = field(default_factory=dict)

    def __post_init__(self):
        for key, a in self.availability.items():
            if a < 0:
                raise DomainError(f"negative availability for {key}")
        for key, p in self.prices.items():
            if p <= 0:
                raise DomainError(f"non-positive price for {key}")

    def price(self, region: str, config: str):
        return self.prices.get((region, config))

    def available(self, region: str, config: str) -> int:
        return self.availability.get((region, config), 0)

    def regions(self) -> list:
        return sorted({r for r, _ in self.prices} | {r for r, _ in self.availability})


@dataclass(frozen=True)
class InstanceInfo:
    iid: str
    region: str
    template_id: str
    load: int = 0


@dataclass
class RunningState:
    """Running serving instances (allocation.py:37-53)."""

    instances: list = field(default_factory=list)

    def counts(self) -> dict:
        out: dict = {}
        for inst in self.instances:
            key = (inst.region, inst.template_id)
            out[key] = out.get(key, 0) + 1
        return out


@dataclass
class AllocationProblem:
    milp: MilpModel
    var_map: dict
    prices: dict
    demand: object
    market: object
    library: object
    running_counts: dict
    k_init: float
    meta: dict = field(default_factory=dict)
    csr: object = None


@dataclass
class AllocationCSR:
    """The model as arrays (variable order = MilpModel insertion order of the nu vars):
    per variable (region, template ordinal) key, ub, price (objective) and throughput
    (its demand-row coefficient); capacity rows (region, config) as CSR over the nu
    vars with the node counts as coefficients."""

    mp: np.ndarray
    region: np.ndarray
    combo_key: np.ndarray
    ub: np.ndarray
    price: np.ndarray
    throughput: np.ndarray
    cap_rows: list            # [(region name, config name)] in row order
    cap_rhs: np.ndarray
    cap_ptr: np.ndarray
    cap_idx: np.ndarray
    cap_val: np.ndarray


def _device_problem(library):
    prob = getattr(library, "_prob", None) or (library if hasattr(library, "h") and hasattr(library, "cfg_by_rank")
                                               else None)
    if prob is None or prob.h is None:
        raise DomainError("the device allocation model needs a device-backed library "
                          "(build_library(..., lazy=True) or a Stage1Problem)")
    return prob


def _demand_of(demand, model, phase) -> float:
    return float(demand.get(model, phase)) if hasattr(demand, "get") and not isinstance(demand, dict) \
        else float(demand.get((model, phase), 0.0))


def _tokens(keys: np.ndarray):
    shifts = np.array([9 * (_native.MAX_NODES - 1 - t) for t in range(_native.MAX_NODES)], dtype=np.uint64)
    toks = ((keys[:, None] >> shifts[None, :]) & np.uint64(511)).astype(np.int64)
    return (toks >> 3) - 1, toks & 7   # str rank (-1 = empty slot), count


def build_allocation_model(library, demand, market, running, k_init: float,
                           prune_ratio: float = 3.0) -> AllocationProblem:
    """allocation.py:108-195 on the device records of `library` (see module doc)."""
    prob = _device_problem(library)
    NP = len(prob.phases)
    nmp = len(prob.models) * NP
    mname = [prob.models[mp // NP].name for mp in range(nmp)]
    pname = [prob.phases[mp % NP] for mp in range(nmp)]
    order = sorted(range(nmp), key=lambda mp: (mname[mp], pname[mp]))
    regions = list(market.regions())
    cfgs = prob.configs                       # name order (config index order)
    K = len(cfgs)
    pm = np.full((len(regions), K), np.nan)
    av = np.zeros((len(regions), K), dtype=np.int64)
    for i, r in enumerate(regions):
        for k, c in enumerate(cfgs):
            p = market.price(r, c.name)
            if p is not None:
                pm[i, k] = float(p)
            av[i, k] = int(market.available(r, c.name))
    dem = np.array([_demand_of(demand, mname[mp], pname[mp]) for mp in range(nmp)])
    run_counts = running.counts()
    # running (region, template id) -> (mp, region index, packed key) of this library
    mp_of = {(mname[mp], pname[mp]): mp for mp in range(nmp)}
    rank_of = {c.name: r for r, c in enumerate(prob.cfg_by_rank)}
    reg_of = {r: i for i, r in enumerate(regions)}
    rmp, rreg, rkey = [], [], []
    for (r, tid), n in run_counts.items():
        if n <= 0 or r not in reg_of:
            continue
        model, phase, combo = tid.split("|", 2)
        mp = mp_of.get((model, phase))
        try:
            toks = [t.rsplit("*", 1) for t in combo.split("+")]
            key = 0
            for name, cnt in toks:
                key = (key << 9) | ((rank_of[name] + 1) << 3) | int(cnt)
            key <<= 9 * (_native.MAX_NODES - len(toks))
        except (KeyError, ValueError):
            continue
        if mp is not None:
            rmp.append(mp)
            rreg.append(reg_of[r])
            rkey.append(key)
    vars_, pruned, best = prob.h.allocation_model(pm, av, dem, order, prune_ratio, rmp, rreg, rkey)

    # ---- host: the reference's MilpModel in its insertion order ------------------
    ranks, cnts = _tokens(vars_["combo_key"])
    names_by_rank = [c.name for c in prob.cfg_by_rank]
    cidx_by_rank = np.array([cfgs.index(c) for c in prob.cfg_by_rank], dtype=np.int64)
    combo_cache: dict = {}
    m = MilpModel(name="allocation")
    var_map, prices = {}, {}
    mps = vars_["mp"].tolist()
    regs = vars_["region"].tolist()
    keys = vars_["combo_key"].tolist()
    ubs = vars_["ub"].tolist()
    pv = vars_["price_usd_h"].tolist()
    tv = vars_["throughput_tps"].tolist()
    rk_l, ck_l = ranks.tolist(), cnts.tolist()
    vids = []
    rows: dict = {}
    demand_rows: dict = {}
    for mp in order:
        if dem[mp] > 0 and math.isfinite(best[mp]):
            demand_rows[(mname[mp], pname[mp])] = {}
    for i in range(len(keys)):
        key = keys[i]
        cs = combo_cache.get(key)
        if cs is None:
            cs = combo_cache[key] = "+".join(f"{names_by_rank[r]}*{c}" for r, c in zip(rk_l[i], ck_l[i]) if c)
        mp = mps[i]
        r = regions[regs[i]]
        tid = f"{mname[mp]}|{pname[mp]}|{cs}"
        vid = f"nu[{r}][{tid}]"
        m.add_var(vid, INTEGER, ub=float(ubs[i]))
        var_map[vid] = (r, tid)
        prices[(r, tid)] = pv[i]
        demand_rows[(mname[mp], pname[mp])][vid] = tv[i]
        for rr_, c in zip(rk_l[i], ck_l[i]):
            if c:
                rows.setdefault((r, names_by_rank[rr_]), {})[vid] = float(c)
        vids.append(vid)
    for (r, cname), coeffs in sorted(rows.items()):
        m.add_constraint(f"cap[{r}][{cname}]", coeffs, LE, float(market.available(r, cname)))
    for (model, phase), row in sorted(demand_rows.items()):
        m.add_constraint(f"demand[{model}][{phase}]", row, GE, _demand_of(demand, model, phase))
    objective = {vid: prices[var_map[vid]] for vid in vids}
    if k_init > 0:
        for vid in vids:
            r, tid = var_map[vid]
            p = prices[(r, tid)]
            iid = f"init[{r}][{tid}]"
            m.add_var(iid, CONTINUOUS)
            nu_prev = run_counts.get((r, tid), 0)
            m.add_constraint(f"pen[{r}][{tid}]", {iid: 1.0, vid: -p * k_init}, GE, -p * k_init * nu_prev)
            objective[iid] = 1.0
    m.set_objective(objective, "min")
    rates = getattr(demand, "rates", demand)
    uncovered = sorted(k for k in rates if rates[k] > 0 and not demand_rows.get(k))

    # ---- CSR view of the capacity rows (stable: variable order within a row) --------
    row_keys = sorted(rows)
    ridx = {rc: i for i, rc in enumerate(row_keys)}
    nz_var, nz_row, nz_val = [], [], []
    cfg_of_rank = cidx_by_rank
    for i in range(len(keys)):
        for rr_, c in zip(rk_l[i], ck_l[i]):
            if c:
                nz_var.append(i)
                nz_row.append(ridx[(regions[regs[i]], cfgs[cfg_of_rank[rr_]].name)])
                nz_val.append(float(c))
    nz_row = np.asarray(nz_row, dtype=np.int64)
    perm = np.argsort(nz_row, kind="stable")
    csr = AllocationCSR(mp=vars_["mp"].copy(), region=vars_["region"].copy(), combo_key=vars_["combo_key"].copy(),
                        ub=vars_["ub"].copy(), price=vars_["price_usd_h"].copy(),
                        throughput=vars_["throughput_tps"].copy(), cap_rows=row_keys,
                        cap_rhs=np.array([float(market.available(r, c)) for r, c in row_keys]),
                        cap_ptr=np.concatenate([[0], np.cumsum(np.bincount(nz_row, minlength=len(row_keys)))]),
                        cap_idx=np.asarray(nz_var, dtype=np.int64)[perm],
                        cap_val=np.asarray(nz_val)[perm])
    return AllocationProblem(
        milp=m, var_map=var_map, prices=prices, demand=demand, market=market, library=library,
        running_counts=run_counts, k_init=k_init,
        meta={"pruned_vars": int(pruned), "uncovered_demands": uncovered,
              "num_vars": len(m.variables), "num_constraints": len(m.constraints)},
        csr=csr)


__all__ = ["AllocationCSR", "AllocationProblem", "Constraint", "DemandSpec", "InstanceInfo", "MarketState",
           "MilpModel", "MilpVar", "RunningState", "build_allocation_model"]
