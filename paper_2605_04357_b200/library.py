"""Drop-in stage-1 generator: `build_library` and friends on the B200.

Mirrors the reference's public operator surface of
/root/reference/pkg/src/hetserve/templates.py:
  LibraryCaps (:38-49), GenContext (:52-65), LibraryGenError (:34-35),
  stage_budget_s (:68-80), throughput_table (:83-96), enumerate_combos (:99-113),
  TemplateLibrary (:329-401) and build_library (:417-505),
with the same argument meaning, ordering and error behaviour. Every number is
computed by the CUDA library (libcoral_s1.so) through the C ABI; this module only
packs spec tables into arrays and turns device records into template objects.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .specs import (PHASES, PREFILL, DomainError, GpuSpec, NodeComboKey, NodeConfig,
                    PerfParams, Placement, ServingTemplate, SloSpec)

LIBRARY_FORMAT = "hetserve-template-library"
LIBRARY_VERSION = 1
NEG_INF = _native.NEG_INF


class _no_gc:
    """Pause the cyclic GC while building many small immutable objects (the collector
    otherwise re-traverses the growing young generation hundreds of times)."""

    def __enter__(self):
        import gc
        self._was = gc.isenabled()
        gc.disable()

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()


class LibraryGenError(RuntimeError):
    """A (model, phase) pair yielded no feasible template at all (templates.py:34-35)."""


@dataclass(frozen=True)
class LibraryCaps:
    """Enumeration caps: max nodes per combo, memory cap as a model-size multiple."""

    n_max: int = 6
    rho: float = 12.0

    def __post_init__(self):
        if self.n_max < 1:
            raise DomainError("n_max must be >= 1")
        if self.rho <= 1:
            raise DomainError("rho must be > 1")


@dataclass(frozen=True)
class GenContext:
    """Generation context (templates.py:52-65)."""

    perf: PerfParams = field(default_factory=PerfParams)
    profile: object = None
    net_gbps: float = 12.5
    net_latency_ms: float = 0.5
    granularity: int = 0

    def layer_granularity(self, model) -> int:
        if self.granularity:
            return self.granularity
        return 2 if model.num_layers >= 80 and model.num_layers % 2 == 0 else 1


# ---------------------------------------------------------------------------------
# spec tables -> C ABI arrays
# ---------------------------------------------------------------------------------

def str_ranks(names) -> np.ndarray:
    """Rank of each name under (name + '*') code-point order.

    str(NodeComboKey) joins "name*count" tokens with '+'; comparing two such
    strings token by token compares names as if terminated by '*', and counts as
    digit strings. Packing (rank, count) tokens into a u64 therefore sorts exactly
    like the reference's str order (templates.py:112, 340).
    """
    order = sorted(range(len(names)), key=lambda i: names[i] + "*")
    ranks = np.zeros(len(names), dtype=np.int32)
    for r, i in enumerate(order):
        ranks[i] = r
    return ranks


def _pack_problem(configs, models, slos, phases, caps, ctx):
    names = [c.name for c in configs]
    if len(set(names)) != len(names):
        raise DomainError("two distinct configs share a name")
    mnames = [m.name for m in models]
    if len(set(mnames)) != len(mnames):
        raise DomainError("duplicate model names")
    for ph in phases:
        if ph not in _native.PHASE_CODE:
            raise DomainError(f"phase must be one of {PHASES}")
    perf = ctx.perf
    arrays = {
        "cfg_gpu_count": [c.gpu_count for c in configs],
        "cfg_mem_gb": [c.gpu.mem_gb for c in configs],
        "cfg_bw_tbps": [c.gpu.bw_tbps for c in configs],
        "cfg_tflops": [c.gpu.tflops for c in configs],
        "cfg_str_rank": str_ranks(names),
        "mdl_num_layers": [m.num_layers for m in models],
        "mdl_granularity": [ctx.layer_granularity(m) for m in models],
        "mdl_params_total_b": [m.params_total_b for m in models],
        "mdl_params_active_b": [m.params_active_b for m in models],
        "mdl_hidden_size": [m.hidden_size for m in models],
        "mdl_bytes_per_param": [m.bytes_per_param for m in models],
        "mdl_kv_bytes": [m.kv_bytes_per_token_per_layer for m in models],
        "slo_prefill_ms": [slos[m.name].prefill_ms for m in models],
        "slo_decode_ms": [slos[m.name].decode_ms for m in models],
        "phases": [_native.PHASE_CODE[p] for p in phases],
    }
    prof = {k: [] for k in ("prof_model", "prof_phase", "prof_cfg", "prof_j", "prof_bucket", "prof_tps")}
    if ctx.profile is not None:
        cidx = {n: i for i, n in enumerate(names)}
        midx = {n: i for i, n in enumerate(mnames)}
        for (cfg, mdl, phase, j, bucket), tps in ctx.profile.entries.items():
            if cfg in cidx and mdl in midx and phase in _native.PHASE_CODE:
                for key, v in (("prof_model", midx[mdl]), ("prof_phase", _native.PHASE_CODE[phase]),
                               ("prof_cfg", cidx[cfg]), ("prof_j", j), ("prof_bucket", bucket),
                               ("prof_tps", tps)):
                    prof[key].append(v)
    arrays.update(prof)
    scalars = dict(num_configs=len(configs), num_models=len(models), num_phases=len(phases),
                   mfu=perf.mfu, mbu=perf.mbu, net_eff=perf.net_eff,
                   fixed_overhead_ms=perf.fixed_overhead_ms,
                   avg_prompt_tokens=perf.avg_prompt_tokens, avg_ctx_tokens=perf.avg_ctx_tokens,
                   slo_budget_frac=perf.slo_budget_frac, net_gbps=ctx.net_gbps,
                   net_latency_ms=ctx.net_latency_ms, n_max=caps.n_max, rho=float(caps.rho),
                   num_profile=len(prof["prof_tps"]))
    return arrays, scalars


def decode_key(key: int):
    """Packed combo key -> [(str rank, count)] tokens in combo (name) order."""
    out = []
    for t in range(_native.MAX_NODES):
        tok = (int(key) >> (9 * (_native.MAX_NODES - 1 - t))) & 511
        if not tok:
            break
        out.append(((tok >> 3) - 1, tok & 7))
    return out


class Stage1Problem:
    """One stage-1 solve on one device: spec tables in, device records out.

    The problem leases its own device handle (_native.acquire) for its lifetime, so
    other solves or T-hat queries issued while it is alive (a FrontierSession between
    epochs, a lazy library before save) never touch its device state. close() (or
    garbage collection) returns the handle to the per-device pool."""

    def __init__(self, configs, models, slos, caps, ctx=None, phases=PHASES, device=None):
        self.ctx = ctx or GenContext()
        self.caps = caps
        self.configs = sorted(configs, key=lambda c: c.name)   # templates.py:429
        self.models = list(models)
        self.slos = slos
        self.phases = tuple(phases)
        self.arrays, self.scalars = _pack_problem(self.configs, self.models, slos, self.phases,
                                                  caps, self.ctx)
        rank = self.arrays["cfg_str_rank"]
        self.cfg_by_rank = [None] * len(self.configs)
        for i, r in enumerate(rank):
            self.cfg_by_rank[r] = self.configs[i]
        self.h = None
        self.h = _native.acquire(device)
        self.h.set_problem(self.arrays, self.scalars)
        self.counts = None
        self.cand_off = None

    def signature(self) -> str:
        """Digest of the packed spec tables (the problem's identity for memoised plans)."""
        if getattr(self, "_sig", None) is None:
            import hashlib
            d = hashlib.sha1()
            for k in sorted(self.arrays):
                d.update(k.encode())
                d.update(np.ascontiguousarray(self.arrays[k]).tobytes())
            d.update(repr(sorted(self.scalars.items())).encode())
            self._sig = d.hexdigest()
        return self._sig

    def close(self) -> None:
        h, self.h = self.h, None
        if h is not None:
            _native.release(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    # -- device stages ------------------------------------------------------------
    def run(self, shard=None):
        """T-hat tables, enumeration, then the evaluator over all candidates, or
        over the `shard` = (lo, hi) range of the global candidate list."""
        h = self.h
        h.tables()
        h.enumerate()
        self.counts = h.num_combos()
        NP = len(self.phases)
        self.cand_off = np.zeros(len(self.models) * NP + 1, dtype=np.int64)
        for mp in range(len(self.models) * NP):
            self.cand_off[mp + 1] = self.cand_off[mp] + self.counts[mp // NP]
        lo, hi = (0, -1) if shard is None else shard
        h.evaluate(lo, hi)
        return self

    @property
    def num_candidates(self) -> int:
        return int(self.cand_off[-1])

    def keys(self, m: int) -> np.ndarray:
        return self.h.get_combos(m, False, int(self.counts[m]))

    def records(self, mp: int) -> np.ndarray:
        return self.h.get_records(mp, int(self.counts[mp // len(self.phases)]))

    def check_feasible(self):
        """templates.py:499-502: LibraryGenError when a (model, phase) has no feasible
        template (counted on the device; CORAL_S1_ENOTEMPLATE)."""
        counts, bad = self.h.feasible_counts()
        if bad:
            NP = len(self.phases)
            missing = [(self.models[mp // NP].name, self.phases[mp % NP])
                       for mp in range(len(counts)) if counts[mp] == 0]
            raise LibraryGenError(f"no feasible template for: {sorted(missing)}")
        return counts

    # -- host materialisation -------------------------------------------------------
    def combo_objects(self, keys: np.ndarray) -> list:
        """Packed keys -> NodeComboKey objects (token decode vectorised in numpy)."""
        keys = np.asarray(keys, dtype=np.uint64)
        shifts = np.array([9 * (_native.MAX_NODES - 1 - t) for t in range(_native.MAX_NODES)],
                          dtype=np.uint64)
        toks = ((keys[:, None] >> shifts[None, :]) & np.uint64(511)).astype(np.int64)
        ranks = ((toks >> 3) - 1).tolist()
        cnts = (toks & 7).tolist()
        cbr = self.cfg_by_rank
        new = object.__new__
        out = []
        for rk, ct in zip(ranks, cnts):
            obj = new(NodeComboKey)
            obj.__dict__["items"] = tuple((cbr[r], c) for r, c in zip(rk, ct) if c)
            out.append(obj)
        return out

    def make_template(self, model, phase, combo, rec) -> ServingTemplate:
        S = int(rec["num_stages"])
        nn = int(rec["num_nodes"])
        pl = object.__new__(Placement)
        pl.__dict__.update(num_stages=S,
                           layers_per_stage=tuple(int(x) for x in rec["layers_per_stage"][:S]),
                           stage_of_node=tuple(int(x) for x in rec["stage_of_node"][:nn]))
        t = object.__new__(ServingTemplate)
        t.__dict__.update(model=model.name, phase=phase, slo=self.slos[model.name], combo=combo,
                          placement=pl, throughput_tps=float(rec["throughput_tps"]))
        return t

    def library_entries(self):
        """All feasible templates in TemplateLibrary order (templates.py:340)."""
        with _no_gc():
            return self._library_entries()

    def _library_entries(self):
        from ._lib import _materialize
        NP = len(self.phases)
        nmp = len(self.models) * NP
        self.check_feasible()
        recs_by_mp = [self.records(mp) for mp in range(nmp)]
        order = sorted(range(nmp), key=lambda mp: (self.models[mp // NP].name, self.phases[mp % NP]))
        caches, keys = {}, {}
        entries = []
        for mp in order:
            m, ph = mp // NP, self.phases[mp % NP]
            model = self.models[m]
            g = self.ctx.layer_granularity(model)
            recs = recs_by_mp[mp]
            if model.num_layers % g and np.any(recs["num_stages"] > 0):
                raise DomainError(f"stage layers sum to {(model.num_layers // g) * g}, "
                                  f"model has {model.num_layers}")
            if m not in keys:
                keys[m] = np.ascontiguousarray(self.keys(m), dtype=np.uint64)
                caches[m] = {}
            entries += _materialize.build_templates(
                np.ascontiguousarray(recs).tobytes(), keys[m].tobytes(), list(self.cfg_by_rank),
                model.name, ph, self.slos[model.name], caches[m], ServingTemplate, Placement, NodeComboKey)
        return entries


# ---------------------------------------------------------------------------------
# TemplateLibrary (templates.py:329-401)
# ---------------------------------------------------------------------------------

def _config_meta(cfg) -> dict:
    return {"gpu": {"name": cfg.gpu.name, "mem_gb": cfg.gpu.mem_gb, "bw_tbps": cfg.gpu.bw_tbps,
                    "tflops": cfg.gpu.tflops, "rel_cost": cfg.gpu.rel_cost},
            "gpu_count": cfg.gpu_count,
            "intra_node_interconnect_gbps": cfg.intra_node_interconnect_gbps}


def _config_from_meta(spec: dict) -> NodeConfig:
    return NodeConfig(GpuSpec(**spec["gpu"]), spec["gpu_count"],
                      spec["intra_node_interconnect_gbps"])


def library_meta(configs, models, slos, caps, ctx) -> dict:
    """Library header (templates.py:528-540)."""
    return {
        "format": LIBRARY_FORMAT,
        "version": LIBRARY_VERSION,
        "caps": {"n_max": caps.n_max, "rho": caps.rho},
        "perf_digest": ctx.perf.digest(),
        "perf": dict(ctx.perf.__dict__),
        "net": {"gbps": ctx.net_gbps, "latency_ms": ctx.net_latency_ms},
        "granularity": {m.name: ctx.layer_granularity(m) for m in models},
        "configs": {c.name: _config_meta(c) for c in configs},
        "models": {m.name: dict(m.__dict__) for m in models},
        "slos": {name: [s.prefill_ms, s.decode_ms] for name, s in slos.items()},
    }


class TemplateLibrary:
    """Template collection indexed by (model, phase) and template id.

    Same interface as the reference (templates.py:329-401). Entries are kept in
    (model, phase, str(combo)) order; the id index is built on first use.
    """

    def __init__(self, entries=None, meta=None, _presorted: bool = False):
        self.entries = list(entries or [])
        self.meta = dict(meta or {})
        self._by_mp: dict = {}
        self._by_id = None
        self.reindex(_presorted)

    def reindex(self, _presorted: bool = False) -> None:
        if not _presorted:
            self.entries.sort(key=lambda t: (t.model, t.phase, str(t.combo)))
        self._by_mp = {}
        for t in self.entries:
            self._by_mp.setdefault((t.model, t.phase), []).append(t)
        self._by_id = None
        if not _presorted:
            self._index_ids()

    def _index_ids(self) -> dict:
        if self._by_id is None:
            by_id = {}
            for t in self.entries:
                tid = t.template_id
                if tid in by_id:
                    raise DomainError(f"duplicate template {tid}")
                by_id[tid] = t
            self._by_id = by_id
        return self._by_id

    def templates_for(self, model: str, phase: str) -> list:
        return self._by_mp.get((model, phase), [])

    def get(self, template_id: str) -> ServingTemplate:
        return self._index_ids()[template_id]

    def __len__(self) -> int:
        return len(self.entries)

    def model_phases(self) -> list:
        return sorted(self._by_mp)

    def counts_by_model_phase(self) -> dict:
        return {k: len(v) for k, v in sorted(self._by_mp.items())}

    def save(self, path: str) -> None:
        dumps = json.dumps
        with open(path, "w") as fh:
            fh.write(dumps(self.meta, sort_keys=True) + "\n")
            for t in self.entries:
                fh.write(dumps({
                    "model": t.model, "phase": t.phase,
                    "slo": [t.slo.prefill_ms, t.slo.decode_ms],
                    "combo": [[c.name, n] for c, n in t.combo.items],
                    "num_stages": t.placement.num_stages,
                    "layers_per_stage": list(t.placement.layers_per_stage),
                    "stage_of_node": list(t.placement.stage_of_node),
                    "throughput_tps": t.throughput_tps,
                }, sort_keys=True) + "\n")

    @classmethod
    def load(cls, path: str) -> "TemplateLibrary":
        """Read a library written by save (templates.py:379-401). The JSON-lines parse
        and object construction run in the CPython extension (csrc/materialize.c)."""
        from ._lib import _materialize
        with open(path) as fh:
            header = json.loads(fh.readline())
        if header.get("format") != LIBRARY_FORMAT:
            raise DomainError(f"{path} is not a template library file")
        configs = {name: _config_from_meta(spec) for name, spec in header["configs"].items()}
        with _no_gc():
            _, entries, in_order = _materialize.load_library(path, configs, ServingTemplate, Placement,
                                                             NodeComboKey, SloSpec)
        return cls(entries=entries, meta=header, _presorted=bool(in_order))


# ---------------------------------------------------------------------------------
# public operators
# ---------------------------------------------------------------------------------

def build_library(configs, models, slos, caps, ctx=None, workers: int = 1,
                  method: str = "search", phases=PHASES, lazy: bool = False):
    """Generate the full template library on the GPU (templates.py:417-505).

    `workers` is accepted for signature compatibility and ignored (the device is the
    parallelism). `method` must be "search": the reference's ILP path
    (templates.py:455-456) is a test oracle, not part of the stage-1 hot path.
    `lazy=True` returns a LazyTemplateLibrary (same interface, objects built on
    access, native byte-identical save).
    """
    del workers
    ctx = ctx or GenContext()
    if method != "search":
        raise DomainError("the GPU stage-1 path implements method='search' only")
    t0 = time.monotonic()
    configs_sorted = sorted(configs, key=lambda c: c.name)
    meta = library_meta(configs_sorted, models, slos, caps, ctx)
    del t0
    if not models:
        return TemplateLibrary(entries=[], meta=meta)
    prob = Stage1Problem(configs, models, slos, caps, ctx, phases)
    prob.run()
    if lazy:  # array-backed: objects on access, native save
        return LazyTemplateLibrary(prob, meta)
    return TemplateLibrary(entries=prob.library_entries(), meta=meta, _presorted=True)


def enumerate_combos(configs, model, caps) -> list:
    """Node multisets of 1..n_max nodes inside the memory window, in the reference's
    (num_nodes, str) order (templates.py:99-113). Runs on the GPU."""
    ctx = GenContext()
    prob = Stage1Problem(configs, [model], {model.name: SloSpec(1.0, 1.0)}, caps, ctx, (PREFILL,))
    prob.h.enumerate()
    n = int(prob.h.num_combos()[0])
    keys = prob.h.get_combos(0, True, n)
    return prob.combo_objects(keys)


def _tables_for(h, configs, model, slo, phase, S, ctx):
    caps = LibraryCaps(n_max=max(1, S), rho=2.0)
    arrays, scalars = _pack_problem(list(configs), [model], {model.name: slo}, (phase,), caps, ctx)
    h.set_problem(arrays, scalars)
    h.tables()


def throughput_table(configs, model, slo, phase, S, ctx) -> np.ndarray:
    """T-hat rows per config (given order) for every layer-unit count at stage
    count S (templates.py:83-96), computed on the GPU."""
    g = ctx.layer_granularity(model)
    lsteps = model.num_layers // g
    if S < 1:
        raise DomainError("S must be >= 1")
    if S > min(_native.MAX_NODES, model.num_layers):
        raise DomainError(f"GPU T-hat tables cover S <= min({_native.MAX_NODES}, num_layers)")
    with _native.lease() as h:
        _tables_for(h, configs, model, slo, phase, S, ctx)
        tab, offs, ls = h.get_tables()
    K = len(configs)
    block = tab[offs[0]:offs[1]].reshape(-1, K, lsteps)
    return block[S - 1].copy()


def stage_budget_s(model, slo, phase, S, ctx) -> float:
    """Per-stage latency budget (templates.py:68-80), evaluated on the GPU."""
    if not 1 <= S <= min(_native.MAX_NODES, model.num_layers):
        raise DomainError(f"GPU stage budgets cover 1 <= S <= min({_native.MAX_NODES}, num_layers)")
    cfg = NodeConfig(GpuSpec("probe", 1.0, 1.0, 1.0, 1.0), 1)
    with _native.lease() as h:
        _tables_for(h, [cfg], model, slo, phase, S, ctx)
        return float(h.get_budgets()[0, S - 1])


class LazyTemplateLibrary:
    """Array-backed TemplateLibrary over one device solve.

    Same interface as TemplateLibrary (templates.py:329-401): entries, meta,
    templates_for, get, model_phases, counts_by_model_phase, __len__, save. Template
    objects are built per (model, phase) on first access; save() streams the records
    straight from device memory through the native writer, byte-identical to the
    reference's TemplateLibrary.save.
    """

    def __init__(self, prob: "Stage1Problem", meta: dict):
        self._prob = prob
        self.meta = meta
        NP = len(prob.phases)
        self._mp_of = {(m.name, ph): mi * NP + pi for mi, m in enumerate(prob.models)
                       for pi, ph in enumerate(prob.phases)}
        prob.check_feasible()
        self._recs = {mp: prob.records(mp) for mp in self._mp_of.values()}
        self._feas = {mp: np.nonzero(r["num_stages"] > 0)[0] for mp, r in self._recs.items()}
        for (mname, ph), mp in self._mp_of.items():
            model = prob.models[mp // NP]
            g = prob.ctx.layer_granularity(model)
            if model.num_layers % g:
                raise DomainError(f"stage layers sum to {(model.num_layers // g) * g}, "
                                  f"model has {model.num_layers}")
        self._keys = {}
        self._combos = {}
        self._segments = {}
        self._entries = None
        self._rank_of = {c.name: r for r, c in enumerate(prob.cfg_by_rank)}

    def _model_keys(self, m):
        if m not in self._keys:
            self._keys[m] = self._prob.keys(m)
        return self._keys[m]

    def model_phases(self) -> list:
        return sorted(self._mp_of)

    def counts_by_model_phase(self) -> dict:
        return {k: int(len(self._feas[self._mp_of[k]])) for k in self.model_phases()}

    def __len__(self) -> int:
        return int(sum(len(f) for f in self._feas.values()))

    def templates_for(self, model: str, phase: str) -> list:
        key = (model, phase)
        if key not in self._mp_of:
            return []
        if key not in self._segments:
            mp = self._mp_of[key]
            NP = len(self._prob.phases)
            m = mp // NP
            if m not in self._combos:
                self._combos[m] = self._prob.combo_objects(self._model_keys(m))
            combos = self._combos[m]
            recs, feas = self._recs[mp], self._feas[mp]
            mdl = self._prob.models[m]
            self._segments[key] = [self._prob.make_template(mdl, phase, combos[i], recs[i])
                                   for i in feas.tolist()]
        return self._segments[key]

    @property
    def entries(self) -> list:
        if self._entries is None:
            self._entries = [t for k in self.model_phases() for t in self.templates_for(*k)]
        return self._entries

    def get(self, template_id: str) -> ServingTemplate:
        model, phase, combo = template_id.split("|", 2)
        mp = self._mp_of.get((model, phase))
        if mp is None:
            raise KeyError(template_id)
        key = 0
        toks = combo.split("+")
        try:
            for tok in toks:
                name, n = tok.rsplit("*", 1)
                key = (key << 9) | ((self._rank_of[name] + 1) << 3) | int(n)
        except (KeyError, ValueError):
            raise KeyError(template_id) from None
        key <<= 9 * (_native.MAX_NODES - len(toks))
        NP = len(self._prob.phases)
        keys = self._model_keys(mp // NP)
        i = int(np.searchsorted(keys, np.uint64(key)))
        if i >= len(keys) or int(keys[i]) != key or self._recs[mp]["num_stages"][i] == 0:
            raise KeyError(template_id)
        m = mp // NP
        combo_obj = self._prob.combo_objects(keys[i:i + 1])[0]
        return self._prob.make_template(self._prob.models[m], phase, combo_obj, self._recs[mp][i])

    def reindex(self) -> None:
        pass

    def save(self, path: str) -> int:
        """Native JSONL writer; returns the number of templates written."""
        prob = self._prob
        NP = len(prob.phases)
        order = [self._mp_of[k] for k in self.model_phases()]
        header = json.dumps(self.meta, sort_keys=True)
        model_json = [json.dumps(m.name) for m in prob.models]
        phase_json = [json.dumps(p) for p in prob.phases]
        slo_json = [json.dumps([prob.slos[m.name].prefill_ms, prob.slos[m.name].decode_ms])
                    for m in prob.models]
        cfg_json = [json.dumps(c.name) for c in prob.configs]
        del NP
        return prob.h.write_library(path, header, order, model_json, phase_json, slo_json, cfg_json)
