"""Spec tables and the BASELINE.json workloads (configs c1-c5) for stage 1.

The GPU/model/SLO numbers are the reference's datasheet tables
(/root/reference/pkg/src/hetserve/catalog.py:15-53, Table 1 of the paper); config
lists, region price factors and the workload-average perf parameters follow
catalog.py:55-114. Scenario builders return only what stage 1 consumes
(SURVEY.md 8d): configs, models, SLOs, caps, the generation context and the
per-region prices the frontier is priced with.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .specs import GpuSpec, ModelSpec, NodeConfig, PerfParams, Region, SloSpec

GPU_CATALOG = {g.name: g for g in (
    GpuSpec("H100", mem_gb=80, bw_tbps=3.35, tflops=989, rel_cost=7.6),
    GpuSpec("A100", mem_gb=80, bw_tbps=2.04, tflops=312, rel_cost=3.5),
    GpuSpec("L40S", mem_gb=48, bw_tbps=0.86, tflops=362, rel_cost=2.2),
    GpuSpec("L4", mem_gb=24, bw_tbps=0.30, tflops=121, rel_cost=1.0),
    GpuSpec("A10G", mem_gb=24, bw_tbps=0.60, tflops=70, rel_cost=1.2),
)}

MODEL_CATALOG = {m.name: m for m in (
    ModelSpec("phi4-14b", 40, 14.7, 14.7, 5120, kv_bytes_per_token_per_layer=4096),
    ModelSpec("gpt-oss-20b", 24, 20.9, 3.6, 2880, kv_bytes_per_token_per_layer=2048,
              is_moe=True, is_hybrid_attn=True),
    ModelSpec("qwen3-32b", 64, 32.8, 32.8, 5120, kv_bytes_per_token_per_layer=4096),
    ModelSpec("llama3-70b", 80, 70.6, 70.6, 8192, kv_bytes_per_token_per_layer=4096),
    ModelSpec("gpt-oss-120b", 36, 116.8, 5.1, 2880, kv_bytes_per_token_per_layer=2048,
              is_moe=True, is_hybrid_attn=True),
    ModelSpec("qwen3-235b", 94, 235.0, 22.0, 4096, kv_bytes_per_token_per_layer=2048,
              is_moe=True),
    # BASELINE config 1
    ModelSpec("llama3-8b", 32, 8.03, 8.03, 4096, kv_bytes_per_token_per_layer=4096),
)}

SLO_CATALOG = {
    "phi4-14b": SloSpec(1200, 60),
    "gpt-oss-20b": SloSpec(900, 30),
    "qwen3-32b": SloSpec(1600, 100),
    "llama3-70b": SloSpec(1500, 80),
    "gpt-oss-120b": SloSpec(1000, 40),
    "qwen3-235b": SloSpec(1800, 120),
    "llama3-8b": SloSpec(1500, 80),
}

CORE_MODELS = ["qwen3-32b", "gpt-oss-20b", "phi4-14b"]
CORE_GPUS = ["L40S", "L4", "A10G"]
EXTENDED_MODELS = CORE_MODELS + ["qwen3-235b", "gpt-oss-120b", "llama3-70b"]
EXTENDED_GPUS = CORE_GPUS + ["H100", "A100"]
GPU_COUNTS = (1, 2, 4, 8)
REGION_PRICE_FACTOR = {"us-east": 1.0, "ap-northeast": 1.08, "us-central": 0.95}


def make_configs(gpus, counts=GPU_COUNTS) -> list:
    """Every (GPU, count) node config, sorted by name (catalog.py:65-72)."""
    out = []
    for gname in gpus:
        gpu = gname if isinstance(gname, GpuSpec) else GPU_CATALOG[gname]
        link = 600.0 if gpu.mem_gb >= 80 else 64.0
        out.extend(NodeConfig(gpu, n, link) for n in counts)
    return sorted(out, key=lambda c: c.name)


def make_prices(configs, regions, base_usd: float = 1.0) -> dict:
    """(region, config) -> USD/h, rounded to 4 decimals (catalog.py:75-83)."""
    return {(r.name, c.name): round(base_usd * c.gpu.rel_cost * c.gpu_count
                                    * REGION_PRICE_FACTOR.get(r.name, 1.0), 4)
            for r in regions for c in configs}


def perf_for_workload(n_models: int = 1, prompt_median=1024.0, prompt_sigma=0.5,
                      output_median=256.0, output_sigma=0.5,
                      slo_budget_frac: float = 0.55) -> PerfParams:
    """Log-normal trace means as the planner's workload averages (catalog.py:92-114).

    The reference averages per-model means of identical synthetic specs, so the
    model count only matters through the float summation order.
    """
    prompt = sum(prompt_median * math.exp(prompt_sigma ** 2 / 2) for _ in range(n_models)) / n_models
    output = sum(output_median * math.exp(output_sigma ** 2 / 2) for _ in range(n_models)) / n_models
    return PerfParams(avg_prompt_tokens=round(prompt, 1), avg_output_tokens=round(output, 1),
                      avg_ctx_tokens=round(prompt + output / 2, 1),
                      slo_budget_frac=slo_budget_frac)


@dataclass
class Stage1Workload:
    """Everything stage 1 reads for one BASELINE config."""

    name: str
    configs: list
    models: list
    slos: dict
    n_max: int = 6
    rho: float = 12.0
    perf: PerfParams = field(default_factory=PerfParams)
    granularity: int = 0
    regions: list = field(default_factory=list)
    prices: dict = field(default_factory=dict)

    def caps(self):
        from .library import LibraryCaps
        return LibraryCaps(self.n_max, self.rho)

    def ctx(self):
        from .library import GenContext
        return GenContext(perf=self.perf, granularity=self.granularity)


def _catalog_workload(name, models, gpus, regions, granularity=0) -> Stage1Workload:
    configs = make_configs(gpus)
    regs = [Region(r) for r in regions]
    return Stage1Workload(
        name=name, configs=configs, models=[MODEL_CATALOG[m] for m in models],
        slos={m: SLO_CATALOG[m] for m in models},
        perf=perf_for_workload(len(models)), granularity=granularity,
        regions=regs, prices=make_prices(configs, regs))


def core_workload() -> Stage1Workload:
    """catalog.core_scenario(): 3 models x 12 configs x 2 regions (catalog.py:117-140)."""
    return _catalog_workload("core", CORE_MODELS, CORE_GPUS, ["us-east", "ap-northeast"])


def extended_workload() -> Stage1Workload:
    """BASELINE config 2 = catalog.extended_scenario(): 6 x 20 x 3 (catalog.py:143-165)."""
    return _catalog_workload("extended", EXTENDED_MODELS, EXTENDED_GPUS,
                             ["us-east", "ap-northeast", "us-central"])


def c1_workload() -> Stage1Workload:
    """BASELINE config 1: llama3-8b x {A100, L4} x {1,2,4,8}, one region."""
    return _catalog_workload("c1", ["llama3-8b"], ["A100", "L4"], ["us-east"])


def c3_workload() -> Stage1Workload:
    """BASELINE config 3: llama3-70b on the 20 extended configs at granularity 1 (Lu = 80).

    perf comes from the extended scenario (6-model averages) as in SURVEY.md 8d.
    """
    w = extended_workload()
    return Stage1Workload(name="c3", configs=w.configs, models=[MODEL_CATALOG["llama3-70b"]],
                          slos={"llama3-70b": SLO_CATALOG["llama3-70b"]}, perf=w.perf,
                          granularity=1, regions=w.regions, prices=w.prices)


def c5_workload(seed: int = 0, n_models: int = 50) -> Stage1Workload:
    """BASELINE config 5: synthetic 50 models x 40 configs.

    40 configs = 10 GPU types x {1,2,4,8}: the 5 catalog GPUs plus 5 variants with
    mem in {16, 32, 40, 64, 96} GiB and bw/tflops/rel_cost jittered +-30%.
    """
    rng = np.random.default_rng(seed)
    gpus = list(GPU_CATALOG.values())
    for i, mem in enumerate((16, 32, 40, 64, 96)):
        base = gpus[i]
        jit = rng.uniform(0.7, 1.3, size=3)
        gpus.append(GpuSpec(f"X{i}{base.name}", float(mem), round(base.bw_tbps * jit[0], 3),
                            round(base.tflops * jit[1], 1), round(base.rel_cost * jit[2], 3)))
    configs = make_configs(gpus)
    models, slos = [], {}
    for k in range(n_models):
        L = int(rng.choice([24, 32, 36, 40, 48, 64, 80, 94]))
        total = float(round(math.exp(rng.uniform(math.log(7), math.log(400))), 2))
        moe = bool(rng.random() < 0.3)
        active = float(round(total * rng.uniform(0.05, 0.25), 2)) if moe else total
        hidden = int(rng.choice([2880, 4096, 5120, 8192]))
        kv = float(rng.choice([2048, 4096]))
        name = f"syn{k:02d}"
        models.append(ModelSpec(name, L, total, active, hidden,
                                kv_bytes_per_token_per_layer=kv, is_moe=moe))
        slos[name] = SloSpec(float(round(rng.uniform(800, 2000))), float(round(rng.uniform(30, 120))))
    regs = [Region("us-east"), Region("ap-northeast"), Region("us-central")]
    return Stage1Workload(name="c5", configs=configs, models=models, slos=slos,
                          perf=perf_for_workload(n_models), regions=regs,
                          prices=make_prices(configs, regs))


def c4_epoch_prices(w: Stage1Workload, epoch: int) -> dict:
    """BASELINE config 4 price path: per (region, config) the base
    price times exp(0.1 z), z ~ N(0, 1) from default_rng(1000 + epoch), drawn in
    (region, config) name order."""
    rng = np.random.default_rng(1000 + epoch)
    out = {}
    for r in sorted(w.regions, key=lambda r: r.name):
        for c in sorted(w.configs, key=lambda c: c.name):
            base = w.prices[(r.name, c.name)]
            out[(r.name, c.name)] = base * math.exp(0.1 * rng.standard_normal())
    return out


WORKLOADS = {"c1": c1_workload, "core": core_workload, "extended": extended_workload,
             "c2": extended_workload, "c3": c3_workload, "c5": c5_workload}
