"""B200-native stage-1 Serving-Template generator for Coral (arXiv 2605.04357).

Drop-in for the reference's candidate generator (hetserve.templates.build_library):
same spec tables in, same template objects out, plus the per-(model, phase, region)
throughput-vs-cost frontier that feeds the unchanged stage-2 MILP. All computation
runs in libcoral_s1.so (hand-written sm_100a CUDA behind a C ABI, include/coral_s1.h).
"""

from .frontier import FrontierEntry, FrontierSession, TemplateFrontier, build_frontier
from .kernels import NEG_INF, placement_search, placement_search_batch
from .library import (GenContext, LibraryCaps, LibraryGenError, Stage1Problem, TemplateLibrary,
                      build_library, enumerate_combos, stage_budget_s, throughput_table)
from .roofline import (node_max_throughput, planned_batch, planned_batch_and_tput,
                       recompute_throughput, stage_node_weights)
from .specs import (DECODE, PHASES, PREFILL, DomainError, GpuSpec, ModelSpec, NodeComboKey,
                    NodeConfig, PerfParams, Placement, ProfileTable, Region, ServingTemplate,
                    SloSpec, combo_key)

__version__ = "0.1.0"
