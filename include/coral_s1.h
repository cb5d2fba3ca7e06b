/*
 * coral_s1.h — C ABI of the B200-native stage-1 Serving-Template generator.
 *
 * The hot path replaced is Coral's stage 1 (arXiv 2605.04357), implemented in the
 * reference by `hetserve.templates.build_library`
 * (/root/reference/pkg/src/hetserve/templates.py:417-505). Every entry point below
 * names the reference function whose behaviour it reproduces. All arguments are
 * plain pointers and sizes; no torch types cross this boundary. Device work runs on
 * the stream given to coral_s1_set_stream (default: the legacy stream).
 *
 * Error convention: every call returns an int status.
 *   CORAL_S1_OK (0)              success
 *   CORAL_S1_EINVAL (1)          invalid argument      -> DomainError / ValueError
 *   CORAL_S1_ENOTEMPLATE (2)     a (model, phase) has no feasible template
 *                                                      -> LibraryGenError
 *   CORAL_S1_ECUDA (3)           CUDA failure          -> RuntimeError
 *   CORAL_S1_EUNSUPPORTED (4)    input outside the GPU path's envelope
 *                                (n_max > 7, > 63 configs, > 128 layer units)
 * The message of the last failure on the calling thread is coral_s1_last_error().
 * The library never aborts the process.
 */
#ifndef CORAL_S1_H
#define CORAL_S1_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CORAL_S1_OK 0
#define CORAL_S1_EINVAL 1
#define CORAL_S1_ENOTEMPLATE 2
#define CORAL_S1_ECUDA 3
#define CORAL_S1_EUNSUPPORTED 4

#define CORAL_S1_PHASE_PREFILL 0
#define CORAL_S1_PHASE_DECODE 1

/* Largest envelope of the GPU path. n_max <= 7 (the reference's own acceptance sweep
 * reaches (7, 14), pkg/tests/test_acceptance.py:320-348) keeps every node multiset's
 * sub-multiset lattice within 128 codes (kernels.py:147-150: M = prod(counts+1)) and
 * the packed combo key within 7 tokens x 9 bits = 63 bits. */
#define CORAL_S1_MAX_NODES 7
#define CORAL_S1_MAX_CONFIGS 63
#define CORAL_S1_MAX_LAYER_UNITS 128

typedef struct coral_s1_handle coral_s1_handle;

/* Spec tables in (SoA). Mirrors the reference inputs of build_library
 * (templates.py:417-421): NodeConfig (domain.py:32-50), ModelSpec
 * (domain.py:64-88), SloSpec (domain.py:91-101), PerfParams (perf.py:17-54),
 * GenContext (templates.py:52-65), LibraryCaps (templates.py:38-49), and the
 * optional ProfileTable overrides (perf.py:94-116). */
typedef struct coral_s1_problem {
  /* node configs, sorted by name (templates.py:429) */
  int32_t num_configs;
  const int32_t* cfg_gpu_count;   /* NodeConfig.gpu_count */
  const double* cfg_mem_gb;       /* GpuSpec.mem_gb (GiB per GPU) */
  const double* cfg_bw_tbps;      /* GpuSpec.bw_tbps */
  const double* cfg_tflops;       /* GpuSpec.tflops */
  const int32_t* cfg_str_rank;    /* rank of (name + '*') in code-point order:
                                     makes the packed combo key sort exactly like
                                     str(NodeComboKey) (domain.py:127-129) */
  /* models, in the caller's order */
  int32_t num_models;
  const int32_t* mdl_num_layers;
  const int32_t* mdl_granularity; /* resolved GenContext.layer_granularity */
  const double* mdl_params_total_b;
  const double* mdl_params_active_b;
  const double* mdl_hidden_size;
  const double* mdl_bytes_per_param;
  const double* mdl_kv_bytes;     /* kv_bytes_per_token_per_layer */
  const double* slo_prefill_ms;   /* SloSpec of each model */
  const double* slo_decode_ms;
  /* phases, in the caller's order (templates.py:441) */
  int32_t num_phases;
  const int32_t* phases;          /* CORAL_S1_PHASE_* */
  /* PerfParams */
  double mfu, mbu, net_eff, fixed_overhead_ms;
  double avg_prompt_tokens, avg_ctx_tokens, slo_budget_frac;
  /* GenContext network assumption */
  double net_gbps, net_latency_ms;
  /* LibraryCaps */
  int32_t n_max;
  double rho;
  /* ProfileTable overrides (perf.py:110-116); bucket -1 matches any budget */
  int32_t num_profile;
  const int32_t* prof_model;
  const int32_t* prof_phase;
  const int32_t* prof_cfg;
  const int32_t* prof_j;          /* layers (not units) */
  const int32_t* prof_bucket;     /* integer milliseconds or -1 */
  const double* prof_tps;
} coral_s1_problem;

/* One evaluated candidate (model, phase, combo): the ServingTemplate payload
 * (domain.py:183-202) in canonical placement form (templates.py:209-228).
 * num_stages == 0 means "no feasible template" (templates.py:487-490). */
typedef struct coral_s1_record {
  double throughput_tps;
  uint8_t num_stages;
  uint8_t num_nodes;
  uint16_t layers_per_stage[CORAL_S1_MAX_NODES];
  uint8_t stage_of_node[CORAL_S1_MAX_NODES];
  uint8_t _pad[1]; /* explicit, always zero: records compare bytewise */
} coral_s1_record; /* 32 bytes */

/* One frontier survivor (new output). */
typedef struct coral_s1_frontier_item {
  double price_usd_h;             /* allocation.py:91-98 sequential sum */
  double throughput_tps;
  uint64_t combo_key;             /* packed tokens, str(combo) order */
  int32_t mp;                     /* model * num_phases + phase slot */
  int32_t region;
  coral_s1_record rec;
} coral_s1_frontier_item; /* 64 bytes */

/* One stage-2 allocation variable nu[region][template] (allocation.py:154-163). */
typedef struct coral_s1_alloc_var {
  uint64_t combo_key;             /* template's packed combo key */
  int32_t mp;                     /* model * num_phases + phase slot */
  int32_t region;                 /* index into the caller's region list */
  int64_t ub;                     /* min(availability cap, ceil(demand / T)) >= 1 */
  double price_usd_h;             /* allocation.py:91-98 */
  double throughput_tps;
} coral_s1_alloc_var; /* 40 bytes */

/* ---- lifecycle -------------------------------------------------------- */
int coral_s1_create(int device, coral_s1_handle** out);
int coral_s1_destroy(coral_s1_handle* h);
const char* coral_s1_last_error(void);
int coral_s1_version(void);
int coral_s1_set_stream(coral_s1_handle* h, void* cuda_stream);
/* number of kernel launches issued on the handle since creation */
int64_t coral_s1_launch_count(const coral_s1_handle* h);

/* ---- problem ---------------------------------------------------------- */
/* Upload the spec tables (host -> device). Validates like the reference
 * constructors (LibraryCaps.__post_init__ templates.py:45-49). */
int coral_s1_set_problem(coral_s1_handle* h, const coral_s1_problem* p);

/* ---- T-hat tables: throughput_table (templates.py:83-96) for every
 * (model, phase, S = 1..min(n_max, L)), node_max_throughput (perf.py:159-175)
 * and stage_budget_s (templates.py:68-80) on device. */
int coral_s1_tables(coral_s1_handle* h);
/* layout: per mp = model*num_phases + phase slot, S-major, config, layer unit.
 * offsets[mp] (num_models*num_phases + 1 entries) index into the flat table. */
int coral_s1_table_layout(const coral_s1_handle* h, int64_t* offsets, int32_t* lsteps,
                          int32_t* smax);
int coral_s1_get_tables(coral_s1_handle* h, double* out, int64_t n);
int coral_s1_get_budgets(coral_s1_handle* h, double* out, int64_t n); /* [mp][n_max] */
/* fraction of positive T-hat entries per (mp, S), [mp][n_max] (S > smax: 0); input of
 * the multi-GPU shard cost model (paper_2605_04357_b200/shard.py) */
int coral_s1_table_posfrac(coral_s1_handle* h, double* out, int64_t n);

/* ---- enumeration: enumerate_combos (templates.py:99-113) -------------- */
int coral_s1_enumerate(coral_s1_handle* h);
int coral_s1_num_combos(const coral_s1_handle* h, int64_t* counts /* [num_models] */);
/* keys of model m in str(combo) order (the library order, templates.py:340);
 * with enumeration_order != 0 in the reference's (num_nodes, str) order
 * (templates.py:112). key = 7 tokens x 9 bits, token = (rank'+1)<<3 | count,
 * first token most significant, zero padded. */
int coral_s1_get_combos(coral_s1_handle* h, int model, int enumeration_order,
                        uint64_t* keys, int64_t n);

/* ---- evaluation: _solve_chunk (templates.py:308-326) over candidates
 * [lo, hi) of the global (model, phase, combo) list (mp-major, library order);
 * hi < 0 means all. Placement DP = _placement_dp_nb (kernels.py:143-276). */
int coral_s1_evaluate(coral_s1_handle* h, int64_t lo, int64_t hi);
/* multi-GPU units: smask[mp] bit S set = evaluate stage count S of (model, phase)
 * mp; records hold each candidate's best over the given S values (ties -> fewer
 * stages), so disjoint masks on different ranks merge exactly. */
int coral_s1_evaluate_units(coral_s1_handle* h, const uint32_t* smask);
/* multi-GPU pieces (the (model, GPU-type combination) axis): piece i
 * evaluates stage counts smask[i] (bit S) of slot mp[i] for the model's candidates
 * [lo[i], hi[i]) (library order; hi < 0 = to the end). Ranks take disjoint pieces. */
int coral_s1_evaluate_pieces(coral_s1_handle* h, int n, const int32_t* mp, const uint32_t* smask,
                             const int64_t* lo, const int64_t* hi);
int coral_s1_num_candidates(const coral_s1_handle* h, int64_t* n);
/* records of one (model, phase slot), library order; n = its combo count */
int coral_s1_get_records(coral_s1_handle* h, int mp, coral_s1_record* out, int64_t n);

/* ---- frontier (new): per (model, phase, region) the skyline of
 * (price ascending, throughput descending, key ascending) over the evaluated
 * candidates; prices[r * num_configs + c] in USD/h, NaN = not offered
 * (allocation.py:91-98 returns None). */
int coral_s1_frontier(coral_s1_handle* h, int num_regions, const double* prices,
                      int64_t* num_survivors);
int coral_s1_get_frontier(coral_s1_handle* h, coral_s1_frontier_item* out, int64_t n);
/* multi-GPU: copy the local survivors into a device buffer (capacity cap), and
 * re-run the skyline over n gathered device items (from all ranks). */
int coral_s1_frontier_export_device(coral_s1_handle* h, void* dev_items, int64_t cap,
                                    int64_t* n);
int coral_s1_frontier_merge_device(coral_s1_handle* h, const void* dev_items, int64_t n,
                                   int64_t* num_survivors);
/* Multi-GPU merge from one all-gather: `parts` partial frontiers laid out at
 * dev_base + p * stride_bytes + item_offset_bytes (counts[p] items each, host array),
 * merged with the same skyline as coral_s1_frontier_merge_device. */
int coral_s1_frontier_merge_parts(coral_s1_handle* h, const void* dev_base, int parts, int64_t stride_bytes,
                                  int64_t item_offset_bytes, const int64_t* counts, int64_t* num_survivors);
/* The exact bucketed prefilter of coral_s1_frontier without the final skyline: the
 * candidates that no strictly cheaper item of this shard dominates, ready for
 * coral_s1_frontier_export_device (multi-GPU: the merge takes the skyline of the union,
 * which equals the global skyline). */
int coral_s1_frontier_candidates(coral_s1_handle* h, int num_regions, const double* prices,
                                 int64_t* num_candidates);
/* Multi-GPU without host round trips: the prefilter's candidates written straight into
 * this rank's slot of an all-gather send buffer (device memory): the int64 item count at
 * dev_part (it may exceed cap: overflow, only the first cap items are written), the
 * items at dev_part + item_offset_bytes. Enqueued on the handle's stream; no sync. */
int coral_s1_frontier_candidates_into(coral_s1_handle* h, int num_regions, const double* prices,
                                      void* dev_part, int64_t item_offset_bytes, int64_t cap);
/* The merge of a gathered buffer of such slots (part p at dev_base + p * stride_bytes),
 * counts read on the device. *max_count = the largest part count; if it exceeds cap the
 * merge is void (*num_survivors = -1): every rank sees the same headers, so all grow
 * cap and repeat candidates_into + all-gather + merge. */
int coral_s1_frontier_merge_gathered(coral_s1_handle* h, const void* dev_base, int parts,
                                     int64_t stride_bytes, int64_t item_offset_bytes, int64_t cap,
                                     int64_t* num_survivors, int64_t* max_count);

/* ---- operator: placement_search (kernels.py:279-295), batched ----------
 * case i: counts[i*7 .. +C_i) (int64), C_i = ncfg[i] <= 7, tput rows at
 * tput + tput_off[i] (C_i x L_i doubles, row-major), S_i. Outputs raw (not
 * canonicalised) results exactly as the numba kernel returns them:
 * best[i] (NEG_INF = -1e300 when infeasible), stage_j[i*7 + s],
 * stage_counts[(i*7 + s)*7 + c] (7 = CORAL_S1_MAX_NODES). Host buffers. */
int coral_s1_placement_search(coral_s1_handle* h, int64_t ncases, const int32_t* ncfg,
                              const int64_t* counts, const int32_t* lsteps,
                              const int64_t* tput_off, const double* tput,
                              int64_t tput_len, const int32_t* S, double* best,
                              int64_t* stage_j, int64_t* stage_counts);

/* ---- timing: device milliseconds of the last call of each stage ---------- */
int coral_s1_stage_ms(const coral_s1_handle* h, double* tables_ms, double* enumerate_ms,
                      double* evaluate_ms, double* frontier_ms);

/* ---- persistence: TemplateLibrary.save (templates.py:364-377)
 * streamed from device records. header = json.dumps(meta, sort_keys=True); mp_order
 * lists (model, phase) slots in library order; model_json[m] = json.dumps(name),
 * phase_json[p] = json.dumps(phase), slo_json[m] = json.dumps([prefill_ms, decode_ms]),
 * cfg_json[c] = json.dumps(config name) (config index order). Byte-identical to the
 * reference's file for the same templates. */
int coral_s1_write_library(coral_s1_handle* h, const char* path, const char* header, int n_mp,
                           const int32_t* mp_order, const char* const* model_json,
                           const char* const* phase_json, const char* const* slo_json,
                           const char* const* cfg_json, int64_t* n_written);
/* ---- caps sweep (cli.py:233-272 cmd_sweep): for caps entries
 * (n_max[k], rho[k]) inside the solved caps, the template count and the best
 * tokens/s per USD-h (price = min over regions, prices[r*K + c], NaN = not offered)
 * over phases in phase_mask (bit = phase slot), from ONE evaluated solve. */
int coral_s1_sweep(coral_s1_handle* h, int ncaps, const int32_t* n_max, const double* rho,
                   int num_regions, const double* prices, uint32_t phase_mask, int64_t* counts,
                   double* best, int64_t* unpriced, int64_t* mp_counts);
/* unpriced[k] (may be NULL): counted templates with a config unpriced in some region (the
 * reference's cmd_sweep raises KeyError on those, cli.py:255); mp_counts[k * NM*NP + mp]
 * (may be NULL): templates per (model, phase) slot at caps entry k (build_library raises
 * LibraryGenError when one is zero, templates.py:499-502). */
/* ---- feasibility check of build_library (templates.py:499-502): feasible templates per
 * (model, phase) slot of the last evaluate into counts[NM*NP]; returns
 * CORAL_S1_ENOTEMPLATE (slots listed in coral_s1_last_error) when an evaluated slot has
 * none. */
int coral_s1_feasible_counts(coral_s1_handle* h, int64_t* counts, int64_t n);
/* ---- T-hat queries (simulator reuse): node_max_throughput
 * (perf.py:159-175, use_profile != 0) or planned_batch_and_tput (perf.py:186-230) for
 * n (config, model, phase code, j layers, budget s) against the current problem's
 * spec tables; host buffers. */
int coral_s1_node_queries(coral_s1_handle* h, int64_t n, const int32_t* cfg, const int32_t* model,
                          const int32_t* phase, const int32_t* j, const double* budget, int use_profile,
                          double* tput, int64_t* batch);
/* ---- stage-2 model construction: build_allocation_model
 * (allocation.py:108-195) over the evaluated records. prices / avail are [R*K] (NaN =
 * unpriced), demand[NM*NP] (<= 0: the slot is skipped), mp_order lists the (model,
 * phase) slots in library order, prune_ratio 0 disables the prune, running (mp, region,
 * combo key) triples are exempt from it. Variables (*num_vars, reference insertion
 * order: slot, template, region) stay on the device for coral_s1_get_allocation_vars;
 * *num_pruned is the reference's meta["pruned_vars"]; best_eff[NM*NP] (may be NULL) the
 * slot's best USD-h per token/s, +inf when it has no priced template (no demand row). */
int coral_s1_allocation_model(coral_s1_handle* h, int num_regions, const double* prices, const int64_t* avail,
                              const double* demand, int n_mp, const int32_t* mp_order, double prune_ratio,
                              int64_t n_running, const int32_t* run_mp, const int32_t* run_region,
                              const uint64_t* run_key, int64_t* num_vars, int64_t* num_pruned,
                              double* best_eff);
int coral_s1_get_allocation_vars(coral_s1_handle* h, coral_s1_alloc_var* out, int64_t n);
/* CPython repr(float) of v into out (cap >= 40); host-only helper, no device needed */
int coral_s1_format_double(double v, char* out, int cap);

/* device time of the last evaluate's lattice kernels of one kind (0 top cells,
 * 1 layers, 2 value tables, 3 decode, 4 sub-multiset ranks): summed CUDA-event time of each launch on its stream */
int coral_s1_kernel_stats(const coral_s1_handle* h, int kind, double* total_ms, int64_t* launches);
/* device time (CUDA events on the handle's stream) and algorithmic bytes of the last
 * enumerate's window_select_kernel, the per-model memory-window compaction of
 * templates.py:110-111 (bench roofline of the streaming path); ms = -1 if none ran */
int coral_s1_window_select_stats(const coral_s1_handle* h, double* ms, int64_t* alg_bytes);
/* per-launch timing events of the lattice kernels (kernel_stats / kernel_timeline /
 * kernel_launches read them): off by default -- the evaluate then records no
 * per-launch events -- on for diagnostics, the bench roofline pass and the multi-GPU
 * cost calibration */
int coral_s1_set_timing(coral_s1_handle* h, int on);
/* per-launch timeline of the last evaluate's lattice kernels (kinds as above plus
 * 3 decode, 4 sub-multiset ranks): side-stream slot and begin/end in ms from the
 * evaluate's start event; up to cap launches, count in *n (diagnostics) */
int coral_s1_kernel_timeline(const coral_s1_handle* h, int64_t cap, int32_t* kind, int32_t* stream,
                             double* begin_ms, double* end_ms, int64_t* n);
/* the last evaluate's timed lattice launches: kind (as coral_s1_kernel_stats), (model,
 * phase) slot, device ms (cost calibration of the multi-GPU split, shard.py) */
int coral_s1_kernel_launches(const coral_s1_handle* h, int64_t cap, int32_t* kind, int32_t* mp, double* ms,
                             int64_t* n);
/* layer-kernel census for the bench roofline: while on, each evaluate counts the
 * algorithmic bytes of its lat_layer_kernel launches (10 B per f/choice cell written +
 * one read of each computed state's value_S and f_{sg-1} rows + 8 B per valid
 * sub-table entry); off (default) passes no counter to the kernel */
int coral_s1_set_census(coral_s1_handle* h, int on);
int coral_s1_census(coral_s1_handle* h, int64_t* layer_bytes);
/* all census counters of the last evaluate: [0] layer-kernel algorithmic bytes, [1] layer
 * (u, l) pairs, [2] top-cell (u, S) pairs searched, [3] reserved */
int coral_s1_census_all(coral_s1_handle* h, int64_t* out, int n);
/* chain streams used by evaluate (1..8; 0 = the default, 4 or CORAL_S1_STREAMS): 1
 * serialises the lattice kernels (bench.py times the roofline launches that way) */
int coral_s1_set_streams(coral_s1_handle* h, int n);

#ifdef __cplusplus
}
#endif
#endif /* CORAL_S1_H */
