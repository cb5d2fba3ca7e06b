// roofline.cuh — bit-exact fp64 restatement of the reference's analytic
// per-node throughput model (T-hat) for sm_100a.
//
// Reference: /root/reference/pkg/src/hetserve/perf.py:57-91 (per-layer bytes,
// iteration_time, transfer_time), :144-230 (max_batch_by_memory,
// node_max_throughput, planned_batch_and_tput) and templates.py:68-80
// (stage_budget_s). Python evaluates every expression left to right in IEEE
// double without contraction, so every multiply/add/divide below goes through
// the explicit round-to-nearest intrinsics (no FMA), in the reference's
// operation order. The file is compiled with -fmad=false as a second guard.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coral {

constexpr int kPrefill = 0;
constexpr int kDecode = 1;
constexpr double kGiB = 1073741824.0;  // domain.py GIB = 2**30
constexpr double kNegInf = -1e300;     // kernels.py:31 NEG_INF

__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }

// Device view of coral_s1_problem (all arrays device-resident).
struct DevProblem {
  int K, NM, NP, n_max;
  double rho;
  const int* gc;
  const double* mem_gb;
  const double* bw;
  const double* tflops;
  const double* mem_bytes;  // (gc * mem_gb) * GIB per config, domain.py:48-50
  const int* rank1;         // str rank + 1 per config (token name field)
  const int* inv_rank;      // rank -> config index
  const int* L;
  const int* g;
  const int* Lu;
  const int* smax;          // min(n_max, L): tables exist for S = 1..smax
  const double* ptb;
  const double* pab;
  const double* hidden;
  const double* bpp;
  const double* kv;
  const double* slo_pf;
  const double* slo_dc;
  const int* phases;
  double mfu, mbu, net_eff, fixed_ms, prompt, ctxd, frac, gbps, lat_ms;
  int nprof;
  const int* pm;
  const int* pp;
  const int* pc;
  const int* pj;
  const int* pb;
  const double* pt;
};

// templates.py:68-80 stage_budget_s (with transfer_time, perf.py:87-91)
__device__ __forceinline__ double stage_budget(const DevProblem& P, int m, int phase, int S) {
  const double slo = (phase == kPrefill) ? P.slo_pf[m] : P.slo_dc[m];
  double total = rn_mul(rn_div(slo, 1e3), P.frac);
  if (phase == kPrefill && S > 1) {
    const double act = rn_mul(rn_mul(P.prompt, P.hidden[m]), P.bpp[m]);
    const double hop = rn_add(rn_div(P.lat_ms, 1e3), rn_div(act, rn_mul(rn_mul(P.gbps, 1e9), P.net_eff)));
    total = rn_sub(total, rn_mul((double)(S - 1), hop));
  }
  return rn_div(total, (double)S);
}

// perf.py:110-116 ProfileTable.lookup: exact (config, model, phase, j, bucket)
// hit first, then the bucket -1 wildcard. Returns true on a hit.
__device__ __forceinline__ bool profile_lookup(const DevProblem& P, int c, int m, int phase,
                                               int j, double budget, double* out) {
  if (P.nprof == 0) return false;
  // Python int(round(x)): round half to even == rint in the default mode
  const long long bucket = (long long)rint(rn_mul(budget, 1e3));
  int wild = -1;
  for (int i = 0; i < P.nprof; ++i) {
    if (P.pm[i] != m || P.pp[i] != phase || P.pc[i] != c || P.pj[i] != j) continue;
    if ((long long)P.pb[i] == bucket) { *out = P.pt[i]; return true; }
    if (P.pb[i] == -1) wild = i;
  }
  if (wild >= 0) { *out = P.pt[wild]; return true; }
  return false;
}

struct NodeModel {
  double jd, tpr, ctx, kv, wbpl, abfpl, cden, mden, d;
  // perf.py:66-84 iteration_time(node, model, j, b*tpr, b, phase)
  __device__ __forceinline__ double iter_t(long long b) const {
    const double bd = (double)b;
    const double bt = rn_mul(bd, tpr);
    const double compute = rn_div(rn_mul(rn_mul(rn_mul(2.0, abfpl), jd), bt), cden);
    const double memory = rn_div(rn_mul(jd, rn_add(wbpl, rn_mul(rn_mul(bd, kv), ctx))), mden);
    return rn_add(memory > compute ? memory : compute, d);
  }
};

// perf.py:186-230 planned_batch_and_tput: returns the throughput, *b_out the batch.
// j is in layers (jj * granularity), budget > 0.
__device__ double planned_batch_and_tput(const DevProblem& P, int c, int m, int phase, int j,
                                         double budget, long long* b_out) {
  *b_out = 0;
  const double gcd = (double)P.gc[c];
  const double Ld = (double)P.L[m];
  NodeModel nm;
  nm.jd = (double)j;
  nm.ctx = (phase == kPrefill) ? P.prompt : P.ctxd;          // PerfParams.phase_ctx
  nm.kv = P.kv[m];
  const double wbytes = rn_mul(rn_mul(P.ptb[m], 1e9), P.bpp[m]);  // ModelSpec.weight_bytes
  nm.wbpl = rn_div(wbytes, Ld);                                 // weight_bytes_per_layer
  nm.abfpl = rn_div(rn_mul(P.pab[m], 1e9), Ld);                   // active_bytes_flops_per_layer
  // max_batch_by_memory (perf.py:149-156)
  const double freeb = rn_sub(P.mem_bytes[c], rn_mul(nm.jd, nm.wbpl));
  if (freeb <= 0.0) return 0.0;
  const double per_req = rn_mul(rn_mul(nm.jd, nm.kv), nm.ctx);
  double q = trunc(rn_div(freeb, per_req));
  if (q > 9.0e15) q = 9.0e15;  // Python int is unbounded; any value this large is capped by b_lat
  const long long b_mem = (long long)q;
  if (b_mem < 1) return 0.0;
  nm.tpr = (phase == kPrefill) ? P.prompt : 1.0;              // _tokens_per_request
  nm.cden = rn_mul(rn_mul(rn_mul(gcd, P.tflops[c]), 1e12), P.mfu);
  nm.mden = rn_mul(rn_mul(rn_mul(gcd, P.bw[c]), 1e12), P.mbu);
  const double a = rn_div(rn_mul(rn_mul(rn_mul(2.0, nm.abfpl), nm.jd), nm.tpr), nm.cden);
  const double w = rn_div(rn_mul(nm.jd, nm.wbpl), nm.mden);
  const double k = rn_div(rn_mul(rn_mul(nm.jd, nm.kv), nm.ctx), nm.mden);
  nm.d = rn_div(P.fixed_ms, 1e3);
  const double slack = rn_sub(budget, nm.d);
  if (slack <= 0.0) return 0.0;
  double b_lat = __longlong_as_double(0x7ff0000000000000ll);  // math.inf
  if (a > 0.0) { const double x = rn_div(slack, a); if (x < b_lat) b_lat = x; }
  if (k > 0.0) {
    const double x = rn_div(rn_sub(slack, w), k);
    if (x < b_lat) b_lat = x;
  } else if (w > slack) {
    return 0.0;
  }
  long long b;
  if (!isfinite(b_lat)) {
    b = b_mem;
  } else {
    const double fl = floor(rn_add(b_lat, 1e-9));
    if (fl >= (double)b_mem) b = b_mem;
    else if (fl < -1.0) b = -1;
    else b = (long long)fl;
  }
  if (b < 1) return 0.0;
  const double lim = rn_add(budget, 1e-12);
  // local fix-up so the closed form agrees exactly with an integer search
  while (b >= 1 && nm.iter_t(b) > lim) --b;
  while (b < b_mem && nm.iter_t(b + 1) <= lim) ++b;
  if (b < 1) return 0.0;
  *b_out = b;
  return rn_div(rn_mul((double)b, nm.tpr), nm.iter_t(b));
}

// perf.py:159-175 node_max_throughput: a profile hit wins verbatim.
__device__ double node_max_throughput(const DevProblem& P, int c, int m, int phase, int j,
                                      double budget) {
  double hit;
  if (profile_lookup(P, c, m, phase, j, budget, &hit)) return hit;
  long long b;
  return planned_batch_and_tput(P, c, m, phase, j, budget, &b);
}

}  // namespace coral
