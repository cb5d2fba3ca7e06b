// coral_s1.cu — B200-native stage-1 Serving-Template generator: kernels + C ABI.
//
// Pipeline:
//   tables_kernel        T-hat rows per (model, phase, S, config)      templates.py:83-96
//   enum_count_kernel    unrank every multiset once, directly in str(combo) order: key +
//                        memory sum + per-model window counts         templates.py:99-112, 340
//   window_select        per-model memory window, stable compaction   templates.py:110-111
//   lattice kernels      (lattice.cuh) per (model, phase, S) chains on 4 streams: the
//                        DP of every candidate over shared sub-multiset tables,
//                        best S, decode                               templates.py:308-326
//   evaluate_kernel      exact per-candidate DP (memory-limited route) kernels.py:143-276
//   frontier             price per (candidate, region) -> bucketed exact prefilter ->
//                        stable merge sort -> segmented running max -> compaction
//                                                                     SURVEY.md 8c
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/coral_s1.h"
#include "lattice.cuh"
#include "pyrepr.h"
#include "placement_dp.cuh"
#include "roofline.cuh"

using namespace coral;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(CORAL_S1_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define LAUNCH_CHECK(h)                                                               \
  do {                                                                                \
    (h)->launches++;                                                                  \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess)                                                            \
      return fail(CORAL_S1_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kKeyTokenBits = 9;

__constant__ unsigned long long c_binom[160][8];  // C(N, k), N < 160, k <= 7

inline unsigned long long next_alloc_id() {  // process-wide, never reused
  static std::atomic<unsigned long long> n{0};
  return ++n;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  unsigned long long id = 0;  // changes with every allocation (a freed address may come back)
  // upload_same: the bytes last copied in (host-written, device-read-only buffers only)
  std::vector<unsigned char> shadow;
  unsigned long long shadow_id = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }  // locals free on every early return
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) return fail(CORAL_S1_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    cap = want;
    id = next_alloc_id();
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    id = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

struct coral_s1_handle {
  int device = 0;
  int num_sms = 148, ranks_blocks_per_sm = 1;
  size_t dp_smem_limit = 0;  // dynamic shared memory the per-candidate DP kernels may use
  cudaStream_t stream = nullptr;
  long long launches = 0;
  bool have_problem = false, have_tables = false, have_enum = false, have_eval = false;
  // host copy of the problem shape
  int K = 0, NM = 0, NP = 0, n_max = 0;
  std::vector<int> L, g, Lu, smax, phases;
  std::vector<int64_t> tab_off;  // [NM*NP + 1]
  int maxLu = 0;
  int64_t U = 0;                 // multiset universe size per model
  std::vector<int64_t> counts;   // combos per model
  std::vector<int64_t> koff;     // [NM+1] first key of each model (compacted)
  std::vector<int64_t> cand_off; // [NM*NP + 1]
  int64_t ncand = 0;
  int64_t nfront = 0;
  int num_regions = 0;
  DevProblem dp{};
  // device buffers
  DevBuf prob, tab, flags, budget, keys, koff_d, nvalid, cand_off_d, rec, cub_tmp;
  DevBuf items, items_sorted, sort_a, sort_b, segk, scanv, flagsel, nsel, front,
      prices, ukey_s, umem_s, blkcnt, blkoff;
  DevBuf op_in, op_out, tab_off_d, fbucket, segbuf, avars, pcounts;
  int64_t navars = 0;
  // lattice (lattice.cuh): shared state tables + per-model maxn + per-stream workspaces
  static constexpr int kStreams = 8;
  static constexpr int kDefaultStreams = 4;
  int default_streams = kDefaultStreams;  // CORAL_S1_STREAMS
  int nstreams = kDefaultStreams;  // side streams in use
  int lat_streams = kStreams;  // streams whose lattice workspace fits in device memory
  bool lat_ok = true;          // false: every unit runs the exact per-candidate kernel
  size_t mem_limit = 0;        // CORAL_S1_MEM_LIMIT: cap on usable device memory (tests)
  long long lat_fit_ns = -1, lat_fit_pitch = -1;  // table shape of the last fit decision
  long long lat_states = 0;
  std::vector<long long> lat_base;     // [R + 2]
  DevBuf lat_base_d, lat_binom_d, lat_key, lat_nsub, lat_off, lat_sub, lat_maxn, lat_flags_h;
  DevBuf ws_value[kStreams], ws_f0[kStreams], ws_ch[kStreams], ws_ranks[kStreams], ws_win[kStreams];
  cudaStream_t side[kStreams] = {};
  cudaEvent_t side_ev[kStreams] = {};
  cudaEvent_t fork_ev = nullptr;
  cudaEvent_t prep_ev = nullptr;  // lattice tables prepared on side[0] during enumerate
  bool lat_ready = false, flags_ready = false;
  std::vector<unsigned char> flags_h;
  std::vector<char> model_used;
  std::vector<char> own_mp;  // (model, phase) chains with records from the last evaluate
  DevBuf run_off_d, run_mp_d, run_ph_d;
  DevBuf tokp;  // [R][512] token prices of the last frontier
  DevBuf rect;  // per candidate: the record's throughput (0 = no template), for the frontier passes
  std::vector<double> memb_h, wbytes_h;  // config memory bytes, model weight bytes
  std::vector<int> inv_rank_h;           // str rank -> config index
  double rho = 0;
  DevBuf lat_sums, lat_soff;
  // per-launch timing of the lattice kernels (coral_s1_kernel_stats)
  static constexpr int kTimedMax = 2048;  // events created on first use
  cudaEvent_t tev[kTimedMax][2] = {};
  int tkind[kTimedMax] = {};
  int tslot[kTimedMax] = {};
  int tmp[kTimedMax] = {};   // (model, phase) slot of the launch (rank tables: the model's first)
  bool timing = false;       // per-launch events on (coral_s1_set_timing); off: no event records
  int cur_mp = -1;
  int ntimed = 0;
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_ws[2] = {};  // around the last window_select_kernel launch (bench roofline)
  bool ws_timed = false;
  int64_t ws_bytes = 0;
  float ms[4] = {0, 0, 0, 0};
  // layer-kernel census (coral_s1_set_census): algorithmic bytes of the last evaluate
  bool census_on = false;
  DevBuf census;
  DevBuf poscnt;  // positive T-hat entries per (mp, S)
  DevBuf prep_tmp;  // CUB scratch of lattice_prepare (side stream)
  // memoised achievable-memory-sum table of lattice_prepare (key -> flat sums, offsets)
  std::vector<double> sums_key_mem, sums_flat;
  double sums_key_cap = -1.0;
  int sums_key_kmax = -1;
  std::vector<int> sums_off;
};

namespace {

// --------------------------------------------------------------------------------
// T-hat tables. One block per (mp, S, config); threads over layer units jj.
// Also the per-row monotone flags kernels.py:291 needs:
//   bit0: all(diff <= 1e-12) (the reference's test), bit1: all(diff <= 0).
// --------------------------------------------------------------------------------
__global__ void tables_kernel(DevProblem P, const int64_t* __restrict__ tab_off,
                              double* __restrict__ tab, unsigned char* __restrict__ flags,
                              double* __restrict__ budgets, unsigned* __restrict__ poscnt) {
  __shared__ unsigned npos;
  const int c = blockIdx.x;
  const int S = blockIdx.y + 1;
  const int mp = blockIdx.z;
  const int m = mp / P.NP;
  const int phase = P.phases[mp % P.NP];
  if (S > P.smax[m]) return;
  const int Lu = P.Lu[m];
  const int g = P.g[m];
  const double budget = stage_budget(P, m, phase, S);
  if (c == 0 && threadIdx.x == 0) budgets[mp * P.n_max + (S - 1)] = budget;
  double* row = tab + tab_off[mp] + ((int64_t)(S - 1) * P.K + c) * Lu;
  for (int jj = threadIdx.x; jj < Lu; jj += blockDim.x) {
    // templates.py:89-95: zeros when the budget is exhausted
    row[jj] = (budget <= 0.0) ? 0.0 : node_max_throughput(P, c, m, phase, (jj + 1) * g, budget);
  }
  if (threadIdx.x == 0) npos = 0;
  __syncthreads();
  unsigned mine = 0;  // positive entries (shard cost model, coral_s1_table_posfrac)
  for (int jj = threadIdx.x; jj < Lu; jj += blockDim.x) mine += row[jj] > 0.0;
  if (mine) atomicAdd(&npos, mine);
  int tol = 1, exact = 1;
  for (int jj = threadIdx.x; jj + 1 < Lu; jj += blockDim.x) {
    const double d = rn_sub(row[jj + 1], row[jj]);  // np.diff
    tol &= (d <= 1e-12);
    exact &= (d <= 0.0);
  }
  tol = __syncthreads_and(tol);
  exact = __syncthreads_and(exact);
  if (threadIdx.x == 0) {
    flags[((int64_t)mp * P.n_max + (S - 1)) * P.K + c] = (unsigned char)(tol | (exact << 1));
    if (npos) atomicAdd(poscnt + (int64_t)mp * P.n_max + (S - 1), npos);
  }
}

// --------------------------------------------------------------------------------
// Enumeration: thread per (model, universe rank). Universe = multisets of 1..n_max
// of K configs, ranked size-major, lexicographic within a size (stars and bars).
// --------------------------------------------------------------------------------
constexpr int kEnumBinomRows = 72;  // N = K + n - 1 < 63 + 7 in the GPU envelope


// Enumeration (templates.py:99-113) in two streaming passes, with no sort. The universe
// of node multisets is model-independent, and it is unranked DIRECTLY in packed-key order
// (= str(combo) order): each model's window test (weight <= mem <
// rho * weight) is then a stable compaction of that order -- model-major, library order
// within a model.
//
// Key order: tokens ((r + 1) << 3 | count) with strictly increasing str rank r, first token
// most significant, zero padded. Rest(r0, m) = token sequences over ranks >= r0 with total
// count <= m, the empty one first; |Rest(r0, m)| = C(K - r0 + m, m) (multisets of size
// <= m from K - r0 types). The sequences whose first rank is >= r number C(K - r + m, m) - 1,
// and those with first token (r, c) number C(K - r - 1 + m - c, m - c).

constexpr int kEnumThreads = 256, kEnumItems = 4;  // one block = 1024 consecutive ranks
constexpr int kEnumBlock = kEnumThreads * kEnumItems;

// universe element `idx` (0-based among the non-empty sequences, key order) -> packed key
// and memory sum, summed over the picks in config (name) order (templates.py:103-109)
__device__ __forceinline__ void unrank_key(const unsigned long long (*B)[8], const DevProblem& P,
                                           unsigned long long idx, unsigned long long& key, double& mem) {
  const int K = P.K;
  int m = P.n_max, r0 = 0, ntok = 0;
  int tcfg[kMaxC], tcnt[kMaxC];
  key = 0ull;
  for (;;) {
    // first rank r: the largest r with #(first rank < r) <= idx
    const unsigned long long tot0 = B[K - r0 + m][m] - 1ull;
    int lo = r0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tot0 - (B[K - mid + m][m] - 1ull) <= idx) lo = mid; else hi = mid - 1;
    }
    const int r = lo;
    idx -= tot0 - (B[K - r + m][m] - 1ull);
    int c = 1;
    for (;; ++c) {  // first token (r, c): blocks of C(K - r - 1 + m - c, m - c)
      const unsigned long long blk = B[K - r - 1 + m - c][m - c];
      if (idx < blk) break;
      idx -= blk;
    }
    key = (key << kKeyTokenBits) | ((unsigned long long)(r + 1) << 3) | (unsigned long long)c;
    tcfg[ntok] = P.inv_rank[r];
    tcnt[ntok] = c;
    ++ntok;
    if (idx == 0ull) break;  // the empty rest
    --idx;
    r0 = r + 1;
    m -= c;
  }
  key <<= kKeyTokenBits * (kMaxC - ntok);
  // picks in config-index (name) order: sort the <= 7 tokens by config
  for (int a = 1; a < ntok; ++a)
    for (int b = a; b > 0 && tcfg[b - 1] > tcfg[b]; --b) {
      const int t0 = tcfg[b], t1 = tcnt[b];
      tcfg[b] = tcfg[b - 1];
      tcnt[b] = tcnt[b - 1];
      tcfg[b - 1] = t0;
      tcnt[b - 1] = t1;
    }
  mem = 0.0;
  for (int t = 0; t < ntok; ++t)
    for (int k = 0; k < tcnt[t]; ++k) mem = rn_add(mem, P.mem_bytes[tcfg[t]]);
}

// templates.py:110-111 window of model m, in the reference's arithmetic
__device__ __forceinline__ void model_window(const DevProblem& P, int m, double& lo, double& hi) {
  const double wbytes = rn_mul(rn_mul(P.ptb[m], 1e9), P.bpp[m]);
  lo = wbytes;
  hi = rn_mul(P.rho, wbytes);
}

// Both passes count and compact per 128-element chunk (one warp's share of a block):
// chunk c = elements c * 128 .. c * 128 + 127, so the compaction needs no block-wide
// scan, no shared-memory staging and no barrier -- a warp's survivors of a model go out
// at the chunk's scanned offset in 4 coalesced stores.
constexpr int kEnumChunk = 32 * kEnumItems, kEnumChunksPerBlock = kEnumBlock / kEnumChunk;

// pass 1: thread t of block b unranks elements b * 1024 + 4t .. +3 (key order), stores
// their keys and memory sums (16 B each, read once by pass 2) and counts each model's
// window survivors per chunk: chkcnt[m * nchunk + c] (model-major)
__global__ void __launch_bounds__(kEnumThreads) enum_count_kernel(
    DevProblem P, int64_t U, int64_t nchunk, unsigned long long* __restrict__ ukey, double* __restrict__ umem,
    unsigned long long* __restrict__ chkcnt) {
  __shared__ unsigned long long s_binom[kEnumBinomRows][8];
  const int rows = min(kEnumBinomRows, P.K + P.n_max + 1);
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) s_binom[i >> 3][i & 7] = c_binom[i >> 3][i & 7];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t e0 = (int64_t)blockIdx.x * kEnumBlock + (int64_t)threadIdx.x * kEnumItems;
  const int64_t chunk = (int64_t)blockIdx.x * kEnumChunksPerBlock + (threadIdx.x >> 5);
  unsigned long long k4[kEnumItems];
  double m4[kEnumItems];
#pragma unroll
  for (int k = 0; k < kEnumItems; ++k) {
    k4[k] = 0ull;
    m4[k] = -1.0;  // past the end: in no window (weights are > 0)
    if (e0 + k < U) unrank_key(s_binom, P, (unsigned long long)(e0 + k), k4[k], m4[k]);
  }
  if (e0 + kEnumItems <= U) {  // 32-byte aligned: vector stores
    reinterpret_cast<ulonglong2*>(ukey + e0)[0] = make_ulonglong2(k4[0], k4[1]);
    reinterpret_cast<ulonglong2*>(ukey + e0)[1] = make_ulonglong2(k4[2], k4[3]);
    reinterpret_cast<double2*>(umem + e0)[0] = make_double2(m4[0], m4[1]);
    reinterpret_cast<double2*>(umem + e0)[1] = make_double2(m4[2], m4[3]);
  } else {
    for (int k = 0; k < kEnumItems; ++k)
      if (e0 + k < U) {
        ukey[e0 + k] = k4[k];
        umem[e0 + k] = m4[k];
      }
  }
  if (chunk >= nchunk) return;  // warp-uniform
  for (int m = 0; m < P.NM; ++m) {
    double lo, hi;
    model_window(P, m, lo, hi);
    int c = 0;
#pragma unroll
    for (int k = 0; k < kEnumItems; ++k) c += lo <= m4[k] && m4[k] < hi;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == (m & 31)) chkcnt[(int64_t)m * nchunk + chunk] = (unsigned long long)c;
  }
}

// pass 2: ONE read of the chunk's keys and memory sums (element c * 128 + 32k + lane:
// coalesced), then every model's stable compaction at its scanned chunk offset: per k a
// ballot, and the warp's survivors of that k land contiguously (coalesced store)
__global__ void __launch_bounds__(kEnumThreads) window_select_kernel(
    DevProblem P, int64_t U, const unsigned long long* __restrict__ ukey, const double* __restrict__ umem,
    int64_t nchunk, const unsigned long long* __restrict__ chkoff, unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * kEnumChunksPerBlock + (threadIdx.x >> 5);
  if (chunk >= nchunk) return;
  const int64_t e0 = chunk * kEnumChunk + lane;
  unsigned long long k4[kEnumItems];
  double m4[kEnumItems];
#pragma unroll
  for (int k = 0; k < kEnumItems; ++k) {
    const int64_t e = e0 + 32 * k;
    k4[k] = e < U ? ukey[e] : 0ull;
    m4[k] = e < U ? umem[e] : -1.0;
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int m = 0; m < P.NM; ++m) {
    double lo, hi;
    model_window(P, m, lo, hi);
    unsigned bal[kEnumItems];
    int tot = 0;
#pragma unroll
    for (int k = 0; k < kEnumItems; ++k) {
      bal[k] = __ballot_sync(0xffffffffu, lo <= m4[k] && m4[k] < hi);
      tot += __popc(bal[k]);
    }
    if (!tot) continue;  // warp-uniform
    unsigned long long* out = keys + chkoff[(int64_t)m * nchunk + chunk];
    int at = 0;
#pragma unroll
    for (int k = 0; k < kEnumItems; ++k) {
      if ((bal[k] >> lane) & 1u) out[at + __popc(bal[k] & lt)] = k4[k];
      at += __popc(bal[k]);
    }
  }
}

// per-model survivor counts from the scanned chunk offsets (offset array has NM*nchunk+1)
__global__ void window_totals_kernel(int NM, int64_t nchunk, const unsigned long long* __restrict__ chkoff,
                                     unsigned long long* __restrict__ nvalid) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < NM) nvalid[m] = chkoff[(int64_t)(m + 1) * nchunk] - chkoff[(int64_t)m * nchunk];
}


__device__ __forceinline__ int decode_key(const DevProblem& P, unsigned long long key,
                                          int* cfg, int* cnt) {
  int C = 0;
  for (int t = 0; t < kMaxC; ++t) {
    const unsigned tok = (unsigned)(key >> (kKeyTokenBits * (kMaxC - 1 - t))) & 511u;
    if (!tok) break;
    cfg[C] = P.inv_rank[(tok >> 3) - 1];
    cnt[C] = tok & 7u;
    ++C;
  }
  return C;
}

// --------------------------------------------------------------------------------
// Canonical placement (templates.py:209-228): stages ordered by (-j, -counts tuple),
// layers = j * g, nodes assigned config by config in combo order.
// stage_cnt[s][c] = nodes of combo config c in raw stage s.
// --------------------------------------------------------------------------------
__device__ void canonical_record(int S, const int* stage_j, const int (*stage_cnt)[kMaxC], int C,
                                 const int* cnt, int g, double val, int n, coral_s1_record* rec) {
  int order[kMaxC];
  for (int s = 0; s < S; ++s) order[s] = s;
  for (int a = 1; a < S; ++a) {  // stable insertion sort == sorted(range(S), key=...)
    const int x = order[a];
    int b = a - 1;
    while (b >= 0) {
      const int y = order[b];
      bool less;  // key(x) < key(y)
      if (stage_j[x] != stage_j[y]) less = stage_j[x] > stage_j[y];
      else {
        less = false;
        for (int c = 0; c < C; ++c)
          if (stage_cnt[x][c] != stage_cnt[y][c]) { less = stage_cnt[x][c] > stage_cnt[y][c]; break; }
      }
      if (!less) break;
      order[b + 1] = y;
      --b;
    }
    order[b + 1] = x;
  }
  int next_free[kMaxC];
  int offc = 0;
  for (int c = 0; c < C; ++c) { next_free[c] = offc; offc += cnt[c]; }
  coral_s1_record r;
  memset(&r, 0, sizeof(r));
  r.throughput_tps = val;
  r.num_stages = (unsigned char)S;
  r.num_nodes = (unsigned char)n;
  for (int pos = 0; pos < S; ++pos) {
    const int s = order[pos];
    r.layers_per_stage[pos] = (unsigned short)(stage_j[s] * g);
    for (int c = 0; c < C; ++c)
      for (int k = 0; k < stage_cnt[s][c]; ++k) r.stage_of_node[next_free[c]++] = (unsigned char)pos;
  }
  *rec = r;
}

__device__ __forceinline__ double record_best(const coral_s1_record& r) {
  return r.num_stages ? r.throughput_tps : kNegInf;
}

// templates.py:317-324 keeps S if val > best and val > 1e-9 while S ascends; the
// equivalent order-independent rule also prefers the smaller S on an exact tie.
__device__ __forceinline__ bool better_S(double val, int S, double best, int bestS) {
  return val > 1e-9 && (val > best || (val == best && bestS > 0 && S < bestS));
}

// --------------------------------------------------------------------------------
// Per-candidate evaluator (exact fallback): one CTA per candidate (model, phase,
// combo) for S in [S_lo, S_hi], continuing from the candidate's current record.
// templates.py:308-326 for the S loop and best-S rule (strictly better, > 1e-9),
// kernels.py:143-276 for the DP (placement_dp.cuh). Used where the lattice path
// does not apply (a row outside the monotone test at this S) and for sub-ranges.
// --------------------------------------------------------------------------------
struct EvalArgs {
  DevProblem P;
  const unsigned long long* keys;  // model m's combos at koff[m], str(combo) order
  const int64_t* koff;
  const int64_t* cand_off;         // [NMP+1]
  int NMP;
  int64_t lo, hi, stride;          // candidates lo, lo+stride, ... < hi
  int S_lo, S_hi;
  const double* tab;
  const int64_t* tab_off;
  const unsigned char* flags;
  coral_s1_record* rec;            // indexed by global candidate index
  double* rect;                    // its throughput (frontier passes)
};

__global__ void __launch_bounds__(kDpThreads) evaluate_kernel(EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ DpShared sh;
  __shared__ int s_mp, s_cfg[kMaxC];
  __shared__ double s_best;
  __shared__ int s_bestS;
  __shared__ coral_s1_record s_rec;
  const int64_t ci = A.lo + (int64_t)blockIdx.x * A.stride;
  if (ci >= A.hi) return;
  const int tid = threadIdx.x;
  const DevProblem& P = A.P;
  if (tid == 0) {
    int lo = 0, hi = A.NMP;  // last mp with cand_off[mp] <= ci
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (A.cand_off[mid] <= ci) lo = mid; else hi = mid;
    }
    s_mp = lo;
    const int m = lo / P.NP;
    const int64_t idx = ci - A.cand_off[lo];
    int cfg[kMaxC], cnt[kMaxC];
    const int C = decode_key(P, A.keys[A.koff[m] + idx], cfg, cnt);
    sh.C = C;
    for (int c = 0; c < C; ++c) { s_cfg[c] = cfg[c]; sh.cnt[c] = cnt[c]; }
    sh.Lu = P.Lu[m];
    sh.LuP = sh.Lu + 1;
    s_rec = A.rec[ci];
    s_best = record_best(s_rec);
    s_bestS = s_rec.num_stages;
  }
  __syncthreads();
  dp_setup_lattice(sh);
  const int mp = s_mp;
  const int m = mp / P.NP;
  const int K = P.K;
  const int Lu = sh.Lu, LuP = sh.LuP, C = sh.C, M = sh.M, n = sh.n;
  const DpBuffers B = dp_carve(smem, M, LuP, Lu, n - 2);
  const int Smax = min(min(n, Lu), A.S_hi);
  for (int S = A.S_lo; S <= Smax; ++S) {
    // tables[S][cfg_rows, :] (templates.py:320)
    const double* base = A.tab + A.tab_off[mp] + (int64_t)(S - 1) * K * Lu;
    for (int idx = tid; idx < C * Lu; idx += blockDim.x) {
      const int c = idx / Lu;
      const int jj = idx - c * Lu;
      B.tputS[idx] = base[(int64_t)s_cfg[c] * Lu + jj];
    }
    if (tid == 0) {
      int mono = 1;
      for (int c = 0; c < C; ++c)
        mono &= A.flags[((int64_t)mp * P.n_max + (S - 1)) * K + s_cfg[c]] & 1;
      sh.mono = mono;
    }
    __syncthreads();
    dp_build_value(sh, B);
    __syncthreads();
    double val;
    if (S == 1) {
      val = B.value[(M - 1) * LuP + Lu];  // f[1][L][full]
      if (tid == 0) { sh.top_val = val; sh.top_u = M - 1; sh.top_j = Lu; }
    } else {
      dp_run(sh, B, S);
      val = sh.top_val;
    }
    // templates.py:322: strictly better and > 1e-9, ties keep the smaller S
    // (order-independent form, so S values may be evaluated by different kernels)
    if (tid == 0 && better_S(val, S, s_best, s_bestS)) {
      s_best = val;
      s_bestS = S;
      if (S == 1) { sh.stage_j[0] = Lu; sh.stage_u[0] = M - 1; }
      else dp_decode(sh, B, S);
      int stage_cnt[kMaxC][kMaxC];
      for (int s = 0; s < S; ++s)
        for (int c = 0; c < C; ++c) stage_cnt[s][c] = sh.digits[sh.stage_u[s]][c];
      canonical_record(S, sh.stage_j, stage_cnt, C, sh.cnt, P.g[m], val, n, &s_rec);
    }
    __syncthreads();
  }
  if (tid == 0) {
    A.rec[ci] = s_rec;
    A.rect[ci] = s_rec.num_stages ? s_rec.throughput_tps : 0.0;
  }
}

// Warp-wide (value desc, code asc) selection of the reference tie rule with the
// hardware reductions: candidate values are >= 0 (or kNegInf for an empty lane, which
// never wins), and non-negative doubles order like their bit patterns, so the max is
// the lexicographic max of (hi word, lo word); ties go to the smallest code. All
// lanes receive the winner's (value, code, j).
__device__ __forceinline__ void warp_argmax_code(double& v, int& code, int& j) {
  const bool ok = v >= 0.0;
  const unsigned long long b = ok ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  const unsigned c = __reduce_min_sync(0xffffffffu, top ? (unsigned)code : 0xffffffffu);
  const unsigned who = __ballot_sync(0xffffffffu, top && (unsigned)code == c);
  const int src = __ffs(who) - 1;
  const double wv = __shfl_sync(0xffffffffu, v, src);
  j = __shfl_sync(0xffffffffu, j, src);
  code = (int)c;
  v = wv;
}

// warp_argmax_code with the lane's (code, j) packed as code << 10 | j: among the lanes
// holding the max value the smallest packed word is the smallest code (each code lives
// on one lane), so one min-reduction carries the winner's j along.
__device__ __forceinline__ void warp_argmax_packed(double& v, unsigned& bc) {
  const bool ok = v >= 0.0;
  const unsigned long long b = ok ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  bc = __reduce_min_sync(0xffffffffu, top ? bc : 0xFFFFFFFFu);
  v = __hiloint2double((int)mhi, (int)mlo);
}

// --------------------------------------------------------------------------------
// Lattice top cells: one warp per candidate of one (model, phase), every S in smask.
// f_S[S][Lu][full] = max over u (lanes) of the crossing with f_S[S-1][.][full-u]
// (value_S when S == 2), reduced with the reference tie rule (value desc, u code
// asc); best S by better_S; the winning S's choices are walked back through its
// lattice layers into the canonical record.
// --------------------------------------------------------------------------------
struct TopArgs {
  LatModel L;
  const int* inv_rank;
  const unsigned long long* keys;   // this model's combos (library order)
  long long ncombo;
  unsigned smask;                   // S values of this chain
  unsigned xmask;                   // S values whose rows are exactly monotone
  unsigned long long nonmono[8];    // per S: configs whose row fails kernels.py:291
  int K, Lu, g;
  const double* tab_mp;             // [S][K][Lu]
  LatWork W;
  const unsigned long long* state_key;
  const long long* off;
  const uint2* subtab;
  coral_s1_record* rec;             // this (model, phase)'s records
  double* rect;                     // their throughputs (frontier passes)
  int4* win;                        // per candidate: best value (lo, hi), S, u code << 10 | j
  const unsigned* ranks;            // [candidate][64] from lat_ranks_kernel
  unsigned long long* census;       // census on: [2] += (u, S) pairs searched
};

// One 32-byte read-only load (LDG.E.ENL2.256 on sm_100a): a row summary of LatWork.
__device__ __forceinline__ double4 ld_sum(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// dp_pair (placement_dp.cuh, kernels.py:210-239) for a top cell (l = Lu), with g(1),
// g(jmax), h(1), h(jmax) and the caps J, K taken from the two row summaries (one load
// each) instead of five scattered loads: the same shortcuts, bracket, probes and result.
__device__ __forceinline__ void top_pair(const double* __restrict__ gv, const double* __restrict__ hv,
                                         double g1, double gm, double h1, double hm, int J, int K, int l,
                                         int jmax, bool cap, double floor, double& cand, int& cj) {
  if (g1 <= h1) { cand = g1; cj = 1; return; }
  if (gm >= hm) { cand = hm; cj = jmax; return; }
  // the bound min(g(1), h(jmax)) holds for exactly monotone rows only (cap): rows
  // monotone within 1e-12 may exceed it by that much
  if (cap && (g1 < hm ? g1 : hm) <= floor) { cand = kNegInf; cj = 0; return; }
  // h(lo) and g(hi) of the final bracket are tracked instead of re-loaded: g(jmax) is
  // in the summary and g(J + 1) == 0 (J is the row's last positive column, values are
  // >= 0), so g(hi) is always known; h(lo) is known for lo == 1 or a probed lo
  int lo = 1, hi = jmax;
  double vhi = gm, vlo = h1;
  bool lo_known = true;
  if (cap) {
    hi = min(jmax, J + 1);
    lo = max(1, min(min(J, l - K - 1), hi - 1));
    if (hi < jmax) vhi = 0.0;
    lo_known = lo == 1;
  }
  const double* __restrict__ hl = hv + l;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    const double gmid = gv[mid], hmid = hl[-mid];
    if (gmid > hmid) { lo = mid; vlo = hmid; lo_known = true; } else { hi = mid; vhi = gmid; }
  }
  if (!lo_known) vlo = hl[-lo];
  if (vlo >= vhi) { cand = vlo; cj = lo; } else { cand = vhi; cj = hi; }
}

// kSlots code slots per lane (codes lane + 1 + 32k): 2 for candidates of <= 6 nodes
// (M <= 64), 4 when a model has 7-node candidates (M <= 128).
template <int kSlots, bool kScan>
__global__ void __launch_bounds__(128, 12) lat_top_kernel(TopArgs A) {
  const int lane = threadIdx.x & 31;
  const long long ci = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ci >= A.ncombo) return;
  const int Lu = A.Lu, LuP = lat_pitch(Lu);
  // one pass over the key's tokens (combo order; no per-thread arrays): M, n, the
  // config mask and the S = 1 value (f[1][L][full] = value[full][L], the same sum order)
  int M = 1, n = 0;
  unsigned long long cmask = 0ull;  // the candidate's configs
  double v1 = 0.0;
  {
    const unsigned long long key = A.keys[ci];
#pragma unroll
    for (int t = 0; t < kMaxC; ++t) {
      const unsigned tok = (unsigned)(key >> (9 * (kMaxC - 1 - t))) & 511u;
      if (!tok) break;
      const int cfg = A.inv_rank[(tok >> 3) - 1], cnt = (int)(tok & 7u);
      M *= cnt + 1;
      n += cnt;
      cmask |= 1ull << cfg;
      v1 = rn_add(v1, rn_mul((double)cnt, A.tab_mp[cfg * Lu + (Lu - 1)]));
    }
  }
  const int Smax = min(n, Lu);
  // this lane's u codes (lane+1, lane+33): size, idx(u), idx(full-u) from the model's
  // rank table (code M-1-c is the complement of code c)
  int su[kSlots];
  unsigned iu[kSlots], iy[kSlots];
  const unsigned* rk = A.ranks + ci * kRankStride;
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int code = lane + 1 + 32 * k;
    su[k] = 1 << 20;
    iu[k] = iy[k] = 0;
    if (code < M) {
      const unsigned e = rk[code], ec = rk[M - 1 - code];
      su[k] = (int)(e >> 24);
      iu[k] = e & 0xFFFFFFu;
      iy[k] = ec & 0xFFFFFFu;
    }
  }
  // S ascending; strict improvement (templates.py:322) -> smaller S on ties
  double tbest = kNegInf;
  int twin = 0, tbc = 0, npairs = 0;  // tbc: winner's u code << 10 | j
  if ((A.smask & 2u) && Smax >= 1 && !kScan && v1 > 1e-9) { tbest = v1; twin = 1; }  // S = 1
  for (int S = 2; S <= Smax; ++S) {
    if (!((A.smask >> S) & 1u)) continue;
    if (((cmask & A.nonmono[S]) != 0ull) != kScan) continue;  // the other pass's candidates at S
    const double* val = A.W.val(S);
    const double* lay = A.W.lay(S, S - 1);
    const double* vsum = A.W.vs(S);
    const double* hsum = S == 2 ? vsum : A.W.fs(S);
    double best = kNegInf;
    unsigned bc = 0xFFFFFFFFu;  // this lane's best: u code << 10 | j (code order = bc order)
    // S == 2 reads value rows on both sides: symmetric, search the lower half only
    const int chalf = (S == 2 && ((A.xmask >> 2) & 1u)) ? (M - 1) / 2 : M;
    const bool cap = (A.xmask >> S) & 1u;  // exactly monotone rows: capped crossing search
    const int jmax = Lu - (S - 1);
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      if (su[k] > n - (S - 1) || lane + 1 + 32 * k > chalf) continue;
      const double4 gs = ld_sum(vsum + (size_t)iu[k] * 4);
      const double4 hs = ld_sum(hsum + (size_t)iy[k] * 4);
      // S == 2: h(j) = value_2[Y][Lu - j]: h(1) = v[Lu-1] (.w), h(jmax) = v[1] (.y);
      // S > 2:  h(j) = f_S[S-1][Y][Lu - j]: h(1) = f[Lu-1] (.z), h(jmax) = f[S-1] (.y)
      double cand;
      int cj;
      if (kScan) {  // kernels.py:240-249 full scan (no bound: rows are not monotone)
        dp_pair(val + (size_t)iu[k] * LuP, lay + (size_t)iy[k] * LuP, Lu, jmax, false, cand, cj);
      } else {
        // only values above the best earlier S (and 1e-9) can matter (templates.py:322)
        top_pair(val + (size_t)iu[k] * LuP, lay + (size_t)iy[k] * LuP, gs.y, gs.z, S == 2 ? hs.w : hs.z, hs.y,
                 __double2loint(gs.x), __double2loint(hs.x), Lu, jmax, cap, tbest > 1e-9 ? tbest : 1e-9, cand, cj);
      }
      ++npairs;
      if (cand > best) { best = cand; bc = ((unsigned)(lane + 1 + 32 * k) << 10) | (unsigned)cj; }
    }
    // an S only matters if some lane beats the best so far (strict, templates.py:322);
    // otherwise its winning code / j are never used: skip the reduction
    if (!__any_sync(0xffffffffu, best > tbest && best > 1e-9)) continue;
    warp_argmax_packed(best, bc);
    if (best > tbest && best > 1e-9) { tbest = best; twin = S; tbc = (int)bc; }
  }
  if (A.census) {
    const unsigned np = __reduce_add_sync(0xffffffffu, (unsigned)npairs);
    if (lane == 0) atomicAdd(A.census + 2, (unsigned long long)np);
  }
  if (lane) return;
  A.win[ci] = make_int4(__double2loint(tbest), __double2hiint(tbest), twin, tbc);
}

// Walk-back of each candidate's winning S (kernels.py:258-275) into its canonical
// record (templates.py:209-228), one thread per candidate so that the dependent
// table lookups of 32 candidates overlap. Applies better_S against the record.
__global__ void __launch_bounds__(256) lat_decode_kernel(TopArgs A) {
  const long long ci = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= A.ncombo) return;
  const int4 w = A.win[ci];
  const int twin = w.z;
  if (!twin) return;
  const double tbest = __hiloint2double(w.y, w.x);
  coral_s1_record r = A.rec[ci];
  if (!better_S(tbest, twin, record_best(r), r.num_stages)) return;
  int cfg[kMaxC], cnt[kMaxC];
  const int C = lat_tokens(A.inv_rank, A.keys[ci], cfg, cnt);
  int n = 0;
  for (int c = 0; c < C; ++c) n += cnt[c];
  const int Lu = A.Lu, LuP = lat_pitch(Lu);
  int sj[kMaxC], sc[kMaxC][kMaxC];
  if (twin == 1) {
    sj[0] = Lu;
    for (int c = 0; c < C; ++c) sc[0][c] = cnt[c];
  } else {
    const int tcode = w.w >> 10, tj = w.w & 1023;
    int e[kMaxC], rest = tcode;
    for (int c = 0; c < C; ++c) { sc[0][c] = rest % (cnt[c] + 1); rest /= cnt[c] + 1; e[c] = cnt[c] - sc[0][c]; }
    sj[0] = tj;
    int sr;
    long long X = lat_rank_tokens(A.L, cfg, e, C, &sr);
    int l = Lu - tj;
    for (int s = 1; s < twin; ++s) {
      const int sg = twin - s;
      // independent loads first: state tokens, choice, sub-table offset
      const unsigned long long xkey = A.state_key[X];
      const unsigned short chv = sg > 1 ? A.W.chl(twin, sg)[X * LuP + l] : 0;
      const long long xo = A.off[X];
      int xc[kMaxC], xn[kMaxC];
      const int XC = lat_tokens(A.inv_rank, xkey, xc, xn);
      int uc = -1, j = l;
      if (sg > 1) { uc = chv >> 10; j = chv & 1023; }
      int ud[kMaxC];
      if (uc < 0) { for (int t = 0; t < XC; ++t) ud[t] = xn[t]; }
      else {
        int q = uc;
        for (int t = 0; t < XC; ++t) { ud[t] = q % (xn[t] + 1); q /= xn[t] + 1; }
      }
      for (int c = 0; c < C; ++c) {
        sc[s][c] = 0;
        for (int t = 0; t < XC; ++t) if (xc[t] == cfg[c]) sc[s][c] = ud[t];
      }
      sj[s] = j;
      if (uc >= 0) X = A.subtab[xo + uc].y;
      l -= j;
    }
  }
  canonical_record(twin, sj, sc, C, cnt, A.g, tbest, n, &A.rec[ci]);
  A.rect[ci] = tbest;
}

// --------------------------------------------------------------------------------
// placement_search operator (kernels.py:279-295), one CTA per case, raw outputs.
// --------------------------------------------------------------------------------
struct OpArgs {
  const int* ncfg;
  const long long* counts;  // [n*6]
  const int* lsteps;
  const long long* tput_off;
  const double* tput;
  const int* S;
  double* best;
  long long* stage_j;       // [n*6]
  long long* stage_counts;  // [n*36]
  int64_t ncases;
};

__global__ void __launch_bounds__(kDpThreads) placement_op_kernel(OpArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ DpShared sh;
  const int64_t i = blockIdx.x;
  if (i >= A.ncases) return;
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh.C = A.ncfg[i];
    for (int c = 0; c < sh.C; ++c) sh.cnt[c] = (int)A.counts[i * kMaxC + c];
    sh.Lu = A.lsteps[i];
    sh.LuP = sh.Lu + 1;
  }
  __syncthreads();
  dp_setup_lattice(sh);
  const int S = A.S[i];
  const int Lu = sh.Lu, LuP = sh.LuP, C = sh.C, M = sh.M, n = sh.n;
  for (int s = tid; s < kMaxC; s += blockDim.x) {
    A.stage_j[i * kMaxC + s] = 0;
    for (int c = 0; c < kMaxC; ++c) A.stage_counts[(i * kMaxC + s) * kMaxC + c] = 0;
  }
  if (S > n || S > Lu || S < 1) {  // kernels.py:174-175
    if (tid == 0) A.best[i] = kNegInf;
    return;
  }
  const DpBuffers B = dp_carve(smem, M, LuP, Lu, n - 2);
  const double* rows = A.tput + A.tput_off[i];
  for (int idx = tid; idx < C * Lu; idx += blockDim.x) B.tputS[idx] = rows[idx];
  __syncthreads();
  if (tid == 0) {
    int mono = 1;  // kernels.py:291
    for (int c = 0; c < C; ++c)
      for (int j = 0; j + 1 < Lu; ++j) mono &= (rn_sub(B.tputS[c * Lu + j + 1], B.tputS[c * Lu + j]) <= 1e-12);
    sh.mono = mono;
  }
  dp_build_value(sh, B);
  __syncthreads();
  if (S == 1) {
    if (tid == 0) { sh.top_val = B.value[(M - 1) * LuP + Lu]; sh.top_u = M - 1; sh.top_j = Lu; }
    __syncthreads();
  } else {
    dp_run(sh, B, S);
  }
  if (tid == 0) {
    const double best = sh.top_val;
    if (best <= kNegInf / 2) { A.best[i] = kNegInf; return; }
    if (S == 1) { sh.stage_j[0] = Lu; sh.stage_u[0] = M - 1; }
    else dp_decode(sh, B, S);
    A.best[i] = best;
    for (int s = 0; s < S; ++s) {
      A.stage_j[i * kMaxC + s] = sh.stage_j[s];
      for (int c = 0; c < C; ++c) A.stage_counts[(i * kMaxC + s) * kMaxC + c] = sh.digits[sh.stage_u[s]][c];
    }
  }
}

// --------------------------------------------------------------------------------
// Frontier
// --------------------------------------------------------------------------------
struct FrontArgs {
  DevProblem P;
  const unsigned long long* keys;
  const int64_t* koff;
  const int64_t* cand_off;
  int NMP;
  const coral_s1_record* rec;
  int64_t ncand;
  const double* prices;  // [R][K], NaN = not offered
  const double* tok_price = nullptr;  // [R][512] count x price per packed token (frontier passes)
  int R;
  coral_s1_frontier_item* items;
  unsigned long long* nitems;
  unsigned long long cap = 0;      // items capacity (frontier_items_kernel counts past it)
  // the prefilter passes run over the models this device evaluated (one or both of
  // their phases): run k (model run_mp[k], phase mask run_ph[k]) owns blocks
  // run_boff[k] .. run_boff[k+1] - 1, kFrontBlock of the model's candidates each
  const int64_t* run_boff = nullptr;
  const double* rect = nullptr;    // per candidate: the record's throughput, 0 = no template
  const int64_t* run_off = nullptr;
  const int* run_mp = nullptr;
  const unsigned char* run_ph = nullptr;
  int nrun = 0;
  int64_t ntot = 0;
};

// The frontier passes: thread t of a block serves the model candidates base + k * 256 + t,
// k < kFrontItems (coalesced per k; all loads issued before the dependent pricing). A
// candidate's key is read and priced once for both phases -- a combo costs the same in
// both -- and its records' throughputs come from the compact per-phase arrays (8 B), the
// 32-byte records being re-read for survivors only.
constexpr int kFrontPhases = 2, kFrontItems = 4, kFrontBlock = 256 * kFrontItems;

// The block's run (one binary search per block, not per thread).
__device__ __forceinline__ int frontier_block_run(const FrontArgs& A) {
  __shared__ int s_run;
  if (threadIdx.x == 0) {
    int lo = 0, hi = A.nrun;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (A.run_boff[mid] <= (int64_t)blockIdx.x) lo = mid; else hi = mid;
    }
    s_run = lo;
  }
  __syncthreads();
  return s_run;
}

// This thread's candidates of the block's run: model m, the index of the first, and per
// item the phase throughputs (0 = no template or phase not evaluated here) and the key
// (0 when no phase has a template).
struct FrontItems {
  int m;
  int64_t idx0;
  double T[kFrontItems][kFrontPhases];
  unsigned long long key[kFrontItems];
};
__device__ __forceinline__ void frontier_load(const FrontArgs& A, FrontItems& F) {
  const int run = frontier_block_run(A);
  const int m = A.run_mp[run];
  const unsigned own = A.run_ph[run];
  const int NP = A.P.NP;
  F.m = m;
  F.idx0 = ((int64_t)blockIdx.x - A.run_boff[run]) * kFrontBlock + threadIdx.x;
  const int64_t n = A.cand_off[m * NP + 1] - A.cand_off[m * NP];
#pragma unroll
  for (int k = 0; k < kFrontItems; ++k) {
    const int64_t idx = F.idx0 + (int64_t)k * 256;
#pragma unroll
    for (int p = 0; p < kFrontPhases; ++p)
      F.T[k][p] = (idx < n && p < NP && ((own >> p) & 1u)) ? A.rect[A.cand_off[m * NP + p] + idx] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kFrontItems; ++k) {
    const int64_t idx = F.idx0 + (int64_t)k * 256;
    F.key[k] = (F.T[k][0] > 0.0 || F.T[k][1] > 0.0) ? A.keys[A.koff[m] + idx] : 0ull;
  }
}
// Token prices of every region, tp[r * 512 + token] = count x the config's price in
// region r (rn_mul on the host: the same IEEE product allocation.py:97 computes as n * p;
// NaN when the config is unpriced there, which then propagates through the sum), read
// through the read-only cache: one load + add per token instead of a config lookup, a
// price load and a multiply.
// allocation.py:91-98 _template_price of the candidate in region r (combo order,
// sequential); false when a config is not offered there (price None). Tokens are
// contiguous from the top of the key: the first zero token ends the combo.
__device__ __forceinline__ bool frontier_price(const FrontArgs& A, unsigned long long key, int r, double& total) {
  total = 0.0;
  const double* __restrict__ row = A.tok_price + r * 512;
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) {
    const unsigned tok = (unsigned)(key >> (kKeyTokenBits * (kMaxC - 1 - c))) & 511u;
    if (tok) total = rn_add(total, __ldg(row + tok));
  }
  return !isnan(total);
}
__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);  // monotone for x >= 0
}

// price bucket: top bits of the (non-negative) price's bit pattern relative to the range
// start, clamped to [0, nb) -- a non-decreasing map of the price
__device__ __forceinline__ int bucket_of(double price, int shift, unsigned long long base, int nb) {
  const unsigned long long q = dbits(price) >> shift;
  if (q <= base) return 0;
  const unsigned long long d = q - base;
  return d >= (unsigned long long)nb ? nb - 1 : (int)d;
}

// pass 1: per (segment, price bucket) the max throughput (bit pattern, T > 0)
__global__ void __launch_bounds__(256) frontier_bucket_kernel(FrontArgs A, int shift, unsigned long long base,
                                                              int nb, unsigned long long* __restrict__ bmax) {
  FrontItems F;
  frontier_load(A, F);
  const int NP = A.P.NP;
#pragma unroll
  for (int k = 0; k < kFrontItems; ++k) {
    if (!F.key[k]) continue;
    for (int r = 0; r < A.R; ++r) {
      double price;
      if (!frontier_price(A, F.key[k], r, price)) continue;
      const int b = bucket_of(price, shift, base, nb);
#pragma unroll
      for (int p = 0; p < kFrontPhases; ++p) {
        if (!(F.T[k][p] > 0.0)) continue;
        const unsigned long long tb = dbits(F.T[k][p]);
        // most items do not raise their bucket: read first (an unconditional atomic per
        // item serialises on the hot buckets, 2.5x slower at config 5)
        unsigned long long* slot = bmax + ((int64_t)(F.m * NP + p) * A.R + r) * nb + b;
        if (*slot < tb) atomicMax(slot, tb);
      }
    }
  }
}
// pass 2: exclusive prefix max over the buckets of each segment (block per segment)
__global__ void frontier_prefix_kernel(int nb, unsigned long long* __restrict__ bmax) {
  typedef cub::BlockScan<unsigned long long, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  unsigned long long* row = bmax + (int64_t)blockIdx.x * nb;
  const int per = (nb + 255) / 256;
  const int b0 = threadIdx.x * per;
  unsigned long long local = 0;
  for (int b = b0; b < min(b0 + per, nb); ++b) local = max(local, row[b]);
  unsigned long long excl;
  Scan(tmp).ExclusiveScan(local, excl, 0ull, cub::Max());
  __syncthreads();
  unsigned long long run = excl;
  for (int b = b0; b < min(b0 + per, nb); ++b) {
    const unsigned long long v = row[b];
    row[b] = run;  // max over strictly cheaper buckets
    run = max(run, v);
  }
}

// pass 3: write the items that can still be on the frontier: T must exceed every
// throughput of a strictly cheaper bucket, else a cheaper candidate dominates it
// (SURVEY.md 8c keep rule: T > running max of the earlier items).
__global__ void __launch_bounds__(256) frontier_items_kernel(FrontArgs A, int shift, unsigned long long base,
                                                             int nb, const unsigned long long* __restrict__ pmax) {
  FrontItems F;
  frontier_load(A, F);
  const int lane = threadIdx.x & 31;
  const int NP = A.P.NP;
#pragma unroll
  for (int k = 0; k < kFrontItems; ++k) {
    if (!__any_sync(0xffffffffu, F.key[k] != 0ull)) continue;  // warp-uniform
    for (int r = 0; r < A.R; ++r) {  // uniform over the warp: ballots stay converged
      double price = 0.0;
      const bool priced = F.key[k] && frontier_price(A, F.key[k], r, price);
      const int b = priced && nb > 0 ? bucket_of(price, shift, base, nb) : 0;
#pragma unroll
      for (int p = 0; p < kFrontPhases; ++p) {
        if (p >= NP) break;
        const int mp = F.m * NP + p;
        bool keep = priced && F.T[k][p] > 0.0;
        if (keep && nb > 0) keep = dbits(F.T[k][p]) > pmax[((int64_t)mp * A.R + r) * nb + b];
        const unsigned ballot = __ballot_sync(0xffffffffu, keep);
        if (!ballot) continue;
        unsigned long long pos = 0;
        if (lane == __ffs(ballot) - 1) pos = atomicAdd(A.nitems, (unsigned long long)__popc(ballot));
        pos = __shfl_sync(0xffffffffu, pos, __ffs(ballot) - 1);
        if (keep && pos + __popc(ballot & ((1u << lane) - 1u)) < A.cap) {  // bounded buffer: count the rest
          coral_s1_frontier_item it;
          it.price_usd_h = price;
          it.throughput_tps = F.T[k][p];
          it.combo_key = F.key[k];
          it.mp = mp;
          it.region = r;
          it.rec = A.rec[A.cand_off[mp] + F.idx0 + (int64_t)k * 256];
          A.items[pos + __popc(ballot & ((1u << lane) - 1u))] = it;
        }
      }
    }
  }
}
// cmd_sweep statistics (cli.py:233-272) for several LibraryCaps at once from one
// solve at the widest caps: DP records do not depend on the caps, only the
// enumeration window does (templates.py:107-111). Per candidate: window test per caps
// entry, price = min over regions of the combo-order sum (regions with an unpriced
// config skipped), efficiency T / price; per entry count + max efficiency.
__global__ void sweep_kernel(FrontArgs A, int ncaps, const int* __restrict__ cap_n,
                             const double* __restrict__ cap_rho, unsigned phase_mask,
                             unsigned long long* __restrict__ counts,
                             unsigned long long* __restrict__ best_bits,
                             unsigned long long* __restrict__ unpriced,
                             unsigned long long* __restrict__ mp_counts) {
  const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= A.ncand) return;
  const coral_s1_record rc = A.rec[ci];
  if (rc.num_stages == 0) return;
  int lo = 0, hi = A.NMP;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (A.cand_off[mid] <= ci) lo = mid; else hi = mid;
  }
  if (!((phase_mask >> (lo % A.P.NP)) & 1u)) return;
  const int m = lo / A.P.NP;
  const unsigned long long key = A.keys[A.koff[m] + (ci - A.cand_off[lo])];
  int cfg[kMaxC], cnt[kMaxC];
  const int C = decode_key(A.P, key, cfg, cnt);
  double mem = 0.0;
  int n = 0;
  for (int c = 0; c < C; ++c) {
    n += cnt[c];
    for (int k = 0; k < cnt[c]; ++k) mem = rn_add(mem, A.P.mem_bytes[cfg[c]]);
  }
  // cli.py:253-258: min over every region of the combo-order sum; the reference indexes
  // scenario.prices[(region, config)] directly, so an unpriced config is an error there
  double price = __longlong_as_double(0x7ff0000000000000ll);
  bool all_priced = A.R > 0;
  for (int r = 0; r < A.R; ++r) {
    double total = 0.0;
    bool ok = true;
    for (int c = 0; c < C; ++c) {
      const double p = A.prices[(int64_t)r * A.P.K + cfg[c]];
      if (isnan(p)) { ok = false; break; }
      total = rn_add(total, rn_mul((double)cnt[c], p));
    }
    all_priced &= ok;
    if (ok && total < price) price = total;
  }
  const bool priced = isfinite(price);
  const double eff = priced ? rn_div(rc.throughput_tps, price) : 0.0;
  const double w = rn_mul(rn_mul(A.P.ptb[m], 1e9), A.P.bpp[m]);
  for (int k = 0; k < ncaps; ++k) {
    if (n > cap_n[k] || !(w <= mem && mem < rn_mul(cap_rho[k], w))) continue;
    atomicAdd(counts + k, 1ull);
    atomicAdd(mp_counts + (int64_t)k * A.NMP + lo, 1ull);
    if (!all_priced) atomicAdd(unpriced + k, 1ull);
    if (priced) atomicMax(best_bits + k, (unsigned long long)__double_as_longlong(eff));
  }
}

// feasible templates per (model, phase) of the last evaluate (templates.py:499-502 check)
__global__ void feasible_count_kernel(const coral_s1_record* __restrict__ rec, const int64_t* __restrict__ cand_off,
                                      int NMP, int64_t ncand, unsigned long long* __restrict__ out) {
  const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool f = ci < ncand && rec[ci].num_stages != 0;
  int mp = 0;
  if (ci < ncand) {
    int lo = 0, hi = NMP;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (cand_off[mid] <= ci) lo = mid; else hi = mid;
    }
    mp = lo;
  }
  // one atomic per run of equal mp in the warp
  const unsigned peers = __match_any_sync(0xffffffffu, f ? mp : -1);
  if (f && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(out + mp, (unsigned long long)__popc(peers));
}

// --------------------------------------------------------------------------------
// Stage-2 model construction: build_allocation_model
// (allocation.py:108-195) over the device records. Per (model, phase) slot with demand
// > 0, every (template, region) with a price is a candidate variable: eff = p / T, the
// slot's best eff, the prune rule (eff > ratio x best unless already running), the
// availability cap min over the combo of avail // n, and ub = min(cap, ceil(demand / T));
// ub <= 0 drops it. Variables come out in the reference's insertion order: slots in
// library order, templates in library (str) order, regions in market order.
// --------------------------------------------------------------------------------
struct AllocArgs {
  DevProblem P;
  const unsigned long long* keys;
  const int64_t* koff;
  const int64_t* cand_off;
  const coral_s1_record* rec;
  const double* prices;           // [R][K], NaN = unpriced (allocation.py:91-98 None)
  const long long* avail;         // [R][K] MarketState.available
  const double* demand;           // [NMP]
  int R;
  double prune_ratio;
  // running (region, template) pairs, sorted by (mp, key, region)
  const int* run_mp;
  const int* run_region;
  const unsigned long long* run_key;
  long long nrunning;
  // slots in library order with their candidates: thread t -> run k -> mp = runs_mp[k]
  const int64_t* runs_off;
  const int* runs_mp;
  int nruns;
  int64_t ntot;
  unsigned long long* best_bits;  // [NMP] min eff (bit pattern; eff >= 0)
  unsigned* flags;                // [ntot] region bit mask of kept variables
  unsigned long long* blkcnt;     // per block kept count
  unsigned long long* npruned;    // meta["pruned_vars"] (allocation.py:146-148)
  coral_s1_alloc_var* out;
  const unsigned long long* blkoff;
};

struct AllocCand {
  int mp, C;
  unsigned long long key;
  double T;
  int cfg[kMaxC], cnt[kMaxC];
};

__device__ __forceinline__ bool alloc_cand(const AllocArgs& A, int64_t t, AllocCand& f) {
  if (t >= A.ntot) return false;
  int lo = 0, hi = A.nruns;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (A.runs_off[mid] <= t) lo = mid; else hi = mid;
  }
  f.mp = A.runs_mp[lo];
  const int64_t idx = t - A.runs_off[lo];
  const coral_s1_record& r = A.rec[A.cand_off[f.mp] + idx];
  if (r.num_stages == 0) return false;  // not a template
  f.T = r.throughput_tps;
  f.key = A.keys[A.koff[f.mp / A.P.NP] + idx];
  f.C = decode_key(A.P, f.key, f.cfg, f.cnt);
  return true;
}

__device__ __forceinline__ bool alloc_price(const AllocArgs& A, const AllocCand& f, int r, double& p) {
  p = 0.0;
  for (int c = 0; c < f.C; ++c) {
    const double x = A.prices[(int64_t)r * A.P.K + f.cfg[c]];
    if (isnan(x)) return false;
    p = rn_add(p, rn_mul((double)f.cnt[c], x));
  }
  return true;
}

__global__ void alloc_best_kernel(AllocArgs A) {
  AllocCand f;
  if (!alloc_cand(A, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, f)) return;
  for (int r = 0; r < A.R; ++r) {
    double p;
    if (!alloc_price(A, f, r, p)) continue;
    const unsigned long long e = (unsigned long long)__double_as_longlong(rn_div(p, f.T));
    if (e < A.best_bits[f.mp]) atomicMin(A.best_bits + f.mp, e);
  }
}

__device__ __forceinline__ bool alloc_running(const AllocArgs& A, int mp, unsigned long long key, int r) {
  long long lo = 0, hi = A.nrunning;  // first entry >= (mp, key, r)
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    const bool less = A.run_mp[mid] != mp ? A.run_mp[mid] < mp
                    : A.run_key[mid] != key ? A.run_key[mid] < key : A.run_region[mid] < r;
    if (less) lo = mid + 1; else hi = mid;
  }
  return lo < A.nrunning && A.run_mp[lo] == mp && A.run_key[lo] == key && A.run_region[lo] == r;
}

// the variable (f, r) if it is kept: its ub
// -1: pruned (allocation.py:143-148)
__device__ __forceinline__ long long alloc_ub(const AllocArgs& A, const AllocCand& f, int r, double p) {
  const double eff = rn_div(p, f.T);
  const double best = __longlong_as_double((long long)A.best_bits[f.mp]);
  if (A.prune_ratio != 0.0 && eff > rn_mul(A.prune_ratio, best) && !alloc_running(A, f.mp, f.key, r)) return -1;
  long long cap = LLONG_MAX;
  for (int c = 0; c < f.C; ++c) {
    const long long a = A.avail[(int64_t)r * A.P.K + f.cfg[c]];
    const long long q = a >= 0 ? a / f.cnt[c] : -((-a + f.cnt[c] - 1) / f.cnt[c]);  // Python //
    cap = q < cap ? q : cap;
  }
  const double need = ceil(rn_div(A.demand[f.mp], f.T));
  const long long ub = (double)cap < need ? cap : (long long)need;
  return ub;
}

constexpr int kAllocThreads = 256;

__global__ void __launch_bounds__(kAllocThreads) alloc_count_kernel(AllocArgs A) {
  __shared__ int ws[kAllocThreads / 32];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  AllocCand f;
  unsigned mask = 0u;
  if (alloc_cand(A, t, f))
    for (int r = 0; r < A.R; ++r) {
      double p;
      if (!alloc_price(A, f, r, p)) continue;
      const long long ub = alloc_ub(A, f, r, p);
      if (ub > 0) mask |= 1u << r;
      else if (ub < 0) atomicAdd(A.npruned, 1ull);
    }
  if (t < A.ntot) A.flags[t] = mask;
  int c = __reduce_add_sync(0xffffffffu, __popc(mask));
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kAllocThreads / 32; ++w) s += ws[w];
    A.blkcnt[blockIdx.x] = (unsigned long long)s;
  }
}

__global__ void __launch_bounds__(kAllocThreads) alloc_emit_kernel(AllocArgs A) {
  __shared__ int ws[kAllocThreads / 32];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned mask = t < A.ntot ? A.flags[t] : 0u;
  const int c = __popc(mask);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (!mask) return;
  int before = 0;
  for (int w = 0; w < warp; ++w) before += ws[w];
  unsigned long long o = A.blkoff[blockIdx.x] + (unsigned long long)(before + incl - c);
  AllocCand f;
  alloc_cand(A, t, f);
  for (int r = 0; r < A.R; ++r) {
    if (!((mask >> r) & 1u)) continue;
    double p;
    alloc_price(A, f, r, p);
    coral_s1_alloc_var v;
    v.combo_key = f.key;
    v.mp = f.mp;
    v.region = r;
    v.ub = alloc_ub(A, f, r, p);
    v.price_usd_h = p;
    v.throughput_tps = f.T;
    A.out[o++] = v;
  }
}

// Batched T-hat queries (perf.py:159-230) against the current spec tables: the
// simulator-side reuse of the roofline model.
__global__ void node_query_kernel(DevProblem P, int64_t n, const int* __restrict__ cfg,
                                  const int* __restrict__ model, const int* __restrict__ phase,
                                  const int* __restrict__ j, const double* __restrict__ budget,
                                  int use_profile, double* __restrict__ tput, long long* __restrict__ batch) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long b = 0;
  double t;
  double hit;
  if (use_profile && profile_lookup(P, cfg[i], model[i], phase[i], j[i], budget[i], &hit)) t = hit;
  else t = planned_batch_and_tput(P, cfg[i], model[i], phase[i], j[i], budget[i], &b);
  tput[i] = t;
  batch[i] = b;
}

// Frontier order: segment asc, price asc, T desc, combo key asc,
// stages asc -- the last only separates the per-rank partial records of one
// (model, phase, combo) in the multi-GPU merge (fewer stages first, the
// templates.py:322 tie rule). One 40-byte composite key, compared lexicographically.
struct FrontKey {
  unsigned seg, idx;            // segment = mp * R + region; idx = position in items
  unsigned long long price;     // bit pattern of price >= 0 (orders like the value)
  unsigned long long neg_t;     // ~bits(T), T > 0: ascending = T descending
  unsigned long long key;       // packed combo key (63 bits)
  unsigned stages, pad;         // num_stages
};

struct FrontLess {
  __device__ __forceinline__ bool operator()(const FrontKey& a, const FrontKey& b) const {
    if (a.seg != b.seg) return a.seg < b.seg;
    if (a.price != b.price) return a.price < b.price;
    if (a.neg_t != b.neg_t) return a.neg_t < b.neg_t;
    if (a.key != b.key) return a.key < b.key;
    return a.stages < b.stages;
  }
};

__global__ void front_keys_kernel(const coral_s1_frontier_item* __restrict__ items, int64_t n, int R,
                                  FrontKey* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const coral_s1_frontier_item& it = items[i];
  FrontKey k;
  k.seg = (unsigned)it.mp * (unsigned)R + (unsigned)it.region;
  k.idx = (unsigned)i;
  k.price = (unsigned long long)__double_as_longlong(it.price_usd_h);
  k.neg_t = ~(unsigned long long)__double_as_longlong(it.throughput_tps);
  k.key = it.combo_key;
  k.stages = it.rec.num_stages;
  k.pad = 0u;
  out[i] = k;
}

__global__ void gather_items_kernel(const coral_s1_frontier_item* __restrict__ in,
                                    const FrontKey* __restrict__ order, int64_t n,
                                    coral_s1_frontier_item* __restrict__ out,
                                    unsigned long long* __restrict__ seg, double* __restrict__ tv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const FrontKey k = order[i];
  const coral_s1_frontier_item it = in[k.idx];
  out[i] = it;
  seg[i] = k.seg;
  tv[i] = it.throughput_tps;
}

struct MaxOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return b > a ? b : a; }
};

// keep iff T > running max of the earlier items of the segment (strict)
__global__ void skyline_flags_kernel(const unsigned long long* __restrict__ seg,
                                     const double* __restrict__ tv, const double* __restrict__ incl,
                                     int64_t n, unsigned char* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || seg[i] != seg[i - 1] || tv[i] > incl[i - 1]) ? 1 : 0;
}

// ---- Frontier skyline, hand-written: one CTA per segment -----------------
// The CTA of segment s collects its items from every part (one part on one GPU; the
// gathered per-rank partial frontiers in the multi-GPU merge) into shared memory, sorts
// them (bitonic) by (price asc, T desc, combo key asc, stages asc), keeps an item iff its
// T exceeds the running max of the items before it (block max-scan), and stages the
// survivors' ordinals; front_emit_kernel writes them compacted, segment by segment.
// Segments larger than kSegCap items take the general path (frontier_from_items_general).
constexpr int kSegThreads = 1024, kSegCap = 4096, kMaxParts = 32;
constexpr int kSegPrefilter = 512;  // segments above this take a bucket prefilter before the sort

struct SegKey {
  unsigned long long price;  // bit pattern of price >= 0 (orders like the value)
  unsigned long long neg_t;  // ~bits(T), T > 0: ascending = T descending
  unsigned long long key;    // packed combo key
  unsigned long long s_ord;  // num_stages << 32 | item ordinal (fewer stages first)
};

__device__ __forceinline__ bool seg_less(const SegKey& a, const SegKey& b) {
  if (a.price != b.price) return a.price < b.price;
  if (a.neg_t != b.neg_t) return a.neg_t < b.neg_t;
  if (a.key != b.key) return a.key < b.key;
  return a.s_ord < b.s_ord;
}

struct FrontParts {
  const unsigned char* base;  // part p's items at base + p * stride + offset
  long long stride, offset;
  int nparts, R;
  long long n[kMaxParts];     // items per part
  long long first[kMaxParts + 1];  // ordinal of each part's first item
  // device-side counts instead (parts_counts_kernel: n at dn[p], first at dn[kMaxParts + p]),
  // so a gathered buffer merges without a host round trip for its headers
  const long long* dn = nullptr;
  __device__ __forceinline__ long long cnt(int p) const { return dn ? dn[p] : n[p]; }
  __device__ __forceinline__ long long fst(int p) const { return dn ? dn[kMaxParts + p] : first[p]; }
  __device__ __forceinline__ const coral_s1_frontier_item& item(int p, long long i) const {
    return reinterpret_cast<const coral_s1_frontier_item*>(base + p * stride + offset)[i];
  }
  __device__ __forceinline__ const coral_s1_frontier_item& by_ord(long long o) const {
    int p = 0;
    while (p + 1 < nparts && fst(p + 1) <= o) ++p;
    return item(p, o - fst(p));
  }
};

constexpr int kPartsCountsLen = 2 * kMaxParts + 2;

// Headers of a gathered buffer (int64 item count at base + p * stride; a count above
// `cap` means that part overflowed its slot) -> dn: n[p] = min(count, cap), first[p],
// and dn[2 * kMaxParts + 1] = the largest count (the host checks it for overflow).
__global__ void parts_counts_kernel(const unsigned char* __restrict__ base, long long stride, int nparts,
                                    long long cap, long long* __restrict__ dn) {
  if (threadIdx.x) return;
  long long at = 0, mx = 0;
  for (int p = 0; p < nparts; ++p) {
    const long long c = *reinterpret_cast<const long long*>(base + p * stride);
    mx = c > mx ? c : mx;
    const long long k = c < cap ? c : cap;
    dn[p] = k;
    dn[kMaxParts + p] = at;
    at += k;
  }
  dn[kMaxParts + nparts] = at;
  dn[2 * kMaxParts + 1] = mx;
}

// block-wide exclusive scan (sum or max) of one value per thread; 1024 threads
template <bool kMax>
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* s_warp,
                                                             unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = kMax ? (t > incl ? t : incl) : incl + t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = s_warp[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi = kMax ? (t > wi ? t : wi) : wi + t;
    }
    s_warp[lane] = wi;  // inclusive over warps
  }
  __syncthreads();
  const unsigned long long before = warp ? s_warp[warp - 1] : 0ull;
  unsigned long long ex;
  if (kMax) {  // exclusive max: the previous lane's inclusive value, then the earlier warps
    const unsigned long long up = __shfl_up_sync(0xffffffffu, incl, 1);
    const unsigned long long lanepre = lane ? up : 0ull;
    ex = lanepre > before ? lanepre : before;
  } else {
    ex = before + incl - v;
  }
  if (total) *total = s_warp[31];
  __syncthreads();
  return ex;
}

__global__ void __launch_bounds__(kSegThreads) front_segment_kernel(FrontParts F, int nseg,
                                                                    unsigned* __restrict__ staged,
                                                                    unsigned* __restrict__ surv,
                                                                    unsigned* __restrict__ overflow) {
  extern __shared__ SegKey s_keys[];  // [kSegCap]
  __shared__ unsigned s_cnt;
  __shared__ unsigned long long s_warp[32];
  const int seg = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) s_cnt = 0u;
  __syncthreads();
  for (int p = 0; p < F.nparts; ++p) {
    const long long np = F.cnt(p), fp = F.fst(p);
    for (long long i = tid; i < np; i += kSegThreads) {
      const coral_s1_frontier_item& it = F.item(p, i);
      const int2 mr = *reinterpret_cast<const int2*>(&it.mp);  // (mp, region)
      if (mr.x * F.R + mr.y != seg) continue;
      const unsigned pos = atomicAdd(&s_cnt, 1u);
      if (pos < kSegCap) {
        SegKey k;
        k.price = (unsigned long long)__double_as_longlong(it.price_usd_h);
        k.neg_t = ~(unsigned long long)__double_as_longlong(it.throughput_tps);
        k.key = it.combo_key;
        k.s_ord = ((unsigned long long)it.rec.num_stages << 32) | (unsigned long long)(fp + i);
        s_keys[pos] = k;
      }
    }
  }
  __syncthreads();
  int cnt = (int)s_cnt;
  if (cnt > kSegCap) {
    if (tid == 0) { atomicOr(overflow, 1u); surv[seg] = 0u; }
    return;
  }
  if (cnt > kSegPrefilter) {
    // a large segment (few segments, many items: the multi-GPU merge of a one-model
    // config): the exact bucket prefilter of the frontier passes again, over this
    // segment's union, before its sort -- per price bucket (top bits of the price's bit
    // pattern over the segment's own range: a non-decreasing map) the max T; an item
    // goes only if a strictly cheaper bucket holds a T >= its T (a cheaper item that
    // precedes and dominates it). The kept set contains every survivor, so the sort
    // and running-max skyline below stay exact on fewer items.
    __shared__ unsigned long long s_bkt[kSegThreads];
    unsigned long long lmx = 0ull, lmn = 0ull;  // max price bits, max of ~price bits
    for (int i = tid; i < cnt; i += kSegThreads) {
      const unsigned long long pb = s_keys[i].price;
      lmx = pb > lmx ? pb : lmx;
      lmn = ~pb > lmn ? ~pb : lmn;
    }
    unsigned long long hi_b = 0ull, lo_nb = 0ull;
    block_excl_scan<true>(lmx, s_warp, &hi_b);
    block_excl_scan<true>(lmn, s_warp, &lo_nb);
    const unsigned long long lo_b = ~lo_nb;
    int shift = 0;  // block-uniform
    while (((hi_b >> shift) - (lo_b >> shift)) >= (unsigned long long)kSegThreads) ++shift;
    const unsigned long long base = lo_b >> shift;
    s_bkt[tid] = 0ull;
    __syncthreads();
    for (int i = tid; i < cnt; i += kSegThreads) {
      const int b = (int)((s_keys[i].price >> shift) - base);
      const unsigned long long tb = ~s_keys[i].neg_t;
      if (s_bkt[b] < tb) atomicMax(&s_bkt[b], tb);
    }
    __syncthreads();
    const unsigned long long pre = block_excl_scan<true>(s_bkt[tid], s_warp, nullptr);  // strictly cheaper
    s_bkt[tid] = pre;
    __syncthreads();
    constexpr int kPer = kSegCap / kSegThreads;
    SegKey mine[kPer];
    unsigned live = 0u;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int i = tid + r * kSegThreads;
      if (i < cnt) {
        mine[r] = s_keys[i];
        if (~mine[r].neg_t > s_bkt[(int)((mine[r].price >> shift) - base)]) live |= 1u << r;
      }
    }
    unsigned long long total = 0ull;
    unsigned o = (unsigned)block_excl_scan<false>((unsigned long long)__popc(live), s_warp, &total);  // syncs
#pragma unroll
    for (int r = 0; r < kPer; ++r)
      if ((live >> r) & 1u) s_keys[o++] = mine[r];
    __syncthreads();
    cnt = (int)total;
  }
  int np2 = 1;
  while (np2 < cnt) np2 <<= 1;
  for (int i = cnt + tid; i < np2; i += kSegThreads) {
    SegKey k;
    k.price = k.neg_t = k.key = k.s_ord = ~0ull;  // sentinel: sorts last
    s_keys[i] = k;
  }
  __syncthreads();
  // bitonic sort of np2 keys
  for (int size = 2; size <= np2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < (np2 >> 1); t += kSegThreads) {
        const int i = 2 * t - (t & (stride - 1));  // lower index of the pair
        const int j = i + stride;
        const bool up = (i & size) == 0;
        SegKey a = s_keys[i], b = s_keys[j];
        if (seg_less(b, a) == up) { s_keys[i] = b; s_keys[j] = a; }
      }
      __syncthreads();
    }
  }
  // skyline: thread t owns sorted positions [t*per, t*per + per)
  const int per = (cnt + kSegThreads - 1) / kSegThreads;
  const int b0 = min(tid * per, cnt), b1 = min(b0 + per, cnt);
  unsigned long long lmax = 0ull;  // T bits; every T > 0
  for (int i = b0; i < b1; ++i) {
    const unsigned long long tb = ~s_keys[i].neg_t;
    lmax = tb > lmax ? tb : lmax;
  }
  unsigned long long run = block_excl_scan<true>(lmax, s_warp, nullptr);
  unsigned keep = 0u;  // bit k: position b0 + k survives (per <= 4)
  for (int i = b0; i < b1; ++i) {
    const unsigned long long tb = ~s_keys[i].neg_t;
    if (tb > run) { keep |= 1u << (i - b0); run = tb; }
  }
  unsigned long long total = 0ull;
  const unsigned long long at = block_excl_scan<false>((unsigned long long)__popc(keep), s_warp, &total);
  unsigned o = (unsigned)at;
  for (int i = b0; i < b1; ++i)
    if ((keep >> (i - b0)) & 1u) staged[(long long)seg * kSegCap + o++] = (unsigned)(s_keys[i].s_ord & 0xFFFFFFFFull);
  if (tid == 0) surv[seg] = (unsigned)total;
}

// survivors of segment s -> out at the sum of the earlier segments' survivor counts
__global__ void __launch_bounds__(256) front_emit_kernel(FrontParts F, int nseg, const unsigned* __restrict__ staged,
                                                         const unsigned* __restrict__ surv,
                                                         coral_s1_frontier_item* __restrict__ out,
                                                         long long* __restrict__ ntotal) {
  __shared__ unsigned long long s_part[8];
  const int seg = blockIdx.x;
  unsigned long long pre = 0ull;
  for (int s = threadIdx.x; s < seg; s += blockDim.x) pre += surv[s];
  pre = __reduce_add_sync(0xffffffffu, (unsigned)pre);  // < 2^32 survivors
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = pre;
  __syncthreads();
  unsigned long long base = 0ull;
  for (int w = 0; w < 8; ++w) base += s_part[w];
  const unsigned ns = surv[seg];
  for (unsigned k = threadIdx.x; k < ns; k += blockDim.x)
    out[base + k] = F.by_ord(staged[(long long)seg * kSegCap + k]);
  if (seg == nseg - 1 && threadIdx.x == 0) *ntotal = (long long)(base + ns);
}

int ensure_tmp(coral_s1_handle* h, size_t bytes) { return h->cub_tmp.ensure(bytes); }

// General frontier over n items already in h->items (any segment size: stable merge sort
// + segmented max scan + compaction); survivors -> h->front, count -> h->nfront.
int frontier_from_items_general(coral_s1_handle* h, int64_t n, int R) {
  cudaStream_t st = h->stream;
  h->nfront = 0;
  if (n == 0) return 0;
  int rc;
  if ((rc = h->sort_a.ensure(n * sizeof(FrontKey))) || (rc = h->sort_b.ensure(n * 8)) ||
      (rc = h->items_sorted.ensure(n * sizeof(coral_s1_frontier_item))) ||
      (rc = h->segk.ensure(n * 8)) || (rc = h->scanv.ensure(n * 8)) ||
      (rc = h->flagsel.ensure(n)) || (rc = h->nsel.ensure(32)))
    return rc;
  const int TB = 256;
  const unsigned gb = (unsigned)((n + TB - 1) / TB);
  const coral_s1_frontier_item* items = h->items.as<coral_s1_frontier_item>();
  FrontKey* keys = h->sort_a.as<FrontKey>();
  front_keys_kernel<<<gb, TB, 0, st>>>(items, n, R, keys);
  LAUNCH_CHECK(h);
  {
    size_t tmp = 0;
    cub::DeviceMergeSort::StableSortKeys(nullptr, tmp, keys, n, FrontLess(), st);
    if ((rc = ensure_tmp(h, tmp))) return rc;
    CUDA_TRY(cub::DeviceMergeSort::StableSortKeys(h->cub_tmp.p, tmp, keys, n, FrontLess(), st));
    h->launches += 3;
  }
  coral_s1_frontier_item* sorted = h->items_sorted.as<coral_s1_frontier_item>();
  gather_items_kernel<<<gb, TB, 0, st>>>(items, keys, n, sorted, h->segk.as<unsigned long long>(),
                                         h->sort_b.as<double>());
  LAUNCH_CHECK(h);
  size_t tmp = 0;
  cub::DeviceScan::InclusiveScanByKey(nullptr, tmp, h->segk.as<unsigned long long>(),
                                      h->sort_b.as<double>(), h->scanv.as<double>(), MaxOp(),
                                      (int)n, cub::Equality(), st);
  if ((rc = ensure_tmp(h, tmp))) return rc;
  CUDA_TRY(cub::DeviceScan::InclusiveScanByKey(h->cub_tmp.p, tmp, h->segk.as<unsigned long long>(),
                                               h->sort_b.as<double>(), h->scanv.as<double>(),
                                               MaxOp(), (int)n, cub::Equality(), st));
  h->launches += 2;
  skyline_flags_kernel<<<gb, TB, 0, st>>>(h->segk.as<unsigned long long>(), h->sort_b.as<double>(),
                                          h->scanv.as<double>(), n, h->flagsel.as<unsigned char>());
  LAUNCH_CHECK(h);
  if ((rc = h->front.ensure(n * sizeof(coral_s1_frontier_item)))) return rc;
  tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, sorted, h->flagsel.as<unsigned char>(),
                             h->front.as<coral_s1_frontier_item>(), h->nsel.as<long long>(),
                             (int)n, st);
  if ((rc = ensure_tmp(h, tmp))) return rc;
  CUDA_TRY(cub::DeviceSelect::Flagged(h->cub_tmp.p, tmp, sorted, h->flagsel.as<unsigned char>(),
                                      h->front.as<coral_s1_frontier_item>(),
                                      h->nsel.as<long long>(), (int)n, st));
  h->launches += 2;
  long long ns = 0;
  CUDA_TRY(cudaMemcpyAsync(&ns, h->nsel.p, sizeof(ns), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  h->nfront = ns;
  return 0;
}

// Frontier over the items of `F` (nseg = mp x region segments): the per-segment CTA path;
// if some segment holds more than kSegCap items, the items are made contiguous in
// h->items (when they are not already) and the general path runs instead.
int frontier_segments(coral_s1_handle* h, const FrontParts& Fin, int64_t ntot, bool items_are_contiguous,
                      long long* dn_host = nullptr) {
  cudaStream_t st = h->stream;
  h->nfront = 0;
  if (ntot == 0) return 0;
  FrontParts F = Fin;
  const int nseg = h->NM * h->NP * F.R;
  int rc;
  const size_t o_surv = (size_t)nseg * kSegCap * 4, o_flag = o_surv + (size_t)nseg * 4 + 16;
  if ((rc = h->segbuf.ensure(o_flag + 16)) || (rc = h->front.ensure(ntot * sizeof(coral_s1_frontier_item))))
    return rc;
  unsigned char* sb = h->segbuf.as<unsigned char>();
  CUDA_TRY(cudaMemsetAsync(sb + o_flag, 0, 16, st));
  front_segment_kernel<<<(unsigned)nseg, kSegThreads, kSegCap * sizeof(SegKey), st>>>(
      F, nseg, (unsigned*)sb, (unsigned*)(sb + o_surv), (unsigned*)(sb + o_flag));
  LAUNCH_CHECK(h);
  front_emit_kernel<<<(unsigned)nseg, 256, 0, st>>>(F, nseg, (const unsigned*)sb, (const unsigned*)(sb + o_surv),
                                                    h->front.as<coral_s1_frontier_item>(), (long long*)(sb + o_flag + 8));
  LAUNCH_CHECK(h);
  long long res[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(res, sb + o_flag, 16, cudaMemcpyDeviceToHost, st));
  if (F.dn) CUDA_TRY(cudaMemcpyAsync(dn_host, F.dn, kPartsCountsLen * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (F.dn) {  // the counts the kernels used, for the general path below
    for (int p = 0; p < F.nparts; ++p) { F.n[p] = dn_host[p]; F.first[p] = dn_host[kMaxParts + p]; }
    F.first[F.nparts] = dn_host[kMaxParts + F.nparts];
    ntot = F.first[F.nparts];
    F.dn = nullptr;
  }
  if ((res[0] & 0xFFFFFFFFll) == 0) {
    h->nfront = res[1];
    return 0;
  }
  // a segment beyond kSegCap items: the general path over contiguous items
  if (!items_are_contiguous) {
    if ((rc = h->items.ensure(ntot * sizeof(coral_s1_frontier_item)))) return rc;
    for (int p = 0; p < F.nparts; ++p)
      if (F.n[p])
        CUDA_TRY(cudaMemcpyAsync(h->items.as<coral_s1_frontier_item>() + F.first[p], F.base + p * F.stride + F.offset,
                                 F.n[p] * sizeof(coral_s1_frontier_item), cudaMemcpyDeviceToDevice, st));
  }
  return frontier_from_items_general(h, ntot, F.R);
}

FrontParts one_part(const void* items, int64_t n, int R) {
  FrontParts F{};
  F.base = static_cast<const unsigned char*>(items);
  F.stride = 0;
  F.offset = 0;
  F.nparts = 1;
  F.R = R;
  F.n[0] = n;
  F.first[0] = 0;
  F.first[1] = n;
  return F;
}

template <class T>
int upload(coral_s1_handle* h, DevBuf& buf, const std::vector<T>& v, cudaStream_t st = nullptr) {
  int rc = buf.ensure(std::max<size_t>(v.size() * sizeof(T), 8));
  if (rc) return rc;
  if (!v.empty())
    CUDA_TRY(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st ? st : h->stream));
  return 0;
}

// upload() that skips the copy when the buffer still holds exactly these bytes: for the
// host-written, device-read-only tables a repeat solve re-sends unchanged (offsets, run
// lists, the frontier's token prices); the allocation id guards against a freed
// address coming back
template <class T>
int upload_same(coral_s1_handle* h, DevBuf& buf, const std::vector<T>& v, cudaStream_t st = nullptr) {
  const size_t nb = v.size() * sizeof(T);
  if (buf.id && buf.id == buf.shadow_id && buf.shadow.size() == nb &&
      (nb == 0 || !std::memcmp(buf.shadow.data(), v.data(), nb)))
    return 0;
  int rc = upload(h, buf, v, st);
  if (rc) return rc;
  buf.shadow.assign(reinterpret_cast<const unsigned char*>(v.data()), reinterpret_cast<const unsigned char*>(v.data()) + nb);
  buf.shadow_id = buf.id;
  return 0;
}

int64_t universe_size(int K, int n_max) {
  // sum_{n=1}^{n_max} C(K+n-1, n)
  int64_t tot = 0;
  for (int n = 1; n <= n_max; ++n) {
    long double c = 1;
    for (int i = 1; i <= n; ++i) c = c * (K + n - 1 - n + i) / i;
    tot += (int64_t)(c + 0.5L);
  }
  return tot;
}

}  // namespace

// ================================================================================
// C ABI
// ================================================================================
static int lattice_prepare(coral_s1_handle* h, cudaStream_t st);  // below: lattice state tables

extern "C" {

const char* coral_s1_last_error(void) { return g_err.c_str(); }
int coral_s1_version(void) { return 1; }

int coral_s1_create(int device, coral_s1_handle** out) {
  if (!out) return fail(CORAL_S1_EINVAL, "out is null");
  *out = nullptr;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(CORAL_S1_EINVAL, "bad device ordinal");
  CUDA_TRY(cudaSetDevice(device));
  auto* h = new coral_s1_handle();
  h->device = device;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->ranks_blocks_per_sm, lat_ranks_kernel, kRanksWarps * 32, 0);
  h->ranks_blocks_per_sm = std::max(h->ranks_blocks_per_sm, 1);
  static unsigned long long tab[160][8];
  for (int N = 0; N < 160; ++N)
    for (int k = 0; k < 8; ++k) {
      if (k > N) { tab[N][k] = 0; continue; }
      unsigned long long c = 1;
      for (int i = 1; i <= k; ++i) c = c * (unsigned long long)(N - k + i) / (unsigned long long)i;
      tab[N][k] = c;
    }
  cudaError_t e = cudaMemcpyToSymbol(c_binom, tab, sizeof(tab));
  if (e != cudaSuccess) { delete h; return fail(CORAL_S1_ECUDA, cudaGetErrorString(e)); }
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  for (auto& ev : h->ev_ws) cudaEventCreate(&ev);
  for (int i = 0; i < coral_s1_handle::kStreams; ++i) {
    cudaStreamCreateWithFlags(&h->side[i], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&h->side_ev[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->prep_ev, cudaEventDisableTiming);
  if (const char* e = getenv("CORAL_S1_STREAMS")) h->nstreams = std::max(1, std::min(atoi(e), coral_s1_handle::kStreams));
  h->default_streams = h->nstreams;
  if (const char* e = getenv("CORAL_S1_MEM_LIMIT")) h->mem_limit = (size_t)strtoull(e, nullptr, 10);
  if (h->lat_binom_d.ensure(sizeof(tab)) == 0)
    cudaMemcpy(h->lat_binom_d.p, tab, sizeof(tab), cudaMemcpyHostToDevice);
  {  // the per-candidate DP kernels may take all the shared memory their statics leave
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, evaluate_kernel);
    h->dp_smem_limit = (size_t)std::max(0, optin - (int)fa.sharedSizeBytes);
    cudaFuncGetAttributes(&fa, placement_op_kernel);
    h->dp_smem_limit = std::min(h->dp_smem_limit, (size_t)std::max(0, optin - (int)fa.sharedSizeBytes));
    cudaFuncSetAttribute(evaluate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->dp_smem_limit);
    cudaFuncSetAttribute(placement_op_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->dp_smem_limit);
  }
  cudaFuncSetAttribute(front_segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSegCap * sizeof(SegKey)));
  e = cudaGetLastError();
  if (e != cudaSuccess) { delete h; return fail(CORAL_S1_ECUDA, cudaGetErrorString(e)); }
  *out = h;
  return 0;
}

int coral_s1_destroy(coral_s1_handle* h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  DevBuf* bufs[] = {&h->prob, &h->tab, &h->flags, &h->budget, &h->keys, &h->koff_d,
                    &h->nvalid, &h->cand_off_d, &h->rec, &h->cub_tmp, &h->items, &h->items_sorted,
                    &h->sort_a, &h->sort_b, &h->segk, &h->scanv,
                    &h->flagsel, &h->nsel, &h->front, &h->prices, &h->ukey_s, &h->umem_s, &h->blkcnt, &h->blkoff, &h->op_in, &h->op_out, &h->tab_off_d, &h->fbucket, &h->segbuf, &h->avars, &h->pcounts,
                    &h->lat_base_d, &h->lat_binom_d, &h->lat_key, &h->lat_nsub, &h->lat_off,
                    &h->lat_sub, &h->lat_maxn, &h->census, &h->poscnt, &h->prep_tmp, &h->lat_flags_h, &h->lat_sums, &h->lat_soff, &h->run_off_d, &h->run_mp_d, &h->run_ph_d, &h->rect, &h->tokp};
  for (DevBuf* b : bufs) b->release();
  for (int i = 0; i < coral_s1_handle::kStreams; ++i) {
    h->ws_value[i].release(); h->ws_f0[i].release(); h->ws_ch[i].release(); h->ws_ranks[i].release();
    h->ws_win[i].release();
    if (h->side[i]) cudaStreamDestroy(h->side[i]);
    if (h->side_ev[i]) cudaEventDestroy(h->side_ev[i]);
  }
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  for (auto& ev : h->ev_ws)
    if (ev) cudaEventDestroy(ev);
  if (h->prep_ev) cudaEventDestroy(h->prep_ev);
  for (int i = 0; i < coral_s1_handle::kTimedMax; ++i) {
    if (h->tev[i][0]) cudaEventDestroy(h->tev[i][0]);
    if (h->tev[i][1]) cudaEventDestroy(h->tev[i][1]);
  }
  for (auto& ev : h->ev) if (ev) cudaEventDestroy(ev);
  delete h;
  return 0;
}

int coral_s1_set_stream(coral_s1_handle* h, void* stream) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  h->stream = reinterpret_cast<cudaStream_t>(stream);
  return 0;
}

int64_t coral_s1_launch_count(const coral_s1_handle* h) { return h ? h->launches : 0; }

int coral_s1_set_problem(coral_s1_handle* h, const coral_s1_problem* p) {
  if (!h || !p) return fail(CORAL_S1_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  // LibraryCaps.__post_init__ (templates.py:45-49)
  if (p->n_max < 1) return fail(CORAL_S1_EINVAL, "n_max must be >= 1");
  if (!(p->rho > 1)) return fail(CORAL_S1_EINVAL, "rho must be > 1");
  if (p->n_max > CORAL_S1_MAX_NODES)
    return fail(CORAL_S1_EUNSUPPORTED, "GPU path supports n_max <= 7");
  if (p->num_configs < 0 || p->num_configs > CORAL_S1_MAX_CONFIGS)
    return fail(CORAL_S1_EUNSUPPORTED, "GPU path supports <= 63 node configs");
  if (p->num_models < 0 || p->num_phases < 0 || p->num_phases > 2)
    return fail(CORAL_S1_EINVAL, "bad model/phase count");
  const int K = p->num_configs, NM = p->num_models, NP = p->num_phases;
  h->K = K; h->NM = NM; h->NP = NP; h->n_max = p->n_max;
  h->L.assign(NM, 0); h->g.assign(NM, 1); h->Lu.assign(NM, 0); h->smax.assign(NM, 0);
  h->phases.assign(p->phases, p->phases + NP);
  for (int i = 0; i < NP; ++i)
    if (h->phases[i] != CORAL_S1_PHASE_PREFILL && h->phases[i] != CORAL_S1_PHASE_DECODE)
      return fail(CORAL_S1_EINVAL, "phase must be prefill or decode");
  h->maxLu = 1;
  for (int m = 0; m < NM; ++m) {
    h->L[m] = p->mdl_num_layers[m];
    h->g[m] = p->mdl_granularity[m];
    if (h->L[m] < 1 || h->g[m] < 1) return fail(CORAL_S1_EINVAL, "num_layers and granularity must be >= 1");
    h->Lu[m] = h->L[m] / h->g[m];
    if (h->Lu[m] < 1) return fail(CORAL_S1_EINVAL, "granularity larger than num_layers");
    if (h->Lu[m] > CORAL_S1_MAX_LAYER_UNITS)
      return fail(CORAL_S1_EUNSUPPORTED, "GPU path supports <= 128 layer units per model");
    h->smax[m] = std::min(p->n_max, h->L[m]);
    h->maxLu = std::max(h->maxLu, h->Lu[m]);
  }
  h->tab_off.assign(NM * NP + 1, 0);
  for (int mp = 0; mp < NM * NP; ++mp) {
    const int m = mp / std::max(NP, 1);
    h->tab_off[mp + 1] = h->tab_off[mp] + (int64_t)p->n_max * K * h->Lu[m];
  }
  std::vector<double> memb(K);
  std::vector<int> inv(64, 0), rank1(K);
  for (int c = 0; c < K; ++c) {
    if (p->cfg_gpu_count[c] < 1) return fail(CORAL_S1_EINVAL, "gpu_count must be >= 1");
    memb[c] = ((double)p->cfg_gpu_count[c] * p->cfg_mem_gb[c]) * 1073741824.0;
    const int r = p->cfg_str_rank[c];
    if (r < 0 || r >= K) return fail(CORAL_S1_EINVAL, "cfg_str_rank out of range");
    rank1[c] = r + 1;
    inv[r] = c;
  }
  // pack every array into one device blob
  std::vector<unsigned char> blob;
  auto put = [&](const void* src, size_t bytes) {
    size_t off = (blob.size() + 15) & ~(size_t)15;
    blob.resize(off + std::max<size_t>(bytes, 8));
    if (bytes) memcpy(blob.data() + off, src, bytes);
    return off;
  };
  std::vector<int> ph(h->phases);
  const size_t o_gc = put(p->cfg_gpu_count, K * 4), o_mem = put(p->cfg_mem_gb, K * 8),
               o_bw = put(p->cfg_bw_tbps, K * 8), o_tf = put(p->cfg_tflops, K * 8),
               o_memb = put(memb.data(), K * 8), o_rank = put(rank1.data(), K * 4),
               o_inv = put(inv.data(), 64 * 4), o_L = put(h->L.data(), NM * 4),
               o_g = put(h->g.data(), NM * 4), o_Lu = put(h->Lu.data(), NM * 4),
               o_smax = put(h->smax.data(), NM * 4), o_ptb = put(p->mdl_params_total_b, NM * 8),
               o_pab = put(p->mdl_params_active_b, NM * 8), o_hid = put(p->mdl_hidden_size, NM * 8),
               o_bpp = put(p->mdl_bytes_per_param, NM * 8), o_kv = put(p->mdl_kv_bytes, NM * 8),
               o_spf = put(p->slo_prefill_ms, NM * 8), o_sdc = put(p->slo_decode_ms, NM * 8),
               o_ph = put(ph.data(), NP * 4);
  const int NPR = std::max(p->num_profile, 0);
  const size_t o_pm = put(p->prof_model, NPR * 4), o_pp = put(p->prof_phase, NPR * 4),
               o_pc = put(p->prof_cfg, NPR * 4), o_pj = put(p->prof_j, NPR * 4),
               o_pb = put(p->prof_bucket, NPR * 4), o_pt = put(p->prof_tps, NPR * 8);
  int rc = h->prob.ensure(blob.size());
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(h->prob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, h->stream));
  auto* b = h->prob.as<unsigned char>();
  DevProblem& d = h->dp;
  d.K = K; d.NM = NM; d.NP = NP; d.n_max = p->n_max; d.rho = p->rho;
  d.gc = (const int*)(b + o_gc); d.mem_gb = (const double*)(b + o_mem);
  d.bw = (const double*)(b + o_bw); d.tflops = (const double*)(b + o_tf);
  d.mem_bytes = (const double*)(b + o_memb); d.rank1 = (const int*)(b + o_rank);
  d.inv_rank = (const int*)(b + o_inv); d.L = (const int*)(b + o_L); d.g = (const int*)(b + o_g);
  d.Lu = (const int*)(b + o_Lu); d.smax = (const int*)(b + o_smax);
  d.ptb = (const double*)(b + o_ptb); d.pab = (const double*)(b + o_pab);
  d.hidden = (const double*)(b + o_hid); d.bpp = (const double*)(b + o_bpp);
  d.kv = (const double*)(b + o_kv); d.slo_pf = (const double*)(b + o_spf);
  d.slo_dc = (const double*)(b + o_sdc); d.phases = (const int*)(b + o_ph);
  d.mfu = p->mfu; d.mbu = p->mbu; d.net_eff = p->net_eff; d.fixed_ms = p->fixed_overhead_ms;
  d.prompt = p->avg_prompt_tokens; d.ctxd = p->avg_ctx_tokens; d.frac = p->slo_budget_frac;
  d.gbps = p->net_gbps; d.lat_ms = p->net_latency_ms;
  d.nprof = NPR;
  d.pm = (const int*)(b + o_pm); d.pp = (const int*)(b + o_pp); d.pc = (const int*)(b + o_pc);
  d.pj = (const int*)(b + o_pj); d.pb = (const int*)(b + o_pb); d.pt = (const double*)(b + o_pt);
  h->U = universe_size(K, p->n_max);
  h->memb_h = memb;
  h->inv_rank_h.assign(inv.begin(), inv.begin() + std::max(K, 1));
  h->rho = p->rho;
  h->wbytes_h.assign(NM, 0.0);
  for (int m = 0; m < NM; ++m) h->wbytes_h[m] = (p->mdl_params_total_b[m] * 1e9) * p->mdl_bytes_per_param[m];
  h->have_problem = true;
  h->have_tables = h->have_enum = h->have_eval = false;
  h->nfront = 0;
  return 0;
}

int coral_s1_tables(coral_s1_handle* h) {
  if (!h || !h->have_problem) return fail(CORAL_S1_EINVAL, "set_problem first");
  CUDA_TRY(cudaSetDevice(h->device));
  const int NMP = h->NM * h->NP;
  int rc;
  if ((rc = h->tab.ensure(std::max<int64_t>(h->tab_off[NMP], 1) * 8)) ||
      (rc = h->flags.ensure(std::max<int64_t>((int64_t)NMP * h->n_max * h->K, 1))) ||
      (rc = h->budget.ensure(std::max<int64_t>((int64_t)NMP * h->n_max, 1) * 8)) ||
      (rc = h->poscnt.ensure(std::max<int64_t>((int64_t)NMP * h->n_max, 1) * 4)) ||
      (rc = upload_same(h, h->tab_off_d, h->tab_off)))
    return rc;
  CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
  if (NMP > 0 && h->K > 0) {
    CUDA_TRY(cudaMemsetAsync(h->budget.p, 0, (size_t)NMP * h->n_max * 8, h->stream));
    CUDA_TRY(cudaMemsetAsync(h->poscnt.p, 0, (size_t)NMP * h->n_max * 4, h->stream));
    const int tpb = std::min(128, ((h->maxLu + 31) / 32) * 32);
    dim3 grid(h->K, h->n_max, NMP);
    tables_kernel<<<grid, tpb, 0, h->stream>>>(h->dp, h->tab_off_d.as<int64_t>(), h->tab.as<double>(),
                                               h->flags.as<unsigned char>(), h->budget.as<double>(),
                                               h->poscnt.as<unsigned>());
    LAUNCH_CHECK(h);
  }
  CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
  h->have_tables = true;
  h->have_eval = false;
  h->lat_ready = h->flags_ready = false;
  return 0;
}

int coral_s1_table_posfrac(coral_s1_handle* h, double* out, int64_t n) {
  if (!h || !h->have_tables) return fail(CORAL_S1_EINVAL, "tables first");
  const int NMP = h->NM * h->NP;
  if (n < (int64_t)NMP * h->n_max) return fail(CORAL_S1_EINVAL, "output too small");
  std::vector<unsigned> cnt((size_t)NMP * h->n_max, 0u);
  if (!cnt.empty())
    CUDA_TRY(cudaMemcpyAsync(cnt.data(), h->poscnt.p, cnt.size() * 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int mp = 0; mp < NMP; ++mp) {
    const int m = mp / h->NP;
    const double cells = (double)h->K * h->Lu[m];
    for (int S = 1; S <= h->n_max; ++S)
      out[(size_t)mp * h->n_max + S - 1] = cells > 0 ? cnt[(size_t)mp * h->n_max + S - 1] / cells : 0.0;
  }
  return 0;
}

int coral_s1_table_layout(const coral_s1_handle* h, int64_t* offsets, int32_t* lsteps,
                          int32_t* smax) {
  if (!h || !h->have_problem) return fail(CORAL_S1_EINVAL, "set_problem first");
  const int NMP = h->NM * h->NP;
  if (offsets) for (int i = 0; i <= NMP; ++i) offsets[i] = h->tab_off[i];
  if (lsteps) for (int m = 0; m < h->NM; ++m) lsteps[m] = h->Lu[m];
  if (smax) for (int m = 0; m < h->NM; ++m) smax[m] = h->smax[m];
  return 0;
}

int coral_s1_get_tables(coral_s1_handle* h, double* out, int64_t n) {
  if (!h || !h->have_tables) return fail(CORAL_S1_EINVAL, "tables not computed");
  const int64_t tot = h->tab_off[h->NM * h->NP];
  if (n < tot) return fail(CORAL_S1_EINVAL, "output too small");
  if (tot) CUDA_TRY(cudaMemcpyAsync(out, h->tab.p, tot * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int coral_s1_get_budgets(coral_s1_handle* h, double* out, int64_t n) {
  if (!h || !h->have_tables) return fail(CORAL_S1_EINVAL, "tables not computed");
  const int64_t tot = (int64_t)h->NM * h->NP * h->n_max;
  if (n < tot) return fail(CORAL_S1_EINVAL, "output too small");
  if (tot) CUDA_TRY(cudaMemcpyAsync(out, h->budget.p, tot * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int coral_s1_enumerate(coral_s1_handle* h) {
  if (!h || !h->have_problem) return fail(CORAL_S1_EINVAL, "set_problem first");
  CUDA_TRY(cudaSetDevice(h->device));
  const int NM = h->NM;
  const int64_t U = h->U;
  int rc;
  if ((rc = h->nvalid.ensure(std::max(NM, 1) * 8 + 16))) return rc;
  cudaStream_t st = h->stream;
  CUDA_TRY(cudaEventRecord(h->ev[2], st));
  h->counts.assign(NM, 0);
  h->koff.assign(NM + 1, 0);
  if (NM > 0 && U > 0) {
    const int64_t nblk64 = (U + kEnumBlock - 1) / kEnumBlock;
    const int nblk = (int)std::min<int64_t>(nblk64, INT32_MAX);
    const int64_t nchunk = (U + kEnumChunk - 1) / kEnumChunk;
    const int64_t nb = (int64_t)NM * nchunk;
    if (nb + 1 > (int64_t)INT32_MAX || nblk64 > INT32_MAX)  // one 32-bit-indexed scan over (model, chunk)
      return fail(CORAL_S1_EUNSUPPORTED, "enumerate: models x universe chunks exceed 2^31");
    if ((rc = h->ukey_s.ensure(U * 8)) || (rc = h->umem_s.ensure(U * 8)) ||
        (rc = h->blkcnt.ensure((nb + 1) * 8)) || (rc = h->blkoff.ensure((nb + 1) * 8)))
      return rc;
    // the universe once, unranked in key order: keys + memory sums + per-model window
    // counts per block; one scan -> block offsets and model totals
    enum_count_kernel<<<(unsigned)nblk, kEnumThreads, 0, st>>>(
        h->dp, U, nchunk, h->ukey_s.as<unsigned long long>(), h->umem_s.as<double>(),
        h->blkcnt.as<unsigned long long>());
    LAUNCH_CHECK(h);
    CUDA_TRY(cudaMemsetAsync(h->blkcnt.as<unsigned long long>() + nb, 0, 8, st));
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, h->blkcnt.as<unsigned long long>(),
                                  h->blkoff.as<unsigned long long>(), (int)(nb + 1), st);
    if ((rc = ensure_tmp(h, tmp))) return rc;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(h->cub_tmp.p, tmp, h->blkcnt.as<unsigned long long>(),
                                           h->blkoff.as<unsigned long long>(), (int)(nb + 1), st));
    window_totals_kernel<<<(NM + 127) / 128, 128, 0, st>>>(NM, nchunk, h->blkoff.as<unsigned long long>(),
                                                           h->nvalid.as<unsigned long long>());
    LAUNCH_CHECK(h);
    h->launches += 2;
    std::vector<unsigned long long> nv(NM);
    CUDA_TRY(cudaMemcpyAsync(nv.data(), h->nvalid.p, NM * 8, cudaMemcpyDeviceToHost, st));
    // the evaluator's T-hat monotonicity flags ride on this round trip
    const int NMPf = NM * h->NP;
    h->flags_h.assign((size_t)std::max(NMPf, 1) * h->n_max * h->K, 0);
    if (h->have_tables && NMPf && h->K)
      CUDA_TRY(cudaMemcpyAsync(h->flags_h.data(), h->flags.p, (size_t)NMPf * h->n_max * h->K,
                               cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    h->flags_ready = h->have_tables;
    for (int m = 0; m < NM; ++m) {
      h->counts[m] = (int64_t)nv[m];
      h->koff[m + 1] = h->koff[m] + h->counts[m];
    }
    const int64_t nk = h->koff[NM];
    if ((rc = h->keys.ensure(std::max<int64_t>(nk, 1) * 8))) return rc;
    h->ws_timed = false;
    if (nk > 0) {  // model-major, str(combo) order within a model: the library order
      CUDA_TRY(cudaEventRecord(h->ev_ws[0], st));
      window_select_kernel<<<(unsigned)nblk, kEnumThreads, 0, st>>>(
          h->dp, U, h->ukey_s.as<unsigned long long>(), h->umem_s.as<double>(), nchunk,
          h->blkoff.as<unsigned long long>(), h->keys.as<unsigned long long>());
      LAUNCH_CHECK(h);
      CUDA_TRY(cudaEventRecord(h->ev_ws[1], st));
      // its algorithmic bytes: one read of every universe key and memory sum (16 B) and
      // one write of each model's survivor keys (8 B)
      h->ws_bytes = U * 16 + nk * 8;
      h->ws_timed = true;
    }
    // lattice state tables for every model with candidates, on side stream 0; enqueued
    // after the compaction above, so the device compacts while the host prepares
    h->model_used.assign(NM, 0);
    for (int m = 0; m < NM; ++m) h->model_used[m] = h->counts[m] > 0;
    h->lat_ready = false;
    if (h->n_max >= 2 && h->have_tables) {
      if ((rc = lattice_prepare(h, h->side[0]))) return rc;
      CUDA_TRY(cudaEventRecord(h->prep_ev, h->side[0]));
      h->lat_ready = true;
    }
  }
  CUDA_TRY(cudaEventRecord(h->ev[3], st));
  // candidate list: mp-major, library order within each (model, phase)
  const int NMP = NM * h->NP;
  h->cand_off.assign(NMP + 1, 0);
  for (int mp = 0; mp < NMP; ++mp) h->cand_off[mp + 1] = h->cand_off[mp] + h->counts[mp / h->NP];
  h->ncand = h->cand_off[NMP];
  if ((rc = upload_same(h, h->cand_off_d, h->cand_off)) || (rc = upload_same(h, h->koff_d, h->koff))) return rc;
  h->have_enum = true;
  h->have_eval = false;
  return 0;
}

int coral_s1_num_combos(const coral_s1_handle* h, int64_t* counts) {
  if (!h || !h->have_enum) return fail(CORAL_S1_EINVAL, "enumerate first");
  for (int m = 0; m < h->NM; ++m) counts[m] = h->counts[m];
  return 0;
}

int coral_s1_get_combos(coral_s1_handle* h, int model, int enumeration_order, uint64_t* keys,
                        int64_t n) {
  if (!h || !h->have_enum) return fail(CORAL_S1_EINVAL, "enumerate first");
  if (model < 0 || model >= h->NM) return fail(CORAL_S1_EINVAL, "bad model index");
  const int64_t cnt = h->counts[model];
  if (n < cnt) return fail(CORAL_S1_EINVAL, "output too small");
  if (cnt)
    CUDA_TRY(cudaMemcpyAsync(keys, h->keys.as<unsigned long long>() + h->koff[model], cnt * 8,
                             cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (enumeration_order) {
    // templates.py:112 (num_nodes, str): stable partition of the str-sorted list
    std::stable_sort(keys, keys + cnt, [](uint64_t a, uint64_t b) {
      auto nodes = [](uint64_t k) {
        int s = 0;
        for (int t = 0; t < kMaxC; ++t) s += (int)((k >> (kKeyTokenBits * t)) & 7u);
        return s;
      };
      return nodes(a) < nodes(b);
    });
  }
  return 0;
}

int coral_s1_num_candidates(const coral_s1_handle* h, int64_t* n) {
  if (!h || !h->have_enum) return fail(CORAL_S1_EINVAL, "enumerate first");
  *n = h->ncand;
  return 0;
}

}  // extern "C"

// Per-combo kernel over candidates lo, lo+stride, ... < hi for S in [S_lo, S_hi].
static int launch_percombo(coral_s1_handle* h, cudaStream_t st, int64_t lo, int64_t hi, int64_t stride,
                           int S_lo, int S_hi) {
  if (hi <= lo) return 0;
  EvalArgs A;
  A.P = h->dp;
  A.keys = h->keys.as<unsigned long long>();
  A.koff = h->koff_d.as<int64_t>();
  A.cand_off = h->cand_off_d.as<int64_t>();
  A.NMP = h->NM * h->NP;
  A.hi = hi;
  A.stride = stride;
  A.S_lo = S_lo;
  A.S_hi = S_hi;
  A.tab = h->tab.as<double>();
  A.tab_off = h->tab_off_d.as<int64_t>();
  A.flags = h->flags.as<unsigned char>();
  A.rec = h->rec.as<coral_s1_record>();
  A.rect = h->rect.as<double>();
  const size_t smem = dp_smem_bytes(std::min(kMaxM, 1 << h->n_max), h->maxLu + 1, h->maxLu, h->n_max - 2);
  if (smem > h->dp_smem_limit)
    return fail(CORAL_S1_EUNSUPPORTED, "per-candidate placement DP: n_max " + std::to_string(h->n_max) +
                                           " with " + std::to_string(h->maxLu) +
                                           " layer units exceeds shared memory (the lattice path covers it)");
  const int64_t nblocks = (hi - lo + stride - 1) / stride;
  const int64_t chunk = 1ll << 30;
  for (int64_t b0 = 0; b0 < nblocks; b0 += chunk) {
    A.lo = lo + b0 * stride;
    const int64_t nb = std::min(chunk, nblocks - b0);
    evaluate_kernel<<<(unsigned)nb, kDpThreads, smem, st>>>(A);
    LAUNCH_CHECK(h);
  }
  return 0;
}

// Bracket one launch on stream st with a timing-event pair of kind `kind`
// (0 = lat_top_kernel, 1 = lat_layer_kernel, 2 = lat_value_kernel, 3 = lat_decode_kernel,
// 4 = lat_ranks_kernel).
static int timed_begin(coral_s1_handle* h, cudaStream_t st, int kind, int mp = -2) {
  if (!h->timing) return -1;  // two event records per launch cost ~2 us of host time each
  if (h->ntimed >= coral_s1_handle::kTimedMax) return -1;
  const int i = h->ntimed;
  if (!h->tev[i][0] && (cudaEventCreate(&h->tev[i][0]) != cudaSuccess || cudaEventCreate(&h->tev[i][1]) != cudaSuccess))
    return -1;
  h->ntimed++;
  h->tkind[i] = kind;
  h->tmp[i] = mp == -2 ? h->cur_mp : mp;
  h->tslot[i] = -1;
  for (int k = 0; k < coral_s1_handle::kStreams; ++k)
    if (h->side[k] == st) h->tslot[i] = k;
  cudaEventRecord(h->tev[i][0], st);
  return i;
}
static void timed_end(coral_s1_handle* h, cudaStream_t st, int i) {
  if (i >= 0) cudaEventRecord(h->tev[i][1], st);
}

// State tables shared by all models (depend on K and n_max only) + per-model maxn.
static int lattice_prepare(coral_s1_handle* h, cudaStream_t st) {
  const int K = h->K, R = h->n_max - 1;
  h->lat_base.assign(R + 2, 0);
  for (int sz = 1; sz <= R; ++sz) {
    long double c = 1;
    for (int i = 1; i <= sz; ++i) c = c * (K + i - 1) / i;  // C(K+sz-1, sz)
    h->lat_base[sz + 1] = h->lat_base[sz] + (long long)(c + 0.5L);
  }
  h->lat_states = h->lat_base[R + 1];
  int rc;
  if (h->lat_states >= (1ll << 24)) {  // state indices are packed in 24 bits (rank tables,
    h->lat_ok = false;                 // sub-tables): beyond that every unit takes the exact
    h->lat_states = 0;                 // per-candidate kernel
    return 0;
  }
  if ((rc = upload_same(h, h->lat_base_d, h->lat_base, st))) return rc;
  if (h->lat_states == 0) return 0;
  const long long ns = h->lat_states;
  if ((rc = h->lat_key.ensure(ns * 8)) || (rc = h->lat_nsub.ensure((ns + 1) * 8)) ||
      (rc = h->lat_off.ensure((ns + 1) * 8)) ||
      (rc = h->lat_maxn.ensure((size_t)std::max(h->NM, 1) * ns * 4)))
    return rc;
  LatModel L{K, R, h->lat_base_d.as<long long>(), h->lat_binom_d.as<unsigned long long>()};
  const unsigned gb = (unsigned)((ns + 255) / 256);
  lat_state_keys_kernel<<<gb, 256, 0, st>>>(L, h->dp.rank1, h->lat_key.as<unsigned long long>());
  LAUNCH_CHECK(h);
  lat_nsub_kernel<<<(unsigned)((ns + 256) / 256), 256, 0, st>>>(L, h->lat_key.as<unsigned long long>(),
                                                                h->lat_nsub.as<long long>());
  LAUNCH_CHECK(h);
  size_t tmp = 0;  // own scratch: may run beside the enumeration's CUB calls
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, h->lat_nsub.as<long long>(), h->lat_off.as<long long>(),
                                (int)(ns + 1), st);
  if ((rc = h->prep_tmp.ensure(std::max<size_t>(tmp, 8)))) return rc;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(h->prep_tmp.p, tmp, h->lat_nsub.as<long long>(),
                                         h->lat_off.as<long long>(), (int)(ns + 1), st));
  h->launches += 2;
  // upper bound (every state has at most 2^R sub-multiset codes): no host round trip
  if ((rc = h->lat_sub.ensure(std::max<long long>(ns << R, 1) * sizeof(uint2)))) return rc;
  lat_subtab_kernel<<<(unsigned)((ns * 32 + 255) / 256), 256, 0, st>>>(L, h->dp.inv_rank, h->lat_key.as<unsigned long long>(),
                                        h->lat_off.as<long long>(), h->lat_sub.as<uint2>());
  LAUNCH_CHECK(h);
  // maxn per model in closed form from the achievable memory sums of k configs
  {
    std::vector<double> mem(h->memb_h);
    std::sort(mem.begin(), mem.end());
    mem.erase(std::unique(mem.begin(), mem.end()), mem.end());
    double cap = 0;  // sums at or above the largest window top never matter
    for (int m = 0; m < h->NM; ++m)
      if (h->model_used[m]) cap = std::max(cap, h->rho * h->wbytes_h[m]);
    cap *= 1.0 + 1e-6;
    const int kmax = h->n_max - 1;  // a state holds >= 1 config
    // the sum table is a pure function of (memory sizes, cap, kmax): memoised per handle
    if (!(h->sums_key_mem == mem && h->sums_key_cap == cap && h->sums_key_kmax == kmax)) {
      std::vector<std::vector<double>> sums(kmax + 1);
      sums[0].push_back(0.0);
      for (int k = 1; k <= kmax; ++k) {
        for (double prev : sums[k - 1])
          for (double v : mem)
            if (prev + v < cap) sums[k].push_back(prev + v);
        std::sort(sums[k].begin(), sums[k].end());
        sums[k].erase(std::unique(sums[k].begin(), sums[k].end()), sums[k].end());
      }
      h->sums_flat.clear();
      h->sums_off.assign(kmax + 2, 0);
      for (int k = 0; k <= kmax; ++k) {
        h->sums_off[k] = (int)h->sums_flat.size();
        h->sums_flat.insert(h->sums_flat.end(), sums[k].begin(), sums[k].end());
      }
      h->sums_off[kmax + 1] = (int)h->sums_flat.size();
      h->sums_key_mem = mem;
      h->sums_key_cap = cap;
      h->sums_key_kmax = kmax;
    }
    const std::vector<double>& flat = h->sums_flat;
    const std::vector<int>& soff = h->sums_off;
    if ((rc = upload_same(h, h->lat_sums, flat, st)) || (rc = upload_same(h, h->lat_soff, soff, st))) return rc;
    for (int m = 0; m < h->NM; ++m) {
      if (!h->counts[m] || !h->model_used[m]) continue;
      const double lo = h->wbytes_h[m], hi = h->rho * lo;
      lat_maxn_closed_kernel<<<gb, 256, 0, st>>>(L, h->dp.inv_rank, h->lat_key.as<unsigned long long>(),
                                                 h->dp.mem_bytes, h->lat_sums.as<double>(),
                                                 h->lat_soff.as<int>(), lo, hi, 1e-9 * hi, h->n_max,
                                                 h->lat_maxn.as<unsigned>() + (size_t)m * ns);
      LAUNCH_CHECK(h);
    }
  }
  // workspaces: one chain per stream, as many streams as fit in device memory (the
  // tables grow as C(K + n_max - 2, n_max - 1) x Lu); none fitting -> every unit takes
  // the exact per-candidate kernel (no lattice tables needed)
  const long long LuP = lat_pitch(h->maxLu);
  const long long nS = std::max(h->n_max - 1, 1);                         // S = 2..n_max
  const long long nch = std::max((h->n_max - 2) * (h->n_max - 1) / 2, 1);  // (S, sg) choice layers
  // value tables + their row summaries (nS x states x 32 B); f tables + theirs
  const size_t want_v = (size_t)(nS * ns * LuP * 8) + (size_t)(nS * ns * 32) + 32,
               want_f = (size_t)(2 * nS * ns * LuP * 8) + (size_t)(nS * ns * 32) + 32,
               want_c = (size_t)(nch * ns * LuP * 2);
  {  // already allocated: no memory query (cudaMemGetInfo can stall the step)
    int have = 0;
    while (have < h->nstreams && h->ws_value[have].cap >= want_v && h->ws_f0[have].cap >= want_f &&
           h->ws_ch[have].cap >= want_c)
      ++have;
    if (have == h->nstreams) {  // every stream fits
      h->lat_streams = have;
      h->lat_ok = true;
      return 0;
    }
    if (h->lat_ok && h->lat_fit_ns == ns && h->lat_fit_pitch == LuP && have >= h->lat_streams)
      return 0;  // same tables as the last, memory-limited decision
  }
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  if (h->mem_limit) {
    size_t used = 0;  // what this handle already holds counts as used against the cap
    for (int i = 0; i < coral_s1_handle::kStreams; ++i) used += h->ws_value[i].cap + h->ws_f0[i].cap + h->ws_ch[i].cap;
    free_b = std::min(free_b, h->mem_limit > used ? h->mem_limit - used : (size_t)0);
  }
  // the evaluate's own buffers come after the lattice workspaces: records (32 B per
  // candidate), and per chain stream the rank table (256 B) and winners (16 B) per
  // candidate of the largest model; plus the bounded frontier item buffer (64 MiB)
  size_t reserve = (size_t)64 << 20;
  {
    int64_t nc = 0, maxc = 1;
    for (int m = 0; m < h->NM; ++m) { nc += h->counts[m] * h->NP; maxc = std::max<int64_t>(maxc, h->counts[m]); }
    const size_t have_rec = h->rec.cap, want_rec = (size_t)nc * sizeof(coral_s1_record);
    reserve += want_rec > have_rec ? want_rec - have_rec : 0;
    for (int i = 0; i < h->nstreams; ++i) {
      const size_t want = (size_t)maxc * (kRankStride * sizeof(unsigned) + sizeof(int4)), have = h->ws_ranks[i].cap + h->ws_win[i].cap;
      reserve += want > have ? want - have : 0;
    }
  }
  const size_t avail = free_b / 10 * 9;  // 10% headroom for CUB scratch and the frontier sort
  const size_t budget = avail > reserve ? avail - reserve : 0;
  int fit = 0;
  size_t extra = 0;
  for (int i = 0; i < h->nstreams; ++i) {
    auto more = [](const DevBuf& b, size_t w) { return b.cap >= w ? (size_t)0 : w; };
    const size_t add = more(h->ws_value[i], want_v) + more(h->ws_f0[i], want_f) + more(h->ws_ch[i], want_c);
    if (extra + add > budget) break;
    extra += add;
    ++fit;
  }
  h->lat_streams = std::max(fit, 1);
  h->lat_ok = fit > 0;
  h->lat_fit_ns = ns;
  h->lat_fit_pitch = LuP;
  for (int i = 0; i < fit; ++i) {
    if ((rc = h->ws_value[i].ensure(want_v)) || (rc = h->ws_f0[i].ensure(want_f)) ||
        (rc = h->ws_ch[i].ensure(want_c)))
      return rc;
  }
  return 0;
}

// One (model, phase) chain on stream `slot`: lattice for every monotone S of the
// chain, the exact per-candidate kernel for the others.
// One lattice pass of a (model, phase) chain over the S values in smask: value tables,
// DP layers, top cells, decode. scan = the reference's full-scan variant (kernels.py:
// 240-249) for the candidates whose rows fail the monotone test at S; otherwise the
// binary-search crossing (kernels.py:210-239) for the candidates whose rows pass it.
static int lattice_pass(coral_s1_handle* h, int mp, int slot, const unsigned* ranks, unsigned smask,
                        unsigned xmask, bool scan, const unsigned long long* nonmono, int64_t lo, int64_t hi) {
  cudaStream_t st = h->side[slot];
  const int m = mp / h->NP;
  const int K = h->K, Lu = h->Lu[m];
  const long long ns = h->lat_states, LuP = lat_pitch(h->maxLu);
  const long long ncombo = hi - lo;  // the top cells of candidates [lo, hi) of the model
  LatModel L{K, h->n_max - 1, h->lat_base_d.as<long long>(), h->lat_binom_d.as<unsigned long long>()};
  int Smax = 0;
  for (int S = 1; S <= CORAL_S1_MAX_NODES; ++S)
    if ((smask >> S) & 1u) Smax = S;
  LatWork W;
  W.value = h->ws_value[slot].as<double>();
  W.f = h->ws_f0[slot].as<double>();
  W.ch = h->ws_ch[slot].as<unsigned short>();
  W.stride = ns * lat_pitch(Lu);
  {
    const long long nS = std::max(h->n_max - 1, 1);  // summaries sit after the maxLu-pitched tables
    // 32-byte aligned: lat_top_kernel reads a summary with one 256-bit load
    W.vsum = h->ws_value[slot].as<double>() + ((nS * ns * LuP + 3) & ~3ll);
    W.fsum = h->ws_f0[slot].as<double>() + ((2 * nS * ns * LuP + 3) & ~3ll);
    W.sstride = ns * 4;
  }
  const double* tab_mp = h->tab.as<double>() + h->tab_off[mp];
  if (Smax >= 2 && ns > 0 && !scan) {  // value tables do not depend on the variant
    const int ti = timed_begin(h, st, 2);
    lat_value_kernel<<<dim3((unsigned)((ns * 32 + 255) / 256), Smax - 1), 256, 0, st>>>(
        L, h->dp.inv_rank, h->lat_key.as<unsigned long long>(), h->lat_maxn.as<unsigned>() + (size_t)m * ns,
        tab_mp, K, Lu, 2, smask, W);
    timed_end(h, st, ti);
    LAUNCH_CHECK(h);
  }
  for (int sg = 2; sg <= Smax - 1; ++sg) {
    const long long nst = h->lat_base[h->n_max - 1 + 1] - h->lat_base[sg];
    if (nst <= 0) continue;
    const int ti = timed_begin(h, st, 1);
    const dim3 lgrid((unsigned)((nst * 32 + 255) / 256), Smax - sg);
    unsigned long long* cen = h->census_on ? h->census.as<unsigned long long>() : nullptr;
    const unsigned* maxn = h->lat_maxn.as<unsigned>() + (size_t)m * ns;
    const long long* off = h->lat_off.as<long long>();
    const uint2* sub = h->lat_sub.as<uint2>();
    // states of 6 configs (n_max = 7): up to 63 sub-multiset codes -> 2 slots per lane
    // one launch per search mode (exact: capped search; tolerance-monotone: literal
    // search; scan pass: full scan), each over the S values of that mode
    const unsigned m_exact = scan ? 0u : (smask & xmask), m_tol = scan ? 0u : (smask & ~xmask),
                   m_scan = scan ? smask : 0u;
#define CORAL_LAYER(SL, MODE, MASK) \
    lat_layer_kernel<SL, MODE><<<lgrid, 256, 0, st>>>(L, sg, sg + 1, MASK, xmask, h->n_max, Lu, maxn, off, sub, W, cen)
#define CORAL_LAYER_RUN(SL, MASK) \
    lat_layer_run_kernel<SL><<<lgrid, 256, 0, st>>>(L, sg, sg + 1, MASK, xmask, h->n_max, Lu, maxn, off, sub, W, cen)
    const bool run = Lu >= kLayerRunMinLu;  // exact rows of a long model: two cells per lane
    if (h->n_max >= 7) {
      if (m_exact) { if (run) CORAL_LAYER_RUN(2, m_exact); else CORAL_LAYER(2, 1, m_exact); }
      if (m_tol) CORAL_LAYER(2, 0, m_tol);
      if (m_scan) CORAL_LAYER(2, 2, m_scan);
    } else {
      if (m_exact) { if (run) CORAL_LAYER_RUN(1, m_exact); else CORAL_LAYER(1, 1, m_exact); }
      if (m_tol) CORAL_LAYER(1, 0, m_tol);
      if (m_scan) CORAL_LAYER(1, 2, m_scan);
    }
#undef CORAL_LAYER_RUN
#undef CORAL_LAYER
    timed_end(h, st, ti);
    LAUNCH_CHECK(h);
  }
  TopArgs T;
  T.L = L;
  T.inv_rank = h->dp.inv_rank;
  T.keys = h->keys.as<unsigned long long>() + h->koff[m] + lo;
  T.ncombo = ncombo;
  T.smask = smask;
  T.xmask = xmask;
  for (int S = 0; S < 8; ++S) T.nonmono[S] = nonmono[S];
  T.K = K;
  T.Lu = Lu;
  T.g = h->g[m];
  T.tab_mp = tab_mp;
  T.W = W;
  T.state_key = h->lat_key.as<unsigned long long>();
  T.off = h->lat_off.as<long long>();
  T.subtab = h->lat_sub.as<uint2>();
  T.rec = h->rec.as<coral_s1_record>() + h->cand_off[mp] + lo;
  T.rect = h->rect.as<double>() + h->cand_off[mp] + lo;
  T.win = h->ws_win[slot].as<int4>();
  T.ranks = ranks;
  T.census = h->census_on ? h->census.as<unsigned long long>() : nullptr;
  const int ti = timed_begin(h, st, 0);
  const unsigned tg = (unsigned)((ncombo * 32 + 127) / 128);  // 4 candidates (warps) per CTA
  if (h->n_max >= 7) {
    if (scan) lat_top_kernel<4, true><<<tg, 128, 0, st>>>(T);
    else lat_top_kernel<4, false><<<tg, 128, 0, st>>>(T);
  } else {
    if (scan) lat_top_kernel<2, true><<<tg, 128, 0, st>>>(T);
    else lat_top_kernel<2, false><<<tg, 128, 0, st>>>(T);
  }
  timed_end(h, st, ti);
  LAUNCH_CHECK(h);
  const int td = timed_begin(h, st, 3);
  lat_decode_kernel<<<(unsigned)((ncombo + 255) / 256), 256, 0, st>>>(T);
  timed_end(h, st, td);
  LAUNCH_CHECK(h);
  return 0;
}

// One (model, phase) chain on stream `slot`. Each candidate's DP mode at S follows its
// own rows (kernels.py:291: np.all(np.diff(tput) <= 1e-12) over the combo's configs):
// pass A runs the search variant for the candidates that pass the test, pass B the
// full-scan variant (only for the S values where some config row fails it) for the
// others. Without lattice tables (memory) every S takes the exact per-candidate kernel.
static int lattice_units(coral_s1_handle* h, int mp, const std::vector<int>& Ss, int slot,
                         const unsigned* ranks, int64_t lo, int64_t hi) {
  const int K = h->K;
  if (hi <= lo) return 0;
  unsigned smask = 0, xmask = 0, scanmask = 0;
  unsigned long long nonmono[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int S : Ss) {
    if (!h->lat_ok) {  // exact per-candidate kernel for this S
      int rc = launch_percombo(h, h->side[slot], h->cand_off[mp] + lo, h->cand_off[mp] + hi, 1, S, S);
      if (rc) return rc;
      continue;
    }
    smask |= 1u << S;
    bool exact = true;  // bit 1 of the row flags: all diffs <= 0
    for (int c = 0; c < K; ++c) {
      const unsigned char f = h->flags_h[((size_t)mp * h->n_max + (S - 1)) * K + c];
      exact &= (f & 2) != 0;
      if (!(f & 1)) nonmono[S] |= 1ull << c;
    }
    if (exact) xmask |= 1u << S;
    if (nonmono[S] && S >= 2) scanmask |= 1u << S;
  }
  if (!smask) return 0;
  int rc = lattice_pass(h, mp, slot, ranks, smask, xmask, false, nonmono, lo, hi);
  if (!rc && scanmask) rc = lattice_pass(h, mp, slot, ranks, scanmask, 0u, true, nonmono, lo, hi);
  return rc;
}

// One piece of evaluation work: stage counts `smask` of (model, phase) slot mp for the
// candidates [lo, hi) of the model (library order). Multi-GPU ranks take disjoint
// pieces: whole (mp, S) units, or a unit's candidates split by range (the north star's
// (model, GPU-type combination) axis); records hold each candidate's best over the S
// values evaluated, so pieces merge exactly.
struct Piece {
  int mp;
  unsigned smask;
  int64_t lo, hi;
};

static int evaluate_pieces(coral_s1_handle* h, std::vector<Piece> pieces) {
  if (!h || !h->have_tables || !h->have_enum) return fail(CORAL_S1_EINVAL, "tables and enumerate first");
  CUDA_TRY(cudaSetDevice(h->device));
  int rc;
  if ((rc = h->rec.ensure(std::max<int64_t>(h->ncand, 1) * sizeof(coral_s1_record))) ||
      (rc = h->rect.ensure(std::max<int64_t>(h->ncand, 1) * sizeof(double))))
    return rc;
  cudaStream_t st = h->stream;
  const int NMP = h->NM * h->NP;
  h->own_mp.assign(NMP, 0);
  std::vector<Piece> ok;
  for (Piece p : pieces) {
    if (p.mp < 0 || p.mp >= NMP) return fail(CORAL_S1_EINVAL, "piece: bad mp");
    if (p.smask) h->own_mp[p.mp] = 1;  // requested: feasibility is checked even with no candidates
    const int m = p.mp / h->NP;
    p.lo = std::max<int64_t>(p.lo, 0);
    p.hi = (p.hi < 0 || p.hi > h->counts[m]) ? h->counts[m] : p.hi;
    unsigned mk = 0;
    for (int S = 1; S <= std::min(h->smax[m], h->Lu[m]); ++S) mk |= p.smask & (1u << S);
    p.smask = mk;
    if (!mk || p.hi <= p.lo) continue;
    h->own_mp[p.mp] = 1;
    ok.push_back(p);
  }
  const bool flags_were_ready = h->flags_ready;
  if (!flags_were_ready) {
    h->flags_h.assign((size_t)std::max(NMP, 1) * h->n_max * h->K, 0);
    if (NMP && h->K)
      CUDA_TRY(cudaMemcpyAsync(h->flags_h.data(), h->flags.p, (size_t)NMP * h->n_max * h->K,
                               cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaEventRecord(h->ev[4], st));
  h->ntimed = 0;
  // records not improved by any piece read as infeasible (num_stages 0)
  CUDA_TRY(cudaMemsetAsync(h->rec.p, 0, std::max<int64_t>(h->ncand, 1) * sizeof(coral_s1_record), st));
  CUDA_TRY(cudaMemsetAsync(h->rect.p, 0, std::max<int64_t>(h->ncand, 1) * sizeof(double), st));
  if (h->census_on) CUDA_TRY(cudaMemsetAsync(h->census.p, 0, 32, st));
  if (h->lat_ready) {  // prepared on side[0] during enumerate (every model with candidates)
    CUDA_TRY(cudaStreamWaitEvent(st, h->prep_ev, 0));
  } else {
    h->model_used.assign(h->NM, 0);  // lattice tables only for the models this call evaluates
    for (const Piece& p : ok) h->model_used[p.mp / h->NP] = 1;
    if ((rc = lattice_prepare(h, st))) return rc;
  }
  if (!flags_were_ready) CUDA_TRY(cudaStreamSynchronize(st));  // flags_h valid
  CUDA_TRY(cudaEventRecord(h->fork_ev, st));
  for (int i = 0; i < coral_s1_handle::kStreams; ++i) CUDA_TRY(cudaStreamWaitEvent(h->side[i], h->fork_ev, 0));
  // Pieces of one (model, phase) slot run back to back on one stream: their candidate
  // ranges may overlap (different S), and the decode of each read-modify-writes the
  // records. The two phases of a model (disjoint records) share a stream -- and the rank
  // table of an equal range -- unless there are fewer such groups than chain streams,
  // in which case each phase takes its own stream and both run concurrently.
  const int nslots = std::max(1, h->lat_ok ? std::min(h->lat_streams, h->nstreams) : h->nstreams);
  struct Group { int m; std::vector<int> idx; double w; };
  std::vector<Group> groups;
  {
    std::vector<Group> per_mp;
    for (int i = 0; i < (int)ok.size(); ++i) {
      Group* g = nullptr;
      for (Group& x : per_mp)
        if (ok[x.idx[0]].mp == ok[i].mp) g = &x;
      if (!g) { per_mp.push_back(Group{ok[i].mp / h->NP, {}, 0.0}); g = &per_mp.back(); }
      g->idx.push_back(i);
      g->w += (double)(ok[i].hi - ok[i].lo) * h->Lu[ok[i].mp / h->NP] * __builtin_popcount(ok[i].smask);
    }
    int nmodels = 0;
    for (size_t i = 0; i < per_mp.size(); ++i) {
      bool seen = false;
      for (size_t j = 0; j < i; ++j) seen |= per_mp[j].m == per_mp[i].m;
      nmodels += !seen;
    }
    const bool by_model = nmodels >= nslots;
    for (Group& g : per_mp) {
      Group* t = nullptr;
      if (by_model)
        for (Group& x : groups)
          if (x.m == g.m) t = &x;
      if (!t) { groups.push_back(Group{g.m, {}, 0.0}); t = &groups.back(); }
      t->idx.insert(t->idx.end(), g.idx.begin(), g.idx.end());
      t->w += g.w;
    }
    // within a group, equal ranges back to back (one rank table each)
    for (Group& g : groups)
      std::stable_sort(g.idx.begin(), g.idx.end(), [&](int x, int y) {
        return ok[x].lo != ok[y].lo ? ok[x].lo < ok[y].lo : ok[x].hi < ok[y].hi;
      });
  }
  std::stable_sort(groups.begin(), groups.end(), [](const Group& a, const Group& b) { return a.w > b.w; });
  int64_t maxc = 1;
  for (const Piece& p : ok) maxc = std::max<int64_t>(maxc, p.hi - p.lo);
  // per chain stream: the rank table of the group's range and the top cells' winners
  // (stream-ordered within a group, so one buffer per stream suffices)
  // chain streams in rotation: the lattice workspaces that fit, at most the streams asked for
  for (int i = 0; i < nslots; ++i)
    if ((rc = h->ws_ranks[i].ensure(maxc * kRankStride * sizeof(unsigned))) || (rc = h->ws_win[i].ensure(maxc * sizeof(int4))))
      return rc;
  int slot = 0;
  for (const Group& g : groups) {
    const int m = g.m;
    unsigned* ranks = h->ws_ranks[slot].as<unsigned>();
    int64_t rlo = -1, rhi = -1;  // range of the rank table on this stream
    for (int i : g.idx) {
      if ((ok[i].lo != rlo || ok[i].hi != rhi) && h->n_max >= 2 && h->lat_states > 0 && h->lat_ok) {
        LatModel L{h->K, h->n_max - 1, h->lat_base_d.as<long long>(), h->lat_binom_d.as<unsigned long long>()};
        const long long n = ok[i].hi - ok[i].lo;
        const long long rb = std::min<long long>((n + kRanksWarps - 1) / kRanksWarps, (long long)h->num_sms * h->ranks_blocks_per_sm);
        const int tr = timed_begin(h, h->side[slot], 4, ok[i].mp);
        lat_ranks_kernel<<<(unsigned)rb, kRanksWarps * 32, 0, h->side[slot]>>>(
            L, h->dp.inv_rank, h->keys.as<unsigned long long>() + h->koff[m] + ok[i].lo, n, ranks);
        timed_end(h, h->side[slot], tr);
        LAUNCH_CHECK(h);
        rlo = ok[i].lo;
        rhi = ok[i].hi;
      }
      std::vector<int> Ss;
      for (int S = 1; S <= CORAL_S1_MAX_NODES; ++S)
        if ((ok[i].smask >> S) & 1u) Ss.push_back(S);
      h->cur_mp = ok[i].mp;
      if ((rc = lattice_units(h, ok[i].mp, Ss, slot, ranks, ok[i].lo, ok[i].hi))) return rc;
    }
    slot = (slot + 1) % nslots;
  }
  for (int i = 0; i < coral_s1_handle::kStreams; ++i) {
    CUDA_TRY(cudaEventRecord(h->side_ev[i], h->side[i]));
    CUDA_TRY(cudaStreamWaitEvent(st, h->side_ev[i], 0));
  }
  CUDA_TRY(cudaEventRecord(h->ev[5], st));
  h->have_eval = true;
  return 0;
}

// (mp, S) units selected by take(mp, S), every candidate
template <class Take>
static int evaluate_units(coral_s1_handle* h, Take take) {
  if (!h || !h->have_tables || !h->have_enum) return fail(CORAL_S1_EINVAL, "tables and enumerate first");
  std::vector<Piece> pieces;
  for (int mp = 0; mp < h->NM * h->NP; ++mp) {
    unsigned mk = 0;
    for (int S = 1; S <= CORAL_S1_MAX_NODES; ++S)
      if (take(mp, S)) mk |= 1u << S;
    if (mk) pieces.push_back(Piece{mp, mk, 0, -1});
  }
  return evaluate_pieces(h, pieces);
}

extern "C" {

int coral_s1_evaluate(coral_s1_handle* h, int64_t lo, int64_t hi) {
  if (!h || !h->have_tables || !h->have_enum) return fail(CORAL_S1_EINVAL, "tables and enumerate first");
  if (hi < 0 || hi > h->ncand) hi = h->ncand;
  if (lo < 0) lo = 0;
  if (lo == 0 && hi == h->ncand) return evaluate_units(h, [](int, int) { return true; });
  // a sub-range: per-candidate kernel over [lo, hi), every S
  CUDA_TRY(cudaSetDevice(h->device));
  int rc;
  if ((rc = h->rec.ensure(std::max<int64_t>(h->ncand, 1) * sizeof(coral_s1_record))) ||
      (rc = h->rect.ensure(std::max<int64_t>(h->ncand, 1) * sizeof(double))))
    return rc;
  h->own_mp.assign((size_t)h->NM * h->NP, 1);
  CUDA_TRY(cudaEventRecord(h->ev[4], h->stream));
  CUDA_TRY(cudaMemsetAsync(h->rec.p, 0, std::max<int64_t>(h->ncand, 1) * sizeof(coral_s1_record), h->stream));
  CUDA_TRY(cudaMemsetAsync(h->rect.p, 0, std::max<int64_t>(h->ncand, 1) * sizeof(double), h->stream));
  if (h->census_on) CUDA_TRY(cudaMemsetAsync(h->census.p, 0, 32, h->stream));
  if ((rc = launch_percombo(h, h->stream, lo, hi, 1, 1, CORAL_S1_MAX_NODES))) return rc;
  CUDA_TRY(cudaEventRecord(h->ev[5], h->stream));
  h->have_eval = true;
  return 0;
}

// Evaluate the (model, phase, S) units given as one S bit-mask per mp (bit S set =
// evaluate stage count S). Multi-GPU ranks pass disjoint masks (paper_2605_04357_b200/
// shard.py assigns them); records then hold each candidate's best over its S subset.
int coral_s1_evaluate_units(coral_s1_handle* h, const uint32_t* smask) {
  if (!h || !h->have_enum) return fail(CORAL_S1_EINVAL, "enumerate first");
  if (!smask) return fail(CORAL_S1_EINVAL, "null mask");
  std::vector<uint32_t> mk(smask, smask + (size_t)h->NM * h->NP);
  return evaluate_units(h, [&](int mp, int S) { return ((mk[mp] >> S) & 1u) != 0; });
}

int coral_s1_evaluate_pieces(coral_s1_handle* h, int n, const int32_t* mp, const uint32_t* smask,
                             const int64_t* lo, const int64_t* hi) {
  if (!h || !h->have_enum) return fail(CORAL_S1_EINVAL, "enumerate first");
  if (n < 0 || (n && (!mp || !smask || !lo || !hi))) return fail(CORAL_S1_EINVAL, "bad pieces");
  std::vector<Piece> pieces;
  for (int i = 0; i < n; ++i) pieces.push_back(Piece{mp[i], smask[i], lo[i], hi[i]});
  return evaluate_pieces(h, pieces);
}

int coral_s1_kernel_launches(const coral_s1_handle* h, int64_t cap, int32_t* kind, int32_t* mp, double* ms,
                             int64_t* n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  const int64_t k = std::min<int64_t>(cap, h->ntimed);
  for (int64_t i = 0; i < k; ++i) {
    float t = 0;
    CUDA_TRY(cudaEventSynchronize(h->tev[i][1]));
    CUDA_TRY(cudaEventElapsedTime(&t, h->tev[i][0], h->tev[i][1]));
    kind[i] = h->tkind[i];
    mp[i] = h->tmp[i];
    ms[i] = t;
  }
  if (n) *n = k;
  return 0;
}

int coral_s1_get_records(coral_s1_handle* h, int mp, coral_s1_record* out, int64_t n) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  if (mp < 0 || mp >= h->NM * h->NP) return fail(CORAL_S1_EINVAL, "bad mp index");
  const int64_t cnt = h->cand_off[mp + 1] - h->cand_off[mp];
  if (n < cnt) return fail(CORAL_S1_EINVAL, "output too small");
  if (cnt)
    CUDA_TRY(cudaMemcpyAsync(out, h->rec.as<coral_s1_record>() + h->cand_off[mp],
                             cnt * sizeof(coral_s1_record), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

static int frontier_run(coral_s1_handle* h, int num_regions, const double* prices, bool skyline,
                        int64_t* num_survivors, void* dst_part = nullptr, int64_t dst_item_off = 0,
                        int64_t dst_cap = 0) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  if (num_regions < 0) return fail(CORAL_S1_EINVAL, "num_regions < 0");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  h->num_regions = num_regions;
  CUDA_TRY(cudaEventRecord(h->ev[6], st));
  const int64_t nmax = h->ncand * num_regions;
  int rc;
  std::vector<double> pv(prices, prices + (size_t)num_regions * h->K);
  // the prefilter keeps a few thousand items per solve (c5: ~1e5 of 1.4e9), so the item
  // buffer is bounded: it starts at 1 Mi items, the items pass counts past its end, and
  // only an overflow grows it (to the exact count) and re-runs that pass
  const int64_t icap0 = std::max<int64_t>(std::min<int64_t>(nmax, 1 << 20), (int64_t)(h->items.cap / sizeof(coral_s1_frontier_item)));
  if ((rc = h->items.ensure(std::max<int64_t>(icap0, 1) * sizeof(coral_s1_frontier_item))) ||
      (rc = h->nsel.ensure(32)))
    return rc;
  int64_t n = 0;
  if (dst_part && nmax == 0) {  // nothing to price: an empty slot (count 0)
    CUDA_TRY(cudaMemsetAsync(dst_part, 0, 8, st));
    h->nfront = 0;
    CUDA_TRY(cudaEventRecord(h->ev[7], st));
    if (num_survivors) *num_survivors = -1;
    return 0;
  }
  if (nmax > 0) {
    CUDA_TRY(cudaMemsetAsync(h->nsel.p, 0, 8, st));
    FrontArgs A;
    A.P = h->dp;
    A.keys = h->keys.as<unsigned long long>();
    A.koff = h->koff_d.as<int64_t>();
    A.cand_off = h->cand_off_d.as<int64_t>();
    A.NMP = h->NM * h->NP;
    A.rec = h->rec.as<coral_s1_record>();
    A.ncand = h->ncand;
    A.prices = nullptr;  // the passes price through the token table (tok_price)
    A.R = num_regions;
    A.items = h->items.as<coral_s1_frontier_item>();
    A.nitems = h->nsel.as<unsigned long long>();
    int64_t nblocks = 0;
    {  // only the models this device evaluated (all of them on one GPU), kFrontBlock per block;
       // a run serves the model's evaluated phases together
      if (h->NP > kFrontPhases) return fail(CORAL_S1_EUNSUPPORTED, "frontier: at most 2 phases");
      std::vector<int64_t> boff(1, 0);
      std::vector<int> rm;
      std::vector<unsigned char> rph;
      for (int m = 0; m < h->NM; ++m) {
        const int64_t c = h->counts[m];
        unsigned char ph = 0;
        for (int p = 0; p < h->NP; ++p) {
          const int mp = m * h->NP + p;
          if (mp >= (int)h->own_mp.size() || h->own_mp[mp]) ph |= (unsigned char)(1u << p);
        }
        if (!c || !ph) continue;
        rm.push_back(m);
        rph.push_back(ph);
        boff.push_back(boff.back() + (c + kFrontBlock - 1) / kFrontBlock);
      }
      if (rm.empty()) { rm.push_back(0); rph.push_back(0); boff.push_back(0); }  // non-empty device arrays
      rph.resize((rph.size() + 7) & ~size_t(7), 0);
      if ((rc = upload_same(h, h->run_off_d, boff)) || (rc = upload_same(h, h->run_mp_d, rm)) ||
          (rc = upload_same(h, h->run_ph_d, rph)))
        return rc;
      A.run_boff = h->run_off_d.as<int64_t>();
      A.run_mp = h->run_mp_d.as<int>();
      A.run_ph = h->run_ph_d.as<unsigned char>();
      A.nrun = (int)rm.size();
      A.rect = h->rect.as<double>();
      nblocks = boff.back();
      std::vector<double> tp((size_t)std::max(num_regions, 1) * 512, 0.0);
      for (int r = 0; r < num_regions; ++r)
        for (int tok = 0; tok < 512; ++tok) {
          const int rank1 = tok >> 3, cnt = tok & 7;
          if (rank1 >= 1 && rank1 <= h->K && cnt > 0)
            tp[(size_t)r * 512 + tok] = (double)cnt * pv[(size_t)r * h->K + h->inv_rank_h[rank1 - 1]];
        }
      if ((rc = upload_same(h, h->tokp, tp))) return rc;
      A.tok_price = h->tokp.as<double>();
    }
    // exact prefilter: per (segment, price bucket) max T -> prefix max. The bucket range
    // only has to contain every item price (any non-decreasing price -> bucket map keeps
    // the filter exact), so it comes from the price matrix on the host: a combo costs at
    // least the cheapest offered config and at most n_max x the dearest (with margin for
    // rounding; bucket indices are clamped, which keeps the map non-decreasing).
    const unsigned gb = (unsigned)std::max<int64_t>(nblocks, 1);  // kFrontItems candidates per thread, regions looped
    unsigned long long range[2] = {~0ull, 0ull};
    {
      double pmin = HUGE_VAL, pmax = 0.0;
      for (double p : pv)
        if (!std::isnan(p)) { pmin = std::min(pmin, p); pmax = std::max(pmax, p); }
      if (pmin <= pmax && pmax > 0.0) {
        const double lo = pmin > 0.0 ? pmin * (1.0 - 1e-9) : 0.0, hi = pmax * h->n_max * (1.0 + 1e-9);
        std::memcpy(&range[0], &lo, 8);
        std::memcpy(&range[1], &hi, 8);
      }
    }
    int shift = 0, nb = 0;
    unsigned long long base = 0;
    const int64_t nseg = (int64_t)h->NM * h->NP * num_regions;
    if (range[1] >= range[0] && range[1]) {
      shift = 40;  // 11 exponent + 12 mantissa bits; coarser until <= 4096 buckets
      while (((range[1] >> shift) - (range[0] >> shift)) + 1 > 4096) ++shift;
      base = range[0] >> shift;
      nb = (int)(((range[1] >> shift) - base) + 1);
      if ((rc = h->fbucket.ensure(std::max<int64_t>(nseg * nb, 1) * 8))) return rc;
      CUDA_TRY(cudaMemsetAsync(h->fbucket.p, 0, nseg * nb * 8, st));
      frontier_bucket_kernel<<<gb, 256, 0, st>>>(A, shift, base, nb, h->fbucket.as<unsigned long long>());
      LAUNCH_CHECK(h);
      frontier_prefix_kernel<<<(unsigned)nseg, 256, 0, st>>>(nb, h->fbucket.as<unsigned long long>());
      LAUNCH_CHECK(h);
    }
    if (dst_part) {  // straight into the caller's slot: count at dst_part, no host round trip
      A.items = reinterpret_cast<coral_s1_frontier_item*>(static_cast<unsigned char*>(dst_part) + dst_item_off);
      A.cap = (unsigned long long)dst_cap;
      A.nitems = static_cast<unsigned long long*>(dst_part);
      CUDA_TRY(cudaMemsetAsync(dst_part, 0, 8, st));
      frontier_items_kernel<<<gb, 256, 0, st>>>(A, shift, base, nb, h->fbucket.as<unsigned long long>());
      LAUNCH_CHECK(h);
      h->nfront = 0;
      CUDA_TRY(cudaEventRecord(h->ev[7], st));
      if (num_survivors) *num_survivors = -1;
      return 0;
    }
    unsigned long long ni = 0;
    for (int pass = 0; pass < 2; ++pass) {
      A.items = h->items.as<coral_s1_frontier_item>();
      A.cap = h->items.cap / sizeof(coral_s1_frontier_item);
      frontier_items_kernel<<<gb, 256, 0, st>>>(A, shift, base, nb, h->fbucket.as<unsigned long long>());
      LAUNCH_CHECK(h);
      CUDA_TRY(cudaMemcpyAsync(&ni, h->nsel.p, 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (ni <= A.cap) break;
      if ((rc = h->items.ensure(ni * sizeof(coral_s1_frontier_item)))) return rc;  // overflow: exact size
      CUDA_TRY(cudaMemsetAsync(h->nsel.p, 0, 8, st));
    }
    n = (int64_t)ni;
  }
  if (skyline) {
    if ((rc = frontier_segments(h, one_part(h->items.p, n, num_regions), n, true))) return rc;
  } else {  // prefiltered candidates only (their skyline is taken after the multi-GPU merge)
    if ((rc = h->front.ensure(std::max<int64_t>(n, 1) * sizeof(coral_s1_frontier_item)))) return rc;
    if (n)
      CUDA_TRY(cudaMemcpyAsync(h->front.p, h->items.p, n * sizeof(coral_s1_frontier_item),
                               cudaMemcpyDeviceToDevice, st));
    h->nfront = n;
  }
  CUDA_TRY(cudaEventRecord(h->ev[7], st));
  if (num_survivors) *num_survivors = h->nfront;
  return 0;
}

int coral_s1_frontier(coral_s1_handle* h, int num_regions, const double* prices, int64_t* num_survivors) {
  return frontier_run(h, num_regions, prices, true, num_survivors);
}

int coral_s1_frontier_candidates(coral_s1_handle* h, int num_regions, const double* prices,
                                 int64_t* num_candidates) {
  return frontier_run(h, num_regions, prices, false, num_candidates);
}

int coral_s1_frontier_candidates_into(coral_s1_handle* h, int num_regions, const double* prices, void* dev_part,
                                      int64_t item_offset_bytes, int64_t cap) {
  if (!dev_part || cap < 0 || item_offset_bytes < 8 || item_offset_bytes % 8)
    return fail(CORAL_S1_EINVAL, "candidates_into: bad slot");
  return frontier_run(h, num_regions, prices, false, nullptr, dev_part, item_offset_bytes, cap);
}

int coral_s1_frontier_merge_gathered(coral_s1_handle* h, const void* dev_base, int parts, int64_t stride_bytes,
                                     int64_t item_offset_bytes, int64_t cap, int64_t* num_survivors,
                                     int64_t* max_count) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (parts < 1 || !dev_base || cap < 0 || item_offset_bytes < 8) return fail(CORAL_S1_EINVAL, "bad parts");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  if (parts > kMaxParts) {  // headers to the host, then the host-count merge
    std::vector<int64_t> c(parts);
    CUDA_TRY(cudaMemcpy2DAsync(c.data(), 8, dev_base, stride_bytes, 8, parts, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int64_t mx = 0;
    for (int64_t v : c) mx = std::max(mx, v);
    if (max_count) *max_count = mx;
    if (mx > cap) { h->nfront = 0; if (num_survivors) *num_survivors = -1; return 0; }
    return coral_s1_frontier_merge_parts(h, dev_base, parts, stride_bytes, item_offset_bytes, c.data(), num_survivors);
  }
  int rc;
  if ((rc = h->pcounts.ensure(kPartsCountsLen * 8))) return rc;
  parts_counts_kernel<<<1, 32, 0, st>>>(static_cast<const unsigned char*>(dev_base), stride_bytes, parts, cap,
                                        h->pcounts.as<long long>());
  LAUNCH_CHECK(h);
  FrontParts F{};
  F.base = static_cast<const unsigned char*>(dev_base);
  F.stride = stride_bytes;
  F.offset = item_offset_bytes;
  F.nparts = parts;
  F.R = h->num_regions;
  F.dn = h->pcounts.as<long long>();
  long long dn[kPartsCountsLen] = {};
  if ((rc = frontier_segments(h, F, (int64_t)parts * cap, false, dn))) return rc;
  const long long mx = dn[2 * kMaxParts + 1];
  if (max_count) *max_count = mx;
  if (mx > cap) { h->nfront = 0; if (num_survivors) *num_survivors = -1; return 0; }
  if (num_survivors) *num_survivors = h->nfront;
  return 0;
}

int coral_s1_get_frontier(coral_s1_handle* h, coral_s1_frontier_item* out, int64_t n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (n < h->nfront) return fail(CORAL_S1_EINVAL, "output too small");
  if (h->nfront)
    CUDA_TRY(cudaMemcpyAsync(out, h->front.p, h->nfront * sizeof(coral_s1_frontier_item),
                             cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int coral_s1_frontier_export_device(coral_s1_handle* h, void* dev_items, int64_t cap, int64_t* n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (n) *n = h->nfront;
  if (cap < h->nfront) return fail(CORAL_S1_EINVAL, "export capacity too small");
  if (h->nfront)
    CUDA_TRY(cudaMemcpyAsync(dev_items, h->front.p, h->nfront * sizeof(coral_s1_frontier_item),
                             cudaMemcpyDeviceToDevice, h->stream));
  return 0;
}

int coral_s1_frontier_merge_device(coral_s1_handle* h, const void* dev_items, int64_t n,
                                   int64_t* num_survivors) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (n < 0 || (n && !dev_items)) return fail(CORAL_S1_EINVAL, "bad items");
  CUDA_TRY(cudaSetDevice(h->device));
  int rc;
  if ((rc = frontier_segments(h, one_part(dev_items, n, h->num_regions), n, dev_items == h->items.p))) return rc;
  if (num_survivors) *num_survivors = h->nfront;
  return 0;
}

int coral_s1_frontier_merge_parts(coral_s1_handle* h, const void* dev_base, int parts, int64_t stride_bytes,
                                  int64_t item_offset_bytes, const int64_t* counts, int64_t* num_survivors) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (parts < 0 || (parts && !dev_base) || (parts && !counts)) return fail(CORAL_S1_EINVAL, "bad parts");
  CUDA_TRY(cudaSetDevice(h->device));
  int64_t n = 0;
  for (int p = 0; p < parts; ++p) {
    if (counts[p] < 0) return fail(CORAL_S1_EINVAL, "negative part count");
    n += counts[p];
  }
  int rc;
  if (parts <= kMaxParts) {  // the gathered buffer is read in place
    FrontParts F{};
    F.base = static_cast<const unsigned char*>(dev_base);
    F.stride = stride_bytes;
    F.offset = item_offset_bytes;
    F.nparts = parts;
    F.R = h->num_regions;
    F.first[0] = 0;
    for (int p = 0; p < parts; ++p) { F.n[p] = counts[p]; F.first[p + 1] = F.first[p] + counts[p]; }
    if ((rc = frontier_segments(h, F, n, false))) return rc;
  } else {
    if ((rc = h->items.ensure(std::max<int64_t>(n, 1) * sizeof(coral_s1_frontier_item)))) return rc;
    int64_t at = 0;
    for (int p = 0; p < parts; ++p) {
      if (!counts[p]) continue;
      const char* src = static_cast<const char*>(dev_base) + p * stride_bytes + item_offset_bytes;
      CUDA_TRY(cudaMemcpyAsync(h->items.as<coral_s1_frontier_item>() + at, src,
                               counts[p] * sizeof(coral_s1_frontier_item), cudaMemcpyDeviceToDevice, h->stream));
      at += counts[p];
    }
    if ((rc = frontier_segments(h, one_part(h->items.p, n, h->num_regions), n, true))) return rc;
  }
  if (num_survivors) *num_survivors = h->nfront;
  return 0;
}

int coral_s1_placement_search(coral_s1_handle* h, int64_t ncases, const int32_t* ncfg,
                              const int64_t* counts, const int32_t* lsteps, const int64_t* tput_off,
                              const double* tput, int64_t tput_len, const int32_t* S, double* best,
                              int64_t* stage_j, int64_t* stage_counts) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (ncases <= 0) return 0;
  CUDA_TRY(cudaSetDevice(h->device));
  int maxLu = 1, maxM = 1, maxN = 0;
  for (int64_t i = 0; i < ncases; ++i) {
    if (ncfg[i] < 1 || ncfg[i] > kMaxC) return fail(CORAL_S1_EUNSUPPORTED, "placement_search: 1..7 configs");
    long long M = 1;
    for (int c = 0; c < ncfg[i]; ++c) {
      if (counts[i * kMaxC + c] < 0) return fail(CORAL_S1_EINVAL, "negative count");
      M *= counts[i * kMaxC + c] + 1;
    }
    if (M > kMaxM) return fail(CORAL_S1_EUNSUPPORTED, "placement_search: prod(counts+1) must be <= 128");
    long long nodes = 0;
    for (int c = 0; c < ncfg[i]; ++c) nodes += counts[i * kMaxC + c];
    if (nodes > CORAL_S1_MAX_NODES)  // the DP's per-size tables hold <= 7 nodes
      return fail(CORAL_S1_EUNSUPPORTED, "placement_search: at most 7 nodes per multiset");
    maxM = std::max(maxM, (int)M);
    maxN = std::max(maxN, (int)nodes);
    if (lsteps[i] < 1 || lsteps[i] > CORAL_S1_MAX_LAYER_UNITS)
      return fail(CORAL_S1_EUNSUPPORTED, "placement_search: 1..128 layer units");
    if (tput_off[i] < 0 || tput_off[i] + (int64_t)ncfg[i] * lsteps[i] > tput_len)
      return fail(CORAL_S1_EINVAL, "tput offset out of range");
    maxLu = std::max(maxLu, (int)lsteps[i]);
  }
  for (int64_t i = 0; i < tput_len; ++i)
    if (tput[i] < 0) return fail(CORAL_S1_EINVAL, "throughput table must be non-negative");
  cudaStream_t st = h->stream;
  // pack inputs: ncfg | lsteps | S | counts | tput_off | tput
  const size_t b_ncfg = ncases * 4, b_counts = ncases * kMaxC * 8, b_off = ncases * 8,
               b_tput = std::max<int64_t>(tput_len, 1) * 8;
  size_t o = 0;
  const size_t o_ncfg = o; o += (b_ncfg + 15) & ~15ull;
  const size_t o_ls = o; o += (b_ncfg + 15) & ~15ull;
  const size_t o_S = o; o += (b_ncfg + 15) & ~15ull;
  const size_t o_cnt = o; o += (b_counts + 15) & ~15ull;
  const size_t o_off = o; o += (b_off + 15) & ~15ull;
  const size_t o_tp = o; o += b_tput;
  const size_t ob_best = 0, ob_sj = (ncases * 8 + 15) & ~15ull,
               ob_sc = ob_sj + ((ncases * kMaxC * 8 + 15) & ~15ull),
               ob_end = ob_sc + ncases * kMaxC * kMaxC * 8;
  int rc;
  if ((rc = h->op_in.ensure(o)) || (rc = h->op_out.ensure(ob_end))) return rc;
  auto* in = h->op_in.as<unsigned char>();
  CUDA_TRY(cudaMemcpyAsync(in + o_ncfg, ncfg, b_ncfg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(in + o_ls, lsteps, b_ncfg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(in + o_S, S, b_ncfg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(in + o_cnt, counts, b_counts, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(in + o_off, tput_off, b_off, cudaMemcpyHostToDevice, st));
  if (tput_len) CUDA_TRY(cudaMemcpyAsync(in + o_tp, tput, tput_len * 8, cudaMemcpyHostToDevice, st));
  auto* out = h->op_out.as<unsigned char>();
  OpArgs A;
  A.ncfg = (const int*)(in + o_ncfg);
  A.lsteps = (const int*)(in + o_ls);
  A.S = (const int*)(in + o_S);
  A.counts = (const long long*)(in + o_cnt);
  A.tput_off = (const long long*)(in + o_off);
  A.tput = (const double*)(in + o_tp);
  A.best = (double*)(out + ob_best);
  A.stage_j = (long long*)(out + ob_sj);
  A.stage_counts = (long long*)(out + ob_sc);
  A.ncases = ncases;
  const size_t smem = dp_smem_bytes(maxM, maxLu + 1, maxLu, maxN - 2);
  if (smem > h->dp_smem_limit)
    return fail(CORAL_S1_EUNSUPPORTED, "placement_search: multiset x layer units exceed shared memory");
  placement_op_kernel<<<(unsigned)ncases, kDpThreads, smem, st>>>(A);
  LAUNCH_CHECK(h);
  CUDA_TRY(cudaMemcpyAsync(best, out + ob_best, ncases * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(stage_j, out + ob_sj, ncases * kMaxC * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(stage_counts, out + ob_sc, ncases * kMaxC * kMaxC * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return 0;
}

int coral_s1_sweep(coral_s1_handle* h, int ncaps, const int32_t* n_max, const double* rho,
                   int num_regions, const double* prices, uint32_t phase_mask, int64_t* counts,
                   double* best, int64_t* unpriced, int64_t* mp_counts) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  if (ncaps < 0 || num_regions < 0) return fail(CORAL_S1_EINVAL, "bad sizes");
  for (int k = 0; k < ncaps; ++k)
    if (n_max[k] > h->n_max) return fail(CORAL_S1_EINVAL, "sweep caps must lie inside the solved caps");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  int rc;
  const int NMP = h->NM * h->NP;
  std::vector<double> pv(prices, prices + (size_t)num_regions * h->K);
  std::vector<int> nv(n_max, n_max + ncaps);
  std::vector<double> rv(rho, rho + ncaps);
  DevBuf capn, caprho, out;
  const size_t nout = (size_t)std::max(ncaps, 1) * (3 + NMP);  // counts | best | unpriced | [caps][mp]
  if ((rc = upload(h, h->prices, pv)) || (rc = upload(h, capn, nv)) || (rc = upload(h, caprho, rv)) ||
      (rc = out.ensure(nout * 8)))
    return rc;
  CUDA_TRY(cudaMemsetAsync(out.p, 0, nout * 8, st));
  FrontArgs A;
  A.P = h->dp;
  A.keys = h->keys.as<unsigned long long>();
  A.koff = h->koff_d.as<int64_t>();
  A.cand_off = h->cand_off_d.as<int64_t>();
  A.NMP = NMP;
  A.rec = h->rec.as<coral_s1_record>();
  A.ncand = h->ncand;
  A.prices = h->prices.as<double>();
  A.R = num_regions;
  A.items = nullptr;
  A.nitems = nullptr;
  unsigned long long* o = out.as<unsigned long long>();
  const int nc = std::max(ncaps, 1);
  if (h->ncand > 0 && ncaps > 0) {
    sweep_kernel<<<(unsigned)((h->ncand + 255) / 256), 256, 0, st>>>(A, ncaps, capn.as<int>(), caprho.as<double>(),
                                                                    phase_mask, o, o + nc, o + 2 * nc, o + 3 * nc);
    LAUNCH_CHECK(h);
  }
  std::vector<unsigned long long> hv(nout);
  CUDA_TRY(cudaMemcpyAsync(hv.data(), out.p, nout * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int k = 0; k < ncaps; ++k) {
    counts[k] = (int64_t)hv[k];
    unsigned long long b = hv[nc + k];
    double d;
    memcpy(&d, &b, 8);
    best[k] = d;
    if (unpriced) unpriced[k] = (int64_t)hv[2 * nc + k];
    if (mp_counts)
      for (int mp = 0; mp < NMP; ++mp) mp_counts[(size_t)k * NMP + mp] = (int64_t)hv[3 * nc + (size_t)k * NMP + mp];
  }
  return 0;
}

int coral_s1_feasible_counts(coral_s1_handle* h, int64_t* counts, int64_t n) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  const int NMP = h->NM * h->NP;
  if (n < NMP) return fail(CORAL_S1_EINVAL, "output too small");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  DevBuf out;
  int rc;
  if ((rc = out.ensure((size_t)std::max(NMP, 1) * 8))) return rc;
  CUDA_TRY(cudaMemsetAsync(out.p, 0, (size_t)std::max(NMP, 1) * 8, st));
  if (h->ncand > 0) {
    feasible_count_kernel<<<(unsigned)((h->ncand + 255) / 256), 256, 0, st>>>(
        h->rec.as<coral_s1_record>(), h->cand_off_d.as<int64_t>(), NMP, h->ncand, out.as<unsigned long long>());
    LAUNCH_CHECK(h);
  }
  std::vector<unsigned long long> hv(std::max(NMP, 1));
  CUDA_TRY(cudaMemcpyAsync(hv.data(), out.p, hv.size() * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::string missing;
  for (int mp = 0; mp < NMP; ++mp) {
    counts[mp] = (int64_t)hv[mp];
    const bool owned = mp >= (int)h->own_mp.size() || h->own_mp[mp];
    if (!hv[mp] && owned) missing += (missing.empty() ? "" : ",") + std::to_string(mp);
  }
  // templates.py:499-502: a (model, phase) with no feasible template at all
  if (!missing.empty()) return fail(CORAL_S1_ENOTEMPLATE, "no feasible template for (model, phase) slots " + missing);
  return 0;
}

int coral_s1_allocation_model(coral_s1_handle* h, int num_regions, const double* prices, const int64_t* avail,
                              const double* demand, int n_mp, const int32_t* mp_order, double prune_ratio,
                              int64_t n_running, const int32_t* run_mp, const int32_t* run_region,
                              const uint64_t* run_key, int64_t* num_vars, int64_t* num_pruned,
                              double* best_eff) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  if (num_regions < 0 || num_regions > 32) return fail(CORAL_S1_EUNSUPPORTED, "allocation model: 0..32 regions");
  if (n_mp < 0 || n_running < 0 || (n_running && (!run_mp || !run_region || !run_key)))
    return fail(CORAL_S1_EINVAL, "bad allocation inputs");
  const int NMP = h->NM * h->NP;
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const int K = h->K;
  for (int64_t i = 0; i < (int64_t)num_regions * K; ++i)
    if (avail[i] < 0) return fail(CORAL_S1_EINVAL, "negative availability");
  // slots with demand > 0, library order (allocation.py:128-130)
  std::vector<int64_t> roff(1, 0);
  std::vector<int> rmp;
  for (int i = 0; i < n_mp; ++i) {
    const int mp = mp_order[i];
    if (mp < 0 || mp >= NMP) return fail(CORAL_S1_EINVAL, "bad mp in order");
    if (!(demand[mp] > 0.0)) continue;
    rmp.push_back(mp);
    roff.push_back(roff.back() + (h->cand_off[mp + 1] - h->cand_off[mp]));
  }
  if (rmp.empty()) rmp.push_back(0);
  const int64_t ntot = roff.back();
  // running pairs sorted by (mp, key, region) for the device lookup
  std::vector<int64_t> ord((size_t)n_running);
  for (int64_t i = 0; i < n_running; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    if (run_mp[a] != run_mp[b]) return run_mp[a] < run_mp[b];
    if (run_key[a] != run_key[b]) return run_key[a] < run_key[b];
    return run_region[a] < run_region[b];
  });
  std::vector<int> rm(std::max<int64_t>(n_running, 1)), rr(std::max<int64_t>(n_running, 1));
  std::vector<unsigned long long> rk(std::max<int64_t>(n_running, 1));
  for (int64_t i = 0; i < n_running; ++i) { rm[i] = run_mp[ord[i]]; rr[i] = run_region[ord[i]]; rk[i] = run_key[ord[i]]; }
  std::vector<double> pv(prices, prices + (size_t)num_regions * K), dv(demand, demand + NMP);
  std::vector<long long> av(avail, avail + (size_t)num_regions * K);
  const int64_t nblk = (std::max<int64_t>(ntot, 1) + kAllocThreads - 1) / kAllocThreads;
  DevBuf d_av, d_dem, d_rm, d_rr, d_rk, d_roff, d_rmp, d_best, d_flags, d_cnt, d_off, d_np;
  int rc;
  if ((rc = upload(h, h->prices, pv)) || (rc = upload(h, d_av, av)) || (rc = upload(h, d_dem, dv)) ||
      (rc = upload(h, d_rm, rm)) || (rc = upload(h, d_rr, rr)) || (rc = upload(h, d_rk, rk)) ||
      (rc = upload(h, d_roff, roff)) || (rc = upload(h, d_rmp, rmp)) ||
      (rc = d_best.ensure((size_t)std::max(NMP, 1) * 8)) || (rc = d_flags.ensure((size_t)std::max<int64_t>(ntot, 1) * 4)) ||
      (rc = d_cnt.ensure((size_t)(nblk + 1) * 8)) || (rc = d_off.ensure((size_t)(nblk + 1) * 8)) || (rc = d_np.ensure(8)))
    return rc;
  CUDA_TRY(cudaMemsetAsync(d_best.p, 0xFF, (size_t)std::max(NMP, 1) * 8, st));
  CUDA_TRY(cudaMemsetAsync(d_np.p, 0, 8, st));
  CUDA_TRY(cudaMemsetAsync(d_cnt.as<unsigned long long>() + nblk, 0, 8, st));
  AllocArgs A;
  A.P = h->dp;
  A.keys = h->keys.as<unsigned long long>();
  A.koff = h->koff_d.as<int64_t>();
  A.cand_off = h->cand_off_d.as<int64_t>();
  A.rec = h->rec.as<coral_s1_record>();
  A.prices = h->prices.as<double>();
  A.avail = d_av.as<long long>();
  A.demand = d_dem.as<double>();
  A.R = num_regions;
  A.prune_ratio = prune_ratio;
  A.run_mp = d_rm.as<int>();
  A.run_region = d_rr.as<int>();
  A.run_key = d_rk.as<unsigned long long>();
  A.nrunning = n_running;
  A.runs_off = d_roff.as<int64_t>();
  A.runs_mp = d_rmp.as<int>();
  A.nruns = (int)roff.size() - 1;
  A.ntot = ntot;
  A.best_bits = d_best.as<unsigned long long>();
  A.flags = d_flags.as<unsigned>();
  A.blkcnt = d_cnt.as<unsigned long long>();
  A.npruned = d_np.as<unsigned long long>();
  A.out = nullptr;
  A.blkoff = d_off.as<unsigned long long>();
  if (ntot > 0) {
    alloc_best_kernel<<<(unsigned)nblk, kAllocThreads, 0, st>>>(A);
    LAUNCH_CHECK(h);
    alloc_count_kernel<<<(unsigned)nblk, kAllocThreads, 0, st>>>(A);
    LAUNCH_CHECK(h);
  } else {
    CUDA_TRY(cudaMemsetAsync(d_cnt.p, 0, (size_t)(nblk + 1) * 8, st));
  }
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt.as<unsigned long long>(), d_off.as<unsigned long long>(),
                                (int)(nblk + 1), st);
  if ((rc = ensure_tmp(h, tmp))) return rc;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(h->cub_tmp.p, tmp, d_cnt.as<unsigned long long>(),
                                         d_off.as<unsigned long long>(), (int)(nblk + 1), st));
  unsigned long long res[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(&res[0], d_off.as<unsigned long long>() + nblk, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&res[1], d_np.p, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nv = (int64_t)res[0];
  if ((rc = h->avars.ensure((size_t)std::max<int64_t>(nv, 1) * sizeof(coral_s1_alloc_var)))) return rc;
  A.out = h->avars.as<coral_s1_alloc_var>();
  if (nv > 0) {
    alloc_emit_kernel<<<(unsigned)nblk, kAllocThreads, 0, st>>>(A);
    LAUNCH_CHECK(h);
  }
  if (best_eff) {  // per slot min eff; +inf when the slot had no priced template
    std::vector<unsigned long long> bb((size_t)std::max(NMP, 1));
    CUDA_TRY(cudaMemcpyAsync(bb.data(), d_best.p, bb.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int mp = 0; mp < NMP; ++mp) {
      double v = HUGE_VAL;
      if (bb[mp] != ~0ull) memcpy(&v, &bb[mp], 8);
      best_eff[mp] = v;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  h->navars = nv;
  if (num_vars) *num_vars = nv;
  if (num_pruned) *num_pruned = (int64_t)res[1];
  return 0;
}

int coral_s1_get_allocation_vars(coral_s1_handle* h, coral_s1_alloc_var* out, int64_t n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (n < h->navars) return fail(CORAL_S1_EINVAL, "output too small");
  if (h->navars)
    CUDA_TRY(cudaMemcpyAsync(out, h->avars.p, h->navars * sizeof(coral_s1_alloc_var), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int coral_s1_node_queries(coral_s1_handle* h, int64_t n, const int32_t* cfg, const int32_t* model,
                          const int32_t* phase, const int32_t* j, const double* budget, int use_profile,
                          double* tput, int64_t* batch) {
  if (!h || !h->have_problem) return fail(CORAL_S1_EINVAL, "set_problem first");
  if (n <= 0) return 0;
  for (int64_t i = 0; i < n; ++i) {
    if (cfg[i] < 0 || cfg[i] >= h->K || model[i] < 0 || model[i] >= h->NM || j[i] < 1 || !(budget[i] > 0) ||
        (phase[i] != CORAL_S1_PHASE_PREFILL && phase[i] != CORAL_S1_PHASE_DECODE))
      return fail(CORAL_S1_EINVAL, "node query out of range (perf.py:189 asserts budget > 0, j >= 1)");
  }
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  DevBuf in, out;
  const size_t bi = (size_t)n * 4;
  int rc;
  if ((rc = in.ensure(4 * ((bi + 15) & ~15ull) + n * 8)) || (rc = out.ensure(n * 16))) return rc;
  auto* b = in.as<unsigned char>();
  const size_t step = (bi + 15) & ~15ull;
  CUDA_TRY(cudaMemcpyAsync(b, cfg, bi, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b + step, model, bi, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b + 2 * step, phase, bi, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b + 3 * step, j, bi, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b + 4 * step, budget, n * 8, cudaMemcpyHostToDevice, st));
  node_query_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
      h->dp, n, (const int*)b, (const int*)(b + step), (const int*)(b + 2 * step), (const int*)(b + 3 * step),
      (const double*)(b + 4 * step), use_profile, out.as<double>(), (long long*)(out.as<double>() + n));
  LAUNCH_CHECK(h);
  CUDA_TRY(cudaMemcpyAsync(tput, out.p, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(batch, out.as<double>() + n, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  in.release();
  out.release();
  return 0;
}

int coral_s1_format_double(double v, char* out, int cap) {
  if (!out || cap < 40) return fail(CORAL_S1_EINVAL, "buffer too small");
  py_repr_double(v, out);
  return 0;
}

// Stream the evaluated library as the reference's JSONL (templates.py:364-377):
// header line, then one json.dumps(record, sort_keys=True) line per feasible
// template, (model, phase) in mp_order, combos in str order. JSON string fragments
// (json.dumps of names, SLO lists) come from the caller so escaping and number
// types match Python exactly.
int coral_s1_write_library(coral_s1_handle* h, const char* path, const char* header, int n_mp,
                           const int32_t* mp_order, const char* const* model_json,
                           const char* const* phase_json, const char* const* slo_json,
                           const char* const* cfg_json, int64_t* n_written) {
  if (!h || !h->have_eval) return fail(CORAL_S1_EINVAL, "evaluate first");
  if (!path || !header) return fail(CORAL_S1_EINVAL, "null path/header");
  CUDA_TRY(cudaSetDevice(h->device));
  FILE* f = fopen(path, "wb");
  if (!f) return fail(CORAL_S1_EINVAL, std::string("cannot open ") + path);
  std::vector<char> out;
  out.reserve(1 << 24);
  auto put = [&](const char* s, size_t n) { out.insert(out.end(), s, s + n); };
  auto puts_ = [&](const char* s) { put(s, strlen(s)); };
  auto flush = [&]() {
    if (!out.empty()) fwrite(out.data(), 1, out.size(), f);
    out.clear();
  };
  puts_(header);
  put("\n", 1);
  int64_t written = 0;
  std::vector<coral_s1_record> rec;
  std::vector<unsigned long long> keys;
  int keys_model = -1;
  char num[64];
  for (int i = 0; i < n_mp; ++i) {
    const int mp = mp_order[i];
    if (mp < 0 || mp >= h->NM * h->NP) { fclose(f); return fail(CORAL_S1_EINVAL, "bad mp in order"); }
    const int m = mp / h->NP, ph = mp % h->NP;
    const int64_t cnt = h->counts[m];
    if (m != keys_model) {
      keys.resize(cnt);
      if (cnt)
        CUDA_TRY(cudaMemcpyAsync(keys.data(), h->keys.as<unsigned long long>() + h->koff[m], cnt * 8,
                                 cudaMemcpyDeviceToHost, h->stream));
      keys_model = m;
    }
    rec.resize(cnt);
    if (cnt)
      CUDA_TRY(cudaMemcpyAsync(rec.data(), h->rec.as<coral_s1_record>() + h->cand_off[mp],
                               cnt * sizeof(coral_s1_record), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (int64_t c = 0; c < cnt; ++c) {
      const coral_s1_record& r = rec[c];
      if (!r.num_stages) continue;
      puts_("{\"combo\": [");
      for (int t = 0; t < kMaxC; ++t) {
        const unsigned tok = (unsigned)(keys[c] >> (kKeyTokenBits * (kMaxC - 1 - t))) & 511u;
        if (!tok) break;
        if (t) puts_(", ");
        puts_("[");
        puts_(cfg_json[h->inv_rank_h[(tok >> 3) - 1]]);
        put(num, sprintf(num, ", %u]", tok & 7u));
      }
      puts_("], \"layers_per_stage\": [");
      for (int s2 = 0; s2 < r.num_stages; ++s2) put(num, sprintf(num, s2 ? ", %u" : "%u", r.layers_per_stage[s2]));
      puts_("], \"model\": ");
      puts_(model_json[m]);
      put(num, sprintf(num, ", \"num_stages\": %u, \"phase\": ", r.num_stages));
      puts_(phase_json[ph]);
      puts_(", \"slo\": ");
      puts_(slo_json[m]);
      puts_(", \"stage_of_node\": [");
      for (int k = 0; k < r.num_nodes; ++k) put(num, sprintf(num, k ? ", %u" : "%u", r.stage_of_node[k]));
      puts_("], \"throughput_tps\": ");
      put(num, py_repr_double(r.throughput_tps, num));
      puts_("}\n");
      ++written;
      if (out.size() > (1u << 24)) flush();
    }
  }
  flush();
  const bool ok = fclose(f) == 0;
  if (n_written) *n_written = written;
  return ok ? 0 : fail(CORAL_S1_EINVAL, "write failed");
}

int coral_s1_kernel_stats(const coral_s1_handle* h, int kind, double* total_ms, int64_t* launches) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  double tot = 0;
  int64_t n = 0;
  for (int i = 0; i < h->ntimed; ++i) {
    if (h->tkind[i] != kind) continue;
    float t = 0;
    CUDA_TRY(cudaEventSynchronize(h->tev[i][1]));
    CUDA_TRY(cudaEventElapsedTime(&t, h->tev[i][0], h->tev[i][1]));
    tot += t;
    ++n;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = n;
  return 0;
}

int coral_s1_set_census(coral_s1_handle* h, int on) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  int rc;
  if (on && (rc = h->census.ensure(32))) return rc;
  h->census_on = on != 0;
  return 0;
}

int coral_s1_census(coral_s1_handle* h, int64_t* layer_bytes) {
  int64_t v[4] = {0, 0, 0, 0};
  const int rc = coral_s1_census_all(h, v, 4);
  if (layer_bytes) *layer_bytes = v[0];
  return rc;
}

int coral_s1_census_all(coral_s1_handle* h, int64_t* out, int n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  unsigned long long v[4] = {0, 0, 0, 0};
  if (h->census_on) {
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    CUDA_TRY(cudaMemcpy(v, h->census.p, 32, cudaMemcpyDeviceToHost));
  }
  for (int i = 0; i < n && i < 4; ++i) out[i] = (int64_t)v[i];
  return 0;
}

int coral_s1_set_timing(coral_s1_handle* h, int on) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  h->timing = on != 0;
  return 0;
}

int coral_s1_set_streams(coral_s1_handle* h, int n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  if (n < 0 || n > coral_s1_handle::kStreams) return fail(CORAL_S1_EINVAL, "streams must be 0 (default) .. 8");
  h->nstreams = n ? n : h->default_streams;
  return 0;
}

int coral_s1_kernel_timeline(const coral_s1_handle* h, int64_t cap, int32_t* kind, int32_t* stream,
                             double* begin_ms, double* end_ms, int64_t* n) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  const int64_t m = std::min<int64_t>(cap, h->ntimed);
  for (int64_t i = 0; i < m; ++i) {
    float b = 0, e = 0;
    CUDA_TRY(cudaEventSynchronize(h->tev[i][1]));
    CUDA_TRY(cudaEventElapsedTime(&b, h->ev[4], h->tev[i][0]));
    CUDA_TRY(cudaEventElapsedTime(&e, h->ev[4], h->tev[i][1]));
    kind[i] = h->tkind[i];
    stream[i] = h->tslot[i];
    begin_ms[i] = b;
    end_ms[i] = e;
  }
  if (n) *n = m;
  return 0;
}

int coral_s1_window_select_stats(const coral_s1_handle* h, double* ms, int64_t* alg_bytes) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  float t = 0;
  if (h->ws_timed) {
    CUDA_TRY(cudaEventSynchronize(h->ev_ws[1]));
    CUDA_TRY(cudaEventElapsedTime(&t, h->ev_ws[0], h->ev_ws[1]));
  }
  if (ms) *ms = h->ws_timed ? t : -1.0;
  if (alg_bytes) *alg_bytes = h->ws_timed ? h->ws_bytes : 0;
  return 0;
}

int coral_s1_stage_ms(const coral_s1_handle* h, double* tables_ms, double* enumerate_ms,
                      double* evaluate_ms, double* frontier_ms) {
  if (!h) return fail(CORAL_S1_EINVAL, "null handle");
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  float t = 0;
  double* outs[4] = {tables_ms, enumerate_ms, evaluate_ms, frontier_ms};
  for (int i = 0; i < 4; ++i) {
    if (!outs[i]) continue;
    *outs[i] = -1.0;
    if (cudaEventElapsedTime(&t, h->ev[2 * i], h->ev[2 * i + 1]) == cudaSuccess) *outs[i] = t;
    else cudaGetLastError();
  }
  return 0;
}

}  // extern "C"
