// lattice.cuh — the placement DP evaluated once per sub-multiset, shared by every
// candidate combo that contains it.
//
// The reference (kernels.py:143-276, _placement_dp_nb) runs an independent DP per
// candidate combo: f[sg][l][rem] over the combo's sub-multisets rem. Nothing in a
// cell depends on the enclosing combo:
//   * value[u][j] = sum over u's configs (name order) of digit * tput[c][j-1]
//     (kernels.py:164-170; zero digits add +0.0), a function of u alone;
//   * the u loop visits sub-multisets of rem in increasing mixed-radix code order
//     (kernels.py:204), which is lexicographic with the highest-named config most
//     significant — identical for every combo containing rem;
//   * the size filter (:207) and the crossing rule (:210-253) read only u, rem-u.
// So f_S[sg][X][l] and its (u, j) choice are functions of the multiset X, and one
// table per (model, phase, S, sg) over all multisets X serves every candidate:
// 9.6e8 (u, l) pairs for BASELINE config 2 instead of 1.56e11 in the reference
// (measured in DESIGN.md).
//
// Cells computed per (S, sg): X with sg <= |X| <= maxn(X) - (S - sg), l in
// [sg, Lu - (S - sg)], where maxn(X) is the largest candidate containing X — exactly
// the cells some candidate's DP can reach. The top cell (S, Lu, full) is per
// candidate. Choices are stored per cell (u as X-local code, j) and walked back for
// the candidates whose best S improves.
//
// States: multisets of 1..R = n_max-1 configs, indexed size-major and colex within a
// size: idx = base[s] + sum_i C(a_i + i, i + 1) for sorted picks a_0 <= ... <= a_{s-1}.
#pragma once
#include "placement_dp.cuh"

namespace coral {

constexpr int kLatMaxState = kMaxC - 1;  // lattice tables hold |X| <= n_max - 1 <= 6
constexpr int kRankStride = kMaxM;       // rank-table entries per candidate (codes < 2^n)

// Row pitch of the lattice value / f / choice tables: Lu + 1 rounded up to even, so
// every row starts 16-byte aligned and dp_pair's capped search fetches (J, g[1]) with
// one vector load (column 0 holds J / K, columns 1..Lu the values).
__host__ __device__ constexpr int lat_pitch(int Lu) { return (Lu + 2) & ~1; }

struct LatModel {
  int K, R;                 // configs, largest state size (n_max - 1)
  const long long* base;    // [R + 2]: first index of each size (base[1] = 0), base[R+1] = total
  const unsigned long long* binom;  // [160][8]
};

__device__ __forceinline__ unsigned long long lat_binom(const LatModel& L, int N, int k) {
  if (k < 0 || N < k) return 0ull;
  return L.binom[N * 8 + k];
}

// colex index of the multiset given by ascending picks
__device__ __forceinline__ long long lat_rank(const LatModel& L, const int* picks, int s) {
  unsigned long long r = 0;
  for (int i = 0; i < s; ++i) r += lat_binom(L, picks[i] + i, i + 1);
  return L.base[s] + (long long)r;
}

// index of the multiset sum_t d[t] x cfg[t] (tokens in ascending config order)
__device__ __forceinline__ long long lat_rank_tokens(const LatModel& L, const int* cfg, const int* d,
                                                     int ntok, int* size_out) {
  int picks[kMaxC];
  int s = 0;
  for (int t = 0; t < ntok; ++t)
    for (int k = 0; k < d[t]; ++k) picks[s++] = cfg[t];
  *size_out = s;
  return s ? lat_rank(L, picks, s) : -1;
}

// ---- per-model state tables -------------------------------------------------

// state_key[idx] = packed token key of state idx (same token format as combos).
__global__ void lat_state_keys_kernel(LatModel L, const int* __restrict__ rank1,
                                      unsigned long long* __restrict__ state_key) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L.base[L.R + 1]) return;
  int s = 1;
  while (idx >= L.base[s + 1]) ++s;
  unsigned long long r = (unsigned long long)(idx - L.base[s]);
  int b[kMaxC];
  for (int i = s - 1; i >= 0; --i) {  // colex unrank
    int v = i;
    while (lat_binom(L, v + 1, i + 1) <= r) ++v;
    b[i] = v;
    r -= lat_binom(L, v, i + 1);
  }
  unsigned long long key = 0;
  int ntok = 0;
  for (int i = 0; i < s;) {
    const int a = b[i] - i;
    int j = i;
    while (j < s && b[j] - j == a) ++j;
    key = (key << 9) | ((unsigned long long)rank1[a] << 3) | (unsigned long long)(j - i);
    ++ntok;
    i = j;
  }
  state_key[idx] = key << (9 * (kMaxC - ntok));
}

// decode a packed key into ascending config indices + counts
__device__ __forceinline__ int lat_tokens(const int* __restrict__ inv_rank, unsigned long long key,
                                          int* cfg, int* cnt) {
  int C = 0;
  for (int t = 0; t < kMaxC; ++t) {
    const unsigned tok = (unsigned)(key >> (9 * (kMaxC - 1 - t))) & 511u;
    if (!tok) break;
    cfg[C] = inv_rank[(tok >> 3) - 1];
    cnt[C] = tok & 7u;
    ++C;
  }
  return C;
}

// Closed form of maxn (a superset of the exact one, so it can only add cells):
// maxn(X) = |X| + max k such that some k configs E make lo <= mem(X)+mem(E) < hi
// (templates.py:107-111 window), with a relative slack eps; sums[soff[k]..soff[k+1])
// are the sorted achievable memories of k-config multisets. 0 if none.
__global__ void lat_maxn_closed_kernel(LatModel L, const int* __restrict__ inv_rank,
                                       const unsigned long long* __restrict__ state_key,
                                       const double* __restrict__ mem_bytes,
                                       const double* __restrict__ sums, const int* __restrict__ soff,
                                       double lo, double hi, double eps, int n_max,
                                       unsigned* __restrict__ maxn) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L.base[L.R + 1]) return;
  int cfg[kMaxC], cnt[kMaxC];
  const int C = lat_tokens(inv_rank, state_key[idx], cfg, cnt);
  double m = 0.0;
  int s = 0;
  for (int c = 0; c < C; ++c) { s += cnt[c]; for (int k = 0; k < cnt[c]; ++k) m += mem_bytes[cfg[c]]; }
  unsigned best = 0;
  for (int k = min(n_max - s, n_max - 1); k >= 0 && !best; --k) {
    const double a = lo - m - eps, b = hi - m + eps;  // need some sum in [a, b)
    int l = soff[k], r = soff[k + 1];                  // first sum >= a
    while (l < r) { const int mid = (l + r) >> 1; if (sums[mid] < a) l = mid + 1; else r = mid; }
    if (l < soff[k + 1] && sums[l] < b) best = (unsigned)(s + k);
  }
  maxn[idx] = best;
}

// ceil(2^16 / r) for radices r = 1..8: q = (x * kLatMagic[r]) >> 16 equals x / r for
// every x < 2^16 / 8 (the error term x * (m r - 2^16) stays below 2^16), and sub-multiset
// codes are < 128.
__constant__ unsigned kLatMagic[9] = {0u, 65536u, 32768u, 21846u, 16384u, 13108u, 10923u, 9363u, 8192u};

// Colex sums of the sub-multiset u = digits(code) of the packed key (token 0 is the
// least significant mixed-radix digit, radix count + 1 -- the code order of
// kernels.py:204) and, with kRest, of its complement key - u. The picks of u are
// d_t copies of cfg_t in token order, so pick i contributes C(cfg_t + i, i + 1)
// (lat_rank); a token's run of picks telescopes to two table entries. Registers only:
// the token loop is unrolled and digits come from a multiply-high, not a division.
template <bool kRest>
__device__ __forceinline__ int lat_code_ranks(const LatModel& L, const int* __restrict__ inv_rank,
                                              unsigned long long key, unsigned code, int* su,
                                              unsigned long long* au, int* sr, unsigned long long* ar) {
  unsigned rest = code;
  int M = 1, pu = 0, pr = 0;
  unsigned long long accu = 0, accr = 0;
#pragma unroll
  for (int t = 0; t < kMaxC; ++t) {
    const unsigned tok = (unsigned)(key >> (9 * (kMaxC - 1 - t))) & 511u;
    if (tok) {
      const int cfg = __ldg(inv_rank + (tok >> 3) - 1);
      const unsigned c = tok & 7u, radix = c + 1u;
      const unsigned q = (rest * kLatMagic[radix]) >> 16;
      const unsigned d = rest - q * radix;
      rest = q;
      M *= (int)radix;
      // picks p..p+d-1 of value a add sum_{j=p+1}^{p+d} C(a-1+j, j)
      //   = C(a+p+d, p+d) - C(a+p, p)   (hockey stick; 0 for a = 0)
      accu += __ldg(L.binom + (cfg + pu + (int)d) * 8 + pu + (int)d) - __ldg(L.binom + (cfg + pu) * 8 + pu);
      pu += (int)d;
      if (kRest) {
        const int e = (int)(c - d);
        accr += __ldg(L.binom + (cfg + pr + e) * 8 + pr + e) - __ldg(L.binom + (cfg + pr) * 8 + pr);
        pr += e;
      }
    }
  }
  *su = pu;
  *au = accu;
  if (kRest) {
    *sr = pr;
    *ar = accr;
  }
  return M;
}

// Per candidate and u code < M: size(u) << 24 | idx(u) (idx 0 when |u| > R; entries
// past M are never read). The top cells read idx(full - u) as the entry of code
// M-1-code. Shared by both phases of a model. Persistent warps, one candidate per
// warp iteration (next key prefetched), lane = code (two rounds when M > 32). Every
// table entry lat_code_ranks' telescoped sums touch is C(cfg + k, k) with cfg < K and
// k <= n_max, so the block stages those rows (32-bit: C(62 + 6, 6) < 2^32) and the
// config ranks in shared memory once; the (cfg + p) * 8 + p addresses of a warp's
// lanes fall in distinct banks.
constexpr int kRanksWarps = 8;
constexpr int kRanksRows = CORAL_S1_MAX_CONFIGS + kMaxC + 1;
__global__ void __launch_bounds__(kRanksWarps * 32) lat_ranks_kernel(
    LatModel L, const int* __restrict__ inv_rank, const unsigned long long* __restrict__ keys,
    long long ncombo, unsigned* __restrict__ ranks) {
  __shared__ unsigned sBin[kRanksRows * 8];  // [N][k] flattened: C(N, k) at N * 8 + k
  __shared__ int sInv[CORAL_S1_MAX_CONFIGS];
  for (int e = threadIdx.x; e < (L.K + kMaxC + 1) * 8; e += blockDim.x) sBin[e] = (unsigned)L.binom[e];
  for (int e = threadIdx.x; e < L.K; e += blockDim.x) sInv[e] = inv_rank[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * kRanksWarps;
  long long ci = (long long)blockIdx.x * kRanksWarps + (threadIdx.x >> 5);
  unsigned long long key = ci < ncombo ? keys[ci] : 0ull;
  for (; ci < ncombo; ci += nwarps) {
    const unsigned long long cur = key;
    if (ci + nwarps < ncombo) key = keys[ci + nwarps];
    // per token: table row base cfg * 8, radix, multiply-high constant. An empty slot
    // has radix 1 (digit 0), so it adds C(N, p) - C(N, p) = 0: no branches below.
    unsigned cb[kMaxC], radix[kMaxC], magic[kMaxC];
    int M = 1;
#pragma unroll
    for (int t = 0; t < kMaxC; ++t) {
      const unsigned tok = (unsigned)(cur >> (9 * (kMaxC - 1 - t))) & 511u;
      cb[t] = (unsigned)sInv[max((int)(tok >> 3) - 1, 0)] * 8u;
      radix[t] = (tok & 7u) + 1u;
      magic[t] = kLatMagic[radix[t]];
      M *= (int)radix[t];
    }
    unsigned* out = ranks + ci * kRankStride;
    for (unsigned code = lane; (int)code < M; code += 32) {
      unsigned rest = code, acc = 0, p9 = 0;  // p9 = 9 * picks so far: C(cfg + p, p) at cb + 9p
#pragma unroll
      for (int t = 0; t < kMaxC; ++t) {
        const unsigned q = (rest * magic[t]) >> 16;
        const unsigned d9 = (rest - q * radix[t]) * 9u;
        rest = q;
        acc += sBin[cb[t] + p9 + d9] - sBin[cb[t] + p9];
        p9 += d9;
      }
      const int pu = (int)(p9 / 9u);
      out[code] = ((unsigned)pu << 24) | (pu >= 1 && pu <= L.R ? (unsigned)(L.base[pu] + (long long)acc) : 0u);
    }
  }
}

// nsub[idx] = M(X) = prod(counts + 1)
__global__ void lat_nsub_kernel(LatModel L, const unsigned long long* __restrict__ state_key,
                                long long* __restrict__ nsub) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = L.base[L.R + 1];
  if (idx > tot) return;
  if (idx == tot) { nsub[idx] = 0; return; }
  const unsigned long long key = state_key[idx];
  long long M = 1;
  for (int t = 0; t < kMaxC; ++t) {
    const unsigned tok = (unsigned)(key >> (9 * (kMaxC - 1 - t))) & 511u;
    if (!tok) break;
    M *= (tok & 7u) + 1;
  }
  nsub[idx] = M;
}

// subtab[off[X] + code] = {size(u) << 24 | idx(u), idx(X - u)} for code in [0, M(X)).
// Warp per state X, lane = code (+32): |X| <= R <= 6 gives M(X) <= 64.
__global__ void lat_subtab_kernel(LatModel L, const int* __restrict__ inv_rank,
                                  const unsigned long long* __restrict__ state_key,
                                  const long long* __restrict__ off, uint2* __restrict__ subtab) {
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (idx >= L.base[L.R + 1]) return;
  const unsigned long long key = state_key[idx];
  for (unsigned code = threadIdx.x & 31u;; code += 32u) {
    int su, sr;
    unsigned long long au, ar;
    const int M = lat_code_ranks<true>(L, inv_rank, key, code, &su, &au, &sr, &ar);
    if ((int)code >= M) break;
    subtab[off[idx] + code] =
        make_uint2(((unsigned)su << 24) | (su ? (unsigned)(L.base[su] + (long long)au) : 0u),
                   sr ? (unsigned)(L.base[sr] + (long long)ar) : 0u);
  }
}

// ---- per (model, phase): every S at once ----------------------------------------

// Workspace of one (model, phase) chain: per S = 2..n_max a value table and two
// ping-pong f layers, plus one choice layer per (S, sg), sg = 2..S-1.
struct LatWork {
  double* value;          // [S-2][states][LuP]
  double* f;              // [S-2][2][states][LuP]
  unsigned short* ch;     // [tri(S) + sg-2][states][LuP]
  long long stride;       // states * LuP
  // per-row summaries the top cells read with ONE 32-byte load each (lat_top_kernel):
  //   vsum(S)[X] = {J, value_S[X][1], value_S[X][Lu-S+1], value_S[X][Lu-1]}
  //   fsum(S)[X] = {K, f_S[S-1][X][S-1], f_S[S-1][X][Lu-1], 0}
  double* vsum;           // [S-2][states][4]
  double* fsum;           // [S-2][states][4]
  long long sstride;      // states * 4
  __device__ __forceinline__ double* vs(int S) const { return vsum + (long long)(S - 2) * sstride; }
  __device__ __forceinline__ double* fs(int S) const { return fsum + (long long)(S - 2) * sstride; }
  __device__ __forceinline__ double* val(int S) const { return value + (long long)(S - 2) * stride; }
  __device__ __forceinline__ double* lay(int S, int sg) const {
    return sg == 1 ? val(S) : f + ((long long)(S - 2) * 2 + (sg & 1)) * stride;
  }
  __device__ __forceinline__ unsigned short* chl(int S, int sg) const {
    return ch + ((long long)((S - 3) * (S - 2) / 2) + (sg - 2)) * stride;
  }
};

// value_S[idx][j], j = 1..Lu (kernels.py:164-170) for S in [S_lo, S_lo + gridDim.y);
// warp per row, lanes over j. Column 0 (never read as a value) receives J, the last j
// with value > 0, for dp_pair's search cap.
// Only rows some reader can touch: u is one stage of a candidate whose other S - 1
// stages hold >= 1 node each, so |candidate| >= |u| + S - 1 <= maxn(u) -- true for
// every u the layers (maxn(u) >= maxn(X)), the layer-2 X - u side and the top cell
// read; maxn is a superset bound, so no needed row is skipped.
__global__ void lat_value_kernel(LatModel L, const int* __restrict__ inv_rank,
                                 const unsigned long long* __restrict__ state_key,
                                 const unsigned* __restrict__ maxn,
                                 const double* __restrict__ tab_mp /* [S][K][Lu] */, int K, int Lu,
                                 int S_lo, unsigned smask, LatWork W) {
  const int S = S_lo + blockIdx.y;
  if (!((smask >> S) & 1u)) return;
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= L.base[L.R + 1]) return;
  const unsigned long long key = state_key[idx];
  int n = 0;
  for (int t = 0; t < kMaxC; ++t) n += (int)((key >> (9 * t)) & 7u);
  if ((int)maxn[idx] < n + S - 1) return;  // uniform per warp
  const double* tabS = tab_mp + (long long)(S - 1) * K * Lu;
  int cfg[kMaxC], cnt[kMaxC];
  const int C = lat_tokens(inv_rank, key, cfg, cnt);
  double* row = W.val(S) + idx * lat_pitch(Lu);
  double* sum = W.vs(S) + idx * 4;
  int J = 0;
  for (int j0 = 1; j0 <= Lu; j0 += 32) {
    const int j = j0 + lane;
    double v = 0.0;
    if (j <= Lu) {
      for (int c = 0; c < C; ++c) v = rn_add(v, rn_mul((double)cnt[c], tabS[cfg[c] * Lu + (j - 1)]));
      row[j] = v;
      if (j == 1) sum[1] = v;
      if (j == Lu - S + 1) sum[2] = v;
      if (j == Lu - 1) sum[3] = v;
    }
    const unsigned pos = __ballot_sync(0xffffffffu, j <= Lu && v > 0.0);
    if (pos) J = j0 + 31 - __clz(pos);
  }
  if (lane == 0) {
    row[0] = __longlong_as_double((long long)J);  // J as integer bits
    sum[0] = row[0];
  }
}

// Exactly monotone rows (kMode 1): the crossing count t(l) = #{j <= jmax(l) : g(j) >
// f[l - j]} of one (u, X-u) pair moves by 0 or 1 from cell l - 1 to cell l (g and f are
// non-increasing: t(l) >= t(l-1) since f[l-j] <= f[l-1-j]; t(l) <= t(l-1) + 1 since
// g(j) <= g(j-1) <= f[l-j] past it), and the step test g(t+1) > f[l-1-t] reads exactly
// the two values cell l - 1 loaded for its own result. So a lane that owns kRun
// consecutive cells bisects once (the capped bracket of dp_pair) and then walks: per
// cell the two shortcut tests and two loads, no search. The result of every cell is
// dp_pair's (kernels.py:210-239): shortcut 1 (g(1) <= h(1)) <=> t == 0, shortcut 2,
// else (lo, hi) = (t, t + 1), the unique boundary the reference's bisection finds.
template <int kRun>
__device__ __forceinline__ void layer_run(const double* __restrict__ gv, const double* __restrict__ fr, int l1,
                                          int lmax, int sg, int code, double* best, int* bc) {
  const double2 g01 = *reinterpret_cast<const double2*>(gv);  // (J as integer bits, g(1))
  const int J = __double2loint(g01.x);
  const double g1 = g01.y;
  const double hm = fr[sg - 1];             // h(jmax) = f[l - jmax] = f[sg - 1] for every l
  const int K = __double2loint(fr[0]);      // last l with f > 0
  int t = 0;
  double gt1 = g1, ft = 0.0;                // g(t + 1) and f[l - t] of the previous cell
#pragma unroll
  for (int r = 0; r < kRun; ++r) {
    const int l = l1 + r;
    if (l > lmax) break;
    const int jmax = l - (sg - 1);
    if (r == 0) {
      // cold start: t by the capped bisection (P(j) true below min(J, l-K-1), false
      // above J; P(1) decides t == 0)
      const double h1 = fr[l - 1];
      if (g1 <= h1) {
        t = 0;
      } else {
        int lo = max(1, min(min(J, l - K - 1), jmax));
        int hi = min(J, jmax) + 1;  // P(hi) false (or past jmax)
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (gv[mid] > fr[l - mid]) lo = mid; else hi = mid;
        }
        t = lo;
      }
    } else if (t + 1 <= jmax) {
      t += gt1 > ft ? 1 : 0;  // P_l(t + 1) = g(t + 1) > f[(l - 1) - t]
    }
    if (t == 0) {  // shortcut 1: g(1) <= h(1)
      if (g1 > best[r]) { best[r] = g1; bc[r] = (code << 10) | 1; }
      gt1 = g1;
      if (r + 1 < kRun && l < lmax) ft = fr[l];  // f[l - 0] for the next step
      continue;
    }
    const double gm = gv[jmax];
    const double vlo = fr[l - t];
    const double vhi = gv[t + 1];  // t <= jmax < Lu
    double c;
    int j;
    if (gm >= hm) { c = hm; j = jmax; }  // shortcut 2
    else if (vlo >= vhi) { c = vlo; j = t; }
    else { c = vhi; j = t + 1; }
    if (c > best[r]) { best[r] = c; bc[r] = (code << 10) | j; }
    gt1 = vhi;
    ft = vlo;
  }
}

// DP layer sg for every S in [S_lo, S_lo + gridDim.y) with S > sg: warp per state X,
// lanes over l. Cells: sg <= |X| <= maxn(X) - (S - sg), sg <= l <= Lu - (S - sg).
// kSlots = ceil((M(X) - 1) / 32) code slots per lane: 1 while n_max <= 6 (|X| <= 5),
// 2 for n_max = 7 (|X| <= 6, M(X) <= 64). kMode: 1 = exactly monotone rows (capped
// crossing search, u <-> X-u symmetry at layer 2), 0 = rows monotone only within the
// 1e-12 tolerance (the literal [1, jmax] search), 2 = the full-scan variant (rows that
// fail the monotone test, kernels.py:240-249). One launch per mode; each launch's smask
// holds only the S values of its mode.
template <int kSlots, int kMode, int kLayerRun>
__device__ __forceinline__ void lat_layer_body(
    LatModel L, int sg, int S_lo, unsigned smask, unsigned xmask, int n_max, int Lu,
    const unsigned* __restrict__ maxn, const long long* __restrict__ off,
    const uint2* __restrict__ subtab, LatWork W, unsigned long long* __restrict__ census) {
  const int S = S_lo + blockIdx.y;
  if (!((smask >> S) & 1u) || S <= sg) return;
  const int lane = threadIdx.x & 31;
  const int smaxsz = min(L.R, n_max - (S - sg));
  const long long idx = L.base[sg] + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (smaxsz < sg || idx >= L.base[smaxsz + 1]) return;
  int s = sg;
  while (idx >= L.base[s + 1]) ++s;
  if (s > (int)maxn[idx] - (S - sg)) return;  // no candidate reaches this cell
  const int LuP = lat_pitch(Lu);
  const int lmax = Lu - (S - sg);
  const int usz = s - (sg - 1);  // |u| <= |X| - (sg - 1)
  const long long o = off[idx];
  const long long M = off[idx + 1] - o;
  // Layer 2 reads value rows on both sides: with exactly monotone rows the crossing
  // is the true max, so cand(u) == cand(X-u) (j <-> l-j); the smallest maximising
  // code lies in the lower half (code(X-u) = M-1-code(u)) and only it is searched.
  const long long cmax = (sg == 2 && kMode == 1) ? (M - 1) / 2 + 1 : M;
  (void)xmask;
  // the row bases stay in registers (the compiler would re-derive them from the launch
  // parameters inside the search loop)
  const double* __restrict__ value = W.val(S);
  const double* __restrict__ fprev = W.lay(S, sg - 1);
  asm volatile("" : "+l"(value));
  asm volatile("" : "+l"(fprev));
  double* __restrict__ fout = W.lay(S, sg);
  unsigned short* __restrict__ chout = W.chl(S, sg);
  // u codes of X that pass the size filter: slot k of a lane holds code lane + 1 + 32k;
  // ballot per slot, then compaction (valid code #i at lane i & 31, slot i >> 5)
  uint2 myent[kSlots];
  unsigned vm[kSlots];
  int nv = 0;
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int code = lane + 1 + 32 * k;
    myent[k] = make_uint2(0u, 0u);
    bool ok = false;
    if (code < cmax) {
      myent[k] = subtab[o + code];
      ok = (int)(myent[k].x >> 24) <= usz;
    }
    vm[k] = __ballot_sync(0xffffffffu, ok);
    nv += __popc(vm[k]);
  }
  int kpos = 0;  // last l with f > 0 -> column 0 of the f row (dp_pair's search cap)
  // compacted slot r of a lane: the 32-bit row offsets of its value_S[u] and f[X-u]
  // rows (< 2^32 in the envelope) and its code
  unsigned cvo[kSlots], cfo[kSlots];
  int ccode[kSlots];
#pragma unroll
  for (int r = 0; r < kSlots; ++r) {
    const int i = lane + 32 * r;  // valid code #i
    int before = 0, src = 0, word = 0;
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      const int cnt = __popc(vm[k]);
      if (i >= before && i < before + cnt) { word = k; src = (int)__fns(vm[k], 0, i - before + 1); }
      before += cnt;
    }
    unsigned ex = 0u, ey = 0u;
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      const unsigned x = __shfl_sync(0xffffffffu, myent[k].x, src);
      const unsigned y = __shfl_sync(0xffffffffu, myent[k].y, src);
      if (k == word) { ex = x; ey = y; }
    }
    cvo[r] = (ex & 0xFFFFFFu) * (unsigned)LuP;
    cfo[r] = ey * (unsigned)LuP;
    ccode[r] = src + 1 + 32 * word;
  }
  // census (bench roofline, off in timed runs): algorithmic bytes of this state = its
  // f + choice cells written (10 B each), one read of its value_S and f_{sg-1} rows
  // and of its valid sub-table entries
  if (census && lane == 0) {
    atomicAdd(census, (unsigned long long)(10 * (lmax - sg + 1) + 16 * (Lu + 1) + 8 * nv));
    atomicAdd(census + 1, (unsigned long long)nv * (unsigned long long)(lmax - sg + 1));  // (u, l) pairs
  }
  if (kMode == 1 && kLayerRun > 1) {
    // exactly monotone rows: each lane owns kLayerRun consecutive cells (layer_run)
    for (int l0 = sg; l0 <= lmax; l0 += 32 * kLayerRun) {
      const int wc = min(32 * kLayerRun, lmax - l0 + 1);  // cells of this chunk
      const int wl = (wc + kLayerRun - 1) / kLayerRun;     // lanes they need
      int lw = 0;
      while ((1 << lw) < wl) ++lw;
      const int wp = 1 << lw;
      const int G = 32 >> lw;
      const int g = lane >> lw, i = lane & (wp - 1);
      const int l1 = l0 + i * kLayerRun;
      const bool act = i < wl;
      double best[kLayerRun];
      int bc[kLayerRun];  // code << 10 | j of the best
#pragma unroll
      for (int r = 0; r < kLayerRun; ++r) { best[r] = kNegInf; bc[r] = (1 << 20) << 10; }
      const int T = (nv + G - 1) >> (5 - lw);
      for (int t = 0; t < T; ++t) {
        const int kk = t * G + g;
        const int src = (kk < nv ? kk : 0) & 31, slot = kSlots > 1 && kk < nv ? kk >> 5 : 0;
        unsigned vo = 0u, fo = 0u;
        int code = 0;
#pragma unroll
        for (int r = 0; r < kSlots; ++r) {
          const unsigned a = __shfl_sync(0xffffffffu, cvo[r], src);
          const unsigned b = __shfl_sync(0xffffffffu, cfo[r], src);
          const int c = __shfl_sync(0xffffffffu, ccode[r], src);
          if (r == slot) { vo = a; fo = b; code = c; }
        }
        if (!act || kk >= nv) continue;
        layer_run<kLayerRun>(value + vo, fprev + fo, l1, lmax, sg, code, best, bc);
      }
      int lastpos = 0;
#pragma unroll
      for (int r = 0; r < kLayerRun; ++r) {
        // merge the groups of each cell: value desc, then smallest code
        for (int ofs = wp; ofs < 32; ofs <<= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best[r], ofs);
          const int oc = __shfl_xor_sync(0xffffffffu, bc[r], ofs);
          // value desc, then smallest code (bc orders by code first: j < 1024)
          if (ob > best[r] || (ob == best[r] && oc < bc[r])) { best[r] = ob; bc[r] = oc; }
        }
        const int l = l1 + r;
        if (act && g == 0 && l <= lmax) {
          fout[idx * LuP + l] = best[r];
          chout[idx * LuP + l] = (unsigned short)bc[r];
          if (sg == S - 1) {  // the layer the top cells read: its summary entries
            if (l == S - 1) W.fs(S)[idx * 4 + 1] = best[r];
            if (l == Lu - 1) W.fs(S)[idx * 4 + 2] = best[r];
          }
          if (best[r] > 0.0) lastpos = l;
        }
      }
      kpos = max(kpos, (int)__reduce_max_sync(0xffffffffu, (unsigned)lastpos));
    }
  } else
  for (int l0 = sg; l0 <= lmax; l0 += 32) {
    // lanes = G groups x wp positions; group g takes valid codes g, g+G, g+2G, ...
    const int w = min(32, lmax - l0 + 1);
    int lw = 0;  // wp = 2^lw >= w (powers of two: shifts, not divisions)
    while ((1 << lw) < w) ++lw;
    const int wp = 1 << lw;
    const int G = 32 >> lw;
    const int g = lane >> lw, i = lane & (wp - 1);
    const int l = l0 + i;
    const bool act = i < w;
    const int jmax = l - (sg - 1);
    double best = kNegInf;
    int bc = (1 << 20) << 10;  // best u code << 10 | j
    const int T = (nv + G - 1) >> (5 - lw);
    for (int t = 0; t < T; ++t) {
      const int kk = t * G + g;  // this group's kk-th valid code (ascending per group)
      const int src = (kk < nv ? kk : 0) & 31, slot = kSlots > 1 && kk < nv ? kk >> 5 : 0;
      unsigned vo = 0u, fo = 0u;
      int code = 0;
#pragma unroll
      for (int r = 0; r < kSlots; ++r) {
        const unsigned a = __shfl_sync(0xffffffffu, cvo[r], src);
        const unsigned b = __shfl_sync(0xffffffffu, cfo[r], src);
        const int c = __shfl_sync(0xffffffffu, ccode[r], src);
        if (r == slot) { vo = a; fo = b; code = c; }
      }
      if (!act || kk >= nv) continue;
      double cand;
      int cj;
      dp_pair(value + vo, fprev + fo, l, jmax, kMode != 2, cand, cj, kMode == 1);  // 2: kernels.py:240-249
      if (cand > best) { best = cand; bc = (code << 10) | cj; }
    }
    // merge the groups of each l: value desc, then smallest code (the reference's
    // first strictly better u over the ascending code sequence)
    for (int ofs = wp; ofs < 32; ofs <<= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, ofs);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, ofs);
      if (ob > best || (ob == best && oc < bc)) { best = ob; bc = oc; }  // code first: j < 1024
    }
    if (act && g == 0) {
      fout[idx * LuP + l] = best;
      chout[idx * LuP + l] = (unsigned short)bc;
      if (sg == S - 1) {  // the layer the top cells read: its summary entries
        if (l == S - 1) W.fs(S)[idx * 4 + 1] = best;
        if (l == Lu - 1) W.fs(S)[idx * 4 + 2] = best;
      }
    }
    const unsigned pos = __ballot_sync(0xffffffffu, act && g == 0 && best > 0.0);  // group 0 = lanes 0..wp-1
    if (pos) kpos = l0 + 31 - __clz(pos);
  }
  if (lane == 0) {
    fout[idx * LuP] = __longlong_as_double((long long)kpos);  // K as integer bits
    if (sg == S - 1) W.fs(S)[idx * 4] = fout[idx * LuP];
  }
}

// The layer kernel: one launch per (sg, search mode); lanes own one cell each.
template <int kSlots, int kMode>
__global__ void __launch_bounds__(256, 8) lat_layer_kernel(
    LatModel L, int sg, int S_lo, unsigned smask, unsigned xmask, int n_max, int Lu,
    const unsigned* __restrict__ maxn, const long long* __restrict__ off,
    const uint2* __restrict__ subtab, LatWork W, unsigned long long* __restrict__ census) {
  lat_layer_body<kSlots, kMode, 1>(L, sg, S_lo, smask, xmask, n_max, Lu, maxn, off, subtab, W, census);
}

// Exactly monotone rows of long models (Lu >= kLayerRunMinLu): lanes own two consecutive
// cells (layer_run: one bisection, then the free staircase step; the running best kept
// as value + packed (code, j)) -- fewer probes where the crossing brackets are wide
// (BASELINE config 3, Lu = 80: evaluate 3.56 -> 3.16 ms); with short rows the capped
// bisection is already cheap and the one-cell kernel is faster.
constexpr int kLayerRunMinLu = 56;
template <int kSlots>
__global__ void __launch_bounds__(256, 8) lat_layer_run_kernel(
    LatModel L, int sg, int S_lo, unsigned smask, unsigned xmask, int n_max, int Lu,
    const unsigned* __restrict__ maxn, const long long* __restrict__ off,
    const uint2* __restrict__ subtab, LatWork W, unsigned long long* __restrict__ census) {
  lat_layer_body<kSlots, 1, 2>(L, sg, S_lo, smask, xmask, n_max, Lu, maxn, off, subtab, W, census);
}

}  // namespace coral
