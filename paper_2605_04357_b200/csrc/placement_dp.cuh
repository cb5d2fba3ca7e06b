// placement_dp.cuh — CTA-cooperative exact placement DP for one node multiset.
//
// Reference: _placement_dp_nb, /root/reference/pkg/src/hetserve/kernels.py:143-276
// (numba, the default path; tie rules are defined against it).
//
//   value[u][j]        = sum_c digit_c(u) * tput[c][j-1], summed in c order   (:164-170)
//   f[1][l][rem]       = value[rem][l]                                          (:181-183)
//   f[sg][l][rem]      = max_{u subset rem, |rem|-|u| >= sg-1} cand(u)          (:195-256)
//   cand(u)            = crossing of value[u][.] and f[sg-1][l-.][rem-u],
//                        binary search when tput is monotone (:210-239),
//                        full scan otherwise (:240-249); first strictly better u wins.
//
// B200 restructuring (same values, same tie choices on the decode path):
//  * Only cells the answer can reach are computed: at layer sg < S the cell
//    (l, rem) needs sg <= |rem| <= n-(S-sg) and sg <= l <= Lu-(S-sg); the top layer
//    is the single cell (Lu, full). Every computed cell runs the reference's exact
//    per-cell rule, so the values and the (u, j) choices along the decode path are
//    identical to the full table the reference fills.
//  * f lives in ONE shared-memory buffer updated in place: layer sg writes
//    multiset sizes from large to small, and a cell of size s only reads sizes < s.
//  * Warp task = (rem, 32 consecutive l): the u-loop is warp-uniform (no divergence
//    in trip count); lanes differ only in the binary-search path.
//  * The top cell is split over lanes by u and reduced with the reference's
//    tie rule (largest value, then smallest u code).
//  * Choices are kept as u16 (u << 8 | j) only for layers 2..S-1 (u < 128 codes,
//    j <= 128 layer units).
#pragma once
#include "roofline.cuh"

namespace coral {

constexpr int kMaxC = CORAL_S1_MAX_NODES;  // tokens per key, nodes per multiset, stages
constexpr int kMaxM = 1 << kMaxC;          // sub-multiset codes: prod(counts + 1) <= 2^n
constexpr int kDpWarps = 8;
constexpr int kDpThreads = kDpWarps * 32;

struct DpShared {
  int C, n, M, Lu, LuP, S;
  int cnt[kMaxC];
  int mono;  // np.all(np.diff(tput, axis=1) <= 1e-12) over the rows in use (kernels.py:291)
  unsigned char digits[kMaxM][kMaxC];
  unsigned char sizes[kMaxM];
  unsigned long long contain[kMaxM][2];  // bit u set <=> u is a sub-multiset of rem (128 bits)
  unsigned long long size_le[kMaxC + 2][2];
  unsigned char bysize[kMaxC + 1][kMaxM];
  int nbysize[kMaxC + 1];
  // top-cell result
  double top_val;
  int top_u, top_j;
  // decoded raw placement (kernels.py:258-275)
  int stage_j[kMaxC];
  int stage_u[kMaxC];
};

// Dynamic shared memory carve-up for one CTA.
struct DpBuffers {
  double* value;       // [M][LuP]
  double* f;           // [M][LuP]
  unsigned short* ch;  // [n-2][M][LuP]
  double* tputS;       // [C][Lu]
};
// (choices: [n - 2][M][LuP], layer sg at (sg - 2))

// nlayers = choice layers kept (stage counts S <= n need layers 2..S-1: n - 2)
__host__ __device__ inline size_t dp_smem_bytes(int maxM, int maxLuP, int maxLu, int nlayers) {
  size_t b = 0;
  b += (size_t)maxM * maxLuP * sizeof(double) * 2;
  b += (size_t)(nlayers > 0 ? nlayers : 0) * maxM * maxLuP * sizeof(unsigned short);
  b = (b + 15) & ~(size_t)15;
  b += (size_t)kMaxC * maxLu * sizeof(double);
  return b;
}

__device__ inline DpBuffers dp_carve(unsigned char* smem, int M, int LuP, int Lu, int nlayers) {
  DpBuffers B;
  B.value = reinterpret_cast<double*>(smem);
  B.f = B.value + (size_t)M * LuP;
  B.ch = reinterpret_cast<unsigned short*>(B.f + (size_t)M * LuP);
  size_t off = (size_t)M * LuP * sizeof(double) * 2 +
               (size_t)(nlayers > 0 ? nlayers : 0) * M * LuP * sizeof(unsigned short);
  off = (off + 15) & ~(size_t)15;
  B.tputS = reinterpret_cast<double*>(smem + off);
  (void)Lu;
  return B;
}

// Mixed-radix sub-multiset lattice of the combo (kernels.py:147-162, 185-193).
// Requires sh.C, sh.cnt set; all threads call.
__device__ inline void dp_setup_lattice(DpShared& sh) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    int M = 1, n = 0;
    for (int c = 0; c < sh.C; ++c) { M *= sh.cnt[c] + 1; n += sh.cnt[c]; }
    sh.M = M;
    sh.n = n;
  }
  __syncthreads();
  const int M = sh.M;
  for (int code = tid; code < M; code += blockDim.x) {
    int rest = code, tot = 0;
    for (int c = 0; c < kMaxC; ++c) {
      int d = 0;
      if (c < sh.C) { d = rest % (sh.cnt[c] + 1); rest /= sh.cnt[c] + 1; }
      sh.digits[code][c] = (unsigned char)d;
      tot += d;
    }
    sh.sizes[code] = (unsigned char)tot;
  }
  __syncthreads();
  for (int rem = tid; rem < M; rem += blockDim.x) {
    unsigned long long mask[2] = {0ull, 0ull};
    for (int u = 0; u <= rem; ++u) {
      bool ok = true;
      for (int c = 0; c < sh.C; ++c) ok &= sh.digits[u][c] <= sh.digits[rem][c];
      if (ok) mask[u >> 6] |= 1ull << (u & 63);
    }
    sh.contain[rem][0] = mask[0];
    sh.contain[rem][1] = mask[1];
  }
  if (tid < kMaxC + 2) {
    unsigned long long mask[2] = {0ull, 0ull};
    for (int u = 0; u < M; ++u)
      if (sh.sizes[u] <= tid) mask[u >> 6] |= 1ull << (u & 63);
    sh.size_le[tid][0] = mask[0];
    sh.size_le[tid][1] = mask[1];
  }
  if (tid == 0) {
    for (int s = 0; s <= kMaxC; ++s) sh.nbysize[s] = 0;
    for (int code = 0; code < M; ++code) {
      const int s = sh.sizes[code];
      sh.bysize[s][sh.nbysize[s]++] = (unsigned char)code;
    }
  }
  __syncthreads();
}

// value[u][j] (kernels.py:164-170): v = 0.0; v += digit * tput[c][j-1] in c order.
// Zero digits add an exact +0.0 to a non-negative sum, so they are skipped.
__device__ inline void dp_build_value(const DpShared& sh, const DpBuffers& B) {
  const int M = sh.M, Lu = sh.Lu, LuP = sh.LuP, C = sh.C;
  for (int idx = threadIdx.x; idx < M * Lu; idx += blockDim.x) {
    const int u = idx / Lu;
    const int j = idx - u * Lu + 1;
    double v = 0.0;
    for (int c = 0; c < C; ++c) {
      const int d = sh.digits[u][c];
      if (d) v = rn_add(v, rn_mul((double)d, B.tputS[c * Lu + (j - 1)]));
    }
    B.value[u * LuP + j] = v;
  }
}

// One (u, l) pair of the reference's per-cell rule: crossing of g(j) = gv[j]
// (non-increasing) and h(j) = hv[l-j] (non-decreasing) for j in [1, jmax].
// kernels.py:210-249, literally (including the branch order and tie choices).
//
// cap (lattice tables with exactly non-increasing rows only): column 0 of every value
// and f row holds its last positive index (J for g = value[u], K for the h source row:
// f[Y][m] = 0 for m > K, and every DP cell is >= 0). So P(j) = g(j) > h(j) is false
// for j > J (g = 0 <= h) and true for j <= J with j < l - K (g > 0 = h). With exactly
// monotone rows P is monotone and its boundary unique, so searching from
// lo = min(J, l - K - 1), hi = J + 1 (clamped to [1, jmax]) returns the reference
// search's (lo, hi) in fewer probes. (Past the two shortcuts P(1) is true and P(jmax)
// false, so J >= 1 and the clamped bracket is never empty.)
//
// floor (callers that keep only strictly better values): with g non-increasing and h
// non-decreasing no j gives more than min(g(1), h(jmax)); a pair whose bound is <= floor
// cannot change the caller's result, so it returns -inf without searching.
template <bool kFloor = false>
__device__ __forceinline__ void dp_pair(const double* __restrict__ gv,
                                        const double* __restrict__ hv, int l, int jmax,
                                        bool mono, double& cand, int& cj, bool cap = false,
                                        double floor = kNegInf) {
  if (mono) {
    const double* __restrict__ hl = hv + l;  // hv[l - j] == hl[-j]: one address op per probe
    // capped rows are 16-byte aligned (lat_pitch): (J, g[1]) in one vector load; J and
    // K are stored as integer bits in the double slots
    double g0 = 0.0, g1, h0 = 0.0;
    if (cap) {
      const double2 g01 = *reinterpret_cast<const double2*>(gv);
      g0 = g01.x;
      g1 = g01.y;
      h0 = hv[0];
    } else {
      g1 = gv[1];
    }
    const double h1 = hl[-1];
    if (g1 <= h1) { cand = g1; cj = 1; return; }
    const double gm = gv[jmax];
    const double hm = hl[-jmax];
    if (gm >= hm) { cand = hm; cj = jmax; return; }
    if (kFloor && (g1 < hm ? g1 : hm) <= floor) { cand = kNegInf; cj = 0; return; }
    int lo = 1, hi = jmax;
    if (cap) {
      const int J = __double2loint(g0), K = __double2loint(h0);
      hi = min(jmax, J + 1);
      lo = max(1, min(min(J, l - K - 1), hi - 1));
    }
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (gv[mid] > hl[-mid]) lo = mid; else hi = mid;
    }
    const double vlo = hl[-lo];
    const double vhi = gv[hi];
    if (vlo >= vhi) { cand = vlo; cj = lo; } else { cand = vhi; cj = hi; }
  } else {
    cand = kNegInf;
    cj = 0;
    for (int j = 1; j <= jmax; ++j) {
      const double v = gv[j];
      const double h = hv[l - j];
      const double mv = v < h ? v : h;
      if (mv > cand) { cand = mv; cj = j; }
    }
  }
}

// Run the DP for stage count S (2 <= S <= min(n, Lu)) on the value table already
// in B.value. Leaves the answer in sh.top_val/top_u/top_j and the choices of
// layers 2..S-1 in B.ch. All threads call.
__device__ inline void dp_run(DpShared& sh, const DpBuffers& B, int S) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int n = sh.n, Lu = sh.Lu, LuP = sh.LuP, M = sh.M;
  const bool mono = sh.mono != 0;
  for (int sg = 2; sg <= S - 1; ++sg) {
    const double* fprev = (sg == 2) ? B.value : B.f;
    unsigned short* chl = B.ch + (size_t)(sg - 2) * M * LuP;
    const int smin = sg, smaxsz = n - (S - sg);
    const int lmax = Lu - (S - sg);
    const int nl = lmax - sg + 1;
    const int nchunks = (nl + 31) >> 5;
    for (int s = smaxsz; s >= smin; --s) {
      const int nrem = sh.nbysize[s];
      const int ntasks = nrem * nchunks;
      const unsigned long long umask0 = sh.size_le[s - (sg - 1)][0] & ~1ull, umask1 = sh.size_le[s - (sg - 1)][1];
      for (int t = warp; t < ntasks; t += nwarps) {
        const int ri = t / nchunks;
        const int rem = sh.bysize[s][ri];
        const int l = sg + (t - ri * nchunks) * 32 + lane;
        const bool act = l <= lmax;
        const int jmax = l - (sg - 1);
        double best = kNegInf;
        int bu = 0, bj = 0;
        for (int w = 0; w < 2; ++w) {  // u ascending over the 128-bit sub-multiset mask
          unsigned long long mask = sh.contain[rem][w] & (w ? umask1 : umask0);
          while (mask) {
            const int u = (w << 6) + __ffsll((long long)mask) - 1;
            mask &= mask - 1;
            if (act) {
              double cand;
              int cj;
              dp_pair(B.value + u * LuP, fprev + (rem - u) * LuP, l, jmax, mono, cand, cj);
              if (cand > best) { best = cand; bu = u; bj = cj; }
            }
          }
        }
        if (act) {
          B.f[rem * LuP + l] = best;
          chl[rem * LuP + l] = (unsigned short)((bu << 8) | bj);
        }
      }
      __syncthreads();
    }
  }
  // top cell (S, Lu, full): lanes split u, reduce with (value desc, u asc)
  if (warp == 0) {
    const double* fprev = (S == 2) ? B.value : B.f;
    const int full = M - 1;
    const int l = Lu;
    const int jmax = l - (S - 1);
    const int umax_size = n - (S - 1);
    double best = kNegInf;
    int bu = 1 << 20, bj = 0;
    for (int u = lane + 1; u < M; u += 32) {
      if (sh.sizes[u] > umax_size) continue;
      double cand;
      int cj;
      dp_pair(B.value + u * LuP, fprev + (full - u) * LuP, l, jmax, mono, cand, cj);
      if (cand > best) { best = cand; bu = u; bj = cj; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, off);
      const int ou = __shfl_down_sync(0xffffffffu, bu, off);
      const int oj = __shfl_down_sync(0xffffffffu, bj, off);
      if (ob > best || (ob == best && ou < bu)) { best = ob; bu = ou; bj = oj; }
    }
    if (lane == 0) { sh.top_val = best; sh.top_u = bu; sh.top_j = bj; }
  }
  __syncthreads();
}

// Walk the choices from (S, Lu, full) (kernels.py:258-275). Thread 0 only.
__device__ inline void dp_decode(DpShared& sh, const DpBuffers& B, int S) {
  const int LuP = sh.LuP, M = sh.M;
  int l = sh.Lu, rem = M - 1;
  for (int s = 0; s < S; ++s) {
    const int sg = S - s;
    int u, j;
    if (sg == 1) {
      u = rem; j = l;
    } else if (sg == S) {
      u = sh.top_u; j = sh.top_j;
    } else {
      const unsigned short c = B.ch[(size_t)(sg - 2) * M * LuP + rem * LuP + l];
      u = c >> 8; j = c & 255;
    }
    sh.stage_j[s] = j;
    sh.stage_u[s] = u;
    l -= j;
    rem -= u;
  }
}

}  // namespace coral
