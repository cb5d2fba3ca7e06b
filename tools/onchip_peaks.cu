// On-chip peaks of one B200 for the evaluator's roofline (the lattice
// search kernels read L2/L1-resident fp64 tables, so HBM is not their bound and
// MEASURED_PEAKS.json has no on-chip figure). Measured the way the HBM peak is: CUDA
// events around a kernel, best of several runs, after warm-up.
//   l2_read_gbs       : 32 MB buffer (L2-resident), 16-byte ld.global.cg reads, all SMs
//   l1_gather_lanes_s : per-lane 8-byte loads to distinct 128-B lines of a per-block
//                       L1-resident 32 KB slab (the lat_top_kernel probe pattern: one
//                       L1 wavefront per lane) -> lane-loads per second, whole GPU
//   l1_coalesced_gbs  : the same slab read with consecutive lanes (1 wavefront per
//                       warp-wide 8-byte load)
//   smem_gbs          : conflict-free 8-byte shared-memory reads
//   fp64_minmax_ops_s : fp64 fmax/fmin (DSETP.MAX/MIN + selects on sm_100a; the DP max-min)
// Build + run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/onchip_peaks.cu
//              -o /tmp/onchip && /tmp/onchip  (prints one JSON object)
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void l2_read(const double2* __restrict__ a, size_t n, int passes, double* out) {
  double s = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 12345.678) *out = s;
}

// slab: per block 4096 doubles (32 KB). gather: lane l of iteration i reads line
// ((l * 7 + i * 13) & 255), word (i & 15): 32 distinct lines per warp load.
template <bool kGather>
__global__ void l1_read(const double* __restrict__ a, int iters, double* out) {
  const double* slab = a + (size_t)blockIdx.x * 4096;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; i += 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ii = i + k + w;
      const int idx = kGather ? (((lane * 7 + ii * 13) & 255) << 4) | (ii & 15)
                              : ((ii * 32 + lane) & 4095);
      const double v = slab[idx];
      if (k == 0) s0 += v; else if (k == 1) s1 += v; else if (k == 2) s2 += v; else s3 += v;
    }
  }
  const double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) *out = s;
}

__global__ void smem_read(int iters, double* out) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 0.5;
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; i += 4) {
    s0 += sm[((i + 0) * 32 + threadIdx.x) & 4095];
    s1 += sm[((i + 1) * 32 + threadIdx.x) & 4095];
    s2 += sm[((i + 2) * 32 + threadIdx.x) & 4095];
    s3 += sm[((i + 3) * 32 + threadIdx.x) & 4095];
  }
  const double s = s0 + s1 + s2 + s3;
  if (s == 12345.678) *out = s;
}

// the DP's inner step, best = max(best, min(a, b)), rotated over 3 registers per group
// (4 independent groups) so the compiler cannot fold repeated clamps
__global__ void dmnmx(int iters, double seed, double* out) {
  double a[4], b[4], c[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { a[k] = seed + threadIdx.x + k; b[k] = seed * (k + 2); c[k] = seed - k; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 6 ops per group
      a[k] = fmax(a[k], fmin(b[k], c[k]));
      b[k] = fmax(b[k], fmin(c[k], a[k]));
      c[k] = fmin(c[k], fmax(a[k], b[k]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += a[k] + b[k] + c[k];
  if (s == 12345.678) *out = s;
}

template <typename F>
static float best_ms(F launch, int reps = 7) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 8));
  // L2: 32 MB resident buffer, 64 passes
  const size_t n2 = (32u << 20) / 16;
  double2* a2;
  CK(cudaMalloc(&a2, n2 * 16));
  CK(cudaMemset(a2, 0, n2 * 16));
  const int passes = 64;
  float ms = best_ms([&] { l2_read<<<sms * 4, 512>>>(a2, n2, passes, out); });
  const double l2_gbs = (double)n2 * 16 * passes / (ms * 1e-3) / 1e9;
  // L1: one 32 KB slab per block, 4 blocks of 256 threads per SM
  const int blocks = sms * 4, iters = 4096;
  double* a1;
  CK(cudaMalloc(&a1, (size_t)blocks * 4096 * 8));
  CK(cudaMemset(a1, 0, (size_t)blocks * 4096 * 8));
  ms = best_ms([&] { l1_read<true><<<blocks, 256>>>(a1, iters, out); });
  const double gather = (double)blocks * 256 * iters / (ms * 1e-3);
  ms = best_ms([&] { l1_read<false><<<blocks, 256>>>(a1, iters, out); });
  const double coal = (double)blocks * 256 * iters * 8 / (ms * 1e-3) / 1e9;
  ms = best_ms([&] { smem_read<<<blocks, 256>>>(iters, out); });
  const double smem = (double)blocks * 256 * iters * 8 / (ms * 1e-3) / 1e9;
  const int it3 = 8192;
  ms = best_ms([&] { dmnmx<<<sms * 8, 256>>>(it3, 1.5, out); });
  const double dm = (double)sms * 8 * 256 * it3 * 24 / (ms * 1e-3);
  CK(cudaGetLastError());
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_nominal\": %d, "
         "\"l2_read_gbs\": %.1f, \"l1_gather_lanes_s\": %.4g, \"l1_gather_lanes_per_sm_clk\": %.3f, "
         "\"l1_coalesced_gbs\": %.1f, \"smem_gbs\": %.1f, \"fp64_minmax_ops_s\": %.4g}\n",
         p.name, sms, clk / 1000, l2_gbs, gather, gather / sms / (clk * 1e3), coal, smem, dm);
  return 0;
}
