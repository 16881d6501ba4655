// Does a shared-memory (or L1) 128-bit load whose lanes share addresses cost fewer
// crossbar cycles?  Throughput of LDS.128 / LDS.64 / LDG.128 (L1 hit) per warp
// instruction for lane -> address patterns: all distinct, pairs (L, L ^ 16), pairs
// (2m, 2m + 1), quads, all equal.  Decides whether two ciphertexts sharing a key
// value in one warp instruction halve the key-read traffic of the FFT ladder.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_bcast_bench tools/lds_bcast_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 8192;

__device__ __forceinline__ int lane_slot(int pat, int L) {
  switch (pat) {
    case 0: return L;             // distinct
    case 1: return L & 15;        // pairs (L, L ^ 16)
    case 2: return L >> 1;        // pairs (2m, 2m + 1)
    case 3: return L >> 2;        // quads
    default: return 0;            // all equal
  }
}

template <int KIND>   // 0 = LDS.128, 1 = LDS.64, 2 = LDG.128 (L1-resident)
__global__ void __launch_bounds__(256) ld_kernel(unsigned *out, const uint4 *g, int pat) {
  __shared__ uint4 buf[2048];
  const int t = threadIdx.x, L = t & 31;
  for (int i = t; i < 2048; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  unsigned a = t, b = t * 7, c = t * 11, d = t * 13;
  const int lo = lane_slot(pat, L);
  int row = (t >> 5) & 7;
#pragma unroll 8
  for (int it = 0; it < ITERS; ++it) {
    const int idx = (row << 5) | lo;
    if (KIND == 0) {
      const uint4 v = buf[idx];
      a ^= v.x; b += v.y; c ^= v.z; d += v.w;
    } else if (KIND == 1) {
      const uint2 v = reinterpret_cast<const uint2 *>(buf)[idx];
      a ^= v.x; b += v.y;
    } else {
      const uint4 v = __ldg(&g[idx]);
      a ^= v.x; b += v.y; c ^= v.z; d += v.w;
    }
    row = (row + 1 + (a & 0)) & 63;
  }
  out[blockIdx.x * blockDim.x + t] = a ^ b ^ c ^ d;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned *out;
  uint4 *g;
  cudaMalloc(&out, (size_t)sms * 8 * 256 * 4);
  cudaMalloc(&g, 2048 * 16);
  cudaMemset(g, 1, 2048 * 16);
  const char *kinds[3] = {"LDS.128", "LDS.64 ", "LDG.128"};
  const char *pats[5] = {"distinct", "pairs L^16", "pairs 2m,2m+1", "quads", "all equal"};
  for (int kind = 0; kind < 3; ++kind)
    for (int pat = 0; pat < 5; ++pat) {
      cudaEvent_t s, e;
      cudaEventCreate(&s);
      cudaEventCreate(&e);
      auto launch = [&] {
        if (kind == 0) ld_kernel<0><<<sms * 8, 256>>>(out, g, pat);
        if (kind == 1) ld_kernel<1><<<sms * 8, 256>>>(out, g, pat);
        if (kind == 2) ld_kernel<2><<<sms * 8, 256>>>(out, g, pat);
      };
      launch();
      cudaEventRecord(s);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      ms /= 5;
      const double warp_instr_per_sm = 8.0 * 8 * ITERS;   // 8 CTAs x 8 warps x ITERS
      const double cyc = ms * 1e-3 * clk * 1e3;
      printf("%s %-14s %.3f ms  %.2f cycles per warp instruction per SM\n", kinds[kind], pats[pat], ms,
             cyc / warp_instr_per_sm);
    }
  return 0;
}
