// Shared-memory vs warp-shuffle throughput, and whether they share a datapath:
// LDS.128 alone, SHFL alone, both interleaved in the same warps; plus dependent
// DFMA / DADD latency.  Decides whether shuffle-based transposes can take load off
// the shared-memory crossbar in the FFT ladder.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mio_bench tools/mio_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>   // 0 = LDS.128, 1 = SHFL.32 x4, 2 = both
__global__ void mio_kernel(unsigned *out) {
  __shared__ uint4 buf[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  unsigned a = t, b = t * 7, c = t * 11, d = t * 13;
  int idx = t & 1023;
#pragma unroll 8
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0 || MODE == 2) {
      const uint4 v = buf[idx];
      a ^= v.x; b += v.y; c ^= v.z; d += v.w;
      idx = (idx + 32) & 1023;
    }
    if (MODE == 1 || MODE == 2) {
      a = __shfl_xor_sync(0xffffffffu, a, 1) + 1;
      b = __shfl_xor_sync(0xffffffffu, b, 2) ^ 3;
      c = __shfl_xor_sync(0xffffffffu, c, 4) + 5;
      d = __shfl_xor_sync(0xffffffffu, d, 8) ^ 7;
    }
  }
  out[blockIdx.x * blockDim.x + t] = a ^ b ^ c ^ d;
}

template <int OP>   // 0 = DFMA chain, 1 = DADD chain
__global__ void lat_kernel(double *out, long long *cyc, double x0) {
  double x = x0 + threadIdx.x;
  const long long s = clock64();
#pragma unroll 16
  for (int it = 0; it < ITERS; ++it) x = OP == 0 ? fma(x, 0.999999, 1e-9) : x + 1e-9;
  const long long e = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = e - s;
}

template <typename K>
static float time_it(K k, int grid, int block, unsigned *out) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  k<<<grid, block>>>(out);
  cudaEventRecord(s);
  for (int r = 0; r < 5; ++r) k<<<grid, block>>>(out);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  return ms / 5;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned *out;
  cudaMalloc(&out, sizeof(unsigned) * sms * 8 * 512);
  for (int warps = 8; warps <= 32; warps *= 2) {
    const int grid = sms * (warps / 8), block = 256;
    const float t0 = time_it(mio_kernel<0>, grid, block, out);
    const float t1 = time_it(mio_kernel<1>, grid, block, out);
    const float t2 = time_it(mio_kernel<2>, grid, block, out);
    const double cyc = clk * 1e3 * 1e-3;   // cycles per ms at the rated clock
    const double warp_iters = (double)warps * ITERS;
    printf("warps/SM %2d: LDS.128 %.3f ms (%.2f cyc per warp-LDS.128/SM), SHFLx4 %.3f ms (%.2f cyc per warp-SHFL/SM), "
           "both %.3f ms (sum %.3f, max %.3f)\n",
           warps, t0, t0 * cyc / warp_iters, t1, t1 * cyc / (warp_iters * 4), t2, t0 + t1, t0 > t1 ? t0 : t1);
  }
  double *dout;
  long long *dc, hc;
  cudaMalloc(&dout, 1024 * sizeof(double));
  cudaMalloc(&dc, sizeof(long long));
  lat_kernel<0><<<1, 32>>>(dout, dc, 1.0);
  lat_kernel<0><<<1, 32>>>(dout, dc, 1.0);
  cudaMemcpy(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency %.2f cyc\n", (double)hc / ITERS);
  lat_kernel<1><<<1, 32>>>(dout, dc, 1.0);
  cudaMemcpy(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("DADD dependent latency %.2f cyc\n", (double)hc / ITERS);
  return 0;
}
