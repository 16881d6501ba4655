// Integer pipe throughput microbenchmarks on B200 (sm_100a): warp instructions
// per cycle per SM for IMAD, IMAD.HI, IMAD.WIDE, IADD3, LOP3 and mixes.  Used to
// choose the instruction mix of the NTT butterflies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pmb tools/pipe_microbench.cu && /tmp/pmb
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent chains per thread
constexpr int ITERS = 4096;

template <int OP>
__global__ void bench(uint32_t *sink, uint32_t a, uint32_t b) {
  uint32_t x[CH], y[CH];
  double xd[CH], yd[CH];
  const double ad = 1.0000001 + a * 1e-12, wp = (double)a / 357900289.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) { x[k] = threadIdx.x + k; y[k] = blockIdx.x * 7 + k; xd[k] = x[k]; yd[k] = y[k]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (OP == 0) x[k] = x[k] * a + y[k];                      // IMAD
      if (OP == 1) x[k] = __umulhi(x[k], a) ^ y[k];             // IMAD.HI (+LOP3)
      if (OP == 2) { uint64_t t = (uint64_t)x[k] * a; x[k] = (uint32_t)t + (uint32_t)(t >> 32); }  // IMAD.WIDE
      if (OP == 3) x[k] = x[k] + y[k] + a;                      // IADD3
      if (OP == 4) { uint32_t q = __umulhi(x[k], a); x[k] = x[k] * b - q * 7u; }   // Shoup-like
      if (OP == 5) x[k] = (x[k] ^ y[k]) & a;                    // LOP3
      if (OP == 6) { x[k] = x[k] * a + y[k]; y[k] = y[k] + x[k] + b; }  // IMAD + IADD3 mix
      if (OP == 7) xd[k] = fma(xd[k], ad, yd[k]);                // DFMA
      if (OP == 8) { x[k] = x[k] * a + y[k]; xd[k] = fma(xd[k], ad, yd[k]); }   // IMAD || DFMA
      if (OP == 9) {   // hybrid modmul: quotient on the FP64 pipe, remainder with 2 IMADs
        const double qd = fma(xd[k], wp, 6755399441055744.0);   // 1.5 * 2^52: round to integer
        const uint32_t q = (uint32_t)__double2loint(qd);
        uint32_t r = x[k] * a - q * 357900289u;
        r = min(r, r + 357900289u);
        x[k] = r;
        xd[k] = __hiloint2double(0x43300000, r) - 4503599627370496.0;
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s ^= x[k] ^ y[k] ^ (uint32_t)__double2loint(xd[k]);
  if (s == 0x9e3779b9u) sink[0] = s;
}

template <int OP>
void run(const char *name, int ops_per_inner, int sms) {
  uint32_t *sink;
  cudaMalloc(&sink, 4);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<OP><<<blocks, threads>>>(sink, 0x9e3779b9u, 12345u);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    bench<OP><<<blocks, threads>>>(sink, 0x9e3779b9u, 12345u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_ops = (double)blocks * (threads / 32) * ITERS * CH * ops_per_inner;
  const double per_s = warp_ops / (best * 1e-3);
  printf("%-28s %8.2f T warp-op/s   %6.3f warp-op/clk/SM at %d MHz (%.3f ms)\n", name, per_s / 1e12,
         per_s / sms / (clk_khz * 1e3), clk_khz / 1000, best);
  cudaFree(sink);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("IMAD (dependent per chain)", 1, sms);
  run<1>("IMAD.HI + LOP3", 2, sms);
  run<2>("IMAD.WIDE + IADD", 2, sms);
  run<3>("IADD3", 1, sms);
  run<4>("Shoup (HI + 2 IMAD)", 3, sms);
  run<5>("LOP3", 1, sms);
  run<6>("IMAD + IADD3", 2, sms);
  run<7>("DFMA", 1, sms);
  run<8>("IMAD || DFMA (independent)", 2, sms);
  run<9>("hybrid modmul (DFMA q, 2 IMAD)", 1, sms);
  return 0;
}
