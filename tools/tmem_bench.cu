// TMEM bandwidth from the SIMT side: tcgen05.ld / tcgen05.st of 32x32b.x32 blocks
// (32 columns per thread), alone and interleaved with LDS.128 traffic -- decides
// whether per-thread accumulators can live in TMEM next to a shared-memory-bound
// FFT ladder.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

#define LD32(r, addr)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                  \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),         \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),     \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),  \
                 "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),  \
                 "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                       \
               : "r"(addr))
#define ST32(r, addr)                                                                                      \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
               "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),       \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),        \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),  \
               "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),            \
               "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),            \
               "r"(r[30]), "r"(r[31]))

// MODE bit 0: tcgen05.ld, bit 1: tcgen05.st, bit 2: LDS.128 traffic
template <int MODE, int COLS>
__global__ void __launch_bounds__(128) tmem_kernel(unsigned *out) {
  __shared__ uint32_t slot;
  __shared__ uint4 buf[2048];
  const int t = threadIdx.x, w = t / 32;
  for (int i = t; i < 2048; i += 128) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                 "r"((uint32_t)COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)(32 * (w & 3)) << 16);
  uint32_t r[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) r[k] = t * 32 + k;
  uint32_t acc = 0;
  int idx = t;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t col = (uint32_t)((it * 32) % COLS);
    if (MODE & 1) {
      LD32(r, base + col);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 32; ++k) r[k] += 1;
    }
    if (MODE & 2) {
      ST32(r, base + col);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (MODE & 4) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {   // 8 x 512 B per warp = 4 KB, as the 32-column TMEM block
        const uint4 v = buf[idx];
        acc += v.x ^ v.w;
        idx = (idx + 128) & 2047;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) acc += r[k];
  out[blockIdx.x * 128 + t] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"((uint32_t)COLS));
}

template <typename K>
static float time_it(K k, int grid, unsigned *out) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  k<<<grid, 128>>>(out);
  cudaEventRecord(s);
  for (int r = 0; r < 5; ++r) k<<<grid, 128>>>(out);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
  return ms / 5;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned *out;
  cudaMalloc(&out, sizeof(unsigned) * sms * 4 * 128);
  const double cyc_per_ms = clk * 1.0;   // kHz -> cycles per ms
  for (int ctas = 1; ctas <= 4; ctas *= 2) {   // CTAs per SM (256 columns each at 2, 128 at 4)
    const int grid = sms * ctas;
    float tl, ts, tls, tx, tlx;
    if (ctas == 1) {
      tl = time_it(tmem_kernel<1, 512>, grid, out);
      ts = time_it(tmem_kernel<2, 512>, grid, out);
      tls = time_it(tmem_kernel<3, 512>, grid, out);
      tx = time_it(tmem_kernel<4, 512>, grid, out);
      tlx = time_it(tmem_kernel<7, 512>, grid, out);
    } else if (ctas == 2) {
      tl = time_it(tmem_kernel<1, 256>, grid, out);
      ts = time_it(tmem_kernel<2, 256>, grid, out);
      tls = time_it(tmem_kernel<3, 256>, grid, out);
      tx = time_it(tmem_kernel<4, 256>, grid, out);
      tlx = time_it(tmem_kernel<7, 256>, grid, out);
    } else {
      tl = time_it(tmem_kernel<1, 128>, grid, out);
      ts = time_it(tmem_kernel<2, 128>, grid, out);
      tls = time_it(tmem_kernel<3, 128>, grid, out);
      tx = time_it(tmem_kernel<4, 128>, grid, out);
      tlx = time_it(tmem_kernel<7, 128>, grid, out);
    }
    // bytes per SM per run: ctas x 128 threads x 128 B per ITER
    const double bytes = (double)ctas * 128 * 128 * ITERS;
    printf("CTAs/SM %d: ld %.3f ms (%.1f B/clk/SM)  st %.3f ms (%.1f)  ld+st %.3f ms  LDS-only %.3f ms (%.1f B/clk)  "
           "ld+st+LDS %.3f ms\n",
           ctas, tl, bytes / (tl * cyc_per_ms), ts, bytes / (ts * cyc_per_ms), tls, tx, bytes / (tx * cyc_per_ms), tlx);
  }
  return 0;
}
