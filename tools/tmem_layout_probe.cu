// Probe the thread <-> (lane, column) mapping of the tcgen05.ld shapes 16x64b,
// 16x128b, 16x256b and 16x32bx2 on the hardware: every lane holds (lane << 8) | column
// in columns 0..63 (written with 32x32b), then each shape loads from lane base 0 and
// 16 and each thread prints what it received.  Decides whether TMEM can serve as a
// warp-local transpose medium for the FFT.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(uint32_t *out) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t / 32, L = t % 32;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(64u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)(32 * (w & 3)) << 16);
  for (int c = 0; c < 64; c += 4) {
    const uint32_t v0 = (L << 8) | c, v1 = (L << 8) | (c + 1), v2 = (L << 8) | (c + 2), v3 = (L << 8) | (c + 3);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(base + c), "r"(v0), "r"(v1),
                 "r"(v2), "r"(v3)
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t *o = out + t * 64;
  for (int half = 0; half < 2; ++half) {
    const uint32_t a = base + ((uint32_t)(16 * half) << 16);
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    o[half * 32 + 0] = r[0];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    o[half * 32 + 1] = r[0];
    o[half * 32 + 2] = r[1];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 4; ++k) o[half * 32 + 3 + k] = r[k];
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x1.b32 {%0}, [%1], 8;" : "=r"(r[0]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    o[half * 32 + 7] = r[0];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 8; ++k) o[half * 32 + 8 + k] = r[k];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 4; ++k) o[half * 32 + 16 + k] = r[k];
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    o[half * 32 + 20] = r[0];
    o[half * 32 + 21] = r[1];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(64u));
  }
}

static void pr(const char *name, const uint32_t *h, int half, int off, int n) {
  printf("%s (lane base %d): thread: (lane,col)...\n", name, 16 * half);
  for (int t = 0; t < 32; ++t) {
    printf("  t%2d:", t);
    for (int k = 0; k < n; ++k) {
      const uint32_t v = h[t * 64 + half * 32 + off + k];
      printf(" (%u,%u)", v >> 8, v & 255);
    }
    printf("\n");
  }
}

int main() {
  uint32_t *d, h[128 * 64];
  cudaMalloc(&d, sizeof(h));
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  for (int half = 0; half < 2; ++half) {
    pr("16x64b.x1", h, half, 0, 1);
    pr("16x128b.x1", h, half, 1, 2);
    pr("16x256b.x1", h, half, 3, 4);
    pr("16x32bx2.x1 (imm 8)", h, half, 7, 1);
    pr("16x256b.x2", h, half, 8, 8);
    pr("16x128b.x2", h, half, 16, 4);
    pr("16x64b.x2", h, half, 20, 2);
  }
  return 0;
}
