// hwb_tc.cuh — LWE key switch on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// The key switch (hw/tfhe.py:377-401, SURVEY §8(a) last row) is the contraction
//     out[b][c] = (c < n ? 0 : in[b][N]) - sum_k D[b][k] * KSK[k][c]   (mod 2^32)
// with k = j*l_ks + t (input coefficient j, gadget level t), D the signed gadget digits
// (|d| <= beta/2 <= 128 for base_log <= 8, i.e. exact int8) and KSK 32-bit words.
// Splitting each key word into four bytes KSK = sum_q K_q 2^(8q) turns it into one
// int8 x uint8 GEMM with N_mma = 4 limbs x 64 output columns:
//     S_q[b][c] = sum_k D[b][k] K_q[k][c]            (exact in int32: K*128*255 < 2^31)
//     sum_k D K  = S_0 + S_1 2^8 + S_2 2^16 + S_3 2^24 (mod 2^32)
// so the result is bit-exact by construction.
//
// Operands are pre-tiled in HBM in the tensor core's canonical K-major, no-swizzle layout
// (8-row x 16-byte core matrices), so one 1-D TMA bulk copy moves a whole tile:
//   digit tile  (mt, kb): 128 items x 128 K-bytes = 16 KiB, [c 8][g 16][r 8][16 B]
//   key tile    (ct, kb): 256 rows (limb*64 + col) x 128 K-bytes = 32 KiB, [c 8][g 32][r 8][16 B]
// One CTA = 128 items x 64 output columns; 4-stage TMA -> tcgen05.mma pipeline on
// mbarriers, one elected thread issues the MMAs (M=128, N=256, K=32 per instruction),
// the int32 accumulators live in TMEM (256 columns) and the 4 warps' epilogue reads
// them back with tcgen05.ld, recombines the limbs mod 2^32 and writes the LWE rows.
#pragma once

#include <cstdint>

namespace hwb {

constexpr int TC_M = 128;          // items per CTA (TMEM lanes)
constexpr int TC_COLS = 64;        // output columns per CTA
constexpr int TC_N = 4 * TC_COLS;  // MMA N: 4 byte limbs x 64 columns
constexpr int TC_KB = 128;         // K bytes per pipeline stage (4 MMAs of K = 32)
constexpr int TC_STAGES = 4;
constexpr int TC_A_BYTES = TC_M * TC_KB;   // 16 KiB
constexpr int TC_B_BYTES = TC_N * TC_KB;   // 32 KiB
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + 1024;

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a lost arrival traps (error surfaced to the host) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) __trap();   // 2 s
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// smem matrix descriptor, K-major, no swizzle: LBO = stride between 16-byte K chunks,
// SBO = stride between 8-row groups (both in bytes), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor: D s32, A s8 (signed), B u8 (unsigned), both K-major, M=128, N=256
constexpr uint32_t kTcIdesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(kTcIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

// ---- operand tiling ----------------------------------------------------------------------
// byte offset of (row, kbyte) inside a K-major no-swizzle tile with `groups` 8-row groups
__host__ __device__ __forceinline__ uint32_t tc_tile_off(uint32_t row, uint32_t kbyte, uint32_t groups) {
  return ((((kbyte >> 4) * groups + (row >> 3)) * 8u + (row & 7u)) << 4) | (kbyte & 15u);
}

// KSK [K][ncol] u32 -> key tiles [ct][kb] (32 KiB each).  One thread per 16-byte row chunk.
__global__ void ksk_to_tc_kernel(const uint32_t *__restrict__ ksk, uint4 *out, int K, int ncol, int nct) {
  const int nkb = K / TC_KB;
  const int64_t total = (int64_t)nct * nkb * (TC_B_BYTES / 16);
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int R = (int)(idx % (TC_B_BYTES / 16));    // (c*32 + g)*8 + r
  const int64_t tile = idx / (TC_B_BYTES / 16);
  const int kb = (int)(tile % nkb), ct = (int)(tile / nkb);
  const int c = R >> 8, n = R & 255;               // n = g*8 + r
  const int limb = n >> 6, col = ct * TC_COLS + (n & 63);
  const int k0 = kb * TC_KB + c * 16;
  uint32_t w[4] = {0, 0, 0, 0};
  if (col < ncol) {
    for (int b = 0; b < 16; ++b) {
      const uint32_t byte = (ksk[(size_t)(k0 + b) * ncol + col] >> (8 * limb)) & 0xFFu;
      w[b >> 2] |= byte << (8 * (b & 3));
    }
  }
  out[idx] = make_uint4(w[0], w[1], w[2], w[3]);
}

// Gadget digits of the input LWE masks -> digit tiles [mt][kb] (16 KiB each), int8.
// One thread per (item, 16-byte K chunk); rows past B are zero.
__global__ void ks_digits_kernel(const uint32_t *__restrict__ in, uint4 *dig, int64_t B, int N, int K,
                                 Gadget gk) {
  const int nch = K / 16, nkb = K / TC_KB;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int m_in = (int)(idx % TC_M);
  const int64_t rest = idx / TC_M;
  const int cg = (int)(rest % nch);
  const int64_t mt = rest / nch;
  const int64_t m = mt * TC_M + m_in;
  const int64_t ntiles_m = (B + TC_M - 1) / TC_M;
  if (mt >= ntiles_m) return;
  const int kb = cg / (TC_KB / 16), c = cg % (TC_KB / 16);
  uint32_t w[4] = {0, 0, 0, 0};
  if (m < B) {
    const int L = (int)gk.levels;
    const int k0 = cg * 16;
    int j = k0 / L, t = k0 - j * L;
    const uint32_t *row = in + m * (int64_t)(N + 1);
    uint32_t v = decomp_prep(row[j], gk);
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const uint32_t sh = gk.base_log * (uint32_t)(L - 1 - t);
      const uint32_t d = (((v >> sh) & gk.mask) - gk.half) & 0xFFu;
      w[b >> 2] |= d << (8 * (b & 3));
      if (++t == L && b < 15) {
        t = 0;
        v = decomp_prep(row[++j], gk);
      }
    }
  }
  const size_t tile = (size_t)mt * nkb + kb;
  dig[tile * (TC_A_BYTES / 16) + (tc_tile_off((uint32_t)m_in, (uint32_t)c * 16, TC_M / 8) >> 4)] =
      make_uint4(w[0], w[1], w[2], w[3]);
}

// grid (ceil(B/128), nct); 128 threads; TC_SMEM dynamic shared memory.
__global__ void __launch_bounds__(128, 1)
    keyswitch_tc_kernel(const uint8_t *__restrict__ dig, const uint8_t *__restrict__ key,
                        const uint32_t *__restrict__ in, uint32_t *out, int64_t B, int N, int n, int K) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t *base = (uint8_t *)(((uintptr_t)tc_smem + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[TC_STAGES], empty[TC_STAGES], done;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, ct = blockIdx.y;
  const int nkb = K / TC_KB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"((uint32_t)TC_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {
    // producer: TMA bulk copies of the pre-tiled operands
    const uint8_t *ga = dig + (size_t)mt * nkb * TC_A_BYTES;
    const uint8_t *gb = key + (size_t)ct * nkb * TC_B_BYTES;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % TC_STAGES;
      if (kb >= TC_STAGES) mbar_wait(&empty[s], ((kb / TC_STAGES) - 1) & 1);
      uint8_t *sa = base + (size_t)s * TC_STAGE_BYTES;
      mbar_expect_tx(&full[s], TC_STAGE_BYTES);
      bulk_g2s(sa, ga + (size_t)kb * TC_A_BYTES, TC_A_BYTES, &full[s]);
      bulk_g2s(sa + TC_A_BYTES, gb + (size_t)kb * TC_B_BYTES, TC_B_BYTES, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % TC_STAGES;
      mbar_wait(&full[s], (kb / TC_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sa = smem_u32(base + (size_t)s * TC_STAGE_BYTES);
      const uint32_t sb = sa + TC_A_BYTES;
#pragma unroll
      for (int k = 0; k < TC_KB / 32; ++k) {
        const uint64_t da = umma_desc(sa + k * 2 * (TC_M / 8) * 128, (TC_M / 8) * 128, 128);
        const uint64_t db = umma_desc(sb + k * 2 * (TC_N / 8) * 128, (TC_N / 8) * 128, 128);
        umma_i8(tmem, da, db, (kb | k) != 0);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(&done);
  }
  __syncwarp();

  // epilogue: warp w owns TMEM lanes 32w..32w+31 = items mt*128 + 32w + lane
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int64_t m = (int64_t)mt * TC_M + warp * 32 + lane;
  const uint32_t bval = m < B ? in[m * (int64_t)(N + 1) + N] : 0u;
  const int ncol = n + 1;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
  for (int cc = 0; cc < TC_COLS; cc += 16) {
    uint32_t s0[16], s1[16], s2[16], s3[16];
    tmem_ld16(lane_addr + 0 * TC_COLS + cc, s0);
    tmem_ld16(lane_addr + 1 * TC_COLS + cc, s1);
    tmem_ld16(lane_addr + 2 * TC_COLS + cc, s2);
    tmem_ld16(lane_addr + 3 * TC_COLS + cc, s3);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (m < B) {
      uint32_t *o = out + m * (int64_t)ncol;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = ct * TC_COLS + cc + i;
        const uint32_t acc = s0[i] + (s1[i] << 8) + (s2[i] << 16) + (s3[i] << 24);
        if (col < ncol) o[col] = (col == n ? bval : 0u) - acc;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TC_N));
  }
}

// Throughput probe of the shipped MMA shape (kind::i8, M128 N256 K32, operands in
// shared memory, accumulator in TMEM): one CTA per SM, `iters` x 4 back-to-back MMAs
// into one accumulator, the same issue pattern as keyswitch_tc_kernel's K loop.
// Its rate is P_i8 (int8 MACs/s), the tensor-core roofline denominator.
__global__ void __launch_bounds__(128, 1) probe_i8mma_kernel(uint32_t *sink, int iters) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t *base = (uint8_t *)(((uintptr_t)tc_smem + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < TC_STAGE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(base)[i] = make_uint4(i, i * 3u, i * 5u, i * 7u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"((uint32_t)TC_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(base), sb = sa + TC_A_BYTES;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < TC_KB / 32; ++k) {
        const uint64_t da = umma_desc(sa + k * 2 * (TC_M / 8) * 128, (TC_M / 8) * 128, 128);
        const uint64_t db = umma_desc(sb + k * 2 * (TC_N / 8) * 128, (TC_N / 8) * 128, 128);
        umma_i8(tmem, da, db, (it | k) != 0);
      }
    }
    umma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  if (s == 0x12345678u) sink[0] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TC_N));
  }
}

}  // namespace hwb
