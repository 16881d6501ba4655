// Device building blocks for exact negacyclic arithmetic mod 2^32 on sm_100a.
//
// Exactness strategy: the external product's true integer
// coefficients satisfy |sum_r d_r (*) g_r| <= 2l * N * beta/2 * 2^31 < 2^54 for
// every BASELINE config, so they are recovered exactly from their residues
// modulo two 28.4-bit NTT primes (P = p0*p1 ~ 2^56.8) by CRT and a centred lift,
// then reduced mod 2^32.  One warp owns one (polynomial, prime) pair and keeps
// the 1024 (2048) coefficients in registers, 32 (64) per lane; butterflies with
// span >= 32 are lane-local in layout A (i = lane + 32 j), the rest are
// lane-local in layout B (i = C*lane + j) after one swizzled shared-memory
// transpose per transform.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace hwb {

constexpr uint32_t kP0 = 357900289u;   // 0x15552001 = 43690*2^13 + 1
constexpr uint32_t kP1 = 357818369u;   // 0x1553e001 = 43680*2^13 + 1

// per-prime constants (index = prime)
struct PrimeConst {
  uint32_t p, two_p, pinv;   // pinv = p^-1 mod 2^32 (signed Montgomery REDC)
};

// Twiddle tables.  Uniform-stage twiddles (span >= 32) live in constant memory,
// indexed [n_variant][dir][prime][k] as (W, floor(W*2^32/p)) pairs; k < 64.
// Per-lane twiddles (span < 32) live in global memory (L1-resident, 31 or 62
// slots x 32 lanes per prime/dir), see hwb_kernels.cu for the slot order.
struct DeviceTables {
  const uint2 *lane_fwd[2][2];   // [n_variant][prime] -> [slot][32]
  const uint2 *lane_inv[2][2];
};

// Single translation unit (hwb_kernels.cu) includes this header.
__constant__ uint2 c_tw[2][2][2][64];
__constant__ PrimeConst c_prime[2];
__constant__ uint32_t c_crt[4];   // {inv = p0^-1 mod p1, inv_shoup, P mod 2^32, p1/2}
__constant__ uint32_t c_r2ninv[2][2];   // [n_variant][prime]: R^2 N^-1 mod p

template <int C> struct Log2 { static constexpr int v = (C <= 1) ? 0 : 1 + Log2<C / 2>::v; };

template <int N> struct NVar { static constexpr int v = (N == 1024) ? 0 : 1; };

__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

// a*W mod p in [0, 2p) for any 32-bit a (Shoup, W' = floor(W 2^32 / p)).
__device__ __forceinline__ uint32_t shoup_mul(uint32_t a, uint32_t w, uint32_t wq, uint32_t p) {
  uint32_t q = __umulhi(a, wq);
  return a * w - q * p;
}

// Signed Montgomery product a*b*2^-32 mod p in (0, 2p) for a < 2^32, b < p.
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv) {
  uint64_t t = (uint64_t)a * b;
  uint32_t lo = (uint32_t)t, hi = (uint32_t)(t >> 32);
  uint32_t m = lo * pinv;
  return hi - __umulhi(m, p) + p;
}

// Harvey lazy Cooley-Tukey butterfly: X, Y in [0, 4p) -> [0, 4p).
__device__ __forceinline__ void ct_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wq,
                                        uint32_t p, uint32_t two_p) {
  uint32_t x = umin(X, X - two_p);
  uint32_t t = shoup_mul(Y, w, wq, p);
  X = x + t;
  Y = x - t + two_p;
}

// Harvey lazy Gentleman-Sande butterfly: X, Y in [0, 2p) -> [0, 2p).
__device__ __forceinline__ void gs_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wq,
                                        uint32_t p, uint32_t two_p) {
  uint32_t x = X, y = Y;
  uint32_t s = x + y;
  X = umin(s, s - two_p);
  Y = shoup_mul(x - y + two_p, w, wq, p);
}

// Swizzled position of coefficient i in a warp's N-word transpose scratch:
// conflict-free both for layout-A writes/reads and layout-B reads/writes.
template <int N>
__device__ __forceinline__ int swz(int i) {
  constexpr int G = N / 1024;   // rows per lane group in layout B
  int r = i >> 5;
  return (r << 5) | ((i & 31) ^ ((r / G) & 31));
}

template <int N>
__device__ __forceinline__ void transpose_a_to_b(uint32_t (&x)[N / 32], uint32_t *scr, int lane) {
  constexpr int C = N / 32;
#pragma unroll
  for (int j = 0; j < C; ++j) scr[swz<N>(lane + 32 * j)] = x[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < C; ++j) x[j] = scr[swz<N>(C * lane + j)];
  __syncwarp();
}

template <int N>
__device__ __forceinline__ void transpose_b_to_a(uint32_t (&x)[N / 32], uint32_t *scr, int lane) {
  constexpr int C = N / 32;
#pragma unroll
  for (int j = 0; j < C; ++j) scr[swz<N>(C * lane + j)] = x[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < C; ++j) x[j] = scr[swz<N>(lane + 32 * j)];
  __syncwarp();
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Forward negacyclic NTT (merged psi twist, CT, natural -> bit-reversed).
// In: layout A, values in [0, 4p).  Out: layout B (lane holds NTT positions
// C*lane + j), values in [0, 4p).
template <int N>
__device__ __forceinline__ void fwd_ntt(uint32_t (&x)[N / 32], uint32_t *scr, int lane, int prime,
                                        const uint2 *__restrict__ lane_tw) {
  constexpr int C = N / 32;
  constexpr int NV = NVar<N>::v;
  const uint32_t p = c_prime[prime].p, two_p = c_prime[prime].two_p;
  // span t = 32h >= 32: m = C/(2h) blocks, twiddle psi_rev[m + blk], lane-uniform
  static_for<0, Log2<C>::v>([&](auto S) {
    constexpr int h = (C / 2) >> decltype(S)::value;
    constexpr int m = 1 << decltype(S)::value;
#pragma unroll
    for (int blk = 0; blk < m; ++blk) {
      const uint2 w = c_tw[NV][0][prime][m + blk];
#pragma unroll
      for (int jj = 0; jj < h; ++jj) ct_bfly(x[blk * 2 * h + jj], x[blk * 2 * h + jj + h], w.x, w.y, p, two_p);
    }
  });
  transpose_a_to_b<N>(x, scr, lane);
  // span t < 32: each lane covers C/(2t) blocks, per-lane twiddles
  static_for<0, 5>([&](auto S) {
    constexpr int t = 16 >> decltype(S)::value;
    constexpr int nb = C / (2 * t);
    constexpr int slot = (C / 32) * ((1 << decltype(S)::value) - 1);   // sum of earlier nb
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      const uint2 w = __ldg(&lane_tw[(slot + u) * 32 + lane]);
#pragma unroll
      for (int jj = 0; jj < t; ++jj) ct_bfly(x[u * 2 * t + jj], x[u * 2 * t + jj + t], w.x, w.y, p, two_p);
    }
  });
}

// Inverse negacyclic NTT (GS, bit-reversed -> natural, N^-1 folded into the
// GGSW).  In: layout B, values in [0, 2p).  Out: layout A, values in [0, 2p).
template <int N>
__device__ __forceinline__ void inv_ntt(uint32_t (&x)[N / 32], uint32_t *scr, int lane, int prime,
                                        const uint2 *__restrict__ lane_tw) {
  constexpr int C = N / 32;
  constexpr int NV = NVar<N>::v;
  const uint32_t p = c_prime[prime].p, two_p = c_prime[prime].two_p;
  static_for<0, 5>([&](auto S) {
    constexpr int t = 1 << decltype(S)::value;
    constexpr int nb = C / (2 * t);
    constexpr int slot = C - 2 * nb;   // sum of earlier nb: C/2 + C/4 + ... (S terms)
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      const uint2 w = __ldg(&lane_tw[(slot + u) * 32 + lane]);
#pragma unroll
      for (int jj = 0; jj < t; ++jj) gs_bfly(x[u * 2 * t + jj], x[u * 2 * t + jj + t], w.x, w.y, p, two_p);
    }
  });
  transpose_b_to_a<N>(x, scr, lane);
  static_for<0, Log2<C>::v>([&](auto S) {
    constexpr int h = 1 << decltype(S)::value;
    constexpr int m = C / (2 * h);
#pragma unroll
    for (int blk = 0; blk < m; ++blk) {
      const uint2 w = c_tw[NV][1][prime][m + blk];
#pragma unroll
      for (int jj = 0; jj < h; ++jj) gs_bfly(x[blk * 2 * h + jj], x[blk * 2 * h + jj + h], w.x, w.y, p, two_p);
    }
  });
}

// Offset of NTT position (lane, j) inside one N-word lane-interleaved slice:
// uint4 index (j/4)*32 + lane, element j%4.  A warp's uint4 load for fixed j/4
// covers 512 contiguous bytes.
template <int N>
__device__ __forceinline__ const uint4 *slice_vec(const uint32_t *slice, int lane, int jq) {
  return reinterpret_cast<const uint4 *>(slice) + jq * 32 + lane;
}

// CRT of (r0 mod p0, r1 mod p1), both canonical, to the centred integer mod 2^32.
__device__ __forceinline__ uint32_t crt_lift(uint32_t r0, uint32_t r1) {
  const uint32_t p0 = kP0, p1 = kP1;
  uint32_t d = r1 + 2u * p1 - r0;                      // (0, 3 p1)
  uint32_t t = shoup_mul(d, c_crt[0], c_crt[1], p1);   // [0, 2 p1)
  t = umin(t, t - p1);                                 // [0, p1)
  uint32_t res = r0 + p0 * t;                          // X = r0 + p0 t mod 2^32
  return (t > c_crt[3]) ? res - c_crt[2] : res;        // X >= P/2: X - P
}

// Gadget decomposition at q = 2^32 (hw/ring.py:126-151) in closed form:
// v = round(x / 2^(32 - l w)) + sum_k beta/2 beta^k; digit t (weight q/beta^(t+1))
// = ((v >> w (l-1-t)) & (beta-1)) - beta/2.  Equality with the reference's
// LSB-first carry loop is checked exhaustively over edge values in the tests.
struct Gadget {
  uint32_t round_add, shift, hsum, mask, half, base_log, levels;
};

__device__ __forceinline__ uint32_t decomp_prep(uint32_t x, const Gadget &g) {
  return ((x + g.round_add) >> g.shift) + g.hsum;
}

}  // namespace hwb
