// Device building blocks for exact negacyclic arithmetic mod 2^32 on sm_100a.
//
// Exactness strategy: the external product's true integer
// coefficients satisfy |sum_r d_r (*) g_r| <= 2l * N * beta/2 * 2^31 < 2^54 for
// every BASELINE config, so they are recovered exactly from their residues
// modulo two 28.4-bit NTT primes (P = p0*p1 ~ 2^56.8) by CRT and a centred lift,
// then reduced mod 2^32.
//
// Thread mapping: a group of TPP threads owns one (polynomial, prime) pair and
// keeps its N coefficients in registers, C = N/TPP per thread.  Every NTT
// stage pairs index bit s; it is thread-local in one of three layouts, each a
// bit permutation of (thread t, register j):
//   A (natural):  i = t + TPP*j                      stages s >= T   (T = log2 TPP)
//   M (middle):   i = t_lo | j << LO | t_hi << T     stages LOGC <= s < T
//   B (bit-rev):  i = j + C*t                        stages s < min(LOGC, T)
// with LO = T - LOGC.  Layout changes go through a swizzled shared-memory
// scratch (conflict-free for all three layouts, see swz_mask) and a named
// barrier over the group.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace hwb {

constexpr uint32_t kP0 = 357900289u;   // 0x15552001 = 43690*2^13 + 1
constexpr uint32_t kP1 = 357818369u;   // 0x1553e001 = 43680*2^13 + 1

struct PrimeConst {
  uint32_t p, two_p, pinv;   // pinv = p^-1 mod 2^32 (signed Montgomery REDC)
};

// Single translation unit (hwb_kernels.cu) includes this header.
// Uniform-stage twiddles (W, floor(W 2^32/p)) indexed [n_variant][dir][prime][k].
__constant__ uint2 c_tw[2][2][2][64];
__constant__ PrimeConst c_prime[2];
__constant__ uint32_t c_crt[4];        // {p0^-1 mod p1, its Shoup quotient, P mod 2^32, p1/2}
__constant__ uint32_t c_r2ninv[2][2];  // [n_variant][prime]: R^2 N^-1 mod p
// Always 0 (written by the host).  Two-operand adds written as x + y + c_zero
// compile to one IADD3 with a constant-bank operand on the ALU pipe; plain
// x + y is often emitted as IMAD.IADD, which occupies the FMA-heavy pipe the
// modular products are bound by.
__constant__ uint32_t c_zero;
#ifndef HWB_CZERO
#define HWB_CZERO 1
#endif
#if HWB_CZERO
#define HWB_Z + c_zero
#else
#define HWB_Z
#endif

template <int C> struct Log2 { static constexpr int v = (C <= 1) ? 0 : 1 + Log2<C / 2>::v; };
template <int N> struct NVar { static constexpr int v = (N == 1024) ? 0 : 1; };

template <int N, int TPP>
struct Geo {
  static constexpr int LOGN = Log2<N>::v;
  static constexpr int T = Log2<TPP>::v;
  static constexpr int C = N / TPP;
  static constexpr int LOGC = Log2<C>::v;
  static constexpr int LO = T - LOGC;            // > 0 iff a middle layout exists
  static constexpr bool HAS_M = LO > 0;
  static constexpr int B_TOP = LOGC < T ? LOGC : T;
  static constexpr int M_SLOTS = HAS_M ? (1 << LO) - 1 : 0;
  static constexpr int B_SLOTS = C - (C >> B_TOP);
  static constexpr int SLOTS = M_SLOTS + B_SLOTS;   // per-thread twiddles per transform
  static_assert(LOGN == T + LOGC, "N must be TPP * C");
  static_assert(LO <= LOGC, "three layouts cannot cover this (N, TPP)");
  static_assert(C % 4 == 0, "vectorised GGSW loads need C % 4 == 0");
};

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

__device__ __forceinline__ void prefetch_l2(const void *ptr) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}
__device__ __forceinline__ void prefetch_l1(const void *ptr) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
}

// Harvey lazy Cooley-Tukey butterfly: X, Y in [0, 4p) -> [0, 4p).
__device__ __forceinline__ void ct_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wq,
                                        uint32_t p, uint32_t two_p) {
  uint32_t x = umin(X, X - two_p);
  uint32_t t = shoup_mul(Y, w, wq, p);
  X = x + t HWB_Z;
  Y = x - t + two_p;
}

// Lazier CT butterfly for the forward transform.  Outputs are < x_bound + 2p
// (Shoup's t < 2p for any 32-bit input), so from inputs < 2p the bound grows
// by 2p per stage and reaches 12p after 5 stages; RED stages (execution index
// 5 and 10) first bring x from < 12p down to < 2p.  All values stay < 12p <
// 2^32 (p < 2^32/12), replacing 10-11 reductions per transform with 1-2.
template <bool RED>
__device__ __forceinline__ void ct_bfly_lazy(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wq,
                                             uint32_t p, uint32_t two_p) {
  uint32_t x = X;
  if (RED) {
    x = umin(x, x - 4 * two_p);
    x = umin(x, x - 2 * two_p);
    x = umin(x, x - two_p);
  }
  uint32_t t = shoup_mul(Y, w, wq, p);
  X = x + t HWB_Z;
  Y = x - t + two_p;
}

// Harvey lazy Gentleman-Sande butterfly: X, Y in [0, 2p) -> [0, 2p).
__device__ __forceinline__ void gs_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wq,
                                        uint32_t p, uint32_t two_p) {
  uint32_t x = X, y = Y;
  uint32_t s = x + y HWB_Z;
  X = umin(s, s - two_p);
  Y = shoup_mul(x - y + two_p, w, wq, p);
}

// Bank swizzle: XOR into the bank bits a GF(2)-linear image of the row bits
// (i >> 5).  Found by search; conflict-free for every layout of every
// (N, TPP) in {1024, 2048} x {32, 64, 128}.  Linearity lets the thread and
// register parts of an index be swizzled separately (pos = BT ^ OJ).
__host__ __device__ constexpr uint32_t swz_mask(uint32_t row) {
  constexpr uint32_t m[6] = {13, 27, 12, 31, 6, 24};
  uint32_t r = 0;
  for (int k = 0; k < 6; ++k)
    if ((row >> k) & 1u) r ^= m[k];
  return r;
}
__host__ __device__ constexpr uint32_t swz(uint32_t i) { return i ^ swz_mask(i >> 5); }

enum Layout { LAY_A = 0, LAY_M = 1, LAY_B = 2 };

// index offset contributed by register j in a layout (thread part excluded)
template <int N, int TPP, int LAY>
__host__ __device__ constexpr uint32_t joff(int j) {
  using G = Geo<N, TPP>;
  return LAY == LAY_A ? (uint32_t)(TPP * j) : (LAY == LAY_M ? (uint32_t)j << (G::LO > 0 ? G::LO : 0) : (uint32_t)j);
}

// index offset contributed by thread t in a layout
template <int N, int TPP, int LAY>
__device__ __forceinline__ uint32_t toff(int t) {
  using G = Geo<N, TPP>;
  if (LAY == LAY_A) return (uint32_t)t;
  if (LAY == LAY_B) return (uint32_t)(G::C * t);
  constexpr int LO = G::LO > 0 ? G::LO : 0;
  return ((uint32_t)t & ((1u << LO) - 1)) | (((uint32_t)t >> LO) << G::T);
}

// Swizzled thread bases of the three layouts (computed once per thread).
struct LayBase {
  uint32_t a, m, b;
};

template <int N, int TPP>
__device__ __forceinline__ LayBase make_lay(int t) {
  LayBase L;
  L.a = swz(toff<N, TPP, LAY_A>(t));
  L.m = swz(toff<N, TPP, LAY_M>(t));
  L.b = swz(toff<N, TPP, LAY_B>(t));
  return L;
}

template <int N, int TPP, int LAY>
__device__ __forceinline__ uint32_t lay_base(const LayBase &L) {
  return LAY == LAY_A ? L.a : (LAY == LAY_M ? L.m : L.b);
}

// Synchronise the TPP threads of one group (named barrier id 1 + group).
template <int TPP>
__device__ __forceinline__ void group_sync(int group) {
  if (TPP == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(TPP) : "memory");
  }
}

template <int N, int TPP, int FROM, int TO>
__device__ __forceinline__ void relayout(uint32_t (&x)[N / TPP], uint32_t *scr, const LayBase &L, int group) {
  constexpr int C = N / TPP;
  const uint32_t bf = lay_base<N, TPP, FROM>(L), bt = lay_base<N, TPP, TO>(L);
#pragma unroll
  for (int j = 0; j < C; ++j) scr[bf ^ swz(joff<N, TPP, FROM>(j))] = x[j];
  group_sync<TPP>(group);
#pragma unroll
  for (int j = 0; j < C; ++j) x[j] = scr[bt ^ swz(joff<N, TPP, TO>(j))];
  group_sync<TPP>(group);
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Per-thread twiddle load that the compiler may not hoist out of the digit
// loop (hoisting every loop-invariant twiddle into registers costs ~70
// registers per thread and halves occupancy); the table is L1-resident.
__device__ __forceinline__ uint2 ld_tw(const uint2 *ptr) {
  uint2 v;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(ptr));
  return v;
}

// One NTT stage on the register bit JB (partner j ^ 2^JB).  Twiddles: uniform
// (constant bank, index MBASE + u) or per thread (table slot SLOT + u).
// PRIME >= 0 specialises the code for one prime (uniform twiddles become
// direct constant-bank operands); PRIME < 0 takes the prime at run time, so
// both groups of a CTA share one copy of the code (smaller I-cache footprint).
template <int N, int TPP, int PRIME, bool FWD, int JB, bool UNIFORM, int MBASE, int SLOT, bool RED = true>
__device__ __forceinline__ void ntt_stage(uint32_t (&x)[N / TPP], int t, int prime, const uint2 *__restrict__ tw) {
  constexpr int C = N / TPP;
  constexpr int NBT = C >> (JB + 1);
  constexpr int HALF = 1 << JB;
  const int pr = PRIME >= 0 ? PRIME : prime;
  const uint32_t p = PRIME >= 0 ? (PRIME ? kP1 : kP0) : c_prime[pr].p;
  const uint32_t two_p = 2 * p;
#pragma unroll
  for (int u = 0; u < NBT; ++u) {
    const uint2 w = UNIFORM ? c_tw[NVar<N>::v][FWD ? 0 : 1][pr][MBASE + u]
                            : (PRIME >= 0 ? ld_tw(&tw[(SLOT + u) * TPP + t]) : __ldg(&tw[(SLOT + u) * TPP + t]));
#pragma unroll
    for (int lo = 0; lo < HALF; ++lo) {
      const int j = (u << (JB + 1)) | lo;
      if (FWD)
        ct_bfly_lazy<RED>(x[j], x[j + HALF], w.x, w.y, p, two_p);
      else
        gs_bfly(x[j], x[j + HALF], w.x, w.y, p, two_p);
    }
  }
}

// Forward negacyclic NTT (merged psi twist, CT, natural -> bit-reversed).
// In: layout A, values < 2p.  Out: layout B, values < 12p (lazy reduction:
// x is reduced only on execution stages 5 and 10 -- see ct_bfly_lazy).
// Per-thread twiddle slots: M stages s = T-1..LOGC, then B stages s = B_TOP-1..0.
template <int N, int TPP, int PRIME>
__device__ __forceinline__ void fwd_ntt(uint32_t (&x)[N / TPP], uint32_t *scr, const LayBase &L, int t, int prime,
                                        const uint2 *__restrict__ tw) {
  using G = Geo<N, TPP>;
  const int group = PRIME >= 0 ? PRIME : prime;
  static_for<0, G::LOGN - G::T>([&](auto K) {          // A stages s = LOGN-1 .. T
    constexpr int s = G::LOGN - 1 - decltype(K)::value;
    constexpr bool red = (G::LOGN - 1 - s) % 5 == 0 && s != G::LOGN - 1;
    ntt_stage<N, TPP, PRIME, true, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0, red>(x, t, prime, tw);
  });
  if constexpr (G::HAS_M) {
    relayout<N, TPP, LAY_A, LAY_M>(x, scr, L, group);
    static_for<0, G::T - G::LOGC>([&](auto K) {        // M stages s = T-1 .. LOGC
      constexpr int s = G::T - 1 - decltype(K)::value;
      constexpr int slot = (1 << decltype(K)::value) - 1;
      constexpr bool red = (G::LOGN - 1 - s) % 5 == 0 && s != G::LOGN - 1;
      ntt_stage<N, TPP, PRIME, true, s - G::LO, false, 0, slot, red>(x, t, prime, tw);
    });
    relayout<N, TPP, LAY_M, LAY_B>(x, scr, L, group);
  } else {
    relayout<N, TPP, LAY_A, LAY_B>(x, scr, L, group);
  }
  static_for<0, G::B_TOP>([&](auto K) {                  // B stages s = B_TOP-1 .. 0
    constexpr int s = G::B_TOP - 1 - decltype(K)::value;
    constexpr int slot = G::M_SLOTS + (G::C >> G::B_TOP) * ((1 << decltype(K)::value) - 1);
    constexpr bool red = (G::LOGN - 1 - s) % 5 == 0 && s != G::LOGN - 1;
    ntt_stage<N, TPP, PRIME, true, s, false, 0, slot, red>(x, t, prime, tw);
  });
}

// Inverse negacyclic NTT (GS, bit-reversed -> natural; N^-1 is folded into the
// GGSW).  In: layout B, values in [0, 2p).  Out: layout A, values in [0, 2p).
// Per-thread twiddle slots: B stages s = 0..B_TOP-1, then M stages s = LOGC..T-1.
template <int N, int TPP, int PRIME>
__device__ __forceinline__ void inv_ntt(uint32_t (&x)[N / TPP], uint32_t *scr, const LayBase &L, int t, int prime,
                                        const uint2 *__restrict__ tw, int bar_group = -1) {
  using G = Geo<N, TPP>;
  // named-barrier group of the TPP threads (TPP > 32): the prime unless overridden
  const int group = bar_group >= 0 ? bar_group : (PRIME >= 0 ? PRIME : prime);
  static_for<0, G::B_TOP>([&](auto K) {                  // B stages s = 0 .. B_TOP-1
    constexpr int s = decltype(K)::value;
    constexpr int slot = G::C - 2 * (G::C >> (s + 1));   // C/2 + C/4 + ... (s terms)
    ntt_stage<N, TPP, PRIME, false, s, false, 0, slot>(x, t, prime, tw);
  });
  if constexpr (G::HAS_M) {
    relayout<N, TPP, LAY_B, LAY_M>(x, scr, L, group);
    static_for<0, G::T - G::LOGC>([&](auto K) {        // M stages s = LOGC .. T-1
      constexpr int s = G::LOGC + decltype(K)::value;
      constexpr int slot = G::B_SLOTS + (1 << (G::T - G::LOGC)) - (1 << (G::T - s));
      ntt_stage<N, TPP, PRIME, false, s - G::LO, false, 0, slot>(x, t, prime, tw);
    });
    relayout<N, TPP, LAY_M, LAY_A>(x, scr, L, group);
  } else {
    relayout<N, TPP, LAY_B, LAY_A>(x, scr, L, group);
  }
  static_for<0, G::LOGN - G::T>([&](auto K) {          // A stages s = T .. LOGN-1
    constexpr int s = G::T + decltype(K)::value;
    ntt_stage<N, TPP, PRIME, false, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x, t, prime, tw);
  });
}

// NTT-domain polynomial slice: position (t, j) of layout B stored at uint4
// index (j/4)*TPP + t, element j%4 -- a group's uint4 load for fixed j/4 covers
// TPP*16 contiguous bytes.
template <int TPP>
__device__ __forceinline__ const uint4 *slice_vec(const uint32_t *slice, int t, int jq) {
  return reinterpret_cast<const uint4 *>(slice) + jq * TPP + t;
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
// LSB-first carry loop is checked against reference fixtures in the tests.
struct Gadget {
  uint32_t round_add, shift, hsum, mask, half, base_log, levels;
};

__device__ __forceinline__ uint32_t decomp_prep(uint32_t x, const Gadget &g) {
  return ((x + g.round_add) >> g.shift) + g.hsum;
}

}  // namespace hwb
