// hwb_fft.cuh — FP64 negacyclic FFT for the CMUX ladder (N = 1024), exact by rounding.
//
// The limb-exact route of the reference's FFT engine (hw/fft.py:88-119): the key
// words (signed 32-bit) are split into signed 16-bit halves G = lo + 2^16 hi, each
// product sum_t d_t * G_t is computed separately for lo and hi in double-precision
// complex arithmetic, rounded to the nearest integer and recombined mod 2^32.  The
// true sums are integers below 2l * N * beta/2 * 2^15 <= 2^37.6 and the FFT error is
// below 2^-13 (tests measure the margin), so rounding recovers them exactly: the
// result is bit-identical to the NTT ladder and to the reference's schoolbook.
//
// Folding: a real negacyclic polynomial a (degree < N) becomes the complex vector
// z_i = a_i + i a_{i+N/2} (i < H = N/2), i.e. a polynomial mod Y^H - i.  Its
// transform is the merged-twist Cooley-Tukey recursion on the roots of Y^H - i
// (root of block (level, m) = zeta^{E(level, m)/2}, zeta = e^{i pi / N}), the same
// block/twiddle indexing as the NTT (hwb_device.cuh); the inverse is the
// Gentleman-Sande recursion with conjugate twiddles, 1/H folded into the key.
//
// Thread mapping: one transform on 64 threads (2 warps), 8 complex values per thread,
// the A/M/B layouts of Geo<512, 64> (2 shared-memory transposes per transform).
#pragma once

#include <cstdint>

// Timing-only sensitivity switches (wrong results; tools/ab_variants.sh builds only):
// HWB_X_NOTRANS skips the transposes' shared-memory traffic, HWB_X_NOTW the per-thread
// twiddle loads, HWB_X_NOKEY the key-slice reads of the TMEM ladders' MAC.
#ifndef HWB_X_NOTRANS
#define HWB_X_NOTRANS 0
#endif
#ifndef HWB_X_NOTW
#define HWB_X_NOTW 0
#endif
#ifndef HWB_X_NOKEY
#define HWB_X_NOKEY 0
#endif

namespace hwb {

constexpr int FH = 512;       // complex points per folded polynomial (N = 1024)
constexpr int FT = 64;        // threads per transform
constexpr int FC = FH / FT;   // complex values per thread
using FGeo = Geo<FH, FT>;

// uniform A-stage twiddles [row][forward / inverse (conjugate)][k]: row 0 = the
// N = 1024 transform, rows 1 + g = half g of the N = 2048 transform (FFT2 below)
__constant__ double2 c_ftw[3][2][8];
__constant__ double2 c_fw0[2];   // FFT2 level-0 twiddle: [0] forward (cos, tan), [1] inverse (conjugate)

__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
#ifndef HWB_FFT_TAN
#define HWB_FFT_TAN 1
#endif
// (X, Y) -> (X + w Y, X - w Y).  Forward twiddles are stored in tangent form
// (cos t, tan t) (no forward twiddle has cos t = 0: the angles are odd multiples of
// pi / 2^k, k >= 2): w Y = cos t * (Y.x - tan t Y.y, Y.y + tan t Y.x), six DFMA per
// butterfly in two dependent steps instead of DMUL -> DFMA -> DADD.  The rounding
// error stays below 2^-52 (|cos t| + |sin t|) |Y| per step, as for the plain form.
__device__ __forceinline__ void fft_ct(double2 &X, double2 &Y, double2 w) {
#if HWB_FFT_TAN
  const double ux = fma(-w.y, Y.y, Y.x), uy = fma(w.y, Y.x, Y.y);
  Y = make_double2(fma(-w.x, ux, X.x), fma(-w.x, uy, X.y));
  X = make_double2(fma(w.x, ux, X.x), fma(w.x, uy, X.y));
#else
  const double2 t = cmul(Y, w);
  Y = make_double2(X.x - t.x, X.y - t.y);
  X = make_double2(X.x + t.x, X.y + t.y);
#endif
}
// (X, Y) -> (X + Y, (X - Y) conj(w_fwd)), the twiddle passed already conjugated
__device__ __forceinline__ void fft_gs(double2 &X, double2 &Y, double2 w) {
  const double2 d = make_double2(X.x - Y.x, X.y - Y.y);
  X = make_double2(X.x + Y.x, X.y + Y.y);
  Y = cmul(d, w);
}
// Sibling twiddles: blocks 2m and 2m + 1 of a level have roots r and -r, so their
// butterfly twiddles (square roots) differ by exactly i: w(2m+1) = i w(2m) (checked on
// the host table, fft_twiddles).  The odd block's butterfly is formed from the even
// block's twiddle at the same cost -- half the per-thread twiddle loads.
// forward, twiddle i w (w in tangent form): (X + i w Y, X - i w Y)
__device__ __forceinline__ void fft_ct_i(double2 &X, double2 &Y, double2 w) {
#if HWB_FFT_TAN
  const double ux = fma(-w.y, Y.y, Y.x), uy = fma(w.y, Y.x, Y.y);   // w Y = cos (ux, uy); i w Y = cos (-uy, ux)
  Y = make_double2(fma(w.x, uy, X.x), fma(-w.x, ux, X.y));
  X = make_double2(fma(-w.x, uy, X.x), fma(w.x, ux, X.y));
#else
  const double2 t = cmul(Y, w);
  Y = make_double2(X.x + t.y, X.y - t.x);
  X = make_double2(X.x - t.y, X.y + t.x);
#endif
}
// inverse, conj(i w) = -i conj(w): (X + Y, -i (X - Y) conj(w)), w passed conjugated
__device__ __forceinline__ void fft_gs_i(double2 &X, double2 &Y, double2 w) {
  const double2 d = make_double2(X.x - Y.x, X.y - Y.y);
  X = make_double2(X.x + Y.x, X.y + Y.y);
  Y = make_double2(fma(d.x, w.y, d.y * w.x), fma(-d.x, w.x, d.y * w.y));   // -i (d w) = (Im, -Re)
}
#ifndef HWB_FFT_SIB
#define HWB_FFT_SIB 1
#endif

// Compact per-thread twiddle table (CT = true, e.g. staged in shared memory): only the
// slots fft_stage loads -- the even u of every stage, siblings dropped -- in the order
// of the full table: forward slots {0, 1, 3, 5, 7, 8, 10, 12}, inverse {0, 2, 4, 6, 7,
// 9, 11, 13} of Geo<512, 64>'s 14 (hwb_kernels.cu: thread_table_of).
constexpr int kTwc = 8;
template <bool FWD>
__host__ __device__ constexpr int twc_slot(int s) {
  return FWD ? (s < 7 ? (s + 1) / 2 : 4 + (s - 6) / 2) : (s < 7 ? s / 2 : 4 + (s - 7) / 2);
}
template <bool FWD>
__host__ __device__ constexpr int twc_full(int c) {   // inverse map: compact slot -> full slot
  return FWD ? (c < 5 ? (c == 0 ? 0 : 2 * c - 1) : 6 + 2 * (c - 4)) : (c < 4 ? 2 * c : 7 + 2 * (c - 4));
}

template <bool FWD, int JB, bool UNIFORM, int MBASE, int SLOT, bool CT = false>
__device__ __forceinline__ void fft_stage(double2 (&x)[FC], int t, const double2 *__restrict__ tw, int cg = 0) {
  constexpr int NBT = FC >> (JB + 1);
  constexpr int HALF = 1 << JB;
  double2 w;
#pragma unroll
  for (int u = 0; u < NBT; ++u) {
    // per-thread twiddles: consecutive u are consecutive blocks of one level, the
    // odd one reuses the even one's twiddle (fft_ct_i / fft_gs_i)
    const bool sib = !UNIFORM && HWB_FFT_SIB && (u & 1);
#if HWB_X_NOTW   // timing-only sensitivity build: per-thread twiddles replaced by constants
    w = c_ftw[cg][FWD ? 0 : 1][(MBASE + u + SLOT) & 7];
#else
    if (!sib)
      w = UNIFORM ? c_ftw[cg][FWD ? 0 : 1][MBASE + u]
                  : (CT ? tw[twc_slot<FWD>(SLOT + u) * FT + t] : __ldg(&tw[(SLOT + u) * FT + t]));
#endif
#pragma unroll
    for (int lo = 0; lo < HALF; ++lo) {
      const int j = (u << (JB + 1)) | lo;
      if (FWD) {
        if (sib)
          fft_ct_i(x[j], x[j + HALF], w);
        else
          fft_ct(x[j], x[j + HALF], w);
      } else {
        if (sib)
          fft_gs_i(x[j], x[j + HALF], w);
        else
          fft_gs(x[j], x[j + HALF], w);
      }
    }
  }
}

// Bank swizzle for 16-byte elements: a quarter-warp's 8 accesses must hit distinct
// element slots mod 8.  e ^ ((e >> 3) & 7) achieves it in all three layouts (A and M
// already differ in e & 7 across a quarter-warp; B = 8t + j needs the row bits t
// folded in), and being GF(2)-linear it splits into thread and register parts.
__host__ __device__ constexpr uint32_t fswz(uint32_t e) { return e ^ ((e >> 3) & 7u); }

struct FLay {
  uint32_t a, m, b;
};
__device__ __forceinline__ FLay make_flay(int t) {
  return FLay{fswz(toff<FH, FT, LAY_A>(t)), fswz(toff<FH, FT, LAY_M>(t)), fswz(toff<FH, FT, LAY_B>(t))};
}
template <int LAY>
__device__ __forceinline__ uint32_t flay_base(const FLay &L) {
  return LAY == LAY_A ? L.a : (LAY == LAY_M ? L.m : L.b);
}

// The M <-> B transposes are warp-local.  Layout M is i = (t & 7) | (j << 3) | ((t >> 3) << 6)
// and layout B is i = 8 t + j: both keep index bits 6..8 in t >> 3 (and the swizzle only
// touches bits 0..2), so a value only ever moves between the 8 threads that share t >> 3.
// Every FFT kernel maps those 8 threads (of one ciphertext) into one warp (t = tid % 64,
// 16 hpos + (lane >> 1) or 8 w + (lane >> 2)), so the stores are ordered before the loads
// by __syncwarp() alone -- no CTA or named barrier over the transform's 2 to 8 warps.
// HWB_MB_LOCAL=0 restores the barrier.
#ifndef HWB_MB_LOCAL
#define HWB_MB_LOCAL 1
#endif
template <int FROM, int TO>
constexpr bool kMbLocal = HWB_MB_LOCAL && ((FROM == LAY_M && TO == LAY_B) || (FROM == LAY_B && TO == LAY_M));

// Barrier of the 64 threads of one transform: the whole CTA (bar == 0) or a named
// barrier when a CTA holds several transform groups.
__device__ __forceinline__ void fsync(int bar) {
  if (bar == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
}

// The CTA is exactly the 64 threads of the transform: CTA barriers.  `after_first`
// runs once all threads have passed the first barrier (everyone finished the
// previous consumer of any shared buffer -- the key-slice prefetch hook).
// TRAIL = false drops the trailing barrier.  Legal for the FIRST transpose of a
// transform (A -> M forward, B -> M inverse): the second transpose then stores each
// thread's values to exactly the addresses that thread loaded in the first (its
// middle-layout slots), so no thread can overwrite a location another thread has yet
// to read; the second transpose's own barrier orders everything after it.
template <int FROM, int TO, typename F, bool TRAIL = true>
__device__ __forceinline__ void frelayout(double2 (&x)[FC], double2 *scr, const FLay &L, F &&after_first,
                                          int bar = 0) {
  const uint32_t bf = flay_base<FROM>(L), bt = flay_base<TO>(L);
#pragma unroll
  for (int j = 0; j < FC; ++j) scr[bf ^ fswz(joff<FH, FT, FROM>(j))] = x[j];
  if (kMbLocal<FROM, TO>)
    __syncwarp();
  else
    fsync(bar);
  after_first();
#pragma unroll
  for (int j = 0; j < FC; ++j) x[j] = scr[bt ^ fswz(joff<FH, FT, TO>(j))];
  if (TRAIL) fsync(bar);
}
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// natural (layout A) -> block order (layout B); per-thread twiddle slots as fwd_ntt
template <typename F = NoHook>
__device__ __forceinline__ void fwd_fft(double2 (&x)[FC], double2 *scr, const FLay &L, int t,
                                        const double2 *__restrict__ tw, F &&hook = F(), int bar = 0, int cg = 0) {
  using G = FGeo;
  static_for<0, G::LOGN - G::T>([&](auto K) {
    constexpr int s = G::LOGN - 1 - decltype(K)::value;
    fft_stage<true, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x, t, tw, cg);
  });
  frelayout<LAY_A, LAY_M, F &, false>(x, scr, L, hook, bar);
  static_for<0, G::T - G::LOGC>([&](auto K) {
    constexpr int s = G::T - 1 - decltype(K)::value;
    constexpr int slot = (1 << decltype(K)::value) - 1;
    fft_stage<true, s - G::LO, false, 0, slot>(x, t, tw, cg);
  });
  frelayout<LAY_M, LAY_B>(x, scr, L, NoHook(), bar);
  static_for<0, G::B_TOP>([&](auto K) {
    constexpr int s = G::B_TOP - 1 - decltype(K)::value;
    constexpr int slot = G::M_SLOTS + (G::C >> G::B_TOP) * ((1 << decltype(K)::value) - 1);
    fft_stage<true, s, false, 0, slot>(x, t, tw, cg);
  });
}

// block order (layout B) -> natural (layout A), unscaled (1/H is in the key)
__device__ __forceinline__ void inv_fft(double2 (&x)[FC], double2 *scr, const FLay &L, int t,
                                        const double2 *__restrict__ tw, int bar = 0, int cg = 0) {
  using G = FGeo;
  static_for<0, G::B_TOP>([&](auto K) {
    constexpr int s = decltype(K)::value;
    constexpr int slot = G::C - 2 * (G::C >> (s + 1));
    fft_stage<false, s, false, 0, slot>(x, t, tw, cg);
  });
  frelayout<LAY_B, LAY_M, NoHook, false>(x, scr, L, NoHook(), bar);
  static_for<0, G::T - G::LOGC>([&](auto K) {
    constexpr int s = G::LOGC + decltype(K)::value;
    constexpr int slot = G::B_SLOTS + (1 << (G::T - G::LOGC)) - (1 << (G::T - s));
    fft_stage<false, s - G::LO, false, 0, slot>(x, t, tw, cg);
  });
  frelayout<LAY_M, LAY_A>(x, scr, L, NoHook(), bar);
  static_for<0, G::LOGN - G::T>([&](auto K) {
    constexpr int s = G::T + decltype(K)::value;
    fft_stage<false, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x, t, tw, cg);
  });
}

// K independent inverse transforms in lockstep (the four accumulators of a CMUX
// step): one pair of barriers per transpose for all K, K times the ILP per stage.
// scr holds K * FH elements.
template <int K, int FROM, int TO, typename F = NoHook, bool TRAIL = true>
__device__ __forceinline__ void frelayout_k(double2 (*x)[FC], double2 *scr, const FLay &L, F &&after_first = F()) {
  const uint32_t bf = flay_base<FROM>(L), bt = flay_base<TO>(L);
#if HWB_X_NOTRANS   // timing-only sensitivity build: barriers kept, no shared-memory round trip
  __syncthreads();
  after_first();
  __syncthreads();
  return;
#endif
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) scr[k * FH + (bf ^ fswz(joff<FH, FT, FROM>(j)))] = x[k][j];
  if (kMbLocal<FROM, TO>)
    __syncwarp();
  else
    __syncthreads();
  after_first();
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) x[k][j] = scr[k * FH + (bt ^ fswz(joff<FH, FT, TO>(j)))];
  if (TRAIL) __syncthreads();
}

// K independent forward transforms in lockstep (the two key halves of a GGSW row;
// two ciphertexts of the TMEM ladder); `hook` as in fwd_fft
template <int K, bool CT = false, typename F = NoHook>
__device__ __forceinline__ void fwd_fft_k(double2 (*x)[FC], double2 *scr, const FLay &L, int t,
                                          const double2 *__restrict__ tw, int cg = 0, F &&hook = F()) {
  using G = FGeo;
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::LOGN - 1 - decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw, cg);
  });
  frelayout_k<K, LAY_A, LAY_M, F &, false>(x, scr, L, hook);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::T - 1 - decltype(Q)::value;
    constexpr int slot = (1 << decltype(Q)::value) - 1;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::LO, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  frelayout_k<K, LAY_M, LAY_B>(x, scr, L);
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = G::B_TOP - 1 - decltype(Q)::value;
    constexpr int slot = G::M_SLOTS + (G::C >> G::B_TOP) * ((1 << decltype(Q)::value) - 1);
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s, false, 0, slot, CT>(x[k], t, tw, cg);
  });
}

template <int K, bool CT = false>
__device__ __forceinline__ void inv_fft_k(double2 (*x)[FC], double2 *scr, const FLay &L, int t,
                                          const double2 *__restrict__ tw, int cg = 0) {
  using G = FGeo;
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = decltype(Q)::value;
    constexpr int slot = G::C - 2 * (G::C >> (s + 1));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  frelayout_k<K, LAY_B, LAY_M, NoHook, false>(x, scr, L);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::LOGC + decltype(Q)::value;
    constexpr int slot = G::B_SLOTS + (1 << (G::T - G::LOGC)) - (1 << (G::T - s));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::LO, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  frelayout_k<K, LAY_M, LAY_A>(x, scr, L);
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::T + decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw, cg);
  });
}

// exact small integer -> double without a conversion instruction: 2^52 + u - (2^52 + off)
__device__ __forceinline__ double u2d_minus(uint32_t u, double two52_plus_off) {
  return __hiloint2double(0x43300000, (int)u) - two52_plus_off;
}
// Rounding-margin instrumentation (the build of libhwb200_margin.so, -DHWB_FFT_MARGIN=1):
// every rounded FFT output records |y - rint(y)| into g_fft_margin (the bit pattern of
// a non-negative double orders like an integer), read back by hwb_fft_margin().  The
// exactness argument needs this to stay well below 1/2; tests assert < 2^-6.
#ifndef HWB_FFT_MARGIN
#define HWB_FFT_MARGIN 0
#endif
#if HWB_FFT_MARGIN
__device__ unsigned long long g_fft_margin;
#endif
// round to nearest and reduce mod 2^32 (|y| < 2^51): low word of y + 1.5 * 2^52
__device__ __forceinline__ uint32_t round_u32(double y) {
  const double r = y + 6755399441055744.0;
#if HWB_FFT_MARGIN
  const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(y - (r - 6755399441055744.0)));
  if (bits > *(volatile unsigned long long *)&g_fft_margin) atomicMax(&g_fft_margin, bits);
#endif
  return (uint32_t)__double2loint(r);
}

}  // namespace hwb

namespace hwb {

// ---- ping-pong transforms (group-local named barriers, one barrier per transpose) ----
// The two transposes of a transform use two different scratch buffers (s0: the first,
// s1: the second), so a transpose needs no trailing barrier: the next write into a
// buffer always follows the barrier of the other buffer's transpose, which every
// reader of the first passed only after its loads.  `bar` is a named barrier over the
// NT threads of the transform group; per-thread twiddles come from the compact table
// (CT) or the full global table.
template <int NT>
__device__ __forceinline__ void gsync(int bar) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");
}

template <int K, int FROM, int TO, int NT, typename F = NoHook>
__device__ __forceinline__ void frelayout_pp(double2 (*x)[FC], double2 *scr, const FLay &L, int bar,
                                             F &&after_first = F()) {
  const uint32_t bf = flay_base<FROM>(L), bt = flay_base<TO>(L);
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) scr[k * FH + (bf ^ fswz(joff<FH, FT, FROM>(j)))] = x[k][j];
  gsync<NT>(bar);
  after_first();
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) x[k][j] = scr[k * FH + (bt ^ fswz(joff<FH, FT, TO>(j)))];
}

template <int K, int NT, bool CT = false, typename F = NoHook>
__device__ __forceinline__ void fwd_fft_pp(double2 (*x)[FC], double2 *s0, double2 *s1, const FLay &L, int t,
                                           const double2 *__restrict__ tw, int bar, F &&hook = F()) {
  using G = FGeo;
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::LOGN - 1 - decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw);
  });
  frelayout_pp<K, LAY_A, LAY_M, NT>(x, s0, L, bar, hook);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::T - 1 - decltype(Q)::value;
    constexpr int slot = (1 << decltype(Q)::value) - 1;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::LO, false, 0, slot, CT>(x[k], t, tw);
  });
  frelayout_pp<K, LAY_M, LAY_B, NT>(x, s1, L, bar);
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = G::B_TOP - 1 - decltype(Q)::value;
    constexpr int slot = G::M_SLOTS + (G::C >> G::B_TOP) * ((1 << decltype(Q)::value) - 1);
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s, false, 0, slot, CT>(x[k], t, tw);
  });
}

template <int K, int NT, bool CT = false>
__device__ __forceinline__ void inv_fft_pp(double2 (*x)[FC], double2 *s0, double2 *s1, const FLay &L, int t,
                                           const double2 *__restrict__ tw, int bar) {
  using G = FGeo;
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = decltype(Q)::value;
    constexpr int slot = G::C - 2 * (G::C >> (s + 1));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s, false, 0, slot, CT>(x[k], t, tw);
  });
  frelayout_pp<K, LAY_B, LAY_M, NT>(x, s0, L, bar);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::LOGC + decltype(Q)::value;
    constexpr int slot = G::B_SLOTS + (1 << (G::T - G::LOGC)) - (1 << (G::T - s));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::LO, false, 0, slot, CT>(x[k], t, tw);
  });
  frelayout_pp<K, LAY_M, LAY_A, NT>(x, s1, L, bar);
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::T + decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw);
  });
}

}  // namespace hwb

namespace hwb {

// frelayout_k with a named barrier over NT threads (both barriers kept: one scratch)
template <int K, int FROM, int TO, int NT, bool TRAIL = true>
__device__ __forceinline__ void frelayout_hk(double2 (*x)[FC], double2 *scr, const FLay &L, int bar) {
  const uint32_t bf = flay_base<FROM>(L), bt = flay_base<TO>(L);
#if HWB_X_NOTRANS   // timing-only sensitivity build: barriers kept, no shared-memory round trip
  gsync<NT>(bar);
  if (TRAIL) gsync<NT>(bar);
  return;
#endif
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) scr[k * FH + (bf ^ fswz(joff<FH, FT, FROM>(j)))] = x[k][j];
  if (kMbLocal<FROM, TO>)
    __syncwarp();
  else
    gsync<NT>(bar);
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < FC; ++j) x[k][j] = scr[k * FH + (bt ^ fswz(joff<FH, FT, TO>(j)))];
  if (TRAIL) gsync<NT>(bar);
}

// TRAIL2 = false drops the trailing barrier of the second transpose: the caller
// guarantees a group barrier before the next write into scr.
// `pre` runs right before the first store into scr (the split scratch-free wait of the
// mode-5 ladder's HWB_TD_SPLITBAR build).
template <int K, int NT, bool CT = false, bool TRAIL2 = true, typename F = NoHook>
__device__ __forceinline__ void fwd_fft_hk(double2 (*x)[FC], double2 *scr, const FLay &L, int t,
                                           const double2 *__restrict__ tw, int bar, int cg = 0, F &&pre = F()) {
  using G = FGeo;
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::LOGN - 1 - decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw, cg);
  });
  pre();
  frelayout_hk<K, LAY_A, LAY_M, NT, false>(x, scr, L, bar);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::T - 1 - decltype(Q)::value;
    constexpr int slot = (1 << decltype(Q)::value) - 1;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s - G::LO, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  frelayout_hk<K, LAY_M, LAY_B, NT, TRAIL2>(x, scr, L, bar);
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = G::B_TOP - 1 - decltype(Q)::value;
    constexpr int slot = G::M_SLOTS + (G::C >> G::B_TOP) * ((1 << decltype(Q)::value) - 1);
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<true, s, false, 0, slot, CT>(x[k], t, tw, cg);
  });
}

template <int K, int NT, bool CT = false, bool TRAIL2 = true, typename F = NoHook>
__device__ __forceinline__ void inv_fft_hk(double2 (*x)[FC], double2 *scr, const FLay &L, int t,
                                           const double2 *__restrict__ tw, int bar, int cg = 0, F &&pre = F()) {
  using G = FGeo;
  static_for<0, G::B_TOP>([&](auto Q) {
    constexpr int s = decltype(Q)::value;
    constexpr int slot = G::C - 2 * (G::C >> (s + 1));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  pre();
  frelayout_hk<K, LAY_B, LAY_M, NT, false>(x, scr, L, bar);
  static_for<0, G::T - G::LOGC>([&](auto Q) {
    constexpr int s = G::LOGC + decltype(Q)::value;
    constexpr int slot = G::B_SLOTS + (1 << (G::T - G::LOGC)) - (1 << (G::T - s));
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::LO, false, 0, slot, CT>(x[k], t, tw, cg);
  });
  frelayout_hk<K, LAY_M, LAY_A, NT, TRAIL2>(x, scr, L, bar);
  static_for<0, G::LOGN - G::T>([&](auto Q) {
    constexpr int s = G::T + decltype(Q)::value;
#pragma unroll
    for (int k = 0; k < K; ++k) fft_stage<false, s - G::T, true, (1 << (G::LOGN - 1 - s)), 0>(x[k], t, tw, cg);
  });
}

// ---------------------------------------------------------------------------
// Wide-thread transform: the same 512-point merged-twist network on 32 threads with 16
// complex values each (FFT mode 7, blind_rotate_fft_w_kernel).  Nine levels = 4 (layout
// A16) + 4 (layout M16) + 1 (partner exchange): ONE shared-memory transpose per
// transform instead of two, and the last level's pairs (i, i + 1) meet through warp
// shuffles.  Index bits i8..i0 of the in-place array:
//   A16: thread t = i4..i0, slot j = i8..i5          (levels 0-3, uniform twiddles)
//   M16: thread u = (i8..i5) << 1 | i0, slot jj = i4..i1   (levels 4-7)
//   X16: thread u, b = u & 1: slots s < 8 hold i0 = 0, s + 8 hold i0 = 1 of the pairs
//        with i4 = b, (i3 i2 i1) = s & 7, i.e. i = (u >> 1) << 5 | b << 4 | (s & 7) << 1 | s >> 3
// Level L, block m uses the twiddle k = 2^L + m of fft_twiddles (as every other ladder),
// and the network is in place, so array position i of the spectrum holds what it holds in
// the 64-thread transforms: the FFT key is read in its usual [c][h][j][t] layout at
// (j, t) = (i & 7, i >> 3).
constexpr int WT = 32;   // threads per transform
constexpr int WC = 16;   // complex values per thread

__constant__ double2 c_w16[2][16];   // twiddles k = 1..15 (levels 0-3): [0] forward (cos, tan), [1] inverse (conjugate)

// 16-byte-element swizzle of the one transpose: a quarter-warp (4 threads x the two
// lane-paired ciphertexts, the odd one XOR 4) must hit 8 distinct slots mod 8.  In A16 the
// 4 threads differ in (i0, i1), in M16 in (i0, i5): folding i5 into bit 1 serves both.
__host__ __device__ constexpr uint32_t wswz(uint32_t i) { return i ^ (((i >> 5) & 1u) << 1); }
// array index of slot s of thread u in the final (X16) layout
__host__ __device__ constexpr int w16_index(int u, int s) {
  return ((u >> 1) << 5) | ((u & 1) << 4) | ((s & 7) << 1) | (s >> 3);
}
// Per-thread twiddle tables of one direction, [kW16Tab] double2: twm[slot][u >> 1] (slots:
// level 4 -> 0, level 5 -> 1, level 6 -> 2, 3, level 7 -> 4..7; even blocks only, the odd
// sibling reuses them) then tw8[slot][u] (level 8, blocks 8 u + {0, 2, 4, 6}).
constexpr int kW16Twm = 8 * 16, kW16Tab = kW16Twm + 4 * WT;

// one level on the thread's 16 values: pairs (v, v + 2^P); block b = v >> (P + 1) uses
// tw(b); SIB: odd blocks reuse the even block's twiddle (fft_ct_i / fft_gs_i)
template <bool FWD, int P, bool SIB, typename TW>
__device__ __forceinline__ void stage16(double2 (&x)[WC], TW &&tw) {
  constexpr int NB = WC >> (P + 1), HALF = 1 << P;
  double2 w = make_double2(0.0, 0.0);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const bool sib = SIB && (b & 1);
    if (!sib) w = tw(b);
#pragma unroll
    for (int lo = 0; lo < HALF; ++lo) {
      const int v = (b << (P + 1)) | lo;
      if (FWD) {
        if (sib)
          fft_ct_i(x[v], x[v + HALF], w);
        else
          fft_ct(x[v], x[v + HALF], w);
      } else {
        if (sib)
          fft_gs_i(x[v], x[v + HALF], w);
        else
          fft_gs(x[v], x[v + HALF], w);
      }
    }
  }
}

// the partner exchange between M16 and X16 (its own inverse): the thread with i0 = b
// keeps slots s < 8 (b = 0) or s >= 8 (b = 1) and swaps the others with lane ^ 2
__device__ __forceinline__ void w16_exchange(double2 (&x)[WC], bool b) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const double2 snd = b ? x[s] : x[s + 8];
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, snd.x, 2);
    r.y = __shfl_xor_sync(0xffffffffu, snd.y, 2);
    if (b)
      x[s] = r;
    else
      x[s + 8] = r;
  }
}

// natural order (A16) -> spectrum (X16).  ea / em: the thread's swizzled element bases in
// the two layouts (make_w16_bases), tab: the forward table (shared memory), `bar`: named
// barrier of the transform's 64 threads (2 warps x 2 lane-paired ciphertexts).
__device__ __forceinline__ void fwd_fft16(double2 (&x)[WC], double2 *scr, uint32_t ea, uint32_t em, int u,
                                          const double2 *__restrict__ tab, int bar) {
  static_for<0, 4>([&](auto Q) {
    constexpr int L = decltype(Q)::value;
    stage16<true, 3 - L, false>(x, [&](int b) { return c_w16[0][(1 << L) + b]; });
  });
#pragma unroll
  for (int j = 0; j < WC; ++j) scr[ea ^ wswz((uint32_t)(WT * j))] = x[j];
  gsync<64>(bar);
#pragma unroll
  for (int jj = 0; jj < WC; ++jj) x[jj] = scr[em ^ (uint32_t)(jj << 1)];
  const double2 *tm = tab + (u >> 1), *tw8 = tab + kW16Twm + u;
  stage16<true, 3, true>(x, [&](int) { return tm[0 * 16]; });
  stage16<true, 2, true>(x, [&](int) { return tm[1 * 16]; });
  stage16<true, 1, true>(x, [&](int b) { return tm[(2 + (b >> 1)) * 16]; });
  stage16<true, 0, true>(x, [&](int b) { return tm[(4 + (b >> 1)) * 16]; });
  w16_exchange(x, u & 1);
  double2 w = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < 8; ++s) {   // level 8: one butterfly per block, siblings in pairs
    if (s & 1) {
      fft_ct_i(x[s], x[s + 8], w);
    } else {
      w = tw8[(s >> 1) * WT];
      fft_ct(x[s], x[s + 8], w);
    }
  }
}

// spectrum (X16) -> natural order (A16), unscaled (1/H is in the key); trail: trailing
// barrier (the next writer of scr may be the other warp)
__device__ __forceinline__ void inv_fft16(double2 (&x)[WC], double2 *scr, uint32_t ea, uint32_t em, int u,
                                          const double2 *__restrict__ tab, int bar, bool trail) {
  const double2 *tm = tab + (u >> 1), *tw8 = tab + kW16Twm + u;
  double2 w = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (s & 1) {
      fft_gs_i(x[s], x[s + 8], w);
    } else {
      w = tw8[(s >> 1) * WT];
      fft_gs(x[s], x[s + 8], w);
    }
  }
  w16_exchange(x, u & 1);
  stage16<false, 0, true>(x, [&](int b) { return tm[(4 + (b >> 1)) * 16]; });
  stage16<false, 1, true>(x, [&](int b) { return tm[(2 + (b >> 1)) * 16]; });
  stage16<false, 2, true>(x, [&](int) { return tm[1 * 16]; });
  stage16<false, 3, true>(x, [&](int) { return tm[0 * 16]; });
#pragma unroll
  for (int jj = 0; jj < WC; ++jj) scr[em ^ (uint32_t)(jj << 1)] = x[jj];
  gsync<64>(bar);
#pragma unroll
  for (int j = 0; j < WC; ++j) x[j] = scr[ea ^ wswz((uint32_t)(WT * j))];
  static_for<0, 4>([&](auto Q) {
    constexpr int L = 3 - decltype(Q)::value;
    stage16<false, 3 - L, false>(x, [&](int b) { return c_w16[1][(1 << L) + b]; });
  });
  if (trail) gsync<64>(bar);   // (after the last levels, as in mode 5: 54.3 -> 52.4 ms there)
}


}  // namespace hwb
