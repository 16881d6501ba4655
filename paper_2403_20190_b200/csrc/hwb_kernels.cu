// libhwb200: batched TFHE bootstrapping kernels for B200 (sm_100a) and their C ABI.
//
// Kernels:
//   ggsw_to_ntt_kernel  GGSW -> NTT domain (Montgomery form, N^-1 folded)
//   cmux_kernel<MODE>   batched external product / CMUX / CDEMUX, one item per CTA
//   blind_rotate_kernel fused CMUX ladder (hw/tfhe.py:340-349), all L steps in one
//                       launch with the accumulator resident in shared memory;
//                       PBS mode adds mod switch, TV rotation and extraction
//   extract_kernel      sample extraction (hw/tfhe.py:352-361)
//   keyswitch_kernel    LWE key switch as a tiled integer contraction mod 2^32
//
// CTA shape for the ladder/CMUX kernels: 2 groups of TPP threads = one
// ciphertext; group g works modulo prime p_g on both GLWE components, then the
// groups exchange residues through shared memory and group g lifts component g
// by CRT.  TPP = 32 (N = 1024) or 64 (N = 2048): 32 coefficients per thread.
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hwb.h"
#include "hwb_device.cuh"
#include "hwb_tc.cuh"
#include "hwb_fft.cuh"

namespace hwb {

static thread_local std::string g_err;
// kernel variant: selects the register/occupancy build of the ladder kernels
// (0 = default, 1 = alternative); both bit-identical, for A/B measurement.
static thread_local int g_variant = 0;
// batches up to this size run the latency-mode ladder (blind_rotate_lat_kernel);
// -1 = automatic (3 x the SM count: up to three waves of 2 CTAs per SM).
static thread_local int64_t g_lat_max_batch = -1;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

// Per-ring-degree launch shape.  32 threads per (polynomial, prime) at N = 1024
// and 64 at N = 2048 (32 coefficients per thread either way).  Measured on
// B200 (profiles/r01_*): 64 threads at N = 1024 (16 coefficients, a middle
// layout, 2 transposes per NTT) was 8-20% slower than 32 threads.
// Kernel variants (hwb_set_variant): V0 = prime taken at run time (one code
// copy shared by both groups), V1 = V0 with a register cap for HWB_V1_MINB
// resident CTAs/SM.  (A per-prime specialised build -- uniform twiddles as
// constant-bank operands, twice the code -- measured 2x slower: I-cache.)
#ifndef HWB_V1_MINB
#define HWB_V1_MINB 6
#endif
template <int N> struct Cfg {
  static constexpr int TPP = (N == 1024) ? 32 : 64;
  static constexpr int THREADS = 2 * TPP;
  __host__ __device__ static constexpr bool spec(int v) { return v == 2; }
  __host__ __device__ static constexpr int minb(int v) { return v == 1 ? HWB_V1_MINB : 1; }
};

// ---------------------------------------------------------------------------
// host-side table construction

static uint32_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  b %= m;
  while (e) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return (uint32_t)r;
}

static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

static uint2 shoup_pair(uint32_t w, uint32_t p) {
  return make_uint2(w, (uint32_t)(((uint64_t)w << 32) / p));
}

struct DevState {
  bool ready = false;
  int sms = 148;
  uint2 *lane_fwd[2][2] = {};   // [n_variant][prime] -> [slot][TPP]
  uint2 *lane_inv[2][2] = {};
  uint2 *lane_inv64[2] = {};    // N = 1024 inverse transform on 64 threads (latency ladder)
  double2 *fft_fwd = nullptr, *fft_inv = nullptr;   // FP64 FFT per-thread twiddles
  double2 *fft_w16 = nullptr;   // wide-thread transform (mode 7): [forward, inverse][kW16Tab]
  double2 *fft2_fwd[2] = {}, *fft2_inv[2] = {};     // N = 2048: the sub-transform of half g
};

static std::mutex g_mu;
static DevState g_state[64];

// Per-thread twiddle table in the slot order fwd_ntt/inv_ntt consume
// (hwb_device.cuh): twiddle index of stage s, block b is m + b, m = N/2^(s+1).
// Per-thread twiddle table in the slot order the transforms consume: entry
// (slot, t) holds val(k) for the twiddle index k of that slot and thread.
template <int N, int TPP, typename V, typename F>
static std::vector<V> thread_table_of(F val, bool fwd) {
  using G = Geo<N, TPP>;
  std::vector<V> tab((size_t)G::SLOTS * TPP);
  int slot = 0;
  auto m_stage = [&](int s) {   // middle layout: block = t_hi 2^(T-s-1) + u
    const int nb = 1 << (G::T - s - 1);
    for (int u = 0; u < nb; ++u)
      for (int t = 0; t < TPP; ++t)
        tab[(size_t)(slot + u) * TPP + t] = val((N >> (s + 1)) + (t >> G::LO) * nb + u);
    slot += nb;
  };
  auto b_stage = [&](int s) {   // bit-reversed layout: block = t C/2^(s+1) + u
    const int nb = G::C >> (s + 1);
    for (int u = 0; u < nb; ++u)
      for (int t = 0; t < TPP; ++t)
        tab[(size_t)(slot + u) * TPP + t] = val((N >> (s + 1)) + t * nb + u);
    slot += nb;
  };
  if (fwd) {
    if (G::HAS_M)
      for (int s = G::T - 1; s >= G::LOGC; --s) m_stage(s);
    for (int s = G::B_TOP - 1; s >= 0; --s) b_stage(s);
  } else {
    for (int s = 0; s < G::B_TOP; ++s) b_stage(s);
    if (G::HAS_M)
      for (int s = G::LOGC; s < G::T; ++s) m_stage(s);
  }
  return tab;
}

template <int N, int TPP = Cfg<N>::TPP>
static std::vector<uint2> thread_table(const std::vector<uint32_t> &w, uint32_t p, bool fwd) {
  return thread_table_of<N, TPP, uint2>([&](int k) { return shoup_pair(w[k], p); }, fwd);
}

// FFT twiddles (hwb_fft.cuh): k = 2^level + m -> zeta^{E(level, m)/2}, zeta = e^{i pi/(2H)},
// E(0, 0) = H and E(level+1, {2m, 2m+1}) = {E/2, E/2 + 2H} (mod 4H): the roots of the
// factors of Y^H - i.  Computed in long double, rounded once to double.
static std::vector<double2> fft_twiddles(bool conj, int H = FH) {
  std::vector<long> E(2 * H, 0);
  E[1] = H;
  for (int k = 1; k < H; ++k) {
    E[2 * k] = (E[k] / 2) % (4 * H);
    E[2 * k + 1] = (E[k] / 2 + 2 * H) % (4 * H);
  }
  std::vector<double2> w(H);
  for (int k = 1; k < H; ++k) {
    const long double ang = acosl(-1.0L) * (long double)(E[k] / 2) / (long double)(2 * H);
    w[k] = make_double2((double)cosl(ang), (double)(conj ? -sinl(ang) : sinl(ang)));
#if HWB_FFT_TAN
    if (!conj) w[k] = make_double2((double)cosl(ang), (double)tanl(ang));   // tangent form (fft_ct)
#endif
  }
  w[0] = make_double2(1.0, 0.0);
  return w;
}

static int init_device(DevState **out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(HWB_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  if (dev < 0 || dev >= 64) return fail(HWB_ECUDA, "device index out of range");
  std::lock_guard<std::mutex> lk(g_mu);
  DevState &st = g_state[dev];
  if (st.ready) {
    *out = &st;
    return HWB_OK;
  }
  const uint32_t primes[2] = {kP0, kP1};
  cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev);
  static uint2 h_tw[2][2][2][64];
  uint32_t h_r2ninv[2][2];
  PrimeConst h_prime[2];
  for (int pr = 0; pr < 2; ++pr) {
    uint32_t p = primes[pr];
    uint32_t inv = 1;   // p^-1 mod 2^32 by Newton
    for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    h_prime[pr] = PrimeConst{p, 2u * p, inv};
  }
  for (int nv = 0; nv < 2; ++nv) {
    const int N = nv == 0 ? 1024 : 2048;
    const int logN = nv == 0 ? 10 : 11;
    for (int pr = 0; pr < 2; ++pr) {
      const uint32_t p = primes[pr];
      uint32_t psi = 0;
      for (uint32_t a = 2; a < 1000; ++a) {
        uint32_t c = powmod(a, (p - 1) / (2 * N), p);
        if (powmod(c, N, p) == p - 1) {
          psi = c;
          break;
        }
      }
      if (!psi) return fail(HWB_ECUDA, "no 2N-th root of unity");
      const uint32_t psi_inv = powmod(psi, p - 2, p);
      std::vector<uint32_t> fw(N), iw(N);
      for (int k = 0; k < N; ++k) {
        fw[k] = powmod(psi, bitrev(k, logN), p);
        iw[k] = powmod(psi_inv, bitrev(k, logN), p);
      }
      for (int k = 0; k < 64; ++k) {
        h_tw[nv][0][pr][k] = shoup_pair(fw[k], p);
        h_tw[nv][1][pr][k] = shoup_pair(iw[k], p);
      }
      std::vector<uint2> lf = nv == 0 ? thread_table<1024>(fw, p, true) : thread_table<2048>(fw, p, true);
      std::vector<uint2> li = nv == 0 ? thread_table<1024>(iw, p, false) : thread_table<2048>(iw, p, false);
      const size_t bytes = sizeof(uint2) * lf.size();
      cudaError_t e1 = cudaMalloc(&st.lane_fwd[nv][pr], bytes);
      cudaError_t e2 = cudaMalloc(&st.lane_inv[nv][pr], bytes);
      if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(HWB_ECUDA, "cudaMalloc twiddle tables failed");
      e1 = cudaMemcpy(st.lane_fwd[nv][pr], lf.data(), bytes, cudaMemcpyHostToDevice);
      e2 = cudaMemcpy(st.lane_inv[nv][pr], li.data(), bytes, cudaMemcpyHostToDevice);
      if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(HWB_ECUDA, "twiddle upload failed");
      if (nv == 0) {
        std::vector<uint2> l64 = thread_table<1024, 64>(iw, p, false);
        const size_t b64 = sizeof(uint2) * l64.size();
        e1 = cudaMalloc(&st.lane_inv64[pr], b64);
        if (e1 == cudaSuccess) e1 = cudaMemcpy(st.lane_inv64[pr], l64.data(), b64, cudaMemcpyHostToDevice);
        if (e1 != cudaSuccess) return fail(HWB_ECUDA, "twiddle upload failed");
      }
      // Montgomery form with N^-1: x -> x * R * N^-1 via mont_mul(x, R^2 N^-1)
      uint64_t R = ((uint64_t)1 << 32) % p;
      uint64_t r2 = R * R % p;
      uint64_t ninv = powmod(N, p - 2, p);
      h_r2ninv[nv][pr] = (uint32_t)(r2 * ninv % p);
    }
  }
  const uint32_t crt_inv = powmod(kP0, kP1 - 2, kP1);
  const uint2 crt_pair = shoup_pair(crt_inv, kP1);
  uint32_t h_crt[4] = {crt_pair.x, crt_pair.y, (uint32_t)((uint64_t)kP0 * kP1), kP1 / 2};
  {
    const std::vector<double2> wf = fft_twiddles(false), wi = fft_twiddles(true);
    const std::vector<double2> lf = thread_table_of<FH, FT, double2>([&](int k) { return wf[k]; }, true);
    const std::vector<double2> li = thread_table_of<FH, FT, double2>([&](int k) { return wi[k]; }, false);
    const size_t fb = sizeof(double2) * lf.size();
    cudaError_t e1 = cudaMalloc(&st.fft_fwd, fb), e2 = cudaMalloc(&st.fft_inv, fb);
    if (e1 == cudaSuccess) e1 = cudaMemcpy(st.fft_fwd, lf.data(), fb, cudaMemcpyHostToDevice);
    if (e2 == cudaSuccess) e2 = cudaMemcpy(st.fft_inv, li.data(), fb, cudaMemcpyHostToDevice);
    double2 h_ftw[3][2][8];
    for (int k = 0; k < 8; ++k) {
      h_ftw[0][0][k] = wf[k];
      h_ftw[0][1][k] = wi[k];
    }
    {   // wide-thread transform (hwb_fft.cuh: fwd_fft16 / inv_fft16)
      std::vector<double2> w16(2 * kW16Tab);
      double2 h_w16[2][16];
      for (int d = 0; d < 2; ++d) {
        const std::vector<double2> &w = d == 0 ? wf : wi;
        double2 *tab = w16.data() + d * kW16Tab;
        for (int v = 0; v < 16; ++v) {
          tab[0 * 16 + v] = w[16 + v];                                              // level 4, block v
          tab[1 * 16 + v] = w[32 + 2 * v];                                          // level 5, block 2 v
          for (int b = 0; b < 2; ++b) tab[(2 + b) * 16 + v] = w[64 + 4 * v + 2 * b];    // level 6
          for (int b = 0; b < 4; ++b) tab[(4 + b) * 16 + v] = w[128 + 8 * v + 2 * b];   // level 7
        }
        for (int b = 0; b < 4; ++b)
          for (int uu = 0; uu < WT; ++uu) tab[kW16Twm + b * WT + uu] = w[256 + 8 * uu + 2 * b];   // level 8
        for (int k = 0; k < 16; ++k) h_w16[d][k] = w[k];
      }
      if (e1 == cudaSuccess) e1 = cudaMalloc(&st.fft_w16, sizeof(double2) * w16.size());
      if (e1 == cudaSuccess)
        e1 = cudaMemcpy(st.fft_w16, w16.data(), sizeof(double2) * w16.size(), cudaMemcpyHostToDevice);
      if (e1 == cudaSuccess) e1 = cudaMemcpyToSymbol(c_w16, h_w16, sizeof(h_w16));
    }
    // N = 2048 (FFT2): the 1024-point folded transform's first stage (level 0,
    // twiddle k = 1) is done by hand; half g is a 512-point transform whose local
    // twiddle k' = 2^l' + m' is the full one at level l' + 1, block g 2^l' + m'
    const std::vector<double2> wf2 = fft_twiddles(false, 2 * FH), wi2 = fft_twiddles(true, 2 * FH);
    auto sub = [](const std::vector<double2> &w, int g, int k) {
      if (k == 0) return w[0];
      int lv = 0;
      while ((2 << lv) <= k) ++lv;
      return w[k + (1 + g) * (1 << lv)];
    };
    for (int g = 0; g < 2 && e1 == cudaSuccess && e2 == cudaSuccess; ++g) {
      const std::vector<double2> gf = thread_table_of<FH, FT, double2>([&](int k) { return sub(wf2, g, k); }, true);
      const std::vector<double2> gi = thread_table_of<FH, FT, double2>([&](int k) { return sub(wi2, g, k); }, false);
      e1 = cudaMalloc(&st.fft2_fwd[g], fb);
      e2 = cudaMalloc(&st.fft2_inv[g], fb);
      if (e1 == cudaSuccess) e1 = cudaMemcpy(st.fft2_fwd[g], gf.data(), fb, cudaMemcpyHostToDevice);
      if (e2 == cudaSuccess) e2 = cudaMemcpy(st.fft2_inv[g], gi.data(), fb, cudaMemcpyHostToDevice);
      for (int k = 0; k < 8; ++k) {
        h_ftw[1 + g][0][k] = sub(wf2, g, k);
        h_ftw[1 + g][1][k] = sub(wi2, g, k);
      }
    }
    const double2 w0[2] = {wf2[1], wi2[1]};   // level-0 twiddle (forward tangent form, inverse conjugate)
    if (e1 == cudaSuccess && e2 == cudaSuccess) e1 = cudaMemcpyToSymbol(c_fw0, w0, sizeof(w0));
    if (e1 == cudaSuccess && e2 == cudaSuccess) e1 = cudaMemcpyToSymbol(c_ftw, h_ftw, sizeof(h_ftw));
    if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(HWB_ECUDA, "FFT twiddle upload failed");
  }
  const uint32_t zero = 0;
  cudaError_t ec = cudaMemcpyToSymbol(c_tw, h_tw, sizeof(h_tw));
  if (ec == cudaSuccess) ec = cudaMemcpyToSymbol(c_zero, &zero, sizeof(zero));
  if (ec == cudaSuccess) ec = cudaMemcpyToSymbol(c_prime, h_prime, sizeof(h_prime));
  if (ec == cudaSuccess) ec = cudaMemcpyToSymbol(c_crt, h_crt, sizeof(h_crt));
  if (ec == cudaSuccess) ec = cudaMemcpyToSymbol(c_r2ninv, h_r2ninv, sizeof(h_r2ninv));
  if (ec != cudaSuccess) return fail(HWB_ECUDA, std::string("constant upload: ") + cudaGetErrorString(ec));
  st.ready = true;
  *out = &st;
  return HWB_OK;
}

// ---------------------------------------------------------------------------
// kernels

template <int N>
struct Smem {
  uint32_t acc[2 * N];   // working ciphertext (a, b)
  uint32_t v[2 * N];     // decomposition-ready input; then the residue exchange
  uint32_t scr[2][N];    // per-group transpose scratch
};

struct Tw {
  const uint2 *fwd[2];
  const uint2 *inv[2];
  const uint2 *inv64[2];   // N = 1024, 64 threads per transform
};

// Thread coordinates inside a ciphertext CTA.
template <int N>
struct Who {
  static constexpr int TPP = Cfg<N>::TPP;
  int tid, grp, t;
  LayBase lay;
  __device__ __forceinline__ Who() : tid(threadIdx.x), grp(threadIdx.x / TPP), t(threadIdx.x % TPP) {
    lay = make_lay<N, TPP>(t);
  }
};

// One external product for the CTA's item.  Pre: sm.v holds decomp_prep() of
// the input (both components) and a barrier has passed.  Post (after the
// internal barriers): x holds, in layout A, the canonical residues mod p_grp of
// component grp, and sm.v[grp*N + i] holds those mod p_{1-grp} of component grp.
template <int N, int PRIME, bool PF>
__device__ __forceinline__ void ext_product_core_p(Smem<N> &sm, const uint32_t *__restrict__ G, const Gadget &g,
                                                   const Who<N> &me, const Tw &tw, uint32_t (&x)[N / Cfg<N>::TPP],
                                                   const uint32_t *Gnext) {
  constexpr int TPP = Cfg<N>::TPP;
  constexpr int C = N / TPP;
  const int w = PRIME >= 0 ? PRIME : me.grp;
  const int t = me.t;
  const uint32_t p = PRIME >= 0 ? (PRIME ? kP1 : kP0) : c_prime[w].p, two_p = 2 * p;
  const uint32_t pinv = c_prime[w].pinv;
  const uint32_t off = p - g.half;
  const int L = (int)g.levels;
  const uint2 *twf = w ? tw.fwd[1] : tw.fwd[0];
  const uint2 *twi = w ? tw.inv[1] : tw.inv[0];
  uint32_t a0[C], a1[C];
#pragma unroll
  for (int j = 0; j < C; ++j) a0[j] = a1[j] = 0;

#pragma unroll 1
  for (int r = 0; r < 2 * L; ++r) {
    // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
    const int comp = r < L ? 1 : 0;
    const int tt = r < L ? r : r - L;
    const uint32_t sh = g.base_log * (uint32_t)(L - 1 - tt);
    const uint32_t *vs = sm.v + comp * N + t;
    {   // prefetch the GGSW rows the next digit (or the next step's first digit)
        // multiplies by while this digit's transform runs: per-item GGSWs come
        // from HBM, not L2 (rotation ladders of vertical packing, IVP levels)
      const uint32_t *gn = r + 1 < 2 * L ? G + (size_t)(r + 1) * 4 * N : Gnext;
      if (PF && gn) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int q = t; q < N / 32; q += TPP) prefetch_l2(gn + ((size_t)c * 2 + w) * N + q * 32);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) x[j] = ((vs[TPP * j] >> sh) & g.mask) + off;
    fwd_ntt<N, TPP, PRIME>(x, sm.scr[w], me.lay, t, w, twf);
    const uint32_t *g0 = G + ((size_t)(r * 2 + 0) * 2 + w) * N;
    const uint32_t *g1 = G + ((size_t)(r * 2 + 1) * 2 + w) * N;
#pragma unroll
    for (int jq = 0; jq < C / 4; ++jq) {
      const uint4 G0 = __ldg(slice_vec<TPP>(g0, t, jq));
      const uint4 G1 = __ldg(slice_vec<TPP>(g1, t, jq));
      a0[4 * jq + 0] += mont_mul(x[4 * jq + 0], G0.x, p, pinv);
      a0[4 * jq + 1] += mont_mul(x[4 * jq + 1], G0.y, p, pinv);
      a0[4 * jq + 2] += mont_mul(x[4 * jq + 2], G0.z, p, pinv);
      a0[4 * jq + 3] += mont_mul(x[4 * jq + 3], G0.w, p, pinv);
      a1[4 * jq + 0] += mont_mul(x[4 * jq + 0], G1.x, p, pinv);
      a1[4 * jq + 1] += mont_mul(x[4 * jq + 1], G1.y, p, pinv);
      a1[4 * jq + 2] += mont_mul(x[4 * jq + 2], G1.z, p, pinv);
      a1[4 * jq + 3] += mont_mul(x[4 * jq + 3], G1.w, p, pinv);
    }
  }
  // 2l <= 6 terms in (0, 2p): sums < 12p < 2^32; reduce to [0, 2p)
#pragma unroll
  for (int j = 0; j < C; ++j) {
    uint32_t u = a0[j], v = a1[j];
    u = umin(u, u - 4 * two_p); v = umin(v, v - 4 * two_p);
    u = umin(u, u - 2 * two_p); v = umin(v, v - 2 * two_p);
    u = umin(u, u - two_p);     v = umin(v, v - two_p);
    a0[j] = u; a1[j] = v;
  }
  __syncthreads();   // both groups are done reading sm.v: it becomes the exchange buffer
#pragma unroll 1
  for (int it = 0; it < 2; ++it) {
    const int c = it == 0 ? 1 - w : w;
#pragma unroll
    for (int j = 0; j < C; ++j) x[j] = c ? a1[j] : a0[j];
    inv_ntt<N, TPP, PRIME>(x, sm.scr[w], me.lay, t, w, twi);
#pragma unroll
    for (int j = 0; j < C; ++j) x[j] = umin(x[j], x[j] - p);
    if (it == 0) {
#pragma unroll
      for (int j = 0; j < C; ++j) sm.v[c * N + t + TPP * j] = x[j];
    }
  }
  __syncthreads();   // exchange complete
}

// SPEC: each group runs its own instantiation (the prime, hence every uniform
// twiddle and modulus, is a compile-time constant); otherwise one shared copy.
template <int N, bool SPEC, bool PF = true>
__device__ __forceinline__ void ext_product_core(Smem<N> &sm, const uint32_t *__restrict__ G, const Gadget &g,
                                                 const Who<N> &me, const Tw &tw, uint32_t (&x)[N / Cfg<N>::TPP],
                                                 const uint32_t *Gnext = nullptr) {
  if (!SPEC)
    ext_product_core_p<N, -1, PF>(sm, G, g, me, tw, x, Gnext);
  else if (me.grp == 0)
    ext_product_core_p<N, 0, PF>(sm, G, g, me, tw, x, Gnext);
  else
    ext_product_core_p<N, 1, PF>(sm, G, g, me, tw, x, Gnext);
}

__device__ __forceinline__ uint32_t lift(int w, uint32_t own, uint32_t other) {
  return w == 0 ? crt_lift(own, other) : crt_lift(other, own);
}

// negacyclic rotation read: (x * X^e)[i] with e in [0, 2N)
template <int N>
__device__ __forceinline__ uint32_t rot_read(const uint32_t *poly, int i, int e) {
  const int src = (i - e) & (2 * N - 1);
  const uint32_t val = poly[src & (N - 1)];
  return src >= N ? 0u - val : val;
}

// MODE_IVP_LEVEL / MODE_VP_LEVEL process one level of the inverse / forward
// vertical-packing tree (hw/lut.py:294-313 / 233-247) for B items of m (resp.
// 2m) polynomials each; block = item*m + sub, the GGSW is per item.
enum { MODE_EXT = 0, MODE_CMUX = 1, MODE_CDEMUX = 2, MODE_IVP_LEVEL = 3, MODE_VP_LEVEL = 4 };

template <int N, int MODE, int V>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::minb(V))
    cmux_kernel(const uint32_t *__restrict__ ggsw, size_t ggsw_words, const int32_t *__restrict__ gidx,
                const uint32_t *in, const uint32_t *c1, const int32_t *__restrict__ rot, uint32_t *out,
                uint32_t *out_hi, int m, Gadget g, Tw tw) {
  constexpr int TPP = Cfg<N>::TPP, NT = Cfg<N>::THREADS;
  constexpr bool LEVEL = MODE == MODE_IVP_LEVEL || MODE == MODE_VP_LEVEL;
  constexpr bool MUX = MODE == MODE_CMUX || MODE == MODE_VP_LEVEL;
  extern __shared__ uint4 smem_raw[];
  Smem<N> &sm = *reinterpret_cast<Smem<N> *>(smem_raw);
  const int64_t b = blockIdx.x;
  const int64_t item = LEVEL ? b / m : b, sub = LEVEL ? b % m : 0;
  const Who<N> me;
  const int tid = me.tid;
  const uint32_t *G = ggsw + (size_t)(gidx ? gidx[item] : 0) * ggsw_words;
  // operand / result addresses (see the mode comment above)
  const uint32_t *src = in + (MODE == MODE_VP_LEVEL ? (item * 2 * m + sub) : b) * 2 * N;
  const uint32_t *s1 = MODE == MODE_VP_LEVEL ? in + (item * 2 * m + m + sub) * 2 * N : (c1 ? c1 + b * 2 * N : nullptr);
  uint32_t *o_lo = out + (MODE == MODE_IVP_LEVEL ? (item * 2 * m + sub) : b) * 2 * N;
  uint32_t *o_hi = MODE == MODE_IVP_LEVEL ? out + (item * 2 * m + m + sub) * 2 * N : (out_hi ? out_hi + b * 2 * N : nullptr);
  if (MODE == MODE_EXT) {
    for (int k = tid; k < 2 * N; k += NT) sm.v[k] = decomp_prep(src[k], g);
  } else {
    for (int k = tid; k < 2 * N; k += NT) sm.acc[k] = src[k];
    __syncthreads();
    if (MUX) {
      if (s1) {
        for (int k = tid; k < 2 * N; k += NT) sm.v[k] = decomp_prep(s1[k] - sm.acc[k], g);
      } else {
        const int e = ((rot[b] % (2 * N)) + 2 * N) % (2 * N);
        for (int k = tid; k < 2 * N; k += NT) {
          const int c = k >= N, i = k & (N - 1);
          sm.v[k] = decomp_prep(rot_read<N>(sm.acc + c * N, i, e) - sm.acc[k], g);
        }
      }
    } else {
      for (int k = tid; k < 2 * N; k += NT) sm.v[k] = decomp_prep(sm.acc[k], g);
    }
  }
  __syncthreads();
  uint32_t x[N / TPP];
  ext_product_core<N, Cfg<N>::spec(V)>(sm, G, g, me, tw, x);
  const int w = me.grp;
#pragma unroll
  for (int j = 0; j < N / TPP; ++j) {
    const int i = w * N + me.t + TPP * j;
    const uint32_t val = lift(w, x[j], sm.v[i]);
    if (MODE == MODE_EXT) {
      o_lo[i] = val;
    } else if (MUX) {
      o_lo[i] = sm.acc[i] + val;
    } else {
      o_hi[i] = val;
      o_lo[i] = sm.acc[i] - val;
    }
  }
}

// dst[k] += sum_{i < count} src[i * words + k] mod 2^32: the rows of `count`
// samples added into the model in one pass (hw/hewnn.py:213).
__global__ void accumulate_rows_kernel(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, int64_t words,
                                       int count) {
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k >= words) return;
  if (k + 4 <= words && (words & 3) == 0) {
    uint4 acc = *reinterpret_cast<const uint4 *>(dst + k);
    for (int i = 0; i < count; ++i) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src + (int64_t)i * words + k));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    *reinterpret_cast<uint4 *>(dst + k) = acc;
  } else {
    for (int64_t kk = k; kk < k + 4 && kk < words; ++kk) {
      uint32_t a = dst[kk];
      for (int i = 0; i < count; ++i) a += src[(int64_t)i * words + kk];
      dst[kk] = a;
    }
  }
}

// x_b * X^(e_b) per item (hw/lut.py:317-325), e_b taken mod 2N; in may not alias out.
template <int N>
__global__ void monomial_gather_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                       const int32_t *__restrict__ exps, int64_t B) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * 2 * N) return;
  const int64_t b = idx / (2 * N);
  const int k = (int)(idx % (2 * N));
  const int e = ((exps[b] % (2 * N)) + 2 * N) % (2 * N);
  const int c = k >= N, i = k & (N - 1);
  out[idx] = rot_read<N>(in + b * 2 * N + c * N, i, e);
}

// dst[k] += sign * src[k] mod 2^32 (exact ring addition for model accumulation,
// hw/hewnn.py:213, 264-271); src is indexed k mod src_words (broadcast rows).
__global__ void accumulate_kernel(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, int64_t words,
                                  int64_t src_words, int negate) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= words) return;
  const uint32_t v = src[k % src_words];
  dst[k] += negate ? 0u - v : v;
}

// LWE linear combination (the affine steps between bootstraps of the PBS inference
// pipeline): out[b][k] = ((cx[b] x[b][k] + cy[b] y[b][k]) << shift) + [k == W-1] cb[b]
// mod 2^32; a NULL multiplier is 1 (cx) or 0 (y NULL), a NULL constant 0.
__global__ void lwe_lincomb_kernel(const uint32_t *__restrict__ x, const uint32_t *__restrict__ y,
                                   uint32_t *__restrict__ out, const int32_t *__restrict__ cx,
                                   const int32_t *__restrict__ cy, const uint32_t *__restrict__ cb, int64_t B,
                                   int32_t W, int32_t shift) {
  const int64_t b = blockIdx.y * (int64_t)gridDim.z + blockIdx.z;
  if (b >= B) return;
  const uint32_t mx = cx ? (uint32_t)cx[b] : 1u, my = cy ? (uint32_t)cy[b] : 0u;
  const uint32_t c = cb ? cb[b] : 0u;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < W; k += gridDim.x * blockDim.x) {
    uint32_t v = mx * x[b * W + k];
    if (y) v += my * y[b * W + k];
    v <<= shift;
    if (k == W - 1) v += c;
    out[b * W + k] = v;
  }
}

// out[b] = table[idx[b]] (rows of `row_words` words): per-item test polynomials
// drawn from a small table of LUTs.
__global__ void gather_rows_kernel(const uint32_t *__restrict__ table, const int32_t *__restrict__ idx,
                                   uint32_t *__restrict__ out, int64_t B, int32_t row_words) {
  const int64_t b = blockIdx.y * (int64_t)gridDim.z + blockIdx.z;
  if (b >= B) return;
  const uint4 *src = reinterpret_cast<const uint4 *>(table + (int64_t)idx[b] * row_words);
  uint4 *dst = reinterpret_cast<uint4 *>(out + b * row_words);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < row_words / 4; k += gridDim.x * blockDim.x) dst[k] = src[k];
}

// numpy's Philox4x64-10 (Random123 rounds; numpy/random/src/philox): block g of a draw
// is philox(ctr + 1 + g, key) -- numpy increments the counter before each block --
// and its 4 uint64 outputs give the uint32 stream low half, high half (next_uint32).
// Generator.bytes(4 n) is that uint32 stream (hw/tfhe.py:38-40 uniform_u64 at 4-byte
// words).  `prefix` holds the words still buffered in the host generator.
__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c[0], hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c[0]);
    const uint64_t lo1 = 0xCA5A826395121157ull * c[2], hi1 = __umul64hi(0xCA5A826395121157ull, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// out[r][0][j] = word r N + j of the stream (prefix words first), out[r][1][j] = b[r][j]:
// the RGSW rows of enc_rgsw_batch (a drawn by rng.bytes, hw/tfhe.py:246-263) rebuilt
// from the generator state and the shipped b half.
__global__ void philox_rgsw_kernel(hwb_philox st, const uint32_t *__restrict__ b_rows,
                                   const uint32_t *__restrict__ a0fix, int32_t levels, uint32_t *__restrict__ out,
                                   int64_t rows, int32_t N, int32_t pair) {
  const int64_t rs = pair ? 2 * (int64_t)N : N;     // row stride of out
  const int64_t nwords = rows * N;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nblocks = (nwords - st.nprefix + 7) / 8;
  if (g < nblocks) {
    uint64_t c[4];
    const uint64_t add = (uint64_t)g + 1;
    c[0] = st.ctr[0] + add;
    uint64_t carry = c[0] < add;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      c[i] = st.ctr[i] + carry;
      carry = carry && c[i] == 0;
    }
    philox4x64_10(c, st.key[0], st.key[1]);
    // rows l..2l-1 of each RGSW carry the gadget term m g_t on a[0] (hw/tfhe.py:259-262):
    // those words ship explicitly (a0fix [rows / 2l][l]) and are written instead of the
    // regenerated ones (by the thread that owns the word: no second writer)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t w = st.nprefix + 8 * g + q;
      if (w < nwords) {
        const uint64_t u = c[q >> 1];
        const int64_t r = w / N, col = w % N;
        uint32_t v = (q & 1) ? (uint32_t)(u >> 32) : (uint32_t)u;
        if (a0fix && col == 0 && (r % (2 * levels)) >= levels)
          v = a0fix[(r / (2 * levels)) * levels + (r % (2 * levels)) - levels];
        out[r * rs + col] = v;
      }
    }
  }
  if (g < st.nprefix && g < nwords) {
    const int64_t r = g / N, col = g % N;
    uint32_t v = st.prefix[g];
    if (a0fix && col == 0 && (r % (2 * levels)) >= levels)
      v = a0fix[(r / (2 * levels)) * levels + (r % (2 * levels)) - levels];
    out[r * rs + col] = v;
  }
  if (b_rows && pair)
    for (int64_t w = g; w < nwords; w += (int64_t)gridDim.x * blockDim.x) out[(w / N) * 2 * N + N + w % N] = b_rows[w];
}

__device__ __forceinline__ int mod_switch(uint32_t x, int log2m) {
  return (int)((x + (1u << (31 - log2m))) >> (32 - log2m));
}

// Fused blind rotation.  PBS = false: acc_io [B][2][N] in/out, exps [B][L] are
// the reference's I values (rotation X^-I); step s uses GGSW s of `bsk`, or,
// with gidx [B][L], GGSW gidx[b][s] (< 0: the step is skipped) -- the per-item
// CMUX ladders of vertical packing (hw/lut.py:249-260, 280-291).  PBS = true:
// lwe_in [B][L+1]; acc = TV * X^-b~, rotation X^{a~_i} (I_i = -a~_i), output the
// coefficient-0 extraction [B][N+1].
template <int N, bool PBS, int V>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::minb(V))
    blind_rotate_kernel(const uint32_t *__restrict__ bsk, size_t ggsw_words, const int32_t *__restrict__ gidx,
                        const int32_t *__restrict__ exps, const uint32_t *__restrict__ lwe_in,
                        const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *acc_io, uint32_t *lwe_out, int L,
                        Gadget g, Tw tw) {
  constexpr int TPP = Cfg<N>::TPP, NT = Cfg<N>::THREADS;
  extern __shared__ uint4 smem_raw[];
  Smem<N> &sm = *reinterpret_cast<Smem<N> *>(smem_raw);
  constexpr int LOG2M = (N == 1024) ? 11 : 12;
  const int64_t b = blockIdx.x;
  const Who<N> me;
  const int tid = me.tid, w = me.grp;
  const uint32_t *row = PBS ? lwe_in + b * (int64_t)(L + 1) : nullptr;
  if (PBS) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      sm.acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = tid; k < 2 * N; k += NT) sm.acc[k] = acc_io[b * 2 * N + k];
  }
  __syncthreads();
  uint32_t x[N / TPP];
#pragma unroll 1
  for (int s = 0; s < L; ++s) {
    int e;
    if (PBS) {
      e = mod_switch(row[s], LOG2M);   // X^{a~_s}
    } else {
      e = (int)((-(int64_t)exps[b * L + s]) % (2 * N));
      if (e < 0) e += 2 * N;
    }
    if (e == 0) continue;   // zero difference -> zero product: exact skip
    int gi = s;
    if (!PBS && gidx) {
      gi = gidx[b * L + s];
      if (gi < 0) continue;   // clear selector bit: handled by the caller
    }
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      sm.v[k] = decomp_prep(rot_read<N>(sm.acc + c * N, i, e) - sm.acc[k], g);
    }
    __syncthreads();
    const uint32_t *gnext = nullptr;
    if (s + 1 < L) {
      const int gn = (!PBS && gidx) ? gidx[b * L + s + 1] : s + 1;
      if (gn >= 0) gnext = bsk + (size_t)gn * ggsw_words;
    }
    // prefetching pays for per-item GGSWs (HBM); the PBS key is L2-resident
    ext_product_core<N, Cfg<N>::spec(V), !PBS>(sm, bsk + (size_t)gi * ggsw_words, g, me, tw, x, gnext);
#pragma unroll
    for (int j = 0; j < N / TPP; ++j) {
      const int i = me.t + TPP * j;
      sm.acc[w * N + i] += lift(w, x[j], sm.v[w * N + i]);
    }
    __syncthreads();
  }
  if (PBS) {
    uint32_t *o = lwe_out + b * (int64_t)(N + 1);
    for (int k = tid; k < N; k += NT) o[k] = k == 0 ? sm.acc[0] : 0u - sm.acc[N - k];
    if (tid == 0) o[N] = sm.acc[N];
  } else {
    for (int k = tid; k < 2 * N; k += NT) acc_io[b * 2 * N + k] = sm.acc[k];
  }
}

// Latency-mode ladder (small batches): one ciphertext per CTA of 4*LV warps, one
// warp per (digit row r, prime w).  Same arithmetic and bit-exact results as
// blind_rotate_kernel; each CMUX step runs as
//   (a) all threads: v = decomp_prep(acc * X^e - acc)
//   (b) warp (r, w): forward NTT of digit r mod p_w, Montgomery products with the
//       GGSW row r, red.shared.add into the spectra accumulators macc[c][w]
//       (<= 2l terms in (0, 2p): sums < 12p < 2^32)
//   (c) warps (c, w), c, w in {0,1}: reduce, inverse NTT, canonical residues
//   (d) all threads: acc += CRT(macc[c][0], macc[c][1]); macc = 0
// so the 12 forward transforms of a step run concurrently on 12 warps instead of
// 6 + 6 sequentially on 2 -- a single PBS finishes ~3x sooner.
template <int N, int LV>
struct SmemLat {
  uint32_t acc[2 * N];
  uint32_t v[2 * N];
  uint32_t macc[2][2][N];          // [component][prime], NTT domain
  uint32_t scr[4 * LV][N];         // per-warp transpose scratch
};

// MINB = resident CTAs per SM the build targets: 1 (168 registers, lowest
// single-ciphertext latency) or 2 (80 registers, higher per-SM throughput).
template <int N, int LV, bool PBS, int MINB>
__global__ void __launch_bounds__(128 * LV, MINB)
    blind_rotate_lat_kernel(const uint32_t *__restrict__ bsk, size_t ggsw_words,
                            const int32_t *__restrict__ exps, const uint32_t *__restrict__ lwe_in,
                            const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *acc_io, uint32_t *lwe_out,
                            int L, Gadget g, Tw tw) {
  static_assert(N == 1024, "latency mode: one warp per transform (TPP = 32)");
  constexpr int TPP = 32, C = N / TPP, NT = 128 * LV;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  SmemLat<N, LV> &sm = *reinterpret_cast<SmemLat<N, LV> *>(smem_raw);
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, wi = tid >> 5, t = tid & 31;
  const int w = wi & 1, r = wi >> 1;                 // forward phase: digit row r, prime w
  const LayBase lay = make_lay<N, TPP>(t);
  const uint32_t p = c_prime[w].p, pinv = c_prime[w].pinv;
  const uint32_t off = p - g.half;
  const uint32_t *row = PBS ? lwe_in + b * (int64_t)(L + 1) : nullptr;
  if (PBS) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      sm.acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = tid; k < 2 * N; k += NT) sm.acc[k] = acc_io[b * 2 * N + k];
  }
  for (int k = tid; k < 4 * N; k += NT) (&sm.macc[0][0][0])[k] = 0u;
  __syncthreads();
  uint32_t x[C];
#pragma unroll 1
  for (int s = 0; s < L; ++s) {
    int e;
    if (PBS) {
      e = mod_switch(row[s], LOG2M);
    } else {
      e = (int)((-(int64_t)exps[b * L + s]) % (2 * N));
      if (e < 0) e += 2 * N;
    }
    if (e == 0) continue;
    // (a)
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      sm.v[k] = decomp_prep(rot_read<N>(sm.acc + c * N, i, e) - sm.acc[k], g);
    }
    __syncthreads();
    const uint32_t *G = bsk + (size_t)s * ggsw_words;
    if (r < 2 * LV && r < 2 * (int)g.levels) {
      // (b) digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < (int)g.levels ? 1 : 0;
      const int tt = r < (int)g.levels ? r : r - (int)g.levels;
      const uint32_t sh = g.base_log * (uint32_t)((int)g.levels - 1 - tt);
      const uint32_t *vs = sm.v + comp * N + t;
#pragma unroll
      for (int c = 0; c < 2; ++c) prefetch_l2(G + ((size_t)(r * 2 + c) * 2 + w) * N + t * 32);
#pragma unroll
      for (int j = 0; j < C; ++j) x[j] = ((vs[TPP * j] >> sh) & g.mask) + off HWB_Z;
      fwd_ntt<N, TPP, -1>(x, sm.scr[wi], lay, t, w, w ? tw.fwd[1] : tw.fwd[0]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t *gs = G + ((size_t)(r * 2 + c) * 2 + w) * N;
        uint32_t *dst = sm.macc[c][w];
#pragma unroll
        for (int jq = 0; jq < C / 4; ++jq) {
          const uint4 Gv = __ldg(slice_vec<TPP>(gs, t, jq));
          uint32_t *d = dst + jq * 4 * TPP + t;      // element k of lane t at k*32 + t: conflict-free
          atomicAdd(d + 0 * TPP, mont_mul(x[4 * jq + 0], Gv.x, p, pinv));
          atomicAdd(d + 1 * TPP, mont_mul(x[4 * jq + 1], Gv.y, p, pinv));
          atomicAdd(d + 2 * TPP, mont_mul(x[4 * jq + 2], Gv.z, p, pinv));
          atomicAdd(d + 3 * TPP, mont_mul(x[4 * jq + 3], Gv.w, p, pinv));
        }
      }
    }
    __syncthreads();
    if (LV >= 2 && MINB == 1) {
      // (c) 8 warps: warp pair q = (component q >> 1, prime q & 1) shares one
      // inverse transform on 64 threads (named barrier 1 + q).  (The 2-CTA/SM
      // build keeps 4 warps: there the other CTA fills the idle slots.)
      if (wi < 8) {
        constexpr int T2 = 64, C2 = N / T2;
        const int q = wi >> 1, c = q >> 1, w2 = q & 1, t2 = ((wi & 1) << 5) | t;
        const uint32_t p2 = c_prime[w2].p, two_p2 = 2 * p2;
        uint32_t *src = sm.macc[c][w2];
        uint32_t y[C2];
#pragma unroll
        for (int j = 0; j < C2; ++j) {
          // layout-B index i = C2*t2 + j of the 64-thread transform; the spectra were
          // accumulated in the 32-thread order: (t32, j32) = (i / 32, i % 32) at
          // (j32 / 4) * 128 + (j32 % 4) * 32 + t32
          const int i = C2 * t2 + j, j32 = i & 31, t32 = i >> 5;
          uint32_t u = src[(j32 >> 2) * 128 + (j32 & 3) * 32 + t32];
          u = umin(u, u - 4 * two_p2);
          u = umin(u, u - 2 * two_p2);
          u = umin(u, u - two_p2);
          y[j] = u;
        }
        const LayBase lay2 = make_lay<N, T2>(t2);
        inv_ntt<N, T2, -1>(y, sm.scr[2 * q], lay2, t2, w2, tw.inv64[w2], q);
#pragma unroll
        for (int j = 0; j < C2; ++j) src[t2 + T2 * j] = umin(y[j], y[j] - p2);
      }
    } else if (wi < 4) {
      // (c) component c = wi >> 1, prime w
      const int c = wi >> 1;
      uint32_t *src = sm.macc[c][w];
      const uint32_t two_p = 2 * p;
#pragma unroll
      for (int j = 0; j < C; ++j) x[j] = src[j * TPP + t];
#pragma unroll
      for (int j = 0; j < C; ++j) {
        uint32_t u = x[j];
        u = umin(u, u - 4 * two_p);
        u = umin(u, u - 2 * two_p);
        u = umin(u, u - two_p);
        x[j] = u;
      }
      inv_ntt<N, TPP, -1>(x, sm.scr[wi], lay, t, w, w ? tw.inv[1] : tw.inv[0]);
#pragma unroll
      for (int j = 0; j < C; ++j) src[t + TPP * j] = umin(x[j], x[j] - p);
    }
    __syncthreads();
    // (d)
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      sm.acc[k] = sm.acc[k] + crt_lift(sm.macc[c][0][i], sm.macc[c][1][i]) HWB_Z;
      sm.macc[c][0][i] = 0u;
      sm.macc[c][1][i] = 0u;
    }
    __syncthreads();
  }
  if (PBS) {
    uint32_t *o = lwe_out + b * (int64_t)(N + 1);
    for (int k = tid; k < N; k += NT) o[k] = k == 0 ? sm.acc[0] : 0u - sm.acc[N - k];
    if (tid == 0) o[N] = sm.acc[N];
  } else {
    for (int k = tid; k < 2 * N; k += NT) acc_io[b * 2 * N + k] = sm.acc[k];
  }
}

// ---------------------------------------------------------------------------
// FP64 FFT ladder (hwb_fft.cuh), N = 1024: one ciphertext per CTA of 64 threads.
// Thread t owns the spectrum positions (t, j) of layout B for every transform, so
// the 2l digit spectra are multiplied into the four accumulators Y[c][h] (component
// c, key half h) in registers, and after the inverse transforms each thread owns the
// coefficients i = t + 64 j and i + 512 of both halves: no exchange between threads.

// BSK [n][2l][2][N] u32 -> FFT domain [n][2l][2][2 halves][FC][FT] double2 (scaled 1/H).
__global__ void __launch_bounds__(FT) bsk_to_fft_kernel(const uint32_t *__restrict__ in, double2 *out,
                                                         const double2 *__restrict__ twf) {
  __shared__ double2 scr[2 * FH];
  const int t = threadIdx.x;
  const int64_t poly = blockIdx.x;
  const uint32_t *a = in + poly * (2 * FH);
  const FLay lay = make_flay(t);
  double2 x[2][FC];   // [half][j]: both halves transformed in lockstep
#pragma unroll
  for (int j = 0; j < FC; ++j) {
    const int i = t + FT * j;
    double lo[2], hi[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t gword = (int32_t)a[i + q * FH];               // signed 32-bit key word
      const int64_t l16 = ((gword + 32768) & 0xFFFF) - 32768;      // [-2^15, 2^15)
      lo[q] = (double)l16;
      hi[q] = (double)((gword - l16) >> 16);
    }
    x[0][j] = make_double2(lo[0], lo[1]);
    x[1][j] = make_double2(hi[0], hi[1]);
  }
  fwd_fft_k<2>(x, scr, lay, t, twf);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 *o = out + (poly * 2 + h) * (FC * FT);
#pragma unroll
    for (int j = 0; j < FC; ++j) o[j * FT + t] = make_double2(x[h][j].x * (1.0 / FH), x[h][j].y * (1.0 / FH));
  }
}

// CPB ciphertexts per CTA (64 threads each) share one staged key slice per digit:
// the slice is written into shared memory once and read CPB times.
#ifndef HWB_FFT_DIG
#define HWB_FFT_DIG 1
#endif
constexpr int FDR = 6;   // digit rows 2l staged per product (FFT path: l <= 3, byte digits)
// staging slots per thread: 2l rows of 16 byte digits (base_log <= 8).  Wide gadgets
// (base_log > 8) extract their digits on the fly instead: 8 slots would grow the CTA past
// the 4 CTAs/SM that the register ladder needs (measured: B = 592 at 13.9 vs 10.0 ms).
constexpr int FDS = FDR;
template <int CPB>
struct FSmemT {
  uint32_t acc[CPB][2 * 2 * FH];
  double2 scr[CPB][FH];
#if HWB_FFT_DIG
  uint4 dig[CPB][FDS * FT];       // the product's digits, biased bytes / halfwords [slot][thread]
#endif
  double2 key[2 * 2 * FC * FT];   // the current digit's key slice [c][h][j][t] (32 KB, TMA)
  uint64_t key_full;              // mbarrier: slice landed
};
using FSmem = FSmemT<1>;

// One exact external product on the FFT path for the CTA's item.  prep(c, i) gives
// the decomposition-ready value (decomp_prep) of component c, coefficient i; G is the
// item's GGSW in the FFT domain [2l rows][2 comps][2 halves][FC][FT]; sink(c, i, v)
// receives coefficient i of component c of the product for this thread's positions
// i = t + 64 j and i + 512 (every thread owns the same positions in all transforms,
// so no exchange is needed).  Each digit's 32 KB key slice is staged in shared
// memory by a TMA bulk copy issued after the digit transform's first barrier.
template <int CPB = 1, typename Prep, typename Sink>
__device__ __forceinline__ void fft_ext_product(FSmemT<CPB> &sm, const double2 *__restrict__ G, const Gadget &g,
                                                int t, const FLay &lay, const double2 *__restrict__ twf,
                                                const double2 *__restrict__ twi, uint32_t &key_phase, Prep &&prep,
                                                Sink &&sink, int grp = 0) {
  double2 *scr = sm.scr[grp];
  const int bar = CPB == 1 ? 0 : 1 + grp;
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;   // 2^52 + beta/2
#if HWB_FFT_DIG
  // The whole decomposition once per product: each prep word (rotation, difference,
  // rounding) is formed once and its l digits, biased into [0, beta), are stored as
  // bytes -- row r, thread t: 16 bytes, byte 2j + q for position t + 64 j + 512 q.
  // Each thread reads back only its own slots, so no barrier is needed.
  // Wide gadgets (base_log > 8, the full-precision 2 x 16 sets) skip the staging and
  // extract each row's digits from prep on the fly (below).
  uint4 *dig = sm.dig[grp];
  const bool wide = g.base_log > 8;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (wide) break;
    uint32_t pw[2 * FC];
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      pw[2 * j] = prep(c, t + FT * j);
      pw[2 * j + 1] = prep(c, t + FT * j + FH);
    }
    const uint32_t bmask = g.mask * 0x01010101u;
#pragma unroll 1
    for (int tt = 0; tt < lv; ++tt) {
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const int row = (c == 1 ? 0 : lv) + tt;
      uint32_t wd[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint32_t lo = __byte_perm(pw[4 * m] >> sh, pw[4 * m + 1] >> sh, 0x0040);
        const uint32_t hi = __byte_perm(pw[4 * m + 2] >> sh, pw[4 * m + 3] >> sh, 0x0040);
        wd[m] = __byte_perm(lo, hi, 0x5410) & bmask;
      }
      dig[row * FT + t] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
  }
#endif
  double2 Y[2][2][FC];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < FC; ++j) Y[c][h][j] = make_double2(0.0, 0.0);
#pragma unroll 1
  for (int r = 0; r < 2 * lv; ++r) {
    // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
    const double2 *gr = G + (size_t)r * (2 * 2 * FC * FT);
    double2 x[FC];
#if HWB_FFT_DIG
    if (wide) {
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        x[j] = make_double2(u2d_minus((prep(comp, i) >> sh) & g.mask, dig_off),
                            u2d_minus((prep(comp, i + FH) >> sh) & g.mask, dig_off));
      }
    } else {
      const uint4 dv = dig[r * FT + t];
      const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const uint32_t w = dw[j >> 1], k = 2 * (j & 1);
        x[j] = make_double2(u2d_minus(__byte_perm(w, 0, 0x4440 + k), dig_off),
                            u2d_minus(__byte_perm(w, 0, 0x4441 + k), dig_off));
      }
    }
#else
    const int comp = r < lv ? 1 : 0;
    const int tt = r < lv ? r : r - lv;
    const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const int i = t + FT * j;
      const uint32_t p0 = prep(comp, i), p1 = prep(comp, i + FH);
      x[j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
    }
#endif
    auto stage_key = [&] {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full, kSliceBytes);
        bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
      }
    };
    if (CPB == 1) {
      // issued after the transform's first barrier: every thread is past the MAC
      // that read the previous slice
      fwd_fft(x, scr, lay, t, twf, stage_key);
    } else {
      __syncthreads();   // all groups are past the previous slice's MAC
      stage_key();
      fwd_fft(x, scr, lay, t, twf, NoHook(), bar);
    }
    mbar_wait(&sm.key_full, key_phase);
    key_phase ^= 1u;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const double2 k = sm.key[((c * 2 + h) * FC + j) * FT + t];
          double2 &y = Y[c][h][j];
          y.x = fma(x[j].x, k.x, fma(-x[j].y, k.y, y.x));
          y.y = fma(x[j].x, k.y, fma(x[j].y, k.x, y.y));
        }
  }
  if (CPB == 1) {
    // the four inverse transforms in lockstep, their transposes in the (now idle)
    // key buffer
    __syncthreads();   // every thread has finished reading the last key slice
    inv_fft_k<4>(&Y[0][0], sm.key, lay, t, twi);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) inv_fft((&Y[0][0])[q], scr, lay, t, twi, bar);
  }
  // rounding and recombination of the halves
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const int i = t + FT * j;
      sink(c, i, round_u32(Y[c][0][j].x) + (round_u32(Y[c][1][j].x) << 16));
      sink(c, i + FH, round_u32(Y[c][0][j].y) + (round_u32(Y[c][1][j].y) << 16));
    }
}

__device__ __forceinline__ void fft_smem_init(FSmem &sm, int t) {
  if (t == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// The CMUX ladder on the FFT path.  PBS: lwe_in [B][L+1], the accumulator starts as
// TV * X^-b~ (at s0 == 0), rotation X^{a~_s} with GGSW s, coefficient-0 extraction
// at s1 == L; steps [s0, s1) per launch, the accumulator resting in acc_io between
// launches -- running the ladder in segments keeps the segment's slice of the FFT key
// (192 KB per step, 121 MB in all at cfg2) L2-resident for the whole batch.
// !PBS: acc_io [B][2][N] in/out, exps [B][L] (rotation X^-I), GGSW gidx[b][s] (< 0:
// skip) or s -- the per-item rotation ladders of vertical packing.
template <bool PBS, int CPB = 1>
__global__ void __launch_bounds__(FT * CPB, 1)
    blind_rotate_fft_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                            const int32_t *__restrict__ exps, const uint32_t *__restrict__ lwe_in,
                            const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                            const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                            int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemT<CPB> &sm = *reinterpret_cast<FSmemT<CPB> *>(smem_raw);
  const int grp = threadIdx.x / FT, t = threadIdx.x % FT;
  // groups past the end of the batch run a clamped copy of the last ciphertext (they
  // must take part in every CTA barrier) and write nothing
  const int64_t bb = (int64_t)blockIdx.x * CPB + grp;
  const bool valid = bb < B;
  const int64_t b = valid ? bb : B - 1;
  uint32_t *acc = sm.acc[grp];
  const FLay lay = make_flay(t);
  const uint32_t *row = PBS ? lwe_in + b * (int64_t)(L + 1) : nullptr;
  if (PBS && s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = t; k < 2 * N; k += FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = t; k < 2 * N; k += FT) acc[k] = acc_io[b * 2 * N + k];
  }
  if (threadIdx.x == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t key_phase = 0;
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;   // double2 per GGSW
  uint32_t a_nx = PBS ? row[s0] : 0u;   // the next step's mask word, loaded a step ahead
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    int e, gi = s;
    if (PBS) {
      e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
      a_nx = row[s + 1];
    } else {
      e = (int)((-(int64_t)exps[b * L + s]) % (2 * N));
      if (e < 0) e += 2 * N;
      if (gidx) gi = gidx[b * L + s];
    }
    if (CPB == 1 && (e == 0 || gi < 0)) continue;
    const bool skip = e == 0 || gi < 0;
    // (CPB > 1: every group runs the step -- the key slices and barriers are shared --
    // and a group whose step is an exact no-op discards the product)
    fft_ext_product<CPB>(
        sm, ggsw + (size_t)(gi < 0 ? 0 : gi) * ggsw_f, g, t, lay, twf, twi, key_phase,
        [&](int c, int i) {   // digits of (acc X^e - acc), straight from the accumulator
          const uint32_t *ac = acc + c * N;
          return decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
        },
        [&](int c, int i, uint32_t v) {
          if (!skip) acc[c * N + i] += v;
        },
        grp);
    if (CPB == 1)
      __syncthreads();
    else
      fsync(1 + grp);
  }
  if (!valid) return;
  if (!PBS || s1 < L) {
    for (int k = t; k < 2 * N; k += FT) acc_io[b * 2 * N + k] = acc[k];
    return;
  }
  uint32_t *o = lwe_out + b * (int64_t)(N + 1);
  for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
  if (t == 0) o[N] = acc[N];
}

// ---------------------------------------------------------------------------
// PBS ladder with the accumulators in tensor memory (TMEM).  The register ladder
// above keeps the four spectra accumulators Y[c][h] in registers (128 of 254), so
// each thread serves one ciphertext and every staged key value is read once per
// ciphertext.  Here they live in TMEM (2 KB per thread per ... 256 columns per
// 128-lane CTA; SIMT tcgen05.ld/st move 500-700 B/clk/SM, beside the shared-memory
// crossbar that bounds the ladder): each thread transforms the digits of TWO
// ciphertexts in lockstep and applies every key value it reads from shared memory
// to both, and one TMA-staged 32 KB key slice serves the CTA's four ciphertexts.
// Shared-memory bytes per ciphertext-step drop by the key share.
// TMEM layout: lane = threadIdx.x, columns ((q 2 + c) 2 + h) 32 + 4 j + {re.lo,
// re.hi, im.lo, im.hi} for ciphertext q in {0, 1} of the thread's group.

constexpr int TMC = 4;          // ciphertexts per CTA (2 groups x 2 per thread)
constexpr uint32_t TM_COLS = 256;

struct FSmemTM {
  uint32_t acc[TMC][2 * 2 * FH];
  double2 scr[2][2 * FH];         // forward scratch of group g (2 transforms); all 32 KB: group 1's inverse scratch
  double2 key[2 * 2 * FC * FT];   // the digit's key slice (TMA); group 0's inverse scratch
  uint64_t key_full;
  uint64_t in_full;               // level kernels: the inputs' bulk copies landed
  uint32_t tmem_slot;
};

__device__ __forceinline__ void tm_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(addr));
}
__device__ __forceinline__ void tm_st32(uint32_t addr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
               "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
               "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
               "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
               : "memory");
}
__device__ __forceinline__ void tm_st_f64(uint32_t addr, double v) {   // one double: 2 columns
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(__double2loint(v)),
               "r"(__double2hiint(v))
               : "memory");
}
__device__ __forceinline__ void tm_st_c64(uint32_t addr, double2 v) {   // one complex: 4 columns
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
#ifndef HWB_TM_ST4
#define HWB_TM_ST4 0
#endif
// store one complex accumulator value: x4 (one STTM) or two x2 halves
__device__ __forceinline__ void tm_st_acc(uint32_t addr, double2 v) {
#if HWB_TM_ST4
  tm_st_c64(addr, v);
#else
  tm_st_f64(addr, v.x);
  tm_st_f64(addr + 2, v.y);
#endif
}
__device__ __forceinline__ void tm_zero32(uint32_t addr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
               "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(0u)
               : "memory");
}
__device__ __forceinline__ double2 tm_get(const uint32_t (&r)[32], int j) {
  return make_double2(__hiloint2double((int)r[4 * j + 1], (int)r[4 * j]),
                      __hiloint2double((int)r[4 * j + 3], (int)r[4 * j + 2]));
}
__device__ __forceinline__ void tm_put(uint32_t (&r)[32], int j, double2 v) {
  r[4 * j] = (uint32_t)__double2loint(v.x);
  r[4 * j + 1] = (uint32_t)__double2hiint(v.x);
  r[4 * j + 2] = (uint32_t)__double2loint(v.y);
  r[4 * j + 3] = (uint32_t)__double2hiint(v.y);
}

// One external product per ciphertext for the CTA's four ciphertexts (thread group
// grp holds q = 0, 1), all against the same GGSW G: prep(q, c, i) gives the
// decomposition-ready word of component c, coefficient i; sink(q, c, i, v) receives
// the product's coefficients (i = t + 64 j and + 512).  The TMEM accumulators are
// zero on entry and left zero on exit.
template <typename Prep, typename Sink>
__device__ __forceinline__ void tm_ext_product(FSmemTM &sm, const double2 *__restrict__ G, const Gadget &g, int grp,
                                               int t, const FLay &lay, const double2 *__restrict__ twf,
                                               const double2 *__restrict__ twi, uint32_t lane_addr,
                                               uint32_t &key_phase, Prep &&prep, Sink &&sink) {
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;
#pragma unroll 1
  for (int r = 0; r < 2 * lv; ++r) {
    // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
    const int comp = r < lv ? 1 : 0;
    const int tt = r < lv ? r : r - lv;
    const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
    double2 x[2][FC];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        const uint32_t p0 = prep(q, comp, i), p1 = prep(q, comp, i + FH);
        x[q][j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
      }
    const double2 *gr = G + (size_t)r * (2 * 2 * FC * FT);
    fwd_fft_k<2>(x, sm.scr[grp], lay, t, twf, 0, [&] {
      if (threadIdx.x == 0) {   // every thread is past the previous reader of the key buffer
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full, kSliceBytes);
        bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
      }
    });
    mbar_wait(&sm.key_full, key_phase);
    key_phase ^= 1u;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      const uint32_t a0 = lane_addr + (uint32_t)((0 * 4 + ch) * 32), a1 = lane_addr + (uint32_t)((1 * 4 + ch) * 32);
      uint32_t y0[32], y1[32];
      tm_ld32(a0, y0);
      tm_ld32(a1, y1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const double2 k = sm.key[(ch * FC + j) * FT + t];
        double2 u = tm_get(y0, j), v = tm_get(y1, j);
        u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
        u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
        v.x = fma(x[1][j].x, k.x, fma(-x[1][j].y, k.y, v.x));
        v.y = fma(x[1][j].x, k.y, fma(x[1][j].y, k.x, v.y));
        // per-double stores: the results stay in whatever registers the DFMAs chose
        // (32-register block stores made ptxas move them)
        tm_st_acc(a0 + 4 * j, u);
        tm_st_acc(a1 + 4 * j, v);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // inverse transforms, one ciphertext at a time (both groups in lockstep);
  // group 0's scratch is the idle key buffer, group 1's the forward scratch
  __syncthreads();
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    double2 Y[4][FC];
    {
      uint32_t y[4][32];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) tm_ld32(lane_addr + (uint32_t)((q * 4 + ch) * 32), y[ch]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) tm_zero32(lane_addr + (uint32_t)((q * 4 + ch) * 32));   // next product
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
#pragma unroll
        for (int j = 0; j < FC; ++j) Y[ch][j] = tm_get(y[ch], j);
    }
    inv_fft_k<4>(Y, grp == 0 ? sm.key : &sm.scr[0][0], lay, t, twi);
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        sink(q, c, i, round_u32(Y[2 * c][j].x) + (round_u32(Y[2 * c + 1][j].x) << 16));
        sink(q, c, i + FH, round_u32(Y[2 * c][j].y) + (round_u32(Y[2 * c + 1][j].y) << 16));
      }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// TMEM allocation of a 128-thread CTA (warp 0 allocates, every thread sees the base)
__device__ __forceinline__ uint32_t tm_alloc_cta(FSmemTM &sm) {
  if (threadIdx.x / 32 == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
#pragma unroll
  for (int k = 0; k < 8; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  return lane_addr;
}
__device__ __forceinline__ void tm_free_cta(FSmemTM &sm) {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x / 32 == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(TM_COLS));
  }
}

__global__ void __launch_bounds__(2 * FT, 2)
    blind_rotate_fft_tm_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                               int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemTM &sm = *reinterpret_cast<FSmemTM *>(smem_raw);
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT, warp = tid / 32;
  const FLay lay = make_flay(t);
  int64_t bq[2];
  bool vq[2];
  const uint32_t *row[2];
  uint32_t *acc[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    // items past the end of the batch run a clamped copy of the last ciphertext
    // (they take part in every barrier) and write nothing
    const int64_t bb = (int64_t)blockIdx.x * TMC + grp * 2 + q;
    vq[q] = bb < B;
    bq[q] = vq[q] ? bb : B - 1;
    row[q] = lwe_in + bq[q] * (int64_t)(L + 1);
    acc[q] = sm.acc[grp * 2 + q];
    if (s0 == 0) {
      const int bt = mod_switch(row[q][L], LOG2M);
      const uint32_t *tp = tv + (tv_per_item ? bq[q] * 2 * N : 0);
      const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
      for (int k = t; k < 2 * N; k += FT) {
        const int c = k >= N, i = k & (N - 1);
        acc[q][k] = rot_read<N>(tp + c * N, i, e);
      }
    } else {
      for (int k = t; k < 2 * N; k += FT) acc[q][k] = acc_io[bq[q] * 2 * N + k];
    }
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int k = 0; k < 8; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t key_phase = 0;
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;
  uint32_t a_nx[2] = {row[0][s0], row[1][s0]};   // the next step's mask words, loaded a step ahead
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    int e[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      e[q] = mod_switch(a_nx[q], LOG2M);   // X^{a~_s}
      a_nx[q] = row[q][s + 1];
    }
    // the CTA runs the step when any of its ciphertexts needs it (shared key
    // slices and barriers); an exact no-op product (e = 0) is discarded
    if (!__syncthreads_or((e[0] | e[1]) != 0)) continue;
    const double2 *G = ggsw + (size_t)s * ggsw_f;
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      double2 x[2][FC];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t *ac = acc[q] + comp * N;
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          const uint32_t p0 = decomp_prep(rot_read<N>(ac, i, e[q]) - ac[i], g);
          const uint32_t p1 = decomp_prep(rot_read<N>(ac, i + FH, e[q]) - ac[i + FH], g);
          x[q][j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
        }
      }
      const double2 *gr = G + (size_t)r * (2 * 2 * FC * FT);
      fwd_fft_k<2>(x, sm.scr[grp], lay, t, twf, 0, [&] {
        if (tid == 0) {   // every thread is past the previous reader of the key buffer
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&sm.key_full, kSliceBytes);
          bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
        }
      });
      mbar_wait(&sm.key_full, key_phase);
      key_phase ^= 1u;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a0 = lane_addr + (uint32_t)((0 * 4 + ch) * 32), a1 = lane_addr + (uint32_t)((1 * 4 + ch) * 32);
        uint32_t y0[32], y1[32];
        tm_ld32(a0, y0);   // zeroed at the end of the previous product
        tm_ld32(a1, y1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = sm.key[(ch * FC + j) * FT + t];
#endif
          double2 u = tm_get(y0, j), v = tm_get(y1, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          v.x = fma(x[1][j].x, k.x, fma(-x[1][j].y, k.y, v.x));
          v.y = fma(x[1][j].x, k.y, fma(x[1][j].y, k.x, v.y));
          // per-double stores: the results stay in whatever registers the DFMAs chose
          tm_st_acc(a0 + 4 * j, u);
          tm_st_acc(a1 + 4 * j, v);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms, one ciphertext at a time (both groups in lockstep);
    // group 0's scratch is the idle key buffer, group 1's the forward scratch
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      double2 Y[4][FC];
      {
        uint32_t y[4][32];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tm_ld32(lane_addr + (uint32_t)((q * 4 + ch) * 32), y[ch]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tm_zero32(lane_addr + (uint32_t)((q * 4 + ch) * 32));   // next product
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[ch][j] = tm_get(y[ch], j);
      }
      inv_fft_k<4>(Y, grp == 0 ? sm.key : &sm.scr[0][0], lay, t, twi);
      if (e[q] != 0) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const int i = t + FT * j;
            acc[q][c * N + i] += round_u32(Y[2 * c][j].x) + (round_u32(Y[2 * c + 1][j].x) << 16);
            acc[q][c * N + i + FH] += round_u32(Y[2 * c][j].y) + (round_u32(Y[2 * c + 1][j].y) << 16);
          }
      }
    }
    __syncthreads();
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(TM_COLS));
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (!vq[q]) continue;
    if (s1 < L) {
      for (int k = t; k < 2 * N; k += FT) acc_io[bq[q] * 2 * N + k] = acc[q][k];
    } else {
      uint32_t *o = lwe_out + bq[q] * (int64_t)(N + 1);
      for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[q][0] : 0u - acc[q][N - k];
      if (t == 0) o[N] = acc[q][N];
    }
  }
}

// ---------------------------------------------------------------------------
// TMEM ladder, one ciphertext per thread (`blind_rotate_fft_tx_kernel`, FFT mode 2).
//
// The TMEM ladder above runs 8 warps per SM: TMEM (256 KB) holds the spectral
// accumulators of exactly 8 ciphertexts, and each thread carries two of them.  Here
// each 64-thread group owns ONE ciphertext (8 complex values per thread), so the same
// 8 ciphertexts per SM run on 16 warps at <= 128 registers: twice the warps to hide
// the FFT's dependency and shared-memory latencies, at the price of reading each
// key value once per ciphertext instead of once per two.  CTA = 4 groups (256
// threads, 4 ciphertexts, one TMA-staged key slice per digit row shared by all four);
// 2 CTAs per SM.  The decomposition-ready words of a component are computed once per
// step (rotation and difference), and its l digit rows are extracted from registers.
// TMEM: group q's warps 2q, 2q+1 sit in sub-partitions (2q) % 4 and (2q+1) % 4, so
// groups q and q + 2 share lanes and split the CTA's 256 columns: column
// (q >> 1) 128 + ((c 2 + h) 32) + 4 j + {re.lo, re.hi, im.lo, im.hi}.
// Inverse: the two halves (lo, hi) of one component at a time (two transforms in
// lockstep), scratch = the forward scratch (groups 0, 1) or the idle key buffer
// (groups 2, 3).  Bit-identical to the other FFT ladders.

constexpr int TXC = 4;   // ciphertexts (64-thread groups) per CTA

struct FSmemTX {
  uint32_t acc[TXC][2 * 2 * FH];
  double2 scr[2][2 * FH];          // forward scratch of groups 0..3 (8 KB each); inverse: groups 0, 1
  double2 key[2 * 2 * FC * FT];    // the digit's key slice (TMA); inverse scratch of groups 2, 3
  uint64_t key_full;
  uint32_t tmem_slot;
};

#ifndef HWB_TX_HOIST
#define HWB_TX_HOIST 1
#endif

__global__ void __launch_bounds__(TXC * FT, 2)
    blind_rotate_fft_tx_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                               int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemTX &sm = *reinterpret_cast<FSmemTX *>(smem_raw);
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT, warp = tid / 32;
  const FLay lay = make_flay(t);
  // items past the end of the batch run a clamped copy of the last ciphertext
  // (they take part in every barrier) and write nothing
  const int64_t bb = (int64_t)blockIdx.x * TXC + grp;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[grp];
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = t; k < 2 * N; k += FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = t; k < 2 * N; k += FT) acc[k] = acc_io[bq * 2 * N + k];
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((grp >> 1) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t key_phase = 0;
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = &sm.scr[0][0] + grp * FH;                               // forward: 8 KB per group
  double2 *iscr = grp < 2 ? &sm.scr[0][0] + grp * 2 * FH : sm.key + (grp - 2) * 2 * FH;   // inverse: 16 KB
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead (s + 1 <= L)
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
    // the CTA runs the step when any of its ciphertexts needs it (shared key
    // slices and barriers); an exact no-op product (e = 0) is discarded
    if (!__syncthreads_or(e != 0)) continue;
    const double2 *G = ggsw + (size_t)s * ggsw_f;
#if HWB_TX_HOIST
    uint32_t pw[2][FC];   // decomposition-ready words of the current component
#endif
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[1][FC];
#if HWB_TX_HOIST
      if (tt == 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          pw[0][j] = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
          pw[1][j] = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        }
      }
#pragma unroll
      for (int j = 0; j < FC; ++j)
        x[0][j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                               u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
#else
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        const uint32_t p0 = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
        const uint32_t p1 = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        x[0][j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
      }
#endif
      const double2 *gr = G + (size_t)r * (2 * 2 * FC * FT);
      fwd_fft_k<1>(x, fscr, lay, t, twf, 0, [&] {
        if (tid == 0) {   // every thread is past the previous reader of the key buffer
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&sm.key_full, kSliceBytes);
          bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
        }
      });
      mbar_wait(&sm.key_full, key_phase);
      key_phase ^= 1u;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a = lane_addr + (uint32_t)(ch * 32);
        uint32_t y[32];
        tm_ld32(a, y);   // zeroed at the end of the previous product
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = sm.key[(ch * FC + j) * FT + t];
#endif
          double2 u = tm_get(y, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          tm_st_acc(a + 4 * j, u);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms: the two halves of one component at a time; groups 2, 3
    // use the idle key buffer as scratch, so every thread must be past its MAC
    __syncthreads();
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      double2 Y[2][FC];
      {
        uint32_t y[2][32];
#pragma unroll
        for (int h = 0; h < 2; ++h) tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y[h]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) tm_zero32(lane_addr + (uint32_t)((c * 2 + h) * 32));   // next product
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[h][j] = tm_get(y[h], j);
      }
      inv_fft_k<2>(Y, iscr, lay, t, twi);
      if (e != 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          acc[c * N + i] += round_u32(Y[0][j].x) + (round_u32(Y[1][j].x) << 16);
          acc[c * N + i + FH] += round_u32(Y[0][j].y) + (round_u32(Y[1][j].y) << 16);
        }
      }
    }
    __syncthreads();
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(TM_COLS));
  }
  if (!valid) return;
  if (s1 < L) {
    for (int k = t; k < 2 * N; k += FT) acc_io[bq * 2 * N + k] = acc[k];
  } else {
    uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
    for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
    if (t == 0) o[N] = acc[N];
  }
}

// ---------------------------------------------------------------------------
// TMEM ladder, lane-paired (`blind_rotate_fft_tp_kernel`, FFT mode 3).
//
// Mode 2's layout (one ciphertext per thread, 16 warps per SM) with the two
// ciphertexts of a lane pair (2m, 2m + 1) at the SAME spectral position: the key
// value and the twiddles a pair needs sit at one shared-memory address, and a
// quarter-warp LDS.128 that serves 4 addresses to 8 lanes costs 2.4 instead of 4
// crossbar cycles (tools/lds_bcast_bench.cu).  Thread (warp w, lane L): ciphertext
// q = 2 (w & 1) + (L & 1), transform position t = 16 (w >> 1) + (L >> 1) -- each
// transform spans half the lanes of 4 warps.  Bank offsets keep the pairs
// conflict-free: odd ciphertexts' transpose scratch is displaced by 64 B (4 of the 8
// 16-byte bank groups), their accumulators by 16 words.  The per-thread twiddles
// (compact: sibling slots dropped, hwb_fft.cuh) are staged in shared memory.

constexpr int TPC = 4;                   // ciphertexts per CTA
constexpr int TP_ACC = 2 * 2 * FH + 16;  // words per accumulator (+16: pair bank offset)

struct FSmemTP {
  uint32_t acc[TPC][TP_ACC];
  double2 scr[4 * (FH + 4)];            // forward scratch (8 KB per ciphertext); inverse: ciphertexts 0, 1
  double2 key[2 * 2 * FC * FT + 4];     // the digit's key slice (TMA); inverse scratch of ciphertexts 2, 3
  double2 twf[kTwc * FT], twi[kTwc * FT];
  uint64_t key_full;
  uint32_t key_cnt;   // mode 5: halves done with the key buffer
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(TPC * FT, 2)
    blind_rotate_fft_tp_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                               int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemTP &sm = *reinterpret_cast<FSmemTP *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int q = 2 * (warp & 1) + (lane & 1), t = 16 * (warp >> 1) + (lane >> 1);
  const FLay lay = make_flay(t);
  const int64_t bb = (int64_t)blockIdx.x * TPC + q;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[q];
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = t; k < 2 * N; k += FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = t; k < 2 * N; k += FT) acc[k] = acc_io[bq * 2 * N + k];
  }
  for (int k = tid; k < kTwc * FT; k += TPC * FT) {
    sm.twf[k] = twf[twc_full<true>(k / FT) * FT + k % FT];
    sm.twi[k] = twi[twc_full<false>(k / FT) * FT + k % FT];
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t key_phase = 0;
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = sm.scr + q * (FH + 4);                                                      // 8 KB
  double2 *iscr = (q < 2 ? sm.scr : sm.key) + (q & 1) * (2 * FH + 4);                        // 16 KB
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead (s + 1 <= L)
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
    if (!__syncthreads_or(e != 0)) continue;
    const double2 *G = ggsw + (size_t)s * ggsw_f;
    uint32_t pw[2][FC];   // decomposition-ready words of the current component
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[1][FC];
      if (tt == 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          pw[0][j] = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
          pw[1][j] = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        }
      }
#pragma unroll
      for (int j = 0; j < FC; ++j)
        x[0][j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                               u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
      const double2 *gr = G + (size_t)r * (2 * 2 * FC * FT);
      fwd_fft_k<1, true>(x, fscr, lay, t, sm.twf, 0, [&] {
        if (tid == 0) {   // every thread is past the previous reader of the key buffer
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&sm.key_full, kSliceBytes);
          bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
        }
      });
      mbar_wait(&sm.key_full, key_phase);
      key_phase ^= 1u;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a = lane_addr + (uint32_t)(ch * 32);
        uint32_t y[32];
        tm_ld32(a, y);   // zeroed at the end of the previous product
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = sm.key[(ch * FC + j) * FT + t];
#endif
          double2 u = tm_get(y, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          tm_st_acc(a + 4 * j, u);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms: the two halves of one component at a time; ciphertexts 2, 3
    // use the idle key buffer as scratch, so every thread must be past its MAC
    __syncthreads();
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      double2 Y[2][FC];
      {
        uint32_t y[2][32];
#pragma unroll
        for (int h = 0; h < 2; ++h) tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y[h]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) tm_zero32(lane_addr + (uint32_t)((c * 2 + h) * 32));   // next product
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[h][j] = tm_get(y[h], j);
      }
      inv_fft_k<2, true>(Y, iscr, lay, t, sm.twi);
      if (e != 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          acc[c * N + i] += round_u32(Y[0][j].x) + (round_u32(Y[1][j].x) << 16);
          acc[c * N + i + FH] += round_u32(Y[0][j].y) + (round_u32(Y[1][j].y) << 16);
        }
      }
    }
    __syncthreads();
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(TM_COLS));
  }
  if (!valid) return;
  if (s1 < L) {
    for (int k = t; k < 2 * N; k += FT) acc_io[bq * 2 * N + k] = acc[k];
  } else {
    uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
    for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
    if (t == 0) o[N] = acc[N];
  }
}

// ---------------------------------------------------------------------------
// TMEM ladder, lane-paired, decoupled halves (`blind_rotate_fft_td_kernel`, FFT mode 5).
//
// Mode 3 with its two halves (warps w & 1 = 0: ciphertexts 0, 1; w & 1 = 1: 2, 3)
// synchronising only among their own 128 threads (named barriers).  They share the
// TMA-staged key slice: each half releases it after its MAC and the second release
// issues the next row's copy (it lands while the halves run their next digit
// transforms).  The inverse runs one accumulator at a time in the ciphertext's own
// 8 KB scratch, so the halves share nothing else.

// Shape of the inverse phase / instruction footprint of the step loop (A/B, cfg2 B = 4096,
// DESIGN.md 3b).  HWB_TD_ONEINV: 0 = the trailing barrier inside the inverse, right after its
// last loads from the scratch (two instantiations for h = 1: 2,808 instructions, 54.3 ms);
// 1 = one instantiation per h, the barrier after the inverse's last three levels, skipped at
// run time for the last inverse (2,344 instructions, **52.4 ms**, default); 2 = 1 with the h
// loop rolled (one instantiation, 1,992 instructions: 54.3 ms); 3 = the barrier at the latest
// point, before the next inverse's first store (53.0 ms); 4 = after the rounding (53.0 ms).
// HWB_TD_MACROLL: 1 / 2 = the MAC's accumulator loop rolled / unrolled by 2 (53.8 / 52.8 ms).
#ifndef HWB_TD_ONEINV
#define HWB_TD_ONEINV 1
#endif
#ifndef HWB_TD_MACROLL
#define HWB_TD_MACROLL 0
#endif
constexpr int kTdMacUnroll = HWB_TD_MACROLL == 1 ? 1 : (HWB_TD_MACROLL == 2 ? 2 : 4),
              kTdInvUnroll = HWB_TD_ONEINV == 2 ? 1 : 2;

template <int NG, int KS>
struct FSmemTDT {
  uint32_t acc[2 * NG][TP_ACC];     // working ciphertexts; odd ones 16 words further (TP_ACC)
  double2 scr[2 * NG][FH];          // transpose scratch per ciphertext (odd: addresses XOR 4)
  double2 key[KS][2 * 2 * FC * FT];   // key-slice ring (TMA)
  double2 twf[kTwc * FT], twi[kTwc * FT];
  uint64_t key_full[KS];
  uint64_t in_full;                 // level kernel: the inputs' bulk copies landed
  uint64_t scr_free[NG];            // mode 5/6: a group's 4 warps are past their reads of scr (split barrier)
  uint32_t key_cnt[KS];             // warps (HWB_TD_SPLITBAR) or groups done with the slot's slice
  uint32_t tmem_slot;
};

// NG groups of 4 warps (2 lane-paired ciphertexts each), KS key slots: <2, 1> = mode 5
// (2 CTAs per SM), <4, 2> = mode 6 (one 16-warp CTA per SM, the slice shared by 8).
template <int NG, int KS>
__global__ void __launch_bounds__(NG * 128, NG == 2 ? 2 : 1)
    blind_rotate_fft_td_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                               int s0_arg, int s1_arg, int64_t B, uint32_t *progress) {
  constexpr int N = 2 * FH;
  // One launch per segment (progress == nullptr: steps [s0_arg, s1_arg), group blockIdx.x) or
  // ONE launch for the whole ladder (progress != nullptr, s1_arg - s0_arg = segment length):
  // CTA b runs segment b / groups of group b % groups, so a segment's partial last wave is
  // filled with the next segment's first groups.  A group's segment s waits until
  // progress[group] == s (its accumulator rests in acc_io; normally done `groups` CTAs ago)
  // and publishes s + 1.  CTAs start in blockIdx order, so a CTA only ever waits for one
  // that is running or done; the wait is bounded and traps instead of hanging.  All of it
  // derives from blockIdx: uniform values, no registers across the steps.
  constexpr int kPerCta = 2 * NG;
  const uint32_t groups = progress ? (uint32_t)((B + 2 * NG - 1) / (2 * NG)) : gridDim.x;
  const uint32_t seg = blockIdx.x / groups, grp = blockIdx.x % groups;
  const int s0 = progress ? (int)seg * (s1_arg - s0_arg) : s0_arg;
  const int s1 = progress ? (s0 + (s1_arg - s0_arg) < L ? s0 + (s1_arg - s0_arg) : L) : s1_arg;
  // (a compile-time SINGLE flag instead of the run-time test measured slower: 52.2 vs 51.9 ms)
  constexpr int LOG2M = 11;
  constexpr int GT = 128;   // threads per half (named barriers)
  extern __shared__ uint4 smem_raw[];
  FSmemTDT<NG, KS> &sm = *reinterpret_cast<FSmemTDT<NG, KS> *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
#ifndef HWB_TD_SPLIT
#define HWB_TD_SPLIT 1
#endif
  // HWB_TD_SPLIT: half = warp >> 2, so every scheduler (warp % 4) runs one warp of each
  // half (independent instruction streams); 0: half = warp & 1 (a scheduler's warps in
  // lockstep)
  const int hsel = HWB_TD_SPLIT || NG != 2 ? (warp >> 2) : (warp & 1),
            hpos = HWB_TD_SPLIT || NG != 2 ? (warp & 3) : (warp >> 1);
  const int q = 2 * hsel + (lane & 1), t = 16 * hpos + (lane >> 1);
  FLay lay = make_flay(t);
  if (q & 1) {   // pair partner: the other half of the 8 bank groups
    lay.a ^= 4u;
    lay.m ^= 4u;
    lay.b ^= 4u;
  }
  const int64_t bb = (int64_t)grp * (2 * NG) + q;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[q];   // TP_ACC stride: odd ciphertexts 16 banks over
  if (progress && seg > 0) {   // the group's previous segment
    if (tid == 0) {
      uint32_t done, spins = 0;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(done) : "l"(progress + grp) : "memory");
        if (done >= seg) break;
        __nanosleep(256);
        if (++spins > (1u << 24)) __trap();   // (seconds: a lost predecessor surfaces as an error)
      }
    }
    __syncthreads();
  }
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = t; k < 2 * N; k += FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = t; k < 2 * N; k += FT) acc[k] = __ldcg(&acc_io[bq * 2 * N + k]);   // (another SM wrote it)
  }
  for (int k = tid; k < kTwc * FT; k += NG * 128) {
    sm.twf[k] = twf[twc_full<true>(k / FT) * FT + k % FT];
    sm.twi[k] = twi[twc_full<false>(k / FT) * FT + k % FT];
  }
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  const int rows = (s1 - s0) * 2 * lv;   // key-slice rows of this launch, u = (s - s0) 2l + r
  auto slice = [&](int u) {
    return ggsw + (size_t)(s0 + u / (2 * lv)) * ggsw_f + (size_t)(u % (2 * lv)) * (2 * 2 * FC * FT);
  };
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      mbar_init(&sm.key_full[k], 1);
      sm.key_cnt[k] = 0;
    }
#pragma unroll
    for (int k = 0; k < NG; ++k) mbar_init(&sm.scr_free[k], 4);   // one arrival per warp of the group
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int k = 0; k < KS; ++k)   // the first KS rows' slices
      if (k < rows) {
        mbar_expect_tx(&sm.key_full[k], kSliceBytes);
        bulk_g2s(sm.key[k], slice(k), kSliceBytes, &sm.key_full[k]);
      }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"((uint32_t)(NG * 128)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const int half = hsel, hbar = 1 + half;
  const bool leader = lane == 0 && hpos == 0;
  // a half is done with the key buffer (slice or, for half 1, inverse scratch):
  // the second half to finish issues the next row's slice
#ifndef HWB_TD_SPLITBAR
#define HWB_TD_SPLITBAR 0
#endif
#ifndef HWB_TD_LATEWAIT
#define HWB_TD_LATEWAIT 0
#endif
  // HWB_TD_SPLITBAR: the barriers that only guard buffer REUSE become split barriers.
  // (a) Key slot: every warp counts itself out after its MAC (its key loads have returned:
  // the tcgen05.st of their products have issued) and the last of the CTA's warps issues
  // the next slice's copy -- nobody waits.  (b) Transpose scratch: a warp arrives on the
  // group's scr_free mbarrier once its last loads from scr are consumed (the stages after
  // the transform's second transpose) and waits on it only right before the next
  // transform's first store, a whole stage group later.  The barriers between a
  // transpose's stores and loads (a data dependency) stay.
  auto release = [&](int u) {   // the last warp / group done with slot u % KS fetches row u + KS
#if HWB_TD_SPLITBAR
    __syncwarp();
    if (lane != 0) return;
    constexpr uint32_t kLast = NG * 4 - 1;
#else
    if (!leader) return;
    constexpr uint32_t kLast = NG - 1;
#endif
    __threadfence_block();
    if (atomicAdd(&sm.key_cnt[u % KS], 1u) == kLast) {
      sm.key_cnt[u % KS] = 0;
      if (u + KS < rows) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full[u % KS], kSliceBytes);
        bulk_g2s(sm.key[u % KS], slice(u + KS), kSliceBytes, &sm.key_full[u % KS]);
      }
    }
  };
#if HWB_TD_SPLITBAR
  uint32_t sf_phase = 0;   // completed scr_free phases this thread has waited for
  auto scr_arrive = [&] {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.scr_free[half]);
  };
  auto scr_wait = [&] {
    mbar_wait(&sm.scr_free[half], sf_phase & 1u);
    ++sf_phase;
  };
#endif

  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = sm.scr[q];   // 8 KB
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead (s + 1 <= L)
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
      uint32_t pw[2][FC];   // decomposition-ready words of the current component
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[1][FC];
      if (tt == 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          pw[0][j] = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
          pw[1][j] = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        }
      }
#pragma unroll
      for (int j = 0; j < FC; ++j)
        x[0][j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                               u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
      // (no trailing barrier on the second transpose: the release barrier after the MAC
      // precedes the next write into fscr)
#if HWB_TD_SPLITBAR
      fwd_fft_hk<1, GT, true, false>(x, fscr, lay, t, sm.twf, hbar, 0, [&] {
        if (r != 0) scr_wait();   // (row 0 follows the end-of-step barrier)
      });
      scr_arrive();   // the last stages consumed every value loaded from fscr
#else
      fwd_fft_hk<1, GT, true, false>(x, fscr, lay, t, sm.twf, hbar);
#endif
      const int u = (s - s0) * 2 * lv + r;   // this row's slot u % KS, use u / KS
      mbar_wait(&sm.key_full[u % KS], (uint32_t)(u / KS) & 1u);
      const double2 *key = sm.key[u % KS];
#if HWB_TD_LATEWAIT   // the previous row's (or the inverse's zeroing) stores: drained during the transform
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#endif
#pragma unroll kTdMacUnroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a = lane_addr + (uint32_t)(ch * 32);
        uint32_t y[32];
        tm_ld32(a, y);   // zeroed at the end of the previous product
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = key[(ch * FC + j) * FT + t];
#endif
          double2 u = tm_get(y, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          tm_st_acc(a + 4 * j, u);
        }
      }
#if !HWB_TD_SPLITBAR
      gsync<GT>(hbar);   // the half is past the slice
#endif
      release(u);
#if !HWB_TD_LATEWAIT
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#endif
    }
#if HWB_TD_LATEWAIT
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");   // the last row's products
#endif
    // inverse transforms, one accumulator at a time (lo then hi of each component), in
    // the ciphertext's own forward scratch: the key buffer only ever holds slices
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t lo[2][FC] = {};
#pragma unroll kTdInvUnroll
      for (int h = 0; h < 2; ++h) {
        double2 Y[1][FC];
        {
          uint32_t y[32];
          tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tm_zero32(lane_addr + (uint32_t)((c * 2 + h) * 32));   // next product
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[0][j] = tm_get(y, j);
        }
#if HWB_TD_SPLITBAR
        inv_fft_hk<1, GT, true, false>(Y, fscr, lay, t, sm.twi, hbar, 0, [&] { scr_wait(); });
        if (!(c == 1 && h == 1)) scr_arrive();   // (the end-of-step barrier follows the last one)
#else
#if HWB_TD_ONEINV == 3
        // the scratch-reuse barrier as late as it can be: right before this inverse's first
        // store into fscr, after its TMEM load and first three levels (the first inverse
        // follows the MAC's barrier and needs none)
        inv_fft_hk<1, GT, true, false>(Y, fscr, lay, t, sm.twi, hbar, 0, [&] {
          if (h == 1 || c == 1) gsync<GT>(hbar);
        });
#elif HWB_TD_ONEINV   // one copy of the inverse per h: the trailing barrier as a runtime-skipped call after it
        inv_fft_hk<1, GT, true, false>(Y, fscr, lay, t, sm.twi, hbar);
        if (HWB_TD_ONEINV != 4 && !(c == 1 && h == 1)) gsync<GT>(hbar);   // (the end-of-step barrier follows the last inverse)
#else
        if (c == 1 && h == 1)   // the end-of-step barrier precedes the next write into fscr
          inv_fft_hk<1, GT, true, false>(Y, fscr, lay, t, sm.twi, hbar);
        else
          inv_fft_hk<1, GT, true>(Y, fscr, lay, t, sm.twi, hbar);
#endif
#endif
        if (h == 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            lo[0][j] = round_u32(Y[0][j].x);
            lo[1][j] = round_u32(Y[0][j].y);
          }
        } else if (e != 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const int i = t + FT * j;
            acc[c * N + i] += lo[0][j] + (round_u32(Y[0][j].x) << 16);
            acc[c * N + i + FH] += lo[1][j] + (round_u32(Y[0][j].y) << 16);
          }
        }
        if (HWB_TD_ONEINV == 4 && !(c == 1 && h == 1)) gsync<GT>(hbar);   // (variant: after the rounding)
      }
    }
    gsync<GT>(hbar);   // the half's accumulator updates before the next step's digits
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot),
                 "r"((uint32_t)(NG * 128)));
  }
  if (valid) {
    if (s1 < L) {
      for (int k = t; k < 2 * N; k += FT) acc_io[bq * 2 * N + k] = acc[k];
    } else {
      uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
      for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
      if (t == 0) o[N] = acc[N];
    }
  }
  if (progress) {   // publish after every thread's accumulator stores
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      // (recomputed from blockIdx: nothing of the protocol stays live across the steps)
      const uint32_t groups2 = (uint32_t)((B + kPerCta - 1) / kPerCta);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(progress + blockIdx.x % groups2),
                   "r"(blockIdx.x / groups2 + 1)
                   : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// TMEM ladder on wide threads (`blind_rotate_fft_w_kernel`, FFT mode 7).
//
// Mode 5's structure (lane-paired ciphertexts, decoupled groups, the TMA-staged key slice
// shared by the CTA's 4 ciphertexts, spectra accumulators in tensor memory) on the
// 32-thread transform of hwb_fft.cuh (fwd_fft16 / inv_fft16): 16 complex values per
// thread, so a transform has ONE shared-memory transpose (16 KB of traffic instead of
// 32 KB) plus 16 register exchanges with the neighbouring position through shuffles.  A
// CTA is 4 warps = 2 groups of 2 warps; a group carries two lane-paired ciphertexts
// (lanes 2m, 2m + 1: the same position u = 16 (warp & 1) + m of ciphertexts 2 g, 2 g + 1)
// and synchronises on its own 64-thread named barrier.  Each thread owns 256 TMEM
// columns (4 accumulators x 16 complex), a CTA the 4 lane quadrants x 256 columns; two
// CTAs per SM fill the tensor memory with 8 ciphertexts, as in mode 5.  The key is read
// in its usual layout at (j, t) = (i & 7, i >> 3), i = w16_index(u, s): 4 positions of a
// quarter-warp read 4 distinct 16-byte bank groups, each serving a lane pair.

#ifndef HWB_W_ROLL   // 1: the MAC's accumulator loop rolled (instruction-cache footprint: 61.5 -> 59.4 ms)
#define HWB_W_ROLL 1
#endif
// (The four inverses stay unrolled.  A rolled loop carries `lo` from the h = 0 iteration to
// the h = 1 one; with `lo` uninitialised at loop entry that build returned wrong results --
// the loop-carried value has an undefined incoming edge -- hence the `= {}` below and in the
// other ladders' rolled variants.)
constexpr int kWUnroll = HWB_W_ROLL ? 1 : 4, kWUnrollInv = 4;

struct FSmemW {
  uint32_t acc[4][TP_ACC];          // working ciphertexts; odd ones 16 words further (TP_ACC)
  double2 scr[4][FH];               // transpose scratch per ciphertext (odd: addresses XOR 4)
  double2 key[2 * 2 * FC * FT];     // the row's key slice (TMA), shared by both groups
  double2 twf[kW16Tab], twi[kW16Tab];
  uint64_t key_full;
  uint32_t key_cnt;                 // groups done with the slice
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(128, 2)
    blind_rotate_fft_w_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                              const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                              const double2 *__restrict__ w16tab, uint32_t *acc_io, int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemW &sm = *reinterpret_cast<FSmemW *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int grp = warp >> 1, bar = 1 + grp;
  const int q = 2 * grp + (lane & 1), u = 16 * (warp & 1) + (lane >> 1);
  // swizzled element bases of the thread in layouts A16 (i = u + 32 j) and M16
  // (i = (u >> 1) << 5 | jj << 1 | (u & 1)); the pair partner takes the other half of the
  // 8 bank groups
  const uint32_t px = (q & 1) ? 4u : 0u;
  const uint32_t ea = wswz((uint32_t)u) ^ px, em = wswz((uint32_t)(((u >> 1) << 5) | (u & 1))) ^ px;
  const int64_t bb = (int64_t)blockIdx.x * 4 + q;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[q];
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = u; k < 2 * N; k += WT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = u; k < 2 * N; k += WT) acc[k] = acc_io[bq * 2 * N + k];
  }
  for (int k = tid; k < kW16Tab; k += 128) {
    sm.twf[k] = w16tab[k];
    sm.twi[k] = w16tab[kW16Tab + k];
  }
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  const int rows = (s1 - s0) * 2 * lv;   // key-slice rows of this launch, r_abs = (s - s0) 2l + r
  auto slice = [&](int ra) {
    return ggsw + (size_t)(s0 + ra / (2 * lv)) * ggsw_f + (size_t)(ra % (2 * lv)) * (2 * 2 * FC * FT);
  };
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    sm.key_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&sm.key_full, kSliceBytes);
    bulk_g2s(sm.key, slice(0), kSliceBytes, &sm.key_full);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // lane quadrant = warp (4 warps); columns (ch 16 + s) 4 + {re.lo, re.hi, im.lo, im.hi}
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int k = 0; k < 8; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const bool leader = lane == 0 && (warp & 1) == 0;
  // a group is done with the slice: the second one issues the next row's copy
  auto release = [&](int ra) {
    if (!leader) return;
    __threadfence_block();
    if (atomicAdd(&sm.key_cnt, 1u) == 1u) {
      sm.key_cnt = 0;
      if (ra + 1 < rows) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full, kSliceBytes);
        bulk_g2s(sm.key, slice(ra + 1), kSliceBytes, &sm.key_full);
      }
    }
  };

  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = sm.scr[q];   // 8 KB
  // key address of slot s: (j, t) = (i & 7, i >> 3), i = w16_index(u, s): t = 2 u + ((s >> 2) & 1)
  const double2 *keyu = sm.key + 2 * u;
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead (s + 1 <= L)
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
    uint32_t pw[2][WC];   // decomposition-ready words of the current component
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[WC];
      if (tt == 0) {
#pragma unroll
        for (int j = 0; j < WC; ++j) {
          const int i = u + WT * j;
          pw[0][j] = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
          pw[1][j] = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        }
      }
#pragma unroll
      for (int j = 0; j < WC; ++j)
        x[j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                            u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
      // (no trailing barrier: the release barrier after the MAC precedes the next write
      // into fscr)
      fwd_fft16(x, fscr, ea, em, u, sm.twf, bar);
      const int ra = (s - s0) * 2 * lv + r;
      mbar_wait(&sm.key_full, (uint32_t)ra & 1u);
#pragma unroll kWUnroll
      for (int ch = 0; ch < 4; ++ch) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const uint32_t a = lane_addr + (uint32_t)(ch * 64 + hf * 32);
          uint32_t y[32];
          tm_ld32(a, y);   // zeroed at the end of the previous product
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int s8 = 0; s8 < 8; ++s8) {
            const int sl = hf * 8 + s8;
            const int kj = ((sl & 3) << 1) | (sl >> 3), kt = (sl >> 2) & 1;
#if HWB_X_NOKEY
            const double2 k = make_double2(1.0 + sl + ch, 0.5 * r);
#else
            const double2 k = keyu[(ch * FC + kj) * FT + kt];
#endif
            double2 v = tm_get(y, s8);
            v.x = fma(x[sl].x, k.x, fma(-x[sl].y, k.y, v.x));
            v.y = fma(x[sl].x, k.y, fma(x[sl].y, k.x, v.y));
            tm_st_acc(a + 4 * s8, v);
          }
        }
      }
      gsync<64>(bar);   // the group is past the slice (and its reads of fscr)
      release(ra);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms, one accumulator at a time (lo then hi of each component)
    uint32_t lo[2][WC] = {};
#pragma unroll kWUnrollInv
    for (int ci = 0; ci < 4; ++ci) {
      const int c = ci >> 1, h = ci & 1;
      double2 Y[WC];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t a = lane_addr + (uint32_t)(ci * 64 + hf * 32);
        uint32_t y[32];
        tm_ld32(a, y);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tm_zero32(a);   // next product
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) Y[hf * 8 + s8] = tm_get(y, s8);
      }
      // (the end-of-step barrier follows the last inverse)
      inv_fft16(Y, fscr, ea, em, u, sm.twi, bar, ci != 3);
      if (h == 0) {
#pragma unroll
        for (int j = 0; j < WC; ++j) {
          lo[0][j] = round_u32(Y[j].x);
          lo[1][j] = round_u32(Y[j].y);
        }
      } else {
        // (a skipped step, e == 0, adds 0: no branch, the pair's two ciphertexts -- lanes of
        // one warp with different e -- never diverge ahead of the named barriers)
        const uint32_t keep = e != 0 ? 0xFFFFFFFFu : 0u;
#pragma unroll
        for (int j = 0; j < WC; ++j) {
          const int i = u + WT * j;
          acc[c * N + i] += (lo[0][j] + (round_u32(Y[j].x) << 16)) & keep;
          acc[c * N + i + FH] += (lo[1][j] + (round_u32(Y[j].y) << 16)) & keep;
        }
      }
    }
    gsync<64>(bar);   // the group's accumulator updates before the next step's digits
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(256u));
  }
  if (!valid) return;
  if (s1 < L) {
    for (int k = u; k < 2 * N; k += WT) acc_io[bq * 2 * N + k] = acc[k];
  } else {
    uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
    for (int k = u; k < N; k += WT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
    if (u == 0) o[N] = acc[N];
  }
}

// ---------------------------------------------------------------------------
// TMEM ladder, decoupled lane-paired groups (`blind_rotate_fft_tq_kernel`, FFT mode 4).
//
// One CTA of 16 warps per SM holds 8 ciphertexts (the TMEM capacity) as 4 independent
// groups of 4 warps; a group carries two lane-paired ciphertexts (mode 3's mapping:
// lanes 2m, 2m + 1 share a spectral position, so they read one key address).  Groups
// synchronise only among their own 128 threads (named barriers), and each transpose
// has one barrier instead of two: the two transposes of a transform use two scratch
// buffers (fwd_fft_pp / inv_fft_pp).  All 8 ciphertexts share one TMA-staged key
// slice: the last group to finish a row's MAC (shared counter) issues the next row's
// copy, which lands while the groups run their digit transforms.  The inverse runs
// one accumulator at a time.  Odd ciphertexts' transpose addresses are XOR-ed with 4
// (the 16-byte bank group's top bit) so a pair never conflicts.

constexpr int TQC = 8;   // ciphertexts per CTA
constexpr int TQG = 4;   // groups (4 warps, 2 ciphertexts each)

struct FSmemTQ {
  uint32_t acc[TQC][2 * 2 * FH];
  double2 buf[2][TQC][FH];          // ping-pong transpose scratch, 8 KB per ciphertext each
  double2 key[2 * 2 * FC * FT];     // the row's key slice (TMA), shared by all groups
  uint64_t key_full;
  uint32_t key_cnt;                 // groups done with the current slice
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(TQG * 4 * 32, 1)
    blind_rotate_fft_tq_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi, uint32_t *acc_io,
                               int s0, int s1, int64_t B) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  constexpr int GT = 128;   // threads per group
  extern __shared__ uint4 smem_raw[];
  FSmemTQ &sm = *reinterpret_cast<FSmemTQ *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int grp = warp >> 2, bar = 1 + grp;
  const int q = 2 * grp + (lane & 1), t = 16 * (warp & 3) + (lane >> 1);
  FLay lay = make_flay(t);
  if (q & 1) {   // pair partner: the other half of the 8 bank groups
    lay.a ^= 4u;
    lay.m ^= 4u;
    lay.b ^= 4u;
  }
  const int64_t bb = (int64_t)blockIdx.x * TQC + q;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[q];
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = t; k < 2 * N; k += FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = t; k < 2 * N; k += FT) acc[k] = acc_io[bq * 2 * N + k];
  }
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    sm.key_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&sm.key_full, kSliceBytes);   // the first row's slice
    bulk_g2s(sm.key, ggsw + (size_t)s0 * ggsw_f, kSliceBytes, &sm.key_full);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t key_phase = 0;
  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *b0 = sm.buf[0][q], *b1 = sm.buf[1][q];
  const bool leader = (tid % GT) == 0;
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead (s + 1 <= L)
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
    uint32_t pw[2][FC];   // decomposition-ready words of the current component
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[1][FC];
      if (tt == 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          pw[0][j] = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
          pw[1][j] = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        }
      }
#pragma unroll
      for (int j = 0; j < FC; ++j)
        x[0][j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                               u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
      fwd_fft_pp<1, GT>(x, b0, b1, lay, t, twf, bar);
      mbar_wait(&sm.key_full, key_phase);
      key_phase ^= 1u;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a = lane_addr + (uint32_t)(ch * 32);
        uint32_t y[32];
        tm_ld32(a, y);   // zeroed at the end of the previous product
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = sm.key[(ch * FC + j) * FT + t];
#endif
          double2 u = tm_get(y, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          tm_st_acc(a + 4 * j, u);
        }
      }
      // the group is done with the slice; the last group fetches the next row's
      gsync<GT>(bar);
      if (leader) {
        __threadfence_block();
        const uint32_t done = atomicAdd(&sm.key_cnt, 1u);
        if (done == TQG - 1) {
          sm.key_cnt = 0;
          const int nr = r + 1 < 2 * lv ? r + 1 : 0, ns = r + 1 < 2 * lv ? s : s + 1;
          if (ns < s1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.key_full, kSliceBytes);
            bulk_g2s(sm.key, ggsw + (size_t)ns * ggsw_f + (size_t)nr * (2 * 2 * FC * FT), kSliceBytes,
                     &sm.key_full);
          }
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms, one accumulator at a time (lo then hi of each component)
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t lo[2][FC];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 Y[1][FC];
        {
          uint32_t y[32];
          tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tm_zero32(lane_addr + (uint32_t)((c * 2 + h) * 32));   // next product
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[0][j] = tm_get(y, j);
        }
        inv_fft_pp<1, GT>(Y, b0, b1, lay, t, twi, bar);
        if (h == 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            lo[0][j] = round_u32(Y[0][j].x);
            lo[1][j] = round_u32(Y[0][j].y);
          }
        } else if (e != 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const int i = t + FT * j;
            acc[c * N + i] += lo[0][j] + (round_u32(Y[0][j].x) << 16);
            acc[c * N + i + FH] += lo[1][j] + (round_u32(Y[0][j].y) << 16);
          }
        }
      }
    }
    gsync<GT>(bar);   // the group's accumulator updates before the next step's digits
  }
  // the last step's zeroing stores (tm_zero32) must land before the columns are freed
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(512u));
  }
  if (!valid) return;
  if (s1 < L) {
    for (int k = t; k < 2 * N; k += FT) acc_io[bq * 2 * N + k] = acc[k];
  } else {
    uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
    for (int k = t; k < N; k += FT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
    if (t == 0) o[N] = acc[N];
  }
}

// One IVP (CDEMUX) / VP (CMUX) tree level on the TMEM path: the four
// sub-ciphertexts 4k .. 4k+3 of an item share its GGSW (levels with m >= 4).
template <int MODE>
__global__ void __launch_bounds__(2 * FT, 2)
    level_fft_tm_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                        const uint32_t *__restrict__ in, uint32_t *out, int m, Gadget g,
                        const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  extern __shared__ uint4 smem_raw[];
  FSmemTM &sm = *reinterpret_cast<FSmemTM *>(smem_raw);
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT;
  const FLay lay = make_flay(t);
  const int64_t cta = blockIdx.x, per_item = m / TMC, item = cta / per_item;
  const int64_t sub0 = (cta % per_item) * TMC + grp * 2;   // this thread's subs sub0, sub0 + 1
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const double2 *G = ggsw + (size_t)gidx[item] * ggsw_f;
  // inputs: IVP -- the CTA's 4 consecutive sub-ciphertexts are one contiguous 32 KB
  // run, fetched by one bulk copy; VP -- c1 - c0 with every 16-byte load in flight at once
  // (the element-wise copy loop it replaces exposed one global latency per word: 26% of
  // the kernel's stall samples, profiles/r02b_ncu_lvl.txt)
  if (MODE != MODE_IVP_LEVEL) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint4 *a = reinterpret_cast<uint4 *>(sm.acc[grp * 2 + q]);
      const int64_t sub = sub0 + q;
      const uint4 *c0 = reinterpret_cast<const uint4 *>(in + (item * 2 * m + sub) * 2 * N);
      const uint4 *c1 = reinterpret_cast<const uint4 *>(in + (item * 2 * m + m + sub) * 2 * N);
      uint4 v0[2 * N / 4 / FT], v1[2 * N / 4 / FT];
#pragma unroll
      for (int k = 0; k < 2 * N / 4 / FT; ++k) {
        v0[k] = c0[t + FT * k];
        v1[k] = c1[t + FT * k];
      }
#pragma unroll
      for (int k = 0; k < 2 * N / 4 / FT; ++k)
        a[t + FT * k] = make_uint4(v1[k].x - v0[k].x, v1[k].y - v0[k].y, v1[k].z - v0[k].z, v1[k].w - v0[k].w);
    }
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    mbar_init(&sm.in_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE == MODE_IVP_LEVEL) {
      const uint32_t *d = in + (item * m + (cta % per_item) * TMC) * 2 * N;
      mbar_expect_tx(&sm.in_full, (uint32_t)sizeof(sm.acc));
      bulk_g2s(&sm.acc[0][0], d, (uint32_t)sizeof(sm.acc), &sm.in_full);
    }
  }
  const uint32_t lane_addr = tm_alloc_cta(sm);   // (its barrier also publishes the inputs)
  if (MODE == MODE_IVP_LEVEL) mbar_wait(&sm.in_full, 0);
  uint32_t key_phase = 0;
  tm_ext_product(
      sm, G, g, grp, t, lay, twf, twi, lane_addr, key_phase,
      [&](int q, int c, int i) { return decomp_prep(sm.acc[grp * 2 + q][c * N + i], g); },
      [&](int q, int c, int i, uint32_t v) {
        const int64_t sub = sub0 + q;
        if (MODE == MODE_IVP_LEVEL) {
          // CDEMUX (hw/lut.py:113-119, 294-313): hi = C (*) d, lo = d - hi
          out[(item * 2 * m + m + sub) * 2 * N + c * N + i] = v;
          out[(item * 2 * m + sub) * 2 * N + c * N + i] = sm.acc[grp * 2 + q][c * N + i] - v;
        } else {
          // CMUX (hw/lut.py:130-136, 233-247): next = c0 + C (*) (c1 - c0)
          const uint32_t *c0 = in + (item * 2 * m + sub) * 2 * N;
          out[(item * m + sub) * 2 * N + c * N + i] = c0[c * N + i] + v;
        }
      });
  tm_free_cta(sm);
}

// Global -> shared copies of a ciphertext with every 16-byte load in flight at once
// (element-wise copy loops exposed one global latency per word in the level kernels).
template <int WORDS, int NT>
__device__ __forceinline__ void ld_vec(uint32_t *dst, const uint32_t *src, int tid) {
  constexpr int V = WORDS / 4 / NT;
  static_assert(V * 4 * NT == WORDS, "ld_vec shape");
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  uint4 *d4 = reinterpret_cast<uint4 *>(dst);
  uint4 r[V];
#pragma unroll
  for (int k = 0; k < V; ++k) r[k] = s4[tid + NT * k];
#pragma unroll
  for (int k = 0; k < V; ++k) d4[tid + NT * k] = r[k];
}
template <int WORDS, int NT>   // dst = c1 - c0
__device__ __forceinline__ void ld_vec_diff(uint32_t *dst, const uint32_t *c1, const uint32_t *c0, int tid) {
  constexpr int V = WORDS / 4 / NT;
  static_assert(V * 4 * NT == WORDS, "ld_vec shape");
  const uint4 *a4 = reinterpret_cast<const uint4 *>(c1), *b4 = reinterpret_cast<const uint4 *>(c0);
  uint4 *d4 = reinterpret_cast<uint4 *>(dst);
  uint4 x[V], y[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    x[k] = a4[tid + NT * k];
    y[k] = b4[tid + NT * k];
  }
#pragma unroll
  for (int k = 0; k < V; ++k) d4[tid + NT * k] = make_uint4(x[k].x - y[k].x, x[k].y - y[k].y, x[k].z - y[k].z, x[k].w - y[k].w);
}

// One IVP / VP tree level on mode 5's layout (`level_fft_td_kernel`, FFT mode >= 5): the
// CTA's 4 sub-ciphertexts 4k .. 4k + 3 of an item share its GGSW; two decoupled halves
// of two lane-paired ciphertexts each (blind_rotate_fft_td_kernel's mapping), one
// product per CTA.  The inputs (IVP: one bulk copy) and the first key slice are
// fetched at once; per-thread twiddles from the global table.
template <int MODE>
__global__ void __launch_bounds__(256, 2)
    level_fft_td_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                        const uint32_t *__restrict__ in, uint32_t *out, int m, Gadget g,
                        const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  constexpr int GT = 128;
  extern __shared__ uint4 smem_raw[];
  FSmemTDT<2, 1> &sm = *reinterpret_cast<FSmemTDT<2, 1> *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int half = warp >> 2, hbar = 1 + half;
  const int q = 2 * half + (lane & 1), t = 16 * (warp & 3) + (lane >> 1);
  FLay lay = make_flay(t);
  if (q & 1) {
    lay.a ^= 4u;
    lay.m ^= 4u;
    lay.b ^= 4u;
  }
  const int64_t cta = blockIdx.x, per_item = m / 4, item = cta / per_item;
  const int64_t sub0 = (cta % per_item) * 4, sub = sub0 + q;
  const int lv = (int)g.levels;
  const size_t ggsw_f = (size_t)2 * lv * 2 * 2 * FC * FT;
  const double2 *G = ggsw + (size_t)gidx[item] * ggsw_f;
  constexpr uint32_t kSliceBytes = 2 * 2 * FC * FT * sizeof(double2);
  uint32_t *acc = sm.acc[q];   // TP_ACC stride
  if (MODE != MODE_IVP_LEVEL) {
    const uint32_t *c0 = in + (item * 2 * m + sub) * 2 * N, *c1 = in + (item * 2 * m + m + sub) * 2 * N;
    ld_vec_diff<2 * N, FT>(acc, c1, c0, t);
  }
  if (tid == 0) {
    mbar_init(&sm.key_full[0], 1);
    mbar_init(&sm.in_full, 1);
    sm.key_cnt[0] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&sm.key_full[0], kSliceBytes);
    bulk_g2s(sm.key[0], G, kSliceBytes, &sm.key_full[0]);
    if (MODE == MODE_IVP_LEVEL) {   // 4 contiguous sub-ciphertexts into the padded slots
      mbar_expect_tx(&sm.in_full, 4 * 2 * N * 4);
#pragma unroll 1
      for (int k = 0; k < 4; ++k)
        bulk_g2s(sm.acc[k], in + (item * m + sub0 + k) * 2 * N, 2 * N * 4, &sm.in_full);
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  if (MODE == MODE_IVP_LEVEL) mbar_wait(&sm.in_full, 0);
  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = sm.scr[q];
  const bool leader = lane == 0 && (warp & 3) == 0;
  uint32_t pw[2][FC];
#pragma unroll 1
  for (int r = 0; r < 2 * lv; ++r) {
    // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
    const int comp = r < lv ? 1 : 0;
    const int tt = r < lv ? r : r - lv;
    const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
    double2 x[1][FC];
    if (tt == 0) {
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        pw[0][j] = decomp_prep(acc[comp * N + i], g);
        pw[1][j] = decomp_prep(acc[comp * N + i + FH], g);
      }
    }
#pragma unroll
    for (int j = 0; j < FC; ++j)
      x[0][j] = make_double2(u2d_minus((pw[0][j] >> sh) & g.mask, dig_off),
                             u2d_minus((pw[1][j] >> sh) & g.mask, dig_off));
    fwd_fft_hk<1, GT, false, false>(x, fscr, lay, t, twf, hbar);
    mbar_wait(&sm.key_full[0], (uint32_t)r & 1u);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      const uint32_t a = lane_addr + (uint32_t)(ch * 32);
      uint32_t y[32];
      tm_ld32(a, y);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const double2 k = sm.key[0][(ch * FC + j) * FT + t];
        double2 u = tm_get(y, j);
        u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
        u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
        tm_st_acc(a + 4 * j, u);
      }
    }
    gsync<GT>(hbar);   // the half is past the slice; the second half fetches the next row's
    if (leader) {
      __threadfence_block();
      if (atomicAdd(&sm.key_cnt[0], 1u) == 1u) {
        sm.key_cnt[0] = 0;
        if (r + 1 < 2 * lv) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&sm.key_full[0], kSliceBytes);
          bulk_g2s(sm.key[0], G + (size_t)(r + 1) * (2 * 2 * FC * FT), kSliceBytes, &sm.key_full[0]);
        }
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    uint32_t lo[2][FC];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 Y[1][FC];
      {
        uint32_t y[32];
        tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) Y[0][j] = tm_get(y, j);
      }
      // (scratch-reuse barrier after the inverse's last levels, none after the last inverse:
      // blind_rotate_fft_td_kernel's HWB_TD_ONEINV placement)
      inv_fft_hk<1, GT, false, false>(Y, fscr, lay, t, twi, hbar);
      if (!(c == 1 && h == 1)) gsync<GT>(hbar);
      if (h == 0) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          lo[0][j] = round_u32(Y[0][j].x);
          lo[1][j] = round_u32(Y[0][j].y);
        }
      } else {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            const int i = t + FT * j + FH * u2;
            const uint32_t v = lo[u2][j] + (round_u32(u2 ? Y[0][j].y : Y[0][j].x) << 16);
            if (MODE == MODE_IVP_LEVEL) {
              // CDEMUX (hw/lut.py:113-119, 294-313): hi = C (*) d, lo = d - hi
              out[(item * 2 * m + m + sub) * 2 * N + c * N + i] = v;
              out[(item * 2 * m + sub) * 2 * N + c * N + i] = acc[c * N + i] - v;
            } else {
              // CMUX (hw/lut.py:130-136, 233-247): next = c0 + C (*) (c1 - c0)
              const uint32_t *c0 = in + (item * 2 * m + sub) * 2 * N;
              out[(item * m + sub) * 2 * N + c * N + i] = c0[c * N + i] + v;
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(256u));
  }
}

// One tree level of vertical packing on the FFT path (cmux_kernel's MODE_IVP_LEVEL /
// MODE_VP_LEVEL): block = item * m + sub, GGSW gidx[item].
template <int MODE>
__global__ void __launch_bounds__(FT, 1)
    level_fft_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                     const uint32_t *__restrict__ in, uint32_t *out, int m, Gadget g,
                     const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  extern __shared__ uint4 smem_raw[];
  FSmem &sm = *reinterpret_cast<FSmem *>(smem_raw);
  const int64_t b = blockIdx.x, item = b / m, sub = b % m;
  const int t = threadIdx.x;
  const FLay lay = make_flay(t);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * FC * FT;
  const double2 *G = ggsw + (size_t)gidx[item] * ggsw_f;
  uint32_t key_phase = 0;
  if (MODE == MODE_IVP_LEVEL) {
    // CDEMUX (hw/lut.py:113-119, 294-313): hi = C (*) d, lo = d - hi
    const uint32_t *d = in + (item * m + sub) * 2 * N;
    uint32_t *o_lo = out + (item * 2 * m + sub) * 2 * N, *o_hi = out + (item * 2 * m + m + sub) * 2 * N;
    ld_vec<2 * N, FT>(sm.acc[0], d, t);
    fft_smem_init(sm, t);
    __syncthreads();
    fft_ext_product(
        sm, G, g, t, lay, twf, twi, key_phase, [&](int c, int i) { return decomp_prep(sm.acc[0][c * N + i], g); },
        [&](int c, int i, uint32_t v) {
          o_hi[c * N + i] = v;
          o_lo[c * N + i] = sm.acc[0][c * N + i] - v;
        });
  } else {
    // CMUX (hw/lut.py:130-136, 233-247): next = c0 + C (*) (c1 - c0)
    const uint32_t *c0 = in + (item * 2 * m + sub) * 2 * N, *c1 = in + (item * 2 * m + m + sub) * 2 * N;
    uint32_t *o = out + (item * m + sub) * 2 * N;
    ld_vec_diff<2 * N, FT>(sm.acc[0], c1, c0, t);
    fft_smem_init(sm, t);
    __syncthreads();
    fft_ext_product(
        sm, G, g, t, lay, twf, twi, key_phase, [&](int c, int i) { return decomp_prep(sm.acc[0][c * N + i], g); },
        [&](int c, int i, uint32_t v) { o[c * N + i] = c0[c * N + i] + v; });
  }
}

// ---------------------------------------------------------------------------
// Latency-mode FFT ladder (small batches, N = 1024): one ciphertext per CTA of 2l
// groups of 64 threads.  Per CMUX step: (1) thread 0 stages the key rows
// r in [l, 2l) (l x 32 KB, one TMA bulk copy) while groups 0..3 load their rows
// r < l straight into registers; (2) group r extracts digit row r and runs its
// forward transform (named barrier per group); (3) the 2l digit spectra meet in
// shared memory; (4) group q = (c, h) < 4 forms accumulator Y[c][h] = sum_r D_r K[r][c][h]
// and inverse-transforms it; (5) the h = 1 groups hand their rounded words to
// the h = 0 groups, which update the accumulator.  Bit-identical to the
// throughput ladder (same exact rounding).

#ifndef HWB_FFT_LAT_PF
#define HWB_FFT_LAT_PF 3   // steps of L2 prefetch ahead in the FFT latency ladder
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

struct FSmemL {
  uint32_t acc[2 * 2 * FH];
  double2 D[FDR][FH];                 // digit spectra, layout-B position j * 64 + t
  double2 scr[FDR][FH];               // per-group transpose scratch (scr[4] also hands over the hi words)
  double2 key[FDR / 2][2][2][FC * FT];   // key rows [l, 2l) of the step (TMA)
  uint64_t key_full;
};

__global__ void __launch_bounds__(FDR * FT, 1)
    blind_rotate_fft_lat_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                                const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L,
                                Gadget g, const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemL &sm = *reinterpret_cast<FSmemL *>(smem_raw);
  const int lv = (int)g.levels, ng = 2 * lv, nt = ng * FT;
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT;
  const int64_t b = blockIdx.x;
  uint32_t *acc = sm.acc;
  const FLay lay = make_flay(t);
  const uint32_t *row = lwe_in + b * (int64_t)(L + 1);
  {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = tid; k < 2 * N; k += nt) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t ggsw_f = (size_t)2 * lv * 2 * 2 * FC * FT;
  const size_t row_f = (size_t)2 * 2 * FC * FT;   // double2 per key row r
  const uint32_t smem_rows_bytes = (uint32_t)(lv * row_f * sizeof(double2));
  const double dig_off = 4503599627370496.0 + (double)g.half;
  const int mc = grp >> 1, mh = grp & 1;          // accumulator of a MAC group (grp < 4)
  uint32_t key_phase = 0;
  uint32_t *hi_words = reinterpret_cast<uint32_t *>(sm.scr[4]);   // [2 comps][N]
#pragma unroll 1
  for (int s = 0; s < L; ++s) {
    const int e = mod_switch(row[s], LOG2M);   // X^{a~_s}
    if (e == 0) continue;
    const double2 *G = ggsw + (size_t)s * ggsw_f;
    if (tid == 0) {
      // a lone ciphertext streams the whole key from HBM: pull the GGSW of step
      // s + HWB_FFT_LAT_PF into L2 now (one bulk prefetch), so its loads hit L2
      if (s + HWB_FFT_LAT_PF < L)
        bulk_prefetch_l2(ggsw + (size_t)(s + HWB_FFT_LAT_PF) * ggsw_f, (uint32_t)(ggsw_f * sizeof(double2)));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&sm.key_full, smem_rows_bytes);
      bulk_g2s(&sm.key[0][0][0][0], G + lv * row_f, smem_rows_bytes, &sm.key_full);
    }
    double2 kreg[FDR / 2][FC];
    if (grp < 4) {
#pragma unroll
      for (int r = 0; r < FDR / 2; ++r)
        if (r < lv) {
          const double2 *src = G + r * row_f + (mc * 2 + mh) * (FC * FT) + t;
#pragma unroll
          for (int j = 0; j < FC; ++j) kreg[r][j] = __ldg(src + j * FT);
        }
    }
    // digit row grp (hw/tfhe.py:290-298: rows 0..l-1 = digits of b, l..2l-1 of a)
    {
      const int comp = grp < lv ? 1 : 0;
      const int tt = grp < lv ? grp : grp - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + comp * N;
      double2 x[FC];
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        const uint32_t p0 = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
        const uint32_t p1 = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        x[j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
      }
      fwd_fft(x, sm.scr[grp], lay, t, twf, NoHook(), 1 + grp);
#pragma unroll
      for (int j = 0; j < FC; ++j) sm.D[grp][j * FT + t] = x[j];
    }
    __syncthreads();
    double2 Y[FC];
    if (grp < 4) {
#pragma unroll
      for (int j = 0; j < FC; ++j) Y[j] = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < FDR / 2; ++r)
        if (r < lv) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const double2 x = sm.D[r][j * FT + t], k = kreg[r][j];
            Y[j].x = fma(x.x, k.x, fma(-x.y, k.y, Y[j].x));
            Y[j].y = fma(x.x, k.y, fma(x.y, k.x, Y[j].y));
          }
        }
      mbar_wait(&sm.key_full, key_phase);
#pragma unroll 1
      for (int r = lv; r < 2 * lv; ++r) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const double2 x = sm.D[r][j * FT + t], k = sm.key[r - lv][mc][mh][j * FT + t];
          Y[j].x = fma(x.x, k.x, fma(-x.y, k.y, Y[j].x));
          Y[j].y = fma(x.x, k.y, fma(x.y, k.x, Y[j].y));
        }
      }
      inv_fft(Y, sm.scr[grp], lay, t, twi, 1 + grp);
      if (mh == 1) {
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          hi_words[mc * N + i] = round_u32(Y[j].x) << 16;
          hi_words[mc * N + i + FH] = round_u32(Y[j].y) << 16;
        }
      }
    }
    __syncthreads();
    if (grp < 4 && mh == 0) {
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        acc[mc * N + i] += round_u32(Y[j].x) + hi_words[mc * N + i];
        acc[mc * N + i + FH] += round_u32(Y[j].y) + hi_words[mc * N + i + FH];
      }
    }
    key_phase ^= 1u;
    __syncthreads();
  }
  uint32_t *o = lwe_out + b * (int64_t)(N + 1);
  for (int k = tid; k < N; k += nt) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
  if (tid == 0) o[N] = acc[N];
}

// ---------------------------------------------------------------------------
// Cluster latency ladder (single ciphertexts, N = 1024): one ciphertext per
// CLUSTER of 2l CTAs (64 threads each), so the 192 KB of key per CMUX step streams
// through 2l SMs instead of one (a lone CTA gets ~27 GB/s).  CTA r
// owns digit row r: it TMA-stages its key row K[r] (32 KB, one step ahead, double
// buffered), transforms its digits and forms the four partial products
// P_r[q] = D_r K[r][q] in its shared memory; CTA q < 4 (accumulator (c, h) = (q/2,
// q%2)) sums P_0..P_{2l-1}[q] over distributed shared memory, inverse-transforms
// it and rounds; CTA 2c + 1 hands its high words to CTA 2c, which owns the
// master copy of component c and adds both; every CTA then copies the component
// its digit row decomposes.  Three cluster barriers per step.  Bit-identical.

namespace cg = cooperative_groups;

struct FSmemC {
  // owner q: the partial products P_r[q] of every CTA r (<= 8), double-buffered by
  // executed-step parity: a push for step s+2 is causally after every owner's read of
  // step s (it needs this CTA's component of step s+1, whose owners needed every
  // CTA's push of step s+1, each issued after that CTA's owner section of step s);
  // a single buffer would let a push for s+1 overwrite a slow owner of the OTHER
  // component still reading step s
  double2 Pin[2][FDR + 2][FC * FT];
  double2 key[2][4][FC * FT];     // K[r] of the current / next step (TMA, double buffered)
  double2 scr[FH];                // transpose scratch
  uint32_t acc[2 * FH];           // this CTA's copy of component c(r); owners add their words into it
  uint64_t key_full[2];
  uint64_t pin_full[2], acc_full; // arrival of pushed data (st.async / red.async complete_tx)
};

__device__ __forceinline__ uint32_t mapa_u32(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// remote shared-memory store that completes `bytes` on the remote CTA's mbarrier
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(v.x), "d"(v.y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
// remote shared-memory add (mod 2^32) that completes 4 bytes on the remote mbarrier
__device__ __forceinline__ void red_async_add_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.add.u32 [%0], %1, [%2];" ::"r"(
                   raddr),
               "r"(v), "r"(rbar)
               : "memory");
}
// (CTA-scope acquire: the pushed data is async-proxy shared-memory traffic completed
// through this CTA's own mbarrier; a cluster-scope acquire adds an L1 invalidate,
// CCTL.IVALL, to every poll -- 13% of the cluster ladder's stall samples)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
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

// Exchanges are pushes to the consumer: st.async / red.async remote operations that
// complete bytes on the receiver's mbarrier, so a CTA waits only for the data it
// consumes -- no cluster barrier, no memory fence.  Two hops per step: every CTA r
// pushes P_r[q] to accumulator CTA q; CTA q = (c, h) sums, inverse-transforms,
// rounds and ADDS its words (lo, or hi << 16) into every copy of component c
// (red.async.add, mod 2^32 -- the two halves commute).  Buffer reuse is safe by
// causality: a producer's next push depends on the receiver having consumed the
// previous one.  (Measured variants: a master CTA per component combining the
// halves, 3 hops, 2.60 ms per cfg2 PBS; one owner per component doing both
// inverses, 2.85 ms.)
__global__ void __launch_bounds__(FT, 1)
    blind_rotate_fft_cl_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                               const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                               const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemC &sm = *reinterpret_cast<FSmemC *>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int lv = (int)g.levels, ng = 2 * lv;
  const int r = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / ng;
  const int t = threadIdx.x;
  const FLay lay = make_flay(t);
  const uint32_t *row = lwe_in + b * (int64_t)(L + 1);
  const int comp = r < lv ? 1 : 0;                  // component this digit row decomposes
  const int tt = r < lv ? r : r - lv;
  const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
  const double dig_off = 4503599627370496.0 + (double)g.half;
  const bool owner = r < 4;
  const int mc = r >> 1, mh = r & 1;                // accumulator (c, h) of an owner
  const size_t ggsw_f = (size_t)2 * lv * 2 * 2 * FC * FT;
  const size_t row_f = (size_t)2 * 2 * FC * FT;
  constexpr uint32_t kRowBytes = 2 * 2 * FC * FT * sizeof(double2);
  const uint32_t pin_bytes = (uint32_t)(ng * FC * FT * sizeof(double2)), delta_bytes = (uint32_t)(2 * N * 4);
  {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);       // X^-b~
    for (int i = t; i < N; i += FT) sm.acc[i] = rot_read<N>(tp + comp * N, i, e);
  }
  auto next_step = [&](int s) {   // zero-exponent steps are exact no-ops
    while (s < L && mod_switch(row[s], LOG2M) == 0) ++s;
    return s;
  };
  if (t == 0) {
    mbar_init(&sm.key_full[0], 1);
    mbar_init(&sm.key_full[1], 1);
    mbar_init(&sm.pin_full[0], 1);
    mbar_init(&sm.pin_full[1], 1);
    mbar_init(&sm.acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (owner) {
      mbar_expect_tx(&sm.pin_full[0], pin_bytes);
      mbar_expect_tx(&sm.pin_full[1], pin_bytes);
    }
    mbar_expect_tx(&sm.acc_full, delta_bytes);
  }
  int s = next_step(0);
  if (t == 0 && s < L) {
    mbar_expect_tx(&sm.key_full[0], kRowBytes);
    bulk_g2s(&sm.key[0][0][0], ggsw + (size_t)s * ggsw_f + r * row_f, kRowBytes, &sm.key_full[0]);
  }
  uint32_t pin_dst[4], pin_bar[4];                  // my slot in owner q's Pin[0] and its mbarrier
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    pin_dst[q] = mapa_u32(&sm.Pin[0][r][0], (uint32_t)q);
    pin_bar[q] = mapa_u32(&sm.pin_full[0], (uint32_t)q);
  }
  constexpr uint32_t kPinBufBytes = (uint32_t)sizeof(sm.Pin[0]);
  uint32_t kphase[2] = {0u, 0u}, pphase[2] = {0u, 0u}, aphase = 0u;
  int buf = 0, pb = 0;                              // key buffer, Pin buffer (executed-step parity)
  cluster.sync();                                   // barriers initialised and armed cluster-wide
  bool first = true;
  while (s < L) {
    const int e = mod_switch(row[s], LOG2M);        // X^{a~_s}
    const int sn = next_step(s + 1);
    if (!first) {
      mbar_wait_cluster(&sm.acc_full, aphase);      // both halves of the previous step's product added
      aphase ^= 1u;
      __syncthreads();                              // every thread past the wait before re-arming
      if (t == 0) mbar_expect_tx(&sm.acc_full, delta_bytes);
    }
    first = false;
    if (t == 0 && sn < L) {
      // the other key buffer's last reader (step s - 1) is done
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&sm.key_full[buf ^ 1], kRowBytes);
      bulk_g2s(&sm.key[buf ^ 1][0][0], ggsw + (size_t)sn * ggsw_f + r * row_f, kRowBytes, &sm.key_full[buf ^ 1]);
    }
    double2 x[FC];
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const int i = t + FT * j;
      const uint32_t p0 = decomp_prep(rot_read<N>(sm.acc, i, e) - sm.acc[i], g);
      const uint32_t p1 = decomp_prep(rot_read<N>(sm.acc, i + FH, e) - sm.acc[i + FH], g);
      x[j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
    }
    fwd_fft(x, sm.scr, lay, t, twf);
    mbar_wait(&sm.key_full[buf], kphase[buf]);
    kphase[buf] ^= 1u;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const double2 k = sm.key[buf][q][j * FT + t];
        st_async_f64x2(pin_dst[q] + pb * kPinBufBytes + (uint32_t)((j * FT + t) * sizeof(double2)),
                       make_double2(fma(x[j].x, k.x, -x[j].y * k.y), fma(x[j].x, k.y, x[j].y * k.x)),
                       pin_bar[q] + pb * (uint32_t)sizeof(uint64_t));
      }
    if (owner) {
      mbar_wait_cluster(&sm.pin_full[pb], pphase[pb]);   // P_0..P_{2l-1}[q] have landed
      pphase[pb] ^= 1u;
      double2 Y[FC];
#pragma unroll
      for (int j = 0; j < FC; ++j) Y[j] = sm.Pin[pb][0][j * FT + t];
#pragma unroll
      for (int rr = 1; rr < FDR + 2; ++rr)
        if (rr < ng) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const double2 v = sm.Pin[pb][rr][j * FT + t];
            Y[j].x += v.x;
            Y[j].y += v.y;
          }
        }
      __syncthreads();                              // Pin[pb] consumed by every thread
      if (t == 0) mbar_expect_tx(&sm.pin_full[pb], pin_bytes);
      inv_fft(Y, sm.scr, lay, t, twi);
      const uint32_t shift = mh ? 16u : 0u;
      uint32_t w0[FC], w1[FC];
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        w0[j] = round_u32(Y[j].x) << shift;
        w1[j] = round_u32(Y[j].y) << shift;
      }
      // add this half of component mc into every copy of it (CTAs r0 .. r0 + l - 1)
      const int r0 = mc == 1 ? 0 : lv;
#pragma unroll 1
      for (int rr = r0; rr < r0 + lv; ++rr) {
        const uint32_t dst = mapa_u32(sm.acc, (uint32_t)rr), bar = mapa_u32(&sm.acc_full, (uint32_t)rr);
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          red_async_add_u32(dst + (uint32_t)(i * 4), w0[j], bar);
          red_async_add_u32(dst + (uint32_t)((i + FH) * 4), w1[j], bar);
        }
      }
    }
    buf ^= 1;
    pb ^= 1;
    s = sn;
  }
  if (!first) {
    mbar_wait_cluster(&sm.acc_full, aphase);        // the last step's halves
  }
  // extraction (coefficient 0): a' from component 0 (CTA l), b' = b[0] from component 1 (CTA 0)
  cluster.sync();
  if (r == lv) {
    uint32_t *o = lwe_out + b * (int64_t)(N + 1);
    for (int k = t; k < N; k += FT) o[k] = k == 0 ? sm.acc[0] : 0u - sm.acc[N - k];
    if (t == 0) o[N] = cluster.map_shared_rank(sm.acc, 0)[0];
  }
  cluster.sync();                                   // remote reads done before any CTA exits
}

// Four-CTA cluster variant: CTA q = (c, h) transforms ALL 2l digit rows itself (2l
// groups of 64 threads), multiplies them by its key slices K[r][c][h] (48 KB per
// step, TMA, double-buffered), sums the partials in shared memory, inverse-transforms
// Y[c][h] and adds its rounded words into every CTA's copy of component c
// (red.async).  The only cross-SM traffic per step is 4 KB per CTA pair (vs 48 KB of
// partial products into each accumulator CTA above); a "free" mbarrier (one remote
// arrival per peer after its digit extraction) keeps a fast CTA from adding step
// s+1's words before a slow peer has read step s's component.
struct FSmemC4 {
  uint32_t acc[2][2 * FH];            // both components
  double2 key[2][FDR][FC * FT];       // K[r][c][h] of the current / next step, r < 2l
  double2 part[FDR][FC * FT];         // per-row partial products
  double2 scr[FDR][FH];               // per-group transpose scratch
  uint64_t key_full[2], acc_full, free_bar;
};

__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}

__global__ void __launch_bounds__(FDR * FT, 1)
    blind_rotate_fft_cl4_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                                const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                                const double2 *__restrict__ twf, const double2 *__restrict__ twi) {
  constexpr int N = 2 * FH;
  constexpr int LOG2M = 11;
  extern __shared__ uint4 smem_raw[];
  FSmemC4 &sm = *reinterpret_cast<FSmemC4 *>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int lv = (int)g.levels, ng = 2 * lv;
  const int q = (int)cluster.block_rank(), qc = q >> 1, qh = q & 1;
  const int64_t b = blockIdx.x / 4;
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT;
  const FLay lay = make_flay(t);
  const uint32_t *row = lwe_in + b * (int64_t)(L + 1);
  const int comp = grp < lv ? 1 : 0;
  const int tt = grp < lv ? grp : grp - lv;
  const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
  const double dig_off = 4503599627370496.0 + (double)g.half;
  const size_t ggsw_f = (size_t)2 * lv * 2 * 2 * FC * FT;
  const size_t row_f = (size_t)2 * 2 * FC * FT;
  constexpr uint32_t kSliceBytes = FC * FT * sizeof(double2);   // one (r, c, h) key polynomial
  const uint32_t key_bytes = (uint32_t)(ng * kSliceBytes), delta_bytes = (uint32_t)(4 * N * 4);
  {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);       // X^-b~
    for (int k = tid; k < 2 * N; k += ng * FT) sm.acc[k >> 10][k & (N - 1)] = rot_read<N>(tp + (k >> 10) * N, k & (N - 1), e);
  }
  auto next_step = [&](int s) {
    while (s < L && mod_switch(row[s], LOG2M) == 0) ++s;
    return s;
  };
  auto stage_key = [&](int s, int bf) {             // thread 0: the 2l slices (r, qc, qh) of GGSW s
    mbar_expect_tx(&sm.key_full[bf], key_bytes);
    const double2 *G = ggsw + (size_t)s * ggsw_f + (qc * 2 + qh) * (FC * FT);
    for (int r = 0; r < ng; ++r) bulk_g2s(&sm.key[bf][r][0], G + r * row_f, kSliceBytes, &sm.key_full[bf]);
  };
  if (tid == 0) {
    mbar_init(&sm.key_full[0], 1);
    mbar_init(&sm.key_full[1], 1);
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.free_bar, 3);                     // one arrival per peer per step
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&sm.acc_full, delta_bytes);
  }
  int s = next_step(0);
  if (tid == 0 && s < L) stage_key(s, 0);
  uint32_t acc_dst[4], acc_bar[4], free_rbar[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    acc_dst[p] = mapa_u32(&sm.acc[qc][0], (uint32_t)p);
    acc_bar[p] = mapa_u32(&sm.acc_full, (uint32_t)p);
    free_rbar[p] = mapa_u32(&sm.free_bar, (uint32_t)p);
  }
  uint32_t kphase[2] = {0u, 0u}, aphase = 0u, fphase = 0u;
  int buf = 0;
  cluster.sync();
  bool first = true;
  while (s < L) {
    const int e = mod_switch(row[s], LOG2M);
    const int sn = next_step(s + 1);
    if (!first) {
      mbar_wait_cluster(&sm.acc_full, aphase);      // all four quarters of the previous product added
      aphase ^= 1u;
    }
    __syncthreads();
    if (tid == 0) {
      if (!first) mbar_expect_tx(&sm.acc_full, delta_bytes);
      if (sn < L) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_key(sn, buf ^ 1);
      }
    }
    first = false;
    // group grp: digit row grp of component comp
    double2 x[FC];
    {
      const uint32_t *ac = sm.acc[comp];
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int i = t + FT * j;
        const uint32_t p0 = decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
        const uint32_t p1 = decomp_prep(rot_read<N>(ac, i + FH, e) - ac[i + FH], g);
        x[j] = make_double2(u2d_minus((p0 >> sh) & g.mask, dig_off), u2d_minus((p1 >> sh) & g.mask, dig_off));
      }
    }
    __syncthreads();                                // every group has read the component
    if (tid == 0)
      for (int p = 0; p < 4; ++p)
        if (p != q) mbar_arrive_remote(free_rbar[p]);   // peers may add this step's words now
    fwd_fft(x, sm.scr[grp], lay, t, twf, NoHook(), 1 + grp);
    mbar_wait(&sm.key_full[buf], kphase[buf]);
    kphase[buf] ^= 1u;
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const double2 k = sm.key[buf][grp][j * FT + t];
      sm.part[grp][j * FT + t] = make_double2(fma(x[j].x, k.x, -x[j].y * k.y), fma(x[j].x, k.y, x[j].y * k.x));
    }
    __syncthreads();
    if (grp == 0) {
      double2 Y[FC];
#pragma unroll
      for (int j = 0; j < FC; ++j) Y[j] = sm.part[0][j * FT + t];
#pragma unroll
      for (int r = 1; r < FDR; ++r)
        if (r < ng) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const double2 v = sm.part[r][j * FT + t];
            Y[j].x += v.x;
            Y[j].y += v.y;
          }
        }
      inv_fft(Y, sm.scr[0], lay, t, twi, 1);
      const uint32_t shift = qh ? 16u : 0u;
      uint32_t w0[FC], w1[FC];
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        w0[j] = round_u32(Y[j].x) << shift;
        w1[j] = round_u32(Y[j].y) << shift;
      }
      mbar_wait_cluster(&sm.free_bar, fphase);      // every peer has read this step's component
#pragma unroll 1
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const int i = t + FT * j;
          red_async_add_u32(acc_dst[p] + (uint32_t)(i * 4), w0[j], acc_bar[p]);
          red_async_add_u32(acc_dst[p] + (uint32_t)((i + FH) * 4), w1[j], acc_bar[p]);
        }
    }
    fphase ^= 1u;
    buf ^= 1;
    s = sn;
  }
  if (!first) mbar_wait_cluster(&sm.acc_full, aphase);
  if (q == 0) {
    uint32_t *o = lwe_out + b * (int64_t)(N + 1);
    for (int k = tid; k < N; k += ng * FT) o[k] = k == 0 ? sm.acc[0][0] : 0u - sm.acc[0][N - k];
    if (tid == 0) o[N] = sm.acc[1][0];
  }
  cluster.sync();
}

// ---------------------------------------------------------------------------
// FP64 FFT ladder at N = 2048 (FFT2): the folded polynomial has H = 1024 points
// (z_i = a_i + i a_{i+1024}, a polynomial mod Y^1024 - i).  Its first
// Cooley-Tukey stage (level 0: z_k +/- w0 z_{k+512}, w0 = e^{i pi/4}) is formed
// while the digits are read, after which half g is an independent 512-point
// merged-twist transform -- the N = 1024 machinery on 64 threads, with the
// twiddles of the subtree under block (1, g) (tables fft2_*[g], c_ftw row 1 + g).
// One ciphertext per CTA of 128 threads (group g = half g).  The inverse runs the
// two 512-point inverses, then the level-0 Gentleman-Sande stage across the
// halves through shared memory.  Thread (g, t) owns folded points g 512 + t + 64 j,
// i.e. coefficients g 512 + t + 64 j and + 1024 of the product.
// Digits: l <= 2 rows per component, base_log <= 15 (signed 16-bit), biased
// halfwords [row][j][g][t]: word g holds positions k + 512 (2g) (low) and
// k + 512 (2g + 1) (high), k = t + 64 j.

constexpr int F2R = 4;   // digit rows 2l staged per product (l <= 2)

#ifndef HWB_FFT2_ONFLY
#define HWB_FFT2_ONFLY 0
#endif
struct FSmem2 {
  uint32_t acc[2 * 4 * FH];        // working ciphertext (a, b), N = 2048
  double2 scr[2][FH];              // per-half transpose scratch
#if !HWB_FFT2_ONFLY
  uint32_t dig[F2R * FC * 2 * FT]; // the product's digits (biased halfwords)
#endif
  double2 key[2 * 2 * 2 * FC * FT];   // the digit's key slice [c][h][g][j][t] (64 KB, TMA)
  uint64_t key_full;
};

// (X, Y) -> X + w0 Y (g = 0) or X - w0 Y (g = 1), w0 in tangent form
__device__ __forceinline__ double2 fft2_first(double2 X, double2 Y, int grp) {
  const double2 w = c_fw0[0];
  const double ux = fma(-w.y, Y.y, Y.x), uy = fma(w.y, Y.x, Y.y);
  const double c = grp ? -w.x : w.x;
  return make_double2(fma(c, ux, X.x), fma(c, uy, X.y));
}

template <typename Prep, typename Sink>
__device__ __forceinline__ void fft2_ext_product(FSmem2 &sm, const double2 *__restrict__ G, const Gadget &g,
                                                 int grp, int t, const FLay &lay, const double2 *__restrict__ twf,
                                                 const double2 *__restrict__ twi, uint32_t &key_phase, Prep &&prep,
                                                 Sink &&sink) {
  constexpr uint32_t kSliceBytes = 2 * 2 * 2 * FC * FT * sizeof(double2);
  const int lv = (int)g.levels;
  const double dig_off = 4503599627370496.0 + (double)g.half;   // 2^52 + beta/2
#if !HWB_FFT2_ONFLY
  // the decomposition once per product: thread (grp, t) forms the prep words of
  // positions k + 512 q, q = 2 grp + {0, 1}
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pw[2 * FC];
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const int k = t + FT * j;
      pw[2 * j] = prep(c, k + FH * (2 * grp));
      pw[2 * j + 1] = prep(c, k + FH * (2 * grp + 1));
    }
#pragma unroll 1
    for (int tt = 0; tt < lv; ++tt) {
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const int r = (c == 1 ? 0 : lv) + tt;
#pragma unroll
      for (int j = 0; j < FC; ++j)
        sm.dig[((r * FC + j) * 2 + grp) * FT + t] = ((pw[2 * j] >> sh) & g.mask) | (((pw[2 * j + 1] >> sh) & g.mask) << 16);
    }
  }
  __syncthreads();
#endif
  double2 Y[2][2][FC];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < FC; ++j) Y[c][h][j] = make_double2(0.0, 0.0);
#pragma unroll 1
  for (int r = 0; r < 2 * lv; ++r) {
    const double2 *gr = G + (size_t)r * (2 * 2 * 2 * FC * FT);
    double2 x[FC];
#if HWB_FFT2_ONFLY
    {
      // digits straight from the accumulator (no staging buffer: 16 KB more L1 for the
      // per-thread twiddle tables)
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int k = t + FT * j;
        const uint32_t d0 = (prep(comp, k) >> sh) & g.mask, d1 = (prep(comp, k + FH) >> sh) & g.mask;
        const uint32_t d2 = (prep(comp, k + 2 * FH) >> sh) & g.mask, d3 = (prep(comp, k + 3 * FH) >> sh) & g.mask;
        const double2 zk = make_double2(u2d_minus(d0, dig_off), u2d_minus(d2, dig_off));
        const double2 zh = make_double2(u2d_minus(d1, dig_off), u2d_minus(d3, dig_off));
        x[j] = fft2_first(zk, zh, grp);
      }
    }
#else
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const uint32_t w0 = sm.dig[((r * FC + j) * 2) * FT + t], w1 = sm.dig[((r * FC + j) * 2 + 1) * FT + t];
      const double2 zk = make_double2(u2d_minus(w0 & 0xFFFFu, dig_off), u2d_minus(w1 & 0xFFFFu, dig_off));
      const double2 zh = make_double2(u2d_minus(w0 >> 16, dig_off), u2d_minus(w1 >> 16, dig_off));
      x[j] = fft2_first(zk, zh, grp);
    }
#endif
    auto stage_key = [&] {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full, kSliceBytes);
        bulk_g2s(sm.key, gr, kSliceBytes, &sm.key_full);
      }
    };
    // CTA-wide barriers: the hook runs once both halves are past the previous MAC
    fwd_fft(x, sm.scr[grp], lay, t, twf, stage_key, 0, 1 + grp);
    mbar_wait(&sm.key_full, key_phase);
    key_phase ^= 1u;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          const double2 k = sm.key[(((c * 2 + h) * 2 + grp) * FC + j) * FT + t];
          double2 &y = Y[c][h][j];
          y.x = fma(x[j].x, k.x, fma(-x[j].y, k.y, y.x));
          y.y = fma(x[j].x, k.y, fma(x[j].y, k.x, y.y));
        }
  }
  __syncthreads();   // every thread has finished reading the last key slice
  inv_fft_k<4>(&Y[0][0], sm.key + grp * 4 * FH, lay, t, twi, 1 + grp);
  // level-0 Gentleman-Sande stage across the halves: (X, Y) -> (X + Y, (X - Y) conj(w0))
  double2 *xb = sm.key;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < FC; ++j) xb[((grp * 4 + q) * FC + j) * FT + t] = (&Y[0][0])[q][j];
  __syncthreads();
  const double2 wi = c_fw0[1];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const double2 o = xb[(((1 - grp) * 4 + q) * FC + j) * FT + t];
      double2 &y = (&Y[0][0])[q][j];
      if (grp == 0)
        y = make_double2(y.x + o.x, y.y + o.y);
      else
        y = cmul(make_double2(o.x - y.x, o.y - y.y), wi);
    }
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < FC; ++j) {
      const int f = grp * FH + t + FT * j;   // folded point: coefficients f and f + 1024
      sink(c, f, round_u32(Y[c][0][j].x) + (round_u32(Y[c][1][j].x) << 16));
      sink(c, f + 2 * FH, round_u32(Y[c][0][j].y) + (round_u32(Y[c][1][j].y) << 16));
    }
}

// BSK/GGSW polynomials [count][2048] u32 -> FFT2 domain [count][2 halves][2 g][FC][FT]
// double2 (scaled 1/1024): 128 threads per polynomial, both key halves in lockstep.
__global__ void __launch_bounds__(2 * FT) bsk_to_fft2_kernel(const uint32_t *__restrict__ in, double2 *out,
                                                              const double2 *__restrict__ twf0,
                                                              const double2 *__restrict__ twf1) {
  __shared__ double2 scr[2][2 * FH];
  const int grp = threadIdx.x / FT, t = threadIdx.x % FT;
  const int64_t poly = blockIdx.x;
  const uint32_t *a = in + poly * (4 * FH);
  const FLay lay = make_flay(t);
  double2 x[2][FC];
#pragma unroll
  for (int j = 0; j < FC; ++j) {
    const int k = t + FT * j;
    double lo[4], hi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {   // positions k, k + 512, k + 1024, k + 1536
      const int64_t gword = (int32_t)a[k + q * FH];
      const int64_t l16 = ((gword + 32768) & 0xFFFF) - 32768;
      lo[q] = (double)l16;
      hi[q] = (double)((gword - l16) >> 16);
    }
    x[0][j] = fft2_first(make_double2(lo[0], lo[2]), make_double2(lo[1], lo[3]), grp);
    x[1][j] = fft2_first(make_double2(hi[0], hi[2]), make_double2(hi[1], hi[3]), grp);
  }
  fwd_fft_k<2>(x, scr[grp], lay, t, grp ? twf1 : twf0, 1 + grp);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 *o = out + (poly * 2 + h) * (2 * FC * FT) + grp * (FC * FT);
#pragma unroll
    for (int j = 0; j < FC; ++j)
      o[j * FT + t] = make_double2(x[h][j].x * (1.0 / (2 * FH)), x[h][j].y * (1.0 / (2 * FH)));
  }
}

// The CMUX ladder on the FFT2 path: as blind_rotate_fft_kernel (PBS: mod switch to
// 2N = 4096, TV X^-b~, steps [s0, s1) per launch, extraction at the end; !PBS: the
// per-item rotation ladders of vertical packing), one ciphertext per 128-thread CTA.
template <bool PBS>
__global__ void __launch_bounds__(2 * FT, 1)
    blind_rotate_fft2_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                             const int32_t *__restrict__ exps, const uint32_t *__restrict__ lwe_in,
                             const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                             const double2 *__restrict__ twf0, const double2 *__restrict__ twf1,
                             const double2 *__restrict__ twi0, const double2 *__restrict__ twi1, uint32_t *acc_io,
                             int s0, int s1, int64_t B) {
  constexpr int N = 4 * FH;
  constexpr int LOG2M = 12;
  constexpr int NT = 2 * FT;
  extern __shared__ uint4 smem_raw[];
  FSmem2 &sm = *reinterpret_cast<FSmem2 *>(smem_raw);
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT;
  const int64_t b = blockIdx.x;
  uint32_t *acc = sm.acc;
  const FLay lay = make_flay(t);
  const double2 *twf = grp ? twf1 : twf0, *twi = grp ? twi1 : twi0;
  const uint32_t *row = PBS ? lwe_in + b * (int64_t)(L + 1) : nullptr;
  if (PBS && s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? b * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = tid; k < 2 * N; k += NT) {
      const int c = k >= N, i = k & (N - 1);
      acc[k] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = tid; k < 2 * N; k += NT) acc[k] = acc_io[b * 2 * N + k];
  }
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t key_phase = 0;
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * 2 * FC * FT;   // double2 per GGSW
  uint32_t a_nx = PBS ? row[s0] : 0u;   // the next step's mask word, loaded a step ahead
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    int e, gi = s;
    if (PBS) {
      e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
      a_nx = row[s + 1];
    } else {
      e = (int)((-(int64_t)exps[b * L + s]) % (2 * N));
      if (e < 0) e += 2 * N;
      if (gidx) gi = gidx[b * L + s];
    }
    if (e == 0 || gi < 0) continue;
    fft2_ext_product(
        sm, ggsw + (size_t)gi * ggsw_f, g, grp, t, lay, twf, twi, key_phase,
        [&](int c, int i) {   // digits of (acc X^e - acc), straight from the accumulator
          const uint32_t *ac = acc + c * N;
          return decomp_prep(rot_read<N>(ac, i, e) - ac[i], g);
        },
        [&](int c, int i, uint32_t v) { acc[c * N + i] += v; });
    __syncthreads();
  }
  if (!PBS || s1 < L) {
    for (int k = tid; k < 2 * N; k += NT) acc_io[b * 2 * N + k] = acc[k];
    return;
  }
  uint32_t *o = lwe_out + b * (int64_t)(N + 1);
  for (int k = tid; k < N; k += NT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
  if (tid == 0) o[N] = acc[N];
}

// ---------------------------------------------------------------------------
// N = 2048 TMEM ladder (`blind_rotate_fft2_td_kernel`, FFT mode >= 1 at N = 2048).
//
// The register FFT2 ladder above holds one ciphertext's 4 spectral accumulators in
// registers (2 ciphertexts per SM) and stages a 64 KB key slice per ciphertext.  Here
// the accumulators live in TMEM (64 KB per ciphertext: 4 per SM) and one CTA of 16
// warps runs 4 ciphertexts as two decoupled lane-paired pairs (mode 5's layout at
// N = 2048): warp w carries pair P = w >> 3, half g = (w >> 2) & 1 of the folded
// 1024-point transform, positions t = 16 (w & 3) + (lane >> 1), ciphertext
// q = 2 P + (lane & 1).  All 4 ciphertexts share each TMA-staged 64 KB key slice
// (released per pair; the second release issues the next row's copy), a lane pair
// reads each key value and twiddle at one address, and every scheduler (w % 4) runs
// one warp of each (pair, half).  The level-0 stage joins the halves: forward, each
// thread forms it from the four quarter positions of its digits; inverse, the halves
// exchange their values through the transpose scratch.

constexpr int T2C = 4;   // ciphertexts per CTA
#ifndef HWB_T2_MACUNROLL   // instruction-cache footprint switches (as HWB_TD_*)
#define HWB_T2_MACUNROLL 4
#endif
#ifndef HWB_T2_INVUNROLL
#define HWB_T2_INVUNROLL 2
#endif
constexpr int kT2MacUnroll = HWB_T2_MACUNROLL, kT2InvUnroll = HWB_T2_INVUNROLL;
#ifndef HWB_T2_LATEBAR
#define HWB_T2_LATEBAR 0
#endif
constexpr int T2_COMP = 4 * FH + 48;   // words per padded component (t2_off)

struct FSmem2TD {
  // working ciphertexts (a, b), N = 2048, padded (t2_off): each 512-coefficient block
  // starts 8 banks after the previous one (offsets 0, 8, 40, 48 words), odd ciphertexts 16
  // banks further (the row stride).  A lane quad's 4 (ciphertext, half) accesses then land on
  // 4 different bank octets both in the digit reads (halves 1024 apart) and in the
  // accumulator update after the inverse (halves 512 apart; 4-way conflicts before:
  // profiles/r02c_smem_lines_f2td.txt)
  uint32_t acc[T2C][2 * T2_COMP + 16];
  double2 scr[T2C][2][FH];         // transpose / level-0 scratch per (ciphertext, half)
  // the row's key slice [c][h][g][j][t] (64 KB, 8 TMA chunks of 8 KB at a stride of
  // 8 KB + 64 B, so a lane quad's two halves hit different bank groups)
  double2 key[8 * (FC * FT + 4)];
  double2 twf[2][kTwc * FT + 4], twi[2][kTwc * FT + 4];   // compact per-thread twiddles of half g (+64 B)
  uint64_t key_full;
  uint32_t key_cnt;
  uint32_t tmem_slot;
};

static_assert(sizeof(FSmem2TD) <= 232448, "FSmem2TD exceeds the 227 KB of shared memory a CTA can opt into");
__device__ __forceinline__ int t2_off(int i) { return i + 8 * ((i >> 9) & 1) + 40 * (i >> 10); }
__device__ __forceinline__ int t2_pad(int c, int i) { return c * T2_COMP + t2_off(i); }
// rot_read on a t2_pad-ded component
__device__ __forceinline__ uint32_t rot_read_t2(const uint32_t *poly, int i, int e) {
  constexpr int N = 4 * FH;
  const int src = (i - e) & (2 * N - 1), idx = src & (N - 1);
  const uint32_t val = poly[t2_off(idx)];
  return src >= N ? 0u - val : val;
}

template <bool SINGLE>
__global__ void __launch_bounds__(16 * 32, 1)
    blind_rotate_fft2_td_kernel(const double2 *__restrict__ ggsw, const uint32_t *__restrict__ lwe_in,
                                const uint32_t *__restrict__ tv, int tv_per_item, uint32_t *lwe_out, int L, Gadget g,
                                const double2 *__restrict__ twf0, const double2 *__restrict__ twf1,
                                const double2 *__restrict__ twi0, const double2 *__restrict__ twi1, uint32_t *acc_io,
                                int s0_arg, int s1_arg, int64_t B, uint32_t *progress) {
  constexpr int N = 4 * FH;
  constexpr int LOG2M = 12;
  constexpr int GT = 256;   // threads per pair (named barrier)
  // SINGLE: one launch for the whole ladder, CTA = (segment, group) in segment-major order,
  // s1_arg = the segment length (blind_rotate_fft_td_kernel has the protocol)
  constexpr int kPerCta = T2C;
  const uint32_t groups = SINGLE ? (uint32_t)((B + T2C - 1) / T2C) : gridDim.x;
  const uint32_t seg = blockIdx.x / groups, grp = blockIdx.x % groups;
  const int s0 = SINGLE ? (int)seg * s1_arg : s0_arg;
  const int s1 = SINGLE ? (s0 + s1_arg < L ? s0 + s1_arg : L) : s1_arg;
  extern __shared__ uint4 smem_raw[];
  FSmem2TD &sm = *reinterpret_cast<FSmem2TD *>(smem_raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // lane quad (4m .. 4m + 3) = position t for both ciphertexts of the pair (lane bit 0)
  // and both halves (lane bit 1): key and twiddle addresses shared by lane bit 0, the
  // halves' exchanges (level-0 digits forward, level-0 stage inverse) by shuffles
  const int pr = warp >> 3, hf = (lane >> 1) & 1, bar = 1 + pr;
  const int q = 2 * pr + (lane & 1), t = 8 * (warp & 7) + (lane >> 2), tq = hf * FT + t;
  FLay lay = make_flay(t);
  {   // the quad's four (ciphertext, half) buffers on distinct 16-byte bank groups
    const uint32_t xo = (uint32_t)((q & 1) * 4 + hf * 2);
    lay.a ^= xo;
    lay.m ^= xo;
    lay.b ^= xo;
  }
  const int64_t bb = (int64_t)grp * T2C + q;
  const bool valid = bb < B;
  const int64_t bq = valid ? bb : B - 1;
  const uint32_t *row = lwe_in + bq * (int64_t)(L + 1);
  uint32_t *acc = sm.acc[q];   // row stride = 16 mod 32 words: odd ciphertexts 16 banks over
  if (SINGLE && seg > 0) {   // the group's previous segment
    if (tid == 0) {
      uint32_t done, spins = 0;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(done) : "l"(progress + grp) : "memory");
        if (done >= seg) break;
        __nanosleep(256);
        if (++spins > (1u << 24)) __trap();
      }
    }
    __syncthreads();
  }
  if (s0 == 0) {
    const int bt = mod_switch(row[L], LOG2M);
    const uint32_t *tp = tv + (tv_per_item ? bq * 2 * N : 0);
    const int e = (2 * N - bt) & (2 * N - 1);   // X^-b~
    for (int k = tq; k < 2 * N; k += 2 * FT) {
      const int c = k >= N, i = k & (N - 1);
      acc[t2_pad(c, i)] = rot_read<N>(tp + c * N, i, e);
    }
  } else {
    for (int k = tq; k < 2 * N; k += 2 * FT) acc[t2_pad(k >= N, k & (N - 1))] = __ldcg(&acc_io[bq * 2 * N + k]);
  }
  for (int k = tid; k < kTwc * FT; k += 16 * 32) {
    const int fs = twc_full<true>(k / FT) * FT + k % FT, is = twc_full<false>(k / FT) * FT + k % FT;
    sm.twf[0][k] = twf0[fs];
    sm.twf[1][k] = twf1[fs];
    sm.twi[0][k] = twi0[is];
    sm.twi[1][k] = twi1[is];
  }
  constexpr uint32_t kSliceBytes = 2 * 2 * 2 * FC * FT * sizeof(double2);
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * 2 * FC * FT;
  const int lv = (int)g.levels;
  auto key_chunks = [&](const double2 *src) {   // 8 chunks [c][h][g] of 8 KB
#pragma unroll 1
    for (int c8 = 0; c8 < 8; ++c8)
      bulk_g2s(sm.key + c8 * (FC * FT + 4), src + c8 * FC * FT, FC * FT * sizeof(double2), &sm.key_full);
  };
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    sm.key_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&sm.key_full, kSliceBytes);   // the first row's slice
    key_chunks(ggsw + (size_t)s0 * ggsw_f);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane_addr = sm.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll
  for (int k = 0; k < 4; ++k) tm_zero32(lane_addr + (uint32_t)(k * 32));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t key_phase = 0;
  const double dig_off = 4503599627370496.0 + (double)g.half;
  double2 *fscr = sm.scr[q][hf];
  const bool leader = lane == 0 && (warp & 7) == 0;   // warps 0 and 8
  auto release = [&](int s_, int r_) {   // the second pair to finish the slice fetches the next
    if (!leader) return;
    __threadfence_block();
    if (atomicAdd(&sm.key_cnt, 1u) == 1u) {
      sm.key_cnt = 0;
      const int nr = r_ + 1 < 2 * lv ? r_ + 1 : 0, ns = r_ + 1 < 2 * lv ? s_ : s_ + 1;
      if (ns < s1) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.key_full, kSliceBytes);
        key_chunks(ggsw + (size_t)ns * ggsw_f + (size_t)nr * (2 * 2 * 2 * FC * FT));
      }
    }
  };
  const double2 wi0 = c_fw0[1];
  uint32_t a_nx = row[s0];   // the next step's mask word, loaded a step ahead
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const int e = mod_switch(a_nx, LOG2M);   // X^{a~_s}
    a_nx = row[s + 1];
    uint32_t nxt[FC];   // packed digits of the component's next row (two-row gadgets)
#pragma unroll 1
    for (int r = 0; r < 2 * lv; ++r) {
      // digit order (hw/tfhe.py:290-298): rows 0..l-1 = digits of b, l..2l-1 of a
      const int comp = r < lv ? 1 : 0;
      const int tt = r < lv ? r : r - lv;
      const uint32_t sh = g.base_log * (uint32_t)(lv - 1 - tt);
      const uint32_t *ac = acc + t2_pad(comp, 0);
      double2 x[1][FC];
      // two-row gadgets (cfg4): the second row's digits are extracted with the first's
      // and kept packed (one word per position) -- the decomposition once per component
      const bool reuse = lv == 2 && tt == 1;
#pragma unroll
      for (int j = 0; j < FC; ++j) {
        const int k = t + FT * j;
        // this half's two quarter positions k + 512 (2 hf + {0, 1}); the partner half
        // (lane ^ 2) forms the other two
        uint32_t own = 0;
        if (reuse) {
          own = nxt[j];
        } else {
          uint32_t o1 = 0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int i = k + FH * (2 * hf + u);
            const uint32_t pw = decomp_prep(rot_read_t2(ac, i, e) - ac[i + 8 * u + 40 * hf], g);   // = t2_off(i)
            own |= ((pw >> sh) & g.mask) << (16 * u);
            o1 |= ((pw >> (sh - g.base_log)) & g.mask) << (16 * u);   // row tt + 1 (used iff lv == 2)
          }
          nxt[j] = o1;
        }
        const uint32_t par = __shfl_xor_sync(0xffffffffu, own, 2);
        const uint32_t q01 = hf ? par : own, q23 = hf ? own : par;
        const double2 zk = make_double2(u2d_minus(q01 & 0xFFFFu, dig_off), u2d_minus(q23 & 0xFFFFu, dig_off));
        const double2 zh = make_double2(u2d_minus(q01 >> 16, dig_off), u2d_minus(q23 >> 16, dig_off));
        x[0][j] = fft2_first(zk, zh, hf);
      }
      // (no trailing barrier on the second transpose: the release barrier after the MAC
      // precedes the next write into fscr)
      fwd_fft_hk<1, GT, true, false>(x, fscr, lay, t, sm.twf[hf], bar, 1 + hf);
      mbar_wait(&sm.key_full, key_phase);
      key_phase ^= 1u;
#pragma unroll kT2MacUnroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t a = lane_addr + (uint32_t)(ch * 32);
        uint32_t y[32];
        tm_ld32(a, y);   // zeroed at the end of the previous product
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < FC; ++j) {
#if HWB_X_NOKEY
          const double2 k = make_double2(1.0 + j + ch, 0.5 * r);
#else
          const double2 k = sm.key[(ch * 2 + hf) * (FC * FT + 4) + j * FT + t];
#endif
          double2 u = tm_get(y, j);
          u.x = fma(x[0][j].x, k.x, fma(-x[0][j].y, k.y, u.x));
          u.y = fma(x[0][j].x, k.y, fma(x[0][j].y, k.x, u.y));
          tm_st_acc(a + 4 * j, u);
        }
      }
      gsync<GT>(bar);   // the pair is past the slice
      release(s, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // inverse transforms, one accumulator at a time: the half's 512-point inverse, then
    // the level-0 Gentleman-Sande stage across the halves, (X, Y) -> (X + Y, (X - Y) conj(w0))
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t lo[2][FC] = {};   // (defined on every path: a rolled h loop carries it)
#pragma unroll kT2InvUnroll
      for (int h = 0; h < 2; ++h) {
        double2 Y[1][FC];
        {
          uint32_t y[32];
          tm_ld32(lane_addr + (uint32_t)((c * 2 + h) * 32), y);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tm_zero32(lane_addr + (uint32_t)((c * 2 + h) * 32));   // next product
#pragma unroll
          for (int j = 0; j < FC; ++j) Y[0][j] = tm_get(y, j);
        }
#if HWB_T2_LATEBAR   // the scratch-reuse barrier after the inverse's last levels and the level-0 stage
        inv_fft_hk<1, GT, true, false>(Y, fscr, lay, t, sm.twi[hf], bar, 1 + hf);
#else
        inv_fft_hk<1, GT, true>(Y, fscr, lay, t, sm.twi[hf], bar, 1 + hf);
#endif
#pragma unroll
        for (int j = 0; j < FC; ++j) {   // the partner half's value at the same position (lane ^ 2)
          double2 o;
          o.x = __shfl_xor_sync(0xffffffffu, Y[0][j].x, 2);
          o.y = __shfl_xor_sync(0xffffffffu, Y[0][j].y, 2);
          Y[0][j] = hf == 0 ? make_double2(Y[0][j].x + o.x, Y[0][j].y + o.y)
                            : cmul(make_double2(o.x - Y[0][j].x, o.y - Y[0][j].y), wi0);
        }
#if HWB_T2_LATEBAR
        if (!(c == 1 && h == 1)) gsync<GT>(bar);   // (the end-of-step barrier follows the last inverse)
#endif
        if (h == 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            lo[0][j] = round_u32(Y[0][j].x);
            lo[1][j] = round_u32(Y[0][j].y);
          }
        } else if (e != 0) {
#pragma unroll
          for (int j = 0; j < FC; ++j) {
            const int f = hf * FH + t + FT * j;   // folded point: coefficients f and f + 1024
            uint32_t *af = acc + c * T2_COMP + f + 8 * hf;   // t2_pad(c, f), f < 1024 in block hf
            af[0] += lo[0][j] + (round_u32(Y[0][j].x) << 16);
            af[2 * FH + 40] += lo[1][j] + (round_u32(Y[0][j].y) << 16);   // t2_pad(c, f + 1024)
          }
        }
      }
    }
    gsync<GT>(bar);   // the pair's accumulator updates before the next step's digits
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_slot), "r"(512u));
  }
  if (valid) {
    if (s1 < L) {
      for (int k = tq; k < 2 * N; k += 2 * FT) acc_io[bq * 2 * N + k] = acc[t2_pad(k >= N, k & (N - 1))];
    } else {
      uint32_t *o = lwe_out + bq * (int64_t)(N + 1);
      for (int k = tq; k < N; k += 2 * FT) o[k] = k == 0 ? acc[0] : 0u - acc[t2_pad(0, N - k)];
      if (tq == 0) o[N] = acc[t2_pad(1, 0)];
    }
  }
  if (SINGLE) {   // publish after every thread's accumulator stores
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      // (recomputed from blockIdx: nothing of the protocol stays live across the steps)
      const uint32_t groups2 = (uint32_t)((B + kPerCta - 1) / kPerCta);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(progress + blockIdx.x % groups2),
                   "r"(blockIdx.x / groups2 + 1)
                   : "memory");
    }
  }
}

// One vertical-packing tree level on the FFT2 path (level_fft_kernel at N = 2048).
template <int MODE>
__global__ void __launch_bounds__(2 * FT, 1)
    level_fft2_kernel(const double2 *__restrict__ ggsw, const int32_t *__restrict__ gidx,
                      const uint32_t *__restrict__ in, uint32_t *out, int m, Gadget g,
                      const double2 *__restrict__ twf0, const double2 *__restrict__ twf1,
                      const double2 *__restrict__ twi0, const double2 *__restrict__ twi1) {
  constexpr int N = 4 * FH;
  constexpr int NT = 2 * FT;
  extern __shared__ uint4 smem_raw[];
  FSmem2 &sm = *reinterpret_cast<FSmem2 *>(smem_raw);
  const int64_t b = blockIdx.x, item = b / m, sub = b % m;
  const int tid = threadIdx.x, grp = tid / FT, t = tid % FT;
  const FLay lay = make_flay(t);
  const double2 *twf = grp ? twf1 : twf0, *twi = grp ? twi1 : twi0;
  const size_t ggsw_f = (size_t)2 * g.levels * 2 * 2 * 2 * FC * FT;
  const double2 *G = ggsw + (size_t)gidx[item] * ggsw_f;
  uint32_t key_phase = 0;
  if (tid == 0) {
    mbar_init(&sm.key_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == MODE_IVP_LEVEL) {
    // CDEMUX (hw/lut.py:113-119, 294-313): hi = C (*) d, lo = d - hi
    const uint32_t *d = in + (item * m + sub) * 2 * N;
    uint32_t *o_lo = out + (item * 2 * m + sub) * 2 * N, *o_hi = out + (item * 2 * m + m + sub) * 2 * N;
    ld_vec<2 * N, NT>(sm.acc, d, tid);
    __syncthreads();
    fft2_ext_product(
        sm, G, g, grp, t, lay, twf, twi, key_phase, [&](int c, int i) { return decomp_prep(sm.acc[c * N + i], g); },
        [&](int c, int i, uint32_t v) {
          o_hi[c * N + i] = v;
          o_lo[c * N + i] = sm.acc[c * N + i] - v;
        });
  } else {
    // CMUX (hw/lut.py:130-136, 233-247): next = c0 + C (*) (c1 - c0)
    const uint32_t *c0 = in + (item * 2 * m + sub) * 2 * N, *c1 = in + (item * 2 * m + m + sub) * 2 * N;
    uint32_t *o = out + (item * m + sub) * 2 * N;
    ld_vec_diff<2 * N, NT>(sm.acc, c1, c0, tid);
    __syncthreads();
    fft2_ext_product(
        sm, G, g, grp, t, lay, twf, twi, key_phase, [&](int c, int i) { return decomp_prep(sm.acc[c * N + i], g); },
        [&](int c, int i, uint32_t v) { o[c * N + i] = c0[c * N + i] + v; });
  }
}

template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) ggsw_to_ntt_kernel(const uint32_t *__restrict__ in,
                                                                      uint32_t *out, Tw tw) {
  constexpr int TPP = Cfg<N>::TPP;
  constexpr int C = N / TPP;
  constexpr int NV = NVar<N>::v;
  __shared__ uint32_t scr[2][N];
  const int64_t poly = blockIdx.x;
  const Who<N> me;
  const int w = me.grp, t = me.t;
  const uint32_t p = c_prime[w].p, pinv = c_prime[w].pinv;
  uint32_t x[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    int32_t s = (int32_t)in[poly * N + t + TPP * j];   // centred coefficient
    int32_t r = s % (int32_t)p;
    x[j] = (uint32_t)(r < 0 ? r + (int32_t)p : r);
  }
  fwd_ntt<N, TPP, -1>(x, scr[w], me.lay, t, w, w ? tw.fwd[1] : tw.fwd[0]);
  const uint32_t k = c_r2ninv[NV][w];
  uint4 *o = reinterpret_cast<uint4 *>(out + (poly * 2 + w) * N);
#pragma unroll
  for (int jq = 0; jq < C / 4; ++jq) {
    uint32_t y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t v = mont_mul(x[4 * jq + q], k, p, pinv);   // (0, 2p)
      y[q] = umin(v, v - p);
    }
    o[jq * TPP + t] = make_uint4(y[0], y[1], y[2], y[3]);
  }
}

// Client-side key product (hw/tfhe.py:69-78 SecretKey._key_mul; used by
// enc_rgsw_batch, hw/tfhe.py:246-263): out[b] = in[b] (*) s + add[b] mod 2^32
// for a small key s given in the NTT domain (key_ntt: [2 primes][N], as
// ggsw_to_ntt lays out one polynomial).  Exact while N * 2^31 * max|s| < P/2.
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) key_mul_kernel(const uint32_t *__restrict__ in,
                                                                  const uint32_t *__restrict__ key_ntt,
                                                                  const uint32_t *__restrict__ add, uint32_t *out,
                                                                  Tw tw) {
  constexpr int TPP = Cfg<N>::TPP, NT = Cfg<N>::THREADS;
  constexpr int C = N / TPP;
  __shared__ uint32_t scr[2][N];
  __shared__ uint32_t ex[2][N];
  const int64_t poly = blockIdx.x;
  const Who<N> me;
  const int w = me.grp, t = me.t;
  const uint32_t p = c_prime[w].p, pinv = c_prime[w].pinv;
  uint32_t x[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    int32_t s = (int32_t)in[poly * N + t + TPP * j];   // centred coefficient
    int32_t r = s % (int32_t)p;
    x[j] = (uint32_t)(r < 0 ? r + (int32_t)p : r);
  }
  fwd_ntt<N, TPP, -1>(x, scr[w], me.lay, t, w, w ? tw.fwd[1] : tw.fwd[0]);
  const uint32_t *ks = key_ntt + (size_t)w * N;
#pragma unroll
  for (int jq = 0; jq < C / 4; ++jq) {
    const uint4 K = __ldg(slice_vec<TPP>(ks, t, jq));
    x[4 * jq + 0] = mont_mul(x[4 * jq + 0], K.x, p, pinv);
    x[4 * jq + 1] = mont_mul(x[4 * jq + 1], K.y, p, pinv);
    x[4 * jq + 2] = mont_mul(x[4 * jq + 2], K.z, p, pinv);
    x[4 * jq + 3] = mont_mul(x[4 * jq + 3], K.w, p, pinv);
  }
  inv_ntt<N, TPP, -1>(x, scr[w], me.lay, t, w, w ? tw.inv[1] : tw.inv[0]);
#pragma unroll
  for (int j = 0; j < C; ++j) ex[w][t + TPP * j] = umin(x[j], x[j] - p);
  __syncthreads();
  for (int i = me.tid; i < N; i += NT) {
    uint32_t v = crt_lift(ex[0][i], ex[1][i]);
    if (add) v += add[poly * N + i];
    out[poly * N + i] = v;
  }
}

// Packing key switch (hw/tfhe.py:390-439 pack_batch), phase 1: for output b
// and a chunk of key rows j, accumulate in the NTT domain
//   sum_{j in chunk} sum_t D_{j,t} * KSK[j,t][c],  D_{j,t}(X) = sum_i digit_t(a^(i)_j) X^i,
// where apolys[b][j][i] = a^(i)_j (the transposed a-stack, zero past k).
// Partial sums (both components, this CTA's prime) go to part[b][chunk][c][prime][N].
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) pack_ks_partial_kernel(
    const uint32_t *__restrict__ apolys, const uint32_t *__restrict__ ksk_ntt, uint32_t *part, int rows_j,
    Gadget gk, Tw tw) {
  constexpr int TPP = Cfg<N>::TPP;
  constexpr int C = N / TPP;
  __shared__ uint32_t scr[2][N];
  const int64_t b = blockIdx.y;
  const int chunk = blockIdx.x, nchunks = gridDim.x;
  const Who<N> me;
  const int w = me.grp, t = me.t;
  const uint32_t p = c_prime[w].p, two_p = 2 * p, pinv = c_prime[w].pinv;
  const uint32_t off = p - gk.half;
  const int L = (int)gk.levels;
  const uint2 *twf = w ? tw.fwd[1] : tw.fwd[0];
  uint32_t a0[C], a1[C], v[C], x[C];
#pragma unroll
  for (int j = 0; j < C; ++j) a0[j] = a1[j] = 0;
  const int j0 = chunk * rows_j, j1 = min(N, j0 + rows_j);
#pragma unroll 1
  for (int jr = j0; jr < j1; ++jr) {
    const uint32_t *src = apolys + ((int64_t)b * N + jr) * N + t;
#pragma unroll
    for (int jj = 0; jj < C; ++jj) v[jj] = decomp_prep(src[TPP * jj], gk);
#pragma unroll 1
    for (int tt = 0; tt < L; ++tt) {
      const uint32_t sh = gk.base_log * (uint32_t)(L - 1 - tt);
#pragma unroll
      for (int jj = 0; jj < C; ++jj) x[jj] = ((v[jj] >> sh) & gk.mask) + off;
      fwd_ntt<N, TPP, -1>(x, scr[w], me.lay, t, w, twf);
      const uint32_t *k0 = ksk_ntt + (((size_t)(jr * L + tt) * 2 + 0) * 2 + w) * N;
      const uint32_t *k1 = ksk_ntt + (((size_t)(jr * L + tt) * 2 + 1) * 2 + w) * N;
#pragma unroll
      for (int jq = 0; jq < C / 4; ++jq) {
        const uint4 K0 = __ldg(slice_vec<TPP>(k0, t, jq));
        const uint4 K1 = __ldg(slice_vec<TPP>(k1, t, jq));
        const uint32_t k0v[4] = {K0.x, K0.y, K0.z, K0.w}, k1v[4] = {K1.x, K1.y, K1.z, K1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t u0 = a0[4 * jq + q] + mont_mul(x[4 * jq + q], k0v[q], p, pinv);
          uint32_t u1 = a1[4 * jq + q] + mont_mul(x[4 * jq + q], k1v[q], p, pinv);
          a0[4 * jq + q] = umin(u0, u0 - two_p);
          a1[4 * jq + q] = umin(u1, u1 - two_p);
        }
      }
    }
  }
  uint4 *o0 = reinterpret_cast<uint4 *>(part + ((((int64_t)b * nchunks + chunk) * 2 + 0) * 2 + w) * N);
  uint4 *o1 = reinterpret_cast<uint4 *>(part + ((((int64_t)b * nchunks + chunk) * 2 + 1) * 2 + w) * N);
#pragma unroll
  for (int jq = 0; jq < C / 4; ++jq) {
    o0[jq * TPP + t] = make_uint4(a0[4 * jq], a0[4 * jq + 1], a0[4 * jq + 2], a0[4 * jq + 3]);
    o1[jq * TPP + t] = make_uint4(a1[4 * jq], a1[4 * jq + 1], a1[4 * jq + 2], a1[4 * jq + 3]);
  }
}

// Packing key switch phase 2: each chunk's partial sum is bounded (rows_j *
// levels * N * beta/2 * 2^31 < P/2), so it is inverse-transformed and CRT-lifted
// on its own; the lifted chunks are added mod 2^32 and
// out[b] = (-acc_a, b_poly - acc_b) (hw/tfhe.py:418-419).
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) pack_ks_finish_kernel(const uint32_t *__restrict__ part,
                                                                         int nchunks,
                                                                         const uint32_t *__restrict__ b_polys,
                                                                         uint32_t *out, Tw tw) {
  constexpr int TPP = Cfg<N>::TPP, NT = Cfg<N>::THREADS;
  constexpr int C = N / TPP;
  constexpr int PER = 2 * N / NT;   // output words per thread
  __shared__ uint32_t scr[2][N];
  __shared__ uint32_t ex[2][2][N];   // [comp][prime][i]
  const int64_t b = blockIdx.x;
  const Who<N> me;
  const int w = me.grp, t = me.t;
  const uint32_t p = c_prime[w].p;
  uint32_t x[C], acc[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) acc[k] = 0;
#pragma unroll 1
  for (int ch = 0; ch < nchunks; ++ch) {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      const uint32_t *src = part + ((((int64_t)b * nchunks + ch) * 2 + c) * 2 + w) * N;
#pragma unroll
      for (int jq = 0; jq < C / 4; ++jq) {
        const uint4 P4 = __ldg(slice_vec<TPP>(src, t, jq));
        x[4 * jq] = P4.x; x[4 * jq + 1] = P4.y; x[4 * jq + 2] = P4.z; x[4 * jq + 3] = P4.w;
      }
      inv_ntt<N, TPP, -1>(x, scr[w], me.lay, t, w, w ? tw.inv[1] : tw.inv[0]);
#pragma unroll
      for (int j = 0; j < C; ++j) ex[c][w][t + TPP * j] = umin(x[j], x[j] - p);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int kk = me.tid + NT * k, c = kk >= N, i = kk & (N - 1);
      acc[k] += crt_lift(ex[c][0][i], ex[c][1][i]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int kk = me.tid + NT * k, c = kk >= N, i = kk & (N - 1);
    out[b * 2 * N + kk] = c ? b_polys[b * N + i] - acc[k] : 0u - acc[k];
  }
}

// RGSW gadget term (hw/tfhe.py:259-262): rows t get m * q/beta^(t+1) on the b
// constant coefficient, rows l+t on the a constant coefficient.
__global__ void rgsw_gadget_kernel(uint32_t *rgsw, const int32_t *__restrict__ bits, int64_t B, int N, int levels,
                                   int base_log) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * levels) return;
  const int64_t b = idx / levels;
  const int t = (int)(idx % levels);
  const uint32_t gt = bits[b] ? (1u << (32 - (t + 1) * base_log)) : 0u;
  uint32_t *g = rgsw + b * (int64_t)(2 * levels) * 2 * N;
  g[((int64_t)t * 2 + 1) * N] += gt;              // row t, component b, coefficient 0
  g[((int64_t)(levels + t) * 2 + 0) * N] += gt;   // row l+t, component a, coefficient 0
}

// hw/tfhe.py:352-361: LWE of coefficient i: a'[j] = a[i-j] (j <= i),
// -a[N+i-j] (j > i); b' = b[i].
template <int N>
__global__ void extract_kernel(const uint32_t *__restrict__ rlwe, uint32_t *lwe, int64_t B, int coeff) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * (N + 1)) return;
  const int64_t b = idx / (N + 1);
  const int k = (int)(idx % (N + 1));
  const uint32_t *a = rlwe + b * 2 * N;
  lwe[idx] = k == N ? a[N + coeff] : (k <= coeff ? a[coeff - k] : 0u - a[N + coeff - k]);
}
// LWE key switch: out[b][c] = (c < n ? 0 : in[b][N]) - sum_{j,t} d[b][j][t] * ksk[j][t][c]
// CTA tile: 64 items x 64 output columns, K chunked by KS_TJ input coefficients.
constexpr int KS_TB = 64, KS_TC = 64, KS_TJ = 4, KS_MAXL = 16;

__global__ void __launch_bounds__(256) keyswitch_kernel(const uint32_t *__restrict__ ksk,
                                                        const uint32_t *__restrict__ in, uint32_t *out,
                                                        int64_t B, int N, int n, Gadget gk) {
  __shared__ int32_t dig[KS_TJ * KS_MAXL][KS_TB];
  __shared__ uint32_t kt[KS_TJ * KS_MAXL][KS_TC];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t b0 = (int64_t)blockIdx.x * KS_TB;
  const int c0 = blockIdx.y * KS_TC;
  const int L = (int)gk.levels;
  const int rows = KS_TJ * L;
  const int ncol = n + 1;
  uint32_t acc[4][4] = {};
  for (int jc = 0; jc < N; jc += KS_TJ) {
    {   // digits of a'_j for 64 items x KS_TJ coefficients: one per thread
      const int item = tid & 63, jj = tid >> 6;
      const int64_t bi = b0 + item;
      uint32_t a = (bi < B && jc + jj < N) ? in[bi * (N + 1) + jc + jj] : 0u;
      const uint32_t v = decomp_prep(a, gk);
      for (int t = 0; t < L; ++t) {
        const uint32_t sh = gk.base_log * (uint32_t)(L - 1 - t);
        dig[jj * L + t][item] = (int32_t)((v >> sh) & gk.mask) - (int32_t)gk.half;
      }
    }
    for (int e = tid; e < rows * KS_TC; e += 256) {
      const int r = e / KS_TC, cc = e % KS_TC;
      const int col = c0 + cc;
      kt[r][cc] = col < ncol ? ksk[((size_t)jc * L + r) * ncol + col] : 0u;
    }
    __syncthreads();
    for (int r = 0; r < rows; ++r) {
      const int4 dv = *reinterpret_cast<const int4 *>(&dig[r][ty * 4]);
      const uint4 kv = *reinterpret_cast<const uint4 *>(&kt[r][tx * 4]);
      const uint32_t d[4] = {(uint32_t)dv.x, (uint32_t)dv.y, (uint32_t)dv.z, (uint32_t)dv.w};
      const uint32_t k[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] += d[i] * k[q];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t bi = b0 + ty * 4 + i;
    if (bi >= B) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = c0 + tx * 4 + q;
      if (col >= ncol) continue;
      out[bi * ncol + col] = (col < n ? 0u : in[bi * (N + 1) + N]) - acc[i][q];
    }
  }
}

// Register-only throughput probe of the shipped modular multiplication: each
// thread runs 8 independent chains; one "RNS modmul" = one Shoup product mod p0
// and one mod p1 (the two-prime counterpart of a 64-bit-prime modmul).  Gives
// P_mm, the denominator of the integer roofline.
__global__ void __launch_bounds__(256) probe_modmul_kernel(uint32_t *sink, int iters) {
  const uint32_t p0 = kP0, p1 = kP1;
  const uint32_t w0 = 123456789u % kP0, w1 = 987654321u % kP1;
  const uint32_t q0 = (uint32_t)(((uint64_t)w0 << 32) / kP0), q1 = (uint32_t)(((uint64_t)w1 << 32) / kP1);
  uint32_t a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = b[k] = threadIdx.x * 8 + k + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a[k] = shoup_mul(a[k], w0, q0, p0);
      b[k] = shoup_mul(b[k], w1, q1, p1);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k] ^ b[k];
  if (s == 0x12345678u) sink[0] = s;
}
// FP64 pipe probe: 8 independent DFMA chains per thread (the FFT ladder's
// denominator P_fp64, in FP64 instructions per second).
__global__ void __launch_bounds__(256) probe_fp64_kernel(uint32_t *sink, int iters) {
  double a[8];
  const double m = 1.0000000001, c = 1e-9 * (threadIdx.x + 1);
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 8 + k + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 0.123) sink[0] = 1u;
}
// ---------------------------------------------------------------------------
// host helpers

static Gadget make_gadget(uint32_t levels, uint32_t base_log) {
  Gadget g;
  const uint32_t total = levels * base_log;
  g.round_add = total < 32 ? (1u << (31 - total)) : 0u;
  g.shift = 32 - total;
  uint32_t h = 0;
  for (uint32_t k = 0; k < levels; ++k) h += (1u << (base_log - 1)) << (base_log * k);
  g.hsum = h;
  g.mask = base_log >= 32 ? 0xFFFFFFFFu : ((1u << base_log) - 1u);
  g.half = 1u << (base_log - 1);
  g.base_log = base_log;
  g.levels = levels;
  return g;
}

// ring and gadget shape shared by both exact formulations
static int check_ring(const hwb_params *p) {
  if (!p) return fail(HWB_EINVAL, "null params");
  if (p->q_bits != 32) return fail(HWB_EINVAL, "q_bits must be 32");
  if (p->k != 1) return fail(HWB_EINVAL, "only GLWE dimension k = 1 is supported");
  if (p->N != 1024 && p->N != 2048) return fail(HWB_EINVAL, "ring degree N must be 1024 or 2048");
  if (p->l < 1 || p->l > 3) return fail(HWB_EINVAL, "gadget levels must be in [1, 3]");
  if (p->base_log < 1 || p->l * p->base_log > 32) return fail(HWB_EINVAL, "gadget spans more than 32 bits");
  return HWB_OK;
}

static int check_glwe(const hwb_params *p) {
  int rc = check_ring(p);
  if (rc) return rc;
  // exactness of the two-prime RNS: max |sum| = 2l * N * beta/2 * 2^31 < P/2
  const double bound = 2.0 * p->l * p->N * std::ldexp(1.0, (int)p->base_log - 1) * std::ldexp(1.0, 31);
  const double halfP = 0.5 * (double)kP0 * (double)kP1;
  if (!(bound < halfP)) return fail(HWB_EINVAL, "gadget/ring too wide for the exact 2-prime NTT (2l N beta/2 2^31 >= P/2)");
  return HWB_OK;
}

static int check_ks(const hwb_params *p) {
  if (p->ks_l < 1 || p->ks_l > (uint32_t)KS_MAXL) return fail(HWB_EINVAL, "key-switch levels must be in [1, 16]");
  if (p->ks_base_log < 1 || p->ks_l * p->ks_base_log > 32) return fail(HWB_EINVAL, "key-switch gadget spans more than 32 bits");
  if (p->n < 1) return fail(HWB_EINVAL, "LWE dimension n must be positive");
  return HWB_OK;
}

static int post_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HWB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HWB_OK;
}

static Tw make_tw(DevState *st, int N) {
  const int nv = N == 1024 ? 0 : 1;
  Tw tw;
  for (int pr = 0; pr < 2; ++pr) {
    tw.fwd[pr] = st->lane_fwd[nv][pr];
    tw.inv[pr] = st->lane_inv[nv][pr];
    tw.inv64[pr] = st->lane_inv64[pr];
  }
  return tw;
}

template <typename K>
static int set_smem(K kernel, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(HWB_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  return HWB_OK;
}


// blocks = items (MODE < MODE_IVP_LEVEL) or items * m (tree levels)
template <int N, int MODE>
static int launch_cmux(const hwb_params *p, DevState *st, const uint32_t *ggsw, const int32_t *gidx,
                       const uint32_t *in, const uint32_t *c1, const int32_t *rot, uint32_t *out,
                       uint32_t *out_hi, int64_t blocks, int m, cudaStream_t s) {
  const size_t smem = sizeof(Smem<N>);
  const size_t words = hwb_ggsw_ntt_words(p);
  const Gadget g = make_gadget(p->l, p->base_log);
  int rc;
  if (g_variant == 1) {
    if ((rc = set_smem(cmux_kernel<N, MODE, 1>, smem))) return rc;
    cmux_kernel<N, MODE, 1><<<(unsigned)blocks, Cfg<N>::THREADS, smem, s>>>(ggsw, words, gidx, in, c1, rot, out,
                                                                            out_hi, m, g, make_tw(st, N));
  } else {
    if ((rc = set_smem(cmux_kernel<N, MODE, 0>, smem))) return rc;
    cmux_kernel<N, MODE, 0><<<(unsigned)blocks, Cfg<N>::THREADS, smem, s>>>(ggsw, words, gidx, in, c1, rot, out,
                                                                            out_hi, m, g, make_tw(st, N));
  }
  return post_launch("cmux_kernel");
}

template <int LV, bool PBS, int MINB>
static int launch_br_lat(const hwb_params *p, DevState *st, const uint32_t *bsk, const int32_t *exps,
                         const uint32_t *lwe_in, const uint32_t *tv, int tv_per_item, uint32_t *acc,
                         uint32_t *lwe_out, int L, int64_t B, cudaStream_t s) {
  constexpr int N = 1024;
  const size_t smem = sizeof(SmemLat<N, LV>);
  int rc;
  if ((rc = set_smem(blind_rotate_lat_kernel<N, LV, PBS, MINB>, smem))) return rc;
  blind_rotate_lat_kernel<N, LV, PBS, MINB><<<(unsigned)B, 128 * LV, smem, s>>>(
      bsk, hwb_ggsw_ntt_words(p), exps, lwe_in, tv, tv_per_item, acc, lwe_out, L,
      make_gadget(p->l, p->base_log), make_tw(st, N));
  return post_launch("blind_rotate_lat_kernel");
}

template <int LV, bool PBS>
static int launch_br_lat_b(const hwb_params *p, DevState *st, const uint32_t *bsk, const int32_t *exps,
                           const uint32_t *lwe_in, const uint32_t *tv, int tv_per_item, uint32_t *acc,
                           uint32_t *lwe_out, int L, int64_t B, cudaStream_t s) {
  if (B <= st->sms)   // one wave of 1-CTA/SM ciphertexts: the lowest-latency build
    return launch_br_lat<LV, PBS, 1>(p, st, bsk, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, B, s);
  return launch_br_lat<LV, PBS, 2>(p, st, bsk, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, B, s);
}

template <int N, bool PBS>
static int launch_br(const hwb_params *p, DevState *st, const uint32_t *bsk, const int32_t *gidx,
                     const int32_t *exps, const uint32_t *lwe_in, const uint32_t *tv, int tv_per_item,
                     uint32_t *acc, uint32_t *lwe_out, int L, int64_t B, cudaStream_t s) {
  const size_t smem = sizeof(Smem<N>);
  const Gadget g = make_gadget(p->l, p->base_log);
  const size_t words = hwb_ggsw_ntt_words(p);
  int rc;
  const int64_t lat_max = g_lat_max_batch >= 0 ? g_lat_max_batch : 3 * (int64_t)st->sms;
  if (N == 1024 && !gidx && B <= lat_max) {   // latency mode (small batches)
    if (p->l == 1) return launch_br_lat_b<1, PBS>(p, st, bsk, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, B, s);
    if (p->l == 2) return launch_br_lat_b<2, PBS>(p, st, bsk, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, B, s);
    return launch_br_lat_b<3, PBS>(p, st, bsk, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, B, s);
  }
  if (g_variant == 1) {
    if ((rc = set_smem(blind_rotate_kernel<N, PBS, 1>, smem))) return rc;
    blind_rotate_kernel<N, PBS, 1><<<(unsigned)B, Cfg<N>::THREADS, smem, s>>>(
        bsk, words, gidx, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, g, make_tw(st, N));
  } else {
    if ((rc = set_smem(blind_rotate_kernel<N, PBS, 0>, smem))) return rc;
    blind_rotate_kernel<N, PBS, 0><<<(unsigned)B, Cfg<N>::THREADS, smem, s>>>(
        bsk, words, gidx, exps, lwe_in, tv, tv_per_item, acc, lwe_out, L, g, make_tw(st, N));
  }
  return post_launch("blind_rotate_kernel");
}

static int keyswitch_launch(const hwb_params *p, const uint32_t *ksk, const uint32_t *in, uint32_t *out,
                            int64_t B, cudaStream_t s) {
  dim3 grid((unsigned)((B + KS_TB - 1) / KS_TB), (unsigned)((p->n + 1 + KS_TC - 1) / KS_TC));
  keyswitch_kernel<<<grid, 256, 0, s>>>(ksk, in, out, B, (int)p->N, (int)p->n,
                                        make_gadget(p->ks_l, p->ks_base_log));
  return post_launch("keyswitch_kernel");
}

// tensor-core key switch: supported shapes and launch (hwb_tc.cuh)
static int check_ks_tc(const hwb_params *p) {
  int rc = check_ks(p);
  if (rc) return rc;
  if (p->ks_base_log > 8) return fail(HWB_EINVAL, "tensor-core key switch needs ks_base_log <= 8 (int8 digits)");
  const int64_t K = (int64_t)p->N * p->ks_l;
  if (p->N < 1 || K % TC_KB) return fail(HWB_EINVAL, "tensor-core key switch needs N*ks_l % 128 == 0");
  if (K * 128 * 255 >= (int64_t)1 << 31) return fail(HWB_EINVAL, "tensor-core key switch: N*ks_l too large for int32 limbs");
  return HWB_OK;
}

static size_t ks_tc_digit_bytes(const hwb_params *p, int64_t B) {
  return (size_t)((B + TC_M - 1) / TC_M) * TC_M * (size_t)p->N * p->ks_l;
}

static int keyswitch_tc_launch(const hwb_params *p, const void *ksk_tc, const uint32_t *in, uint32_t *out,
                               int64_t B, void *digits, cudaStream_t s) {
  const int K = (int)(p->N * p->ks_l);
  const int64_t mtiles = (B + TC_M - 1) / TC_M;
  const int64_t threads = mtiles * TC_M * (K / 16);
  ks_digits_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(in, (uint4 *)digits, B, (int)p->N, K,
                                                                      make_gadget(p->ks_l, p->ks_base_log));
  int rc = post_launch("ks_digits_kernel");
  if (rc) return rc;
  if ((rc = set_smem(keyswitch_tc_kernel, TC_SMEM))) return rc;
  const int nct = (int)((p->n + 1 + TC_COLS - 1) / TC_COLS);
  keyswitch_tc_kernel<<<dim3((unsigned)mtiles, (unsigned)nct), 128, TC_SMEM, s>>>(
      (const uint8_t *)digits, (const uint8_t *)ksk_tc, in, out, B, (int)p->N, (int)p->n, K);
  return post_launch("keyswitch_tc_kernel");
}

}  // namespace hwb
using namespace hwb;

extern "C" {

int hwb_version(void) { return 1; }

int64_t hwb_probe_modmul(uint32_t *sink, int32_t blocks, int32_t iters, void *stream) {
  if (blocks < 1 || iters < 1) return -fail(HWB_EINVAL, "probe needs positive blocks and iters");
  probe_modmul_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters);
  if (post_launch("probe_modmul_kernel")) return -HWB_ECUDA;
  return (int64_t)blocks * 256 * 8 * iters;
}

int hwb_fft_margin(double *out, int reset) {
#if HWB_FFT_MARGIN
  unsigned long long bits = 0;
  if (out) {
    if (cudaMemcpyFromSymbol(&bits, g_fft_margin, sizeof(bits)) != cudaSuccess)
      return fail(HWB_ECUDA, std::string("hwb_fft_margin: ") + cudaGetErrorString(cudaGetLastError()));
    memcpy(out, &bits, sizeof(bits));
  }
  if (reset) {
    bits = 0;
    if (cudaMemcpyToSymbol(g_fft_margin, &bits, sizeof(bits)) != cudaSuccess)
      return fail(HWB_ECUDA, std::string("hwb_fft_margin: ") + cudaGetErrorString(cudaGetLastError()));
  }
  return HWB_OK;
#else
  (void)out;
  (void)reset;
  return fail(HWB_EINVAL, "built without HWB_FFT_MARGIN (use libhwb200_margin.so)");
#endif
}

int64_t hwb_probe_fp64(uint32_t *sink, int32_t blocks, int32_t iters, void *stream) {
  if (blocks < 1 || iters < 1) return -fail(HWB_EINVAL, "probe needs positive blocks and iters");
  probe_fp64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters);
  if (post_launch("probe_fp64_kernel")) return -HWB_ECUDA;
  return (int64_t)blocks * 256 * 8 * iters;
}

int64_t hwb_probe_i8mma(uint32_t *sink, int32_t blocks, int32_t iters, void *stream) {
  if (blocks < 1 || iters < 1) return -fail(HWB_EINVAL, "probe needs positive blocks and iters");
  if (set_smem(probe_i8mma_kernel, TC_SMEM)) return -HWB_ECUDA;
  probe_i8mma_kernel<<<blocks, 128, TC_SMEM, (cudaStream_t)stream>>>(sink, iters);
  if (post_launch("probe_i8mma_kernel")) return -HWB_ECUDA;
  return (int64_t)blocks * iters * (TC_KB / 32) * TC_M * TC_N * 32;
}

int64_t hwb_set_latency_batch(int64_t max_batch) {
  const int64_t prev = g_lat_max_batch;
  if (max_batch >= -1) g_lat_max_batch = max_batch;
  return prev;
}

int hwb_set_variant(int v) {
  if (v < 0 || v > 1) return fail(HWB_EINVAL, "unknown kernel variant");
  g_variant = v;
  return HWB_OK;
}

const char *hwb_last_error(void) { return g_err.c_str(); }

size_t hwb_ggsw_ntt_words(const hwb_params *p) {
  if (!p) return 0;
  return (size_t)2 * p->l * 2 * 2 * p->N;
}

int hwb_ggsw_to_ntt(const hwb_params *p, const uint32_t *ggsw, uint32_t *ggsw_ntt, int64_t count,
                    void *stream) {
  int rc = check_glwe(p);
  if (rc) return rc;
  if (count < 0) return fail(HWB_EINVAL, "negative count");
  if (count == 0) return HWB_OK;
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  const int64_t polys = count * 2 * p->l * 2;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024)
    ggsw_to_ntt_kernel<1024><<<(unsigned)polys, Cfg<1024>::THREADS, 0, s>>>(ggsw, ggsw_ntt, make_tw(st, 1024));
  else
    ggsw_to_ntt_kernel<2048><<<(unsigned)polys, Cfg<2048>::THREADS, 0, s>>>(ggsw, ggsw_ntt, make_tw(st, 2048));
  return post_launch("ggsw_to_ntt_kernel");
}

extern "C++" {
template <int N>
static int launch_mode(int mode, const hwb_params *p, DevState *st, const uint32_t *ggsw, const int32_t *gidx,
                       const uint32_t *in, const uint32_t *c1, const int32_t *rot, uint32_t *out,
                       uint32_t *out_hi, int64_t blocks, int m, cudaStream_t s) {
  switch (mode) {
    case MODE_EXT: return launch_cmux<N, MODE_EXT>(p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
    case MODE_CMUX: return launch_cmux<N, MODE_CMUX>(p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
    case MODE_CDEMUX: return launch_cmux<N, MODE_CDEMUX>(p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
    case MODE_IVP_LEVEL:
      return launch_cmux<N, MODE_IVP_LEVEL>(p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
    default: return launch_cmux<N, MODE_VP_LEVEL>(p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
  }
}
}  // extern "C++"

static int cmux_dispatch(int mode, const hwb_params *p, const uint32_t *ggsw, const int32_t *gidx,
                         const uint32_t *in, const uint32_t *c1, const int32_t *rot, uint32_t *out,
                         uint32_t *out_hi, int64_t B, void *stream, int m = 1) {
  int rc = check_glwe(p);
  if (rc) return rc;
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (m < 1) return fail(HWB_EINVAL, "tree level needs m >= 1 polynomials per item");
  if (B == 0) return HWB_OK;
  const int64_t blocks = B * m;
  if (blocks > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024) return launch_mode<1024>(mode, p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
  return launch_mode<2048>(mode, p, st, ggsw, gidx, in, c1, rot, out, out_hi, blocks, m, s);
}

int hwb_ivp_level(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx, const uint32_t *cur,
                  uint32_t *next, int32_t m, int64_t B, void *stream) {
  return cmux_dispatch(MODE_IVP_LEVEL, p, ggsw_ntt, ggsw_idx, cur, nullptr, nullptr, next, nullptr, B, stream, m);
}

int hwb_vp_level(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx, const uint32_t *cur,
                 uint32_t *next, int32_t m, int64_t B, void *stream) {
  return cmux_dispatch(MODE_VP_LEVEL, p, ggsw_ntt, ggsw_idx, cur, nullptr, nullptr, next, nullptr, B, stream, m);
}

int hwb_monomial_gather(const hwb_params *p, const uint32_t *in, uint32_t *out, const int32_t *exps, int64_t B,
                        void *stream) {
  int rc = check_ring(p);
  if (rc) return rc;
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if (in == out) return fail(HWB_EINVAL, "monomial_gather cannot run in place");
  const int64_t total = B * 2 * p->N;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024)
    monomial_gather_kernel<1024><<<blocks, 256, 0, s>>>(in, out, exps, B);
  else
    monomial_gather_kernel<2048><<<blocks, 256, 0, s>>>(in, out, exps, B);
  return post_launch("monomial_gather_kernel");
}

int hwb_poly_to_ntt(const hwb_params *p, const uint32_t *in, uint32_t *out, int64_t npolys, void *stream) {
  int rc = check_ring(p);
  if (rc) return rc;
  if (npolys < 0) return fail(HWB_EINVAL, "negative count");
  if (npolys == 0) return HWB_OK;
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024)
    ggsw_to_ntt_kernel<1024><<<(unsigned)npolys, Cfg<1024>::THREADS, 0, s>>>(in, out, make_tw(st, 1024));
  else
    ggsw_to_ntt_kernel<2048><<<(unsigned)npolys, Cfg<2048>::THREADS, 0, s>>>(in, out, make_tw(st, 2048));
  return post_launch("poly_to_ntt");
}

int hwb_key_mul(const hwb_params *p, const uint32_t *key_ntt, const uint32_t *in, const uint32_t *add, uint32_t *out,
                int64_t npolys, void *stream) {
  int rc = check_ring(p);
  if (rc) return rc;
  if (npolys < 0) return fail(HWB_EINVAL, "negative count");
  if (npolys == 0) return HWB_OK;
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024)
    key_mul_kernel<1024><<<(unsigned)npolys, Cfg<1024>::THREADS, 0, s>>>(in, key_ntt, add, out, make_tw(st, 1024));
  else
    key_mul_kernel<2048><<<(unsigned)npolys, Cfg<2048>::THREADS, 0, s>>>(in, key_ntt, add, out, make_tw(st, 2048));
  return post_launch("key_mul_kernel");
}

static const int kPackRowsJ = 32;   // key rows j per partial-sum CTA

size_t hwb_pack_ks_workspace_bytes(const hwb_params *p, int64_t B) {
  if (!p || B <= 0) return 0;
  const int64_t chunks = (p->N + kPackRowsJ - 1) / kPackRowsJ;
  return sizeof(uint32_t) * (size_t)B * chunks * 2 * 2 * p->N;
}

int hwb_pack_ks(const hwb_params *p, int32_t levels, int32_t base_log, const uint32_t *ksk_ntt,
                const uint32_t *apolys, const uint32_t *b_polys, uint32_t *out, int64_t B, void *workspace,
                void *stream) {
  int rc = check_ring(p);   // the external-product gadget is not used here: only the packing one
  if (rc) return rc;
  if (levels < 1 || base_log < 1 || levels * base_log > 32)
    return fail(HWB_EINVAL, "packing gadget spans more than 32 bits");
  // exactness of one chunk: rows_j key rows x levels digits x N LWEs x beta/2 x 2^31 < P/2
  const double bound = (double)kPackRowsJ * levels * p->N * std::ldexp(1.0, base_log - 1) * std::ldexp(1.0, 31);
  if (!(bound < 0.5 * (double)kP0 * (double)kP1))
    return fail(HWB_EINVAL, "packing gadget too wide for the exact 2-prime NTT");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if (!workspace) return fail(HWB_EINVAL, "hwb_pack_ks needs a workspace");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int chunks = (int)((p->N + kPackRowsJ - 1) / kPackRowsJ);
  const Gadget gk = make_gadget(levels, base_log);
  uint32_t *part = (uint32_t *)workspace;
  dim3 grid(chunks, (unsigned)B);
  if (p->N == 1024) {
    pack_ks_partial_kernel<1024><<<grid, Cfg<1024>::THREADS, 0, s>>>(apolys, ksk_ntt, part, kPackRowsJ, gk,
                                                                     make_tw(st, 1024));
    if ((rc = post_launch("pack_ks_partial_kernel"))) return rc;
    pack_ks_finish_kernel<1024><<<(unsigned)B, Cfg<1024>::THREADS, 0, s>>>(part, chunks, b_polys, out,
                                                                           make_tw(st, 1024));
  } else {
    pack_ks_partial_kernel<2048><<<grid, Cfg<2048>::THREADS, 0, s>>>(apolys, ksk_ntt, part, kPackRowsJ, gk,
                                                                     make_tw(st, 2048));
    if ((rc = post_launch("pack_ks_partial_kernel"))) return rc;
    pack_ks_finish_kernel<2048><<<(unsigned)B, Cfg<2048>::THREADS, 0, s>>>(part, chunks, b_polys, out,
                                                                           make_tw(st, 2048));
  }
  return post_launch("pack_ks_finish_kernel");
}

int hwb_rgsw_add_gadget(const hwb_params *p, uint32_t *rgsw, const int32_t *bits, int64_t B, void *stream) {
  int rc = check_ring(p);
  if (rc) return rc;
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  const int64_t total = B * p->l;
  rgsw_gadget_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(rgsw, bits, B, (int)p->N,
                                                                                         (int)p->l, (int)p->base_log);
  return post_launch("rgsw_gadget_kernel");
}

int hwb_accumulate_rows(uint32_t *dst, const uint32_t *src, int64_t words, int32_t count, void *stream) {
  if (words < 0 || count < 0) return fail(HWB_EINVAL, "accumulate_rows: negative size");
  if (words == 0 || count == 0) return HWB_OK;
  if (((uintptr_t)dst | (uintptr_t)src) & 15) return fail(HWB_EINVAL, "accumulate_rows: pointers must be 16-byte aligned");
  const int64_t threads = (words + 3) / 4;
  accumulate_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dst, src, words, count);
  return post_launch("accumulate_rows_kernel");
}

int hwb_accumulate(uint32_t *dst, const uint32_t *src, int64_t words, int64_t src_words, int negate, void *stream) {
  if (words < 0 || src_words < 1 || (words > 0 && (words % src_words) != 0))
    return fail(HWB_EINVAL, "accumulate: words must be a multiple of src_words");
  if (words == 0) return HWB_OK;
  accumulate_kernel<<<(unsigned)((words + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dst, src, words, src_words,
                                                                                         negate);
  return post_launch("accumulate_kernel");
}

int hwb_philox_rgsw(const hwb_philox *st, const uint32_t *b_rows, const uint32_t *a0fix, int32_t levels,
                    uint32_t *out, int64_t rows, int32_t N, int32_t pair, void *stream) {
  if (!st || !out || rows < 0 || N < 1 || st->nprefix < 0 || st->nprefix > 9)
    return fail(HWB_EINVAL, "philox_rgsw: bad arguments");
  if (a0fix && (levels < 1 || rows % (2 * levels))) return fail(HWB_EINVAL, "philox_rgsw: rows not whole RGSWs");
  if (rows == 0) return HWB_OK;
  const int64_t nblocks = (rows * N + 7) / 8 + 1;
  philox_rgsw_kernel<<<(unsigned)((nblocks + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*st, b_rows, a0fix, levels,
                                                                                          out, rows, N, pair);
  return post_launch("philox_rgsw_kernel");
}

static dim3 rows_grid(int64_t B, int x_blocks) {
  // B rows over (y, z) so batches beyond 65535 rows launch
  const int64_t z = B < 65535 ? B : 65535;
  return dim3((unsigned)x_blocks, (unsigned)((B + z - 1) / z), (unsigned)z);
}

int hwb_lwe_lincomb(const uint32_t *x, const uint32_t *y, uint32_t *out, const int32_t *cx, const int32_t *cy,
                    const uint32_t *cb, int64_t B, int32_t width, int32_t shift, void *stream) {
  if (B < 0 || width < 1 || shift < 0 || shift > 31) return fail(HWB_EINVAL, "lwe_lincomb: bad shape or shift");
  if (B == 0) return HWB_OK;
  if (!x || !out) return fail(HWB_EINVAL, "lwe_lincomb: null pointer");
  lwe_lincomb_kernel<<<rows_grid(B, (width + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, y, out, cx, cy, cb, B,
                                                                                          width, shift);
  return post_launch("lwe_lincomb_kernel");
}

int hwb_gather_rows(const uint32_t *table, const int32_t *idx, uint32_t *out, int64_t B, int32_t row_words,
                    void *stream) {
  if (B < 0 || row_words < 4 || (row_words & 3)) return fail(HWB_EINVAL, "gather_rows: row_words must be a multiple of 4");
  if (B == 0) return HWB_OK;
  if (!table || !idx || !out) return fail(HWB_EINVAL, "gather_rows: null pointer");
  if (((uintptr_t)table | (uintptr_t)out) & 15) return fail(HWB_EINVAL, "gather_rows: 16-byte alignment");
  gather_rows_kernel<<<rows_grid(B, (row_words / 4 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(table, idx, out,
                                                                                                  B, row_words);
  return post_launch("gather_rows_kernel");
}

int hwb_ext_product(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
                    const uint32_t *in, uint32_t *out, int64_t B, void *stream) {
  return cmux_dispatch(MODE_EXT, p, ggsw_ntt, ggsw_idx, in, nullptr, nullptr, out, nullptr, B, stream);
}

int hwb_cmux(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx, const uint32_t *c1,
             const uint32_t *c0, const int32_t *rot, uint32_t *out, int64_t B, void *stream) {
  if (!c1 && !rot) return fail(HWB_EINVAL, "cmux needs c1 or a rotation vector");
  return cmux_dispatch(MODE_CMUX, p, ggsw_ntt, ggsw_idx, c0, c1, rot, out, nullptr, B, stream);
}

int hwb_cdemux(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx, const uint32_t *d,
               uint32_t *lo, uint32_t *hi, int64_t B, void *stream) {
  return cmux_dispatch(MODE_CDEMUX, p, ggsw_ntt, ggsw_idx, d, nullptr, nullptr, lo, hi, B, stream);
}

int hwb_blind_rotate(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx, const int32_t *exps,
                     uint32_t *acc, int32_t L, int64_t B, void *stream) {
  int rc = check_glwe(p);
  if (rc) return rc;
  if (B < 0 || L < 0) return fail(HWB_EINVAL, "negative batch or length");
  if (B == 0) return HWB_OK;
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->N == 1024)
    return launch_br<1024, false>(p, st, ggsw_ntt, ggsw_idx, exps, nullptr, nullptr, 0, acc, nullptr, L, B, s);
  return launch_br<2048, false>(p, st, ggsw_ntt, ggsw_idx, exps, nullptr, nullptr, 0, acc, nullptr, L, B, s);
}

int hwb_sample_extract(const hwb_params *p, const uint32_t *rlwe, uint32_t *lwe, int64_t B, int32_t coeff,
                       void *stream) {
  int rc = check_ring(p);
  if (rc) return rc;
  if (coeff < 0 || coeff >= (int32_t)p->N) return fail(HWB_EINVAL, "coefficient index out of range");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = B * (p->N + 1);
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (p->N == 1024)
    extract_kernel<1024><<<blocks, 256, 0, s>>>(rlwe, lwe, B, coeff);
  else
    extract_kernel<2048><<<blocks, 256, 0, s>>>(rlwe, lwe, B, coeff);
  return post_launch("extract_kernel");
}

int hwb_keyswitch(const hwb_params *p, const uint32_t *ksk, const uint32_t *in, uint32_t *out, int64_t B,
                  void *stream) {
  if (!p) return fail(HWB_EINVAL, "null params");
  int rc = check_ks(p);
  if (rc) return rc;
  if (p->N < 1) return fail(HWB_EINVAL, "N must be positive");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  return keyswitch_launch(p, ksk, in, out, B, (cudaStream_t)stream);
}

size_t hwb_pbs_workspace_bytes(const hwb_params *p, int64_t B) {
  if (!p || B <= 0) return 0;
  return sizeof(uint32_t) * (size_t)B * (p->N + 1);
}

int hwb_pbs(const hwb_params *p, const uint32_t *bsk_ntt, const uint32_t *ksk, const uint32_t *tv,
            int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out, int64_t B, void *workspace,
            void *stream) {
  int rc = check_glwe(p);
  if (rc) return rc;
  if (ksk && (rc = check_ks(p))) return rc;
  if (p->n < 1) return fail(HWB_EINVAL, "LWE dimension n must be positive");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if (B > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (ksk && !workspace) return fail(HWB_EINVAL, "hwb_pbs with key switch needs a workspace");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t *ext = ksk ? (uint32_t *)workspace : lwe_out;
  if (p->N == 1024)
    rc = launch_br<1024, true>(p, st, bsk_ntt, nullptr, nullptr, lwe_in, tv, tv_per_item, nullptr, ext, (int)p->n, B, s);
  else
    rc = launch_br<2048, true>(p, st, bsk_ntt, nullptr, nullptr, lwe_in, tv, tv_per_item, nullptr, ext, (int)p->n, B, s);
  if (rc || !ksk) return rc;
  return keyswitch_launch(p, ksk, ext, lwe_out, B, s);
}

static size_t pbs_ext_bytes(const hwb_params *p, int64_t B) {
  return ((sizeof(uint32_t) * (size_t)B * (p->N + 1)) + 255) & ~(size_t)255;
}

// accumulators between segments [B][2][N], then the single-launch ladder's progress words
// (segments done per CTA-group of 4 ciphertexts)
static size_t fft_accs_only_bytes(const hwb_params *p, int64_t B) { return ((size_t)B * 2 * p->N * 4 + 255) & ~(size_t)255; }
static size_t fft_queue_bytes(int64_t B) { return (((size_t)(B + 3) / 4) * 4 + 255) & ~(size_t)255; }
static size_t fft_acc_bytes(const hwb_params *p, int64_t B) { return fft_accs_only_bytes(p, B) + fft_queue_bytes(B); }
// ladder steps per launch of the FFT ladder (L2 residency of the key slice)
static thread_local int g_fft_segment = 64;
// the single-launch ladders' segment while hwb_set_fft_segment has not been called: shorter
// segments fill the launch's only tail more finely (cfg2 B = 4096: 51.5 ms at 48 steps, 52.0 at
// 64, 51.7 at 32; cfg1 31.7 / 31.8; tools/seg_sweep.py), the per-segment modes keep 64
static thread_local bool g_fft_segment_set = false;
constexpr int kSingleLaunchSegment = 48;
// ciphertexts per CTA of the FFT PBS ladder (sharing each staged key slice)
static thread_local int g_fft_cpb = 1;
// batches of at most this many ciphertexts run the FFT latency ladder (-1: one per SM)
static thread_local int64_t g_fft_lat_max_batch = -1;
// cluster latency ladder shape: 0 = 2l CTAs (one digit row each), 1 = 4 CTAs (one
// accumulator quarter each, all digit rows per CTA)
static thread_local int g_fft_cluster_mode = 0;
int hwb_set_fft_cluster_mode(int mode) {
  if (mode != 0 && mode != 1) return fail(HWB_EINVAL, "cluster mode must be 0 or 1");
  g_fft_cluster_mode = mode;
  return HWB_OK;
}
// batches of at most this many ciphertexts run the cluster latency ladder (2l SMs
// each); -1: as many as fit co-resident (hwb_fft_cluster_capacity)
static thread_local int64_t g_fft_cluster_max_batch = -1;

int64_t hwb_set_fft_cluster_batch(int64_t max_batch) {
  const int64_t prev = g_fft_cluster_max_batch;
  if (max_batch >= -1) g_fft_cluster_max_batch = max_batch;
  return prev;
}
// FFT PBS ladder (batches of >= 8 ciphertexts per SM; smaller ones use the register
// ladder): 0 = registers (g_fft_cpb ciphertexts per CTA), 1 = TMEM accumulators, two
// ciphertexts per thread; 2 = TMEM, one per thread (16 warps/SM); 3 = 2 with lane-paired
// ciphertexts; 4 = 3 as one 16-warp CTA of decoupled groups; 5 = 3 with decoupled halves
// and the whole ladder in ONE launch (default: cfg2 B = 4096 in 51.5 ms vs 61.0 / 60.1 /
// 59.6 / 63.2 ms for modes 1-4); 6 = 5 as one 16-warp CTA with a two-slot key ring
// (62.1 ms; 62.5 vs 61.8 ms at full waves, B = 4736); 7 = 5 on 32-thread transforms, one
// transpose per transform (59.4 ms); 8 = 5 with one launch per segment (53.2 ms),
// DESIGN.md §3b.  All bit-identical.
static thread_local int g_fft_mode = 5;
// smallest batch (ciphertexts per SM) for the mode-5 TMEM ladder: from 4 per SM (one
// CTA) it beats the register ladder (cfg2 B = 592: 9.27 vs 9.97 ms; 1036: 16.2 vs 19.4;
// 444: 9.29 vs 8.84)
constexpr int64_t g_fft_tmem_min = 4;

int hwb_set_fft_mode(int mode) {
  if (mode < 0 || mode > 8)
    return fail(HWB_EINVAL, "FFT ladder mode must be 0 (registers), 1 (TMEM), 2 (TMEM, one ciphertext per thread) "
                            "3 (TMEM, lane-paired), 4 (TMEM, decoupled groups), 5 (TMEM, lane-paired, decoupled halves) or 6 (5 as one "
                            "16-warp CTA with a two-slot key ring) 7 (5 on 32-thread transforms: one transpose per transform) or 8 (5 with one launch per segment "
                            "instead of one launch for the whole ladder)");
  g_fft_mode = mode;
  return HWB_OK;
}

int64_t hwb_set_fft_latency_batch(int64_t max_batch) {
  const int64_t prev = g_fft_lat_max_batch;
  if (max_batch >= -1) g_fft_lat_max_batch = max_batch;
  return prev;
}

extern "C++" {
template <int CPB>
static int launch_pbs_fft(const void *bsk_fft, const uint32_t *lwe_in, const uint32_t *tv, int tv_per_item,
                          uint32_t *ext, int L, const Gadget &g, DevState *st, uint32_t *acc, int s0, int s1,
                          int64_t B, cudaStream_t s) {
  const size_t smem = sizeof(FSmemT<CPB>);
  int rc;
  if ((rc = set_smem(blind_rotate_fft_kernel<true, CPB>, smem))) return rc;
  blind_rotate_fft_kernel<true, CPB><<<(unsigned)((B + CPB - 1) / CPB), FT * CPB, smem, s>>>(
      (const double2 *)bsk_fft, nullptr, nullptr, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc,
      s0, s1, B);
  return post_launch("blind_rotate_fft_kernel");
}
}  // extern "C++"

static int check_fft(const hwb_params *p) {
  // the FFT ladders do not use the two-prime CRT, so the NTT's range bound does not apply
  // (full-precision 2 x 16 gadgets run here); their own exactness is the rounding margin:
  // measured max |y - rint(y)| 2^-21 (N = 1024, 8-bit digits) and 2^-18 (N = 2048,
  // 10-bit digits), growing linearly with the digit size -- 16-bit digits stay below 2^-12
  // (tests/test_gpu_fullsize.py measures every supported width)
  int rc = check_ring(p);
  if (rc) return rc;
  if (p->N == 4 * FH) {
    // FFT2: biased halfword digits, 2l <= F2R rows
    if (2 * p->l > (uint32_t)F2R || p->base_log > 16)
      return fail(HWB_EINVAL, "the N = 2048 FFT ladder needs l <= 2 and base_log <= 16");
    return HWB_OK;
  }
  if (p->N != 2 * FH) return fail(HWB_EINVAL, "the FFT ladder supports N = 1024 and 2048");
  if (p->base_log > 16) return fail(HWB_EINVAL, "the FFT ladder needs base_log <= 16");
#if HWB_FFT_DIG
  // staged byte digits (base_log <= 8) or on-the-fly extraction (base_log <= 16), 2l <= FDR
  if (2 * p->l > (uint32_t)FDR) return fail(HWB_EINVAL, "the FFT ladder needs l <= 3");
#endif
  return HWB_OK;
}

size_t hwb_bsk_fft_bytes(const hwb_params *p) {
  if (!p || check_fft(p)) return 0;
  return (size_t)p->n * 2 * p->l * 2 * 2 * (p->N / 2) * sizeof(double2);
}

static int launch_to_fft(const hwb_params *p, const uint32_t *in, void *out, int64_t polys, DevState *st,
                         cudaStream_t s) {
  if (p->N == 4 * FH) {
    bsk_to_fft2_kernel<<<(unsigned)polys, 2 * FT, 0, s>>>(in, (double2 *)out, st->fft2_fwd[0], st->fft2_fwd[1]);
    return post_launch("bsk_to_fft2_kernel");
  }
  bsk_to_fft_kernel<<<(unsigned)polys, FT, 0, s>>>(in, (double2 *)out, st->fft_fwd);
  return post_launch("bsk_to_fft_kernel");
}

int hwb_bsk_to_fft(const hwb_params *p, const uint32_t *bsk, void *bsk_fft, void *stream) {
  int rc = check_fft(p);
  if (rc) return rc;
  if (p->n < 1) return fail(HWB_EINVAL, "LWE dimension n must be positive");
  if (!bsk || !bsk_fft) return fail(HWB_EINVAL, "null key pointer");
  if ((uintptr_t)bsk_fft & 15) return fail(HWB_EINVAL, "bsk_fft must be 16-byte aligned");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  const int64_t polys = (int64_t)p->n * 2 * p->l * 2;
  return launch_to_fft(p, bsk, bsk_fft, polys, st, (cudaStream_t)stream);
}

int64_t hwb_fft_cluster_capacity(const hwb_params *p) {
  static int64_t cache[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  if (!p || check_fft(p) || p->N != 2 * FH || p->l < 2 || 2 * p->l > 8) return 0;
  std::lock_guard<std::mutex> lk(g_mu);
  if (cache[p->l] >= 0) return cache[p->l];
  const size_t smem = sizeof(FSmemC);
  if (cudaFuncSetAttribute(blind_rotate_fft_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * p->l * 64));
  cfg.blockDim = dim3(FT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * p->l;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, blind_rotate_fft_cl_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[p->l] = n;
  return n;
}

int hwb_pbs_fft(const hwb_params *p, const void *bsk_fft, const void *ksk_tc, const uint32_t *tv,
                int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out, int64_t B, void *workspace,
                void *stream) {
  int rc = check_fft(p);
  if (rc) return rc;
  if (ksk_tc && (rc = check_ks_tc(p))) return rc;
  if (p->n < 1) return fail(HWB_EINVAL, "LWE dimension n must be positive");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if (B > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (!bsk_fft) return fail(HWB_EINVAL, "null key pointer");
  if (ksk_tc && (((uintptr_t)ksk_tc | (uintptr_t)workspace) & 15))
    return fail(HWB_EINVAL, "ksk_tc/workspace must be 16-byte aligned");
  if (!workspace) return fail(HWB_EINVAL, "hwb_pbs_fft needs a workspace (hwb_pbs_fft_workspace_bytes)");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)workspace;
  uint32_t *acc = (uint32_t *)ws;                               // [B][2][N] between segments
  uint32_t *ext = ksk_tc ? (uint32_t *)(ws + fft_acc_bytes(p, B)) : lwe_out;
  const Gadget g = make_gadget(p->l, p->base_log);
  const int L = (int)p->n;
  const int64_t lat_max = g_fft_lat_max_batch >= 0 ? g_fft_lat_max_batch : (int64_t)st->sms;
  const int64_t cl_max = g_fft_cluster_max_batch >= 0 ? g_fft_cluster_max_batch : hwb_fft_cluster_capacity(p);
  if (p->N == 2 * FH && B <= cl_max && p->l >= 2 && 2 * p->l <= 8) {
    // cluster latency ladder: 2l (or 4) CTAs (SMs) per ciphertext
    const bool c4 = g_fft_cluster_mode == 1;
    const size_t smem = c4 ? sizeof(FSmemC4) : sizeof(FSmemC);
    if ((rc = c4 ? set_smem(blind_rotate_fft_cl4_kernel, smem) : set_smem(blind_rotate_fft_cl_kernel, smem)))
      return rc;
    const int csize = c4 ? 4 : 2 * (int)p->l;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * csize));
    cfg.blockDim = dim3(c4 ? 2 * p->l * FT : FT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, c4 ? blind_rotate_fft_cl4_kernel : blind_rotate_fft_cl_kernel,
                                             (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g,
                                             (const double2 *)st->fft_fwd, (const double2 *)st->fft_inv);
    if (e != cudaSuccess) return fail(HWB_ECUDA, std::string("cluster launch: ") + cudaGetErrorString(e));
    if ((rc = post_launch("blind_rotate_fft_cl_kernel"))) return rc;
    if (!ksk_tc) return HWB_OK;
    return keyswitch_tc_launch(p, ksk_tc, ext, lwe_out, B, ws + fft_acc_bytes(p, B) + pbs_ext_bytes(p, B), s);
  }
  if (p->N == 2 * FH && B <= lat_max) {
    // latency mode: 2l groups of 64 threads per ciphertext, the whole ladder in one launch
    const size_t smem = sizeof(FSmemL);
    if ((rc = set_smem(blind_rotate_fft_lat_kernel, smem))) return rc;
    blind_rotate_fft_lat_kernel<<<(unsigned)B, 2 * p->l * FT, smem, s>>>(
        (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv);
    if ((rc = post_launch("blind_rotate_fft_lat_kernel"))) return rc;
    if (!ksk_tc) return HWB_OK;
    return keyswitch_tc_launch(p, ksk_tc, ext, lwe_out, B, ws + fft_acc_bytes(p, B) + pbs_ext_bytes(p, B), s);
  }
  // mode 5: ONE launch for the whole ladder, CTA = (segment, group) in segment-major order,
  // so a segment's partial last wave overlaps the next segment (mode 8: one launch per
  // segment, each with its own tail)
  const bool single = p->N == 2 * FH && g_fft_mode == 5 && B >= g_fft_tmem_min * (int64_t)st->sms;
  if (single) {
    uint32_t *progress = (uint32_t *)(ws + fft_accs_only_bytes(p, B));
    const cudaError_t e = cudaMemsetAsync(progress, 0, fft_queue_bytes(B), s);
    if (e != cudaSuccess) return fail(HWB_ECUDA, std::string("progress memset: ") + cudaGetErrorString(e));
    const int seg_len = g_fft_segment_set ? g_fft_segment : kSingleLaunchSegment;
    const int64_t ctas = ((B + 3) / 4) * (int64_t)((L + seg_len - 1) / seg_len);
    if (ctas > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
    const size_t smem = sizeof(FSmemTDT<2, 1>);
    if ((rc = set_smem(blind_rotate_fft_td_kernel<2, 1>, smem))) return rc;
    blind_rotate_fft_td_kernel<2, 1><<<(unsigned)ctas, 256, smem, s>>>(
        (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, 0, seg_len, B,
        progress);
    if ((rc = post_launch("blind_rotate_fft_td_kernel (single launch)"))) return rc;
  }
  const bool single2 = p->N == 4 * FH && g_fft_mode == 5 && B >= (int64_t)T2C * st->sms;
  if (single2) {   // the N = 2048 TMEM ladder, same single-launch protocol
    uint32_t *progress = (uint32_t *)(ws + fft_accs_only_bytes(p, B));
    const cudaError_t e = cudaMemsetAsync(progress, 0, fft_queue_bytes(B), s);
    if (e != cudaSuccess) return fail(HWB_ECUDA, std::string("progress memset: ") + cudaGetErrorString(e));
    const int seg_len = g_fft_segment_set ? g_fft_segment : kSingleLaunchSegment;
    const int64_t ctas = ((B + T2C - 1) / T2C) * (int64_t)((L + seg_len - 1) / seg_len);
    if (ctas > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
    const size_t smem = sizeof(FSmem2TD);
    if ((rc = set_smem(blind_rotate_fft2_td_kernel<true>, smem))) return rc;
    blind_rotate_fft2_td_kernel<true><<<(unsigned)ctas, 16 * 32, smem, s>>>(
        (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft2_fwd[0], st->fft2_fwd[1],
        st->fft2_inv[0], st->fft2_inv[1], acc, 0, seg_len, B, progress);
    if ((rc = post_launch("blind_rotate_fft2_td_kernel (single launch)"))) return rc;
  }
  for (int s0 = 0; s0 < L && !single && !single2; s0 += g_fft_segment) {
    const int s1 = s0 + g_fft_segment < L ? s0 + g_fft_segment : L;
    if (p->N == 4 * FH && g_fft_mode >= 1 && B >= (int64_t)T2C * st->sms) {
      // TMEM ladder: 4 ciphertexts per SM (one 16-warp CTA) sharing each key slice
      const size_t smem = sizeof(FSmem2TD);
      if ((rc = set_smem(blind_rotate_fft2_td_kernel<false>, smem))) return rc;
      blind_rotate_fft2_td_kernel<false><<<(unsigned)((B + T2C - 1) / T2C), 16 * 32, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft2_fwd[0], st->fft2_fwd[1],
          st->fft2_inv[0], st->fft2_inv[1], acc, s0, s1, B, nullptr);
      rc = post_launch("blind_rotate_fft2_td_kernel");
    } else if (p->N == 4 * FH) {
      const size_t smem = sizeof(FSmem2);
      if ((rc = set_smem(blind_rotate_fft2_kernel<true>, smem))) return rc;
      blind_rotate_fft2_kernel<true><<<(unsigned)B, 2 * FT, smem, s>>>(
          (const double2 *)bsk_fft, nullptr, nullptr, lwe_in, tv, tv_per_item, ext, L, g, st->fft2_fwd[0],
          st->fft2_fwd[1], st->fft2_inv[0], st->fft2_inv[1], acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft2_kernel");
    } else if (g_fft_mode == 7 && B >= g_fft_tmem_min * (int64_t)st->sms) {
      const size_t smem = sizeof(FSmemW);
      if ((rc = set_smem(blind_rotate_fft_w_kernel, smem))) return rc;
      blind_rotate_fft_w_kernel<<<(unsigned)((B + 3) / 4), 128, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_w16, acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft_w_kernel");
    } else if (g_fft_mode == 6 && B >= 8 * (int64_t)st->sms) {
      const size_t smem = sizeof(FSmemTDT<4, 2>);
      if ((rc = set_smem(blind_rotate_fft_td_kernel<4, 2>, smem))) return rc;
      blind_rotate_fft_td_kernel<4, 2><<<(unsigned)((B + 7) / 8), 512, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B,
          nullptr);
      rc = post_launch("blind_rotate_fft_td_kernel<4,2>");
    } else if (g_fft_mode >= 5 && B >= g_fft_tmem_min * (int64_t)st->sms) {
      const size_t smem = sizeof(FSmemTDT<2, 1>);
      if ((rc = set_smem(blind_rotate_fft_td_kernel<2, 1>, smem))) return rc;
      blind_rotate_fft_td_kernel<2, 1><<<(unsigned)((B + 3) / 4), 256, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B,
          nullptr);
      rc = post_launch("blind_rotate_fft_td_kernel");
    } else if (g_fft_mode == 4 && B >= (int64_t)TQC * st->sms) {
      const size_t smem = sizeof(FSmemTQ);
      if ((rc = set_smem(blind_rotate_fft_tq_kernel, smem))) return rc;
      blind_rotate_fft_tq_kernel<<<(unsigned)((B + TQC - 1) / TQC), TQG * 4 * 32, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft_tq_kernel");
    } else if (g_fft_mode == 3 && B >= (int64_t)2 * TPC * st->sms) {
      const size_t smem = sizeof(FSmemTP);
      if ((rc = set_smem(blind_rotate_fft_tp_kernel, smem))) return rc;
      blind_rotate_fft_tp_kernel<<<(unsigned)((B + TPC - 1) / TPC), TPC * FT, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft_tp_kernel");
    } else if (g_fft_mode == 2 && B >= (int64_t)2 * TXC * st->sms) {
      const size_t smem = sizeof(FSmemTX);
      if ((rc = set_smem(blind_rotate_fft_tx_kernel, smem))) return rc;
      blind_rotate_fft_tx_kernel<<<(unsigned)((B + TXC - 1) / TXC), TXC * FT, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft_tx_kernel");
    } else if (g_fft_mode == 1 && B >= (int64_t)2 * TMC * st->sms) {
      // TMEM ladder only when it fills two CTAs (8 ciphertexts) per SM; smaller
      // batches keep more CTAs per SM on the register ladder
      const size_t smem = sizeof(FSmemTM);
      if ((rc = set_smem(blind_rotate_fft_tm_kernel, smem))) return rc;
      blind_rotate_fft_tm_kernel<<<(unsigned)((B + TMC - 1) / TMC), 2 * FT, smem, s>>>(
          (const double2 *)bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st->fft_fwd, st->fft_inv, acc, s0, s1, B);
      rc = post_launch("blind_rotate_fft_tm_kernel");
    } else if (g_fft_cpb == 4)
      rc = launch_pbs_fft<4>(bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st, acc, s0, s1, B, s);
    else if (g_fft_cpb == 2)
      rc = launch_pbs_fft<2>(bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st, acc, s0, s1, B, s);
    else
      rc = launch_pbs_fft<1>(bsk_fft, lwe_in, tv, tv_per_item, ext, L, g, st, acc, s0, s1, B, s);
    if (rc) return rc;
  }
  if (!ksk_tc) return HWB_OK;
  return keyswitch_tc_launch(p, ksk_tc, ext, lwe_out, B,
                             ws + fft_acc_bytes(p, B) + pbs_ext_bytes(p, B), s);
}

size_t hwb_ggsw_fft_bytes(const hwb_params *p) {
  if (!p || check_fft(p)) return 0;
  return (size_t)2 * p->l * 2 * 2 * (p->N / 2) * sizeof(double2);
}

int hwb_ggsw_to_fft(const hwb_params *p, const uint32_t *ggsw, void *ggsw_fft, int64_t count, void *stream) {
  int rc = check_fft(p);
  if (rc) return rc;
  if (count < 0) return fail(HWB_EINVAL, "negative count");
  if (count == 0) return HWB_OK;
  if (!ggsw || !ggsw_fft) return fail(HWB_EINVAL, "null pointer");
  if ((uintptr_t)ggsw_fft & 15) return fail(HWB_EINVAL, "ggsw_fft must be 16-byte aligned");
  const int64_t polys = count * 2 * p->l * 2;
  if (polys > 0x7FFFFFFF) return fail(HWB_EINVAL, "too many GGSWs");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  return launch_to_fft(p, ggsw, ggsw_fft, polys, st, (cudaStream_t)stream);
}

int hwb_blind_rotate_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const int32_t *exps,
                         uint32_t *acc, int32_t L, int64_t B, void *stream) {
  int rc = check_fft(p);
  if (rc) return rc;
  if (L < 0 || B < 0) return fail(HWB_EINVAL, "negative size");
  if (L == 0 || B == 0) return HWB_OK;
  if (B > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (!ggsw_fft || !exps || !acc) return fail(HWB_EINVAL, "null pointer");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  if (p->N == 4 * FH) {
    const size_t smem = sizeof(FSmem2);
    if ((rc = set_smem(blind_rotate_fft2_kernel<false>, smem))) return rc;
    blind_rotate_fft2_kernel<false><<<(unsigned)B, 2 * FT, smem, (cudaStream_t)stream>>>(
        (const double2 *)ggsw_fft, ggsw_idx, exps, nullptr, nullptr, 0, nullptr, L, make_gadget(p->l, p->base_log),
        st->fft2_fwd[0], st->fft2_fwd[1], st->fft2_inv[0], st->fft2_inv[1], acc, 0, L, B);
    return post_launch("blind_rotate_fft2_kernel");
  }
  const size_t smem = sizeof(FSmem);
  if ((rc = set_smem(blind_rotate_fft_kernel<false>, smem))) return rc;
  blind_rotate_fft_kernel<false><<<(unsigned)B, FT, smem, (cudaStream_t)stream>>>(
      (const double2 *)ggsw_fft, ggsw_idx, exps, nullptr, nullptr, 0, nullptr, L, make_gadget(p->l, p->base_log),
      st->fft_fwd, st->fft_inv, acc, 0, L, B);
  return post_launch("blind_rotate_fft_kernel");
}

extern "C++" {
template <int MODE>
static int level_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const uint32_t *cur,
                     uint32_t *next, int32_t m, int64_t B, void *stream) {
  int rc = check_fft(p);
  if (rc) return rc;
  if (m < 1 || B < 0) return fail(HWB_EINVAL, "bad level shape");
  if (B == 0) return HWB_OK;
  if (B * m > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (!ggsw_fft || !ggsw_idx || !cur || !next) return fail(HWB_EINVAL, "null pointer");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  if (p->N == 4 * FH) {
    const size_t smem = sizeof(FSmem2);
    if ((rc = set_smem(level_fft2_kernel<MODE>, smem))) return rc;
    level_fft2_kernel<MODE><<<(unsigned)(B * m), 2 * FT, smem, (cudaStream_t)stream>>>(
        (const double2 *)ggsw_fft, ggsw_idx, cur, next, m, make_gadget(p->l, p->base_log), st->fft2_fwd[0],
        st->fft2_fwd[1], st->fft2_inv[0], st->fft2_inv[1]);
    return post_launch("level_fft2_kernel");
  }
#ifndef HWB_LEVEL_TD
#define HWB_LEVEL_TD 1   // bit 0: IVP levels, bit 1: VP levels on level_fft_td_kernel
#endif
  if ((HWB_LEVEL_TD >> (MODE == MODE_IVP_LEVEL ? 0 : 1)) & 1 && g_fft_mode >= 5 && m % 4 == 0 &&
      B * m >= (int64_t)8 * st->sms) {
    const size_t smem_td = sizeof(FSmemTDT<2, 1>);
    if ((rc = set_smem(level_fft_td_kernel<MODE>, smem_td))) return rc;
    level_fft_td_kernel<MODE><<<(unsigned)(B * m / 4), 256, smem_td, (cudaStream_t)stream>>>(
        (const double2 *)ggsw_fft, ggsw_idx, cur, next, m, make_gadget(p->l, p->base_log), st->fft_fwd, st->fft_inv);
    return post_launch("level_fft_td_kernel");
  }
  if (g_fft_mode >= 1 && m % TMC == 0 && B * m >= (int64_t)2 * TMC * st->sms) {
    // sub-ciphertexts of an item share its GGSW: four per CTA on the TMEM path
    const size_t smem_tm = sizeof(FSmemTM);
    if ((rc = set_smem(level_fft_tm_kernel<MODE>, smem_tm))) return rc;
    level_fft_tm_kernel<MODE><<<(unsigned)(B * m / TMC), 2 * FT, smem_tm, (cudaStream_t)stream>>>(
        (const double2 *)ggsw_fft, ggsw_idx, cur, next, m, make_gadget(p->l, p->base_log), st->fft_fwd, st->fft_inv);
    return post_launch("level_fft_tm_kernel");
  }
  const size_t smem = sizeof(FSmem);
  if ((rc = set_smem(level_fft_kernel<MODE>, smem))) return rc;
  level_fft_kernel<MODE><<<(unsigned)(B * m), FT, smem, (cudaStream_t)stream>>>(
      (const double2 *)ggsw_fft, ggsw_idx, cur, next, m, make_gadget(p->l, p->base_log), st->fft_fwd, st->fft_inv);
  return post_launch("level_fft_kernel");
}
}  // extern "C++"

int hwb_ivp_level_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const uint32_t *cur,
                      uint32_t *next, int32_t m, int64_t B, void *stream) {
  return level_fft<MODE_IVP_LEVEL>(p, ggsw_fft, ggsw_idx, cur, next, m, B, stream);
}

int hwb_vp_level_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const uint32_t *cur,
                     uint32_t *next, int32_t m, int64_t B, void *stream) {
  return level_fft<MODE_VP_LEVEL>(p, ggsw_fft, ggsw_idx, cur, next, m, B, stream);
}

size_t hwb_pbs_fft_workspace_bytes(const hwb_params *p, int64_t B, int with_keyswitch) {
  if (!p || B <= 0 || check_fft(p)) return 0;
  size_t bytes = fft_acc_bytes(p, B);
  if (with_keyswitch) {
    if (check_ks_tc(p)) return 0;
    bytes += pbs_ext_bytes(p, B) + ks_tc_digit_bytes(p, B);
  }
  return bytes;
}

int hwb_set_fft_group(int ciphertexts_per_cta) {
  if (ciphertexts_per_cta != 1 && ciphertexts_per_cta != 2 && ciphertexts_per_cta != 4)
    return fail(HWB_EINVAL, "ciphertexts per CTA must be 1, 2 or 4");
  g_fft_cpb = ciphertexts_per_cta;
  return HWB_OK;
}

int hwb_set_fft_segment(int steps) {
  if (steps < 1) return fail(HWB_EINVAL, "segment must be >= 1 step");
  g_fft_segment = steps;
  g_fft_segment_set = true;
  return HWB_OK;
}

size_t hwb_ksk_tc_bytes(const hwb_params *p) {
  if (!p || check_ks_tc(p)) return 0;
  const size_t nct = (p->n + 1 + TC_COLS - 1) / TC_COLS;
  return nct * ((size_t)p->N * p->ks_l / TC_KB) * TC_B_BYTES;
}

int hwb_ksk_to_tc(const hwb_params *p, const uint32_t *ksk, void *ksk_tc, void *stream) {
  if (!p) return fail(HWB_EINVAL, "null params");
  int rc = check_ks_tc(p);
  if (rc) return rc;
  if (!ksk || !ksk_tc) return fail(HWB_EINVAL, "null key pointer");
  if ((uintptr_t)ksk_tc & 15) return fail(HWB_EINVAL, "ksk_tc must be 16-byte aligned");
  const int K = (int)(p->N * p->ks_l);
  const int nct = (int)((p->n + 1 + TC_COLS - 1) / TC_COLS);
  const int64_t total = (int64_t)nct * (K / TC_KB) * (TC_B_BYTES / 16);
  ksk_to_tc_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(ksk, (uint4 *)ksk_tc, K,
                                                                                       (int)p->n + 1, nct);
  return post_launch("ksk_to_tc_kernel");
}

size_t hwb_keyswitch_tc_workspace_bytes(const hwb_params *p, int64_t B) {
  if (!p || B <= 0 || check_ks_tc(p)) return 0;
  return ks_tc_digit_bytes(p, B);
}

int hwb_keyswitch_tc(const hwb_params *p, const void *ksk_tc, const uint32_t *in, uint32_t *out, int64_t B,
                     void *workspace, void *stream) {
  if (!p) return fail(HWB_EINVAL, "null params");
  int rc = check_ks_tc(p);
  if (rc) return rc;
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if ((B + TC_M - 1) / TC_M > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (!ksk_tc || !workspace) return fail(HWB_EINVAL, "hwb_keyswitch_tc needs ksk_tc and a workspace");
  if (((uintptr_t)ksk_tc | (uintptr_t)workspace) & 15) return fail(HWB_EINVAL, "ksk_tc/workspace must be 16-byte aligned");
  return keyswitch_tc_launch(p, ksk_tc, in, out, B, workspace, (cudaStream_t)stream);
}


size_t hwb_pbs_tc_workspace_bytes(const hwb_params *p, int64_t B) {
  if (!p || B <= 0 || check_ks_tc(p)) return 0;
  return pbs_ext_bytes(p, B) + ks_tc_digit_bytes(p, B);
}

int hwb_pbs_tc(const hwb_params *p, const uint32_t *bsk_ntt, const void *ksk_tc, const uint32_t *tv,
               int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out, int64_t B, void *workspace,
               void *stream) {
  int rc = check_glwe(p);
  if (rc) return rc;
  if ((rc = check_ks_tc(p))) return rc;
  if (p->n < 1) return fail(HWB_EINVAL, "LWE dimension n must be positive");
  if (B < 0) return fail(HWB_EINVAL, "negative batch");
  if (B == 0) return HWB_OK;
  if (B > 0x7FFFFFFF) return fail(HWB_EINVAL, "batch too large");
  if (!ksk_tc || !workspace) return fail(HWB_EINVAL, "hwb_pbs_tc needs ksk_tc and a workspace");
  if (((uintptr_t)ksk_tc | (uintptr_t)workspace) & 15) return fail(HWB_EINVAL, "ksk_tc/workspace must be 16-byte aligned");
  DevState *st;
  if ((rc = init_device(&st))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t *ext = (uint32_t *)workspace;
  void *digits = (uint8_t *)workspace + pbs_ext_bytes(p, B);
  if (p->N == 1024)
    rc = launch_br<1024, true>(p, st, bsk_ntt, nullptr, nullptr, lwe_in, tv, tv_per_item, nullptr, ext, (int)p->n, B, s);
  else
    rc = launch_br<2048, true>(p, st, bsk_ntt, nullptr, nullptr, lwe_in, tv, tv_per_item, nullptr, ext, (int)p->n, B, s);
  if (rc) return rc;
  return keyswitch_tc_launch(p, ksk_tc, ext, lwe_out, B, digits, s);
}

}  // extern "C"
