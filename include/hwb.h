/*
 * hwb.h -- C ABI of libhwb200.so, the B200 (sm_100a) batched TFHE bootstrapping
 * library.  Flat extern "C" entry points over plain pointers and sizes; no C++
 * or torch types cross the boundary.
 *
 * The reference (`hewisard`, pure Python over numpy uint64) has no FFI; its
 * drop-in boundary is the Python module API.  Each entry point below names the
 * reference function whose computation it replaces (hw/ = pkg/src/hewisard/).
 * The Python mirror of that API lives in paper_2403_20190_b200/ and binds these
 * symbols with ctypes (see INTEGRATION.md for the binding a maintainer adds).
 *
 * Conventions
 *   - q = 2^32.  Ciphertext words are little-endian uint32, C-contiguous, with
 *     the reference axis orders: RLWE [a, b] (hw/tfhe.py:124), RGSW rows
 *     b-gadget then a-gadget (hw/tfhe.py:148-152), LWE [a_0..a_{n-1}, b].
 *   - All data pointers are DEVICE pointers owned by the caller (e.g. torch
 *     tensors' data_ptr()); the library never allocates or frees caller memory.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous on it.
 *   - Return 0 on success; HWB_EINVAL for shape/parameter errors (the Python
 *     layer raises TfheError, as the reference does, hw/tfhe.py:25-30);
 *     HWB_ECUDA for launch/async CUDA errors (RuntimeError).  Nothing throws or
 *     exits across the ABI.  hwb_last_error() describes the last failure of the
 *     calling thread.
 *   - Threading: calls are re-entrant and asynchronous on their
 *     stream; there are no host threads in the library.  The tuning setters
 *     (hwb_set_variant, hwb_set_*_batch, hwb_set_fft_*) are THREAD-LOCAL: they
 *     change kernel selection for the calling thread only, so two threads
 *     driving two streams never see each other's settings.  Kernel selection
 *     never changes results (every ladder is bit-identical).
 *   - Supported envelope: N in {1024, 2048}; gadget levels <= 3 and
 *     2*levels * N * beta/2 * 2^31 < 2^55 (exact two-prime RNS NTT); see DESIGN.md.
 */
#ifndef HWB_H
#define HWB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HWB_OK 0
#define HWB_EINVAL 1
#define HWB_ECUDA 2

/* Parameter block (hw/params.py:47-82 at q = 2^32, plus the PBS LWE side). */
typedef struct hwb_params {
    uint32_t q_bits;      /* must be 32 */
    uint32_t n;           /* LWE dimension (BSK length) */
    uint32_t N;           /* ring degree */
    uint32_t k;           /* GLWE dimension, must be 1 */
    uint32_t l;           /* external-product gadget levels (GadgetSpec.levels) */
    uint32_t base_log;    /* external-product gadget log2(beta) */
    uint32_t ks_l;        /* LWE key-switch gadget levels */
    uint32_t ks_base_log; /* LWE key-switch gadget log2(beta_ks) */
} hwb_params;

int hwb_version(void);
const char *hwb_last_error(void);

/* Select the CMUX-ladder kernel build: 0 = unconstrained registers (default),
 * 1 = 128-register cap for twice the resident CTAs.  Both are bit-identical;
 * the switch exists for A/B measurement (bench.py --variant). */
int hwb_set_variant(int v);

/* Batches of at most max_batch ciphertexts (N = 1024, no per-item GGSW index)
 * run the latency-mode ladder: one ciphertext per CTA of 4l warps, one warp per
 * (digit, prime) transform.  Bit-identical to the throughput kernel.  -1 selects
 * the automatic threshold (3 x SM count, the default); < -1 only queries.
 * Returns the previous setting. */
int64_t hwb_set_latency_batch(int64_t max_batch);

/* Measurement probe (not a reference function): launches a register-only
 * kernel of `blocks` x 256 threads doing `iters` x 8 independent RNS modular
 * multiplications each (one Shoup product per prime).  Returns the number of
 * RNS modmuls enqueued (the caller times the stream), or -HWB_E* on error.
 * Its rate is P_mm, the integer-pipe roofline denominator. */
int64_t hwb_probe_modmul(uint32_t *sink, int32_t blocks, int32_t iters, void *stream);

/* FP64 pipe probe (NEW): `blocks` x 256 threads, `iters` x 8 independent DFMA
 * chains each.  Returns the FP64 instructions enqueued; its rate is P_fp64, the
 * FFT ladder's roofline denominator. */
int64_t hwb_probe_fp64(uint32_t *sink, int32_t blocks, int32_t iters, void *stream);

/* FFT rounding margin (NEW, test instrumentation): in the build compiled with
 * -DHWB_FFT_MARGIN=1 (libhwb200_margin.so) every FP64 ladder records the largest
 * |y - rint(y)| over all rounded FFT outputs; *out receives it (synchronous) and
 * reset != 0 clears it.  The exactness of the FFT ladders needs it below 1/2.
 * The production build returns HWB_EINVAL. */
int hwb_fft_margin(double *out, int reset);

/* Tensor-core throughput probe (NEW): `blocks` CTAs (one per SM) each issue
 * iters x 4 tcgen05.mma kind::i8 M128 N256 K32 from shared memory into TMEM,
 * the key switch's MMA shape.  Returns the int8 MACs enqueued (the caller times
 * the stream), or -HWB_E* on error.  Its rate is P_i8. */
int64_t hwb_probe_i8mma(uint32_t *sink, int32_t blocks, int32_t iters, void *stream);

/* Number of uint32 words of one GGSW in the NTT domain used by every kernel:
 * 2l rows x 2 components x 2 RNS primes x N. */
size_t hwb_ggsw_ntt_words(const hwb_params *p);

/* Forward transform of `count` GGSWs (coefficient domain, [count][2l][2][N] u32)
 * into the NTT domain ([count][hwb_ggsw_ntt_words] u32).  Replaces the cached
 * spectra of RgswCiphertext.spectra()/rgsw_rep (hw/tfhe.py:158-162, 322-324);
 * used for the bootstrapping key (enc_rgsw_batch of s0, hw/tfhe.py:246-263). */
int hwb_ggsw_to_ntt(const hwb_params *p, const uint32_t *ggsw, uint32_t *ggsw_ntt,
                    int64_t count, void *stream);

/* Batched external product (hw/tfhe.py:301-319 ext_product_batch):
 *   out[b] = sum_r digit_r(in[b]) (*) G[idx[b]][r]
 * ggsw_ntt: NTT-domain GGSWs; ggsw_idx: [B] int32 or NULL (broadcast GGSW 0);
 * in/out: [B][2][N].  in and out may alias. */
int hwb_ext_product(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
                    const uint32_t *in, uint32_t *out, int64_t B, void *stream);

/* Batched CMUX (hw/tfhe.py:334-337 cmux; hw/lut.py:200-206 _cmux_sub):
 *   out[b] = c0[b] + G[idx[b]] (*) (c1[b] - c0[b])
 * If c1 == NULL, c1[b] = c0[b] * X^(rot[b]) (the rotated branch of blind_rotate,
 * hw/tfhe.py:347, and of vp/ivp_batch, hw/lut.py:258, 289); rot may be NULL
 * only when c1 != NULL.  out may alias c0. */
int hwb_cmux(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
             const uint32_t *c1, const uint32_t *c0, const int32_t *rot, uint32_t *out,
             int64_t B, void *stream);

/* Batched CDEMUX (hw/lut.py:113-119): hi = G (*) d, lo = d - hi.
 * d, lo, hi: [B][2][N]; lo may alias d. */
int hwb_cdemux(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
               const uint32_t *d, uint32_t *lo, uint32_t *hi, int64_t B, void *stream);

/* One level of the inverse-vertical-packing CDEMUX tree (hw/lut.py:294-313):
 * for item b < B and poly i < m, with C = G[idx[b]] (the item's tree bit):
 *   hi = C (*) cur[b][i];  next[b][i] = cur[b][i] - hi;  next[b][m+i] = hi.
 * cur: [B][m][2][N], next: [B][2m][2][N]. */
int hwb_ivp_level(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
                  const uint32_t *cur, uint32_t *next, int32_t m, int64_t B, void *stream);

/* One level of the vertical-packing CMUX tree (hw/lut.py:233-247, 130-136):
 *   next[b][i] = cmux(G[idx[b]], cur[b][m+i], cur[b][i]) for i < m.
 * cur: [B][2m][2][N], next: [B][m][2][N]. */
int hwb_vp_level(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
                 const uint32_t *cur, uint32_t *next, int32_t m, int64_t B, void *stream);

/* Per-item negacyclic monomial product out[b] = in[b] * X^(exps[b]) (exponents
 * mod 2N; hw/lut.py:317-325 monomial_gather, hw/ring.py:106-113).  in, out:
 * [B][2][N], must not alias. */
int hwb_monomial_gather(const hwb_params *p, const uint32_t *in, uint32_t *out, const int32_t *exps,
                        int64_t B, void *stream);

/* Forward transform of npolys coefficient-domain polynomials [npolys][N] into
 * the NTT layout of one GGSW row ([npolys][2 primes][N]); used for the secret
 * key of hwb_key_mul. */
int hwb_poly_to_ntt(const hwb_params *p, const uint32_t *in, uint32_t *out, int64_t npolys, void *stream);

/* Client-side key product (hw/tfhe.py:69-78 SecretKey._key_mul, the core of
 * enc_rgsw_batch hw/tfhe.py:246-263): out[i] = in[i] (*) s + add[i] mod 2^32,
 * s given as hwb_poly_to_ntt(s); add may be NULL.  Exact for binary keys. */
int hwb_key_mul(const hwb_params *p, const uint32_t *key_ntt, const uint32_t *in, const uint32_t *add,
                uint32_t *out, int64_t npolys, void *stream);

/* LWE linear combination (NEW; the affine steps between the bootstraps of the
 * PBS inference pipeline, paper_2403_20190_b200/infer_pbs.py): for b < B, k < width
 *   out[b][k] = ((cx[b] x[b][k] + cy[b] y[b][k]) << shift) + (k == width-1 ? cb[b] : 0)
 * mod 2^32.  cx NULL = 1; y NULL (or cy NULL) drops the y term; cb NULL = 0.
 * out may alias x or y.  The word at width-1 is the LWE body b. */
int hwb_lwe_lincomb(const uint32_t *x, const uint32_t *y, uint32_t *out, const int32_t *cx, const int32_t *cy,
                    const uint32_t *cb, int64_t B, int32_t width, int32_t shift, void *stream);

/* numpy Philox4x64-10 generator state at the start of a uniform draw (NEW): the
 * next words of Generator.bytes() are prefix[0 .. nprefix) (still buffered in the
 * host generator), then the uint32 stream of blocks philox(ctr + 1 + g, key). */
typedef struct hwb_philox {
    uint64_t key[2];
    uint64_t ctr[4];
    uint32_t prefix[9];
    int32_t nprefix;
} hwb_philox;

/* Rebuild RGSW rows from a seeded encryption (NEW): pair != 0: out [rows][2][N],
 * out[r][0][j] = word r*N + j of the uniform stream (the a half drawn by
 * enc_rgsw_batch, hw/tfhe.py:246-263, with the 4-byte rng.bytes idiom of
 * hw/tfhe.py:38-40) and out[r][1][j] = b_rows[r][j] (b_rows NULL: untouched);
 * pair == 0: out [rows][N] receives the a words only.  a0fix (NULL: none) holds,
 * per RGSW (2*levels rows), the levels words a[l+t][0] that carry the gadget term
 * m g_t (hw/tfhe.py:259-262); they replace the regenerated words.  Bit-identical
 * to the host draw. */
int hwb_philox_rgsw(const hwb_philox *st, const uint32_t *b_rows, const uint32_t *a0fix, int32_t levels,
                    uint32_t *out, int64_t rows, int32_t N, int32_t pair, void *stream);

/* Row gather out[b] = table[idx[b]] (rows of row_words words, a multiple of 4,
 * 16-byte aligned): per-item test polynomials drawn from a table of LUTs. */
int hwb_gather_rows(const uint32_t *table, const int32_t *idx, uint32_t *out, int64_t B, int32_t row_words,
                    void *stream);

/* Add the RGSW gadget term m * q/beta^(t+1) (hw/tfhe.py:259-262) to B RGSW
 * ciphertexts [B][2l][2][N] for selector bits[B] in {0, 1}. */
int hwb_rgsw_add_gadget(const hwb_params *p, uint32_t *rgsw, const int32_t *bits, int64_t B, void *stream);

/* Packing key switch (hw/tfhe.py:390-439 pack_batch): B outputs, each packing
 * up to N extracted LWEs into one RLWE whose coefficient i carries LWE i:
 *   out[b] = (-sum_{j,t} D_{j,t} (*) K[j,t,0],  b_polys[b] - sum_{j,t} D_{j,t} (*) K[j,t,1]),
 *   D_{j,t}(X) = sum_i digit_t(a^(i)_j) X^i  (gadget `levels` x `base_log`).
 * ksk_ntt: hwb_poly_to_ntt of the packing key [N][levels][2][N] (N*levels*2 polys);
 * apolys: [B][N][N] with apolys[b][j][i] = a^(i)_j (zero for i >= number of LWEs);
 * b_polys: [B][N]; out: [B][2][N]; workspace: hwb_pack_ks_workspace_bytes. */
size_t hwb_pack_ks_workspace_bytes(const hwb_params *p, int64_t B);
int hwb_pack_ks(const hwb_params *p, int32_t levels, int32_t base_log, const uint32_t *ksk_ntt,
                const uint32_t *apolys, const uint32_t *b_polys, uint32_t *out, int64_t B, void *workspace,
                void *stream);

/* dst[k] += sum_{i < count} src[i*words + k] mod 2^32: the IVP rows of `count`
 * samples added into an encrypted model in one pass (hw/hewnn.py:213).
 * 16-byte aligned pointers. */
int hwb_accumulate_rows(uint32_t *dst, const uint32_t *src, int64_t words, int32_t count, void *stream);

/* dst[k] += (negate ? -1 : 1) * src[k mod src_words] mod 2^32 for k < words: exact
 * ciphertext addition for model accumulation and federated merge
 * (hw/hewnn.py:213, 264-271). */
int hwb_accumulate(uint32_t *dst, const uint32_t *src, int64_t words, int64_t src_words, int negate,
                   void *stream);

/* Fused blind rotation (hw/tfhe.py:340-349 blind_rotate), one launch for all L
 * steps: acc[b] <- cmux(G, acc[b] * X^(-I[b][i]), acc[b]) for i < L, with
 * G = ggsw_ntt[i] (ggsw_idx == NULL: L GGSWs shared by the batch, the BSK) or
 * G = ggsw_ntt[ggsw_idx[b][i]] (per-item selector ladders of vertical packing,
 * hw/lut.py:249-260, 280-291; an index < 0 skips the step).
 * exps: [B][L] int32 I values; acc: [B][2][N] in/out. */
int hwb_blind_rotate(const hwb_params *p, const uint32_t *ggsw_ntt, const int32_t *ggsw_idx,
                     const int32_t *exps, uint32_t *acc, int32_t L, int64_t B, void *stream);

/* Batched sample extraction of coefficient `coeff` (hw/tfhe.py:352-361; the
 * batched coefficient-0 form is hw/lut.py:263-266): rlwe [B][2][N] ->
 * lwe [B][N+1] (b last), under the coefficient vector of S1. */
int hwb_sample_extract(const hwb_params *p, const uint32_t *rlwe, uint32_t *lwe, int64_t B,
                       int32_t coeff, void *stream);

/* LWE key switch N -> n (NEW; algebra of pack_batch hw/tfhe.py:397-420):
 * ksk [N][ks_l][n+1], in [B][N+1], out [B][n+1]. */
int hwb_keyswitch(const hwb_params *p, const uint32_t *ksk, const uint32_t *in, uint32_t *out,
                  int64_t B, void *stream);

/* Device workspace bytes hwb_pbs needs for a batch of B. */
size_t hwb_pbs_workspace_bytes(const hwb_params *p, int64_t B);

/* Programmable bootstrapping (NEW composition): mod switch ->
 * acc = TV * X^(-b~) -> blind rotation with I_i = -a~_i -> extract -> key switch.
 * tv: [2][N] (tv_per_item = 0) or [B][2][N]; lwe_in/lwe_out: [B][n+1].
 * If ksk == NULL the key switch is skipped and lwe_out is [B][N+1]. */
int hwb_pbs(const hwb_params *p, const uint32_t *bsk_ntt, const uint32_t *ksk,
            const uint32_t *tv, int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out,
            int64_t B, void *workspace, void *stream);

/* ---- Tensor-core key switch (tcgen05 kind::i8; same result as hwb_keyswitch) ----
 * The key words are split into 4 byte limbs and pre-tiled for the tensor cores
 * (64 output columns x 128 K-bytes per tile).  Available when ks_base_log <= 8
 * (digits are exact int8); hwb_ksk_tc_bytes returns 0 otherwise. */
size_t hwb_ksk_tc_bytes(const hwb_params *p);
/* ksk [N][ks_l][n+1] u32 -> ksk_tc (hwb_ksk_tc_bytes bytes, 16-byte aligned). */
int hwb_ksk_to_tc(const hwb_params *p, const uint32_t *ksk, void *ksk_tc, void *stream);
/* Workspace for hwb_keyswitch_tc: the int8 digit tiles of a batch of B. */
size_t hwb_keyswitch_tc_workspace_bytes(const hwb_params *p, int64_t B);
int hwb_keyswitch_tc(const hwb_params *p, const void *ksk_tc, const uint32_t *in, uint32_t *out,
                     int64_t B, void *workspace, void *stream);
/* hwb_pbs with the tensor-core key switch (ksk_tc from hwb_ksk_to_tc). */
size_t hwb_pbs_tc_workspace_bytes(const hwb_params *p, int64_t B);
int hwb_pbs_tc(const hwb_params *p, const uint32_t *bsk_ntt, const void *ksk_tc,
               const uint32_t *tv, int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out,
               int64_t B, void *workspace, void *stream);

/* ---- FP64 FFT ladder (N = 1024; same results as hwb_pbs) ----
 * The key words are split into signed 16-bit halves whose double-precision FFT
 * spectra form the key; the products are rounded to integers, which is exact
 * (|sum| < 2^37.6, FFT error < 2^-13).  Requires l * 2^base_log < 2^19. */
size_t hwb_bsk_fft_bytes(const hwb_params *p);
/* bsk [n][2l][2][N] u32 (coefficient domain) -> bsk_fft (hwb_bsk_fft_bytes bytes). */
int hwb_bsk_to_fft(const hwb_params *p, const uint32_t *bsk, void *bsk_fft, void *stream);
/* FFT-domain GGSWs for the vertical-packing ladders (training / inference):
 * bytes per GGSW, and the transform of `count` GGSWs [count][2l][2][N] u32. */
size_t hwb_ggsw_fft_bytes(const hwb_params *p);
int hwb_ggsw_to_fft(const hwb_params *p, const uint32_t *ggsw, void *ggsw_fft, int64_t count, void *stream);
/* hwb_blind_rotate / hwb_ivp_level / hwb_vp_level on the FFT path (same results;
 * ggsw_fft from hwb_ggsw_to_fft, indices as in the NTT versions). */
int hwb_blind_rotate_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const int32_t *exps,
                         uint32_t *acc, int32_t L, int64_t B, void *stream);
int hwb_ivp_level_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const uint32_t *cur,
                      uint32_t *next, int32_t m, int64_t B, void *stream);
int hwb_vp_level_fft(const hwb_params *p, const void *ggsw_fft, const int32_t *ggsw_idx, const uint32_t *cur,
                     uint32_t *next, int32_t m, int64_t B, void *stream);
/* Workspace of hwb_pbs_fft: the accumulators between ladder segments and the
 * single-launch ladders' progress words (one per group of 4 ciphertexts, cleared by
 * hwb_pbs_fft on the caller's stream), plus the key switch's buffers when
 * with_keyswitch.  One workspace serves one call at a time (one per stream). */
size_t hwb_pbs_fft_workspace_bytes(const hwb_params *p, int64_t B, int with_keyswitch);
/* Ladder steps per segment (per calling thread): a segment's key slices stay L2-resident.
 * Default 64 for the modes that launch once per segment and 48 for the single-launch
 * ladders (FFT mode 5) until this is called; afterwards `steps` for both. */
int hwb_set_fft_segment(int steps);
/* Ciphertexts per CTA of the FFT PBS ladder (1, 2 or 4): they share every staged key
 * slice (one shared-memory write, several reads). */
int hwb_set_fft_group(int ciphertexts_per_cta);
/* Batches of at most max_batch ciphertexts (-1: one per SM, the default) run the
 * FFT latency ladder at N = 1024: one ciphertext per CTA of 2l groups of 64
 * threads (one digit transform per group, the four accumulators on four groups),
 * the whole ladder in one launch.  Bit-identical to the throughput ladder.
 * Returns the previous setting (the reference has no counterpart). */
int64_t hwb_set_fft_latency_batch(int64_t max_batch);
/* FFT PBS ladder shape (per calling thread): 0 = register accumulators
 * (hwb_set_fft_group ciphertexts per CTA); tensor-memory accumulators with
 * 1 = two ciphertexts per thread (8 warps/SM), 2 = one per thread (16 warps/SM),
 * 3 = lane-paired ciphertexts (a lane pair reads each key value / twiddle at one
 * address), 4 = 3 as one 16-warp CTA of decoupled groups, 5 = 3 with decoupled halves
 * (default; from 4 ciphertexts per SM), 6 = 5 as one 16-warp CTA with a two-slot key
 * ring, 7 = 5 on 32-thread transforms with 16 values per thread (one shared-memory
 * transpose per transform), 8 = 5 with one launch per segment (5 runs the whole ladder
 * as one launch whose CTAs are (segment, ciphertext group) pairs in segment-major order).  At N = 2048 any mode >= 1 selects the N = 2048 TMEM ladder
 * (from 4 per SM).  All bit-identical; EINVAL outside 0..8 (the reference has no counterpart). */
int hwb_set_fft_mode(int mode);
/* Batches of at most max_batch ciphertexts (default -1: the cluster capacity) run the cluster latency
 * ladder at N = 1024: one ciphertext per cluster of 2l CTAs on 2l SMs (digit row r
 * on CTA r, partial products summed over distributed shared memory), so the key
 * streams through 2l SMs.  Returns the previous setting (max_batch < -1: query only). */
int64_t hwb_set_fft_cluster_batch(int64_t max_batch);
/* Clusters of the cluster latency ladder that fit co-resident on the device for
 * these parameters (cudaOccupancyMaxActiveClusters; 0 where the ladder does not
 * apply): the default batch limit of that ladder. */
int64_t hwb_fft_cluster_capacity(const hwb_params *p);
/* Shape of the cluster latency ladder: 0 = 2l CTAs, one digit row each (default);
 * 1 = 4 CTAs, one accumulator quarter each, every CTA transforming all digit rows. */
int hwb_set_fft_cluster_mode(int mode);
/* hwb_pbs on the FFT ladder with the tensor-core key switch (ksk_tc from
 * hwb_ksk_to_tc); ksk_tc == NULL skips the key switch (lwe_out [B][N+1]). */
int hwb_pbs_fft(const hwb_params *p, const void *bsk_fft, const void *ksk_tc, const uint32_t *tv,
                int tv_per_item, const uint32_t *lwe_in, uint32_t *lwe_out, int64_t B, void *workspace,
                void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HWB_H */
