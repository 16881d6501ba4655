/*
 * CPU oracle for batched TFHE bootstrapping at q = 2^32 -- TEST INFRASTRUCTURE.
 *
 * Plain-C restatement of the reference's exact path (/root/reference/pkg/src/
 * hewisard, cited hw/<file>:<line>) used by tests/ as the checker at sizes the
 * Python oracle cannot reach, and by bench.py's CPU-baseline leg.  It is never
 * linked into the product.
 *
 * All arithmetic is uint32 wrap-around, which IS arithmetic mod q = 2^32, so the
 * schoolbook negacyclic products (hw/ring.py:92-98) are exact without big ints.
 * Pinned against the reference-generated fixtures in tests/golden/ by
 * tests/test_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* hw/ring.py:126-151: signed digits in [-beta/2, beta/2), LSB-first with carry;
 * d[t] carries q / beta^(t+1). */
static void decompose(uint32_t x, int levels, int w, int32_t *d)
{
    int total = levels * w;
    int64_t u;
    if (total < 32)
        u = (int64_t)((uint32_t)(x + (1u << (31 - total))) >> (32 - total));
    else
        u = (int64_t)x;
    int64_t beta = (int64_t)1 << w, half = beta >> 1, mask = beta - 1;
    for (int t = levels - 1; t >= 0; --t) {
        int64_t dd = u & mask;
        if (dd >= half) dd -= beta;
        u = (u - dd) >> w;
        d[t] = (int32_t)dd;
    }
}

/* out += d (*) g negacyclic, d small signed, g u32 (hw/ring.py:92-98). */
static void negacyclic_mac(uint32_t *out, const int32_t *d, const uint32_t *g, int N)
{
    for (int j = 0; j < N; ++j) {
        uint32_t dj = (uint32_t)d[j];
        if (!dj) continue;
        uint32_t *o = out + j;
        for (int k = 0; k < N - j; ++k) o[k] += dj * g[k];
        const uint32_t *gw = g + N - j;
        for (int k = 0; k < j; ++k) out[k] -= dj * gw[k];
    }
}

/* hw/tfhe.py:290-298 + 301-315 for one item: out = sum_r digit_r (*) G[r]. */
static void ext_product_one(int N, int levels, int w, const uint32_t *ggsw,
                            const uint32_t *ct, uint32_t *out, int32_t *dig)
{
    /* dig: (2*levels, N); rows 0..l-1 = digits of b, rows l..2l-1 = digits of a */
    int32_t tmp[32];
    for (int c = 0; c < 2; ++c)
        for (int i = 0; i < N; ++i) {
            decompose(ct[c * N + i], levels, w, tmp);
            int base = (c == 1) ? 0 : levels;
            for (int t = 0; t < levels; ++t) dig[(base + t) * N + i] = tmp[t];
        }
    memset(out, 0, sizeof(uint32_t) * 2 * N);
    for (int r = 0; r < 2 * levels; ++r)
        for (int c = 0; c < 2; ++c)
            negacyclic_mac(out + c * N, dig + r * N, ggsw + ((size_t)r * 2 + c) * N, N);
}

static void set_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* rgsw: (B|1, 2l, 2, N); cts/out: (B, 2, N). */
void orc_ext_product(int N, int levels, int w, const uint32_t *rgsw, int rgsw_bcast,
                     const uint32_t *cts, uint32_t *out, int64_t B, int nthreads)
{
    set_threads(nthreads);
    size_t gsz = (size_t)2 * levels * 2 * N;
#pragma omp parallel
    {
        int32_t *dig = (int32_t *)malloc(sizeof(int32_t) * 2 * levels * N);
#pragma omp for schedule(dynamic)
        for (int64_t b = 0; b < B; ++b)
            ext_product_one(N, levels, w, rgsw + (rgsw_bcast ? 0 : b * gsz),
                            cts + b * 2 * N, out + b * 2 * N, dig);
        free(dig);
    }
}

/* x * X^e (hw/ring.py:106-113), e mod 2N. */
static void monomial(const uint32_t *x, int64_t e, uint32_t *out, int N)
{
    int64_t m = 2 * (int64_t)N;
    e = ((e % m) + m) % m;
    for (int i = 0; i < N; ++i) {
        int64_t src = ((int64_t)i - e + m) % m;
        out[i] = src < N ? x[src] : (uint32_t)(0u - x[src - N]);
    }
}

static void blind_rotate_one(int N, int levels, int w, const uint32_t *bsk,
                             const int32_t *exps, int L, uint32_t *acc,
                             uint32_t *work, int32_t *dig)
{
    size_t gsz = (size_t)2 * levels * 2 * N;
    uint32_t *diff = work, *prod = work + 2 * N;
    for (int i = 0; i < L; ++i) {
        /* hw/tfhe.py:346-348: acc = acc + C_i (*) (acc X^(-I_i) - acc) */
        for (int c = 0; c < 2; ++c) monomial(acc + c * N, -(int64_t)exps[i], diff + c * N, N);
        for (int k = 0; k < 2 * N; ++k) diff[k] -= acc[k];
        ext_product_one(N, levels, w, bsk + i * gsz, diff, prod, dig);
        for (int k = 0; k < 2 * N; ++k) acc[k] += prod[k];
    }
}

/* hw/tfhe.py:340-349 per item: bsk (L, 2l, 2, N) shared, exps (B, L), acc (B, 2, N). */
void orc_blind_rotate(int N, int levels, int w, const uint32_t *bsk, const int32_t *exps,
                      uint32_t *acc, int L, int64_t B, int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel
    {
        uint32_t *work = (uint32_t *)malloc(sizeof(uint32_t) * 4 * N);
        int32_t *dig = (int32_t *)malloc(sizeof(int32_t) * 2 * levels * N);
#pragma omp for schedule(dynamic)
        for (int64_t b = 0; b < B; ++b)
            blind_rotate_one(N, levels, w, bsk, exps + b * L, L, acc + b * 2 * N, work, dig);
        free(work);
        free(dig);
    }
}

/* NEW: LWE key switch (algebra of hw/tfhe.py:397-420).
 * ksk (N, lks, n+1); in (B, N+1); out (B, n+1). */
static void keyswitch_one(int N, int n, int lks, int wks, const uint32_t *ksk,
                          const uint32_t *in, uint32_t *out)
{
    int32_t d[32];
    memset(out, 0, sizeof(uint32_t) * (n + 1));
    for (int j = 0; j < N; ++j) {
        decompose(in[j], lks, wks, d);
        for (int t = 0; t < lks; ++t) {
            uint32_t dt = (uint32_t)d[t];
            if (!dt) continue;
            const uint32_t *row = ksk + ((size_t)j * lks + t) * (n + 1);
            for (int k = 0; k <= n; ++k) out[k] += dt * row[k];
        }
    }
    for (int k = 0; k < n; ++k) out[k] = 0u - out[k];
    out[n] = in[N] - out[n];
}

void orc_keyswitch(int N, int n, int lks, int wks, const uint32_t *ksk, const uint32_t *in,
                   uint32_t *out, int64_t B, int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b)
        keyswitch_one(N, n, lks, wks, ksk, in + b * (N + 1), out + b * (n + 1));
}

/* Packing key switch, hw/tfhe.py:390-420 (exact branch): for output b,
 * acc[c] = sum_{j<N} sum_{t<l} D_{j,t} (*) ksk[j][t][c] with D_{j,t}(X) =
 * sum_{i<k} digit_t(a^(i)_j) X^i; out = (-acc[0], b_poly - acc[1]).
 * ksk (N, l, 2, N); a_stacks (B, k, N); b_polys (B, N); out (B, 2, N). */
void orc_pack_ks(int N, int levels, int w, const uint32_t *ksk, const uint32_t *a_stacks,
                 const uint32_t *b_polys, uint32_t *out, int64_t B, int k, int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel
    {
        uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * 2 * N);
        int32_t d[32];
#pragma omp for schedule(dynamic)
        for (int64_t b = 0; b < B; ++b) {
            memset(acc, 0, sizeof(uint32_t) * 2 * N);
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < k; ++i) {
                    decompose(a_stacks[((size_t)b * k + i) * N + j], levels, w, d);
                    for (int t = 0; t < levels; ++t) {
                        uint32_t dt = (uint32_t)d[t];
                        if (!dt) continue;
                        for (int c = 0; c < 2; ++c) {   /* acc[c] += dt X^i (*) K */
                            const uint32_t *K = ksk + (((size_t)j * levels + t) * 2 + c) * N;
                            uint32_t *o = acc + c * N;
                            for (int m = 0; m < N - i; ++m) o[i + m] += dt * K[m];
                            for (int m = N - i; m < N; ++m) o[i + m - N] -= dt * K[m];
                        }
                    }
                }
            for (int m = 0; m < N; ++m) {
                out[(size_t)b * 2 * N + m] = 0u - acc[m];
                out[(size_t)b * 2 * N + N + m] = b_polys[(size_t)b * N + m] - acc[N + m];
            }
        }
        free(acc);
    }
}

/* NEW: mod switch round(x 2N / q) mod 2N (rounding idiom hw/ring.py:139-140). */
static int32_t mod_switch(uint32_t x, int N)
{
    int logm = 0;
    while ((1 << logm) < 2 * N) ++logm;
    return (int32_t)((uint32_t)(x + (1u << (31 - logm))) >> (32 - logm));
}

/* NEW composition: mod switch, TV * X^(-b~), blind rotation with
 * I_i = -a~_i, extract coefficient 0 (hw/tfhe.py:352-361), optional key switch.
 * lwe_in (B, n+1); tv (2, N) or (B, 2, N); lwe_out (B, n+1) or (B, N+1) w/o KS. */
void orc_pbs(int N, int n, int levels, int w, int lks, int wks, const uint32_t *bsk,
             const uint32_t *ksk, const uint32_t *tv, int tv_per_item,
             const uint32_t *lwe_in, uint32_t *lwe_out, int64_t B, int do_ks, int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel
    {
        uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * 2 * N);
        uint32_t *work = (uint32_t *)malloc(sizeof(uint32_t) * 4 * N);
        uint32_t *ext = (uint32_t *)malloc(sizeof(uint32_t) * (N + 1));
        int32_t *dig = (int32_t *)malloc(sizeof(int32_t) * 2 * levels * N);
        int32_t *exps = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
#pragma omp for schedule(dynamic)
        for (int64_t b = 0; b < B; ++b) {
            const uint32_t *row = lwe_in + b * (n + 1);
            const uint32_t *t = tv + (tv_per_item ? b * 2 * N : 0);
            int32_t bt = mod_switch(row[n], N);
            for (int c = 0; c < 2; ++c) monomial(t + c * N, -(int64_t)bt, acc + c * N, N);
            for (int i = 0; i < n; ++i) exps[i] = -mod_switch(row[i], N);
            blind_rotate_one(N, levels, w, bsk, exps, n, acc, work, dig);
            ext[0] = acc[0];
            for (int j = 1; j < N; ++j) ext[j] = 0u - acc[N - j];
            ext[N] = acc[N];
            if (do_ks)
                keyswitch_one(N, n, lks, wks, ksk, ext, lwe_out + b * (n + 1));
            else
                memcpy(lwe_out + b * (N + 1), ext, sizeof(uint32_t) * (N + 1));
        }
        free(acc); free(work); free(ext); free(dig); free(exps);
    }
}
