/*
 * synth/gen.c -- seeded synthetic edge streams shaped like the paper's workloads (INPUTS ONLY: no part of
 * the method's arithmetic lives here; shared by the oracle tests and the CUDA path's tests / bench, the one
 * thing the two sides may share).  Recipe: DESIGN.md "Input recipe"; BASELINE.json configs.
 *
 * Counter-based and thread-count independent: every random number is a keyed hash of (stream id, index),
 * so the output depends only on the arguments.  Every stream is a simple graph (self-loops and undirected
 * duplicates dropped), vertex ids relabelled by a keyed permutation, delivered in a keyed pseudo-random
 * order with each edge's orientation flipped by a hash bit.
 *
 *   gen_rmat      R-MAT(a, b, c, d): per draw, one quadrant choice per bit level (probabilities quantised
 *                 to 1/65536), ndraws draws, dedup
 *   gen_chung_lu  Chung-Lu: weights (i + i0)^(-1/(gamma-1)), i0 set so that the largest expected degree is
 *                 dmax; endpoints i.i.d. proportional to weight; draws until m unique, m of them kept
 *
 * Permutations are cycle-walking balanced Feistel networks (4 rounds, keyed hash round function) on the
 * smallest even bit width covering the domain: bijections of [0, n) without an O(n) table.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) { /* splitmix64 finaliser */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t i) {
    return mix64(mix64(seed ^ (stream * 0xD6E8FEB86659FD93ull)) ^ mix64(i + 0x632BE59BD9B4E019ull * stream));
}

/* ---------------- keyed permutation of [0, n) ---------------- */
typedef struct { uint64_t n; uint32_t half; uint64_t k[4]; } perm_t;

static void perm_init(perm_t *p, uint64_t n, uint64_t seed, uint64_t stream) {
    uint32_t bits = 0;
    while ((1ull << bits) < n) ++bits;
    if (bits & 1) ++bits;
    if (bits < 2) bits = 2;
    p->n = n;
    p->half = bits / 2;
    for (int r = 0; r < 4; ++r) p->k[r] = rnd(seed, stream, 0x5EED0000ull + (uint64_t)r);
}
static inline uint64_t feistel(const perm_t *p, uint64_t x) {
    const uint64_t m = (1ull << p->half) - 1;
    uint64_t L = x >> p->half, R = x & m;
    for (int r = 0; r < 4; ++r) {
        uint64_t t = L ^ (mix64(R ^ p->k[r]) & m);
        L = R;
        R = t;
    }
    return (L << p->half) | R;
}
static inline uint64_t perm_apply(const perm_t *p, uint64_t x) { /* cycle walking stays inside [0, n) */
    do { x = feistel(p, x); } while (x >= p->n);
    return x;
}

/* ---------------- parallel LSD radix sort of u64 keys on their low `bits` bits ---------------- */
static int radix_sort_u64(uint64_t *a, uint64_t n, int bits) {
    uint64_t *tmp = (uint64_t *)malloc(8 * (n ? n : 1));
    if (!tmp) return -1;
    const int D = 11, NB = 1 << D;
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    uint64_t *hist = (uint64_t *)calloc((size_t)nt * NB, 8);
    if (!hist) { free(tmp); return -1; }
    uint64_t *src = a, *dst = tmp;
    int passes = 0;
    for (int sh = 0; sh < bits; sh += D, ++passes) {
        memset(hist, 0, (size_t)nt * NB * 8);
#pragma omp parallel num_threads(nt)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            uint64_t lo = n * (uint64_t)t / (uint64_t)nt, hi = n * (uint64_t)(t + 1) / (uint64_t)nt;
            uint64_t *h = hist + (size_t)t * NB;
            for (uint64_t i = lo; i < hi; ++i) h[(src[i] >> sh) & (NB - 1)]++;
#pragma omp barrier
#pragma omp single
            {
                uint64_t run = 0;
                for (int d = 0; d < NB; ++d)
                    for (int q = 0; q < nt; ++q) {
                        uint64_t c = hist[(size_t)q * NB + d];
                        hist[(size_t)q * NB + d] = run;
                        run += c;
                    }
            }
            for (uint64_t i = lo; i < hi; ++i) dst[h[(src[i] >> sh) & (NB - 1)]++] = src[i];
        }
        uint64_t *x = src; src = dst; dst = x;
    }
    if (passes & 1) memcpy(a, src, 8 * n);
    free(hist);
    free(tmp);
    return 0;
}

static uint64_t unique_u64(uint64_t *a, uint64_t n) {
    if (!n) return 0;
    uint64_t k = 1;
    for (uint64_t i = 1; i < n; ++i)
        if (a[i] != a[k - 1]) a[k++] = a[i];
    return k;
}

/* Keys (lo << vbits | hi), sorted and unique, -> out[0 .. take) in keyed pseudo-random order and random
   orientation: element i goes to position pi(i); elements with pi(i) >= take are dropped (a uniformly
   chosen subset when take < nkeys). */
static void emit(const uint64_t *keys, uint64_t nkeys, uint64_t take, int vbits, uint64_t seed, uint32_t *out) {
    perm_t P;
    perm_init(&P, nkeys, seed, 7);
    const uint64_t vm = (1ull << vbits) - 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)nkeys; ++i) {
        uint64_t j = perm_apply(&P, (uint64_t)i);
        if (j >= take) continue;
        uint32_t lo = (uint32_t)(keys[i] >> vbits), hi = (uint32_t)(keys[i] & vm);
        int flip = (int)(rnd(seed, 8, j) & 1);
        out[2 * j] = flip ? hi : lo;
        out[2 * j + 1] = flip ? lo : hi;
    }
}

/* R-MAT: returns the number of unique edges written to out (capacity 2 * ndraws uint32), or -1. */
int64_t gen_rmat(int scale, uint64_t ndraws, uint64_t seed, double a, double b, double c, uint32_t *out) {
    if (scale < 1 || scale > 31) return -1;
    const uint32_t ta = (uint32_t)llround(a * 65536.0), tab = (uint32_t)llround((a + b) * 65536.0),
                   tabc = (uint32_t)llround((a + b + c) * 65536.0);
    uint64_t *keys = (uint64_t *)malloc(8 * (ndraws ? ndraws : 1));
    if (!keys) return -1;
    perm_t V;
    perm_init(&V, 1ull << scale, seed, 2);
    const int nh = (scale + 3) / 4;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)ndraws; ++i) {
        uint32_t u = 0, v = 0;
        for (int h = 0; h < nh; ++h) {
            uint64_t x = rnd(seed, 1, (uint64_t)i * (uint64_t)nh + (uint64_t)h);
            for (int q = 0; q < 4 && 4 * h + q < scale; ++q) {
                uint32_t r16 = (uint32_t)(x >> (16 * q)) & 0xFFFFu;
                uint32_t ub = r16 >= tab, vb = (r16 >= ta && r16 < tab) || r16 >= tabc;
                u |= ub << (4 * h + q);
                v |= vb << (4 * h + q);
            }
        }
        uint64_t pu = perm_apply(&V, u), pv = perm_apply(&V, v);
        uint64_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
        keys[i] = lo == hi ? ~0ull : (lo << scale) | hi;  /* self-loops sort last and are cut below */
    }
    if (radix_sort_u64(keys, ndraws, 2 * scale + 1) != 0) { free(keys); return -1; }
    uint64_t k = unique_u64(keys, ndraws);
    if (k && keys[k - 1] == ~0ull) --k;
    emit(keys, k, k, scale, seed, out);
    free(keys);
    return (int64_t)k;
}

/* Chung-Lu: exactly m unique edges into out (capacity 2 * m uint32); returns m or -1. */
int64_t gen_chung_lu(uint64_t n, uint64_t m, double gamma, double dmax, uint64_t seed, uint32_t *out) {
    if (n < 2 || n > 0xFFFFFFFEull || m > n * (n - 1) / 2) return -1;
    double *cdf = (double *)malloc(8 * n);
    if (!cdf) return -1;
    const double ex = -1.0 / (gamma - 1.0);
    double lo_i0 = 1e-3, hi_i0 = 1e7;
    for (int it = 0; it < 80; ++it) { /* the largest expected degree 2 m w_0 / sum w decreases in i0 */
        double mid = sqrt(lo_i0 * hi_i0), sum = 0.0;
#pragma omp parallel for schedule(static) reduction(+:sum)
        for (int64_t i = 0; i < (int64_t)n; ++i) sum += pow((double)i + mid, ex);
        if (2.0 * (double)m * pow(mid, ex) / sum > dmax) lo_i0 = mid; else hi_i0 = mid;
    }
    double run = 0.0;
    for (uint64_t i = 0; i < n; ++i) { run += pow((double)i + hi_i0, ex); cdf[i] = run; }
    for (uint64_t i = 0; i < n; ++i) cdf[i] /= run;
    int vbits = 1;
    while ((1ull << vbits) < n) ++vbits;
    perm_t V;
    perm_init(&V, n, seed, 2);
    uint64_t cap = m + m / 4 + 4096, have = 0, drawn = 0;
    uint64_t *keys = (uint64_t *)malloc(8 * cap);
    if (!keys) { free(cdf); return -1; }
    for (int round = 0; have < m && round < 64; ++round) {
        uint64_t k = (uint64_t)((double)(m - have) * 1.15) + 1024;
        if (have + k > cap) {
            cap = have + k;
            uint64_t *nk = (uint64_t *)realloc(keys, 8 * cap);
            if (!nk) { free(keys); free(cdf); return -1; }
            keys = nk;
        }
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < (int64_t)k; ++t) {
            uint32_t e[2];
            for (int s = 0; s < 2; ++s) {
                double U = (double)(rnd(seed, 3 + s, drawn + (uint64_t)t) >> 11) * 0x1.0p-53;
                uint64_t L = 0, H = n - 1; /* first i with cdf[i] > U */
                while (L < H) { uint64_t M = (L + H) / 2; if (cdf[M] > U) H = M; else L = M + 1; }
                e[s] = (uint32_t)perm_apply(&V, L);
            }
            uint64_t a = e[0] < e[1] ? e[0] : e[1], b = e[0] < e[1] ? e[1] : e[0];
            keys[have + (uint64_t)t] = a == b ? ~0ull : (a << vbits) | b;
        }
        drawn += k;
        if (radix_sort_u64(keys, have + k, 2 * vbits + 1) != 0) { free(keys); free(cdf); return -1; }
        have = unique_u64(keys, have + k);
        if (have && keys[have - 1] == ~0ull) --have;
    }
    free(cdf);
    if (have < m) { free(keys); return -1; }
    emit(keys, have, m, vbits, seed, out);
    free(keys);
    return (int64_t)m;
}

int gen_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
