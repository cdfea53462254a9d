/*
 * oracle/indexed.c -- the paper's *bulk* algorithm, bulkUpdateAll, on the CPU.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_1308_2166_b200/csrc).
 *
 * Plain and literal, following PAPER.md §4 (lines 484-845) step by step:
 *   Step 1: map(randInt(|W|+|E|)) -> idx[]; extract + combine.
 *   Step 2: rankAll(W) = build F (2 records per edge),
 *          sort by (src asc, pos desc), rank by the App. B scan with resets;
 *          Q1 multisearch (u, p) -> ld, rd; chi+ = ld + rd; one draw; Q2 (src, a) -> f2.
 *   Step 3: edges sorted by (src, dst); multisearch the closing
 *          edge; accept if its pos is after f2.
 * Multisearch is done by binary search over the sorted sequence (a library-grade
 * primitive standing for the paper's exactMultiSearch / predEQMultiSearch); the
 * sort is qsort (the comparison order is total, so stability is moot).
 * Estimator loops are OpenMP "parallel for" -- each estimator's update is a map.
 *
 * Randomness: Philox4x32-10 + Lemire, readings R7/R8 (the paper is silent,
 * PAPER.md:988-989); implemented here independently of the CUDA path.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EMPTY_V 0xFFFFFFFFu
#define EMPTY_P UINT64_MAX
#define C_MAX 0x7FFFFFFFull

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ENOMEM = -2, ORC_ESELFLOOP = -3, ORC_EDUP = -4, ORC_EOVERFLOW = -5 };

/* ---------------- Philox4x32-10 (Salmon et al. SC'11) ---------------- */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int rnd = 0; rnd < 10; ++rnd) {
        if (rnd) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void block_words(uint64_t seed, uint64_t i, uint32_t b, uint32_t w, uint64_t *lo, uint64_t *hi) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), b, w};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox(ctr, key, o);
    *lo = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
    *hi = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
}

/* Lemire: p = x*n; reject while low64(p) < (2^64 - n) mod n; return high64(p).
   retry t uses ctr.w = base + t, low word. */
static uint64_t lemire(uint64_t n, uint64_t x, uint64_t seed, uint64_t i, uint32_t b, uint32_t base) {
    unsigned __int128 p = (unsigned __int128)x * n;
    uint64_t l = (uint64_t)p;
    if (l < n) {
        uint64_t t = (0 - n) % n;
        uint32_t k = 0;
        while (l < t) {
            uint64_t lo, hi;
            ++k;
            block_words(seed, i, b, base + k, &lo, &hi);
            p = (unsigned __int128)lo * n;
            l = (uint64_t)p;
        }
    }
    return (uint64_t)(p >> 64);
}

uint64_t orc_lemire_words(uint64_t n, uint64_t x, uint64_t seed, uint64_t i, uint32_t b, uint32_t base) {
    return lemire(n, x, seed, i, b, base);
}

/* ---------------- state ---------------- */
typedef struct {
    uint64_t r, seed, first, count;
    uint64_t m;   /* |E|: edges seen */
    uint32_t b;   /* non-empty batches seen */
    uint32_t *r1; /* 2*count: lo, hi */
    uint32_t *r2;
    uint64_t *p1, *p2;
    uint32_t *c;
    uint8_t *closed;
    /* per-step trace of the last accepted batch (test wiring, orc_set_trace): Step 1's replacement index j
       (UINT32_MAX = f1 retained), chi^- after Step 1, rank(u->v) and rank(v->u) (chi^+ = ld + rd), Step 2's
       draw d2 (UINT64_MAX = no draw), the batch position of the new f2 (UINT32_MAX = kept), Step 3's flag */
    int trace;
    uint32_t *t_j, *t_chim, *t_ld, *t_rd, *t_k2;
    uint64_t *t_d2;
    uint8_t *t_closed;
} orc;

orc *orc_create(uint64_t r, uint64_t seed, uint64_t first, uint64_t count) {
    if (r == 0 || first + count > r) return NULL;
    orc *o = (orc *)calloc(1, sizeof(orc));
    if (!o) return NULL;
    o->r = r; o->seed = seed; o->first = first; o->count = count;
    uint64_t n = count ? count : 1;
    o->r1 = (uint32_t *)malloc(8 * n); o->r2 = (uint32_t *)malloc(8 * n);
    o->p1 = (uint64_t *)malloc(8 * n); o->p2 = (uint64_t *)malloc(8 * n);
    o->c = (uint32_t *)calloc(n, 4); o->closed = (uint8_t *)calloc(n, 1);
    if (!o->r1 || !o->r2 || !o->p1 || !o->p2 || !o->c || !o->closed) return NULL;
    for (uint64_t i = 0; i < count; ++i) {
        o->r1[2 * i] = o->r1[2 * i + 1] = EMPTY_V;
        o->r2[2 * i] = o->r2[2 * i + 1] = EMPTY_V;
        o->p1[i] = o->p2[i] = EMPTY_P;
    }
    return o;
}

void orc_destroy(orc *o) {
    if (!o) return;
    free(o->t_j); free(o->t_chim); free(o->t_ld); free(o->t_rd); free(o->t_k2); free(o->t_d2); free(o->t_closed);
    free(o->r1); free(o->r2); free(o->p1); free(o->p2); free(o->c); free(o->closed);
    free(o);
}

/* ---------------- rankAll (Lemma rank-all) ---------------- */
typedef struct { uint32_t src, dst; int64_t pos; uint32_t rank; } arc_rec;

static int cmp_src_posdesc(const void *a, const void *b) {
    const arc_rec *x = (const arc_rec *)a, *y = (const arc_rec *)b;
    if (x->src != y->src) return x->src < y->src ? -1 : 1;
    if (x->pos != y->pos) return x->pos > y->pos ? -1 : 1; /* decreasing pos */
    return 0;
}

typedef struct { uint32_t src, dst; int64_t pos; } edge_rec;

static int cmp_src_dst(const void *a, const void *b) {
    const edge_rec *x = (const edge_rec *)a, *y = (const edge_rec *)b;
    if (x->src != y->src) return x->src < y->src ? -1 : 1;
    if (x->dst != y->dst) return x->dst < y->dst ? -1 : 1;
    return 0;
}

/* first index in F[0..n) with src >= u */
static int64_t lower_src(const arc_rec *F, int64_t n, uint32_t u) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (F[mid].src < u) lo = mid + 1; else hi = mid; }
    return lo;
}

/* first index in F[0..n) with src > u */
static int64_t upper_src(const arc_rec *F, int64_t n, uint32_t u) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (F[mid].src <= u) lo = mid + 1; else hi = mid; }
    return lo;
}

/* (Q1) (u, p): the arc with src = u and the least pos >= p; -1 if none.
   Within the src group pos is decreasing, so it is the last index with pos >= p. */
static int64_t q1(const arc_rec *F, int64_t n, uint32_t u, int64_t p) {
    int64_t g0 = lower_src(F, n, u), g1 = upper_src(F, n, u);
    if (g0 >= g1) return -1;
    int64_t lo = g0, hi = g1; /* find first index with pos < p */
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (F[mid].pos >= p) lo = mid + 1; else hi = mid; }
    return lo - 1 >= g0 ? lo - 1 : -1;
}

/* (Q2) (u, a): the arc with src = u and rank a: observation 2
   orders a src group by increasing rank, so it is group start + a. */
static int64_t q2(const arc_rec *F, int64_t n, uint32_t u, uint32_t a) {
    int64_t g0 = lower_src(F, n, u);
    int64_t k = g0 + a;
    if (k >= n || F[k].src != u || F[k].rank != a) return -1;
    return k;
}

static int64_t find_edge(const edge_rec *S, int64_t n, uint32_t a, uint32_t z) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (S[mid].src < a || (S[mid].src == a && S[mid].dst < z)) lo = mid + 1; else hi = mid;
    }
    if (lo < n && S[lo].src == a && S[lo].dst == z) return lo;
    return -1;
}

/* bulkUpdateAll for one batch; edges = 2*w uint32 (u, v) in arrival order, any orientation.
   forced_d1 / forced_d2 (test wiring, may be NULL): per estimator, the value of Step 1's draw
   randInt(|W|+|E|) and of Step 2's draw over chi^- + chi^+ instead of the Philox + Lemire draw;
   an out-of-range forced value rejects the batch with ORC_EINVAL (nothing is mutated). */
static int push_batch_impl(orc *o, const uint32_t *edges, uint64_t w, const uint64_t *forced_d1,
                           const uint64_t *forced_d2) {
    if (w == 0) return ORC_OK;
    int err_inval = 0, err_loop = 0, err_dup = 0;
    uint32_t *E = (uint32_t *)malloc(8 * w);           /* normalized W */
    edge_rec *S = (edge_rec *)malloc(sizeof(edge_rec) * w);
    arc_rec *F = (arc_rec *)malloc(sizeof(arc_rec) * 2 * w);
    int64_t *idx = (int64_t *)malloc(8 * (o->count ? o->count : 1));
    if (!E || !S || !F || !idx) { free(E); free(S); free(F); free(idx); return ORC_ENOMEM; }
    for (uint64_t k = 0; k < w; ++k) {
        uint32_t u = edges[2 * k], v = edges[2 * k + 1];
        if (u == EMPTY_V || v == EMPTY_V) err_inval = 1;
        if (u == v) err_loop = 1;
        E[2 * k] = u < v ? u : v;
        E[2 * k + 1] = u < v ? v : u;
    }
    /* Step 3's "edges" array, built up front so a duplicate rejects the batch
       before any state changes. */
    for (uint64_t k = 0; k < w; ++k) { S[k].src = E[2 * k]; S[k].dst = E[2 * k + 1]; S[k].pos = (int64_t)k; }
    qsort(S, w, sizeof(edge_rec), cmp_src_dst);
    for (uint64_t k = 1; k < w; ++k)
        if (S[k].src == S[k - 1].src && S[k].dst == S[k - 1].dst) err_dup = 1;
    int code = err_inval ? ORC_EINVAL : err_loop ? ORC_ESELFLOOP : err_dup ? ORC_EDUP : ORC_OK;

    /* rankAll(W): F, sort by (src, -pos), scan with resets */
    for (uint64_t k = 0; k < w; ++k) {
        F[2 * k].src = E[2 * k]; F[2 * k].dst = E[2 * k + 1]; F[2 * k].pos = (int64_t)k;
        F[2 * k + 1].src = E[2 * k + 1]; F[2 * k + 1].dst = E[2 * k]; F[2 * k + 1].pos = (int64_t)k;
    }
    int64_t nF = (int64_t)(2 * w);
    qsort(F, (size_t)nF, sizeof(arc_rec), cmp_src_posdesc);
    {   /* App. B loop: out[i] = sum; if A[i] is the reset: sum = 0 else sum += 1, where the reset
           marks the last record of each src group (reading R14). */
        uint32_t sum = 0;
        for (int64_t i = 0; i < nF; ++i) {
            F[i].rank = sum;
            int last = (i + 1 == nF) || F[i + 1].src != F[i].src;
            if (last) sum = 0; else sum += 1;
        }
    }
    if (code != ORC_OK) { free(E); free(S); free(F); free(idx); return code; }

    const uint64_t m_prev = o->m, seed = o->seed, first = o->first;
    const uint32_t b = o->b;
    const int64_t cnt = (int64_t)o->count;
    /* all-or-nothing: the state is snapshotted and restored if some estimator's chi overflows
       (reading R13) or a forced draw is out of range */
    const uint64_t n = o->count ? o->count : 1;
    uint32_t *s_r1 = (uint32_t *)malloc(8 * n), *s_r2 = (uint32_t *)malloc(8 * n), *s_c = (uint32_t *)malloc(4 * n);
    uint64_t *s_p1 = (uint64_t *)malloc(8 * n), *s_p2 = (uint64_t *)malloc(8 * n);
    uint8_t *s_cl = (uint8_t *)malloc(n);
    if (!s_r1 || !s_r2 || !s_c || !s_p1 || !s_p2 || !s_cl) {
        free(s_r1); free(s_r2); free(s_c); free(s_p1); free(s_p2); free(s_cl);
        free(E); free(S); free(F); free(idx);
        return ORC_ENOMEM;
    }
    memcpy(s_r1, o->r1, 8 * o->count); memcpy(s_r2, o->r2, 8 * o->count); memcpy(s_c, o->c, 4 * o->count);
    memcpy(s_p1, o->p1, 8 * o->count); memcpy(s_p2, o->p2, 8 * o->count); memcpy(s_cl, o->closed, o->count);
    int ovf = 0, bad_draw = 0;

    /* ---- Step 1: idx[i] = randInt(|W|+|E|) - |E| or null ---- */
#pragma omp parallel for schedule(static) reduction(|:bad_draw)
    for (int64_t i = 0; i < cnt; ++i) {
        uint64_t xlo, xhi, d1;
        if (forced_d1) {
            d1 = forced_d1[i];
            if (d1 >= m_prev + w) { bad_draw = 1; d1 = 0; }
        } else {
            block_words(seed, first + (uint64_t)i, b, 0, &xlo, &xhi);
            d1 = lemire(m_prev + w, xlo, seed, first + (uint64_t)i, b, 0x10000u);
        }
        idx[i] = d1 >= m_prev ? (int64_t)(d1 - m_prev) : -1;
        if (o->trace) o->t_j[i] = idx[i] >= 0 ? (uint32_t)idx[i] : UINT32_MAX;
    }
    /* extract + combine */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        if (idx[i] < 0) continue;
        int64_t j = idx[i];
        o->r1[2 * i] = E[2 * j]; o->r1[2 * i + 1] = E[2 * j + 1];
        o->p1[i] = m_prev + (uint64_t)j;
        o->c[i] = 0;
        o->r2[2 * i] = o->r2[2 * i + 1] = EMPTY_V; o->p2[i] = EMPTY_P; o->closed[i] = 0;
    }

    /* ---- Step 2 ---- */
#pragma omp parallel for schedule(static) reduction(|:ovf, bad_draw)
    for (int64_t i = 0; i < cnt; ++i) {
        uint32_t u = o->r1[2 * i], v = o->r1[2 * i + 1]; /* u = min (reading R1) */
        int64_t p = idx[i] >= 0 ? idx[i] : -1;        /* footnote PAPER.md:818-821 */
        int64_t au = q1(F, nF, u, p), av = q1(F, nF, v, p);
        uint64_t ld = au < 0 ? 0 : (p >= 0 ? F[au].rank : (uint64_t)F[au].rank + 1);
        uint64_t rd = av < 0 ? 0 : (p >= 0 ? F[av].rank : (uint64_t)F[av].rank + 1);
        uint64_t chi_m = o->c[i], chi_p = ld + rd;
        if (o->trace) {
            o->t_chim[i] = (uint32_t)chi_m; o->t_ld[i] = (uint32_t)ld; o->t_rd[i] = (uint32_t)rd;
            o->t_d2[i] = UINT64_MAX; o->t_k2[i] = UINT32_MAX;
        }
        if (chi_p == 0) continue;
        uint64_t xlo, xhi, d2;
        if (forced_d2) {
            d2 = forced_d2[i];
            if (d2 >= chi_m + chi_p) { bad_draw = 1; d2 = 0; }
        } else {
            block_words(seed, first + (uint64_t)i, b, 0, &xlo, &xhi);
            d2 = lemire(chi_m + chi_p, xhi, seed, first + (uint64_t)i, b, 0x20000u);
        }
        if (o->trace) o->t_d2[i] = d2;
        if (d2 >= chi_m) {
            uint64_t phi = d2 - chi_m;
            uint32_t src = phi < ld ? u : v;
            uint32_t a = (uint32_t)(phi < ld ? phi : phi - ld);
            int64_t k = q2(F, nF, src, a);
            if (k < 0) abort(); /* cannot happen: the naming is a bijection */
            uint32_t x = F[k].src, y = F[k].dst;
            o->r2[2 * i] = x < y ? x : y; o->r2[2 * i + 1] = x < y ? y : x;
            o->p2[i] = m_prev + (uint64_t)F[k].pos;
            o->closed[i] = 0;
            if (o->trace) o->t_k2[i] = (uint32_t)F[k].pos;
        }
        /* overflow guard (reading R13): chi^- + chi^+ in 64 bits; chi must fit 31 bits (bit 31 of the
           GPU's packed word is the closed flag).  m and positions are uint64 and not limited. */
        if (chi_m + chi_p > C_MAX) ovf = 1;
        o->c[i] = (uint32_t)(chi_m + chi_p);
    }

    /* ---- Step 3 ---- */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        if (o->r2[2 * i] == EMPTY_V || o->closed[i]) continue;
        uint32_t a1 = o->r1[2 * i], b1 = o->r1[2 * i + 1], a2 = o->r2[2 * i], b2 = o->r2[2 * i + 1];
        /* non-shared endpoints of f1 and f2 */
        uint32_t x = (a1 == a2 || a1 == b2) ? b1 : a1;
        uint32_t z = (a2 == a1 || a2 == b1) ? b2 : a2;
        uint32_t lo = x < z ? x : z, hi = x < z ? z : x;
        int64_t k = find_edge(S, (int64_t)w, lo, hi);
        if (k >= 0 && m_prev + (uint64_t)S[k].pos > o->p2[i]) o->closed[i] = 1;
    }

    if (o->trace) memcpy(o->t_closed, o->closed, o->count);
    code = bad_draw ? ORC_EINVAL : ovf ? ORC_EOVERFLOW : ORC_OK;
    if (code != ORC_OK) {  /* reject the whole batch: restore the snapshot */
        memcpy(o->r1, s_r1, 8 * o->count); memcpy(o->r2, s_r2, 8 * o->count); memcpy(o->c, s_c, 4 * o->count);
        memcpy(o->p1, s_p1, 8 * o->count); memcpy(o->p2, s_p2, 8 * o->count); memcpy(o->closed, s_cl, o->count);
    } else {
        o->m += w;
        o->b += 1;
    }
    free(s_r1); free(s_r2); free(s_c); free(s_p1); free(s_p2); free(s_cl);
    free(E); free(S); free(F); free(idx);
    return code;
}

int orc_push_batch(orc *o, const uint32_t *edges, uint64_t w) { return push_batch_impl(o, edges, w, NULL, NULL); }

/* Test wiring: the same batch update with the two draws of every estimator supplied (forced). */
int orc_push_batch_forced(orc *o, const uint32_t *edges, uint64_t w, const uint64_t *d1, const uint64_t *d2) {
    if (!d1 || !d2) return ORC_EINVAL;
    return push_batch_impl(o, edges, w, d1, d2);
}

/* Test wiring: overwrite estimator i's state / the counters (e.g. a chi near 2^31 or m past 2^32, to
   exercise the overflow guard without streaming billions of edges).  No validation: tests only. */
void orc_set_estimator(orc *o, uint64_t i, const uint32_t r1[2], uint64_t p1, const uint32_t r2[2], uint64_t p2,
                       uint32_t c, uint8_t closed) {
    o->r1[2 * i] = r1[0]; o->r1[2 * i + 1] = r1[1]; o->p1[i] = p1;
    o->r2[2 * i] = r2[0]; o->r2[2 * i + 1] = r2[1]; o->p2[i] = p2;
    o->c[i] = c; o->closed[i] = closed;
}

void orc_set_counters(orc *o, uint64_t m, uint32_t b) { o->m = m; o->b = b; }

/* Test wiring: record the per-step values of every later batch (see the orc fields); 0 on success. */
int orc_set_trace(orc *o, int on) {
    if (on && !o->t_j) {
        uint64_t n = o->count ? o->count : 1;
        o->t_j = (uint32_t *)calloc(n, 4); o->t_chim = (uint32_t *)calloc(n, 4); o->t_ld = (uint32_t *)calloc(n, 4);
        o->t_rd = (uint32_t *)calloc(n, 4); o->t_k2 = (uint32_t *)calloc(n, 4); o->t_d2 = (uint64_t *)calloc(n, 8);
        o->t_closed = (uint8_t *)calloc(n, 1);
        if (!o->t_j || !o->t_chim || !o->t_ld || !o->t_rd || !o->t_k2 || !o->t_d2 || !o->t_closed) return ORC_ENOMEM;
    }
    o->trace = on;
    return ORC_OK;
}

void orc_get_trace(const orc *o, uint32_t *j, uint32_t *chim, uint32_t *ld, uint32_t *rd, uint64_t *d2, uint32_t *k2,
                   uint8_t *closed) {
    memcpy(j, o->t_j, 4 * o->count); memcpy(chim, o->t_chim, 4 * o->count); memcpy(ld, o->t_ld, 4 * o->count);
    memcpy(rd, o->t_rd, 4 * o->count); memcpy(d2, o->t_d2, 8 * o->count); memcpy(k2, o->t_k2, 4 * o->count);
    memcpy(closed, o->t_closed, o->count);
}

void orc_get_state(const orc *o, uint32_t *r1, uint64_t *p1, uint32_t *r2, uint64_t *p2, uint32_t *c,
                   uint8_t *closed) {
    memcpy(r1, o->r1, 8 * o->count); memcpy(r2, o->r2, 8 * o->count);
    memcpy(p1, o->p1, 8 * o->count); memcpy(p2, o->p2, 8 * o->count);
    memcpy(c, o->c, 4 * o->count); memcpy(closed, o->closed, o->count);
}

uint64_t orc_closed_sum(const orc *o) {
    uint64_t s = 0;
    for (uint64_t i = 0; i < o->count; ++i) if (o->closed[i]) s += o->c[i];
    return s;
}

void orc_counters(const orc *o, uint64_t *m, uint32_t *b) { *m = o->m; *b = o->b; }

int orc_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
