// ed.c -- event-driven oracle, fast form: each estimator's skip-sampled neighborhood sampling walked event by
// event over the whole stream prefix (reading R17).
//
// TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pinned to oracle/ed.py (the plain per-edge form of the
// same rule, itself pinned by exact enumeration) by tests/test_oracle_ed_c.py.
//
// For one estimator the sequential rule of oracle/ed.py reduces to (times are 1-based stream positions):
//   J = 1; repeat while J <= m:                         -- clause 1 fires at t = J
//       t1 = J; J = next_after(t1);  f1 = e_t1 = (u, v); B = deg_t1(u) + deg_t1(v); K = 1; f2 = none
//       the epoch of this f1 ends at h = min(J - 1, m); chi(t) = deg_t(u) + deg_t(v) - B counts Gamma(f1)
//       (clause 2; no edge but f1 touches both u and v in a simple graph)
//       while the K-th edge of Gamma(f1) exists at a time P <= h:   -- clause 3 fires when chi reaches K
//           f2 = e_P, t2 = P, K = next_after(K)
//       closed = (the closing edge of (f1, f2) arrives at a time in (t2, h])       -- clause 4
//   chi = deg_m(u) + deg_m(v) - B for the last f1.
// The random words are consumed in event-time order, as in the per-edge form: next_after(t1) when f1 is taken
// (before that epoch's f2 events), next_after(K) when f2 is taken.
//
// Data: the vertices' arrival-time lists (vertex -> sorted times, a counting sort in stream order) give
// deg_t(x) by binary search and the K-th neighbour by a binary search over time; a hash map gives the time of
// every edge (the closing-edge lookup).
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HMAX 0x7FFFFFFFu
#define INF 0xFFFFFFFFu
#define EMPTYV 0xFFFFFFFFu

typedef unsigned __int128 u128;

static void philox(uint32_t c[4], const uint32_t key[2]) {
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n1 = (uint32_t)p1, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1,
                       n3 = (uint32_t)p0;
        c[0] = n0;
        c[1] = n1;
        c[2] = n2;
        c[3] = n3;
    }
}

typedef struct {
    uint64_t id, seed, ev;
} Words;

static uint64_t next_word(Words *w) {
    const uint64_t n = w->ev++;
    uint32_t c[4] = {(uint32_t)w->id, (uint32_t)(w->id >> 32), (uint32_t)(n >> 1), 0xED5A0000u};
    const uint32_t key[2] = {(uint32_t)w->seed, (uint32_t)(w->seed >> 32)};
    philox(c, key);
    return (n & 1) ? ((uint64_t)c[2] | ((uint64_t)c[3] << 32)) : ((uint64_t)c[0] | ((uint64_t)c[1] << 32));
}

// U[0, n), n >= 1 (Lemire; a rejected word is replaced by the next word of the stream)
static uint64_t uniform(uint64_t n, Words *w) {
    u128 p = (u128)next_word(w) * n;
    if ((uint64_t)p < n) {
        const uint64_t thr = (0ull - n) % n;
        while ((uint64_t)p < thr) p = (u128)next_word(w) * n;
    }
    return (uint64_t)(p >> 64);
}

// reading R17: P(T > s) = t / s
static uint32_t next_after(uint64_t t, Words *w) {
    if (t == 0) return 1;
    const uint64_t x = next_word(w);
    if (x == 0) return INF;
    const int k = __builtin_ctzll(x);
    if (k >= 31) return INF;
    const uint64_t L = t << k;
    if (L > HMAX) return INF;
    for (;;) {
        const uint64_t s = L + 1 + uniform(L, w);
        if (uniform(s - 1, w) >= L) continue;
        if (uniform(s, w) >= L + 1) continue;
        return s <= HMAX ? (uint32_t)s : INF;
    }
}

uint32_t orc_ed_next_after(uint64_t t, uint64_t id, uint64_t seed, uint64_t ev_in, uint64_t *ev_out) {
    Words w = {id, seed, ev_in};
    const uint32_t s = next_after(t, &w);
    *ev_out = w.ev;
    return s;
}

// ---- stream index -------------------------------------------------------------------------------------------
static uint64_t mix64(uint64_t x) {
    x ^= x >> 31;
    x *= 0x7fb5d329728ea185ull;
    x ^= x >> 27;
    x *= 0x81dadef4bc2dd44dull;
    x ^= x >> 33;
    return x;
}

typedef struct {
    uint64_t cap;
    uint64_t *key;
    uint32_t *val;
} Map;

static int map_init(Map *M, uint64_t n) {
    M->cap = 16;
    while (M->cap < 2 * n + 16) M->cap <<= 1;
    M->key = (uint64_t *)malloc(M->cap * sizeof(uint64_t));
    M->val = (uint32_t *)malloc(M->cap * sizeof(uint32_t));
    if (!M->key || !M->val) return -1;
    memset(M->key, 0xFF, M->cap * sizeof(uint64_t));
    return 0;
}
static void map_free(Map *M) {
    free(M->key);
    free(M->val);
}
// returns the slot of key (inserted with val if absent; *fresh = 1 then)
static uint64_t map_put(Map *M, uint64_t key, uint32_t val, int *fresh) {
    uint64_t i = mix64(key) & (M->cap - 1);
    for (;;) {
        if (M->key[i] == key) {
            *fresh = 0;
            return i;
        }
        if (M->key[i] == ~0ull) {
            M->key[i] = key;
            M->val[i] = val;
            *fresh = 1;
            return i;
        }
        i = (i + 1) & (M->cap - 1);
    }
}
static int map_get(const Map *M, uint64_t key, uint32_t *val) {
    uint64_t i = mix64(key) & (M->cap - 1);
    for (;;) {
        if (M->key[i] == key) {
            *val = M->val[i];
            return 1;
        }
        if (M->key[i] == ~0ull) return 0;
        i = (i + 1) & (M->cap - 1);
    }
}

typedef struct {
    uint64_t m;
    const uint32_t *lo, *hi;  // normalised edges, index t-1
    Map vid;                  // vertex -> dense index
    uint64_t *off;            // [nv + 1] list offsets
    uint32_t *times;          // [2m] arrival times per vertex, ascending
    Map pair;                 // (lo, hi) -> time
} Stream;

// number of arrivals of x at times <= t
static uint64_t deg_at(const Stream *S, uint32_t xi, uint64_t t) {
    uint64_t a = S->off[xi], b = S->off[xi + 1];
    while (a < b) {
        const uint64_t mid = (a + b) / 2;
        if (S->times[mid] <= t) a = mid + 1;
        else b = mid;
    }
    return a - S->off[xi];
}

// time of the n-th (n >= 1) arrival at u or v strictly after t1, or 0 if there are fewer than n
static uint64_t kth_after(const Stream *S, uint32_t ui, uint32_t vi, uint64_t t1, uint64_t n) {
    const uint64_t cu = deg_at(S, ui, t1), cv = deg_at(S, vi, t1);
    const uint64_t du = S->off[ui + 1] - S->off[ui], dv = S->off[vi + 1] - S->off[vi];
    if ((du - cu) + (dv - cv) < n) return 0;
    uint64_t a = t1 + 1, b = S->m;  // smallest P with count(t1, P] >= n
    while (a < b) {
        const uint64_t mid = (a + b) / 2;
        if ((deg_at(S, ui, mid) - cu) + (deg_at(S, vi, mid) - cv) >= n) b = mid;
        else a = mid + 1;
    }
    return a;
}

// Runs estimators [first, first + count) over the m-edge stream (edges[2t], edges[2t+1]; validated by the
// caller: no self loops, no duplicate edges).  Outputs per estimator: t1, t2 (1-based times, 0 = empty), chi,
// closed, J, K (INF = none), ev (words used).  Returns 0, or -1 on allocation failure.
int orc_ed_run(const uint32_t *edges, uint64_t m, uint64_t seed, uint64_t first, uint64_t count, uint32_t *t1o,
               uint32_t *t2o, uint32_t *chio, uint8_t *closedo, uint32_t *Jo, uint32_t *Ko, uint64_t *evo) {
    Stream S;
    memset(&S, 0, sizeof(S));
    S.m = m;
    uint32_t *lo = (uint32_t *)malloc((m + 1) * sizeof(uint32_t)), *hi = (uint32_t *)malloc((m + 1) * sizeof(uint32_t));
    uint32_t *vix = (uint32_t *)malloc((2 * m + 1) * sizeof(uint32_t));
    if (!lo || !hi || !vix || map_init(&S.vid, 2 * m) || map_init(&S.pair, m)) return -1;
    uint32_t nv = 0;
    for (uint64_t t = 0; t < m; ++t) {
        const uint32_t a = edges[2 * t], b = edges[2 * t + 1];
        lo[t] = a < b ? a : b;
        hi[t] = a < b ? b : a;
        int fresh;
        const uint64_t s0 = map_put(&S.vid, lo[t], nv, &fresh);
        nv += fresh;
        vix[2 * t] = S.vid.val[s0];
        const uint64_t s1 = map_put(&S.vid, hi[t], nv, &fresh);
        nv += fresh;
        vix[2 * t + 1] = S.vid.val[s1];
        map_put(&S.pair, ((uint64_t)lo[t] << 32) | hi[t], (uint32_t)(t + 1), &fresh);
    }
    S.lo = lo;
    S.hi = hi;
    S.off = (uint64_t *)calloc(nv + 1, sizeof(uint64_t));
    S.times = (uint32_t *)malloc((2 * m + 1) * sizeof(uint32_t));
    uint64_t *fill = (uint64_t *)malloc((nv + 1) * sizeof(uint64_t));
    if (!S.off || !S.times || !fill) return -1;
    for (uint64_t i = 0; i < 2 * m; ++i) S.off[vix[i] + 1]++;
    for (uint32_t x = 0; x < nv; ++x) S.off[x + 1] += S.off[x];
    memcpy(fill, S.off, (nv + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < 2 * m; ++i) S.times[fill[vix[i]]++] = (uint32_t)(i / 2 + 1);  // stream order

#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < (int64_t)count; ++j) {
        Words w = {first + (uint64_t)j, seed, 0};
        uint64_t J = 1, t1 = 0, t2 = 0, K = INF, B = 0;
        uint32_t ui = 0, vi = 0, closed = 0;
        while (J <= m) {
            t1 = J;
            J = next_after(t1, &w);
            ui = vix[2 * (t1 - 1)];
            vi = vix[2 * (t1 - 1) + 1];
            B = deg_at(&S, ui, t1) + deg_at(&S, vi, t1);
            K = 1;
            t2 = 0;
            closed = 0;
            const uint64_t h = J <= m ? J - 1 : m;
            for (;;) {
                if (K == INF) break;
                const uint64_t P = kth_after(&S, ui, vi, t1, K);
                if (P == 0 || P > h) break;
                t2 = P;
                K = next_after(K, &w);
            }
            if (t2) {
                const uint32_t u = lo[t1 - 1], v = hi[t1 - 1], a = lo[t2 - 1], b = hi[t2 - 1];
                const uint32_t shared = (a == u || b == u) ? u : v;
                const uint32_t z = shared == u ? v : u, y = a == shared ? b : a;
                const uint64_t key = z < y ? (((uint64_t)z << 32) | y) : (((uint64_t)y << 32) | z);
                uint32_t tc;
                closed = map_get(&S.pair, key, &tc) && tc > t2 && tc <= h;
            }
        }
        t1o[j] = (uint32_t)t1;
        t2o[j] = (uint32_t)t2;
        chio[j] = t1 ? (uint32_t)(deg_at(&S, ui, m) + deg_at(&S, vi, m) - B) : 0u;
        closedo[j] = (uint8_t)closed;
        Jo[j] = (uint32_t)(J > HMAX ? INF : J);
        Ko[j] = t1 ? (uint32_t)K : INF;
        evo[j] = w.ev;
    }
    free(lo);
    free(hi);
    free(vix);
    free(fill);
    free(S.off);
    free(S.times);
    map_free(&S.vid);
    map_free(&S.pair);
    return 0;
}

int orc_ed_threads(void) { return omp_get_max_threads(); }
