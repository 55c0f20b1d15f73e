/* TEST INFRASTRUCTURE ONLY — the CPU checker, never linked into the product.
 *
 * Plain-C restatement of the reference NN-Descent path for squared L2
 * (reference: /root/reference/proj/include/knng/, cited below as file:line).
 * Compiled with -ffp-contract=off: every fused multiply-add the reference's
 * compiled kernels perform is written out explicitly with fmaf(), every
 * unfused one as a separate multiply and add, so the arithmetic is pinned and
 * does not depend on this compiler's contraction decisions.
 *
 * Parity status: PINNED.  tests/test_oracle_pins.py checks this file against
 * the reference itself (oracle/_ref/libknng_ref.so built from the unmodified
 * headers) bit for bit, and against the golden fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#define _POSIX_C_SOURCE 200809L
#include "knng_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* oracle_last_error(void) { return g_err; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* Rng = std::mt19937_64 (dataset.hpp:23), the engine specified by the C++  */
/* standard [rand.eng.mers] with the mt19937_64 parameters.                  */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t mt[MT_N];
    int idx;
} Mt64;

static void mt_seed(Mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static uint64_t mt_next(Mt64* r) {
    if (r->idx >= MT_N) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* std::uniform_int_distribution<uint32_t>(a, b) over a 64-bit engine as
 * implemented by GCC's libstdc++ (the reference's toolchain):
 * Lemire's nearly-divisionless downscaling in 128-bit arithmetic. */
static uint32_t uniform_u32(Mt64* r, uint32_t a, uint32_t b) {
    const uint64_t range = (uint64_t)b - (uint64_t)a + 1ULL;
    unsigned __int128 product = (unsigned __int128)mt_next(r) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        const uint64_t threshold = (0ULL - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)mt_next(r) * range;
            low = (uint64_t)product;
        }
    }
    return (uint32_t)(product >> 64) + a;
}

/* std::uniform_real_distribution<double>(0, 1) = generate_canonical<double,53>
 * with one 64-bit draw (libstdc++ random.tcc), clamped below 1. */
static double unit_double(Mt64* r) {
    double x = (double)mt_next(r) / 18446744073709551616.0;
    if (x >= 1.0) x = nextafter(1.0, 0.0);
    return x;
}

/* ------------------------------------------------------------------------ */
/* Distance kernels (distance.hpp)                                          */
/* ------------------------------------------------------------------------ */

/* reduce_lanes (distance.hpp:29-31) */
static float reduce_lanes(const float* acc) {
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

/* l2_sq_core (distance.hpp:35-51): 8 strided lanes, UNFUSED square-accumulate. */
static float l2_scalar(const float* a, const float* b, uint32_t d) {
    float acc[8] = {0};
    const uint32_t chunks = d / 8;
    for (uint32_t c = 0; c < chunks; ++c)
        for (uint32_t l = 0; l < 8; ++l) {
            const float diff = a[c * 8 + l] - b[c * 8 + l];
            const float sq = diff * diff;
            acc[l] = acc[l] + sq;
        }
    float tail = 0.0f;
    for (uint32_t j = chunks * 8; j < d; ++j) {
        const float diff = a[j] - b[j];
        const float sq = diff * diff;
        tail = tail + sq;
    }
    return reduce_lanes(acc) + tail;
}

/* block_core<5,5> (distance.hpp:55-88) and tri_core5 (:96-121): same lanes,
 * but the compiled tiles FUSE the square-accumulate (pinned by
 * tests against the reference harness). */
static float l2_tile(const float* a, const float* b, uint32_t d) {
    float acc[8] = {0};
    const uint32_t chunks = d / 8;
    for (uint32_t c = 0; c < chunks; ++c)
        for (uint32_t l = 0; l < 8; ++l) {
            const float diff = a[c * 8 + l] - b[c * 8 + l];
            acc[l] = fmaf(diff, diff, acc[l]);
        }
    float tail = 0.0f;
    for (uint32_t j = chunks * 8; j < d; ++j) {
        const float diff = a[j] - b[j];
        tail = fmaf(diff, diff, tail);
    }
    return reduce_lanes(acc) + tail;
}

static const uint8_t kTri[10][2] = {{0, 1}, {0, 2}, {0, 3}, {0, 4}, {1, 2},
                                    {1, 3}, {1, 4}, {2, 3}, {2, 4}, {3, 4}};

/* ------------------------------------------------------------------------ */
/* Graph state (graph.hpp)                                                  */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t n, k;
    uint32_t* ids;
    float* dists;
    uint8_t* flags;
    uint32_t* rev;   /* reverse_degree_ = k + in-degree */
    float* row_max;  /* cached root distance */
    uint64_t changes;
} Graph;

static int graph_alloc(Graph* g, uint32_t n, uint32_t k) {
    g->n = n;
    g->k = k;
    g->ids = malloc(sizeof(uint32_t) * (size_t)n * k);
    g->dists = malloc(sizeof(float) * (size_t)n * k);
    g->flags = malloc((size_t)n * k);
    g->rev = malloc(sizeof(uint32_t) * n);
    g->row_max = malloc(sizeof(float) * n);
    g->changes = 0;
    return g->ids && g->dists && g->flags && g->rev && g->row_max;
}

static void graph_free(Graph* g) {
    free(g->ids);
    free(g->dists);
    free(g->flags);
    free(g->rev);
    free(g->row_max);
    memset(g, 0, sizeof *g);
}

/* sift_down (graph.hpp:197-214) on row base p */
static void sift_down(Graph* g, size_t p, uint32_t i) {
    const uint32_t k = g->k;
    const uint32_t mid = g->ids[p + i];
    const float mdist = g->dists[p + i];
    const uint8_t mflag = g->flags[p + i];
    for (;;) {
        uint32_t largest = i;
        const uint32_t left = 2 * i + 1, right = left + 1;
        float largest_dist = mdist;
        if (left < k && g->dists[p + left] > largest_dist) {
            largest = left;
            largest_dist = g->dists[p + left];
        }
        if (right < k && g->dists[p + right] > largest_dist) largest = right;
        if (largest == i) break;
        g->ids[p + i] = g->ids[p + largest];
        g->dists[p + i] = g->dists[p + largest];
        g->flags[p + i] = g->flags[p + largest];
        i = largest;
    }
    g->ids[p + i] = mid;
    g->dists[p + i] = mdist;
    g->flags[p + i] = mflag;
}

/* heapify_row (graph.hpp:191-195) */
static void heapify_row(Graph* g, uint32_t u) {
    const size_t p = (size_t)u * g->k;
    for (uint32_t i = g->k / 2; i-- > 0;) sift_down(g, p, i);
    g->row_max[u] = g->dists[p];
}

/* try_insert (graph.hpp:116-129) */
static int try_insert(Graph* g, uint32_t u, uint32_t v, float dist) {
    if (dist >= g->row_max[u] || u == v) return 0;
    const size_t p = (size_t)u * g->k;
    for (uint32_t i = 0; i < g->k; ++i)
        if (g->ids[p + i] == v) return 0;
    --g->rev[g->ids[p]];
    ++g->rev[v];
    g->ids[p] = v;
    g->dists[p] = dist;
    g->flags[p] = 1;
    sift_down(g, p, 0);
    g->row_max[u] = g->dists[p];
    ++g->changes;
    return 1;
}

/* flag_consumed (graph.hpp:133-143) */
static void flag_consumed(Graph* g, uint32_t u, const uint32_t* ids, uint32_t count) {
    const size_t p = (size_t)u * g->k;
    for (uint32_t c = 0; c < count; ++c)
        for (uint32_t i = 0; i < g->k; ++i)
            if (g->ids[p + i] == ids[c]) {
                g->flags[p + i] = 0;
                break;
            }
}

/* Padded dataset rows, stride = ceil8(d) (dataset.hpp:61-77). */
typedef struct {
    uint32_t n, d, stride;
    float* v;
} Data;

static int data_make(Data* ds, const float* src, uint32_t n, uint32_t d) {
    ds->n = n;
    ds->d = d;
    ds->stride = (d + 7) / 8 * 8;
    ds->v = calloc((size_t)n * ds->stride, sizeof(float));
    if (!ds->v) return 0;
    for (uint32_t i = 0; i < n; ++i)
        memcpy(ds->v + (size_t)i * ds->stride, src + (size_t)i * d, sizeof(float) * d);
    return 1;
}

static const float* row(const Data* ds, uint32_t i) { return ds->v + (size_t)i * ds->stride; }

/* KnnGraph::init_random (graph.hpp:34-67) */
static int init_random(Graph* g, const Data* ds, uint32_t k, uint64_t seed, uint64_t* evals) {
    const uint32_t n = ds->n;
    if (k < 2) return fail(1, "init_random: k must be at least 2");
    if (k >= n) return fail(1, "init_random: k must be smaller than n");
    if (!graph_alloc(g, n, k)) return fail(2, "init_random: out of memory");
    for (uint32_t u = 0; u < n; ++u) g->rev[u] = k;
    Mt64 rng;
    mt_seed(&rng, seed);
    uint32_t* chosen = malloc(sizeof(uint32_t) * k);
    for (uint32_t u = 0; u < n; ++u) {
        for (uint32_t i = 0; i < k; ++i) {
            uint32_t v;
            int fresh;
            do {
                v = uniform_u32(&rng, 0, n - 1);
                fresh = v != u;
                for (uint32_t j = 0; fresh && j < i; ++j) fresh = chosen[j] != v;
            } while (!fresh);
            chosen[i] = v;
            const size_t p = (size_t)u * k + i;
            g->ids[p] = v;
            g->dists[p] = l2_scalar(row(ds, u), row(ds, v), ds->stride);
            g->flags[p] = 1;
            ++g->rev[v];
            ++*evals;
        }
        heapify_row(g, u);
    }
    free(chosen);
    return 0;
}

/* KnnGraph::from_rows (graph.hpp:70-93) */
static int from_rows(Graph* g, uint32_t n, uint32_t k, const uint32_t* ids, const float* dists,
                     const uint8_t* flags) {
    if (k < 2 || k >= n) return fail(1, "from_rows: need 2 <= k < n");
    if (!graph_alloc(g, n, k)) return fail(2, "from_rows: out of memory");
    for (uint32_t u = 0; u < n; ++u) g->rev[u] = k;
    for (uint32_t u = 0; u < n; ++u) {
        for (uint32_t i = 0; i < k; ++i) {
            const size_t p = (size_t)u * k + i;
            if (ids[p] == u) return fail(1, "from_rows: self loop");
            if (ids[p] >= n) return fail(1, "from_rows: id out of range");
            for (uint32_t j = 0; j < i; ++j)
                if (ids[(size_t)u * k + j] == ids[p]) return fail(1, "from_rows: duplicate id");
            g->ids[p] = ids[p];
            g->dists[p] = dists[p];
            g->flags[p] = flags[p] ? 1 : 0;
            ++g->rev[ids[p]];
        }
        heapify_row(g, u);
    }
    return 0;
}

static void export_graph(const Graph* g, uint32_t* ids, float* dists, uint8_t* flags,
                         uint32_t* rev) {
    const size_t nk = (size_t)g->n * g->k;
    if (ids) memcpy(ids, g->ids, sizeof(uint32_t) * nk);
    if (dists) memcpy(dists, g->dists, sizeof(float) * nk);
    if (flags) memcpy(flags, g->flags, nk);
    if (rev) memcpy(rev, g->rev, sizeof(uint32_t) * g->n);
}

/* ------------------------------------------------------------------------ */
/* CandidateSet (selection.hpp:22-89): per node 2*cap ids, new then old.     */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t n, cap;
    uint32_t* ids;
    uint32_t* nc;
    uint32_t* oc;
} Cands;

static int cands_alloc(Cands* c, uint32_t n, uint32_t cap) {
    if (cap == 0) return fail(1, "CandidateSet: cap must be positive");
    c->n = n;
    c->cap = cap;
    c->ids = malloc(sizeof(uint32_t) * (size_t)n * 2 * cap);
    c->nc = calloc(n, sizeof(uint32_t));
    c->oc = calloc(n, sizeof(uint32_t));
    return (c->ids && c->nc && c->oc) ? 0 : fail(2, "CandidateSet: out of memory");
}

static void cands_free(Cands* c) {
    free(c->ids);
    free(c->nc);
    free(c->oc);
    memset(c, 0, sizeof *c);
}

static uint32_t* new_data(const Cands* c, uint32_t u) { return c->ids + (size_t)u * 2 * c->cap; }
static uint32_t* old_data(const Cands* c, uint32_t u) {
    return c->ids + (size_t)u * 2 * c->cap + c->cap;
}

static void export_cands(const Cands* c, uint32_t* cand_ids, uint32_t* nc, uint32_t* oc) {
    for (uint32_t u = 0; u < c->n; ++u) {
        uint32_t* block = cand_ids + (size_t)u * 2 * c->cap;
        for (uint32_t i = 0; i < 2 * c->cap; ++i) block[i] = 0xffffffffu;
        memcpy(block, new_data(c, u), sizeof(uint32_t) * c->nc[u]);
        memcpy(block + c->cap, old_data(c, u), sizeof(uint32_t) * c->oc[u]);
        nc[u] = c->nc[u];
        oc[u] = c->oc[u];
    }
}

/* select_turbo offer (selection.hpp:296-309) */
static void turbo_offer(const Graph* g, Cands* c, Mt64* rng, uint32_t target, uint32_t id,
                        int is_new) {
    const uint32_t degree = g->rev[target];
    if (degree > c->cap && unit_double(rng) * (double)degree >= (double)c->cap) return;
    const uint32_t* nd = new_data(c, target);
    const uint32_t* od = old_data(c, target);
    for (uint32_t i = 0; i < c->nc[target]; ++i)
        if (nd[i] == id) return;
    for (uint32_t i = 0; i < c->oc[target]; ++i)
        if (od[i] == id) return;
    uint32_t* ids = is_new ? new_data(c, target) : old_data(c, target);
    uint32_t* size = is_new ? &c->nc[target] : &c->oc[target];
    if (*size < c->cap)
        ids[(*size)++] = id;
    else
        ids[uniform_u32(rng, 0, c->cap - 1)] = id;
}

/* select_turbo (selection.hpp:282-320) */
static void select_turbo(const Graph* g, uint64_t seed, Cands* c) {
    memset(c->nc, 0, sizeof(uint32_t) * c->n);
    memset(c->oc, 0, sizeof(uint32_t) * c->n);
    Mt64 rng;
    mt_seed(&rng, seed);
    for (uint32_t u = 0; u < g->n; ++u)
        for (uint32_t i = 0; i < g->k; ++i) {
            const size_t p = (size_t)u * g->k + i;
            const uint32_t v = g->ids[p];
            const int f = g->flags[p];
            turbo_offer(g, c, &rng, u, v, f);
            turbo_offer(g, c, &rng, v, u, f);
        }
}

/* ------------------------------------------------------------------------ */
/* compute_step (descent.hpp:82-153) and compute_step_flat (:159-182)        */
/* ------------------------------------------------------------------------ */

static uint64_t compute_step(Graph* g, const Cands* c, const Data* ds, uint64_t* evals) {
    uint64_t changes = 0;
    const uint32_t stride = ds->stride;
    const uint32_t cap = c->cap;
    float* new_max = malloc(sizeof(float) * cap);
    float* old_max = malloc(sizeof(float) * cap);
    for (uint32_t u = 0; u < g->n; ++u) {
        const uint32_t nn = c->nc[u];
        if (nn == 0) continue;
        const uint32_t no = c->oc[u];
        const uint32_t* nid = new_data(c, u);
        const uint32_t* oid = old_data(c, u);
        for (uint32_t i = 0; i < nn; ++i) new_max[i] = g->row_max[nid[i]];

#define CONSUME(I, J, D)                                                                  \
    do {                                                                                  \
        const float dd = (D);                                                             \
        if (dd < new_max[I] && try_insert(g, nid[I], nid[J], dd)) {                      \
            new_max[I] = g->row_max[nid[I]];                                              \
            ++changes;                                                                    \
        }                                                                                 \
        if (dd < new_max[J] && try_insert(g, nid[J], nid[I], dd)) {                      \
            new_max[J] = g->row_max[nid[J]];                                              \
            ++changes;                                                                    \
        }                                                                                 \
    } while (0)

        /* mutual_block_distances (distance.hpp:157-190) */
        if (nn >= 2) {
            const uint32_t full = nn - nn % 5;
            for (uint32_t gi = 0; gi < full; gi += 5) {
                float tri[10];
                for (int p = 0; p < 10; ++p)
                    tri[p] = l2_tile(row(ds, nid[gi + kTri[p][0]]), row(ds, nid[gi + kTri[p][1]]),
                                     stride);
                *evals += 10;
                for (int p = 0; p < 10; ++p) CONSUME(gi + kTri[p][0], gi + kTri[p][1], tri[p]);
                for (uint32_t gj = gi + 5; gj < full; gj += 5) {
                    float tile[25];
                    for (uint32_t x = 0; x < 5; ++x)
                        for (uint32_t y = 0; y < 5; ++y)
                            tile[x * 5 + y] =
                                l2_tile(row(ds, nid[gi + x]), row(ds, nid[gj + y]), stride);
                    *evals += 25;
                    for (uint32_t x = 0; x < 5; ++x)
                        for (uint32_t y = 0; y < 5; ++y) CONSUME(gi + x, gj + y, tile[x * 5 + y]);
                }
            }
            for (uint32_t r = full; r < nn; ++r)
                for (uint32_t q = 0; q < r; ++q) {
                    *evals += 1;
                    CONSUME(q, r, l2_scalar(row(ds, nid[q]), row(ds, nid[r]), stride));
                }
        }
#undef CONSUME
        if (no == 0) continue;
        for (uint32_t j = 0; j < no; ++j) old_max[j] = g->row_max[oid[j]];
        /* 5x5 tiles over new x old via block_l2_sq (distance.hpp:134-151) */
        for (uint32_t i0 = 0; i0 < nn; i0 += 5) {
            const uint32_t na = nn - i0 < 5 ? nn - i0 : 5;
            for (uint32_t j0 = 0; j0 < no; j0 += 5) {
                const uint32_t nb = no - j0 < 5 ? no - j0 : 5;
                const int full_tile = na == 5 && nb == 5;
                float tile[25];
                for (uint32_t a = 0; a < na; ++a)
                    for (uint32_t b = 0; b < nb; ++b) {
                        const float* ra = row(ds, nid[i0 + a]);
                        const float* rb = row(ds, oid[j0 + b]);
                        tile[a * nb + b] = full_tile ? l2_tile(ra, rb, stride)
                                                     : l2_scalar(ra, rb, stride);
                    }
                *evals += (uint64_t)na * nb;
                for (uint32_t a = 0; a < na; ++a)
                    for (uint32_t b = 0; b < nb; ++b) {
                        const uint32_t x = nid[i0 + a], y = oid[j0 + b];
                        const float dist = tile[a * nb + b];
                        if (dist < new_max[i0 + a] && try_insert(g, x, y, dist)) {
                            new_max[i0 + a] = g->row_max[x];
                            ++changes;
                        }
                        if (dist < old_max[j0 + b] && try_insert(g, y, x, dist)) {
                            old_max[j0 + b] = g->row_max[y];
                            ++changes;
                        }
                    }
            }
        }
    }
    free(new_max);
    free(old_max);
    return changes;
}

static uint64_t compute_step_flat(Graph* g, const Cands* c, const Data* ds, uint64_t* evals) {
    uint64_t changes = 0;
    for (uint32_t u = 0; u < g->n; ++u) {
        const uint32_t nn = c->nc[u];
        if (nn == 0) continue;
        const uint32_t no = c->oc[u];
        const uint32_t* nid = new_data(c, u);
        const uint32_t* oid = old_data(c, u);
        for (uint32_t i = 0; i < nn; ++i) {
            for (uint32_t j = i + 1; j < nn; ++j) {
                const float dist = l2_scalar(row(ds, nid[i]), row(ds, nid[j]), ds->stride);
                ++*evals;
                changes += (uint64_t)try_insert(g, nid[i], nid[j], dist);
                changes += (uint64_t)try_insert(g, nid[j], nid[i], dist);
            }
            for (uint32_t j = 0; j < no; ++j) {
                const float dist = l2_scalar(row(ds, nid[i]), row(ds, oid[j]), ds->stride);
                ++*evals;
                changes += (uint64_t)try_insert(g, nid[i], oid[j], dist);
                changes += (uint64_t)try_insert(g, oid[j], nid[i], dist);
            }
        }
    }
    return changes;
}

/* ------------------------------------------------------------------------ */
/* greedy_cluster (reorder.hpp:22-50), apply_permutation (dataset.hpp:      */
/* 237-245), KnnGraph::remap (graph.hpp:150-166)                             */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t id;
    float dist;
} Adj;

static int adj_cmp(const void* pa, const void* pb) {
    const Adj* a = pa;
    const Adj* b = pb;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

static void greedy_cluster(const Graph* g, uint32_t* sigma, uint32_t* sigma_inv) {
    const uint32_t n = g->n, k = g->k;
    for (uint32_t i = 0; i < n; ++i) sigma[i] = sigma_inv[i] = i;
    Adj* adj = malloc(sizeof(Adj) * k);
    for (uint32_t i = 0; i < n; ++i) {
        const size_t p = (size_t)sigma_inv[i] * k;
        for (uint32_t j = 0; j < k; ++j) {
            adj[j].id = g->ids[p + j];
            adj[j].dist = g->dists[p + j];
        }
        qsort(adj, k, sizeof(Adj), adj_cmp);
        for (uint32_t j = 0; j < k; ++j) {
            const uint32_t node = adj[j].id;
            const uint32_t spot = sigma[node];
            if (spot < i + 1) continue;
            if (spot == i + 1) break;
            const uint32_t occupant = sigma_inv[i + 1];
            uint32_t t = sigma[node];
            sigma[node] = sigma[occupant];
            sigma[occupant] = t;
            t = sigma_inv[spot];
            sigma_inv[spot] = sigma_inv[i + 1];
            sigma_inv[i + 1] = t;
            break;
        }
    }
    free(adj);
}

static int apply_permutation(const Data* in, const uint32_t* sigma, Data* out) {
    out->n = in->n;
    out->d = in->d;
    out->stride = in->stride;
    out->v = malloc(sizeof(float) * (size_t)in->n * in->stride);
    if (!out->v) return 0;
    for (uint32_t i = 0; i < in->n; ++i)
        memcpy(out->v + (size_t)sigma[i] * in->stride, in->v + (size_t)i * in->stride,
               sizeof(float) * in->stride);
    return 1;
}

static int remap(Graph* g, const uint32_t* sigma) {
    Graph r;
    if (!graph_alloc(&r, g->n, g->k)) return 0;
    const uint32_t k = g->k;
    for (uint32_t u = 0; u < g->n; ++u) {
        const size_t dst = (size_t)sigma[u] * k, src = (size_t)u * k;
        for (uint32_t i = 0; i < k; ++i) {
            r.ids[dst + i] = sigma[g->ids[src + i]];
            r.dists[dst + i] = g->dists[src + i];
            r.flags[dst + i] = g->flags[src + i];
        }
        r.rev[sigma[u]] = g->rev[u];
        r.row_max[sigma[u]] = g->row_max[u];
    }
    r.changes = g->changes;
    graph_free(g);
    *g = r;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Entry points                                                             */
/* ------------------------------------------------------------------------ */

/* run (descent.hpp:193-255) with strategy = turbo, blocked compute. */
int oracle_run(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap, double delta,
               uint32_t max_iterations, int reorder, uint32_t reorder_after, uint64_t seed,
               uint32_t* out_ids, float* out_dists, uint8_t* out_flags, uint64_t* iter_evals,
               uint64_t* iter_changes, double* iter_wall, uint32_t* n_rows, double* total_wall,
               uint32_t* sigma_out) {
    /* RunParams::validate (descent.hpp:29-35) and the n > k check (:197) */
    if (k < 2) return fail(1, "RunParams: k must be at least 2");
    if (cap < k) return fail(1, "RunParams: max_candidates must be at least k");
    if (!(delta > 0.0 && delta < 1.0))
        return fail(1, "RunParams: termination_delta must be in (0,1)");
    if (n <= k) return fail(1, "run: need n > k");
    if (n < 2 || d < 1) return fail(1, "Dataset: degenerate shape");

    Data ds, permuted = {0, 0, 0, NULL};
    if (!data_make(&ds, data, n, d)) return fail(2, "run: out of memory");
    const Data* active = &ds;
    Mt64 master;
    mt_seed(&master, seed);
    uint64_t evals = 0;
    double t0 = now_s();
    const uint64_t init_seed = mt_next(&master);
    Graph g;
    int rc = init_random(&g, &ds, k, init_seed, &evals);
    if (rc) {
        free(ds.v);
        return rc;
    }
    double t1 = now_s();
    uint32_t rows = 0;
    double total = 0.0;
#define PUSH_ROW(EV, CH, W)                        \
    do {                                           \
        if (iter_evals) iter_evals[rows] = (EV);   \
        if (iter_changes) iter_changes[rows] = (CH); \
        if (iter_wall) iter_wall[rows] = (W);      \
        total += (W);                              \
        ++rows;                                    \
    } while (0)
    PUSH_ROW(evals, 0, t1 - t0);

    Cands c;
    rc = cands_alloc(&c, n, cap);
    if (rc) {
        graph_free(&g);
        free(ds.v);
        return rc;
    }
    uint32_t* sigma = NULL;
    uint32_t* sigma_inv = NULL;
    const double threshold = delta * (double)n * (double)k;
    for (uint32_t iter = 1; iter <= max_iterations; ++iter) {
        t0 = now_s();
        const uint64_t iter_seed = mt_next(&master);
        g.changes = 0;
        select_turbo(&g, iter_seed, &c);
        for (uint32_t u = 0; u < n; ++u) flag_consumed(&g, u, new_data(&c, u), c.nc[u]);
        uint64_t step_evals = 0;
        const uint64_t changes = compute_step(&g, &c, active, &step_evals);
        if (reorder && !sigma && iter == reorder_after) {
            sigma = malloc(sizeof(uint32_t) * n);
            sigma_inv = malloc(sizeof(uint32_t) * n);
            greedy_cluster(&g, sigma, sigma_inv);
            apply_permutation(active, sigma, &permuted);
            active = &permuted;
            remap(&g, sigma);
        }
        t1 = now_s();
        PUSH_ROW(step_evals, changes, t1 - t0);
        if ((double)changes < threshold) break;
    }
#undef PUSH_ROW
    if (sigma) remap(&g, sigma_inv);
    export_graph(&g, out_ids, out_dists, out_flags, NULL);
    if (n_rows) *n_rows = rows;
    if (total_wall) *total_wall = total;
    if (sigma_out && sigma) memcpy(sigma_out, sigma, sizeof(uint32_t) * n);
    free(sigma);
    free(sigma_inv);
    free(permuted.v);
    cands_free(&c);
    graph_free(&g);
    free(ds.v);
    return 0;
}

int oracle_capture_step(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                        uint64_t seed, uint32_t t, uint32_t* in_ids, float* in_dists,
                        uint8_t* in_flags, uint32_t* in_rev_deg, uint32_t* cand_ids,
                        uint32_t* new_counts, uint32_t* old_counts, uint32_t* out_ids,
                        float* out_dists, uint8_t* out_flags, uint32_t* out_rev_deg,
                        uint64_t* changes, uint64_t* evals) {
    if (t < 1) return fail(1, "oracle_capture_step: t must be >= 1");
    Data ds;
    if (!data_make(&ds, data, n, d)) return fail(2, "out of memory");
    Mt64 master;
    mt_seed(&master, seed);
    uint64_t ev = 0;
    Graph g;
    int rc = init_random(&g, &ds, k, mt_next(&master), &ev);
    if (rc) {
        free(ds.v);
        return rc;
    }
    Cands c;
    rc = cands_alloc(&c, n, cap);
    if (rc) {
        graph_free(&g);
        free(ds.v);
        return rc;
    }
    for (uint32_t iter = 1; iter <= t; ++iter) {
        const uint64_t iter_seed = mt_next(&master);
        g.changes = 0;
        select_turbo(&g, iter_seed, &c);
        for (uint32_t u = 0; u < n; ++u) flag_consumed(&g, u, new_data(&c, u), c.nc[u]);
        if (iter == t) {
            export_graph(&g, in_ids, in_dists, in_flags, in_rev_deg);
            export_cands(&c, cand_ids, new_counts, old_counts);
        }
        uint64_t step_evals = 0;
        const uint64_t ch = compute_step(&g, &c, &ds, &step_evals);
        if (iter == t) {
            export_graph(&g, out_ids, out_dists, out_flags, out_rev_deg);
            if (changes) *changes = ch;
            if (evals) *evals = step_evals;
        }
    }
    cands_free(&c);
    graph_free(&g);
    free(ds.v);
    return 0;
}

int oracle_compute_step(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                        const uint32_t* in_ids, const float* in_dists, const uint8_t* in_flags,
                        const uint32_t* cand_ids, const uint32_t* new_counts,
                        const uint32_t* old_counts, int flat, uint32_t* out_ids,
                        float* out_dists, uint8_t* out_flags, uint32_t* out_rev_deg,
                        uint64_t* changes, uint64_t* evals) {
    Data ds;
    if (!data_make(&ds, data, n, d)) return fail(2, "out of memory");
    Graph g;
    int rc = from_rows(&g, n, k, in_ids, in_dists, in_flags);
    if (rc) {
        graph_free(&g);
        free(ds.v);
        return rc;
    }
    Cands c;
    rc = cands_alloc(&c, n, cap);
    if (rc) {
        graph_free(&g);
        free(ds.v);
        return rc;
    }
    for (uint32_t u = 0; u < n; ++u) {
        if (new_counts[u] > cap || old_counts[u] > cap) {
            cands_free(&c);
            graph_free(&g);
            free(ds.v);
            return fail(1, "compute_step: candidate count exceeds cap");
        }
        c.nc[u] = new_counts[u];
        c.oc[u] = old_counts[u];
        memcpy(new_data(&c, u), cand_ids + (size_t)u * 2 * cap, sizeof(uint32_t) * new_counts[u]);
        memcpy(old_data(&c, u), cand_ids + (size_t)u * 2 * cap + cap,
               sizeof(uint32_t) * old_counts[u]);
    }
    uint64_t ev = 0;
    const uint64_t ch = flat ? compute_step_flat(&g, &c, &ds, &ev) : compute_step(&g, &c, &ds, &ev);
    export_graph(&g, out_ids, out_dists, out_flags, out_rev_deg);
    if (changes) *changes = ch;
    if (evals) *evals = ev;
    cands_free(&c);
    graph_free(&g);
    free(ds.v);
    return 0;
}

int oracle_init_random(const float* data, uint32_t n, uint32_t d, uint32_t k, uint64_t seed,
                       uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
                       uint32_t* out_rev_deg, uint64_t* evals) {
    Data ds;
    if (n < 2 || d < 1) return fail(1, "Dataset: degenerate shape");
    if (!data_make(&ds, data, n, d)) return fail(2, "out of memory");
    Graph g;
    uint64_t ev = 0;
    const int rc = init_random(&g, &ds, k, seed, &ev);
    if (!rc) export_graph(&g, out_ids, out_dists, out_flags, out_rev_deg);
    if (evals) *evals = ev;
    graph_free(&g);
    free(ds.v);
    return rc;
}

int oracle_select_turbo(uint32_t n, uint32_t k, uint32_t cap, const uint32_t* in_ids,
                        const float* in_dists, const uint8_t* in_flags, uint64_t seed,
                        uint32_t* cand_ids, uint32_t* new_counts, uint32_t* old_counts,
                        uint8_t* out_flags_after_consume) {
    Graph g;
    int rc = from_rows(&g, n, k, in_ids, in_dists, in_flags);
    if (rc) {
        graph_free(&g);
        return rc;
    }
    Cands c;
    rc = cands_alloc(&c, n, cap);
    if (rc) {
        graph_free(&g);
        return rc;
    }
    select_turbo(&g, seed, &c);
    export_cands(&c, cand_ids, new_counts, old_counts);
    if (out_flags_after_consume) {
        for (uint32_t u = 0; u < n; ++u) flag_consumed(&g, u, new_data(&c, u), c.nc[u]);
        for (uint32_t u = 0; u < n; ++u)
            for (uint32_t i = 0; i < k; ++i) {
                const uint32_t id = in_ids[(size_t)u * k + i];
                for (uint32_t j = 0; j < k; ++j)
                    if (g.ids[(size_t)u * k + j] == id)
                        out_flags_after_consume[(size_t)u * k + i] = g.flags[(size_t)u * k + j];
            }
    }
    cands_free(&c);
    graph_free(&g);
    return 0;
}

/* brute_force_knng (oracle.hpp:92-127): double accumulation in 8 lanes over
 * the TRUE dimension d (l2_sq_double, oracle.hpp:50-66), (dist,id) order.
 * The reference's compiled double loop FUSES the square-accumulate (pinned
 * against the reference harness in tests/test_oracle_pins.py). */
static double l2_double(const float* a, const float* b, uint32_t d) {
    double acc[8] = {0};
    uint32_t j = 0;
    for (; j + 8 <= d; j += 8)
        for (uint32_t l = 0; l < 8; ++l) {
            const double diff = (double)a[j + l] - (double)b[j + l];
            acc[l] = fma(diff, diff, acc[l]);
        }
    double tail = 0.0;
    for (; j < d; ++j) {
        const double diff = (double)a[j] - (double)b[j];
        tail = fma(diff, diff, tail);
    }
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7])) + tail;
}

typedef struct {
    double dist;
    uint32_t id;
} Exact;

static int exact_less(Exact a, Exact b) {
    return a.dist != b.dist ? a.dist < b.dist : a.id < b.id;
}

/* exact_insert (oracle.hpp:78-86) */
static void exact_insert(Exact* list, uint32_t k, Exact cand) {
    if (!exact_less(cand, list[k - 1])) return;
    uint32_t i = k - 1;
    while (i > 0 && exact_less(cand, list[i - 1])) {
        list[i] = list[i - 1];
        --i;
    }
    list[i] = cand;
}

int oracle_brute_force(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t* out_ids,
                       double* out_dists) {
    if (k == 0 || k >= n) return fail(1, "brute_force_knng: need 0 < k < n");
    Data ds;
    if (!data_make(&ds, data, n, d)) return fail(2, "out of memory");
    Exact* best = malloc(sizeof(Exact) * (size_t)n * k);
    for (size_t p = 0; p < (size_t)n * k; ++p) {
        best[p].dist = INFINITY;
        best[p].id = 0xffffffffu;
    }
    for (uint32_t ib = 0; ib < n; ib += 256) {
        const uint32_t ie = ib + 256 < n ? ib + 256 : n;
        for (uint32_t j = ib + 1; j < n; ++j) {
            const uint32_t lim = ie < j ? ie : j;
            for (uint32_t i = ib; i < lim; ++i) {
                const double dist = l2_double(row(&ds, i), row(&ds, j), d);
                exact_insert(best + (size_t)i * k, k, (Exact){dist, j});
                exact_insert(best + (size_t)j * k, k, (Exact){dist, i});
            }
        }
    }
    for (size_t p = 0; p < (size_t)n * k; ++p) {
        out_ids[p] = best[p].id;
        if (out_dists) out_dists[p] = best[p].dist;
    }
    free(best);
    free(ds.v);
    return 0;
}

static int u32_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* recall (oracle.hpp:131-144): membership by id. */
int oracle_recall(uint32_t n, uint32_t k, const uint32_t* approx_ids, const float* approx_dists,
                  const uint32_t* exact_ids, double* out) {
    (void)approx_dists;
    uint32_t* truth = malloc(sizeof(uint32_t) * k);
    uint64_t hits = 0;
    for (uint32_t u = 0; u < n; ++u) {
        memcpy(truth, exact_ids + (size_t)u * k, sizeof(uint32_t) * k);
        qsort(truth, k, sizeof(uint32_t), u32_cmp);
        for (uint32_t i = 0; i < k; ++i)
            if (bsearch(&approx_ids[(size_t)u * k + i], truth, k, sizeof(uint32_t), u32_cmp))
                ++hits;
    }
    free(truth);
    *out = (double)hits / ((double)n * (double)k);
    return 0;
}

int oracle_greedy_cluster(uint32_t n, uint32_t k, const uint32_t* ids, const float* dists,
                          const uint8_t* flags, uint32_t* sigma, uint32_t* sigma_inv) {
    Graph g;
    const int rc = from_rows(&g, n, k, ids, dists, flags);
    if (!rc) greedy_cluster(&g, sigma, sigma_inv);
    graph_free(&g);
    return rc;
}

float oracle_l2_sq(const float* a, const float* b, uint32_t d) { return l2_scalar(a, b, d); }

int oracle_block_l2_sq(const float* rows_a, uint32_t na, const float* rows_b, uint32_t nb,
                       uint32_t d, float* out) {
    if (na == 0 || nb == 0) return fail(1, "block_l2_sq: empty tile");
    if (na > 5 || nb > 5) return fail(1, "block_l2_sq: tile larger than 5x5");
    const int full = na == 5 && nb == 5;
    for (uint32_t i = 0; i < na; ++i)
        for (uint32_t j = 0; j < nb; ++j) {
            const float* a = rows_a + (size_t)i * d;
            const float* b = rows_b + (size_t)j * d;
            out[i * nb + j] = full ? l2_tile(a, b, d) : l2_scalar(a, b, d);
        }
    return 0;
}

int oracle_mutual_block(const float* rows, uint32_t m, uint32_t d, float* out_matrix,
                        uint32_t* visit_pairs, uint64_t* n_visits) {
    uint64_t count = 0;
#define VISIT(I, J, D)                                              \
    do {                                                            \
        const float dv = (D);                                       \
        out_matrix[(size_t)(I) * m + (J)] = dv;                     \
        out_matrix[(size_t)(J) * m + (I)] = dv;                     \
        if (visit_pairs) {                                          \
            visit_pairs[2 * count] = (I);                           \
            visit_pairs[2 * count + 1] = (J);                       \
        }                                                           \
        ++count;                                                    \
    } while (0)
    if (m >= 2) {
        const uint32_t full = m - m % 5;
        for (uint32_t gi = 0; gi < full; gi += 5) {
            for (int p = 0; p < 10; ++p) {
                const uint32_t x = gi + kTri[p][0], y = gi + kTri[p][1];
                VISIT(x, y, l2_tile(rows + (size_t)x * d, rows + (size_t)y * d, d));
            }
            for (uint32_t gj = gi + 5; gj < full; gj += 5)
                for (uint32_t x = 0; x < 5; ++x)
                    for (uint32_t y = 0; y < 5; ++y)
                        VISIT(gi + x, gj + y,
                              l2_tile(rows + (size_t)(gi + x) * d, rows + (size_t)(gj + y) * d, d));
        }
        for (uint32_t r = full; r < m; ++r)
            for (uint32_t q = 0; q < r; ++q)
                VISIT(q, r, l2_scalar(rows + (size_t)q * d, rows + (size_t)r * d, d));
    }
#undef VISIT
    if (n_visits) *n_visits = count;
    return 0;
}

void oracle_mt64_stream(uint64_t seed, uint64_t* out, uint32_t count) {
    Mt64 r;
    mt_seed(&r, seed);
    for (uint32_t i = 0; i < count; ++i) out[i] = mt_next(&r);
}
