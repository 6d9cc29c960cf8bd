/* ORACLE / TEST INFRASTRUCTURE ONLY — see gpufaas_oracle.h.
 *
 * Deliberately naive plain-C restatement of the reference simulator's
 * control plane. Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). It shares no code with the
 * product (paper_2303_05601_b200/csrc): model locations are re-derived by
 * scanning caches, the global queue is a flat array, and every scheduling
 * pass works on snapshots exactly as the reference does.
 */
#define _POSIX_C_SOURCE 200809L
#include "gpufaas_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------- */
/* errors                                                                     */

static __thread char g_err[512];
static __thread int g_failed;

static void fail(const char* fmt, ...) {
    if (g_failed) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_failed = 1;
}
const char* orc_sim_last_error(void) { return g_err; }
void orc_free(void* p) { free(p); }

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}
static void* xrealloc(void* p, size_t s) {
    void* q = realloc(p, s ? s : 1);
    if (!q) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return q;
}

/* ------------------------------------------------------------------------- */
/* mt19937_64 (std::mt19937_64 parameters), Rng wrapper: include/gpufaas/rng.hpp:11-30 */

typedef struct { uint64_t mt[312]; int mti; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:24-26: raw % n */
static int64_t mt64_uniform_below(mt64* s, int64_t n) { return (int64_t)(mt64_next(s) % (uint64_t)n); }
/* rng.hpp:28-30: (raw >> 11) * 2^-53 */
static double mt64_uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

void orc_mt19937_64(uint64_t seed, int64_t n, uint64_t* out) {
    mt64 s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = mt64_next(&s);
}

/* ------------------------------------------------------------------------- */
/* catalog: include/gpufaas/catalog.hpp:15-48, src/catalog.cpp:45-111       */

#define ORC_ID_MAX 96

typedef struct {
    char id[ORC_ID_MAX];
    double occupation_mb;
    int64_t load_us, infer_us;
} orc_model;

typedef struct {
    orc_model* m;
    int n;
} orc_catalog;

/* sim_time.hpp:15-17 */
static int64_t seconds_to_us(double s) { return (int64_t)llround(s * 1e6); }

/* split on ',' dropping '\r' (catalog.cpp:28-41) */
static int split_fields(const char* line, size_t len, char fields[][ORC_ID_MAX], int maxf) {
    int nf = 0;
    size_t pos = 0;
    fields[0][0] = 0;
    for (size_t i = 0; i < len; ++i) {
        char c = line[i];
        if (c == ',') {
            fields[nf][pos] = 0;
            if (++nf >= maxf) return -1;
            pos = 0;
            fields[nf][0] = 0;
        } else if (c != '\r') {
            if (pos + 1 < ORC_ID_MAX) fields[nf][pos++] = c;
        }
    }
    fields[nf][pos] = 0;
    return nf + 1;
}

/* std::stod semantics used by catalog.cpp:16-26: whole field must parse */
static int parse_double(const char* s, double* out) {
    if (!*s) return 0;
    char* end = NULL;
    double v = strtod(s, &end);
    if (end == s || *end) return 0;
    *out = v;
    return 1;
}

/* iterate lines of a text buffer */
typedef struct { const char* p; } line_iter;
static int next_line(line_iter* it, const char** line, size_t* len) {
    if (!it->p || !*it->p) return 0;
    const char* e = strchr(it->p, '\n');
    *line = it->p;
    if (e) { *len = (size_t)(e - it->p); it->p = e + 1; }
    else { *len = strlen(it->p); it->p = it->p + *len; }
    return 1;
}

/* parse_catalog_csv: catalog.cpp:71-105 */
static int parse_catalog(const char* text, orc_catalog* cat) {
    line_iter it = {text};
    const char* line;
    size_t len;
    char f[8][ORC_ID_MAX];
    memset(cat, 0, sizeof *cat);
    if (!next_line(&it, &line, &len)) { fail("catalog: empty catalog file"); return 0; }
    int nf = split_fields(line, len, f, 8);
    if (nf != 4 || strcmp(f[0], "model_id") || strcmp(f[1], "occupation_mb") ||
        strcmp(f[2], "load_time_s") || strcmp(f[3], "infer_time_s")) {
        fail("catalog:1: bad header");
        return 0;
    }
    int cap = 16, lineno = 1;
    cat->m = xcalloc((size_t)cap, sizeof(orc_model));
    while (next_line(&it, &line, &len)) {
        ++lineno;
        if (len == 0 || (len == 1 && line[0] == '\r')) continue;
        nf = split_fields(line, len, f, 8);
        if (nf != 4) { fail("catalog:%d: expected 4 fields", lineno); return 0; }
        orc_model m;
        memset(&m, 0, sizeof m);
        snprintf(m.id, sizeof m.id, "%s", f[0]);
        double a, b, c;
        if (!parse_double(f[1], &a) || !parse_double(f[2], &b) || !parse_double(f[3], &c)) {
            fail("catalog:%d: bad value", lineno);
            return 0;
        }
        m.occupation_mb = a;
        m.load_us = seconds_to_us(b);
        m.infer_us = seconds_to_us(c);
        if (!m.id[0]) { fail("catalog:%d: empty model_id", lineno); return 0; }
        if (m.occupation_mb <= 0 || m.load_us <= 0 || m.infer_us <= 0) {
            fail("catalog:%d: non-positive value for model '%s'", lineno, m.id);
            return 0;
        }
        for (int i = 0; i < cat->n; ++i)
            if (!strcmp(cat->m[i].id, m.id)) { fail("catalog: duplicate model_id '%s'", m.id); return 0; }
        if (cat->n == cap) { cap *= 2; cat->m = xrealloc(cat->m, (size_t)cap * sizeof(orc_model)); }
        cat->m[cat->n++] = m;
    }
    if (cat->n == 0) { fail("catalog: catalog has no model rows"); return 0; }
    return 1;
}

/* ------------------------------------------------------------------------- */
/* trace: include/gpufaas/trace.hpp, src/trace.cpp                           */

typedef struct {
    char (*fn)[ORC_ID_MAX];
    int64_t* counts; /* [rows][minutes] */
    int rows, minutes;
} orc_trace;

static void trace_free(orc_trace* t) { free(t->fn); free(t->counts); memset(t, 0, sizeof *t); }

/* parse_trace_csv: trace.cpp:56-102 */
static int parse_trace(const char* text, orc_trace* t) {
    line_iter it = {text};
    const char* line;
    size_t len;
    memset(t, 0, sizeof *t);
    if (!next_line(&it, &line, &len)) { fail("trace: empty trace file"); return 0; }
    /* header: function_id,m1..mN */
    int cols = 1;
    for (size_t i = 0; i < len; ++i) cols += line[i] == ',';
    if (cols > 100000) { fail("trace: too many columns"); return 0; }
    char (*f)[ORC_ID_MAX] = xcalloc((size_t)cols + 1, ORC_ID_MAX);
    int nf = split_fields(line, len, f, cols + 1);
    if (nf < 2 || strcmp(f[0], "function_id")) { free(f); fail("trace:1: bad header"); return 0; }
    for (int i = 1; i < nf; ++i) {
        char want[32];
        snprintf(want, sizeof want, "m%d", i);
        if (strcmp(f[i], want)) { free(f); fail("trace:1: bad minute column"); return 0; }
    }
    t->minutes = nf - 1;
    int cap = 64, lineno = 1;
    t->fn = xcalloc((size_t)cap, ORC_ID_MAX);
    t->counts = xcalloc((size_t)cap * (size_t)t->minutes, sizeof(int64_t));
    while (next_line(&it, &line, &len)) {
        ++lineno;
        if (len == 0 || (len == 1 && line[0] == '\r')) continue;
        int n2 = split_fields(line, len, f, cols + 1);
        if (n2 != nf) { free(f); fail("trace:%d: field count", lineno); return 0; }
        if (!f[0][0]) { free(f); fail("trace:%d: empty function_id", lineno); return 0; }
        for (int r = 0; r < t->rows; ++r)
            if (!strcmp(t->fn[r], f[0])) { free(f); fail("trace:%d: duplicate function_id", lineno); return 0; }
        if (t->rows == cap) {
            cap *= 2;
            t->fn = xrealloc(t->fn, (size_t)cap * ORC_ID_MAX);
            t->counts = xrealloc(t->counts, (size_t)cap * (size_t)t->minutes * sizeof(int64_t));
        }
        memcpy(t->fn[t->rows], f[0], ORC_ID_MAX);
        for (int m = 0; m < t->minutes; ++m) {
            char* end = NULL;
            const char* s = f[m + 1];
            long long v = strtoll(s, &end, 10);
            if (!*s || *end || v < 0) { free(f); fail("trace:%d: bad count", lineno); return 0; }
            t->counts[(size_t)t->rows * (size_t)t->minutes + (size_t)m] = v;
        }
        t->rows++;
    }
    free(f);
    if (!t->rows) { fail("trace: trace has no function rows"); return 0; }
    return 1;
}

/* make_synthetic_trace: trace.cpp:156-192 */
static int synthetic_trace(int function_count, int minutes, int draws, double zipf, uint64_t seed,
                           orc_trace* t) {
    memset(t, 0, sizeof *t);
    if (function_count <= 0 || minutes <= 0 || draws <= 0) { fail("synthetic trace: all sizes must be positive"); return 0; }
    if (zipf < 0) { fail("synthetic trace: zipf_exponent must be non-negative"); return 0; }
    size_t n = (size_t)function_count;
    double* cdf = xcalloc(n, sizeof(double));
    double sum = 0.0;
    for (size_t r = 0; r < n; ++r) {
        sum += pow((double)(r + 1), -zipf);
        cdf[r] = sum;
    }
    for (size_t r = 0; r < n; ++r) cdf[r] /= sum;
    cdf[n - 1] = 1.0;
    t->rows = function_count;
    t->minutes = minutes;
    t->fn = xcalloc(n, ORC_ID_MAX);
    t->counts = xcalloc(n * (size_t)minutes, sizeof(int64_t));
    for (size_t r = 0; r < n; ++r) snprintf(t->fn[r], ORC_ID_MAX, "f%03zu", r);
    mt64 rng;
    mt64_seed(&rng, seed);
    for (int m = 0; m < minutes; ++m) {
        for (int d = 0; d < draws; ++d) {
            double u = mt64_uniform01(&rng);
            /* std::upper_bound: first cdf[i] > u */
            size_t lo = 0, hi = n;
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (u < cdf[mid]) hi = mid; else lo = mid + 1;
            }
            size_t idx = lo;
            if (idx >= n) idx = n - 1;
            t->counts[idx * (size_t)minutes + (size_t)m]++;
        }
    }
    free(cdf);
    return 1;
}

char* orc_synthetic_trace_csv(int function_count, int minutes, int draws, double zipf, uint64_t seed) {
    g_failed = 0;
    orc_trace t;
    if (!synthetic_trace(function_count, minutes, draws, zipf, seed, &t)) return NULL;
    size_t cap = 64 + (size_t)t.rows * (size_t)(t.minutes + 1) * 24;
    char* out = xcalloc(cap, 1);
    size_t pos = (size_t)snprintf(out, cap, "function_id");
    for (int m = 1; m <= t.minutes; ++m) pos += (size_t)snprintf(out + pos, cap - pos, ",m%d", m);
    pos += (size_t)snprintf(out + pos, cap - pos, "\n");
    for (int r = 0; r < t.rows; ++r) {
        pos += (size_t)snprintf(out + pos, cap - pos, "%s", t.fn[r]);
        for (int m = 0; m < t.minutes; ++m)
            pos += (size_t)snprintf(out + pos, cap - pos, ",%lld",
                                    (long long)t.counts[(size_t)r * (size_t)t.minutes + (size_t)m]);
        pos += (size_t)snprintf(out + pos, cap - pos, "\n");
    }
    trace_free(&t);
    return out;
}

static int64_t trace_total(const orc_trace* t, int r) {
    int64_t s = 0;
    for (int m = 0; m < t->minutes; ++m) s += t->counts[(size_t)r * (size_t)t->minutes + (size_t)m];
    return s;
}

/* top_function_rows: trace.cpp:130-146 — totals desc, function_id asc */
static const orc_trace* g_sort_trace;
static int64_t* g_sort_totals;
static int cmp_top(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    if (g_sort_totals[x] != g_sort_totals[y]) return g_sort_totals[x] > g_sort_totals[y] ? -1 : 1;
    return strcmp(g_sort_trace->fn[x], g_sort_trace->fn[y]);
}

/* ------------------------------------------------------------------------- */
/* workload: src/workload.cpp                                                 */

typedef struct {
    int model;          /* catalog index */
    int64_t arrival_us;
    int skip_count;     /* workload.hpp:19 */
    int64_t dispatched_at_us, completed_at_us;
} orc_request;

/* largest_remainder_allocate: workload.cpp:11-42 (stable sort by remainder desc) */
static int64_t* g_rem;
static int cmp_rem(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    if (g_rem[x] != g_rem[y]) return g_rem[x] > g_rem[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}
static int lra(const int64_t* counts, int n, int64_t total, int64_t* alloc) {
    if (total < 0) { fail("largest_remainder_allocate: negative total"); return 0; }
    int64_t base = 0;
    for (int i = 0; i < n; ++i) base += counts[i];
    for (int i = 0; i < n; ++i) if (counts[i] < 0) { fail("largest_remainder_allocate: negative count"); return 0; }
    if (base == 0) {
        if (total == 0) { memset(alloc, 0, (size_t)n * sizeof(int64_t)); return 1; }
        fail("largest_remainder_allocate: all counts are zero");
        return 0;
    }
    int64_t* rem = xcalloc((size_t)n, sizeof(int64_t));
    int* order = xcalloc((size_t)n, sizeof(int));
    int64_t assigned = 0;
    for (int i = 0; i < n; ++i) {
        int64_t num = counts[i] * total;
        alloc[i] = num / base;
        rem[i] = num % base;
        assigned += alloc[i];
        order[i] = i;
    }
    g_rem = rem;
    qsort(order, (size_t)n, sizeof(int), cmp_rem);
    for (size_t j = 0; assigned < total; ++j) {
        alloc[order[j % (size_t)n]] += 1;
        ++assigned;
    }
    free(rem);
    free(order);
    return 1;
}

/* interleave_catalog_by_size: workload.cpp:44-62 — sort (occupation, id) asc, then lo/hi */
static const orc_catalog* g_sort_cat;
static int cmp_size(const void* a, const void* b) {
    const orc_model* x = &g_sort_cat->m[*(const int*)a];
    const orc_model* y = &g_sort_cat->m[*(const int*)b];
    if (x->occupation_mb != y->occupation_mb) return x->occupation_mb < y->occupation_mb ? -1 : 1;
    return strcmp(x->id, y->id);
}

typedef struct { int64_t arrival; uint64_t seq; int model; } orc_draw;
static int cmp_draw(const void* a, const void* b) {
    const orc_draw* x = a;
    const orc_draw* y = b;
    if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* synthesize_workload: workload.cpp:86-157 */
static int synthesize(const orc_trace* t, const orc_sim_config* c, const orc_catalog* cat,
                      orc_request** out, int* n_out) {
    if (c->working_set <= 0) { fail("workload: working_set_size must be positive"); return 0; }
    if (c->per_minute_total <= 0) { fail("workload: per_minute_total must be positive"); return 0; }
    if (c->duration_minutes <= 0) { fail("workload: duration_minutes must be positive"); return 0; }
    if (c->duration_minutes > t->minutes) { fail("workload: duration exceeds trace length"); return 0; }
    int k = c->working_set;
    if (k > t->rows) { fail("top_function_rows: k exceeds trace function count"); return 0; }
    int* rows = xcalloc((size_t)t->rows, sizeof(int));
    int64_t* totals = xcalloc((size_t)t->rows, sizeof(int64_t));
    for (int r = 0; r < t->rows; ++r) { rows[r] = r; totals[r] = trace_total(t, r); }
    g_sort_trace = t;
    g_sort_totals = totals;
    qsort(rows, (size_t)t->rows, sizeof(int), cmp_top);

    /* build_model_mapping: workload.cpp:64-77 */
    if (cat->n == 0) { fail("model mapping: empty catalog"); return 0; }
    if (k > 2 * cat->n) { fail("model mapping: working set needs more than two passes over the catalog"); return 0; }
    int* sorted = xcalloc((size_t)cat->n, sizeof(int));
    for (int i = 0; i < cat->n; ++i) sorted[i] = i;
    g_sort_cat = cat;
    qsort(sorted, (size_t)cat->n, sizeof(int), cmp_size);
    int* inter = xcalloc((size_t)cat->n, sizeof(int));
    int lo = 0, hi = cat->n, w = 0;
    while (lo < hi) {
        inter[w++] = sorted[lo++];
        if (lo < hi) inter[w++] = sorted[--hi];
    }
    int* fn_model = xcalloc((size_t)k, sizeof(int));
    for (int r = 0; r < k; ++r) fn_model[r] = inter[r % cat->n];

    size_t cap = (size_t)c->per_minute_total * (size_t)c->duration_minutes;
    orc_draw* draws = xcalloc(cap, sizeof(orc_draw));
    size_t nd = 0;
    mt64 rng;
    mt64_seed(&rng, c->seed);
    uint64_t seq = 0;
    int64_t* mc = xcalloc((size_t)k, sizeof(int64_t));
    int64_t* alloc = xcalloc((size_t)k, sizeof(int64_t));
    int ok = 1;
    for (int m = 0; m < c->duration_minutes && ok; ++m) {
        int64_t sum = 0;
        for (int r = 0; r < k; ++r) { mc[r] = t->counts[(size_t)rows[r] * (size_t)t->minutes + (size_t)m]; sum += mc[r]; }
        if (sum == 0) { fail("workload: working set has no invocations in minute %d", m + 1); ok = 0; break; }
        if (!lra(mc, k, c->per_minute_total, alloc)) { ok = 0; break; }
        int64_t minute_start = (int64_t)m * 60000000LL;
        for (int r = 0; r < k; ++r) {
            for (int64_t i = 0; i < alloc[r]; ++i) {
                if (nd == cap) { cap *= 2; draws = xrealloc(draws, cap * sizeof(orc_draw)); }
                draws[nd].arrival = minute_start + mt64_uniform_below(&rng, 60000000LL);
                draws[nd].seq = seq++;
                draws[nd].model = fn_model[r];
                nd++;
            }
        }
    }
    if (ok) {
        qsort(draws, nd, sizeof(orc_draw), cmp_draw);
        orc_request* reqs = xcalloc(nd, sizeof(orc_request));
        for (size_t i = 0; i < nd; ++i) {
            reqs[i].model = draws[i].model;
            reqs[i].arrival_us = draws[i].arrival;
            reqs[i].dispatched_at_us = -1;
            reqs[i].completed_at_us = -1;
        }
        *out = reqs;
        *n_out = (int)nd;
    }
    free(rows); free(totals); free(sorted); free(inter); free(fn_model); free(draws); free(mc); free(alloc);
    return ok;
}

/* ------------------------------------------------------------------------- */
/* cluster: include/gpufaas/cluster.hpp, src/cluster.cpp                     */

typedef struct { int model; double occupation_mb; uint64_t last_use_tick; int64_t uses; } orc_cached;
typedef struct { int request; int model; int64_t infer_us; } orc_local;

typedef struct {
    orc_cached* cache;   /* index 0 = MRU (cluster.hpp:79) */
    int ncache, capcache;
    double capacity_mb, cached_mb;  /* incrementally updated doubles (cluster.cpp:112,121) */
    int64_t hotness;
    orc_local* lq;
    int nlq, caplq, lq_head;
    int64_t lq_infer_us;
    int running_req, running_model;  /* -1 idle */
    int64_t busy_until;
    /* Extension (pipelined GPUs; product: SchedulerConfig::pipeline): one task
     * staged behind the running one; copy_free = end of the last load here. */
    int staged_req, staged_model;    /* -1 none */
    int64_t staged_until, copy_free;
    int* pins;  /* per catalog model */
} orc_gpu;

typedef struct {
    orc_gpu* g;
    int n;
    uint64_t use_ticks;
    int nmodels;
    int pipeline;
    double headroom_mb;  /* largest catalog model */
} orc_cluster;

/* can a dispatch start on g now? reference: idle. Pipelined: nothing staged,
 * and while running, unpinned memory for any catalog model (summed MRU -> LRU) */
static int accepting(const orc_cluster* c, const orc_gpu* g) {
    if (!c->pipeline) return g->running_req < 0;
    if (g->staged_req >= 0) return 0;
    if (g->running_req < 0) return 1;
    double pinned = 0.0;
    for (int i = 0; i < g->ncache; ++i)
        if (g->pins[g->cache[i].model] > 0) pinned += g->cache[i].occupation_mb;
    return g->capacity_mb - pinned >= c->headroom_mb;
}
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

static int gpu_find(const orc_gpu* g, int model) {
    for (int i = 0; i < g->ncache; ++i) if (g->cache[i].model == model) return i;
    return -1;
}

/* locations derived by scanning (cluster.cpp:69-83) */
static int locations(const orc_cluster* c, int model, int* out) {
    int n = 0;
    for (int g = 0; g < c->n; ++g) if (gpu_find(&c->g[g], model) >= 0) out[n++] = g;
    return n;
}
static int cached_anywhere_except(const orc_cluster* c, int model, int gpu) {
    for (int g = 0; g < c->n; ++g) if (g != gpu && gpu_find(&c->g[g], model) >= 0) return 1;
    return 0;
}

/* estimate_finish_time: cluster.cpp:85-93 */
static int64_t estimate_finish(const orc_cluster* c, int gpu, int64_t now) {
    const orc_gpu* g = &c->g[gpu];
    int64_t rem = 0;
    if (g->running_req >= 0) {
        rem = (g->staged_req >= 0 ? g->staged_until : g->busy_until) - now;
        if (rem < 0) fail("cluster invariant violated: running task finished in the past");
    }
    return rem + g->lq_infer_us;
}

/* touch: cluster.cpp:95-102 */
static void touch(orc_cluster* c, orc_gpu* g, int model) {
    int i = gpu_find(g, model);
    orc_cached e = g->cache[i];
    e.uses += 1;
    e.last_use_tick = ++c->use_ticks;
    g->hotness += 1;
    memmove(&g->cache[1], &g->cache[0], (size_t)i * sizeof(orc_cached));
    g->cache[0] = e;
}

/* insert_model: cluster.cpp:104-115 */
static void insert_model(orc_cluster* c, orc_gpu* g, int model, double mb) {
    if (g->cached_mb + mb > g->capacity_mb) fail("cluster invariant violated: insert would exceed capacity");
    if (g->ncache == g->capcache) {
        g->capcache = g->capcache ? g->capcache * 2 : 8;
        g->cache = xrealloc(g->cache, (size_t)g->capcache * sizeof(orc_cached));
    }
    memmove(&g->cache[1], &g->cache[0], (size_t)g->ncache * sizeof(orc_cached));
    g->cache[0].model = model;
    g->cache[0].occupation_mb = mb;
    g->cache[0].last_use_tick = ++c->use_ticks;
    g->cache[0].uses = 1;
    g->ncache++;
    g->cached_mb += mb;
    g->hotness += 1;
}

/* evict_one: cluster.cpp:117-129 */
static void evict_one(orc_gpu* g, int model) {
    int i = gpu_find(g, model);
    if (i < 0) { fail("cluster invariant violated: evict of non-resident model"); return; }
    if (g->pins[model] > 0) { fail("cluster invariant violated: evict of pinned model"); return; }
    g->cached_mb -= g->cache[i].occupation_mb;
    g->hotness -= g->cache[i].uses;
    memmove(&g->cache[i], &g->cache[i + 1], (size_t)(g->ncache - i - 1) * sizeof(orc_cached));
    g->ncache--;
}

/* select_victims: cluster.cpp:131-148 — walk LRU tail to head skipping pinned */
static int select_victims(const orc_gpu* g, int gpu_id, double needed, int* victims) {
    if (needed > g->capacity_mb) { fail("model of %f MB cannot fit on a %f MB gpu", needed, g->capacity_mb); return -1; }
    int nv = 0;
    double free_mb = g->capacity_mb - g->cached_mb;
    for (int i = g->ncache - 1; i >= 0 && free_mb < needed; --i) {
        if (g->pins[g->cache[i].model] > 0) continue;
        victims[nv++] = g->cache[i].model;
        free_mb += g->cache[i].occupation_mb;
    }
    if (free_mb < needed) { fail("gpu %d cannot free enough memory: pinned models occupy the cache", gpu_id); return -1; }
    return nv;
}

/* ------------------------------------------------------------------------- */
/* decisions (sched.hpp:31-53)                                                */

typedef struct {
    int kind; /* 0 hit_idle, 1 miss_idle, 2 enqueue_local */
    int request, gpu, from_local, false_miss, skip;
    int64_t completion_us, load_us, infer_us;
    int nev, ev_off;
} orc_decision;

typedef struct {
    orc_decision* d;
    int64_t n, cap;
    int* ev;
    int64_t nev, capev;
} orc_dlist;

static orc_decision* dl_push(orc_dlist* l) {
    if (l->n == l->cap) { l->cap = l->cap ? l->cap * 2 : 256; l->d = xrealloc(l->d, (size_t)l->cap * sizeof(orc_decision)); }
    orc_decision* d = &l->d[l->n++];
    memset(d, 0, sizeof *d);
    d->completion_us = -1;
    return d;
}
static void dl_push_ev(orc_dlist* l, int model) {
    if (l->nev == l->capev) { l->capev = l->capev ? l->capev * 2 : 256; l->ev = xrealloc(l->ev, (size_t)l->capev * sizeof(int)); }
    l->ev[l->nev++] = model;
}

/* ------------------------------------------------------------------------- */
/* global queue (sched.cpp:44-67): arrival-ordered flat array                 */

typedef struct { int* ids; int n, cap; } orc_queue;
static void q_push(orc_queue* q, int id) {
    if (q->n == q->cap) { q->cap = q->cap ? q->cap * 2 : 256; q->ids = xrealloc(q->ids, (size_t)q->cap * sizeof(int)); }
    q->ids[q->n++] = id;
}
static int q_find(const orc_queue* q, int id) {
    for (int i = 0; i < q->n; ++i) if (q->ids[i] == id) return i;
    return -1;
}
static void q_remove(orc_queue* q, int id) {
    int i = q_find(q, id);
    if (i < 0) { fail("queue invariant violated: request %d not queued", id); return; }
    memmove(&q->ids[i], &q->ids[i + 1], (size_t)(q->n - i - 1) * sizeof(int));
    q->n--;
}

/* ------------------------------------------------------------------------- */
/* scheduler: src/sched.cpp                                                    */

typedef struct {
    orc_cluster* cl;
    orc_queue* q;
    orc_request* req;
    const orc_catalog* cat;
    int64_t now;
    int policy, limit;
    orc_dlist* out;
} orc_ctx;

/* ClusterState::begin_execution: cluster.cpp:150-174; returns completion */
static int64_t begin_execution(orc_ctx* x, int gpu, int request, int* hit, orc_decision* d) {
    orc_gpu* g = &x->cl->g[gpu];
    if (!accepting(x->cl, g)) { fail("cluster invariant violated: begin_execution on busy gpu %d", gpu); return 0; }
    int model = x->req[request].model;
    const orc_model* p = &x->cat->m[model];
    int64_t completion;
    int behind = g->running_req >= 0;  /* pipelined: staged behind the running task */
    *hit = gpu_find(g, model) >= 0;
    if (*hit) {
        touch(x->cl, g, model);
        completion = (behind ? max64(x->now, g->busy_until) : x->now) + p->infer_us;
    } else {
        int* victims = xcalloc((size_t)g->ncache + 1, sizeof(int));
        int nv = select_victims(g, gpu, p->occupation_mb, victims);
        if (nv < 0) { free(victims); return 0; }
        d->ev_off = (int)x->out->nev;
        d->nev = nv;
        for (int i = 0; i < nv; ++i) { dl_push_ev(x->out, victims[i]); evict_one(g, victims[i]); }
        free(victims);
        insert_model(x->cl, g, model, p->occupation_mb);
        /* load on the copy engine once the previous load here is done; the
         * inference once the load and the running task are */
        int64_t load_end = (behind ? max64(x->now, g->copy_free) : x->now) + p->load_us;
        g->copy_free = load_end;
        completion = (behind ? max64(load_end, g->busy_until) : load_end) + p->infer_us;
    }
    if (behind) {
        g->staged_req = request;
        g->staged_model = model;
        g->staged_until = completion;
    } else {
        g->running_req = request;
        g->running_model = model;
        g->busy_until = completion;
    }
    g->pins[model] += 1;
    return completion;
}

/* Scheduler::dispatch: sched.cpp:113-134 */
static void dispatch(orc_ctx* x, int gpu, int request, int from_local) {
    orc_request* r = &x->req[request];
    if (!from_local) q_remove(x->q, request);
    int elsewhere = cached_anywhere_except(x->cl, r->model, gpu);
    orc_decision* d = dl_push(x->out);
    int hit = 0;
    int64_t completion = begin_execution(x, gpu, request, &hit, d);
    r->dispatched_at_us = x->now;
    const orc_model* p = &x->cat->m[r->model];
    d->kind = hit ? 0 : 1;
    d->request = request;
    d->gpu = gpu;
    d->from_local = from_local;
    d->false_miss = !hit && elsewhere;
    d->skip = r->skip_count;
    d->completion_us = completion;
    d->load_us = hit ? 0 : p->load_us;
    d->infer_us = p->infer_us;
}

/* Scheduler::locality_load_balance: sched.cpp:187-241 */
static int llb(orc_ctx* x, int gpu, int request) {
    orc_request* r = &x->req[request];
    const orc_model* p = &x->cat->m[r->model];
    int locs[1024];
    int nl = locations(x->cl, r->model, locs);
    if (nl == 0) { dispatch(x, gpu, request, 0); return 1; }
    int best_idle = -1, best_running = 0;
    uint64_t best_tick = 0;
    for (int i = 0; i < nl; ++i) {
        const orc_gpu* g = &x->cl->g[locs[i]];
        if (!accepting(x->cl, g)) continue;
        uint64_t tick = g->cache[gpu_find(g, r->model)].last_use_tick;
        int running = g->running_req >= 0;  /* pipelined: idle holders first */
        if (best_idle == -1 || (running == best_running ? tick > best_tick : !running)) {
            best_idle = locs[i]; best_tick = tick; best_running = running;
        }
    }
    if (best_idle != -1) { dispatch(x, best_idle, request, 0); return best_idle == gpu; }
    int best_busy = -1;
    int64_t best_est = 0;
    for (int i = 0; i < nl; ++i) {
        int64_t est = estimate_finish(x->cl, locs[i], x->now);
        if (best_busy == -1 || est < best_est) { best_busy = locs[i]; best_est = est; }
    }
    if (best_est < p->load_us) {
        q_remove(x->q, request);
        /* ClusterState::push_local: cluster.cpp:189-198 */
        orc_gpu* g = &x->cl->g[best_busy];
        if (gpu_find(g, r->model) < 0) { fail("cluster invariant violated: local enqueue for non-resident model"); return 0; }
        if (g->nlq == g->caplq) { g->caplq = g->caplq ? g->caplq * 2 : 16; g->lq = xrealloc(g->lq, (size_t)g->caplq * sizeof(orc_local)); }
        g->lq[g->nlq].request = request;
        g->lq[g->nlq].model = r->model;
        g->lq[g->nlq].infer_us = p->infer_us;
        g->nlq++;
        g->lq_infer_us += p->infer_us;
        g->pins[r->model] += 1;
        orc_decision* d = dl_push(x->out);
        d->kind = 2;
        d->request = request;
        d->gpu = best_busy;
        d->skip = r->skip_count;
        d->infer_us = 0;
        return 0;
    }
    dispatch(x, gpu, request, 0);
    return 1;
}

/* Scheduler::schedule_idle_gpu: sched.cpp:136-185 */
static void schedule_idle_gpu(orc_ctx* x, int gpu) {
    orc_gpu* g = &x->cl->g[gpu];
    if (g->nlq - g->lq_head > 0) {
        /* pop_local: cluster.cpp:200-208 */
        orc_local e = g->lq[g->lq_head++];
        g->lq_infer_us -= e.infer_us;
        g->pins[e.model] -= 1;
        dispatch(x, gpu, e.request, 1);
        if (x->out->d[x->out->n - 1].kind != 0) fail("locally queued request missed its pinned model");
        return;
    }
    if (x->q->n == 0) return;
    if (x->policy == 0) { dispatch(x, gpu, x->q->ids[0], 0); return; }

    /* Pass 1 over a snapshot (sched.cpp:161-176) */
    int n = x->q->n;
    if (n <= 0) return;
    int* scan = xcalloc((size_t)n, sizeof(int));
    memcpy(scan, x->q->ids, (size_t)n * sizeof(int));
    int* bypassed = xcalloc((size_t)n, sizeof(int));
    int nb = 0;
    for (int i = 0; i < n && !g_failed; ++i) {
        int rid = scan[i];
        if (q_find(x->q, rid) < 0) continue;
        orc_request* r = &x->req[rid];
        if (gpu_find(g, r->model) >= 0) {
            for (int b = 0; b < nb; ++b) x->req[bypassed[b]].skip_count += 1;
            dispatch(x, gpu, rid, 0);
            free(scan); free(bypassed);
            return;
        }
        if (r->skip_count >= x->limit) {
            if (llb(x, gpu, rid)) { free(scan); free(bypassed); return; }
            continue;
        }
        bypassed[nb++] = rid;
    }
    free(scan);
    free(bypassed);
    /* Pass 2 over a fresh snapshot (sched.cpp:180-184) */
    n = x->q->n;
    if (n <= 0) return;
    int* rest = xcalloc((size_t)n, sizeof(int));
    memcpy(rest, x->q->ids, (size_t)n * sizeof(int));
    for (int i = 0; i < n && !g_failed; ++i) {
        if (q_find(x->q, rest[i]) < 0) continue;
        if (llb(x, gpu, rest[i])) break;
    }
    free(rest);
}

/* idle_gpus_in_service_order + on_scheduling_point: sched.cpp:93-111
 * (hotness re-summed from cache contents, like tests/support/reference_scheduler.cpp:39-43) */
static void on_scheduling_point(orc_ctx* x) {
    int G = x->cl->n;
    int* idle = xcalloc((size_t)G, sizeof(int));
    int64_t* hot = xcalloc((size_t)G, sizeof(int64_t));
    int ni = 0;
    for (int g = 0; g < G; ++g) {
        if (!accepting(x->cl, &x->cl->g[g])) continue;
        int64_t h = 0;
        for (int i = 0; i < x->cl->g[g].ncache; ++i) h += x->cl->g[g].cache[i].uses;
        if (h != x->cl->g[g].hotness) fail("oracle: hotness drift");
        idle[ni] = g;
        hot[ni] = h;
        ni++;
    }
    /* stable insertion sort: (pipelined: idle before running), hotness desc,
     * ties keep ascending id */
    for (int i = 1; i < ni; ++i) {
        int gi = idle[i];
        int64_t hi = hot[i];
        int ri = x->cl->g[gi].running_req >= 0;
        int j = i - 1;
        while (j >= 0) {
            int rj = x->cl->g[idle[j]].running_req >= 0;
            if (!(rj > ri || (rj == ri && hot[j] < hi))) break;
            idle[j + 1] = idle[j]; hot[j + 1] = hot[j]; --j;
        }
        idle[j + 1] = gi;
        hot[j + 1] = hi;
    }
    for (int i = 0; i < ni && !g_failed; ++i) {
        if (!accepting(x->cl, &x->cl->g[idle[i]])) continue;
        schedule_idle_gpu(x, idle[i]);
    }
    free(idle);
    free(hot);
}

/* ------------------------------------------------------------------------- */
/* event log (engine.cpp:63-98): nlohmann dump with sorted keys              */

typedef struct { char* s; size_t n, cap; } sbuf;
static void sb_put(sbuf* b, const char* s, size_t n) {
    if (b->n + n + 1 > b->cap) {
        b->cap = (b->n + n + 1) * 2;
        b->s = xrealloc(b->s, b->cap);
    }
    memcpy(b->s + b->n, s, n);
    b->n += n;
    b->s[b->n] = 0;
}
static void sb_str(sbuf* b, const char* s) { sb_put(b, s, strlen(s)); }
static void sb_fmt(sbuf* b, const char* fmt, ...) {
    char tmp[256];
    va_list ap;
    va_start(ap, fmt);
    int k = vsnprintf(tmp, sizeof tmp, fmt, ap);
    va_end(ap);
    sb_put(b, tmp, (size_t)k);
}
static void sb_json_string(sbuf* b, const char* s) {
    sb_put(b, "\"", 1);
    for (; *s; ++s) {
        unsigned char c = (unsigned char)*s;
        if (c == '"') sb_str(b, "\\\"");
        else if (c == '\\') sb_str(b, "\\\\");
        else if (c == '\n') sb_str(b, "\\n");
        else if (c == '\t') sb_str(b, "\\t");
        else if (c == '\r') sb_str(b, "\\r");
        else if (c == '\b') sb_str(b, "\\b");
        else if (c == '\f') sb_str(b, "\\f");
        else if (c < 0x20) sb_fmt(b, "\\u%04x", c);
        else sb_put(b, (const char*)&c, 1);
    }
    sb_put(b, "\"", 1);
}
static void log_caches(sbuf* b, const orc_cluster* cl, const orc_catalog* cat) {
    sb_str(b, "\"caches\":[");
    for (int g = 0; g < cl->n; ++g) {
        if (g) sb_put(b, ",", 1);
        sb_put(b, "[", 1);
        for (int i = 0; i < cl->g[g].ncache; ++i) {
            if (i) sb_put(b, ",", 1);
            sb_json_string(b, cat->m[cl->g[g].cache[i].model].id);
        }
        sb_put(b, "]", 1);
    }
    sb_str(b, "],");
}

/* ------------------------------------------------------------------------- */
/* engine: run_stream (engine.cpp:100-173) + metrics (metrics.cpp:23-107)    */

typedef struct { int64_t t; int kind; uint64_t seq; int payload; } orc_event;
typedef struct { orc_event* e; size_t n, cap; } orc_heap;
static int ev_less(const orc_event* a, const orc_event* b) {  /* engine.cpp:21-25 */
    if (a->t != b->t) return a->t < b->t;
    if (a->kind != b->kind) return a->kind < b->kind;
    return a->seq < b->seq;
}
static void heap_push(orc_heap* h, orc_event v) {
    if (h->n == h->cap) { h->cap = h->cap ? h->cap * 2 : 1024; h->e = xrealloc(h->e, h->cap * sizeof(orc_event)); }
    size_t i = h->n++;
    h->e[i] = v;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!ev_less(&h->e[i], &h->e[p])) break;
        orc_event t = h->e[i]; h->e[i] = h->e[p]; h->e[p] = t;
        i = p;
    }
}
static orc_event heap_pop(orc_heap* h) {
    orc_event top = h->e[0];
    h->e[0] = h->e[--h->n];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && ev_less(&h->e[l], &h->e[m])) m = l;
        if (r < h->n && ev_less(&h->e[r], &h->e[m])) m = r;
        if (m == i) break;
        orc_event t = h->e[i]; h->e[i] = h->e[m]; h->e[m] = t;
        i = m;
    }
    return top;
}

typedef struct {
    orc_catalog cat;
    orc_request* req;
    int nreq;
    orc_dlist dl;
    orc_report rep;
    sbuf log;
    double run_ns;
} orc_handle;

static const char* kind_name(int k) { return k == 0 ? "hit_idle" : k == 1 ? "miss_idle" : "enqueue_local"; }

static int run_stream(orc_handle* H, const orc_sim_config* c) {
    const orc_catalog* cat = &H->cat;
    orc_request* req = H->req;
    int n = H->nreq;
    if (c->gpu_count <= 0) { fail("cluster: gpu_count must be positive"); return 0; }
    if (c->capacity_mb <= 0) { fail("cluster: capacity_mb must be positive"); return 0; }
    if (c->o3_limit < 0) { fail("scheduler: o3_limit must be >= 0"); return 0; }
    /* validate_stream: engine.cpp:28-45 */
    int64_t prev = 0;
    for (int i = 0; i < n; ++i) {
        if (req[i].arrival_us < prev) { fail("request stream: arrivals must be sorted"); return 0; }
        prev = req[i].arrival_us;
        if (req[i].model < 0 || req[i].model >= cat->n) { fail("catalog: unknown model"); return 0; }
        if (cat->m[req[i].model].occupation_mb > c->capacity_mb) { fail("model '%s' cannot fit in gpu memory", cat->m[req[i].model].id); return 0; }
    }
    /* most_requested_model: engine.cpp:47-59 — max count, ties lexicographically first id */
    int64_t* counts = xcalloc((size_t)cat->n, sizeof(int64_t));
    for (int i = 0; i < n; ++i) counts[req[i].model]++;
    int top = -1;
    for (int m = 0; m < cat->n; ++m) {
        if (!counts[m]) continue;
        if (top < 0 || counts[m] > counts[top] || (counts[m] == counts[top] && strcmp(cat->m[m].id, cat->m[top].id) < 0)) top = m;
    }
    free(counts);

    orc_cluster cl;
    cl.n = c->gpu_count;
    cl.use_ticks = 0;
    cl.nmodels = cat->n;
    cl.pipeline = c->pipeline != 0;
    cl.headroom_mb = 0.0;
    for (int m = 0; m < cat->n; ++m)
        if (cat->m[m].occupation_mb > cl.headroom_mb) cl.headroom_mb = cat->m[m].occupation_mb;
    cl.g = xcalloc((size_t)cl.n, sizeof(orc_gpu));
    for (int g = 0; g < cl.n; ++g) {
        cl.g[g].capacity_mb = c->capacity_mb;
        cl.g[g].running_req = -1;
        cl.g[g].running_model = -1;
        cl.g[g].staged_req = -1;
        cl.g[g].staged_model = -1;
        cl.g[g].pins = xcalloc((size_t)cat->n, sizeof(int));
    }
    orc_queue q = {0};
    orc_ctx x = {&cl, &q, req, cat, 0, c->policy, c->policy == 2 ? c->o3_limit : 0, &H->dl};

    /* metrics accumulator state (metrics.hpp:72-85) */
    int64_t hits = 0, misses = 0, false_misses = 0, local_enq = 0, evictions = 0, busy_us = 0, infer_us = 0;
    int max_skip = 0;
    double copy_area = 0.0;
    int64_t copies_since = 0;
    int current_copies = 0;

    orc_heap heap = {0};
    uint64_t seq = 0;
    for (int i = 0; i < n; ++i) heap_push(&heap, (orc_event){req[i].arrival_us, 1, seq++, i});
    int64_t now = 0;
    int log = c->log_events;
    while (heap.n && !g_failed) {
        orc_event ev = heap_pop(&heap);
        if (ev.t < now) { fail("engine: event time went backwards"); break; }
        now = ev.t;
        x.now = now;
        if (ev.kind == 0) {
            /* ClusterState::complete: cluster.cpp:176-187 */
            orc_gpu* g = &cl.g[ev.payload];
            if (g->running_req < 0 || g->busy_until != now) { fail("cluster invariant violated: completion"); break; }
            int rid = g->running_req;
            g->pins[g->running_model] -= 1;
            g->running_req = -1;
            g->running_model = -1;
            g->busy_until = 0;
            if (g->staged_req >= 0) {  /* pipelined: the staged task runs now */
                g->running_req = g->staged_req;
                g->running_model = g->staged_model;
                g->busy_until = g->staged_until;
                g->staged_req = -1;
                g->staged_model = -1;
                g->staged_until = 0;
            }
            req[rid].completed_at_us = now;
            if (log) {
                sb_str(&H->log, "{");
                if (log == 2) log_caches(&H->log, &cl, cat);
                sb_fmt(&H->log, "\"event\":\"completion\",\"gpu_id\":%d,\"request_id\":%d,\"t_us\":%lld}\n",
                       ev.payload, rid, (long long)now);
            }
        } else {
            q_push(&q, ev.payload);
            if (log)
                sb_fmt(&H->log, "{\"event\":\"arrival\",\"request_id\":%d,\"t_us\":%lld}\n", ev.payload, (long long)now);
        }
        int64_t first = H->dl.n;
        on_scheduling_point(&x);
        for (int64_t i = first; i < H->dl.n && !g_failed; ++i) {
            orc_decision* d = &H->dl.d[i];
            if (d->kind == 0 || d->kind == 1) heap_push(&heap, (orc_event){d->completion_us, 0, seq++, d->gpu});
            /* record_decision: metrics.cpp:23-49 */
            if (d->skip > max_skip) max_skip = d->skip;
            if (d->kind == 0 || d->kind == 1) {
                if (d->kind == 0) hits++;
                else { misses++; if (d->false_miss) false_misses++; }
                evictions += d->nev;
                busy_us += d->load_us + d->infer_us;
                infer_us += d->infer_us;
            } else {
                local_enq++;
            }
            if (log) {
                sb_str(&H->log, "{");
                if (log == 2) log_caches(&H->log, &cl, cat);
                sb_fmt(&H->log, "\"decision\":\"%s\",\"event\":\"decision\",", kind_name(d->kind));
                if (d->kind != 2) sb_fmt(&H->log, "\"false_miss\":%s,", d->false_miss ? "true" : "false");
                sb_fmt(&H->log, "\"gpu_id\":%d,", d->gpu);
                if (d->kind != 2) sb_fmt(&H->log, "\"hit\":%s,", d->kind == 0 ? "true" : "false");
                sb_fmt(&H->log, "\"request_id\":%d,\"skip_count\":%d,\"t_us\":%lld}\n", d->request, d->skip, (long long)now);
            }
        }
        /* record_top_model_copies: metrics.cpp:51-56 */
        int cp = 0;
        for (int g = 0; g < cl.n; ++g) if (top >= 0 && gpu_find(&cl.g[g], top) >= 0) cp++;
        copy_area += (double)(now - copies_since) * current_copies;
        copies_since = now;
        current_copies = cp;
    }
    int ok = !g_failed;
    if (ok && q.n) { fail("engine: requests still queued after the last event"); ok = 0; }
    for (int g = 0; ok && g < cl.n; ++g)
        if (cl.g[g].running_req >= 0 || cl.g[g].staged_req >= 0 || cl.g[g].nlq - cl.g[g].lq_head > 0) { fail("engine: cluster not drained"); ok = 0; }
    for (int i = 0; ok && i < n; ++i) {
        if (req[i].completed_at_us < 0) { fail("engine: request %d never completed", i); ok = 0; }
        if (req[i].skip_count > x.limit) { fail("engine: request %d bypassed too often", i); ok = 0; }
    }
    if (ok) {
        /* finalize: metrics.cpp:58-107 */
        orc_report* r = &H->rep;
        memset(r, 0, sizeof *r);
        r->request_count = n;
        r->total_sim_time_s = (double)now / 1e6;
        r->hits = hits; r->misses = misses; r->false_misses = false_misses;
        r->local_enqueues = local_enq; r->evictions = evictions; r->max_skip_count = max_skip;
        r->top_model_idx = top;
        int64_t dispatches = hits + misses;
        if (dispatches != n) { fail("metrics: dispatched %lld of %d requests", (long long)dispatches, n); ok = 0; }
        if (dispatches > 0) {
            r->has_ratios = 1;
            r->cache_miss_ratio = (double)misses / (double)dispatches;
            r->false_miss_ratio = (double)false_misses / (double)dispatches;
        }
        if (n > 0) {
            double sum = 0.0;
            for (int i = 0; i < n; ++i) sum += (double)(req[i].completed_at_us - req[i].arrival_us) / 1e6;
            double mean = sum / (double)n;
            double var = 0.0;
            for (int i = 0; i < n; ++i) {
                double d = (double)(req[i].completed_at_us - req[i].arrival_us) / 1e6 - mean;
                var += d * d;
            }
            r->has_latency = 1;
            r->avg_latency_s = mean;
            r->latency_variance_s2 = var / (double)n;
        }
        if (now > 0) {
            copy_area += (double)(now - copies_since) * current_copies;
            r->has_time = 1;
            r->avg_top_model_duplicates = copy_area / (double)now;
            double cluster_time = (double)now * c->gpu_count;
            r->utilization_busy = (double)busy_us / cluster_time;
            r->utilization_infer_only = (double)infer_us / cluster_time;
        }
    }
    for (int g = 0; g < cl.n; ++g) { free(cl.g[g].cache); free(cl.g[g].lq); free(cl.g[g].pins); }
    free(cl.g);
    free(q.ids);
    free(heap.e);
    return ok && !g_failed;
}

static double now_ns(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec * 1e9 + (double)ts.tv_nsec;
}

static void handle_free(orc_handle* H) {
    if (!H) return;
    free(H->cat.m);
    free(H->req);
    free(H->dl.d);
    free(H->dl.ev);
    free(H->log.s);
    free(H);
}

void* orc_sim_run(const char* catalog_csv, const char* trace_csv, const orc_sim_config* c) {
    g_failed = 0;
    g_err[0] = 0;
    orc_handle* H = xcalloc(1, sizeof(orc_handle));
    orc_trace t;
    int ok = parse_catalog(catalog_csv, &H->cat);
    if (ok) {
        if (trace_csv && !c->use_synthetic_trace) ok = parse_trace(trace_csv, &t);
        else ok = synthetic_trace(c->syn_function_count, c->syn_minutes, c->syn_draws_per_minute,
                                  c->syn_zipf_exponent, c->syn_seed, &t);
        if (ok) {
            ok = synthesize(&t, c, &H->cat, &H->req, &H->nreq);
            trace_free(&t);
        }
    }
    if (ok) {
        double t0 = now_ns();
        ok = run_stream(H, c);
        H->run_ns = now_ns() - t0;
    }
    if (!ok) { handle_free(H); return NULL; }
    return H;
}

void* orc_sim_run_stream(const char* catalog_csv, const orc_sim_config* c, int n,
                         const int32_t* model_idx, const int64_t* arrival_us) {
    g_failed = 0;
    g_err[0] = 0;
    orc_handle* H = xcalloc(1, sizeof(orc_handle));
    int ok = parse_catalog(catalog_csv, &H->cat);
    if (ok) {
        H->nreq = n;
        H->req = xcalloc((size_t)n, sizeof(orc_request));
        for (int i = 0; i < n; ++i) {
            H->req[i].model = model_idx[i];
            H->req[i].arrival_us = arrival_us[i];
            H->req[i].dispatched_at_us = -1;
            H->req[i].completed_at_us = -1;
        }
        double t0 = now_ns();
        ok = run_stream(H, c);
        H->run_ns = now_ns() - t0;
    }
    if (!ok) { handle_free(H); return NULL; }
    return H;
}

int64_t orc_sim_num_decisions(void* h) { return ((orc_handle*)h)->dl.n; }
int64_t orc_sim_num_requests(void* h) { return ((orc_handle*)h)->nreq; }
double orc_sim_run_ns(void* h) { return ((orc_handle*)h)->run_ns; }

void orc_sim_get_decisions(void* h, int32_t* ints, int64_t* times) {
    orc_handle* H = h;
    for (int64_t i = 0; i < H->dl.n; ++i) {
        const orc_decision* d = &H->dl.d[i];
        int32_t* o = ints + 7 * i;
        o[0] = d->kind; o[1] = d->request; o[2] = d->gpu; o[3] = d->from_local;
        o[4] = d->false_miss; o[5] = d->skip; o[6] = d->nev;
        times[3 * i] = d->completion_us;
        times[3 * i + 1] = d->load_us;
        times[3 * i + 2] = d->infer_us;
    }
}

int32_t orc_sim_get_evicted(void* h, int64_t i, int32_t* out, int32_t cap) {
    orc_handle* H = h;
    const orc_decision* d = &H->dl.d[i];
    for (int k = 0; k < d->nev && k < cap; ++k) out[k] = H->dl.ev[d->ev_off + k];
    return d->nev;
}

void orc_sim_get_requests(void* h, int32_t* model_idx, int64_t* arrival, int64_t* dispatched,
                          int64_t* completed, int32_t* skip) {
    orc_handle* H = h;
    for (int i = 0; i < H->nreq; ++i) {
        model_idx[i] = H->req[i].model;
        arrival[i] = H->req[i].arrival_us;
        dispatched[i] = H->req[i].dispatched_at_us;
        completed[i] = H->req[i].completed_at_us;
        skip[i] = H->req[i].skip_count;
    }
}

void orc_sim_get_report(void* h, orc_report* out) { *out = ((orc_handle*)h)->rep; }

static uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = p;
    for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ULL; }
    return h;
}
#define FNV_BASIS 14695981039346656037ULL

uint64_t orc_sim_decision_digest(void* h) {
    orc_handle* H = h;
    uint64_t x = FNV_BASIS;
    for (int64_t i = 0; i < H->dl.n; ++i) {
        const orc_decision* d = &H->dl.d[i];
        int32_t a[6] = {d->kind, d->request, d->gpu, d->from_local, d->false_miss, d->skip};
        for (int k = 0; k < 6; ++k) x = fnv(x, &a[k], 4);
        x = fnv(x, &d->completion_us, 8);
        x = fnv(x, &d->load_us, 8);
        x = fnv(x, &d->infer_us, 8);
        int32_t nev = d->nev;
        x = fnv(x, &nev, 4);
        for (int k = 0; k < d->nev; ++k) {
            const char* s = H->cat.m[H->dl.ev[d->ev_off + k]].id;
            x = fnv(x, s, strlen(s) + 1);
        }
    }
    return x;
}

uint64_t orc_sim_request_digest(void* h) {
    orc_handle* H = h;
    uint64_t x = FNV_BASIS;
    for (int i = 0; i < H->nreq; ++i) {
        x = fnv(x, &H->req[i].dispatched_at_us, 8);
        x = fnv(x, &H->req[i].completed_at_us, 8);
        int32_t s = H->req[i].skip_count;
        x = fnv(x, &s, 4);
    }
    return x;
}

uint64_t orc_sim_log_digest(void* h) {
    orc_handle* H = h;
    return fnv(FNV_BASIS, H->log.s ? H->log.s : "", H->log.n);
}
int64_t orc_sim_log_size(void* h) { return (int64_t)((orc_handle*)h)->log.n; }
const char* orc_sim_log(void* h) { orc_handle* H = h; return H->log.s ? H->log.s : ""; }
void orc_sim_free(void* h) { handle_free(h); }
