/*
 * gd_oracle.c -- CPU restatement of the reference's dynamic-graph hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.  The product (paper_2507_11094_b200/) never links or calls it.
 *
 * It restates, single-threaded and in plain C, the algorithm of the reference
 * package /root/reference/pkg (graphdyn v0.1.0):
 *   - the diff-CSR store:   src/graphdyn/graph/{csr,dynamic}.py and
 *                           runtime/graphdyn_rt.h:215-511
 *   - dynamic SSSP:         src/graphdyn/programs/sssp_dynamic.sp:8-158,
 *                           tests/golden/sssp_dynamic_omp.cc:10-261
 *   - dynamic PageRank:     src/graphdyn/programs/pr_dynamic.sp:7-102,
 *                           tests/golden/pr_dynamic_omp.cc:9-138
 *   - dynamic triangles:    src/graphdyn/programs/tc_dynamic.sp:7-115,
 *                           tests/golden/tc_dynamic_omp.cc:8-148
 *   - flag flooding:        src/graphdyn/engine/interp.py:70-109,
 *                           runtime/graphdyn_rt.h:595-633
 * Loops run in the order the emitted code runs them with --threads 1, so PR
 * results are bit-identical to pr_bin --threads 1 (same summation order).
 *
 * Parity pinning: tests/test_oracle_golden.py checks this file against the
 * fixtures in tests/golden/ (made by tests/golden/make_golden.py from the
 * reference Python package and the reference's own emitted OpenMP binaries).
 *
 * Return codes follow include/gd_capi.h: 0 ok, -1 malformed input,
 * -2 contract violation, -3 configuration, -4 exec error, -5 diverged.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_SENT INT64_MAX /* csr.py:14 SENTINEL */
#define OR_INF INT64_MAX  /* properties.py:20 INT_INF */

#define OR_OK 0
#define OR_MALFORMED (-1)
#define OR_CONTRACT (-2)
#define OR_CONFIG (-3)
#define OR_EXEC (-4)
#define OR_DIVERGED (-5)

static char or_err[512];
const char* or_last_error(void) { return or_err; }
static int fail(int code, const char* msg) {
    snprintf(or_err, sizeof or_err, "%s", msg);
    return code;
}

/* graphdyn_rt.h:40-44 / interp.py:181-185 */
static int64_t sat_add(int64_t a, int64_t b) {
    if (a >= OR_INF || b >= OR_INF) return OR_INF;
    return a + b;
}

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "gd_oracle: out of memory\n");
        abort();
    }
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) {
        fprintf(stderr, "gd_oracle: out of memory\n");
        abort();
    }
    return p;
}

/* ------------------------------------------------------------------------ */
/* store: csr.py:17-80, dynamic.py:46-334, graphdyn_rt.h:215-511             */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t* off;   /* n+1 */
    int64_t* coord; /* nslots, SENTINEL marks a deleted slot */
    int64_t* w;     /* nslots or NULL when unweighted */
    int64_t nslots;
} or_seg;

typedef struct {
    int64_t src;
    int32_t seg;
    int64_t idx;
} or_rev;

typedef struct {
    or_rev* a;
    int64_t len, cap;
} or_revlist;

typedef struct or_graph {
    int64_t n;
    int directed, weighted, with_reverse;
    int64_t merge_interval;
    int nseg, segcap;
    or_seg* segs; /* [0] is the base, then deltas in creation order */
    int64_t live;
    int64_t version, merge_epoch;
    or_revlist* rev; /* per-node reverse entries, NULL without reverse */
    int64_t nclaims, claimcap;
    int32_t* claim_seg;
    int64_t* claim_idx;
} or_graph;

typedef struct {
    int64_t s, d, w;
} or_arc;

/* Csr.from_buckets (csr.py:27-50): counting sort by src, stable per src. */
static or_seg seg_from_arcs(int64_t n, const or_arc* arcs, int64_t m, int weighted) {
    or_seg s;
    s.nslots = m;
    s.off = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
    s.coord = (int64_t*)xmalloc((size_t)m * sizeof(int64_t));
    s.w = weighted ? (int64_t*)xmalloc((size_t)m * sizeof(int64_t)) : NULL;
    for (int64_t i = 0; i < m; ++i) s.off[arcs[i].s + 1]++;
    for (int64_t v = 0; v < n; ++v) s.off[v + 1] += s.off[v];
    int64_t* cur = (int64_t*)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
    memcpy(cur, s.off, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) {
        int64_t p = cur[arcs[i].s]++;
        s.coord[p] = arcs[i].d;
        if (weighted) s.w[p] = arcs[i].w;
    }
    free(cur);
    return s;
}

static void seg_free(or_seg* s) {
    free(s->off);
    free(s->coord);
    free(s->w);
}

static void push_seg(or_graph* g, or_seg s) {
    if (g->nseg == g->segcap) {
        g->segcap = g->segcap ? 2 * g->segcap : 4;
        g->segs = (or_seg*)realloc(g->segs, (size_t)g->segcap * sizeof(or_seg));
    }
    g->segs[g->nseg++] = s;
}

static void rev_push(or_revlist* l, int64_t src, int32_t seg, int64_t idx) {
    if (l->len == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 4;
        l->a = (or_rev*)realloc(l->a, (size_t)l->cap * sizeof(or_rev));
    }
    l->a[l->len].src = src;
    l->a[l->len].seg = seg;
    l->a[l->len].idx = idx;
    l->len++;
}

/* graphdyn_rt.h:474-482 drop_rev: erase the entry naming (seg, idx). */
static void rev_drop(or_revlist* l, int32_t seg, int64_t idx) {
    for (int64_t k = 0; k < l->len; ++k) {
        if (l->a[k].seg == seg && l->a[k].idx == idx) {
            memmove(&l->a[k], &l->a[k + 1], (size_t)(l->len - k - 1) * sizeof(or_rev));
            l->len--;
            return;
        }
    }
}

/* dynamic.py:319-329 _rebuild_reverse: per segment, per node, per slot. */
static void rebuild_reverse(or_graph* g) {
    if (!g->rev) g->rev = (or_revlist*)xcalloc((size_t)(g->n ? g->n : 1), sizeof(or_revlist));
    for (int64_t v = 0; v < g->n; ++v) g->rev[v].len = 0;
    for (int sg = 0; sg < g->nseg; ++sg) {
        or_seg* s = &g->segs[sg];
        for (int64_t v = 0; v < g->n; ++v)
            for (int64_t i = s->off[v]; i < s->off[v + 1]; ++i)
                if (s->coord[i] != OR_SENT) rev_push(&g->rev[s->coord[i]], v, sg, i);
    }
}

/* DynamicGraph.build (dynamic.py:89-120). */
int or_graph_build(int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
                   int directed, int weighted, int with_reverse, int64_t merge_interval,
                   or_graph** out) {
    if (n < 0 || n >= OR_SENT) return fail(OR_CONTRACT, "node_count collides with the deletion sentinel");
    if (merge_interval < 1) return fail(OR_CONTRACT, "merge_interval must be >= 1");
    int64_t na = directed ? m : 2 * m;
    or_arc* arcs = (or_arc*)xmalloc((size_t)(na ? na : 1) * sizeof(or_arc));
    int64_t k = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t wi = w ? w[i] : 1;
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) {
            free(arcs);
            snprintf(or_err, sizeof or_err, "edge %lld: node id out of range (src=%lld, dst=%lld, node_count=%lld)",
                     (long long)i, (long long)src[i], (long long)dst[i], (long long)n);
            return OR_MALFORMED;
        }
        if (weighted && wi < 0) {
            free(arcs);
            snprintf(or_err, sizeof or_err, "edge %lld: negative weight %lld", (long long)i, (long long)wi);
            return OR_MALFORMED;
        }
        arcs[k].s = src[i];
        arcs[k].d = dst[i];
        arcs[k].w = wi;
        k++;
        if (!directed) {
            arcs[k].s = dst[i];
            arcs[k].d = src[i];
            arcs[k].w = wi;
            k++;
        }
    }
    or_graph* g = (or_graph*)xcalloc(1, sizeof(or_graph));
    g->n = n;
    g->directed = directed;
    g->weighted = weighted;
    g->with_reverse = with_reverse;
    g->merge_interval = merge_interval;
    /* arcs.sort(key=src) is stable; the counting sort in from_buckets is too */
    push_seg(g, seg_from_arcs(n, arcs, na, weighted));
    free(arcs);
    g->live = na;
    if (with_reverse) rebuild_reverse(g);
    *out = g;
    return OR_OK;
}

void or_graph_free(or_graph* g) {
    if (!g) return;
    for (int i = 0; i < g->nseg; ++i) seg_free(&g->segs[i]);
    free(g->segs);
    if (g->rev) {
        for (int64_t v = 0; v < g->n; ++v) free(g->rev[v].a);
        free(g->rev);
    }
    free(g->claim_seg);
    free(g->claim_idx);
    free(g);
}

static int64_t slot_weight(const or_seg* s, int64_t i) { return s->w ? s->w[i] : 1; }

/* dynamic.py:188-196 _find_live_slot: oldest (base-first) live slot src->dst,
 * skipping (skip_seg, skip_idx). */
static int find_live_slot(const or_graph* g, int64_t src, int64_t dst, int skip_seg, int64_t skip_idx,
                          int* seg_out, int64_t* idx_out) {
    for (int sg = 0; sg < g->nseg; ++sg) {
        const or_seg* s = &g->segs[sg];
        for (int64_t i = s->off[src]; i < s->off[src + 1]; ++i) {
            if (s->coord[i] == dst && !(sg == skip_seg && i == skip_idx)) {
                *seg_out = sg;
                *idx_out = i;
                return 1;
            }
        }
    }
    return 0;
}

/* dynamic.py:316-317 _slot_source */
static int64_t slot_source(const or_seg* s, int64_t n, int64_t idx) {
    int64_t lo = 0, hi = n; /* last v with off[v] <= idx */
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (s->off[mid] <= idx) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

static void kill_slot(or_graph* g, int sg, int64_t i) {
    or_seg* s = &g->segs[sg];
    int64_t dst = s->coord[i];
    s->coord[i] = OR_SENT;
    g->live--;
    if (g->rev) rev_drop(&g->rev[dst], sg, i);
}

/* update_csr_del (dynamic.py:208-244).  miss_flags (nullable) gets 1 per
 * record that found no live slot. */
int or_graph_delete(or_graph* g, const int64_t* src, const int64_t* dst, int64_t k, int64_t* applied,
                    int64_t* misses, uint8_t* miss_flags) {
    for (int64_t r = 0; r < k; ++r)
        if (src[r] < 0 || src[r] >= g->n || dst[r] < 0 || dst[r] >= g->n) {
            snprintf(or_err, sizeof or_err, "node id %lld out of range [0, %lld)",
                     (long long)((src[r] < 0 || src[r] >= g->n) ? src[r] : dst[r]), (long long)g->n);
            return OR_CONTRACT;
        }
    int64_t ap = 0, ms = 0;
    for (int64_t r = 0; r < k; ++r) {
        int sg;
        int64_t i;
        if (miss_flags) miss_flags[r] = 0;
        if (!find_live_slot(g, src[r], dst[r], -1, -1, &sg, &i)) {
            ms++;
            if (miss_flags) miss_flags[r] = 1;
            continue;
        }
        int sg2 = -1;
        int64_t i2 = -1;
        int have2 = 0;
        if (!g->directed && src[r] != dst[r]) {
            have2 = find_live_slot(g, dst[r], src[r], -1, -1, &sg2, &i2);
        } else if (!g->directed) {
            have2 = find_live_slot(g, src[r], dst[r], sg, i, &sg2, &i2);
        }
        kill_slot(g, sg, i);
        if (have2) kill_slot(g, sg2, i2);
        ap++;
    }
    g->version++;
    if (applied) *applied = ap;
    if (misses) *misses = ms;
    return OR_OK;
}

static void claim_push(or_graph* g, int32_t sg, int64_t idx) {
    if (g->nclaims == g->claimcap) {
        g->claimcap = g->claimcap ? 2 * g->claimcap : 16;
        g->claim_seg = (int32_t*)realloc(g->claim_seg, (size_t)g->claimcap * sizeof(int32_t));
        g->claim_idx = (int64_t*)realloc(g->claim_idx, (size_t)g->claimcap * sizeof(int64_t));
    }
    g->claim_seg[g->nclaims] = sg;
    g->claim_idx[g->nclaims] = idx;
    g->nclaims++;
}

/* update_csr_add (dynamic.py:249-286): claim the first vacant slot of src
 * (base first, then deltas), else spill into one new delta per call. */
int or_graph_add(or_graph* g, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t k) {
    for (int64_t r = 0; r < k; ++r)
        if (src[r] < 0 || src[r] >= g->n || dst[r] < 0 || dst[r] >= g->n) {
            snprintf(or_err, sizeof or_err, "node id %lld out of range [0, %lld)",
                     (long long)((src[r] < 0 || src[r] >= g->n) ? src[r] : dst[r]), (long long)g->n);
            return OR_CONTRACT;
        }
    or_arc* left = (or_arc*)xmalloc((size_t)(2 * k + 1) * sizeof(or_arc));
    int64_t nl = 0;
    for (int64_t r = 0; r < k; ++r) {
        int64_t wr = w ? w[r] : 1;
        for (int dir = 0; dir < (g->directed ? 1 : 2); ++dir) {
            int64_t s = dir ? dst[r] : src[r];
            int64_t d = dir ? src[r] : dst[r];
            int placed = 0;
            for (int sg = 0; sg < g->nseg && !placed; ++sg) {
                or_seg* S = &g->segs[sg];
                for (int64_t i = S->off[s]; i < S->off[s + 1]; ++i) {
                    if (S->coord[i] == OR_SENT) {
                        S->coord[i] = d;
                        if (S->w) S->w[i] = wr;
                        claim_push(g, sg, i);
                        if (g->rev) rev_push(&g->rev[d], s, sg, i);
                        placed = 1;
                        break;
                    }
                }
            }
            if (!placed) {
                left[nl].s = s;
                left[nl].d = d;
                left[nl].w = wr;
                nl++;
            }
            g->live++;
        }
    }
    if (nl) {
        or_seg delta = seg_from_arcs(g->n, left, nl, g->weighted);
        push_seg(g, delta);
        int sg = g->nseg - 1;
        if (g->rev) {
            or_seg* S = &g->segs[sg];
            for (int64_t i = 0; i < S->nslots; ++i)
                rev_push(&g->rev[S->coord[i]], slot_source(S, g->n, i), sg, i);
        }
    }
    free(left);
    g->version++;
    return OR_OK;
}

/* merge_deltas (dynamic.py:290-317): compact every live arc, in
 * neighbors() order, into one clean base; rebuild the reverse. */
int or_graph_merge(or_graph* g) {
    or_arc* arcs = (or_arc*)xmalloc((size_t)(g->live + 1) * sizeof(or_arc));
    int64_t m = 0;
    for (int64_t v = 0; v < g->n; ++v)
        for (int sg = 0; sg < g->nseg; ++sg) {
            or_seg* s = &g->segs[sg];
            for (int64_t i = s->off[v]; i < s->off[v + 1]; ++i)
                if (s->coord[i] != OR_SENT) {
                    arcs[m].s = v;
                    arcs[m].d = s->coord[i];
                    arcs[m].w = slot_weight(s, i);
                    m++;
                }
        }
    or_seg base = seg_from_arcs(g->n, arcs, m, g->weighted);
    free(arcs);
    for (int i = 0; i < g->nseg; ++i) seg_free(&g->segs[i]);
    g->nseg = 0;
    push_seg(g, base);
    g->live = m;
    g->nclaims = 0;
    g->version++;
    g->merge_epoch++;
    if (g->with_reverse) rebuild_reverse(g);
    return OR_OK;
}

/* -- inspection (for the store tests) -- */
int64_t or_graph_live(const or_graph* g) { return g->live; }
int or_graph_nseg(const or_graph* g) { return g->nseg; }
int64_t or_graph_seg_slots(const or_graph* g, int sg) { return g->segs[sg].nslots; }
void or_graph_export_seg(const or_graph* g, int sg, int64_t* off, int64_t* coord, int64_t* w) {
    const or_seg* s = &g->segs[sg];
    memcpy(off, s->off, (size_t)(g->n + 1) * sizeof(int64_t));
    memcpy(coord, s->coord, (size_t)s->nslots * sizeof(int64_t));
    if (w) {
        for (int64_t i = 0; i < s->nslots; ++i) w[i] = slot_weight(s, i);
    }
}
/* reverse lists flattened: rev_off[n+1], rev_src[], rev_w[] in list order */
int64_t or_graph_rev_total(const or_graph* g) {
    int64_t t = 0;
    if (!g->rev) return -1;
    for (int64_t v = 0; v < g->n; ++v) t += g->rev[v].len;
    return t;
}
void or_graph_export_rev(const or_graph* g, int64_t* off, int64_t* src, int64_t* w) {
    int64_t p = 0;
    off[0] = 0;
    for (int64_t v = 0; v < g->n; ++v) {
        for (int64_t k = 0; k < g->rev[v].len; ++k) {
            const or_rev* e = &g->rev[v].a[k];
            src[p] = e->src;
            w[p] = slot_weight(&g->segs[e->seg], e->idx);
            p++;
        }
        off[v + 1] = p;
    }
}

/* ------------------------------------------------------------------------ */
/* batch records                                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t *s, *d, *w;
    int64_t k;
} or_recs;

/* UpdateBatch.deletes / .adds (updates.py:42-48): filter in stream order */
static or_recs pick(const uint8_t* kind, const int64_t* s, const int64_t* d, const int64_t* w, int64_t k,
                    uint8_t want) {
    or_recs r;
    r.s = (int64_t*)xmalloc((size_t)(k + 1) * sizeof(int64_t));
    r.d = (int64_t*)xmalloc((size_t)(k + 1) * sizeof(int64_t));
    r.w = (int64_t*)xmalloc((size_t)(k + 1) * sizeof(int64_t));
    r.k = 0;
    for (int64_t i = 0; i < k; ++i)
        if (kind[i] == want) {
            r.s[r.k] = s[i];
            r.d[r.k] = d[i];
            r.w[r.k] = (want == 'a' && w) ? w[i] : 1;
            r.k++;
        }
    return r;
}
static void recs_free(or_recs* r) {
    free(r->s);
    free(r->d);
    free(r->w);
}

/* interp.py:563-570 _validate_batch */
static int validate(const or_graph* g, const uint8_t* kind, const int64_t* s, const int64_t* d, int64_t k) {
    for (int64_t i = 0; i < k; ++i) {
        if (kind[i] != 'a' && kind[i] != 'd') return fail(OR_MALFORMED, "unknown update kind");
        if (s[i] < 0 || s[i] >= g->n || d[i] < 0 || d[i] >= g->n) {
            snprintf(or_err, sizeof or_err, "update record %c %lld %lld references a node outside [0, %lld)",
                     kind[i], (long long)s[i], (long long)d[i], (long long)g->n);
            return OR_EXEC;
        }
    }
    return OR_OK;
}

/* in-edge iteration over the maintained reverse lists (graphdyn_rt.h:362-371) */
#define FOR_IN(g, v, SRC, W, BODY)                                                 \
    for (int64_t _k = 0; _k < (g)->rev[v].len; ++_k) {                             \
        const or_rev* _e = &(g)->rev[v].a[_k];                                     \
        int64_t SRC = _e->src;                                                     \
        int64_t W = slot_weight(&(g)->segs[_e->seg], _e->idx);                     \
        BODY                                                                       \
    }
/* neighbors(v): base then deltas, skipping sentinels (graphdyn_rt.h:329-360) */
#define FOR_OUT(g, v, DST, W, BODY)                                                \
    for (int _sg = 0; _sg < (g)->nseg; ++_sg) {                                    \
        const or_seg* _s = &(g)->segs[_sg];                                        \
        for (int64_t _i = _s->off[v]; _i < _s->off[(v) + 1]; ++_i) {               \
            if (_s->coord[_i] == OR_SENT) continue;                                \
            int64_t DST = _s->coord[_i];                                           \
            int64_t W = slot_weight(_s, _i);                                       \
            (void)W;                                                               \
            BODY                                                                   \
        }                                                                          \
    }

static int any_set(const uint8_t* f, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (f[i]) return 1;
    return 0;
}
/* graphdyn_rt.h:538-544 swap_clear */
static void swap_clear(uint8_t* base, uint8_t* nxt, int64_t n) {
    memcpy(base, nxt, (size_t)n);
    memset(nxt, 0, (size_t)n);
}

/* ------------------------------------------------------------------------ */
/* SSSP: sssp_dynamic.sp / sssp_dynamic_omp.cc                              */
/* ------------------------------------------------------------------------ */

typedef struct or_sssp {
    or_graph* g;
    int64_t src;
    int64_t *dist, *parent;
    int64_t iters; /* fixedPoint iterations, summed */
} or_sssp;

/* parent = min-id in-neighbour closing the distance (sssp_dynamic.sp:23-34) */
static void fix_parent(or_sssp* S, int64_t v) {
    or_graph* g = S->g;
    if (v != S->src && S->dist[v] < OR_INF) {
        S->parent[v] = -1;
        FOR_IN(g, v, u, w, {
            if (sat_add(S->dist[u], w) == S->dist[v])
                if (S->parent[v] == -1 || u < S->parent[v]) S->parent[v] = u;
        })
    }
}

/* staticSSSP: sssp_dynamic_omp.cc:10-59 */
static int sssp_static(or_sssp* S) {
    or_graph* g = S->g;
    int64_t n = g->n;
    uint8_t* mod = (uint8_t*)xcalloc((size_t)n, 1);
    uint8_t* nxt = (uint8_t*)xcalloc((size_t)n, 1);
    for (int64_t v = 0; v < n; ++v) {
        S->dist[v] = OR_INF;
        S->parent[v] = -1;
    }
    S->dist[S->src] = 0;
    mod[S->src] = 1;
    int64_t it = 0, cap = 10 * n;
    while (any_set(mod, n)) {
        if (it >= cap) {
            free(mod);
            free(nxt);
            return fail(OR_DIVERGED, "fixed point diverged");
        }
        for (int64_t v = 0; v < n; ++v) {
            if (!mod[v]) continue;
            FOR_OUT(g, v, t, w, {
                int64_t c = sat_add(S->dist[v], w);
                if (c < S->dist[t]) {
                    S->dist[t] = c;
                    nxt[t] = 1;
                }
            })
        }
        swap_clear(mod, nxt, n);
        ++it;
    }
    S->iters += it;
    for (int64_t v = 0; v < n; ++v) fix_parent(S, v);
    free(mod);
    free(nxt);
    return OR_OK;
}

/* decrementalSSSP: sssp_dynamic_omp.cc:61-159 */
static int sssp_decremental(or_sssp* S, uint8_t* mod) {
    or_graph* g = S->g;
    int64_t n = g->n, cap = 10 * n;
    uint8_t* nxt = (uint8_t*)xcalloc((size_t)n, 1);
    uint8_t* stale = (uint8_t*)xcalloc((size_t)n, 1);
    uint8_t* changed = (uint8_t*)xcalloc((size_t)n, 1);
    int rc = OR_OK;
    S->dist[S->src] = 0;
    for (int64_t v = 0; v < n; ++v)
        if (mod[v]) stale[v] = 1;
    int64_t it = 0;
    while (any_set(mod, n)) { /* walk the tree downstream */
        if (it >= cap) {
            rc = fail(OR_DIVERGED, "fixed point diverged");
            goto done;
        }
        for (int64_t v = 0; v < n; ++v) {
            if (!mod[v]) continue;
            FOR_OUT(g, v, t, w, {
                if (S->parent[t] == v) {
                    S->dist[t] = OR_INF;
                    S->parent[t] = -1;
                    stale[t] = 1;
                    nxt[t] = 1;
                }
            })
        }
        swap_clear(mod, nxt, n);
        ++it;
    }
    S->iters += it;
    S->dist[S->src] = 0;
    for (int64_t v = 0; v < n; ++v)
        if (stale[v]) mod[v] = 1;
    it = 0;
    while (any_set(mod, n)) { /* pull from in-neighbours */
        if (it >= cap) {
            rc = fail(OR_DIVERGED, "fixed point diverged");
            goto done;
        }
        for (int64_t v = 0; v < n; ++v) {
            if (!mod[v]) continue;
            FOR_IN(g, v, u, w, {
                int64_t c = sat_add(S->dist[u], w);
                if (c < S->dist[v]) {
                    S->dist[v] = c;
                    changed[v] = 1;
                }
            })
        }
        for (int64_t v = 0; v < n; ++v) {
            if (!changed[v]) continue;
            changed[v] = 0;
            FOR_OUT(g, v, t, w, {
                if (stale[t]) nxt[t] = 1;
            })
        }
        swap_clear(mod, nxt, n);
        ++it;
    }
    S->iters += it;
    for (int64_t v = 0; v < n; ++v)
        if (stale[v]) fix_parent(S, v);
done:
    free(nxt);
    free(stale);
    free(changed);
    return rc;
}

/* incrementalSSSP: sssp_dynamic_omp.cc:161-215 */
static int sssp_incremental(or_sssp* S, uint8_t* mod) {
    or_graph* g = S->g;
    int64_t n = g->n, cap = 10 * n;
    uint8_t* nxt = (uint8_t*)xcalloc((size_t)n, 1);
    uint8_t* touched = (uint8_t*)xcalloc((size_t)n, 1);
    for (int64_t v = 0; v < n; ++v)
        if (mod[v]) touched[v] = 1;
    int64_t it = 0;
    while (any_set(mod, n)) {
        if (it >= cap) {
            free(nxt);
            free(touched);
            return fail(OR_DIVERGED, "fixed point diverged");
        }
        for (int64_t v = 0; v < n; ++v) {
            if (!mod[v]) continue;
            FOR_OUT(g, v, t, w, {
                int64_t c = sat_add(S->dist[v], w);
                if (c < S->dist[t]) {
                    S->dist[t] = c;
                    nxt[t] = 1;
                    touched[t] = 1;
                }
            })
        }
        swap_clear(mod, nxt, n);
        ++it;
    }
    S->iters += it;
    for (int64_t v = 0; v < n; ++v)
        if (touched[v]) fix_parent(S, v);
    free(nxt);
    free(touched);
    return OR_OK;
}

int or_sssp_create(or_graph* g, int64_t src, or_sssp** out) {
    if (!g->rev) return fail(OR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
    if (src < 0 || src >= g->n) return fail(OR_EXEC, "source node out of range");
    or_sssp* S = (or_sssp*)xcalloc(1, sizeof(or_sssp));
    S->g = g;
    S->src = src;
    S->dist = (int64_t*)xmalloc((size_t)(g->n ? g->n : 1) * sizeof(int64_t));
    S->parent = (int64_t*)xmalloc((size_t)(g->n ? g->n : 1) * sizeof(int64_t));
    int rc = sssp_static(S);
    if (rc) {
        free(S->dist);
        free(S->parent);
        free(S);
        return rc;
    }
    *out = S;
    return OR_OK;
}

/* one Batch body of dynamicSSSP (sssp_dynamic_omp.cc:217-261) */
int or_sssp_batch(or_sssp* S, const uint8_t* kind, const int64_t* s, const int64_t* d, const int64_t* w,
                  int64_t k, int64_t batch_index) {
    or_graph* g = S->g;
    int64_t n = g->n;
    int rc = validate(g, kind, s, d, k);
    if (rc) return rc;
    uint8_t* onDel = (uint8_t*)xcalloc((size_t)n, 1);
    uint8_t* onAdd = (uint8_t*)xcalloc((size_t)n, 1);
    or_recs dl = pick(kind, s, d, w, k, 'd');
    or_recs ad = pick(kind, s, d, w, k, 'a');
    for (int64_t i = 0; i < dl.k; ++i) {
        if (S->parent[dl.d[i]] == dl.s[i]) {
            S->dist[dl.d[i]] = OR_INF;
            S->parent[dl.d[i]] = -1;
            onDel[dl.d[i]] = 1;
        }
    }
    or_graph_delete(g, dl.s, dl.d, dl.k, NULL, NULL, NULL);
    rc = sssp_decremental(S, onDel);
    if (!rc) {
        for (int64_t i = 0; i < ad.k; ++i) {
            int64_t c = sat_add(S->dist[ad.s[i]], ad.w[i]);
            if (c < S->dist[ad.d[i]]) {
                S->dist[ad.d[i]] = c;
                onAdd[ad.d[i]] = 1;
            }
        }
        or_graph_add(g, ad.s, ad.d, ad.w, ad.k);
        rc = sssp_incremental(S, onAdd);
    }
    if (!rc && (batch_index + 1) % g->merge_interval == 0) or_graph_merge(g);
    recs_free(&dl);
    recs_free(&ad);
    free(onDel);
    free(onAdd);
    return rc;
}

void or_sssp_read(const or_sssp* S, int64_t* dist, int64_t* parent) {
    memcpy(dist, S->dist, (size_t)S->g->n * sizeof(int64_t));
    memcpy(parent, S->parent, (size_t)S->g->n * sizeof(int64_t));
}
int64_t or_sssp_iters(const or_sssp* S) { return S->iters; }
void or_sssp_free(or_sssp* S) {
    if (!S) return;
    free(S->dist);
    free(S->parent);
    free(S);
}

/* ------------------------------------------------------------------------ */
/* flag flooding over weak components (interp.py:70-109)                    */
/* ------------------------------------------------------------------------ */

int64_t or_propagate_flags(or_graph* g, uint8_t* flag) {
    int64_t n = g->n;
    int64_t* fr = (int64_t*)xmalloc((size_t)(n + 1) * sizeof(int64_t));
    int64_t* nx = (int64_t*)xmalloc((size_t)(n + 1) * sizeof(int64_t));
    int64_t nf = 0, rounds = 0;
    for (int64_t v = 0; v < n; ++v)
        if (flag[v]) fr[nf++] = v;
    while (nf) {
        ++rounds;
        int64_t nn = 0;
        for (int64_t k = 0; k < nf; ++k) {
            int64_t v = fr[k];
            FOR_OUT(g, v, t, w, {
                if (!flag[t]) {
                    flag[t] = 1;
                    nx[nn++] = t;
                }
            })
            if (g->directed) {
                FOR_IN(g, v, u, w, {
                    (void)w;
                    if (!flag[u]) {
                        flag[u] = 1;
                        nx[nn++] = u;
                    }
                })
            }
        }
        int64_t* tmp = fr;
        fr = nx;
        nx = tmp;
        nf = nn;
    }
    free(fr);
    free(nx);
    return rounds;
}

/* ------------------------------------------------------------------------ */
/* PageRank: pr_dynamic.sp / pr_dynamic_omp.cc                              */
/* ------------------------------------------------------------------------ */

typedef struct or_pr {
    or_graph* g;
    double damping, beta;
    int64_t maxiter;
    double* rank;
    int64_t* outdeg;
    double* rank_new;
    int64_t sweeps; /* while-loop iterations, summed */
} or_pr;

/* one while-loop of staticPR / incrementalPR (pr_dynamic_omp.cc:27-60,70-100);
 * affected == NULL means every node */
static void pr_loop(or_pr* P, const uint8_t* affected) {
    or_graph* g = P->g;
    int64_t n = g->n;
    int64_t iter = 0;
    double diff = P->beta + 1.0;
    while (diff >= P->beta && iter < P->maxiter) {
        double dangling = 0.0;
        for (int64_t v = 0; v < n; ++v)
            if (P->outdeg[v] == 0) dangling += P->rank[v];
        diff = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            if (affected && !affected[v]) continue;
            double incoming = 0.0;
            FOR_IN(g, v, u, w, {
                (void)w;
                incoming += P->rank[u] / (double)P->outdeg[u];
            })
            double nr = ((1.0 - P->damping) / (double)n) + (P->damping * (incoming + (dangling / (double)n)));
            double delta = nr - P->rank[v];
            if (delta < 0.0) delta = 0.0 - delta;
            if (delta > diff) diff = delta;
            P->rank_new[v] = nr;
        }
        for (int64_t v = 0; v < n; ++v) {
            if (affected && !affected[v]) continue;
            P->rank[v] = P->rank_new[v];
        }
        iter++;
    }
    P->sweeps += iter;
}

int or_pr_create(or_graph* g, double damping, double beta, int64_t maxiter, or_pr** out) {
    if (!g->rev) return fail(OR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
    or_pr* P = (or_pr*)xcalloc(1, sizeof(or_pr));
    int64_t n = g->n;
    P->g = g;
    P->damping = damping;
    P->beta = beta;
    P->maxiter = maxiter;
    P->rank = (double*)xmalloc((size_t)(n ? n : 1) * sizeof(double));
    P->rank_new = (double*)xcalloc((size_t)(n ? n : 1), sizeof(double));
    P->outdeg = (int64_t*)xcalloc((size_t)(n ? n : 1), sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) P->rank[v] = 1.0 / (double)n;
    for (int64_t v = 0; v < n; ++v) {
        int64_t deg = 0;
        FOR_OUT(g, v, t, w, {
            (void)t;
            deg += 1;
        })
        P->outdeg[v] = deg;
    }
    pr_loop(P, NULL);
    *out = P;
    return OR_OK;
}

/* one Batch body of dynamicPR (pr_dynamic_omp.cc:103-138) */
int or_pr_batch(or_pr* P, const uint8_t* kind, const int64_t* s, const int64_t* d, const int64_t* w, int64_t k,
                int64_t batch_index) {
    or_graph* g = P->g;
    int rc = validate(g, kind, s, d, k);
    if (rc) return rc;
    uint8_t* aff = (uint8_t*)xcalloc((size_t)(g->n ? g->n : 1), 1);
    or_recs dl = pick(kind, s, d, w, k, 'd');
    or_recs ad = pick(kind, s, d, w, k, 'a');
    for (int64_t i = 0; i < dl.k; ++i) {
        aff[dl.s[i]] = 1;
        aff[dl.d[i]] = 1;
        P->outdeg[dl.s[i]] -= 1;
    }
    or_graph_delete(g, dl.s, dl.d, dl.k, NULL, NULL, NULL);
    for (int64_t i = 0; i < ad.k; ++i) {
        aff[ad.s[i]] = 1;
        aff[ad.d[i]] = 1;
        P->outdeg[ad.s[i]] += 1;
    }
    or_graph_add(g, ad.s, ad.d, ad.w, ad.k);
    or_propagate_flags(g, aff);
    pr_loop(P, aff);
    if ((batch_index + 1) % g->merge_interval == 0) or_graph_merge(g);
    recs_free(&dl);
    recs_free(&ad);
    free(aff);
    return OR_OK;
}

void or_pr_read(const or_pr* P, double* rank, int64_t* outdeg) {
    memcpy(rank, P->rank, (size_t)P->g->n * sizeof(double));
    if (outdeg) memcpy(outdeg, P->outdeg, (size_t)P->g->n * sizeof(int64_t));
}
int64_t or_pr_sweeps(const or_pr* P) { return P->sweeps; }
void or_pr_free(or_pr* P) {
    if (!P) return;
    free(P->rank);
    free(P->rank_new);
    free(P->outdeg);
    free(P);
}

/* ------------------------------------------------------------------------ */
/* Triangle counting: tc_dynamic.sp / tc_dynamic_omp.cc                     */
/* ------------------------------------------------------------------------ */

typedef struct or_tc {
    or_graph* g;
    int64_t count;
} or_tc;

/* staticTC (tc_dynamic_omp.cc:8-24) */
static int64_t tc_static(or_graph* g) {
    int64_t t = 0;
    for (int64_t v = 0; v < g->n; ++v) {
        FOR_OUT(g, v, a, w1, {
            if (a > v) {
                for (int sg2 = 0; sg2 < g->nseg; ++sg2) {
                    const or_seg* s2 = &g->segs[sg2];
                    for (int64_t j = s2->off[a]; j < s2->off[a + 1]; ++j) {
                        int64_t b = s2->coord[j];
                        if (b == OR_SENT || !(b > a)) continue;
                        FOR_OUT(g, v, c, w3, {
                            if (c == b) t += 1;
                        })
                    }
                }
            }
        })
    }
    return t;
}

/* Per-slot edge marks, as EdgeProp (graphdyn_rt.h:548-589).  Attached at
 * batch start; a claimed slot resets to the default when it is reused
 * (graphdyn_rt.h:573-576), new deltas extend with defaults. */
typedef struct {
    uint8_t** mark;
    int64_t** rank;
    int nseg;
} or_eprop;

static void eprop_attach(or_eprop* p, const or_graph* g) {
    p->nseg = g->nseg;
    p->mark = (uint8_t**)xcalloc((size_t)g->nseg, sizeof(uint8_t*));
    p->rank = (int64_t**)xcalloc((size_t)g->nseg, sizeof(int64_t*));
    for (int i = 0; i < g->nseg; ++i) {
        p->mark[i] = (uint8_t*)xcalloc((size_t)g->segs[i].nslots + 1, 1);
        p->rank[i] = (int64_t*)xcalloc((size_t)g->segs[i].nslots + 1, sizeof(int64_t));
    }
}
static void eprop_free(or_eprop* p) {
    for (int i = 0; i < p->nseg; ++i) {
        free(p->mark[i]);
        free(p->rank[i]);
    }
    free(p->mark);
    free(p->rank);
}

static int64_t pair_rank(int64_t a, int64_t b, int64_t n) {
    return a < b ? sat_add(a * n, b) : sat_add(b * n, a);
}

/* mark every slot holding a batch edge (tc_dynamic_omp.cc:46-66) */
static void tc_mark(or_graph* g, or_eprop* P, const or_recs* R) {
    for (int64_t r = 0; r < R->k; ++r) {
        int64_t u = R->s[r], v = R->d[r];
        int64_t rk = pair_rank(u, v, g->n);
        for (int dir = 0; dir < 2; ++dir) {
            int64_t a = dir ? v : u, b = dir ? u : v;
            for (int sg = 0; sg < g->nseg; ++sg) {
                const or_seg* s = &g->segs[sg];
                for (int64_t i = s->off[a]; i < s->off[a + 1]; ++i)
                    if (s->coord[i] == b) {
                        P->mark[sg][i] = 1;
                        P->rank[sg][i] = rk;
                    }
            }
        }
    }
}

/* count triangles through each batch edge, charged to the smallest-rank batch
 * edge of the triangle (tc_dynamic_omp.cc:67-93) */
static int64_t tc_count(or_graph* g, or_eprop* P, const or_recs* R) {
    int64_t t = 0;
    for (int64_t r = 0; r < R->k; ++r) {
        int64_t u = R->s[r], v = R->d[r];
        int64_t rk = pair_rank(u, v, g->n);
        for (int sg2 = 0; sg2 < g->nseg; ++sg2) {
            const or_seg* s2 = &g->segs[sg2];
            for (int64_t i = s2->off[u]; i < s2->off[u + 1]; ++i) {
                int64_t x = s2->coord[i];
                if (x == OR_SENT || x == v) continue;
                for (int sg3 = 0; sg3 < g->nseg; ++sg3) {
                    const or_seg* s3 = &g->segs[sg3];
                    for (int64_t j = s3->off[v]; j < s3->off[v + 1]; ++j) {
                        if (s3->coord[j] != x) continue;
                        int skip = 0;
                        if (P->mark[sg2][i] && P->rank[sg2][i] < rk) skip = 1;
                        if (P->mark[sg3][j] && P->rank[sg3][j] < rk) skip = 1;
                        if (!skip) t += 1;
                    }
                }
            }
        }
    }
    return t;
}

int or_tc_create(or_graph* g, or_tc** out) {
    or_tc* T = (or_tc*)xcalloc(1, sizeof(or_tc));
    T->g = g;
    T->count = tc_static(g);
    *out = T;
    return OR_OK;
}

/* one Batch body of dynamicTC (tc_dynamic_omp.cc:36-146) */
int or_tc_batch(or_tc* T, const uint8_t* kind, const int64_t* s, const int64_t* d, const int64_t* w, int64_t k,
                int64_t batch_index) {
    or_graph* g = T->g;
    int rc = validate(g, kind, s, d, k);
    if (rc) return rc;
    or_recs dl = pick(kind, s, d, w, k, 'd');
    or_recs ad = pick(kind, s, d, w, k, 'a');
    or_eprop del;
    eprop_attach(&del, g);
    tc_mark(g, &del, &dl);
    T->count -= tc_count(g, &del, &dl);
    eprop_free(&del);
    or_graph_delete(g, dl.s, dl.d, dl.k, NULL, NULL, NULL);
    or_graph_add(g, ad.s, ad.d, ad.w, ad.k);
    or_eprop add; /* attached after the update: reused slots read as default */
    eprop_attach(&add, g);
    tc_mark(g, &add, &ad);
    T->count += tc_count(g, &add, &ad);
    eprop_free(&add);
    if ((batch_index + 1) % g->merge_interval == 0) or_graph_merge(g);
    recs_free(&dl);
    recs_free(&ad);
    return OR_OK;
}

int64_t or_tc_read(const or_tc* T) { return T->count; }
void or_tc_free(or_tc* T) { free(T); }
