/*
 * oracle.c — CPU restatement of the reference resharding path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Never linked into the product; the
 * product (paper_2605_18815_b200/csrc) is an independent C++/CUDA implementation.
 *
 * Planner functions restate /root/reference/proj/include/reshard/ headers; every
 * function cites the file:line it follows. Differences are only in data
 * structures and complexity: interval set operations use linear / binary-search
 * sweeps instead of the reference's O(n*m) loops (region.hpp:126-158), which is
 * safe because normalized interval lists are a unique normal form of a set.
 * Box set operations keep the reference's exact algorithm (order-sensitive).
 *
 * Executor / verify / oracle_reshard restate SPEC.md:346-426 (no reference code).
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <pthread.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ basics */

typedef struct { int64_t lo, hi; } iv_t;
typedef struct { iv_t d[4]; } box_t;
typedef struct { box_t* v; int n, cap; } blist;
typedef struct { iv_t* v; int64_t n, cap; } ilist;

typedef struct {
    char id[128];
    int nd;
    int64_t shape[4];
    int layer, tp_axis, expert_axis, dtype;
    int64_t off, numel;
} tens_t;

typedef struct {
    int dp, tp, pp, ep, zero;
    char order_str[64];
} cfg_t;

struct or_scenario {
    tens_t* t;
    int nt, layers, experts;
    int64_t total;
    uint64_t fp;
    int* by_id; /* tensor indices sorted by id (std::map<std::string,...> order) */
    cfg_t src, dst;
    int *src_phys, *dst_phys;
    int nsrc, ndst, has_world;
    int nodes, rpn;
    int migrate, balance;
    int64_t scalar_words;
};

typedef struct {
    jmp_buf jb;
    char msg[512];
} ctx_t;

static void fail(ctx_t* c, int code, const char* fmt, ...) {
    va_list a;
    va_start(a, fmt);
    vsnprintf(c->msg, sizeof c->msg, fmt, a);
    va_end(a);
    longjmp(c->jb, code);
}

static void* xrealloc(void* p, size_t n) {
    void* q = realloc(p, n ? n : 1);
    if (!q) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return q;
}

static void bl_push(blist* l, const box_t* b) {
    if (l->n == l->cap) { l->cap = l->cap ? 2 * l->cap : 4; l->v = xrealloc(l->v, sizeof(box_t) * l->cap); }
    l->v[l->n++] = *b;
}
static void il_push(ilist* l, int64_t lo, int64_t hi) {
    if (l->n == l->cap) { l->cap = l->cap ? 2 * l->cap : 16; l->v = xrealloc(l->v, sizeof(iv_t) * l->cap); }
    l->v[l->n].lo = lo;
    l->v[l->n].hi = hi;
    l->n++;
}
static void bl_free(blist* l) { free(l->v); l->v = NULL; l->n = l->cap = 0; }
static void il_free(ilist* l) { free(l->v); l->v = NULL; l->n = l->cap = 0; }

/* common.hpp:66-72 splitmix64 finalizer; common.hpp:77-80 canon_value */
static uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
uint64_t or_canon(uint64_t seed, int64_t element, int kind) {
    return mix64(mix64(seed ^ (uint64_t)element * 0xD6E8FEB86659FD93ull) ^
                 ((uint64_t)kind + 1) * 0xA5A5A5A5A5A5A5A5ull);
}

/* ------------------------------------------------------------ interval ops */

static int iv_cmp(const void* a, const void* b) {
    const iv_t *x = a, *y = b;
    if (x->lo != y->lo) return x->lo < y->lo ? -1 : 1;
    if (x->hi != y->hi) return x->hi < y->hi ? -1 : 1;
    return 0;
}

/* region.hpp:104-117 normalize_intervals: drop empties, sort, merge runs with
 * lo <= back.hi (overlapping or abutting). In place. */
static void il_normalize(ilist* l) {
    int64_t w = 0;
    for (int64_t i = 0; i < l->n; ++i)
        if (l->v[i].lo < l->v[i].hi) l->v[w++] = l->v[i];
    l->n = w;
    if (w > 1) qsort(l->v, (size_t)w, sizeof(iv_t), iv_cmp);
    int64_t o = 0;
    for (int64_t i = 0; i < l->n; ++i) {
        if (o > 0 && l->v[i].lo <= l->v[o - 1].hi) {
            if (l->v[i].hi > l->v[o - 1].hi) l->v[o - 1].hi = l->v[i].hi;
        } else {
            l->v[o++] = l->v[i];
        }
    }
    l->n = o;
}

/* region.hpp:126-135 intervals_intersect, as a two-pointer sweep over normalized inputs */
static ilist il_intersect(const ilist* a, const ilist* b) {
    ilist out = {0};
    int64_t i = 0, j = 0;
    while (i < a->n && j < b->n) {
        int64_t lo = a->v[i].lo > b->v[j].lo ? a->v[i].lo : b->v[j].lo;
        int64_t hi = a->v[i].hi < b->v[j].hi ? a->v[i].hi : b->v[j].hi;
        if (lo < hi) il_push(&out, lo, hi);
        if (a->v[i].hi < b->v[j].hi) ++i; else ++j;
    }
    il_normalize(&out);
    return out;
}

/* region.hpp:137-158 intervals_diff (a \ b) as a sweep over normalized inputs */
static ilist il_diff(const ilist* a, const ilist* b) {
    ilist out = {0};
    int64_t j = 0;
    for (int64_t i = 0; i < a->n; ++i) {
        int64_t cur = a->v[i].lo, end = a->v[i].hi;
        while (j < b->n && b->v[j].hi <= cur) ++j;
        int64_t k = j;
        while (cur < end) {
            if (k >= b->n || b->v[k].lo >= end) { il_push(&out, cur, end); break; }
            if (b->v[k].lo > cur) il_push(&out, cur, b->v[k].lo);
            if (b->v[k].hi > cur) cur = b->v[k].hi;
            ++k;
        }
    }
    il_normalize(&out);
    return out;
}

/* pieces of normalized list a inside [lo,hi): binary search + scan
 * (the single-interval case of region.hpp:126-135 used at routing.hpp:323) */
static int64_t il_lower(const ilist* a, int64_t lo) {
    int64_t L = 0, R = a->n;
    while (L < R) {
        int64_t m = (L + R) / 2;
        if (a->v[m].hi <= lo) L = m + 1; else R = m;
    }
    return L;
}

static int64_t il_length(const ilist* l) {
    int64_t n = 0;
    for (int64_t i = 0; i < l->n; ++i) n += l->v[i].hi - l->v[i].lo;
    return n;
}

/* ------------------------------------------------------------------ box ops */

static int box_empty(const box_t* b, int nd) {
    if (nd == 0) return 1;
    for (int i = 0; i < nd; ++i)
        if (b->d[i].lo >= b->d[i].hi) return 1;
    return 0;
}
static int64_t box_numel(const box_t* b, int nd) {
    int64_t n = 1;
    for (int i = 0; i < nd; ++i) n *= (b->d[i].hi > b->d[i].lo ? b->d[i].hi - b->d[i].lo : 0);
    return nd ? n : 0;
}
static box_t box_isect(const box_t* a, const box_t* b, int nd) {
    box_t r;
    memset(&r, 0, sizeof r);
    for (int i = 0; i < nd; ++i) {
        r.d[i].lo = a->d[i].lo > b->d[i].lo ? a->d[i].lo : b->d[i].lo;
        r.d[i].hi = a->d[i].hi < b->d[i].hi ? a->d[i].hi : b->d[i].hi;
    }
    return r;
}
/* Box operator<=> (region.hpp:63): lexicographic over dims, Interval by (lo,hi) */
static int box_cmp_nd(const box_t* a, const box_t* b, int nd) {
    for (int i = 0; i < nd; ++i) {
        if (a->d[i].lo != b->d[i].lo) return a->d[i].lo < b->d[i].lo ? -1 : 1;
        if (a->d[i].hi != b->d[i].hi) return a->d[i].hi < b->d[i].hi ? -1 : 1;
    }
    return 0;
}
static int g_sort_nd;
static int box_cmp_q(const void* a, const void* b) { return box_cmp_nd(a, b, g_sort_nd); }
static void box_sort(blist* l, int nd) {
    g_sort_nd = nd;
    /* insertion sort: stable and tiny lists; std::sort result is the same since keys are unique */
    for (int i = 1; i < l->n; ++i) {
        box_t x = l->v[i];
        int j = i - 1;
        while (j >= 0 && box_cmp_nd(&l->v[j], &x, nd) > 0) { l->v[j + 1] = l->v[j]; --j; }
        l->v[j + 1] = x;
    }
    (void)box_cmp_q;
}

/* region.hpp:79-100 box_diff: a \ b by per-axis carve, pieces in carve order */
static void box_diff(const box_t* a, const box_t* b, int nd, blist* out) {
    if (box_empty(a, nd)) return;
    box_t ov = box_isect(a, b, nd);
    if (box_empty(&ov, nd)) { bl_push(out, a); return; }
    box_t cur = *a;
    for (int d = 0; d < nd; ++d) {
        iv_t o = ov.d[d];
        if (cur.d[d].lo < o.lo) { box_t p = cur; p.d[d].hi = o.lo; bl_push(out, &p); }
        if (o.hi < cur.d[d].hi) { box_t p = cur; p.d[d].lo = o.hi; bl_push(out, &p); }
        cur.d[d] = o;
    }
}

/* region.hpp:172-213 normalize_boxes: disjoint-ify against earlier boxes, sort,
 * coalesce the first pair (i<j) equal on all axes but one and abutting there,
 * re-sort, repeat to fixpoint. Consumes `in`. */
static blist normalize_boxes(blist* in_list, int nd) {
    blist acc = {0};
    for (int i = 0; i < in_list->n; ++i) {
        if (box_empty(&in_list->v[i], nd)) continue;
        blist pieces = {0};
        bl_push(&pieces, &in_list->v[i]);
        for (int h = 0; h < acc.n; ++h) {
            blist next = {0};
            for (int p = 0; p < pieces.n; ++p) box_diff(&pieces.v[p], &acc.v[h], nd, &next);
            bl_free(&pieces);
            pieces = next;
        }
        for (int p = 0; p < pieces.n; ++p) bl_push(&acc, &pieces.v[p]);
        bl_free(&pieces);
    }
    bl_free(in_list);
    box_sort(&acc, nd);
    int merged = 1;
    while (merged) {
        merged = 0;
        for (int i = 0; i < acc.n && !merged; ++i) {
            for (int j = i + 1; j < acc.n && !merged; ++j) {
                int axis = -1, ok = 1;
                for (int d = 0; d < nd; ++d) {
                    if (acc.v[i].d[d].lo == acc.v[j].d[d].lo && acc.v[i].d[d].hi == acc.v[j].d[d].hi) continue;
                    if (axis >= 0) { ok = 0; break; }
                    axis = d;
                }
                if (!ok || axis < 0) continue;
                iv_t x = acc.v[i].d[axis], y = acc.v[j].d[axis];
                if (x.hi == y.lo || y.hi == x.lo) {
                    acc.v[i].d[axis].lo = x.lo < y.lo ? x.lo : y.lo;
                    acc.v[i].d[axis].hi = x.hi > y.hi ? x.hi : y.hi;
                    memmove(&acc.v[j], &acc.v[j + 1], sizeof(box_t) * (size_t)(acc.n - j - 1));
                    acc.n--;
                    box_sort(&acc, nd);
                    merged = 1;
                }
            }
        }
    }
    return acc;
}

static blist bl_copy(const blist* a) {
    blist r = {0};
    for (int i = 0; i < a->n; ++i) bl_push(&r, &a->v[i]);
    return r;
}

/* region.hpp:215-226 boxes_diff */
static blist boxes_diff(const blist* a, const blist* b, int nd) {
    blist rem = bl_copy(a);
    for (int y = 0; y < b->n; ++y) {
        blist next = {0};
        for (int r = 0; r < rem.n; ++r) box_diff(&rem.v[r], &b->v[y], nd, &next);
        bl_free(&rem);
        rem = next;
    }
    return normalize_boxes(&rem, nd);
}

/* region.hpp:228-237 boxes_intersect */
static blist boxes_intersect(const blist* a, const blist* b, int nd) {
    blist out = {0};
    for (int x = 0; x < a->n; ++x)
        for (int y = 0; y < b->n; ++y) {
            box_t i = box_isect(&a->v[x], &b->v[y], nd);
            if (!box_empty(&i, nd)) bl_push(&out, &i);
        }
    return normalize_boxes(&out, nd);
}

/* --------------------------------------------------------------- RegionSet */

/* region.hpp:252-289: per-tensor box lists (index = tensor) + flat intervals */
typedef struct {
    blist* tb;
    ilist flat;
    int nt;
} region_t;

static region_t rg_new(int nt) {
    region_t r;
    r.nt = nt;
    r.tb = calloc((size_t)nt, sizeof(blist));
    memset(&r.flat, 0, sizeof r.flat);
    return r;
}
static void rg_free(region_t* r) {
    if (r->tb)
        for (int i = 0; i < r->nt; ++i) bl_free(&r->tb[i]);
    free(r->tb);
    r->tb = NULL;
    il_free(&r->flat);
}
static region_t rg_copy(const region_t* a) {
    region_t r = rg_new(a->nt);
    for (int i = 0; i < a->nt; ++i) r.tb[i] = bl_copy(&a->tb[i]);
    for (int64_t i = 0; i < a->flat.n; ++i) il_push(&r.flat, a->flat.v[i].lo, a->flat.v[i].hi);
    return r;
}

/* region.hpp:311-323 region_diff */
static region_t rg_diff(const or_scenario* s, const region_t* a, const region_t* b) {
    region_t r = rg_new(s->nt);
    for (int t = 0; t < s->nt; ++t) {
        if (a->tb[t].n == 0) continue;
        if (b->tb[t].n == 0) {
            blist c = bl_copy(&a->tb[t]);
            r.tb[t] = normalize_boxes(&c, s->t[t].nd);
        } else {
            r.tb[t] = boxes_diff(&a->tb[t], &b->tb[t], s->t[t].nd);
        }
    }
    r.flat = il_diff(&a->flat, &b->flat);
    return r;
}

/* region.hpp:297-309 region_intersect */
static region_t rg_intersect(const or_scenario* s, const region_t* a, const region_t* b) {
    region_t r = rg_new(s->nt);
    for (int t = 0; t < s->nt; ++t) {
        if (a->tb[t].n == 0 || b->tb[t].n == 0) continue;
        r.tb[t] = boxes_intersect(&a->tb[t], &b->tb[t], s->t[t].nd);
    }
    r.flat = il_intersect(&a->flat, &b->flat);
    return r;
}

/* region.hpp:345-352 region_contains_box */
static int rg_contains_box(const or_scenario* s, const region_t* r, int t, const box_t* box) {
    if (r->tb[t].n == 0) return box_empty(box, s->t[t].nd);
    blist one = {0};
    bl_push(&one, box);
    blist rem = boxes_diff(&one, &r->tb[t], s->t[t].nd);
    bl_free(&one);
    int contained = rem.n == 0;
    bl_free(&rem);
    return contained;
}

/* ----------------------------------------------------------------- parsing */

static int parse_list(const char* s, int64_t* out, int maxn) {
    int n = 0;
    while (*s) {
        if (n == maxn) return -1;
        char* end;
        out[n++] = strtoll(s, &end, 10);
        if (end == s) return -1;
        s = end;
        if (*s == ',') ++s;
        else if (*s) return -1;
    }
    return n;
}

static int parse_cfg(char** tok, int ntok, cfg_t* c) {
    c->dp = c->tp = c->pp = c->ep = 1;
    c->zero = 0;
    strcpy(c->order_str, "pp-dp-tp");
    for (int i = 1; i < ntok; ++i) {
        char* eq = strchr(tok[i], '=');
        if (!eq) return -1;
        *eq = 0;
        const char *k = tok[i], *v = eq + 1;
        if (!strcmp(k, "dp")) c->dp = atoi(v);
        else if (!strcmp(k, "tp")) c->tp = atoi(v);
        else if (!strcmp(k, "pp")) c->pp = atoi(v);
        else if (!strcmp(k, "ep")) c->ep = atoi(v);
        else if (!strcmp(k, "zero")) c->zero = atoi(v) != 0;
        else if (!strcmp(k, "order")) { snprintf(c->order_str, sizeof c->order_str, "%s", v); }
        else return -1;
    }
    return 0;
}

static const char* g_sort_names_base;
static or_scenario* g_sort_scn;
static int id_cmp(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return strcmp(g_sort_scn->t[x].id, g_sort_scn->t[y].id);
}

static int parse_phys(const char* v, int** out) {
    int64_t tmp[4096];
    int n = 0;
    if (*v) {
        n = parse_list(v, tmp, 4096);
        if (n < 0) return -1;
    }
    *out = xrealloc(NULL, sizeof(int) * (size_t)(n ? n : 1));
    for (int i = 0; i < n; ++i) (*out)[i] = (int)tmp[i];
    return n;
}

/* Scenario text (format documented in DESIGN.md §5); model invariants per
 * model.hpp:95-123 validate_model, offsets and fingerprint per model.hpp:127-144. */
or_scenario* or_scenario_parse(const char* text, char* err, size_t errlen) {
    or_scenario* s = calloc(1, sizeof *s);
    s->layers = 1;
    s->experts = 1;
    s->nodes = 1;
    s->rpn = 8;
    s->scalar_words = 8;
    s->src.dp = s->src.tp = s->src.pp = s->src.ep = 1;
    s->dst = s->src;
    strcpy(s->src.order_str, "pp-dp-tp");
    strcpy(s->dst.order_str, "pp-dp-tp");
    int cap = 0;
    char* buf = strdup(text);
    char* save = NULL;
    int lineno = 0;
#define PERR(...) do { snprintf(err, errlen, __VA_ARGS__); free(buf); or_scenario_free(s); return NULL; } while (0)
    for (char* line = strtok_r(buf, "\n", &save); line; line = strtok_r(NULL, "\n", &save)) {
        ++lineno;
        char* tok[32];
        int ntok = 0;
        char* sv = NULL;
        for (char* w = strtok_r(line, " \t\r", &sv); w && ntok < 32; w = strtok_r(NULL, " \t\r", &sv)) tok[ntok++] = w;
        if (ntok == 0 || tok[0][0] == '#') continue;
        if (!strcmp(tok[0], "version")) continue;
        if (!strcmp(tok[0], "seed")) continue;
        if (!strcmp(tok[0], "model")) {
            for (int i = 1; i < ntok; ++i) {
                if (!strncmp(tok[i], "layers=", 7)) s->layers = atoi(tok[i] + 7);
                else if (!strncmp(tok[i], "experts=", 8)) s->experts = atoi(tok[i] + 8);
                else PERR("line %d: bad model key '%s'", lineno, tok[i]);
            }
        } else if (!strcmp(tok[0], "tensor")) {
            if (ntok < 3) PERR("line %d: tensor needs id and shape", lineno);
            if (s->nt == cap) { cap = cap ? 2 * cap : 64; s->t = xrealloc(s->t, sizeof(tens_t) * (size_t)cap); }
            tens_t* t = &s->t[s->nt++];
            memset(t, 0, sizeof *t);
            snprintf(t->id, sizeof t->id, "%s", tok[1]);
            int nd = parse_list(tok[2], t->shape, 4);
            if (nd <= 0) PERR("line %d: bad shape '%s'", lineno, tok[2]);
            t->nd = nd;
            t->tp_axis = -1;
            t->expert_axis = -1;
            t->dtype = 2;
            for (int i = 3; i < ntok; ++i) {
                char* eq = strchr(tok[i], '=');
                if (!eq) PERR("line %d: bad tensor attribute '%s'", lineno, tok[i]);
                *eq = 0;
                if (!strcmp(tok[i], "layer")) t->layer = atoi(eq + 1);
                else if (!strcmp(tok[i], "tp")) t->tp_axis = atoi(eq + 1);
                else if (!strcmp(tok[i], "expert")) t->expert_axis = atoi(eq + 1);
                else if (!strcmp(tok[i], "dtype")) t->dtype = atoi(eq + 1);
                else PERR("line %d: bad tensor attribute '%s'", lineno, tok[i]);
            }
        } else if (!strcmp(tok[0], "src") || !strcmp(tok[0], "dst")) {
            if (parse_cfg(tok, ntok, tok[0][0] == 's' ? &s->src : &s->dst)) PERR("line %d: bad config", lineno);
        } else if (!strcmp(tok[0], "world")) {
            s->has_world = 1;
            for (int i = 1; i < ntok; ++i) {
                if (!strncmp(tok[i], "src=", 4)) { s->nsrc = parse_phys(tok[i] + 4, &s->src_phys); if (s->nsrc < 0) PERR("line %d: bad world", lineno); }
                else if (!strncmp(tok[i], "dst=", 4)) { s->ndst = parse_phys(tok[i] + 4, &s->dst_phys); if (s->ndst < 0) PERR("line %d: bad world", lineno); }
                else PERR("line %d: bad world key", lineno);
            }
        } else if (!strcmp(tok[0], "topology")) {
            for (int i = 1; i < ntok; ++i) {
                if (!strncmp(tok[i], "nodes=", 6)) s->nodes = atoi(tok[i] + 6);
                else if (!strncmp(tok[i], "rpn=", 4)) s->rpn = atoi(tok[i] + 4);
                else PERR("line %d: bad topology key", lineno);
            }
        } else if (!strcmp(tok[0], "options")) {
            for (int i = 1; i < ntok; ++i) {
                if (!strcmp(tok[i], "grads=drop")) s->migrate = 0;
                else if (!strcmp(tok[i], "grads=migrate")) s->migrate = 1;
                else if (!strncmp(tok[i], "balance=", 8)) s->balance = atoi(tok[i] + 8) != 0;
                else if (!strncmp(tok[i], "scalar_words=", 13)) s->scalar_words = atoll(tok[i] + 13);
                else PERR("line %d: bad option '%s'", lineno, tok[i]);
            }
        } else {
            PERR("line %d: unknown keyword '%s'", lineno, tok[0]);
        }
    }
    free(buf);
    buf = NULL;
    /* model.hpp:95-123 validate_model */
    if (s->layers < 1) PERR("num_layers must be positive");
    if (s->experts < 1) PERR("num_experts must be positive");
    for (int i = 0; i < s->nt; ++i) {
        tens_t* t = &s->t[i];
        for (int j = 0; j < i; ++j)
            if (!strcmp(s->t[j].id, t->id)) PERR("duplicate tensor_id '%s'", t->id);
        for (int d = 0; d < t->nd; ++d)
            if (t->shape[d] < 1) PERR("tensor '%s' has zero extent", t->id);
        if (t->layer < 0 || t->layer >= s->layers) PERR("tensor '%s' layer out of range", t->id);
        if (t->tp_axis >= t->nd || t->tp_axis < -1) PERR("tensor '%s' tp_shard_axis out of range", t->id);
        if (t->expert_axis >= 0) {
            if (t->expert_axis >= t->nd) PERR("tensor '%s' expert_axis out of range", t->id);
            if (t->tp_axis >= 0 && t->tp_axis == t->expert_axis) PERR("tensor '%s' expert_axis equals tp_shard_axis", t->id);
            if (t->shape[t->expert_axis] != s->experts) PERR("tensor '%s' expert extent != num_experts", t->id);
        }
        if (t->dtype < 1) PERR("tensor '%s' dtype_bytes must be positive", t->id);
    }
    /* model.hpp:127-144 build_model_space: declaration-order offsets, FNV-1a fingerprint */
    uint64_t fp = 0xcbf29ce484222325ull;
#define FEED(v) (fp = (fp ^ (uint64_t)(v)) * 0x100000001b3ull)
    int64_t off = 0;
    for (int i = 0; i < s->nt; ++i) {
        tens_t* t = &s->t[i];
        t->off = off;
        t->numel = 1;
        for (int d = 0; d < t->nd; ++d) t->numel *= t->shape[d];
        off += t->numel;
        for (const char* c = t->id; *c; ++c) FEED((unsigned char)*c);
        for (int d = 0; d < t->nd; ++d) FEED(t->shape[d]);
        FEED(t->layer);
    }
    FEED(s->layers);
    FEED(s->experts);
#undef FEED
    s->total = off;
    s->fp = fp;
    s->by_id = xrealloc(NULL, sizeof(int) * (size_t)(s->nt > 0 ? s->nt : 1));
    for (int i = 0; i < s->nt; ++i) s->by_id[i] = i;
    g_sort_scn = s;
    (void)g_sort_names_base;
    if (s->nt > 1) qsort(s->by_id, (size_t)s->nt, sizeof(int), id_cmp);
    return s;
#undef PERR
}

void or_scenario_free(or_scenario* s) {
    if (!s) return;
    free(s->t);
    free(s->by_id);
    free(s->src_phys);
    free(s->dst_phys);
    free(s);
}
int or_scenario_num_tensors(const or_scenario* s) { return s->nt; }
const char* or_scenario_tensor_id(const or_scenario* s, int t) { return s->t[t].id; }
int64_t or_scenario_total_numel(const or_scenario* s) { return s->total; }
uint64_t or_scenario_fingerprint(const or_scenario* s) { return s->fp; }
void or_free(void* p) { free(p); }

/* --------------------------------------------------- parallel coordinates */

typedef struct { int pp, dp, tp, ep, edp; } coord_t;

/* parallel.hpp:61-84 order_axes (same token loop, same acceptance quirks) */
static void order_axes(ctx_t* c, const cfg_t* cfg, char tags[3], int deg[3]) {
    const char* o = cfg->order_str;
    size_t len = strlen(o), pos = 0;
    int found = 0;
    while (pos < len && found < 3) {
        const char* dash = strchr(o + pos, '-');
        size_t tl = dash ? (size_t)(dash - (o + pos)) : len - pos;
        char tok[64];
        if (tl >= sizeof tok) tl = sizeof tok - 1;
        memcpy(tok, o + pos, tl);
        tok[tl] = 0;
        if (!strcmp(tok, "pp")) { tags[found] = 'p'; deg[found] = cfg->pp; }
        else if (!strcmp(tok, "dp")) { tags[found] = 'd'; deg[found] = cfg->dp; }
        else if (!strcmp(tok, "tp")) { tags[found] = 't'; deg[found] = cfg->tp; }
        else fail(c, 2, "bad rank_order token '%s'", tok);
        ++found;
        pos = dash ? (size_t)(dash - o) + 1 : len;
    }
    if (found != 3 || pos != len) fail(c, 2, "rank_order must name pp, dp and tp exactly once: '%s'", o);
    if (tags[0] == tags[1] || tags[1] == tags[2] || tags[0] == tags[2]) fail(c, 2, "rank_order repeats a dimension: '%s'", o);
}

static int world_size(const cfg_t* c) { return c->dp * c->tp * c->pp; }

/* parallel.hpp:88-106 rank_coord */
static coord_t rank_coord(ctx_t* c, const cfg_t* cfg, int rank) {
    if (rank < 0 || rank >= world_size(cfg)) fail(c, 2, "rank %d out of range (world %d)", rank, world_size(cfg));
    char tags[3];
    int deg[3];
    order_axes(c, cfg, tags, deg);
    coord_t k = {0, 0, 0, 0, 0};
    int rem = rank;
    for (int i = 2; i >= 0; --i) {
        int v = rem % deg[i];
        rem /= deg[i];
        if (tags[i] == 'p') k.pp = v;
        else if (tags[i] == 'd') k.dp = v;
        else k.tp = v;
    }
    k.ep = k.dp % cfg->ep;
    k.edp = k.dp / cfg->ep;
    return k;
}

/* parallel.hpp:120-126 stage_layer_range (remainder-first) */
static void stage_range(int layers, int pp, int r, int* lo, int* hi) {
    int base = layers / pp, extra = layers % pp;
    *lo = r * base + (r < extra ? r : extra);
    *hi = *lo + base + (r < extra ? 1 : 0);
}

/* parallel.hpp:130-146 validate_config */
static void validate_config(ctx_t* c, const or_scenario* s, const cfg_t* cfg) {
    if (cfg->dp < 1 || cfg->tp < 1 || cfg->pp < 1 || cfg->ep < 1)
        fail(c, 2, "parallel degrees must be positive: dp=%d tp=%d pp=%d ep=%d", cfg->dp, cfg->tp, cfg->pp, cfg->ep);
    char tags[3];
    int deg[3];
    order_axes(c, cfg, tags, deg);
    if (cfg->dp % cfg->ep != 0) fail(c, 2, "ep=%d does not divide dp=%d", cfg->ep, cfg->dp);
    if (s->experts % cfg->ep != 0) fail(c, 2, "ep=%d does not divide num_experts=%d", cfg->ep, s->experts);
    if (cfg->pp > s->layers) fail(c, 2, "pp=%d exceeds num_layers=%d", cfg->pp, s->layers);
    for (int i = 0; i < s->nt; ++i) {
        const tens_t* t = &s->t[i];
        if (t->tp_axis >= 0 && t->shape[t->tp_axis] % cfg->tp != 0)
            fail(c, 2, "tp=%d does not divide extent %lld of tensor '%s'", cfg->tp, (long long)t->shape[t->tp_axis], t->id);
    }
}

/* --------------------------------------------------------------- projection */

/* project.hpp:44-74 project: PP visibility, TP slice, expert block, DP replicate */
static region_t project(ctx_t* c, const or_scenario* s, const cfg_t* cfg, int rank) {
    coord_t k = rank_coord(c, cfg, rank);
    int lo, hi;
    stage_range(s->layers, cfg->pp, k.pp, &lo, &hi);
    region_t r = rg_new(s->nt);
    for (int i = 0; i < s->nt; ++i) {
        const tens_t* t = &s->t[i];
        if (t->layer < lo || t->layer >= hi) continue;
        box_t b;
        memset(&b, 0, sizeof b);
        for (int d = 0; d < t->nd; ++d) { b.d[d].lo = 0; b.d[d].hi = t->shape[d]; }
        if (t->tp_axis >= 0) {
            int64_t ext = t->shape[t->tp_axis];
            if (ext % cfg->tp != 0)
                fail(c, 2, "tp=%d does not divide extent %lld of tensor '%s'", cfg->tp, (long long)ext, t->id);
            int64_t w = ext / cfg->tp;
            b.d[t->tp_axis].lo = k.tp * w;
            b.d[t->tp_axis].hi = (k.tp + 1) * w;
        }
        if (t->expert_axis >= 0) {
            if (s->experts % cfg->ep != 0) fail(c, 2, "ep=%d does not divide num_experts=%d", cfg->ep, s->experts);
            int64_t w = s->experts / cfg->ep;
            b.d[t->expert_axis].lo = k.ep * w;
            b.d[t->expert_axis].hi = (k.ep + 1) * w;
        }
        bl_push(&r.tb[i], &b);
    }
    return r;
}

/* project.hpp:77-112 LocalSegment / local_layout: visible boxes in declaration
 * order, dense span and expert span indexed separately */
typedef struct {
    int t;
    box_t box;
    int64_t lo, hi;
} seg_t;
typedef struct {
    seg_t* dense;
    seg_t* expert;
    int nd_, ne_;
    int64_t dense_len, expert_len;
} layout_t;

static layout_t local_layout(ctx_t* c, const or_scenario* s, const cfg_t* cfg, int rank) {
    region_t r = project(c, s, cfg, rank);
    layout_t L;
    memset(&L, 0, sizeof L);
    L.dense = xrealloc(NULL, sizeof(seg_t) * (size_t)(s->nt + 1));
    L.expert = xrealloc(NULL, sizeof(seg_t) * (size_t)(s->nt + 1));
    for (int i = 0; i < s->nt; ++i) {
        for (int b = 0; b < r.tb[i].n; ++b) {
            int64_t n = box_numel(&r.tb[i].v[b], s->t[i].nd);
            if (s->t[i].expert_axis >= 0) {
                L.expert[L.ne_++] = (seg_t){i, r.tb[i].v[b], L.expert_len, L.expert_len + n};
                L.expert_len += n;
            } else {
                L.dense[L.nd_++] = (seg_t){i, r.tb[i].v[b], L.dense_len, L.dense_len + n};
                L.dense_len += n;
            }
        }
    }
    rg_free(&r);
    return L;
}
static void layout_free(layout_t* L) { free(L->dense); free(L->expert); }

/* project.hpp:118-124 shard_range: ceil chunk, trailing shard truncated */
static iv_t shard_range(int64_t len, int parts, int index) {
    iv_t r = {0, 0};
    if (len == 0) return r;
    int64_t chunk = (len + parts - 1) / parts;
    r.lo = (int64_t)index * chunk < len ? (int64_t)index * chunk : len;
    r.hi = r.lo + chunk < len ? r.lo + chunk : len;
    return r;
}

/* region.hpp:391-417 box_subrange_flat_runs: [a,b) of the box's row-major
 * enumeration as global flat runs (one per box row), appended to out */
static void box_subrange_runs(const or_scenario* s, int ti, const box_t* box, int64_t a0, int64_t b0, ilist* out) {
    const tens_t* t = &s->t[ti];
    int d = t->nd;
    if (box_empty(box, d) || a0 >= b0) return;
    int64_t stride[4];
    stride[d - 1] = 1;
    for (int i = d - 1; i > 0; --i) stride[i - 1] = stride[i] * t->shape[i];
    int64_t width = box->d[d - 1].hi - box->d[d - 1].lo;
    for (int64_t row = a0 / width; row * width < b0; ++row) {
        int64_t a = a0 - row * width > 0 ? a0 - row * width : 0;
        int64_t b = b0 - row * width < width ? b0 - row * width : width;
        if (a >= b) continue;
        int64_t rem = row, base = t->off + box->d[d - 1].lo;
        for (int i = d - 1; i-- > 0;) {
            int64_t len = box->d[i].hi - box->d[i].lo;
            base += (box->d[i].lo + rem % len) * stride[i];
            rem /= len;
        }
        il_push(out, base + a, base + b);
    }
}

/* project.hpp:126-135 invert_segments */
static void invert_segments(const or_scenario* s, const seg_t* segs, int n, iv_t shard, ilist* out) {
    for (int i = 0; i < n; ++i) {
        int64_t lo = segs[i].lo > shard.lo ? segs[i].lo : shard.lo;
        int64_t hi = segs[i].hi < shard.hi ? segs[i].hi : shard.hi;
        if (lo >= hi) continue;
        box_subrange_runs(s, segs[i].t, &segs[i].box, lo - segs[i].lo, hi - segs[i].lo, out);
    }
}

/* project.hpp:146-159 project_optimizer */
static region_t project_optimizer(ctx_t* c, const or_scenario* s, const cfg_t* cfg, int rank) {
    if (!cfg->zero) fail(c, 2, "no sharded optimizer: zero_enabled is false");
    coord_t k = rank_coord(c, cfg, rank);
    layout_t L = local_layout(c, s, cfg, rank);
    region_t r = rg_new(s->nt);
    invert_segments(s, L.dense, L.nd_, shard_range(L.dense_len, cfg->dp, k.dp), &r.flat);
    int edp = cfg->dp / cfg->ep;
    invert_segments(s, L.expert, L.ne_, shard_range(L.expert_len, edp, k.edp), &r.flat);
    il_normalize(&r.flat);
    layout_free(&L);
    return r;
}

/* project.hpp:174-196 split_by_projection_grid */
static void split_axis(blist* cells, int axis, int64_t width) {
    blist next = {0};
    for (int i = 0; i < cells->n; ++i) {
        iv_t iv = cells->v[i].d[axis];
        for (int64_t cut = (iv.lo / width) * width; cut < iv.hi; cut += width) {
            int64_t lo = iv.lo > cut ? iv.lo : cut;
            int64_t hi = iv.hi < cut + width ? iv.hi : cut + width;
            if (lo >= hi) continue;
            box_t nb = cells->v[i];
            nb.d[axis].lo = lo;
            nb.d[axis].hi = hi;
            bl_push(&next, &nb);
        }
    }
    bl_free(cells);
    *cells = next;
}
static blist split_by_projection_grid(const or_scenario* s, const cfg_t* cfg, int ti, const box_t* box) {
    const tens_t* t = &s->t[ti];
    blist cells = {0};
    bl_push(&cells, box);
    if (t->tp_axis >= 0) split_axis(&cells, t->tp_axis, t->shape[t->tp_axis] / cfg->tp);
    if (t->expert_axis >= 0) split_axis(&cells, t->expert_axis, s->experts / cfg->ep);
    return cells;
}

/* ------------------------------------------------------------------ planner */

typedef struct {
    region_t src, dst, send, recv, retain;
} catset_t;

typedef struct {
    int phys, src_rank, dst_rank;
    catset_t params, optim;
} route_t;

typedef struct {
    int kind, t, flat;
    box_t box;
    iv_t iv;
    int dst_phys, dst_rank;
    int64_t cand_off;
    int ncand;
} pending_t;

struct or_plan {
    const or_scenario* s;
    route_t* routes;
    int nroutes;
    pending_t* pend;
    int64_t npend, pcap;
    int* cands;
    int64_t ncands, ccap;
    or_transfer* tr;
    int64_t ntr;
    int has_scalars;
    int root_phys;
    int nscalar_recv;
    int* scalar_recv;
    int64_t scalar_bytes_per_rank;
    int* src_phys;
    int* dst_phys;
    int nsrc, ndst;
};

static void push_pending(or_plan* p, int kind, int t, int flat, const box_t* box, iv_t iv, int dst_phys, int dst_rank,
                         const int* cands, int ncand) {
    if (p->npend == p->pcap) { p->pcap = p->pcap ? 2 * p->pcap : 1024; p->pend = xrealloc(p->pend, sizeof(pending_t) * (size_t)p->pcap); }
    if (p->ncands + ncand > p->ccap) {
        while (p->ncands + ncand > p->ccap) p->ccap = p->ccap ? 2 * p->ccap : 1024;
        p->cands = xrealloc(p->cands, sizeof(int) * (size_t)p->ccap);
    }
    pending_t* q = &p->pend[p->npend++];
    memset(q, 0, sizeof *q);
    q->kind = kind;
    q->t = t;
    q->flat = flat;
    if (box) q->box = *box;
    q->iv = iv;
    q->dst_phys = dst_phys;
    q->dst_rank = dst_rank;
    q->cand_off = p->ncands;
    q->ncand = ncand;
    memcpy(p->cands + p->ncands, cands, sizeof(int) * (size_t)ncand);
    p->ncands += ncand;
}

/* routing.hpp:185-193 decompose */
static catset_t decompose(const or_scenario* s, const region_t* src, const region_t* dst) {
    catset_t c;
    c.src = rg_copy(src);
    c.dst = rg_copy(dst);
    c.send = rg_diff(s, src, dst);
    c.recv = rg_diff(s, dst, src);
    c.retain = rg_intersect(s, src, dst);
    return c;
}
static void catset_free(catset_t* c) {
    rg_free(&c->src); rg_free(&c->dst); rg_free(&c->send); rg_free(&c->recv); rg_free(&c->retain);
}
static catset_t catset_copy(const catset_t* a) {
    catset_t c;
    c.src = rg_copy(&a->src); c.dst = rg_copy(&a->dst); c.send = rg_copy(&a->send);
    c.recv = rg_copy(&a->recv); c.retain = rg_copy(&a->retain);
    return c;
}

static void format_box_s(char* out, size_t n, const box_t* b, int nd) {
    size_t o = 0;
    o += (size_t)snprintf(out + o, n - o, "[");
    for (int i = 0; i < nd; ++i) o += (size_t)snprintf(out + o, n - o, "%s%lld:%lld", i ? "," : "", (long long)b->d[i].lo, (long long)b->d[i].hi);
    snprintf(out + o, n - o, "]");
}

/* routing.hpp:205-222 queue_box_recvs (+ box_candidates :197-203) */
static void queue_box_recvs(ctx_t* c, or_plan* p, const cfg_t* src_cfg, const region_t* src_regions, int nsrc, int kind,
                            const route_t* route, const region_t* recv) {
    const or_scenario* s = p->s;
    int* cands = xrealloc(NULL, sizeof(int) * (size_t)(nsrc + 1));
    for (int oi = 0; oi < s->nt; ++oi) {
        int t = s->by_id[oi];
        for (int b = 0; b < recv->tb[t].n; ++b) {
            blist cells = split_by_projection_grid(s, src_cfg, t, &recv->tb[t].v[b]);
            for (int ci = 0; ci < cells.n; ++ci) {
                int nc = 0;
                for (int j = 0; j < nsrc; ++j)
                    if (rg_contains_box(s, &src_regions[j], t, &cells.v[ci])) cands[nc++] = j;
                if (nc == 0) {
                    char bx[256];
                    format_box_s(bx, sizeof bx, &cells.v[ci], s->t[t].nd);
                    free(cands);
                    fail(c, 2, "unreachable state: no source holds %s %s needed by device %d", s->t[t].id, bx, route->phys);
                }
                iv_t z = {0, 0};
                push_pending(p, kind, t, 0, &cells.v[ci], z, route->phys, route->dst_rank, cands, nc);
            }
            bl_free(&cells);
        }
    }
    free(cands);
}

static int int_cmp(const void* a, const void* b) { int x = *(const int*)a, y = *(const int*)b; return (x > y) - (x < y); }

/* worldmap.hpp:30-79: identity default, participants, validate */
static void setup_world(ctx_t* c, const or_scenario* s, or_plan* p) {
    if (s->has_world) {
        p->nsrc = s->nsrc;
        p->ndst = s->ndst;
        p->src_phys = xrealloc(NULL, sizeof(int) * (size_t)(s->nsrc + 1));
        p->dst_phys = xrealloc(NULL, sizeof(int) * (size_t)(s->ndst + 1));
        memcpy(p->src_phys, s->src_phys, sizeof(int) * (size_t)s->nsrc);
        memcpy(p->dst_phys, s->dst_phys, sizeof(int) * (size_t)s->ndst);
    } else {
        p->nsrc = world_size(&s->src);
        p->ndst = world_size(&s->dst);
        p->src_phys = xrealloc(NULL, sizeof(int) * (size_t)(p->nsrc + 1));
        p->dst_phys = xrealloc(NULL, sizeof(int) * (size_t)(p->ndst + 1));
        for (int i = 0; i < p->nsrc; ++i) p->src_phys[i] = i;
        for (int i = 0; i < p->ndst; ++i) p->dst_phys[i] = i;
    }
    /* worldmap.hpp:68-78 validate */
    for (int side = 0; side < 2; ++side) {
        int n = side ? p->ndst : p->nsrc;
        int* v = xrealloc(NULL, sizeof(int) * (size_t)(n + 1));
        memcpy(v, side ? p->dst_phys : p->src_phys, sizeof(int) * (size_t)n);
        qsort(v, (size_t)n, sizeof(int), int_cmp);
        for (int i = 1; i < n; ++i)
            if (v[i] == v[i - 1]) { free(v); fail(c, 2, "%s maps two ranks to one device", side ? "dst world" : "src world"); }
        if (n && v[0] < 0) { free(v); fail(c, 2, "negative device id"); }
        free(v);
    }
}

static int src_rank_of(const or_plan* p, int phys) {
    for (int i = 0; i < p->nsrc; ++i) if (p->src_phys[i] == phys) return i;
    return -1;
}
static int dst_rank_of(const or_plan* p, int phys) {
    for (int i = 0; i < p->ndst; ++i) if (p->dst_phys[i] == phys) return i;
    return -1;
}

/* routing.hpp:231-279 plan_parameters */
static void plan_parameters(ctx_t* c, or_plan* p) {
    const or_scenario* s = p->s;
    setup_world(c, s, p);
    if (p->nsrc != world_size(&s->src)) fail(c, 2, "world map src size does not match src config");
    if (p->ndst != world_size(&s->dst)) fail(c, 2, "world map dst size does not match dst config");
    int ns = world_size(&s->src), nd = world_size(&s->dst);
    region_t* srcr = xrealloc(NULL, sizeof(region_t) * (size_t)ns);
    region_t* dstr = xrealloc(NULL, sizeof(region_t) * (size_t)nd);
    for (int i = 0; i < ns; ++i) srcr[i] = project(c, s, &s->src, i);
    for (int j = 0; j < nd; ++j) dstr[j] = project(c, s, &s->dst, j);
    /* participants: sorted unique union (worldmap.hpp:46-52) */
    int* parts = xrealloc(NULL, sizeof(int) * (size_t)(ns + nd + 1));
    int np = 0;
    for (int i = 0; i < ns; ++i) parts[np++] = p->src_phys[i];
    for (int i = 0; i < nd; ++i) parts[np++] = p->dst_phys[i];
    qsort(parts, (size_t)np, sizeof(int), int_cmp);
    int u = 0;
    for (int i = 0; i < np; ++i) if (u == 0 || parts[u - 1] != parts[i]) parts[u++] = parts[i];
    np = u;
    p->routes = calloc((size_t)(np + 1), sizeof(route_t));
    p->nroutes = np;
    region_t empty = rg_new(s->nt);
    for (int k = 0; k < np; ++k) {
        route_t* r = &p->routes[k];
        r->phys = parts[k];
        r->src_rank = src_rank_of(p, r->phys);
        r->dst_rank = dst_rank_of(p, r->phys);
        const region_t* rs = r->src_rank >= 0 ? &srcr[r->src_rank] : &empty;
        const region_t* rd = r->dst_rank >= 0 ? &dstr[r->dst_rank] : &empty;
        r->params = decompose(s, rs, rd);
        if (r->dst_rank >= 0) queue_box_recvs(c, p, &s->src, srcr, ns, 0, r, &r->params.recv);
    }
    if (s->migrate) {
        int64_t n = p->npend;
        for (int64_t i = 0; i < n; ++i)
            if (p->pend[i].kind == 0) {
                pending_t q = p->pend[i];
                push_pending(p, 2, q.t, q.flat, &q.box, q.iv, q.dst_phys, q.dst_rank, p->cands + q.cand_off, q.ncand);
            }
    }
    rg_free(&empty);
    for (int i = 0; i < ns; ++i) rg_free(&srcr[i]);
    for (int j = 0; j < nd; ++j) rg_free(&dstr[j]);
    free(srcr);
    free(dstr);
    free(parts);
}

/* routing.hpp:287-337 plan_optimizer. allow_oversourced enables the documented
 * D2 extension: an over-sourced recv interval is split into
 * maximal runs with a uniform candidate set, resolved later by resolve_peers. */
static void plan_optimizer(ctx_t* c, or_plan* p, int allow_oversourced) {
    const or_scenario* s = p->s;
    if (s->src.zero != s->dst.zero) fail(c, 2, "transitions toggling zero_enabled are unsupported");
    int ns = world_size(&s->src), nd = world_size(&s->dst);
    if (!s->src.zero) {
        region_t* srcr = xrealloc(NULL, sizeof(region_t) * (size_t)ns);
        for (int i = 0; i < ns; ++i) srcr[i] = project(c, s, &s->src, i);
        for (int k = 0; k < p->nroutes; ++k) {
            route_t* r = &p->routes[k];
            r->optim = catset_copy(&r->params);
            if (r->dst_rank >= 0) queue_box_recvs(c, p, &s->src, srcr, ns, 1, r, &r->optim.recv);
        }
        for (int i = 0; i < ns; ++i) rg_free(&srcr[i]);
        free(srcr);
        return;
    }
    region_t* ss = xrealloc(NULL, sizeof(region_t) * (size_t)ns);
    region_t* ds = xrealloc(NULL, sizeof(region_t) * (size_t)nd);
    for (int i = 0; i < ns; ++i) ss[i] = project_optimizer(c, s, &s->src, i);
    for (int j = 0; j < nd; ++j) ds[j] = project_optimizer(c, s, &s->dst, j);
    region_t empty = rg_new(s->nt);
    ilist pieces = {0};
    int* owners = NULL;
    int64_t ocap = 0;
    int* cset = xrealloc(NULL, sizeof(int) * (size_t)(ns + 1));
    for (int k = 0; k < p->nroutes; ++k) {
        route_t* r = &p->routes[k];
        const region_t* rs = r->src_rank >= 0 ? &ss[r->src_rank] : &empty;
        const region_t* rd = r->dst_rank >= 0 ? &ds[r->dst_rank] : &empty;
        r->optim = decompose(s, rs, rd);
        for (int64_t q = 0; q < r->optim.recv.flat.n; ++q) {
            iv_t iv = r->optim.recv.flat.v[q];
            pieces.n = 0;
            int64_t np = 0;
            for (int j = 0; j < ns; ++j) {
                const ilist* sh = &ss[j].flat;
                for (int64_t a = il_lower(sh, iv.lo); a < sh->n && sh->v[a].lo < iv.hi; ++a) {
                    int64_t lo = sh->v[a].lo > iv.lo ? sh->v[a].lo : iv.lo;
                    int64_t hi = sh->v[a].hi < iv.hi ? sh->v[a].hi : iv.hi;
                    if (lo >= hi) continue;
                    il_push(&pieces, lo, hi);
                    if (np == ocap) { ocap = ocap ? 2 * ocap : 64; owners = xrealloc(owners, sizeof(int) * (size_t)ocap); }
                    owners[np++] = j;
                }
            }
            int64_t total = il_length(&pieces);
            int64_t len = iv.hi - iv.lo;
            if (total == len) {
                for (int64_t a = 0; a < np; ++a)
                    push_pending(p, 1, -1, 1, NULL, pieces.v[a], r->phys, r->dst_rank, &owners[a], 1);
                continue;
            }
            if (!allow_oversourced || total < len)
                fail(c, 2, "unreachable state: optimizer interval [%lld:%lld] for device %d not fully sourced",
                     (long long)iv.lo, (long long)iv.hi, r->phys);
            /* D2 extension: elementary segments between all piece boundaries */
            int64_t nb = 0;
            int64_t* bnd = xrealloc(NULL, sizeof(int64_t) * (size_t)(2 * np + 2));
            bnd[nb++] = iv.lo;
            bnd[nb++] = iv.hi;
            for (int64_t a = 0; a < np; ++a) { bnd[nb++] = pieces.v[a].lo; bnd[nb++] = pieces.v[a].hi; }
            for (int64_t x = 1; x < nb; ++x) {
                int64_t v = bnd[x], y = x - 1;
                while (y >= 0 && bnd[y] > v) { bnd[y + 1] = bnd[y]; --y; }
                bnd[y + 1] = v;
            }
            int64_t run_lo = -1, run_hi = -1;
            int run_n = 0;
            int* run_c = xrealloc(NULL, sizeof(int) * (size_t)(ns + 1));
            for (int64_t x = 0; x + 1 < nb; ++x) {
                int64_t lo = bnd[x], hi = bnd[x + 1];
                if (lo >= hi) continue;
                int ncs = 0;
                for (int64_t a = 0; a < np; ++a)
                    if (pieces.v[a].lo <= lo && hi <= pieces.v[a].hi) {
                        int dup = 0;
                        for (int z = 0; z < ncs; ++z) dup |= cset[z] == owners[a];
                        if (!dup) cset[ncs++] = owners[a];
                    }
                qsort(cset, (size_t)ncs, sizeof(int), int_cmp);
                if (ncs == 0) { free(bnd); free(run_c); fail(c, 2, "unreachable state: optimizer interval [%lld:%lld] for device %d not fully sourced", (long long)iv.lo, (long long)iv.hi, r->phys); }
                if (run_n == ncs && run_hi == lo && !memcmp(run_c, cset, sizeof(int) * (size_t)ncs)) {
                    run_hi = hi;
                } else {
                    if (run_n) { iv_t z = {run_lo, run_hi}; push_pending(p, 1, -1, 1, NULL, z, r->phys, r->dst_rank, run_c, run_n); }
                    run_lo = lo; run_hi = hi; run_n = ncs;
                    memcpy(run_c, cset, sizeof(int) * (size_t)ncs);
                }
            }
            if (run_n) { iv_t z = {run_lo, run_hi}; push_pending(p, 1, -1, 1, NULL, z, r->phys, r->dst_rank, run_c, run_n); }
            free(run_c);
            free(bnd);
        }
    }
    free(cset);
    free(owners);
    il_free(&pieces);
    rg_free(&empty);
    for (int i = 0; i < ns; ++i) rg_free(&ss[i]);
    for (int j = 0; j < nd; ++j) rg_free(&ds[j]);
    free(ss);
    free(ds);
}

/* routing.hpp:341-353 plan_scalars */
static void plan_scalars(or_plan* p) {
    if (p->nsrc == 0) return;
    p->has_scalars = 1;
    p->root_phys = p->src_phys[0];
    p->scalar_bytes_per_rank = p->s->scalar_words * 8;
    p->scalar_recv = xrealloc(NULL, sizeof(int) * (size_t)(p->ndst + 1));
    p->nscalar_recv = 0;
    for (int j = 0; j < p->ndst; ++j)
        if (p->dst_phys[j] != p->root_phys) p->scalar_recv[p->nscalar_recv++] = p->dst_phys[j];
    qsort(p->scalar_recv, (size_t)p->nscalar_recv, sizeof(int), int_cmp);
}

/* routing.hpp:79-84 transfer_order_less: (src, dst, kind, tensor_id, region key) */
static const or_scenario* g_cmp_scn;
static int tr_cmp(const void* A, const void* B) {
    const or_transfer *a = A, *b = B;
    if (a->src_rank != b->src_rank) return a->src_rank < b->src_rank ? -1 : 1;
    if (a->dst_rank != b->dst_rank) return a->dst_rank < b->dst_rank ? -1 : 1;
    if (a->kind != b->kind) return a->kind < b->kind ? -1 : 1;
    const char* ia = a->tensor >= 0 ? g_cmp_scn->t[a->tensor].id : "";
    const char* ib = b->tensor >= 0 ? g_cmp_scn->t[b->tensor].id : "";
    int sc = strcmp(ia, ib);
    if (sc) return sc < 0 ? -1 : 1;
    int na = a->flat ? 1 : a->nd, nb = b->flat ? 1 : b->nd;
    for (int i = 0; i < na && i < nb; ++i) {
        if (a->lo[i] != b->lo[i]) return a->lo[i] < b->lo[i] ? -1 : 1;
        if (a->hi[i] != b->hi[i]) return a->hi[i] < b->hi[i] ? -1 : 1;
    }
    return (na > nb) - (na < nb);
}

/* routing.hpp:360-396 resolve_peers (D1 fixed: byte widths from the model space,
 * routing.hpp:174-183 payload_bytes) */
static void resolve_peers(or_plan* p) {
    const or_scenario* s = p->s;
    int64_t cursor = 0;
    p->tr = xrealloc(NULL, sizeof(or_transfer) * (size_t)(p->npend + 1));
    p->ntr = 0;
    for (int64_t i = 0; i < p->npend; ++i) {
        const pending_t* q = &p->pend[i];
        const int* cands = p->cands + q->cand_off;
        int chosen;
        if (s->balance && q->ncand > 1) {
            chosen = cands[(size_t)(cursor++) % (size_t)q->ncand];
        } else {
            chosen = -1;
            for (int k = 0; k < q->ncand; ++k) {
                int cp = p->src_phys[cands[k]];
                if (cp / s->rpn == q->dst_phys / s->rpn) { chosen = cands[k]; break; }
            }
            if (chosen < 0) chosen = cands[0];
        }
        or_transfer* t = &p->tr[p->ntr++];
        memset(t, 0, sizeof *t);
        t->kind = q->kind;
        t->tensor = q->flat ? -1 : q->t;
        t->flat = q->flat;
        if (q->flat) {
            t->nd = 1;
            t->lo[0] = q->iv.lo;
            t->hi[0] = q->iv.hi;
            t->count = q->iv.hi - q->iv.lo;
        } else {
            t->nd = s->t[q->t].nd;
            for (int d = 0; d < t->nd; ++d) { t->lo[d] = q->box.d[d].lo; t->hi[d] = q->box.d[d].hi; }
            t->count = box_numel(&q->box, t->nd);
        }
        t->src_rank = chosen;
        t->src_phys = p->src_phys[chosen];
        t->dst_rank = q->dst_rank;
        t->dst_phys = q->dst_phys;
        int w = q->kind == 0 ? s->t[q->t].dtype : q->kind == 1 ? 12 : q->kind == 2 ? 4 : 8;
        t->bytes = t->count * w;
    }
    free(p->pend); p->pend = NULL; p->npend = p->pcap = 0;
    free(p->cands); p->cands = NULL; p->ncands = p->ccap = 0;
    g_cmp_scn = s;
    qsort(p->tr, (size_t)p->ntr, sizeof(or_transfer), tr_cmp);
}

int or_plan_build(const or_scenario* s, int allow_oversourced, or_plan** out, char* err, size_t errlen) {
    *out = NULL;
    ctx_t* c = calloc(1, sizeof *c);
    or_plan* volatile p = calloc(1, sizeof *p);
    p->s = s;
    int code = setjmp(c->jb);
    if (code) {
        snprintf(err, errlen, "%s", c->msg);
        free(c);
        or_plan_free(p);
        return code;
    }
    /* CLI order: validate_config x2, then the planner passes */
    validate_config(c, s, &s->src);
    validate_config(c, s, &s->dst);
    plan_parameters(c, p);
    plan_optimizer(c, p, allow_oversourced);
    plan_scalars(p);
    resolve_peers(p);
    free(c);
    *out = p;
    return 0;
}

void or_plan_free(or_plan* p) {
    if (!p) return;
    for (int k = 0; k < p->nroutes; ++k) {
        route_t* r = &p->routes[k];
        if (r->params.src.tb) catset_free(&r->params);
        if (r->optim.src.tb) catset_free(&r->optim);
    }
    free(p->routes);
    free(p->pend);
    free(p->cands);
    free(p->tr);
    free(p->scalar_recv);
    free(p->src_phys);
    free(p->dst_phys);
    free(p);
}

int64_t or_plan_num_transfers(const or_plan* p) { return p->ntr; }
const or_transfer* or_plan_transfers(const or_plan* p) { return p->tr; }

/* routing.hpp:151-156 bytes_moved */
int64_t or_plan_bytes_moved(const or_plan* p) {
    int64_t n = 0;
    for (int64_t i = 0; i < p->ntr; ++i) n += p->tr[i].bytes;
    if (p->has_scalars) n += p->scalar_bytes_per_rank * p->nscalar_recv;
    return n;
}

/* routing.hpp:157-169 bytes_retained */
int64_t or_plan_bytes_retained(const or_plan* p) {
    const or_scenario* s = p->s;
    int64_t n = 0;
    for (int k = 0; k < p->nroutes; ++k) {
        const route_t* r = &p->routes[k];
        for (int t = 0; t < s->nt; ++t)
            for (int b = 0; b < r->params.retain.tb[t].n; ++b)
                n += box_numel(&r->params.retain.tb[t].v[b], s->t[t].nd) * s->t[t].dtype;
        n += il_length(&r->optim.retain.flat) * 12;
        for (int t = 0; t < s->nt; ++t)
            for (int b = 0; b < r->optim.retain.tb[t].n; ++b)
                n += box_numel(&r->optim.retain.tb[t].v[b], s->t[t].nd) * 12;
    }
    return n;
}

/* routing.hpp:86-90 format_transfer */
static const char* kind_name(int k) { return k == 0 ? "param" : k == 1 ? "optim" : k == 2 ? "grad" : "scalar"; }

char* or_plan_dump(const or_plan* p) {
    size_t cap = 1 << 16, len = 0;
    char* out = xrealloc(NULL, cap);
    out[0] = 0;
    char line[1024], reg[512];
    for (int64_t i = 0; i < p->ntr; ++i) {
        const or_transfer* t = &p->tr[i];
        if (t->flat) snprintf(reg, sizeof reg, "[%lld:%lld]", (long long)t->lo[0], (long long)t->hi[0]);
        else {
            box_t b;
            memset(&b, 0, sizeof b);
            for (int d = 0; d < t->nd; ++d) { b.d[d].lo = t->lo[d]; b.d[d].hi = t->hi[d]; }
            format_box_s(reg, sizeof reg, &b, t->nd);
        }
        int n = snprintf(line, sizeof line, "%s %s %s src=%d dst=%d bytes=%lld\n", kind_name(t->kind),
                         t->tensor >= 0 ? p->s->t[t->tensor].id : "-", reg, t->src_rank, t->dst_rank, (long long)t->bytes);
        if (len + (size_t)n + 1 > cap) { while (len + (size_t)n + 1 > cap) cap *= 2; out = xrealloc(out, cap); }
        memcpy(out + len, line, (size_t)n + 1);
        len += (size_t)n;
    }
    return out;
}

/* ------------------------------------------------------------ regions dump */

typedef struct { char* b; size_t len, cap; } sbuf;
static void sb_printf(sbuf* s, const char* fmt, ...) {
    char tmp[1024];
    va_list a;
    va_start(a, fmt);
    int n = vsnprintf(tmp, sizeof tmp, fmt, a);
    va_end(a);
    if (s->len + (size_t)n + 1 > s->cap) { s->cap = (s->cap + (size_t)n + 1) * 2; s->b = xrealloc(s->b, s->cap); }
    memcpy(s->b + s->len, tmp, (size_t)n + 1);
    s->len += (size_t)n;
}

char* or_regions_dump(const or_scenario* s, int which, char* err, size_t errlen) {
    ctx_t* c = calloc(1, sizeof *c);
    sbuf sb = {0};
    sb_printf(&sb, "");
    int code = setjmp(c->jb);
    if (code) { snprintf(err, errlen, "%s", c->msg); free(c); free(sb.b); return NULL; }
    const cfg_t* cfg = which ? &s->dst : &s->src;
    validate_config(c, s, cfg);
    char bx[512];
    for (int r = 0; r < world_size(cfg); ++r) {
        region_t reg = project(c, s, cfg, r);
        for (int oi = 0; oi < s->nt; ++oi) {
            int t = s->by_id[oi];
            for (int b = 0; b < reg.tb[t].n; ++b) {
                format_box_s(bx, sizeof bx, &reg.tb[t].v[b], s->t[t].nd);
                sb_printf(&sb, "rank %d param %s %s\n", r, s->t[t].id, bx);
            }
        }
        rg_free(&reg);
        layout_t L = local_layout(c, s, cfg, r);
        for (int i = 0; i < L.nd_; ++i) {
            format_box_s(bx, sizeof bx, &L.dense[i].box, s->t[L.dense[i].t].nd);
            sb_printf(&sb, "rank %d layout dense %s %s %lld %lld\n", r, s->t[L.dense[i].t].id, bx, (long long)L.dense[i].lo, (long long)L.dense[i].hi);
        }
        for (int i = 0; i < L.ne_; ++i) {
            format_box_s(bx, sizeof bx, &L.expert[i].box, s->t[L.expert[i].t].nd);
            sb_printf(&sb, "rank %d layout expert %s %s %lld %lld\n", r, s->t[L.expert[i].t].id, bx, (long long)L.expert[i].lo, (long long)L.expert[i].hi);
        }
        layout_free(&L);
        if (cfg->zero) {
            region_t o = project_optimizer(c, s, cfg, r);
            for (int64_t i = 0; i < o.flat.n; ++i) sb_printf(&sb, "rank %d optim [%lld:%lld]\n", r, (long long)o.flat.v[i].lo, (long long)o.flat.v[i].hi);
            rg_free(&o);
        }
    }
    free(c);
    return sb.b;
}

/* ----------------------------------------------------------------- executor */

/* Physical layout per virtual rank (SURVEY §8a contract):
 *  param : local_layout segments, dense then expert, dtype_bytes per element
 *  grad  : same segments, 4 B per element
 *  optim : ZeRO -> [dense shard | expert shard] of the local index spaces;
 *          no ZeRO -> dense_len + expert_len elements; SoA master/m/v, 4 B each
 *  scalars: scalar_words x 8 B */
typedef struct {
    layout_t L;
    int64_t* seg_byte_off; /* per segment (dense..., expert...) param byte offset */
    int64_t param_bytes, nelem;
    iv_t dshard, eshard;
    int64_t optim_len;
    uint8_t* buf[6];
    int64_t bytes[6];
} rstate_t;

struct or_state {
    const or_scenario* s;
    const cfg_t* cfg;
    int which, nranks, with_grads;
    rstate_t* r;
};

static seg_t* rs_seg(const rstate_t* R, int i) { return i < R->L.nd_ ? &R->L.dense[i] : &R->L.expert[i - R->L.nd_]; }
static int rs_nseg(const rstate_t* R) { return R->L.nd_ + R->L.ne_; }

or_state* or_state_create(const or_scenario* s, int which, int with_grads, char* err, size_t errlen) {
    ctx_t* c = calloc(1, sizeof *c);
    or_state* volatile st = calloc(1, sizeof *st);
    int code = setjmp(c->jb);
    if (code) { snprintf(err, errlen, "%s", c->msg); free(c); or_state_free(st); return NULL; }
    st->s = s;
    st->which = which;
    st->cfg = which ? &s->dst : &s->src;
    st->with_grads = with_grads;
    validate_config(c, s, st->cfg);
    st->nranks = world_size(st->cfg);
    st->r = calloc((size_t)st->nranks, sizeof(rstate_t));
    for (int r = 0; r < st->nranks; ++r) {
        rstate_t* R = &st->r[r];
        R->L = local_layout(c, s, st->cfg, r);
        int ns = rs_nseg(R);
        R->seg_byte_off = xrealloc(NULL, sizeof(int64_t) * (size_t)(ns + 1));
        int64_t bo = 0;
        for (int i = 0; i < ns; ++i) {
            seg_t* g = rs_seg(R, i);
            bo = (bo + 15) / 16 * 16; /* segments start 16-B aligned */
            R->seg_byte_off[i] = bo;
            bo += (g->hi - g->lo) * s->t[g->t].dtype;
        }
        R->param_bytes = bo;
        R->nelem = R->L.dense_len + R->L.expert_len;
        coord_t k = rank_coord(c, st->cfg, r);
        if (st->cfg->zero) {
            R->dshard = shard_range(R->L.dense_len, st->cfg->dp, k.dp);
            R->eshard = shard_range(R->L.expert_len, st->cfg->dp / st->cfg->ep, k.edp);
        } else {
            R->dshard = (iv_t){0, R->L.dense_len};
            R->eshard = (iv_t){0, R->L.expert_len};
        }
        R->optim_len = (R->dshard.hi - R->dshard.lo) + (R->eshard.hi - R->eshard.lo);
        R->bytes[0] = R->param_bytes;
        R->bytes[1] = R->bytes[2] = R->bytes[3] = R->optim_len * 4;
        R->bytes[4] = with_grads ? R->nelem * 4 : 0;
        R->bytes[5] = s->scalar_words * 8;
        for (int b = 0; b < 6; ++b) R->buf[b] = calloc((size_t)(R->bytes[b] ? R->bytes[b] : 1), 1);
    }
    free(c);
    return st;
}

void or_state_free(or_state* st) {
    if (!st) return;
    if (st->r)
        for (int r = 0; r < st->nranks; ++r) {
            layout_free(&st->r[r].L);
            free(st->r[r].seg_byte_off);
            for (int b = 0; b < 6; ++b) free(st->r[r].buf[b]);
        }
    free(st->r);
    free(st);
}
int or_state_num_ranks(const or_state* st) { return st->nranks; }
void* or_state_buffer(or_state* st, int rank, int buf, int64_t* bytes) {
    if (rank < 0 || rank >= st->nranks || buf < 0 || buf > 5) { *bytes = 0; return NULL; }
    *bytes = st->r[rank].bytes[buf];
    return st->r[rank].buf[buf];
}
void or_state_clear(or_state* st) {
    for (int r = 0; r < st->nranks; ++r)
        for (int b = 0; b < 6; ++b) memset(st->r[r].buf[b], 0, (size_t)st->r[r].bytes[b]);
}

/* optim position of local element index li (dense idx if !expert) or -1 */
static int64_t optim_pos(const rstate_t* R, int expert, int64_t li) {
    if (!expert) return (li >= R->dshard.lo && li < R->dshard.hi) ? li - R->dshard.lo : -1;
    if (li >= R->eshard.lo && li < R->eshard.hi) return (R->dshard.hi - R->dshard.lo) + li - R->eshard.lo;
    return -1;
}

static void put_param(uint8_t* p, int w, uint64_t v) { memcpy(p, &v, (size_t)w); } /* little-endian low bytes */
static uint64_t get_param(const uint8_t* p, int w) { uint64_t v = 0; memcpy(&v, p, (size_t)w); return v; }

typedef void (*elem_fn)(void* ctx, int rank, rstate_t* R, int seg, int64_t li_in_seg, int64_t k);

/* visit every element a rank holds, row-major per segment, with its global flat index */
static void for_each_elem(or_state* st, int rank, elem_fn fn, void* ctx) {
    const or_scenario* s = st->s;
    rstate_t* R = &st->r[rank];
    for (int i = 0; i < rs_nseg(R); ++i) {
        seg_t* g = rs_seg(R, i);
        const tens_t* t = &s->t[g->t];
        int d = t->nd;
        int64_t stride[4];
        stride[d - 1] = 1;
        for (int a = d - 1; a > 0; --a) stride[a - 1] = stride[a] * t->shape[a];
        int64_t n = g->hi - g->lo, idx[4];
        for (int a = 0; a < d; ++a) idx[a] = g->box.d[a].lo;
        for (int64_t e = 0; e < n; ++e) {
            int64_t k = t->off;
            for (int a = 0; a < d; ++a) k += idx[a] * stride[a];
            fn(ctx, rank, R, i, e, k);
            for (int a = d - 1; a >= 0; --a) {
                if (++idx[a] < g->box.d[a].hi) break;
                idx[a] = g->box.d[a].lo;
            }
        }
    }
}

typedef struct { or_state* st; uint64_t seed; int64_t bad; char* err; size_t errlen; } lv_ctx;

static void load_fn(void* cx, int rank, rstate_t* R, int si, int64_t e, int64_t k) {
    lv_ctx* c = cx;
    (void)rank;
    seg_t* g = rs_seg(R, si);
    int w = c->st->s->t[g->t].dtype;
    put_param(R->buf[0] + R->seg_byte_off[si] + e * w, w, or_canon(c->seed, k, 0));
    int expert = si >= R->L.nd_;
    int64_t li = g->lo + e;
    if (c->st->with_grads) {
        uint32_t gv = (uint32_t)or_canon(c->seed, k, 2);
        memcpy(R->buf[4] + ((expert ? R->L.dense_len : 0) + li) * 4, &gv, 4);
    }
    int64_t op = optim_pos(R, expert, li);
    if (op >= 0) {
        uint64_t o = or_canon(c->seed, k, 1);
        uint32_t mst = (uint32_t)o, m = (uint32_t)(o >> 32), v = (uint32_t)or_canon(c->seed ^ 0x5eedull, k, 1);
        memcpy(R->buf[1] + op * 4, &mst, 4);
        memcpy(R->buf[2] + op * 4, &m, 4);
        memcpy(R->buf[3] + op * 4, &v, 4);
    }
}

/* load_state; ranks are independent, so they load in parallel */
typedef struct { or_state* st; uint64_t seed; int rank; } load_job;
static void* load_worker(void* a) {
    load_job* j = a;
    lv_ctx c = {j->st, j->seed, 0, NULL, 0};
    for_each_elem(j->st, j->rank, load_fn, &c);
    for (int64_t w = 0; w < j->st->s->scalar_words; ++w) {
        uint64_t v = or_canon(j->seed, w, 3);
        memcpy(j->st->r[j->rank].buf[5] + w * 8, &v, 8);
    }
    return NULL;
}
void or_state_load(or_state* st, uint64_t seed) {
    pthread_t* th = xrealloc(NULL, sizeof(pthread_t) * (size_t)st->nranks);
    load_job* jobs = xrealloc(NULL, sizeof(load_job) * (size_t)st->nranks);
    for (int r = 0; r < st->nranks; ++r) {
        jobs[r] = (load_job){st, seed, r};
        pthread_create(&th[r], NULL, load_worker, &jobs[r]);
    }
    for (int r = 0; r < st->nranks; ++r) pthread_join(th[r], NULL);
    free(th);
    free(jobs);
}

static void verify_fn(void* cx, int rank, rstate_t* R, int si, int64_t e, int64_t k) {
    lv_ctx* c = cx;
    seg_t* g = rs_seg(R, si);
    int w = c->st->s->t[g->t].dtype;
    uint64_t mask = w >= 8 ? ~0ull : ((1ull << (8 * w)) - 1);
    uint64_t got = get_param(R->buf[0] + R->seg_byte_off[si] + e * w, w);
    int expert = si >= R->L.nd_;
    int64_t li = g->lo + e;
#define BAD(kind)                                                                                             \
    do {                                                                                                      \
        if (c->bad++ == 0 && c->err)                                                                          \
            snprintf(c->err, c->errlen, "rank %d %s element %lld mismatch", rank, kind, (long long)k);         \
    } while (0)
    if (got != (or_canon(c->seed, k, 0) & mask)) BAD("param");
    if (c->st->with_grads) {
        uint32_t gv;
        memcpy(&gv, R->buf[4] + ((expert ? R->L.dense_len : 0) + li) * 4, 4);
        if (gv != (uint32_t)or_canon(c->seed, k, 2)) BAD("grad");
    }
    int64_t op = optim_pos(R, expert, li);
    if (op >= 0) {
        uint64_t o = or_canon(c->seed, k, 1);
        uint32_t a, b, v;
        memcpy(&a, R->buf[1] + op * 4, 4);
        memcpy(&b, R->buf[2] + op * 4, 4);
        memcpy(&v, R->buf[3] + op * 4, 4);
        if (a != (uint32_t)o || b != (uint32_t)(o >> 32) || v != (uint32_t)or_canon(c->seed ^ 0x5eedull, k, 1)) BAD("optim");
    }
#undef BAD
}

/* verify_state; ranks checked in parallel, first violation by rank order */
typedef struct { or_state* st; uint64_t seed; int rank; int64_t bad; char msg[256]; } verify_job;
static void* verify_worker(void* a) {
    verify_job* j = a;
    lv_ctx c = {j->st, j->seed, 0, j->msg, sizeof j->msg};
    j->msg[0] = 0;
    for_each_elem(j->st, j->rank, verify_fn, &c);
    for (int64_t w = 0; w < j->st->s->scalar_words; ++w) {
        uint64_t v;
        memcpy(&v, j->st->r[j->rank].buf[5] + w * 8, 8);
        if (v != or_canon(j->seed, w, 3) && c.bad++ == 0)
            snprintf(j->msg, sizeof j->msg, "rank %d scalar word %lld mismatch", j->rank, (long long)w);
    }
    j->bad = c.bad;
    return NULL;
}
int64_t or_verify(const or_state* stc, uint64_t seed, char* err, size_t errlen) {
    or_state* st = (or_state*)stc;
    if (err && errlen) err[0] = 0;
    pthread_t* th = xrealloc(NULL, sizeof(pthread_t) * (size_t)st->nranks);
    verify_job* jobs = xrealloc(NULL, sizeof(verify_job) * (size_t)st->nranks);
    for (int r = 0; r < st->nranks; ++r) {
        jobs[r].st = st;
        jobs[r].seed = seed;
        jobs[r].rank = r;
        jobs[r].bad = 0;
        pthread_create(&th[r], NULL, verify_worker, &jobs[r]);
    }
    int64_t bad = 0;
    for (int r = 0; r < st->nranks; ++r) {
        pthread_join(th[r], NULL);
        if (jobs[r].bad && bad == 0 && err) snprintf(err, errlen, "%s", jobs[r].msg);
        bad += jobs[r].bad;
    }
    free(th);
    free(jobs);
    return bad;
}

/* locate global coordinate c (tensor t) inside rank R's segment: returns segment
 * index and row-major local offset within it, or -1 */
static int find_seg(const rstate_t* R, int t) {
    for (int i = 0; i < rs_nseg(R); ++i)
        if (rs_seg(R, i)->t == t) return i;
    return -1;
}
static int64_t seg_offset(const or_scenario* s, const seg_t* g, const int64_t* coord) {
    const tens_t* t = &s->t[g->t];
    int64_t o = 0;
    for (int a = 0; a < t->nd; ++a) o = o * (g->box.d[a].hi - g->box.d[a].lo) + (coord[a] - g->box.d[a].lo);
    return o;
}
static int tensor_of(const or_scenario* s, int64_t k) {
    int L = 0, R = s->nt - 1;
    while (L < R) {
        int m = (L + R + 1) / 2;
        if (s->t[m].off <= k) L = m; else R = m - 1;
    }
    return L;
}

typedef struct { int kind; const or_transfer* t; int64_t lo, hi; } work_t; /* kind 0 box rows [lo,hi), 1 flat [lo,hi) */

typedef struct {
    const or_plan* p;
    const or_state* src;
    or_state* dst;
    work_t* w;
    int64_t nw;
    int64_t next;
    pthread_mutex_t mu;
    int bad;
    char msg[256];
} exec_ctx;

/* copy rows [r0, r1) of a box transfer (rows = all coords but the last axis) */
static int copy_box_rows(exec_ctx* E, const or_transfer* tr, int64_t r0, int64_t r1) {
    const or_scenario* s = E->p->s;
    int ti = tr->tensor;
    const tens_t* t = &s->t[ti];
    const rstate_t* S = &E->src->r[tr->src_rank];
    rstate_t* D = &E->dst->r[tr->dst_rank];
    int ssi = find_seg(S, ti), dsi = find_seg(D, ti);
    if (ssi < 0 || dsi < 0) return -1;
    const seg_t *sg = rs_seg(S, ssi), *dg = rs_seg(D, dsi);
    int nd = t->nd;
    int64_t width = tr->hi[nd - 1] - tr->lo[nd - 1];
    int64_t coord[4];
    for (int64_t row = r0; row < r1; ++row) {
        int64_t rem = row;
        for (int a = nd - 2; a >= 0; --a) {
            int64_t len = tr->hi[a] - tr->lo[a];
            coord[a] = tr->lo[a] + rem % len;
            rem /= len;
        }
        coord[nd - 1] = tr->lo[nd - 1];
        int64_t so = seg_offset(s, sg, coord), dof = seg_offset(s, dg, coord);
        if (tr->kind == 0) {
            int w = t->dtype;
            memcpy(D->buf[0] + D->seg_byte_off[dsi] + dof * w, S->buf[0] + S->seg_byte_off[ssi] + so * w, (size_t)(width * w));
        } else if (tr->kind == 2) {
            int64_t sl = (ssi >= S->L.nd_ ? S->L.dense_len : 0) + sg->lo + so;
            int64_t dl = (dsi >= D->L.nd_ ? D->L.dense_len : 0) + dg->lo + dof;
            memcpy(D->buf[4] + dl * 4, S->buf[4] + sl * 4, (size_t)(width * 4));
        } else {
            int64_t sp = optim_pos(S, ssi >= S->L.nd_, sg->lo + so);
            int64_t dp = optim_pos(D, dsi >= D->L.nd_, dg->lo + dof);
            int64_t spe = optim_pos(S, ssi >= S->L.nd_, sg->lo + so + width - 1);
            int64_t dpe = optim_pos(D, dsi >= D->L.nd_, dg->lo + dof + width - 1);
            if (sp < 0 || dp < 0 || spe != sp + width - 1 || dpe != dp + width - 1) return -1;
            for (int b = 1; b <= 3; ++b) memcpy(D->buf[b] + dp * 4, S->buf[b] + sp * 4, (size_t)(width * 4));
        }
    }
    return 0;
}

/* copy flat ZeRO optimizer interval [lo,hi) from src rank to dst rank */
static int copy_flat(exec_ctx* E, int sr, int dr, int64_t lo, int64_t hi) {
    const or_scenario* s = E->p->s;
    const rstate_t* S = &E->src->r[sr];
    rstate_t* D = &E->dst->r[dr];
    int64_t k = lo;
    int64_t coord[4];
    while (k < hi) {
        int ti = tensor_of(s, k);
        const tens_t* t = &s->t[ti];
        int ssi = find_seg(S, ti), dsi = find_seg(D, ti);
        if (ssi < 0 || dsi < 0) return -1;
        const seg_t *sg = rs_seg(S, ssi), *dg = rs_seg(D, dsi);
        int64_t rem = k - t->off;
        for (int a = t->nd - 1; a >= 0; --a) { coord[a] = rem % t->shape[a]; rem /= t->shape[a]; }
        int64_t last = coord[t->nd - 1];
        int64_t n = hi - k;
        if (sg->box.d[t->nd - 1].hi - last < n) n = sg->box.d[t->nd - 1].hi - last;
        if (dg->box.d[t->nd - 1].hi - last < n) n = dg->box.d[t->nd - 1].hi - last;
        if (n <= 0) return -1;
        int64_t sp = optim_pos(S, ssi >= S->L.nd_, sg->lo + seg_offset(s, sg, coord));
        int64_t dp = optim_pos(D, dsi >= D->L.nd_, dg->lo + seg_offset(s, dg, coord));
        if (sp < 0 || dp < 0 || sp + n > S->optim_len || dp + n > D->optim_len) return -1;
        for (int b = 1; b <= 3; ++b) memcpy(D->buf[b] + dp * 4, S->buf[b] + sp * 4, (size_t)(n * 4));
        k += n;
    }
    return 0;
}

static void* exec_worker(void* arg) {
    exec_ctx* E = arg;
    for (;;) {
        pthread_mutex_lock(&E->mu);
        int64_t i = E->next++;
        pthread_mutex_unlock(&E->mu);
        if (i >= E->nw) break;
        work_t* w = &E->w[i];
        int rc = w->kind == 0 ? copy_box_rows(E, w->t, w->lo, w->hi)
                              : copy_flat(E, w->t->src_rank, w->t->dst_rank, w->lo, w->hi);
        if (rc) {
            pthread_mutex_lock(&E->mu);
            if (!E->bad) snprintf(E->msg, sizeof E->msg, "transfer outside the physical layout");
            E->bad = 1;
            pthread_mutex_unlock(&E->mu);
        }
    }
    return NULL;
}

/* execute. Plan transfers + retained regions (routing.hpp:98
 * retain = R_src ∩ R_dst) + scalar broadcast (routing.hpp:341-353). Work items
 * are independent (disjoint destination ranges), so threads need no ordering. */
int or_execute(const or_plan* p, const or_state* src, or_state* dst, int nthreads, char* err, size_t errlen) {
    const or_scenario* s = p->s;
    exec_ctx E;
    memset(&E, 0, sizeof E);
    E.p = p;
    E.src = src;
    E.dst = dst;
    int64_t cap = 1024;
    E.w = xrealloc(NULL, sizeof(work_t) * (size_t)cap);
    /* retained regions expressed as synthetic transfers (same device) */
    int64_t nret = 0, rcap = 256;
    or_transfer* ret = xrealloc(NULL, sizeof(or_transfer) * (size_t)rcap);
#define PUSH_RET(T) do { if (nret == rcap) { rcap *= 2; ret = xrealloc(ret, sizeof(or_transfer) * (size_t)rcap); } ret[nret++] = (T); } while (0)
    for (int k = 0; k < p->nroutes; ++k) {
        const route_t* r = &p->routes[k];
        if (r->src_rank < 0 || r->dst_rank < 0) continue;
        for (int kind = 0; kind < 3; ++kind) {
            if (kind == 2 && !s->migrate) continue;
            const region_t* reg = kind == 1 ? &r->optim.retain : &r->params.retain;
            for (int t = 0; t < s->nt; ++t)
                for (int b = 0; b < reg->tb[t].n; ++b) {
                    or_transfer tr;
                    memset(&tr, 0, sizeof tr);
                    tr.kind = kind;
                    tr.tensor = t;
                    tr.nd = s->t[t].nd;
                    for (int d = 0; d < tr.nd; ++d) { tr.lo[d] = reg->tb[t].v[b].d[d].lo; tr.hi[d] = reg->tb[t].v[b].d[d].hi; }
                    tr.src_rank = r->src_rank;
                    tr.dst_rank = r->dst_rank;
                    PUSH_RET(tr);
                }
            if (kind == 1)
                for (int64_t i = 0; i < reg->flat.n; ++i) {
                    or_transfer tr;
                    memset(&tr, 0, sizeof tr);
                    tr.kind = 1;
                    tr.tensor = -1;
                    tr.flat = 1;
                    tr.nd = 1;
                    tr.lo[0] = reg->flat.v[i].lo;
                    tr.hi[0] = reg->flat.v[i].hi;
                    tr.src_rank = r->src_rank;
                    tr.dst_rank = r->dst_rank;
                    PUSH_RET(tr);
                }
        }
    }
#undef PUSH_RET
    const int64_t kChunk = 1 << 20;
    for (int pass = 0; pass < 2; ++pass) {
        const or_transfer* arr = pass ? ret : p->tr;
        int64_t n = pass ? nret : p->ntr;
        for (int64_t i = 0; i < n; ++i) {
            const or_transfer* t = &arr[i];
            int64_t total, per;
            if (t->flat) { total = t->hi[0] - t->lo[0]; per = kChunk; }
            else {
                total = 1;
                for (int d = 0; d + 1 < t->nd; ++d) total *= t->hi[d] - t->lo[d];
                int64_t width = t->hi[t->nd - 1] - t->lo[t->nd - 1];
                per = kChunk / (width ? width : 1);
                if (per < 1) per = 1;
            }
            for (int64_t a = 0; a < total; a += per) {
                if (E.nw == cap) { cap *= 2; E.w = xrealloc(E.w, sizeof(work_t) * (size_t)cap); }
                int64_t b = a + per < total ? a + per : total;
                E.w[E.nw++] = t->flat ? (work_t){1, t, t->lo[0] + a, t->lo[0] + b} : (work_t){0, t, a, b};
            }
        }
    }
    pthread_mutex_init(&E.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = xrealloc(NULL, sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, exec_worker, &E);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&E.mu);
    /* scalar broadcast from src world rank 0 to every dst rank */
    if (p->has_scalars)
        for (int j = 0; j < dst->nranks; ++j)
            memcpy(dst->r[j].buf[5], src->r[0].buf[5], (size_t)(s->scalar_words * 8));
    free(E.w);
    free(ret);
    if (E.bad) { snprintf(err, errlen, "%s", E.msg); return 1; }
    return 0;
}

/* oracle_reshard: gather every element from any src replica,
 * then distribute by the dst layout. Ignores plans entirely. */
typedef struct { uint64_t* param; uint32_t *grad, *mst, *m, *v; uint8_t *has_p, *has_o; int64_t missing; } gather_t;
typedef struct { or_state* st; gather_t* g; } gctx;

static void gather_fn(void* cx, int rank, rstate_t* R, int si, int64_t e, int64_t k) {
    gctx* c = cx;
    (void)rank;
    seg_t* sg = rs_seg(R, si);
    int w = c->st->s->t[sg->t].dtype;
    c->g->param[k] = get_param(R->buf[0] + R->seg_byte_off[si] + e * w, w);
    c->g->has_p[k] = 1;
    int expert = si >= R->L.nd_;
    int64_t li = sg->lo + e;
    if (c->st->with_grads) memcpy(&c->g->grad[k], R->buf[4] + ((expert ? R->L.dense_len : 0) + li) * 4, 4);
    int64_t op = optim_pos(R, expert, li);
    if (op >= 0) {
        memcpy(&c->g->mst[k], R->buf[1] + op * 4, 4);
        memcpy(&c->g->m[k], R->buf[2] + op * 4, 4);
        memcpy(&c->g->v[k], R->buf[3] + op * 4, 4);
        c->g->has_o[k] = 1;
    }
}
static void scatter_fn(void* cx, int rank, rstate_t* R, int si, int64_t e, int64_t k) {
    gctx* c = cx;
    (void)rank;
    seg_t* sg = rs_seg(R, si);
    int w = c->st->s->t[sg->t].dtype;
    if (!c->g->has_p[k]) c->g->missing++;
    put_param(R->buf[0] + R->seg_byte_off[si] + e * w, w, c->g->param[k]);
    int expert = si >= R->L.nd_;
    int64_t li = sg->lo + e;
    if (c->st->with_grads) memcpy(R->buf[4] + ((expert ? R->L.dense_len : 0) + li) * 4, &c->g->grad[k], 4);
    int64_t op = optim_pos(R, expert, li);
    if (op >= 0) {
        if (!c->g->has_o[k]) c->g->missing++;
        memcpy(R->buf[1] + op * 4, &c->g->mst[k], 4);
        memcpy(R->buf[2] + op * 4, &c->g->m[k], 4);
        memcpy(R->buf[3] + op * 4, &c->g->v[k], 4);
    }
}

int or_oracle_reshard(const or_scenario* s, const or_state* src, or_state* dst, char* err, size_t errlen) {
    gather_t g;
    memset(&g, 0, sizeof g);
    size_t n = (size_t)(s->total ? s->total : 1);
    g.param = calloc(n, 8);
    g.grad = calloc(n, 4);
    g.mst = calloc(n, 4);
    g.m = calloc(n, 4);
    g.v = calloc(n, 4);
    g.has_p = calloc(n, 1);
    g.has_o = calloc(n, 1);
    gctx c1 = {(or_state*)src, &g};
    for (int r = 0; r < src->nranks; ++r) for_each_elem((or_state*)src, r, gather_fn, &c1);
    gctx c2 = {dst, &g};
    for (int r = 0; r < dst->nranks; ++r) {
        for_each_elem(dst, r, scatter_fn, &c2);
        memcpy(dst->r[r].buf[5], src->r[0].buf[5], (size_t)(s->scalar_words * 8));
    }
    free(g.param); free(g.grad); free(g.mst); free(g.m); free(g.v); free(g.has_p); free(g.has_o);
    if (g.missing) { snprintf(err, errlen, "%lld destination elements have no source", (long long)g.missing); return 1; }
    return 0;
}

int or_state_equal(const or_state* a, const or_state* b) {
    if (a->nranks != b->nranks) return 0;
    for (int r = 0; r < a->nranks; ++r)
        for (int k = 0; k < 6; ++k) {
            if (a->r[r].bytes[k] != b->r[r].bytes[k]) return 0;
            if (memcmp(a->r[r].buf[k], b->r[r].buf[k], (size_t)a->r[r].bytes[k])) return 0;
        }
    return 1;
}
