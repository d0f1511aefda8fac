/*
 * mwt_oracle.c -- CPU restatement of the reference ray-query hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_2112_05570_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the product
 * never links, imports or falls back to it.
 *
 * It restates, scalar fp64 with NO FMA contraction (built -ffp-contract=off),
 * the pure-Python reference package `mintri` (/root/reference/pkg/src/mintri):
 *   geometry.py:81-83   signed_area2
 *   geometry.py:136-166 ray_segment_intersect
 *   geometry.py:56-59   Segment.param_of
 *   accel.py:64-98      SceneIndex / canonical
 *   accel.py:101-132    brute_force_closest
 *   accel.py:138-213    traverse_triangulation (orc_trace_ex also returns the
 *                       final triangle: the loop variable `cur` when it returns)
 *   accel.py:219-353    _contains, _resolve_tie, locate_brute_force, TriLocator
 *   trimesh.py:386-436  Triangulation.locate (anchor seeds)
 *   accel.py:460-518    _ray_box, bvh_intersect
 *   accel.py:712-832    RopedKdTree.locate_leaf, kd_intersect
 * and the engine's own seeded ray generator (no reference counterpart; its
 * device twin lives in the CUDA engine, its numpy twin in oracle/raygen.py).
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if defined(__FP_FAST_FMA) && !defined(ORACLE_ALLOW_FMA)
/* the explicit fma() calls below are exact-product helpers only */
#endif

/* status bits: mirror include/mwt.h */
#define ST_ERROR 1u
#define ST_FALLBACK 2u
#define ST_GRAZING 4u
#define ST_CANON 8u
#define ST_PARALLEL 16u
#define ST_ZERO_SIDE 32u
#define ST_MULTI 64u
#define ST_LOC_TIE 128u
#define ST_LOC_BRUTE 256u
#define ST_LOC_OUTSIDE 512u
#define ST_OVERFLOW 1024u

#define INTERNAL (-1)

/* ------------------------------------------------------------------ */
/* correctly rounded hypot (Python's math.hypot is correctly rounded;  */
/* glibc's is not).  Exact decision by Shewchuk expansion arithmetic.  */

static void two_sum(double a, double b, double *s, double *e) {
    double x = a + b;
    double bv = x - a;
    double av = x - bv;
    *s = x;
    *e = (a - av) + (b - bv);
}

/* sign of the exact sum of n doubles */
static int exact_sign(const double *v, int n) {
    double h[32];
    int m = 0;
    for (int k = 0; k < n; k++) {
        double q = v[k];
        int mm = 0;
        for (int i = 0; i < m; i++) {
            double s, e;
            two_sum(q, h[i], &s, &e);
            if (e != 0.0) h[mm++] = e;
            q = s;
        }
        if (q != 0.0) h[mm++] = q;
        m = mm;
    }
    if (m == 0) return 0;
    return h[m - 1] > 0.0 ? 1 : -1;
}

/* sign of (x^2 + y^2) - (c + d)^2 with d = +-2^k exactly (midpoint test) */
static int cmp_mid(double x, double y, double c, double d) {
    double v[8];
    double sh = x * x, th = y * y;
    v[0] = sh;
    v[1] = fma(x, x, -sh);
    v[2] = th;
    v[3] = fma(y, y, -th);
    double ph = c * c;
    v[4] = -ph;
    v[5] = -fma(c, c, -ph);
    v[6] = -(2.0 * c * d); /* exact: c times a power of two */
    v[7] = -(d * d);       /* exact */
    return exact_sign(v, 8);
}

double orc_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return NAN;
    if (x < y) { double t = x; x = y; y = t; }
    if (y == 0.0) return x;
    double scale = 1.0;
    if (x > 0x1p+500) { x *= 0x1p-600; y *= 0x1p-600; scale = 0x1p+600; }
    else if (x < 0x1p-500) { x *= 0x1p+600; y *= 0x1p+600; scale = 0x1p-600; }
    double c = sqrt(x * x + y * y);
    for (int it = 0; it < 4; it++) {
        double up = nextafter(c, INFINITY);
        double dn = nextafter(c, 0.0);
        int su = cmp_mid(x, y, c, 0.5 * (up - c));
        if (su > 0) { c = up; continue; }
        int sd = cmp_mid(x, y, c, -0.5 * (c - dn));
        if (sd < 0) { c = dn; continue; }
        if (su == 0) { /* exact tie with the upper midpoint: round half even */
            uint64_t b; memcpy(&b, &c, 8);
            if (b & 1) c = up;
        } else if (sd == 0) {
            uint64_t b; memcpy(&b, &c, 8);
            if (b & 1) c = dn;
        }
        break;
    }
    return c * scale;
}

/* ------------------------------------------------------------------ */
/* seeded ray generator (engine-defined)  */

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
#define GOLDEN 0x9E3779B97F4A7C15ull

uint64_t orc_ray_key(uint64_t seed, uint64_t stream) {
    return mix64(mix64(seed + GOLDEN) ^ (stream * 0xD1B54A32D192ED03ull));
}
/* A mode word (include/mwt.h): base | group_log2 << 8 | cell_bits << 16.
 * Base 0: box-entry isotropic line rays; 1: interior origins.  With
 * cell_bits c > 0 ("coherent" order) every draw k of ray i takes the top c
 * bits of each 32-bit half from draw k of its group's stream (group =
 * i >> group_log2, stream key mix64(key ^ GROUP_SALT)). */
#define GROUP_SALT 0x6A09E667F3BCC909ull

typedef struct {
    int base, gshift;
    uint64_t cmask, key, gkey;
} orc_gen;

static int orc_gen_init(int mode, uint64_t seed, orc_gen *g) {
    unsigned w = (unsigned)mode, base = w & 0xFFu, gs = (w >> 8) & 0xFFu, c = (w >> 16) & 0xFFu;
    if ((w >> 24) || base > 1u || gs > 40u || c > 16u) return 0;
    uint64_t h = c ? (((1ull << c) - 1ull) << (32 - c)) : 0ull;
    g->base = (int)base;
    g->gshift = (int)gs;
    g->cmask = (h << 32) | h;
    g->key = orc_ray_key(seed, base);
    g->gkey = mix64(g->key ^ GROUP_SALT);
    return 1;
}

/* draw k of ray idx: mix64(s0 + (k + 1) * golden), group bits spliced in */
static inline uint64_t orc_draw(const orc_gen *g, uint64_t s0, uint64_t gs, unsigned k) {
    uint64_t z = mix64(s0 + (uint64_t)(k + 1) * GOLDEN);
    if (!g->cmask) return z;
    return (z & ~g->cmask) | (mix64(gs + (uint64_t)(k + 1) * GOLDEN) & g->cmask);
}

static void orc_raygen_gen(const orc_gen *g, const double box[4], uint64_t idx, double out[4]) {
    uint64_t s0 = g->key ^ idx; /* per-ray SplitMix64 stream: mix64(s0 + (k + 1) * golden) */
    uint64_t gs = g->gkey ^ (idx >> g->gshift);
    double x = 1.0, y = 0.0, r2 = 1.0;
    int ok = 0;
    for (int a = 0; a < 64; a++) {
        /* one 64-bit draw per attempt -> two 32-bit coordinates in [-1, 1) */
        uint64_t z = orc_draw(g, s0, gs, (unsigned)a);
        x = 2.0 * ((double)(uint32_t)(z >> 32) * 0x1p-32) - 1.0;
        y = 2.0 * ((double)(uint32_t)(z & 0xffffffffull) * 0x1p-32) - 1.0;
        r2 = x * x + y * y;
        if (r2 <= 1.0 && r2 > 0x1p-60) { ok = 1; break; }
    }
    double dx = 1.0, dy = 0.0;
    if (ok) { /* angle doubling: (x^2 - y^2, 2xy) / r2 */
        double inv = 1.0 / r2;
        dx = (x * x - y * y) * inv;
        dy = (2.0 * x * y) * inv;
    }
    double x0 = box[0], y0 = box[1], x1 = box[2], y1 = box[3];
    double W = x1 - x0, H = y1 - y0;
    uint64_t zuv = orc_draw(g, s0, gs, 128u); /* draw 128: u, v = its 32-bit halves * 2^-32 */
    double u = (double)(uint32_t)(zuv >> 32) * 0x1p-32, v = (double)(uint32_t)zuv * 0x1p-32;
    double ox, oy;
    if (g->base == 1) {
        ox = x0 + W * u;
        oy = y0 + H * v;
    } else {
        /* entry side by projected length, uniform position along it */
        double wx = H * fabs(dx), wy = W * fabs(dy);
        if (u * (wx + wy) < wx) {
            ox = dx > 0.0 ? x0 : x1;
            oy = y0 + H * v;
        } else {
            oy = dy > 0.0 ? y0 : y1;
            ox = x0 + W * v;
        }
    }
    out[0] = ox; out[1] = oy; out[2] = dx; out[3] = dy;
}

/* returns 0, or -1 for a malformed mode word */
int orc_raygen(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n, double *out) {
    orc_gen g;
    if (!orc_gen_init(mode, seed, &g)) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) orc_raygen_gen(&g, box, first + (uint64_t)i, out + 4 * i);
    return 0;
}

/* ------------------------------------------------------------------ */
/* mesh / scene model (reference data model, trimesh.py:39-60)          */

typedef struct {
    int nv, nt, ns;
    const double *vx, *vy;
    const int32_t *tv, *tn, *tf; /* 3 per triangle; tn -1 = None */
    const double *sax, *say, *sbx, *sby;
    const uint8_t *skind; /* 0 geometry, 1 boundary */
    /* SceneIndex.endpoint_map (accel.py:77-80) as a sorted table */
    int nep;
    double *epx, *epy;
    int32_t *epsid;
    /* TriLocator anchors (accel.py:263-282) */
    int res;
    int32_t *anchor;
} orc_mesh;

static inline double sa2(double ax, double ay, double bx, double by, double cx, double cy) {
    /* geometry.py:81-83 */
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
}

/* geometry.py:136-166; returns 1 and (t,u) on a forward hit; *par set when
 * the parallel branch was taken */
static int rsi(double ox, double oy, double dx, double dy,
               double ax, double ay, double bx, double by,
               double *t, double *u, int *par) {
    double ex = bx - ax, ey = by - ay;
    double denom = dx * ey - dy * ex;
    double wx = ax - ox, wy = ay - oy;
    if (denom == 0.0) {
        if (par) *par = 1;
        if (wx * dy - wy * dx != 0.0) return 0;
        double ta = wx * dx + wy * dy;
        double tb = (bx - ox) * dx + (by - oy) * dy;
        if (ta < 0.0 && tb < 0.0) return 0;
        if (ta < 0.0) { *t = tb; *u = 1.0; return 1; }
        if (tb < 0.0) { *t = ta; *u = 0.0; return 1; }
        if (ta <= tb) { *t = ta; *u = 0.0; } else { *t = tb; *u = 1.0; }
        return 1;
    }
    double tt = (wx * ey - wy * ex) / denom;
    double uu = (wx * dy - wy * dx) / denom;
    if (tt < 0.0 || uu < 0.0 || uu > 1.0) return 0;
    *t = tt;
    *u = uu;
    return 1;
}

int orc_ray_segment_intersect(const double ray[4], const double seg[4], double *t, double *u) {
    return rsi(ray[0], ray[1], ray[2], ray[3], seg[0], seg[1], seg[2], seg[3], t, u, NULL);
}

static int ep_cmp(const orc_mesh *m, int i, int j) {
    if (m->epx[i] < m->epx[j]) return -1;
    if (m->epx[i] > m->epx[j]) return 1;
    if (m->epy[i] < m->epy[j]) return -1;
    if (m->epy[i] > m->epy[j]) return 1;
    return m->epsid[i] < m->epsid[j] ? -1 : (m->epsid[i] > m->epsid[j]);
}

static void build_endpoints(orc_mesh *m) {
    int n = 0;
    for (int s = 0; s < m->ns; s++) n += m->skind[s] == 0 ? 2 : 0;
    m->nep = n;
    m->epx = (double *)malloc(sizeof(double) * (n + 1));
    m->epy = (double *)malloc(sizeof(double) * (n + 1));
    m->epsid = (int32_t *)malloc(sizeof(int32_t) * (n + 1));
    int k = 0;
    for (int s = 0; s < m->ns; s++) {
        if (m->skind[s] != 0) continue;
        m->epx[k] = m->sax[s]; m->epy[k] = m->say[s]; m->epsid[k] = s; k++;
        m->epx[k] = m->sbx[s]; m->epy[k] = m->sby[s]; m->epsid[k] = s; k++;
    }
    /* insertion sort is too slow for 30k; simple merge sort on an index */
    int *idx = (int *)malloc(sizeof(int) * (n + 1)), *tmp = (int *)malloc(sizeof(int) * (n + 1));
    for (int i = 0; i < n; i++) idx[i] = i;
    for (int w = 1; w < n; w *= 2) {
        for (int lo = 0; lo < n; lo += 2 * w) {
            int mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int a = lo, b = mid, o = lo;
            while (a < mid && b < hi) tmp[o++] = ep_cmp(m, idx[a], idx[b]) <= 0 ? idx[a++] : idx[b++];
            while (a < mid) tmp[o++] = idx[a++];
            while (b < hi) tmp[o++] = idx[b++];
        }
        int *sw = idx; idx = tmp; tmp = sw;
    }
    double *x2 = (double *)malloc(sizeof(double) * (n + 1)), *y2 = (double *)malloc(sizeof(double) * (n + 1));
    int32_t *s2 = (int32_t *)malloc(sizeof(int32_t) * (n + 1));
    for (int i = 0; i < n; i++) { x2[i] = m->epx[idx[i]]; y2[i] = m->epy[idx[i]]; s2[i] = m->epsid[idx[i]]; }
    free(m->epx); free(m->epy); free(m->epsid); free(idx); free(tmp);
    m->epx = x2; m->epy = y2; m->epsid = s2;
}

/* first index with (epx,epy) >= (x,y) */
static int ep_lower(const orc_mesh *m, double x, double y) {
    int lo = 0, hi = m->nep;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        int less = m->epx[mid] < x || (m->epx[mid] == x && m->epy[mid] < y);
        if (less) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* accel.py:82-98 */
static int canonical(const orc_mesh *m, const double ray[4], int sid, double t, double u,
                     double *ot, double *ou) {
    int best_sid = sid;
    double best_t = t, best_u = u;
    if (u <= 1e-9 || u >= 1.0 - 1e-9) {
        double px = u <= 1e-9 ? m->sax[sid] : m->sbx[sid];
        double py = u <= 1e-9 ? m->say[sid] : m->sby[sid];
        for (int k = ep_lower(m, px, py); k < m->nep && m->epx[k] == px && m->epy[k] == py; k++) {
            int sid2 = m->epsid[k];
            if (sid2 >= best_sid) continue;
            double t2, u2;
            if (!rsi(ray[0], ray[1], ray[2], ray[3], m->sax[sid2], m->say[sid2], m->sbx[sid2],
                     m->sby[sid2], &t2, &u2, NULL))
                continue;
            double at = fabs(t);
            if (fabs(t2 - t) <= 1e-9 * (at > 1.0 ? at : 1.0)) {
                best_sid = sid2; best_t = t2; best_u = u2;
            }
        }
    }
    *ot = best_t;
    *ou = best_u;
    return best_sid;
}

/* ------------------------------------------------------------------ */
/* triangulation walk, accel.py:138-213                                  */

static inline double side_of(const orc_mesh *m, int vid, double ox, double oy, double dx, double dy) {
    return dx * (m->vy[vid] - oy) - dy * (m->vx[vid] - ox);
}

/* returns status; *seg = -1 on a miss */
/* *end (may be NULL): the triangle the walk ended in -- the one whose exit
 * edge is constrained or has no neighbour (the loop variable `cur` of
 * accel.py:161-211 when it returns); -1 after a TraversalError */
uint32_t orc_trace_one(const orc_mesh *m, const double ray[4], int start, int *seg, double *tout,
                       double *uout, int *steps, int *end) {
    double ox = ray[0], oy = ray[1], dx = ray[2], dy = ray[3];
    uint32_t st = 0;
    int cur = start;
    int ea = -1, eb = -1; /* entry edge vertex pair (frozenset) */
    int nsteps = 0;
    long cap = 4L * m->nt + 16; /* > number of distinct (tri, entry) states */
    *seg = -1;
    *tout = NAN;
    *uout = NAN;
    for (;;) {
        if (nsteps >= cap) { st |= ST_ERROR; break; } /* revisit => TraversalError */
        nsteps++;
        const int32_t *v = m->tv + 3 * cur;
        int best_i = -1, fb_i = -1, ncand = 0;
        double best_trans = 0.0, fb_trans = 0.0;
        for (int i = 0; i < 3; i++) {
            int p = v[(i + 1) % 3], q = v[(i + 2) % 3];
            if (ea >= 0 && ((p == ea && q == eb) || (p == eb && q == ea))) continue;
            double sp = side_of(m, p, ox, oy, dx, dy), sq = side_of(m, q, ox, oy, dx, dy);
            double trans = sq - sp;
            if (trans > fb_trans) { fb_trans = trans; fb_i = i; }
            if (sp <= 0.0 && 0.0 <= sq) {
                ncand++;
                if (sp == 0.0 || sq == 0.0) st |= ST_ZERO_SIDE;
                if (trans > best_trans) { best_trans = trans; best_i = i; }
            }
        }
        if (ncand > 1) st |= ST_MULTI;
        if (best_i < 0) {
            best_i = fb_i;
            if (best_i >= 0) st |= ST_FALLBACK;
        }
        if (best_i < 0) { st |= ST_ERROR; break; }
        int flag = m->tf[3 * cur + best_i];
        int a = v[(best_i + 1) % 3], b = v[(best_i + 2) % 3];
        if (flag != INTERNAL) {
            if (m->skind[flag] != 0) break; /* boundary: no hit */
            double t, u;
            int par = 0;
            int ok = rsi(ox, oy, dx, dy, m->sax[flag], m->say[flag], m->sbx[flag], m->sby[flag], &t, &u, &par);
            if (par) st |= ST_PARALLEL;
            if (!ok) {
                st |= ST_GRAZING;
                double sp = side_of(m, a, ox, oy, dx, dy), sq = side_of(m, b, ox, oy, dx, dy);
                double w = sp != sq ? sp / (sp - sq) : 0.5;
                double x = m->vx[a] + w * (m->vx[b] - m->vx[a]);
                double y = m->vy[a] + w * (m->vy[b] - m->vy[a]);
                t = (x - ox) * dx + (y - oy) * dy;
                double ex = m->sbx[flag] - m->sax[flag], ey = m->sby[flag] - m->say[flag];
                u = ((x - m->sax[flag]) * ex + (y - m->say[flag]) * ey) / (ex * ex + ey * ey);
            }
            int s2 = canonical(m, ray, flag, t, u, tout, uout);
            if (s2 != flag) st |= ST_CANON;
            *seg = s2;
            break;
        }
        int nxt = m->tn[3 * cur + best_i];
        if (nxt < 0) break;
        ea = a;
        eb = b;
        cur = nxt;
    }
    *steps = nsteps;
    if (end) *end = (st & ST_ERROR) ? -1 : cur;
    return st;
}

/* ------------------------------------------------------------------ */
/* point location                                                       */

static int contains(const orc_mesh *m, int tid, double px, double py) {
    /* accel.py:219-223 */
    const int32_t *v = m->tv + 3 * tid;
    for (int i = 0; i < 3; i++) {
        int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
        if (!(sa2(m->vx[a], m->vy[a], m->vx[b], m->vy[b], px, py) >= -1e-15)) return 0;
    }
    return 1;
}

/* trimesh.py:386-416 (Triangulation.locate; tid only) */
static int tri_locate(const orc_mesh *m, double px, double py, int hint) {
    int tid = (hint >= 0 && hint < m->nt) ? hint : 0;
    long cap = 4L * m->nt + 16;
    for (long visited = 0; visited < cap; visited++) {
        const int32_t *v = m->tv + 3 * tid;
        int worst = -1;
        double worst_val = 0.0;
        for (int i = 0; i < 3; i++) {
            int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
            double s = sa2(m->vx[a], m->vy[a], m->vx[b], m->vy[b], px, py);
            if (s < worst_val) { worst_val = s; worst = i; }
        }
        if (worst < 0) return tid;
        int n = m->tn[3 * tid + worst];
        if (n < 0) return tid;
        tid = n;
    }
    /* _locate_scan, trimesh.py:428-436 */
    for (int t = 0; t < m->nt; t++)
        if (contains(m, t, px, py)) return t;
    return -1;
}

static void build_anchors(orc_mesh *m) {
    int nt = m->nt > 4 ? m->nt : 4;
    int res = (int)sqrt(nt / 2.0); /* accel.py:265-266 */
    if (res < 2) res = 2;
    m->res = res;
    m->anchor = (int32_t *)malloc(sizeof(int32_t) * res * res);
    int hint = -1;
    /* eager row-major fill with hint chaining (the reference fills lazily in
     * query order; both agree whenever a cell centre is strictly inside a
     * triangle -- checked by the engine's packer) */
    for (int cy = 0; cy < res; cy++)
        for (int cx = 0; cx < res; cx++) {
            double px = (cx + 0.5) / res, py = (cy + 0.5) / res;
            int tid = tri_locate(m, px, py, hint);
            hint = tid;
            m->anchor[cy * res + cx] = tid;
        }
}

/* accel.py:291-330 */
static int tl_walk(const orc_mesh *m, double sx, double sy, int tid, double px, double py) {
    double dx = px - sx, dy = py - sy;
    double norm = orc_hypot(dx, dy);
    if (norm == 0.0) return tid;
    dx = dx / norm;
    dy = dy / norm;
    int cur = tid, ea = -1, eb = -1;
    long cap = 4L * m->nt + 16;
    for (long it = 0; it < cap; it++) {
        if (contains(m, cur, px, py)) return cur;
        const int32_t *v = m->tv + 3 * cur;
        int best_i = -1;
        double best_trans = 0.0;
        for (int i = 0; i < 3; i++) {
            int p = v[(i + 1) % 3], q = v[(i + 2) % 3];
            if (ea >= 0 && ((p == ea && q == eb) || (p == eb && q == ea))) continue;
            double sp = dx * (m->vy[p] - sy) - dy * (m->vx[p] - sx);
            double sq = dx * (m->vy[q] - sy) - dy * (m->vx[q] - sx);
            if (sp <= 0.0 && 0.0 <= sq && sq - sp > best_trans) { best_trans = sq - sp; best_i = i; }
        }
        if (best_i < 0) return -1;
        int nxt = m->tn[3 * cur + best_i];
        if (nxt < 0) return -1;
        ea = v[(best_i + 1) % 3];
        eb = v[(best_i + 2) % 3];
        cur = nxt;
    }
    return -1;
}

/* accel.py:226-238; returns min tid; *nvis = flood size */
static int resolve_tie(const orc_mesh *m, int tid, double px, double py, int *nvis) {
    int cap = 64, n = 1, top = 1;
    int *seen = (int *)malloc(sizeof(int) * cap);
    int *stack = (int *)malloc(sizeof(int) * cap);
    seen[0] = tid;
    stack[0] = tid;
    int best = tid;
    while (top > 0) {
        int cur = stack[--top];
        if (cur < best) best = cur;
        for (int i = 0; i < 3; i++) {
            int nb = m->tn[3 * cur + i];
            if (nb < 0) continue;
            int dup = 0;
            for (int k = 0; k < n; k++) if (seen[k] == nb) { dup = 1; break; }
            if (dup || !contains(m, nb, px, py)) continue;
            if (n == cap) {
                cap *= 2;
                seen = (int *)realloc(seen, sizeof(int) * cap);
                stack = (int *)realloc(stack, sizeof(int) * cap);
            }
            seen[n++] = nb;
            stack[top++] = nb;
        }
    }
    free(seen);
    free(stack);
    *nvis = n;
    return best;
}

/* accel.py:241-253 */
static int locate_brute(const orc_mesh *m, double px, double py, uint32_t *st) {
    for (int t = 0; t < m->nt; t++)
        if (contains(m, t, px, py)) return t;
    *st |= ST_LOC_OUTSIDE;
    int best = 0;
    double bd = INFINITY;
    for (int t = 0; t < m->nt; t++) {
        const int32_t *v = m->tv + 3 * t;
        double cx = (m->vx[v[0]] + m->vx[v[1]] + m->vx[v[2]]) / 3.0;
        double cy = (m->vy[v[0]] + m->vy[v[1]] + m->vy[v[2]]) / 3.0;
        double d = orc_hypot(cx - px, cy - py);
        if (d < bd) { bd = d; best = t; }
    }
    return best;
}

/* TriLocator.locate, accel.py:284-289 */
int orc_locate_one(const orc_mesh *m, double px, double py, uint32_t *st) {
    int res = m->res;
    double vxr = px * res, vyr = py * res;
    int cx = vxr < 0.0 ? 0 : (vxr >= res ? res - 1 : (int)vxr);
    int cy = vyr < 0.0 ? 0 : (vyr >= res ? res - 1 : (int)vyr);
    if (!(vxr == vxr)) cx = 0; /* NaN guard */
    if (!(vyr == vyr)) cy = 0;
    double ax = (cx + 0.5) / res, ay = (cy + 0.5) / res;
    int cur = tl_walk(m, ax, ay, m->anchor[cy * res + cx], px, py);
    if (cur < 0 || !contains(m, cur, px, py)) {
        *st |= ST_LOC_BRUTE;
        cur = locate_brute(m, px, py, st);
    }
    int nvis = 1;
    int r = resolve_tie(m, cur, px, py, &nvis);
    if (nvis > 1) *st |= ST_LOC_TIE;
    return r;
}

/* ------------------------------------------------------------------ */
/* public oracle API                                                    */

void *orc_mesh_create(int nv, const double *vx, const double *vy, int nt, const int32_t *tv,
                      const int32_t *tn, const int32_t *tf, int ns, const double *sax, const double *say,
                      const double *sbx, const double *sby, const uint8_t *skind) {
    orc_mesh *m = (orc_mesh *)calloc(1, sizeof(orc_mesh));
    m->nv = nv; m->nt = nt; m->ns = ns;
    m->vx = vx; m->vy = vy; m->tv = tv; m->tn = tn; m->tf = tf;
    m->sax = sax; m->say = say; m->sbx = sbx; m->sby = sby; m->skind = skind;
    build_endpoints(m);
    if (nt > 0) build_anchors(m);
    return m;
}

void orc_mesh_destroy(void *h) {
    orc_mesh *m = (orc_mesh *)h;
    if (!m) return;
    free(m->epx); free(m->epy); free(m->epsid); free(m->anchor);
    free(m);
}

int orc_anchor_res(void *h) { return ((orc_mesh *)h)->res; }
void orc_anchors(void *h, int32_t *out) {
    orc_mesh *m = (orc_mesh *)h;
    memcpy(out, m->anchor, sizeof(int32_t) * m->res * m->res);
}

void orc_locate(void *h, const double *pts, int64_t n, int32_t *out_tid, uint32_t *out_st) {
    const orc_mesh *m = (const orc_mesh *)h;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        uint32_t st = 0;
        out_tid[i] = orc_locate_one(m, pts[2 * i], pts[2 * i + 1], &st);
        out_st[i] = st;
    }
}

/* start == NULL: locate each origin first (TriLocator.locate) */
void orc_trace_ex(void *h, const double *rays, const int32_t *start, int64_t n, int32_t *out_start,
                  int32_t *out_seg, double *out_t, double *out_u, int32_t *out_steps,
                  uint32_t *out_st, int32_t *out_end);

void orc_trace(void *h, const double *rays, const int32_t *start, int64_t n, int32_t *out_start,
               int32_t *out_seg, double *out_t, double *out_u, int32_t *out_steps, uint32_t *out_st) {
    orc_trace_ex(h, rays, start, n, out_start, out_seg, out_t, out_u, out_steps, out_st, NULL);
}

void orc_trace_ex(void *h, const double *rays, const int32_t *start, int64_t n, int32_t *out_start,
                  int32_t *out_seg, double *out_t, double *out_u, int32_t *out_steps,
                  uint32_t *out_st, int32_t *out_end) {
    const orc_mesh *m = (const orc_mesh *)h;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        const double *r = rays + 4 * i;
        uint32_t st = 0;
        int s = start ? start[i] : orc_locate_one(m, r[0], r[1], &st);
        if (out_start) out_start[i] = s;
        int seg = -1, steps = 0, end = -1;
        double t = NAN, u = NAN;
        if (s < 0 || s >= m->nt) st |= ST_ERROR; /* no such start triangle */
        else st |= orc_trace_one(m, r, s, &seg, &t, &u, &steps, &end);
        if (out_end) out_end[i] = end;
        out_seg[i] = seg;
        out_t[i] = t;
        if (out_u) out_u[i] = u;
        out_steps[i] = steps;
        out_st[i] = st;
    }
}

/* accel.py:101-132 */
void orc_brute_force(void *h, const double *rays, int64_t n, int32_t *out_seg, double *out_t, double *out_u) {
    const orc_mesh *m = (const orc_mesh *)h;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        const double *r = rays + 4 * i;
        double ox = r[0], oy = r[1], dx = r[2], dy = r[3];
        int have = 0, bsid = -1;
        double bt = 0.0, bu = 0.0;
        /* vectorised pass: first minimal t among valid (np.argmin) */
        for (int s = 0; s < m->ns; s++) {
            if (m->skind[s] != 0) continue;
            double ax = m->sax[s], ay = m->say[s];
            double ex = m->sbx[s] - ax, ey = m->sby[s] - ay;
            double wx = ax - ox, wy = ay - oy;
            double denom = dx * ey - dy * ex;
            if (denom == 0.0) continue;
            double t = (wx * ey - wy * ex) / denom;
            double u = (wx * dy - wy * dx) / denom;
            if (t >= 0.0 && u >= 0.0 && u <= 1.0 && (!have || t < bt)) {
                have = 1; bt = t; bsid = s; bu = u;
            }
        }
        /* collinear fallback */
        for (int s = 0; s < m->ns; s++) {
            if (m->skind[s] != 0) continue;
            double ax = m->sax[s], ay = m->say[s];
            double ex = m->sbx[s] - ax, ey = m->sby[s] - ay;
            double wx = ax - ox, wy = ay - oy;
            double denom = dx * ey - dy * ex;
            if (!(denom == 0.0 && wx * dy - wy * dx == 0.0)) continue;
            double t, u;
            if (rsi(ox, oy, dx, dy, ax, ay, m->sbx[s], m->sby[s], &t, &u, NULL) && (!have || t < bt)) {
                have = 1; bt = t; bsid = s; bu = u;
            }
        }
        if (!have) { out_seg[i] = -1; out_t[i] = NAN; if (out_u) out_u[i] = NAN; continue; }
        double t2, u2;
        out_seg[i] = canonical(m, r, bsid, bt, bu, &t2, &u2);
        out_t[i] = t2;
        if (out_u) out_u[i] = u2;
    }
}

/* ------------------------------------------------------------------ */
/* BVH, accel.py:460-518 (flattened: fixtures/gen_fixtures.py)          */

static int ray_box(double ox, double oy, double dx, double dy, const double *b, double *tn) {
    double tmin = 0.0, tmax = INFINITY;
    double o[2] = {ox, oy}, d[2] = {dx, dy}, lo[2] = {b[0], b[1]}, hi[2] = {b[2], b[3]};
    for (int k = 0; k < 2; k++) {
        if (d[k] == 0.0) {
            if (o[k] < lo[k] || o[k] > hi[k]) return 0;
            continue;
        }
        double t1 = (lo[k] - o[k]) / d[k], t2 = (hi[k] - o[k]) / d[k];
        if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
        tmin = t1 > tmin ? t1 : tmin; /* Python max(tmin, t1) */
        tmax = t2 < tmax ? t2 : tmax; /* Python min(tmax, t2) */
        if (tmin > tmax) return 0;
    }
    *tn = tmin;
    return 1;
}

typedef struct {
    int nnodes;
    const double *box; /* 4 per node */
    const int32_t *left, *right, *poff, *pcnt, *prims;
} orc_bvh;

void *orc_bvh_create(int nnodes, const double *box, const int32_t *left, const int32_t *right,
                     const int32_t *poff, const int32_t *pcnt, const int32_t *prims) {
    orc_bvh *b = (orc_bvh *)calloc(1, sizeof(orc_bvh));
    b->nnodes = nnodes; b->box = box; b->left = left; b->right = right;
    b->poff = poff; b->pcnt = pcnt; b->prims = prims;
    return b;
}
void orc_bvh_destroy(void *h) { free(h); }

void orc_bvh_trace(void *mh, void *bh, const double *rays, int64_t n, int32_t *out_seg, double *out_t,
                   double *out_u, int32_t *out_node_tests, int32_t *out_prim_tests) {
    const orc_mesh *m = (const orc_mesh *)mh;
    const orc_bvh *b = (const orc_bvh *)bh;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        const double *r = rays + 4 * i;
        double ox = r[0], oy = r[1], dx = r[2], dy = r[3];
        int nodes = 1, prims = 0, have = 0, bsid = -1;
        double bt = 0.0, bu = 0.0, tn;
        out_seg[i] = -1; out_t[i] = NAN; if (out_u) out_u[i] = NAN;
        if (ray_box(ox, oy, dx, dy, b->box, &tn)) {
            double st_t[256];
            int st_n[256], top = 0;
            st_t[top] = tn; st_n[top] = 0; top++;
            while (top > 0) {
                top--;
                double tnear = st_t[top];
                int node = st_n[top];
                if (have && tnear > bt + 1e-12) continue;
                if (b->left[node] < 0) {
                    for (int k = 0; k < b->pcnt[node]; k++) {
                        int sid = b->prims[b->poff[node] + k];
                        prims++;
                        double t, u;
                        if (!rsi(ox, oy, dx, dy, m->sax[sid], m->say[sid], m->sbx[sid], m->sby[sid], &t, &u, NULL))
                            continue;
                        if (!have || t < bt) { have = 1; bt = t; bsid = sid; bu = u; }
                    }
                    continue;
                }
                double ct[2];
                int cn[2], nc = 0;
                int ch[2] = {b->left[node], b->right[node]};
                for (int c = 0; c < 2; c++) {
                    nodes++;
                    double s;
                    if (ray_box(ox, oy, dx, dy, b->box + 4 * ch[c], &s) && (!have || s <= bt + 1e-12)) {
                        ct[nc] = s; cn[nc] = ch[c]; nc++;
                    }
                }
                /* stable sort descending then extend: equal keys keep order */
                if (nc == 2 && ct[1] > ct[0]) {
                    double tt = ct[0]; ct[0] = ct[1]; ct[1] = tt;
                    int tc = cn[0]; cn[0] = cn[1]; cn[1] = tc;
                }
                for (int c = 0; c < nc && top < 256; c++) { st_t[top] = ct[c]; st_n[top] = cn[c]; top++; }
            }
            if (have) {
                double t2, u2;
                out_seg[i] = canonical(m, r, bsid, bt, bu, &t2, &u2);
                out_t[i] = t2;
                if (out_u) out_u[i] = u2;
            }
        }
        out_node_tests[i] = nodes;
        out_prim_tests[i] = prims;
    }
}

/* ------------------------------------------------------------------ */
/* roped kd-tree, accel.py:712-832                                       */

typedef struct {
    int nnodes, nleaves;
    const int32_t *axis, *left, *right, *ropes, *rope_cost, *poff, *pcnt, *prims;
    const double *pos, *box;
} orc_kd;

void *orc_kd_create(int nnodes, int nleaves, const int32_t *axis, const double *pos, const int32_t *left,
                    const int32_t *right, const double *box, const int32_t *ropes, const int32_t *rope_cost,
                    const int32_t *poff, const int32_t *pcnt, const int32_t *prims) {
    orc_kd *k = (orc_kd *)calloc(1, sizeof(orc_kd));
    k->nnodes = nnodes; k->nleaves = nleaves; k->axis = axis; k->pos = pos; k->left = left;
    k->right = right; k->box = box; k->ropes = ropes; k->rope_cost = rope_cost;
    k->poff = poff; k->pcnt = pcnt; k->prims = prims;
    return k;
}
void orc_kd_destroy(void *h) { free(h); }

void orc_kd_trace(void *mh, void *kh, const double *rays, int64_t n, int32_t *out_seg, double *out_t,
                  double *out_u, int32_t *out_nodes, int32_t *out_ropes, int32_t *out_prims, uint32_t *out_st) {
    const orc_mesh *m = (const orc_mesh *)mh;
    const orc_kd *kd = (const orc_kd *)kh;
#pragma omp parallel
    {
        uint8_t *tested = (uint8_t *)calloc((size_t)m->ns + 1, 1);
        int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * ((size_t)m->ns + 1));
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; i++) {
            const double *r = rays + 4 * i;
            double ox = r[0], oy = r[1], dx = r[2], dy = r[3];
            int nodes = 0, ropes = 0, prims = 0, ntouched = 0, have = 0, bsid = -1;
            uint32_t st = 0;
            double bt = 0.0, bu = 0.0;
            out_seg[i] = -1; out_t[i] = NAN; if (out_u) out_u[i] = NAN;
            /* locate_leaf with direction tie-break (uncounted) */
            int cur = 0;
            while (kd->axis[cur] >= 0) {
                double coord = kd->axis[cur] == 0 ? ox : oy;
                if (coord < kd->pos[cur]) cur = kd->left[cur];
                else if (coord > kd->pos[cur]) cur = kd->right[cur];
                else {
                    double d = kd->axis[cur] == 0 ? dx : dy;
                    cur = d > 0.0 ? kd->right[cur] : kd->left[cur];
                }
            }
            long guard = 4L * kd->nleaves + 16;
            int done = 0;
            while (guard > 0) {
                guard--;
                nodes++;
                const double *bb = kd->box + 4 * cur;
                double t_exit = INFINITY;
                int side = -1;
                if (dx > 0.0) { double tx = (bb[2] - ox) / dx; if (tx < t_exit) { t_exit = tx; side = 1; } }
                else if (dx < 0.0) { double tx = (bb[0] - ox) / dx; if (tx < t_exit) { t_exit = tx; side = 0; } }
                if (dy > 0.0) { double ty = (bb[3] - oy) / dy; if (ty < t_exit) { t_exit = ty; side = 3; } }
                else if (dy < 0.0) { double ty = (bb[1] - oy) / dy; if (ty < t_exit) { t_exit = ty; side = 2; } }
                for (int k = 0; k < kd->pcnt[cur]; k++) {
                    int sid = kd->prims[kd->poff[cur] + k];
                    if (tested[sid]) continue;
                    tested[sid] = 1;
                    touched[ntouched++] = sid;
                    prims++;
                    double t, u;
                    if (!rsi(ox, oy, dx, dy, m->sax[sid], m->say[sid], m->sbx[sid], m->sby[sid], &t, &u, NULL))
                        continue;
                    if (!have || t < bt) { have = 1; bt = t; bsid = sid; bu = u; }
                }
                if (have && bt <= t_exit + 1e-12) {
                    double t2, u2;
                    out_seg[i] = canonical(m, r, bsid, bt, bu, &t2, &u2);
                    out_t[i] = t2;
                    if (out_u) out_u[i] = u2;
                    done = 1;
                    break;
                }
                if (side < 0) { done = 1; break; }
                int rope = kd->ropes[4 * cur + side];
                if (rope < 0) { done = 1; break; }
                ropes += kd->rope_cost[4 * cur + side];
                double px = ox + t_exit * dx, py = oy + t_exit * dy;
                int node = rope;
                while (kd->axis[node] >= 0) {
                    nodes++;
                    double coord = kd->axis[node] == 0 ? px : py;
                    if (coord < kd->pos[node]) node = kd->left[node];
                    else if (coord > kd->pos[node]) node = kd->right[node];
                    else {
                        double d = kd->axis[node] == 0 ? dx : dy;
                        node = d > 0.0 ? kd->right[node] : kd->left[node];
                    }
                }
                cur = node;
            }
            if (!done) st |= ST_ERROR;
            for (int k = 0; k < ntouched; k++) tested[touched[k]] = 0;
            out_nodes[i] = nodes; out_ropes[i] = ropes; out_prims[i] = prims; out_st[i] = st;
        }
        free(tested);
        free(touched);
    }
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* the thread count of later parallel regions (launchers such as torchrun set
   OMP_NUM_THREADS=1 per rank; the CPU baseline uses every host thread) */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
