// B200 (sm_100a) kernels of the batched 2D ray-query engine.
//
//   K2 raygen      seeded isotropic rays (engine-defined, twin: oracle/raygen.py)
//   K3 locate      TriLocator.locate            accel.py:219-330
//   K4 walk        traverse_triangulation       accel.py:138-213
//   K5 bvh         bvh_intersect                accel.py:460-518
//   K6 kd          kd_intersect                 accel.py:712-832
//   K7 histogram   per-ray results -> step / hit / status counters
//   brute          brute_force_closest          accel.py:101-132
//
// Bit-exactness: CPython evaluates every + - * / in IEEE binary64 with no
// fusion.  This translation unit is compiled with -fmad=false so no a*b+c is
// contracted; fma() appears only where an EXACT product error term is wanted
// (correctly rounded hypot).  Operation order follows the reference
// expression by expression.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "mwt_internal.h"

namespace mwt {

#define ST_ERROR MWT_ST_ERROR
#define ST_FALLBACK MWT_ST_FALLBACK
#define ST_GRAZING MWT_ST_GRAZING
#define ST_CANON MWT_ST_CANON
#define ST_PARALLEL MWT_ST_PARALLEL
#define ST_ZERO_SIDE MWT_ST_ZERO_SIDE
#define ST_MULTI MWT_ST_MULTI
#define ST_LOC_TIE MWT_ST_LOC_TIE
#define ST_LOC_BRUTE MWT_ST_LOC_BRUTE
#define ST_LOC_OUTSIDE MWT_ST_LOC_OUTSIDE
#define ST_OVERFLOW MWT_ST_OVERFLOW

constexpr int kThreads = 256;
constexpr int kFloodCap = 32;
constexpr int kBvhStack = 128;
constexpr int kKdMailbox = 512;

struct Ray {
    double ox, oy, dx, dy;
};

// 32-B read-only load as two 16-B vector loads (no __ldg overload for double4)
__device__ __forceinline__ double4 ldg4d(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// ---------------------------------------------------------------------------
// correctly rounded hypot (CPython's math.hypot is correctly rounded; the
// CUDA libm hypot is not).  Fast filtered decision; exact expansion fallback.

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    double x = a + b;
    double bv = x - a;
    double av = x - bv;
    s = x;
    e = (a - av) + (b - bv);
}

__device__ __noinline__ int exact_sign8(const double *v) {
    double h[16];
    int m = 0;
    for (int k = 0; k < 8; k++) {
        double q = v[k];
        int mm = 0;
        for (int i = 0; i < m; i++) {
            double s, e;
            two_sum(q, h[i], s, e);
            if (e != 0.0) h[mm++] = e;
            q = s;
        }
        if (q != 0.0) h[mm++] = q;
        m = mm;
    }
    if (m == 0) return 0;
    return h[m - 1] > 0.0 ? 1 : -1;
}

// sign of (x^2 + y^2) - (c + d)^2, d = +-2^k
__device__ __noinline__ int cmp_mid_exact(double x, double y, double c, double d) {
    double v[8];
    double sh = x * x, th = y * y, ph = c * c;
    v[0] = sh;
    v[1] = fma(x, x, -sh);
    v[2] = th;
    v[3] = fma(y, y, -th);
    v[4] = -ph;
    v[5] = -fma(c, c, -ph);
    v[6] = -(2.0 * c * d);
    v[7] = -(d * d);
    return exact_sign8(v);
}

__device__ double cr_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    if (isinf(x) || isinf(y)) return CUDART_INF;
    if (isnan(x) || isnan(y)) return CUDART_NAN;
    if (x < y) {
        double t = x;
        x = y;
        y = t;
    }
    if (y == 0.0) return x;
    double scale = 1.0;
    if (x > 0x1p+500) {
        x *= 0x1p-600; y *= 0x1p-600; scale = 0x1p+600;
    } else if (x < 0x1p-500) {
        x *= 0x1p+600; y *= 0x1p+600; scale = 0x1p-600;
    }
    double sh = x * x, sl = fma(x, x, -sh);
    double th = y * y, tl = fma(y, y, -th);
    double S, es;
    two_sum(sh, th, S, es);
    double c = sqrt(S);
    for (int it = 0; it < 4; it++) {
        double ph = c * c, pl = fma(c, c, -ph);
        double d1 = S - ph;  // exact: c*c within a few ulp of S (Sterbenz)
        double delta = d1 + (((es + sl) + tl) - pl);  // ~ (x^2+y^2) - c^2
        double up = nextafter(c, CUDART_INF), dn = nextafter(c, 0.0);
        double hu = 0.5 * (up - c), hd = 0.5 * (c - dn);
        double Tu = 2.0 * c * hu + hu * hu;  // (c+hu)^2 - c^2
        double Td = 2.0 * c * hd - hd * hd;  // c^2 - (c-hd)^2
        double margin = 0x1p-40 * Tu;
        if (delta > Tu + margin) { c = up; continue; }
        if (delta < -Td - margin) { c = dn; continue; }
        if (fabs(delta - Tu) <= margin || fabs(delta + Td) <= margin) {
            int su = cmp_mid_exact(x, y, c, hu);
            if (su > 0) { c = up; continue; }
            int sd = cmp_mid_exact(x, y, c, -hd);
            if (sd < 0) { c = dn; continue; }
            unsigned long long b = (unsigned long long)__double_as_longlong(c);
            if (su == 0 && (b & 1ull)) c = up;
            else if (sd == 0 && (b & 1ull)) c = dn;
        }
        break;
    }
    return c * scale;
}

// ---------------------------------------------------------------------------
// K2: ray generator (twin: oracle/raygen.py, oracle/mwt_oracle.c orc_raygen)

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static unsigned long long ray_key(unsigned long long seed, unsigned long long stream) {
    return mix64(mix64(seed + kGolden) ^ (stream * 0xD1B54A32D192ED03ull));
}

__device__ __forceinline__ double u01(unsigned long long s0, unsigned long long k) {
    return (double)(mix64(s0 + (k + 1ull) * kGolden) >> 11) * 0x1p-53;
}

struct Box {
    double x0, y0, x1, y1;
};

__device__ __forceinline__ Ray gen_ray(int mode, const Box &b, unsigned long long key,
                                       unsigned long long idx) {
    unsigned long long s0 = mix64(key ^ idx);
    double x = 1.0, y = 0.0, r2 = 1.0;
    bool ok = false;
    for (int a = 0; a < 64; a++) {
        x = 2.0 * u01(s0, 2 * a) - 1.0;
        y = 2.0 * u01(s0, 2 * a + 1) - 1.0;
        r2 = x * x + y * y;
        if (r2 <= 1.0 && r2 > 0x1p-60) { ok = true; break; }
    }
    Ray r;
    r.dx = 1.0;
    r.dy = 0.0;
    if (ok) {
        double n = sqrt(r2);
        r.dx = x / n;
        r.dy = y / n;
    }
    double W = b.x1 - b.x0, H = b.y1 - b.y0;
    if (mode == MWT_RAYS_INTERIOR) {
        r.ox = b.x0 + W * u01(s0, 128);
        r.oy = b.y0 + H * u01(s0, 129);
    } else {
        double cx = b.x0 + 0.5 * W, cy = b.y0 + 0.5 * H;
        double nx = -r.dy, ny = r.dx;
        double w = 0.5 * (fabs(nx) * W + fabs(ny) * H);
        double s = w * (2.0 * u01(s0, 128) - 1.0);
        double px = cx + s * nx, py = cy + s * ny;
        double tx = -CUDART_INF, ty = -CUDART_INF;
        if (r.dx > 0.0) tx = (b.x0 - px) / r.dx;
        else if (r.dx < 0.0) tx = (b.x1 - px) / r.dx;
        if (r.dy > 0.0) ty = (b.y0 - py) / r.dy;
        else if (r.dy < 0.0) ty = (b.y1 - py) / r.dy;
        if (tx >= ty) {
            r.ox = r.dx > 0.0 ? b.x0 : b.x1;
            double oy = py + tx * r.dy;
            r.oy = oy < b.y0 ? b.y0 : (oy > b.y1 ? b.y1 : oy);
        } else {
            r.oy = r.dy > 0.0 ? b.y0 : b.y1;
            double ox = px + ty * r.dx;
            r.ox = ox < b.x0 ? b.x0 : (ox > b.x1 ? b.x1 : ox);
        }
    }
    return r;
}

// ---------------------------------------------------------------------------
// geometry (geometry.py)

__device__ __forceinline__ double sa2(double2 a, double2 b, double px, double py) {
    // geometry.py:81-83 signed_area2(a, b, p)
    return (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);
}

__device__ __forceinline__ double side_of(const Ray &r, double2 v) {
    // accel.py:157
    return r.dx * (v.y - r.oy) - r.dy * (v.x - r.ox);
}

// geometry.py:136-166
__device__ __forceinline__ bool rsi(const Ray &r, double4 s, double &t, double &u, bool &par) {
    double ex = s.z - s.x, ey = s.w - s.y;
    double denom = r.dx * ey - r.dy * ex;
    double wx = s.x - r.ox, wy = s.y - r.oy;
    if (denom == 0.0) {
        par = true;
        if (wx * r.dy - wy * r.dx != 0.0) return false;
        double ta = wx * r.dx + wy * r.dy;
        double tb = (s.z - r.ox) * r.dx + (s.w - r.oy) * r.dy;
        if (ta < 0.0 && tb < 0.0) return false;
        if (ta < 0.0) { t = tb; u = 1.0; return true; }
        if (tb < 0.0) { t = ta; u = 0.0; return true; }
        if (ta <= tb) { t = ta; u = 0.0; } else { t = tb; u = 1.0; }
        return true;
    }
    double tt = (wx * ey - wy * ex) / denom;
    double uu = (wx * r.dy - wy * r.dx) / denom;
    if (tt < 0.0 || uu < 0.0 || uu > 1.0) return false;
    t = tt;
    u = uu;
    return true;
}

// accel.py:82-98 SceneIndex.canonical
__device__ int canonical(const MeshDev &M, const Ray &r, int sid, double t, double u, double &ot,
                         double &ou) {
    int best = sid;
    double bt = t, bu = u;
    if (u <= 1e-9 || u >= 1.0 - 1e-9) {
        int e = 2 * sid + (u <= 1e-9 ? 0 : 1);
        int2 rg = __ldg(M.ep_range + e);
        double at = fabs(t);
        double tol = 1e-9 * (at > 1.0 ? at : 1.0);
        for (int k = 0; k < rg.y; k++) {
            int sid2 = __ldg(M.ep_ids + rg.x + k);
            if (sid2 >= best) continue;
            double t2, u2;
            bool par = false;
            if (!rsi(r, ldg4d(M.seg + sid2), t2, u2, par)) continue;
            if (fabs(t2 - t) <= tol) {
                best = sid2;
                bt = t2;
                bu = u2;
            }
        }
    }
    ot = bt;
    ou = bu;
    return best;
}

__device__ __forceinline__ uint32_t pick(int4 L, int i) {
    return (uint32_t)(i == 0 ? L.x : (i == 1 ? L.y : L.z));
}

// ---------------------------------------------------------------------------
// K4: the walk, accel.py:138-213.  One ray per thread.  State between steps:
// current triangle, entry mirror j, and the side values (a, b) of the two
// shared corners; each step loads link[cur] (16 B) and the apex corner
// cxy[3*cur + j] (16 B), both addressed by (cur, j) only.

struct WalkOut {
    int seg, steps;
    double t, u;
};

__device__ __noinline__ void walk_terminal(const MeshDev &M, const Ray &r, int cur, int ei,
                                           uint32_t w, double sp, double sq, WalkOut &o,
                                           uint32_t &st) {
    if (w == kOpenWord || (w & kBoundaryBit)) return;  // no hit (accel.py:196-197, :210-211)
    int sid = (int)(w & kSidMask);
    double4 S = ldg4d(M.seg + sid);
    double t, u;
    bool par = false;
    bool ok = rsi(r, S, t, u, par);
    if (par) st |= ST_PARALLEL;
    if (!ok) {
        // grazing numerical corner, accel.py:199-207
        st |= ST_GRAZING;
        double2 pa = __ldg(M.cxy + 3 * cur + (ei + 1) % 3);
        double2 pb = __ldg(M.cxy + 3 * cur + (ei + 2) % 3);
        double wq = sp != sq ? sp / (sp - sq) : 0.5;
        double x = pa.x + wq * (pb.x - pa.x);
        double y = pa.y + wq * (pb.y - pa.y);
        t = (x - r.ox) * r.dx + (y - r.oy) * r.dy;
        double ex = S.z - S.x, ey = S.w - S.y;
        u = ((x - S.x) * ex + (y - S.y) * ey) / (ex * ex + ey * ey);  // Segment.param_of
    }
    int s2 = canonical(M, r, sid, t, u, o.t, o.u);
    if (s2 != sid) st |= ST_CANON;
    o.seg = s2;
}

__device__ __forceinline__ void walk(const MeshDev &M, const Ray &r, int start, WalkOut &o,
                                     uint32_t &st) {
    o.seg = -1;
    o.t = CUDART_NAN;
    o.u = CUDART_NAN;
    const long long cap = 4LL * M.nt + 16;
    int cur = start;
    long long steps = 1;
    int4 L = __ldg(M.link + cur);
    double2 P0 = __ldg(M.cxy + 3 * cur), P1 = __ldg(M.cxy + 3 * cur + 1),
            P2 = __ldg(M.cxy + 3 * cur + 2);
    double s0 = side_of(r, P0), s1 = side_of(r, P1), s2 = side_of(r, P2);
    // first triangle: edges 0 (s1,s2), 1 (s2,s0), 2 (s0,s1) in order, none skipped
    int best = -1, fb = -1, ncand = 0;
    double bt = 0.0, ft = 0.0;
#define MWT_SCAN(I, SP, SQ)                                     \
    {                                                           \
        double tr = (SQ) - (SP);                                \
        if (tr > ft) { ft = tr; fb = I; }                       \
        if ((SP) <= 0.0 && 0.0 <= (SQ)) {                       \
            ncand++;                                            \
            if ((SP) == 0.0 || (SQ) == 0.0) st |= ST_ZERO_SIDE; \
            if (tr > bt) { bt = tr; best = I; }                 \
        }                                                       \
    }
    MWT_SCAN(0, s1, s2)
    MWT_SCAN(1, s2, s0)
    MWT_SCAN(2, s0, s1)
#undef MWT_SCAN
    if (ncand > 1) st |= ST_MULTI;
    if (best < 0) {
        best = fb;
        if (best >= 0) st |= ST_FALLBACK;
    }
    if (best < 0) {
        st |= ST_ERROR;
        o.steps = 1;
        return;
    }
    double sp = best == 0 ? s1 : (best == 1 ? s2 : s0);
    double sq = best == 0 ? s2 : (best == 1 ? s0 : s1);
    int ei = best;
    uint32_t w = pick(L, best);
    while (!(w & kStopBit)) {
        if (steps >= cap) {  // revisited (triangle, entry) state => TraversalError
            st |= ST_ERROR;
            o.steps = (int)steps;
            return;
        }
        steps++;
        cur = (int)(w >> 2);
        int j = (int)(w & 3u);
        double a = sq, b = sp;  // sides of corners (j+1)%3 and (j+2)%3
        L = __ldg(M.link + cur);
        double c = side_of(r, __ldg(M.cxy + 3 * cur + j));
        // E1 = edge (j+1)%3: (sp, sq) = (b, c);  E2 = edge (j+2)%3: (c, a)
        // reference scan order: ascending edge index -> E2 first iff j == 1
        bool sw = (j == 1);
        double spF = sw ? c : b, sqF = sw ? a : c;
        double spS = sw ? b : c, sqS = sw ? c : a;
        double trF = sqF - spF, trS = sqS - spS;
        bool cF = spF <= 0.0 && 0.0 <= sqF;
        bool cS = spS <= 0.0 && 0.0 <= sqS;
        int eF = sw ? (j + 2) % 3 : (j + 1) % 3;
        int eS = sw ? (j + 1) % 3 : (j + 2) % 3;
        int sel = -1;
        double btr = 0.0;
        if (cF && trF > btr) { sel = 0; btr = trF; }
        if (cS && trS > btr) sel = 1;
        if (cF && cS) st |= ST_MULTI;
        if ((cF && (spF == 0.0 || sqF == 0.0)) || (cS && (spS == 0.0 || sqS == 0.0)))
            st |= ST_ZERO_SIDE;
        if (sel < 0) {
            double ftr = 0.0;
            if (trF > ftr) { sel = 0; ftr = trF; }
            if (trS > ftr) sel = 1;
            if (sel < 0) {
                st |= ST_ERROR;
                o.steps = (int)steps;
                return;
            }
            st |= ST_FALLBACK;
        }
        sp = sel ? spS : spF;
        sq = sel ? sqS : sqF;
        ei = sel ? eS : eF;
        w = pick(L, ei);
    }
    o.steps = (int)steps;
    walk_terminal(M, r, cur, ei, w, sp, sq, o, st);
}

// ---------------------------------------------------------------------------
// K3: point location, accel.py:219-330

__device__ __forceinline__ void corners(const MeshDev &M, int t, double2 &P0, double2 &P1,
                                        double2 &P2) {
    P0 = __ldg(M.cxy + 3 * t);
    P1 = __ldg(M.cxy + 3 * t + 1);
    P2 = __ldg(M.cxy + 3 * t + 2);
}

__device__ __forceinline__ bool contains3(double2 P0, double2 P1, double2 P2, double px, double py,
                                          double &e0, double &e1, double &e2) {
    // accel.py:219-223 (all three evaluated; no side effects)
    e0 = sa2(P1, P2, px, py);
    e1 = sa2(P2, P0, px, py);
    e2 = sa2(P0, P1, px, py);
    return e0 >= -1e-15 && e1 >= -1e-15 && e2 >= -1e-15;
}

__device__ __forceinline__ bool contains_t(const MeshDev &M, int t, double px, double py) {
    double2 P0, P1, P2;
    corners(M, t, P0, P1, P2);
    double e0, e1, e2;
    return contains3(P0, P1, P2, px, py, e0, e1, e2);
}

// TriLocator._walk, accel.py:291-330
__device__ int loc_walk(const MeshDev &M, double sx, double sy, int tid, double px, double py) {
    double dx = px - sx, dy = py - sy;
    double norm = cr_hypot(dx, dy);
    if (norm == 0.0) return tid;
    dx = dx / norm;
    dy = dy / norm;
    int cur = tid, ent = -1;
    const long long cap = 4LL * M.nt + 16;
    for (long long it = 0; it < cap; it++) {
        double2 P[3];
        corners(M, cur, P[0], P[1], P[2]);
        double e0, e1, e2;
        if (contains3(P[0], P[1], P[2], px, py, e0, e1, e2)) return cur;
        int4 NB = __ldg(M.lnbr + cur);
        double s[3];
#pragma unroll
        for (int k = 0; k < 3; k++) s[k] = dx * (P[k].y - sy) - dy * (P[k].x - sx);
        int best = -1;
        double bt = 0.0;
#pragma unroll
        for (int i = 0; i < 3; i++) {
            if (i == ent) continue;
            double spv = s[(i + 1) % 3], sqv = s[(i + 2) % 3];
            if (spv <= 0.0 && 0.0 <= sqv && sqv - spv > bt) {
                bt = sqv - spv;
                best = i;
            }
        }
        if (best < 0) return -1;
        int word = (int)pick(NB, best);
        if (word < 0) return -1;
        cur = word >> 2;
        ent = word & 3;
    }
    return -1;
}

// locate_brute_force, accel.py:241-253
__device__ __noinline__ int loc_brute(const MeshDev &M, double px, double py, uint32_t &st) {
    for (int t = 0; t < M.nt; t++)
        if (contains_t(M, t, px, py)) return t;
    st |= ST_LOC_OUTSIDE;
    int best = 0;
    double bd = CUDART_INF;
    for (int t = 0; t < M.nt; t++) {
        double2 P0, P1, P2;
        corners(M, t, P0, P1, P2);
        double cx = ((P0.x + P1.x) + P2.x) / 3.0;
        double cy = ((P0.y + P1.y) + P2.y) / 3.0;
        double d = cr_hypot(cx - px, cy - py);
        if (d < bd) {
            bd = d;
            best = t;
        }
    }
    return best;
}

// _resolve_tie, accel.py:226-238: min tid over the neighbour-connected set of
// triangles containing p.  A neighbour across edge i can contain p only if
// this triangle's own value for edge i is <= ~1e-14 (the two are rounded
// negations of one exact number), so larger values skip the exact test.
__device__ int flood(const MeshDev &M, int tid, double px, double py, bool filt, uint32_t &st) {
    int seen[kFloodCap];
    int stack[kFloodCap];
    int nseen = 1, top = 1, best = tid;
    seen[0] = tid;
    stack[0] = tid;
    while (top > 0) {
        int cur = stack[--top];
        if (cur < best) best = cur;
        double2 P0, P1, P2;
        corners(M, cur, P0, P1, P2);
        double e[3];
        contains3(P0, P1, P2, px, py, e[0], e[1], e[2]);
        int4 NB = __ldg(M.lnbr + cur);
#pragma unroll
        for (int i = 0; i < 3; i++) {
            int word = (int)pick(NB, i);
            if (word < 0) continue;
            if (filt && e[i] > 1e-12) continue;
            int nb = word >> 2;
            bool dup = false;
            for (int k = 0; k < nseen; k++) dup |= (seen[k] == nb);
            if (dup || !contains_t(M, nb, px, py)) continue;
            if (nseen == kFloodCap) {
                st |= ST_OVERFLOW;
                return best;
            }
            seen[nseen++] = nb;
            stack[top++] = nb;
        }
    }
    if (nseen > 1) st |= ST_LOC_TIE;
    return best;
}

// TriLocator.locate, accel.py:284-289
__device__ int locate(const MeshDev &M, double px, double py, uint32_t &st) {
    int res = M.res;
    double dres = (double)res;
    double vx = px * dres, vy = py * dres;
    int cx = vx < 0.0 ? 0 : (vx >= dres ? res - 1 : (int)vx);
    int cy = vy < 0.0 ? 0 : (vy >= dres ? res - 1 : (int)vy);
    if (!(vx == vx)) cx = 0;
    if (!(vy == vy)) cy = 0;
    double ax = ((double)cx + 0.5) / dres, ay = ((double)cy + 0.5) / dres;
    int cur = loc_walk(M, ax, ay, __ldg(M.anchor + cy * res + cx), px, py);
    if (cur < 0 || !contains_t(M, cur, px, py)) {
        st |= ST_LOC_BRUTE;
        cur = loc_brute(M, px, py, st);
    }
    bool filt = fabs(px) <= 4.0 && fabs(py) <= 4.0;
    return flood(M, cur, px, py, filt, st);
}

// ---------------------------------------------------------------------------
// kernels

__device__ __forceinline__ Ray load_ray(const double *rays, long long i) {
    const double2 *p = reinterpret_cast<const double2 *>(rays) + 2 * i;
    double2 a = __ldg(p), b = __ldg(p + 1);
    Ray r;
    r.ox = a.x;
    r.oy = a.y;
    r.dx = b.x;
    r.dy = b.y;
    return r;
}

__global__ void __launch_bounds__(kThreads) k_raygen(int mode, Box box, unsigned long long key,
                                                     unsigned long long first, long long n,
                                                     double *rays) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = gen_ray(mode, box, key, first + (unsigned long long)i);
        double2 *p = reinterpret_cast<double2 *>(rays) + 2 * i;
        p[0] = make_double2(r.ox, r.oy);
        p[1] = make_double2(r.dx, r.dy);
    }
}

__global__ void __launch_bounds__(kThreads) k_locate(MeshDev M, const double *pts, long long n,
                                                     int32_t *tid, uint32_t *st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double2 p = __ldg(reinterpret_cast<const double2 *>(pts) + i);
        uint32_t s = 0;
        int t = locate(M, p.x, p.y, s);
        if (tid) tid[i] = t;
        if (st) st[i] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_trace(MeshDev M, const double *rays,
                                                    const int32_t *start, long long n,
                                                    int32_t *o_start, int32_t *o_seg, double *o_t,
                                                    double *o_u, int32_t *o_steps, uint32_t *o_st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = load_ray(rays, i);
        uint32_t st = 0;
        int s = start ? __ldg(start + i) : locate(M, r.ox, r.oy, st);
        WalkOut o;
        if (s < 0 || s >= M.nt) {
            st |= ST_ERROR;
            o.seg = -1; o.t = CUDART_NAN; o.u = CUDART_NAN; o.steps = 0;
        } else {
            walk(M, r, s, o, st);
        }
        if (o_start) o_start[i] = s;
        if (o_seg) o_seg[i] = o.seg;
        if (o_t) o_t[i] = o.t;
        if (o_u) o_u[i] = o.u;
        if (o_steps) o_steps[i] = o.steps;
        if (o_st) o_st[i] = st;
    }
}

// K7 histogram accumulation (block-private shared counters, one global flush)
struct BlockHist {
    unsigned int *h;  // shared, MWT_HIST_LEN
};

__device__ __forceinline__ void hist_init(unsigned int *h) {
    for (int k = threadIdx.x; k < MWT_HIST_LEN; k += blockDim.x) h[k] = 0u;
    __syncthreads();
}

__device__ __forceinline__ void hist_add(unsigned int *h, int seg, int steps, uint32_t st) {
    int bin = steps < MWT_HIST_STEP_BINS - 1 ? (steps < 0 ? 0 : steps) : MWT_HIST_STEP_BINS - 1;
    atomicAdd(h + bin, 1u);
    atomicAdd(h + (seg >= 0 ? MWT_HIST_HIT : MWT_HIST_MISS), 1u);
    if (st) {
        for (int b = 0; b < 11; b++)
            if (st & (1u << b)) atomicAdd(h + MWT_HIST_STATUS0 + b, 1u);
    }
}

__device__ __forceinline__ void hist_flush(unsigned int *h, unsigned long long steps_sum,
                                           long long *hist) {
    // warp-reduce the 64-bit step sum
    for (int o = 16; o > 0; o >>= 1) steps_sum += __shfl_down_sync(0xffffffffu, steps_sum, o);
    if ((threadIdx.x & 31) == 0 && steps_sum)
        atomicAdd(reinterpret_cast<unsigned long long *>(hist + MWT_HIST_STEPS_SUM), steps_sum);
    __syncthreads();
    for (int k = threadIdx.x; k < MWT_HIST_LEN; k += blockDim.x)
        if (h[k] && k != MWT_HIST_STEPS_SUM)
            atomicAdd(reinterpret_cast<unsigned long long *>(hist + k), (unsigned long long)h[k]);
}

__global__ void __launch_bounds__(kThreads) k_trace_generated(MeshDev M, int mode, Box box,
                                                              unsigned long long key,
                                                              unsigned long long first, long long n,
                                                              int32_t *o_seg, double *o_t,
                                                              int32_t *o_steps, long long *hist) {
    __shared__ unsigned int h[MWT_HIST_LEN];
    if (hist) hist_init(h);
    unsigned long long steps_sum = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = gen_ray(mode, box, key, first + (unsigned long long)i);
        uint32_t st = 0;
        int s = locate(M, r.ox, r.oy, st);
        WalkOut o;
        walk(M, r, s, o, st);
        if (o_seg) o_seg[i] = o.seg;
        if (o_t) o_t[i] = o.t;
        if (o_steps) o_steps[i] = o.steps;
        if (hist) {
            hist_add(h, o.seg, o.steps, st);
            steps_sum += (unsigned long long)o.steps;
        }
    }
    if (hist) hist_flush(h, steps_sum, hist);
}

__global__ void __launch_bounds__(kThreads) k_histogram(const int32_t *seg, const int32_t *steps,
                                                        const uint32_t *status, long long n,
                                                        long long *hist) {
    __shared__ unsigned int h[MWT_HIST_LEN];
    hist_init(h);
    unsigned long long steps_sum = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int s = steps[i];
        hist_add(h, seg[i], s, status ? status[i] : 0u);
        steps_sum += (unsigned long long)(s > 0 ? s : 0);
    }
    hist_flush(h, steps_sum, hist);
}

// ---------------------------------------------------------------------------
// K5: BVH, accel.py:460-518

__device__ __forceinline__ bool ray_box(const Ray &r, double4 b, double &tn) {
    double tmin = 0.0, tmax = CUDART_INF;
    // x slab then y slab; Python max/min keep the first operand on ties
    if (r.dx == 0.0) {
        if (r.ox < b.x || r.ox > b.z) return false;
    } else {
        double t1 = (b.x - r.ox) / r.dx, t2 = (b.z - r.ox) / r.dx;
        if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
        tmin = t1 > tmin ? t1 : tmin;
        tmax = t2 < tmax ? t2 : tmax;
        if (tmin > tmax) return false;
    }
    if (r.dy == 0.0) {
        if (r.oy < b.y || r.oy > b.w) return false;
    } else {
        double t1 = (b.y - r.oy) / r.dy, t2 = (b.w - r.oy) / r.dy;
        if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
        tmin = t1 > tmin ? t1 : tmin;
        tmax = t2 < tmax ? t2 : tmax;
        if (tmin > tmax) return false;
    }
    tn = tmin;
    return true;
}

__global__ void __launch_bounds__(kThreads) k_bvh(MeshDev M, BvhDev B, const double *rays,
                                                  long long n, int32_t *o_seg, double *o_t,
                                                  double *o_u, int32_t *o_nodes, int32_t *o_prims,
                                                  uint32_t *o_st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = load_ray(rays, i);
        int nodes = 1, prims = 0, bsid = -1;
        bool have = false;
        uint32_t st = 0;
        double bt = 0.0, bu = 0.0, tn;
        int seg = -1;
        double ot = CUDART_NAN, ou = CUDART_NAN;
        if (ray_box(r, ldg4d(B.box), tn)) {
            double st_t[kBvhStack];
            int st_n[kBvhStack];
            int top = 0;
            st_t[0] = tn;
            st_n[0] = 0;
            top = 1;
            while (top > 0) {
                top--;
                double tnear = st_t[top];
                int node = st_n[top];
                if (have && tnear > bt + 1e-12) continue;
                int2 ch = __ldg(B.child + node);
                if (ch.x < 0) {
                    int2 pr = __ldg(B.prange + node);
                    for (int k = 0; k < pr.y; k++) {
                        int sid = __ldg(B.prims + pr.x + k);
                        prims++;
                        double t, u;
                        bool par = false;
                        if (!rsi(r, ldg4d(M.seg + sid), t, u, par)) continue;
                        if (!have || t < bt) { have = true; bt = t; bsid = sid; bu = u; }
                    }
                    continue;
                }
                double tl = 0.0, tr = 0.0;
                nodes += 2;
                bool hl = ray_box(r, ldg4d(B.box + ch.x), tl) && (!have || tl <= bt + 1e-12);
                bool hr = ray_box(r, ldg4d(B.box + ch.y), tr) && (!have || tr <= bt + 1e-12);
                if (top + 2 > kBvhStack) { st |= ST_OVERFLOW; break; }
                // children sorted by tnear descending (stable) then pushed: the
                // nearer pops first; on equal tnear the right child pops first
                if (hl && hr) {
                    if (tr > tl) {
                        st_t[top] = tr; st_n[top] = ch.y; top++;
                        st_t[top] = tl; st_n[top] = ch.x; top++;
                    } else {
                        st_t[top] = tl; st_n[top] = ch.x; top++;
                        st_t[top] = tr; st_n[top] = ch.y; top++;
                    }
                } else if (hl) {
                    st_t[top] = tl; st_n[top] = ch.x; top++;
                } else if (hr) {
                    st_t[top] = tr; st_n[top] = ch.y; top++;
                }
            }
            if (have) seg = canonical(M, r, bsid, bt, bu, ot, ou);
        }
        if (o_seg) o_seg[i] = seg;
        if (o_t) o_t[i] = ot;
        if (o_u) o_u[i] = ou;
        if (o_nodes) o_nodes[i] = nodes;
        if (o_prims) o_prims[i] = prims;
        if (o_st) o_st[i] = st;
    }
}

// ---------------------------------------------------------------------------
// K6: roped kd-tree, accel.py:712-832

__device__ __forceinline__ int kd_descend(const KdDev &K, int node, double px, double py, double dx,
                                          double dy, int &nodes, bool count) {
    int a;
    while ((a = __ldg(K.axis + node)) >= 0) {
        if (count) nodes++;
        double coord = a == 0 ? px : py;
        double pos = __ldg(K.pos + node);
        int2 ch = __ldg(K.child + node);
        if (coord < pos) node = ch.x;
        else if (coord > pos) node = ch.y;
        else {
            double d = a == 0 ? dx : dy;
            node = d > 0.0 ? ch.y : ch.x;
        }
    }
    return node;
}

__global__ void __launch_bounds__(kThreads) k_kd(MeshDev M, KdDev K, const double *rays,
                                                 long long n, int32_t *o_seg, double *o_t,
                                                 double *o_u, int32_t *o_nodes, int32_t *o_ropes,
                                                 int32_t *o_prims, uint32_t *o_st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = load_ray(rays, i);
        int nodes = 0, ropes = 0, prims = 0, bsid = -1, seg = -1;
        bool have = false, done = false;
        uint32_t st = 0;
        double bt = 0.0, bu = 0.0, ot = CUDART_NAN, ou = CUDART_NAN;
        int tested[kKdMailbox];
        int ntested = 0;
        int dummy = 0;
        int cur = kd_descend(K, 0, r.ox, r.oy, r.dx, r.dy, dummy, false);  // locate_leaf
        long long guard = 4LL * K.nleaves + 16;
        while (guard > 0 && !done) {
            guard--;
            nodes++;
            double4 bb = ldg4d(K.box + cur);
            double t_exit = CUDART_INF;
            int side = -1;
            if (r.dx > 0.0) {
                double tx = (bb.z - r.ox) / r.dx;
                if (tx < t_exit) { t_exit = tx; side = 1; }
            } else if (r.dx < 0.0) {
                double tx = (bb.x - r.ox) / r.dx;
                if (tx < t_exit) { t_exit = tx; side = 0; }
            }
            if (r.dy > 0.0) {
                double ty = (bb.w - r.oy) / r.dy;
                if (ty < t_exit) { t_exit = ty; side = 3; }
            } else if (r.dy < 0.0) {
                double ty = (bb.y - r.oy) / r.dy;
                if (ty < t_exit) { t_exit = ty; side = 2; }
            }
            int2 pr = __ldg(K.prange + cur);
            for (int k = 0; k < pr.y; k++) {
                int sid = __ldg(K.prims + pr.x + k);
                bool dup = false;
                for (int q = 0; q < ntested; q++) dup |= (tested[q] == sid);
                if (dup) continue;
                if (ntested == kKdMailbox) { st |= ST_OVERFLOW; done = true; break; }
                tested[ntested++] = sid;
                prims++;
                double t, u;
                bool par = false;
                if (!rsi(r, ldg4d(M.seg + sid), t, u, par)) continue;
                if (!have || t < bt) { have = true; bt = t; bsid = sid; bu = u; }
            }
            if (done) break;
            if (have && bt <= t_exit + 1e-12) {
                seg = canonical(M, r, bsid, bt, bu, ot, ou);
                done = true;
                break;
            }
            if (side < 0) { done = true; break; }
            int rope = ((const int *)(K.ropes + cur))[side];
            if (rope < 0) { done = true; break; }
            ropes += ((const int *)(K.rope_cost + cur))[side];
            double px = r.ox + t_exit * r.dx, py = r.oy + t_exit * r.dy;
            cur = kd_descend(K, rope, px, py, r.dx, r.dy, nodes, true);
        }
        if (!done) st |= ST_ERROR;
        if (o_seg) o_seg[i] = seg;
        if (o_t) o_t[i] = ot;
        if (o_u) o_u[i] = ou;
        if (o_nodes) o_nodes[i] = nodes;
        if (o_ropes) o_ropes[i] = ropes;
        if (o_prims) o_prims[i] = prims;
        if (o_st) o_st[i] = st;
    }
}

// ---------------------------------------------------------------------------
// brute force, accel.py:101-132

__global__ void __launch_bounds__(kThreads) k_brute(MeshDev M, const double *rays, long long n,
                                                    int32_t *o_seg, double *o_t, double *o_u) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = load_ray(rays, i);
        bool have = false;
        int bsid = -1;
        double bt = 0.0, bu = 0.0;
        for (int s = 0; s < M.ns; s++) {
            if (__ldg(M.segkind + s) != 0) continue;
            double4 S = ldg4d(M.seg + s);
            double ex = S.z - S.x, ey = S.w - S.y;
            double wx = S.x - r.ox, wy = S.y - r.oy;
            double denom = r.dx * ey - r.dy * ex;
            if (denom == 0.0) continue;
            double t = (wx * ey - wy * ex) / denom;
            double u = (wx * r.dy - wy * r.dx) / denom;
            if (t >= 0.0 && u >= 0.0 && u <= 1.0 && (!have || t < bt)) {
                have = true; bt = t; bsid = s; bu = u;
            }
        }
        for (int s = 0; s < M.ns; s++) {  // collinear fallback
            if (__ldg(M.segkind + s) != 0) continue;
            double4 S = ldg4d(M.seg + s);
            double ex = S.z - S.x, ey = S.w - S.y;
            double wx = S.x - r.ox, wy = S.y - r.oy;
            double denom = r.dx * ey - r.dy * ex;
            if (!(denom == 0.0 && wx * r.dy - wy * r.dx == 0.0)) continue;
            double t, u;
            bool par = false;
            if (rsi(r, S, t, u, par) && (!have || t < bt)) {
                have = true; bt = t; bsid = s; bu = u;
            }
        }
        int seg = -1;
        double ot = CUDART_NAN, ou = CUDART_NAN;
        if (have) seg = canonical(M, r, bsid, bt, bu, ot, ou);
        if (o_seg) o_seg[i] = seg;
        if (o_t) o_t[i] = ot;
        if (o_u) o_u[i] = ou;
    }
}

// ---------------------------------------------------------------------------
// launchers

static int grid_for(long long n) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    long long blocks = (n + kThreads - 1) / kThreads;
    long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

#define MWT_LAUNCH_RET return (int)cudaGetLastError()

int launch_raygen(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n,
                  double *rays, void *stream) {
    if (n <= 0) return 0;
    Box b{box[0], box[1], box[2], box[3]};
    k_raygen<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(mode, b, ray_key(seed, mode), first,
                                                                 n, rays);
    MWT_LAUNCH_RET;
}

int launch_locate(const MeshDev &m, const double *pts, int64_t n, int32_t *tid, uint32_t *st,
                  void *stream) {
    if (n <= 0) return 0;
    k_locate<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, pts, n, tid, st);
    MWT_LAUNCH_RET;
}

int launch_trace(const MeshDev &m, const double *rays, const int32_t *start, int64_t n,
                 int32_t *o_start, int32_t *o_seg, double *o_t, double *o_u, int32_t *o_steps,
                 uint32_t *o_st, void *stream) {
    if (n <= 0) return 0;
    k_trace<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, rays, start, n, o_start, o_seg,
                                                                o_t, o_u, o_steps, o_st);
    MWT_LAUNCH_RET;
}

int launch_trace_generated(const MeshDev &m, int mode, const double *box, uint64_t seed,
                           uint64_t first, int64_t n, int32_t *o_seg, double *o_t,
                           int32_t *o_steps, long long *hist, void *stream) {
    if (n <= 0) return 0;
    Box b{box[0], box[1], box[2], box[3]};
    k_trace_generated<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        m, mode, b, ray_key(seed, mode), first, n, o_seg, o_t, o_steps, hist);
    MWT_LAUNCH_RET;
}

int launch_histogram(const int32_t *seg, const int32_t *steps, const uint32_t *st, int64_t n,
                     long long *hist, void *stream) {
    if (n <= 0) return 0;
    k_histogram<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(seg, steps, st, n, hist);
    MWT_LAUNCH_RET;
}

int launch_bvh(const MeshDev &m, const BvhDev &b, const double *rays, int64_t n, int32_t *o_seg,
               double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_prims, uint32_t *o_st,
               void *stream) {
    if (n <= 0) return 0;
    k_bvh<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, b, rays, n, o_seg, o_t, o_u,
                                                              o_nodes, o_prims, o_st);
    MWT_LAUNCH_RET;
}

int launch_kd(const MeshDev &m, const KdDev &k, const double *rays, int64_t n, int32_t *o_seg,
              double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_ropes, int32_t *o_prims,
              uint32_t *o_st, void *stream) {
    if (n <= 0) return 0;
    k_kd<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, k, rays, n, o_seg, o_t, o_u,
                                                             o_nodes, o_ropes, o_prims, o_st);
    MWT_LAUNCH_RET;
}

int launch_brute(const MeshDev &m, const double *rays, int64_t n, int32_t *o_seg, double *o_t,
                 double *o_u, void *stream) {
    if (n <= 0) return 0;
    k_brute<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, rays, n, o_seg, o_t, o_u);
    MWT_LAUNCH_RET;
}

}  // namespace mwt
