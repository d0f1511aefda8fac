#pragma once
// Device helpers shared by the B200 (sm_100a) kernels of the ray-query engine.
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
constexpr int kFloodCap = 160;  // > the largest vertex fan of every fixture (64, FloorPlan corner)
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

static __device__ __noinline__ int exact_sign8(const double *v) {
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
static __device__ __noinline__ int cmp_mid_exact(double x, double y, double c, double d) {
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

static __device__ __noinline__ double cr_hypot(double x, double y) {
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
// K2: ray generator (its host twins live in the test oracle: oracle/raygen.py)

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline unsigned long long ray_key(unsigned long long seed, unsigned long long stream) {
    return mix64(mix64(seed + kGolden) ^ (stream * 0xD1B54A32D192ED03ull));
}
constexpr unsigned long long kGroupSalt = 0x6A09E667F3BCC909ull;

struct Box {
    double x0, y0, x1, y1;
};

// A generator specification (mode word of include/mwt.h, decoded on the host).
// Coherent mode (cmask != 0): every 64-bit draw k of ray i has the top c bits
// of each 32-bit half replaced by draw k of its group's stream (group =
// i >> gshift).  Each ray's draws stay uniform 64-bit words (bits from two
// independent uniform streams), so every ray has exactly the iid
// distribution; rays of one group share a cell of the disk-rejection square
// (direction) and of the side / position draw (entry point).
struct RayGen {
    int mode;  // MWT_RAYS_BOX_ENTRY / MWT_RAYS_INTERIOR
    int gshift;
    unsigned long long cmask;  // 0: iid
    Box box;
    unsigned long long key, gkey;
};

// decode an include/mwt.h mode word; false if malformed
static inline bool make_raygen(int mode_word, const double *box, unsigned long long seed, RayGen &g) {
    const unsigned w = (unsigned)mode_word;
    const int base = (int)(w & 0xFFu), gs = (int)((w >> 8) & 0xFFu), c = (int)((w >> 16) & 0xFFu);
    if ((w >> 24) != 0u || (base != MWT_RAYS_BOX_ENTRY && base != MWT_RAYS_INTERIOR) || gs > 40 || c > 16)
        return false;
    g.mode = base;
    g.gshift = gs;
    const unsigned long long h = c ? (((1ull << c) - 1ull) << (32 - c)) : 0ull;
    g.cmask = (h << 32) | h;
    g.box = Box{box[0], box[1], box[2], box[3]};
    g.key = ray_key(seed, (unsigned long long)base);
    g.gkey = mix64(g.key ^ kGroupSalt);
    return true;
}

// draw k (0-based) of a ray: mix64(s0 + (k + 1) * golden), group bits spliced in
__device__ __forceinline__ unsigned long long draw(const RayGen &g, unsigned long long s0,
                                                   unsigned long long gs, unsigned k) {
    const unsigned long long z = mix64(s0 + (unsigned long long)(k + 1) * kGolden);
    if (!g.cmask) return z;
    return (z & ~g.cmask) | (mix64(gs + (unsigned long long)(k + 1) * kGolden) & g.cmask);
}

// 64-bit draw -> two 32-bit coordinates in [-1, 1): x = 2 * (hi * 2^-32) - 1,
// built without an integer conversion: the double 2 + hi * 2^-31 has hi in its
// top mantissa bits, and subtracting 3 is exact (both forms are exact, so the
// bits agree with the host twins)
__device__ __forceinline__ void disk_point(unsigned long long z, double &x, double &y, double &r2) {
    const unsigned hi = (unsigned)(z >> 32), lo = (unsigned)z;
    x = __hiloint2double((int)(0x40000000u | (hi >> 12)), (int)(hi << 20)) - 3.0;
    y = __hiloint2double((int)(0x40000000u | (lo >> 12)), (int)(lo << 20)) - 3.0;
    r2 = x * x + y * y;
}

// rejection attempt a: one 64-bit draw -> two 32-bit coordinates in [-1, 1)
__device__ __forceinline__ void disk_try(const RayGen &g, unsigned long long s0, unsigned long long gs,
                                         int a, double &x, double &y, double &r2) {
    disk_point(draw(g, s0, gs, (unsigned)a), x, y, r2);
}

// Group words of draws 0 and 128 for the calling lanes (coherent order).  The
// lanes of one refill batch take consecutive ray indices, so nearly always
// they share one group: the first two active lanes compute its two words
// (one mix64 pass for the warp instead of two) and broadcast them; lanes of
// another group (a batch across a group boundary) compute their own.
__device__ __forceinline__ void group_words(unsigned long long gs, unsigned long long &w0,
                                            unsigned long long &w128) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int l0 = __ffs(m) - 1;
    const unsigned m1 = m & (m - 1u);
    const int l1 = m1 ? __ffs(m1) - 1 : l0;
    const unsigned long long gl = __shfl_sync(m, gs, l0);
    // lane l1 computes draw 128 of the leader's group, every other lane draw 0
    const unsigned long long v = mix64(gl + ((lane == l1 && l1 != l0) ? 129ull : 1ull) * kGolden);
    w0 = __shfl_sync(m, v, l0);
    w128 = __shfl_sync(m, v, l1);
    if (l1 == l0) w128 = mix64(gl + 129ull * kGolden);  // a single active lane
    if (gs != gl) {  // (rare) a lane of another group
        w0 = mix64(gs + kGolden);
        w128 = mix64(gs + 129ull * kGolden);
    }
}

// gw (coherent order, may be NULL): a warp's cached group words {group's
// stream, draw 0, draw 128} of one group (k_trace fills it per grab)
__device__ __forceinline__ Ray gen_ray(const RayGen &g, unsigned long long idx,
                                       const unsigned long long *gw = nullptr) {
    // per-ray SplitMix64 stream: draws mix64(s0 + (k + 1) * golden), s0 = key ^ index
    const unsigned long long s0 = g.key ^ idx;
    const unsigned long long gs = g.gkey ^ (idx >> g.gshift);  // the group's stream
    const Box &b = g.box;
    const unsigned m = __activemask();
    unsigned long long G0 = 0ull, G128 = 0ull;
    if (g.cmask) {
        if (gw && gw[0] == gs) {
            G0 = gw[1];
            G128 = gw[2];
        } else {
            group_words(gs, G0, G128);
        }
    }
    // unit-disk rejection: the first accepted attempt a in 0..63.  Later
    // attempts run while any lane of the warp still needs one, so the warp
    // stays converged (iid order: attempt 1 always -- nearly every warp needs
    // it; coherent order: only a group whose attempt-0 cell missed the disk).
    double x, y, r2;
    disk_point((mix64(s0 + kGolden) & ~g.cmask) | (G0 & g.cmask), x, y, r2);
    bool ok = r2 <= 1.0 && r2 > 0x1p-60;
    int a0 = 1;
    if (!g.cmask) {
        // iid order: attempt 1 unconditionally (nearly every warp needs it)
        double xb, yb, rb;
        disk_point(mix64(s0 + 2ull * kGolden), xb, yb, rb);
        x = ok ? x : xb;
        y = ok ? y : yb;
        r2 = ok ? r2 : rb;
        ok = ok || (rb <= 1.0 && rb > 0x1p-60);
        a0 = 2;
    }
    for (int a = a0; a < 64 && __any_sync(m, !ok); a++) {
        if (!ok) {
            double xa, ya, ra;
            disk_try(g, s0, gs, a, xa, ya, ra);
            ok = ra <= 1.0 && ra > 0x1p-60;
            x = xa;
            y = ya;
            r2 = ra;
        }
    }
    Ray r;
    {
        // angle doubling: (x, y) = rho (cos phi, sin phi) uniform in the disk has
        // phi ~ U[0, 2pi), so (x^2 - y^2, 2xy) / r2 = (cos 2phi, sin 2phi) is
        // isotropic and unit up to rounding -- no sqrt, one division
        const double inv = 1.0 / (ok ? r2 : 1.0);
        r.dx = ok ? (x * x - y * y) * inv : 1.0;
        r.dy = ok ? (2.0 * x * y) * inv : 0.0;
    }
    const double W = b.x1 - b.x0, H = b.y1 - b.y0;
    // u, v: the two 32-bit halves of draw 128 (hi * 2^-32, lo * 2^-32), built
    // as 1 + h * 2^-32 - 1 (exact)
    const unsigned long long zuv = (mix64(s0 + 129ull * kGolden) & ~g.cmask) | (G128 & g.cmask);
    const unsigned uh = (unsigned)(zuv >> 32), vl = (unsigned)zuv;
    const double u = __hiloint2double((int)(0x3FF00000u | (uh >> 12)), (int)(uh << 20)) - 1.0;
    const double v = __hiloint2double((int)(0x3FF00000u | (vl >> 12)), (int)(vl << 20)) - 1.0;
    if (g.mode == MWT_RAYS_INTERIOR) {
        r.ox = b.x0 + W * u;
        r.oy = b.y0 + H * v;
    } else {
        // lines of direction d with a uniform perpendicular offset enter the box
        // through the side facing -d in x with probability H|dx| / (H|dx| + W|dy|),
        // else through the side facing -d in y, uniformly along that side
        const double wx = H * fabs(r.dx), wy = W * fabs(r.dy);
        const bool xside = u * (wx + wy) < wx;  // (selects, not a divergent branch)
        const double along = xside ? b.y0 + H * v : b.x0 + W * v;
        r.ox = xside ? (r.dx > 0.0 ? b.x0 : b.x1) : along;
        r.oy = xside ? along : (r.dy > 0.0 ? b.y0 : b.y1);
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

// a / b correctly rounded from y = RN(1/b), so that several quotients by one
// divisor cost one IEEE division: q = RN(a y) is within one ulp of a / b,
// r = a - b q is exact (one FMA) and RN(q + r y) = RN(a / b) (Markstein's
// theorem; round-to-nearest, no under- or overflow in any step).  The range
// guards keep every step normal: |b|, |a| in [2^-400, 2^400] (or a = 0);
// outside them the IEEE division itself.  Bit-identical to a / b.
struct Rcp {
    double b, y;
    bool ok;
};

__device__ __forceinline__ Rcp make_rcp(double b) {
    const double ab = fabs(b);
    Rcp R;
    R.b = b;
    R.ok = ab >= 0x1p-400 && ab <= 0x1p400;
    R.y = 1.0 / (R.ok ? b : 1.0);
    return R;
}

__device__ __forceinline__ double div_rcp(double a, const Rcp &R) {
    const double q = a * R.y;
    const double r = __fma_rn(-q, R.b, a);
    const double q1 = __fma_rn(r, R.y, q);
    const double aa = fabs(a);
    if (R.ok && (aa == 0.0 || (aa >= 0x1p-400 && aa <= 0x1p400))) return q1;
    return a / R.b;
}

// geometry.py:136-166.  RCP: both quotients from one reciprocal (div_rcp);
// the walk's epilogue keeps two IEEE divisions (fewer live registers there).
template <bool RCP = true>
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
    // (wx * ey - wy * ex) / denom and (wx * dy - wy * dx) / denom, one division
    double tt, uu;
    if (RCP) {
        const Rcp R = make_rcp(denom);
        tt = div_rcp(wx * ey - wy * ex, R);
        uu = div_rcp(wx * r.dy - wy * r.dx, R);
    } else {
        tt = (wx * ey - wy * ex) / denom;
        uu = (wx * r.dy - wy * r.dx) / denom;
    }
    if (tt < 0.0 || uu < 0.0 || uu > 1.0) return false;
    t = tt;
    u = uu;
    return true;
}

// accel.py:82-98 SceneIndex.canonical
template <bool RCP = true>
__device__ __forceinline__ int canonical(const MeshDev &M, const Ray &r, int sid, double t, double u, double &ot,
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
            if (!rsi<RCP>(r, ldg4d(M.seg + sid2), t2, u2, par)) continue;
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

int grid_for(long long n);

}  // namespace mwt
