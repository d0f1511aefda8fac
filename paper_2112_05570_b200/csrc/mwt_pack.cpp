// K1 -- host mesh packer: reference triangulation + scene -> device layout.
//
// Input is the reference data model as loaded by load_triangulation
// (trimesh.py:1309-1337) and parse_scene (scene.py:135-165).  The packer
//  * validates indices and neighbour symmetry (the subset of
//    Triangulation.validate_topology, trimesh.py:283-311, the walk relies on),
//  * computes each internal edge's mirror index (Triangulation.mirror,
//    trimesh.py:154-163) so the walk skips its entry edge by index -- on a
//    valid mesh identical to the reference's vertex-set test (accel.py:178),
//  * builds SceneIndex.endpoint_map (accel.py:77-80) as per-endpoint ranges,
//  * fills TriLocator's anchor grid (accel.py:263-282) with
//    Triangulation.locate (trimesh.py:386-416), eagerly in row-major order.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "mwt_internal.h"

namespace mwt {
namespace {

inline double sa2(double ax, double ay, double bx, double by, double cx, double cy) {
    // geometry.py:81-83; this TU is compiled with -ffp-contract=off
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
}

// Doubles in a totally ordered integer key (-0.0 and +0.0 share key 0).
inline int64_t dkey(double x) {
    int64_t b;
    std::memcpy(&b, &x, 8);
    return b >= 0 ? b : INT64_MIN - b;
}
inline double dval(int64_t k) {
    const int64_t b = k >= 0 ? k : INT64_MIN - k;
    double x;
    std::memcpy(&x, &b, 8);
    return x;
}

// The box-entry start test (device boundary_start) for an origin o strictly
// inside boundary edge PQ of triangle T (apex A) on the side line:
//   _contains (accel.py:219-223): ej = sa2(P, Q, o) >= -1e-15 and the flood
//   bound (accel.py:226-238) on the other two: e1 = sa2(Q, A, o) > 1e-12,
//   e2 = sa2(A, P, o) > 1e-12.
// When P and Q lie exactly on the side line (coordinate c), o = (u, c) or
// (c, u) makes ej = +-0 and reduces e1, e2 to a constant combined with ONE
// rounded product of a rounded difference in u -- each a monotone function of
// u under IEEE rounding.  So the test holds exactly on one interval of
// doubles, found here by bisection with the device's own expressions; the
// kernel then compares u against its bounds instead of evaluating the test.
// Returns the open interval (L, H) (L >= H: empty).
struct OpenIv {
    double lo, hi;
};
OpenIv start_interval(int axis, double c, double umin, double umax, double px, double py, double qx,
                      double qy, double ax, double ay) {
    auto at = [&](int64_t k, int which) {
        const double u = dval(k);
        const double ox = axis == 0 ? u : c, oy = axis == 0 ? c : u;
        if (which == 0) return sa2(qx, qy, ax, ay, ox, oy) > 1e-12;
        if (which == 1) return sa2(ax, ay, px, py, ox, oy) > 1e-12;
        return sa2(px, py, qx, qy, ox, oy) >= -1e-15;
    };
    int64_t lo = dkey(umin) + 1, hi = dkey(umax) - 1;  // the doubles strictly inside
    if (lo > hi) return {umax, umax};
    for (int which = 0; which < 3; which++) {
        const bool fl = at(lo, which), fh = at(hi, which);
        if (fl && fh) continue;
        if (!fl && !fh) return {umax, umax};
        int64_t a = lo, b = hi;  // monotone: bisect for the switch point
        if (!fl) {  // false ... true: smallest true
            while (a + 1 < b) {
                const int64_t m = a + (b - a) / 2;
                (at(m, which) ? b : a) = m;
            }
            lo = b;
        } else {  // true ... false: largest true
            while (a + 1 < b) {
                const int64_t m = a + (b - a) / 2;
                (at(m, which) ? a : b) = m;
            }
            hi = a;
        }
        if (lo > hi) return {umax, umax};
    }
    return {dval(lo - 1), dval(hi + 1)};
}

struct Ctx {
    const double *vx, *vy;
    const int32_t *tv, *tn;
    int32_t nt;
};

bool contains(const Ctx &c, int tid, double px, double py) {
    const int32_t *v = c.tv + 3 * tid;
    for (int i = 0; i < 3; i++) {
        int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
        if (!(sa2(c.vx[a], c.vy[a], c.vx[b], c.vy[b], px, py) >= -1e-15)) return false;
    }
    return true;
}

// trimesh.py:386-416; returns tid, sets *strict when p is strictly inside
int tri_locate(const Ctx &c, double px, double py, int hint, bool *strict) {
    int tid = (hint >= 0 && hint < c.nt) ? hint : 0;
    long cap = 4L * c.nt + 16;
    for (long visited = 0; visited < cap; visited++) {
        const int32_t *v = c.tv + 3 * tid;
        int worst = -1;
        double worst_val = 0.0;
        bool all_pos = true;
        for (int i = 0; i < 3; i++) {
            int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
            double s = sa2(c.vx[a], c.vy[a], c.vx[b], c.vy[b], px, py);
            if (!(s > 0.0)) all_pos = false;
            if (s < worst_val) {
                worst_val = s;
                worst = i;
            }
        }
        if (worst < 0) {
            *strict = all_pos;
            return tid;
        }
        int n = c.tn[3 * tid + worst];
        if (n < 0) {
            *strict = false;
            return tid;
        }
        tid = n;
    }
    *strict = false;
    for (int t = 0; t < c.nt; t++)  // _locate_scan, trimesh.py:428-436
        if (contains(c, t, px, py)) return t;
    return 0;
}

}  // namespace

int pack_mesh(const double *vx, const double *vy, int32_t nv, const int32_t *tv, const int32_t *tn,
              const int32_t *tf, int32_t nt, const double *seg_xy, const uint8_t *seg_kind,
              int32_t ns, HostPacked *out, std::string *err) {
    if (nt < 0 || nv < 0 || ns < 0 || (nt > 0 && (!vx || !vy || !tv || !tn || !tf)) ||
        (ns > 0 && (!seg_xy || !seg_kind))) {
        *err = "mesh_create: negative count or NULL array";
        return MWT_E_INVALID;
    }
    if (nt >= (1 << 29) || ns >= (1 << 30)) {  // 3*nt record indices < 2^31
        *err = "mesh_create: triangulation too large for the 30-bit edge words";
        return MWT_E_INVALID;
    }
    HostPacked &P = *out;
    P.nv = nv;
    P.nt = nt;
    P.ns = ns;
    for (int64_t k = 0; k < 3LL * nt; k++) {
        if (tv[k] < 0 || tv[k] >= nv || tn[k] < -1 || tn[k] >= nt || tf[k] < -1 || tf[k] >= ns) {
            *err = "mesh_create: index out of range in triangle " + std::to_string(k / 3);
            return MWT_E_INVALID;
        }
    }
    P.link.assign(4LL * nt, 0);
    P.lnbr.assign(4LL * nt, -1);
    P.cxy.resize(6LL * nt);
    for (int t = 0; t < nt; t++) {
        const int32_t *v = tv + 3 * t;
        for (int k = 0; k < 3; k++) {
            P.cxy[6LL * t + 2 * k] = vx[v[k]];
            P.cxy[6LL * t + 2 * k + 1] = vy[v[k]];
        }
        for (int i = 0; i < 3; i++) {
            int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
            int n = tn[3 * t + i];
            int j = -1;
            if (n >= 0) {
                const int32_t *u = tv + 3 * n;
                for (int jj = 0; jj < 3; jj++)
                    if (u[(jj + 1) % 3] == b && u[(jj + 2) % 3] == a) j = jj;
                if (j < 0 || tn[3 * n + j] != t) {
                    *err = "mesh_create: neighbor symmetry broken at " + std::to_string(t) + ":" +
                           std::to_string(i) + " -> " + std::to_string(n);
                    return MWT_E_TOPOLOGY;
                }
                P.lnbr[4LL * t + i] = (n << 2) | j;
            }
            int f = tf[3 * t + i];
            uint32_t w;
            if (f != -1) {
                w = kStopBit | (seg_kind[f] ? kBoundaryBit : 0u) | (uint32_t)f;
            } else if (n < 0) {
                w = kOpenWord;
            } else {
                w = 3u * (uint32_t)n + (uint32_t)j;  // step record of neighbour n entered via its edge j
            }
            P.link[4LL * t + i] = (int32_t)w;
        }
    }
    // per-(triangle, entry edge) step records
    P.step.assign(8LL * 3 * nt, 0);
    for (int t = 0; t < nt; t++)
        for (int j = 0; j < 3; j++) {
            int32_t *r = P.step.data() + 8LL * (3LL * t + j);
            r[0] = P.link[4LL * t + (j + 1) % 3];
            r[1] = P.link[4LL * t + (j + 2) % 3];
            std::memcpy(r + 4, &P.cxy[6LL * t + 2 * j], 16);
        }
    // compact walk table (same record indices, vertex-indexed apex)
    if (3LL * nt < (1LL << 17) && nv < (1 << 14) && ns < 0xFFFF) {
        auto cw = [](uint32_t w) -> uint32_t {
            if (!(w & kStopBit)) return w;
            if (w == kOpenWord) return kCOpen;
            return kCStop | ((w & kBoundaryBit) ? kCBoundary : 0u) | (w & kSidMask);
        };
        const int64_t nrec = 3LL * nt, padded = (nrec + 1) & ~1LL;
        P.crec.assign(2 * padded, 0u);
        for (int t = 0; t < nt; t++)
            for (int j = 0; j < 3; j++) {
                const int64_t k = 3LL * t + j;
                P.crec[2 * k] = cw((uint32_t)P.link[4LL * t + (j + 1) % 3]) |
                                ((uint32_t)tv[3 * t + j] << kCVidShift);
                P.crec[2 * k + 1] = cw((uint32_t)P.link[4LL * t + (j + 2) % 3]);
            }
        P.ctri.assign(4LL * nt, 0u);
        for (int t = 0; t < nt; t++)
            for (int i = 0; i < 3; i++)
                P.ctri[4LL * t + i] = cw((uint32_t)P.link[4LL * t + i]) | ((uint32_t)tv[3 * t + i] << kCVidShift);
        P.vxy.resize(2LL * nv);
        for (int v = 0; v < nv; v++) {
            P.vxy[2LL * v] = vx[v];
            P.vxy[2LL * v + 1] = vy[v];
        }
    }
    P.seg.assign(seg_xy, seg_xy + 4LL * ns);
    P.segkind.assign(seg_kind, seg_kind + ns);

    // SceneIndex.endpoint_map: exact (x, y) -> ascending geometry sids
    struct Ep {
        double x, y;
        int32_t sid, end;
    };
    std::vector<Ep> eps;
    for (int s = 0; s < ns; s++) {
        if (seg_kind[s] != 0) continue;
        eps.push_back({seg_xy[4LL * s], seg_xy[4LL * s + 1], s, 0});
        eps.push_back({seg_xy[4LL * s + 2], seg_xy[4LL * s + 3], s, 1});
    }
    std::sort(eps.begin(), eps.end(), [](const Ep &p, const Ep &q) {
        if (p.x < q.x) return true;
        if (q.x < p.x) return false;
        if (p.y < q.y) return true;
        if (q.y < p.y) return false;
        return p.sid < q.sid;
    });
    P.ep_range.assign(4LL * ns, 0);
    P.ep_ids.clear();
    for (size_t g = 0; g < eps.size();) {
        size_t h = g;
        while (h < eps.size() && eps[h].x == eps[g].x && eps[h].y == eps[g].y) h++;
        int32_t off = (int32_t)P.ep_ids.size();
        for (size_t k = g; k < h; k++) P.ep_ids.push_back(eps[k].sid);
        for (size_t k = g; k < h; k++) {
            int e = 2 * eps[k].sid + eps[k].end;
            P.ep_range[2LL * e] = off;
            P.ep_range[2LL * e + 1] = (int32_t)(h - g);
        }
        g = h;
    }
    if (P.ep_ids.empty()) P.ep_ids.push_back(0);

    // boundary-edge table: for each axis-aligned boundary segment (a side of
    // the square), its constrained mesh edges sorted along the side, with the
    // triangle they bound and a bucket index for O(1) lookup
    P.nbsides = 0;
    for (int f = 0; f < ns && P.nbsides < 4; f++) {
        if (seg_kind[f] == 0) continue;
        const double ax = seg_xy[4LL * f], ay = seg_xy[4LL * f + 1];
        const double bx = seg_xy[4LL * f + 2], by = seg_xy[4LL * f + 3];
        int axis;
        if (ay == by) axis = 0;       // horizontal: u = x
        else if (ax == bx) axis = 1;  // vertical: u = y
        else continue;
        struct E {
            double umin, umax, px, py, qx, qy;
            int32_t word;
            double ax, ay;  // apex (corner opposite the edge)
        };
        std::vector<E> es;
        bool ok = true;
        for (int t = 0; t < nt && ok; t++)
            for (int i = 0; i < 3; i++) {
                if (tf[3 * t + i] != f) continue;
                const int a = tv[3 * t + (i + 1) % 3], b = tv[3 * t + (i + 2) % 3];
                // endpoints may sit a rounding off the side line (the CDT splits
                // boundary edges at points within its tolerance); the device
                // tests containment with the actual coordinates
                const double ua = axis == 0 ? vx[a] : vy[a], ub = axis == 0 ? vx[b] : vy[b];
                const int ap = tv[3 * t + i];
                es.push_back({std::min(ua, ub), std::max(ua, ub), vx[a], vy[a], vx[b], vy[b],
                              (int32_t)(3 * t + i), vx[ap], vy[ap]});
            }
        if (!ok || es.empty()) continue;
        std::sort(es.begin(), es.end(), [](const E &p, const E &q) { return p.umin < q.umin; });
        bool tiled = true;  // the edges must tile the side without gaps or overlaps
        for (size_t k = 1; k < es.size(); k++)
            if (es[k].umin != es[k - 1].umax) tiled = false;
        if (!tiled) continue;
        HostPacked::Side &S = P.sides[P.nbsides++];
        S.axis = axis;
        S.c = axis == 0 ? ay : ax;
        S.lo = es.front().umin;
        S.hi = es.back().umax;
        S.off = (int32_t)P.bword.size();
        S.cnt = (int32_t)es.size();
        S.nb = 8 * S.cnt;
        S.scale = S.nb / (S.hi - S.lo);
        S.boff = (int32_t)P.bbucket.size();
        for (const E &e : es) {
            // bu: the exact start interval when P and Q lie on the side line,
            // else the edge's extent with kBExact set on the word (the
            // kernel then evaluates the test itself)
            const bool online = axis == 0 ? (e.py == S.c && e.qy == S.c) : (e.px == S.c && e.qx == S.c);
            const OpenIv iv = online ? start_interval(axis, S.c, e.umin, e.umax, e.px, e.py, e.qx, e.qy,
                                                      e.ax, e.ay)
                                     : OpenIv{e.umin, e.umax};
            P.bu.push_back(iv.lo);
            P.bu.push_back(iv.hi);
            P.bpq.push_back(e.px);
            P.bpq.push_back(e.py);
            P.bpq.push_back(e.qx);
            P.bpq.push_back(e.qy);
            P.bword.push_back(online ? e.word : (int32_t)((uint32_t)e.word | kBExact));
        }
        int k = 0;
        for (int b = 0; b < S.nb; b++) {
            const double start = S.lo + b / S.scale;
            while (k < S.cnt - 1 && es[k].umax <= start) k++;
            P.bbucket.push_back(k);
        }
    }
    // the unit square (every mintri scene, scene.py:18-23): order the sides
    // bottom, right, top, left so the device picks the side from the origin
    P.unit_sides = 0;
    if (P.nbsides == 4) {
        int order[4] = {-1, -1, -1, -1};
        for (int k = 0; k < 4; k++) {
            const HostPacked::Side &S = P.sides[k];
            int slot = -1;
            if (S.axis == 0 && S.c == 0.0) slot = 0;
            else if (S.axis == 1 && S.c == 1.0) slot = 1;
            else if (S.axis == 0 && S.c == 1.0) slot = 2;
            else if (S.axis == 1 && S.c == 0.0) slot = 3;
            if (slot >= 0 && order[slot] < 0) order[slot] = k;
        }
        if (order[0] >= 0 && order[1] >= 0 && order[2] >= 0 && order[3] >= 0) {
            HostPacked::Side tmp[4];
            for (int k = 0; k < 4; k++) tmp[k] = P.sides[order[k]];
            for (int k = 0; k < 4; k++) P.sides[k] = tmp[k];
            P.unit_sides = 1;
        }
    }
    if (P.bword.empty()) {  // keep device pointers valid
        P.bu.assign(2, 0.0);
        P.bpq.assign(4, 0.0);
        P.bword.assign(1, 0);
        P.bbucket.assign(1, 0);
    }

    if (nt == 0) {  // scene-only mesh (BVH / kd / brute force); no walk, no locate
        P.res = 0;
        P.anchor.assign(1, 0);
        return MWT_OK;
    }
    // flood pre-filter is valid while coordinates stay within [-4, 4]
    P.flood_filter = 1;
    for (int k = 0; k < nv; k++)
        if (!(std::fabs(vx[k]) <= 4.0 && std::fabs(vy[k]) <= 4.0)) P.flood_filter = 0;
    P.coord_small = 1;
    for (int k = 0; k < nv; k++)
        if (!(std::fabs(vx[k]) <= 0x1p500 && std::fabs(vy[k]) <= 0x1p500)) P.coord_small = 0;
    // seed grid: the reference's TriLocator uses max(2, int(sqrt(T/2))) cells
    // per side (accel.py:265-266); the device uses a 24x finer grid (~290 cells
    // per triangle; Lines-1024: 1080^2 cells, 4.7 MB, L2-resident) so the seed
    // cell's triangle almost always contains the origin (measured on the
    // interior-ray launch: 4x -> 12x -6%, 12x -> 24x -3%), capped at 2^23
    // cells.  Any containing triangle seeds the same lowest-id flood
    // (accel.py:226-238).
    int ntc = nt > 4 ? nt : 4;
    int res = 24 * (int)std::sqrt(ntc / 2.0);
    if ((long long)res * res > (1LL << 23)) res = 2896;  // floor(sqrt(2^23))
    if (res < 2) res = 2;
    P.res = res;
    P.anchor.assign((size_t)res * res, 0);
    P.anchors_not_strict = 0;
    Ctx c{vx, vy, tv, tn, nt};
    int hint = -1;
    for (int cy = 0; cy < res; cy++)
        for (int cx = 0; cx < res; cx++) {
            const double inv = 1.0 / res;  // the device seeds walks from the same points
            double px = (cx + 0.5) * inv, py = (cy + 0.5) * inv;
            bool strict = false;
            int tid = tri_locate(c, px, py, hint, &strict);
            if (!strict) P.anchors_not_strict++;
            hint = tid;
            P.anchor[(size_t)cy * res + cx] = tid;
        }
    return MWT_OK;
}

}  // namespace mwt
