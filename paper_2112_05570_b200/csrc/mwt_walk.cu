// K2 ray generation, K3 point location, K4 the MWT walk and K7 histograms
// for B200 (sm_100a).  Compiled with -fmad=false: every fp64 expression is
// evaluated in the reference's operation order with no contraction.
//
// Execution model (K4): one persistent CTA per SM (896 threads, 72
// registers).  The CTA stages the mesh's compact walk table, the boundary-edge
// table and the segments in shared memory when they fit, owns a contiguous
// range of rays and hands them to its warps 128 at a time.  In a warp, a lane
// whose ray has terminated goes idle; once at most `refill_below` lanes are
// still walking, the finished lanes run the epilogue (hit test, outputs,
// histogram) and the idle lanes the prologue of their next rays (raygen or
// load, box-entry start or locate, first triangle) as one batch.  Between
// batches the walking lanes run a predicated loop of one-candidate steps.
// Everything is inlined: out-of-line calls spilled ~140 B per ray.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include "mwt_device.cuh"

namespace mwt {

// ---------------------------------------------------------------------------
// K3: point location.  Result = TriLocator.locate (accel.py:284-289): the
// lowest id among the neighbour-connected triangles that _contains p
// (accel.py:219-238).  Any containing triangle seeds the same flood, so the
// seed search here is the engine's own: a fine grid of cell-centre triangles
// (packer) and a straight walk toward p with the reference's exit rule
// (accel.py:314-322, direction left unnormalised), brute-force scan on
// failure (accel.py:287-288).

__device__ __forceinline__ void corners(const MeshDev &M, int t, double2 &P0, double2 &P1,
                                        double2 &P2) {
    P0 = __ldg(M.cxy + 3 * t);
    P1 = __ldg(M.cxy + 3 * t + 1);
    P2 = __ldg(M.cxy + 3 * t + 2);
}

// compact stop word (shared-memory table) -> full walk word
__device__ __forceinline__ uint32_t expand_cword(uint32_t c) {
    if (c == kCOpen) return kOpenWord;
    return kStopBit | ((c & kCBoundary) ? kBoundaryBit : 0u) | (c & 0xFFFFu);
}

// corners from the shared-memory walk table when staged (record 3t+k holds
// the vertex id of corner k), else from cxy
__device__ __forceinline__ void corners2(const MeshDev &M, const uint2 *srec, const double2 *svxy,
                                         int t, double2 &P0, double2 &P1, double2 &P2) {
    if (srec) {
        P0 = svxy[srec[3 * t].x >> kCVidShift];
        P1 = svxy[srec[3 * t + 1].x >> kCVidShift];
        P2 = svxy[srec[3 * t + 2].x >> kCVidShift];
    } else {
        corners(M, t, P0, P1, P2);
    }
}

// accel.py:219-223 with geometry.py:81-83 per edge i: signed_area2(P[i+1], P[i+2], p)
__device__ __forceinline__ void edge_areas(double2 P0, double2 P1, double2 P2, double px, double py,
                                           double &e0, double &e1, double &e2) {
    e0 = sa2(P1, P2, px, py);
    e1 = sa2(P2, P0, px, py);
    e2 = sa2(P0, P1, px, py);
}

__device__ __forceinline__ bool inside(double e0, double e1, double e2) {
    return e0 >= -1e-15 && e1 >= -1e-15 && e2 >= -1e-15;
}

// locate_brute_force, accel.py:241-253.  Cold path: arguments by value so no
// caller state becomes address-taken.
struct LocRes {
    int tid;
    uint32_t st;
};

__device__ __noinline__ LocRes loc_brute(const double2 *cxy, int nt, double px, double py) {
    for (int t = 0; t < nt; t++) {
        double2 P0 = __ldg(cxy + 3 * t), P1 = __ldg(cxy + 3 * t + 1), P2 = __ldg(cxy + 3 * t + 2);
        double e0, e1, e2;
        e0 = sa2(P1, P2, px, py);
        e1 = sa2(P2, P0, px, py);
        e2 = sa2(P0, P1, px, py);
        if (e0 >= -1e-15 && e1 >= -1e-15 && e2 >= -1e-15) return LocRes{t, 0u};
    }
    int best = 0;
    double bd = CUDART_INF;
    for (int t = 0; t < nt; t++) {
        double2 P0 = __ldg(cxy + 3 * t), P1 = __ldg(cxy + 3 * t + 1), P2 = __ldg(cxy + 3 * t + 2);
        double cx = ((P0.x + P1.x) + P2.x) / 3.0;
        double cy = ((P0.y + P1.y) + P2.y) / 3.0;
        double d = cr_hypot(cx - px, cy - py);
        if (d < bd) {
            bd = d;
            best = t;
        }
    }
    return LocRes{best, (uint32_t)ST_LOC_OUTSIDE};
}

// _resolve_tie, accel.py:226-238, general case (some edge value <= 1e-12):
// min tid over the flood of neighbour triangles containing p.  A neighbour
// across edge i can contain p only if this triangle's value for edge i is
// <= ~1e-14 (both are roundings of one exact quantity of opposite sign), so
// larger values skip the exact test without changing the result.
__device__ __noinline__ LocRes flood(const double2 *cxy, const int4 *lnbr, int filter, int tid,
                                    double px, double py) {
    int seen[kFloodCap];
    int stack[kFloodCap];
    int nseen = 1, top = 1, best = tid;
    seen[0] = tid;
    stack[0] = tid;
    const bool filt = filter && fabs(px) <= 4.0 && fabs(py) <= 4.0;
    while (top > 0) {
        int cur = stack[--top];
        if (cur < best) best = cur;
        double2 P0 = __ldg(cxy + 3 * cur), P1 = __ldg(cxy + 3 * cur + 1), P2 = __ldg(cxy + 3 * cur + 2);
        double e[3];
        e[0] = sa2(P1, P2, px, py);
        e[1] = sa2(P2, P0, px, py);
        e[2] = sa2(P0, P1, px, py);
        int4 NB = __ldg(lnbr + cur);
        for (int i = 0; i < 3; i++) {
            int word = (int)pick(NB, i);
            if (word < 0) continue;
            if (filt && e[i] > 1e-12) continue;
            int nb = word >> 2;
            bool dup = false;
            for (int k = 0; k < nseen; k++) dup |= (seen[k] == nb);
            if (dup) continue;
            double2 Q0 = __ldg(cxy + 3 * nb), Q1 = __ldg(cxy + 3 * nb + 1), Q2 = __ldg(cxy + 3 * nb + 2);
            if (!(sa2(Q1, Q2, px, py) >= -1e-15 && sa2(Q2, Q0, px, py) >= -1e-15 &&
                  sa2(Q0, Q1, px, py) >= -1e-15))
                continue;
            if (nseen == kFloodCap) return LocRes{best, (uint32_t)ST_OVERFLOW};
            seen[nseen++] = nb;
            stack[top++] = nb;
        }
    }
    return LocRes{best, nseen > 1 ? (uint32_t)ST_LOC_TIE : 0u};
}

// returns the start triangle and its corners
__device__ __forceinline__ int locate(const MeshDev &M, double px, double py, uint32_t &st,
                                      double2 &P0, double2 &P1, double2 &P2,
                                      const uint2 *srec = nullptr, const double2 *svxy = nullptr) {
    const int res = M.res;
    const double dres = (double)res;
    double vx = px * dres, vy = py * dres;
    int cx = vx < 0.0 ? 0 : (vx >= dres ? res - 1 : (int)vx);
    int cy = vy < 0.0 ? 0 : (vy >= dres ? res - 1 : (int)vy);
    if (!(vx == vx)) cx = 0;
    if (!(vy == vy)) cy = 0;
    // seed point: the centre of the cell, computed exactly as the packer did
    const double sx = ((double)cx + 0.5) * M.inv_res, sy = ((double)cy + 0.5) * M.inv_res;
    const double dx = px - sx, dy = py - sy;
    int cur = __ldg(M.anchor + cy * res + cx);
    double e0, e1, e2;
    corners2(M, srec, svxy, cur, P0, P1, P2);
    edge_areas(P0, P1, P2, px, py, e0, e1, e2);
    if (!inside(e0, e1, e2)) {  // seed cell centre and p in different triangles
        int ent = -1;
        bool found = false;
        const int cap = 4 * M.nt + 16;
        for (int it = 0; it < cap; it++) {
            // straight walk toward p, exit rule of accel.py:314-322
            double s0 = dx * (P0.y - sy) - dy * (P0.x - sx);
            double s1 = dx * (P1.y - sy) - dy * (P1.x - sx);
            double s2 = dx * (P2.y - sy) - dy * (P2.x - sx);
            int best = -1;
            double bt = 0.0;
            if (ent != 0 && s1 <= 0.0 && 0.0 <= s2 && s2 - s1 > bt) { bt = s2 - s1; best = 0; }
            if (ent != 1 && s2 <= 0.0 && 0.0 <= s0 && s0 - s2 > bt) { bt = s0 - s2; best = 1; }
            if (ent != 2 && s0 <= 0.0 && 0.0 <= s1 && s1 - s0 > bt) { bt = s1 - s0; best = 2; }
            if (best < 0) break;
            int word = (int)pick(__ldg(M.lnbr + cur), best);
            if (word < 0) break;
            cur = word >> 2;
            ent = word & 3;
            corners2(M, srec, svxy, cur, P0, P1, P2);
            edge_areas(P0, P1, P2, px, py, e0, e1, e2);
            if (inside(e0, e1, e2)) {
                found = true;
                break;
            }
        }
        if (!found) {
            const LocRes lr = loc_brute(M.cxy, M.nt, px, py);
            st |= ST_LOC_BRUTE | lr.st;
            cur = lr.tid;
            corners2(M, srec, svxy, cur, P0, P1, P2);
            edge_areas(P0, P1, P2, px, py, e0, e1, e2);
        }
    }
    if (M.flood_filter && fabs(px) <= 4.0 && fabs(py) <= 4.0) {
        // only neighbours across edges with value <= 1e-12 can contain p; a
        // point strictly inside, or on a boundary edge, has none to test
        if (e0 > 1e-12 && e1 > 1e-12 && e2 > 1e-12) return cur;
        const int4 NB = __ldg(M.lnbr + cur);
        if ((e0 > 1e-12 || NB.x < 0) && (e1 > 1e-12 || NB.y < 0) && (e2 > 1e-12 || NB.z < 0))
            return cur;
    }
    const LocRes fr = flood(M.cxy, M.lnbr, M.flood_filter, cur, px, py);
    st |= fr.st;
    const int best = fr.tid;
    if (best != cur) corners2(M, srec, svxy, best, P0, P1, P2);
    return best;
}

// ---------------------------------------------------------------------------
// K4: the walk, accel.py:138-213.  State between steps: current triangle,
// the chosen exit edge word w and whether its endpoints' sides are strict
// (sp < 0 < sq; the values themselves are recomputed where needed).
// Entering neighbour N across w through N's edge j, the two shared corners
// keep their side values (accel.py:153-159 caches them per vertex), so one
// step loads link[N] (16 B) and the apex corner cxy[3N + j] (16 B) -- both
// addressed by (N, j) alone.

// Walk words (packer): an internal edge's word is the index k = 3N + j of the
// step record for entering neighbour N through its edge j; stop words carry
// the stop bit.  The walk state keeps the record index of the current
// triangle (kr) and which candidate it exits through (ch: 0 = edge (j+1)%3,
// 1 = edge (j+2)%3); the triangle id and exit edge are only needed at the
// exit, and are recovered there (cur = kr / 3, ei = (kr % 3 + 1 + ch) % 3).
// The side values (sp, sq) of the chosen exit edge's endpoints decide the
// state (fast: sp < 0 < sq) but are not carried between steps: a step in the
// fast state never reads them, and the rare consumers (the general rule, the
// grazing fallback) recompute them from the edge's corners -- side_of is a
// pure function of the vertex, so the value is the reference's cached one
// (accel.py:153-159).  That keeps four registers and four selects per step
// out of the walk loop.
struct WalkState {
    int kr, ch, steps;
    uint32_t w;     // word of the exit edge just chosen
    double sp, sq;  // (walk_first / boundary_start only) sides of corners (ei+1)%3, (ei+2)%3
    bool fast;      // sp < 0 < sq: the next step may take the one-candidate fast path
};

// the 32-B step record k (words of the two candidate exits, apex corner)
__device__ __forceinline__ void load_step(const MeshDev &M, uint32_t k, int4 &W, double2 &A) {
    const int4 *p = M.step + 2 * (size_t)k;
    unsigned long long w01, w23;
    asm("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
        : "=l"(w01), "=l"(w23), "=d"(A.x), "=d"(A.y)
        : "l"(p));
    W.x = (int)(uint32_t)w01;
    W.y = (int)(uint32_t)(w01 >> 32);
    W.z = (int)(uint32_t)w23;
    W.w = (int)(uint32_t)(w23 >> 32);
}

// the same record as ONE 256-bit load (sm_100 LDG.E.ENL2.256: one L1
// wavefront per lane instead of two); volatile, so it is issued before the side
// test rather than sunk into the branch that consumes the words
template <bool SPLIT = false>
__device__ __forceinline__ void load_step_issue(const MeshDev &M, uint32_t k, int4 &W, double2 &A) {
    const int4 *p = M.step + 2 * (size_t)k;
    if (SPLIT) {
        // the 24 used bytes as an 8-B and a 16-B load (the pad is not read):
        // 6 instead of 8 L1 data-pipe wavefronts per warp when the lanes'
        // records are few (coherent rays), two wavefronts per lane when they
        // are scattered
        uint32_t w0, w1;
        asm volatile("ld.global.nc.v2.b32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "l"(p));
        asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(A.x), "=d"(A.y) : "l"(p + 1));
        W.x = (int)w0;
        W.y = (int)w1;
        W.z = W.w = 0;
    } else {
        unsigned long long w01, w23;
        asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(w01), "=l"(w23), "=d"(A.x), "=d"(A.y)
                     : "l"(p));
        W.x = (int)(uint32_t)w01;
        W.y = (int)(uint32_t)(w01 >> 32);
        W.z = (int)(uint32_t)w23;
        W.w = (int)(uint32_t)(w23 >> 32);
    }
}

// first triangle: edges 0 (s1,s2), 1 (s2,s0), 2 (s0,s1) in order, none skipped
__device__ __forceinline__ bool walk_first(const Ray &r, int t0, int4 L, double2 P0, double2 P1,
                                           double2 P2, WalkState &s, uint32_t &st) {
    double s0 = side_of(r, P0), s1 = side_of(r, P1), s2 = side_of(r, P2);
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
        st |= ST_ERROR;  // no exit edge: TraversalError (accel.py:190-191)
        return false;
    }
    s.sp = best == 0 ? s1 : (best == 1 ? s2 : s0);
    s.sq = best == 0 ? s2 : (best == 1 ? s0 : s1);
    s.fast = s.sp < 0.0 && 0.0 < s.sq;
    // express "exit edge best of t0" as (record, choice 0): j = (best + 2) % 3
    s.kr = 3 * t0 + (best == 0 ? 2 : best - 1);
    s.ch = 0;
    s.w = pick(L, best);
    return true;
}


// General step rule of accel.py:171-191 for the triangle just entered through
// its edge j: a = side of corner (j+1)%3, b = side of corner (j+2)%3 (the
// shared corners, values carried over as the reference's per-vertex cache),
// c = side of the apex corner j.  E1 = edge (j+1)%3 has (sp, sq) = (b, c),
// E2 = edge (j+2)%3 has (c, a); the reference scans ascending edge index, so
// E2 comes first iff j == 1.  Kept out of line: only degenerate or fallback
// configurations reach it.
// Returns the status bits | (choice + 1) << 20 with choice 0 = E1, 1 = E2, -1 = none.
__device__ __noinline__ uint32_t walk_general(int j, double a, double b, double c, uint32_t st) {
    const bool sw = (j == 1);
    const double spF = sw ? c : b, sqF = sw ? a : c;
    const double spS = sw ? b : c, sqS = sw ? c : a;
    const double trF = sqF - spF, trS = sqS - spS;
    const bool cF = spF <= 0.0 && 0.0 <= sqF;
    const bool cS = spS <= 0.0 && 0.0 <= sqS;
    int sel = -1;
    if (cF && trF > 0.0) sel = 0;
    if (cS && trS > (sel == 0 ? trF : 0.0)) sel = 1;
    if (cF && cS) st |= ST_MULTI;
    if ((cF && (spF == 0.0 || sqF == 0.0)) || (cS && (spS == 0.0 || sqS == 0.0))) st |= ST_ZERO_SIDE;
    if (sel < 0) {  // fallback: largest positive trans (accel.py:182-184, :188-189)
        if (trF > 0.0) sel = 0;
        if (trS > (sel == 0 ? trF : 0.0)) sel = 1;
        if (sel < 0) st |= ST_ERROR;
        else st |= ST_FALLBACK;
    }
    const int choice = sel < 0 ? -1 : ((sel != 0) != sw ? 1 : 0);
    return st | ((uint32_t)(choice + 1) << 20);
}

// One step into the neighbour across s.w (an internal word).  Fast path:
// when the exit just taken was a strict candidate (sp < 0 < sq) and the new
// apex side c is nonzero, exactly one edge qualifies -- E1 if c > 0 (its
// trans c - sp > 0), E2 if c < 0 (trans sq - c > 0) -- with no zero side,
// no second candidate and no fallback, which is what the general rule
// yields in that case.
__device__ __forceinline__ bool walk_step(const MeshDev &M, const Ray &r, WalkState &s,
                                          uint32_t &st) {
    if (s.steps >= 4 * M.nt + 16) {  // > #(triangle, entry) states: a revisit => TraversalError
        st |= ST_ERROR;
        return false;
    }
    s.steps++;
    const uint32_t k = s.w;
    // one 32-B step record: both candidate exit words and the apex corner
    int4 W;
    double2 A;
    load_step(M, k, W, A);
    const double c = side_of(r, A);
    s.kr = (int)k;
    if (s.fast && c != 0.0) {
        // E1 -> (sp, c), E2 -> (c, sq): still sp < 0 < sq
        s.w = (uint32_t)(c > 0.0 ? W.x : W.y);
        s.ch = c > 0.0 ? 0 : 1;
        return true;
    }
    // the shared corners' sides, recomputed: a = corner (j+1)%3 (the previous
    // exit's sq), b = corner (j+2)%3 (its sp)
    const int j = (int)(k % 3u), N = (int)(k / 3u);
    const double a = side_of(r, __ldg(M.cxy + 3 * N + (j + 1) % 3));
    const double b = side_of(r, __ldg(M.cxy + 3 * N + (j + 2) % 3));
    const uint32_t g = walk_general(j, a, b, c, st);
    st = g & 0xFFFFFu;
    const int sel = (int)(g >> 20) - 1;
    if (sel < 0) return false;
    const double sp = sel == 0 ? b : c, sq = sel == 0 ? c : a;  // E1: (b, c); E2: (c, a)
    s.w = (uint32_t)(sel == 0 ? W.x : W.y);
    s.ch = sel;
    s.fast = sp < 0.0 && 0.0 < sq;
    return true;
}

#ifndef MWT_TERM_RCP
#define MWT_TERM_RCP 0
#endif
// the hit test's two quotients: IEEE divisions (0) or one reciprocal (1)
constexpr bool kTermRcp = MWT_TERM_RCP;

// constrained / open exit: accel.py:192-211
// (sseg: a shared-memory copy of the segments, or NULL)
__device__ __forceinline__ int walk_terminal(const MeshDev &M, const Ray &r, const WalkState &s,
                                          double &ot, double &ou, uint32_t &st,
                                          const double4 *sseg = nullptr) {
    ot = CUDART_NAN;
    ou = CUDART_NAN;
    if (s.w == kOpenWord || (s.w & kBoundaryBit)) return -1;
    const int sid = (int)(s.w & kSidMask);
    const double4 S = sseg ? sseg[sid] : ldg4d(M.seg + sid);
    double t, u;
    bool par = false;
    bool ok = rsi<kTermRcp>(r, S, t, u, par);
    if (par) st |= ST_PARALLEL;
    if (!ok) {
        // grazing numerical corner, accel.py:199-207
        st |= ST_GRAZING;
        const int cur = s.kr / 3, j = s.kr % 3;
        const int ei = (j + 1 + s.ch) % 3;
        const double2 pa = __ldg(M.cxy + 3 * cur + (ei + 1) % 3);
        const double2 pb = __ldg(M.cxy + 3 * cur + (ei + 2) % 3);
        const double sp = side_of(r, pa), sq = side_of(r, pb);  // the exit edge's sides
        const double wq = sp != sq ? sp / (sp - sq) : 0.5;
        const double x = pa.x + wq * (pb.x - pa.x);
        const double y = pa.y + wq * (pb.y - pa.y);
        t = (x - r.ox) * r.dx + (y - r.oy) * r.dy;
        const double ex = S.z - S.x, ey = S.w - S.y;
        u = ((x - S.x) * ex + (y - S.y) * ey) / (ex * ex + ey * ey);  // Segment.param_of
    }
    const int s2 = canonical<kTermRcp>(M, r, sid, t, u, ot, ou);
    if (s2 != sid) st |= ST_CANON;
    return s2;
}

// ---------------------------------------------------------------------------
// K7 histogram: block-private shared counters, flushed once per block

__device__ __forceinline__ void hist_init(unsigned int *h) {
    for (int k = threadIdx.x; k < MWT_HIST_LEN; k += blockDim.x) h[k] = 0u;
    __syncthreads();
}

__device__ __forceinline__ void hist_add(unsigned int *h, int seg, int steps, uint32_t st) {
    int bin = steps < MWT_HIST_STEP_BINS - 1 ? (steps < 0 ? 0 : steps) : MWT_HIST_STEP_BINS - 1;
    atomicAdd(h + bin, 1u);
    atomicAdd(h + (seg >= 0 ? MWT_HIST_HIT : MWT_HIST_MISS), 1u);
    if (st) {
        for (int b = 0; b < 12; b++)
            if (st & (1u << b)) atomicAdd(h + MWT_HIST_STATUS0 + b, 1u);
    }
}

__device__ __forceinline__ void hist_flush(unsigned int *h, unsigned long long steps_sum,
                                           long long *hist) {
    for (int o = 16; o > 0; o >>= 1) steps_sum += __shfl_down_sync(0xffffffffu, steps_sum, o);
    if ((threadIdx.x & 31) == 0 && steps_sum)
        atomicAdd(reinterpret_cast<unsigned long long *>(hist + MWT_HIST_STEPS_SUM), steps_sum);
    __syncthreads();
    for (int k = threadIdx.x; k < MWT_HIST_LEN; k += blockDim.x)
        if (h[k] && k != MWT_HIST_STEPS_SUM)
            atomicAdd(reinterpret_cast<unsigned long long *>(hist + k), (unsigned long long)h[k]);
}

// ---------------------------------------------------------------------------
// the persistent trace kernel

struct RaySrc {
    RayGen gen;        // generated rays (GEN == true)
    unsigned long long first;
    int box_in4;       // the generator's box lies in [-4, 4]^2 (so does every origin)
    const double *rays;   // loaded rays (GEN == false)
    const int32_t *start; // optional given start triangles
};

struct TraceOut {
    int32_t *start, *seg, *steps;
    double *t, *u;
    uint32_t *st;
    int32_t *end;  // the triangle each walk ended in (-1 after an error)
};

// Per-launch constants: one __grid_constant__ kernel parameter.  The
// out-of-line prologue and epilogue take its address, so they cost neither
// argument registers nor a local copy.
struct Launch {
    RaySrc src;
    TraceOut out;
    // the tight loop may decide the apex side by comparing side_of's two
    // products (see k_trace): the mesh is coord_small and, for generated rays,
    // so is the box (loaded rays are checked per lane)
    int cmp_side;
};

// Per-ray prologue result (raygen or load, locate, first triangle)
struct Init {
    double ox, oy, dx, dy;
    uint32_t w, st;
    int cur, ei, steps, phase, start;
    bool fast;
};

// Box-entry start: for a ray whose origin lies on a side of the square, the
// boundary-edge table gives the triangle T bounded there.  If T is provably
// the ONLY triangle that _contains the origin (accel.py:219-223; the two other
// edge values exceed the flood bound of 1e-12), T is the reference's start
// triangle (accel.py:226-238), and if the edge's endpoints straddle the ray
// (side(Q) < 0 < side(P)) the first-triangle scan of accel.py:171-191 reduces
// to an ordinary step entered through that edge: it is no candidate (sp > 0)
// and has trans < 0, so neither the exit nor the fallback choice can pick it.
struct BTab {  // the boundary-edge table arrays (global or a shared-memory copy)
    const double2 *bu;
    const double4 *bpq;
    const int32_t *bword, *bbucket;
    const MeshDev::BSide *bs;  // the side descriptors (shared-memory copy: lanes index freely)
    const uint2 *srec;  // the staged walk table (corners for locate), or NULL
    const double2 *svxy;
};

// box_in4: the origin is known to lie in [-4, 4]^2 (generated rays of a box inside it)
__device__ __forceinline__ bool boundary_start(const MeshDev &M, const BTab &T, const Ray &r,
                                               WalkState &s, bool box_in4 = false) {
    // one validity flag instead of early returns (fewer divergent branches);
    // indices stay in range when a condition fails
    bool ok = M.flood_filter && (box_in4 || (fabs(r.ox) <= 4.0 && fabs(r.oy) <= 4.0));
    int k = -1;
    if (M.unit_sides) {  // bottom, right, top, left
        k = r.oy == 0.0 ? 0 : (r.ox == 1.0 ? 1 : (r.oy == 1.0 ? 2 : (r.ox == 0.0 ? 3 : -1)));
    } else {
        for (int kk = M.nbsides - 1; kk >= 0; kk--)
            if ((M.bs[kk].axis == 0 ? r.oy : r.ox) == M.bs[kk].c) k = kk;
    }
    ok = ok && k >= 0;
    const MeshDev::BSide &S = T.bs[k < 0 ? 0 : k];
    const double u = S.axis == 0 ? r.ox : r.oy;
    ok = ok && u > S.lo && u < S.hi;
    int b = (int)((u - S.lo) * S.scale);
    b = b < 0 ? 0 : (b >= S.nb ? S.nb - 1 : b);
    int e = T.bbucket[S.boff + b];
    // bu holds each edge's exact start interval (mwt_pack.cpp): u inside it
    // <=> strictly inside the edge and the _contains / flood-bound test holds;
    // a u past it moves on, and then fails the next edge's lower bound
    double2 U = T.bu[S.off + e];
    while (ok && u >= U.y && e < S.cnt - 1) U = T.bu[S.off + (++e)];
    ok = ok && U.x < u && u < U.y;
    const double4 PQ = T.bpq[S.off + e];
    uint32_t word = (uint32_t)T.bword[S.off + e];
    const double2 P = make_double2(PQ.x, PQ.y), Q = make_double2(PQ.z, PQ.w);
    if (word & kBExact) {  // endpoints off the side line: the test in full (rare)
        word &= ~kBExact;
        const double2 A = __ldg(M.cxy + word);  // apex corner j of T: cxy[3T + j], word = 3T + j
        // _contains values in the reference's form: edge i -> (corner i+1, corner i+2)
        const double ej = sa2(P, Q, r.ox, r.oy);
        const double e1 = sa2(Q, A, r.ox, r.oy);
        const double e2 = sa2(A, P, r.ox, r.oy);
        ok = ok && ej >= -1e-15 && e1 > 1e-12 && e2 > 1e-12;
    }
    const double sa = side_of(r, P), sb = side_of(r, Q);
    ok = ok && sb < 0.0 && 0.0 < sa;
    if (ok) {
        s.w = word;
        s.sq = sa;  // side of corner (j+1)%3
        s.sp = sb;  // side of corner (j+2)%3
        s.fast = true;
        s.steps = 0;  // the first walk step enters (counts) T itself
        s.kr = (int)word;
        s.ch = 0;
    }
    return ok;
}

// the walk words of triangle t's three edges: from the staged walk table when
// present (record 3t+2 holds edges 0 and 1, record 3t holds edge 2), else link[t]
__device__ __forceinline__ int4 link_words(const MeshDev &M, const BTab &T, int t) {
    if (!T.srec) return __ldg(M.link + t);
    const uint2 a = T.srec[3 * t + 2], b = T.srec[3 * t];
    const uint32_t w0 = a.x & kCWordMask, w1 = a.y, w2 = b.y;
    return make_int4((int)((w0 & kCStop) ? expand_cword(w0) : w0),
                     (int)((w1 & kCStop) ? expand_cword(w1) : w1),
                     (int)((w2 & kCStop) ? expand_cword(w2) : w2), 0);
}

template <bool GEN>
__device__ __forceinline__ Init prologue_body(const MeshDev &M, const BTab &T, const RaySrc &src,
                                              long long i, const unsigned long long *gw = nullptr) {
    Init o;
    o.st = 0;
    const Ray r = GEN ? gen_ray(src.gen, src.first + (unsigned long long)i, gw)
                      : load_ray(src.rays, i);
    o.ox = r.ox; o.oy = r.oy; o.dx = r.dx; o.dy = r.dy;
    // (generated interior rays never start on the box: skip the table)
    if ((GEN || !src.start) && !(GEN && src.gen.mode == MWT_RAYS_INTERIOR)) {  // (generated: no start ids)
        WalkState bs;
        if (boundary_start(M, T, r, bs, GEN && src.box_in4)) {
            o.start = bs.kr / 3;
            o.w = bs.w; o.cur = bs.kr; o.ei = bs.ch; o.steps = 0;
            o.fast = true;
            o.phase = 1;
            o.st = MWT_ST_BOUNDARY;
            return o;
        }
    }
    double2 P0, P1, P2;
    int t0;
    if (!GEN && src.start) {
        t0 = __ldg(src.start + i);
        if (t0 < 0 || t0 >= M.nt) t0 = -1;
        else corners(M, t0, P0, P1, P2);
    } else {
        t0 = locate(M, r.ox, r.oy, o.st, P0, P1, P2, T.srec, T.svxy);
    }
    o.start = t0;
    WalkState s;
    s.kr = 0;
    s.ch = 0;
    s.steps = 1;
    s.sp = s.sq = 0.0;
    s.w = 0;
    s.fast = false;
    if (t0 < 0) {
        o.st |= ST_ERROR;
        s.steps = 0;
        o.phase = 3;
    } else if (!walk_first(r, t0, link_words(M, T, t0), P0, P1, P2, s, o.st)) {
        o.phase = 3;
    } else {
        o.phase = (s.w & kStopBit) ? 2 : 1;
    }
    o.w = s.w; o.cur = s.kr; o.ei = s.ch; o.steps = s.steps;
    o.fast = s.fast;
    return o;
}

// Block-private histogram: a shared atomic per lane for its step bin,
// warp-aggregated updates for hit / miss / the step sum / each status bit present.
template <int NT>  // threads per CTA
struct HistSm {
    unsigned int bins[MWT_HIST_LEN];
    unsigned long long steps_sum;
    unsigned long long warp_steps[32];  // per-warp partial step sums (owner-only updates)
    unsigned warp_hm[32][2];            // per-warp hit / miss counts (owner-only updates)
    // per-thread counters (owner-only, no collectives): hits | misses << 21 |
    // boundary starts << 42, and the step sum
    unsigned long long lane_cnt[NT];
    unsigned long long lane_steps[NT];
};
constexpr unsigned long long kLaneHit = 1ull, kLaneMiss = 1ull << 21, kLaneBnd = 1ull << 42;

template <int NT>
__device__ __forceinline__ void hist_add_warp(HistSm<NT> *H, int seg, int steps, uint32_t st) {
    const int bin = steps < MWT_HIST_STEP_BINS - 1 ? (steps < 0 ? 0 : steps) : MWT_HIST_STEP_BINS - 1;
    atomicAdd(H->bins + bin, 1u);  // per lane: cheaper than grouping equal bins (match.any)
    // hit / miss / boundary-start counts and the step sum: this thread's own
    // slots (flushed once per CTA)
    H->lane_cnt[threadIdx.x] += (seg >= 0 ? kLaneHit : kLaneMiss) +
                                ((st & MWT_ST_BOUNDARY) ? kLaneBnd : 0ull);
    H->lane_steps[threadIdx.x] += (unsigned long long)(steps > 0 ? steps : 0);
    // the other status bits are rare: warp-aggregated when present
    const unsigned rest = st & 0x7FFu;
    const unsigned m = __activemask();
    if (!__any_sync(m, rest)) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned any = __reduce_or_sync(m, rest);
    while (any) {
        const int b = __ffs(any) - 1;
        any &= any - 1;
        const unsigned c = __ballot_sync(m, (st >> b) & 1u);
        if (lane == leader) atomicAdd(H->bins + MWT_HIST_STATUS0 + b, (unsigned)__popc(c));
    }
}

// Epilogue for a lane whose ray has ended (phase 2: exit edge
// reached; phase 3: TraversalError): hit test, per-ray outputs, histogram.
template <bool END, int NT>
__device__ __forceinline__ void epilogue(const MeshDev *__restrict__ Mg, const Launch *__restrict__ L,
                                      HistSm<NT> *H, const double4 *sseg, long long i, double ox, double oy, double dx,
                                      double dy, int kr, int ch, uint32_t w,
                                      uint32_t st, int steps, int phase) {
    int seg = -1;
    double t = CUDART_NAN, u = CUDART_NAN;
    if (phase == 2) {
        const Ray r{ox, oy, dx, dy};
        WalkState s;
        s.kr = kr;
        s.ch = ch;
        s.w = w;
        seg = walk_terminal(*Mg, r, s, t, u, st, sseg);
    }
    const TraceOut &O = L->out;
    if (O.seg) O.seg[i] = seg;
    if (O.t) O.t[i] = t;
    if (END && O.u) O.u[i] = u;  // (the generated-ray launch writes seg, t and steps only)
    if (O.steps) O.steps[i] = steps;
    if (END && O.st) O.st[i] = st;
    if (END && O.end) O.end[i] = phase == 2 ? kr / 3 : -1;  // loaded rays only (chaining)
    if (H) hist_add_warp(H, seg, steps, st);
}


// The step record k of the tight loop: the two candidate exit words (E1 =
// edge (j+1)%3, E2 = edge (j+2)%3) and the apex corner -- from the staged
// per-record table (SMEM), the staged per-triangle table (SMEM && TRI) or one
// 32-B global record.
template <bool SMEM, bool TRI>
__device__ __forceinline__ void fetch_step(const MeshDev &M, const uint2 *srec, const uint4 *stri,
                                           const double2 *svxy, uint32_t k, uint32_t &wx, uint32_t &wy,
                                           double2 &A) {
    if (SMEM && TRI) {
        // record 3N + j from triangle N's 16-B entry: apex = corner j,
        // exits = edges (j+1)%3, (j+2)%3
        const uint32_t N = __umulhi(k, 0xAAAAAAABu) >> 1;
        const uint32_t j = k - 3u * N;
        const uint4 X = stri[N];
        const uint32_t a = j == 0u ? X.x : (j == 1u ? X.y : X.z);
        const uint32_t b = j == 0u ? X.y : (j == 1u ? X.z : X.x);
        const uint32_t c = j == 0u ? X.z : (j == 1u ? X.x : X.y);
        A = svxy[a >> kCVidShift];
        wx = b & kCWordMask;
        wy = c & kCWordMask;
    } else if (SMEM) {
        const uint2 X = srec[k];
        A = svxy[X.x >> kCVidShift];
        wx = X.x & kCWordMask;
        wy = X.y;
    } else {
        int4 W;
        load_step_issue<TRI>(M, k, W, A);  // (TRI without SMEM: split loads)
        wx = (uint32_t)W.x;
        wy = (uint32_t)W.y;
    }
}

#ifndef MWT_GRAB
#define MWT_GRAB 512
#endif
#ifndef MWT_GRAB_TAIL
#define MWT_GRAB_TAIL 128
#endif
#ifndef MWT_UNROLL
#define MWT_UNROLL 5
#endif
// Rays a warp takes from its CTA's counter at a time: kGrab (a whole
// coherent group of the benchmark order, so a refill batch rarely spans two
// groups or two grabs), kGrabTail once fewer than two big grabs per warp
// are left in the CTA's range (the warps' last grabs stay short: balance).
constexpr int kGrab = MWT_GRAB;
constexpr int kGrabTail = MWT_GRAB_TAIL;
#ifndef MWT_CTA_ALIGN
#define MWT_CTA_ALIGN MWT_GRAB
#endif
constexpr long long kCtaAlign = MWT_CTA_ALIGN;
constexpr int kUnroll = MWT_UNROLL;  // fast steps per warp vote

// The trace kernel.  Each CTA owns a contiguous range of rays; its warps take
// kGrab (kGrabTail) rays at a time from a shared counter (so all warps of a CTA finish
// together), and each warp keeps its lanes busy: once at most `refill_below`
// lanes are still walking, the lanes whose rays ended run the epilogue and
// the idle lanes the prologue of the next rays, both as one batch.
//
// ---------------------------------------------------------------------------
// Staging with the bulk-copy engine (cp.async.bulk, the 1-D TMA path): one
// thread arms an mbarrier with the byte count and issues the copies; every
// thread waits on the barrier's phase.  Sizes and addresses are multiples of 16.

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// stage n pieces (dst, src, bytes) into shared memory; call from all threads
__device__ __forceinline__ void bulk_stage(unsigned long long *bar, int n, void *const *dst,
                                           const void *const *src, const unsigned *bytes) {
    if (threadIdx.x == 0) {
        unsigned total = 0;
        for (int k = 0; k < n; k++) total += bytes[k];
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(smem_u32(bar)), "r"(total) : "memory");
        for (int k = 0; k < n; k++)
            for (unsigned off = 0; off < bytes[k]; off += 65536u) {
                const unsigned b = bytes[k] - off < 65536u ? bytes[k] - off : 65536u;
                bulk_g2s(static_cast<char *>(dst[k]) + off, static_cast<const char *>(src[k]) + off, b,
                         bar);
            }
    }
    __syncthreads();  // the barrier is initialised
    asm volatile(
        "{\n.reg .pred p;\nLAB_WAIT%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra LAB_WAIT%=;\n}\n" :: "r"(smem_u32(bar)) : "memory");
}

// SMEM: the compact walk table (mwt_internal.h) is staged into shared memory
// once per CTA and the tight loop reads it there (one CTA of THREADS per SM);
// otherwise the tight loop reads the 32-B step records from global memory.
// TRI (with SMEM): the per-triangle compact table is staged instead of the
// per-record one (meshes too large for the latter); locate and the
// first-triangle words then read global memory.  TRI without SMEM: the
// global step records are read as 8 + 16 B (load_step_issue<true>; chosen
// for the coherent generator orders, FloorPlan +3%, iid orders -18%).
template <bool GEN, int MINB, int THREADS, bool SMEM, bool STAGE = SMEM, bool TRI = false>
__global__ void __launch_bounds__(THREADS, MINB)
    k_trace(const __grid_constant__ MeshDev M, const __grid_constant__ Launch L, long long n,
            long long *hist, int refill_below) {
    __shared__ HistSm<THREADS> H;
    __shared__ unsigned s_next;
    __shared__ unsigned long long s_gw[GEN ? THREADS / 32 : 1][3];  // per warp: its grab's group words
    extern __shared__ __align__(16) unsigned char dsm[];
    const uint2 *srec = reinterpret_cast<const uint2 *>(dsm);
    const uint4 *stri = reinterpret_cast<const uint4 *>(dsm);
    const int tbytes = !SMEM ? 0 : TRI ? 16 * M.nt : M.crec_bytes;  // the table; vxy follows
    const double2 *svxy = reinterpret_cast<const double2 *>(dsm + tbytes);
    __shared__ MeshDev::BSide sbs[4];
    if (threadIdx.x < 4) sbs[threadIdx.x] = M.bs[threadIdx.x];
    BTab btab{M.bu, M.bpq, M.bword, M.bbucket, sbs, nullptr, nullptr};
    const double4 *sseg = nullptr;
    const int wbytes = !SMEM ? 0 : TRI ? M.tri_smem_bytes : M.smem_bytes;  // the walk table, then the boundary blob, segments
    if (SMEM || STAGE) {
        __shared__ __align__(8) unsigned long long stage_bar;
        void *dst[4];
        const void *src[4];
        unsigned bytes[4];
        int np = 0;
        if (SMEM) {
            dst[np] = dsm; src[np] = TRI ? (const void *)M.ctri : (const void *)M.crec;
            bytes[np++] = (unsigned)tbytes;
            dst[np] = dsm + tbytes; src[np] = M.vxy;
            bytes[np++] = (unsigned)(wbytes - tbytes);
            if (!TRI) {
                btab.srec = srec;
                btab.svxy = svxy;
            }
        }
        if (STAGE) {
            const unsigned char *bb = dsm + wbytes;
            dst[np] = dsm + wbytes; src[np] = M.bblob; bytes[np++] = (unsigned)M.bblob_bytes;
            btab.bu = reinterpret_cast<const double2 *>(bb);
            btab.bpq = reinterpret_cast<const double4 *>(bb + M.bo_bpq);
            btab.bword = reinterpret_cast<const int32_t *>(bb + M.bo_bword);
            btab.bbucket = reinterpret_cast<const int32_t *>(bb + M.bo_bbucket);
            if (SMEM ? (TRI ? M.tri_seg_staged : M.seg_staged) : M.gseg_staged) {
                dst[np] = dsm + wbytes + M.bblob_bytes; src[np] = M.seg;
                bytes[np++] = 32u * (unsigned)M.ns;
                sseg = reinterpret_cast<const double4 *>(dsm + wbytes + M.bblob_bytes);
            }
        }
        bulk_stage(&stage_bar, np, dst, src, bytes);
    }
    // CTA ranges start at multiples of kGrab (MWT_CTA_ALIGN), so a big grab
    // is one aligned block of ray indices -- one coherent group of the
    // benchmark order -- rather than the tails of two
    const long long per = ((n + gridDim.x - 1) / gridDim.x + kCtaAlign - 1) / kCtaAlign * kCtaAlign;
    const long long cbeg = (long long)blockIdx.x * per;
    const long long cend = cbeg + per < n ? cbeg + per : n;
    if (hist) {
        for (int k = threadIdx.x; k < MWT_HIST_LEN; k += THREADS) H.bins[k] = 0u;
        H.lane_cnt[threadIdx.x] = 0ull;
        H.lane_steps[threadIdx.x] = 0ull;
    }
    if (threadIdx.x == 0) {
        H.steps_sum = 0ull;
        for (int w = 0; w < 32; w++) {
            H.warp_steps[w] = 0ull;
            H.warp_hm[w][0] = H.warp_hm[w][1] = 0u;
        }
        s_next = 0u;
    }
    __syncthreads();
    HistSm<THREADS> *Hp = hist ? &H : nullptr;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int lim = 4 * M.nt + 16;  // walk_step's guard
    // ray offsets within the CTA's range (32-bit: a range is < 2^32 rays)
    const unsigned span = (unsigned)(cend > cbeg ? cend - cbeg : 0);
    unsigned next = 0u, end = 0u;   // the warp's current grab
    bool more = span > 0u;          // warp-uniform: the CTA range is not exhausted

    // lane phase: 0 idle, 1 walking, 2 reached its exit edge (epilogue pending),
    // 3 failed (TraversalError pending)
    int phase = 0;
    unsigned idx = 0u;
    Ray r{0.0, 0.0, 0.0, 0.0};
    WalkState s;
    s.kr = 0; s.ch = 0; s.steps = 0; s.w = 0; s.fast = false;
    uint32_t st = 0;

    while (true) {
        unsigned walking = __ballot_sync(FULL, phase == 1);
        if (__popc(walking) <= refill_below) {
            if (phase >= 2) {
                epilogue<!GEN, THREADS>(&M, &L, Hp, sseg, cbeg + (long long)idx, r.ox, r.oy, r.dx, r.dy, s.kr, s.ch, s.w, st,
                         s.steps, phase);
                phase = 0;
            }
            if (more) {
                const unsigned idle = ~walking;
                const int nidle = __popc(idle), rank = __popc(idle & lt_mask);
                // rays for the idle lanes: the rest of the current grab, then a new one
                unsigned nb = end, ne = end;
                const int rem = (int)(end - next);
                if (rem < nidle) {
                    unsigned base = 0u, g = (unsigned)kGrab;
                    if (lane == 0) {
                        const unsigned cur = *reinterpret_cast<volatile unsigned *>(&s_next);
                        if (kGrabTail < kGrab && (cur >= span || span - cur < 2u * (THREADS / 32) * kGrab))
                            g = (unsigned)kGrabTail;
                        base = atomicAdd(&s_next, g);
                    }
                    base = __shfl_sync(FULL, base, 0);
                    g = __shfl_sync(FULL, g, 0);
                    nb = base < span ? base : span;
                    ne = span - nb > g ? nb + g : span;
                    if (GEN && L.src.gen.cmask && nb < ne) {
                        // the group words of the grab's first ray, once per grab
                        // (lane 0: draw 0, lane 1: draw 128); rays of another
                        // group compute their own (gen_ray)
                        const unsigned long long gs =
                            L.src.gen.gkey ^ ((L.src.first + (unsigned long long)(cbeg + nb)) >> L.src.gen.gshift);
                        const unsigned long long v = mix64(gs + (lane == 1 ? 129ull : 1ull) * kGolden);
                        const unsigned long long v1 = __shfl_sync(FULL, v, 1);
                        if (lane == 0) {
                            s_gw[threadIdx.x >> 5][0] = gs;
                            s_gw[threadIdx.x >> 5][1] = v;
                            s_gw[threadIdx.x >> 5][2] = v1;
                        }
                        __syncwarp();
                    }
                }
                if (phase == 0) {
                    const unsigned o = rank < rem ? next + rank : nb + (rank - rem);
                    if (rank < rem || o < ne) {
                        idx = o;
                        const long long i = cbeg + (long long)o;
                        const Init in = prologue_body<GEN>(M, btab, L.src, i, GEN ? s_gw[threadIdx.x >> 5] : nullptr);
                        if (!GEN && L.out.start) L.out.start[i] = in.start;
                        r.ox = in.ox; r.oy = in.oy; r.dx = in.dx; r.dy = in.dy;
                        s.w = in.w; s.kr = in.cur;
                        st = in.st;
                        phase = in.phase;
                        s.fast = in.fast;
                        s.ch = in.ei;
                        s.steps = in.steps;
                    }
                }
                if (rem >= nidle) {
                    next += nidle;
                } else {
                    next = nb + (nidle - rem) < ne ? nb + (nidle - rem) : ne;
                    end = ne;
                    more = next < end || ne < span;
                }
            }
            walking = __ballot_sync(FULL, phase == 1);
            if (walking == 0) {
                if (!more && __ballot_sync(FULL, phase != 0) == 0) break;
                continue;  // pending lanes resolve at the top of the loop
            }
        }
        // Fast steps in a tight loop: lanes in the one-candidate state (see
        // walk_step) step until too few remain to keep the warp busy -- or,
        // once the range is exhausted, until none remains.  A lane leaves on a
        // zero apex side (the general rule decides that step), at its stop
        // edge, or at the step guard (walk_step below flags the error).
        // The guard is checked once per group of kUnroll steps (a lane enters a
        // group only with steps < lim - kUnroll, so no step in it passes the guard;
        // the last few steps before the guard run in walk_step), and the stop
        // edge ends the lane's walk in the loop but its phase is set after it.
        // The apex side c = RN(p - q), p = RN(dx * RN(vy - oy)), q = RN(dy *
        // RN(vx - ox)) (side_of, no contraction), is only compared with 0
        // here, so the loop compares p with q: for finite p, q, RN(p - q) == 0
        // iff p == q (gradual underflow) and it has the sign of p - q.  p and q
        // are finite when the ray's and the mesh's coordinates are bounded by
        // 2^500 (every lane of a bounded launch; a loaded ray outside the bound,
        // or one with a NaN or infinity, takes walk_step's full rule instead).
        const int glim = L.cmp_side ? lim - kUnroll : -1;
        bool fl = phase == 1 && s.fast && s.steps < glim;
        if (!GEN)
            fl = fl && fmax(fmax(fabs(r.ox), fabs(r.oy)), fmax(fabs(r.dx), fabs(r.dy))) <= 0x1p500;
        const bool entered = fl;
        // kn: the record of the triangle the lane enters next.  It stays a
        // valid record index throughout the loop (a lane that left keeps
        // re-reading its last record and commits nothing), so the load needs
        // no select, and only kn and the step count change per step; the exit
        // word, edge and triangle are recovered after the loop from record kn.
        uint32_t kn = fl ? s.w : 0u;
        {
            const int thr = more ? refill_below : 0;
            while (__popc(__ballot_sync(FULL, fl)) > thr) {
#pragma unroll
                for (int u2 = 0; u2 < kUnroll; u2++) {
                    uint32_t wx, wy;
                    double2 A;
                    fetch_step<SMEM, TRI>(M, srec, stri, svxy, kn, wx, wy, A);
                    const double p = r.dx * (A.y - r.oy), q = r.dy * (A.x - r.ox);  // c = p - q
                    const bool ok = fl && p != q;
                    const uint32_t nw = p > q ? wx : wy;  // E1 if c > 0, else E2
                    // (a predicated add: the compiler's own form is an add and a select)
                    asm("{.reg .pred q; setp.ne.b32 q, %1, 0; @q add.s32 %0, %0, 1;}"
                        : "+r"(s.steps) : "r"((int)ok));
                    const bool go = ok && !(nw & (SMEM ? kCStop : kStopBit));
                    kn = go ? nw : kn;
                    fl = go;
                }
                fl = fl && s.steps < glim;
            }
        }
        if (entered) {
            if (fl || s.steps >= glim) {
                s.w = kn;  // left behind in the fast state, or at the guard (walk_step flags it)
            } else {
                // the lane reached its stop edge in record kn, or met a zero
                // apex side there (not counted; the general rule decides it):
                // both are pure functions of the record and the ray
                uint32_t wx, wy;
                double2 A;
                fetch_step<SMEM, TRI>(M, srec, stri, svxy, kn, wx, wy, A);
                const double c = side_of(r, A);
                if (c == 0.0) {
                    s.w = kn;
                } else {
                    const uint32_t nw = c > 0.0 ? wx : wy;
                    s.w = SMEM ? expand_cword(nw) : nw;
                    s.kr = (int)kn;
                    s.ch = c > 0.0 ? 0 : 1;
                    phase = 2;
                }
            }
        }
        // one full-rule step for every lane that left the tight loop still
        // walking (zero side, the general state, the guard); lanes it merely
        // left behind (still in the fast state) continue after the refill
        if (phase == 1 && !fl) {
            if (!walk_step(M, r, s, st)) phase = 3;
            else if (s.w & kStopBit) phase = 2;
        }
    }
    if (hist) {
        {  // this thread's counters into its warp's slots, then the CTA flush
            const unsigned long long c = H.lane_cnt[threadIdx.x];
            unsigned hh = (unsigned)(c & 0x1FFFFFu), mm = (unsigned)((c >> 21) & 0x1FFFFFu),
                     bb = (unsigned)(c >> 42);
            unsigned long long ss = H.lane_steps[threadIdx.x];
            for (int o = 16; o > 0; o >>= 1) {
                hh += __shfl_down_sync(FULL, hh, o);
                mm += __shfl_down_sync(FULL, mm, o);
                bb += __shfl_down_sync(FULL, bb, o);
                ss += __shfl_down_sync(FULL, ss, o);
            }
            if (lane == 0) {
                const int w = threadIdx.x >> 5;
                H.warp_hm[w][0] += hh;
                H.warp_hm[w][1] += mm;
                H.warp_steps[w] += ss;
                if (bb) atomicAdd(H.bins + MWT_HIST_STATUS0 + 11, bb);
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < MWT_HIST_LEN; k += THREADS)
            if (H.bins[k] && k != MWT_HIST_STEPS_SUM)
                atomicAdd(reinterpret_cast<unsigned long long *>(hist + k), (unsigned long long)H.bins[k]);
        if (threadIdx.x == 0) {
            unsigned long long hh = 0, mm = 0;
            for (int w = 0; w < THREADS / 32; w++) {
                hh += H.warp_hm[w][0];
                mm += H.warp_hm[w][1];
            }
            if (hh) atomicAdd(reinterpret_cast<unsigned long long *>(hist + MWT_HIST_HIT), hh);
            if (mm) atomicAdd(reinterpret_cast<unsigned long long *>(hist + MWT_HIST_MISS), mm);
            unsigned long long t = H.steps_sum;
            for (int w = 0; w < THREADS / 32; w++) t += H.warp_steps[w];
            if (t) atomicAdd(reinterpret_cast<unsigned long long *>(hist + MWT_HIST_STEPS_SUM), t);
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_raygen(const __grid_constant__ RayGen g,
                                                     unsigned long long first, long long n,
                                                     double *rays) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Ray r = gen_ray(g, first + (unsigned long long)i);
        double2 *p = reinterpret_cast<double2 *>(rays) + 2 * i;
        p[0] = make_double2(r.ox, r.oy);
        p[1] = make_double2(r.dx, r.dy);
    }
}

// BRUTE: locate_triangle(tri, p, "brute") (accel.py:341-349): the first
// triangle in id order that _contains p -- the lowest containing id, so the
// tie flood from it returns it unchanged -- else the nearest centroid
// (accel.py:241-253; no neighbour of it contains p either)
template <bool BRUTE>
__global__ void __launch_bounds__(kThreads) k_locate(MeshDev M, const double *pts, long long n,
                                                     int32_t *tid, uint32_t *st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double2 p = __ldg(reinterpret_cast<const double2 *>(pts) + i);
        uint32_t s = 0;
        double2 P0, P1, P2;
        int t;
        if (BRUTE) {
            const LocRes lr = loc_brute(M.cxy, M.nt, p.x, p.y);
            t = lr.tid;
            s = ST_LOC_BRUTE | lr.st;
        } else {
            t = locate(M, p.x, p.y, s, P0, P1, P2);
        }
        if (tid) tid[i] = t;
        if (st) st[i] = s;
    }
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
// launchers

#define MWT_LAUNCH_RET return (int)cudaGetLastError()

// rays per k_trace launch: per-CTA ray offsets are 32-bit and the per-thread
// hit / miss counters 21-bit (flushed once per launch), so even a one-CTA grid
// (896 threads) stays in range; the launchers split larger calls
constexpr int64_t kMaxLaunchRays = 1ll << 30;

static int g_refill_below = 6;  // tuned on B200 (tools/breakdown.py): refill when <= 6 lanes still walk
static int g_min_blocks = 4;    // register budget; see launch_k_trace_any
static int g_variant = 2;       // 2: shared-memory staged walk when a compact table fits, else 1; 3: per-triangle table first

// the launch-configuration caches below are process-wide: calls from several
// host threads (one per device or stream) serialise on this lock
static std::mutex g_cfg_mu;

template <typename K>
static int persistent_grid(K kernel, long long n, int threads = kThreads, int smem = 0) {
    // one resident wave: SMs x resident CTAs (cached per kernel, device, smem size)
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    static const void *keys[64];
    static int devs[64], smems[64], waves[64], nkeys = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int wave = 0;
    for (int k = 0; k < nkeys; k++)
        if (keys[k] == (const void *)kernel && devs[k] == dev && smems[k] == smem) wave = waves[k];
    if (wave == 0) {
        int sms = 0, blocks_per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kernel, threads, smem);
        if (blocks_per_sm <= 0) blocks_per_sm = 1;
        if (sms <= 0) sms = 148;
        wave = sms * blocks_per_sm;
        if (nkeys < 64) {
            keys[nkeys] = (const void *)kernel;
            devs[nkeys] = dev;
            smems[nkeys] = smem;
            waves[nkeys] = wave;
            nkeys++;
        }
    }
    long long want = (n + threads - 1) / threads;
    return (int)(want < wave ? (want < 1 ? 1 : want) : wave);
}


template <bool GEN, int MINB, int THREADS, bool SMEM, bool STAGE = SMEM, bool TRI = false>
static bool launch_k_trace(const MeshDev &m, const Launch &L, long long n, long long *hist,
                           void *stream) {
    auto kern = k_trace<GEN, MINB, THREADS, SMEM, STAGE, TRI>;
    const int dyn = SMEM && TRI ? m.tri_smem_bytes + m.bblob_bytes + (m.tri_seg_staged ? 32 * m.ns : 0)
                  : SMEM  ? m.smem_bytes + m.bblob_bytes + (m.seg_staged ? 32 * m.ns : 0)
                  : STAGE ? m.bblob_bytes + (m.gseg_staged ? 32 * m.ns : 0) : 0;
    if (SMEM && (TRI ? m.tri_smem_bytes : m.smem_bytes) <= 0) return false;  // does not fit
    if (STAGE) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64) return false;
        static int attr_set[64] = {};  // per instantiation and device: enabled dynamic size
        std::lock_guard<std::mutex> lk(g_cfg_mu);
        if (attr_set[dev] < dyn) {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) !=
                cudaSuccess) {
                (void)cudaGetLastError();  // does not fit: the caller falls back
                return false;
            }
            attr_set[dev] = dyn;
        }
    }
    kern<<<persistent_grid(kern, n, THREADS, dyn), THREADS, dyn, (cudaStream_t)stream>>>(
        m, L, n, hist, g_refill_below);
    return true;
}

template <bool GEN>
static void launch_k_trace_any(const MeshDev &m, const Launch &L, long long n, long long *hist,
                               void *stream) {
    // shared-memory walk table: one CTA per SM; min_blocks picks its size
    // (3: 768 threads / 80 registers, 4: 896 / 72 (default, measured best),
    // 2: 1024 / 64)
    if (g_variant == 3 && launch_k_trace<GEN, 1, 896, true, true, true>(m, L, n, hist, stream))
        return;  // (A/B knob: the per-triangle table even where the record table fits)
    if (g_variant >= 2) {
        const bool ok = g_min_blocks == 3   ? launch_k_trace<GEN, 1, 768, true>(m, L, n, hist, stream)
                        : g_min_blocks == 2 ? launch_k_trace<GEN, 1, 1024, true>(m, L, n, hist, stream)
                                            : launch_k_trace<GEN, 1, 896, true>(m, L, n, hist, stream);
        if (ok) return;
    }
    // the per-triangle compact table when the record table does not fit
    if (g_variant >= 2 && launch_k_trace<GEN, 1, 896, true, true, true>(m, L, n, hist, stream)) return;
    // global walk records; boundary table (and segments when they fit) staged
    if constexpr (GEN) {
        if (g_variant >= 2 && L.src.gen.cmask && launch_k_trace<true, 1, 896, false, true, true>(m, L, n, hist, stream))
            return;
    }
    if (g_variant >= 2 && launch_k_trace<GEN, 1, 896, false, true>(m, L, n, hist, stream)) return;
    // nothing fits shared memory (Grass-4096's 4,108-edge boundary table): the
    // same 896-thread persistent CTAs reading every table from L1/L2
    if (g_variant >= 2 && launch_k_trace<GEN, 1, 896, false, false>(m, L, n, hist, stream)) return;
    if (g_min_blocks == 3)
        launch_k_trace<GEN, 3, kThreads, false>(m, L, n, hist, stream);
    else if (g_min_blocks == 2)
        launch_k_trace<GEN, 2, kThreads, false>(m, L, n, hist, stream);
    else
        launch_k_trace<GEN, 4, kThreads, false>(m, L, n, hist, stream);
}

int launch_raygen(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n,
                  double *rays, void *stream) {
    if (n <= 0) return 0;
    RayGen g;
    if (!make_raygen(mode, box, seed, g)) return (int)cudaErrorInvalidValue;
    k_raygen<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(g, first, n, rays);
    MWT_LAUNCH_RET;
}

int launch_locate(const MeshDev &m, const double *pts, int64_t n, int32_t *tid, uint32_t *st,
                  void *stream, bool brute) {
    if (n <= 0) return 0;
    if (brute)
        k_locate<true><<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, pts, n, tid, st);
    else
        k_locate<false><<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, pts, n, tid, st);
    MWT_LAUNCH_RET;
}

int launch_trace(const MeshDev &m, const double *rays, const int32_t *start, int64_t n,
                 int32_t *o_start, int32_t *o_seg, double *o_t, double *o_u, int32_t *o_steps,
                 uint32_t *o_st, void *stream, int32_t *o_end) {
    if (n <= 0) return 0;
    // chunked so every launch keeps k_trace's 32-bit per-CTA ray offsets and
    // 21-bit per-thread hit/miss counters in range (kMaxLaunchRays)
    for (int64_t off = 0; off < n; off += kMaxLaunchRays) {
        const int64_t c = n - off < kMaxLaunchRays ? n - off : kMaxLaunchRays;
        auto at = [off](auto *p) { return p ? p + off : p; };
        Launch L{};
        L.src.rays = rays + 4 * off;
        L.src.start = at(start);
        L.out = TraceOut{at(o_start), at(o_seg), at(o_steps), at(o_t), at(o_u), at(o_st), at(o_end)};
        L.cmp_side = m.coord_small;
        launch_k_trace_any<false>(m, L, c, nullptr, stream);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return (int)e;
    }
    return 0;
}

int launch_trace_generated(const MeshDev &m, int mode, const double *box, uint64_t seed,
                           uint64_t first, int64_t n, int32_t *o_seg, double *o_t,
                           int32_t *o_steps, long long *hist, void *stream) {
    if (n <= 0) return 0;
    RayGen g;
    if (!make_raygen(mode, box, seed, g)) return (int)cudaErrorInvalidValue;
    // origins on or inside the box: |o| <= 2^500 when the box is (W * u <= 2^501)
    bool box_small = true, box4 = true;
    for (int k = 0; k < 4; k++) {
        box_small = box_small && std::fabs(box[k]) <= 0x1p499;
        // origins: box corners or x0 + RN(W u), u in [0, 1) -- within a few ulps
        // of the box, so inside [-4, 4] for a box inside [-3.5, 3.5]
        box4 = box4 && std::fabs(box[k]) <= 3.5;
    }
    for (int64_t off = 0; off < n; off += kMaxLaunchRays) {  // see launch_trace
        const int64_t c = n - off < kMaxLaunchRays ? n - off : kMaxLaunchRays;
        auto at = [off](auto *p) { return p ? p + off : p; };
        Launch L{};
        L.src.gen = g;
        L.src.first = first + (uint64_t)off;
        L.src.box_in4 = box4;
        L.out = TraceOut{nullptr, at(o_seg), at(o_steps), at(o_t), nullptr, nullptr, nullptr};
        L.cmp_side = m.coord_small && box_small;  // generated directions have |d| <= 1
        launch_k_trace_any<true>(m, L, c, hist, stream);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return (int)e;
    }
    return 0;
}

int launch_histogram(const int32_t *seg, const int32_t *steps, const uint32_t *st, int64_t n,
                     long long *hist, void *stream) {
    if (n <= 0) return 0;
    k_histogram<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(seg, steps, st, n, hist);
    MWT_LAUNCH_RET;
}

void set_tuning(int refill_below, int min_blocks, int variant) {
    if (refill_below >= 0) g_refill_below = refill_below > 31 ? 31 : refill_below;
    if (min_blocks >= 2 && min_blocks <= 4) g_min_blocks = min_blocks;
    if (variant >= 1 && variant <= 3) g_variant = variant;
}

}  // namespace mwt
