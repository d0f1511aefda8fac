// Internal structures shared by the host packer (mwt_pack.cpp), the kernels
// (mwt_kernels.cu) and the C ABI (mwt_capi.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

#include "mwt.h"

namespace mwt {

// ---------------------------------------------------------------------------
// Packed triangulation (K1).  Layout in HBM (all arrays 16-B aligned):
//
//   link[T]   int4  walk words, one per edge i = 0..2 (edge i is opposite
//                   corner i, endpoints corners (i+1)%3, (i+2)%3 -- trimesh.py:10-13):
//                     bit31 = 0  : internal edge, step-record index 3*nbr + mirror j
//                     bit31 = 1  : walk stops here; bit30 = boundary kind,
//                                  bits 0..29 = scene segment id (geometry hit)
//                     0xFFFFFFFF : internal edge without neighbour (miss)
//                   .w = 0 (pad)
//   cxy[3T]   double2 corner coordinates (x, y) of corner k of triangle t
//                   at 3t+k: the one vertex a walk step does not already know
//                   is corner j of the neighbour -> ONE 16-B load, independent
//                   of the 16-B link load.
//   lnbr[T]   int4  locate words: (nbr << 2) | mirror for every neighbour,
//                   across constrained edges too; -1 = None.  Read only by
//                   point location (accel.py:291-330 ignores flags).
//   seg[S]    double4 (ax, ay, bx, by); segkind[S] uint8 (0 G, 1 B)
//   ep_range[2S] int2 (offset, count) into ep_ids: for endpoint e of
//                   segment s (2s = a, 2s+1 = b), the ascending geometry
//                   segment ids sharing that exact point (SceneIndex.endpoint_map).
//   anchor[res*res] int32 seed grid over [0,1]^2: triangle holding each cell
//                   centre (Triangulation.locate, trimesh.py:386-416), row-major.
//
//   step[3T] 32-B step records, one per (triangle N, entry edge j) at 3N+j:
//                   {word of edge (j+1)%3, word of edge (j+2)%3, 0, 0 | apex
//                   corner j (x, y)} -- everything one walk step needs, in one
//                   32-B sector.  A step reads exactly one record: 32
//                   algorithmic bytes per triangle entered.
// ---------------------------------------------------------------------------

constexpr uint32_t kStopBit = 0x80000000u;
constexpr uint32_t kBoundaryBit = 0x40000000u;
constexpr uint32_t kOpenWord = 0xFFFFFFFFu;
constexpr uint32_t kSidMask = 0x3FFFFFFFu;
// boundary-edge word flag: the edge's endpoints are off the side line, so the
// start test is evaluated on the device (bu then holds the edge's extent)
constexpr uint32_t kBExact = 0x80000000u;

struct HostPacked {
    int32_t nv = 0, nt = 0, ns = 0;
    int32_t res = 0, anchors_not_strict = 0, flood_filter = 1;
    int32_t coord_small = 1;  // every vertex coordinate finite and |.| <= 2^500 (see MeshDev)
    std::vector<int32_t> link;      // 4*nt
    std::vector<double> cxy;        // 6*nt
    std::vector<int32_t> step;      // 8*3*nt (32-B records)
    std::vector<int32_t> lnbr;      // 4*nt
    std::vector<double> seg;        // 4*ns
    std::vector<uint8_t> segkind;   // ns
    std::vector<int32_t> ep_range;  // 2*(2*ns)
    std::vector<int32_t> ep_ids;
    std::vector<int32_t> anchor;    // res*res
    // boundary-edge table (box-entry start triangles), one side per boundary segment
    int32_t nbsides = 0;
    int32_t unit_sides = 0;  // sides are exactly y=0, x=1, y=1, x=0 (in this order)
    struct Side {
        int32_t axis;      // 0: side lies on y = c (u = x); 1: on x = c (u = y)
        double c, lo, hi;  // the line, and the side's u extent
        int32_t off, cnt;  // its edges in bedge order (sorted by umin)
        int32_t boff, nb;  // its buckets
        double scale;      // nb / (hi - lo)
    } sides[4];
    std::vector<double> bu;         // 2 per edge: the open start interval (see mwt_pack.cpp)
    std::vector<double> bpq;        // 4 per edge: P (corner (j+1)%3), Q (corner (j+2)%3)
    std::vector<int32_t> bword;     // 3T + j, j = the boundary edge's index in T (| kBExact)
    std::vector<int32_t> bbucket;   // first edge (side-local) whose umax > bucket start
    // compact walk table (shared-memory staged walk, see kCompact* below); empty
    // when the mesh exceeds the compact word limits
    std::vector<uint32_t> crec;     // 2 per record 3N+j (+ pad to 16 B)
    std::vector<uint32_t> ctri;     // 4 per triangle: cw(edge i) | vid(corner i) << 18, i < 3; 0
    std::vector<double> vxy;        // 2 per vertex
};

// Compact walk table (K4 shared-memory variant).  Record 3N+j is 8 bytes:
//   .x = cw(word of edge (j+1)%3) | vid(corner j) << 18
//   .y = cw(word of edge (j+2)%3)
// with the vertex coordinates in a separate vxy[V] table (16 B per vertex).
// Compact words: internal edges keep their record index 3n+j (< 2^17);
// stop words are bit 17 | boundary kind at bit 16 | segment id (< 0xFFFF);
// 0x3FFFF is the open word.  For Lines-1024 (4,050 triangles, 2,052
// vertices) the table is 97 KB + 33 KB and lives in shared memory; a step then
// reads 8 + 16 bytes from shared memory and never misses.
constexpr uint32_t kCStop = 1u << 17;
constexpr uint32_t kCBoundary = 1u << 16;
constexpr uint32_t kCOpen = 0x3FFFFu;
constexpr uint32_t kCWordMask = 0x3FFFFu;
constexpr int kCVidShift = 18;
constexpr int kSmemWalkMax = 200 * 1024;  // staged only if the table fits this
// Per-triangle compact table (meshes whose record table does not fit): 16 B
// per triangle, word i = cw(edge i) | vid(corner i) << 18.  Entering N through
// its edge j, the step reads word j (apex vid; its own edge word is the entry),
// word (j+1)%3 and word (j+2)%3 -- the record 3N+j rebuilt from one 16-B load.
// 16 B/tri + 16 B/vertex instead of 24 + 16: Hair-512 (7,986 triangles, 4,008
// vertices) fits shared memory this way.

// Build the packed layout; returns MWT_OK or an error code with *err set.
int pack_mesh(const double *vx, const double *vy, int32_t nverts, const int32_t *tri_v,
              const int32_t *tri_nbr, const int32_t *tri_flag, int32_t ntris,
              const double *seg_xy, const uint8_t *seg_kind, int32_t nsegs, HostPacked *out,
              std::string *err);

// Device view passed by value to kernels.
struct MeshDev {
    int32_t nt, ns, res, flood_filter;
    const int4 *link;
    const double2 *cxy;
    const int4 *step;  // record k occupies step[2k] (words) and step[2k+1] (apex as double2)
    const int4 *lnbr;
    const double4 *seg;
    const uint8_t *segkind;
    const int2 *ep_range;
    const int32_t *ep_ids;
    const int32_t *anchor;
    double inv_res;  // 1.0 / res (seed-cell centres: (c + 0.5) * inv_res)
    // boundary-edge table: start triangles of rays whose origin lies on a box side
    int32_t nbsides;
    int32_t unit_sides;  // sides ordered y=0, x=1, y=1, x=0: the side is found without loads
    struct BSide {
        int32_t axis, off, cnt, boff, nb;
        double c, lo, hi, scale;
    } bs[4];
    const double2 *bu;      // the open start interval per edge (mwt_pack.cpp start_interval)
    const double4 *bpq;     // (P.x, P.y, Q.x, Q.y) per edge
    const int32_t *bword;
    const int32_t *bbucket;
    // compact walk table for the shared-memory staged walk (NULL if absent)
    const uint2 *crec;
    const double2 *vxy;
    int32_t crec_bytes;  // 16-B padded size of crec; vxy follows it in shared memory
    int32_t smem_bytes;  // crec_bytes + 16 * nv if the table fits kSmemWalkMax, else 0
    // the boundary-edge table as one blob (staged next to the walk table):
    // bu at 0, bpq at bo_bpq, bword at bo_bword, bbucket at bo_bbucket (bytes)
    const uint4 *bblob;
    int32_t bblob_bytes, bo_bpq, bo_bword, bo_bbucket;
    int32_t seg_staged;  // the segments (32 B each) also fit: staged after the blob
    int32_t gseg_staged;  // without the walk table: the segments fit after the blob
    // per-triangle compact table (staged when the record table does not fit)
    const uint4 *ctri;
    int32_t tri_smem_bytes;  // 16 * nt + 16 * nv if that plus the blob fits kSmemWalkMax, else 0
    int32_t tri_seg_staged;  // ... and the segments fit after it
    // every vertex coordinate is finite with |x|, |y| <= 2^500: for a ray
    // with the same bound (|d| <= 2^500 too) the two products of side_of
    // cannot overflow, and the walk loop decides the apex side by comparing
    // them (k_trace's tight loop)
    int32_t coord_small;
};

// K5 BVH (mwt_bvh_create).  A node visit reads both children's boxes and
// refs from the parent's slots (no dependent load through a child index).
// A ref is the child's node id if internal, ~node id if a leaf.
struct BvhDev {
    int32_t nnodes;
    double4 root;           // the root's box (the walk's first test)
    int32_t root_ref;       // the root's ref
    const double4 *cbox;    // [2n]: boxes of node n's left, right child (internal n)
    const int2 *cref;       // [n]: refs of node n's left, right child (internal n)
    const int2 *prange;     // [n]: (prim_off, prim_cnt) of leaf n
    const int32_t *prims;
    // the four arrays as one blob (cbox at 0), for staging in shared memory
    const void *blob;
    int32_t blob_bytes, o_cref, o_prange, o_prims;
};

// K6 roped kd-tree (mwt_kd_create).  Node words by node id; one 64-B record
// per leaf by leaf slot (the leaf's rank in node order).
struct KdLeaf {
    double4 box;
    int4 ropes;  // rope target node ids per side (-1: none)
    int4 meta;   // (prim_off, prim_cnt, rope cost of side s in bits 8s..8s+7, 0)
};

struct KdDev {
    int32_t nnodes, nleaves;
    const int4 *node;     // internal: (pos lo, pos hi, left, right | axis << 31); leaf: (0, 0, -1, slot)
    const KdLeaf *leaf;   // [nleaves]
    const int32_t *prims;
};

// launchers (mwt_kernels.cu); return cudaError_t as int
int launch_raygen(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n,
                  double *rays, void *stream);
int launch_locate(const MeshDev &m, const double *pts, int64_t n, int32_t *tid, uint32_t *st,
                  void *stream, bool brute = false);
int launch_trace(const MeshDev &m, const double *rays, const int32_t *start, int64_t n,
                 int32_t *o_start, int32_t *o_seg, double *o_t, double *o_u, int32_t *o_steps,
                 uint32_t *o_st, void *stream, int32_t *o_end = nullptr);
int launch_trace_generated(const MeshDev &m, int mode, const double *box, uint64_t seed,
                           uint64_t first, int64_t n, int32_t *o_seg, double *o_t,
                           int32_t *o_steps, long long *hist, void *stream);
void set_tuning(int refill_below, int min_blocks, int variant);
// L2 read-bandwidth probe (the walk's on-chip roof, measured on the box):
// streaming 128-bit ld.global.cg over a bytes-sized buffer, `passes` times
int probe_l2_read(size_t bytes, int passes, float *ms);
int launch_histogram(const int32_t *seg, const int32_t *steps, const uint32_t *st, int64_t n,
                     long long *hist, void *stream);
int launch_bvh(const MeshDev &m, const BvhDev &b, const double *rays, int64_t n, int32_t *o_seg,
               double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_prims, uint32_t *o_st,
               void *stream);
int launch_kd(const MeshDev &m, const KdDev &k, const double *rays, const int32_t *start, int64_t n, int32_t *o_seg,
              double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_ropes, int32_t *o_prims,
              uint32_t *o_st, void *stream);
int launch_brute(const MeshDev &m, const double *rays, int64_t n, int32_t *o_seg, double *o_t,
                 double *o_u, void *stream);

}  // namespace mwt
