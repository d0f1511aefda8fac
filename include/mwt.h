/*
 * mwt.h -- C ABI of the B200 batched 2D ray-query engine (libmwt.so).
 *
 * Drop-in boundary for the hot path of the reference package `mintri`
 * (arXiv 2112.05570): stackless closest-hit traversal of rays through a
 * constrained triangulation, plus the point location that seeds it and the
 * like-for-like roped kd-tree / SAH BVH engines.  The reference exposes this
 * path only as Python functions (it has no native layer); each entry point
 * below names the reference function it replaces.  A ctypes binding of every
 * symbol lives in paper_2112_05570_b200/_lib.py, and INTEGRATION.md shows the
 * shim a `mintri` maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes; no torch / CUDA types in the signatures.
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Functions named *_dev take DEVICE pointers and are asynchronous on
 *    `stream`; functions named *_host take HOST pointers, copy in and out and
 *    synchronise before returning.
 *  - Rays are float64 quadruples (ox, oy, dx, dy), row-major, 32 B per ray.
 *    Directions are used exactly as given (the reference's `Ray` has already
 *    renormalised them, geometry.py:68-74).
 *  - Every function returns 0 on success or a negative MWT_E* code; the
 *    message of the last failure on the calling thread is mwt_last_error().
 *  - Per-ray results: seg (int32, -1 = no hit), t and u (float64, NaN on a
 *    miss), steps (int32), status (uint32 bit set, MWT_ST_*).
 */
#ifndef MWT_H
#define MWT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MWT_ABI_VERSION 3

/* return codes */
#define MWT_OK 0
#define MWT_E_INVALID (-1)   /* bad argument / malformed mesh */
#define MWT_E_CUDA (-2)      /* CUDA runtime failure */
#define MWT_E_NOMEM (-3)
#define MWT_E_TOPOLOGY (-4)  /* neighbour symmetry broken (trimesh.py:283-311) */

/* per-ray status bits (degeneracy enumeration) */
#define MWT_ST_ERROR 1u        /* TraversalError: loop or no exit (accel.py:164-191) */
#define MWT_ST_FALLBACK 2u     /* no candidate exit edge, fallback used (accel.py:188-189) */
#define MWT_ST_GRAZING 4u      /* ray_segment_intersect None at a constrained edge (accel.py:199-207) */
#define MWT_ST_CANON 8u        /* canonical() moved the hit to a lower id (accel.py:82-98) */
#define MWT_ST_PARALLEL 16u    /* parallel branch of ray_segment_intersect (geometry.py:149-161) */
#define MWT_ST_ZERO_SIDE 32u   /* exact-zero side value at an exit candidate */
#define MWT_ST_MULTI 64u       /* more than one exit candidate in one triangle */
#define MWT_ST_LOC_TIE 128u    /* locate flood visited >1 containing triangle (accel.py:226-238) */
#define MWT_ST_LOC_BRUTE 256u  /* anchor walk failed, brute-force scan (accel.py:287-288) */
#define MWT_ST_LOC_OUTSIDE 512u /* point outside every triangle: nearest centroid (accel.py:245-246) */
#define MWT_ST_OVERFLOW 1024u  /* device capacity exceeded (flood/stack); result invalid */
#define MWT_ST_BOUNDARY 2048u  /* engine-side note: start triangle from the boundary-edge table */

/* ray generator modes (engine-defined) */
#define MWT_RAYS_BOX_ENTRY 0   /* isotropic lines through the box, origin at box entry */
#define MWT_RAYS_INTERIOR 1    /* origin uniform in the box, isotropic direction */
/* Coherent ray order: a mode word base | group_log2 << 8 | cell_bits << 16.
 * Every 64-bit draw of ray i keeps its own low bits and takes the top
 * `cell_bits` of each 32-bit half from the same draw of its group's stream
 * (group = i >> group_log2).  Each ray is still an exact draw of the base
 * distribution (its draws remain uniform words); rays of one group share a
 * cell of the direction draw and of the entry-point draw, so a warp's rays run
 * nearly the same line.  cell_bits = 0 is the iid
 * generator; cell_bits <= 16, group_log2 <= 40. */
#define MWT_RAYS_COHERENT(base, group_log2, cell_bits) \
    ((base) | ((group_log2) << 8) | ((cell_bits) << 16))
/* the benchmark's ordering: groups of 512 rays (four warp grabs), 12 shared bits per coordinate */
#define MWT_RAYS_BOX_ENTRY_COHERENT MWT_RAYS_COHERENT(MWT_RAYS_BOX_ENTRY, 9, 12)
#define MWT_RAYS_INTERIOR_COHERENT MWT_RAYS_COHERENT(MWT_RAYS_INTERIOR, 9, 12)

/* histogram layout written by mwt_trace_generated_dev / mwt_histogram_dev */
#define MWT_HIST_STEP_BINS 1024 /* bins 0..1022 exact step counts, 1023 = overflow */
#define MWT_HIST_HIT 1024       /* rays with a hit */
#define MWT_HIST_MISS 1025      /* rays without a hit (boundary / open edge) */
#define MWT_HIST_STEPS_SUM 1026 /* sum of tri_steps */
#define MWT_HIST_STATUS0 1027   /* 12 counters, one per MWT_ST_* bit */
#define MWT_HIST_LEN 1040       /* int64 entries */

typedef struct mwt_mesh mwt_mesh;
typedef struct mwt_bvh mwt_bvh;
typedef struct mwt_kd mwt_kd;

typedef struct {
    int32_t num_vertices, num_triangles, num_segments;
    int32_t anchor_res;            /* TriLocator grid resolution (accel.py:265-266) */
    int32_t anchors_not_strict;    /* anchor centres on an edge/vertex (order-dependent seeds) */
    int32_t device;
    int64_t device_bytes;          /* total device footprint of the packed mesh */
    int64_t walk_record_bytes;     /* algorithmic bytes per triangle step (32) */
    int64_t walk_smem_bytes;       /* compact walk table staged in shared memory per CTA
                                      (0: walk records read from global memory) */
} mwt_mesh_info;

/* Library / error plumbing */
int mwt_abi_version(void);
const char *mwt_last_error(void);

/* Identity of this build: sha256 (hex, first 16 bytes) of the kernel and ABI
 * sources and the nvcc flags they were compiled with -- profiles captured with
 * ncu are keyed to it (bench.py). */
const char *mwt_build_id(void);
int mwt_device_count(int *count);
/* Tuning knobs of the persistent walk kernel (process-wide; -1 = keep).
 * Lanes whose rays ended refill in one batch once at most `refill_below`
 * (default 6) lanes of the warp still walk.  `variant` 2 (default) stages the
 * mesh's compact walk table in shared memory when it fits, one CTA per SM
 * whose size `min_blocks_per_sm` picks (3: 768 threads / 80 registers,
 * 4: 896 / 72 (default), 2: 1024 / 64), else the per-triangle compact table
 * (16 B per triangle) when that fits, else walks the 32-B records from
 * global memory with the boundary table staged (896 threads); variant 3 tries
 * the per-triangle table first (A/B); variant 1 always
 * walks from global memory with 256-thread CTAs, `min_blocks_per_sm` CTAs per SM.
 * With variant 2 or 3, `min_blocks_per_sm` only sizes the record-table CTA:
 * the per-triangle and global-record paths always use 896-thread CTAs. */
int mwt_set_tuning(int refill_below, int min_blocks_per_sm, int variant);

/* Measurement helper (no reference counterpart): L2 read bandwidth of
 * `device`, streaming 128-bit ld.global.cg loads over an L2-resident buffer of
 * `bytes` (1 MiB .. 1 GiB) `passes` times from every SM -- the on-chip roof the
 * walk's algorithmic bytes are compared with.  Synchronous. */
int mwt_probe_l2_read(int device, int64_t bytes, int passes, double *gbs_out);

/* K1 -- mesh packer.
 * Replaces: building `Triangulation` + `SceneIndex` for the walk
 *   (trimesh.py:93-150 data model; accel.py:64-80 SceneIndex; accel.py:263-282 anchors).
 * Inputs are the reference data model exactly as `load_triangulation`
 * (trimesh.py:1309-1337) / `parse_scene` (scene.py:135-165) hold it:
 *   vx, vy[nverts]; tri_v, tri_nbr, tri_flag[3*ntris] (nbr -1 = None,
 *   flag -1 = INTERNAL or a scene segment id); seg_xy[4*nsegs] (ax, ay, bx, by);
 *   seg_kind[nsegs] (0 = GEOMETRY 'G', 1 = BOUNDARY 'B').
 * Host arrays are copied; the handle owns the device copies. */
int mwt_mesh_create(const double *vx, const double *vy, int32_t nverts,
                    const int32_t *tri_v, const int32_t *tri_nbr, const int32_t *tri_flag,
                    int32_t ntris, const double *seg_xy, const uint8_t *seg_kind, int32_t nsegs,
                    int device, mwt_mesh **out);
int mwt_mesh_destroy(mwt_mesh *mesh);
/* Host-only dry run of the packer (no device needed): validates the input
 * exactly as mwt_mesh_create does and optionally returns the packed walk
 * words (4*ntris int32: link[t].x/y/z/w) and locate words (4*ntris int32),
 * plus the seed-grid resolution and its cell-centre triangles
 * (out_anchor: res*res int32, query res first with out_anchor = NULL). */
int mwt_pack_dry_run(const double *vx, const double *vy, int32_t nverts, const int32_t *tri_v,
                     const int32_t *tri_nbr, const int32_t *tri_flag, int32_t ntris,
                     const double *seg_xy, const uint8_t *seg_kind, int32_t nsegs,
                     int32_t *out_link, int32_t *out_lnbr, int32_t *out_res, int32_t *out_anchor);
int mwt_mesh_info_get(const mwt_mesh *mesh, mwt_mesh_info *out);
/* copy the device-side anchor table (res*res int32) to host, for tests */
int mwt_mesh_anchors(const mwt_mesh *mesh, int32_t *out_host);

/* K2 -- seeded ray generator.  No reference counterpart (the reference's
 * sample_rays, experiment.py:29-63, draws interior origins); realises the
 * BASELINE.json ray recipe.  box = (x0, y0, x1, y1); rays for global indices
 * first .. first+n-1 go to rays_out (device, 4*n doubles). */
int mwt_raygen_dev(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n,
                   double *rays_out, void *stream);

/* K3 -- start-triangle location.
 * Replaces: TriLocator(tri).locate(p) / locate_triangle(tri, p, "anchor")
 *   (accel.py:284-289, :333-353).  pts = n (x, y) pairs (device). */
int mwt_locate_dev(const mwt_mesh *mesh, const double *pts, int64_t n, int32_t *out_tid,
                   uint32_t *out_status, void *stream);
/* Replaces: locate_triangle(tri, p, method="brute") (accel.py:341-349): the
 * lowest triangle id that _contains p (a scan in id order), else the nearest
 * centroid (locate_brute_force, accel.py:241-253).  O(triangles) per point. */
int mwt_locate_brute_dev(const mwt_mesh *mesh, const double *pts, int64_t n, int32_t *out_tid,
                         uint32_t *out_status, void *stream);

/* K4 -- the MWT walk.
 * Replaces: traverse_triangulation(tri, ray, start_tri, index) (accel.py:138-213),
 *   with start_tri = TriLocator.locate(origin) when start == NULL
 *   (the per-ray loop of run_experiment, experiment.py:166-171).
 * Any output pointer may be NULL (not written).  out_start receives the
 * start triangle actually used. */
int mwt_trace_dev(const mwt_mesh *mesh, const double *rays, const int32_t *start, int64_t n,
                  int32_t *out_start, int32_t *out_seg, double *out_t, double *out_u,
                  int32_t *out_steps, uint32_t *out_status, void *stream);
/* K4 for chained (secondary) rays: as mwt_trace_dev, and out_end receives the
 * triangle each walk ended in (the one whose exit edge is the hit segment or
 * the boundary; -1 after a TraversalError).  Passing it back as the next ray's
 * start replaces the locate (Ray.start_tri,
 * geometry.py:66, consumed by traverse_triangulation, accel.py:138-160). */
int mwt_trace_chain_dev(const mwt_mesh *mesh, const double *rays, const int32_t *start, int64_t n,
                        int32_t *out_end, int32_t *out_seg, double *out_t, double *out_u,
                        int32_t *out_steps, uint32_t *out_status, void *stream);
/* Same as mwt_trace_dev on HOST buffers (copies in, traces, copies out, syncs). */
int mwt_trace_host(const mwt_mesh *mesh, const double *rays, const int32_t *start, int64_t n,
                   int32_t *out_start, int32_t *out_seg, double *out_t, double *out_u,
                   int32_t *out_steps, uint32_t *out_status);

/* K2+K3+K4+K7 fused: generate rays first..first+n-1 on device, locate, walk,
 * write optional per-ray outputs and ADD into hist (device int64[MWT_HIST_LEN],
 * may be NULL).  This is the benchmark kernel; rays never touch HBM. */
int mwt_trace_generated_dev(const mwt_mesh *mesh, int mode, const double *box, uint64_t seed,
                            uint64_t first, int64_t n, int32_t *out_seg, double *out_t,
                            int32_t *out_steps, int64_t *hist, void *stream);

/* K7 -- accumulate per-ray results into a histogram (device). */
int mwt_histogram_dev(const int32_t *seg, const int32_t *steps, const uint32_t *status, int64_t n,
                      int64_t *hist, void *stream);

/* K5 -- SAH BVH walk.
 * Replaces: bvh_intersect(bvh, ray) / Bvh.intersect (accel.py:482-518, :428).
 * The tree is the reference Bvh flattened in DFS preorder (node 0 = root):
 * box[4*nnodes]; left/right child index or -1 for a leaf; leaf prims
 * prims[prim_off .. prim_off+prim_cnt) in reference order. */
int mwt_bvh_create(const mwt_mesh *mesh, int32_t nnodes, const double *box, const int32_t *left,
                   const int32_t *right, const int32_t *prim_off, const int32_t *prim_cnt,
                   int32_t nprims, const int32_t *prims, mwt_bvh **out);
int mwt_bvh_destroy(mwt_bvh *bvh);
int mwt_bvh_trace_dev(const mwt_bvh *bvh, const double *rays, int64_t n, int32_t *out_seg,
                      double *out_t, double *out_u, int32_t *out_node_tests,
                      int32_t *out_prim_tests, uint32_t *out_status, void *stream);

/* K6 -- roped kd-tree walk.
 * Replaces: kd_intersect(kd, ray) / RopedKdTree.intersect (accel.py:761-832, :726),
 * start leaf by RopedKdTree.locate_leaf(origin, direction) (accel.py:712-724).
 * Node table in DFS preorder: axis (-1 = leaf), pos, left, right, box[4],
 * ropes[4] (node index or -1), rope_cost[4] = max(1, ceil(log2(count))),
 * leaf prims as for the BVH; num_leaves sets the walk guard 4*leaves+16. */
int mwt_kd_create(const mwt_mesh *mesh, int32_t nnodes, int32_t num_leaves, const int32_t *axis,
                  const double *pos, const int32_t *left, const int32_t *right, const double *box,
                  const int32_t *ropes, const int32_t *rope_cost, const int32_t *prim_off,
                  const int32_t *prim_cnt, int32_t nprims, const int32_t *prims, mwt_kd **out);
int mwt_kd_destroy(mwt_kd *kd);
/* start_leaf: NULL (locate_leaf per ray) or per-ray node indices of the
 * leaves to start from -- kd_intersect(kd, ray, start_leaf=...) (accel.py:761-771);
 * an index that is not a leaf gives MWT_ST_ERROR for that ray. */
int mwt_kd_trace_dev(const mwt_kd *kd, const double *rays, const int32_t *start_leaf, int64_t n,
                     int32_t *out_seg, double *out_t, double *out_u, int32_t *out_nodes,
                     int32_t *out_rope_steps, int32_t *out_prim_tests, uint32_t *out_status,
                     void *stream);

/* Brute-force closest hit (the reference's oracle engine).
 * Replaces: brute_force_closest(scene, ray, index) (accel.py:101-132). */
int mwt_brute_force_dev(const mwt_mesh *mesh, const double *rays, int64_t n, int32_t *out_seg,
                        double *out_t, double *out_u, void *stream);

/* One process, several GPUs (SURVEY.md §8b `mwt_run_sharded`; the reference is
 * single-process, accel.py has no counterpart).  `meshes[k]` is the same mesh
 * created on device k (ndev <= 64); rays [first, first + n) -- or the host
 * rays -- split into contiguous near-equal ranges, one per device, each driven
 * by its own host thread and stream; results are those of one device.
 * mwt_trace_generated_sharded sums the per-device histograms into hist_out
 * (host int64[MWT_HIST_LEN]); mwt_trace_host_sharded writes the per-ray host
 * outputs like mwt_trace_host.  Synchronous. */
int mwt_trace_generated_sharded(const mwt_mesh *const *meshes, int ndev, int mode, const double *box,
                                uint64_t seed, uint64_t first, int64_t n, int64_t *hist_out);
int mwt_trace_host_sharded(const mwt_mesh *const *meshes, int ndev, const double *rays,
                           const int32_t *start, int64_t n, int32_t *out_start, int32_t *out_seg,
                           double *out_t, double *out_u, int32_t *out_steps, uint32_t *out_status);

#ifdef __cplusplus
}
#endif
#endif /* MWT_H */
