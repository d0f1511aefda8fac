// K5 BVH, K6 roped kd-tree and brute-force kernels (B200, sm_100a).
// Compiled with -fmad=false: reference operation order, no contraction.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "mwt_device.cuh"

namespace mwt {

#ifndef MWT_STRUCT_MINB
#define MWT_STRUCT_MINB 4
#endif
constexpr int kStructMinB = MWT_STRUCT_MINB;  // resident CTAs per SM the register budget targets

// Ray order of the kd / BVH kernels: each CTA takes a contiguous range of
// rays (a coherent ray order then keeps one SM's working set small), or
// (MWT_STRUCT_CONTIG=0) the grid-stride order.
#ifndef MWT_STRUCT_CONTIG
#define MWT_STRUCT_CONTIG 0
#endif
struct RayRange {
    long long i, end, step;
};
__device__ __forceinline__ RayRange cta_rays(long long n) {
    if (MWT_STRUCT_CONTIG) {
        const long long per = (n + gridDim.x - 1) / gridDim.x, b = blockIdx.x * per;
        return {b + threadIdx.x, b + per < n ? b + per : n, (long long)blockDim.x};
    }
    return {blockIdx.x * (long long)blockDim.x + threadIdx.x, n, (long long)gridDim.x * blockDim.x};
}

// ---------------------------------------------------------------------------
// K5: BVH, accel.py:460-518

// _ray_box (accel.py:460-476).  rx, ry: the ray's reciprocal direction
// components (make_rcp), so each slab bound is a division-free exact quotient.
__device__ __forceinline__ bool ray_box(const Ray &r, const Rcp &rx, const Rcp &ry, double4 b, double &tn) {
    double tmin = 0.0, tmax = CUDART_INF;
    // x slab then y slab; Python max/min keep the first operand on ties
    if (r.dx == 0.0) {
        if (r.ox < b.x || r.ox > b.z) return false;
    } else {
        double t1 = div_rcp(b.x - r.ox, rx), t2 = div_rcp(b.z - r.ox, rx);
        if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
        tmin = t1 > tmin ? t1 : tmin;
        tmax = t2 < tmax ? t2 : tmax;
        if (tmin > tmax) return false;
    }
    if (r.dy == 0.0) {
        if (r.oy < b.y || r.oy > b.w) return false;
    } else {
        double t1 = div_rcp(b.y - r.oy, ry), t2 = div_rcp(b.w - r.oy, ry);
        if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
        tmin = t1 > tmin ? t1 : tmin;
        tmax = t2 < tmax ? t2 : tmax;
        if (tmin > tmax) return false;
    }
    tn = tmin;
    return true;
}

// 32-B / 16-B read-only loads (the tables are immutable for a launch)
__device__ __forceinline__ double4 ld_box(const double4 *p, bool smem) {
    if (smem) return *p;
    return ldg4d(p);
}

// STAGE: the child boxes / refs, leaf ranges and primitive ids (one blob) and
// the segments are copied into shared memory once per CTA (persistent
// grid-stride CTAs) when they fit, as the walk kernel stages its tables.
// Stack of (tnear, ref) in local memory (L1); kBvhStack entries.
template <bool STAGE>
__global__ void __launch_bounds__(kThreads, kStructMinB) k_bvh(MeshDev M, BvhDev B, const double *rays,
                                                               long long n, int32_t *o_seg, double *o_t,
                                                               double *o_u, int32_t *o_nodes, int32_t *o_prims,
                                                               uint32_t *o_st) {
    extern __shared__ __align__(16) unsigned char bsm[];
    if (STAGE) {
        const int nb = B.blob_bytes >> 4, ns2 = 2 * M.ns;
        uint4 *d = reinterpret_cast<uint4 *>(bsm);
        const uint4 *a = reinterpret_cast<const uint4 *>(B.blob);
        const uint4 *sg = reinterpret_cast<const uint4 *>(M.seg);
        for (int k = threadIdx.x; k < nb + ns2; k += blockDim.x)
            d[k] = k < nb ? __ldg(a + k) : __ldg(sg + (k - nb));
        __syncthreads();
        B.cbox = reinterpret_cast<const double4 *>(bsm);
        B.cref = reinterpret_cast<const int2 *>(bsm + B.o_cref);
        B.prange = reinterpret_cast<const int2 *>(bsm + B.o_prange);
        B.prims = reinterpret_cast<const int32_t *>(bsm + B.o_prims);
    }
    // the segments the leaf tests read (canonical keeps the global copy: the
    // segment table itself, rarely read)
    const double4 *segs = STAGE ? reinterpret_cast<const double4 *>(bsm + B.blob_bytes) : M.seg;
    const RayRange rr = cta_rays(n);
    for (long long i = rr.i; i < rr.end; i += rr.step) {
        Ray r = load_ray(rays, i);
        const Rcp rx = make_rcp(r.dx), ry = make_rcp(r.dy);
        int nodes = 1, prims = 0, bsid = -1;
        bool have = false;
        uint32_t st = 0;
        double bt = 0.0, bu = 0.0, tn;
        int seg = -1;
        double ot = CUDART_NAN, ou = CUDART_NAN;
        if (ray_box(r, rx, ry, B.root, tn)) {
            double st_t[kBvhStack];
            int st_n[kBvhStack];
            st_t[0] = tn;
            st_n[0] = B.root_ref;
            int top = 1;
            while (top > 0) {
                top--;
                const double tnear = st_t[top];
                const int ref = st_n[top];
                if (have && tnear > bt + 1e-12) continue;
                if (ref < 0) {  // leaf: accel.py:497-505
                    const int2 pr = STAGE ? B.prange[~ref] : __ldg(B.prange + ~ref);
                    for (int k = 0; k < pr.y; k++) {
                        const int sid = STAGE ? B.prims[pr.x + k] : __ldg(B.prims + pr.x + k);
                        prims++;
                        double t, u;
                        bool par = false;
                        if (!rsi(r, ld_box(segs + sid, STAGE), t, u, par)) continue;
                        if (!have || t < bt) { have = true; bt = t; bsid = sid; bu = u; }
                    }
                    continue;
                }
                // both children's boxes and refs from this node's slots
                const int2 ch = STAGE ? B.cref[ref] : __ldg(B.cref + ref);
                const double4 bl = ld_box(B.cbox + 2 * ref, STAGE), br = ld_box(B.cbox + 2 * ref + 1, STAGE);
                double tl = 0.0, tr = 0.0;
                nodes += 2;
                const bool hl = ray_box(r, rx, ry, bl, tl) && (!have || tl <= bt + 1e-12);
                const bool hr = ray_box(r, rx, ry, br, tr) && (!have || tr <= bt + 1e-12);
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

// locate_leaf / the rope descent (accel.py:712-724, :820-830): one 16-B node
// word per level; returns the leaf's slot
__device__ __forceinline__ int kd_descend(const KdDev &K, int node, double px, double py, double dx,
                                          double dy, int &nodes, bool count) {
    int4 N = __ldg(K.node + node);
    while (N.z >= 0) {
        if (count) nodes++;
        const bool ay = (uint32_t)N.w >> 31;
        const int right = N.w & 0x7FFFFFFF;
        const double pos = __hiloint2double(N.y, N.x);
        const double coord = ay ? py : px;
        if (coord < pos) node = N.z;
        else if (coord > pos) node = right;
        else node = (ay ? dy : dx) > 0.0 ? right : N.z;
        N = __ldg(K.node + node);
    }
    return N.w;
}

// The reference's `tested` set (accel.py:775, :803-806) only decides which
// primitive tests are counted (a repeated test cannot change `best`), but
// the counter is part of the result: per ray, the tested ids in a local list
// (kKdMailbox entries; beyond: ST_OVERFLOW) and a 32-bit filter of them in a
// register, which skips the list scan for most new ids.  (Measured against a
// shared-memory hash table of the ids: the table's shared memory costs L1
// capacity, FloorPlan -20%.)
__device__ __forceinline__ uint32_t mbx_bit(int sid) { return 1u << (((uint32_t)sid * 0x9E3779B1u) >> 27); }

__global__ void __launch_bounds__(kThreads, kStructMinB) k_kd(MeshDev M, KdDev K, const double *rays,
                                                              const int32_t *start, long long n, int32_t *o_seg,
                                                              double *o_t, double *o_u, int32_t *o_nodes,
                                                              int32_t *o_ropes, int32_t *o_prims, uint32_t *o_st) {
    const RayRange rr = cta_rays(n);
    for (long long i = rr.i; i < rr.end; i += rr.step) {
        Ray r = load_ray(rays, i);
        const Rcp rx = make_rcp(r.dx), ry = make_rcp(r.dy);
        int nodes = 0, ropes = 0, prims = 0, bsid = -1, seg = -1;
        bool have = false, done = false;
        uint32_t st = 0;
        double bt = 0.0, bu = 0.0, ot = CUDART_NAN, ou = CUDART_NAN;
        uint32_t filter = 0u;  // bit mbx_bit(sid) of every listed id
        int tested[kKdMailbox];
        int ntested = 0;
        int dummy = 0;
        int cur;
        long long guard = 4LL * K.nleaves + 16;
        if (start) {  // kd_intersect(kd, ray, start_leaf): the given leaf (accel.py:771)
            const int sn = __ldg(start + i);
            const int4 N = sn >= 0 && sn < K.nnodes ? __ldg(K.node + sn) : make_int4(0, 0, 0, 0);
            cur = N.w;
            if (N.z >= 0) {
                cur = 0;
                guard = 0;  // not a leaf: reported as an error
            }
        } else {
            cur = kd_descend(K, 0, r.ox, r.oy, r.dx, r.dy, dummy, false);  // locate_leaf
        }
        while (guard > 0 && !done) {
            guard--;
            nodes++;
            const KdLeaf *lf = K.leaf + cur;
            const double4 bb = ldg4d(&lf->box);
            const int4 meta = __ldg(&lf->meta);
            double t_exit = CUDART_INF;
            int side = -1;
            if (r.dx > 0.0) {
                double tx = div_rcp(bb.z - r.ox, rx);
                if (tx < t_exit) { t_exit = tx; side = 1; }
            } else if (r.dx < 0.0) {
                double tx = div_rcp(bb.x - r.ox, rx);
                if (tx < t_exit) { t_exit = tx; side = 0; }
            }
            if (r.dy > 0.0) {
                double ty = div_rcp(bb.w - r.oy, ry);
                if (ty < t_exit) { t_exit = ty; side = 3; }
            } else if (r.dy < 0.0) {
                double ty = div_rcp(bb.y - r.oy, ry);
                if (ty < t_exit) { t_exit = ty; side = 2; }
            }
            for (int k = 0; k < meta.y; k++) {
                const int sid = __ldg(K.prims + meta.x + k);
                bool dup = false;
                const uint32_t fb = mbx_bit(sid);
                if (filter & fb)
                    for (int q = 0; q < ntested; q++) dup |= (tested[q] == sid);
                if (!dup) {
                    if (ntested == kKdMailbox) { st |= ST_OVERFLOW; done = true; break; }
                    tested[ntested++] = sid;
                    filter |= fb;
                    prims++;
                }
                if (dup) continue;
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
            const int rope = __ldg(reinterpret_cast<const int *>(&lf->ropes) + side);
            if (rope < 0) { done = true; break; }
            ropes += ((uint32_t)meta.z >> (8 * side)) & 0xFFu;
            const double px = r.ox + t_exit * r.dx, py = r.oy + t_exit * r.dy;
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

#define MWT_LAUNCH_RET return (int)cudaGetLastError()

int grid_for(long long n) {
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

int launch_bvh(const MeshDev &m, const BvhDev &b, const double *rays, int64_t n, int32_t *o_seg,
               double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_prims, uint32_t *o_st,
               void *stream) {
    if (n <= 0) return 0;
    const int dyn = b.blob_bytes + 32 * m.ns;
    if (dyn <= 200 * 1024) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaFuncSetAttribute(k_bvh<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) ==
                cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bvh<true>, kThreads, dyn) ==
                cudaSuccess &&
            per > 0) {
            long long want = (n + kThreads - 1) / kThreads, wave = (long long)(sms > 0 ? sms : 148) * per;
            const int grid = (int)(want < wave ? (want < 1 ? 1 : want) : wave);
            k_bvh<true><<<grid, kThreads, dyn, (cudaStream_t)stream>>>(m, b, rays, n, o_seg, o_t, o_u,
                                                                      o_nodes, o_prims, o_st);
            MWT_LAUNCH_RET;
        }
        (void)cudaGetLastError();
    }
    k_bvh<false><<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, b, rays, n, o_seg, o_t, o_u,
                                                                     o_nodes, o_prims, o_st);
    MWT_LAUNCH_RET;
}

int launch_kd(const MeshDev &m, const KdDev &k, const double *rays, const int32_t *start, int64_t n, int32_t *o_seg,
              double *o_t, double *o_u, int32_t *o_nodes, int32_t *o_ropes, int32_t *o_prims,
              uint32_t *o_st, void *stream) {
    if (n <= 0) return 0;
    k_kd<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, k, rays, start, n, o_seg, o_t, o_u, o_nodes,
                                                             o_ropes, o_prims, o_st);
    MWT_LAUNCH_RET;
}

int launch_brute(const MeshDev &m, const double *rays, int64_t n, int32_t *o_seg, double *o_t,
                 double *o_u, void *stream) {
    if (n <= 0) return 0;
    k_brute<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(m, rays, n, o_seg, o_t, o_u);
    MWT_LAUNCH_RET;
}

// ---------------------------------------------------------------------------
// L2 read probe ("streaming 128-bit loads over an 8-32 MB
// buffer, across all SMs"): the roof the bench divides the walk's algorithmic
// bytes by, measured in the same process as the walk.

__global__ void __launch_bounds__(512) k_l2_stream(const uint4 *__restrict__ p, size_t n, int passes,
                                                   unsigned *sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(p + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *sink = acc;  // keeps the loads
}

int probe_l2_read(size_t bytes, int passes, float *ms) {
    uint4 *p = nullptr;
    unsigned *sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&sink, 4);
    if (e == cudaSuccess) e = cudaMemset(p, 1, bytes);
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    if (e == cudaSuccess) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t n = bytes / 16;
        k_l2_stream<<<sms * 4, 512>>>(p, n, 2, sink);  // warm: the buffer into L2
        cudaEventRecord(a);
        k_l2_stream<<<sms * 4, 512>>>(p, n, passes, sink);
        cudaEventRecord(b);
        e = cudaEventSynchronize(b);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaEventElapsedTime(ms, a, b);
    }
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    if (sink) cudaFree(sink);
    if (p) cudaFree(p);
    return (int)e;
}

}  // namespace mwt
