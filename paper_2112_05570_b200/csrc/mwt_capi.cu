// extern "C" ABI of libmwt.so (declared in include/mwt.h).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mwt_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

// a generator mode word of include/mwt.h: base mode, group_log2 <= 40, cell_bits <= 16
bool mode_ok(int mode) {
    const unsigned w = (unsigned)mode;
    const unsigned base = w & 0xFFu, gs = (w >> 8) & 0xFFu, c = (w >> 16) & 0xFFu;
    return (w >> 24) == 0u && (base == MWT_RAYS_BOX_ENTRY || base == MWT_RAYS_INTERIOR) && gs <= 40u &&
           c <= 16u;
}

int cuda_fail(cudaError_t e, const char *where) {
    g_err = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return MWT_E_CUDA;
}

#define CK(expr)                                                \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);     \
    } while (0)

// restores the caller's current device on scope exit
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && (prev == dev || cudaSetDevice(dev) == cudaSuccess))
            ok = true;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// one device allocation, carved into 256-B aligned pieces
struct Arena {
    char *base = nullptr;
    size_t size = 0, used = 0;
    static size_t align(size_t n) { return (n + 255) & ~size_t(255); }
};

template <typename T>
T *carve(Arena &a, size_t count) {
    T *p = reinterpret_cast<T *>(a.base + a.used);
    a.used += Arena::align(count * sizeof(T));
    return p;
}

}  // namespace

constexpr int kHostStreams = 8;
constexpr int64_t kHostChunk = 1 << 19;  // rays per pipelined chunk of mwt_trace_host

struct mwt_mesh {
    int device = 0;
    cudaStream_t hstream[kHostStreams] = {nullptr, nullptr, nullptr};
    mwt::MeshDev dev{};
    mwt_mesh_info info{};
    void *blob = nullptr;
    // scratch for the host-buffer entry point
    std::mutex mu;
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    long long *hist_scratch = nullptr;  // the sharded entry point's per-device histogram (under mu)
    cudaStream_t stream = nullptr;
};

struct mwt_bvh {
    const mwt_mesh *mesh = nullptr;
    mwt::BvhDev dev{};
    void *blob = nullptr;
};

struct mwt_kd {
    const mwt_mesh *mesh = nullptr;
    mwt::KdDev dev{};
    void *blob = nullptr;
};

extern "C" {

int mwt_abi_version(void) { return MWT_ABI_VERSION; }

int mwt_set_tuning(int refill_below, int min_blocks_per_sm, int variant) {
    mwt::set_tuning(refill_below, min_blocks_per_sm, variant);
    return MWT_OK;
}

const char *mwt_last_error(void) { return g_err.c_str(); }

#ifndef MWT_BUILD_ID
#define MWT_BUILD_ID "unknown"
#endif
const char *mwt_build_id(void) { return MWT_BUILD_ID; }

int mwt_probe_l2_read(int device, int64_t bytes, int passes, double *gbs_out) {
    if (!gbs_out || bytes < (1 << 20) || bytes > (int64_t(1) << 30) || passes < 1 || passes > 100000)
        return fail(MWT_E_INVALID, "probe_l2_read: bad argument");
    DeviceGuard g(device);
    if (!g.ok) return fail(MWT_E_INVALID, "probe_l2_read: bad device");
    float ms = 0.f;
    int rc = mwt::probe_l2_read((size_t)bytes, passes, &ms);
    if (rc) return cuda_fail((cudaError_t)rc, "probe_l2_read");
    *gbs_out = (double)bytes * passes / (ms * 1e-3) / 1e9;
    return MWT_OK;
}

int mwt_device_count(int *count) {
    if (!count) return fail(MWT_E_INVALID, "device_count: NULL");
    CK(cudaGetDeviceCount(count));
    return MWT_OK;
}

int mwt_mesh_create(const double *vx, const double *vy, int32_t nverts, const int32_t *tri_v,
                    const int32_t *tri_nbr, const int32_t *tri_flag, int32_t ntris,
                    const double *seg_xy, const uint8_t *seg_kind, int32_t nsegs, int device,
                    mwt_mesh **out) {
    if (!out) return fail(MWT_E_INVALID, "mesh_create: out is NULL");
    *out = nullptr;
    mwt::HostPacked P;
    std::string err;
    int rc = mwt::pack_mesh(vx, vy, nverts, tri_v, tri_nbr, tri_flag, ntris, seg_xy, seg_kind,
                            nsegs, &P, &err);
    if (rc != MWT_OK) return fail(rc, err);
    DeviceGuard g(device);
    if (!g.ok) return fail(MWT_E_CUDA, "mesh_create: cannot select device " + std::to_string(device));
    const size_t nt = P.nt > 0 ? P.nt : 1, ns = P.ns > 0 ? P.ns : 1;
    size_t bytes = Arena::align(nt * 16) + Arena::align(nt * 48) + Arena::align(nt * 16) +
                   Arena::align(nt * 96) +
                   Arena::align(ns * 32) + Arena::align(ns) + Arena::align(ns * 2 * 8) +
                   Arena::align(P.ep_ids.size() * 4) + Arena::align(P.anchor.size() * 4) +
                   Arena::align(P.bu.size() * 8) + Arena::align(P.bpq.size() * 8) +
                   Arena::align(P.bword.size() * 4) + Arena::align(P.bbucket.size() * 4) +
                   Arena::align(P.crec.size() * 4) + Arena::align(P.ctri.size() * 4) +
                   Arena::align((P.bu.size() + P.bpq.size()) * 8 + P.bword.size() * 4 + P.bbucket.size() * 4 + 64) +
                   Arena::align(P.vxy.size() * 8);
    Arena a;
    CK(cudaMalloc(&a.base, bytes));
    a.size = bytes;
    mwt_mesh *m = new mwt_mesh();
    m->device = device;
    m->blob = a.base;
    int4 *link = carve<int4>(a, nt);
    double2 *cxy = carve<double2>(a, 3 * nt);
    int4 *step = carve<int4>(a, 6 * nt);
    int4 *lnbr = carve<int4>(a, nt);
    double4 *seg = carve<double4>(a, ns);
    uint8_t *kind = carve<uint8_t>(a, ns);
    int2 *epr = carve<int2>(a, 2 * ns);
    int32_t *epi = carve<int32_t>(a, P.ep_ids.size());
    int32_t *anc = carve<int32_t>(a, P.anchor.size());
    double *bu = carve<double>(a, P.bu.size());
    double *bpq = carve<double>(a, P.bpq.size());
    int32_t *bword = carve<int32_t>(a, P.bword.size());
    int32_t *bbucket = carve<int32_t>(a, P.bbucket.size());
    uint32_t *crec = carve<uint32_t>(a, P.crec.size());
    uint32_t *ctri = carve<uint32_t>(a, P.ctri.size());
    double *vxy = carve<double>(a, P.vxy.size());
    // boundary blob: bu | bpq | bword | bbucket, each 16-B aligned
    auto a16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
    const size_t bo_bpq = a16(P.bu.size() * 8), bo_bword = bo_bpq + a16(P.bpq.size() * 8),
                 bo_bbucket = bo_bword + a16(P.bword.size() * 4),
                 bblob_bytes = bo_bbucket + a16(P.bbucket.size() * 4);
    std::vector<unsigned char> bblob_host(bblob_bytes, 0);
    std::memcpy(bblob_host.data(), P.bu.data(), P.bu.size() * 8);
    std::memcpy(bblob_host.data() + bo_bpq, P.bpq.data(), P.bpq.size() * 8);
    std::memcpy(bblob_host.data() + bo_bword, P.bword.data(), P.bword.size() * 4);
    std::memcpy(bblob_host.data() + bo_bbucket, P.bbucket.data(), P.bbucket.size() * 4);
    unsigned char *bblob = carve<unsigned char>(a, bblob_bytes);
    cudaError_t e = cudaSuccess;
    auto up = [&](void *dst, const void *src, size_t n) {
        if (e == cudaSuccess && n) e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    };
    up(link, P.link.data(), (size_t)P.nt * 16);
    up(cxy, P.cxy.data(), (size_t)P.nt * 48);
    up(step, P.step.data(), (size_t)P.nt * 96);
    up(lnbr, P.lnbr.data(), (size_t)P.nt * 16);
    up(seg, P.seg.data(), (size_t)P.ns * 32);
    up(kind, P.segkind.data(), (size_t)P.ns);
    up(epr, P.ep_range.data(), (size_t)P.ns * 16);
    up(epi, P.ep_ids.data(), P.ep_ids.size() * 4);
    up(anc, P.anchor.data(), P.anchor.size() * 4);
    up(bu, P.bu.data(), P.bu.size() * 8);
    up(bpq, P.bpq.data(), P.bpq.size() * 8);
    up(bword, P.bword.data(), P.bword.size() * 4);
    up(bbucket, P.bbucket.data(), P.bbucket.size() * 4);
    up(crec, P.crec.data(), P.crec.size() * 4);
    up(ctri, P.ctri.data(), P.ctri.size() * 4);
    up(vxy, P.vxy.data(), P.vxy.size() * 8);
    up(bblob, bblob_host.data(), bblob_bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        cudaFree(a.base);
        delete m;
        return cuda_fail(e, "mesh_create: upload");
    }
    m->dev = mwt::MeshDev{P.nt, P.ns, P.res, P.flood_filter, link, cxy, step, lnbr, seg, kind, epr, epi, anc,
                         P.res > 0 ? 1.0 / P.res : 0.0};
    m->dev.nbsides = P.nbsides;
    m->dev.unit_sides = P.unit_sides;
    m->dev.coord_small = P.coord_small;
    for (int k = 0; k < P.nbsides; k++) {
        const auto &S = P.sides[k];
        m->dev.bs[k] = mwt::MeshDev::BSide{S.axis, S.off, S.cnt, S.boff, S.nb, S.c, S.lo, S.hi, S.scale};
    }
    m->dev.bu = reinterpret_cast<const double2 *>(bu);
    m->dev.bpq = reinterpret_cast<const double4 *>(bpq);
    m->dev.bword = bword;
    m->dev.bbucket = bbucket;
    m->dev.bblob = reinterpret_cast<const uint4 *>(bblob);
    m->dev.bblob_bytes = (int32_t)bblob_bytes;
    m->dev.bo_bpq = (int32_t)bo_bpq;
    m->dev.bo_bword = (int32_t)bo_bword;
    m->dev.bo_bbucket = (int32_t)bo_bbucket;
    m->dev.gseg_staged = (int64_t)bblob_bytes + 32LL * P.ns <= mwt::kSmemWalkMax;
    if (!P.crec.empty()) {
        m->dev.crec = reinterpret_cast<const uint2 *>(crec);
        m->dev.vxy = reinterpret_cast<const double2 *>(vxy);
        m->dev.crec_bytes = (int32_t)(P.crec.size() * 4);
        const int64_t sm = (int64_t)m->dev.crec_bytes + 16LL * P.nv;
        m->dev.smem_bytes = sm + (int64_t)bblob_bytes <= mwt::kSmemWalkMax ? (int32_t)sm : 0;
        m->dev.seg_staged = m->dev.smem_bytes > 0 &&
                            sm + (int64_t)bblob_bytes + 32LL * P.ns <= mwt::kSmemWalkMax;
        m->dev.ctri = reinterpret_cast<const uint4 *>(ctri);
        const int64_t tm = 16LL * P.nt + 16LL * P.nv;
        m->dev.tri_smem_bytes = tm + (int64_t)bblob_bytes <= mwt::kSmemWalkMax ? (int32_t)tm : 0;
        m->dev.tri_seg_staged = m->dev.tri_smem_bytes > 0 &&
                                tm + (int64_t)bblob_bytes + 32LL * P.ns <= mwt::kSmemWalkMax;
    }
    m->info.num_vertices = P.nv;
    m->info.num_triangles = P.nt;
    m->info.num_segments = P.ns;
    m->info.anchor_res = P.res;
    m->info.anchors_not_strict = P.anchors_not_strict;
    m->info.device = device;
    m->info.device_bytes = (int64_t)bytes;
    m->info.walk_record_bytes = 32;
    m->info.walk_smem_bytes = m->dev.smem_bytes ? m->dev.smem_bytes : m->dev.tri_smem_bytes;
    *out = m;
    return MWT_OK;
}

int mwt_pack_dry_run(const double *vx, const double *vy, int32_t nverts, const int32_t *tri_v,
                     const int32_t *tri_nbr, const int32_t *tri_flag, int32_t ntris,
                     const double *seg_xy, const uint8_t *seg_kind, int32_t nsegs,
                     int32_t *out_link, int32_t *out_lnbr, int32_t *out_res, int32_t *out_anchor) {
    mwt::HostPacked P;
    std::string err;
    int rc = mwt::pack_mesh(vx, vy, nverts, tri_v, tri_nbr, tri_flag, ntris, seg_xy, seg_kind,
                            nsegs, &P, &err);
    if (rc != MWT_OK) return fail(rc, err);
    if (out_link) std::memcpy(out_link, P.link.data(), P.link.size() * sizeof(int32_t));
    if (out_lnbr) std::memcpy(out_lnbr, P.lnbr.data(), P.lnbr.size() * sizeof(int32_t));
    if (out_res) *out_res = P.res;
    if (out_anchor && P.res > 0)
        std::memcpy(out_anchor, P.anchor.data(), P.anchor.size() * sizeof(int32_t));
    return MWT_OK;
}

int mwt_mesh_destroy(mwt_mesh *m) {
    if (!m) return MWT_OK;
    DeviceGuard g(m->device);
    if (m->stream) cudaStreamDestroy(m->stream);
    for (int k = 0; k < kHostStreams; k++)
        if (m->hstream[k]) cudaStreamDestroy(m->hstream[k]);
    if (m->scratch) cudaFree(m->scratch);
    if (m->hist_scratch) cudaFree(m->hist_scratch);
    if (m->blob) cudaFree(m->blob);
    delete m;
    return MWT_OK;
}

int mwt_mesh_info_get(const mwt_mesh *m, mwt_mesh_info *out) {
    if (!m || !out) return fail(MWT_E_INVALID, "mesh_info: NULL");
    *out = m->info;
    return MWT_OK;
}

int mwt_mesh_anchors(const mwt_mesh *m, int32_t *out_host) {
    if (!m || !out_host) return fail(MWT_E_INVALID, "mesh_anchors: NULL");
    DeviceGuard g(m->device);
    if (m->dev.res > 0)
        CK(cudaMemcpy(out_host, m->dev.anchor, sizeof(int32_t) * m->dev.res * m->dev.res,
                      cudaMemcpyDeviceToHost));
    return MWT_OK;
}

int mwt_raygen_dev(int mode, const double *box, uint64_t seed, uint64_t first, int64_t n,
                   double *rays_out, void *stream) {
    if (!box || (n > 0 && !rays_out) || n < 0 || !mode_ok(mode))
        return fail(MWT_E_INVALID, "raygen: bad argument");
    int rc = mwt::launch_raygen(mode, box, seed, first, n, rays_out, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "raygen launch");
    return MWT_OK;
}

int mwt_locate_brute_dev(const mwt_mesh *m, const double *pts, int64_t n, int32_t *out_tid,
                         uint32_t *out_status, void *stream) {
    if (!m || n < 0 || (n > 0 && !pts)) return fail(MWT_E_INVALID, "locate_brute: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "locate_brute: mesh has no triangles");
    DeviceGuard g(m->device);
    int rc = mwt::launch_locate(m->dev, pts, n, out_tid, out_status, stream, true);
    if (rc) return cuda_fail((cudaError_t)rc, "locate_brute launch");
    return MWT_OK;
}

int mwt_locate_dev(const mwt_mesh *m, const double *pts, int64_t n, int32_t *out_tid,
                   uint32_t *out_status, void *stream) {
    if (!m || n < 0 || (n > 0 && !pts)) return fail(MWT_E_INVALID, "locate: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "locate: mesh has no triangles");
    DeviceGuard g(m->device);
    int rc = mwt::launch_locate(m->dev, pts, n, out_tid, out_status, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "locate launch");
    return MWT_OK;
}

int mwt_trace_dev(const mwt_mesh *m, const double *rays, const int32_t *start, int64_t n,
                  int32_t *out_start, int32_t *out_seg, double *out_t, double *out_u,
                  int32_t *out_steps, uint32_t *out_status, void *stream) {
    if (!m || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "trace: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "trace: mesh has no triangles");
    DeviceGuard g(m->device);
    int rc = mwt::launch_trace(m->dev, rays, start, n, out_start, out_seg, out_t, out_u, out_steps,
                               out_status, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "trace launch");
    return MWT_OK;
}

int mwt_trace_chain_dev(const mwt_mesh *m, const double *rays, const int32_t *start, int64_t n,
                        int32_t *out_end, int32_t *out_seg, double *out_t, double *out_u,
                        int32_t *out_steps, uint32_t *out_status, void *stream) {
    if (!m || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "trace_chain: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "trace_chain: mesh has no triangles");
    DeviceGuard g(m->device);
    int rc = mwt::launch_trace(m->dev, rays, start, n, nullptr, out_seg, out_t, out_u, out_steps,
                               out_status, stream, out_end);
    if (rc) return cuda_fail((cudaError_t)rc, "trace_chain launch");
    return MWT_OK;
}

int mwt_trace_host(const mwt_mesh *cm, const double *rays, const int32_t *start, int64_t n,
                   int32_t *out_start, int32_t *out_seg, double *out_t, double *out_u,
                   int32_t *out_steps, uint32_t *out_status) {
    mwt_mesh *m = const_cast<mwt_mesh *>(cm);
    if (!m || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "trace_host: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "trace_host: mesh has no triangles");
    if (n == 0) return MWT_OK;
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard g(m->device);
    // Chunked pipeline over kHostStreams streams: chunk k's H2D copy, trace and
    // D2H copies are ordered on stream k % kHostStreams, so host->device and
    // device->host copies of different chunks overlap each other (separate copy
    // engines) and the kernels.  With pinned host buffers the call is bounded by
    // the larger copy direction.
    const int64_t chunk = n < kHostChunk ? n : kHostChunk;
    const size_t slot = Arena::align((size_t)chunk * 32) + 7 * Arena::align((size_t)chunk * 8);
    const size_t need = kHostStreams * slot;
    if (need > m->scratch_bytes) {
        if (m->scratch) cudaFree(m->scratch);
        m->scratch = nullptr;
        m->scratch_bytes = 0;
        CK(cudaMalloc(&m->scratch, need));
        m->scratch_bytes = need;
    }
    for (int k = 0; k < kHostStreams; k++)
        if (!m->hstream[k]) CK(cudaStreamCreateWithFlags(&m->hstream[k], cudaStreamNonBlocking));
    // on an error, wait for the chunks already queued: they read and write the
    // caller's host buffers, which must not be in use after we return
    auto drain = [&](cudaError_t e, const char *what) {
        for (int k = 0; k < kHostStreams; k++)
            if (m->hstream[k]) (void)cudaStreamSynchronize(m->hstream[k]);
        return cuda_fail(e, what);
    };
#define MWT_CKQ(expr)                                  \
    do {                                               \
        cudaError_t _e = (expr);                       \
        if (_e != cudaSuccess) return drain(_e, #expr); \
    } while (0)
    const int64_t nchunks = (n + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks; c++) {
        const int k = (int)(c % kHostStreams);
        const int64_t off = c * chunk, cnt = (n - off) < chunk ? (n - off) : chunk;
        Arena a;
        a.base = (char *)m->scratch + k * slot;
        a.size = slot;
        double *d_rays = carve<double>(a, 4 * (size_t)chunk);
        int32_t *d_start = carve<int32_t>(a, chunk);
        int32_t *d_ostart = carve<int32_t>(a, chunk);
        int32_t *d_seg = carve<int32_t>(a, chunk);
        double *d_t = carve<double>(a, chunk);
        double *d_u = carve<double>(a, chunk);
        int32_t *d_steps = carve<int32_t>(a, chunk);
        uint32_t *d_st = carve<uint32_t>(a, chunk);
        cudaStream_t s = m->hstream[k];
        MWT_CKQ(cudaMemcpyAsync(d_rays, rays + 4 * off, 32 * (size_t)cnt, cudaMemcpyHostToDevice, s));
        if (start) MWT_CKQ(cudaMemcpyAsync(d_start, start + off, 4 * (size_t)cnt, cudaMemcpyHostToDevice, s));
        int rc = mwt::launch_trace(m->dev, d_rays, start ? d_start : nullptr, cnt,
                                   out_start ? d_ostart : nullptr, out_seg ? d_seg : nullptr,
                                   out_t ? d_t : nullptr, out_u ? d_u : nullptr,
                                   out_steps ? d_steps : nullptr, out_status ? d_st : nullptr, s);
        if (rc) return drain((cudaError_t)rc, "trace_host launch");
        if (out_start) MWT_CKQ(cudaMemcpyAsync(out_start + off, d_ostart, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
        if (out_seg) MWT_CKQ(cudaMemcpyAsync(out_seg + off, d_seg, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
        if (out_t) MWT_CKQ(cudaMemcpyAsync(out_t + off, d_t, 8 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
        if (out_u) MWT_CKQ(cudaMemcpyAsync(out_u + off, d_u, 8 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
        if (out_steps) MWT_CKQ(cudaMemcpyAsync(out_steps + off, d_steps, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
        if (out_status) MWT_CKQ(cudaMemcpyAsync(out_status + off, d_st, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
    }
#undef MWT_CKQ
    for (int k = 0; k < kHostStreams; k++) CK(cudaStreamSynchronize(m->hstream[k]));
    return MWT_OK;
}

int mwt_trace_generated_dev(const mwt_mesh *m, int mode, const double *box, uint64_t seed,
                            uint64_t first, int64_t n, int32_t *out_seg, double *out_t,
                            int32_t *out_steps, int64_t *hist, void *stream) {
    if (!m || !box || n < 0 || !mode_ok(mode))
        return fail(MWT_E_INVALID, "trace_generated: bad argument");
    if (m->dev.nt == 0) return fail(MWT_E_INVALID, "trace_generated: mesh has no triangles");
    DeviceGuard g(m->device);
    int rc = mwt::launch_trace_generated(m->dev, mode, box, seed, first, n, out_seg, out_t,
                                         out_steps, reinterpret_cast<long long *>(hist), stream);
    if (rc) return cuda_fail((cudaError_t)rc, "trace_generated launch");
    return MWT_OK;
}

int mwt_histogram_dev(const int32_t *seg, const int32_t *steps, const uint32_t *status, int64_t n,
                      int64_t *hist, void *stream) {
    if (n < 0 || (n > 0 && (!seg || !steps || !hist))) return fail(MWT_E_INVALID, "histogram: bad argument");
    int rc = mwt::launch_histogram(seg, steps, status, n, reinterpret_cast<long long *>(hist), stream);
    if (rc) return cuda_fail((cudaError_t)rc, "histogram launch");
    return MWT_OK;
}

int mwt_bvh_create(const mwt_mesh *mesh, int32_t nnodes, const double *box, const int32_t *left,
                   const int32_t *right, const int32_t *prim_off, const int32_t *prim_cnt,
                   int32_t nprims, const int32_t *prims, mwt_bvh **out) {
    if (!mesh || !out || nnodes <= 0 || !box || !left || !right || !prim_off || !prim_cnt ||
        nprims < 0 || (nprims > 0 && !prims))
        return fail(MWT_E_INVALID, "bvh_create: bad argument");
    *out = nullptr;
    for (int k = 0; k < nnodes; k++) {
        bool leaf = left[k] < 0;
        if ((leaf && (prim_off[k] < 0 || prim_cnt[k] < 0 || prim_off[k] + prim_cnt[k] > nprims)) ||
            (!leaf && (left[k] >= nnodes || right[k] < 0 || right[k] >= nnodes)))
            return fail(MWT_E_INVALID, "bvh_create: node " + std::to_string(k) + " out of range");
    }
    for (int k = 0; k < nprims; k++)
        if (prims[k] < 0 || prims[k] >= mesh->dev.ns)
            return fail(MWT_E_INVALID, "bvh_create: primitive id out of range");
    DeviceGuard g(mesh->device);
    // child refs and boxes in the parent's slots (mwt_internal.h BvhDev)
    auto ref = [&](int c) { return left[c] < 0 ? ~c : c; };
    const size_t nn = nnodes;
    std::vector<double> cbox(8 * nn, 0.0);
    std::vector<int32_t> cref(2 * nn, 0), pr(2 * nn, 0);
    for (size_t k = 0; k < nn; k++) {
        if (left[k] >= 0) {
            const int c[2] = {left[k], right[k]};
            for (int s = 0; s < 2; s++) {
                cref[2 * k + s] = ref(c[s]);
                for (int q = 0; q < 4; q++) cbox[8 * k + 4 * s + q] = box[4 * (size_t)c[s] + q];
            }
        } else {
            pr[2 * k] = prim_off[k];
            pr[2 * k + 1] = prim_cnt[k];
        }
    }
    size_t np = nprims > 0 ? nprims : 1;
    size_t bytes = Arena::align(64 * nn) + 2 * Arena::align(8 * nn) + Arena::align(4 * np);
    Arena a;
    CK(cudaMalloc(&a.base, bytes));
    mwt_bvh *b = new mwt_bvh();
    b->mesh = mesh;
    b->blob = a.base;
    double4 *dbox = carve<double4>(a, 2 * nn);
    int2 *dref = carve<int2>(a, nn);
    int2 *dpr = carve<int2>(a, nn);
    int32_t *dpm = carve<int32_t>(a, np);
    cudaError_t e = cudaMemcpy(dbox, cbox.data(), 64 * nn, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dref, cref.data(), 8 * nn, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dpr, pr.data(), 8 * nn, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nprims > 0) e = cudaMemcpy(dpm, prims, 4 * (size_t)nprims, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(a.base);
        delete b;
        return cuda_fail(e, "bvh_create: upload");
    }
    mwt::BvhDev d{};
    d.nnodes = nnodes;
    d.root = make_double4(box[0], box[1], box[2], box[3]);
    d.root_ref = ref(0);
    d.cbox = dbox;
    d.cref = dref;
    d.prange = dpr;
    d.prims = dpm;
    d.blob = a.base;
    d.blob_bytes = (int32_t)bytes;
    d.o_cref = (int32_t)((char *)dref - (char *)a.base);
    d.o_prange = (int32_t)((char *)dpr - (char *)a.base);
    d.o_prims = (int32_t)((char *)dpm - (char *)a.base);
    b->dev = d;
    *out = b;
    return MWT_OK;
}

int mwt_bvh_destroy(mwt_bvh *b) {
    if (!b) return MWT_OK;
    DeviceGuard g(b->mesh->device);
    cudaFree(b->blob);
    delete b;
    return MWT_OK;
}

int mwt_bvh_trace_dev(const mwt_bvh *b, const double *rays, int64_t n, int32_t *out_seg,
                      double *out_t, double *out_u, int32_t *out_node_tests,
                      int32_t *out_prim_tests, uint32_t *out_status, void *stream) {
    if (!b || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "bvh_trace: bad argument");
    DeviceGuard g(b->mesh->device);
    int rc = mwt::launch_bvh(b->mesh->dev, b->dev, rays, n, out_seg, out_t, out_u, out_node_tests,
                             out_prim_tests, out_status, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "bvh_trace launch");
    return MWT_OK;
}

int mwt_kd_create(const mwt_mesh *mesh, int32_t nnodes, int32_t num_leaves, const int32_t *axis,
                  const double *pos, const int32_t *left, const int32_t *right, const double *box,
                  const int32_t *ropes, const int32_t *rope_cost, const int32_t *prim_off,
                  const int32_t *prim_cnt, int32_t nprims, const int32_t *prims, mwt_kd **out) {
    if (!mesh || !out || nnodes <= 0 || num_leaves <= 0 || !axis || !pos || !left || !right ||
        !box || !ropes || !rope_cost || !prim_off || !prim_cnt || nprims < 0 || (nprims > 0 && !prims))
        return fail(MWT_E_INVALID, "kd_create: bad argument");
    *out = nullptr;
    for (int k = 0; k < nnodes; k++) {
        if (axis[k] >= 0) {
            if (axis[k] > 1 || left[k] < 0 || left[k] >= nnodes || right[k] < 0 || right[k] >= nnodes)
                return fail(MWT_E_INVALID, "kd_create: node " + std::to_string(k) + " out of range");
        } else {
            if (prim_off[k] < 0 || prim_cnt[k] < 0 || prim_off[k] + prim_cnt[k] > nprims)
                return fail(MWT_E_INVALID, "kd_create: leaf " + std::to_string(k) + " prims out of range");
            for (int s = 0; s < 4; s++)
                if (ropes[4 * k + s] < -1 || ropes[4 * k + s] >= nnodes)
                    return fail(MWT_E_INVALID, "kd_create: rope out of range");
        }
    }
    for (int k = 0; k < nprims; k++)
        if (prims[k] < 0 || prims[k] >= mesh->dev.ns)
            return fail(MWT_E_INVALID, "kd_create: primitive id out of range");
    for (int k = 0; k < nnodes; k++)
        if (axis[k] < 0)
            for (int s = 0; s < 4; s++)
                if (rope_cost[4 * k + s] < 0 || rope_cost[4 * k + s] > 255)
                    return fail(MWT_E_INVALID, "kd_create: rope cost out of range");
    DeviceGuard g(mesh->device);
    // mwt_internal.h KdDev: 16-B node words, one 64-B record per leaf
    const size_t nn = nnodes;
    std::vector<int4> node(nn);
    std::vector<mwt::KdLeaf> leaf;
    for (size_t k = 0; k < nn; k++) {
        if (axis[k] >= 0) {
            unsigned long long pb;
            std::memcpy(&pb, pos + k, 8);
            node[k] = make_int4((int)(uint32_t)pb, (int)(uint32_t)(pb >> 32), left[k],
                                (int)((uint32_t)right[k] | ((uint32_t)axis[k] << 31)));
        } else {
            node[k] = make_int4(0, 0, -1, (int)leaf.size());
            uint32_t cost = 0;
            for (int s = 0; s < 4; s++) cost |= (uint32_t)rope_cost[4 * k + s] << (8 * s);
            mwt::KdLeaf L;
            L.box = make_double4(box[4 * k], box[4 * k + 1], box[4 * k + 2], box[4 * k + 3]);
            L.ropes = make_int4(ropes[4 * k], ropes[4 * k + 1], ropes[4 * k + 2], ropes[4 * k + 3]);
            L.meta = make_int4(prim_off[k], prim_cnt[k], (int)cost, 0);
            leaf.push_back(L);
        }
    }
    const size_t nl = leaf.size() > 0 ? leaf.size() : 1;
    size_t np = nprims > 0 ? nprims : 1;
    size_t bytes = Arena::align(16 * nn) + Arena::align(sizeof(mwt::KdLeaf) * nl) + Arena::align(4 * np);
    Arena a;
    CK(cudaMalloc(&a.base, bytes));
    mwt_kd *k = new mwt_kd();
    k->mesh = mesh;
    k->blob = a.base;
    int4 *dnode = carve<int4>(a, nn);
    mwt::KdLeaf *dleaf = carve<mwt::KdLeaf>(a, nl);
    int32_t *dpm = carve<int32_t>(a, np);
    cudaError_t e = cudaSuccess;
    auto up = [&](void *dst, const void *src, size_t n) {
        if (e == cudaSuccess && n) e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    };
    up(dnode, node.data(), 16 * nn);
    up(dleaf, leaf.data(), sizeof(mwt::KdLeaf) * leaf.size());
    up(dpm, prims, 4 * (size_t)nprims);
    if (e != cudaSuccess) {
        cudaFree(a.base);
        delete k;
        return cuda_fail(e, "kd_create: upload");
    }
    k->dev = mwt::KdDev{nnodes, num_leaves, dnode, dleaf, dpm};  // guard: 4 * len(kd._leaves) + 16
    *out = k;
    return MWT_OK;
}

int mwt_kd_destroy(mwt_kd *k) {
    if (!k) return MWT_OK;
    DeviceGuard g(k->mesh->device);
    cudaFree(k->blob);
    delete k;
    return MWT_OK;
}

int mwt_kd_trace_dev(const mwt_kd *k, const double *rays, const int32_t *start_leaf, int64_t n,
                     int32_t *out_seg, double *out_t, double *out_u, int32_t *out_nodes,
                     int32_t *out_rope_steps, int32_t *out_prim_tests, uint32_t *out_status,
                     void *stream) {
    if (!k || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "kd_trace: bad argument");
    DeviceGuard g(k->mesh->device);
    int rc = mwt::launch_kd(k->mesh->dev, k->dev, rays, start_leaf, n, out_seg, out_t, out_u, out_nodes,
                            out_rope_steps, out_prim_tests, out_status, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "kd_trace launch");
    return MWT_OK;
}

int mwt_brute_force_dev(const mwt_mesh *m, const double *rays, int64_t n, int32_t *out_seg,
                        double *out_t, double *out_u, void *stream) {
    if (!m || n < 0 || (n > 0 && !rays)) return fail(MWT_E_INVALID, "brute_force: bad argument");
    DeviceGuard g(m->device);
    int rc = mwt::launch_brute(m->dev, rays, n, out_seg, out_t, out_u, stream);
    if (rc) return cuda_fail((cudaError_t)rc, "brute_force launch");
    return MWT_OK;
}

// ---------------------------------------------------------------------------
// One process, several GPUs (SURVEY.md §8b `mwt_run_sharded`): rays shard by
// global index into contiguous ranges, one host thread per device drives its
// own stream, and the per-device histograms are summed on the host -- the
// single-process counterpart of the bench's one-process-per-GPU NCCL path.

namespace {
struct ShardErr {
    int rc = MWT_OK;
    std::string msg;
};

// contiguous near-equal ranges [floor(k*n/d), floor((k+1)*n/d))
inline int64_t shard_lo(int64_t n, int ndev, int k) { return (int64_t)((__int128)n * k / ndev); }

int shard_args_ok(const mwt_mesh *const *meshes, int ndev) {
    if (!meshes || ndev <= 0 || ndev > 64) return 0;
    for (int k = 0; k < ndev; k++)
        if (!meshes[k] || meshes[k]->dev.nt == 0) return 0;
    return 1;
}
}  // namespace

int mwt_trace_generated_sharded(const mwt_mesh *const *meshes, int ndev, int mode, const double *box,
                                uint64_t seed, uint64_t first, int64_t n, int64_t *hist_out) {
    if (!shard_args_ok(meshes, ndev) || !box || n < 0 || !hist_out ||
        !mode_ok(mode))
        return fail(MWT_E_INVALID, "trace_generated_sharded: bad argument");
    std::vector<std::vector<int64_t>> part(ndev, std::vector<int64_t>(MWT_HIST_LEN, 0));
    std::vector<ShardErr> err(ndev);
    std::vector<std::thread> th;
    for (int k = 0; k < ndev; k++)
        th.emplace_back([&, k]() {
            mwt_mesh *m = const_cast<mwt_mesh *>(meshes[k]);
            const int64_t lo = shard_lo(n, ndev, k), cnt = shard_lo(n, ndev, k + 1) - lo;
            std::lock_guard<std::mutex> lk(m->mu);
            DeviceGuard g(m->device);
            cudaError_t e = g.ok ? cudaSuccess : cudaErrorInvalidDevice;
            // allocated once per mesh handle, kept for later calls
            if (e == cudaSuccess && !m->hist_scratch)
                e = cudaMalloc(&m->hist_scratch, sizeof(long long) * MWT_HIST_LEN);
            long long *dh = m->hist_scratch;
            if (e == cudaSuccess) e = cudaMemsetAsync(dh, 0, sizeof(long long) * MWT_HIST_LEN, m->stream);
            if (e == cudaSuccess && cnt > 0)
                e = (cudaError_t)mwt::launch_trace_generated(m->dev, mode, box, seed, first + (uint64_t)lo,
                                                             cnt, nullptr, nullptr, nullptr, dh, m->stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(part[k].data(), dh, sizeof(long long) * MWT_HIST_LEN,
                                    cudaMemcpyDeviceToHost, m->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
            if (e != cudaSuccess) {
                err[k].rc = MWT_E_CUDA;
                err[k].msg = std::string("device ") + std::to_string(m->device) + ": " + cudaGetErrorName(e);
            }
        });
    for (auto &t : th) t.join();
    for (int k = 0; k < ndev; k++)
        if (err[k].rc) return fail(err[k].rc, "trace_generated_sharded: " + err[k].msg);
    for (int b = 0; b < MWT_HIST_LEN; b++) {
        int64_t sum = 0;
        for (int k = 0; k < ndev; k++) sum += part[k][b];
        hist_out[b] = sum;
    }
    return MWT_OK;
}

int mwt_trace_host_sharded(const mwt_mesh *const *meshes, int ndev, const double *rays,
                           const int32_t *start, int64_t n, int32_t *out_start, int32_t *out_seg,
                           double *out_t, double *out_u, int32_t *out_steps, uint32_t *out_status) {
    if (!shard_args_ok(meshes, ndev) || n < 0 || (n > 0 && !rays))
        return fail(MWT_E_INVALID, "trace_host_sharded: bad argument");
    std::vector<ShardErr> err(ndev);
    std::vector<std::thread> th;
    for (int k = 0; k < ndev; k++)
        th.emplace_back([&, k]() {
            const int64_t lo = shard_lo(n, ndev, k), cnt = shard_lo(n, ndev, k + 1) - lo;
            auto at = [lo](auto *p, int w) { return p ? p + lo * w : p; };
            const int rc = mwt_trace_host(meshes[k], rays + 4 * lo, at(start, 1), cnt, at(out_start, 1),
                                          at(out_seg, 1), at(out_t, 1), at(out_u, 1), at(out_steps, 1),
                                          at(out_status, 1));
            if (rc) {
                err[k].rc = rc;
                err[k].msg = g_err;  // this worker thread's message
            }
        });
    for (auto &t : th) t.join();
    for (int k = 0; k < ndev; k++)
        if (err[k].rc) return fail(err[k].rc, "trace_host_sharded: " + err[k].msg);
    return MWT_OK;
}

}  // extern "C"
