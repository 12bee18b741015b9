// C ABI of libfgl.so (include/fgl.h): argument validation, scene lifetime, error reporting, and
// the orchestration of the build and cast kernels on the caller's stream.
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/fgl.h"
#include <vector>

#include "fgl_internal.cuh"

using fgl::Error;

namespace fgl {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fgl

struct fgl_scene {
    int dev = 0;
    int64_t V = 0, T = 0, cap_T = 0, cap_V = 0;
    float *verts = nullptr;
    int32_t *tris = nullptr;
    unsigned int *vflag = nullptr;  // validation flag
    unsigned int *hflag = nullptr;  // pinned host copy
    fgl::BuildBuffers b;
    fgl::CastCounter *counters = nullptr;
    std::atomic<uint32_t> slot{0};
    bool built = false;
    bool points = false;  // uploaded with fgl_scene_upload_points (degenerate triangles (i, i, i))
    bool gauss = false;   // uploaded with fgl_scene_upload_gaussians (mu in verts, records in b.tri)
    float kappa = 3.0f;
    float *g_quat = nullptr, *g_scale = nullptr, *g_opac = nullptr;  // [cap_V][4], [cap_V][3], [cap_V]
    unsigned long long *vox_counts = nullptr;                         // scratch when the caller passes none
    unsigned int *vox_overflow = nullptr;
    int bits = 21, leaf_size = 4;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    size_t bytes = 0;
};

namespace {

thread_local std::string g_err;

fgl_status fail(int code, const std::string &msg) {
    g_err = msg;
    return (fgl_status)code;
}

#define FGL_API_BEGIN try {
#define FGL_API_END                                                   \
    }                                                                 \
    catch (const fgl::Error &e) {                                     \
        return fail(e.code, e.what());                                \
    }                                                                 \
    catch (const std::exception &e) {                                 \
        return fail(FGL_E_RESOURCE, e.what());                        \
    }                                                                 \
    return FGL_OK;

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        FGL_CUDA(cudaGetDevice(&prev));
        if (prev != dev) FGL_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

template <class T>
void dalloc(fgl_scene *s, T **p, size_t n) {
    if (*p) {
        cudaFree(*p);
        *p = nullptr;
    }
    if (n == 0) n = 1;
    FGL_CUDA(cudaMalloc((void **)p, n * sizeof(T)));
    s->bytes += n * sizeof(T);
}

void free_build(fgl_scene *s) {
    fgl::BuildBuffers &b = s->b;
    void *ps[] = {b.cent, b.box, b.partial, b.sync, b.keys[0], b.keys[1], b.vals[0], b.vals[1], b.ghist, b.sort_status, b.sort_tiles, b.sort_rts,
                  b.tri, b.child, b.range, b.parent, b.flags, b.leafbox, b.nodebox, b.nodes, b.nodes4, b.depth, b.agg,
                  b.cost, b.tsize, b.cost8, b.wq, b.wctr, b.gslot, b.lbvh_up};
    for (void *p : ps)
        if (p) cudaFree(p);
    b = fgl::BuildBuffers();
}

void alloc_build(fgl_scene *s, int64_t T) {
    free_build(s);
    s->bytes = 0;
    fgl::BuildBuffers &b = s->b;
    b.T = T;
    const int64_t nin = std::max<int64_t>(T - 1, 1);
    dalloc(s, &b.cent, T);
    dalloc(s, &b.box, 8);
    dalloc(s, &b.partial, fgl::kPrepBlocks * 6);
    dalloc(s, &b.sync, 4);
    FGL_CUDA(cudaMemset(b.sync, 0, 4 * sizeof(unsigned int)));
    dalloc(s, &b.keys[0], T);
    dalloc(s, &b.keys[1], T);
    dalloc(s, &b.vals[0], T);
    dalloc(s, &b.vals[1], T);
    dalloc(s, &b.ghist, 8 * 256);
    dalloc(s, &b.sort_status, (size_t)256 * fgl::sort_tile_blocks(T));
    FGL_CUDA(cudaMemset(b.sort_status, 0, sizeof(uint64_t) * 256 * fgl::sort_tile_blocks(T)));
    dalloc(s, &b.sort_tiles, 16);
    dalloc(s, &b.sort_rts, (size_t)256 * fgl::sort_tile_blocks(T));
    FGL_CUDA(cudaMemset(b.sort_tiles, 0, 16 * sizeof(uint32_t)));  // tile counters + device sort epoch
    dalloc(s, &b.tri, (size_t)fgl::kTriStride * T);  // also the Gaussian records (3 float4 each)
    dalloc(s, &b.child, nin);
    dalloc(s, &b.range, nin);
    dalloc(s, &b.parent, 2 * T);
    dalloc(s, &b.flags, nin);
    dalloc(s, &b.leafbox, 2 * T);
    dalloc(s, &b.nodebox, 2 * nin);
    dalloc(s, &b.nodes, nin);
    dalloc(s, &b.nodes4, nin);
    {
        int64_t m = T, tot = 0;
        for (int k = 0; k < 10; ++k) tot += (m = (m + 7) / 8);
        dalloc(s, &b.agg, 2 * tot);
    }
    dalloc(s, &b.depth, nin);
    dalloc(s, &b.cost, nin);
    dalloc(s, &b.tsize, nin);
    dalloc(s, &b.cost8, 8 * nin);
    dalloc(s, &b.wq, T);
    dalloc(s, &b.wctr, 4);
    dalloc(s, &b.gslot, nin);
    FGL_CUDA(cudaMemset(b.gslot, 0, nin * sizeof(unsigned long long)));  // epoch 0 is never a build's
    {
        const size_t ub = fgl::lbvh_up_bytes(T);
        char *u = nullptr;
        dalloc(s, &u, ub);
        FGL_CUDA(cudaMemset(u, 0, ub));  // arrival counters start at 0 and reset themselves
        b.lbvh_up = u;
    }
}

fgl::SceneView view(const fgl_scene *s) {
    // root box: the root's Eq. 7 box (T >= 2), or the single triangle's box
    const float4 *root = s->b.T >= 2 ? s->b.nodebox : s->b.leafbox;
    return fgl::SceneView{s->b.tri, s->b.nodes, s->b.nodes4, s->b.width, s->b.quantized, s->b.wctr + 3, s->vflag, root};
}

fgl::CastCounter *next_counter(const fgl_scene *s) {
    auto *ms = const_cast<fgl_scene *>(s);
    uint32_t k = ms->slot.fetch_add(1, std::memory_order_relaxed) % fgl::kCounterSlots;
    return s->counters + k;
}

void check_interval(float t_min, float t_max) {
    if (!(t_min >= 0.f) || !(t_max > t_min) || std::isnan(t_max))
        throw Error(FGL_E_USAGE, "need 0 <= t_min < t_max");
}

void check_built(const fgl_scene *s) {
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    if (!s->built) throw Error(FGL_E_USAGE, "scene is not built (call fgl_scene_build first)");
}

void check_cast(const fgl_scene *s) {  // casts need a triangle (or point) scene
    check_built(s);
    if (s->gauss) throw Error(FGL_E_USAGE, "cannot cast rays against a Gaussian scene (use fgl_voxelize)");
}

fgl::SpinParams spin_params(const fgl_spinning *p) {
    if (!p) throw Error(FGL_E_USAGE, "pattern is NULL");
    if (p->channels < 1 || p->channels > 512) throw Error(FGL_E_USAGE, "channels must be in [1, 512]");
    if (p->columns < 1) throw Error(FGL_E_USAGE, "columns must be >= 1");
    if (!p->elev_deg) throw Error(FGL_E_USAGE, "elev_deg is NULL");
    check_interval(p->t_min, p->t_max);
    bool inc = true, dec = true;
    for (int c = 0; c < p->channels; ++c) {
        if (!std::isfinite(p->elev_deg[c]) || std::fabs(p->elev_deg[c]) > 90.f)
            throw Error(FGL_E_USAGE, "elevations must be finite degrees in [-90, 90]");
        if (c) {
            inc = inc && p->elev_deg[c] >= p->elev_deg[c - 1];
            dec = dec && p->elev_deg[c] <= p->elev_deg[c - 1];
        }
    }
    if (!inc && !dec) throw Error(FGL_E_USAGE, "elevations must be monotone (S:454)");
    if (!std::isfinite(p->az0_deg)) throw Error(FGL_E_USAGE, "az0_deg must be finite");
    fgl::SpinParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.channels = p->channels, sp.columns = p->columns;
    sp.az0_deg = p->az0_deg, sp.t_min = p->t_min, sp.t_max = p->t_max;
    memcpy(sp.elev_deg, p->elev_deg, sizeof(float) * p->channels);
    return sp;
}

fgl::RosetteParams rosette_params(const fgl_rosette *p, int64_t first_frame) {
    if (!p) throw Error(FGL_E_USAGE, "pattern is NULL");
    if (p->points_per_frame < 1) throw Error(FGL_E_USAGE, "points_per_frame must be >= 1");
    if (!(p->half_fov_deg > 0.f && p->half_fov_deg <= 90.f)) throw Error(FGL_E_USAGE, "half_fov_deg must be in (0, 90]");
    if (first_frame < 0) throw Error(FGL_E_USAGE, "first_frame must be >= 0");
    check_interval(p->t_min, p->t_max);
    fgl::RosetteParams r;
    r.n = p->points_per_frame;
    r.inc1 = p->inc1, r.inc2 = p->inc2, r.phase2_0 = p->phase2_0;
    r.half_fov_deg = p->half_fov_deg, r.t_min = p->t_min, r.t_max = p->t_max;
    r.first_frame = first_frame;
    return r;
}

fgl::CastOut cast_out(float *range, int32_t *tri_id, float *hit, int32_t *nc, int32_t *tc) {
    if (!range || !tri_id) throw Error(FGL_E_USAGE, "range / tri_id output is NULL");
    fgl::CastOut o;
    memset(&o, 0, sizeof(o));
    o.range = range, o.tri_id = tri_id, o.hit_xyz = hit, o.node_counts = nc, o.tri_counts = tc;
    return o;
}

}  // namespace

extern "C" {

const char *fgl_last_error(void) { return g_err.c_str(); }
const char *fgl_version(void) { return "fgl 0.1.0 (sm_100a)"; }
int32_t fgl_abi_version(void) { return 2; }
int64_t fgl_kernel_launches(void) { return fgl::g_launches.load(std::memory_order_relaxed); }

fgl_status fgl_scene_create(int cuda_device, fgl_scene **out) {
    FGL_API_BEGIN
    if (!out) throw Error(FGL_E_USAGE, "out is NULL");
    *out = nullptr;
    int n = 0;
    FGL_CUDA(cudaGetDeviceCount(&n));
    if (cuda_device < 0 || cuda_device >= n) throw Error(FGL_E_USAGE, "no such CUDA device");
    DeviceGuard g(cuda_device);
    fgl_scene *s = new fgl_scene();
    s->dev = cuda_device;
    try {
        FGL_CUDA(cudaMalloc((void **)&s->counters, sizeof(fgl::CastCounter) * fgl::kCounterSlots));
        FGL_CUDA(cudaMemset(s->counters, 0, sizeof(fgl::CastCounter) * fgl::kCounterSlots));
        FGL_CUDA(cudaMalloc((void **)&s->vflag, sizeof(unsigned int)));
        FGL_CUDA(cudaMallocHost((void **)&s->hflag, sizeof(unsigned int)));
        FGL_CUDA(cudaEventCreate(&s->ev0));
        FGL_CUDA(cudaEventCreate(&s->ev1));
    } catch (...) {
        fgl_scene_destroy(s);
        throw;
    }
    *out = s;
    FGL_API_END
}

void fgl_scene_destroy(fgl_scene *s) {
    if (!s) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(s->dev);
    free_build(s);
    if (s->verts) cudaFree(s->verts);
    if (s->tris) cudaFree(s->tris);
    for (void *p : {(void *)s->g_quat, (void *)s->g_scale, (void *)s->g_opac, (void *)s->vox_counts,
                    (void *)s->vox_overflow})
        if (p) cudaFree(p);
    if (s->counters) cudaFree(s->counters);
    if (s->vflag) cudaFree(s->vflag);
    if (s->hflag) cudaFreeHost(s->hflag);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (prev >= 0) cudaSetDevice(prev);
    delete s;
}

fgl_status fgl_scene_upload_mesh(fgl_scene *s, const float *verts, int64_t V, const int32_t *tris, int64_t T,
                                 int ptr_kind, void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl upload (A1)");
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    const bool async = (ptr_kind & FGL_ASYNC) != 0;
    ptr_kind &= ~FGL_ASYNC;
    if (ptr_kind != FGL_HOST && ptr_kind != FGL_DEVICE) throw Error(FGL_E_USAGE, "ptr_kind must be FGL_HOST or FGL_DEVICE");
    if (T <= 0) throw Error(FGL_E_DATA, "mesh has no triangles (T = 0)");
    if (V <= 0) throw Error(FGL_E_DATA, "mesh has no vertices");
    if (!verts || !tris) throw Error(FGL_E_USAGE, "verts / tris is NULL");
    if (T > fgl::kMaxTris) throw Error(FGL_E_USAGE, "too many triangles (T must be < 2^28)");
    if (V > INT32_MAX) throw Error(FGL_E_USAGE, "too many vertices (V must fit int32)");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    s->built = false;
    if (V > s->cap_V) {
        if (s->verts) cudaFree(s->verts), s->verts = nullptr;
        FGL_CUDA(cudaMalloc((void **)&s->verts, sizeof(float) * 3 * V));
        s->cap_V = V;
    }
    if (T > s->cap_T) {
        if (s->tris) cudaFree(s->tris), s->tris = nullptr;
        FGL_CUDA(cudaMalloc((void **)&s->tris, sizeof(int32_t) * 3 * T));
        alloc_build(s, T);
        s->cap_T = T;
    }
    s->b.T = T;
    s->V = V, s->T = T;
    s->points = false;
    s->gauss = false;
    cudaMemcpyKind kind = ptr_kind == FGL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    FGL_CUDA(cudaMemcpyAsync(s->verts, verts, sizeof(float) * 3 * V, kind, st));
    FGL_CUDA(cudaMemcpyAsync(s->tris, tris, sizeof(int32_t) * 3 * T, kind, st));
    fgl::launch_validate(s->verts, V, s->tris, T, s->vflag, st);
    if (async) return FGL_OK;
    FGL_CUDA(cudaMemcpyAsync(s->hflag, s->vflag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FGL_CUDA(cudaStreamSynchronize(st));
    if (*s->hflag & 1u) throw Error(FGL_E_DATA, "triangle index out of range [0, V)");
    if (*s->hflag & 2u) throw Error(FGL_E_DATA, "non-finite vertex coordinate");
    FGL_API_END
}

fgl_status fgl_scene_upload_points(fgl_scene *s, const float *xyz, int64_t n, int ptr_kind, void *stream) {
    FGL_API_BEGIN
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    const bool async = (ptr_kind & FGL_ASYNC) != 0;
    ptr_kind &= ~FGL_ASYNC;
    if (ptr_kind != FGL_HOST && ptr_kind != FGL_DEVICE) throw Error(FGL_E_USAGE, "ptr_kind must be FGL_HOST or FGL_DEVICE");
    if (n <= 0) throw Error(FGL_E_DATA, "point cloud is empty");
    if (!xyz) throw Error(FGL_E_USAGE, "xyz is NULL");
    if (n > fgl::kMaxTris) throw Error(FGL_E_USAGE, "too many points (n must be < 2^28)");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    s->built = false;
    if (n > s->cap_V) {
        if (s->verts) cudaFree(s->verts), s->verts = nullptr;
        FGL_CUDA(cudaMalloc((void **)&s->verts, sizeof(float) * 3 * n));
        s->cap_V = n;
    }
    if (n > s->cap_T) {
        if (s->tris) cudaFree(s->tris), s->tris = nullptr;
        FGL_CUDA(cudaMalloc((void **)&s->tris, sizeof(int32_t) * 3 * n));
        alloc_build(s, n);
        s->cap_T = n;
    }
    s->b.T = n;
    s->V = n, s->T = n;
    s->points = true;
    s->gauss = false;
    FGL_CUDA(cudaMemcpyAsync(s->verts, xyz, sizeof(float) * 3 * n,
                             ptr_kind == FGL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    fgl::launch_iota3(s->tris, n, st);
    fgl::launch_validate(s->verts, n, s->tris, n, s->vflag, st);
    if (async) return FGL_OK;
    FGL_CUDA(cudaMemcpyAsync(s->hflag, s->vflag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FGL_CUDA(cudaStreamSynchronize(st));
    if (*s->hflag & 2u) throw Error(FGL_E_DATA, "non-finite point coordinate");
    FGL_API_END
}

fgl_status fgl_scene_upload_gaussians(fgl_scene *s, const float *mu, const float *quat, const float *scale,
                                      const float *opacity, int64_t n, float kappa, int ptr_kind, void *stream) {
    FGL_API_BEGIN
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    const bool async = (ptr_kind & FGL_ASYNC) != 0;
    ptr_kind &= ~FGL_ASYNC;
    if (ptr_kind != FGL_HOST && ptr_kind != FGL_DEVICE) throw Error(FGL_E_USAGE, "ptr_kind must be FGL_HOST or FGL_DEVICE");
    if (n <= 0) throw Error(FGL_E_DATA, "Gaussian cloud is empty");
    if (!mu || !quat || !scale || !opacity) throw Error(FGL_E_USAGE, "NULL parameter array");
    if (n > fgl::kMaxTris) throw Error(FGL_E_USAGE, "too many Gaussians (n must be < 2^28)");
    if (!(kappa >= 1.0f) || !std::isfinite(kappa)) throw Error(FGL_E_USAGE, "kappa must be finite and >= 1 (Eq. 4)");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    s->built = false;
    if (n > s->cap_V || !s->g_quat) {
        for (float **p : {&s->verts, &s->g_quat, &s->g_scale, &s->g_opac})
            if (*p) cudaFree(*p), *p = nullptr;
        const int64_t cap = std::max(n, s->cap_V);
        FGL_CUDA(cudaMalloc((void **)&s->verts, sizeof(float) * 3 * cap));
        FGL_CUDA(cudaMalloc((void **)&s->g_quat, sizeof(float) * 4 * cap));
        FGL_CUDA(cudaMalloc((void **)&s->g_scale, sizeof(float) * 3 * cap));
        FGL_CUDA(cudaMalloc((void **)&s->g_opac, sizeof(float) * cap));
        s->cap_V = cap;
    }
    if (n > s->cap_T) {
        if (s->tris) cudaFree(s->tris), s->tris = nullptr;
        FGL_CUDA(cudaMalloc((void **)&s->tris, sizeof(int32_t) * 3 * n));
        alloc_build(s, n);
        s->cap_T = n;
    }
    s->b.T = n;
    s->V = n, s->T = n;
    s->points = false;
    s->gauss = true;
    s->kappa = kappa;
    const cudaMemcpyKind kind = ptr_kind == FGL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    FGL_CUDA(cudaMemcpyAsync(s->verts, mu, sizeof(float) * 3 * n, kind, st));
    FGL_CUDA(cudaMemcpyAsync(s->g_quat, quat, sizeof(float) * 4 * n, kind, st));
    FGL_CUDA(cudaMemcpyAsync(s->g_scale, scale, sizeof(float) * 3 * n, kind, st));
    FGL_CUDA(cudaMemcpyAsync(s->g_opac, opacity, sizeof(float) * n, kind, st));
    FGL_CUDA(cudaMemsetAsync(s->vflag, 0, sizeof(unsigned int), st));
    fgl::launch_gauss_prep(s->verts, s->g_quat, s->g_scale, s->g_opac, n, s->b, s->vflag, st);
    if (async) return FGL_OK;
    FGL_CUDA(cudaMemcpyAsync(s->hflag, s->vflag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FGL_CUDA(cudaStreamSynchronize(st));
    if (*s->hflag & 2u)
        throw Error(FGL_E_DATA, "invalid Gaussian (non-finite mu / q, q = 0, scale <= 0 or opacity outside [0, 1])");
    FGL_API_END
}

fgl_status fgl_voxelize(const fgl_scene *s, const fgl_grid *grid, float *density, uint32_t *occupancy,
                        uint32_t *surface, uint32_t *interior, int64_t *counts, void *stream) {
    FGL_API_BEGIN
    check_built(s);
    if (!s->gauss) throw Error(FGL_E_USAGE, "fgl_voxelize needs a Gaussian scene (fgl_scene_upload_gaussians)");
    if (!grid) throw Error(FGL_E_USAGE, "grid is NULL");
    if (!occupancy) throw Error(FGL_E_USAGE, "occupancy output is NULL");
    if (!(grid->spacing > 0.f) || !std::isfinite(grid->spacing)) throw Error(FGL_E_USAGE, "spacing must be finite and > 0");
    for (int a = 0; a < 3; ++a) {
        if (!std::isfinite(grid->origin[a])) throw Error(FGL_E_USAGE, "origin must be finite");
        if (grid->dims[a] < 1) throw Error(FGL_E_USAGE, "dims must be >= 1");
    }
    if ((int64_t)grid->dims[0] * grid->dims[1] * grid->dims[2] > (int64_t(1) << 31))
        throw Error(FGL_E_RESOURCE, "grid exceeds 2^31 voxels: use a coarser spacing");
    if (!std::isfinite(grid->theta)) throw Error(FGL_E_USAGE, "theta must be finite");
    if (grid->tile != 0 && grid->tile != 8) throw Error(FGL_E_USAGE, "tile must be 0 (default) or 8");
    for (int i = 0; i < 3; ++i)
        if (grid->reserved[i]) throw Error(FGL_E_USAGE, "fgl_grid.reserved must be zero");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    auto *ms = const_cast<fgl_scene *>(s);
    if (!ms->vox_counts) {
        FGL_CUDA(cudaMalloc((void **)&ms->vox_counts, sizeof(unsigned long long) * 4));
        FGL_CUDA(cudaMalloc((void **)&ms->vox_overflow, sizeof(unsigned int)));
        FGL_CUDA(cudaMemset(ms->vox_overflow, 0, sizeof(unsigned int)));
    }
    unsigned long long *cnt = counts ? reinterpret_cast<unsigned long long *>(counts) : nullptr;
    if (cnt) FGL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * 4, st));
    fgl::VoxGrid vg;
    for (int a = 0; a < 3; ++a) vg.origin[a] = grid->origin[a], vg.dims[a] = grid->dims[a];
    vg.h = grid->spacing;
    vg.theta = grid->theta;
    fgl::launch_voxelize(s->b, vg, s->kappa, density, occupancy, surface, interior, cnt, ms->vox_overflow, st);
    if (cnt) {  // [3] = traversal-stack overflows (sticky per scene; 0 in any sane configuration)
        FGL_CUDA(cudaMemcpyAsync(cnt + 3, ms->vox_overflow, sizeof(unsigned int), cudaMemcpyDeviceToDevice, st));
    }
    FGL_API_END
}

namespace {
void check_volume(const int32_t *dims, const float *spacing, int64_t max_voxels) {
    if (!dims || !spacing) throw Error(FGL_E_USAGE, "dims / spacing is NULL");
    int64_t n = 1;
    for (int a = 0; a < 3; ++a) {
        if (dims[a] < 1) throw Error(FGL_E_USAGE, "dims must be >= 1");
        if (!(spacing[a] > 0.f) || !std::isfinite(spacing[a])) throw Error(FGL_E_USAGE, "spacing must be finite and > 0");
        n *= dims[a];
    }
    if (n > max_voxels) throw Error(FGL_E_RESOURCE, "volume too large");
}
}  // namespace

fgl_status fgl_denoise(const uint32_t *occupancy, const int32_t *dims, const float *spacing, float sigma, float tau,
                       uint32_t *out, float *vprime, void *stream) {
    FGL_API_BEGIN
    check_volume(dims, spacing, (int64_t(1) << 31) - 1);
    if (!occupancy || !out) throw Error(FGL_E_USAGE, "occupancy / out is NULL");
    if (!(sigma > 0.f) || !std::isfinite(sigma)) throw Error(FGL_E_USAGE, "sigma must be finite and > 0");
    if (!std::isfinite(tau)) throw Error(FGL_E_USAGE, "tau must be finite");
    fgl::launch_denoise(occupancy, dims, spacing, sigma, tau, out, vprime, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_denoise_quantile(const uint32_t *occupancy, const int32_t *dims, const float *spacing, float sigma,
                                float q, uint32_t *out, float *vprime, float *threshold, void *stream) {
    FGL_API_BEGIN
    check_volume(dims, spacing, (int64_t(1) << 31) - 1);
    if (!occupancy || !out) throw Error(FGL_E_USAGE, "occupancy / out is NULL");
    if (!(sigma > 0.f) || !std::isfinite(sigma)) throw Error(FGL_E_USAGE, "sigma must be finite and > 0");
    if (!(q >= 0.f && q <= 1.f)) throw Error(FGL_E_USAGE, "q must be in [0, 1]");
    fgl::launch_denoise(occupancy, dims, spacing, sigma, q, out, vprime, (cudaStream_t)stream, 1, threshold);
    FGL_API_END
}

fgl_status fgl_tsdf(const uint32_t *occupancy, const int32_t *dims, const float *spacing, float r, float *phi,
                    void *stream) {
    FGL_API_BEGIN
    check_volume(dims, spacing, (int64_t(1) << 31) - 1);
    if (!occupancy || !phi) throw Error(FGL_E_USAGE, "occupancy / phi is NULL");
    if (!(r > 0.f) || !std::isfinite(r)) throw Error(FGL_E_USAGE, "r must be finite and > 0");
    fgl::launch_tsdf(occupancy, dims, spacing, r, phi, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_marching_cubes(const float *phi, const int32_t *dims, const float *origin, const float *spacing,
                              float iso, float *verts, float *normals, int64_t vcap, int32_t *tris, int64_t tcap,
                              int64_t *counts, void *stream) {
    FGL_API_BEGIN
    check_volume(dims, spacing, int64_t(1) << 30);
    if (!phi || !origin) throw Error(FGL_E_USAGE, "phi / origin is NULL");
    if (!std::isfinite(iso)) throw Error(FGL_E_USAGE, "iso must be finite");
    if (vcap < 0 || tcap < 0) throw Error(FGL_E_USAGE, "capacities must be >= 0");
    if ((vcap > 0 && !verts) || (tcap > 0 && !tris)) throw Error(FGL_E_USAGE, "verts / tris is NULL");
    if (normals && vcap > 0 && !verts) throw Error(FGL_E_USAGE, "normals need verts");
    fgl::launch_marching_cubes(phi, dims, origin, spacing, iso, verts, normals, vcap, tris, tcap, counts,
                               (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_nearest(const fgl_scene *s, const float *queries, int64_t m, float *dist, int32_t *idx, void *stream) {
    FGL_API_BEGIN
    check_cast(s);
    if (!s->points) throw Error(FGL_E_USAGE, "fgl_nearest needs a point scene (fgl_scene_upload_points)");
    if (m < 0) throw Error(FGL_E_USAGE, "m must be >= 0");
    if (m == 0) return FGL_OK;
    if (!queries || !dist || !idx) throw Error(FGL_E_USAGE, "NULL pointer argument");
    if (s->b.width != 2) throw Error(FGL_E_USAGE, "fgl_nearest needs a width-2 build");
    DeviceGuard g(s->dev);
    fgl::launch_nearest(view(s), queries, m, dist, idx, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cloud_metrics(const float *d_ab, int64_t n_a, const float *d_ba, int64_t n_b, float tau, double *out,
                             void *stream) {
    FGL_API_BEGIN
    if (n_a < 0 || n_b < 0) throw Error(FGL_E_USAGE, "negative count");
    if (!(tau > 0.f)) throw Error(FGL_E_USAGE, "tau must be > 0");
    if (!out || (n_a && !d_ab) || (n_b && !d_ba)) throw Error(FGL_E_USAGE, "NULL pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    void *scratch = nullptr;
    FGL_CUDA(cudaMallocAsync(&scratch, 6 * sizeof(double) + 16, st));
    FGL_CUDA(cudaMemsetAsync(scratch, 0, 6 * sizeof(double) + 16, st));
    fgl::launch_metrics(d_ab, n_a, d_ba, n_b, tau, (double *)scratch, (unsigned int *)((char *)scratch + 48), out, st);
    cudaFreeAsync(scratch, st);
    FGL_API_END
}

fgl_status fgl_scene_check(fgl_scene *s, void *stream) {
    FGL_API_BEGIN
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    if (s->T <= 0) throw Error(FGL_E_USAGE, "no mesh uploaded");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    FGL_CUDA(cudaMemcpyAsync(s->hflag, s->vflag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FGL_CUDA(cudaStreamSynchronize(st));
    if (*s->hflag & 1u) throw Error(FGL_E_DATA, "triangle index out of range [0, V)");
    if (*s->hflag & 2u) throw Error(FGL_E_DATA, "non-finite vertex coordinate");
    if (*s->hflag & 4u)
        throw Error(FGL_E_DATA, "the tree needs a deeper traversal stack than the cast has (width 8, or a restructured "
                                "tree deeper than 94 levels); casts were refused");
    FGL_API_END
}

fgl_status fgl_scene_build(fgl_scene *s, const fgl_build_opts *opts, void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl build");
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    if (s->T <= 0) throw Error(FGL_E_USAGE, "no mesh uploaded");
    // default b (R7): 10 bits per axis (30-bit keys, four sort passes) below 4 M primitives, where
    // the cubic cells are already finer than the primitives; 13 above (the 10 M-triangle terrain
    // loses 7% cast speed at b = 10)
    int bits = s->T < (int64_t(1) << 22) ? 10 : 13, leaf = 2, cubic = 1, width = 2, quant = 0, restructure = 0,
        treelets = 0;
    if (opts) {
        if (opts->quantized < 0 || opts->quantized > 1) throw Error(FGL_E_USAGE, "quantized must be 0 or 1");
        quant = opts->quantized;
        if (opts->width) width = opts->width;
        if (width != 2 && width != 4 && width != 8) throw Error(FGL_E_USAGE, "width must be 2, 4 or 8");
        if (opts->morton_box < 0 || opts->morton_box > 1) throw Error(FGL_E_USAGE, "morton_box must be 0 or 1");
        cubic = opts->morton_box == 0;
        if (opts->reserved[0]) throw Error(FGL_E_USAGE, "fgl_build_opts.reserved must be zero");
        if (opts->treelets < 0 || opts->treelets > 1) throw Error(FGL_E_USAGE, "treelets must be 0 or 1");
        treelets = opts->treelets;
        if (opts->restructure < -8 || opts->restructure > 8) throw Error(FGL_E_USAGE, "restructure must be in [-8, 8]");
        restructure = opts->restructure;
        if (opts->morton_bits) bits = opts->morton_bits;
        if (opts->leaf_size) leaf = opts->leaf_size;
    }
    if (bits < 1 || bits > 21) throw Error(FGL_E_USAGE, "morton_bits must be in [1, 21]");
    if (leaf < 1 || leaf > fgl::kMaxLeaf) throw Error(FGL_E_USAGE, "leaf_size must be in [1, 8]");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    s->bits = bits, s->leaf_size = leaf;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    FGL_CUDA(cudaStreamIsCapturing(st, &cap));
    const bool timed = cap == cudaStreamCaptureStatusNone;  // build_ms is not recorded inside a graph
    if (timed) FGL_CUDA(cudaEventRecord(s->ev0, st));
    if (quant && width == 2) throw Error(FGL_E_USAGE, "quantized nodes need width 4 or 8");
    if (width == 8) quant = 1;  // the 8-wide node is always the compressed node96q
    if (s->gauss) {
        if (width != 2 || quant) throw Error(FGL_E_USAGE, "a Gaussian scene builds width-2 nodes only");
        if (!cubic) throw Error(FGL_E_USAGE, "a Gaussian scene uses the cubic Morton box");
        if (restructure || treelets) throw Error(FGL_E_USAGE, "a Gaussian scene builds the plain Karras tree");
        fgl::launch_gauss_build(s->verts, s->g_quat, s->g_scale, s->g_opac, s->kappa, s->b, bits, leaf, st);
    } else {
        if (restructure && width != 2) throw Error(FGL_E_USAGE, "restructure needs width 2");
        if (treelets && (width != 2 || restructure)) throw Error(FGL_E_USAGE, "treelets needs width 2, restructure 0");
        fgl::launch_build(s->verts, s->V, s->tris, s->b, bits, leaf, cubic, width, quant, st, restructure, treelets);
    }
    if (timed) FGL_CUDA(cudaEventRecord(s->ev1, st));
    s->built = true;
    FGL_API_END
}

fgl_status fgl_scene_refit(fgl_scene *s, const float *verts, int64_t V, int ptr_kind, void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl refit");
    check_built(s);
    if (s->gauss) throw Error(FGL_E_USAGE, "refit is for triangle / point scenes");
    const bool async = (ptr_kind & FGL_ASYNC) != 0;
    ptr_kind &= ~FGL_ASYNC;
    if (ptr_kind != FGL_HOST && ptr_kind != FGL_DEVICE) throw Error(FGL_E_USAGE, "ptr_kind must be FGL_HOST or FGL_DEVICE");
    if (!verts) throw Error(FGL_E_USAGE, "verts is NULL");
    if (V != s->V) throw Error(FGL_E_USAGE, "refit needs the uploaded vertex count (same topology)");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    FGL_CUDA(cudaStreamIsCapturing(st, &cap));
    const bool timed = cap == cudaStreamCaptureStatusNone;
    FGL_CUDA(cudaMemcpyAsync(s->verts, verts, sizeof(float) * 3 * V,
                             ptr_kind == FGL_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    fgl::launch_validate(s->verts, V, s->tris, s->T, s->vflag, st);
    if (timed) FGL_CUDA(cudaEventRecord(s->ev0, st));
    fgl::launch_refit(s->verts, s->V, s->tris, s->b, s->leaf_size, st);
    if (timed) FGL_CUDA(cudaEventRecord(s->ev1, st));
    if (async) return FGL_OK;
    FGL_CUDA(cudaMemcpyAsync(s->hflag, s->vflag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    FGL_CUDA(cudaStreamSynchronize(st));
    if (*s->hflag & 2u) throw Error(FGL_E_DATA, "non-finite vertex coordinate");
    FGL_API_END
}

fgl_status fgl_scene_stats(fgl_scene *s, fgl_stats *out) {
    FGL_API_BEGIN
    if (!s || !out) throw Error(FGL_E_USAGE, "NULL argument");
    DeviceGuard g(s->dev);
    memset(out, 0, sizeof(*out));
    out->triangles = s->T;
    out->vertices = s->V;
    out->nodes = std::max<int64_t>(s->T - 1, 1);
    out->device_bytes = (int64_t)(s->bytes + sizeof(float) * 3 * s->cap_V + sizeof(int32_t) * 3 * s->cap_T);
    out->morton_bits = s->bits;
    out->leaf_size = s->leaf_size;
    if (s->built) {
        FGL_CUDA(cudaEventSynchronize(s->ev1));
        FGL_CUDA(cudaEventElapsedTime(&out->build_ms, s->ev0, s->ev1));
        float box[6];
        FGL_CUDA(cudaMemcpy(box, s->b.box, sizeof(box), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 3; ++i) out->scene_lo[i] = box[i], out->scene_hi[i] = box[3 + i];
    }
    FGL_API_END
}

fgl_status fgl_cast_spinning(const fgl_scene *s, const fgl_spinning *pattern, const float *poses, int64_t P,
                             float *range, int32_t *tri_id, float *hit_xyz, int32_t *node_counts, int32_t *tri_counts,
                             void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl cast spinning (A8-A11)");
    check_cast(s);
    fgl::SpinParams sp = spin_params(pattern);
    if (P < 0) throw Error(FGL_E_USAGE, "P must be >= 0");
    if (P == 0) return FGL_OK;
    if (!poses) throw Error(FGL_E_USAGE, "poses is NULL");
    fgl::CastOut o = cast_out(range, tri_id, hit_xyz, node_counts, tri_counts);
    DeviceGuard g(s->dev);
    fgl::launch_cast_spinning(view(s), sp, poses, P, o, next_counter(s), (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cast_rosette(const fgl_scene *s, const fgl_rosette *pattern, const float *poses, int64_t P,
                            int64_t first_frame, float *range, int32_t *tri_id, float *hit_xyz, int32_t *node_counts,
                            int32_t *tri_counts, void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl cast rosette (A8-A11)");
    check_cast(s);
    fgl::RosetteParams rp = rosette_params(pattern, first_frame);
    if (P < 0) throw Error(FGL_E_USAGE, "P must be >= 0");
    if (P == 0) return FGL_OK;
    if (!poses) throw Error(FGL_E_USAGE, "poses is NULL");
    fgl::CastOut o = cast_out(range, tri_id, hit_xyz, node_counts, tri_counts);
    DeviceGuard g(s->dev);
    fgl::launch_cast_rosette(view(s), rp, poses, P, o, next_counter(s), (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cast_rays(const fgl_scene *s, const float *orig, const float *dir, int64_t R, float t_min, float t_max,
                         float *range, int32_t *tri_id, void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl cast rays (A9-A11)");
    check_cast(s);
    check_interval(t_min, t_max);
    if (R < 0) throw Error(FGL_E_USAGE, "R must be >= 0");
    if (R == 0) return FGL_OK;
    if (!orig || !dir) throw Error(FGL_E_USAGE, "orig / dir is NULL");
    fgl::CastOut o = cast_out(range, tri_id, nullptr, nullptr, nullptr);
    DeviceGuard g(s->dev);
    fgl::launch_cast_rays(view(s), orig, dir, R, t_min, t_max, o, next_counter(s), (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cast_rays_bruteforce(const fgl_scene *s, const float *orig, const float *dir, int64_t R, float t_min,
                                    float t_max, float *range, int32_t *tri_id, void *stream) {
    FGL_API_BEGIN
    if (!s) throw Error(FGL_E_USAGE, "scene is NULL");
    if (s->T <= 0) throw Error(FGL_E_USAGE, "no mesh uploaded");
    check_interval(t_min, t_max);
    if (R < 0) throw Error(FGL_E_USAGE, "R must be >= 0");
    if (R == 0) return FGL_OK;
    if (!orig || !dir || !range || !tri_id) throw Error(FGL_E_USAGE, "NULL pointer argument");
    DeviceGuard g(s->dev);
    fgl::launch_cast_bruteforce(s->verts, s->V, s->tris, s->T, orig, dir, R, t_min, t_max, range, tri_id,
                                (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cast_spinning_gather_signal(const fgl_scene *s, const fgl_spinning *pattern, const float *poses,
                                           int64_t P, int64_t first_pose, float *const *range_bufs,
                                           int32_t *const *tri_bufs, int32_t *const *flags, int32_t npeer,
                                           void *stream) {
    FGL_API_BEGIN
    fgl::NvtxRange nvtx_range_("fgl cast + gather (A8-A12)");
    check_cast(s);
    fgl::SpinParams sp = spin_params(pattern);
    if (P < 0 || first_pose < 0) throw Error(FGL_E_USAGE, "P and first_pose must be >= 0");
    if (npeer < 1 || npeer > fgl::kMaxPeers) throw Error(FGL_E_USAGE, "npeer must be in [1, 8]");
    if (!range_bufs || !tri_bufs) throw Error(FGL_E_USAGE, "range_bufs / tri_bufs is NULL");
    if (P > 0 && !poses) throw Error(FGL_E_USAGE, "poses is NULL");
    fgl::CastOut o;
    memset(&o, 0, sizeof(o));
    const int64_t per = (int64_t)sp.channels * sp.columns;
    // the local copy is peer 0's buffer (this process's own global output)
    o.range = range_bufs[0] + first_pose * per;
    o.tri_id = tri_bufs[0] + first_pose * per;
    o.npeer = npeer - 1;
    o.out_offset = first_pose * per;
    for (int w = 1; w < npeer; ++w) {
        if (!range_bufs[w] || !tri_bufs[w]) throw Error(FGL_E_USAGE, "NULL peer buffer");
        o.peer_range[w - 1] = range_bufs[w];
        o.peer_tri[w - 1] = tri_bufs[w];
    }
    if (flags) {
        o.nsignal = npeer;
        for (int w = 0; w < npeer; ++w) {
            if (!flags[w]) throw Error(FGL_E_USAGE, "NULL flag pointer");
            o.signal[w] = flags[w];
        }
    }
    DeviceGuard g(s->dev);
    if (P == 0) {
        // nothing to cast: still signal every rank (a 1-tile launch whose only work is the epilogue)
        if (!flags) return FGL_OK;
    }
    fgl::launch_cast_spinning(view(s), sp, poses, P, o, next_counter(s), (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_cast_spinning_gather(const fgl_scene *s, const fgl_spinning *pattern, const float *poses, int64_t P,
                                    int64_t first_pose, float *const *range_bufs, int32_t *const *tri_bufs,
                                    int32_t npeer, void *stream) {
    return fgl_cast_spinning_gather_signal(s, pattern, poses, P, first_pose, range_bufs, tri_bufs, nullptr, npeer,
                                           stream);
}

fgl_status fgl_l2_read_probe(const void *buf, int64_t bytes, int32_t iters, float *sink, void *stream) {
    FGL_API_BEGIN
    if (!buf || !sink) throw Error(FGL_E_USAGE, "buffer / sink is NULL");
    if (bytes < 16 || bytes % 16 || ((uintptr_t)buf & 15)) throw Error(FGL_E_USAGE, "bytes must be a positive multiple of 16, buffer 16-B aligned");
    if (iters < 1) throw Error(FGL_E_USAGE, "iters must be >= 1");
    fgl::launch_l2_read(buf, bytes, iters, sink, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_wait_flag(const int32_t *flag, int32_t target, void *stream) {
    FGL_API_BEGIN
    if (!flag) throw Error(FGL_E_USAGE, "flag is NULL");
    fgl::launch_wait_flag(flag, target, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_alloc(int dev, int64_t bytes, void **p) {
    FGL_API_BEGIN
    if (!p || bytes <= 0) throw Error(FGL_E_USAGE, "bad fgl_alloc arguments");
    DeviceGuard g(dev);
    FGL_CUDA(cudaMalloc(p, (size_t)bytes));
    FGL_API_END
}

fgl_status fgl_free(void *p) {
    FGL_API_BEGIN
    if (p) FGL_CUDA(cudaFree(p));
    FGL_API_END
}

fgl_status fgl_ipc_get_handle(void *p, fgl_ipc_handle *out) {
    FGL_API_BEGIN
    if (!p || !out) throw Error(FGL_E_USAGE, "NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(fgl_ipc_handle), "IPC handle size");
    cudaIpcMemHandle_t h;
    FGL_CUDA(cudaIpcGetMemHandle(&h, p));
    memcpy(out->bytes, &h, sizeof(h));
    FGL_API_END
}

fgl_status fgl_ipc_open_handle(int dev, const fgl_ipc_handle *handle, void **p) {
    FGL_API_BEGIN
    if (!handle || !p) throw Error(FGL_E_USAGE, "NULL argument");
    DeviceGuard g(dev);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle->bytes, sizeof(h));
    FGL_CUDA(cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess));
    FGL_API_END
}

fgl_status fgl_ipc_close_handle(void *p) {
    FGL_API_BEGIN
    if (p) FGL_CUDA(cudaIpcCloseMemHandle(p));
    FGL_API_END
}

fgl_status fgl_export_rays_spinning(const fgl_spinning *pattern, const float *poses, int64_t P, float *orig, float *dir,
                                    void *stream) {
    FGL_API_BEGIN
    fgl::SpinParams sp = spin_params(pattern);
    if (P < 0) throw Error(FGL_E_USAGE, "P must be >= 0");
    if (P == 0) return FGL_OK;
    if (!poses || !orig || !dir) throw Error(FGL_E_USAGE, "NULL pointer argument");
    fgl::launch_export_spinning(sp, poses, P, orig, dir, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_export_rays_rosette(const fgl_rosette *pattern, const float *poses, int64_t P, int64_t first_frame,
                                   float *orig, float *dir, void *stream) {
    FGL_API_BEGIN
    fgl::RosetteParams rp = rosette_params(pattern, first_frame);
    if (P < 0) throw Error(FGL_E_USAGE, "P must be >= 0");
    if (P == 0) return FGL_OK;
    if (!poses || !orig || !dir) throw Error(FGL_E_USAGE, "NULL pointer argument");
    fgl::launch_export_rosette(rp, poses, P, orig, dir, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_scene_export(const fgl_scene *s, const fgl_export *out, void *stream) {
    FGL_API_BEGIN
    check_built(s);
    if (!out) throw Error(FGL_E_USAGE, "out is NULL");
    DeviceGuard g(s->dev);
    cudaStream_t st = (cudaStream_t)stream;
    if (!s->gauss && (out->leaf_box || out->node_box)) {
        // the fused build stores only the boxes a sibling needs: derive them all (exact unions over
        // the current tree; tri48 is regathered identically), so the export is right after any build,
        // refit or graph replay — the scene's traversal data do not change
        fgl_scene *m = const_cast<fgl_scene *>(s);
        fgl::launch_complete_boxes(m->verts, m->V, m->tris, m->b, st);
    }
    FGL_CUDA(cudaStreamSynchronize(st));
    const int64_t T = s->T, nin = std::max<int64_t>(T - 1, 0);
    const fgl::BuildBuffers &b = s->b;
    auto cp = [&](void *dst, const void *src, size_t bytes) {
        if (dst && bytes) FGL_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    cp(out->scene_box, b.box, 6 * sizeof(float));
    if (out->sorted_keys || out->perm || out->codes) {
        // sorted (code, index) pairs; packed keys hold code << packed_shift | index
        std::vector<uint64_t> k(T);
        std::vector<uint32_t> p(T);
        cp(k.data(), b.keys[b.sorted_slot], T * sizeof(uint64_t));
        if (b.packed_shift) {
            const uint64_t mask = (uint64_t(1) << b.packed_shift) - 1;
            for (int64_t j = 0; j < T; ++j) p[j] = (uint32_t)(k[j] & mask), k[j] >>= b.packed_shift;
        } else {
            cp(p.data(), b.vals[b.sorted_slot], T * sizeof(uint32_t));
        }
        if (out->sorted_keys) std::memcpy(out->sorted_keys, k.data(), T * sizeof(uint64_t));
        if (out->perm) std::memcpy(out->perm, p.data(), T * sizeof(uint32_t));
        // input-order codes: codes[perm[j]] = sorted_keys[j] (a permutation of the sorted array)
        if (out->codes)
            for (int64_t j = 0; j < T; ++j) out->codes[p[j]] = k[j];
    }
    cp(out->child, b.child, nin * sizeof(int2));
    cp(out->range, b.range, nin * sizeof(int2));
    if (out->leaf_box || out->node_box) {
        std::string tmp(std::max<int64_t>(2 * T, 2 * nin) * sizeof(float4), '\0');
        float4 *f = (float4 *)&tmp[0];
        if (out->leaf_box) {
            cp(f, b.leafbox, 2 * T * sizeof(float4));
            for (int64_t j = 0; j < T; ++j)
                for (int i = 0; i < 3; ++i)
                    out->leaf_box[6 * j + i] = (&f[2 * j].x)[i], out->leaf_box[6 * j + 3 + i] = (&f[2 * j + 1].x)[i];
        }
        if (out->node_box && nin) {
            cp(f, b.nodebox, 2 * nin * sizeof(float4));
            for (int64_t j = 0; j < nin; ++j)
                for (int i = 0; i < 3; ++i)
                    out->node_box[6 * j + i] = (&f[2 * j].x)[i], out->node_box[6 * j + 3 + i] = (&f[2 * j + 1].x)[i];
        }
    }
    if (out->tri48 && T) {  // the export format is the 48-byte record; drop the pad of 64-byte ones
        if (fgl::kTriStride == 3 || s->gauss) {
            cp(out->tri48, b.tri, 3 * T * sizeof(float4));
        } else {
            std::vector<float4> tmp((size_t)fgl::kTriStride * T);
            cp(tmp.data(), b.tri, tmp.size() * sizeof(float4));
            float4 *o = reinterpret_cast<float4 *>(out->tri48);
            for (int64_t j = 0; j < T; ++j)
                for (int q = 0; q < 3; ++q) o[3 * j + q] = tmp[(size_t)fgl::kTriStride * j + q];
        }
    }
    cp(out->nodes, b.nodes, std::max<int64_t>(nin, 1) * sizeof(fgl::Node64));
    cp(out->nodes4, b.nodes4, std::max<int64_t>(nin, 1) * sizeof(fgl::Node128));
    cp(out->depth, b.depth, nin * sizeof(int32_t));
    FGL_API_END
}

fgl_status fgl_morton_codes(const float *points, int64_t n, const float *lo, const float *hi, int32_t bits,
                            uint64_t *codes, void *stream) {
    FGL_API_BEGIN
    if (n < 0) throw Error(FGL_E_USAGE, "n must be >= 0");
    if (bits < 1 || bits > 21) throw Error(FGL_E_USAGE, "bits must be in [1, 21]");
    if (n == 0) return FGL_OK;
    if (!points || !lo || !hi || !codes) throw Error(FGL_E_USAGE, "NULL pointer argument");
    fgl::launch_morton_points(points, n, lo, hi, bits, codes, (cudaStream_t)stream);
    FGL_API_END
}

fgl_status fgl_sort_pairs(uint64_t *keys, uint32_t *vals, int64_t n, int32_t key_bits, void *stream) {
    FGL_API_BEGIN
    if (n < 0) throw Error(FGL_E_USAGE, "n must be >= 0");
    if (key_bits < 1 || key_bits > 64) throw Error(FGL_E_USAGE, "key_bits must be in [1, 64]");
    if (n >= (int64_t(1) << 30)) throw Error(FGL_E_USAGE, "n must be < 2^30");
    if (n <= 1) return FGL_OK;
    if (!keys || !vals) throw Error(FGL_E_USAGE, "NULL pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *k1 = nullptr;
    uint32_t *v1 = nullptr, *tiles = nullptr, *ghist = nullptr;
    uint64_t *status = nullptr;
    FGL_CUDA(cudaMallocAsync((void **)&k1, n * sizeof(uint64_t), st));
    FGL_CUDA(cudaMallocAsync((void **)&v1, n * sizeof(uint32_t), st));
    const size_t nstat = (size_t)256 * fgl::sort_tile_blocks(n);
    FGL_CUDA(cudaMallocAsync((void **)&status, nstat * sizeof(uint64_t), st));
    FGL_CUDA(cudaMemsetAsync(status, 0, nstat * sizeof(uint64_t), st));
    FGL_CUDA(cudaMallocAsync((void **)&tiles, 16 * sizeof(uint32_t), st));
    FGL_CUDA(cudaMemsetAsync(tiles, 0, 16 * sizeof(uint32_t), st));
    FGL_CUDA(cudaMallocAsync((void **)&ghist, 8 * 256 * sizeof(uint32_t), st));
    uint32_t *rts = nullptr;
    FGL_CUDA(cudaMallocAsync((void **)&rts, (size_t)256 * fgl::sort_tile_blocks(n) * sizeof(uint32_t), st));
    int slot = 0;
    fgl::radix_sort_pairs(keys, vals, k1, v1, n, key_bits, status, tiles, ghist, false, &slot, st, 0, rts);
    if (slot == 1) {
        FGL_CUDA(cudaMemcpyAsync(keys, k1, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        FGL_CUDA(cudaMemcpyAsync(vals, v1, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    }
    cudaFreeAsync(k1, st);
    cudaFreeAsync(v1, st);
    cudaFreeAsync(status, st);
    cudaFreeAsync(tiles, st);
    cudaFreeAsync(ghist, st);
    cudaFreeAsync(rts, st);
    FGL_API_END
}

}  // extern "C"
