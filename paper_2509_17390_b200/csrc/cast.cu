// LiDAR first-return cast on sm_100a — PAPER.md §IV-C.
//
// One lane per beam, rays generated in registers from the pattern (Eq. 19),
// BVH traversal pruned by the best-so-far t* ("nodes whose entry distance exceeds t* are
// discarded"), leaf triangles tested with the watertight ray/triangle test of Woop,
// Benthin & Wald (JCGT 2013), nearest (t, id) kept lexicographically (Eq. 20 + R4), and the
// result written to its own output slot without locks.
//
// Work distribution: persistent warps; each warp takes 32-ray tiles from a self-resetting atomic
// counter. Spinning tiles are 4 channels x 8 columns (or 2x16 / 1x32) of one pose, so the 32 rays
// of a warp are angular neighbours and walk nearly the same nodes (warp-coherent traversal,
// P:297 "warp-synchronous traversal").
#include <cfloat>
#include <climits>

#include "fgl_internal.cuh"

namespace fgl {

namespace {

constexpr int kCastThreads = 128;
constexpr int kStack = 96;                   // > max depth of a Karras tree over 63-bit keys + index
constexpr float kExpand = 1.0f + 0x1p-20f;   // conservative slab test: tfar * (1 + 2 gamma_3) (Ize 2013)

struct Ray {
    float ox, oy, oz, dx, dy, dz;
};

// per-ray constants of the watertight test and of the slab test
struct Pre {
    float ox, oy, oz;
    float ix, iy, iz;  // 1/d with |d_i| < 2^-80 replaced by +-2^-80 (no 0 * inf in slabs)
    float Sx, Sy, Sz;
    int kx, ky, kz;
};

__device__ __forceinline__ Pre precompute(const Ray &r) {
    Pre p;
    p.ox = r.ox, p.oy = r.oy, p.oz = r.oz;
    const float tiny = 0x1p-80f;
    float dx = fabsf(r.dx) < tiny ? copysignf(tiny, r.dx) : r.dx;
    float dy = fabsf(r.dy) < tiny ? copysignf(tiny, r.dy) : r.dy;
    float dz = fabsf(r.dz) < tiny ? copysignf(tiny, r.dz) : r.dz;
    p.ix = __frcp_rn(dx), p.iy = __frcp_rn(dy), p.iz = __frcp_rn(dz);
    float ax = fabsf(r.dx), ay = fabsf(r.dy), az = fabsf(r.dz);
    int kz = (ax >= ay) ? (ax >= az ? 0 : 2) : (ay >= az ? 1 : 2);
    int kx = kz == 2 ? 0 : kz + 1;
    int ky = kx == 2 ? 0 : kx + 1;
    float dkz = kz == 0 ? r.dx : (kz == 1 ? r.dy : r.dz);
    if (dkz < 0.f) {
        int t = kx;
        kx = ky;
        ky = t;
    }
    float dkx = kx == 0 ? r.dx : (kx == 1 ? r.dy : r.dz);
    float dky = ky == 0 ? r.dx : (ky == 1 ? r.dy : r.dz);
    p.Sx = __fdiv_rn(dkx, dkz);
    p.Sy = __fdiv_rn(dky, dkz);
    p.Sz = __frcp_rn(dkz);
    p.kx = kx, p.ky = ky, p.kz = kz;
    return p;
}

__device__ __forceinline__ float pick(float x, float y, float z, int k) { return k == 0 ? x : (k == 1 ? y : z); }

// Watertight ray/triangle test (two-sided, inclusive edges). Edge functions are evaluated without
// FMA contraction so that the two triangles of a shared edge see exactly opposite values; an
// exactly-zero edge function is re-evaluated in double (float products are exact there).
// Returns true and t when the hit is in [tmin, best_t] and beats (best_t, best_id).
__device__ __forceinline__ bool hit_tri(const Pre &p, float4 a, float4 b, float4 c, float tmin, float best_t,
                                        int32_t best_id, int32_t id, float &t_out) {
    const float Ax0 = a.x - p.ox, Ay0 = a.y - p.oy, Az0 = a.z - p.oz;
    const float Bx0 = b.x - p.ox, By0 = b.y - p.oy, Bz0 = b.z - p.oz;
    const float Cx0 = c.x - p.ox, Cy0 = c.y - p.oy, Cz0 = c.z - p.oz;
    const float Akz = pick(Ax0, Ay0, Az0, p.kz), Bkz = pick(Bx0, By0, Bz0, p.kz), Ckz = pick(Cx0, Cy0, Cz0, p.kz);
    const float Ax = pick(Ax0, Ay0, Az0, p.kx) - p.Sx * Akz;
    const float Ay = pick(Ax0, Ay0, Az0, p.ky) - p.Sy * Akz;
    const float Bx = pick(Bx0, By0, Bz0, p.kx) - p.Sx * Bkz;
    const float By = pick(Bx0, By0, Bz0, p.ky) - p.Sy * Bkz;
    const float Cx = pick(Cx0, Cy0, Cz0, p.kx) - p.Sx * Ckz;
    const float Cy = pick(Cx0, Cy0, Cz0, p.ky) - p.Sy * Ckz;
    float U = __fsub_rn(__fmul_rn(Cx, By), __fmul_rn(Cy, Bx));
    float V = __fsub_rn(__fmul_rn(Ax, Cy), __fmul_rn(Ay, Cx));
    float W = __fsub_rn(__fmul_rn(Bx, Ay), __fmul_rn(By, Ax));
    if (U == 0.f || V == 0.f || W == 0.f) {
        double Ud = (double)Cx * (double)By - (double)Cy * (double)Bx;
        double Vd = (double)Ax * (double)Cy - (double)Ay * (double)Cx;
        double Wd = (double)Bx * (double)Ay - (double)By * (double)Ax;
        if ((Ud < 0.0 || Vd < 0.0 || Wd < 0.0) && (Ud > 0.0 || Vd > 0.0 || Wd > 0.0)) return false;
        U = (float)Ud, V = (float)Vd, W = (float)Wd;
    } else if ((U < 0.f || V < 0.f || W < 0.f) && (U > 0.f || V > 0.f || W > 0.f)) {
        return false;
    }
    const float det = U + V + W;
    if (det == 0.f) return false;
    const float Az = p.Sz * Akz, Bz = p.Sz * Bkz, Cz = p.Sz * Ckz;
    const float T = U * Az + V * Bz + W * Cz;
    const float t = __fdiv_rn(T, det);
    if (!(t >= tmin && t <= best_t)) return false;
    if (t == best_t && id >= best_id) return false;
    t_out = t;
    return true;
}

struct Hit {
    float t;
    int32_t id;
    int32_t nodes, tris;
};

// robust slab test of one child box against [tmin, best_t]; returns entry distance or +inf
__device__ __forceinline__ float slab(const Pre &p, float lx, float hx, float ly, float hy, float lz, float hz,
                                      float tmin, float tmax) {
    const float tx0 = __fmul_rn(__fsub_rn(lx, p.ox), p.ix), tx1 = __fmul_rn(__fsub_rn(hx, p.ox), p.ix);
    const float ty0 = __fmul_rn(__fsub_rn(ly, p.oy), p.iy), ty1 = __fmul_rn(__fsub_rn(hy, p.oy), p.iy);
    const float tz0 = __fmul_rn(__fsub_rn(lz, p.oz), p.iz), tz1 = __fmul_rn(__fsub_rn(hz, p.oz), p.iz);
    const float tn = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), tmin));
    const float tf = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
    return tn <= tf * kExpand ? tn : INFINITY;
}

template <bool kCount>
__device__ __forceinline__ Hit trace(const SceneView &sv, const Ray &r, float tmin, float tmax) {
    const Pre p = precompute(r);
    Hit h{tmax, INT_MAX, 0, 0};
    int32_t st_ref[kStack];
    float st_t[kStack];
    int sp = 0;
    int32_t cur = 0;  // root: internal node 0
    while (true) {
        if (cur >= 0) {
            const float4 *np = reinterpret_cast<const float4 *>(sv.nodes + cur);
            const float4 na = __ldg(np), nb = __ldg(np + 1), nc = __ldg(np + 2);
            const int4 nd = __ldg(reinterpret_cast<const int4 *>(np + 3));
            if (kCount) ++h.nodes;
            const float lim = h.t;
            float t0 = slab(p, na.x, na.y, na.z, na.w, nc.x, nc.y, tmin, lim);
            float t1 = nd.y == kEmptyRef ? INFINITY : slab(p, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, tmin, lim);
            const bool h0 = t0 != INFINITY, h1 = t1 != INFINITY;
            if (h0 && h1) {
                const bool swap = t1 < t0;
                st_ref[sp] = swap ? nd.x : nd.y;
                st_t[sp] = swap ? t0 : t1;
                ++sp;
                cur = swap ? nd.y : nd.x;
                continue;
            }
            if (h0) {
                cur = nd.x;
                continue;
            }
            if (h1) {
                cur = nd.y;
                continue;
            }
        } else {
            const int32_t v = ~cur;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 *tp = sv.tri + 3 * (int64_t)k;
                const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
                const int32_t id = __float_as_int(a.w);
                if (kCount) ++h.tris;
                float t;
                if (hit_tri(p, a, b, c, tmin, h.t, h.id, id, t)) {
                    h.t = t;
                    h.id = id;
                }
            }
        }
        // pop the nearest pending subtree whose entry distance does not exceed t*
        bool found = false;
        while (sp > 0) {
            --sp;
            if (st_t[sp] <= h.t * kExpand) {
                cur = st_ref[sp];
                found = true;
                break;
            }
        }
        if (!found) break;
    }
    return h;
}

__device__ __forceinline__ void write_out(const CastOut &o, int64_t idx, const Ray &r, const Hit &h) {
    const bool miss = h.id == INT_MAX;
    o.range[idx] = miss ? INFINITY : h.t;
    o.tri_id[idx] = miss ? -1 : h.id;
    if (o.hit_xyz) {
        float t = miss ? INFINITY : h.t;
        o.hit_xyz[3 * idx] = miss ? NAN : r.ox + t * r.dx;
        o.hit_xyz[3 * idx + 1] = miss ? NAN : r.oy + t * r.dy;
        o.hit_xyz[3 * idx + 2] = miss ? NAN : r.oz + t * r.dz;
    }
    if (o.node_counts) o.node_counts[idx] = h.nodes;
    if (o.tri_counts) o.tri_counts[idx] = h.tris;
}

// ---- ray generators ---------------------------------------------------------------------------
__device__ __forceinline__ void rotate_pose(const float *__restrict__ pose, float sx, float sy, float sz, Ray &r) {
    const float4 r0 = __ldg(reinterpret_cast<const float4 *>(pose));
    const float4 r1 = __ldg(reinterpret_cast<const float4 *>(pose) + 1);
    const float4 r2 = __ldg(reinterpret_cast<const float4 *>(pose) + 2);
    float dx = r0.x * sx + r0.y * sy + r0.z * sz;
    float dy = r1.x * sx + r1.y * sy + r1.z * sz;
    float dz = r2.x * sx + r2.y * sy + r2.z * sz;
    const float n = sqrtf(dx * dx + dy * dy + dz * dz);
    r.dx = __fdiv_rn(dx, n), r.dy = __fdiv_rn(dy, n), r.dz = __fdiv_rn(dz, n);
    r.ox = r0.w, r.oy = r1.w, r.oz = r2.w;
}

// spinning beam (c, a): d_s = (cos e cos th, cos e sin th, sin e), th = 2 pi a / A + az0 (R11, R12)
__device__ __forceinline__ void spin_ray(const SpinParams &sp, const float *__restrict__ poses, int64_t p, int c, int a,
                                         Ray &r) {
    float se, ce, sa, ca;
    sincospif(__fdiv_rn(sp.elev_deg[c], 180.f), &se, &ce);
    sincospif(__fadd_rn(__fdiv_rn(2.f * (float)a, (float)sp.columns), __fdiv_rn(sp.az0_deg, 180.f)), &sa, &ca);
    rotate_pose(poses + 12 * p, ce * ca, ce * sa, se, r);
}

// rosette sample n of pose p (R20): exact 32-bit phases, two counter-rotating prisms
__device__ __forceinline__ void rosette_ray(const RosetteParams &rp, const float *__restrict__ poses, int64_t p, int k,
                                            Ray &r) {
    const uint64_t n = (uint64_t)(rp.first_frame + p) * (uint64_t)rp.n + (uint64_t)k;
    const uint32_t ph1 = (uint32_t)(n * (uint64_t)rp.inc1);
    const uint32_t ph2 = rp.phase2_0 - (uint32_t)(n * (uint64_t)rp.inc2);
    float s1, c1, s2, c2;
    sincospif(2.f * __uint2float_rn(ph1) * 0x1p-32f, &s1, &c1);
    sincospif(2.f * __uint2float_rn(ph2) * 0x1p-32f, &s2, &c2);
    const float half = 0.5f * rp.half_fov_deg * 0.017453292519943295f;
    const float dx = half * (c1 + c2), dy = half * (s1 + s2);
    const float rho = sqrtf(dx * dx + dy * dy);
    float sr, cr;
    sincosf(rho, &sr, &cr);
    const float s = rho > 0.f ? __fdiv_rn(sr, rho) : 1.f;
    rotate_pose(poses + 12 * p, cr, dx * s, dy * s, r);
}

struct SpinGen {
    SpinParams sp;
    const float *poses;
    int tc, ta, nct, nat;  // tile shape and tiles per pose
    __device__ __forceinline__ bool ray(int64_t tile, int lane, Ray &r, int64_t &idx, float &tmin, float &tmax) const {
        const int64_t per = (int64_t)nct * nat;
        const int64_t p = tile / per;
        const int64_t rem = tile - p * per;
        const int cb = (int)(rem / nat), ab = (int)(rem - (int64_t)cb * nat);
        const int c = cb * tc + lane / ta, a = ab * ta + lane % ta;
        tmin = sp.t_min, tmax = sp.t_max;
        if (c >= sp.channels || a >= sp.columns) return false;
        spin_ray(sp, poses, p, c, a, r);
        idx = (p * sp.channels + c) * (int64_t)sp.columns + a;
        return true;
    }
};

struct RosetteGen {
    RosetteParams rp;
    const float *poses;
    int ntile;  // tiles per pose
    __device__ __forceinline__ bool ray(int64_t tile, int lane, Ray &r, int64_t &idx, float &tmin, float &tmax) const {
        const int64_t p = tile / ntile;
        const int k = (int)(tile - p * ntile) * 32 + lane;
        tmin = rp.t_min, tmax = rp.t_max;
        if (k >= rp.n) return false;
        rosette_ray(rp, poses, p, k, r);
        idx = p * rp.n + k;
        return true;
    }
};

struct RaysGen {
    const float *orig, *dir;
    int64_t R;
    float t_min, t_max;
    __device__ __forceinline__ bool ray(int64_t tile, int lane, Ray &r, int64_t &idx, float &tmin, float &tmax) const {
        idx = tile * 32 + lane;
        tmin = t_min, tmax = t_max;
        if (idx >= R) return false;
        r.ox = orig[3 * idx], r.oy = orig[3 * idx + 1], r.oz = orig[3 * idx + 2];
        r.dx = dir[3 * idx], r.dy = dir[3 * idx + 1], r.dz = dir[3 * idx + 2];
        return true;
    }
};

template <class Gen, bool kCount>
__global__ void __launch_bounds__(kCastThreads) k_cast(const SceneView sv, const Gen gen, int64_t ntiles,
                                                       const CastOut out, CastCounter *ctr) {
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned long long tile = 0;
        if (lane == 0) tile = atomicAdd(&ctr->next, 1ull);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= (unsigned long long)ntiles) break;
        Ray r;
        int64_t idx;
        float tmin, tmax;
        if (gen.ray((int64_t)tile, lane, r, idx, tmin, tmax)) {
            Hit h = trace<kCount>(sv, r, tmin, tmax);
            write_out(out, idx, r, h);
        }
    }
    // self-reset: the last warp to finish clears the counter for the next launch using this slot
    if (lane == 0) {
        const unsigned int total = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(&ctr->done, 1u) == total - 1) {
            ctr->next = 0ull;
            ctr->done = 0u;
            __threadfence();
        }
    }
}

template <class Gen>
void launch_persistent(const SceneView &sv, const Gen &gen, int64_t ntiles, const CastOut &o, CastCounter *ctr,
                       cudaStream_t s) {
    if (ntiles <= 0) return;
    const bool count = o.node_counts || o.tri_counts;
    static int occ[2] = {0, 0};
    static int sms = 0;
    int &oc = occ[count];
    if (!oc) {
        int dev;
        FGL_CUDA(cudaGetDevice(&dev));
        FGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (count)
            FGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, k_cast<Gen, true>, kCastThreads, 0));
        else
            FGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, k_cast<Gen, false>, kCastThreads, 0));
        if (oc < 1) oc = 1;
    }
    const int64_t warps_needed = ntiles;
    int64_t blocks = std::min<int64_t>((int64_t)sms * oc, (warps_needed + kCastThreads / 32 - 1) / (kCastThreads / 32));
    blocks = std::max<int64_t>(blocks, 1);
    if (count)
        k_cast<Gen, true><<<(unsigned)blocks, kCastThreads, 0, s>>>(sv, gen, ntiles, o, ctr);
    else
        k_cast<Gen, false><<<(unsigned)blocks, kCastThreads, 0, s>>>(sv, gen, ntiles, o, ctr);
    FGL_LAUNCHED("k_cast");
}

// ---- brute force: every ray against every triangle, triangles staged in smem -------
constexpr int kBfThreads = 128;
__global__ void __launch_bounds__(kBfThreads) k_bruteforce(const float *__restrict__ verts,
                                                           const int32_t *__restrict__ tris, int64_t T,
                                                           const float *__restrict__ orig,
                                                           const float *__restrict__ dir, int64_t R, float tmin,
                                                           float tmax, float *__restrict__ range,
                                                           int32_t *__restrict__ tri_id) {
    __shared__ float4 st[kBfThreads][3];
    const int64_t i = blockIdx.x * (int64_t)kBfThreads + threadIdx.x;
    const bool live = i < R;
    Ray r{0, 0, 0, 1, 0, 0};
    if (live) {
        r.ox = orig[3 * i], r.oy = orig[3 * i + 1], r.oz = orig[3 * i + 2];
        r.dx = dir[3 * i], r.dy = dir[3 * i + 1], r.dz = dir[3 * i + 2];
    }
    const Pre p = precompute(r);
    float bt = tmax;
    int32_t bid = INT_MAX;
    for (int64_t base = 0; base < T; base += kBfThreads) {
        const int64_t k = base + threadIdx.x;
        if (k < T) {
            for (int v = 0; v < 3; ++v) {
                const int32_t vi = tris[3 * k + v];
                st[threadIdx.x][v] = make_float4(verts[3 * (int64_t)vi], verts[3 * (int64_t)vi + 1],
                                                 verts[3 * (int64_t)vi + 2], 0.f);
            }
        }
        __syncthreads();
        const int n = (int)std::min<int64_t>(kBfThreads, T - base);
        if (live)
            for (int j = 0; j < n; ++j) {
                float t;
                const int32_t id = (int32_t)(base + j);
                if (hit_tri(p, st[j][0], st[j][1], st[j][2], tmin, bt, bid, id, t)) bt = t, bid = id;
            }
        __syncthreads();
    }
    if (live) {
        range[i] = bid == INT_MAX ? INFINITY : bt;
        tri_id[i] = bid == INT_MAX ? -1 : bid;
    }
}

__global__ void k_export_spin(const SpinParams sp, const float *__restrict__ poses, int64_t n, float *orig,
                              float *dir) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t per = (int64_t)sp.channels * sp.columns;
        const int64_t p = g / per;
        const int c = (int)((g - p * per) / sp.columns), a = (int)(g % sp.columns);
        Ray r;
        spin_ray(sp, poses, p, c, a, r);
        orig[3 * g] = r.ox, orig[3 * g + 1] = r.oy, orig[3 * g + 2] = r.oz;
        dir[3 * g] = r.dx, dir[3 * g + 1] = r.dy, dir[3 * g + 2] = r.dz;
    }
}

__global__ void k_export_rosette(const RosetteParams rp, const float *__restrict__ poses, int64_t n, float *orig,
                                 float *dir) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = g / rp.n;
        Ray r;
        rosette_ray(rp, poses, p, (int)(g - p * rp.n), r);
        orig[3 * g] = r.ox, orig[3 * g + 1] = r.oy, orig[3 * g + 2] = r.oz;
        dir[3 * g] = r.dx, dir[3 * g + 1] = r.dy, dir[3 * g + 2] = r.dz;
    }
}

inline int grid_for(int64_t n, int threads = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

}  // namespace

void launch_cast_spinning(const SceneView &sv, const SpinParams &p, const float *poses, int64_t P, const CastOut &o,
                          CastCounter *ctr, cudaStream_t s) {
    SpinGen g;
    g.sp = p;
    g.poses = poses;
    g.tc = p.channels >= 4 ? 4 : (p.channels >= 2 ? 2 : 1);
    g.ta = 32 / g.tc;
    g.nct = (p.channels + g.tc - 1) / g.tc;
    g.nat = (p.columns + g.ta - 1) / g.ta;
    launch_persistent(sv, g, P * (int64_t)g.nct * g.nat, o, ctr, s);
}

void launch_cast_rosette(const SceneView &sv, const RosetteParams &p, const float *poses, int64_t P,
                         const CastOut &o, CastCounter *ctr, cudaStream_t s) {
    RosetteGen g;
    g.rp = p;
    g.poses = poses;
    g.ntile = (p.n + 31) / 32;
    launch_persistent(sv, g, P * (int64_t)g.ntile, o, ctr, s);
}

void launch_cast_rays(const SceneView &sv, const float *orig, const float *dir, int64_t R, float t_min, float t_max,
                      const CastOut &o, CastCounter *ctr, cudaStream_t s) {
    RaysGen g{orig, dir, R, t_min, t_max};
    launch_persistent(sv, g, (R + 31) / 32, o, ctr, s);
}

void launch_cast_bruteforce(const float *verts, const int32_t *tris, int64_t T, const float *orig, const float *dir,
                            int64_t R, float t_min, float t_max, float *range, int32_t *tri_id, cudaStream_t s) {
    if (R <= 0) return;
    k_bruteforce<<<(unsigned)((R + kBfThreads - 1) / kBfThreads), kBfThreads, 0, s>>>(verts, tris, T, orig, dir, R,
                                                                                       t_min, t_max, range, tri_id);
    FGL_LAUNCHED("k_bruteforce");
}

void launch_export_spinning(const SpinParams &p, const float *poses, int64_t P, float *orig, float *dir,
                            cudaStream_t s) {
    const int64_t n = P * p.channels * (int64_t)p.columns;
    if (n <= 0) return;
    k_export_spin<<<grid_for(n), 256, 0, s>>>(p, poses, n, orig, dir);
    FGL_LAUNCHED("k_export_spin");
}

void launch_export_rosette(const RosetteParams &p, const float *poses, int64_t P, float *orig, float *dir,
                           cudaStream_t s) {
    const int64_t n = P * (int64_t)p.n;
    if (n <= 0) return;
    k_export_rosette<<<grid_for(n), 256, 0, s>>>(p, poses, n, orig, dir);
    FGL_LAUNCHED("k_export_rosette");
}

}  // namespace fgl
