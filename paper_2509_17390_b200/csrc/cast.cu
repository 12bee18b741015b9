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
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "fgl_internal.cuh"

namespace fgl {

namespace {

#ifndef FGL_APPROX_PRE
#define FGL_APPROX_PRE 1  // MUFU reciprocals for the per-ray slab / shear constants
#endif
#ifndef FGL_APPROX_NORM
#define FGL_APPROX_NORM 1  // MUFU rsqrt for the direction normalisation (0: exact sqrt + division); the
                           // same in the cast and the ray export; measured max direction error 2^-21.1
                           // either way (tools/raygen_err.py), +1% cast
#endif

#ifndef FGL_LEAF_RCP
#define FGL_LEAF_RCP 1  // leaf test: t = T * rcp(det) instead of the IEEE division (R15)
#endif

#ifndef FGL_CAST_THREADS
#define FGL_CAST_THREADS 128
#endif
constexpr int kCastThreads = FGL_CAST_THREADS;
constexpr int kStack = 96;                   // > max depth of a Karras tree over 63-bit keys + index
constexpr float kExpand = 1.0f + 0x1p-20f;   // conservative slab test: tfar * (1 + 2 gamma_3) (Ize 2013)

struct Ray {
    float ox, oy, oz, dx, dy, dz;
};

// Per-ray constants.
//  * slab test (robust, one FMA per plane): t = fma(x, I, c) with I = 1/d, c = -o I. The rounding
//    of c and of the FMA is bounded by 2u|t| + u|c| (u = 2^-24); the |c| part is folded into two
//    per-axis offsets (clo for the lo plane, chi for the hi plane, pushed outward by 2^-22 |c|)
//    and the relative part into the 1 + 2^-20 factor on t_far. Conservative: never culls a box the
//    exact ray touches.
//  * watertight test (Woop, Benthin, Wald 2013): kz = argmax |d|, shear S; the axis permutation is
//    a cyclic rotation of the coordinates chosen by selects (branch-free); each sheared coordinate
//    carries at most two roundings, identical for a vertex shared by two triangles (watertightness).
struct Pre {
    float ox, oy, oz;
    float Ix, Iy, Iz;
    float clx, chx, cly, chy, clz, chz;
    float Sx, Sy, Sz;  // shear: S_x = d_kx / d_kz, S_y = d_ky / d_kz, S_z = 1 / d_kz
    int kz;            // argmax |d_a|; the shear axes are kx = kz + 1, ky = kz + 2 (mod 3)
};

// 1/x by MUFU.RCP (rcp.approx.ftz.f32, <= 1 ulp); |x| >= 2^-80 here, so no denormal is flushed
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ Pre precompute(const Ray &r) {
    Pre p;
    p.ox = r.ox, p.oy = r.oy, p.oz = r.oz;
    const float tiny = 0x1p-80f;
    const float dx = fabsf(r.dx) < tiny ? copysignf(tiny, r.dx) : r.dx;
    const float dy = fabsf(r.dy) < tiny ? copysignf(tiny, r.dy) : r.dy;
    const float dz = fabsf(r.dz) < tiny ? copysignf(tiny, r.dz) : r.dz;
#if FGL_APPROX_PRE
    // MUFU reciprocals (<= 2 ulp): covered by the slab slack, consistent per ray;
    // the shear S is likewise only required to be consistent per ray (watertightness)
    p.Ix = rcp_approx(dx), p.Iy = rcp_approx(dy), p.Iz = rcp_approx(dz);
#else
    p.Ix = __frcp_rn(dx), p.Iy = __frcp_rn(dy), p.Iz = __frcp_rn(dz);
#endif
    const float cx = -r.ox * p.Ix, cy = -r.oy * p.Iy, cz = -r.oz * p.Iz;
    const float ax = fabsf(cx) * 0x1p-22f, ay = fabsf(cy) * 0x1p-22f, az = fabsf(cz) * 0x1p-22f;
    // lo plane is the near plane when I >= 0: push it towards smaller t; the hi plane the other way
    p.clx = p.Ix >= 0.f ? cx - ax : cx + ax, p.chx = p.Ix >= 0.f ? cx + ax : cx - ax;
    p.cly = p.Iy >= 0.f ? cy - ay : cy + ay, p.chy = p.Iy >= 0.f ? cy + ay : cy - ay;
    p.clz = p.Iz >= 0.f ? cz - az : cz + az, p.chz = p.Iz >= 0.f ? cz + az : cz - az;
    const float fx = fabsf(r.dx), fy = fabsf(r.dy), fz = fabsf(r.dz);
    const int kz = (fx >= fy) ? (fx >= fz ? 0 : 2) : (fy >= fz ? 1 : 2);
    // no kx/ky swap for d_kz < 0: it only orients the winding (see shear), the test is two-sided
    const int kx = kz == 2 ? 0 : kz + 1;
    const int ky = kx == 2 ? 0 : kx + 1;
    const float dkz = kz == 0 ? r.dx : (kz == 1 ? r.dy : r.dz);
    const float dkx = kx == 0 ? r.dx : (kx == 1 ? r.dy : r.dz);
    const float dky = ky == 0 ? r.dx : (ky == 1 ? r.dy : r.dz);
#if FGL_APPROX_PRE
    const float Sz = rcp_approx(dkz), Sx = dkx * Sz, Sy = dky * Sz;
#else
    const float Sx = __fdiv_rn(dkx, dkz), Sy = __fdiv_rn(dky, dkz), Sz = __frcp_rn(dkz);
#endif
    p.Sx = Sx, p.Sy = Sy, p.Sz = Sz;
    p.kz = kz;
    return p;
}

// Per-ray constants of the persistent cast (k_cast_dyn). The slab planes are evaluated as
// t = fma(x, I, c) like precompute's, but every error term is covered by an absolute push of the
// plane constants instead of the relative factor on t_far. With I = 1/d (1 + e), |e| <= 2^-23
// (MUFU), c = -o I (1 + e_c), |e_c| <= 2^-24, and one rounding in the fma, a plane at exact distance
// t is computed within 2^-23 |t| + 2^-24 |c| + 2^-24 |t| < 2^-22.4 |t| + 2^-24 |c|. Only planes with
// |t| <= t_max can decide a box test against [t_min, t*] (a near plane further behind the origin
// stays below t_min, a far plane beyond t_max stays above t*), so pushing the near-plane constant
// down and the far-plane constant up by S = 2^-21 (t_max + |c|) (a margin that also covers the
// rounding of S and of c -/+ S) makes every relevant near-plane t a lower bound and every far-plane
// t an upper bound of the exact one: the box test needs no factor on t_far, and a stacked entry
// distance is a lower bound of the exact entry, so culling it when it exceeds t* is exact (P:279
// "exceeds"). S is 2^-21 of the ray's reach: ~0.1 mm at t_max = 200 m, far below any box.
// (tmax here is the reach R >= every |t| that can decide a test: t_max, or a bound on the distance
// to the farthest point of the scene when t_max is infinite.)
__device__ __forceinline__ Pre precompute_dyn(const Ray &r, float tmax) {
    Pre p = precompute(r);
    const float cx = -r.ox * p.Ix, cy = -r.oy * p.Iy, cz = -r.oz * p.Iz;
    const float sx = (tmax + fabsf(cx)) * 0x1p-21f;
    const float sy = (tmax + fabsf(cy)) * 0x1p-21f;
    const float sz = (tmax + fabsf(cz)) * 0x1p-21f;
    // lo plane is the near plane when I >= 0
    p.clx = p.Ix >= 0.f ? cx - sx : cx + sx, p.chx = p.Ix >= 0.f ? cx + sx : cx - sx;
    p.cly = p.Iy >= 0.f ? cy - sy : cy + sy, p.chy = p.Iy >= 0.f ? cy + sy : cy - sy;
    p.clz = p.Iz >= 0.f ? cz - sz : cz + sz, p.chz = p.Iz >= 0.f ? cz + sz : cz - sz;
    return p;
}

struct V3 {
    float x, y, z;
};

// Sheared coordinates of a vertex relative to the ray origin: (A_kx - Sx A_kz, A_ky - Sy A_kz, Sz A_kz)
// with A = v - o (two roundings per coordinate, the same for every triangle sharing the vertex).
#ifndef FGL_FFMA2
#define FGL_FFMA2 1  // paired FP32 math (FFMA2 / FMUL2 / FADD2, sm_100): slab planes, shear, edge products
#endif
// (fma(lo, I, c_lo), fma(hi, I, c_hi)) — the two planes of one axis in one FFMA2 (fma.rn.f32x2: two
// independent round-to-nearest fmas, bit-identical to two fmaf; I broadcast). The node's lo / hi
// of an axis are adjacent floats (node64 layout), and so are the ray's constants (Pre).
__device__ __forceinline__ void plane_pair(float lo, float hi, float I, float clo, float chi, float &tlo, float &thi) {
#if FGL_FFMA2
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(tlo), "=f"(thi)
        : "f"(lo), "f"(hi), "f"(I), "f"(clo), "f"(chi));
#else
    tlo = fmaf(lo, I, clo), thi = fmaf(hi, I, chi);
#endif
}

// (a0 * b0, a1 * b1) and (a0 + b0, a1 + b1), each lane of the pair rounded to nearest (FMUL2 /
// FADD2: bit-identical to two __fmul_rn / __fadd_rn, never contracted)
#ifndef FGL_PAIR_LEAF
#define FGL_PAIR_LEAF 0  // 1: FMUL2 / FADD2 in the leaf test too (measured -4.6%: the pairs force spills at 48 registers)
#endif
__device__ __forceinline__ void mul_pair(float a0, float a1, float b0, float b1, float &r0, float &r1) {
#if FGL_FFMA2 && FGL_PAIR_LEAF
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
#else
    r0 = __fmul_rn(a0, b0), r1 = __fmul_rn(a1, b1);
#endif
}
__device__ __forceinline__ void sub_pair(float a0, float a1, float b0, float b1, float &r0, float &r1) {
#if FGL_FFMA2 && FGL_PAIR_LEAF
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
#else
    r0 = __fsub_rn(a0, b0), r1 = __fsub_rn(a1, b1);
#endif
}

__device__ __forceinline__ V3 shear(const Pre &p, float4 v) {
    float X, Y;
    sub_pair(v.x, v.y, p.ox, p.oy, X, Y);
    const float Z = v.z - p.oz;
    // (A_kx, A_ky, A_kz) is the cyclic rotation of (X, Y, Z) that ends on kz, by branch-free selects.
    // The swap of kx and ky for d_kz < 0 in Woop et al. only orients the winding: it negates U, V, W,
    // T and det exactly (IEEE negation is exact), so a two-sided test returns the same t without it.
    const bool r0 = p.kz == 0, r1 = p.kz == 1;
    const float Ax = r0 ? Y : (r1 ? Z : X);
    const float Ay = r0 ? Z : (r1 ? X : Y);
    const float Az = r0 ? X : (r1 ? Y : Z);
    return V3{fmaf(-p.Sx, Az, Ax), fmaf(-p.Sy, Az, Ay), p.Sz * Az};
}

// Watertight ray/triangle test (two-sided, inclusive edges). Edge functions are evaluated without
// FMA contraction so that the two triangles of a shared edge see exactly opposite values; an
// exactly-zero edge function is re-evaluated in double (float products are exact there).
// Returns true and t when t is in [tmin, best_t] and (t, id) beats (best_t, best_id).
__device__ __forceinline__ bool hit_tri(const Pre &p, float4 a, float4 b, float4 c, float tmin, float best_t,
                                        int32_t best_id, int32_t id, float &t_out) {
    const V3 A = shear(p, a), B = shear(p, b), C = shear(p, c);
    float u0, u1, v0, v1, w0, w1;
    mul_pair(C.x, C.y, B.y, B.x, u0, u1);
    mul_pair(A.x, A.y, C.y, C.x, v0, v1);
    mul_pair(B.x, B.y, A.y, A.x, w0, w1);
    float U = __fsub_rn(u0, u1);
    float V = __fsub_rn(v0, v1);
    float W = __fsub_rn(w0, w1);
    if ((U < 0.f || V < 0.f || W < 0.f) && (U > 0.f || V > 0.f || W > 0.f)) return false;
    if (U == 0.f || V == 0.f || W == 0.f) {
        const double Ud = (double)C.x * (double)B.y - (double)C.y * (double)B.x;
        const double Vd = (double)A.x * (double)C.y - (double)A.y * (double)C.x;
        const double Wd = (double)B.x * (double)A.y - (double)B.y * (double)A.x;
        if ((Ud < 0.0 || Vd < 0.0 || Wd < 0.0) && (Ud > 0.0 || Vd > 0.0 || Wd > 0.0)) return false;
        U = (float)Ud, V = (float)Vd, W = (float)Wd;
    }
    const float det = U + V + W;
    if (det == 0.f) return false;
    const float T = U * A.z + V * B.z + W * C.z;
#if FGL_LEAF_RCP
    // t = T / det by the MUFU reciprocal (<= 1 ulp) and one rounding: within 2 ulp of the correctly
    // rounded quotient (R15), deterministic, and the same in every kernel that calls hit_tri; a
    // |det| below 2^-100 (where rcp.approx.ftz would flush) takes the IEEE division
    float t = T * rcp_approx(det);
    if (fabsf(det) < 0x1p-100f) t = __fdiv_rn(T, det);
#else
    // cheap conservative reject before the division: t = T/det outside [tmin, best_t] by > 2^-20
    const float ad = fabsf(det), Ts = det < 0.f ? -T : T;
    if (Ts > best_t * ad * (1.f + 0x1p-20f) || Ts < tmin * ad * (1.f - 0x1p-20f)) return false;
    const float t = __fdiv_rn(T, det);
#endif
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

// conservative slab test of one child box against [tmin, tmax]; returns the entry distance or +inf
__device__ __forceinline__ float slab(const Pre &p, float lx, float hx, float ly, float hy, float lz, float hz,
                                      float tmin, float tmax) {
    const float ax = fmaf(lx, p.Ix, p.clx), bx = fmaf(hx, p.Ix, p.chx);
    const float ay = fmaf(ly, p.Iy, p.cly), by = fmaf(hy, p.Iy, p.chy);
    const float az = fmaf(lz, p.Iz, p.clz), bz = fmaf(hz, p.Iz, p.chz);
    const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), tmin));
    const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), tmax));
    return tn <= tf * kExpand ? tn : INFINITY;
}

// the persistent cast's test (constants from precompute_dyn: t_near / t_far are lower / upper
// bounds of the exact plane distances, so no factor on t_far); hit flag and entry distance
// returned separately (no +inf materialisation)
__device__ __forceinline__ bool slab_hit(const Pre &p, float lx, float hx, float ly, float hy, float lz, float hz,
                                         float tmin, float tmax, float &tn_out) {
    float ax, bx, ay, by, az, bz;
    plane_pair(lx, hx, p.Ix, p.clx, p.chx, ax, bx);
    plane_pair(ly, hy, p.Iy, p.cly, p.chy, ay, by);
    plane_pair(lz, hz, p.Iz, p.clz, p.chz, az, bz);
    const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), tmin));
    const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), tmax));
    tn_out = tn;
    return tn <= tf;
}

// Octant-specialised form of slab_hit: when the sign of every I component is known at compile
// time, the near plane of each axis is known (lo iff I >= 0), so the per-axis min/max that orders
// each plane pair disappears: 6 FFMA + 4 FMNMX + 1 FMUL + 1 FSETP per box instead of 6 + 10 + 1 + 1.
// The planes, their constants and the final test are those of slab_hit, so the result is the same
// bit for bit (min/max of the same two values). OCT bit a = (I_a < 0).
template <int OCT>
__device__ __forceinline__ bool slab_oct(const Pre &p, float lx, float hx, float ly, float hy, float lz, float hz,
                                         float tmin, float tmax, float &tn_out) {
    constexpr bool sx = OCT & 1, sy = OCT & 2, sz = OCT & 4;
    float tlx, thx, tly, thy, tlz, thz;
    plane_pair(lx, hx, p.Ix, p.clx, p.chx, tlx, thx);
    plane_pair(ly, hy, p.Iy, p.cly, p.chy, tly, thy);
    plane_pair(lz, hz, p.Iz, p.clz, p.chz, tlz, thz);
    const float nx = sx ? thx : tlx, fx = sx ? tlx : thx;
    const float ny = sy ? thy : tly, fy = sy ? tly : thy;
    const float nz = sz ? thz : tlz, fz = sz ? tlz : thz;
    const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, tmin));
    const float tf = fminf(fminf(fx, fy), fminf(fz, tmax));
    tn_out = tn;
    return tn <= tf;
}

__device__ __forceinline__ int ray_octant(const Pre &p) {
    return (p.Ix < 0.f ? 1 : 0) | (p.Iy < 0.f ? 2 : 0) | (p.Iz < 0.f ? 4 : 0);
}

template <int OCT>
__device__ __forceinline__ bool slab_sel(const Pre &p, float lx, float hx, float ly, float hy, float lz, float hz,
                                         float tmin, float tmax, float &tn_out) {
    if constexpr (OCT < 0)
        return slab_hit(p, lx, hx, ly, hy, lz, hz, tmin, tmax, tn_out);
    else
        return slab_oct<OCT>(p, lx, hx, ly, hy, lz, hz, tmin, tmax, tn_out);
}

constexpr int32_t kDone = INT_MAX;  // "no more work" (never a node index: T - 1 < 2^28)

// Traversal in the "while-while" form of Aila & Laine (HPG 2009): a lane that reaches a leaf
// postpones it and keeps descending internal nodes until every active lane holds a leaf, then the
// warp tests leaves together — leaf tests run with most lanes active instead of a few.
template <bool kCount>
__device__ __forceinline__ Hit trace(const SceneView &sv, const Ray &r, float tmin, float tmax) {
    const Pre p = precompute(r);
    Hit h{tmax, INT_MAX, 0, 0};
    int32_t st_ref[kStack];
    float st_t[kStack];
    int sp = 0;
    int32_t cur = 0;   // next internal node / leaf to visit (root = internal node 0), or kDone
    int32_t leaf = 0;  // postponed leaf (< 0) or none (0)
    auto pop = [&]() -> int32_t {
        while (sp > 0) {
            --sp;
            if (st_t[sp] <= h.t * kExpand) return st_ref[sp];
        }
        return kDone;
    };
    while (true) {
        while (cur >= 0 && cur != kDone) {
            const float4 *np = reinterpret_cast<const float4 *>(sv.nodes + cur);
            const float4 na = __ldg(np), nb = __ldg(np + 1), nc = __ldg(np + 2);
            const int4 nd = __ldg(reinterpret_cast<const int4 *>(np + 3));
            if (kCount) ++h.nodes;
            const float lim = h.t;
            const float t0 = slab(p, na.x, na.y, na.z, na.w, nc.x, nc.y, tmin, lim);
            const float t1 = nd.y == kEmptyRef ? INFINITY : slab(p, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, tmin, lim);
            const bool h0 = t0 != INFINITY, h1 = t1 != INFINITY;
            if (h0 && h1) {
                const bool swap = t1 < t0;
                st_ref[sp] = swap ? nd.x : nd.y;
                st_t[sp] = swap ? t0 : t1;
                ++sp;
                cur = swap ? nd.y : nd.x;
            } else if (h0) {
                cur = nd.x;
            } else if (h1) {
                cur = nd.y;
            } else {
                cur = pop();
            }
            if (cur < 0 && leaf == 0) {
                leaf = cur;
                cur = pop();
            }
            if (!__any_sync(__activemask(), leaf == 0)) break;
        }
        while (leaf < 0) {
            const int32_t v = ~leaf;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 *tp = sv.tri + kTriStride * (int64_t)k;
                const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
                const int32_t id = __float_as_int(a.w);
                if (kCount) ++h.tris;
                float t;
                if (hit_tri(p, a, b, c, tmin, h.t, h.id, id, t)) {
                    h.t = t;
                    h.id = id;
                }
            }
            leaf = 0;
            if (cur < 0) {
                leaf = cur;
                cur = pop();
            }
        }
        if (cur == kDone) break;
    }
    return h;
}

// 4-wide traversal (node128): one fetch brings the four child boxes (SoA, 6 x LDG.128 + refs);
// hit children are sorted by entry distance with a 5-comparator network, the nearest is visited
// next and the others are pushed far-to-near. Same while-while leaf postponing as `trace`.
__device__ __forceinline__ void cswap(float &ta, int32_t &ra, float &tb, int32_t &rb) {
    const bool sw = tb < ta;
    const float t = sw ? tb : ta;
    const int32_t r = sw ? rb : ra;
    tb = sw ? ta : tb;
    rb = sw ? ra : rb;
    ta = t;
    ra = r;
}

template <bool kCount>
__device__ __forceinline__ Hit trace4(const SceneView &sv, const Ray &r, float tmin, float tmax) {
    const Pre p = precompute(r);
    Hit h{tmax, INT_MAX, 0, 0};
    int32_t st_ref[kStack];
    float st_t[kStack];
    int sp = 0;
    int32_t cur = 0;
    int32_t leaf = 0;
    auto pop = [&]() -> int32_t {
        while (sp > 0) {
            --sp;
            if (st_t[sp] <= h.t * kExpand) return st_ref[sp];
        }
        return kDone;
    };
    while (true) {
        while (cur >= 0 && cur != kDone) {
            const float4 *np = reinterpret_cast<const float4 *>(sv.nodes4 + cur);
            const float4 lx = __ldg(np), hx = __ldg(np + 1), ly = __ldg(np + 2), hy = __ldg(np + 3);
            const float4 lz = __ldg(np + 4), hz = __ldg(np + 5);
            const int4 rf = __ldg(reinterpret_cast<const int4 *>(np + 6));
            if (kCount) ++h.nodes;
            const float lim = h.t;
            float t0 = slab(p, lx.x, hx.x, ly.x, hy.x, lz.x, hz.x, tmin, lim);
            float t1 = slab(p, lx.y, hx.y, ly.y, hy.y, lz.y, hz.y, tmin, lim);
            float t2 = slab(p, lx.z, hx.z, ly.z, hy.z, lz.z, hz.z, tmin, lim);
            float t3 = slab(p, lx.w, hx.w, ly.w, hy.w, lz.w, hz.w, tmin, lim);
            int32_t r0 = rf.x, r1 = rf.y, r2 = rf.z, r3 = rf.w;
            cswap(t0, r0, t1, r1);
            cswap(t2, r2, t3, r3);
            cswap(t0, r0, t2, r2);
            cswap(t1, r1, t3, r3);
            cswap(t1, r1, t2, r2);
            if (t3 != INFINITY) st_ref[sp] = r3, st_t[sp] = t3, ++sp;
            if (t2 != INFINITY) st_ref[sp] = r2, st_t[sp] = t2, ++sp;
            if (t1 != INFINITY) st_ref[sp] = r1, st_t[sp] = t1, ++sp;
            cur = t0 != INFINITY ? r0 : pop();
            if (cur < 0 && leaf == 0) {
                leaf = cur;
                cur = pop();
            }
            if (!__any_sync(__activemask(), leaf == 0)) break;
        }
        while (leaf < 0) {
            const int32_t v = ~leaf;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 *tp = sv.tri + kTriStride * (int64_t)k;
                const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
                const int32_t id = __float_as_int(a.w);
                if (kCount) ++h.tris;
                float t;
                if (hit_tri(p, a, b, c, tmin, h.t, h.id, id, t)) {
                    h.t = t;
                    h.id = id;
                }
            }
            leaf = 0;
            if (cur < 0) {
                leaf = cur;
                cur = pop();
            }
        }
        if (cur == kDone) break;
    }
    return h;
}

// 4-wide traversal over 8-bit quantised child boxes (node64q, 4 x LDG.128 per node). A child
// plane x = p + q s is evaluated as t = q (s I) + (p I + c): s I is exact (s a power of two), and the
// per-node offset p I + c is pushed outward by 2^-22 |p I| on top of the per-ray slack, so the test
// stays conservative for the decoded (outward-rounded) box. Bytes become floats with the
// 2^23-mantissa trick (PRMT + FADD).
__device__ __forceinline__ float byte_f(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | (uint32_t)k)) - 8388608.0f;
}

template <bool kCount>
__device__ __forceinline__ Hit trace4q(const SceneView &sv, const Ray &r, float tmin, float tmax) {
    const Pre p = precompute(r);
    Hit h{tmax, INT_MAX, 0, 0};
    int32_t st_ref[kStack];
    float st_t[kStack];
    int sp = 0;
    int32_t cur = 0;
    int32_t leaf = 0;
    const NodeQ *nq = reinterpret_cast<const NodeQ *>(sv.nodes4);
    const float sgx = p.Ix >= 0.f ? 1.f : -1.f, sgy = p.Iy >= 0.f ? 1.f : -1.f, sgz = p.Iz >= 0.f ? 1.f : -1.f;
    auto pop = [&]() -> int32_t {
        while (sp > 0) {
            --sp;
            if (st_t[sp] <= h.t * kExpand) return st_ref[sp];
        }
        return kDone;
    };
    while (true) {
        while (cur >= 0 && cur != kDone) {
            const float4 f0 = __ldg(&nq[cur].f0);
            const int4 q0 = __ldg(&nq[cur].q0), q1 = __ldg(&nq[cur].q1), q2 = __ldg(&nq[cur].q2);
            if (kCount) ++h.nodes;
            const uint32_t bits = __float_as_uint(f0.w);
            const float sx = __uint_as_float((bits & 0xFFu) << 23), sy = __uint_as_float(((bits >> 8) & 0xFFu) << 23);
            const float sz = __uint_as_float(((bits >> 16) & 0xFFu) << 23);
            const uint32_t mask = bits >> 24;
            const float Ax = sx * p.Ix, Ay = sy * p.Iy, Az = sz * p.Iz;
            const float px = f0.x * p.Ix, py = f0.y * p.Iy, pz = f0.z * p.Iz;
            const float ex = fabsf(px) * 0x1p-22f * sgx, ey = fabsf(py) * 0x1p-22f * sgy, ez = fabsf(pz) * 0x1p-22f * sgz;
            const float Blx = fmaf(f0.x, p.Ix, p.clx) - ex, Bhx = fmaf(f0.x, p.Ix, p.chx) + ex;
            const float Bly = fmaf(f0.y, p.Iy, p.cly) - ey, Bhy = fmaf(f0.y, p.Iy, p.chy) + ey;
            const float Blz = fmaf(f0.z, p.Iz, p.clz) - ez, Bhz = fmaf(f0.z, p.Iz, p.chz) + ez;
            const float lim = h.t;
            float t[4];
            int32_t rf[4] = {q1.z, q1.w, q2.x, q2.y};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float ax = fmaf(byte_f((uint32_t)q0.x, k), Ax, Blx), bx = fmaf(byte_f((uint32_t)q0.y, k), Ax, Bhx);
                const float ay = fmaf(byte_f((uint32_t)q0.z, k), Ay, Bly), by = fmaf(byte_f((uint32_t)q0.w, k), Ay, Bhy);
                const float az = fmaf(byte_f((uint32_t)q1.x, k), Az, Blz), bz = fmaf(byte_f((uint32_t)q1.y, k), Az, Bhz);
                const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), tmin));
                const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), lim));
                t[k] = ((mask >> k) & 1u) && tn <= tf * kExpand ? tn : INFINITY;
            }
            cswap(t[0], rf[0], t[1], rf[1]);
            cswap(t[2], rf[2], t[3], rf[3]);
            cswap(t[0], rf[0], t[2], rf[2]);
            cswap(t[1], rf[1], t[3], rf[3]);
            cswap(t[1], rf[1], t[2], rf[2]);
            if (t[3] != INFINITY) st_ref[sp] = rf[3], st_t[sp] = t[3], ++sp;
            if (t[2] != INFINITY) st_ref[sp] = rf[2], st_t[sp] = t[2], ++sp;
            if (t[1] != INFINITY) st_ref[sp] = rf[1], st_t[sp] = t[1], ++sp;
            cur = t[0] != INFINITY ? rf[0] : pop();
            if (cur < 0 && leaf == 0) {
                leaf = cur;
                cur = pop();
            }
            if (!__any_sync(__activemask(), leaf == 0)) break;
        }
        while (leaf < 0) {
            const int32_t v = ~leaf;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 *tp = sv.tri + kTriStride * (int64_t)k;
                const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
                const int32_t id = __float_as_int(a.w);
                if (kCount) ++h.tris;
                float tt;
                if (hit_tri(p, a, b, c, tmin, h.t, h.id, id, tt)) {
                    h.t = tt;
                    h.id = id;
                }
            }
            leaf = 0;
            if (cur < 0) {
                leaf = cur;
                cur = pop();
            }
        }
        if (cur == kDone) break;
    }
    return h;
}

// Packet traversal for coherent pattern tiles (all 32 rays of a warp share the pose origin and
// span ~1.5 degrees): the warp walks ONE node sequence — it descends into a child if any lane's ray
// enters it within that lane's [t_min, t*] — so every node and triangle fetch is a broadcast and
// control never diverges. Children are ordered by a lane vote on which is nearer; a popped subtree
// is skipped when no lane can still improve inside it (per-lane entry distances are kept on the
// stack). Each lane still keeps its own (t*, id) with the same leaf test, so results are identical
// to the per-ray traversal.
template <bool kCount>
__device__ __forceinline__ Hit trace_packet(const SceneView &sv, const Ray &r, float tmin, float tmax,
                                            int32_t *__restrict__ sref) {
    const Pre p = precompute(r);
    Hit h{tmax, INT_MAX, 0, 0};
    float st_t[kStack];
    int sp = 0;
    int32_t cur = 0;
    constexpr unsigned kFull = 0xffffffffu;
    while (true) {
        if (cur >= 0) {
            const float4 *np = reinterpret_cast<const float4 *>(sv.nodes + cur);
            const float4 na = __ldg(np), nb = __ldg(np + 1), nc = __ldg(np + 2);
            const int4 nd = __ldg(reinterpret_cast<const int4 *>(np + 3));
            if (kCount) ++h.nodes;
            const float lim = h.t;
            const float t0 = slab(p, na.x, na.y, na.z, na.w, nc.x, nc.y, tmin, lim);
            const float t1 = nd.y == kEmptyRef ? INFINITY : slab(p, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, tmin, lim);
            const unsigned m0 = __ballot_sync(kFull, t0 != INFINITY), m1 = __ballot_sync(kFull, t1 != INFINITY);
            if (m0 && m1) {
                const unsigned v1 = __ballot_sync(kFull, t1 < t0), v0 = __ballot_sync(kFull, t0 < t1);
                const bool first1 = __popc(v1) > __popc(v0);
                sref[sp] = first1 ? nd.x : nd.y;  // same value from every lane
                st_t[sp] = first1 ? t0 : t1;
                ++sp;
                cur = first1 ? nd.y : nd.x;
                continue;
            }
            if (m0) {
                cur = nd.x;
                continue;
            }
            if (m1) {
                cur = nd.y;
                continue;
            }
        } else {
            const int32_t v = ~cur;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 *tp = sv.tri + kTriStride * (int64_t)k;
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
        cur = kDone;
        while (sp > 0) {
            --sp;
            if (__any_sync(kFull, st_t[sp] <= h.t * kExpand)) {
                cur = sref[sp];
                break;
            }
        }
        if (cur == kDone) break;
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
    // fused all-gather: the same result into every peer's global output (P2P stores over NVLink)
    for (int w = 0; w < o.npeer; ++w) {
        o.peer_range[w][o.out_offset + idx] = miss ? INFINITY : h.t;
        o.peer_tri[w][o.out_offset + idx] = miss ? -1 : h.id;
    }
}

// Kernel epilogue: the last warp to finish resets the work counter for the next launch using this
// slot; with a fused all-gather it also signals every rank (own flag included) after a system-scope
// fence by every warp, so a rank waiting for W signals knows all peers' stores into its buffer landed.
__device__ __forceinline__ void cast_epilogue(const CastOut &out, CastCounter *ctr, int lane) {
    // every lane fences its own peer stores at system scope (a fence orders only the calling thread's
    // accesses), then the warp reconverges before lane 0 counts the warp as done
    if (out.nsignal) __threadfence_system();
    __syncwarp();
    if (lane == 0) {
        const unsigned int total = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(&ctr->done, 1u) == total - 1) {
            ctr->next = 0ull;
            ctr->done = 0u;
            __threadfence();
            if (out.nsignal) {
                __threadfence_system();
                for (int w = 0; w < out.nsignal; ++w) atomicAdd_system(out.signal[w], 1);
            }
        }
    }
}

// ---- ray generators ---------------------------------------------------------------------------
__device__ __forceinline__ void rotate_pose(const float *__restrict__ pose, float sx, float sy, float sz, Ray &r) {
    const float4 r0 = __ldg(reinterpret_cast<const float4 *>(pose));
    const float4 r1 = __ldg(reinterpret_cast<const float4 *>(pose) + 1);
    const float4 r2 = __ldg(reinterpret_cast<const float4 *>(pose) + 2);
    float dx = r0.x * sx + r0.y * sy + r0.z * sz;
    float dy = r1.x * sx + r1.y * sy + r1.z * sz;
    float dz = r2.x * sx + r2.y * sy + r2.z * sz;
#if FGL_APPROX_NORM
    const float rn = rsqrtf(dx * dx + dy * dy + dz * dz);  // MUFU.RSQ (<= 2 ulp), same in cast and export
    r.dx = dx * rn, r.dy = dy * rn, r.dz = dz * rn;
#else
    const float n = sqrtf(dx * dx + dy * dy + dz * dz);
    r.dx = __fdiv_rn(dx, n), r.dy = __fdiv_rn(dy, n), r.dz = __fdiv_rn(dz, n);
#endif
    r.ox = r0.w, r.oy = r1.w, r.oz = r2.w;
}

// spinning beam (c, a): d_s = (cos e cos th, cos e sin th, sin e), th = 2 pi a / A + az0 (R11, R12).
// (sin, cos) of the elevation of channel c and of the azimuth of column a; k_spin_table evaluates
// them once per call into a [C + A] table, so the per-ray generator only rotates and normalises.
__device__ __forceinline__ float2 spin_elev_sc(const SpinParams &sp, int c) {
    float s, co;
    sincospif(__fdiv_rn(sp.elev_deg[c], 180.f), &s, &co);
    return make_float2(s, co);
}
__device__ __forceinline__ float2 spin_az_sc(const SpinParams &sp, int a) {
    float s, co;
    sincospif(__fadd_rn(__fdiv_rn(2.f * (float)a, (float)sp.columns), __fdiv_rn(sp.az0_deg, 180.f)), &s, &co);
    return make_float2(s, co);
}
__device__ __forceinline__ void spin_ray_tab(const float2 *__restrict__ tab, int C, const float *__restrict__ poses,
                                             int64_t p, int c, int a, Ray &r) {
    const float2 e = __ldg(tab + c), z = __ldg(tab + C + a);
    rotate_pose(poses + 12 * p, e.y * z.y, e.y * z.x, e.x, r);
}

// 32-bit division by a launch-invariant divisor (Granlund & Montgomery 1994): for n < 2^31 and
// d >= 2, s = ceil(log2 d), m = ceil(2^(31+s) / d) < 2^32, n / d = umulhi(n, m) >> (s - 1).
struct FastDiv {
    uint32_t d, m, sh;  // sh = s - 1; d = 1 is m = 0 (quotient n)
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{d, 0u, 0u};
    if (d <= 1) return f;
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.m = (uint32_t)(((1ull << (31 + s)) + d - 1) / d);
    f.sh = s - 1;
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    return f.m ? __umulhi(n, f.m) >> f.sh : n;
}

// (sin, cos) of the angle 2 pi ph / 2^32 of an exact 32-bit phase, without rounding the phase to
// float's 24 bits: the top 24 bits are an exact sincospif argument, (ph >> 8) 2^-23 half-turns; the
// low 8 bits (an angle b < 2 pi 2^-24 = 3.8e-7 rad) rotate that result to first order (the dropped
// b^2 / 2 < 7.2e-14 is far below float's resolution).
__device__ __forceinline__ void sincos_phase(uint32_t ph, float &s, float &c) {
    float sc, cc;
    sincospif((float)(ph >> 8) * 0x1p-23f, &sc, &cc);
    const float b = (float)(ph & 0xFFu) * 1.4629180792671596e-09f;  // 2 pi / 2^32
    s = fmaf(cc, b, sc);
    c = fmaf(-sc, b, cc);
}

// rosette sample n of pose p (R20): exact 32-bit phases, two counter-rotating prisms
__device__ __forceinline__ void rosette_ray(const RosetteParams &rp, const float *__restrict__ poses, int64_t p, int k,
                                            Ray &r) {
    const uint64_t n = (uint64_t)(rp.first_frame + p) * (uint64_t)rp.n + (uint64_t)k;
    const uint32_t ph1 = (uint32_t)(n * (uint64_t)rp.inc1);
    const uint32_t ph2 = rp.phase2_0 - (uint32_t)(n * (uint64_t)rp.inc2);
    float s1, c1, s2, c2;
    sincos_phase(ph1, s1, c1);
    sincos_phase(ph2, s2, c2);
    const float half = 0.5f * rp.half_fov_deg * 0.017453292519943295f;
    const float dx = half * (c1 + c2), dy = half * (s1 + s2);
    const float rho = sqrtf(dx * dx + dy * dy);
    float sr, cr;
    sincosf(rho, &sr, &cr);
    const float s = rho > 0.f ? __fdiv_rn(sr, rho) : 1.f;
    rotate_pose(poses + 12 * p, cr, dx * s, dy * s, r);
}

struct SpinGen {
    static constexpr bool kCoherent = true;
    SpinParams sp;
    const float *poses;
    const float2 *tab;     // k_spin_table: [C] elevation (sin, cos), then [A] azimuth (sin, cos)
    int tc, ta, lta;       // tile shape (tc x ta = 32, ta = 2^lta)
    FastDiv per, nat;      // tiles per pose, column tiles per channel tile
    __device__ __forceinline__ bool ray(int64_t tile, int lane, Ray &r, int64_t &idx, float &tmin, float &tmax) const {
        const uint32_t t = (uint32_t)tile;  // < 2^31 (checked at launch)
        const uint32_t p = fdiv(t, per);
        const uint32_t rem = t - p * per.d;
        const uint32_t cb = fdiv(rem, nat), ab = rem - cb * nat.d;
        const int c = (int)cb * tc + (lane >> lta), a = (int)ab * ta + (lane & (ta - 1));
        tmin = sp.t_min, tmax = sp.t_max;
        if (c >= sp.channels || a >= sp.columns) return false;
        spin_ray_tab(tab, sp.channels, poses, p, c, a, r);
        idx = ((int64_t)p * sp.channels + c) * (int64_t)sp.columns + a;
        return true;
    }
    // the same ray / output slot without the index (k_cast_dyn recomputes the index at the write)
    __device__ __forceinline__ bool ray_at(int64_t tile, int lane, Ray &r) const {
        int64_t idx;
        float a, b;
        return ray(tile, lane, r, idx, a, b);
    }
    __device__ __forceinline__ int64_t index(int64_t tile, int lane) const {
        const uint32_t t = (uint32_t)tile;
        const uint32_t p = fdiv(t, per);
        const uint32_t rem = t - p * per.d;
        const uint32_t cb = fdiv(rem, nat), ab = rem - cb * nat.d;
        const int c = (int)cb * tc + (lane >> lta), a = (int)ab * ta + (lane & (ta - 1));
        return ((int64_t)p * sp.channels + c) * (int64_t)sp.columns + a;
    }
    __device__ __forceinline__ float interval_min() const { return sp.t_min; }
    __device__ __forceinline__ float interval_max() const { return sp.t_max; }
};

struct RosetteGen {
    static constexpr bool kCoherent = true;
    RosetteParams rp;
    const float *poses;
    int ntile;      // tiles per pose
    FastDiv ntile_d;  // the same, as a multiply-shift divisor (tile < 2^31, checked at launch)
    __device__ __forceinline__ bool ray(int64_t tile, int lane, Ray &r, int64_t &idx, float &tmin, float &tmax) const {
        const int64_t p = fdiv((uint32_t)tile, ntile_d);
        const int k = (int)(tile - p * ntile) * 32 + lane;
        tmin = rp.t_min, tmax = rp.t_max;
        if (k >= rp.n) return false;
        rosette_ray(rp, poses, p, k, r);
        idx = p * rp.n + k;
        return true;
    }
    __device__ __forceinline__ bool ray_at(int64_t tile, int lane, Ray &r) const {
        int64_t idx;
        float a, b;
        return ray(tile, lane, r, idx, a, b);
    }
    __device__ __forceinline__ int64_t index(int64_t tile, int lane) const {
        const int64_t p = fdiv((uint32_t)tile, ntile_d);
        return p * rp.n + (int)(tile - p * ntile) * 32 + lane;
    }
    __device__ __forceinline__ float interval_min() const { return rp.t_min; }
    __device__ __forceinline__ float interval_max() const { return rp.t_max; }
};

struct RaysGen {
    static constexpr bool kCoherent = false;
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
    __device__ __forceinline__ bool ray_at(int64_t tile, int lane, Ray &r) const {
        int64_t idx;
        float a, b;
        return ray(tile, lane, r, idx, a, b);
    }
    __device__ __forceinline__ int64_t index(int64_t tile, int lane) const { return tile * 32 + lane; }
    __device__ __forceinline__ float interval_min() const { return t_min; }
    __device__ __forceinline__ float interval_max() const { return t_max; }
};

#ifndef FGL_SPECULATE
#define FGL_SPECULATE 1  // while-while: keep descending after a postponed leaf until all lanes hold one
#endif
#ifndef FGL_BRANCHFREE_PUSH
#define FGL_BRANCHFREE_PUSH 0
#endif
#ifndef FGL_CAST_MINBLOCKS
#define FGL_CAST_MINBLOCKS 8
#endif
#ifndef FGL_DYN_MINBLOCKS
#define FGL_DYN_MINBLOCKS 10  // k_cast_dyn: 10 CTAs x 4 warps per SM (48 registers; measured best)
#endif
enum TraversalMode { kRay2 = 0, kPacket2 = 1, kRay4 = 2, kRay4Q = 3, kRay8Q = 4 };

template <class Gen, bool kCount, int kMode>
__global__ void __launch_bounds__(kCastThreads, FGL_CAST_MINBLOCKS)
    k_cast(const SceneView sv, const Gen gen, int64_t ntiles, const CastOut out, CastCounter *ctr) {
    const int lane = threadIdx.x & 31;
    __shared__ int32_t sref_all[kMode == kPacket2 ? kCastThreads / 32 : 1][kMode == kPacket2 ? kStack : 1];
    int32_t *sref = sref_all[kMode == kPacket2 ? threadIdx.x >> 5 : 0];
    while (true) {
        unsigned long long tile = 0;
        if (lane == 0) tile = atomicAdd(&ctr->next, 1ull);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= (unsigned long long)ntiles) break;
        Ray r;
        int64_t idx;
        float tmin, tmax;
        const bool valid = gen.ray((int64_t)tile, lane, r, idx, tmin, tmax);
        if (kMode == kPacket2) {
            if (!valid) {  // a ragged-tile lane rides along with an empty interval
                r = Ray{0.f, 0.f, 0.f, 1.f, 0.f, 0.f};
                tmin = 0.f, tmax = -1.f;
            }
            Hit h = trace_packet<kCount>(sv, r, tmin, tmax, sref);
            if (valid) write_out(out, idx, r, h);
        } else if (valid) {
            Hit h = kMode == kRay4Q ? trace4q<kCount>(sv, r, tmin, tmax)
                    : kMode == kRay4 ? trace4<kCount>(sv, r, tmin, tmax)
                                     : trace<kCount>(sv, r, tmin, tmax);
            write_out(out, idx, r, h);
        }
    }
    // self-reset: the last warp to finish clears the counter for the next launch using this slot
    cast_epilogue(out, ctr, lane);
}

// FGL_TRAVERSAL=packet selects the warp-packet traversal for pattern casts (A/B experiments;
// the default per-ray while-while traversal is faster on the measured workloads).
inline bool packet_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("FGL_TRAVERSAL");
        v = (e && strcmp(e, "packet") == 0) ? 1 : 0;
    }
    return v == 1;
}

#ifndef FGL_CARVEOUT
#define FGL_CARVEOUT 10  // k_cast_dyn shared-memory carveout in percent (-1: driver default); 5-14 measured equal
#endif
#ifndef FGL_DESCEND_UNROLL
#define FGL_DESCEND_UNROLL 2  // node visits between two speculation votes (2: +0.5% over 1 with the
                              // round-2 kernel; the loop form schedules better than a plain body)
#endif
#ifndef FGL_LDG256
#define FGL_LDG256 1
#endif
// One node64 (64 B, 64-B aligned) in two 256-bit loads (sm_100 LDG.E.ENL2.256) instead of four
// 128-bit ones: two fewer load instructions per node visit.
__device__ __forceinline__ void ldg_node(const Node64 *__restrict__ n, float4 &a, float4 &b, float4 &c, float4 &d) {
#if FGL_LDG256
    const float *q = reinterpret_cast<const float *>(n);
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(q));
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w), "=f"(d.x), "=f"(d.y), "=f"(d.z), "=f"(d.w)
        : "l"(q + 8));
#else
    const float4 *np = reinterpret_cast<const float4 *>(n);
    a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2), d = __ldg(np + 3);
#endif
}

#ifndef FGL_SSTACK
#define FGL_SSTACK 0  // traversal-stack entries per lane held in shared memory (0: all in local memory)
#endif
constexpr int kSStack = FGL_SSTACK;
// Per-lane traversal stack of (entry t bits << 32 | node ref) words. The first kSStack entries live
// in shared memory, one column per thread (entry i of thread x at [i][x]: lanes at different depths
// still hit distinct banks), deeper entries in local memory. A local-memory stack costs one 32-B L1
// sector per lane and access when the lanes' depths differ (1.9 useful bytes per sector measured)
// and its lines crowd the nodes and triangles out of L1; the shared part avoids both.
#ifndef FGL_STACK_CACHE
#define FGL_STACK_CACHE 0  // 1 / 2: the top 1 / 2 entries in registers, spilled and refilled lazily
                           // (measured -16% / -34% on C2: branches + spills at 48 registers; off)
#endif
template <int kCap>
struct LaneStackN {
    uint64_t *sh;                                    // &s_stack[0][threadIdx.x]
    uint64_t loc[kCap - kSStack > 0 ? kCap - kSStack : 1];
#if FGL_STACK_CACHE
    // entries: loc[0, spl) then the register cache (sp - spl <= FGL_STACK_CACHE of them, top0 on top):
    // a push spills only when the cache is full, a pop loads only when it is empty
    uint64_t top0 = 0, top1 = 0;
    int spl = 0;
    __device__ __forceinline__ void push(int &sp, uint64_t e) {
        if (sp - spl == FGL_STACK_CACHE) loc[spl++] = FGL_STACK_CACHE == 2 ? top1 : top0;
        if (FGL_STACK_CACHE == 2) top1 = top0;
        top0 = e;
        ++sp;
    }
    __device__ __forceinline__ uint64_t pop(int &sp) {
        uint64_t e;
        if (sp > spl) {
            e = top0;
            if (FGL_STACK_CACHE == 2) top0 = top1;
        } else {
            e = loc[--spl];
        }
        --sp;
        return e;
    }
#else
    __device__ __forceinline__ void push(int &sp, uint64_t e) {
        if (kSStack > 0 && sp < kSStack)
            sh[sp * kCastThreads] = e;
        else
            loc[sp - kSStack] = e;
        ++sp;
    }
    __device__ __forceinline__ uint64_t pop(int &sp) {
        --sp;
        return (kSStack > 0 && sp < kSStack) ? sh[sp * kCastThreads] : loc[sp - kSStack];
    }
#endif
};

#ifndef FGL_FLAT_VISIT
#define FGL_FLAT_VISIT 0  // 1: branch-light node visit (selects, idle lanes re-read the root)
#endif
#ifndef FGL_LEAF_HANDOFF
#define FGL_LEAF_HANDOFF 0  // 1: both children hit, near one a leaf: postpone it, descend the far one (no stack op)
#endif
#ifndef FGL_PREFETCH
#define FGL_PREFETCH 0  // 1: L1-prefetch the children nodes at each visit; 2: also the leaves' first triangle
#endif
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

using LaneStack = LaneStackN<kStack>;
// width 8: every hit child is pushed; the build bounds the depth this needs (k_collapse) and the
// cast refuses a tree that would exceed it (fgl_scene_check reports it)
constexpr int kStack8 = 192;
using LaneStack8 = LaneStackN<kStack8>;

// Pop the nearest stacked subtree that can still hold a hit (entry t <= t* (1 + 2^-20)).
template <class Stack>
__device__ __forceinline__ int32_t pop_live(Stack &st, int &sp, float tlim) {
    while (sp > 0) {
        const uint64_t e = st.pop(sp);
        if (__uint_as_float((uint32_t)(e >> 32)) <= tlim) return (int32_t)(uint32_t)e;
    }
    return kDone;
}

// The descent phase of one while-while iteration (Aila & Laine 2009): internal nodes are visited
// near child first, the far hit child is pushed with its entry distance, and a lane reaching a leaf
// postpones it and keeps descending until every active lane of the warp holds a leaf. OCT >= 0:
// all active lanes travel in ray octant OCT (slab_oct); OCT = -1: mixed octants (slab_hit).
template <int OCT, bool kCount>
__device__ __forceinline__ void descend(const Node64 *__restrict__ nodes, const float4 *__restrict__ tri, const Pre &p,
                                        float tmin, bool active,
                                        Hit &h, float tlim, LaneStack &st, int &sp, int32_t &cur,
                                        int32_t &leaf) {
    while (true) {
        bool go = false;
#pragma unroll
        for (int u = 0; u < FGL_DESCEND_UNROLL; ++u) {  // nodes per warp vote
        go = active && cur >= 0 && cur != kDone;
#if FGL_FLAT_VISIT
        {
            // flat visit: every lane runs the node visit (idle lanes re-read the root, L1-resident, and
            // discard it), decisions by selects; the pops are the only divergent branches
            float4 na, nb, nc, ndf;
            ldg_node(nodes + (go ? cur : 0), na, nb, nc, ndf);
            const int32_t c0 = __float_as_int(ndf.x), c1 = __float_as_int(ndf.y);
            if (kCount && go) ++h.nodes;
            float t0, t1;
            const bool h0 = slab_sel<OCT>(p, na.x, na.y, na.z, na.w, nc.x, nc.y, tmin, h.t, t0) && go;
            const bool h1 = slab_sel<OCT>(p, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, tmin, h.t, t1) && go;
            const bool swap = h1 && (!h0 || t1 < t0);  // the nearer hit child is c1
            const int32_t nearc = swap ? c1 : c0, farc = swap ? c0 : c1;
            if (h0 && h1) st.push(sp, ((uint64_t)__float_as_uint(swap ? t0 : t1) << 32) | (uint32_t)farc);
            if (h0 || h1) cur = nearc;
            bool need = go && !(h0 || h1);
            if ((h0 || h1) && nearc < 0 && leaf == 0) leaf = nearc, need = true;
            if (need) {
                cur = pop_live(st, sp, tlim);
                if (cur < 0 && leaf == 0) {
                    leaf = cur;
                    cur = pop_live(st, sp, tlim);
                }
            }
        }
        if (false) {
#else
        if (go) {
#endif
            float4 na, nb, nc, ndf;
            ldg_node(nodes + cur, na, nb, nc, ndf);
            const int4 nd = make_int4(__float_as_int(ndf.x), __float_as_int(ndf.y), 0, 0);
#if FGL_PREFETCH
            // L1 prefetch of both children as soon as their refs are known: the box test below
            // (~25 issue slots of this warp, interleaved with the SM's other warps) covers most of an
            // L2 round trip, so the next visit's node load usually hits L1
            if (nd.x >= 0) prefetch_l1(nodes + nd.x);
            if (nd.y >= 0) prefetch_l1(nodes + nd.y);
#if FGL_PREFETCH > 1
            if (nd.x < 0 && nd.x != kEmptyRef) prefetch_l1(tri + kTriStride * (int64_t)((~nd.x) >> kLeafShift));
            if (nd.y < 0 && nd.y != kEmptyRef) prefetch_l1(tri + kTriStride * (int64_t)((~nd.y) >> kLeafShift));
#endif
#endif
            if (kCount) ++h.nodes;
            const float lim = h.t;
            float t0, t1;
            const bool h0 = slab_sel<OCT>(p, na.x, na.y, na.z, na.w, nc.x, nc.y, tmin, lim, t0);
            const bool h1 = slab_sel<OCT>(p, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, tmin, lim, t1);
            if (h0 && h1) {
                const bool swap = t1 < t0;
                const int32_t nearc = swap ? nd.y : nd.x, farc = swap ? nd.x : nd.y;
#if FGL_LEAF_HANDOFF
                // the near child is a leaf to postpone: the far child continues the descent at once
                // (instead of a push and an immediate pop of the same entry, which the cull cannot
                // reject: its entry distance is <= t*)
                const bool handoff = nearc < 0 && leaf == 0;
                if (!handoff)
                    st.push(sp, ((uint64_t)__float_as_uint(swap ? t0 : t1) << 32) | (uint32_t)farc);
                cur = handoff ? farc : nearc;
                leaf = handoff ? nearc : leaf;
#else
                st.push(sp, ((uint64_t)__float_as_uint(swap ? t0 : t1) << 32) | (uint32_t)farc);
                cur = nearc;
#endif
            } else if (h0) {
                cur = nd.x;
            } else if (h1) {
                cur = nd.y;
            } else {
                cur = pop_live(st, sp, tlim);
            }
            if (cur < 0 && leaf == 0) {
                leaf = cur;
                cur = pop_live(st, sp, tlim);
            }
        }
        }
        if (!__any_sync(0xffffffffu, go && leaf == 0)) break;
    }
}

// The leaf phase of one while-while iteration: every lane holding a postponed leaf tests its
// triangles (watertight test, (t, id) lexicographic minimum), then takes the next postponed leaf if
// its descent ended on one.
template <bool kCount, class Stack>
__device__ __forceinline__ void leaves(const float4 *__restrict__ tri, const Pre &p, float tmin, bool active, Hit &h,
                                       Stack &st, int &sp, int32_t &cur, int32_t &leaf) {
    if (!active) return;
    while (leaf < 0) {
        const int32_t v = ~leaf;
        const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
        for (int32_t k = first; k < first + cnt; ++k) {
            const float4 *tp = tri + kTriStride * (int64_t)k;
            float4 a, b, c;
            if constexpr (kTriStride == 4) {  // 64-byte records: one 256-bit + one 128-bit load
                asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                    : "l"(tp));
                c = __ldg(tp + 2);
            } else {
                a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
            }
            const int32_t id = __float_as_int(a.w);
            if (kCount) ++h.tris;
            float t;
            if (hit_tri(p, a, b, c, tmin, h.t, h.id, id, t)) {
                h.t = t;
                h.id = id;
            }
        }
        leaf = 0;
        if (cur < 0) {
            leaf = cur;
            // stacked entry distances are lower bounds (precompute_dyn): cull iff > t*
            cur = pop_live(st, sp, h.t);
        }
    }
}

// 8-bit plane byte j of word w as v = 1 + q 2^-15, exactly: one PRMT places q in bits 8..15 of the
// mantissa of 1.0f (no integer-to-float conversion, which runs on a quarter-rate pipe)
__device__ __forceinline__ float qv(uint32_t w, int j) {
    return __uint_as_float(__byte_perm(w, 0x3F800000u, 0x7604u | ((uint32_t)j << 4)));
}

// Per-axis constants of a node96q visit. Plane q of the axis is at p + q 2^e, so its ray parameter
// is t = v A + B with v = 1 + q 2^-15, A = I 2^(e+15) (exact: a power-of-two scaling of I) and
// B = fma(p, I, c) - A. The two extra roundings (fma, subtraction) and the final fma's are each
// <= 2^-24 of |B| + |A| + |t| <= 2 (|B| + 2 |A|), and I's own error adds <= 2^-23 |t|: the near
// plane's B is pushed down and the far plane's up by s = (|B| + 2 |A|) 2^-20, which bounds all of
// them, so the decoded box test stays conservative, like the fp32 slab test.
__device__ __forceinline__ void axis8(float pa, float I, float c_near, float c_far, uint32_t E, float &A, float &Bn,
                                      float &Bf) {
    A = I * __uint_as_float(E << 23);
    const float bn = fmaf(pa, I, c_near) - A, bf = fmaf(pa, I, c_far) - A;
    const float sl = fmaf(fabsf(A), 2.f, fabsf(bn)) * 0x1p-20f;
    Bn = bn - sl;
    Bf = bf + sl;
}

// The descent phase over node96q (width 8): a visit fetches the node in three 256-bit loads, tests
// the eight 8-bit child boxes and pushes every hit child with its entry distance in reverse visiting
// order (Ylitie et al.'s octant order: slot k ^ X(OCT), X with x and y most significant), then pops
// the first one — so the nearest-ordered child is visited next and the rest are culled by t* on pop
// exactly as in the binary traversal. OCT = -1: mixed octants (planes chosen per lane, slot order).
template <int OCT, bool kCount>
__device__ __forceinline__ void descend8(const Node8 *__restrict__ nodes8, const Pre &p, float tmin, bool active,
                                         Hit &h, float tlim, LaneStack8 &st, int &sp, int32_t &cur, int32_t &leaf) {
    while (true) {
        bool go = active && cur >= 0 && cur != kDone;
        if (go) {
            const float *q = reinterpret_cast<const float *>(nodes8 + cur);
            float4 c0a, c0bf, c1af, c1bf, r0f, r1f;
            asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(c0a.x), "=f"(c0a.y), "=f"(c0a.z), "=f"(c0a.w), "=f"(c0bf.x), "=f"(c0bf.y), "=f"(c0bf.z),
                  "=f"(c0bf.w)
                : "l"(q));
            asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(c1af.x), "=f"(c1af.y), "=f"(c1af.z), "=f"(c1af.w), "=f"(c1bf.x), "=f"(c1bf.y), "=f"(c1bf.z),
                  "=f"(c1bf.w)
                : "l"(q + 8));
            asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(r0f.x), "=f"(r0f.y), "=f"(r0f.z), "=f"(r0f.w), "=f"(r1f.x), "=f"(r1f.y), "=f"(r1f.z),
                  "=f"(r1f.w)
                : "l"(q + 16));
            if (kCount) ++h.nodes;
            const uint32_t meta = __float_as_uint(c0a.w);
            const bool nx = OCT >= 0 ? (OCT & 1) != 0 : p.Ix < 0.f;
            const bool ny = OCT >= 0 ? (OCT & 2) != 0 : p.Iy < 0.f;
            const bool nz = OCT >= 0 ? (OCT & 4) != 0 : p.Iz < 0.f;
            float Ax, Bnx, Bfx, Ay, Bny, Bfy, Az, Bnz, Bfz;
            axis8(c0a.x, p.Ix, nx ? p.chx : p.clx, nx ? p.clx : p.chx, meta & 0xFFu, Ax, Bnx, Bfx);
            axis8(c0a.y, p.Iy, ny ? p.chy : p.cly, ny ? p.cly : p.chy, (meta >> 8) & 0xFFu, Ay, Bny, Bfy);
            axis8(c0a.z, p.Iz, nz ? p.chz : p.clz, nz ? p.clz : p.chz, (meta >> 16) & 0xFFu, Az, Bnz, Bfz);
            // plane words (lo / hi bytes of children 0-3 and 4-7); the near plane is lo iff I >= 0
            const uint32_t lx0 = __float_as_uint(c0bf.x), lx1 = __float_as_uint(c0bf.y);
            const uint32_t hx0 = __float_as_uint(c0bf.z), hx1 = __float_as_uint(c0bf.w);
            const uint32_t ly0 = __float_as_uint(c1af.x), ly1 = __float_as_uint(c1af.y);
            const uint32_t hy0 = __float_as_uint(c1af.z), hy1 = __float_as_uint(c1af.w);
            const uint32_t lz0 = __float_as_uint(c1bf.x), lz1 = __float_as_uint(c1bf.y);
            const uint32_t hz0 = __float_as_uint(c1bf.z), hz1 = __float_as_uint(c1bf.w);
            const uint32_t nwx[2] = {nx ? hx0 : lx0, nx ? hx1 : lx1}, fwx[2] = {nx ? lx0 : hx0, nx ? lx1 : hx1};
            const uint32_t nwy[2] = {ny ? hy0 : ly0, ny ? hy1 : ly1}, fwy[2] = {ny ? ly0 : hy0, ny ? ly1 : hy1};
            const uint32_t nwz[2] = {nz ? hz0 : lz0, nz ? hz1 : lz1}, fwz[2] = {nz ? lz0 : hz0, nz ? lz1 : hz1};
            const int32_t ref[8] = {__float_as_int(r0f.x), __float_as_int(r0f.y), __float_as_int(r0f.z),
                                    __float_as_int(r0f.w), __float_as_int(r1f.x), __float_as_int(r1f.y),
                                    __float_as_int(r1f.z), __float_as_int(r1f.w)};
            const float lim = h.t;
            float tk[8];
            bool hk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int w = k >> 2, j = k & 3;
                const float tnx = fmaf(qv(nwx[w], j), Ax, Bnx), tfx = fmaf(qv(fwx[w], j), Ax, Bfx);
                const float tny = fmaf(qv(nwy[w], j), Ay, Bny), tfy = fmaf(qv(fwy[w], j), Ay, Bfy);
                const float tnz = fmaf(qv(nwz[w], j), Az, Bnz), tfz = fmaf(qv(fwz[w], j), Az, Bfz);
                const float tn = fmaxf(fmaxf(tnx, tny), fmaxf(tnz, tmin));
                const float tf = fminf(fminf(tfx, tfy), fminf(tfz, lim));
                hk[k] = tn <= tf && ((meta >> (24 + k)) & 1u);
                tk[k] = tn;
            }
            constexpr int X = OCT >= 0 ? (((OCT & 1) << 2) | (OCT & 2) | ((OCT >> 2) & 1)) : 0;
#pragma unroll
            for (int pos = 7; pos >= 0; --pos) {
                const int k = pos ^ X;
                if (hk[k]) st.push(sp, ((uint64_t)__float_as_uint(tk[k]) << 32) | (uint32_t)ref[k]);
            }
            cur = pop_live(st, sp, tlim);
            if (cur < 0 && leaf == 0) {
                leaf = cur;
                cur = pop_live(st, sp, tlim);
            }
        }
        if (!__any_sync(0xffffffffu, go && leaf == 0)) break;
    }
}

#ifndef FGL_OCTANT
#define FGL_OCTANT 1  // octant-specialised descent when a warp's rays share an octant
#endif
// Per-ray BVH2 traversal, persistent warps: a warp takes a 32-ray tile from a self-resetting global
// counter when all its lanes are done (refilling single lanes earlier was measured slower: it mixes
// rays of distant tiles), generates the rays in registers and runs the while-while traversal of
// Aila & Laine (2009) one outer iteration at a time. The output slot (and, for hit points, the ray)
// is recomputed from (tile, lane) at the write, so neither is held in registers during traversal.
#ifndef FGL_DYN8_MINBLOCKS
#define FGL_DYN8_MINBLOCKS 8  // width 8: 8 CTAs x 4 warps per SM (64 registers: the node96q visit holds more)
#endif
template <class Gen, bool kCount, int kW>
__global__ void __launch_bounds__(kCastThreads, kW == 8 ? FGL_DYN8_MINBLOCKS : FGL_DYN_MINBLOCKS)
    k_cast_dyn(const SceneView sv, const Gen gen, int64_t ntiles, const CastOut out, CastCounter *ctr) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    using Stack = std::conditional_t<kW == 8, LaneStack8, LaneStack>;
    Stack st;
#if FGL_SSTACK > 0
    __shared__ uint64_t s_stack[kSStack][kCastThreads];
    st.sh = &s_stack[0][threadIdx.x];
#else
    st.sh = nullptr;
#endif
    int sp = 0;
    int32_t cur = kDone, leaf = 0;
    Pre p;
    Hit h{0.f, INT_MAX, 0, 0};
    const Node64 *__restrict__ nodes = sv.nodes;
    const Node8 *__restrict__ nodes8 = reinterpret_cast<const Node8 *>(sv.nodes4);
    // a tree whose stack bound exceeds the stack (width 8: k_collapse; restructured width 2: its
    // depth, k_depth_max) is refused, loudly (fgl_scene_check)
    const bool refuse = __ldg(sv.wneed) > (unsigned int)(kW == 8 ? kStack8 : kStack);
    if (refuse && threadIdx.x == 0) atomicOr(sv.err, 4u);
    const float tmin = gen.interval_min();
    bool active = false;  // the lane's ray is still being traversed
    bool valid = false;   // the lane holds a ray of the current tile (result not yet written)
    uint32_t wtile = 0;  // < 2^31 tiles per launch (checked by the launchers)
    while (true) {
        if (!__any_sync(kFull, active)) {
            // the whole tile is done: every lane writes its result now, in one full-warp store per
            // output array (a tile's 8 columns are contiguous), instead of a partial-warp write each
            // time some lane finishes
            if (valid) {
                Ray r{};
                if (out.hit_xyz) gen.ray_at((int64_t)wtile, lane, r);
                write_out(out, gen.index((int64_t)wtile, lane), r, h);
            }
            unsigned long long nt = 0;
            if (lane == 0) nt = atomicAdd(&ctr->next, 1ull);
            // the counter ends below ntiles + (warps of the grid) < 2^31 + 2^20: exact in 32 bits
            wtile = (uint32_t)__shfl_sync(kFull, nt, 0);
            if ((int64_t)wtile >= ntiles || refuse) break;
            Ray r;
            valid = gen.ray_at((int64_t)wtile, lane, r);
            if (valid) {
                // the relevant reach: t_max, or for an unbounded interval the farthest point of the
                // scene (|o| + the largest |coordinate| of the root box, times sqrt 3 > the diagonal)
                float reach = gen.interval_max();
                if (!(reach < INFINITY)) {
                    const float4 blo = __ldg(sv.root_box), bhi = __ldg(sv.root_box + 1);
                    const float m = fmaxf(fmaxf(fmaxf(fabsf(blo.x), fabsf(bhi.x)), fmaxf(fabsf(blo.y), fabsf(bhi.y))),
                                          fmaxf(fabsf(blo.z), fabsf(bhi.z)));
                    const float mo = fmaxf(fmaxf(fabsf(r.ox), fabsf(r.oy)), fabsf(r.oz));
                    reach = 2.f * (m + mo);
                }
                p = precompute_dyn(r, reach);
                h = Hit{gen.interval_max(), INT_MAX, 0, 0};
                sp = 0, cur = 0, leaf = 0;
                active = true;
            }
        }
        // ---- one outer iteration of the while-while traversal ----
        // Every lane of the warp runs the descent loop (idle / finished lanes predicated off), so the
        // speculation vote is a plain full-warp vote. When all active lanes share a ray octant (the
        // usual case: a tile spans ~1.5 degrees) the loop is the octant-specialised instance.
#if FGL_OCTANT
        const unsigned act = __ballot_sync(kFull, active);
        const int oct = ray_octant(p);  // recomputed from p's signs: one register fewer held across the loop
        const int o0 = __shfl_sync(kFull, oct, __ffs(act) - 1);
        if (__all_sync(kFull, !active || oct == o0)) {
            if constexpr (kW == 8) {
                switch (o0) {
                    case 0: descend8<0, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 1: descend8<1, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 2: descend8<2, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 3: descend8<3, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 4: descend8<4, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 5: descend8<5, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 6: descend8<6, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    default: descend8<7, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                }
            } else {
                switch (o0) {
                    case 0: descend<0, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 1: descend<1, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 2: descend<2, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 3: descend<3, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 4: descend<4, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 5: descend<5, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    case 6: descend<6, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                    default: descend<7, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf); break;
                }
            }
        } else
#endif
        {
            if constexpr (kW == 8)
                descend8<-1, kCount>(nodes8, p, tmin, active, h, h.t, st, sp, cur, leaf);
            else
                descend<-1, kCount>(nodes, sv.tri, p, tmin, active, h, h.t, st, sp, cur, leaf);
        }
        leaves<kCount>(sv.tri, p, tmin, active, h, st, sp, cur, leaf);
        if (cur == kDone) active = false;
    }
    cast_epilogue(out, ctr, lane);
}

template <class Gen, bool kCount, int kMode>
void launch_one(const SceneView &sv, const Gen &gen, int64_t ntiles, const CastOut &o, CastCounter *ctr,
                cudaStream_t s) {
    // occupancy and SM count per device (a process may drive several GPUs)
    constexpr int kMaxDev = 64;
    static int oc_dev[kMaxDev] = {0}, sms_dev[kMaxDev] = {0};
    constexpr bool kDyn = kMode == kRay2 || kMode == kRay8Q;
    constexpr int kW = kMode == kRay8Q ? 8 : 2;
    int dev;
    FGL_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) throw Error(1, "CUDA device index out of range");
    int &oc = oc_dev[dev], &sms = sms_dev[dev];
    if (!oc) {
        FGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if constexpr (kDyn) {
#if FGL_CARVEOUT >= 0
            // the largest L1 share that still holds the resident CTAs' shared-memory stacks (plus the
            // 1 KB per CTA the system reserves): node / triangle reuse lives in L1
            const int need = (kW == 8 ? FGL_DYN8_MINBLOCKS : FGL_DYN_MINBLOCKS) * (kSStack * kCastThreads * 8 + 1024);
            const int pct = std::max(FGL_CARVEOUT, (int)((100ll * need + 233471) / 233472));
            FGL_CUDA(cudaFuncSetAttribute(k_cast_dyn<Gen, kCount, kW>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          std::min(pct, 100)));
#endif
            FGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, k_cast_dyn<Gen, kCount, kW>, kCastThreads, 0));
        } else {
            FGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, k_cast<Gen, kCount, kMode>, kCastThreads, 0));
        }
        if (oc < 1) oc = 1;
    }
    int64_t blocks = std::min<int64_t>((int64_t)sms * oc, (ntiles + kCastThreads / 32 - 1) / (kCastThreads / 32));
    blocks = std::max<int64_t>(blocks, 1);
    if constexpr (kDyn)
        k_cast_dyn<Gen, kCount, kW><<<(unsigned)blocks, kCastThreads, 0, s>>>(sv, gen, ntiles, o, ctr);
    else
        k_cast<Gen, kCount, kMode><<<(unsigned)blocks, kCastThreads, 0, s>>>(sv, gen, ntiles, o, ctr);
    FGL_LAUNCHED("k_cast");
}

template <class Gen, bool kCount>
void launch_mode(const SceneView &sv, const Gen &gen, int64_t ntiles, const CastOut &o, CastCounter *ctr,
                 cudaStream_t s) {
    if (sv.width == 8)
        launch_one<Gen, kCount, kRay8Q>(sv, gen, ntiles, o, ctr, s);
    else if (sv.width == 4 && sv.quantized)
        launch_one<Gen, kCount, kRay4Q>(sv, gen, ntiles, o, ctr, s);
    else if (sv.width == 4)
        launch_one<Gen, kCount, kRay4>(sv, gen, ntiles, o, ctr, s);
    else if (Gen::kCoherent && packet_mode())
        launch_one<Gen, kCount, kPacket2>(sv, gen, ntiles, o, ctr, s);
    else
        launch_one<Gen, kCount, kRay2>(sv, gen, ntiles, o, ctr, s);
}

template <class Gen>
void launch_persistent(const SceneView &sv, const Gen &gen, int64_t ntiles, const CastOut &o, CastCounter *ctr,
                       cudaStream_t s) {
    if (ntiles <= 0 && !o.nsignal) return;
    if (o.node_counts || o.tri_counts)
        launch_mode<Gen, true>(sv, gen, ntiles, o, ctr, s);
    else
        launch_mode<Gen, false>(sv, gen, ntiles, o, ctr, s);
}

// ---- brute force: every ray against every triangle, triangles staged in smem -------
constexpr int kBfThreads = 128;
__global__ void __launch_bounds__(kBfThreads) k_bruteforce(const float *__restrict__ verts, int64_t V,
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
                int32_t vi = tris[3 * k + v];
                vi = vi < 0 ? 0 : (vi >= V ? (int32_t)(V - 1) : vi);
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

__global__ void k_spin_table(const SpinParams sp, float2 *tab) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < sp.channels) tab[i] = spin_elev_sc(sp, i);
    else if (i < sp.channels + sp.columns) tab[i] = spin_az_sc(sp, i - sp.channels);
}

__global__ void k_export_spin(const SpinParams sp, const float2 *__restrict__ tab, const float *__restrict__ poses,
                              int64_t n, float *orig, float *dir) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t per = (int64_t)sp.channels * sp.columns;
        const int64_t p = g / per;
        const int c = (int)((g - p * per) / sp.columns), a = (int)(g % sp.columns);
        Ray r;
        spin_ray_tab(tab, sp.channels, poses, p, c, a, r);
        orig[3 * g] = r.ox, orig[3 * g + 1] = r.oy, orig[3 * g + 2] = r.oz;
        dir[3 * g] = r.dx, dir[3 * g + 1] = r.dy, dir[3 * g + 2] = r.dz;
    }
}

// stream-ordered [C + A] sin/cos table for one spinning call (freed on the stream after use)
float2 *spin_table(const SpinParams &p, cudaStream_t s) {
    const int n = p.channels + p.columns;
    float2 *tab = nullptr;
    FGL_CUDA(cudaMallocAsync((void **)&tab, sizeof(float2) * (size_t)n, s));
    k_spin_table<<<(n + 127) / 128, 128, 0, s>>>(p, tab);
    FGL_LAUNCHED("k_spin_table");
    return tab;
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
#ifndef FGL_TILE_C
#define FGL_TILE_C 4
#endif
    g.tc = p.channels >= FGL_TILE_C ? FGL_TILE_C : (p.channels >= 4 ? 4 : (p.channels >= 2 ? 2 : 1));
    g.ta = 32 / g.tc;
    g.lta = __builtin_ctz(g.ta);
    const int64_t nct = (p.channels + g.tc - 1) / g.tc, nat = (p.columns + g.ta - 1) / g.ta;
    const int64_t ntiles = P * nct * nat;
    if (ntiles >= (int64_t(1) << 31)) throw Error(1, "spinning cast: more than 2^31 ray tiles in one call");
    g.per = make_fastdiv((uint32_t)(nct * nat));
    g.nat = make_fastdiv((uint32_t)nat);
    if (ntiles <= 0 && !o.nsignal) return;
    float2 *tab = spin_table(p, s);
    g.tab = tab;
    launch_persistent(sv, g, ntiles, o, ctr, s);
    FGL_CUDA(cudaFreeAsync(tab, s));
}

void launch_cast_rosette(const SceneView &sv, const RosetteParams &p, const float *poses, int64_t P,
                         const CastOut &o, CastCounter *ctr, cudaStream_t s) {
    RosetteGen g;
    g.rp = p;
    g.poses = poses;
    g.ntile = (p.n + 31) / 32;
    g.ntile_d = make_fastdiv((uint32_t)g.ntile);
    if (P * (int64_t)g.ntile >= (int64_t(1) << 31)) throw Error(1, "rosette cast: more than 2^31 ray tiles in one call");
    launch_persistent(sv, g, P * (int64_t)g.ntile, o, ctr, s);
}

void launch_cast_rays(const SceneView &sv, const float *orig, const float *dir, int64_t R, float t_min, float t_max,
                      const CastOut &o, CastCounter *ctr, cudaStream_t s) {
    RaysGen g{orig, dir, R, t_min, t_max};
    if ((R + 31) / 32 >= (int64_t(1) << 31)) throw Error(1, "explicit-ray cast: more than 2^31 ray tiles in one call");
    launch_persistent(sv, g, (R + 31) / 32, o, ctr, s);
}

void launch_cast_bruteforce(const float *verts, int64_t V, const int32_t *tris, int64_t T, const float *orig,
                            const float *dir, int64_t R, float t_min, float t_max, float *range, int32_t *tri_id,
                            cudaStream_t s) {
    if (R <= 0) return;
    k_bruteforce<<<(unsigned)((R + kBfThreads - 1) / kBfThreads), kBfThreads, 0, s>>>(verts, V, tris, T, orig, dir,
                                                                                       R, t_min, t_max, range, tri_id);
    FGL_LAUNCHED("k_bruteforce");
}

__global__ void k_wait_flag(const int32_t *flag, int32_t target) {
    if (threadIdx.x == 0) {
        while (*(volatile const int32_t *)flag < target) __nanosleep(200);
        __threadfence_system();
    }
}

// L2 read-bandwidth probe: grid-stride 128-bit L1-bypassing loads over an L2-resident buffer
__global__ void __launch_bounds__(512) k_l2_read(const float4 *__restrict__ p, int64_t n4, int iters, float *sink) {
    float acc = 0.f;
    for (int it = 0; it < iters; ++it)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(p + i);
            acc += (v.x + v.y) + (v.z + v.w);
        }
    if (acc == 1234.5f) *sink = acc;  // never true for the zero-filled probe buffer; keeps the loads
}

void launch_l2_read(const void *buf, int64_t bytes, int iters, float *sink, cudaStream_t s) {
    int dev, sms;
    FGL_CUDA(cudaGetDevice(&dev));
    FGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    k_l2_read<<<sms * 4, 512, 0, s>>>(reinterpret_cast<const float4 *>(buf), bytes / 16, iters, sink);
    FGL_LAUNCHED("k_l2_read");
}

void launch_wait_flag(const int32_t *flag, int32_t target, cudaStream_t s) {
    k_wait_flag<<<1, 32, 0, s>>>(flag, target);
    FGL_LAUNCHED("k_wait_flag");
}

void launch_export_spinning(const SpinParams &p, const float *poses, int64_t P, float *orig, float *dir,
                            cudaStream_t s) {
    const int64_t n = P * p.channels * (int64_t)p.columns;
    if (n <= 0) return;
    float2 *tab = spin_table(p, s);
    k_export_spin<<<grid_for(n), 256, 0, s>>>(p, tab, poses, n, orig, dir);
    FGL_LAUNCHED("k_export_spin");
    FGL_CUDA(cudaFreeAsync(tab, s));
}

void launch_export_rosette(const RosetteParams &p, const float *poses, int64_t P, float *orig, float *dir,
                           cudaStream_t s) {
    const int64_t n = P * (int64_t)p.n;
    if (n <= 0) return;
    k_export_rosette<<<grid_for(n), 256, 0, s>>>(p, poses, n, orig, dir);
    FGL_LAUNCHED("k_export_rosette");
}

}  // namespace fgl
