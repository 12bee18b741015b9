// Gaussian -> occupancy on sm_100a — PAPER.md §IV-A, SURVEY §8(f) NEXT-2:
//   gauss_prep     : Morton point = the Gaussian centre mu_i, scene box of the centres,
//                    validation of the 3DGS parameters
//   gauss_reorder  : in leaf (Morton) order, the Eq. 4 box b_i = mu_i -+ kappa |R_i| s_i
//                    (rounded outward) and a 48-byte record {mu, f(sigma), Sigma^-1 prescaled for
//                    exp2}; the LBVH itself (Eqs. 5-7) is the mesh build's morton/sort/tree stages
//   voxelize       : one CTA per tile of 8^3 voxels; warp 0 queries the BVH with the tile box
//                    (Eq. 8) into a shared candidate list, all warps accumulate Eq. 9 over it
//                    (R25 truncation at m^2 <= kappa^2), then Eq. 10 thresholds into a bit volume
//   masks          : Eqs. 11-12 on the bit volume, 32 voxels per word
#include <cfloat>

#include "fgl_internal.cuh"

namespace fgl {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// 2^x on the SFU without the library's denormal-result rescaling (x >= -kk > -126 here)
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float wmin(float v) {
    for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float wmax(float v) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// centroids (= mu) + scene box (last-block reduce) + parameter validation (flag bit 2)
__global__ void __launch_bounds__(256) k_gauss_prep(const float *__restrict__ mu, const float *__restrict__ quat,
                                                    const float *__restrict__ scale, const float *__restrict__ opac,
                                                    int64_t n, float4 *__restrict__ cent, float *__restrict__ partial,
                                                    unsigned int *sync, float *__restrict__ box,
                                                    unsigned int *flag) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned int bad = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const float x = mu[3 * k], y = mu[3 * k + 1], z = mu[3 * k + 2];
        const float4 q = reinterpret_cast<const float4 *>(quat)[k];
        const float sx = scale[3 * k], sy = scale[3 * k + 1], sz = scale[3 * k + 2], o = opac[k];
        const float qq = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
        const bool ok = isfinite(x) && isfinite(y) && isfinite(z) && isfinite(qq) && qq > 0.f && sx > 0.f &&
                        sy > 0.f && sz > 0.f && isfinite(sx) && isfinite(sy) && isfinite(sz) && o >= 0.f && o <= 1.f;
        if (!ok) bad |= 2u;
        cent[k] = make_float4(x, y, z, 0.f);
        if (isfinite(x) && isfinite(y) && isfinite(z)) {
            lo[0] = fminf(lo[0], x), lo[1] = fminf(lo[1], y), lo[2] = fminf(lo[2], z);
            hi[0] = fmaxf(hi[0], x), hi[1] = fmaxf(hi[1], y), hi[2] = fmaxf(hi[2], z);
        }
    }
    if (bad && flag) atomicOr(flag, bad);
    __shared__ float s[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < 3; ++i) lo[i] = wmin(lo[i]), hi[i] = wmax(hi[i]);
    if (lane == 0)
        for (int i = 0; i < 3; ++i) s[w][i] = lo[i], s[w][3 + i] = hi[i];
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        partial[blockIdx.x * 6 + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(sync, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    // last block: every thread's partial loads in flight at once (one warp looping over them paid
    // ~28 dependent L2 round trips per component), then warp and block reductions
    float r[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = i < 3 ? INFINITY : -INFINITY;
#pragma unroll
    for (int qb = 0; qb < (kPrepBlocks + 255) / 256; ++qb) {
        const int b = threadIdx.x + qb * (int)blockDim.x;
        if (b < (int)gridDim.x) {
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const float x = __ldcg(partial + b * 6 + i);
                r[i] = i < 3 ? fminf(r[i], x) : fmaxf(r[i], x);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = i < 3 ? wmin(r[i]) : wmax(r[i]);
    __syncthreads();  // s is reused
    if (lane == 0)
        for (int i = 0; i < 6; ++i) s[w][i] = r[i];
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            v = threadIdx.x < 3 ? fminf(v, s[ww][threadIdx.x]) : fmaxf(v, s[ww][threadIdx.x]);
        box[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) *sync = 0u;
}

// Leaf j = Gaussian k = perm(j): Eq. 4 box (outward: every rounding of R, |R| s and mu -+ r is
// covered by a 2^-18 relative pad, so the float box contains the exact kappa ellipsoid) and the
// record r0 = (mu, f(sigma) = sigma [R24]), r1 = (c00, c11, c22, id), r2 = (2 c01, 2 c02, 2 c12,
// 1 / (4 c00))
// with c = (log2 e / 2) Sigma^-1, Sigma^-1 = R diag(1/s^2) R^T, so exp(-m^2 / 2) =
// exp2(-d^T c d). Also the first 8-ary aggregate level of the leaf boxes.
__global__ void __launch_bounds__(256) k_gauss_reorder(const float *__restrict__ mu, const float *__restrict__ quat,
                                                       const float *__restrict__ scale,
                                                       const float *__restrict__ opac, float kappa,
                                                       const uint32_t *__restrict__ perm,
                                                       const uint64_t *__restrict__ pkeys, uint64_t pmask, int64_t n,
                                                       float4 *__restrict__ rec, float4 *__restrict__ leafbox,
                                                       float4 *__restrict__ agg) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
    if (j < n) {
        const uint32_t k = perm ? perm[j] : (uint32_t)(pkeys[j] & pmask);
        const float m[3] = {mu[3 * (int64_t)k], mu[3 * (int64_t)k + 1], mu[3 * (int64_t)k + 2]};
        float4 q = reinterpret_cast<const float4 *>(quat)[k];  // (w, x, y, z)
        const float rn = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
        const float w = q.x * rn, x = q.y * rn, y = q.z * rn, z = q.w * rn;
        float R[3][3];
        R[0][0] = 1.f - 2.f * (y * y + z * z), R[0][1] = 2.f * (x * y - w * z), R[0][2] = 2.f * (x * z + w * y);
        R[1][0] = 2.f * (x * y + w * z), R[1][1] = 1.f - 2.f * (x * x + z * z), R[1][2] = 2.f * (y * z - w * x);
        R[2][0] = 2.f * (x * z - w * y), R[2][1] = 2.f * (y * z + w * x), R[2][2] = 1.f - 2.f * (x * x + y * y);
        const float s[3] = {scale[3 * (int64_t)k], scale[3 * (int64_t)k + 1], scale[3 * (int64_t)k + 2]};
        float l[3], h[3];
        for (int a = 0; a < 3; ++a) {
            float r = 0.f;
            for (int c = 0; c < 3; ++c) r = __fmaf_ru(fabsf(R[a][c]), s[c], r);
            r = __fmul_ru(__fmul_ru(r, kappa), 1.0f + 0x1p-18f);
            l[a] = __fsub_rd(m[a], r);
            h[a] = __fadd_ru(m[a], r);
        }
        lo = make_float4(l[0], l[1], l[2], 0.f);
        hi = make_float4(h[0], h[1], h[2], 0.f);
        leafbox[2 * j] = lo;
        leafbox[2 * j + 1] = hi;
        float is2[3];
        for (int c = 0; c < 3; ++c) is2[c] = 0.5f * kLog2e / (s[c] * s[c]);
        float A[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = a; b < 3; ++b) {
                float v = 0.f;
                for (int c = 0; c < 3; ++c) v = fmaf(R[a][c] * R[b][c], is2[c], v);
                A[a][b] = v;
            }
        rec[3 * j] = make_float4(m[0], m[1], m[2], opac[k]);
        rec[3 * j + 1] = make_float4(A[0][0], A[1][1], A[2][2], __int_as_float((int32_t)k));
        rec[3 * j + 2] = make_float4(2.f * A[0][1], 2.f * A[0][2], 2.f * A[1][2], 0.25f / A[0][0]);
    }
    for (int o = 4; o; o >>= 1) {
        lo.x = fminf(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
        lo.y = fminf(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
        lo.z = fminf(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
        hi.x = fmaxf(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
        hi.y = fmaxf(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
        hi.z = fmaxf(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
    }
    if ((threadIdx.x & 7) == 0 && j < n) {
        agg[2 * (j >> 3)] = lo;
        agg[2 * (j >> 3) + 1] = hi;
    }
}

constexpr int kTileB = 8;                 // tile edge (voxels); B^3 = 512 voxels per CTA
constexpr int kVoxThreads = 128;          // 4 voxels along x per thread
constexpr int kStackCap = 2048;           // warp-0 traversal stack (node indices)
constexpr int kCandCap = 1024;            // candidate indices (leaf positions)
constexpr int kFlushAt = kCandCap - 32 * 2 * kMaxLeaf;  // room for one more 32-node step
constexpr int kBatch = 256;               // records staged in shared memory per accumulation pass

struct VoxArgs {
    double o[3];          // grid origin
    double h;             // spacing
    int nx, ny, nz;
    int tx, ty;           // tiles along x, y
    int rowbytes;         // bytes per occupancy row (4 * ceil(nx / 32))
    float theta;
    float kk;             // (log2 e / 2) kappa^2: the R25 truncation in exp2 units
    float kk_skip;        // kk with a 2^-10 margin: the row-minimum skip test never drops a term
};

__global__ void __launch_bounds__(kVoxThreads) k_voxelize(const Node64 *__restrict__ nodes,
                                                          const float4 *__restrict__ rec, VoxArgs va,
                                                          float *__restrict__ density, uint8_t *__restrict__ occ,
                                                          unsigned long long *__restrict__ counts,
                                                          unsigned int *__restrict__ overflow) {
    __shared__ int s_stack[kStackCap];
    __shared__ int s_cand[kCandCap];
    __shared__ float4 s_rec[kBatch][3];
    __shared__ int s_sp, s_nc;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tile = blockIdx.x;
    const int bx = tile % va.tx, by = (tile / va.tx) % va.ty, bz = tile / (va.tx * va.ty);
    const int x0 = bx * kTileB, y0 = by * kTileB, z0 = bz * kTileB;
    const int x1 = min(x0 + kTileB, va.nx), y1 = min(y0 + kTileB, va.ny), z1 = min(z0 + kTileB, va.nz);
    // reference point c = centre of voxel (x0, y0, z0), in double; offsets are tile-relative floats
    const double cx = va.o[0] + (x0 + 0.5) * va.h, cy = va.o[1] + (y0 + 0.5) * va.h, cz = va.o[2] + (z0 + 0.5) * va.h;
    // Eq. 8 tile box: the span of the tile's voxel centres, rounded outward to float
    const float tlx = __double2float_rd(cx), tly = __double2float_rd(cy), tlz = __double2float_rd(cz);
    const float thx = __double2float_ru(va.o[0] + (x1 - 0.5) * va.h);
    const float thy = __double2float_ru(va.o[1] + (y1 - 0.5) * va.h);
    const float thz = __double2float_ru(va.o[2] + (z1 - 0.5) * va.h);
    // this thread's voxels: x = x0 + xb .. +3, y = y0 + ly, z = z0 + lz
    const int xb = (t & 1) * 4, ly = (t >> 1) & 7, lz = t >> 4;
    const float hf = (float)va.h;
    const float vy = (float)ly * hf, vz = (float)lz * hf;
    float vx[4], D[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 4; ++q) vx[q] = (float)(xb + q) * hf;
    if (t == 0) s_sp = 1, s_nc = 0, s_stack[0] = 0;
    __syncthreads();
    unsigned long long pairs = 0;
    while (true) {
        // ---- Eq. 8: warp 0 walks the BVH with the tile box, 32 stack entries per step ----------
        if (warp == 0) {
            int sp = s_sp, nc = s_nc;
            while (sp > 0 && nc < kFlushAt) {
                const int take = min(32, sp);
                const int node = lane < take ? s_stack[sp - 1 - lane] : -1;
                sp -= take;
                __syncwarp();  // the pushes below reuse the slots just read (memory order within the warp)
                bool ov0 = false, ov1 = false;
                int r0 = 0, r1 = 0;
                if (node >= 0) {
                    const float4 *np = reinterpret_cast<const float4 *>(nodes + node);
                    const float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
                    const int4 d = __ldg(reinterpret_cast<const int4 *>(np + 3));
                    ov0 = a.x <= thx && a.y >= tlx && a.z <= thy && a.w >= tly && c.x <= thz && c.y >= tlz &&
                          d.x != kEmptyRef;
                    ov1 = b.x <= thx && b.y >= tlx && b.z <= thy && b.w >= tly && c.z <= thz && c.w >= tlz &&
                          d.y != kEmptyRef;
                    r0 = d.x, r1 = d.y;
                }
                // push overlapping internal children (ballot-compacted), append leaf ranges
                const bool p0 = ov0 && r0 >= 0, p1 = ov1 && r1 >= 0;
                const unsigned m0 = __ballot_sync(0xffffffffu, p0), m1 = __ballot_sync(0xffffffffu, p1);
                const unsigned lt = (1u << lane) - 1u;
                const int n0 = __popc(m0);
                if (sp + n0 + __popc(m1) > kStackCap) {
                    if (lane == 0) atomicOr(overflow, 1u);
                    sp = 0;
                    break;
                }
                if (p0) s_stack[sp + __popc(m0 & lt)] = r0;
                if (p1) s_stack[sp + n0 + __popc(m1 & lt)] = r1;
                sp += n0 + __popc(m1);
                const int c0 = (ov0 && r0 < 0) ? ((~r0) & (kMaxLeaf - 1)) + 1 : 0;
                const int c1 = (ov1 && r1 < 0) ? ((~r1) & (kMaxLeaf - 1)) + 1 : 0;
                int incl = c0 + c1;  // inclusive warp scan of the leaf counts
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int pos = nc + incl - (c0 + c1);
                for (int k = 0; k < c0; ++k) s_cand[pos++] = ((~r0) >> kLeafShift) + k;
                for (int k = 0; k < c1; ++k) s_cand[pos++] = ((~r1) >> kLeafShift) + k;
                nc += __shfl_sync(0xffffffffu, incl, 31);
                __syncwarp();
            }
            if (lane == 0) s_sp = sp, s_nc = nc;
        }
        __syncthreads();
        const int nc = s_nc;
        // ---- Eq. 9: every voxel of the tile sums its candidates (R25 truncation) ---------------
        for (int b0 = 0; b0 < nc; b0 += kBatch) {
            const int nb = min(kBatch, nc - b0);
            for (int c = t; c < nb; c += kVoxThreads) {
                const int j = s_cand[b0 + c];
                const float4 a = __ldg(rec + 3 * (int64_t)j), b = __ldg(rec + 3 * (int64_t)j + 1),
                             e = __ldg(rec + 3 * (int64_t)j + 2);
                // tile-relative centre: mu - c in double, rounded once to float
                s_rec[c][0] = make_float4((float)((double)a.x - cx), (float)((double)a.y - cy),
                                          (float)((double)a.z - cz), a.w);
                s_rec[c][1] = b;
                s_rec[c][2] = e;
            }
            __syncthreads();
            for (int c = 0; c < nb; ++c) {
                const float4 a = s_rec[c][0], b = s_rec[c][1], e = s_rec[c][2];
                const float dy = vy - a.y, dz = vz - a.z;
                const float P = fmaf(e.x, dy, e.y * dz);                   // 2 c01 dy + 2 c02 dz
                const float Q = fmaf(dy, fmaf(b.y, dy, e.z * dz), b.z * dz * dz);  // c11 dy^2 + 2 c12 dy dz + c22 dz^2
                // the row's quadratic c00 dx^2 + P dx + Q is >= Q - P^2 / (4 c00) for every x: when no
                // lane of the warp can reach the kappa ellipsoid, skip the candidate (warp-uniform)
                if (!__any_sync(0xffffffffu, fmaf(-P * P, e.w, Q) <= va.kk_skip)) continue;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float dx = vx[q] - a.x;
                    const float arg = fmaf(dx, fmaf(b.x, dx, P), Q);
                    if (arg <= va.kk) D[q] = fmaf(a.w, ex2(-arg), D[q]);
                }
            }
            pairs += (unsigned long long)nb;
            __syncthreads();
        }
        const bool more = s_sp > 0;
        __syncthreads();
        if (!more) break;
        if (t == 0) s_nc = 0;
        __syncthreads();
    }
    // ---- outputs: density, Eq. 10 occupancy bits (one byte = 8 voxels along x) ------------------
    const int y = y0 + ly, z = z0 + lz;
    const bool row = y < va.ny && z < va.nz;
    unsigned bits = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = x0 + xb + q;
        if (row && x < va.nx) {
            if (density) density[((int64_t)z * va.ny + y) * va.nx + x] = D[q];
            if (D[q] > va.theta) bits |= 1u << (xb + q);
        }
    }
    bits |= __shfl_xor_sync(0xffffffffu, bits, 1);
    if (row && (t & 1) == 0) occ[((int64_t)z * va.ny + y) * va.rowbytes + bx] = (uint8_t)bits;
    if (counts) {
        unsigned occn = (t & 1) == 0 ? __popc(bits) : 0u;
        for (int o = 16; o; o >>= 1) occn += __shfl_xor_sync(0xffffffffu, occn, o);
        if (lane == 0) atomicAdd(&counts[0], (unsigned long long)occn);
        if (t == 0) {
            const int nvox = (x1 - x0) * (y1 - y0) * (z1 - z0);
            atomicAdd(&counts[2], pairs * (unsigned long long)nvox);
        }
    }
}

// Eqs. 11-12 on 32-voxel words: Int = V and its six neighbours (outside the grid = empty, R27),
// Surf = V and not Int
__global__ void __launch_bounds__(256) k_masks(const uint32_t *__restrict__ occ, int nwx, int ny, int nz,
                                               uint32_t *__restrict__ surf, uint32_t *__restrict__ inter,
                                               unsigned long long *__restrict__ counts) {
    const int64_t nw = (int64_t)nwx * ny * nz;
    unsigned sn = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(i % nwx);
        const int64_t r = i / nwx;
        const int y = (int)(r % ny), z = (int)(r / ny);
        const uint32_t v = occ[i];
        uint32_t in = v;
        if (v) {
            const uint32_t left = w > 0 ? occ[i - 1] >> 31 : 0u, right = w + 1 < nwx ? occ[i + 1] << 31 : 0u;
            in &= (v << 1) | left;   // x - 1 occupied
            in &= (v >> 1) | right;  // x + 1 occupied
            in &= y > 0 ? occ[i - nwx] : 0u;
            in &= y + 1 < ny ? occ[i + nwx] : 0u;
            in &= z > 0 ? occ[i - (int64_t)nwx * ny] : 0u;
            in &= z + 1 < nz ? occ[i + (int64_t)nwx * ny] : 0u;
        }
        if (inter) inter[i] = in;
        if (surf) surf[i] = v & ~in;
        sn += __popc(v & ~in);
    }
    if (counts) {
        for (int o = 16; o; o >>= 1) sn += __shfl_xor_sync(0xffffffffu, sn, o);
        if ((threadIdx.x & 31) == 0 && sn) atomicAdd(&counts[1], (unsigned long long)sn);
    }
}

}  // namespace

void launch_gauss_prep(const float *mu, const float *quat, const float *scale, const float *opac, int64_t n,
                       BuildBuffers &b, unsigned int *flag, cudaStream_t s) {
    k_gauss_prep<<<kPrepBlocks, 256, 0, s>>>(mu, quat, scale, opac, n, b.cent, b.partial, b.sync, b.box, flag);
    FGL_LAUNCHED("k_gauss_prep");
}

void launch_gauss_build(const float *mu, const float *quat, const float *scale, const float *opac, float kappa,
                        BuildBuffers &b, int bits, int leaf_size, cudaStream_t s) {
    const int64_t n = b.T;
    k_gauss_prep<<<kPrepBlocks, 256, 0, s>>>(mu, quat, scale, opac, n, b.cent, b.partial, b.sync, b.box, nullptr);
    FGL_LAUNCHED("k_gauss_prep");
    launch_morton_sort(b, bits, 0, s);
    const int ps = b.packed_shift, slot = b.sorted_slot;
    k_gauss_reorder<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(mu, quat, scale, opac, kappa,
                                                                ps ? nullptr : b.vals[slot], b.keys[slot],
                                                                ps ? (uint64_t(1) << ps) - 1 : 0, n, b.tri,
                                                                b.leafbox, b.agg);
    FGL_LAUNCHED("k_gauss_reorder");
    launch_tree(b, leaf_size, 2, 0, s);
}

void launch_voxelize(const BuildBuffers &b, const VoxGrid &g, float kappa, float *density, uint32_t *occ,
                     uint32_t *surf, uint32_t *inter, unsigned long long *counts, unsigned int *overflow,
                     cudaStream_t s) {
    VoxArgs va;
    for (int a = 0; a < 3; ++a) va.o[a] = g.origin[a];
    va.h = g.h;
    va.nx = g.dims[0], va.ny = g.dims[1], va.nz = g.dims[2];
    va.tx = (va.nx + kTileB - 1) / kTileB;
    va.ty = (va.ny + kTileB - 1) / kTileB;
    const int tz = (va.nz + kTileB - 1) / kTileB;
    const int nwx = (va.nx + 31) / 32;
    va.rowbytes = 4 * nwx;
    va.theta = g.theta;
    va.kk = 0.5f * kLog2e * kappa * kappa;
    va.kk_skip = va.kk * (1.0f + 0x1p-10f) + 0x1p-20f;
    FGL_CUDA(cudaMemsetAsync(occ, 0, sizeof(uint32_t) * (size_t)nwx * va.ny * va.nz, s));
    const int64_t ntiles = (int64_t)va.tx * va.ty * tz;
    k_voxelize<<<(unsigned)ntiles, kVoxThreads, 0, s>>>(b.nodes, b.tri, va, density, reinterpret_cast<uint8_t *>(occ),
                                                        counts, overflow);
    FGL_LAUNCHED("k_voxelize");
    if (surf || inter || counts) {
        const int64_t nw = (int64_t)nwx * va.ny * va.nz;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nw + 255) / 256, 148 * 8));
        k_masks<<<blocks, 256, 0, s>>>(occ, nwx, va.ny, va.nz, surf, inter, counts);
        FGL_LAUNCHED("k_masks");
    }
}

}  // namespace fgl
