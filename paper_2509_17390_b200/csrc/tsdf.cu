// Mesh reconstruction from an occupancy volume on sm_100a — PAPER.md §IV-B,
// SURVEY §8(f) NEXT-3:
//   denoise  : Eq. 13 separable Gaussian blur of V (sigma in metres -> voxels per axis, kernel
//              truncated at ceil(3 sigma), zero outside the grid) + Eq. 14a threshold V' >= tau
//   tsdf     : sign by flood fill from the padded frame (union-find connected components of the
//              free voxels, outside = components touching the grid boundary), S_0 (Eq. 15) and
//              the shells kappa(x) by bitwise 6-neighbour dilation, 32 voxels per word (Eq. 16),
//              phi = clip(s kappa v_min, -r, r) (Eq. 17)
//   mc       : Marching Cubes at iso (Eq. 18): face-consistent cube polygons (table built on the
//              host at first use from the face-walk definition, R34), vertices on
//              crossing edges numbered by global edge id, counts by exclusive scans
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "fgl_internal.cuh"

namespace fgl {

namespace {

// ---- scratch: stream-ordered allocations (capturable in CUDA graphs) -------------------------
// keep freed scratch in the device's default pool (release threshold = max) so a repeated call
// does not re-map memory from the driver every time
void keep_pool() {
    int dev = 0;
    FGL_CUDA(cudaGetDevice(&dev));
    static std::once_flag once[64];
    std::call_once(once[dev & 63], [dev] {
        cudaMemPool_t pool;
        FGL_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = UINT64_MAX;
        FGL_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    });
}

template <class T>
T *salloc(size_t n, cudaStream_t s) {
    keep_pool();
    void *p = nullptr;
    FGL_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s));
    return (T *)p;
}
inline void sfree(void *p, cudaStream_t s) {
    if (p) FGL_CUDA(cudaFreeAsync(p, s));
}

inline unsigned grid1d(int64_t n, int threads = 256, int64_t cap = 148 * 32) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

struct Dims {
    int nx, ny, nz, nwx;
    __host__ __device__ int64_t n() const { return (int64_t)nx * ny * nz; }
    __host__ __device__ int64_t nw() const { return (int64_t)nwx * ny * nz; }
};

// (x, y, z) of linear voxel index i; nx ny nz <= 2^31 (fgl.h), so 32-bit unsigned divisions suffice
// (a 64-bit division is a ~70-instruction software routine)
__device__ __forceinline__ void voxel_xyz(int64_t i, const Dims &d, int &x, int &y, int &z) {
    const uint32_t u = (uint32_t)i, r = u / (uint32_t)d.nx;
    x = (int)(u - r * (uint32_t)d.nx);
    const uint32_t zz = r / (uint32_t)d.ny;
    y = (int)(r - zz * (uint32_t)d.ny), z = (int)zz;
}

__device__ __forceinline__ bool bit_at(const uint32_t *__restrict__ v, const Dims &d, int x, int y, int z) {
    return (v[((int64_t)z * d.ny + y) * d.nwx + (x >> 5)] >> (x & 31)) & 1u;
}

// ---- Eq. 13-14 -------------------------------------------------------------------------------
constexpr int kMaxTaps = 129;  // radius <= 64 voxels
#ifndef FGL_BLUR_TILE
#define FGL_BLUR_TILE 1  // shared-memory tiled y / z blur passes
#endif
struct Taps {
    float w[kMaxTaps];
    int R;
};

// pass 0: bits -> float along x; pass 1, 2: float -> float along y, z. 64 x 4 blocks over
// (x, row = (y, z)), weights read from the parameter bank (staging them in shared memory measured
// slower)
__global__ void __launch_bounds__(256) k_blur(const uint32_t *__restrict__ bits, const float *__restrict__ in,
                                              float *__restrict__ out, Dims d, int axis, Taps t) {
    const int x = blockIdx.x * 64 + threadIdx.x;
    if (x >= d.nx) return;
    for (int row = blockIdx.y * 4 + threadIdx.y; row < d.ny * d.nz; row += gridDim.y * 4) {
        const int y = row % d.ny, z = row / d.ny;
        const int64_t i = (int64_t)row * d.nx + x;
        float acc = 0.f;
        if (axis == 0) {
            const uint32_t *rw = bits + (int64_t)row * d.nwx;
            for (int k = -t.R; k <= t.R; ++k) {
                const int cc = x + k;
                if (cc >= 0 && cc < d.nx && ((__ldg(rw + (cc >> 5)) >> (cc & 31)) & 1u)) acc += t.w[k + t.R];
            }
        } else {
            const int c = axis == 1 ? y : z, n = axis == 1 ? d.ny : d.nz;
            const int64_t stride = axis == 1 ? d.nx : (int64_t)d.nx * d.ny;
            for (int k = -t.R; k <= t.R; ++k) {
                const int cc = c + k;
                if (cc >= 0 && cc < n) acc = fmaf(t.w[k + t.R], __ldg(in + i + (int64_t)k * stride), acc);
            }
        }
        out[i] = acc;
    }
}

// y / z passes, tiled: a 64 x 4 block stages kBlurL output lines of its 64-wide x strip plus the
// 2R halo lines in shared memory (each input read once from global memory instead of 2R + 1 times)
// and sums the taps from there. Same taps, same order, same FMAs as k_blur (a halo line outside
// the volume is staged as 0, and fma(w, 0, acc) = acc for acc >= 0), so the result is identical.
constexpr int kBlurL = 32;
__global__ void __launch_bounds__(256) k_blur_tile(const float *__restrict__ in, float *__restrict__ out, Dims d,
                                                   int axis, Taps t) {
    extern __shared__ float sm[];  // [kBlurL + 2R][64]
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x = blockIdx.x * 64 + tx;
    const int n = axis == 1 ? d.ny : d.nz;
    const int64_t stride = axis == 1 ? d.nx : (int64_t)d.nx * d.ny;
    const int64_t base = axis == 1 ? (int64_t)blockIdx.z * d.nx * d.ny : (int64_t)blockIdx.z * d.nx;
    const int c0 = blockIdx.y * kBlurL, R = t.R, nl = kBlurL + 2 * R;
    for (int l = ty; l < nl; l += 4) {
        const int c = c0 - R + l;
        sm[l * 64 + tx] = (x < d.nx && c >= 0 && c < n) ? __ldg(in + base + (int64_t)c * stride + x) : 0.f;
    }
    __syncthreads();
    if (x >= d.nx) return;
    for (int j = ty; j < kBlurL && c0 + j < n; j += 4) {
        float acc = 0.f;
        for (int k = -R; k <= R; ++k) acc = fmaf(t.w[k + R], sm[(j + k + R) * 64 + tx], acc);
        out[base + (int64_t)(c0 + j) * stride + x] = acc;
    }
}

// x pass from the bit volume, one thread per 32-voxel word (R <= 32, compile time): the word and its
// two neighbours are loaded once, bits outside [0, nx) are cleared, and every tap of every voxel is a
// compile-time bit test + FADD. Same taps in the same order as k_blur (a tap whose bit is 0 or that
// falls outside the row adds nothing there either), so the result is identical. A block covers 256
// consecutive words of the row-major word array, whose voxels form one contiguous output range:
// the outputs are staged in shared memory and written out coalesced.
template <int R>
__global__ void __launch_bounds__(256) k_blur_x(const uint32_t *__restrict__ bits, float *__restrict__ out, Dims d,
                                                Taps t) {
    __shared__ float so[256 * 32];
    const int64_t nw = d.nw();
    const int64_t w0 = (int64_t)blockIdx.x * 256, w = w0 + threadIdx.x;
    float wt[2 * R + 1];
#pragma unroll
    for (int k = 0; k < 2 * R + 1; ++k) wt[k] = t.w[k];
    // output range of the block: voxels of words [w0, w0 + 256) -> [row(w0) nx + x(w0), ...)
    const int64_t row0 = w0 / d.nwx;
    const int64_t o0 = row0 * d.nx + (int64_t)(w0 - row0 * d.nwx) * 32;
    if (w < nw) {
        const int64_t row = w / d.nwx;
        const int q = (int)(w - row * d.nwx);
        const uint32_t *rw = bits + row * d.nwx;
        const int tail = d.nx - 32 * (d.nwx - 1);  // valid bits in a row's last word (1..32)
        const uint32_t last_mask = tail >= 32 ? 0xffffffffu : ((1u << tail) - 1u);
        uint32_t wl = q > 0 ? __ldg(rw + q - 1) : 0u, wc = __ldg(rw + q), wr = q + 1 < d.nwx ? __ldg(rw + q + 1) : 0u;
        if (q == d.nwx - 1) wc &= last_mask;
        if (q + 1 == d.nwx - 1) wr &= last_mask;
        const int64_t ob = row * d.nx + (int64_t)q * 32 - o0;  // offset of this word's voxel 0 in the block range
        const int nv = q == d.nwx - 1 ? tail : 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int k = -R; k <= R; ++k) {
                const int b = j + k;
                const uint32_t word = b < 0 ? wl : (b >= 32 ? wr : wc);
                const int sh = b < 0 ? b + 32 : (b >= 32 ? b - 32 : b);
                if ((word >> sh) & 1u) acc += wt[k + R];
            }
            if (j < nv) so[ob + j] = acc;
        }
    }
    __syncthreads();
    // the block's contiguous output range: up to the voxel after its last word
    const int64_t wl_last = (w0 + 255 < nw ? w0 + 255 : nw - 1);
    const int64_t rowl = wl_last / d.nwx;
    const int ql = (int)(wl_last - rowl * d.nwx);
    const int64_t o1 = rowl * d.nx + (int64_t)ql * 32 + (ql == d.nwx - 1 ? d.nx - 32 * (d.nwx - 1) : 32);
    for (int64_t i = threadIdx.x; i < o1 - o0; i += 256) out[o0 + i] = so[i];
}

// ---- Eq. 14b: Quantile_q(V') by a three-pass radix select over the float bits (V' >= 0, so the
// bit patterns order like the values): 11 + 11 + 10 bits, per-block shared histograms
struct QSel {
    uint32_t prefix;  // selected high bits so far
    uint32_t rank;    // 0-based rank still to find inside the selected bucket
};

__global__ void __launch_bounds__(256) k_qhist(const float *__restrict__ vp, int64_t n, int shift, int bits,
                                               const QSel *__restrict__ sel, uint32_t *__restrict__ ghist) {
    __shared__ uint32_t h[2048];
    const int nb = 1 << bits;
    for (int k = threadIdx.x; k < nb; k += 256) h[k] = 0;
    __syncthreads();
    const uint32_t pre = sel->prefix;
    const int hs = shift + bits;  // bits above this pass must equal the prefix
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = __float_as_uint(__ldg(vp + i));
        if (hs >= 32 || (u >> hs) == pre) atomicAdd(&h[(u >> shift) & (nb - 1)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += 256)
        if (h[k]) atomicAdd(&ghist[k], h[k]);
}

// one block: find the bucket holding the rank, extend the prefix, clear the histogram
__global__ void __launch_bounds__(256) k_qpick(uint32_t *ghist, int bits, QSel *sel) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_bucket, s_before;
    const int nb = 1 << bits, per = nb / 256;  // 8 or 4 buckets per thread
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t c[8], sum = 0;
    for (int k = 0; k < per; ++k) sum += (c[k] = ghist[threadIdx.x * per + k]);
    uint32_t x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int k = 0; k < w; ++k) off += s_w[k];
    uint32_t run = off + x - sum;  // exclusive prefix of this thread's buckets
    const uint32_t r = sel->rank;
    for (int k = 0; k < per; ++k) {
        if (run <= r && r < run + c[k]) s_bucket = threadIdx.x * per + k, s_before = run;
        run += c[k];
    }
    __syncthreads();
    for (int k = 0; k < per; ++k) ghist[threadIdx.x * per + k] = 0u;
    if (threadIdx.x == 0) {
        sel->prefix = (sel->prefix << bits) | s_bucket;
        sel->rank = r - s_before;
    }
}

__global__ void k_qinit(QSel *sel, int64_t n, double q, float *thr_out) {
    // inverted-CDF quantile: the value of 1-based rank max(1, ceil(q n)) in ascending order (R35)
    int64_t k = (int64_t)ceil(q * (double)n);
    if (k < 1) k = 1;
    if (k > n) k = n;
    sel->prefix = 0;
    sel->rank = (uint32_t)(k - 1);
    (void)thr_out;
}

// one warp per output word (its 32 voxels read coalesced, the word is the warp's ballot): V~ = V' >= tau
__device__ __forceinline__ void threshold_words(const float *__restrict__ vp, const Dims &d, float tau,
                                                uint32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < d.nw(); w += nwarps) {
        const int64_t row = w / d.nwx;
        const int x = (int)(w - row * d.nwx) * 32 + lane;
        const bool on = x < d.nx && __ldg(vp + row * d.nx + x) >= tau;
        const uint32_t b = __ballot_sync(0xffffffffu, on);  // padding lanes (x >= nx) vote 0
        if (lane == 0) out[w] = b;
    }
}

__global__ void __launch_bounds__(256) k_threshold_q(const float *__restrict__ vp, Dims d, const QSel *sel,
                                                     uint32_t *__restrict__ out, float *thr_out) {
    const float tau = __uint_as_float(sel->prefix);
    if (thr_out && blockIdx.x == 0 && threadIdx.x == 0) *thr_out = tau;
    threshold_words(vp, d, tau, out);
}

__global__ void __launch_bounds__(256) k_threshold(const float *__restrict__ vp, Dims d, float tau,
                                                   uint32_t *__restrict__ out) {
    threshold_words(vp, d, tau, out);
}

// ---- Eq. 15-17 -------------------------------------------------------------------------------
__device__ __forceinline__ int uf_find(int *lab, int x) {
    int p = __ldcg(lab + x);
    while (p != x) {
        const int g = __ldcg(lab + p);
        if (g != p) atomicCAS(lab + x, p, g);  // path halving (benign race)
        x = p;
        p = g;
    }
    return x;
}

__device__ __forceinline__ void uf_union(int *lab, int a, int b) {
    while (true) {
        a = uf_find(lab, a);
        b = uf_find(lab, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(lab + a, a, b);  // link the larger root under the smaller
        if (old == a) return;
        a = old;
    }
}

// labels start at the first free voxel of each x-run (the run is its own component); one thread
// per voxel, 2-D launch as k_blur
__device__ __forceinline__ bool occ_at(const uint32_t *__restrict__ rw, int x) {
    return (__ldg(rw + (x >> 5)) >> (x & 31)) & 1u;
}
__device__ __forceinline__ int run_start(const uint32_t *__restrict__ rw, int x) {
    // highest occupied voxel below x in the row, + 1 (0 if none)
    int w = x >> 5;
    uint32_t m = __ldg(rw + w) & ((1u << (x & 31)) - 1u);
    while (!m && w > 0) m = __ldg(rw + --w);
    return m ? (w << 5) + (31 - __clz(m)) + 1 : 0;
}

__global__ void __launch_bounds__(256) k_cc_init(const uint32_t *__restrict__ occ, Dims d, int *__restrict__ lab) {
    const int x = blockIdx.x * 64 + threadIdx.x;
    if (x >= d.nx) return;
    for (int row = blockIdx.y * 4 + threadIdx.y; row < d.ny * d.nz; row += gridDim.y * 4) {
        const uint32_t *rw = occ + (int64_t)row * d.nwx;
        const int64_t i = (int64_t)row * d.nx + x;
        lab[i] = occ_at(rw, x) ? -1 : (int)((int64_t)row * d.nx + run_start(rw, x));
    }
}

// The same labels, one warp per row: the start of the run entering each word is a warp prefix max
// over the words' highest occupied voxel, and the row's labels are written coalesced (32 voxels of
// one word per store instruction) instead of one thread per voxel re-scanning the words before it.
__global__ void __launch_bounds__(256) k_cc_init_rows(const uint32_t *__restrict__ occ, Dims d,
                                                      int *__restrict__ lab) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)d.ny * d.nz;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < nrows; row += nwarps) {
        const uint32_t *rw = occ + row * d.nwx;
        int carry = 0;  // (highest occupied voxel before this group of 32 words) + 1, or 0
        for (int q0 = 0; q0 < d.nwx; q0 += 32) {
            const int q = q0 + lane;
            const uint32_t wv = q < d.nwx ? __ldg(rw + q) : 0u;
            int hi = wv ? (q << 5) + 32 - __clz(wv) : 0;  // highest occupied voxel of word q, + 1
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, hi, o);
                if (lane >= o) hi = max(hi, y);
            }
            int before = __shfl_up_sync(kFull, hi, 1);
            before = max(lane == 0 ? 0 : before, carry);  // run start for a voxel with nothing below it in its word
            const int nq = min(32, d.nwx - q0);
            for (int k = 0; k < nq; ++k) {
                const uint32_t wk = __shfl_sync(kFull, wv, k);
                const int bk = __shfl_sync(kFull, before, k);
                const int x = ((q0 + k) << 5) + lane;
                if (x < d.nx) {
                    const uint32_t m = wk & ((1u << lane) - 1u);
                    const int rs = m ? ((q0 + k) << 5) + 32 - __clz(m) : bk;
                    lab[row * d.nx + x] = ((wk >> lane) & 1u) ? -1 : (int)(row * d.nx + rs);
                }
            }
            carry = __shfl_sync(kFull, hi, 31);
        }
    }
}

// union the runs of neighbouring rows (y - 1, z - 1) where they begin to overlap: at x = the later
// of the two run starts, so each overlapping pair of runs is united once
__global__ void __launch_bounds__(256) k_cc_merge(const uint32_t *__restrict__ occ, Dims d, int *lab) {
    const int x = blockIdx.x * 64 + threadIdx.x;
    if (x >= d.nx) return;
    for (int row = blockIdx.y * 4 + threadIdx.y; row < d.ny * d.nz; row += gridDim.y * 4) {
    const int y = row % d.ny, z = row / d.ny;
    const uint32_t *rw = occ + (int64_t)row * d.nwx;
    if (occ_at(rw, x)) continue;
    const int64_t i = (int64_t)row * d.nx + x;
    const bool start = x == 0 || occ_at(rw, x - 1);
    if (y > 0) {
        const uint32_t *rn = rw - d.nwx;
        if (!occ_at(rn, x) && (start || occ_at(rn, x - 1))) uf_union(lab, (int)i, (int)(i - d.nx));
    }
    if (z > 0) {
        const uint32_t *rn = rw - (int64_t)d.nwx * d.ny;
        if (!occ_at(rn, x) && (start || occ_at(rn, x - 1)))
            uf_union(lab, (int)i, (int)(i - (int64_t)d.nx * d.ny));
    }
    }
}

// flatten to roots; free voxels on the grid boundary touch the padded frame: their root is outside
// roots of the run starts (lab[start] = root); free voxels on the grid boundary touch the padded
// frame: their root is outside. Other voxels keep lab = their run start (root = lab[lab[i]]).
__global__ void __launch_bounds__(256) k_cc_flatten(const uint32_t *__restrict__ occ, Dims d, int *lab,
                                                    uint8_t *__restrict__ out_root) {
    const int x = blockIdx.x * 64 + threadIdx.x;
    if (x >= d.nx) return;
    for (int row = blockIdx.y * 4 + threadIdx.y; row < d.ny * d.nz; row += gridDim.y * 4) {
        const uint32_t *rw = occ + (int64_t)row * d.nwx;
        if (occ_at(rw, x)) continue;
        const int y = row % d.ny, z = row / d.ny;
        const bool start = x == 0 || occ_at(rw, x - 1);
        const bool border = x == 0 || y == 0 || z == 0 || x == d.nx - 1 || y == d.ny - 1 || z == d.nz - 1;
        if (!start && !border) continue;
        const int64_t i = (int64_t)row * d.nx + x;
        const int root = uf_find(lab, (int)i);
        if (start) lab[i] = root;
        if (border) out_root[root] = 1;
    }
}

// neighbour words of word w (x: shifted with carries; y, z: whole words, 0 outside the grid)
struct Nb {
    uint32_t c, xm, xp, ym, yp, zm, zp;
};
__device__ __forceinline__ Nb neighbours(const uint32_t *__restrict__ v, const Dims &d, int64_t w) {
    const uint32_t u = (uint32_t)w, r = u / (uint32_t)d.nwx;  // nw <= nx ny nz <= 2^31
    const int wx = (int)(u - r * (uint32_t)d.nwx);
    const int z = (int)(r / (uint32_t)d.ny), y = (int)(r - (uint32_t)z * (uint32_t)d.ny);
    Nb n;
    n.c = v[w];
    n.xm = (n.c << 1) | (wx > 0 ? v[w - 1] >> 31 : 0u);
    n.xp = (n.c >> 1) | (wx + 1 < d.nwx ? v[w + 1] << 31 : 0u);
    n.ym = y > 0 ? v[w - d.nwx] : 0u;
    n.yp = y + 1 < d.ny ? v[w + d.nwx] : 0u;
    const int64_t sl = (int64_t)d.nwx * d.ny;
    n.zm = z > 0 ? v[w - sl] : 0u;
    n.zp = z + 1 < d.nz ? v[w + sl] : 0u;
    return n;
}
__device__ __forceinline__ uint32_t valid_mask(const Dims &d, int64_t w) {
    const int wx = (int)(w % d.nwx);
    const int rem = d.nx - wx * 32;
    return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

// S_0 (Eq. 15, the frame free): kappa = 0 there, 255 elsewhere; vis = S_0
__global__ void __launch_bounds__(256) k_s0(const uint32_t *__restrict__ occ, Dims d, uint32_t *__restrict__ vis,
                                            uint8_t *__restrict__ kappa) {
    // a warp handles 32 consecutive words; the kappa bytes of each word are then written by the 32
    // lanes together (coalesced) instead of 32 scattered byte stores per thread
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31; w0 < d.nw(); w0 += stride) {
        const int64_t w = w0 + lane;
        uint32_t s = 0;
        int64_t base = 0;
        int cnt = 0;
        if (w < d.nw()) {
            const Nb n = neighbours(occ, d, w);
            s = ((n.c ^ n.xm) | (n.c ^ n.xp) | (n.c ^ n.ym) | (n.c ^ n.yp) | (n.c ^ n.zm) | (n.c ^ n.zp)) &
                valid_mask(d, w);
            vis[w] = s;
            const int wx = (int)(w % d.nwx);
            base = (w / d.nwx) * d.nx + wx * 32;
            cnt = min(32, d.nx - wx * 32);
        }
        for (int j = 0; j < 32; ++j) {
            const uint32_t sj = __shfl_sync(0xffffffffu, s, j);
            const int64_t bj = __shfl_sync(0xffffffffu, base, j);
            const int cj = __shfl_sync(0xffffffffu, cnt, j);
            if (lane < cj) kappa[bj + lane] = (sj >> lane) & 1u ? 0 : 255;
        }
    }
}

// one shell (Eq. 16 layered propagation): newly reached voxels get kappa = m
__global__ void __launch_bounds__(256) k_shell(const uint32_t *__restrict__ vin, Dims d, int m,
                                               uint32_t *__restrict__ vout, uint8_t *__restrict__ kappa) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < d.nw(); w += (int64_t)gridDim.x * blockDim.x) {
        const Nb n = neighbours(vin, d, w);
        const uint32_t all = (n.c | n.xm | n.xp | n.ym | n.yp | n.zm | n.zp) & valid_mask(d, w);
        vout[w] = all;
        uint32_t nw = all & ~n.c;
        const int wx = (int)(w % d.nwx);
        const int64_t base = (w / d.nwx) * d.nx + wx * 32;
        while (nw) {
            const int k = __ffs(nw) - 1;
            nw &= nw - 1;
            kappa[base + k] = (uint8_t)m;
        }
    }
}

// Eq. 17: phi = s * min(kappa v_min, r) (float32), s = +1 on outside free voxels
__global__ void __launch_bounds__(256) k_phi(const int *__restrict__ lab, const uint8_t *__restrict__ outside_root,
                                             const uint8_t *__restrict__ kappa, Dims d, float vmin, float r,
                                             float *__restrict__ phi) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n(); i += (int64_t)gridDim.x * blockDim.x) {
        const int l = lab[i];  // run start (or -1), whose label is the component root
        const bool out = l >= 0 && outside_root[lab[l]];
        const int k = kappa[i];
        float dist = k == 255 ? r : __fmul_rn((float)k, vmin);
        dist = fminf(dist, r);
        phi[i] = out ? dist : -dist;
    }
}

// ---- Eq. 18: Marching Cubes table (built once on the host) -----------------------------------
constexpr int kMaxCubeTris = 12, kMaxCent = 2, kMaxLoop = 12;
struct McTable {
    uint8_t ntri[256];
    uint8_t ncent[256];
    uint8_t tri[256][kMaxCubeTris][3];      // 0..11 local edge (rank order), 12 + c = centre vertex c
    uint8_t cent_len[256][kMaxCent];
    uint8_t cent_edges[256][kMaxCent][kMaxLoop];
};
__constant__ McTable c_mc;

// local edge e (rank order (dz, dy, dx, axis) of its lower corner): lower corner and axis
struct LocalEdge {
    int corner, axis;
};

void build_mc_table(McTable &T, LocalEdge (&le)[12]) {
    // corners c = dx + 2 dy + 4 dz; edges = (lower corner with bit a clear, axis a)
    std::vector<std::pair<int, std::pair<int, int>>> es;  // rank key, (corner, axis)
    for (int c = 0; c < 8; ++c)
        for (int a = 0; a < 3; ++a)
            if (!((c >> a) & 1)) {
                const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
                es.push_back({((dz * 2 + dy) * 2 + dx) * 3 + a, {c, a}});
            }
    std::sort(es.begin(), es.end());
    int eidx[8][3];
    for (int e = 0; e < 12; ++e) {
        le[e] = {es[e].second.first, es[e].second.second};
        eidx[le[e].corner][le[e].axis] = e;
    }
    auto edge_of = [&](int a, int b) {  // adjacent corners a, b
        const int lo = a & b, ax = __builtin_ctz(a ^ b);
        return eidx[lo][ax];
    };
    // faces, corners counter-clockwise seen from outside: for axis a, side s, the in-plane axes
    // u = a+1, v = a+2 (mod 3) form a right-handed frame with +a; CCW about the outward normal
    int faces[6][4];
    for (int a = 0; a < 3; ++a)
        for (int s = 0; s < 2; ++s) {
            const int u = (a + 1) % 3, v = (a + 2) % 3;
            const int base = s << a;
            const int q0 = base, q1 = base | (1 << u), q2 = base | (1 << u) | (1 << v), q3 = base | (1 << v);
            int *f = faces[2 * a + s];
            if (s == 1) f[0] = q0, f[1] = q1, f[2] = q2, f[3] = q3;  // CCW about +a
            else f[0] = q0, f[1] = q3, f[2] = q2, f[3] = q1;         // CCW about -a
        }
    auto same_face = [&](int e1, int e2) {
        const int p[4] = {le[e1].corner, le[e1].corner | (1 << le[e1].axis), le[e2].corner,
                          le[e2].corner | (1 << le[e2].axis)};
        for (auto &f : faces) {
            int hit = 0;
            for (int k = 0; k < 4; ++k)
                for (int q = 0; q < 4; ++q)
                    if (p[k] == f[q]) {
                        ++hit;
                        break;
                    }
            if (hit == 4) return true;
        }
        return false;
    };
    memset(&T, 0, sizeof(T));
    for (int cs = 0; cs < 256; ++cs) {
        int nxt[12];
        for (int &x : nxt) x = -1;
        for (auto &f : faces) {
            bool b[4];
            int ni = 0;
            for (int k = 0; k < 4; ++k) ni += (b[k] = (cs >> f[k]) & 1);
            if (ni == 0 || ni == 4) continue;
            for (int s0 = 0; s0 < 4; ++s0) {
                if (!b[s0] || b[(s0 + 3) % 4]) continue;  // a run of inside corners starts at s0
                int t = s0;
                while (b[(t + 1) % 4]) t = (t + 1) % 4;
                const int ein = edge_of(f[(s0 + 3) % 4], f[s0]), eout = edge_of(f[t], f[(t + 1) % 4]);
                if (nxt[ein] != -1) throw Error(4, "marching cubes table: inconsistent face walk");
                nxt[ein] = eout;
            }
        }
        bool used[12] = {};
        int nt = 0, nc = 0;
        for (int e0 = 0; e0 < 12; ++e0) {  // loops start at their lowest-ranked edge
            if (nxt[e0] < 0 || used[e0]) continue;
            int loop[kMaxLoop], m = 0;
            for (int e = e0; !used[e]; e = nxt[e]) {
                if (m == kMaxLoop) throw Error(4, "marching cubes table: loop too long");
                used[e] = true;
                loop[m++] = e;
            }
            bool fan = true;
            for (int k = 2; k <= m - 2; ++k) fan = fan && !same_face(loop[0], loop[k]);
            if (fan) {
                for (int k = 1; k + 1 < m; ++k) {
                    if (nt == kMaxCubeTris) throw Error(4, "marching cubes table: too many triangles");
                    T.tri[cs][nt][0] = (uint8_t)loop[0], T.tri[cs][nt][1] = (uint8_t)loop[k];
                    T.tri[cs][nt][2] = (uint8_t)loop[k + 1];
                    ++nt;
                }
            } else {
                if (nc == kMaxCent) throw Error(4, "marching cubes table: too many centre vertices");
                T.cent_len[cs][nc] = (uint8_t)m;
                for (int k = 0; k < m; ++k) T.cent_edges[cs][nc][k] = (uint8_t)loop[k];
                for (int k = 0; k < m; ++k) {
                    if (nt == kMaxCubeTris) throw Error(4, "marching cubes table: too many triangles");
                    T.tri[cs][nt][0] = (uint8_t)(12 + nc), T.tri[cs][nt][1] = (uint8_t)loop[k];
                    T.tri[cs][nt][2] = (uint8_t)loop[(k + 1) % m];
                    ++nt;
                }
                ++nc;
            }
        }
        T.ntri[cs] = (uint8_t)nt;
        T.ncent[cs] = (uint8_t)nc;
    }
}

struct LocalEdgeArr {
    int8_t corner[12], axis[12];
};
__constant__ LocalEdgeArr c_le;

std::once_flag g_mc_once;
void upload_mc_table() {
    std::call_once(g_mc_once, [] {
        static McTable T;
        LocalEdge le[12];
        build_mc_table(T, le);
        LocalEdgeArr la;
        for (int e = 0; e < 12; ++e) la.corner[e] = (int8_t)le[e].corner, la.axis[e] = (int8_t)le[e].axis;
        FGL_CUDA(cudaMemcpyToSymbol(c_mc, &T, sizeof(T)));
        FGL_CUDA(cudaMemcpyToSymbol(c_le, &la, sizeof(la)));
    });
}

__device__ __forceinline__ int cube_case(const float *__restrict__ phi, const Dims &d, int64_t i, float iso) {
    const int64_t sx = 1, sy = d.nx, sz = (int64_t)d.nx * d.ny;
    int cs = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int64_t o = i + (c & 1) * sx + ((c >> 1) & 1) * sy + ((c >> 2) & 1) * sz;
        if (__ldg(phi + o) < iso) cs |= 1 << c;
    }
    return cs;
}

// per voxel: crossing flags of its +x, +y, +z edges; counts of edge vertices, cube triangles and
// cube centre vertices
__global__ void __launch_bounds__(256) k_mc_count(const float *__restrict__ phi, Dims d, float iso,
                                                  uint8_t *__restrict__ eflag, uint32_t *__restrict__ ecnt,
                                                  uint32_t *__restrict__ tcnt, uint32_t *__restrict__ ccnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n(); i += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        voxel_xyz(i, d, x, y, z);
        const bool in0 = __ldg(phi + i) < iso;
        uint32_t f = 0;
        if (x + 1 < d.nx && ((__ldg(phi + i + 1) < iso) != in0)) f |= 1u;
        if (y + 1 < d.ny && ((__ldg(phi + i + d.nx) < iso) != in0)) f |= 2u;
        if (z + 1 < d.nz && ((__ldg(phi + i + (int64_t)d.nx * d.ny) < iso) != in0)) f |= 4u;
        eflag[i] = (uint8_t)f;
        ecnt[i] = __popc(f);
        uint32_t nt = 0, nc = 0;
        if (x + 1 < d.nx && y + 1 < d.ny && z + 1 < d.nz) {
            const int cs = cube_case(phi, d, i, iso);
            nt = c_mc.ntri[cs];
            nc = c_mc.ncent[cs];
        }
        tcnt[i] = nt;
        ccnt[i] = nc;
    }
}

// ---- exclusive scan of uint32 (three phases; totals in 64 bits) -------------------------------
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long block_excl(unsigned long long v, unsigned long long *s_w,
                                                         unsigned long long &total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    unsigned long long off = 0, tot = 0;
    for (int k = 0; k < kScanThreads / 32; ++k) {
        if (k < w) off += s_w[k];
        tot += s_w[k];
    }
    __syncthreads();
    total = tot;
    return off + x - v;
}

// three arrays scanned together (one pass structure, shared launches)
struct Scan3 {
    uint32_t *a[3];
};

// Blocked layout: thread t of a tile owns the kScanItems consecutive elements [16 t, 16 t + 16),
// read and written as four 128-bit words (arrays are 256-B aligned, tiles 4096 elements); the
// ragged last tile falls back to scalar accesses.
__device__ __forceinline__ void load16(const uint32_t *a, int64_t i, int64_t n, uint32_t (&v)[kScanItems]) {
    if (i + kScanItems <= n) {
        const uint4 *p = reinterpret_cast<const uint4 *>(a + i);
#pragma unroll
        for (int k = 0; k < kScanItems / 4; ++k) {
            const uint4 u = p[k];
            v[4 * k] = u.x, v[4 * k + 1] = u.y, v[4 * k + 2] = u.z, v[4 * k + 3] = u.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = i + k < n ? a[i + k] : 0u;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Scan3 in, int64_t n, unsigned long long *__restrict__ part,
                                                              int nb) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[3][kScanItems];
#pragma unroll
    for (int q = 0; q < 3; ++q) load16(in.a[q], i0, n, v[q]);  // all 12 loads in flight together
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) sum += v[q][k];
        unsigned long long tot;
        block_excl(sum, s_w, tot);
        if (threadIdx.x == 0) part[q * nb + blockIdx.x] = tot;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_parts(unsigned long long *part, int nb,
                                                             unsigned long long *__restrict__ total) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    const int q = blockIdx.x;  // one block per array
    unsigned long long carry = 0;
    for (int b0 = 0; b0 < nb; b0 += kScanThreads) {
        const int idx = b0 + threadIdx.x;
        const unsigned long long v = idx < nb ? part[q * nb + idx] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_excl(v, s_w, tot);
        if (idx < nb) part[q * nb + idx] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) total[q] = carry;
}

// in place: each thread reads its 16 elements before writing them back
__global__ void __launch_bounds__(kScanThreads) k_scan_down(Scan3 io, int64_t n,
                                                            const unsigned long long *__restrict__ part, int nb) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[3][kScanItems];
#pragma unroll
    for (int q = 0; q < 3; ++q) load16(io.a[q], i0, n, v[q]);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) sum += v[q][k];
        unsigned long long tot;
        unsigned long long run = block_excl(sum, s_w, tot) + part[q * nb + blockIdx.x];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t x = v[q][k];
            v[q][k] = (uint32_t)run;
            run += x;
        }
        uint32_t *a = io.a[q];
        if (i0 + kScanItems <= n) {
            uint4 *p = reinterpret_cast<uint4 *>(a + i0);
#pragma unroll
            for (int k = 0; k < kScanItems / 4; ++k)
                p[k] = make_uint4(v[q][4 * k], v[q][4 * k + 1], v[q][4 * k + 2], v[q][4 * k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; ++k)
                if (i0 + k < n) a[i0 + k] = v[q][k];
        }
    }
}

void exclusive_scan3(Scan3 io, int64_t n, unsigned long long *total, unsigned long long *part, cudaStream_t s) {
    const int nb = (int)((n + kScanTile - 1) / kScanTile);
    k_scan_reduce<<<nb, kScanThreads, 0, s>>>(io, n, part, nb);
    FGL_LAUNCHED("k_scan_reduce");
    k_scan_parts<<<3, kScanThreads, 0, s>>>(part, nb, total);
    FGL_LAUNCHED("k_scan_parts");
    k_scan_down<<<nb, kScanThreads, 0, s>>>(io, n, part, nb);
    FGL_LAUNCHED("k_scan_down");
}

struct McArgs {
    float o[3], sp[3];
    float iso;
    int64_t vcap, tcap;
};

__device__ __forceinline__ float grad1(const float *__restrict__ phi, int64_t i, int c, int n, int64_t stride,
                                       float h) {
    if (n < 2) return 0.f;
    if (c == 0) return (__ldg(phi + i + stride) - __ldg(phi + i)) / h;
    if (c == n - 1) return (__ldg(phi + i) - __ldg(phi + i - stride)) / h;
    return (__ldg(phi + i + stride) - __ldg(phi + i - stride)) / (2.f * h);
}

// edge vertices: position p_a + t (p_b - p_a), t = (iso - phi_a) / (phi_b - phi_a); normal =
// normalised interpolated central-difference gradient
__global__ void __launch_bounds__(256) k_mc_verts(const float *__restrict__ phi, Dims d, McArgs a,
                                                  const uint8_t *__restrict__ eflag,
                                                  const uint32_t *__restrict__ ebase, float *__restrict__ verts,
                                                  float *__restrict__ normals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n(); i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = eflag[i];
        if (!f) continue;
        int x, y, z;
        voxel_xyz(i, d, x, y, z);
        const int64_t stride[3] = {1, d.nx, (int64_t)d.nx * d.ny};
        const int c[3] = {x, y, z}, nn[3] = {d.nx, d.ny, d.nz};
        const float pa = __ldg(phi + i);
        float ga[3];
        if (normals)
            for (int q = 0; q < 3; ++q) ga[q] = grad1(phi, i, c[q], nn[q], stride[q], a.sp[q]);
        uint32_t id = ebase[i];
        for (int ax = 0; ax < 3; ++ax) {
            if (!((f >> ax) & 1u)) continue;
            const int64_t j = i + stride[ax];
            const float pb = __ldg(phi + j);
            const float t = (a.iso - pa) / (pb - pa);
            if (id < a.vcap) {
                float p[3];
                for (int q = 0; q < 3; ++q) {
                    const float xa = a.o[q] + ((float)c[q] + 0.5f) * a.sp[q];
                    const float xb = xa + (q == ax ? a.sp[q] : 0.f);
                    p[q] = fmaf(t, xb - xa, xa);
                }
                verts[3 * (int64_t)id] = p[0], verts[3 * (int64_t)id + 1] = p[1], verts[3 * (int64_t)id + 2] = p[2];
                if (normals) {
                    int cb[3] = {x, y, z};
                    cb[ax] += 1;
                    float g[3], l2 = 0.f;
                    for (int q = 0; q < 3; ++q) {
                        const float gb = grad1(phi, j, cb[q], nn[q], stride[q], a.sp[q]);
                        g[q] = fmaf(t, gb - ga[q], ga[q]);
                        l2 = fmaf(g[q], g[q], l2);
                    }
                    const float inv = l2 > 0.f ? rsqrtf(l2) : 0.f;
                    for (int q = 0; q < 3; ++q) normals[3 * (int64_t)id + q] = g[q] * inv;
                }
            }
            ++id;
        }
    }
}

__device__ __forceinline__ uint32_t edge_vertex(const uint8_t *__restrict__ eflag, const uint32_t *__restrict__ ebase,
                                                const Dims &d, int64_t cube, int e) {
    const int corner = c_le.corner[e], ax = c_le.axis[e];
    const int64_t v = cube + (corner & 1) + ((corner >> 1) & 1) * (int64_t)d.nx +
                      ((corner >> 2) & 1) * (int64_t)d.nx * d.ny;
    const uint32_t f = eflag[v];
    return ebase[v] + __popc(f & ((1u << ax) - 1u));
}

// triangles of every cube (table order), centre vertices appended after the edge vertices
__global__ void __launch_bounds__(256) k_mc_tris(const float *__restrict__ phi, Dims d, McArgs a,
                                                 const uint8_t *__restrict__ eflag,
                                                 const uint32_t *__restrict__ ebase,
                                                 const uint32_t *__restrict__ tbase,
                                                 const uint32_t *__restrict__ cbase,
                                                 const unsigned long long *__restrict__ nedge,
                                                 float *__restrict__ verts, float *__restrict__ normals,
                                                 int32_t *__restrict__ tris) {
    const uint32_t ne = (uint32_t)*nedge;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.n(); i += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        voxel_xyz(i, d, x, y, z);
        if (x + 1 >= d.nx || y + 1 >= d.ny || z + 1 >= d.nz) continue;
        const int cs = cube_case(phi, d, i, a.iso);
        const int nt = c_mc.ntri[cs];
        if (!nt) continue;
        const int nc = c_mc.ncent[cs];
        const uint32_t c0 = ne + cbase[i];
        for (int c = 0; c < nc; ++c) {  // centre vertex = mean of its loop's vertices
            const int m = c_mc.cent_len[cs][c];
            float p[3] = {0.f, 0.f, 0.f}, nrm[3] = {0.f, 0.f, 0.f};
            for (int k = 0; k < m; ++k) {
                const uint32_t v = edge_vertex(eflag, ebase, d, i, c_mc.cent_edges[cs][c][k]);
                for (int q = 0; q < 3; ++q) {
                    p[q] += verts[3 * (int64_t)v + q];
                    if (normals) nrm[q] += normals[3 * (int64_t)v + q];
                }
            }
            const uint32_t id = c0 + c;
            if (id < a.vcap) {
                for (int q = 0; q < 3; ++q) verts[3 * (int64_t)id + q] = p[q] / (float)m;
                if (normals) {
                    const float l2 = nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2];
                    const float inv = l2 > 0.f ? rsqrtf(l2) : 0.f;
                    for (int q = 0; q < 3; ++q) normals[3 * (int64_t)id + q] = nrm[q] * inv;
                }
            }
        }
        uint32_t t = tbase[i];
        for (int k = 0; k < nt; ++k, ++t) {
            if (t >= a.tcap) break;
            for (int q = 0; q < 3; ++q) {
                const int ref = c_mc.tri[cs][k][q];
                tris[3 * (int64_t)t + q] = (int32_t)(ref < 12 ? edge_vertex(eflag, ebase, d, i, ref) : c0 + (ref - 12));
            }
        }
    }
}

__global__ void k_mc_totals(const unsigned long long *ne, const unsigned long long *nt, const unsigned long long *nc,
                            int64_t *counts) {
    counts[0] = (int64_t)(*ne + *nc);
    counts[1] = (int64_t)*nt;
}

}  // namespace

// ---- launchers ---------------------------------------------------------------------------------
// 64 x 4 thread blocks over (x, row = (y, z)) for the row-wise kernels
static dim3 grid2d(const Dims &d) {
    return dim3((d.nx + 63) / 64, std::min((d.ny * d.nz + 3) / 4, 65535));
}

static Dims mkdims(const int *dims) {
    Dims d;
    d.nx = dims[0], d.ny = dims[1], d.nz = dims[2];
    d.nwx = (d.nx + 31) / 32;
    return d;
}

void launch_denoise(const uint32_t *occ, const int *dims, const float *spacing, float sigma, float tau,
                    uint32_t *out, float *vprime, cudaStream_t s, int quantile, float *thr_out) {
    const Dims d = mkdims(dims);
    float *a = salloc<float>(d.n(), s), *b = salloc<float>(d.n(), s);
    float *vp = vprime ? vprime : salloc<float>(d.n(), s);
    const float *src = nullptr;
    float *dst[3] = {a, b, vp};
    for (int ax = 0; ax < 3; ++ax) {
        Taps t;
        const double sv = (double)sigma / (double)spacing[ax];
        t.R = std::max(1, (int)std::ceil(3.0 * sv));
        if (2 * t.R + 1 > kMaxTaps) throw Error(1, "denoise: sigma exceeds 21 voxels");
        double sum = 0;
        for (int k = -t.R; k <= t.R; ++k) sum += std::exp(-0.5 * (k / sv) * (k / sv));
        for (int k = -t.R; k <= t.R; ++k) t.w[k + t.R] = (float)(std::exp(-0.5 * (k / sv) * (k / sv)) / sum);
        const int other = ax == 1 ? d.nz : d.ny;
        if (ax > 0 && other <= 65535 && FGL_BLUR_TILE) {
            const int n = ax == 1 ? d.ny : d.nz;
            const dim3 g((d.nx + 63) / 64, (n + kBlurL - 1) / kBlurL, other);
            const size_t smem = sizeof(float) * 64 * (kBlurL + 2 * t.R);
            if (smem > 48 * 1024)
                FGL_CUDA(cudaFuncSetAttribute(k_blur_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_blur_tile<<<g, dim3(64, 4), smem, s>>>(src, dst[ax], d, ax, t);
            FGL_LAUNCHED("k_blur_tile");
        } else if (ax == 0 && t.R <= 4 && FGL_BLUR_TILE) {
            const unsigned nb = (unsigned)((d.nw() + 255) / 256);
            switch (t.R) {
                case 1: k_blur_x<1><<<nb, 256, 0, s>>>(occ, dst[ax], d, t); break;
                case 2: k_blur_x<2><<<nb, 256, 0, s>>>(occ, dst[ax], d, t); break;
                case 3: k_blur_x<3><<<nb, 256, 0, s>>>(occ, dst[ax], d, t); break;
                default: k_blur_x<4><<<nb, 256, 0, s>>>(occ, dst[ax], d, t); break;
            }
            FGL_LAUNCHED("k_blur_x");
        } else {
            k_blur<<<grid2d(d), dim3(64, 4), 0, s>>>(occ, src, dst[ax], d, ax, t);
            FGL_LAUNCHED("k_blur");
        }
        src = dst[ax];
    }
    if (!quantile) {
        k_threshold<<<grid1d(d.nw() * 32), 256, 0, s>>>(vp, d, tau, out);
        FGL_LAUNCHED("k_threshold");
        if (thr_out) FGL_CUDA(cudaMemcpyAsync(thr_out, &tau, sizeof(float), cudaMemcpyHostToDevice, s));
    } else {  // tau is the quantile level q (Eq. 14b)
        QSel *sel = salloc<QSel>(1, s);
        uint32_t *gh = salloc<uint32_t>(2048, s);
        FGL_CUDA(cudaMemsetAsync(gh, 0, 2048 * sizeof(uint32_t), s));
        k_qinit<<<1, 1, 0, s>>>(sel, d.n(), (double)tau, thr_out);
        FGL_LAUNCHED("k_qinit");
        const int pass_shift[3] = {21, 10, 0}, pass_bits[3] = {11, 11, 10};
        for (int p = 0; p < 3; ++p) {
            k_qhist<<<grid1d(d.n(), 256, 148 * 8), 256, 0, s>>>(vp, d.n(), pass_shift[p], pass_bits[p], sel, gh);
            FGL_LAUNCHED("k_qhist");
            k_qpick<<<1, 256, 0, s>>>(gh, pass_bits[p], sel);
            FGL_LAUNCHED("k_qpick");
        }
        k_threshold_q<<<grid1d(d.nw() * 32), 256, 0, s>>>(vp, d, sel, out, thr_out);
        FGL_LAUNCHED("k_threshold_q");
        sfree(sel, s), sfree(gh, s);
    }
    sfree(a, s), sfree(b, s);
    if (!vprime) sfree(vp, s);
}

void launch_tsdf(const uint32_t *occ, const int *dims, const float *spacing, float r, float *phi, cudaStream_t s) {
    const Dims d = mkdims(dims);
    int *lab = salloc<int>(d.n(), s);
    uint8_t *oroot = salloc<uint8_t>(d.n(), s), *kappa = salloc<uint8_t>(d.n(), s);
    uint32_t *v0 = salloc<uint32_t>(d.nw(), s), *v1 = salloc<uint32_t>(d.nw(), s);
    FGL_CUDA(cudaMemsetAsync(oroot, 0, d.n(), s));
    const dim3 g2 = grid2d(d);
    if (FGL_BLUR_TILE)
        k_cc_init_rows<<<grid1d((int64_t)d.ny * d.nz * 32), 256, 0, s>>>(occ, d, lab);
    else
        k_cc_init<<<g2, dim3(64, 4), 0, s>>>(occ, d, lab);
    FGL_LAUNCHED("k_cc_init");
    k_cc_merge<<<g2, dim3(64, 4), 0, s>>>(occ, d, lab);
    FGL_LAUNCHED("k_cc_merge");
    k_cc_flatten<<<g2, dim3(64, 4), 0, s>>>(occ, d, lab, oroot);
    FGL_LAUNCHED("k_cc_flatten");
    k_s0<<<grid1d(d.nw()), 256, 0, s>>>(occ, d, v0, kappa);
    FGL_LAUNCHED("k_s0");
    const float vmin = std::min(spacing[0], std::min(spacing[1], spacing[2]));
    const int m_max = (int)std::ceil((double)r / (double)vmin);
    if (m_max > 254) throw Error(1, "tsdf: band r / v_min must be <= 254 shells");
    for (int m = 1; m <= m_max; ++m) {
        k_shell<<<grid1d(d.nw()), 256, 0, s>>>(v0, d, m, v1, kappa);
        FGL_LAUNCHED("k_shell");
        std::swap(v0, v1);
    }
    k_phi<<<grid1d(d.n()), 256, 0, s>>>(lab, oroot, kappa, d, vmin, r, phi);
    FGL_LAUNCHED("k_phi");
    sfree(lab, s), sfree(oroot, s), sfree(kappa, s), sfree(v0, s), sfree(v1, s);
}

void launch_marching_cubes(const float *phi, const int *dims, const float *origin, const float *spacing, float iso,
                           float *verts, float *normals, int64_t vcap, int32_t *tris, int64_t tcap, int64_t *counts,
                           cudaStream_t s) {
    upload_mc_table();
    const Dims d = mkdims(dims);
    const int64_t n = d.n();
    uint8_t *eflag = salloc<uint8_t>(n, s);
    uint32_t *ecnt = salloc<uint32_t>(n, s), *tcnt = salloc<uint32_t>(n, s), *ccnt = salloc<uint32_t>(n, s);
    const int nb = (int)((n + kScanTile - 1) / kScanTile);
    unsigned long long *part = salloc<unsigned long long>(3 * (size_t)nb, s), *tot = salloc<unsigned long long>(3, s);
    k_mc_count<<<grid1d(n), 256, 0, s>>>(phi, d, iso, eflag, ecnt, tcnt, ccnt);
    FGL_LAUNCHED("k_mc_count");
    Scan3 io;
    io.a[0] = ecnt, io.a[1] = tcnt, io.a[2] = ccnt;
    exclusive_scan3(io, n, tot, part, s);
    McArgs a;
    for (int q = 0; q < 3; ++q) a.o[q] = origin[q], a.sp[q] = spacing[q];
    a.iso = iso, a.vcap = verts ? vcap : 0, a.tcap = tris ? tcap : 0;
    if (a.vcap > 0) {
        k_mc_verts<<<grid1d(n), 256, 0, s>>>(phi, d, a, eflag, ecnt, verts, normals);
        FGL_LAUNCHED("k_mc_verts");
    }
    if (a.vcap > 0 || a.tcap > 0) {
        k_mc_tris<<<grid1d(n), 256, 0, s>>>(phi, d, a, eflag, ecnt, tcnt, ccnt, tot, verts, normals, tris);
        FGL_LAUNCHED("k_mc_tris");
    }
    if (counts) {
        k_mc_totals<<<1, 1, 0, s>>>(tot + 0, tot + 1, tot + 2, counts);
        FGL_LAUNCHED("k_mc_totals");
    }
    sfree(eflag, s), sfree(ecnt, s), sfree(tcnt, s), sfree(ccnt, s), sfree(part, s), sfree(tot, s);
}

}  // namespace fgl
