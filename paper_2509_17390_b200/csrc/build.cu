// LBVH construction over triangles on sm_100a — PAPER.md §IV-A "BVH Construction",
// applied to the cast's triangle mesh (R8):
//   prep     : triangle centroids (the Morton point) + exact scene box [o, o+L] (last-block reduce)
//   morton   : Eq. 5 codes, b bits per axis, x lowest, + the all-pass digit histogram
//   sort     : stable LSD radix sort (sort.cu), "radix sort run massively in parallel"
//   lbvh     : DEFAULT width-2 path, one kernel (k_lbvh): leaf records + Eq. 6 tree + Eq. 7 boxes +
//              node64, built bottom-up in shared memory per chunk of sorted leaves and by the last
//              CTA of each group of chunks above them (see the k_lbvh section); the steps below
//              are the path of the other node widths and of the restructuring passes:
//   reorder  : triangle records (tri48) gathered into sorted (leaf) order
//   karras   : Eq. 6 LCP-split binary radix tree, one thread per internal node,
//              "bitwise operations ... without recursion"
//   refit    : Eq. 7 by its closed form: each node's box is the exact union of its
//              sorted leaf range, read from 8-ary box aggregates (no bottom-up climb)
//   nodes    : traversal nodes (both child boxes per node; subtrees of <= leaf_size triangles
//              become leaves), laid out in Karras (Morton) order ("Morton order").
#include <cstdlib>

#include <cuda/atomic>

#include "fgl_internal.cuh"

#ifndef FGL_SORT_PACKED
#define FGL_SORT_PACKED 1
#endif
#ifndef FGL_TREELET4
#define FGL_TREELET4 1  // parallel restructuring: exhaustive 4-leaf treelets (0: greedy 8-leaf treelets)
#endif
#ifndef FGL_RANGEBOX_DYN
#define FGL_RANGEBOX_DYN 0  // 1: Eq. 7 closed form by loops with exact trip counts (measured slower)
#endif
#ifndef FGL_FUSED_LBVH
#define FGL_FUSED_LBVH 1  // width 2: one bottom-up kernel for leaf records, tree, boxes and node64 (k_lbvh)
#endif
#ifndef FGL_FUSED_NODES
#define FGL_FUSED_NODES 0  // 1: k_karras writes the binary traversal nodes (no separate k_nodes pass)
#endif

namespace fgl {

namespace {

__global__ void k_validate(const float *__restrict__ verts, int64_t V, const int32_t *__restrict__ tris, int64_t T,
                           unsigned int *flag) {
    // 16-byte loads over the (cudaMalloc-aligned, scene-owned) arrays, scalar tails
    unsigned int bad = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt4 = 3 * T / 4, nv4 = 3 * V / 4;
    const int4 *t4 = reinterpret_cast<const int4 *>(tris);
    const float4 *v4 = reinterpret_cast<const float4 *>(verts);
    for (int64_t i = t0; i < nt4; i += stride) {
        const int4 x = t4[i];
        if ((unsigned)x.x >= (uint64_t)V || (unsigned)x.y >= (uint64_t)V || (unsigned)x.z >= (uint64_t)V ||
            (unsigned)x.w >= (uint64_t)V)
            bad |= 1u;
    }
    for (int64_t i = 4 * nt4 + t0; i < 3 * T; i += stride)
        if ((unsigned)tris[i] >= (uint64_t)V) bad |= 1u;
    for (int64_t i = t0; i < nv4; i += stride) {
        const float4 x = v4[i];
        if (!(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w))) bad |= 2u;
    }
    for (int64_t i = 4 * nv4 + t0; i < 3 * V; i += stride)
        if (!isfinite(verts[i])) bad |= 2u;
    if (bad) atomicOr(flag, bad);
}

// vertex gather with the index clamped to [0, V) (memory-safe before validation is checked)
__device__ __forceinline__ int32_t clampv(int32_t i, int64_t V) { return i < 0 ? 0 : (i >= V ? (int32_t)(V - 1) : i); }

// 12-byte rows by one 8-byte and one 4-byte load (row i starts 8-byte aligned iff i is even; the base
// is cudaMalloc-aligned)
__device__ __forceinline__ float3 ldv2(const float *__restrict__ verts, int32_t i) {
    const float *p = verts + 3 * (int64_t)i;
    if (i & 1) {
        const float2 yz = __ldg(reinterpret_cast<const float2 *>(p + 1));
        return make_float3(__ldg(p), yz.x, yz.y);
    }
    const float2 xy = __ldg(reinterpret_cast<const float2 *>(p));
    return make_float3(xy.x, xy.y, __ldg(p + 2));
}
__device__ __forceinline__ int3 ldtri(const int32_t *__restrict__ tris, int64_t k) {
    const int32_t *p = tris + 3 * k;
    if (k & 1) {
        const int2 yz = __ldg(reinterpret_cast<const int2 *>(p + 1));
        return make_int3(__ldg(p), yz.x, yz.y);
    }
    const int2 xy = __ldg(reinterpret_cast<const int2 *>(p));
    return make_int3(xy.x, xy.y, __ldg(p + 2));
}

__device__ __forceinline__ float3 ldv(const float *__restrict__ verts, int32_t i) {
    return make_float3(__ldg(verts + 3 * (int64_t)i), __ldg(verts + 3 * (int64_t)i + 1), __ldg(verts + 3 * (int64_t)i + 2));
}

// centroid c = ((v0 + v1) + v2) / 3, float32 round-to-nearest, no contraction (R8)
__device__ __forceinline__ float centroid1(float a, float b, float c) {
    return __fdiv_rn(__fadd_rn(__fadd_rn(a, b), c), 3.0f);
}

__device__ __forceinline__ float warp_min(float v) {
    for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(256) k_prep(const float *__restrict__ verts, int64_t V,
                                              const int32_t *__restrict__ tris,
                                              int64_t T, float4 *__restrict__ cent, float *__restrict__ partial,
                                              unsigned int *sync, float *__restrict__ box) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i0 = clampv(__ldg(tris + 3 * k), V), i1 = clampv(__ldg(tris + 3 * k + 1), V),
                      i2 = clampv(__ldg(tris + 3 * k + 2), V);
        float3 a = ldv(verts, i0), b = ldv(verts, i1), c = ldv(verts, i2);
        float4 m = make_float4(centroid1(a.x, b.x, c.x), centroid1(a.y, b.y, c.y), centroid1(a.z, b.z, c.z), 0.f);
        cent[k] = m;
        lo[0] = fminf(lo[0], m.x), lo[1] = fminf(lo[1], m.y), lo[2] = fminf(lo[2], m.z);
        hi[0] = fmaxf(hi[0], m.x), hi[1] = fmaxf(hi[1], m.y), hi[2] = fmaxf(hi[2], m.z);
    }
    __shared__ float s[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < 3; ++i) {
        lo[i] = warp_min(lo[i]);
        hi[i] = warp_max(hi[i]);
    }
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
    // last block: reduce all partials (L2 reads, every thread's loads in flight at once — a single
    // warp looping over them paid ~28 dependent L2 round trips per component, most of k_prep at 1 M
    // triangles), publish the box, reset the counter
    float r[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = i < 3 ? INFINITY : -INFINITY;
#pragma unroll
    for (int q = 0; q < (kPrepBlocks + 255) / 256; ++q) {
        const int b = threadIdx.x + q * (int)blockDim.x;
        if (b < (int)gridDim.x) {
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const float x = __ldcg(partial + b * 6 + i);
                r[i] = i < 3 ? fminf(r[i], x) : fmaxf(r[i], x);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = i < 3 ? warp_min(r[i]) : warp_max(r[i]);
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
    if (threadIdx.x == 0) *sync = 0u, sync[2] = 0u, sync[3] += 1u;  // k_lbvh: [2] pending count, [3] slot epoch
}

// spread the low 21 bits of x to every third bit (bit i -> bit 3i)
__device__ __forceinline__ uint64_t spread3(uint32_t x) {
    uint64_t v = x & 0x1fffffu;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

// Eq. 5 quantisation in float32 (the decision is a float one; R7):
// L = hi - lo (cubic box, R22: L = max over axes for every axis); s = L > 0 ? 2^b / L : 0;
// q = min(floor((c - lo) * s), 2^b - 1)
struct MortonBox {
    float lo[3], s[3];
    uint32_t qmax;
};

__device__ __forceinline__ MortonBox morton_box(const float *lo, const float *hi, int bits, int cubic = 0) {
    MortonBox m;
    const float two_b = (float)(1u << bits);
    m.qmax = (1u << bits) - 1u;
    float L[3], Lc = 0.f;
    for (int i = 0; i < 3; ++i) {
        L[i] = __fsub_rn(hi[i], lo[i]);
        Lc = fmaxf(Lc, L[i]);
    }
    for (int i = 0; i < 3; ++i) {
        m.lo[i] = lo[i];
        const float Li = cubic ? Lc : L[i];
        m.s[i] = Li > 0.f ? __fdiv_rn(two_b, Li) : 0.f;
    }
    return m;
}

__device__ __forceinline__ uint64_t morton_code(const MortonBox &m, float x, float y, float z) {
    float c[3] = {x, y, z};
    uint32_t q[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        float f = floorf(__fmul_rn(__fsub_rn(c[i], m.lo[i]), m.s[i]));
        q[i] = f >= (float)m.qmax ? m.qmax : (uint32_t)f;
    }
    return spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
}

// keys[k] = code (vals[k] = k), or packed (vals == nullptr): keys[k] = code << pshift | k
__global__ void __launch_bounds__(256) k_morton(const float4 *__restrict__ cent, int64_t T,
                                                const float *__restrict__ box, int bits, int cubic,
                                                uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                                                int pshift, uint32_t *__restrict__ ghist) {
    __shared__ uint32_t h[8][256];
    __shared__ MortonBox mb;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    if (threadIdx.x == 0) mb = morton_box(box, box + 3, bits, cubic);
    __syncthreads();
    const int npass = (3 * bits + 7) / 8;
    const MortonBox m = mb;
    // (warp-aggregating the digit counts — one atomic when the whole warp shares a digit, or per
    // match_any group — measured slower: 115-120 vs 87 us at 10 M keys)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T; k += (int64_t)gridDim.x * blockDim.x) {
        float4 c = cent[k];
        uint64_t code = morton_code(m, c.x, c.y, c.z);
        if (vals) {
            keys[k] = code;
            vals[k] = (uint32_t)k;
        } else {
            keys[k] = code << pshift | (uint64_t)k;
        }
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(code >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

struct BoxArg {
    float lo[3], hi[3];
};

__global__ void k_morton_points(const float *__restrict__ pts, int64_t n, BoxArg bx, int bits,
                                uint64_t *__restrict__ codes) {
    const MortonBox m = morton_box(bx.lo, bx.hi, bits);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        codes[k] = morton_code(m, pts[3 * k], pts[3 * k + 1], pts[3 * k + 2]);
}

// LCP of augmented keys code_i || i (sorted position fallback for equal codes; R7); -1 outside.
// ki = k[i] is passed in (loaded once per thread).
// With packed keys (code << ks | index), ks strips the index: the tree is the same either way.
// 32-bit positions (T < 2^30); one unsigned compare covers both ends of [0, n).
__device__ __forceinline__ int delta(const uint64_t *__restrict__ k, int n, int i, uint64_t ki, int j, int ks) {
    if ((unsigned)j >= (unsigned)n) return -1;
    const uint64_t x = ki ^ (__ldg(k + j) >> ks);
    return x ? __clzll((long long)x) : 64 + __clz(i ^ j);
}

constexpr float kInf = __builtin_huge_valf();
constexpr int kMaxAgg = 10;  // 8^10 > 2^28 triangles
// level 0 = leaf boxes [n]; levels 1..nlev-1 = unions of 8^k consecutive leaves, stored one after
// the other in `agg` (level k has ceil(n / 8^k) entries)
struct AggLevels {
    const float4 *leaf, *agg;
    int64_t n;
    int nlev;
};

__device__ __forceinline__ void acc(float4 &lo, float4 &hi, const float4 *p, int i) {
    const float4 l = __ldg(p + 2 * i), h = __ldg(p + 2 * i + 1);
    lo.x = fminf(lo.x, l.x), lo.y = fminf(lo.y, l.y), lo.z = fminf(lo.z, l.z);
    hi.x = fmaxf(hi.x, h.x), hi.y = fmaxf(hi.y, h.y), hi.z = fmaxf(hi.z, h.z);
}

// Eq. 7 by its closed form: the box of a node covering sorted leaves [a, b] is the union of their
// boxes (exact: min/max do not round). Evaluated with the 8-ary aggregates: at most 7 + 7 reads per
// level (independent loads, unrolled), <= 8 at the top level.
__device__ __forceinline__ void range_box(const AggLevels &L, int a, int b, float4 &lo, float4 &hi) {
    lo = make_float4(kInf, kInf, kInf, 0.f), hi = make_float4(-kInf, -kInf, -kInf, 0.f);
    int A = a, B = b + 1;  // half-open, in units of the current level
    int cnt = (int)L.n, off = -1;
    for (int lv = 0; lv < L.nlev && A < B; ++lv) {
        const float4 *p = lv == 0 ? L.leaf : L.agg + 2 * off;
        off = lv == 0 ? 0 : off + cnt;
        cnt = (cnt + 7) >> 3;
        if (lv + 1 < L.nlev) {
            const int rem = B - A;
            const int nf = min((8 - (A & 7)) & 7, rem);
#if FGL_RANGEBOX_DYN
            // loops with the exact trip count: a predicated-off unrolled copy still takes an issue slot
            for (int k = 0; k < nf; ++k) acc(lo, hi, p, A + k);
#else
#pragma unroll
            for (int k = 0; k < 7; ++k)
                if (k < nf) acc(lo, hi, p, A + k);
#endif
            A += nf;
            const int nb = min(B & 7, B - A);
#if FGL_RANGEBOX_DYN
            for (int k = 0; k < nb; ++k) acc(lo, hi, p, B - 1 - k);
#else
#pragma unroll
            for (int k = 0; k < 7; ++k)
                if (k < nb) acc(lo, hi, p, B - 1 - k);
#endif
            B -= nb;
            A >>= 3, B >>= 3;
        } else {
#if FGL_RANGEBOX_DYN
            for (int k = A; k < B; ++k) acc(lo, hi, p, k);
#else
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (A + k < B) acc(lo, hi, p, A + k);
#endif
        }
    }
}

// Karras 2012 (Eq. 6 read as the non-recursive LCP split, R7): one thread per internal node i.
// nodes != nullptr (binary traversal nodes wanted, no restructuring): the thread evaluates Eq. 7 for
// its two children (the ranges [f, g] and [g + 1, l] it has just found) instead of for itself, writes
// its own box as their union, and writes its node64 directly — the separate k_nodes pass, a gather of
// both children's boxes per node, disappears.
__global__ void __launch_bounds__(256) k_karras(const uint64_t *__restrict__ k, int n, int ks,
                                                int2 *__restrict__ child, int2 *__restrict__ range,
                                                int32_t *__restrict__ parent, AggLevels L,
                                                float4 *__restrict__ nodebox, Node64 *__restrict__ nodes,
                                                int leaf_size) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // one thread per internal node
    if (i < n - 1) {
        const uint64_t ki = __ldg(k + i) >> ks;
        const int d = (delta(k, n, i, ki, i + 1, ks) - delta(k, n, i, ki, i - 1, ks)) >= 0 ? 1 : -1;
        const int dmin = delta(k, n, i, ki, i - d, ks);
        int lmax = 2;
        while (delta(k, n, i, ki, i + lmax * d, ks) > dmin) lmax <<= 1;
        int l = 0;
        for (int t = lmax >> 1; t >= 1; t >>= 1)
            if (delta(k, n, i, ki, i + (l + t) * d, ks) > dmin) l += t;
        const int j = i + l * d;
        const int dnode = delta(k, n, i, ki, j, ks);
        int s = 0, t = l;
        do {
            t = (t + 1) >> 1;
            if (delta(k, n, i, ki, i + (s + t) * d, ks) > dnode) s += t;
        } while (t > 1);
        const int g = i + s * d + (d < 0 ? -1 : 0);
        const int f = i < j ? i : j, last = i < j ? j : i;
        int32_t left = f == g ? ~g : g;
        int32_t right = last == g + 1 ? ~(g + 1) : g + 1;
        child[i] = make_int2(left, right);
        range[i] = make_int2(f, last);
        parent[left >= 0 ? left : (n - 1) + ~left] = i;
        parent[right >= 0 ? right : (n - 1) + ~right] = i;
        if (i == 0) parent[0] = -1;
#if FGL_FUSED_NODES
        if (nodes) {
            // Eq. 7 boxes of both children by the closed form (exact unions of their leaf ranges)
            float4 l0, h0, l1, h1;
            range_box(L, f, g, l0, h0);
            range_box(L, g + 1, last, l1, h1);
            nodebox[2 * i] = make_float4(fminf(l0.x, l1.x), fminf(l0.y, l1.y), fminf(l0.z, l1.z), 0.f);
            nodebox[2 * i + 1] = make_float4(fmaxf(h0.x, h1.x), fmaxf(h0.y, h1.y), fmaxf(h0.z, h1.z), 0.f);
            const int32_t n0 = g - f + 1, n1 = last - g;
            Node64 nd;
            nd.a = make_float4(l0.x, h0.x, l0.y, h0.y);
            nd.b = make_float4(l1.x, h1.x, l1.y, h1.y);
            nd.c = make_float4(l0.z, h0.z, l1.z, h1.z);
            nd.d = make_int4(n0 <= leaf_size ? make_leaf(f, n0) : left, n1 <= leaf_size ? make_leaf(g + 1, n1) : right,
                             0, 0);
            nodes[i] = nd;
            return;
        }
#endif
        // Eq. 7 box of this node by its closed form (exact union of its leaf range)
        float4 lo, hi;
        range_box(L, f, last, lo, hi);
        nodebox[2 * i] = lo;
        nodebox[2 * i + 1] = hi;
    }
}

// Refit (dynamic meshes): Eq. 7 boxes of every internal node from its stored leaf
// range over the new leaf boxes; the topology (Morton order, Karras tree) is kept.
__global__ void __launch_bounds__(256) k_refit_boxes(int n, const int2 *__restrict__ range, AggLevels L,
                                                     float4 *__restrict__ nodebox) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int2 r = range[i];
    float4 lo, hi;
    range_box(L, r.x, r.y, lo, hi);
    nodebox[2 * i] = lo;
    nodebox[2 * i + 1] = hi;
}

// ---- NEXT-4: agglomerative treelet restructuring (after Karras & Aila 2013, Domingues & Pedrini
// 2015) -------------------------------------------------------------------------------------------
// Bottom-up over the binary tree (one thread per leaf climbing; the second thread to reach a node
// processes it, so a node is handled after both subtrees). At every node whose subtree holds >= 7
// leaves, a treelet of up to 7 leaves is formed by repeatedly opening the treelet leaf with the
// largest surface area; the treelet is re-clustered greedily (merge the pair whose union has the
// smallest area) and the new topology is kept when it lowers the SAH cost
// C(n) = C_i A(n) + C(left) + C(right), C(leaf) = C_t A(leaf). The node boxes stay exact unions.
// Leaves are single triangles (a treelet may regroup any of them).
constexpr float kCi = 1.2f, kCt = 1.0f;
constexpr int kTreeletLeaves = 7;

__device__ __forceinline__ float area(const float4 &lo, const float4 &hi) {
    const float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
    return 2.f * (dx * dy + dy * dz + dz * dx);
}

struct TRef {
    int32_t ref;  // internal node index, or ~leaf
    float4 lo, hi;
    float cost;
    int32_t size;
};

__device__ __forceinline__ void load_ref(TRef &t, int32_t ref, const float4 *nodebox, const float4 *leafbox,
                                         const float *cost, const int32_t *size) {
    t.ref = ref;
    if (ref >= 0) {
        t.lo = __ldcg(nodebox + 2 * (int64_t)ref), t.hi = __ldcg(nodebox + 2 * (int64_t)ref + 1);
        t.cost = __ldcg(cost + ref), t.size = __ldcg(size + ref);
    } else {
        t.lo = __ldg(leafbox + 2 * (int64_t)~ref), t.hi = __ldg(leafbox + 2 * (int64_t)~ref + 1);
        t.cost = kCt * area(t.lo, t.hi), t.size = 1;
    }
}

__device__ __forceinline__ void unite(float4 &lo, float4 &hi, const float4 &l2, const float4 &h2) {
    lo.x = fminf(lo.x, l2.x), lo.y = fminf(lo.y, l2.y), lo.z = fminf(lo.z, l2.z);
    hi.x = fmaxf(hi.x, h2.x), hi.y = fmaxf(hi.y, h2.y), hi.z = fmaxf(hi.z, h2.z);
}

__device__ void treelet_node(int32_t n, int32_t T, int2 *child, int32_t *parent, float4 *nodebox,
                             const float4 *leafbox, float *cost, int32_t *size, bool restructure) {
    // node n's box, cost and size from its (final) children
    const int2 c = __ldcg(child + n);
    TRef a, b;
    load_ref(a, c.x, nodebox, leafbox, cost, size);
    load_ref(b, c.y, nodebox, leafbox, cost, size);
    float4 lo = a.lo, hi = a.hi;
    unite(lo, hi, b.lo, b.hi);
    const float cn = kCi * area(lo, hi) + a.cost + b.cost;
    const int32_t sz = a.size + b.size;
    nodebox[2 * (int64_t)n] = lo, nodebox[2 * (int64_t)n + 1] = hi;
    cost[n] = cn;
    size[n] = sz;
    if (!restructure || sz < kTreeletLeaves) return;
    // form the treelet: open the largest-area internal treelet leaf until there are 7 leaves
    TRef L[kTreeletLeaves];
    int32_t I[kTreeletLeaves - 1];
    int nl = 2, ni = 1;
    L[0] = a, L[1] = b, I[0] = n;
    while (nl < kTreeletLeaves) {
        int best = -1;
        float ba = -1.f;
        for (int k = 0; k < nl; ++k)
            if (L[k].ref >= 0) {
                const float ar = area(L[k].lo, L[k].hi);
                if (ar > ba) ba = ar, best = k;
            }
        if (best < 0) break;
        const int32_t r = L[best].ref;
        I[ni++] = r;
        const int2 cc = __ldcg(child + r);
        load_ref(L[best], cc.x, nodebox, leafbox, cost, size);
        load_ref(L[nl++], cc.y, nodebox, leafbox, cost, size);
    }
    // old cost of the treelet's internal nodes = cost(n) - sum of leaf costs
    float leafsum = 0.f;
    for (int k = 0; k < nl; ++k) leafsum += L[k].cost;
    const float old_internal = cn - leafsum;
    // greedy agglomeration: merge the pair with the smallest union area; internal slots I[ni-1..0]
    // (the last merge takes I[0] = n, so the treelet root keeps its index and parent)
    TRef W[kTreeletLeaves];
    for (int k = 0; k < nl; ++k) W[k] = L[k];
    int nw = nl;
    int2 newc[kTreeletLeaves - 1];
    float new_internal = 0.f;
    int slot = ni - 1;
    float4 nlo[kTreeletLeaves - 1], nhi[kTreeletLeaves - 1];
    float ncost[kTreeletLeaves - 1];
    int32_t nsize[kTreeletLeaves - 1];
    while (nw > 1) {
        int bi = 0, bj = 1;
        float bu = INFINITY;
        for (int i = 0; i < nw; ++i)
            for (int j = i + 1; j < nw; ++j) {
                float4 ul = W[i].lo, uh = W[i].hi;
                unite(ul, uh, W[j].lo, W[j].hi);
                const float u = area(ul, uh);
                if (u < bu) bu = u, bi = i, bj = j;
            }
        TRef m;
        m.lo = W[bi].lo, m.hi = W[bi].hi;
        unite(m.lo, m.hi, W[bj].lo, W[bj].hi);
        const float ic = kCi * area(m.lo, m.hi);
        new_internal += ic;
        m.cost = ic + W[bi].cost + W[bj].cost;
        m.size = W[bi].size + W[bj].size;
        m.ref = I[slot];
        newc[slot] = make_int2(W[bi].ref, W[bj].ref);
        nlo[slot] = m.lo, nhi[slot] = m.hi, ncost[slot] = m.cost, nsize[slot] = m.size;
        --slot;
        W[bi] = m;
        W[bj] = W[--nw];
    }
    if (!(new_internal < old_internal * (1.f - 1e-5f))) return;
    for (int k = 0; k < ni; ++k) {
        const int32_t idx = I[k];
        child[idx] = newc[k];
        nodebox[2 * (int64_t)idx] = nlo[k], nodebox[2 * (int64_t)idx + 1] = nhi[k];
        cost[idx] = ncost[k];
        size[idx] = nsize[k];
        const int32_t r0 = newc[k].x, r1 = newc[k].y;
        parent[r0 >= 0 ? r0 : (T - 1) + ~r0] = idx;
        parent[r1 >= 0 ? r1 : (T - 1) + ~r1] = idx;
    }
}

__global__ void __launch_bounds__(256) k_treelet(int32_t T, int2 *child, int32_t *parent, float4 *nodebox,
                                                 const float4 *__restrict__ leafbox, float *cost, int32_t *size,
                                                 unsigned int *counter, int restructure) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    int32_t n = __ldcg(parent + (T - 1) + j);
    while (n >= 0) {
        __threadfence();
        if (atomicAdd(counter + n, 1u) == 0u) return;  // the sibling subtree is not done yet
        __threadfence();
        treelet_node(n, T, child, parent, nodebox, leafbox, cost, size, restructure != 0);
        __threadfence();
        n = __ldcg(parent + n);
    }
}

// ---- NEXT-4: parallel treelet restructuring over a depth partition ----------------------------
// The internal nodes are partitioned into treelets: a treelet is rooted at every internal node whose
// depth is = off (mod 3) (and at the root) and holds its descendants down to two levels below the
// root; its leaves (<= 8) are triangles or the roots of the next treelets. A treelet's restructuring
// changes only its own internal nodes (child links, boxes, parents of its leaves): its leaves keep
// their subtrees and boxes and its root keeps its box, so every treelet of one pass is independent
// and the pass is ONE launch with no bottom-up dependency chain (the sequential pass above climbs the
// tree, ~2.7 ms at 1 M triangles). Re-clustering: the greedy agglomeration of treelet_node (merge the
// pair with the smallest union area), kept when the treelet's internal SAH area sum drops. Passes at
// offsets 0, 1, 2 move the treelet boundaries; depths are recomputed between passes (k_depth).
__global__ void __launch_bounds__(128) k_treelet_par(int32_t T, int2 *child, int32_t *parent, float4 *nodebox,
                                                     const float4 *__restrict__ leafbox,
                                                     const int32_t *__restrict__ depth, int off) {
    const int32_t n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= T - 1) return;
    if (n != 0 && depth[n] % 3 != off) return;
    if (n == 0 && off != 0) return;
    // gather the treelet: internal nodes I (root first), leaves L with their boxes
    int32_t I[7], Lr[8];
    float4 Ll[8], Lh[8];
    int ni = 0, nl = 0;
    int32_t q[7];
    int qd[7], qh = 0, qt = 0;
    q[qt] = n, qd[qt++] = 0;
    while (qh < qt) {
        const int32_t m = q[qh];
        const int d = qd[qh++];
        I[ni++] = m;
        const int2 c = child[m];
        const int32_t cc[2] = {c.x, c.y};
        for (int k = 0; k < 2; ++k) {
            const int32_t r = cc[k];
            if (r >= 0 && d < 2) {
                q[qt] = r, qd[qt++] = d + 1;
            } else {
                Lr[nl] = r;
                if (r >= 0)
                    Ll[nl] = nodebox[2 * (int64_t)r], Lh[nl] = nodebox[2 * (int64_t)r + 1];
                else
                    Ll[nl] = __ldg(leafbox + 2 * (int64_t)~r), Lh[nl] = __ldg(leafbox + 2 * (int64_t)~r + 1);
                ++nl;
            }
        }
    }
    if (nl <= 2) return;
    float old_cost = 0.f;
    for (int k = 0; k < ni; ++k) old_cost += area(nodebox[2 * (int64_t)I[k]], nodebox[2 * (int64_t)I[k] + 1]);
    // greedy agglomeration; new internal node s takes index I[s] (the last merge -> I[0] = n)
    int32_t Wr[8];
    float4 Wl[8], Wh[8];
    for (int k = 0; k < nl; ++k) Wr[k] = Lr[k], Wl[k] = Ll[k], Wh[k] = Lh[k];
    int nw = nl, slot = ni - 1;
    int2 nc[7];
    float4 nlo[7], nhi[7];
    float new_cost = 0.f;
    while (nw > 1) {
        int bi = 0, bj = 1;
        float bu = INFINITY;
        for (int i = 0; i < nw; ++i)
            for (int j = i + 1; j < nw; ++j) {
                float4 ul = Wl[i], uh = Wh[i];
                unite(ul, uh, Wl[j], Wh[j]);
                const float u = area(ul, uh);
                if (u < bu) bu = u, bi = i, bj = j;
            }
        float4 ml = Wl[bi], mh = Wh[bi];
        unite(ml, mh, Wl[bj], Wh[bj]);
        new_cost += bu;
        nc[slot] = make_int2(Wr[bi], Wr[bj]);
        nlo[slot] = ml, nhi[slot] = mh;
        Wr[bi] = I[slot], Wl[bi] = ml, Wh[bi] = mh;
        --slot;
        --nw;
        Wr[bj] = Wr[nw], Wl[bj] = Wl[nw], Wh[bj] = Wh[nw];
    }
    if (!(new_cost < old_cost * (1.f - 1e-5f))) return;
    for (int k = 0; k < ni; ++k) {
        const int32_t idx = I[k];
        child[idx] = nc[k];
        if (k > 0) nodebox[2 * (int64_t)idx] = nlo[k], nodebox[2 * (int64_t)idx + 1] = nhi[k];
        const int32_t r0 = nc[k].x, r1 = nc[k].y;
        parent[r0 >= 0 ? r0 : (T - 1) + ~r0] = idx;
        parent[r1 >= 0 ? r1 : (T - 1) + ~r1] = idx;
    }
}

// Exhaustive 4-leaf treelets over a depth partition (roots at depth = off mod 2): a root n, its two
// children and their children (the treelet leaves: triangles or the next treelets' roots). With the
// root fixed, 4 leaves have 15 binary topologies (3 pairings 2+2, 12 of the form 1 + (1 + 2)); all
// are costed from the 6 pair and 4 triple unions of the leaf boxes (compile-time code, registers
// only) and the one with the smallest sum of its two non-root internal areas is kept — the root's
// box and the leaves' subtrees are unchanged, so every treelet of a pass is independent (one
// launch, no chain). 3-leaf treelets (one child a leaf) choose among their 3 pairings.
__device__ __forceinline__ float4 fmin4(float4 a, float4 b) {
    return make_float4(fminf(a.x, b.x), fminf(a.y, b.y), fminf(a.z, b.z), 0.f);
}
__device__ __forceinline__ float4 fmax4(float4 a, float4 b) {
    return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), 0.f);
}

__global__ void __launch_bounds__(256) k_treelet4(int32_t T, int2 *child, int32_t *parent, float4 *nodebox,
                                                  const float4 *__restrict__ leafbox,
                                                  const int32_t *__restrict__ depth, int off) {
    const int32_t n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= T - 1 || (depth[n] & 1) != off) return;
    const int2 c = child[n];
    if (c.x < 0 && c.y < 0) return;  // 2 leaves: nothing to choose
    // leaves in fixed slots: children of c.x at 0, 1 (or c.x itself at 0), of c.y at 2, 3
    int32_t L[4];
    int nl;
    int2 g0 = make_int2(0, 0), g1 = make_int2(0, 0);
    if (c.x >= 0) g0 = child[c.x];
    if (c.y >= 0) g1 = child[c.y];
    auto box_of = [&](int32_t r, float4 &lo, float4 &hi) {
        if (r >= 0)
            lo = nodebox[2 * (int64_t)r], hi = nodebox[2 * (int64_t)r + 1];
        else
            lo = __ldg(leafbox + 2 * (int64_t)~r), hi = __ldg(leafbox + 2 * (int64_t)~r + 1);
    };
    float4 lo[4], hi[4];
    if (c.x >= 0 && c.y >= 0) {
        L[0] = g0.x, L[1] = g0.y, L[2] = g1.x, L[3] = g1.y;
        nl = 4;
    } else {  // 3 leaves: the internal child's two children and the leaf child
        const int2 g = c.x >= 0 ? g0 : g1;
        L[0] = g.x, L[1] = g.y, L[2] = c.x >= 0 ? c.y : c.x, L[3] = 0;
        nl = 3;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k < nl) box_of(L[k], lo[k], hi[k]);
    // old: the two non-root internal nodes (4 leaves) or the one (3 leaves)
    const int32_t ia = c.x >= 0 ? c.x : c.y;  // an internal node id to reuse
    const int32_t ib = (c.x >= 0 && c.y >= 0) ? c.y : -1;
    float old_cost = area(nodebox[2 * (int64_t)ia], nodebox[2 * (int64_t)ia + 1]);
    if (ib >= 0) old_cost += area(nodebox[2 * (int64_t)ib], nodebox[2 * (int64_t)ib + 1]);
    // pair unions
    float pa[4][4];
    float4 plo[4][4], phi[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i + 1; j < 4; ++j) {
            plo[i][j] = fmin4(lo[i], lo[j]), phi[i][j] = fmax4(hi[i], hi[j]);
            pa[i][j] = area(plo[i][j], phi[i][j]);
        }
    float best = old_cost;
    int choice = -1;  // 0..2: pairing (0,1|2,3), (0,2|1,3), (0,3|1,2); 3 + 3 x + p: single x, pair p of the rest
    if (nl == 4) {
        const float c2[3] = {pa[0][1] + pa[2][3], pa[0][2] + pa[1][3], pa[0][3] + pa[1][2]};
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (c2[k] < best) best = c2[k], choice = k;
        // 1 + (1 + 2): single x; triple = the other three; inner pair p of the triple
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            int o[3], m = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k != x) o[m++] = k;
            const float4 tlo = fmin4(plo[o[0]][o[1]], lo[o[2]]), thi = fmax4(phi[o[0]][o[1]], hi[o[2]]);
            const float ta = area(tlo, thi);
            const float cp[3] = {pa[o[0]][o[1]], pa[o[0]][o[2]], pa[o[1]][o[2]]};
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (ta + cp[q] < best) best = ta + cp[q], choice = 3 + 3 * x + q;
        }
    } else {
        const float c3[3] = {pa[0][1], pa[0][2], pa[1][2]};
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (c3[k] < best) best = c3[k], choice = k;
    }
    if (choice < 0 || !(best < old_cost * (1.f - 1e-5f))) return;
    // runtime slot picks by select chains (an array indexed at run time would live in local memory)
    auto pick = [&](int i, float4 &l, float4 &h, int32_t &r) {
        l = i == 0 ? lo[0] : (i == 1 ? lo[1] : (i == 2 ? lo[2] : lo[3]));
        h = i == 0 ? hi[0] : (i == 1 ? hi[1] : (i == 2 ? hi[2] : hi[3]));
        r = i == 0 ? L[0] : (i == 1 ? L[1] : (i == 2 ? L[2] : L[3]));
    };
    auto link = [&](int32_t node, int32_t r0, int32_t r1) {
        child[node] = make_int2(r0, r1);
        parent[r0 >= 0 ? r0 : (T - 1) + ~r0] = node;
        parent[r1 >= 0 ? r1 : (T - 1) + ~r1] = node;
    };
    auto setbox = [&](int32_t node, float4 l, float4 h) {
        nodebox[2 * (int64_t)node] = l, nodebox[2 * (int64_t)node + 1] = h;
    };
    float4 l0, h0, l1, h1, l2, h2, l3, h3;
    int32_t r0, r1, r2, r3;
    if (nl == 3) {  // pair (i, j) under ia, the third leaf beside it under n
        const int i = choice == 2 ? 1 : 0, j = choice == 0 ? 1 : 2, r = 3 - i - j;
        pick(i, l0, h0, r0), pick(j, l1, h1, r1), pick(r, l2, h2, r2);
        link(ia, r0, r1);
        setbox(ia, fmin4(l0, l1), fmax4(h0, h1));
        link(n, ia, r2);
        return;
    }
    if (choice < 3) {  // 2 + 2: leaf 0 with leaf choice + 1, the other two together
        const int a1 = choice + 1, b0 = a1 == 1 ? 2 : 1, b1 = a1 == 3 ? 2 : 3;
        pick(0, l0, h0, r0), pick(a1, l1, h1, r1), pick(b0, l2, h2, r2), pick(b1, l3, h3, r3);
        link(ia, r0, r1);
        setbox(ia, fmin4(l0, l1), fmax4(h0, h1));
        link(ib, r2, r3);
        setbox(ib, fmin4(l2, l3), fmax4(h2, h3));
        link(n, ia, ib);
        return;
    }
    // 1 + (1 + 2): single x; the others o0 < o1 < o2; inner pair q of them
    const int x = (choice - 3) / 3, q = (choice - 3) % 3;
    const int o0 = x == 0 ? 1 : 0, o1 = x <= 1 ? 2 : 1, o2 = x <= 2 ? 3 : 2;
    const int p0 = q == 2 ? o1 : o0, p1 = q == 0 ? o1 : o2, r = o0 + o1 + o2 - p0 - p1;
    pick(p0, l0, h0, r0), pick(p1, l1, h1, r1), pick(r, l2, h2, r2), pick(x, l3, h3, r3);
    link(ib, r0, r1);  // inner pair
    const float4 ilo = fmin4(l0, l1), ihi = fmax4(h0, h1);
    setbox(ib, ilo, ihi);
    link(ia, ib, r2);  // triple
    setbox(ia, fmin4(ilo, l2), fmax4(ihi, h2));
    link(n, ia, r3);
}

// the cast's stack bound for a freely restructured binary tree: its depth + 1 (one push per level at
// most), as the maximum over the internal nodes' depths (k_depth), into *need
__global__ void __launch_bounds__(256) k_depth_max(int64_t n, const int32_t *__restrict__ depth, unsigned int *need) {
    int32_t m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n - 1; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, depth[i]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(need, (unsigned int)(m + 2));
}

// traversal nodes for single-triangle leaves from child refs and boxes (any topology)
__global__ void __launch_bounds__(256) k_nodes_free(int64_t n, const int2 *__restrict__ child,
                                                    const float4 *__restrict__ leafbox,
                                                    const float4 *__restrict__ nodebox, Node64 *__restrict__ nodes) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int2 c = child[i];
    const float4 *b0 = c.x >= 0 ? nodebox + 2 * (int64_t)c.x : leafbox + 2 * (int64_t)(~c.x);
    const float4 *b1 = c.y >= 0 ? nodebox + 2 * (int64_t)c.y : leafbox + 2 * (int64_t)(~c.y);
    const float4 l0 = b0[0], h0 = b0[1], l1 = b1[0], h1 = b1[1];
    Node64 nd;
    nd.a = make_float4(l0.x, h0.x, l0.y, h0.y);
    nd.b = make_float4(l1.x, h1.x, l1.y, h1.y);
    nd.c = make_float4(l0.z, h0.z, l1.z, h1.z);
    nd.d = make_int4(c.x >= 0 ? c.x : make_leaf(~c.x, 1), c.y >= 0 ? c.y : make_leaf(~c.y, 1), 0, 0);
    nodes[i] = nd;
}

// Leaf-order gather: tri48[j] = triangle perm[j] {v0.xyz, id}, {v1.xyz, 0}, {v2.xyz, 0}, its exact
// box leafbox[j], and the union of every 8 consecutive leaf boxes (agg[0], 8-lane reduction).
__device__ __forceinline__ void warp_union(float4 &lo, float4 &hi) {
    for (int o = 4; o; o >>= 1) {
        lo.x = fminf(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
        lo.y = fminf(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
        lo.z = fminf(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
        hi.x = fmaxf(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
        hi.y = fmaxf(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
        hi.z = fmaxf(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
    }
}


__global__ void __launch_bounds__(256) k_reorder(const float *__restrict__ verts, int64_t V,
                                                 const int32_t *__restrict__ tris,
                                                 const uint32_t *__restrict__ perm,
                                                 const uint64_t *__restrict__ pkeys, uint64_t pmask, int64_t n,
                                                 float4 *__restrict__ tri, float4 *__restrict__ leafbox,
                                                 float4 *__restrict__ agg) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float4 lo = make_float4(kInf, kInf, kInf, 0.f), hi = make_float4(-kInf, -kInf, -kInf, 0.f);
    if (j < n) {
        const uint32_t k = perm ? perm[j] : (uint32_t)(pkeys[j] & pmask);
        const float3 a = ldv(verts, clampv(__ldg(tris + 3 * (int64_t)k), V)),
                     b = ldv(verts, clampv(__ldg(tris + 3 * (int64_t)k + 1), V)),
                     c = ldv(verts, clampv(__ldg(tris + 3 * (int64_t)k + 2), V));
        tri[kTriStride * j] = make_float4(a.x, a.y, a.z, __int_as_float((int32_t)k));
        tri[kTriStride * j + 1] = make_float4(b.x, b.y, b.z, 0.f);
        tri[kTriStride * j + 2] = make_float4(c.x, c.y, c.z, 0.f);
        lo = make_float4(fminf(a.x, fminf(b.x, c.x)), fminf(a.y, fminf(b.y, c.y)), fminf(a.z, fminf(b.z, c.z)), 0.f);
        hi = make_float4(fmaxf(a.x, fmaxf(b.x, c.x)), fmaxf(a.y, fmaxf(b.y, c.y)), fmaxf(a.z, fmaxf(b.z, c.z)), 0.f);
        leafbox[2 * j] = lo;
        leafbox[2 * j + 1] = hi;
    }
    warp_union(lo, hi);
    if ((threadIdx.x & 7) == 0 && j < n) {
        agg[2 * (j >> 3)] = lo;
        agg[2 * (j >> 3) + 1] = hi;
    }
}

// next aggregate level: union of every 8 consecutive boxes of the level below
__global__ void __launch_bounds__(256) k_aggregate(const float4 *__restrict__ in, int64_t n_in,
                                                   float4 *__restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float4 lo = make_float4(kInf, kInf, kInf, 0.f), hi = make_float4(-kInf, -kInf, -kInf, 0.f);
    if (j < n_in) lo = in[2 * j], hi = in[2 * j + 1];
    warp_union(lo, hi);
    if ((threadIdx.x & 7) == 0 && j < n_in) out[2 * (j >> 3)] = lo, out[2 * (j >> 3) + 1] = hi;
}

// Binary traversal nodes (node64), one thread per internal node, from the children's Eq. 7 boxes
// (leaf boxes / node boxes); subtrees of <= leaf_size triangles become leaves.
__global__ void __launch_bounds__(256) k_nodes(int64_t n, int leaf_size, const int2 *__restrict__ child,
                                               const int2 *__restrict__ range, const float4 *__restrict__ leafbox,
                                               const float4 *__restrict__ nodebox, Node64 *__restrict__ nodes) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int2 c = child[i], r = range[i];
    const int32_t g = c.x >= 0 ? c.x : ~c.x;  // split: left child covers [f, g], right [g + 1, l]
    const float4 *b0 = c.x >= 0 ? nodebox + 2 * (int64_t)c.x : leafbox + 2 * (int64_t)(~c.x);
    const float4 *b1 = c.y >= 0 ? nodebox + 2 * (int64_t)c.y : leafbox + 2 * (int64_t)(~c.y);
    const float4 l0 = b0[0], h0 = b0[1], l1 = b1[0], h1 = b1[1];
    const int32_t n0 = g - r.x + 1, n1 = r.y - g;
    const int32_t ref0 = (c.x < 0 || n0 <= leaf_size) ? make_leaf(r.x, n0) : c.x;
    const int32_t ref1 = (c.y < 0 || n1 <= leaf_size) ? make_leaf(g + 1, n1) : c.y;
    Node64 nd;
    nd.a = make_float4(l0.x, h0.x, l0.y, h0.y);
    nd.b = make_float4(l1.x, h1.x, l1.y, h1.y);
    nd.c = make_float4(l0.z, h0.z, l1.z, h1.z);
    nd.d = make_int4(ref0, ref1, 0, 0);
    nodes[i] = nd;
}

// ---- fused A2 leaf records + A5 Karras tree + A6 Eq. 7 boxes + A7 node64 (width 2, default build) --
// The binary radix tree of Eq. 6 has one internal node per adjacent pair of sorted keys:
// the node split at g (between leaves g and g + 1) covers the maximal run of leaves around g whose
// adjacent LCPs delta(k, k + 1) all exceed delta(g, g + 1). A node covering [l, r] is therefore the
// LEFT child of the node split at r when delta(r, r + 1) > delta(l - 1, l), else the RIGHT child of
// the node split at l - 1 (never equal for distinct augmented keys; delta = -1 outside [0, n)).
// That makes the tree buildable bottom-up with the boxes (after Apetrei 2014): every leaf climbs;
// at a parent the first child to arrive deposits its box and far endpoint and stops, the second
// unites both boxes — Eq. 7, exact min/max — writes the parent's node64 and climbs on.
// Karras's numbering is kept (an internal node is indexed by its right endpoint if it is a left
// child, by its left endpoint if a right child, the root is 0), so a node split at g has children
// g and g + 1 and child / range / parent / node64 are bit-identical to k_karras + k_nodes.
// One CTA per kChunk consecutive leaves, one thread per leaf: parents whose split lies inside the
// chunk meet in shared memory; a node whose parent's range leaves the chunk (the chunk boundaries'
// ancestors, a few per chunk) meets its sibling through a global slot per split — an epoch-tagged
// exchange of the far endpoint, the boxes passed through nodebox / leafbox, fenced. Leaf records
// (tri48) are gathered here in leaf order; leaf and node boxes are stored only where a sibling needs
// them (all_boxes = 1 stores them all; the scene export fills them in on demand otherwise).
#ifndef FGL_LBVH_CHUNK
#define FGL_LBVH_CHUNK 256
#endif
#ifndef FGL_MORTON_BLOCKS
#define FGL_MORTON_BLOCKS (148 * 4)  // k_morton grid (each block adds its 8 x 256 digit counts to the global histogram)
#endif
#ifndef FGL_LBVH_ORDERED
#define FGL_LBVH_ORDERED 0  // 1: round work lists in split order (ballot ranks) instead of atomic appends
                             // (measured: fewer bank conflicts but +32% instructions, C3 k_lbvh 0.73 -> 0.83 ms)
#endif
#ifndef FGL_TREELET_MIN
#define FGL_TREELET_MIN 1  // in-build treelets: only at nodes over at least this many leaves
#endif
#ifndef FGL_LBVH_MINB
#define FGL_LBVH_MINB (1536 / FGL_LBVH_CHUNK)  // resident CTAs per SM the register budget is sized for
#endif
constexpr int kChunk = FGL_LBVH_CHUNK;  // leaves (= threads) per k_lbvh CTA
constexpr int kSlotEmpty = -1, kSlotDone = -2;
constexpr int kMaxRounds = 100;  // > the depth of a Karras tree (delta strictly grows downwards, < 96)

struct Box6 {
    float lx, ly, lz, hx, hy, hz;
};

__device__ __forceinline__ Box6 box_union(const Box6 &a, const Box6 &b) {
    return Box6{fminf(a.lx, b.lx), fminf(a.ly, b.ly), fminf(a.lz, b.lz),
                fmaxf(a.hx, b.hx), fmaxf(a.hy, b.hy), fmaxf(a.hz, b.hz)};
}
__device__ __forceinline__ float box_area(const Box6 &b) {  // half surface area (SAH weight)
    const float dx = b.hx - b.lx, dy = b.hy - b.ly, dz = b.hz - b.lz;
    return dx * dy + dy * dz + dz * dx;
}
// lo.w carries the node's height in the traversal tree (treelet builds; 0 otherwise)
__device__ __forceinline__ void box_store(float4 *p, const Box6 &b, int h = 0) {
    p[0] = make_float4(b.lx, b.ly, b.lz, __int_as_float(h));
    p[1] = make_float4(b.hx, b.hy, b.hz, 0.f);
}
__device__ __forceinline__ Box6 box_load_cg(const float4 *p, int &h) {
    const float4 l = __ldcg(p), hi = __ldcg(p + 1);
    h = __float_as_int(l.w);
    return Box6{l.x, l.y, l.z, hi.x, hi.y, hi.z};
}

// delta(i, i + 1) of the augmented keys (R7), -1 when the pair leaves [0, n)
__device__ __forceinline__ int adj_delta(const uint64_t *__restrict__ k, int n, int i, int ks) {
    if (i < 0 || i + 1 >= n) return -1;
    const uint64_t x = (__ldg(k + i) ^ __ldg(k + i + 1)) >> ks;
    return x ? __clzll((long long)x) : 64 + __clz(i ^ (i + 1));
}

struct LbvhOut {
    int2 *child, *range;
    int32_t *parent;
    float4 *leafbox, *nodebox;
    Node64 *nodes;
    unsigned long long *gslot;
    unsigned int *wneed;  // treelet builds: the traversal-stack bound (height + margin), by the root
    int n, leaf_size, all_boxes;
    uint32_t epoch;
};

// one child of an internal node: child-array ref (internal index / ~leaf), node64 ref (internal
// index / make_leaf(first, count) when the subtree holds <= leaf_size triangles), box, height in
// the traversal tree (0 for node64 leaves)
struct Kid {
    int32_t c, nr;
    Box6 b;
    int h;
};

__device__ __forceinline__ Kid kid_of(const LbvhOut &o, int32_t c, int first, int count, const Box6 &b, int h) {
    return Kid{c, (c < 0 || count <= o.leaf_size) ? make_leaf(first, count) : c, b, (c < 0 || count <= o.leaf_size) ? 0 : h};
}

// write internal node K with children a (slot 0) and b (slot 1): node64, child links, parents
__device__ __forceinline__ void put_kids(const LbvhOut &o, int K, const Kid &a, const Kid &b) {
    o.child[K] = make_int2(a.c, b.c);
    o.parent[a.c >= 0 ? a.c : (o.n - 1) + ~a.c] = K;
    o.parent[b.c >= 0 ? b.c : (o.n - 1) + ~b.c] = K;
    if (K == 0) o.parent[0] = -1;
    Node64 nd;
    nd.a = make_float4(a.b.lx, a.b.hx, a.b.ly, a.b.hy);
    nd.b = make_float4(b.b.lx, b.b.hx, b.b.ly, b.b.hy);
    nd.c = make_float4(a.b.lz, a.b.hz, b.b.lz, b.b.hz);
    nd.d = make_int4(a.nr, b.nr, 0, 0);
    o.nodes[K] = nd;
}

// internal node K = split g over leaves [l, r], children boxes a (left) and b (right), heights ha, hb
__device__ __forceinline__ void put_node(const LbvhOut &o, int K, int g, int l, int r, const Box6 &a, const Box6 &b,
                                         int ha = 0, int hb = 0) {
    const int32_t left = l == g ? ~g : g, right = r == g + 1 ? ~(g + 1) : g + 1;
    o.range[K] = make_int2(l, r);
    put_kids(o, K, kid_of(o, left, l, g - l + 1, a, ha), kid_of(o, right, g + 1, r - g, b, hb));
}

// treelet builds: height of node [l, r] seen by the traversal (0 when it is a node64 leaf)
__device__ __forceinline__ int trav_height(const LbvhOut &o, int l, int r, int h) {
    return r - l + 1 <= o.leaf_size ? 0 : h;
}

// climb from the complete node [l, r] (boundary LCPs dl, dr; height h) through global slots until
// this thread arrives first somewhere or completes the root
template <bool kTreelet>
__device__ __forceinline__ void lbvh_global_climb(const LbvhOut &o, const uint64_t *__restrict__ keys, int ks, int l,
                                                  int r, int dl, int dr, Box6 box, int h, bool published) {
    while (true) {
        const bool left = dr > dl;
        const int gp = left ? r : l - 1;
        if (!published)
            box_store(l == r ? o.leafbox + 2 * (int64_t)l : o.nodebox + 2 * (int64_t)(left ? r : l), box,
                      kTreelet ? trav_height(o, l, r, h) : 0);
        published = false;
        // release this node's box, acquire the sibling's (the first arrival released its own)
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> slot(o.gslot[gp]);
        const unsigned long long old = slot.exchange(((unsigned long long)o.epoch << 32) | (uint32_t)(left ? l : r),
                                                     cuda::std::memory_order_acq_rel);
        if ((uint32_t)(old >> 32) != o.epoch) return;  // first to arrive: the sibling completes gp
        const int other = (int)(uint32_t)old;
        const int sl = left ? gp + 1 : other, sr = left ? other : gp;
        int hs;
        const Box6 sib = box_load_cg(sl == sr ? o.leafbox + 2 * (int64_t)sl : o.nodebox + 2 * (int64_t)(left ? gp + 1 : gp), hs);
        const int hm = kTreelet ? trav_height(o, l, r, h) : 0;
        const Box6 &A = left ? box : sib, &B = left ? sib : box;
        const int L = left ? l : other, R = left ? other : r;
        dl = adj_delta(keys, o.n, L - 1, ks);
        dr = adj_delta(keys, o.n, R, ks);
        const bool root = dl < 0 && dr < 0;
        const Box6 u = box_union(A, B);
        put_node(o, root ? 0 : (dr > dl ? R : L), gp, L, R, A, B, left ? hm : hs, left ? hs : hm);
        h = 1 + max(hm, hs);
        if (root) {
            box_store(o.nodebox, u, h);
            if (kTreelet) *o.wneed = (unsigned int)(h + 1 + 3);  // + 3: refit may split <= 8-triangle leaves
            return;
        }
        box = u, l = L, r = R;
    }
}

constexpr int32_t kNone = INT32_MIN;  // k_lbvh staging: no entry

// boxes in shared memory as six planes (conflict-free for nearby indices; a 24-byte struct array
// takes 2-way bank conflicts on every field)
struct BoxRef {
    float *p;
    __device__ __forceinline__ operator Box6() const {
        return Box6{p[0], p[kChunk], p[2 * kChunk], p[3 * kChunk], p[4 * kChunk], p[5 * kChunk]};
    }
    __device__ __forceinline__ BoxRef &operator=(const Box6 &b) {
        p[0] = b.lx, p[kChunk] = b.ly, p[2 * kChunk] = b.lz, p[3 * kChunk] = b.hx, p[4 * kChunk] = b.hy,
        p[5 * kChunk] = b.hz;
        return *this;
    }
};
struct BoxArr {
    float v[6 * kChunk];
    __device__ __forceinline__ BoxRef operator[](int i) { return BoxRef{v + i}; }
};

// k_lbvh shared memory (dynamic: > 48 KB with the treelet records)
template <bool kTreelet>
struct LbvhSmem {
    int sdelta[kChunk + 1];   // delta(c0 + i - 1, c0 + i), i = 0..cnt
    int sslot[kChunk];        // split c0 + s: first arrival's far endpoint / empty / done
    int wn[kMaxRounds + 1];   // wn[k]: nodes completed in round k - 1
    int spar_int[kChunk];     // staged parent of internal node c0 + i
    int spar_leaf[kChunk];    // staged parent of leaf c0 + i
    int sheight[kTreelet ? kChunk : 1];  // internal node c0 + i: height
    BoxArr slbox;             // leaf c0 + i
    BoxArr snbox;             // internal node c0 + i, once complete
    int2 schild[kChunk];      // staged child refs of internal node c0 + i (kNone: not completed here)
    int2 srange[kChunk];      // staged leaf range of internal node c0 + i
    int4 wl[2][kChunk];       // round work lists: (l, r, split) of nodes to complete
    int smark[kChunk];        // position p starts an output unit ending at smark[p] (kNone: no)
    int2 spos[FGL_LBVH_ORDERED ? kChunk : 1];  // FGL_LBVH_ORDERED: next round's node (L, R) at its split
    int swarp[kChunk / 32 + 1];
    int4 sref[kTreelet ? kChunk : 1];  // internal node c0 + i: (child refs, node64 refs)
};

// ---- levels above the chunks ----------------------------------------------------------------------
// Every chunk's nodes whose parent spans a chunk boundary ("units": maximal subtrees inside the
// chunk, they tile it) are emitted in leaf order; kGroup consecutive chunks form a group one level
// up, whose last CTA to finish (arrival counter) builds the tree over the group's units in shared
// memory exactly as over leaves — units play the leaves, the LCP across a unit boundary is the
// adjacent-key delta there — and emits its own units, and so on until one group holds everything
// and completes the root. A segment with more than kUnitCap units (or a group with more than
// kChunk) sends its units to the global pending list instead (k_lbvh_top climbs those through the
// global slots), and everything above it follows ("poisoned"), so both paths never meet in one node.
constexpr int kUnitCap = 64;
#ifndef FGL_LBVH_GROUP
#define FGL_LBVH_GROUP 16  // max chunks per group; 16 below 2^22 leaves, 8 above (where 16 overflows)
#endif
constexpr int kGroup = FGL_LBVH_GROUP;
static_assert(kGroup <= 32, "one warp reads a group's segment counts");
constexpr int kMaxLevels = 8;
// a unit's boundary LCPs delta(a - 1, a) and delta(b, b + 1) (-1..95), packed in Unit::m.w
__host__ __device__ __forceinline__ int pack_deltas(int dl, int dr) { return (dl + 1) | (dr + 1) << 8; }
__host__ __device__ __forceinline__ int unpack_dl(int w) { return (w & 0xFF) - 1; }
__host__ __device__ __forceinline__ int unpack_dr(int w) { return ((w >> 8) & 0xFF) - 1; }
struct Unit {
    int4 m;  // (a, b, height, packed boundary deltas): leaves [a, b]
    float4 lo, hi;
};
struct UpPlan {
    Unit *units[kMaxLevels];          // level i: nseg[i] segments x kUnitCap units
    int *cnt[kMaxLevels];             // level i, per segment: unit count, -1 = poisoned
    unsigned int *ctr[kMaxLevels];    // level i >= 1, per group: arrivals of its level i-1 segments
    int nseg[kMaxLevels];
    int nlev;                         // nseg[nlev - 1] == 1
    int G;                            // segments per group (<= kGroup)
    int force_global;                 // test hook FGL_LBVH_GLOBAL: 1 = every chunk's units go to the global
                                      // list, 2 = every odd chunk's, 4 = every odd group's (levels >= 1)
};

// segment counts per level and the carve-up of BuildBuffers::lbvh_up (bytes: lbvh_up_bytes)
static UpPlan lbvh_plan(int64_t T, void *base) {
    UpPlan up{};
    // 16-chunk groups save a level (~10 us of tail each); at 10 M triangles their ~17 units per
    // chunk overflow a 256-unit group, so large trees use 8
    up.G = T < (int64_t(1) << 22) ? kGroup : kGroup / 2;
    up.nseg[0] = (int)((T + kChunk - 1) / kChunk);
    up.nlev = 1;
    while (up.nseg[up.nlev - 1] > 1) {
        if (up.nlev == kMaxLevels) throw Error(1, "lbvh: too many levels");
        up.nseg[up.nlev] = (up.nseg[up.nlev - 1] + up.G - 1) / up.G;
        ++up.nlev;
    }
    char *p = static_cast<char *>(base);
    auto take = [&](size_t bytes) {
        char *q = p;
        p += (bytes + 255) & ~size_t(255);
        return q;
    };
    for (int i = 0; i < up.nlev; ++i) {
        up.ctr[i] = reinterpret_cast<unsigned int *>(take(sizeof(unsigned int) * up.nseg[i]));  // zeroed once
        up.cnt[i] = reinterpret_cast<int *>(take(sizeof(int) * up.nseg[i]));
        up.units[i] = i + 1 < up.nlev ? reinterpret_cast<Unit *>(take(sizeof(Unit) * kUnitCap * (size_t)up.nseg[i])) : nullptr;
    }
    if (base == nullptr) up.units[0] = reinterpret_cast<Unit *>(p);  // size query: end pointer
    return up;
}


// append `it` to a shared work list, one shared atomic per warp (called by whole warps)
__device__ __forceinline__ void append_item(int4 *list, int *n, bool push, const int4 &it) {
    const unsigned bal = __ballot_sync(0xffffffffu, push);
    if (!bal) return;
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(n, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (push) list[base + __popc(bal & ((1u << lane) - 1u))] = it;
}

// a unit whose parent will be built by the global climb: publish its box where the sibling looks
// (Karras index by side) and list it for k_lbvh_top
template <bool kTreelet>
__device__ __forceinline__ void lbvh_push_global(const LbvhOut &o, const uint64_t *__restrict__ keys, int ks,
                                                 const Unit &u, int4 *pend, unsigned int *pend_n) {
    const int l = u.m.x, r = u.m.y;
    const int dl = unpack_dl(u.m.w), dr = unpack_dr(u.m.w);
    float4 *dst = l == r ? o.leafbox + 2 * (int64_t)l : o.nodebox + 2 * (int64_t)(dr > dl ? r : l);
    dst[0] = make_float4(u.lo.x, u.lo.y, u.lo.z, __int_as_float(kTreelet ? trav_height(o, l, r, u.m.z) : 0));
    dst[1] = u.hi;
    pend[atomicAdd(pend_n, 1u)] = make_int4(l, r, u.m.z, 0);
}

// Write the marked units (smark[p] = end position, p < P) of segment `seg` at level `lev` in
// position order (block-wide rank by ballots), or poison the segment and push them to the global
// list when they do not fit (or when `poison` is set). All threads of the CTA call this.
template <bool kTreelet, class UnitOf>
__device__ void lbvh_emit(const LbvhOut &o, const uint64_t *__restrict__ keys, int ks, const UpPlan &up, int lev,
                          int seg, int P, const int *smark, int *swarp, UnitOf unit_of, int4 *pend,
                          unsigned int *pend_n, bool poison = false) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const bool has = t < P && smark[t] != kNone;
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    if (lane == 0) swarp[w] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
        const int c = swarp[k];
        before += k < w ? c : 0;
        total += c;
    }
    const int rank = before + __popc(bal & ((1u << lane) - 1u));
    const bool bad = poison || total > kUnitCap;
    if (has) {
        const Unit u = unit_of(t, smark[t]);
        if (bad)
            lbvh_push_global<kTreelet>(o, keys, ks, u, pend, pend_n);
        else
            up.units[lev][(int64_t)seg * kUnitCap + rank] = u;
    }
    if (t == 0) up.cnt[lev][seg] = bad ? -1 : total;
    __syncthreads();  // swarp / smark reuse
}

// The levels above the chunks (see UpPlan). Called by every CTA after its segment is emitted at
// level 0; the last CTA of each group goes on up.
template <bool kTreelet>
__device__ void lbvh_levels(const LbvhOut &o, const uint64_t *__restrict__ keys, int ks, const UpPlan &up, int seg,
                            LbvhSmem<kTreelet> &S, int4 *pend, unsigned int *pend_n, bool arrived) {
    __shared__ int s_last, s_off[kGroup + 1], s_poison;
    const int t = threadIdx.x, n = o.n;
    for (int lev = 1; lev < up.nlev; ++lev) {
        const int group = seg / up.G, first = group * up.G, gsize = min(up.G, up.nseg[lev - 1] - first);
        if (!(lev == 1 && arrived)) {  // (level 1: the caller arrived already, as the last of its group)
            __syncthreads();  // this segment's units / count written (by several threads)
            if (t == 0) {
                __threadfence();  // release them (cumulative over the barrier) before the arrival
                s_last = atomicAdd(up.ctr[lev] + group, 1u) == (unsigned)(gsize - 1);
                if (s_last) up.ctr[lev][group] = 0;  // self-resetting for the next build
            }
            __syncthreads();
            if (!s_last) return;
        }
        if (t == 0) __threadfence();  // acquire the group's segments (the barrier below spreads it)
        __syncthreads();
        seg = group;
        if (t < 32) {  // the segments' counts in parallel (one L2 round trip), prefix by shuffles
            const int c = t < gsize ? __ldcg(up.cnt[lev - 1] + first + t) : 0;
            int x = max(c, 0);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, d);
                if (t >= d) x += y;
            }
            if (t < gsize) s_off[t] = x - max(c, 0);
            const bool poison = __any_sync(0xffffffffu, c < 0);
            const int off = __shfl_sync(0xffffffffu, x, 31);
            if (t == 0) {
                s_off[gsize] = off;
                s_poison = poison || off > kChunk || ((up.force_global & 4) && (group & 1));
            }
        }
        __syncthreads();
        const int m = s_off[gsize];
        // units of the group in order: position v -> segment k, index v - s_off[k]
        auto load_unit = [&](int v) -> Unit {
            int k = 0;
            while (v >= s_off[k + 1]) ++k;
            const Unit *src = up.units[lev - 1] + (int64_t)(first + k) * kUnitCap + (v - s_off[k]);
            Unit r;
            r.m = __ldcg(&src->m), r.lo = __ldcg(&src->lo), r.hi = __ldcg(&src->hi);
            return r;
        };
        if (s_poison) {  // everything here climbs globally (m may exceed the CTA); the segment above is poisoned
            for (int v = t; v < m; v += blockDim.x) lbvh_push_global<kTreelet>(o, keys, ks, load_unit(v), pend, pend_n);
            if (lev + 1 < up.nlev && t == 0) up.cnt[lev][seg] = -1;
            continue;
        }
        Unit u{};
        if (t < m) u = load_unit(t);
        // shared-memory tree over the m units (same scheme as over leaves; unit u plays leaf u)
        int *const sdelta = S.sdelta, *const sslot = S.sslot, *const wn = S.wn, *const smark = S.smark;
        int *const uh = S.spar_int;  // unit heights
        int *const nh = S.spar_leaf;  // node heights (stored like the boxes)
        BoxArr &ubox = S.slbox, &nbox = S.snbox;
        int2 *const uab = S.schild;   // unit leaf ranges
        int4 (*const wl)[kChunk] = S.wl;
        sslot[t] = kSlotEmpty, smark[t] = kNone;
        if (t <= kMaxRounds) wn[t] = 0;
        if (t < m) {
            uab[t] = make_int2(u.m.x, u.m.y);
            uh[t] = u.m.z;
            ubox[t] = Box6{u.lo.x, u.lo.y, u.lo.z, u.hi.x, u.hi.y, u.hi.z};
            sdelta[t] = unpack_dl(u.m.w);  // the unit's boundary LCPs travel with it
            if (t == m - 1) sdelta[m] = unpack_dr(u.m.w);
        }
        __syncthreads();
        int count = m;
        for (int round = 0; count > 0; ++round) {
            int4 next = make_int4(0, 0, 0, 0);
            bool push = false;
            if (t < count) {
                int U = t, W = t;
                if (round > 0) {  // complete the node over units [U2, W2], split at gap gs (second arrival last round)
                    const int4 e = wl[round & 1][t];
                    const int U2 = e.x, W2 = e.y, gs = e.z;
                    const int L = uab[U2].x, R = uab[W2].y, g = uab[gs].y;  // leaves; split after leaf g
                    const Box6 A = U2 == gs ? (Box6)ubox[gs] : (Box6)nbox[gs];
                    const Box6 B = W2 == gs + 1 ? (Box6)ubox[gs + 1] : (Box6)nbox[gs + 1];
                    int ha = 0, hb = 0;
                    if (kTreelet) {
                        ha = trav_height(o, L, g, U2 == gs ? uh[gs] : nh[gs]);
                        hb = trav_height(o, g + 1, R, W2 == gs + 1 ? uh[gs + 1] : nh[gs + 1]);
                    }
                    const int dlp = sdelta[U2], drp = sdelta[W2 + 1];
                    const bool root = dlp < 0 && drp < 0;
                    const Box6 bu = box_union(A, B);
                    put_node(o, root ? 0 : (drp > dlp ? R : L), g, L, R, A, B, ha, hb);
                    const int q = root ? 0 : (drp > dlp ? W2 : U2);
                    nbox[q] = bu;
                    const int hh = 1 + max(ha, hb);
                    if (kTreelet) nh[q] = hh;
                    if (root) {
                        box_store(o.nodebox, bu, kTreelet ? hh : 0);
                        if (kTreelet) *o.wneed = (unsigned int)(hh + 1 + 3);
                    }
                    U = U2, W = W2;
                }
                const int dl = sdelta[U], dr = sdelta[W + 1];
                if (dl >= 0 || dr >= 0) {
                    const bool left = dr > dl;
                    const int gs = left ? W : U - 1;  // the gap between units gs and gs + 1
                    if (gs < 0 || gs > m - 2) {
                        smark[U] = W;
                    } else {
                        const int other = atomicExch(&sslot[gs], left ? U : W);
                        if (other != kSlotEmpty) {
                            sslot[gs] = kSlotDone;
                            next = make_int4(left ? U : other, left ? other : W, gs, 0);
                            push = true;
                        }
                    }
                }
            }
            append_item(wl[(round + 1) & 1], &wn[round + 1], push, next);
            __syncthreads();
            count = wn[round + 1];
        }
        if (t < m - 1) {
            const int f = sslot[t];
            if (f >= 0) {
                if (f <= t)
                    smark[f] = t;
                else
                    smark[t + 1] = f;
            }
        }
        __syncthreads();
        if (lev + 1 >= up.nlev) return;  // the top group: the root is complete
        auto unit_of = [&](int p, int e) -> Unit {
            const int dl = sdelta[p], dr = sdelta[e + 1];
            const int q = p == e ? p : (dr > dl ? e : p);
            const Box6 bx = p == e ? ubox[p] : nbox[q];
            const int hh = p == e ? uh[p] : (kTreelet ? nh[q] : 0);
            return Unit{make_int4(uab[p].x, uab[e].y, hh, pack_deltas(dl, dr)), make_float4(bx.lx, bx.ly, bx.lz, 0.f),
                        make_float4(bx.hx, bx.hy, bx.hz, 0.f)};
        };
        lbvh_emit<kTreelet>(o, keys, ks, up, lev, seg, m, smark, S.swarp, unit_of, pend, pend_n);
    }
}

// kTreelet: after a node completes in shared memory, the treelet of its <= 4 grandchildren is
// re-linked into the lowest-SAH of its binary topologies (3 with 3 leaves, 15 with 4: the 3
// balanced pairings and 12 chains; Karras & Aila 2013's exhaustive treelet search at size 4, done
// bottom-up inside the build) — the node keeps its index and box, its internal children keep
// their indices. The subtree leaf ranges stop being contiguous (range[] is kept for the treelet
// roots only; the scene is marked restructured).
template <bool kTreelet>
__global__ void __launch_bounds__(kChunk, kTreelet ? (kChunk <= 256 ? 4 : 2) : FGL_LBVH_MINB) k_lbvh(const float *__restrict__ verts, int64_t V,
                                                 const int32_t *__restrict__ tris, const uint32_t *__restrict__ perm,
                                                 const uint64_t *__restrict__ keys, int ks, uint64_t pmask,
                                                 float4 *__restrict__ tri, LbvhOut o, int4 *__restrict__ pend,
                                                 unsigned int *pend_n, UpPlan up) {
    extern __shared__ __align__(16) unsigned char lbvh_smem[];
    LbvhSmem<kTreelet> &S = *reinterpret_cast<LbvhSmem<kTreelet> *>(lbvh_smem);
    int *const sdelta = S.sdelta, *const sslot = S.sslot, *const wn = S.wn, *const sheight = S.sheight;
    int *const spar_int = S.spar_int, *const spar_leaf = S.spar_leaf, *const smark = S.smark;
    BoxArr &slbox = S.slbox, &snbox = S.snbox;
    int4 *const sref = S.sref;
    int2 *const schild = S.schild, *const srange = S.srange;
    int4 (*const wl)[kChunk] = S.wl;
    const int n = o.n, t = threadIdx.x, c0 = blockIdx.x * kChunk, cnt = min(kChunk, n - c0), j = c0 + t;
    sslot[t] = kSlotEmpty;
    if (t <= kMaxRounds) wn[t] = 0;
    schild[t] = make_int2(kNone, kNone);
    spar_int[t] = kNone, spar_leaf[t] = kNone, smark[t] = kNone;
#if FGL_LBVH_ORDERED
    S.spos[t] = make_int2(kNone, kNone);
#endif
    // staged parent links: child ref c (internal index or ~leaf, both inside the chunk) -> idx
    auto stage_parent = [&](int32_t c, int idx) {
        if (c >= 0)
            spar_int[c - c0] = idx;
        else
            spar_leaf[~c - c0] = idx;
    };
    Box6 box{};
    if (t < cnt) {
        const uint64_t key = __ldg(keys + j);
        const uint32_t k = perm ? __ldg(perm + j) : (uint32_t)(key & pmask);
        const int3 ti = ldtri(tris, (int64_t)k);
        const float3 a = ldv2(verts, clampv(ti.x, V)), b = ldv2(verts, clampv(ti.y, V)), c = ldv2(verts, clampv(ti.z, V));
        tri[kTriStride * (int64_t)j] = make_float4(a.x, a.y, a.z, __int_as_float((int32_t)k));
        tri[kTriStride * (int64_t)j + 1] = make_float4(b.x, b.y, b.z, 0.f);
        tri[kTriStride * (int64_t)j + 2] = make_float4(c.x, c.y, c.z, 0.f);
        box = Box6{fminf(a.x, fminf(b.x, c.x)), fminf(a.y, fminf(b.y, c.y)), fminf(a.z, fminf(b.z, c.z)),
                   fmaxf(a.x, fmaxf(b.x, c.x)), fmaxf(a.y, fmaxf(b.y, c.y)), fmaxf(a.z, fmaxf(b.z, c.z))};
        slbox[t] = box;
        if (o.all_boxes) box_store(o.leafbox + 2 * (int64_t)j, box);
        sdelta[t] = adj_delta(keys, n, j - 1, ks);
        if (t == cnt - 1) sdelta[cnt] = adj_delta(keys, n, j, ks);
    }
    __syncthreads();
    // phase 1, bottom-up in rounds: round k holds the nodes completed in round k - 1 (round 0: the
    // leaves), compacted onto the first threads, so the climb runs on dense warps; two children meet
    // at their parent's split slot in shared memory, the second completes the parent.
    // a node is completed one round after its second child arrived (after the barrier), so the
    // children's boxes and records are visible without a fence; the exchange at the slot only has to
    // decide who is second
    // leaf pairs (the node split at j covers exactly [j, j + 1]: delta(j, j + 1) exceeds both
    // neighbours' deltas) are completed in round 0 by the left leaf's thread; the right leaf stays idle
    const bool pair_split = t + 1 < cnt && sdelta[t + 1] > sdelta[t] && sdelta[t + 1] > sdelta[t + 2];
    const bool pair_right = t >= 1 && t < cnt && sdelta[t] > sdelta[t - 1] && sdelta[t] > sdelta[t + 1];
    int count = cnt;
    for (int round = 0; count > 0; ++round) {
        int4 next = make_int4(0, 0, 0, 0);
        bool push = false;
        if (t < count && !(round == 0 && pair_right)) {
            int l = j, r = j;
            if (round > 0 || pair_split) {
                const int4 e = round > 0 ? wl[round & 1][t] : make_int4(j, j + 1, j, 0);  // (L, R, split)
                const int L = e.x, R = e.y, gp = e.z;
                int h = 0;
                // both children: [L, gp] and [gp + 1, R]
                const Box6 A = L == gp ? slbox[L - c0] : snbox[gp - c0];
                const Box6 B = R == gp + 1 ? slbox[R - c0] : snbox[gp + 1 - c0];
                const int dlp = sdelta[L - c0], drp = sdelta[R + 1 - c0];
                const bool root = dlp < 0 && drp < 0;
                const int K = root ? 0 : (drp > dlp ? R : L);
                const Box6 u = box_union(A, B);
                srange[K - c0] = make_int2(L, R);
                if (K == 0) spar_int[0] = -1;
                if constexpr (kTreelet) {
                    const int32_t cl = L == gp ? ~gp : gp, cr = R == gp + 1 ? ~(gp + 1) : gp + 1;
                    // children: refs, node64 refs (leaf_size collapse), heights; boxes stay in smem
                    const int nl = gp - L + 1, nrr = R - gp;
                    const bool ia = cl >= 0 && nl > o.leaf_size, ib = cr >= 0 && nrr > o.leaf_size;
                    const int32_t ncl = ia ? cl : make_leaf(L, nl), ncr = ib ? cr : make_leaf(gp + 1, nrr);
                    const int hcl = ia ? sheight[cl - c0] : 0, hcr = ib ? sheight[cr - c0] : 0;
                    auto boxof = [&](int32_t c) -> Box6 { return c >= 0 ? (Box6)snbox[c - c0] : (Box6)slbox[~c - c0]; };
                    auto hof = [&](int32_t c, int32_t nr) -> int { return nr >= 0 ? sheight[c - c0] : 0; };
                    // internal node idx takes children (ca, na, ha) and (cb, nb, hb): staged links,
                    // record, box (children's boxes re-read: a child re-linked just before is current)
                    auto link = [&](int idx, int32_t ca, int32_t na, int ha, int32_t cb, int32_t nb, int hb) {
                        schild[idx - c0] = make_int2(ca, cb);
                        stage_parent(ca, idx);
                        stage_parent(cb, idx);
                        sref[idx - c0] = make_int4(ca, cb, na, nb);
                        snbox[idx - c0] = box_union(boxof(ca), boxof(cb));
                        sheight[idx - c0] = 1 + max(ha, hb);
                    };
                    auto sel4 = [](int i, int v0, int v1, int v2, int v3) { return i == 0 ? v0 : (i == 1 ? v1 : (i == 2 ? v2 : v3)); };
                    int choice = -1;  // -1: keep the Karras topology
                    int xc0 = 0, xc1 = 0, xc2 = 0, xc3 = 0, xn0 = 0, xn1 = 0, xn2 = 0, xn3 = 0;
                    if ((ia || ib) && R - L + 1 >= FGL_TREELET_MIN) {  // small subtrees: little SAH to gain
                        // treelet leaves: x0, x1 under the left child (or the left child), x2, x3 likewise
                        const int4 ra = ia ? sref[cl - c0] : make_int4(cl, cl, ncl, ncl);
                        const int4 rb = ib ? sref[cr - c0] : make_int4(cr, cr, ncr, ncr);
                        xc0 = ra.x, xc1 = ra.y, xn0 = ra.z, xn1 = ra.w, xc2 = rb.x, xc3 = rb.y, xn2 = rb.z, xn3 = rb.w;
                        if (!(ia && ib)) {
                            // 3 leaves y0 y1 y2 (the leaf child at lc): chains only, w alone, the others paired
                            if (!ia) xc1 = xc2, xn1 = xn2, xc2 = xc3, xn2 = xn3;  // y = (leaf, x2, x3)
                            const Box6 y0 = boxof(xc0), y1 = boxof(xc1), y2 = boxof(xc2);
                            const int lc = ia ? 2 : 0;
                            const float a01 = box_area(box_union(y0, y1)), a02 = box_area(box_union(y0, y2)),
                                        a12 = box_area(box_union(y1, y2));
                            float best = (lc == 2 ? a01 : a12) * 0.9999f;
                            if (lc != 0 && a12 < best) best = a12, choice = 0;
                            if (a02 < best) best = a02, choice = 1;
                            if (lc != 2 && a01 < best) best = a01, choice = 2;
                            if (choice >= 0) {
                                const int I0 = ia ? cl : cr;
                                const int p = choice == 0 ? 1 : 0, q = choice == 2 ? 1 : 2;
                                const int cp = sel4(p, xc0, xc1, xc2, 0), np = sel4(p, xn0, xn1, xn2, 0);
                                const int cq = sel4(q, xc0, xc1, xc2, 0), nq = sel4(q, xn0, xn1, xn2, 0);
                                const int cw = sel4(choice, xc0, xc1, xc2, 0), nw = sel4(choice, xn0, xn1, xn2, 0);
                                link(I0, cp, np, hof(cp, np), cq, nq, hof(cq, nq));
                                link(K, cw, nw, hof(cw, nw), I0, I0, sheight[I0 - c0]);
                            }
                        } else {
                            float pa[4][4];
                            {
                                const Box6 xb[4] = {boxof(xc0), boxof(xc1), boxof(xc2), boxof(xc3)};
#pragma unroll
                                for (int a = 0; a < 4; ++a)
#pragma unroll
                                    for (int b = a + 1; b < 4; ++b) pa[a][b] = pa[b][a] = box_area(box_union(xb[a], xb[b]));
                                float best = (pa[0][1] + pa[2][3]) * 0.9999f;
                                // balanced: (0 1 | 2 3) is the current one; (0 2 | 1 3) = 1, (0 3 | 1 2) = 2
                                if (pa[0][2] + pa[1][3] < best) best = pa[0][2] + pa[1][3], choice = 1;
                                if (pa[0][3] + pa[1][2] < best) best = pa[0][3] + pa[1][2], choice = 2;
                                // chains: w alone at the top, z next, the remaining pair at the bottom
#pragma unroll
                                for (int w = 0; w < 4; ++w) {
                                    const int o1 = (w + 1) & 3, o2 = (w + 2) & 3, o3 = (w + 3) & 3;
                                    const float tri_a = box_area(box_union(box_union(xb[o1], xb[o2]), xb[o3]));
                                    if (tri_a + pa[o2][o3] < best) best = tri_a + pa[o2][o3], choice = 3 + 3 * w + 0;
                                    if (tri_a + pa[o1][o3] < best) best = tri_a + pa[o1][o3], choice = 3 + 3 * w + 1;
                                    if (tri_a + pa[o1][o2] < best) best = tri_a + pa[o1][o2], choice = 3 + 3 * w + 2;
                                }
                            }
                            if (choice >= 0) {
                                // leaf slots: pair (s0, s1) under cl, (s2, s3) under cr (balanced); chain:
                                // w alone under K, z with cr under cl, (s2, s3) under cr
                                int s0, s1, s2, s3;
                                if (choice == 1) s0 = 0, s1 = 2, s2 = 1, s3 = 3;
                                else if (choice == 2) s0 = 0, s1 = 3, s2 = 1, s3 = 2;
                                else {
                                    const int w = (choice - 3) / 3, zs = (choice - 3) % 3;
                                    const int o1 = (w + 1) & 3, o2 = (w + 2) & 3, o3 = (w + 3) & 3;
                                    s0 = w, s1 = zs == 0 ? o1 : (zs == 1 ? o2 : o3);
                                    s2 = zs == 0 ? o2 : o1, s3 = zs == 2 ? o2 : o3;
                                }
                                const int c0_ = sel4(s0, xc0, xc1, xc2, xc3), n0_ = sel4(s0, xn0, xn1, xn2, xn3);
                                const int c1_ = sel4(s1, xc0, xc1, xc2, xc3), n1_ = sel4(s1, xn0, xn1, xn2, xn3);
                                const int c2_ = sel4(s2, xc0, xc1, xc2, xc3), n2_ = sel4(s2, xn0, xn1, xn2, xn3);
                                const int c3_ = sel4(s3, xc0, xc1, xc2, xc3), n3_ = sel4(s3, xn0, xn1, xn2, xn3);
                                link(cr, c2_, n2_, hof(c2_, n2_), c3_, n3_, hof(c3_, n3_));
                                if (choice <= 2) {
                                    link(cl, c0_, n0_, hof(c0_, n0_), c1_, n1_, hof(c1_, n1_));
                                    link(K, cl, cl, sheight[cl - c0], cr, cr, sheight[cr - c0]);
                                } else {
                                    link(cl, c1_, n1_, hof(c1_, n1_), cr, cr, sheight[cr - c0]);
                                    link(K, c0_, n0_, hof(c0_, n0_), cl, cl, sheight[cl - c0]);
                                }
                            }
                        }
                    }
                    if (choice < 0) {  // the Karras pair stays: its boxes are in registers already
                        schild[K - c0] = make_int2(cl, cr);
                        stage_parent(cl, K);
                        stage_parent(cr, K);
                        sref[K - c0] = make_int4(cl, cr, ncl, ncr);
                        snbox[K - c0] = u;
                        sheight[K - c0] = 1 + max(hcl, hcr);
                    }
                    h = sheight[K - c0];
                } else {
                    const int32_t cl = L == gp ? ~gp : gp, cr = R == gp + 1 ? ~(gp + 1) : gp + 1;
                    schild[K - c0] = make_int2(cl, cr);
                    stage_parent(cl, K);
                    stage_parent(cr, K);
                    snbox[K - c0] = u;
                }
                if (o.all_boxes || root) box_store(o.nodebox + 2 * (int64_t)K, u, kTreelet ? h : 0);
                if (kTreelet && root) *o.wneed = (unsigned int)(h + 1 + 3);
                l = L, r = R;
            }
            const int dl = sdelta[l - c0], dr = sdelta[r + 1 - c0];
            if (dl >= 0 || dr >= 0) {  // not the root
                const bool left = dr > dl;
                const int gp = left ? r : l - 1;
                if (gp < c0 || gp > c0 + cnt - 2) {  // split on a chunk boundary: an output unit
                    smark[l - c0] = r - c0;
                } else {
                    const int s = gp - c0;
                    const int other = atomicExch(&sslot[s], left ? l : r);
                    if (other != kSlotEmpty) {  // second to arrive: the parent completes next round
                        sslot[s] = kSlotDone;
                        next = make_int4(left ? l : other, left ? other : r, gp, 0);
                        push = true;
                    }
                }
            }
        }
#if FGL_LBVH_ORDERED
        // the next round's items in split order (ranked by ballots), so consecutive threads complete
        // nodes at nearby positions: their shared-memory reads and writes spread over the banks
        if (push) S.spos[next.z - c0] = make_int2(next.x, next.y);
        __syncthreads();
        {
            const int2 e = t < cnt ? S.spos[t] : make_int2(kNone, kNone);
            const bool has = e.x != kNone;
            const unsigned bal = __ballot_sync(0xffffffffu, has);
            const int lane = t & 31, w = t >> 5;
            if (lane == 0) S.swarp[w] = __popc(bal);
            __syncthreads();
            int before = 0, total = 0;
#pragma unroll
            for (int k = 0; k < kChunk / 32; ++k) {
                const int c = S.swarp[k];
                before += k < w ? c : 0;
                total += c;
            }
            if (has) {
                wl[(round + 1) & 1][before + __popc(bal & ((1u << lane) - 1u))] = make_int4(e.x, e.y, c0 + t, 0);
                S.spos[t] = make_int2(kNone, kNone);
            }
            count = total;
        }
        __syncthreads();
#else
        append_item(wl[(round + 1) & 1], &wn[round + 1], push, next);
        __syncthreads();
        count = wn[round + 1];
#endif
    }
    // first arrivals whose sibling never came: their parent spans the chunk boundary (output units)
    if (t < cnt - 1) {
        const int f = sslot[t];
        if (f >= 0) {
            const int g = c0 + t;  // positions relative to the chunk
            if (f <= g)
                smark[f - c0] = t;
            else
                smark[t + 1] = f - c0;
        }
    }
    // write the staged nodes out, node K = c0 + t by thread t (coalesced rows, holes where a node
    // spans the chunk boundary: the levels above write those)
    auto write_out = [&]() {
        if (t < cnt) {
            const int K = c0 + t;
            const int2 ch = schild[t];
            if (ch.x != kNone) {
                o.child[K] = ch;
                o.range[K] = srange[t];
                int32_t r0, r1;
                if constexpr (kTreelet) {
                    const int4 rf = sref[t];
                    r0 = rf.z, r1 = rf.w;
                } else {
                    auto nref = [&](int32_t c) -> int32_t {
                        if (c < 0) return make_leaf(~c, 1);
                        const int2 rg = srange[c - c0];
                        const int count = rg.y - rg.x + 1;
                        return count <= o.leaf_size ? make_leaf(rg.x, count) : c;
                    };
                    r0 = nref(ch.x), r1 = nref(ch.y);
                }
                const Box6 a = ch.x >= 0 ? snbox[ch.x - c0] : slbox[~ch.x - c0];
                const Box6 b = ch.y >= 0 ? snbox[ch.y - c0] : slbox[~ch.y - c0];
                Node64 nd;
                nd.a = make_float4(a.lx, a.hx, a.ly, a.hy);
                nd.b = make_float4(b.lx, b.hx, b.ly, b.hy);
                nd.c = make_float4(a.lz, a.hz, b.lz, b.hz);
                nd.d = make_int4(r0, r1, 0, 0);
                o.nodes[K] = nd;
            }
            if (spar_int[t] != kNone) o.parent[K] = spar_int[t];
            if (spar_leaf[t] != kNone) o.parent[(n - 1) + K] = spar_leaf[t];
        }
    };
    if (up.nlev <= 1) {  // a single chunk: the root completed here
        write_out();
        return;
    }
    __syncthreads();  // smark complete
    // the chunk's units in leaf order; position p = leaf c0 + p; a node [l, r] is stored at its
    // Karras index (r if a left child, l if a right child) - c0
    auto unit_of = [&](int p, int e) -> Unit {
        const int l = c0 + p, r = c0 + e;
        const int dl = sdelta[p], dr = sdelta[e + 1];
        const int q = l == r ? p : (dr > dl ? e : p);
        const Box6 bx = l == r ? slbox[p] : snbox[q];
        const int hh = (kTreelet && l != r) ? sheight[q] : 0;
        return Unit{make_int4(l, r, hh, pack_deltas(dl, dr)), make_float4(bx.lx, bx.ly, bx.lz, 0.f),
                    make_float4(bx.hx, bx.hy, bx.hz, 0.f)};
    };
    const bool force = (up.force_global & 1) || ((up.force_global & 2) && (blockIdx.x & 1));
    lbvh_emit<kTreelet>(o, keys, ks, up, 0, blockIdx.x, cnt, smark, S.swarp, unit_of, pend, pend_n, force);
    // arrive at the group one level up (thread 0: release fence + counter) while the others write
    // the staged nodes out
    __shared__ int s_arr;
    if (t == 0) {
        const int group = blockIdx.x / up.G, gsize = min(up.G, up.nseg[0] - group * up.G);
        __threadfence();
        s_arr = atomicAdd(up.ctr[1] + group, 1u) == (unsigned)(gsize - 1);
        if (s_arr) up.ctr[1][group] = 0;
    }
    write_out();
    __syncthreads();
    if (!s_arr) return;
    lbvh_levels<kTreelet>(o, keys, ks, up, blockIdx.x, S, pend, pend_n, true);
}

// The tree above the chunks: every pending node climbs through the global slots (all chunks' pending
// nodes at once, so the fenced chain is paid once, not per chunk).
template <bool kTreelet>
__global__ void __launch_bounds__(256) k_lbvh_top(const uint64_t *__restrict__ keys, int ks, LbvhOut o,
                                                  const int4 *__restrict__ pend, const unsigned int *pend_n,
                                                  const unsigned int *epoch_p) {
    o.epoch = *epoch_p;
    const unsigned int cnt = *pend_n;
    for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int4 e = pend[i];
        const int l = e.x, r = e.y;
        const int dl = adj_delta(keys, o.n, l - 1, ks), dr = adj_delta(keys, o.n, r, ks);
        int hb;
        const Box6 box = box_load_cg(l == r ? o.leafbox + 2 * (int64_t)l : o.nodebox + 2 * (int64_t)(dr > dl ? r : l), hb);
        lbvh_global_climb<kTreelet>(o, keys, ks, l, r, dl, dr, box, e.z, true);
    }
}

// depth of every internal node (root = 0) by walking the parent links (L2-resident, ~log T steps)
__global__ void __launch_bounds__(256) k_depth(int64_t n, const int32_t *__restrict__ parent,
                                               int32_t *__restrict__ depth) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n - 1; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t d = 0;
        for (int32_t p = __ldg(parent + i); p >= 0; p = __ldg(parent + p)) ++d;
        depth[i] = d;
    }
}

// 4-wide nodes: every even-depth internal node n with more than leaf_size triangles (and the
// root) absorbs its two children; each child is a leaf (<= leaf_size triangles), or is replaced by
// its own two children (leaves, or odd-depth... i.e. the next even-depth wide nodes).
__global__ void __launch_bounds__(256) k_nodes4(int64_t n, int leaf_size, const int2 *__restrict__ child,
                                                const int2 *__restrict__ range, const int32_t *__restrict__ depth,
                                                const float4 *__restrict__ leafbox,
                                                const float4 *__restrict__ nodebox, Node128 *__restrict__ nodes4,
                                                int quantized) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n - 1; i += (int64_t)gridDim.x * blockDim.x) {
        const int2 ri = range[i];
        if (i != 0 && ((depth[i] & 1) || ri.y - ri.x + 1 <= leaf_size)) continue;
        float lo[3][4], hi[3][4];
        int32_t ref[4];
        int k = 0;
        auto emit = [&](int32_t c) {
            float4 l, h;
            if (c < 0) {
                const int32_t j = ~c;
                ref[k] = make_leaf(j, 1);
                l = leafbox[2 * (int64_t)j], h = leafbox[2 * (int64_t)j + 1];
            } else {
                const int2 r = range[c];
                const int32_t cnt = r.y - r.x + 1;
                ref[k] = cnt <= leaf_size ? make_leaf(r.x, cnt) : c;
                l = nodebox[2 * (int64_t)c], h = nodebox[2 * (int64_t)c + 1];
            }
            lo[0][k] = l.x, lo[1][k] = l.y, lo[2][k] = l.z, hi[0][k] = h.x, hi[1][k] = h.y, hi[2][k] = h.z;
            ++k;
        };
        const int2 ci = child[i];
        const int32_t cc[2] = {ci.x, ci.y};
        for (int s = 0; s < 2; ++s) {
            const int32_t c = cc[s];
            bool expand = false;
            if (c >= 0) {
                const int2 r = range[c];
                expand = r.y - r.x + 1 > leaf_size;
            }
            if (!expand) {
                emit(c);
            } else {
                const int2 g = child[c];
                emit(g.x);
                emit(g.y);
            }
        }
        const int valid = k;
        if (quantized) {
            NodeQ q;
            uint32_t bits = 0, qlo[3] = {0, 0, 0}, qhi[3] = {0, 0, 0};
            float p[3];
            for (int a = 0; a < 3; ++a) {
                float plo = lo[a][0], phi = hi[a][0];
                for (int c = 1; c < valid; ++c) plo = fminf(plo, lo[a][c]), phi = fmaxf(phi, hi[a][c]);
                p[a] = plo;
                // smallest e with 255 * 2^e >= the (round-up) extent
                const float ext = __fsub_ru(phi, plo);
                int e = -126;
                if (ext > 0.f) {
                    int x;
                    const float m = frexpf(__fdiv_ru(ext, 255.f), &x);  // r = m 2^x, m in [0.5, 1)
                    e = m == 0.5f ? x - 1 : x;
                    e = e < -126 ? -126 : (e > 127 ? 127 : e);
                }
                bits |= (uint32_t)(e + 127) << (8 * a);
                for (int c = 0; c < valid; ++c) {
                    const float fl = floorf(ldexpf(__fsub_rd(lo[a][c], plo), -e));
                    const float fh = ceilf(ldexpf(__fsub_ru(hi[a][c], plo), -e));
                    const uint32_t bl = fl <= 0.f ? 0u : (fl >= 255.f ? 255u : (uint32_t)fl);
                    const uint32_t bh = fh <= 0.f ? 0u : (fh >= 255.f ? 255u : (uint32_t)fh);
                    qlo[a] |= bl << (8 * c);
                    qhi[a] |= bh << (8 * c);
                }
            }
            bits |= (uint32_t)((1u << valid) - 1u) << 24;
            for (int c = valid; c < 4; ++c) ref[c] = kEmptyRef;
            q.f0 = make_float4(p[0], p[1], p[2], __uint_as_float(bits));
            q.q0 = make_int4((int)qlo[0], (int)qhi[0], (int)qlo[1], (int)qhi[1]);
            q.q1 = make_int4((int)qlo[2], (int)qhi[2], ref[0], ref[1]);
            q.q2 = make_int4(ref[2], ref[3], 0, 0);
            reinterpret_cast<NodeQ *>(nodes4)[i] = q;
            continue;
        }
        for (; k < 4; ++k) {
            ref[k] = kEmptyRef;
            for (int a = 0; a < 3; ++a) lo[a][k] = hi[a][k] = kFarBox;
        }
        Node128 nd;
        for (int a = 0; a < 3; ++a) {
            nd.f[2 * a] = make_float4(lo[a][0], lo[a][1], lo[a][2], lo[a][3]);
            nd.f[2 * a + 1] = make_float4(hi[a][0], hi[a][1], hi[a][2], hi[a][3]);
        }
        nd.ref = make_int4(ref[0], ref[1], ref[2], ref[3]);
        nd.meta = make_int4(valid, depth[i], 0, 0);
        nodes4[i] = nd;
    }
}

// T == 1: a root whose first child is the single leaf and whose other children are empty
__global__ void k_single4(const float4 *__restrict__ leafbox, Node128 *__restrict__ nodes4, int quantized) {
    const float4 lo = leafbox[0], hi = leafbox[1];
    if (quantized) {  // one child covering the whole box: q = (0, 255) on every axis
        NodeQ q;
        uint32_t bits = 1u << 24;
        const float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
        for (int a = 0; a < 3; ++a) {
            const float ext = __fsub_ru(h[a], l[a]);
            int e = -126;
            if (ext > 0.f) {
                int x;
                const float m = frexpf(__fdiv_ru(ext, 255.f), &x);
                e = m == 0.5f ? x - 1 : x;
                e = e < -126 ? -126 : (e > 127 ? 127 : e);
            }
            bits |= (uint32_t)(e + 127) << (8 * a);
        }
        q.f0 = make_float4(lo.x, lo.y, lo.z, __uint_as_float(bits));
        q.q0 = make_int4(0, 255, 0, 255);
        q.q1 = make_int4(0, 255, make_leaf(0, 1), kEmptyRef);
        q.q2 = make_int4(kEmptyRef, kEmptyRef, 0, 0);
        reinterpret_cast<NodeQ *>(nodes4)[0] = q;
        return;
    }
    Node128 nd;
    const float F = kFarBox;
    nd.f[0] = make_float4(lo.x, F, F, F), nd.f[1] = make_float4(hi.x, F, F, F);
    nd.f[2] = make_float4(lo.y, F, F, F), nd.f[3] = make_float4(hi.y, F, F, F);
    nd.f[4] = make_float4(lo.z, F, F, F), nd.f[5] = make_float4(hi.z, F, F, F);
    nd.ref = make_int4(make_leaf(0, 1), kEmptyRef, kEmptyRef, kEmptyRef);
    nd.meta = make_int4(1, 0, 0, 0);
    nodes4[0] = nd;
}

// T == 1: a root whose first child is the single leaf and whose second child is empty
__global__ void k_single(const float4 *__restrict__ leafbox, Node64 *__restrict__ nodes) {
    float4 lo = leafbox[0], hi = leafbox[1];
    Node64 nd;
    nd.a = make_float4(lo.x, hi.x, lo.y, hi.y);
    nd.b = make_float4(kFarBox, kFarBox, kFarBox, kFarBox);
    nd.c = make_float4(lo.z, hi.z, kFarBox, kFarBox);
    nd.d = make_int4(make_leaf(0, 1), kEmptyRef, 0, 0);
    nodes[0] = nd;
}

inline int grid_for(int64_t n, int threads = 256, int max_blocks = 148 * 16) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, max_blocks));
}

}  // namespace

void launch_validate(const float *verts, int64_t V, const int32_t *tris, int64_t T, unsigned int *flag,
                     cudaStream_t s) {
    FGL_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), s));
    k_validate<<<grid_for(3 * std::max(T, V) / 4 + 1), 256, 0, s>>>(verts, V, tris, T, flag);
    FGL_LAUNCHED("k_validate");
}

void launch_morton_points(const float *pts, int64_t n, const float *lo, const float *hi, int bits, uint64_t *codes,
                          cudaStream_t s) {
    if (n <= 0) return;
    BoxArg bx;
    for (int i = 0; i < 3; ++i) bx.lo[i] = lo[i], bx.hi[i] = hi[i];
    k_morton_points<<<grid_for(n), 256, 0, s>>>(pts, n, bx, bits, codes);
    FGL_LAUNCHED("k_morton_points");
}

// Eq. 5 codes of b.cent within b.box, then the stable sort (A3-A4). Sets b.packed_shift and
// b.sorted_slot; the leaf order is then perm_at(b, j).
void launch_morton_sort(BuildBuffers &b, int bits, int cubic, cudaStream_t s) {
    const int64_t T = b.T;
    const int key_bits = 3 * bits;
    FGL_CUDA(cudaMemsetAsync(b.ghist, 0, sizeof(uint32_t) * 8 * 256, s));
    // key-only sort when the triangle index fits below the code: (code << ib) | index sorts like the
    // stable (code, index) pairs and moves 8 instead of 12 bytes per key and pass
    int ib = 1;
    while ((int64_t(1) << ib) < T) ++ib;
    const int ps = (FGL_SORT_PACKED && key_bits + ib <= 64) ? ib : 0;
    b.packed_shift = ps;
    k_morton<<<grid_for(T, 256, FGL_MORTON_BLOCKS), 256, 0, s>>>(b.cent, T, b.box, bits, cubic, b.keys[0], ps ? nullptr : b.vals[0],
                                                       ps, b.ghist);
    FGL_LAUNCHED("k_morton");
    int slot = 0;
    radix_sort_pairs(b.keys[0], ps ? nullptr : b.vals[0], b.keys[1], ps ? nullptr : b.vals[1], T, key_bits,
                     b.sort_status, b.sort_tiles, b.ghist, true, &slot, s, ps, b.sort_rts);
    b.sorted_slot = slot;
}

// Karras tree (A5), Eq. 7 boxes (A6) and traversal nodes (A7) from the leaf boxes and the first
// aggregate level written by the primitive-specific reorder kernel.
static AggLevels launch_aggregates(BuildBuffers &b, cudaStream_t s) {
    const int64_t T = b.T;
    AggLevels L;
    L.leaf = b.leafbox;
    L.agg = b.agg;
    L.n = T;
    L.nlev = 2;
    for (int64_t m = (T + 7) / 8, off = 0; m > 8 && L.nlev <= kMaxAgg; off += m, m = (m + 7) / 8) {
        k_aggregate<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(b.agg + 2 * off, m, b.agg + 2 * (off + m));
        FGL_LAUNCHED("k_aggregate");
        ++L.nlev;
    }
    return L;
}

static void launch_nodes(BuildBuffers &b, int leaf_size, int width, bool depth_known, cudaStream_t s) {
    const int64_t T = b.T;
    if (width == 2) {
        k_nodes<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>(T, leaf_size, b.child, b.range, b.leafbox, b.nodebox,
                                                               b.nodes);
        FGL_LAUNCHED("k_nodes");
    }
    if (width == 4) {
        if (!depth_known) {
            k_depth<<<grid_for(T - 1), 256, 0, s>>>(T, b.parent, b.depth);
            FGL_LAUNCHED("k_depth");
        }
        k_nodes4<<<grid_for(T - 1), 256, 0, s>>>(T, leaf_size, b.child, b.range, b.depth, b.leafbox, b.nodebox,
                                                 b.nodes4, b.quantized);
        FGL_LAUNCHED("k_nodes4");
    }
}

static void launch_single(BuildBuffers &b, int width, cudaStream_t s) {
    if (width == 4) {
        k_single4<<<1, 1, 0, s>>>(b.leafbox, b.nodes4, b.quantized);
        FGL_LAUNCHED("k_single4");
    } else {
        k_single<<<1, 1, 0, s>>>(b.leafbox, b.nodes);
        FGL_LAUNCHED("k_single");
    }
}

// stack bound word (BuildBuffers::wctr[3]) of a restructured width-2 tree: depth + 2 from k_depth
static void launch_stack_bound(BuildBuffers &b, cudaStream_t s) {
    const int64_t T = b.T;
    FGL_CUDA(cudaMemsetAsync(b.wctr + 3, 0, sizeof(unsigned int), s));
    k_depth<<<grid_for(T - 1), 256, 0, s>>>(T, b.parent, b.depth);
    FGL_LAUNCHED("k_depth");
    k_depth_max<<<grid_for(T - 1, 256, 148 * 4), 256, 0, s>>>(T, b.depth, b.wctr + 3);
    FGL_LAUNCHED("k_depth_max");
}

void launch_tree(BuildBuffers &b, int leaf_size, int width, int quantized, cudaStream_t s, int restructure) {
    const int64_t T = b.T;
    // a Karras tree's depth is bounded by its key and index bits (< the cast's stack): no check;
    // restructured and width-8 trees set the bound themselves
    if (width != 8) FGL_CUDA(cudaMemsetAsync(b.wctr + 3, 0, sizeof(unsigned int), s));
    b.width = width;
    b.quantized = width == 4 ? quantized : (width == 8 ? 1 : 0);
    b.restructured = 0;
    AggLevels L = launch_aggregates(b, s);
    if (T == 1) {
        if (width == 8)
            launch_wide8(b, s);
        else
            launch_single(b, width, s);
        return;
    }
    // width 2 without restructuring: k_karras writes the node64s itself (FGL_FUSED_NODES)
    const bool fused = FGL_FUSED_NODES && width == 2 && restructure == 0;
    k_karras<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>(b.keys[b.sorted_slot], (int)T, b.packed_shift, b.child,
                                                            b.range, b.parent, L, b.nodebox,
                                                            fused ? b.nodes : nullptr, leaf_size);
    FGL_LAUNCHED("k_karras");
    if (fused) return;
    if (width == 8) {  // SAH collapse of the Karras tree (single-triangle leaves) to node96q
        launch_wide8(b, s);
        return;
    }
    if (restructure < 0 && width == 2) {
        // -k: k parallel treelet passes over a depth partition, depths recomputed before each
        // (FGL_TREELET4: exhaustive 4-leaf treelets, offsets 0, 1, 0, ...; else greedy 8-leaf
        // treelets, offsets 0, 1, 2, 0, ...); nodes over 1-triangle leaves
        for (int pass = 0; pass < -restructure; ++pass) {
            k_depth<<<grid_for(T - 1), 256, 0, s>>>(T, b.parent, b.depth);
            FGL_LAUNCHED("k_depth");
#if FGL_TREELET4
            k_treelet4<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>((int32_t)T, b.child, b.parent, b.nodebox,
                                                                        b.leafbox, b.depth, pass & 1);
            FGL_LAUNCHED("k_treelet4");
#else
            k_treelet_par<<<(unsigned)((T - 1 + 127) / 128), 128, 0, s>>>((int32_t)T, b.child, b.parent, b.nodebox,
                                                                           b.leafbox, b.depth, pass % 3);
            FGL_LAUNCHED("k_treelet_par");
#endif
        }
        k_nodes_free<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>(T, b.child, b.leafbox, b.nodebox, b.nodes);
        FGL_LAUNCHED("k_nodes_free");
        launch_stack_bound(b, s);
        b.restructured = 1;
        return;
    }
    if (restructure > 0 && width == 2) {
        // costs / sizes bottom-up once, then `restructure` treelet passes; nodes over 1-triangle leaves
        for (int pass = 0; pass <= restructure; ++pass) {
            FGL_CUDA(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * (T - 1), s));
            k_treelet<<<(unsigned)((T + 255) / 256), 256, 0, s>>>((int32_t)T, b.child, b.parent, b.nodebox, b.leafbox,
                                                                  b.cost, b.tsize,
                                                                  reinterpret_cast<unsigned int *>(b.flags), pass);
            FGL_LAUNCHED("k_treelet");
        }
        k_nodes_free<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>(T, b.child, b.leafbox, b.nodebox, b.nodes);
        FGL_LAUNCHED("k_nodes_free");
        launch_stack_bound(b, s);
        b.restructured = 1;
        return;
    }
    launch_nodes(b, leaf_size, width, false, s);
}

// NEXT-4 refit: new vertex positions, same triangles and tree. Leaf records and boxes are regathered
// in the stored leaf order, then aggregates, Eq. 7 node boxes from the stored ranges, and nodes.
void launch_refit(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, int leaf_size,
                  cudaStream_t s) {
    const int64_t T = b.T;
    const int ps = b.packed_shift, slot = b.sorted_slot;
    k_reorder<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(verts, V, tris, ps ? nullptr : b.vals[slot], b.keys[slot],
                                                          ps ? (uint64_t(1) << ps) - 1 : 0, T, b.tri, b.leafbox, b.agg);
    FGL_LAUNCHED("k_reorder");
    AggLevels L = launch_aggregates(b, s);
    if (T == 1) {
        if (b.width == 8)
            launch_wide8(b, s);
        else
            launch_single(b, b.width, s);
        return;
    }
    if (b.restructured) {  // free topology: boxes bottom-up over the kept child links
        FGL_CUDA(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * (T - 1), s));
        k_treelet<<<(unsigned)((T + 255) / 256), 256, 0, s>>>((int32_t)T, b.child, b.parent, b.nodebox, b.leafbox,
                                                              b.cost, b.tsize, reinterpret_cast<unsigned int *>(b.flags),
                                                              0);
        FGL_LAUNCHED("k_treelet");
        k_nodes_free<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>(T, b.child, b.leafbox, b.nodebox, b.nodes);
        FGL_LAUNCHED("k_nodes_free");
        return;
    }
    k_refit_boxes<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>((int)T, b.range, L, b.nodebox);
    FGL_LAUNCHED("k_refit_boxes");
    if (b.width == 8) {  // the binary topology is kept; the SAH collapse is redone over the new boxes
        launch_wide8(b, s);
        return;
    }
    launch_nodes(b, leaf_size, b.width, true, s);
}

void launch_build(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, int bits, int leaf_size,
                  int cubic, int width, int quantized, cudaStream_t s, int restructure, int treelets) {
    const int64_t T = b.T;
    {
        NvtxRange r("fgl build: A2 prep (centroids, scene box)");
        k_prep<<<kPrepBlocks, 256, 0, s>>>(verts, V, tris, T, b.cent, b.partial, b.sync, b.box);
        FGL_LAUNCHED("k_prep");
    }
    {
        NvtxRange r("fgl build: A3-A4 Morton codes + radix sort");
        launch_morton_sort(b, bits, cubic, s);
    }
    const int ps = b.packed_shift, slot = b.sorted_slot;
    if ((FGL_FUSED_LBVH || treelets) && width == 2 && restructure == 0 && T >= 2) {
        // leaf records + Karras tree + Eq. 7 boxes + node64 in one pass (k_lbvh)
        NvtxRange r("fgl build: A2 leaf records + A5-A7 Karras tree, Eq. 7 boxes, node64 (fused)");
        FGL_CUDA(cudaMemsetAsync(b.wctr + 3, 0, sizeof(unsigned int), s));
        b.width = 2, b.quantized = 0, b.restructured = 0;
        static const int all_boxes = [] {
            const char *e = std::getenv("FGL_ALL_BOXES");
            return e && *e == '1' ? 1 : 0;
        }();
        LbvhOut o{b.child, b.range, b.parent, b.leafbox, b.nodebox, b.nodes, b.gslot, b.wctr + 3,
                  (int)T, leaf_size, all_boxes, 0u};
        const uint32_t *perm = ps ? nullptr : b.vals[slot];
        const uint64_t pmask = ps ? (uint64_t(1) << ps) - 1 : 0;
        const unsigned grid = (unsigned)((T + kChunk - 1) / kChunk);
        // pending list: the centroids are dead after the sort; <= 2 x (ceil(T / kChunk) - 1) x 96
        // entries (children of nodes that span a chunk boundary: the boundaries' ancestors) < T
        int4 *pend = reinterpret_cast<int4 *>(b.cent);
        UpPlan up = lbvh_plan(T, b.lbvh_up);
        if (const char *e = std::getenv("FGL_LBVH_GLOBAL")) up.force_global = std::atoi(e);
        const unsigned top_grid = (unsigned)std::min<int64_t>(148 * 8, (T + 255) / 256);
        if (treelets) {
            constexpr int sm = (int)sizeof(LbvhSmem<true>);
            FGL_CUDA(cudaFuncSetAttribute(k_lbvh<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            k_lbvh<true><<<grid, kChunk, sm, s>>>(verts, V, tris, perm, b.keys[slot], ps, pmask, b.tri, o, pend, b.sync + 2, up);
            FGL_LAUNCHED("k_lbvh");
            k_lbvh_top<true><<<top_grid, 256, 0, s>>>(b.keys[slot], ps, o, pend, b.sync + 2, b.sync + 3);
        } else {
            constexpr int sm = (int)sizeof(LbvhSmem<false>);
            FGL_CUDA(cudaFuncSetAttribute(k_lbvh<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            k_lbvh<false><<<grid, kChunk, sm, s>>>(verts, V, tris, perm, b.keys[slot], ps, pmask, b.tri, o, pend, b.sync + 2, up);
            FGL_LAUNCHED("k_lbvh");
            k_lbvh_top<false><<<top_grid, 256, 0, s>>>(b.keys[slot], ps, o, pend, b.sync + 2, b.sync + 3);
        }
        FGL_LAUNCHED("k_lbvh_top");
        b.restructured = treelets ? 1 : 0;
        return;
    }
    {
        // leaf-order records, leaf boxes and the 8-ary box aggregates used by the Eq. 7 boxes
        NvtxRange r("fgl build: A7 leaf-order records + leaf boxes");
        k_reorder<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(verts, V, tris, ps ? nullptr : b.vals[slot], b.keys[slot],
                                                              ps ? (uint64_t(1) << ps) - 1 : 0, T, b.tri, b.leafbox,
                                                              b.agg);
        FGL_LAUNCHED("k_reorder");
    }
    NvtxRange r("fgl build: A5-A7 Karras tree, Eq. 7 boxes, traversal nodes");
    launch_tree(b, leaf_size, width, quantized, s, restructure);
}

size_t lbvh_up_bytes(int64_t T) {
    const UpPlan up = lbvh_plan(std::max<int64_t>(T, 1), nullptr);
    return (size_t)reinterpret_cast<char *>(up.units[0]) + 256;
}

void launch_complete_boxes(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, cudaStream_t s) {
    const int64_t T = b.T;
    const int ps = b.packed_shift, slot = b.sorted_slot;
    k_reorder<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(verts, V, tris, ps ? nullptr : b.vals[slot], b.keys[slot],
                                                          ps ? (uint64_t(1) << ps) - 1 : 0, T, b.tri, b.leafbox, b.agg);
    FGL_LAUNCHED("k_reorder");
    AggLevels L = launch_aggregates(b, s);
    if (T >= 2 && b.restructured) {  // free topology: boxes bottom-up over the child links
        FGL_CUDA(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * (T - 1), s));
        k_treelet<<<(unsigned)((T + 255) / 256), 256, 0, s>>>((int32_t)T, b.child, b.parent, b.nodebox, b.leafbox,
                                                              b.cost, b.tsize, reinterpret_cast<unsigned int *>(b.flags),
                                                              0);
        FGL_LAUNCHED("k_treelet");
    } else if (T >= 2) {
        k_refit_boxes<<<(unsigned)((T - 1 + 255) / 256), 256, 0, s>>>((int)T, b.range, L, b.nodebox);
        FGL_LAUNCHED("k_refit_boxes");
    }
}

}  // namespace fgl
