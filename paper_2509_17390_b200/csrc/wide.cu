// Compressed 8-wide BVH ("node96q") collapsed from the binary Karras tree by SAH — SURVEY.md §8(a)
// A7 and §8(f) NEXT-4 (P:130 node layout "to maximize coalesced memory access", P:297 memory-
// conscious traversal). The collapse is the dynamic program of Ylitie, Karras & Laine (HPG 2017),
// restated here on the Karras tree of build.cu:
//
//   for a binary node n with N(n) triangles and box area A(n), and a slot budget i = 1..8,
//     C(n, i) = least SAH cost of representing n's subtree with at most i children of a wide node
//     leaf(n)       = Ct * A(n) * N(n)                       (only when N(n) <= 3)
//     internal(n)   = Ci * A(n) + min_k [C(l, k) + C(r, 8 - k)]   (n becomes a wide node)
//     C(n, 1)       = min(leaf(n), internal(n))
//     C(n, i >= 2)  = min(C(n, 1), min_{k=1..i-1} [C(l, k) + C(r, i - k)])
//   a single triangle j costs Ct * A(j) for every i.
//
// k_sah_dp evaluates it bottom-up (the second child to finish a node computes it: an atomic arrival
// counter per node); k_collapse then walks the decisions top-down from the root with a device work
// queue: each wide node (identified by the binary node it collapses, so the layout does not depend
// on the queue's scheduling) distributes its 8 slots over its binary descendants, quantises the
// children's Eq. 7 boxes to 8 bits relative to its own box (outward: floor / ceil of the
// directed-rounded offsets over power-of-two steps), assigns the children to octant slots, and
// pushes its internal children.
//
// Node layout (96 B, 3 x 32 B so the cast fetches it with three 256-bit loads):
//   c0: px, py, pz (the box's lo corner), meta = Ex | Ey << 8 | Ez << 16 | valid << 24,
//       qlo_x[8], qhi_x[8]                (child k in byte k % 4 of word k / 4)
//   c1: qlo_y[8], qhi_y[8], qlo_z[8], qhi_z[8]
//   c2: ref[8]   (>= 0: wide node = binary node index; < 0: leaf ~(first << 3 | count - 1); empty:
//                 kEmptyRef)
// Child plane a of slot k is p_a + q * 2^(E_a - 142) with E_a = e_a + 127 + 15 (the step is 2^e_a,
// stored pre-scaled by 2^15 for the cast's byte-to-float conversion, see cast.cu). Slot k's bits
// (x, y, z side of the child's box centre relative to the node's) are (k >> 2, k >> 1, k) & 1, so a
// ray visits positions k ^ X(octant) in increasing order, near side first (Ylitie et al.'s octant
// ordering with x and y most significant: the LiDAR rays are mostly horizontal).
#include "fgl_internal.cuh"

namespace fgl {

namespace {

constexpr float kCi8 = 1.0f;   // cost of one wide-node visit (relative)
constexpr float kCt8 = 0.4f;   // cost of one triangle test relative to a wide-node visit (measured
                               // instruction ratio of the two in the cast kernel)
constexpr int kLeafMax8 = 3;   // triangles per wide leaf

__device__ __forceinline__ float half_area(float4 lo, float4 hi) {
    const float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
    return dx * dy + dy * dz + dz * dx;
}

struct CostRow {
    float c[8];  // c[i - 1] = C(n, i)
};

__device__ __forceinline__ void load_costs(int32_t ref, const float *__restrict__ cost, const float4 *__restrict__ leafbox,
                                           CostRow &r) {
    if (ref < 0) {
        const int32_t j = ~ref;
        const float a = kCt8 * half_area(__ldg(leafbox + 2 * (int64_t)j), __ldg(leafbox + 2 * (int64_t)j + 1));
#pragma unroll
        for (int i = 0; i < 8; ++i) r.c[i] = a;
    } else {
        const float4 *p = reinterpret_cast<const float4 *>(cost + 8 * (int64_t)ref);
        const float4 u = __ldcg(p), v = __ldcg(p + 1);
        r.c[0] = u.x, r.c[1] = u.y, r.c[2] = u.z, r.c[3] = u.w;
        r.c[4] = v.x, r.c[5] = v.y, r.c[6] = v.z, r.c[7] = v.w;
    }
}

// D(i) = min_{k=1..i-1} L(k) + R(i - k), argmin smallest k on ties
__device__ __forceinline__ float distribute(const CostRow &L, const CostRow &R, int i, int &kbest) {
    float best = INFINITY;
    kbest = 1;
    for (int k = 1; k < i; ++k) {
        const float v = L.c[k - 1] + R.c[i - k - 1];
        if (v < best) best = v, kbest = k;
    }
    return best;
}

__device__ __forceinline__ float leaf_cost(int32_t n_tris, float area) {
    return n_tris <= kLeafMax8 ? kCt8 * area * (float)n_tris : INFINITY;
}

// the DP row of internal node n from its children's rows
__device__ void dp_row(int32_t n, const int2 *__restrict__ child, const int2 *__restrict__ range,
                       const float4 *__restrict__ nodebox, const float4 *__restrict__ leafbox, float *cost) {
    const int2 c = __ldcg(child + n), rg = __ldcg(range + n);
    CostRow L, R;
    load_costs(c.x, cost, leafbox, L);
    load_costs(c.y, cost, leafbox, R);
    const float A = half_area(__ldg(nodebox + 2 * (int64_t)n), __ldg(nodebox + 2 * (int64_t)n + 1));
    int k;
    const float internal = kCi8 * A + distribute(L, R, 8, k);
    const float c1 = fminf(leaf_cost(rg.y - rg.x + 1, A), internal);
    float out[8];
    out[0] = c1;
#pragma unroll
    for (int i = 2; i <= 8; ++i) out[i - 1] = fminf(c1, distribute(L, R, i, k));
    float4 *p = reinterpret_cast<float4 *>(cost + 8 * (int64_t)n);
    __stcg(p, make_float4(out[0], out[1], out[2], out[3]));
    __stcg(p + 1, make_float4(out[4], out[5], out[6], out[7]));
}

// bottom-up: one thread per leaf climbs; the second arrival at a node evaluates its row
__global__ void __launch_bounds__(256) k_sah_dp(int32_t T, const int2 *__restrict__ child,
                                                const int2 *__restrict__ range, const int32_t *__restrict__ parent,
                                                const float4 *__restrict__ nodebox,
                                                const float4 *__restrict__ leafbox, unsigned int *flags, float *cost) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    int32_t n = __ldg(parent + (T - 1) + j);
    while (n >= 0) {
        __threadfence();
        if (atomicAdd(flags + n, 1u) == 0u) return;  // the other subtree is not done yet
        __threadfence();
        dp_row(n, child, range, nodebox, leafbox, cost);
        n = __ldg(parent + n);
    }
}

struct Slot {
    int32_t bin;   // binary ref (>= 0 internal node, < 0 ~triangle)
    int32_t kind;  // 0 leaf, 1 internal (wide child)
};

// Slots of the wide node rooted at binary internal node n: its 8 slots distributed over n's two
// children by the DP decisions. Returns the slot count (1..8).
__device__ int collect_slots(int32_t n, const int2 *__restrict__ child, const int2 *__restrict__ range,
                             const float4 *__restrict__ nodebox, const float4 *__restrict__ leafbox,
                             const float *cost, Slot *slots) {
    int32_t sb[8], si[8];  // explicit stack of (binary ref, budget)
    int sp = 0, ns = 0;
    {
        const int2 c = __ldg(child + n);
        CostRow L, R;
        load_costs(c.x, cost, leafbox, L);
        load_costs(c.y, cost, leafbox, R);
        int k;
        distribute(L, R, 8, k);
        sb[sp] = c.y, si[sp++] = 8 - k;
        sb[sp] = c.x, si[sp++] = k;
    }
    while (sp > 0) {
        --sp;
        const int32_t m = sb[sp];
        const int i = si[sp];
        if (m < 0) {  // a single triangle: a one-triangle leaf
            slots[ns++] = Slot{m, 0};
            continue;
        }
        const int2 c = __ldg(child + m), rg = __ldg(range + m);
        CostRow L, R;
        load_costs(c.x, cost, leafbox, L);
        load_costs(c.y, cost, leafbox, R);
        const float A = half_area(__ldg(nodebox + 2 * (int64_t)m), __ldg(nodebox + 2 * (int64_t)m + 1));
        int k8, k;
        const float internal = kCi8 * A + distribute(L, R, 8, k8);
        const float lc = leaf_cost(rg.y - rg.x + 1, A);
        const float c1 = fminf(lc, internal);
        const float d = i >= 2 ? distribute(L, R, i, k) : INFINITY;
        if (c1 <= d) {
            slots[ns++] = Slot{m, lc <= internal ? 0 : 1};
        } else {
            sb[sp] = c.y, si[sp++] = i - k;
            sb[sp] = c.x, si[sp++] = k;
        }
    }
    return ns;
}

// smallest e with 255 * 2^e >= ext (ext rounded up), clamped to the representable range
__device__ __forceinline__ int step_exponent(float ext) {
    int e = -126;
    if (ext > 0.f) {
        int x;
        const float m = frexpf(__fdiv_ru(ext, 255.f), &x);  // ext / 255 = m 2^x, m in [0.5, 1)
        e = m == 0.5f ? x - 1 : x;
        e = e < -126 ? -126 : (e > 112 ? 112 : e);
    }
    return e;
}

__device__ int write_node(int32_t n, const Slot *slots, int ns, const int2 *__restrict__ range,
                          const float4 *__restrict__ nodebox, const float4 *__restrict__ leafbox, Node8 *nodes8,
                          int32_t *children, int &nchild) {
    const float4 plo = __ldg(nodebox + 2 * (int64_t)n), phi = __ldg(nodebox + 2 * (int64_t)n + 1);
    float clo[8][3], chi[8][3];
    int32_t ref[8];
    for (int s = 0; s < ns; ++s) {
        const int32_t m = slots[s].bin;
        float4 l, h;
        if (m < 0) {
            l = __ldg(leafbox + 2 * (int64_t)~m), h = __ldg(leafbox + 2 * (int64_t)~m + 1);
            ref[s] = make_leaf(~m, 1);
        } else {
            l = __ldg(nodebox + 2 * (int64_t)m), h = __ldg(nodebox + 2 * (int64_t)m + 1);
            if (slots[s].kind == 0) {
                const int2 rg = __ldg(range + m);
                ref[s] = make_leaf(rg.x, rg.y - rg.x + 1);
            } else {
                ref[s] = m;
            }
        }
        clo[s][0] = l.x, clo[s][1] = l.y, clo[s][2] = l.z;
        chi[s][0] = h.x, chi[s][1] = h.y, chi[s][2] = h.z;
    }
    // octant slots: greedily give the (child, slot) pair with the largest alignment of the child's
    // box centre offset with the slot's diagonal direction
    const float pc[3] = {0.5f * (plo.x + phi.x), 0.5f * (plo.y + phi.y), 0.5f * (plo.z + phi.z)};
    int slot_of[8];
    unsigned used = 0u, done = 0u;
    for (int round = 0; round < ns; ++round) {
        float best = -INFINITY;
        int bs = 0, bk = 0;
        for (int s = 0; s < ns; ++s) {
            if (done & (1u << s)) continue;
            const float ox = 0.5f * (clo[s][0] + chi[s][0]) - pc[0];
            const float oy = 0.5f * (clo[s][1] + chi[s][1]) - pc[1];
            const float oz = 0.5f * (clo[s][2] + chi[s][2]) - pc[2];
            for (int k = 0; k < 8; ++k) {
                if (used & (1u << k)) continue;
                const float v = ((k & 4) ? ox : -ox) + ((k & 2) ? oy : -oy) + ((k & 1) ? oz : -oz);
                if (v > best) best = v, bs = s, bk = k;
            }
        }
        slot_of[bs] = bk;
        used |= 1u << bk;
        done |= 1u << bs;
    }
    // quantisation relative to the node box (the union of the children)
    const float p[3] = {plo.x, plo.y, plo.z}, q[3] = {phi.x, phi.y, phi.z};
    uint32_t qlo[3][2] = {{0, 0}, {0, 0}, {0, 0}}, qhi[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    uint32_t meta = 0;
    for (int a = 0; a < 3; ++a) {
        const int e = step_exponent(__fsub_ru(q[a], p[a]));
        meta |= (uint32_t)(e + 127 + 15) << (8 * a);
        for (int s = 0; s < ns; ++s) {
            const float fl = floorf(ldexpf(__fsub_rd(clo[s][a], p[a]), -e));
            const float fh = ceilf(ldexpf(__fsub_ru(chi[s][a], p[a]), -e));
            const uint32_t bl = fl <= 0.f ? 0u : (fl >= 255.f ? 255u : (uint32_t)fl);
            const uint32_t bh = fh <= 0.f ? 0u : (fh >= 255.f ? 255u : (uint32_t)fh);
            const int k = slot_of[s];
            qlo[a][k >> 2] |= bl << (8 * (k & 3));
            qhi[a][k >> 2] |= bh << (8 * (k & 3));
        }
    }
    int32_t kref[8];
    for (int k = 0; k < 8; ++k) kref[k] = kEmptyRef;
    for (int s = 0; s < ns; ++s) {
        kref[slot_of[s]] = ref[s];
        meta |= 1u << (24 + slot_of[s]);
        if (ref[s] >= 0) children[nchild++] = ref[s];
    }
    Node8 nd;
    nd.c0a = make_float4(p[0], p[1], p[2], __uint_as_float(meta));
    nd.c0b = make_uint4(qlo[0][0], qlo[0][1], qhi[0][0], qhi[0][1]);
    nd.c1a = make_uint4(qlo[1][0], qlo[1][1], qhi[1][0], qhi[1][1]);
    nd.c1b = make_uint4(qlo[2][0], qlo[2][1], qhi[2][0], qhi[2][1]);
    nd.ref0 = make_int4(kref[0], kref[1], kref[2], kref[3]);
    nd.ref1 = make_int4(kref[4], kref[5], kref[6], kref[7]);
    nodes8[n] = nd;
    return ns;
}

// Top-down collapse over a device work queue of wide-node roots (binary node ids). q[] starts at -1
// with q[0] = 0 (the root); ctr = {head, tail, done, max stack need}. A thread takes the next queue
// index, waits for the entry to be published (or for all work to be finished), builds that wide
// node and appends its internal children. Work ends when every created entry is done.
// need[n] = traversal-stack entries that can be pending when wide node n is visited (the cast
// pushes every hit child of a node and pops one: need(child) = need(n) + children(n) - 1); the
// maximum of need + children over all nodes bounds the cast's stack (checked by the cast kernel).
__global__ void __launch_bounds__(128) k_collapse(const int2 *__restrict__ child, const int2 *__restrict__ range,
                                                  const float4 *__restrict__ nodebox,
                                                  const float4 *__restrict__ leafbox, const float *cost,
                                                  Node8 *nodes8, int32_t *q, unsigned int qcap, unsigned int *ctr,
                                                  int32_t *need) {
    volatile int32_t *vq = q;
    volatile unsigned int *vctr = ctr;
    while (true) {
        const unsigned int idx = atomicAdd(ctr, 1u);
        if (idx >= qcap) return;  // beyond the queue's capacity (>= the number of wide nodes)
        int32_t n;
        while (true) {
            n = vq[idx];
            if (n >= 0) break;
            // finished when every created entry is done and this index lies beyond them
            const unsigned int done = vctr[2];
            __threadfence();
            const unsigned int tail = vctr[1];
            if (done == tail && idx >= tail) return;
            __nanosleep(64);
        }
        __threadfence();
        const int32_t my_need = n == 0 ? 0 : __ldcg(need + n);
        Slot slots[8];
        const int ns = collect_slots(n, child, range, nodebox, leafbox, cost, slots);
        int32_t kids[8];
        int nk = 0;
        write_node(n, slots, ns, range, nodebox, leafbox, nodes8, kids, nk);
        atomicMax(ctr + 3, (unsigned int)(my_need + ns));
        if (nk) {
            for (int k = 0; k < nk; ++k) __stcg(need + kids[k], my_need + ns - 1);
            __threadfence();
            const unsigned int base = atomicAdd(ctr + 1, (unsigned int)nk);
            for (int k = 0; k < nk; ++k) vq[base + k] = kids[k];
        }
        __threadfence();
        atomicAdd(ctr + 2, 1u);
    }
}

__global__ void k_collapse_init(int32_t *q, unsigned int *ctr) {
    q[0] = 0;
    ctr[0] = 0u, ctr[1] = 1u, ctr[2] = 0u, ctr[3] = 0u;
}

// T == 1: a root with the single triangle in slot 0 (box = the triangle's box)
__global__ void k_single8(const float4 *__restrict__ leafbox, Node8 *nodes8) {
    const float4 lo = leafbox[0], hi = leafbox[1];
    const float p[3] = {lo.x, lo.y, lo.z}, q[3] = {hi.x, hi.y, hi.z};
    uint32_t meta = 1u << 24;
    for (int a = 0; a < 3; ++a) meta |= (uint32_t)(step_exponent(__fsub_ru(q[a], p[a])) + 127 + 15) << (8 * a);
    Node8 nd;
    nd.c0a = make_float4(lo.x, lo.y, lo.z, __uint_as_float(meta));
    nd.c0b = make_uint4(0u, 0u, 255u, 0u);
    nd.c1a = make_uint4(0u, 0u, 255u, 0u);
    nd.c1b = make_uint4(0u, 0u, 255u, 0u);
    nd.ref0 = make_int4(make_leaf(0, 1), kEmptyRef, kEmptyRef, kEmptyRef);
    nd.ref1 = make_int4(kEmptyRef, kEmptyRef, kEmptyRef, kEmptyRef);
    nodes8[0] = nd;
}

__global__ void k_need1(unsigned int *ctr) { ctr[3] = 1u; }

}  // namespace

void launch_wide8(BuildBuffers &b, cudaStream_t s) {
    const int64_t T = b.T;
    Node8 *nodes8 = reinterpret_cast<Node8 *>(b.nodes4);
    if (T == 1) {
        k_single8<<<1, 1, 0, s>>>(b.leafbox, nodes8);
        FGL_LAUNCHED("k_single8");
        k_need1<<<1, 1, 0, s>>>(b.wctr);
        FGL_LAUNCHED("k_need1");
        return;
    }
    FGL_CUDA(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * (T - 1), s));
    k_sah_dp<<<(unsigned)((T + 255) / 256), 256, 0, s>>>((int32_t)T, b.child, b.range, b.parent, b.nodebox, b.leafbox,
                                                         reinterpret_cast<unsigned int *>(b.flags), b.cost8);
    FGL_LAUNCHED("k_sah_dp");
    FGL_CUDA(cudaMemsetAsync(b.wq, 0xff, sizeof(int32_t) * T, s));
    k_collapse_init<<<1, 1, 0, s>>>(b.wq, b.wctr);
    FGL_LAUNCHED("k_collapse_init");
    int dev, sms;
    FGL_CUDA(cudaGetDevice(&dev));
    FGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (T + 127) / 128;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
    k_collapse<<<blocks, 128, 0, s>>>(b.child, b.range, b.nodebox, b.leafbox, b.cost8, nodes8, b.wq,
                                        (unsigned int)T, b.wctr, b.tsize);
    FGL_LAUNCHED("k_collapse");
}

}  // namespace fgl
