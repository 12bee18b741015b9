// Point-cloud metrics of §V-A (symmetric Chamfer distance, precision, recall, F-score) on
// sm_100a — SURVEY §8(f) NEXT-1. The reference cloud is indexed by the same LBVH as the cast
// (a "point scene": one degenerate triangle (i, i, i) per point, so the Morton / sort / Karras /
// Eq. 7 build is reused unchanged and every leaf box is the exact point); queries find their exact
// nearest neighbour by a best-first descent pruned by the squared box distance.
#include <cfloat>
#include <climits>

#include "fgl_internal.cuh"

namespace fgl {

namespace {

__global__ void k_iota3(int32_t *__restrict__ tris, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        tris[3 * i] = tris[3 * i + 1] = tris[3 * i + 2] = (int32_t)i;
}

// squared distance from q to a box (0 inside)
__device__ __forceinline__ float box_d2(float qx, float qy, float qz, float lx, float hx, float ly, float hy, float lz,
                                        float hz) {
    const float dx = fmaxf(fmaxf(lx - qx, qx - hx), 0.f);
    const float dy = fmaxf(fmaxf(ly - qy, qy - hy), 0.f);
    const float dz = fmaxf(fmaxf(lz - qz, qz - hz), 0.f);
    return dx * dx + dy * dy + dz * dz;
}

constexpr int kStack = 96;
constexpr float kSlack = 1.0f + 0x1p-18f;  // box pruning tolerates the rounding of box_d2 / best

__global__ void __launch_bounds__(128) k_nearest(const Node64 *__restrict__ nodes, const float4 *__restrict__ pts,
                                                 const float *__restrict__ q, int64_t m, float *__restrict__ dist,
                                                 int32_t *__restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const float qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
    if (!(isfinite(qx) && isfinite(qy) && isfinite(qz))) {  // e.g. the hit point of a missed beam
        dist[i] = NAN;
        idx[i] = -1;
        return;
    }
    float best = INFINITY;
    int32_t bid = INT_MAX;
    uint64_t st[kStack];
    int sp = 0;
    int32_t cur = 0;
    while (true) {
        if (cur >= 0) {
            const float4 *np = reinterpret_cast<const float4 *>(nodes + cur);
            const float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
            const int4 d = __ldg(reinterpret_cast<const int4 *>(np + 3));
            const float d0 = box_d2(qx, qy, qz, a.x, a.y, a.z, a.w, c.x, c.y);
            const float d1 = box_d2(qx, qy, qz, b.x, b.y, b.z, b.w, c.z, c.w);
            const bool h0 = d0 <= best * kSlack, h1 = d1 <= best * kSlack;
            if (h0 && h1) {
                const bool sw = d1 < d0;
                st[sp++] = ((uint64_t)__float_as_uint(sw ? d0 : d1) << 32) | (uint32_t)(sw ? d.x : d.y);
                cur = sw ? d.y : d.x;
                continue;
            }
            if (h0) {
                cur = d.x;
                continue;
            }
            if (h1) {
                cur = d.y;
                continue;
            }
        } else {
            const int32_t v = ~cur;
            const int32_t first = v >> kLeafShift, cnt = (v & (kMaxLeaf - 1)) + 1;
            for (int32_t k = first; k < first + cnt; ++k) {
                const float4 p = __ldg(pts + kTriStride * (int64_t)k);  // tri48 record: v0 = the point, w = its index
                const float dx = p.x - qx, dy = p.y - qy, dz = p.z - qz;
                const float d2 = dx * dx + dy * dy + dz * dz;
                const int32_t id = __float_as_int(p.w);
                if (d2 < best || (d2 == best && id < bid)) best = d2, bid = id;
            }
        }
        cur = INT_MAX;
        while (sp > 0) {
            --sp;
            if (__uint_as_float((uint32_t)(st[sp] >> 32)) <= best * kSlack) {
                cur = (int32_t)(uint32_t)st[sp];
                break;
            }
        }
        if (cur == INT_MAX) break;
    }
    dist[i] = sqrtf(best);
    idx[i] = bid == INT_MAX ? -1 : bid;
}

// sums (double) of the finite distances and of those <= tau, for both directions; the last block
// forms Chamfer, precision, recall and F-score (R23)
__global__ void __launch_bounds__(256) k_metrics(const float *__restrict__ dab, int64_t na,
                                                 const float *__restrict__ dba, int64_t nb, float tau,
                                                 double *__restrict__ acc, unsigned int *sync,
                                                 double *__restrict__ out) {
    double s[6] = {0, 0, 0, 0, 0, 0};  // sum_ab, n_ab, in_ab, sum_ba, n_ba, in_ba
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb; i += (int64_t)gridDim.x * blockDim.x) {
        const bool first = i < na;
        const float d = first ? dab[i] : dba[i - na];
        if (isfinite(d)) {
            const int o = first ? 0 : 3;
            s[o] += d, s[o + 1] += 1.0, s[o + 2] += d <= tau ? 1.0 : 0.0;
        }
    }
    for (int k = 0; k < 6; ++k) {
        double v = s[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&acc[k], v);
    }
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(sync, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    double a[6];
    for (int k = 0; k < 6; ++k) a[k] = __ldcg(&acc[k]), acc[k] = 0.0;
    *sync = 0u;
    const double mab = a[1] > 0 ? a[0] / a[1] : NAN, mba = a[4] > 0 ? a[3] / a[4] : NAN;
    const double prec = a[1] > 0 ? a[2] / a[1] : NAN, rec = a[4] > 0 ? a[5] / a[4] : NAN;
    out[0] = 0.5 * (mab + mba);
    out[1] = prec;
    out[2] = rec;
    out[3] = prec + rec > 0 ? 2.0 * prec * rec / (prec + rec) : 0.0;
    out[4] = a[1];
    out[5] = a[4];
}

}  // namespace

void launch_iota3(int32_t *tris, int64_t n, cudaStream_t s) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_iota3<<<blocks, 256, 0, s>>>(tris, n);
    FGL_LAUNCHED("k_iota3");
}

void launch_nearest(const SceneView &sv, const float *q, int64_t m, float *dist, int32_t *idx, cudaStream_t s) {
    if (m <= 0) return;
    k_nearest<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(sv.nodes, sv.tri, q, m, dist, idx);
    FGL_LAUNCHED("k_nearest");
}

void launch_metrics(const float *dab, int64_t na, const float *dba, int64_t nb, float tau, double *acc,
                    unsigned int *sync, double *out, cudaStream_t s) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((na + nb + 255) / 256, 148 * 4));
    k_metrics<<<blocks, 256, 0, s>>>(dab, na, dba, nb, tau, acc, sync, out);
    FGL_LAUNCHED("k_metrics");
}

}  // namespace fgl
