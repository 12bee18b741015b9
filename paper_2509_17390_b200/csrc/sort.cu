// Stable LSD radix sort of (u64 key, u32 value) pairs, 8-bit digits — the "radix sort run
// massively in parallel" of PAPER.md §IV-A, written for sm_100a.
//
// Per digit pass (reduce-then-scan):
//   upsweep   : each 4096-key tile counts its digits -> counts[digit][tile]
//   scan      : one CTA per digit turns its column into global output offsets
//               (base = keys with a smaller digit, from the all-pass histogram)
//   downsweep : each tile re-reads its keys, ranks them stably (warp match + per-warp counters,
//               warps in key order) and scatters key and value to their final positions.
// The all-pass digit histogram is produced once (fused into the Morton kernel for the build).
#include "fgl_internal.cuh"

namespace fgl {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                      // keys per thread
constexpr int kTile = kThreads * kItems;        // 4096 keys per tile
constexpr int kWarpSpan = kTile / kWarps;       // 512 contiguous keys per warp

__global__ void __launch_bounds__(kThreads) k_digit_hist(const uint64_t *__restrict__ keys, int64_t n, int npass,
                                                         uint32_t *__restrict__ ghist) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        uint64_t k = keys[i];
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += kThreads) {
        uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

__global__ void __launch_bounds__(kThreads) k_upsweep(const uint64_t *__restrict__ keys, int64_t n, int shift,
                                                      uint32_t *__restrict__ counts, int nblk) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int i = 0; i < kItems; ++i) {
        int64_t idx = base + i * kThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

// one CTA per digit: exclusive scan of counts[d][0..nblk) plus the digit's global base
__global__ void __launch_bounds__(1024) k_scan(uint32_t *__restrict__ counts, int nblk,
                                               const uint32_t *__restrict__ hist) {
    __shared__ uint32_t warp_sum[32];
    __shared__ uint32_t s_base;
    const int d = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w == 0) {
        uint32_t s = 0;
        for (int i = lane; i < d; i += 32) s += hist[i];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) s_base = s;
    }
    __syncthreads();
    uint32_t carry = s_base;
    uint32_t *col = counts + (int64_t)d * nblk;
    for (int start = 0; start < nblk; start += 1024) {
        int i = start + threadIdx.x;
        uint32_t v = i < nblk ? col[i] : 0u;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sum[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t s = warp_sum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sum[lane] = s;
        }
        __syncthreads();
        uint32_t excl = carry + (w ? warp_sum[w - 1] : 0u) + x - v;
        if (i < nblk) col[i] = excl;
        carry += warp_sum[31];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_downsweep(const uint64_t *__restrict__ kin,
                                                        const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
                                                        uint32_t *__restrict__ vout, int64_t n, int shift,
                                                        const uint32_t *__restrict__ offsets, int nblk) {
    __shared__ uint32_t wh[kWarps][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&wh[0][0])[i] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * kWarpSpan;
    uint64_t key[kItems];
    uint32_t val[kItems];
    uint32_t rank[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t idx = base + i * 32 + lane;
        bool ok = idx < n;
        key[i] = ok ? kin[idx] : 0ull;
        val[i] = ok ? vin[idx] : 0u;
        uint32_t d = ok ? (uint32_t)((key[i] >> shift) & 0xFF) : 256u + lane;  // invalid lanes match nobody
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = ok ? wh[w][d] : 0u;
        __syncwarp();
        if (ok && (peers & lt) == 0) wh[w][d] = before + __popc(peers);
        __syncwarp();
        rank[i] = before + __popc(peers & lt);
    }
    __syncthreads();
    // exclusive prefix over warps (warps own consecutive key ranges), digit per thread
    {
        const int d = threadIdx.x;
        uint32_t s = offsets[(int64_t)d * nblk + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
            uint32_t c = wh[ww][d];
            wh[ww][d] = s;
            s += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t idx = base + i * 32 + lane;
        if (idx < n) {
            uint32_t d = (uint32_t)((key[i] >> shift) & 0xFF);
            uint32_t pos = wh[w][d] + rank[i];
            kout[pos] = key[i];
            vout[pos] = val[i];
        }
    }
}
}  // namespace

int sort_tile_blocks(int64_t n) { return (int)((n + kTile - 1) / kTile); }

void digit_histograms(const uint64_t *keys, int64_t n, int key_bits, uint32_t *ghist, cudaStream_t s) {
    int npass = (key_bits + 7) / 8;
    FGL_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * 256, s));
    if (n <= 0) return;
    int blocks = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 4);
    k_digit_hist<<<blocks, kThreads, 0, s>>>(keys, n, npass, ghist);
    FGL_LAUNCHED("k_digit_hist");
}

void radix_sort_pairs(uint64_t *keys0, uint32_t *vals0, uint64_t *keys1, uint32_t *vals1, int64_t n, int key_bits,
                      uint32_t *counts, uint32_t *ghist, bool ghist_ready, int *result_slot, cudaStream_t s) {
    *result_slot = 0;
    if (n <= 1) return;
    if (n > (int64_t)UINT32_MAX) throw Error(1, "radix sort: n too large");
    if (!ghist_ready) digit_histograms(keys0, n, key_bits, ghist, s);
    const int npass = (key_bits + 7) / 8;
    const int nblk = sort_tile_blocks(n);
    uint64_t *k[2] = {keys0, keys1};
    uint32_t *v[2] = {vals0, vals1};
    int cur = 0;
    for (int p = 0; p < npass; ++p) {
        const int shift = 8 * p;
        k_upsweep<<<nblk, kThreads, 0, s>>>(k[cur], n, shift, counts, nblk);
        FGL_LAUNCHED("k_upsweep");
        k_scan<<<256, 1024, 0, s>>>(counts, nblk, ghist + 256 * p);
        FGL_LAUNCHED("k_scan");
        k_downsweep<<<nblk, kThreads, 0, s>>>(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], n, shift, counts, nblk);
        FGL_LAUNCHED("k_downsweep");
        cur ^= 1;
    }
    *result_slot = cur;
}

}  // namespace fgl
