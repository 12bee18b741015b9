// Stable LSD radix sort of (u64 key, u32 value) pairs, 8-bit digits — the "radix sort run
// massively in parallel" of PAPER.md §IV-A, written for sm_100a.
//
// One kernel per digit pass, single-pass "onesweep" style (decoupled look-back; Merrill & Garland
// 2016, Adinets & Merrill 2022): a CTA takes the next 4096-key tile from an atomic tile counter,
// ranks its keys stably (warp match + per-warp digit counters, warps in key order), publishes its
// per-digit counts, looks back over earlier tiles' published prefixes to find its global offsets
// (base = keys with a smaller digit, from the all-pass histogram computed once up front — fused
// into the Morton kernel for the build) and scatters keys and values: one read and one write of
// each key per pass. Status words carry a per-pass epoch so they never need clearing; the epoch
// counter lives in device memory and is advanced by k_sort_begin on the stream, so a sort captured
// in a CUDA graph gets fresh epochs on every replay (a host-side epoch would be baked into the
// graph and let a replay accept the previous replay's status words).
#include <cstdlib>

#include <cuda/atomic>

#include "fgl_internal.cuh"

namespace fgl {

namespace {
#ifndef FGL_SORT_THREADS
#define FGL_SORT_THREADS 256
#endif
constexpr int kThreads = FGL_SORT_THREADS;      // >= 256: one look-back thread per digit
constexpr int kWarps = kThreads / 32;
#ifndef FGL_SORT_ITEMS_KV
#define FGL_SORT_ITEMS_KV 8
#endif
#ifndef FGL_SORT_ITEMS_K
#define FGL_SORT_ITEMS_K 12
#endif
#ifndef FGL_SORT_RTS_MIN
#define FGL_SORT_RTS_MIN (1 << 30)  // keys from which a pass runs reduce-then-scan instead of onesweep (measured
                                     // no faster at 10 M keys: 110 vs 99 us per pass; off)
#endif
#ifndef FGL_SORT_MINB
#define FGL_SORT_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
#ifndef FGL_SORT_WIN
#define FGL_SORT_WIN 8  // look-back window: predecessor tiles read per round
#endif
#ifndef FGL_SORT_BACKOFF
#define FGL_SORT_BACKOFF 0
#endif
constexpr int kItemsKV = FGL_SORT_ITEMS_KV;     // keys per thread, key-value passes (34 KB shared)
constexpr int kItemsK = FGL_SORT_ITEMS_K;       // keys per thread, key-only passes (33 KB shared)
constexpr int kMinTile = kThreads * (kItemsKV < kItemsK ? kItemsKV : kItemsK);  // sizes the status array
constexpr uint64_t kAgg = 1ull << 30, kPrefix = 2ull << 30, kValMask = (1ull << 30) - 1;

__global__ void __launch_bounds__(kThreads) k_digit_hist(const uint64_t *__restrict__ keys, int64_t n, int npass,
                                                         int shift0, uint32_t *__restrict__ ghist) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        uint64_t k = keys[i] >> shift0;
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += kThreads) {
        uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

// One digit pass over one tile of kThreads * kIt keys (values optional: kVals = false sorts keys
// that carry their payload in the low bits). Ranking is per warp (match_any + per-warp digit
// counters, warps in key order); the ranked tile is staged in shared memory in digit order so the
// global scatter writes runs of equal digits from consecutive threads (coalesced), after the
// decoupled look-back has produced each digit's global offset.
// kRts (reduce-then-scan, large inputs): the tile's global digit offsets come precomputed in
// offs[digit][tile] (k_tile_hist + k_offs_scan) instead of from the look-back; tile = blockIdx.x.
template <int kIt, bool kVals, bool kRts = false>
__global__ void __launch_bounds__(kThreads, FGL_SORT_MINB) k_onesweep(const uint64_t *__restrict__ kin,
                                                          const uint32_t *__restrict__ vin,
                                                          uint64_t *__restrict__ kout, uint32_t *__restrict__ vout,
                                                          int64_t n, int shift, const uint32_t *__restrict__ hist,
                                                          uint64_t *status, uint32_t *tile_ctr,
                                                          const uint32_t *epoch_end, int pass, int npass,
                                                          const uint32_t *__restrict__ offs = nullptr) {
    static_assert(kThreads == 256, "one thread per digit");
    constexpr int kT = kThreads * kIt, kSpan = kT / kWarps;
    __shared__ uint32_t wh[kWarps][256];
    __shared__ uint32_t s_base[256];   // global start of each digit in this pass's output
    __shared__ uint32_t s_tstart[256];  // start of each digit in the tile's staged (sorted) order
    __shared__ uint32_t s_wsum[kWarps];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_key[kT];
    __shared__ uint32_t s_val[kVals ? kT : 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, d = threadIdx.x;
    // this sort's epochs are (end - npass, end]: written by k_sort_begin earlier on the stream
    const uint32_t epoch = kRts ? 0u : *epoch_end - (uint32_t)npass + 1u + (uint32_t)pass;
    if (threadIdx.x == 0) s_tile = kRts ? blockIdx.x : atomicAdd(tile_ctr, 1u);
    for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&wh[0][0])[i] = 0;
    // block-wide exclusive scan over the 256 digits (one value per thread)
    auto scan256 = [&](uint32_t v) -> uint32_t {
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[w] = x;
        __syncthreads();
        uint32_t off = 0;
        for (int ww = 0; ww < w; ++ww) off += s_wsum[ww];
        __syncthreads();  // s_wsum may be reused by the next scan
        return off + x - v;
    };
    if constexpr (!kRts) s_base[d] = scan256(hist[d]);  // digit bases from the all-pass histogram
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)tile * kT + (int64_t)w * kSpan;
    uint64_t key[kIt];
    uint32_t val[kVals ? kIt : 1];
    uint32_t rank[kIt];
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
        const int64_t idx = base + i * 32 + lane;
        const bool ok = idx < n;
        key[i] = ok ? kin[idx] : 0ull;
        if constexpr (kVals) val[i] = ok ? vin[idx] : 0u;
        const uint32_t dg = ok ? (uint32_t)((key[i] >> shift) & 0xFF) : 256u + lane;  // invalid lanes match nobody
        const uint32_t peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t before = ok ? wh[w][dg] : 0u;
        __syncwarp();
        if (ok && (peers & lt) == 0) wh[w][dg] = before + __popc(peers);
        __syncwarp();
        rank[i] = before + __popc(peers & lt);
    }
    __syncthreads();
    // per digit: tile count (published at once), exclusive prefix over warps, tile start
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
        const uint32_t c = wh[ww][d];
        wh[ww][d] = cnt;
        cnt += c;
    }
    const uint32_t tstart = [&]() {
        if constexpr (kRts) {
            return scan256(cnt);
        } else {
            const uint64_t ep = (uint64_t)epoch << 32;
            // status words carry their own payload, so relaxed (L2-coherent) accesses suffice
            cuda::atomic_ref<uint64_t, cuda::thread_scope_device> mine(status[(int64_t)tile * 256 + d]);
            mine.store(ep | (tile == 0 ? kPrefix : kAgg) | cnt, cuda::std::memory_order_relaxed);
            return scan256(cnt);
        }
    }();
    s_tstart[d] = tstart;
    if constexpr (kRts) {
        s_base[d] = offs[(int64_t)d * gridDim.x + tile] - tstart;  // global start of digit d in this tile
    } else {
    // decoupled look-back: kWin predecessors per round (independent loads in flight), accumulating
    // published tile counts until the nearest published inclusive prefix
    uint32_t excl = 0;
    if (tile != 0) {
        constexpr int kWin = FGL_SORT_WIN;
        int64_t t = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint64_t v[kWin];
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                v[k] = 0;
                if (t - k >= 0) {
                    cuda::atomic_ref<uint64_t, cuda::thread_scope_device> prev(status[(t - k) * 256 + d]);
                    v[k] = prev.load(cuda::std::memory_order_relaxed);
                }
            }
            const int64_t t0 = t;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                if (done || t < 0) break;
                if ((v[k] >> 32) != epoch || (v[k] & (kAgg | kPrefix)) == 0) break;  // not yet: re-poll from t
                excl += (uint32_t)(v[k] & kValMask);
                if (v[k] & kPrefix) done = true;
                --t;
            }
            if (t < 0) done = true;
#if FGL_SORT_BACKOFF
            if (!done && t == t0) __nanosleep(FGL_SORT_BACKOFF);  // predecessor not yet published: yield issue slots
#endif
        }
        cuda::atomic_ref<uint64_t, cuda::thread_scope_device> mine(status[(int64_t)tile * 256 + d]);
        mine.store(((uint64_t)epoch << 32) | kPrefix | (excl + cnt), cuda::std::memory_order_relaxed);
    }
    s_base[d] += excl - tstart;  // global position = s_base[digit] + staged position
    }
    __syncthreads();
    // stage the tile in digit order
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
        if (base + i * 32 + lane < n) {
            const uint32_t dg = (uint32_t)((key[i] >> shift) & 0xFF);
            const uint32_t lp = s_tstart[dg] + wh[w][dg] + rank[i];
            s_key[lp] = key[i];
            if constexpr (kVals) s_val[lp] = val[i];
        }
    }
    __syncthreads();
    // coalesced scatter: consecutive threads write consecutive keys of a digit run
    const int64_t rem = n - (int64_t)tile * kT;
    const int valid = rem < kT ? (int)rem : kT;
    for (int p = threadIdx.x; p < valid; p += kThreads) {
        const uint64_t kk = s_key[p];
        const uint32_t pos = s_base[(kk >> shift) & 0xFF] + p;
        kout[pos] = kk;
        if constexpr (kVals) vout[pos] = s_val[p];
    }
}
// Reduce-then-scan pass, step 1: the digit histogram of every tile (same tile layout as k_onesweep),
// stored digit-major: thist[digit][tile].
template <int kIt>
__global__ void __launch_bounds__(kThreads) k_tile_hist(const uint64_t *__restrict__ kin, int64_t n, int shift,
                                                       uint32_t *__restrict__ thist) {
    constexpr int kT = kThreads * kIt;
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kT;
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
        const int64_t idx = base + i * kThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(kin[idx] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    thist[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// Reduce-then-scan pass, step 2: one CTA per digit d turns its row of tile counts into the tiles'
// global start positions, in place: offs[d][t] = (keys with a smaller digit) + (keys with digit d in
// tiles before t). The digit base comes from the all-pass histogram.
__global__ void __launch_bounds__(kThreads) k_offs_scan(uint32_t *__restrict__ thist, int ntiles,
                                                       const uint32_t *__restrict__ hist) {
    __shared__ uint32_t s_w[kWarps];
    __shared__ uint32_t s_carry;
    const int d = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // digit base: sum of hist[0..d)
    uint32_t b = threadIdx.x < (unsigned)d ? hist[threadIdx.x] : 0u;
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (lane == 0) s_w[w] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < kWarps; ++k) t += s_w[k];
        s_carry = t;
    }
    __syncthreads();
    uint32_t *row = thist + (int64_t)d * ntiles;
    for (int c0 = 0; c0 < ntiles; c0 += kThreads) {
        const int t = c0 + threadIdx.x;
        const uint32_t v = t < ntiles ? row[t] : 0u;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        uint32_t off = s_carry;
        for (int k = 0; k < w; ++k) off += s_w[k];
        if (t < ntiles) row[t] = off + x - v;
        __syncthreads();
        if (threadIdx.x == kThreads - 1) s_carry = off + x;
        __syncthreads();
    }
}

// Per-sort setup on the stream: zero the per-pass tile counters and reserve npass fresh epochs
// (ctl[8] = the last epoch of this sort; epoch 0 marks never-written status words and is skipped
// at wrap-around).
__global__ void k_sort_begin(uint32_t *ctl, int npass) {
    if (threadIdx.x < 8) ctl[threadIdx.x] = 0u;
    if (threadIdx.x == 8) {
        const uint32_t e = ctl[8];
        uint32_t ne = e + (uint32_t)npass;
        if (ne < e) ne = (uint32_t)npass;  // wrapped past 0: restart at 1..npass
        ctl[8] = ne;
    }
}
}  // namespace

int sort_tile_blocks(int64_t n) { return (int)((n + kMinTile - 1) / kMinTile); }

void digit_histograms(const uint64_t *keys, int64_t n, int key_bits, uint32_t *ghist, cudaStream_t s, int shift0) {
    int npass = (key_bits + 7) / 8;
    FGL_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * 8 * 256, s));
    if (n <= 0) return;
    int blocks = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 4);
    k_digit_hist<<<blocks, kThreads, 0, s>>>(keys, n, npass, shift0, ghist);
    FGL_LAUNCHED("k_digit_hist");
}

void radix_sort_pairs(uint64_t *keys0, uint32_t *vals0, uint64_t *keys1, uint32_t *vals1, int64_t n, int key_bits,
                      uint64_t *status, uint32_t *tile_ctr, uint32_t *ghist, bool ghist_ready,
                      int *result_slot, cudaStream_t s, int shift0, uint32_t *rts) {
    *result_slot = 0;
    if (n <= 1) return;
    if (n >= (int64_t)kValMask) throw Error(1, "radix sort: n must be < 2^30");
    if (!ghist_ready) digit_histograms(keys0, n, key_bits, ghist, s, shift0);
    const int npass = (key_bits + 7) / 8;
    const bool kv = vals0 != nullptr;
    const int64_t tile = (int64_t)kThreads * (kv ? kItemsKV : kItemsK);
    const unsigned nblk = (unsigned)((n + tile - 1) / tile);
    k_sort_begin<<<1, 32, 0, s>>>(tile_ctr, npass);
    FGL_LAUNCHED("k_sort_begin");
    uint64_t *k[2] = {keys0, keys1};
    uint32_t *v[2] = {vals0, vals1};
    int cur = 0;
    // large inputs: reduce-then-scan passes (no look-back chain across thousands of tiles)
    // FGL_SORT_RTS_MIN (environment) overrides the compiled threshold: A/B runs and the test of the path
    int64_t rts_min = (int64_t)FGL_SORT_RTS_MIN;
    if (const char *e = getenv("FGL_SORT_RTS_MIN")) rts_min = atoll(e);
    const bool use_rts = rts != nullptr && n >= rts_min;
    for (int p = 0; p < npass; ++p) {
        if (use_rts) {
            const int sh = shift0 + 8 * p;
            if (kv) {
                k_tile_hist<kItemsKV><<<nblk, kThreads, 0, s>>>(k[cur], n, sh, rts);
                FGL_LAUNCHED("k_tile_hist");
                k_offs_scan<<<256, kThreads, 0, s>>>(rts, (int)nblk, ghist + 256 * p);
                FGL_LAUNCHED("k_offs_scan");
                k_onesweep<kItemsKV, true, true><<<nblk, kThreads, 0, s>>>(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], n,
                                                                           sh, ghist + 256 * p, status, tile_ctr + p,
                                                                           tile_ctr + 8, p, npass, rts);
            } else {
                k_tile_hist<kItemsK><<<nblk, kThreads, 0, s>>>(k[cur], n, sh, rts);
                FGL_LAUNCHED("k_tile_hist");
                k_offs_scan<<<256, kThreads, 0, s>>>(rts, (int)nblk, ghist + 256 * p);
                FGL_LAUNCHED("k_offs_scan");
                k_onesweep<kItemsK, false, true><<<nblk, kThreads, 0, s>>>(k[cur], nullptr, k[cur ^ 1], nullptr, n,
                                                                           sh, ghist + 256 * p, status, tile_ctr + p,
                                                                           tile_ctr + 8, p, npass, rts);
            }
            FGL_LAUNCHED("k_onesweep");
            cur ^= 1;
            continue;
        }
        if (kv)
            k_onesweep<kItemsKV, true><<<nblk, kThreads, 0, s>>>(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], n,
                                                                 shift0 + 8 * p, ghist + 256 * p, status,
                                                                 tile_ctr + p, tile_ctr + 8, p, npass);
        else
            k_onesweep<kItemsK, false><<<nblk, kThreads, 0, s>>>(k[cur], nullptr, k[cur ^ 1], nullptr, n,
                                                                 shift0 + 8 * p, ghist + 256 * p, status,
                                                                 tile_ctr + p, tile_ctr + 8, p, npass);
        FGL_LAUNCHED("k_onesweep");
        cur ^= 1;
    }
    *result_slot = cur;
}

}  // namespace fgl
