// Internal declarations shared by the libfgl translation units (never by the oracle).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace fgl {

// ---- errors -----------------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define FGL_CUDA(call)                                                                                  \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) {                                                                        \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? 3 : 4;                                      \
            throw ::fgl::Error(code_, std::string(#call) + ": " + cudaGetErrorString(e_));             \
        }                                                                                               \
    } while (0)

void note_launch();  // process-wide count of libfgl kernel launches (fgl_kernel_launches)

// NVTX range over a scope (host-side enqueue of a build stage or a cast; header-only NVTX v3, a no-op
// unless a profiler injects itself) so an nsys / ncu timeline attributes device work to the call
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define FGL_LAUNCHED(what)                                                                              \
    do {                                                                                                \
        ::fgl::note_launch();                                                                           \
        cudaError_t e_ = cudaGetLastError();                                                            \
        if (e_ != cudaSuccess) throw ::fgl::Error(4, std::string(what) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---- traversal node: binary LBVH node holding both children's boxes ("node64", 4 x 16 B) -------
// a = (c0.lo.x, c0.hi.x, c0.lo.y, c0.hi.y)   b = (c1.lo.x, c1.hi.x, c1.lo.y, c1.hi.y)
// c = (c0.lo.z, c0.hi.z, c1.lo.z, c1.hi.z)   d = (ref0, ref1, 0, 0)
// ref >= 0: internal node index; ref < 0 and != kEmptyRef: leaf, ~ref = first << 3 | (count - 1)
struct __align__(16) Node64 {
    float4 a, b, c;
    int4 d;
};
// 4-wide traversal node ("node128"), children in SoA: f[0]=lo.x[4] f[1]=hi.x[4] f[2]=lo.y[4]
// f[3]=hi.y[4] f[4]=lo.z[4] f[5]=hi.z[4], refs[4], meta = (valid children, depth, 0, 0).
// Stored at the index of the binary node it collapses (even-depth internal nodes).
struct __align__(16) Node128 {
    float4 f[6];
    int4 ref;
    int4 meta;
};
// 4-wide node with 8-bit child boxes ("node64q"): f0 = (origin p = union lo .xyz,
// bits: e_x | e_y << 8 | e_z << 16 | valid-child mask << 24), q0 = (lo.x bytes, hi.x bytes, lo.y,
// hi.y) (child k in byte k), q1 = (lo.z, hi.z, ref0, ref1), q2 = (ref2, ref3, 0, 0). Child planes
// p + q 2^(e-127), quantised outward (floor of the round-down offset / ceil of the round-up one).
struct __align__(16) NodeQ {
    float4 f0;
    int4 q0, q1, q2;
};
// 8-wide compressed node ("node96q", wide.cu): c0a = (px, py, pz, meta = Ex | Ey << 8 | Ez << 16 |
// valid << 24), c0b = (qlo_x[0..3], qlo_x[4..7], qhi_x[0..3], qhi_x[4..7]) bytes, c1a / c1b the same
// for y / z, ref0 / ref1 = child refs of slots 0-3 / 4-7. Child plane = p + q 2^(E - 142).
struct __align__(32) Node8 {
    float4 c0a;
    uint4 c0b, c1a, c1b;
    int4 ref0, ref1;
};
// triangle records in leaf order: kTriStride float4 per triangle ({v0, id}, {v1, 0}, {v2, 0}[, pad]);
// 4 makes each record 64-byte aligned so a leaf test fetches it with one 256-bit + one 128-bit load
#ifndef FGL_TRI_STRIDE
#define FGL_TRI_STRIDE 3
#endif
constexpr int kTriStride = FGL_TRI_STRIDE;
constexpr float kFarBox = 3.0e38f;  // empty child: a degenerate box no ray with t <= t_max reaches
constexpr int32_t kEmptyRef = INT32_MIN;
constexpr int kLeafShift = 3;
constexpr int kMaxLeaf = 8;
constexpr int64_t kMaxTris = (int64_t(1) << 28) - 1;

__host__ __device__ inline int32_t make_leaf(int32_t first, int32_t count) {
    return ~((first << kLeafShift) | (count - 1));
}

// ---- per-call work counters for persistent casts (self-resetting, 64 slots per scene) ----------
struct CastCounter {
    unsigned long long next;
    unsigned int done;
    unsigned int pad;
};
constexpr int kCounterSlots = 64;

// ---- scene build buffers (device) ---------------------------------------------------------------
struct BuildBuffers {
    int64_t T = 0;
    float4 *cent = nullptr;        // [T] centroid (x, y, z, 0)
    float *box = nullptr;          // [6] scene box lo, hi
    float *partial = nullptr;      // [kPrepBlocks][6]
    unsigned int *sync = nullptr;  // [4] last-block counters
    uint64_t *keys[2] = {nullptr, nullptr};
    uint32_t *vals[2] = {nullptr, nullptr};
    uint32_t *ghist = nullptr;     // [8][256] digit histograms
    uint64_t *sort_status = nullptr;  // [nblk][256] look-back status words (epoch | flag | count)
    uint32_t *sort_tiles = nullptr;   // [16]: [0..7] per-pass tile counters, [8] device epoch counter
    uint32_t *sort_rts = nullptr;     // [256][tiles] tile digit counts / offsets (reduce-then-scan passes)
    float4 *tri = nullptr;         // [3T] tri48 in leaf order
    int2 *child = nullptr;         // [T-1]
    int2 *range = nullptr;         // [T-1]
    int32_t *parent = nullptr;     // [2T-1]
    int32_t *flags = nullptr;      // [T-1]
    float4 *leafbox = nullptr;     // [2T]
    float4 *nodebox = nullptr;     // [2(T-1)]
    float4 *agg = nullptr;         // 8-ary box aggregates, level after level (unions of 8^k leaves)
    Node64 *nodes = nullptr;       // [max(T-1,1)]
    Node128 *nodes4 = nullptr;     // [max(T-1,1)] node128, or node64q (stride 64 B) when quantized
    int quantized = 0;
    int32_t *depth = nullptr;      // [T-1]
    int width = 4;
    int sorted_slot = 0;           // which keys/vals buffer holds the sorted result
    int packed_shift = 0;          // > 0: keys hold (code << packed_shift) | triangle index, no vals
    float *cost = nullptr;         // [T-1] SAH cost of each internal node's subtree (restructuring)
    int32_t *tsize = nullptr;      // [T-1] leaves under each internal node (restructuring)
    int restructured = 0;          // 1: treelet-restructured tree (1-triangle leaves, free topology)
    float *cost8 = nullptr;        // [T-1][8] SAH collapse costs C(n, 1..8) (width 8)
    int32_t *wq = nullptr;         // [T] top-down collapse work queue (width 8)
    unsigned int *wctr = nullptr;  // [4] queue head, tail, done, max stack need (width 8)
    unsigned long long *gslot = nullptr;  // [T-1] k_lbvh global meeting slots (epoch << 32 | endpoint), zeroed once
    void *lbvh_up = nullptr;       // k_lbvh levels above the chunks: units, counts, arrival counters (zeroed once)
};

constexpr int kPrepBlocks = 888;  // 6 x 148 SMs (latency-bound gather: more loads in flight)

// ---- launchers ------------------------------------------------------------------------------------
// sort.cu
int sort_tile_blocks(int64_t n);
void radix_sort_pairs(uint64_t *keys0, uint32_t *vals0, uint64_t *keys1, uint32_t *vals1, int64_t n, int key_bits,
                      uint64_t *status, uint32_t *tile_ctr /*[16], zeroed once at allocation*/, uint32_t *ghist,
                      bool ghist_ready, int *result_slot, cudaStream_t s,
                      int shift0 = 0,  // vals0 == nullptr: key-only passes over bits [shift0, shift0 + key_bits)
                      uint32_t *rts = nullptr);  // [256][sort_tile_blocks(n)]: enables reduce-then-scan passes
void digit_histograms(const uint64_t *keys, int64_t n, int key_bits, uint32_t *ghist, cudaStream_t s,
                      int shift0 = 0);

// build.cu
void launch_build(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, int bits, int leaf_size,
                  int cubic, int width, int quantized, cudaStream_t s, int restructure = 0, int treelets = 0);
void launch_validate(const float *verts, int64_t V, const int32_t *tris, int64_t T, unsigned int *flag,
                     cudaStream_t s);
void launch_morton_sort(BuildBuffers &b, int bits, int cubic, cudaStream_t s);
void launch_tree(BuildBuffers &b, int leaf_size, int width, int quantized, cudaStream_t s, int restructure = 0);
void launch_refit(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, int leaf_size, cudaStream_t s);
// leaf boxes + Eq. 7 node boxes of the current tree, recomputed exactly (the fused build stores only
// those a sibling needs; the scene export calls this)
size_t lbvh_up_bytes(int64_t T);  // bytes of BuildBuffers::lbvh_up
void launch_complete_boxes(const float *verts, int64_t V, const int32_t *tris, BuildBuffers &b, cudaStream_t s);
void launch_wide8(BuildBuffers &b, cudaStream_t s);  // wide.cu: SAH collapse to node96q
void launch_morton_points(const float *pts, int64_t n, const float *lo, const float *hi, int bits,
                          uint64_t *codes, cudaStream_t s);

// cast.cu
struct SpinParams {
    int32_t channels, columns;
    float az0_deg, t_min, t_max;
    float elev_deg[512];
};
struct RosetteParams {
    int32_t n;
    uint32_t inc1, inc2, phase2_0;
    float half_fov_deg, t_min, t_max;
    int64_t first_frame;
};
constexpr int kMaxPeers = 8;
struct CastOut {
    float *range;
    int32_t *tri_id;
    float *hit_xyz;
    int32_t *node_counts, *tri_counts;
    // fused cast + all-gather (A12): when npeer > 0, each result is also written at
    // out_offset + idx into every peer buffer (this process's and peers' over NVLink)
    int npeer;
    int64_t out_offset;
    float *peer_range[kMaxPeers];
    int32_t *peer_tri[kMaxPeers];
    // completion signal: the last warp adds 1 to each of these flags (every rank's, own included)
    int nsignal;
    int32_t *signal[kMaxPeers];
};
struct SceneView {
    const float4 *tri;
    const Node64 *nodes;
    const Node128 *nodes4;  // node128 / node64q (width 4) or node96q (width 8, reinterpreted)
    int width;
    int quantized;
    const unsigned int *wneed;  // width 8: the tree's traversal-stack bound (BuildBuffers::wctr[3])
    unsigned int *err;          // sticky scene error flags (bit 2: width-8 stack bound exceeded)
    const float4 *root_box;     // [2] lo, hi of the whole scene (the root's Eq. 7 box)
};
void launch_cast_spinning(const SceneView &sv, const SpinParams &p, const float *poses, int64_t P, const CastOut &o,
                          CastCounter *ctr, cudaStream_t s);
void launch_cast_rosette(const SceneView &sv, const RosetteParams &p, const float *poses, int64_t P,
                         const CastOut &o, CastCounter *ctr, cudaStream_t s);
void launch_cast_rays(const SceneView &sv, const float *orig, const float *dir, int64_t R, float t_min, float t_max,
                      const CastOut &o, CastCounter *ctr, cudaStream_t s);
void launch_cast_bruteforce(const float *verts, int64_t V, const int32_t *tris, int64_t T, const float *orig,
                            const float *dir,
                            int64_t R, float t_min, float t_max, float *range, int32_t *tri_id, cudaStream_t s);
void launch_wait_flag(const int32_t *flag, int32_t target, cudaStream_t s);
void launch_l2_read(const void *buf, int64_t bytes, int iters, float *sink, cudaStream_t s);
// gauss.cu
struct VoxGrid {
    double origin[3];
    double h;
    int dims[3];
    float theta;
};
void launch_gauss_prep(const float *mu, const float *quat, const float *scale, const float *opac, int64_t n,
                       BuildBuffers &b, unsigned int *flag, cudaStream_t s);
void launch_gauss_build(const float *mu, const float *quat, const float *scale, const float *opac, float kappa,
                        BuildBuffers &b, int bits, int leaf_size, cudaStream_t s);
void launch_voxelize(const BuildBuffers &b, const VoxGrid &g, float kappa, float *density, uint32_t *occ,
                     uint32_t *surf, uint32_t *inter, unsigned long long *counts, unsigned int *overflow,
                     cudaStream_t s);
// tsdf.cu
void launch_denoise(const uint32_t *occ, const int *dims, const float *spacing, float sigma, float tau,
                    uint32_t *out, float *vprime, cudaStream_t s, int quantile = 0, float *thr_out = nullptr);
void launch_tsdf(const uint32_t *occ, const int *dims, const float *spacing, float r, float *phi, cudaStream_t s);
void launch_marching_cubes(const float *phi, const int *dims, const float *origin, const float *spacing, float iso,
                           float *verts, float *normals, int64_t vcap, int32_t *tris, int64_t tcap, int64_t *counts,
                           cudaStream_t s);
// points.cu
void launch_iota3(int32_t *tris, int64_t n, cudaStream_t s);
void launch_nearest(const SceneView &sv, const float *q, int64_t m, float *dist, int32_t *idx, cudaStream_t s);
void launch_metrics(const float *dab, int64_t na, const float *dba, int64_t nb, float tau, double *acc,
                    unsigned int *sync, double *out, cudaStream_t s);
void launch_export_spinning(const SpinParams &p, const float *poses, int64_t P, float *orig, float *dir,
                            cudaStream_t s);
void launch_export_rosette(const RosetteParams &p, const float *poses, int64_t P, float *orig, float *dir,
                           cudaStream_t s);

}  // namespace fgl
