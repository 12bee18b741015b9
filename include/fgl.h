/*
 * fgl.h — C ABI of libfgl.so, the B200 (sm_100a) LiDAR first-return ray caster.
 *
 * The operation exposed is the nearest-hit LiDAR measurement of PAPER.md §IV-C
 * (arXiv 2509.17390, "Ray-casting for LiDAR Simulation"):
 *   beam j of a sensor with pose T_s = (R_s | t_s) in SE(3) is the ray r_j(t) = x_s + t d_j,
 *   x_s := t_s, d_j a unit direction from the scanning pattern (Eq. 19);
 *   its return is t_j* = min { tau(r_j, tri_k) : 1 <= k <= T, tau in [t_min, t_max] } over the
 *   triangle mesh M = {tri_k} (Eq. 20), range rho_j = t_j* since ||d_j|| = 1.
 * The acceleration structure is the LBVH of §IV-A: Morton codes (Eq. 5), radix sort,
 * LCP-split radix tree (Eq. 6), bottom-up bound union (Eq. 7), applied to triangle centroids.
 *
 * Conventions shared by every call
 *   - All pointers are plain host or device pointers; the library never frees or retains a
 *     caller pointer after the call returns (output buffers belong to the caller).
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream). Work is enqueued on it and
 *     the call returns without synchronising, except where a call says it synchronises.
 *   - Argument errors are detected synchronously and return FGL_E_USAGE / FGL_E_DATA before any
 *     work is enqueued. The message of the last failing call on the calling thread is
 *     available from fgl_last_error().
 *   - A miss is range = +INF and tri_id = -1. tri_id is the triangle's index in the uploaded
 *     mesh. Ties at equal t go to the smaller tri_id (reading R4).
 *   - The interval [t_min, t_max] is closed (R3). Triangles are two-sided (R2). Degenerate
 *     (zero-area) triangles are never hit (R16).
 *   - A built scene is immutable: casts on different streams may run concurrently (up to 64 in
 *     flight per scene). upload/build must not overlap casts on the same scene.
 */
#ifndef FGL_H
#define FGL_H

#include <stdint.h>

#if defined(__GNUC__)
#define FGL_API __attribute__((visibility("default")))
#else
#define FGL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FGL_OK = 0,
    FGL_E_USAGE = 1,    /* bad argument, NULL pointer, cast before build                     */
    FGL_E_DATA = 2,     /* T = 0, index out of range, NaN/Inf vertex                          */
    FGL_E_RESOURCE = 3, /* out of device memory                                              */
    FGL_E_CUDA = 4      /* any CUDA runtime error; the message carries cudaGetErrorString    */
} fgl_status;

enum { FGL_HOST = 0, FGL_DEVICE = 1, FGL_ASYNC = 4 /* or'ed into ptr_kind: see upload */ };

typedef struct fgl_scene fgl_scene; /* opaque: device copies of the mesh, the BVH and scratch */

typedef struct {
    int32_t morton_bits; /* b of Eq. 5, 1..21; 0 = default: 10 below 2^22 primitives
                            (30-bit keys, 4 sort passes), else 13 (39-bit keys), R7              */
    int32_t leaf_size;   /* max triangles per BVH leaf, 1..8; 0 = default (2)                 */
    int32_t morton_box;  /* 0 = cubic scene box (default): every axis uses L = max_a L_a, the box
                            [o, o+L] read as a cube (isotropic cells; reading R22);
                            1 = per-axis box, L_x, L_y, L_z separately                         */
    int32_t width;       /* traversal node width: 2 (binary "node64", default), 4 ("node128") or 8
                            ("node96q": the Karras tree collapsed by the SAH dynamic program of
                            Ylitie et al. 2017 into 8-wide nodes with 8-bit outward-rounded child
                            boxes and octant-ordered slots, leaves of <= 3 triangles; SURVEY A7 /
                            NEXT-4). Width 8 needs a scene extent below 2^120; a tree
                            deeper than the cast's traversal stack makes casts a no-op and
                            fgl_scene_check report FGL_E_DATA                                   */
    int32_t quantized;   /* width 4: 1 = 8-bit child boxes, outward-rounded ("node64q"); width 8
                            is always 8-bit (0 or 1 accepted)                                  */
    int32_t restructure; /* width 2 only: 0 = plain LBVH (default); k = 1..8 passes of agglomerative
                            treelet restructuring: SAH-guided re-clustering of
                            7-leaf treelets bottom-up, 1-triangle leaves (leaf_size ignored);
                            -k = k PARALLEL passes: treelets of <= 8 leaves over a depth
                            partition (roots at depth = pass mod 3), all re-clustered at once in
                            one launch per pass (no bottom-up chain), 1-triangle leaves        */
    int32_t treelets;    /* width 2, restructure 0: 1 = optimise every 4-leaf treelet bottom-up
                            INSIDE the fused build (each node, as it completes, re-links its <= 4
                            grandchildren into the lowest-SAH of the 3 / 15 binary topologies;
                            after Karras & Aila 2013 at treelet size 4): a better tree for the
                            cast at almost no build cost; leaves keep <= leaf_size triangles, the
                            scene counts as restructured (range[] of re-linked nodes is not a
                            leaf interval). 0 = the Eq. 6 Karras tree (default)               */
    int32_t reserved[1]; /* must be zero                                                     */
} fgl_build_opts;

typedef struct {
    int64_t triangles, vertices;
    int64_t nodes;        /* internal nodes of the binary LBVH (T - 1, or 1 when T = 1)       */
    int64_t device_bytes; /* device memory owned by the scene                                 */
    float scene_lo[3], scene_hi[3]; /* Morton scene box [o, o + L] (centroid bounds)   */
    float build_ms;       /* device time of the last build (synchronises on its end event)   */
    int32_t morton_bits, leaf_size;
} fgl_stats;

/* Spinning multi-beam pattern (R11, R12). Channel c has elevation
 * elev_deg[c] (host array, degrees, monotone); column a has azimuth 2*pi*a/columns + az0
 * (counter-clockwise from sensor +x). Sensor frame: x forward, y left, z up. Ray (p, c, a) is
 * stored at p*channels*columns + c*columns + a. 1 <= channels <= 512, columns >= 1. */
typedef struct {
    int32_t channels, columns;
    const float *elev_deg;
    float az0_deg, t_min, t_max;
} fgl_spinning;

/* Two-prism (Livox-style) non-repetitive pattern (R20; the paper is silent). Sample
 * n = frame*points_per_frame + k has exact 32-bit phases phi1 = n*inc1 mod 2^32,
 * phi2 = phase2_0 - n*inc2 mod 2^32 (turns * 2^32). Ray (p, k) is stored at p*N + k. */
typedef struct {
    int32_t points_per_frame;
    uint32_t inc1, inc2, phase2_0;
    float half_fov_deg, t_min, t_max;
} fgl_rosette;

/* ---- scene lifetime -------------------------------------------------------------------- */
FGL_API fgl_status fgl_scene_create(int cuda_device, fgl_scene **out);
FGL_API void fgl_scene_destroy(fgl_scene *scene);

/* Copy the mesh M = {tri_k} into scene-owned device memory and validate it:
 * verts: float32 [V][3]; tris: int32 [T][3], 0 <= index < V. ptr_kind says whether both pointers
 * are FGL_HOST or FGL_DEVICE. Synchronises `cuda_stream` to report FGL_E_DATA (T = 0, an index out
 * of range, a non-finite vertex). Invalidates any previous build. T must be < 2^28.
 * With FGL_ASYNC or'ed into ptr_kind the call does not synchronise (graph-capturable): the
 * validation result stays on the device and fgl_scene_check reports it; until then the build and
 * casts stay memory-safe (indices are clamped) but their results are unspecified for bad meshes. */
FGL_API fgl_status fgl_scene_upload_mesh(fgl_scene *scene, const float *verts, int64_t V, const int32_t *tris,
                                 int64_t T, int ptr_kind, void *cuda_stream);

/* LBVH build, §IV-A, on the device, enqueued on `cuda_stream`:
 * centroids + scene box -> Morton codes (Eq. 5) -> stable LSD radix sort -> Karras radix tree
 * (Eq. 6) -> bottom-up refit (Eq. 7) -> triangle records reordered into leaf order -> traversal
 * nodes. For width 2 (the default) the last four steps are one kernel that builds the tree and
 * its Eq. 7 boxes bottom-up (the same tree, child links, ranges and nodes, bit for bit). opts may
 * be NULL (defaults). Does no host synchronisation; graph-capturable (every replay rebuilds,
 * also over new vertex data of the same size). */
FGL_API fgl_status fgl_scene_build(fgl_scene *scene, const fgl_build_opts *opts, void *cuda_stream);

/* Synchronises `cuda_stream` and returns FGL_E_DATA if the last upload failed validation. */
FGL_API fgl_status fgl_scene_check(fgl_scene *scene, void *cuda_stream);

/* Refit for a deforming mesh (dynamic scenes are the paper's future work,
 * P:435): new vertex positions verts [V][3] (same V and triangles as the upload, FGL_HOST /
 * FGL_DEVICE | FGL_ASYNC) replace the old ones; the leaf records, leaf boxes, Eq. 7 node boxes
 * (exact unions over each node's stored leaf range) and nodes are recomputed while the Morton
 * order and the tree topology of the last build are kept (casts stay exact; the tree degrades
 * only in quality as the mesh moves away from the built pose). Recorded as build_ms.
 * FGL_E_USAGE: not built, V differs, a Gaussian scene; FGL_E_DATA: non-finite vertex. */
FGL_API fgl_status fgl_scene_refit(fgl_scene *scene, const float *verts, int64_t V, int ptr_kind, void *cuda_stream);

/* Fills *out. Synchronises on the last build's end event (for build_ms and the scene box). */
FGL_API fgl_status fgl_scene_stats(fgl_scene *scene, fgl_stats *out);

/* ---- casts (Eqs. 19-20) ---------------------------------------------------------------- */
/* poses: device float32 [P][3][4] row-major (R | t), sensor -> world (R13). Directions are
 * normalised after rotation. range: device float32 [P][channels][columns]; tri_id: device int32,
 * same shape; hit_xyz: NULL or device float32 [..][3] (x* = x_s + t* d).
 * node_counts / tri_counts: NULL, or device int32 per ray: BVH nodes visited and triangles tested
 * (the N_nodes(r_j) and K_j of Eq. 21). */
FGL_API fgl_status fgl_cast_spinning(const fgl_scene *scene, const fgl_spinning *pattern, const float *poses, int64_t P,
                             float *range, int32_t *tri_id, float *hit_xyz, int32_t *node_counts,
                             int32_t *tri_counts, void *cuda_stream);

/* Rosette: poses[p] is frame first_frame + p; outputs [P][points_per_frame]. */
FGL_API fgl_status fgl_cast_rosette(const fgl_scene *scene, const fgl_rosette *pattern, const float *poses, int64_t P,
                            int64_t first_frame, float *range, int32_t *tri_id, float *hit_xyz,
                            int32_t *node_counts, int32_t *tri_counts, void *cuda_stream);

/* Explicit rays (SPEC first_hit): orig, dir device float32 [R][3]; t is the ray parameter
 * (equal to the range when ||dir|| = 1). 0 <= t_min < t_max. */
FGL_API fgl_status fgl_cast_rays(const fgl_scene *scene, const float *orig, const float *dir, int64_t R, float t_min,
                         float t_max, float *range, int32_t *tri_id, void *cuda_stream);

/* The naive O(N_r T) cast of P:291-294 on the GPU (no BVH; needs only an uploaded mesh), with the
 * same watertight test and tie-break as the BVH cast. A parity bridge and a baseline. */
FGL_API fgl_status fgl_cast_rays_bruteforce(const fgl_scene *scene, const float *orig, const float *dir, int64_t R,
                                    float t_min, float t_max, float *range, int32_t *tri_id, void *cuda_stream);

/* Write the exact float32 rays (origin, unit direction) the cast kernels generate for a pattern,
 * device float32 [R][3] each, in the cast's output order. */
FGL_API fgl_status fgl_export_rays_spinning(const fgl_spinning *pattern, const float *poses, int64_t P, float *orig,
                                    float *dir, void *cuda_stream);
FGL_API fgl_status fgl_export_rays_rosette(const fgl_rosette *pattern, const float *poses, int64_t P, int64_t first_frame,
                                   float *orig, float *dir, void *cuda_stream);

/* ---- fused cast + all-gather over peer memory (A12) ------------------------
 * Device memory owned by the library (allocation bases, so they can be shared by CUDA IPC). */
FGL_API fgl_status fgl_alloc(int cuda_device, int64_t bytes, void **dev_ptr);
FGL_API fgl_status fgl_free(void *dev_ptr);
typedef struct {
    unsigned char bytes[64];
} fgl_ipc_handle;
/* Export an fgl_alloc'ed pointer to another process of the node / open a peer's export in this
 * process (cudaIpcGetMemHandle / cudaIpcOpenMemHandle with peer access). */
FGL_API fgl_status fgl_ipc_get_handle(void *dev_ptr, fgl_ipc_handle *out);
FGL_API fgl_status fgl_ipc_open_handle(int cuda_device, const fgl_ipc_handle *handle, void **dev_ptr);
FGL_API fgl_status fgl_ipc_close_handle(void *dev_ptr);

/* fgl_cast_spinning whose results are written, from inside the cast kernel, into npeer global
 * output buffers at ray index first_pose*channels*columns + (local index): rank r of W casts its
 * pose block and writes straight into every rank's [P_total][C][A] range / tri_id buffers (its own
 * and the peers' opened with fgl_ipc_open_handle), so the all-gather overlaps the cast tile by
 * tile over NVLink. 1 <= npeer <= 8. The caller synchronises the ranks before reading. */
FGL_API fgl_status fgl_cast_spinning_gather(const fgl_scene *scene, const fgl_spinning *pattern, const float *poses,
                                            int64_t P, int64_t first_pose, float *const *range_bufs,
                                            int32_t *const *tri_bufs, int32_t npeer, void *cuda_stream);
/* Device-side completion barrier for the fused gather: `flags` (NULL or [npeer] int32 counters in
 * fgl_alloc'ed memory, index 0 = this rank's own, the others opened by IPC) are each incremented
 * by the cast kernel's last warp after a system-scope fence (pass them to
 * fgl_cast_spinning_gather_signal); fgl_wait_flag makes `cuda_stream` wait until *flag >= target. */
FGL_API fgl_status fgl_cast_spinning_gather_signal(const fgl_scene *scene, const fgl_spinning *pattern,
                                                   const float *poses, int64_t P, int64_t first_pose,
                                                   float *const *range_bufs, int32_t *const *tri_bufs,
                                                   int32_t *const *flags, int32_t npeer, void *cuda_stream);
FGL_API fgl_status fgl_wait_flag(const int32_t *flag, int32_t target, void *cuda_stream);

/* ---- point-cloud metrics (§V-A) --------------------------------
 * A point scene indexes a cloud with the same LBVH (one degenerate triangle (i, i, i) per point;
 * build it with fgl_scene_build, width 2). Same validation / FGL_ASYNC rules as upload_mesh. */
FGL_API fgl_status fgl_scene_upload_points(fgl_scene *scene, const float *xyz, int64_t n, int ptr_kind,
                                           void *cuda_stream);
/* Exact nearest neighbour (Euclidean, float32 distances, ties to the smaller index) in a built
 * point scene for m device query points [m][3]: dist [m] (NaN for a non-finite query), idx [m]. */
FGL_API fgl_status fgl_nearest(const fgl_scene *scene, const float *queries, int64_t m, float *dist, int32_t *idx,
                               void *cuda_stream);
/* From directed nearest-neighbour distances d_ab [n_a] (a -> b) and d_ba [n_b] (device, NaN
 * entries ignored): out (device double [6]) = {symmetric Chamfer distance (mean of the two directed
 * means of unsquared distances), precision = frac(d_ab <= tau), recall = frac(d_ba <= tau),
 * F-score = 2PR/(P+R) (0 if P+R = 0), finite n_a, finite n_b}. Reading R23. */
FGL_API fgl_status fgl_cloud_metrics(const float *d_ab, int64_t n_a, const float *d_ba, int64_t n_b, float tau,
                                     double *out, void *cuda_stream);

/* ---- Gaussian -> occupancy (§IV-A) --------------- */
/* Uploads a 3DGS cloud G = {(mu_i, q_i, s_i, sigma_i)}: mu [n][3], q [n][4] as (w, x, y,
 * z) (normalised on the device), s [n][3] > 0 (activated scales), opacity [n] in [0, 1]
 * (activated), all float32 in `ptr_kind` memory (FGL_HOST / FGL_DEVICE, | FGL_ASYNC as for
 * upload_mesh). kappa >= 1 is the Eq. 4 padding factor (3 = the 3-sigma box). The
 * scene then indexes the Gaussians with the LBVH (fgl_scene_build: Morton codes of mu_i, Eqs.
 * 5-7, width 2, cubic box); it cannot be cast against. FGL_E_DATA: n = 0, non-finite mu / q,
 * q = 0, scale <= 0 or opacity outside [0, 1]. */
FGL_API fgl_status fgl_scene_upload_gaussians(fgl_scene *scene, const float *mu, const float *quat,
                                              const float *scale, const float *opacity, int64_t n, float kappa,
                                              int ptr_kind, void *cuda_stream);

/* Voxel lattice: voxel (i, j, k) has centre origin + (i + 1/2, j + 1/2, k + 1/2) spacing. */
typedef struct {
    float origin[3];
    float spacing;        /* h > 0                                                               */
    int32_t dims[3];      /* nx, ny, nz >= 1, nx * ny * nz <= 2^31                               */
    int32_t tile;         /* B of Eq. 8; 0 = default (8); only 8 is accepted                     */
    float theta;          /* Eq. 10 threshold                                                    */
    int32_t reserved[3];  /* must be zero                                                        */
} fgl_grid;

/* Voxelizes a built Gaussian scene on the caller's stream (no host sync):
 *   Eq. 8  candidates of each B^3 tile = Gaussians whose Eq. 4 box meets the box of the tile's
 *          voxel centres (a BVH overlap query);
 *   Eq. 9  D(v) = sum over candidates of exp(-m^2 / 2) f(sigma), f(sigma) = sigma (R24), with
 *          m^2 = (v - mu)^T Sigma^-1 (v - mu) and contributions beyond m^2 > kappa^2 dropped (R25,
 *          so the result does not depend on B), float32 arithmetic;
 *   Eq. 10 occupancy V = D > theta; Eqs. 11-12 interior = V and its 6 neighbours (outside the grid
 *          = empty, R27), surface = V and not interior.
 * Device outputs: density float [nz][ny][nx] (nullable); occupancy, surface, interior as bit
 * volumes uint32 [nz][ny][ceil(nx / 32)] (bit b of word w = voxel x = 32 w + b; surface and
 * interior nullable); counts int64 [4] (nullable) = {occupied voxels, surface voxels, evaluated
 * (voxel, candidate) pairs, traversal-stack overflow flag (0 unless the result is incomplete)}.
 * FGL_E_USAGE: not a built Gaussian scene, NULL occupancy, bad grid; FGL_E_RESOURCE: > 2^31 voxels. */
FGL_API fgl_status fgl_voxelize(const fgl_scene *scene, const fgl_grid *grid, float *density, uint32_t *occupancy,
                                uint32_t *surface, uint32_t *interior, int64_t *counts, void *cuda_stream);

/* ---- occupancy -> mesh (§IV-B) ---------------------
 * Volumes are device arrays on the current CUDA device, voxel (i, j, k) at linear index
 * (k ny + j) nx + i with centre origin + (i + 1/2, j + 1/2, k + 1/2) spacing; bit volumes are
 * uint32 [nz][ny][ceil(nx / 32)] (bit b of word w = voxel x = 32 w + b), as fgl_voxelize writes.
 * Scratch is stream-ordered (cudaMallocAsync), so the calls are CUDA-graph capturable. */

/* Eq. 13-14a: V' = G_sigma * V (separable, sigma in metres -> sigma / spacing[a] voxels, kernel
 * truncated at ceil(3 sigma) voxels and normalised, zero outside the grid; float32), out = V' >= tau
 * (bit volume). vprime (nullable): float [nz][ny][nx]. FGL_E_USAGE: sigma > 21 voxels, bad sizes. */
FGL_API fgl_status fgl_denoise(const uint32_t *occupancy, const int32_t *dims, const float *spacing, float sigma,
                               float tau, uint32_t *out, float *vprime, void *cuda_stream);

/* Eq. 13-14b: as fgl_denoise, but the threshold is Quantile_q(V') over the whole grid, read as the
 * inverted-CDF quantile: the value of 1-based rank max(1, ceil(q N)) in ascending order (R35),
 * selected on the device by a 3-pass radix select of the float32 V' (so V~ = V' >= that value).
 * threshold (nullable, device float [1]) receives the selected value. q in [0, 1]. */
FGL_API fgl_status fgl_denoise_quantile(const uint32_t *occupancy, const int32_t *dims, const float *spacing,
                                        float sigma, float q, uint32_t *out, float *vprime, float *threshold,
                                        void *cuda_stream);

/* Eqs. 15-17 narrow-band TSDF of a bit volume: s = +1 on free voxels 6-connected to the padded
 * frame (flood fill), -1 elsewhere; kappa = shell index of the 6-neighbour expansion from
 * S_0 = {x : a 6-neighbour differs in V} (the frame counts as free); phi = s min(kappa v_min, r)
 * (float32; s r beyond the band), v_min = min(spacing). phi: float [nz][ny][nx]. The band
 * r / v_min must be <= 254 shells. */
FGL_API fgl_status fgl_tsdf(const uint32_t *occupancy, const int32_t *dims, const float *spacing, float r, float *phi,
                            void *cuda_stream);

/* Eq. 18 Marching Cubes of phi at iso on the voxel-centre lattice (corner inside iff phi < iso):
 * face-consistent cube polygons (R34: inside corners cut off run by run per face, loops
 * fanned from their lowest edge, or around a centre vertex when a fan diagonal would lie in a
 * face), so the mesh is watertight wherever the surface stays inside the grid and consistently
 * oriented (normals towards phi > iso). Vertices: one per crossing edge, numbered by global edge
 * id 3 * voxel + axis, then the centre vertices; verts float [vcap][3], normals (nullable) the
 * normalised interpolated central-difference gradient, tris int32 [tcap][3]; entries beyond a
 * capacity are not written. counts (device int64 [2], nullable) = {vertices, triangles} needed. */
FGL_API fgl_status fgl_marching_cubes(const float *phi, const int32_t *dims, const float *origin, const float *spacing,
                                      float iso, float *verts, float *normals, int64_t vcap, int32_t *tris,
                                      int64_t tcap, int64_t *counts, void *cuda_stream);

/* ---- LBVH internals, for parity tests (host destination pointers; each may be NULL) ----- */
typedef struct {
    float *scene_box;      /* [6]  lo.xyz, hi.xyz                                              */
    uint64_t *codes;       /* [T]  Morton codes in input order (Eq. 5)                          */
    uint64_t *sorted_keys; /* [T]  codes after the stable sort                                  */
    uint32_t *perm;        /* [T]  input triangle index at each sorted position                 */
    int32_t *child;        /* [T-1][2] radix tree (Eq. 6): internal i, or leaf j encoded as ~j  */
    int32_t *range;        /* [T-1][2] first, last sorted position covered by internal node i    */
    float *leaf_box;       /* [T][6]   exact AABB of the triangle at sorted position j          */
    float *node_box;       /* [T-1][6] Eq. 7 union                                              */
    float *tri48;          /* [T][12]  leaf-order triangle records {v0, id}, {v1, 0}, {v2, 0}    */
    float *nodes;          /* [max(T-1,1)][16] binary traversal nodes (DESIGN.md §5 "node64")   */
    float *nodes4;         /* [max(T-1,1)][32] 4-wide traversal nodes at their binary node index
                              (DESIGN.md §5 "node128"; only even-depth slots are meaningful)     */
    int32_t *depth;        /* [T-1] depth of each internal node (root = 0)                      */
} fgl_export;

/* Synchronously copies the requested build arrays of a built scene to host memory. */
FGL_API fgl_status fgl_scene_export(const fgl_scene *scene, const fgl_export *out, void *cuda_stream);

/* Stand-alone build steps on caller device buffers (enqueued on cuda_stream):
 * Eq. 5 Morton codes of n points (device float32 [n][3]) in the box [lo, hi] (host float[3]). */
FGL_API fgl_status fgl_morton_codes(const float *points, int64_t n, const float *lo, const float *hi, int32_t bits,
                            uint64_t *codes, void *cuda_stream);
/* Stable LSD radix sort of (key, value) pairs in place, on the low key_bits bits of the keys
 * (1..64), n < 2^30. Allocates its scratch with cudaMallocAsync on the stream. */
FGL_API fgl_status fgl_sort_pairs(uint64_t *keys, uint32_t *vals, int64_t n, int32_t key_bits, void *cuda_stream);

/* ---- measurement --------------------------------------------------------------------------
 * L2 read-bandwidth probe (the roofline of an L2-resident traversal is the L2, whose
 * bandwidth is measured in the run, not assumed). Enqueues on cuda_stream one kernel that reads the
 * device buffer `buf` (`bytes` >= 16, a multiple of 16, 16-B aligned; pick it well below the L2
 * size so it stays resident) `iters` >= 1 times with 128-bit L1-bypassing loads (ld.global.cg)
 * from every SM, and writes one float (a checksum that keeps the loads alive) to `sink` (device).
 * The caller times the launch with CUDA events: GB/s = bytes * iters / time. Errors: FGL_E_USAGE
 * for NULL pointers / bad sizes, FGL_E_CUDA for launch failures. */
FGL_API fgl_status fgl_l2_read_probe(const void *buf, int64_t bytes, int32_t iters, float *sink, void *cuda_stream);

/* ---- misc ----------------------------------------------------------------------------- */
FGL_API const char *fgl_last_error(void); /* thread-local; valid until the next fgl call on the thread */
FGL_API const char *fgl_version(void);
FGL_API int32_t fgl_abi_version(void);   /* bumped on any incompatible change of this header (2) */
/* Number of kernels libfgl has launched in this process (all devices, all threads). */
FGL_API int64_t fgl_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* FGL_H */
