/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the LiDAR first-return cast path
 * computes, written from PAPER.md (arXiv 2509.17390, §IV-A and §IV-C) in double precision.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library. It shares no code, header, table or constant generator with the CUDA path
 * (paper_2509_17390_b200/csrc): the product never links or calls it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation given alongside).
 * Readings of silent or ambiguous passages are numbered R1..R21 in DESIGN.md §3.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared -ffp-contract=off -fno-fast-math oracle.c -lm
 * (no FMA contraction, IEEE semantics; float arithmetic on x86-64 is SSE single precision).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846

static int g_threads = 0;

void orc_set_threads(int n) { g_threads = n; }

int orc_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------------------------ */
/* Ray model, Eq. 19: r_j(t) = x_s + t d_j, x_s := t_s, d_j = R_s d_j^sensor, unit.   */
/* Pose layout (R13): float32 [3][4] row-major (R | t), sensor -> world.                          */
/* ------------------------------------------------------------------------------------------ */
static void pose_apply(const float *M, const double ds[3], double o[3], double d[3]) {
    double w[3];
    for (int r = 0; r < 3; ++r) {
        w[r] = (double)M[4 * r + 0] * ds[0] + (double)M[4 * r + 1] * ds[1] + (double)M[4 * r + 2] * ds[2];
        o[r] = (double)M[4 * r + 3];
    }
    double n = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    for (int r = 0; r < 3; ++r) d[r] = w[r] / n; /* ||d_j|| = 1 so rho_j = t_j* */
}

/* Spinning pattern (R11, R12): channel c has elevation e_c (degrees), column a has
 * azimuth theta_a = 2 pi a / A + az0 (counter-clockwise from +x); sensor frame x fwd, y left, z up:
 * d = (cos e cos theta, cos e sin theta, sin e). Ray index g = p*C*A + c*A + a (row-major). */
void orc_spinning_rays(const float *elev_deg, int32_t C, int32_t A, double az0_deg,
                       const float *poses, int64_t P, double *orig, double *dir) {
    int64_t n = (int64_t)P * C * A;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
    for (int64_t g = 0; g < n; ++g) {
        int64_t p = g / ((int64_t)C * A);
        int32_t c = (int32_t)((g / A) % C);
        int32_t a = (int32_t)(g % A);
        double e = (double)elev_deg[c] * (ORC_PI / 180.0);
        double th = 2.0 * ORC_PI * (double)a / (double)A + az0_deg * (ORC_PI / 180.0);
        double ds[3] = {cos(e) * cos(th), cos(e) * sin(th), sin(e)};
        pose_apply(poses + 12 * p, ds, orig + 3 * g, dir + 3 * g);
    }
}

/* Rosette (Livox-style, two counter-rotating prisms; the paper is silent, reading R20):
 * global sample n = frame*N + k; exact 32-bit phases
 *   phi1 = (n*inc1 mod 2^32)/2^32,  phi2 = (phase2_0 - n*inc2 mod 2^32)/2^32;
 * delta = (Phi/2) (cos 2pi phi1 + cos 2pi phi2, sin 2pi phi1 + sin 2pi phi2), Phi = half FOV;
 * rho = |delta|; d = (cos rho, delta_x sin(rho)/rho, delta_y sin(rho)/rho). Ray index p*N + k. */
void orc_rosette_rays(int32_t N, uint32_t inc1, uint32_t inc2, uint32_t phase2_0, double half_fov_deg,
                      const float *poses, int64_t P, int64_t first_frame, double *orig, double *dir) {
    int64_t n_all = (int64_t)P * N;
    double Phi = half_fov_deg * (ORC_PI / 180.0);
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
    for (int64_t g = 0; g < n_all; ++g) {
        int64_t p = g / N, k = g % N;
        uint64_t n = (uint64_t)(first_frame + p) * (uint64_t)N + (uint64_t)k;
        uint32_t ph1 = (uint32_t)(n * (uint64_t)inc1);
        uint32_t ph2 = (uint32_t)((uint64_t)phase2_0 - n * (uint64_t)inc2);
        double f1 = (double)ph1 / 4294967296.0, f2 = (double)ph2 / 4294967296.0;
        double dx = 0.5 * Phi * (cos(2.0 * ORC_PI * f1) + cos(2.0 * ORC_PI * f2));
        double dy = 0.5 * Phi * (sin(2.0 * ORC_PI * f1) + sin(2.0 * ORC_PI * f2));
        double rho = sqrt(dx * dx + dy * dy);
        double s = rho > 0.0 ? sin(rho) / rho : 1.0;
        double ds[3] = {cos(rho), dx * s, dy * s};
        pose_apply(poses + 12 * p, ds, orig + 3 * g, dir + 3 * g);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Nearest intersection, Eq. 20, by the naive O(N_r T) scan:            */
/*   t_j* = min { tau(r_j, tri_k) : 1 <= k <= T, tau in [t_min, t_max] }.                        */
/* tau by double-precision Moller-Trumbore, two-sided (R2), inclusive edges, det == 0 -> no hit  */
/* (R16); triangles visited in index order and best replaced only on strict t < best, so equal t */
/* goes to the smaller index (R4). Miss: t = +inf, id = -1 (R6).                                 */
/* ------------------------------------------------------------------------------------------ */
static inline void ldv(const float *verts, int32_t i, double v[3]) {
    v[0] = verts[3 * (int64_t)i];
    v[1] = verts[3 * (int64_t)i + 1];
    v[2] = verts[3 * (int64_t)i + 2];
}

static inline void cross(const double a[3], const double b[3], double c[3]) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

static inline double dot(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* returns 1 and sets *t when the ray hits the triangle (Moller & Trumbore 1997) */
static inline int mt_hit(const double o[3], const double d[3], const double v0[3], const double v1[3],
                         const double v2[3], double *t) {
    double e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
    double e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
    double p[3], q[3];
    cross(d, e2, p);
    double det = dot(e1, p);
    if (det == 0.0) return 0;
    double inv = 1.0 / det;
    double s[3] = {o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]};
    double u = dot(s, p) * inv;
    if (u < 0.0 || u > 1.0) return 0;
    cross(s, e1, q);
    double v = dot(d, q) * inv;
    if (v < 0.0 || u + v > 1.0) return 0;
    *t = dot(e2, q) * inv;
    return 1;
}

void orc_cast(const float *verts, const int32_t *tris, int64_t T, const double *orig, const double *dir,
              int64_t R, double t_min, double t_max, double *t_out, int32_t *id_out) {
#pragma omp parallel for schedule(dynamic, 4) num_threads(orc_get_threads())
    for (int64_t r = 0; r < R; ++r) {
        const double *o = orig + 3 * r, *d = dir + 3 * r;
        double best = INFINITY;
        int32_t bid = -1;
        for (int64_t k = 0; k < T; ++k) {
            double v0[3], v1[3], v2[3], t;
            ldv(verts, tris[3 * k], v0);
            ldv(verts, tris[3 * k + 1], v1);
            ldv(verts, tris[3 * k + 2], v2);
            if (!mt_hit(o, d, v0, v1, v2, &t)) continue;
            if (t < t_min || t > t_max) continue;
            if (t < best) {
                best = t;
                bid = (int32_t)k;
            }
        }
        t_out[r] = best;
        id_out[r] = bid;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Ambiguity classifier (DESIGN.md §4 "acceptance").                                             */
/* Eq. 20 has several correct float answers for rays that pass within rounding distance of a    */
/* triangle boundary or whose nearest depths tie. For each ray and triangle k, in double:        */
/*   eps_k  = eps_rel * max(1 m, max_i |v_ki - o|)   (perturbation of a float32 ray/vertex test)  */
/*   m_k    = signed distance, in the plane orthogonal to d, from the ray to the boundary of the  */
/*            triangle projected along d (>0 inside). m_k < -eps_k: cannot be hit; m_k > eps_k:   */
/*            "solid" (hit under any such perturbation); otherwise "marginal".                    */
/*   depth interval: plane depth +- eps_k (1 + 1/|cos g|), clipped to the vertex depth span +-eps */
/* Firm candidate = solid and depth interval inside [t_min, t_max]. Kept candidates = all with   */
/* t_lo <= min over firm of t_hi (or all, if none is firm). MISS_OK iff no firm candidate.        */
/* Unambiguous iff (kept == {k1}, k1 firm, interval narrow) or (no candidate and strict miss).    */
/* A bounding-sphere prefilter skips triangles that cannot be candidates (conservative).         */
/* ------------------------------------------------------------------------------------------ */
enum {
    ORC_AMBIG = 1,
    ORC_EDGE = 2,
    ORC_BOUNDARY = 4,
    ORC_GRAZE = 8,
    ORC_OVERFLOW = 16,
    ORC_MISS_OK = 32,
    ORC_INCONSISTENT = 64
};

static inline double cross2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }

static double segdist(double ax, double ay, double bx, double by) {
    /* distance from (0,0) to segment a-b */
    double ex = bx - ax, ey = by - ay, L2 = ex * ex + ey * ey;
    double s = L2 > 0 ? -(ax * ex + ay * ey) / L2 : 0.0;
    if (s < 0) s = 0;
    if (s > 1) s = 1;
    double px = ax + s * ex, py = ay + s * ey;
    return sqrt(px * px + py * py);
}

void orc_classify(const float *verts, const int32_t *tris, int64_t T, const double *orig, const double *dir,
                  int64_t R, double t_min, double t_max, double eps_rel, const double *t1, const int32_t *k1,
                  int32_t kmax, int32_t *flags, int32_t *ncand, int32_t *cand_id, double *cand_lo,
                  double *cand_hi) {
#pragma omp parallel num_threads(orc_get_threads())
    {
        int32_t cap = 64;
        int32_t *cid = (int32_t *)malloc(sizeof(int32_t) * cap);
        double *clo = (double *)malloc(sizeof(double) * cap), *chi = (double *)malloc(sizeof(double) * cap);
        char *cfirm = (char *)malloc(cap);
#pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < R; ++r) {
            const double *o = orig + 3 * r;
            double dn = sqrt(dot(dir + 3 * r, dir + 3 * r));
            double dh[3] = {dir[3 * r] / dn, dir[3 * r + 1] / dn, dir[3 * r + 2] / dn};
            /* orthonormal basis e1, e2 of the plane orthogonal to dh */
            double ref[3] = {0, 0, 0};
            int ax = fabs(dh[0]) <= fabs(dh[1]) ? (fabs(dh[0]) <= fabs(dh[2]) ? 0 : 2) : (fabs(dh[1]) <= fabs(dh[2]) ? 1 : 2);
            ref[ax] = 1.0;
            double e1[3], e2[3];
            cross(dh, ref, e1);
            double n1 = sqrt(dot(e1, e1));
            e1[0] /= n1, e1[1] /= n1, e1[2] /= n1;
            cross(dh, e1, e2);
            double zmin = t_min * dn, zmax = t_max * dn;
            int32_t nc = 0;
            for (int64_t k = 0; k < T; ++k) {
                double v[3][3];
                ldv(verts, tris[3 * k], v[0]);
                ldv(verts, tris[3 * k + 1], v[1]);
                ldv(verts, tris[3 * k + 2], v[2]);
                /* conservative bounding-sphere prefilter */
                double c[3], rad = 0;
                for (int i = 0; i < 3; ++i) c[i] = (v[0][i] + v[1][i] + v[2][i]) / 3.0;
                for (int j = 0; j < 3; ++j) {
                    double q[3] = {v[j][0] - c[0], v[j][1] - c[1], v[j][2] - c[2]};
                    double l = sqrt(dot(q, q));
                    if (l > rad) rad = l;
                }
                double w[3] = {c[0] - o[0], c[1] - o[1], c[2] - o[2]};
                double wl = sqrt(dot(w, w));
                double reach = 2.0 * eps_rel * fmax(1.0, wl + rad) + 1e-12;
                double z = dot(w, dh);
                if (z - rad - reach > zmax || z + rad + reach < zmin) continue;
                double q2 = wl * wl - z * z;
                if (q2 > (rad + reach) * (rad + reach)) continue;
                /* projected 2D triangle */
                double a[3][3], px[3], py[3], pz[3], amax = 0;
                for (int j = 0; j < 3; ++j) {
                    for (int i = 0; i < 3; ++i) a[j][i] = v[j][i] - o[i];
                    px[j] = dot(a[j], e1);
                    py[j] = dot(a[j], e2);
                    pz[j] = dot(a[j], dh);
                    double l = sqrt(dot(a[j], a[j]));
                    if (l > amax) amax = l;
                }
                double eps = eps_rel * fmax(1.0, amax);
                double area2 = cross2(px[1] - px[0], py[1] - py[0], px[2] - px[0], py[2] - py[0]);
                double m;
                if (area2 != 0.0) {
                    double sg = area2 > 0 ? 1.0 : -1.0;
                    m = INFINITY;
                    for (int j = 0; j < 3; ++j) {
                        int jn = (j + 1) % 3;
                        double ex = px[jn] - px[j], ey = py[jn] - py[j];
                        double L = sqrt(ex * ex + ey * ey);
                        double s = sg * cross2(ex, ey, -px[j], -py[j]) / L;
                        if (s < m) m = s;
                    }
                } else {
                    double md = INFINITY;
                    for (int j = 0; j < 3; ++j) {
                        int jn = (j + 1) % 3;
                        double s = segdist(px[j], py[j], px[jn], py[jn]);
                        if (s < md) md = s;
                    }
                    m = -md;
                }
                if (m < -eps) continue;
                int solid = m > eps;
                /* depth interval along dh */
                double e_a[3] = {v[1][0] - v[0][0], v[1][1] - v[0][1], v[1][2] - v[0][2]};
                double e_b[3] = {v[2][0] - v[0][0], v[2][1] - v[0][1], v[2][2] - v[0][2]};
                double nrm[3];
                cross(e_a, e_b, nrm);
                double nl = sqrt(dot(nrm, nrm));
                double nd = dot(nrm, dh);
                double cg = nl > 0 ? fabs(nd) / nl : 0.0;
                double zlo = fmin(pz[0], fmin(pz[1], pz[2])) - eps;
                double zhi = fmax(pz[0], fmax(pz[1], pz[2])) + eps;
                double lo = zlo, hi = zhi;
                if (cg > 0) {
                    double zp = dot(nrm, a[0]) / nd;
                    double dz = eps * (1.0 + 1.0 / cg);
                    lo = fmax(zlo, zp - dz);
                    hi = fmin(zhi, zp + dz);
                    if (lo > hi) lo = hi = fmin(fmax(zp, zlo), zhi);
                }
                if (hi < zmin || lo > zmax) continue;
                int inrange = lo >= zmin && hi <= zmax;
                if (nc == cap) {
                    cap *= 2;
                    cid = (int32_t *)realloc(cid, sizeof(int32_t) * cap);
                    clo = (double *)realloc(clo, sizeof(double) * cap);
                    chi = (double *)realloc(chi, sizeof(double) * cap);
                    cfirm = (char *)realloc(cfirm, cap);
                }
                cid[nc] = (int32_t)k;
                clo[nc] = lo / dn;
                chi[nc] = hi / dn;
                cfirm[nc] = (char)(solid && inrange);
                ++nc;
            }
            /* keep candidates that could precede (or tie with) the nearest firm hit */
            double tf = INFINITY;
            int32_t nfirm = 0;
            for (int32_t i = 0; i < nc; ++i)
                if (cfirm[i]) {
                    ++nfirm;
                    if (chi[i] < tf) tf = chi[i];
                }
            int32_t f = 0, kept = 0, k1_kept = 0, k1_firm = 0, boundary = 0;
            double k1_w = 0;
            for (int32_t i = 0; i < nc; ++i) {
                if (nfirm && clo[i] > tf) continue;
                if (clo[i] < t_min || chi[i] > t_max) boundary = 1;
                if (cid[i] == k1[r]) {
                    k1_kept = 1;
                    k1_firm = cfirm[i];
                    k1_w = chi[i] - clo[i];
                }
                if (kept < kmax) {
                    cand_id[r * kmax + kept] = cid[i];
                    cand_lo[r * kmax + kept] = clo[i];
                    cand_hi[r * kmax + kept] = chi[i];
                }
                ++kept;
            }
            if (!nfirm) f |= ORC_MISS_OK;
            if (kept > kmax) f |= ORC_OVERFLOW;
            if (boundary) f |= ORC_BOUNDARY;
            if (kept > 1 || (kept == 1 && !k1_firm)) f |= ORC_EDGE;
            if (k1[r] >= 0 && !k1_kept) f |= ORC_INCONSISTENT;
            if (k1[r] >= 0 && k1_kept && k1_w > 1e-4 * t1[r] + 1e-5) f |= ORC_GRAZE;
            int unamb = 0;
            if (k1[r] >= 0)
                unamb = kept == 1 && k1_kept && k1_firm && !(f & (ORC_GRAZE | ORC_BOUNDARY | ORC_INCONSISTENT));
            else
                unamb = kept == 0;
            if (!unamb) f |= ORC_AMBIG;
            flags[r] = f;
            ncand[r] = kept;
        }
        free(cid);
        free(clo);
        free(chi);
        free(cfirm);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* LBVH build, §IV-A, applied to triangles (R8).                                     */
/* ------------------------------------------------------------------------------------------ */

/* Morton point of a triangle (R8): its centroid, c = ((v0 + v1) + v2) / 3 in float32, RN. */
void orc_centroids(const float *verts, const int32_t *tris, int64_t T, float *cent) {
    for (int64_t k = 0; k < T; ++k)
        for (int i = 0; i < 3; ++i) {
            float a = verts[3 * (int64_t)tris[3 * k] + i], b = verts[3 * (int64_t)tris[3 * k + 1] + i];
            float c = verts[3 * (int64_t)tris[3 * k + 2] + i];
            float s = a + b;
            s = s + c;
            cent[3 * k + i] = s / 3.0f;
        }
}

/* Scene box [o, o+L]: the exact bounds of the Morton points. */
void orc_scene_box(const float *cent, int64_t n, float *lo, float *hi) {
    for (int i = 0; i < 3; ++i) {
        lo[i] = INFINITY;
        hi[i] = -INFINITY;
    }
    for (int64_t k = 0; k < n; ++k)
        for (int i = 0; i < 3; ++i) {
            if (cent[3 * k + i] < lo[i]) lo[i] = cent[3 * k + i];
            if (cent[3 * k + i] > hi[i]) hi[i] = cent[3 * k + i];
        }
}

/* Eq. 5: m = interleave(floor(2^b (mu_x - o_x)/L_x), ... y, ... z), x lowest.
 * The quantisation is a float decision; it is taken in float32 exactly as the kernel does (R7):
 * L = hi - lo; s = (L > 0) ? 2^b / L : 0; x = (c - lo) * s; q = min(floor(x), 2^b - 1).
 * cubic != 0 (reading R22): every axis uses L = max(L_x, L_y, L_z). */
void orc_morton(const float *cent, int64_t n, const float *lo, const float *hi, int bits, int cubic,
                uint64_t *code) {
    float s[3], L[3], Lc = 0.0f;
    float two_b = (float)(1u << bits);
    uint32_t qmax = (1u << bits) - 1u;
    for (int i = 0; i < 3; ++i) {
        L[i] = hi[i] - lo[i];
        if (L[i] > Lc) Lc = L[i];
    }
    for (int i = 0; i < 3; ++i) {
        float Li = cubic ? Lc : L[i];
        s[i] = Li > 0.0f ? two_b / Li : 0.0f;
    }
    for (int64_t k = 0; k < n; ++k) {
        uint32_t q[3];
        for (int i = 0; i < 3; ++i) {
            float d = cent[3 * k + i] - lo[i];
            float x = d * s[i];
            float f = floorf(x);
            q[i] = f >= (float)qmax ? qmax : (uint32_t)f;
        }
        uint64_t m = 0;
        for (int b = 0; b < bits; ++b)
            for (int i = 0; i < 3; ++i) m |= (uint64_t)((q[i] >> b) & 1u) << (3 * b + i);
        code[k] = m;
    }
}

/* "radix sort": the result of a stable sort of (code, index) — the library qsort on
 * (code, original index) pairs, which is the definition of a stable order. */
typedef struct {
    uint64_t key;
    uint32_t idx;
} orc_kv;

static int kv_cmp(const void *a, const void *b) {
    const orc_kv *x = (const orc_kv *)a, *y = (const orc_kv *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

void orc_stable_sort(const uint64_t *keys, const uint32_t *vals, int64_t n, uint64_t *skeys, uint32_t *svals) {
    orc_kv *kv = (orc_kv *)malloc(sizeof(orc_kv) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        kv[i].key = keys[i];
        kv[i].idx = (uint32_t)i;
    }
    qsort(kv, (size_t)n, sizeof(orc_kv), kv_cmp);
    for (int64_t i = 0; i < n; ++i) {
        skeys[i] = kv[i].key;
        svals[i] = vals ? vals[kv[i].idx] : kv[i].idx;
    }
    free(kv);
}

/* Eq. 6: LCP of sorted codes; duplicates broken by the sorted position appended as
 * low-order bits (R7). lambda(i,j) = number of leading equal bits of code_i||i and code_j||j. */
static inline int lcp(const uint64_t *k, int64_t i, int64_t j) {
    if (k[i] != k[j]) return __builtin_clzll(k[i] ^ k[j]);
    return 64 + __builtin_clz((uint32_t)i ^ (uint32_t)j);
}

/* Binary radix tree over n >= 2 sorted keys, by its definition: a node covering [f, l] splits
 * after the last position g whose key shares more than LCP(f, l) leading bits with key f. Node
 * numbering (Karras 2012, the non-recursive construction P:125 reads as — R7): root = 0; the left
 * child of a node split at g is leaf g if g == f else internal g; the right child is leaf g+1 if
 * g+1 == l else internal g+1. Children encode leaf j as ~j (= -1-j). Returns 0 on success. */
int orc_radix_tree(const uint64_t *k, int64_t n, int32_t *child, int32_t *range) {
    if (n < 2) return 0;
    int64_t *stk = (int64_t *)malloc(sizeof(int64_t) * 3 * (size_t)(n + 64));
    int64_t sp = 0;
    stk[sp++] = 0, stk[sp++] = 0, stk[sp++] = n - 1;
    int64_t made = 0;
    while (sp) {
        int64_t l = stk[--sp], f = stk[--sp], id = stk[--sp];
        int lam = lcp(k, f, l);
        int64_t g = f;
        while (g + 1 < l && lcp(k, f, g + 1) > lam) ++g;
        range[2 * id] = (int32_t)f;
        range[2 * id + 1] = (int32_t)l;
        child[2 * id] = g == f ? ~(int32_t)g : (int32_t)g;
        child[2 * id + 1] = g + 1 == l ? ~(int32_t)(g + 1) : (int32_t)(g + 1);
        ++made;
        if (g != f) stk[sp++] = g, stk[sp++] = f, stk[sp++] = g;
        if (g + 1 != l) stk[sp++] = g + 1, stk[sp++] = g + 1, stk[sp++] = l;
    }
    free(stk);
    return made == n - 1 ? 0 : 1;
}

/* Eq. 7: B(n) = B(n_left) U B(n_right); leaf j bounds = the exact float AABB of
 * triangle perm[j]. Boxes are (lo.x, lo.y, lo.z, hi.x, hi.y, hi.z). Computed post-order. */
void orc_refit(const float *verts, const int32_t *tris, const uint32_t *perm, int64_t n, const int32_t *child,
               float *leaf_box, float *node_box) {
    for (int64_t j = 0; j < n; ++j) {
        int64_t k = perm[j];
        for (int i = 0; i < 3; ++i) {
            float a = verts[3 * (int64_t)tris[3 * k] + i], b = verts[3 * (int64_t)tris[3 * k + 1] + i];
            float c = verts[3 * (int64_t)tris[3 * k + 2] + i];
            leaf_box[6 * j + i] = fminf(a, fminf(b, c));
            leaf_box[6 * j + 3 + i] = fmaxf(a, fmaxf(b, c));
        }
    }
    if (n < 2) return;
    /* pre-order list, then reverse it so children come before parents */
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n - 1));
    int32_t *stk = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 64));
    int64_t no = 0, sp = 0;
    stk[sp++] = 0;
    while (sp) {
        int32_t id = stk[--sp];
        order[no++] = id;
        for (int s = 0; s < 2; ++s)
            if (child[2 * id + s] >= 0) stk[sp++] = child[2 * id + s];
    }
    for (int64_t q = no - 1; q >= 0; --q) {
        int32_t id = order[q];
        const float *b[2];
        for (int s = 0; s < 2; ++s) {
            int32_t c = child[2 * id + s];
            b[s] = c >= 0 ? node_box + 6 * (int64_t)c : leaf_box + 6 * (int64_t)(~c);
        }
        for (int i = 0; i < 3; ++i) {
            node_box[6 * (int64_t)id + i] = fminf(b[0][i], b[1][i]);
            node_box[6 * (int64_t)id + 3 + i] = fmaxf(b[0][3 + i], b[1][3 + i]);
        }
    }
    free(order);
    free(stk);
}

/* ------------------------------------------------------------------------------------------ */
/* Point-cloud metrics of §V-A (SPEC evalkit S:527-545): for each query point the exact   */
/* nearest neighbour in a reference cloud by the naive O(m n) scan, Euclidean distance in double, */
/* ties to the smaller index. Chamfer / precision / recall / F-score are formed from these        */
/* distances in oracle/__init__.py (reading R23).                                                 */
/* ------------------------------------------------------------------------------------------ */
void orc_nearest(const float *pts, int64_t n, const float *q, int64_t m, double *dist, int32_t *idx) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(orc_get_threads())
    for (int64_t i = 0; i < m; ++i) {
        double qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
        double best = INFINITY;
        int32_t bi = -1;
        for (int64_t j = 0; j < n; ++j) {
            double dx = (double)pts[3 * j] - qx, dy = (double)pts[3 * j + 1] - qy, dz = (double)pts[3 * j + 2] - qz;
            double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < best) {
                best = d2;
                bi = (int32_t)j;
            }
        }
        dist[i] = sqrt(best);
        idx[i] = bi;
    }
}
