/*
 * rsi_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for segment x triangle-mesh
 * intersection (arXiv 2305.01867).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2305_01867_b200/ and it never imports or links it.
 *
 * What it computes (PAPER.md = P:n, SPEC.md = S:n):
 *   - Problem statement: N_r segments l_i = (r_i^start, r_i^end) against a
 *     mesh of N_t triangles t_j = [t_j1, t_j2, t_j3] over vertices {v_n}
 *     (section 1 "Background").
 *   - The method (BVH + Moller-Trumbore) only prunes; its result is by
 *     definition the EXHAUSTIVE search "comparing N_t triangles with N_r rays"
 *     (P:13).  So this oracle loops over every (ray, triangle) pair.
 *   - Each pair uses the Moller-Trumbore test ([moller1997fast]) in
 *     double precision (the paper's USE_DOUBLE_PRECISION_MOLLER option)
 *     in the fixed operation order of SURVEY.md 8(c).  Build with
 *     -O2 -ffp-contract=off and no fast-math so each * and + rounds once.
 *   - Modes:
 *       boolean         hit[i] = exists j with hit(i,j)
 *       barycentric     nearest hit: lexicographic min of (t, j) over hits;
 *                       tri = j, t, dist = t*|d|, point = O + t*d
 *       intercept_count number of unique intersections: sort hit t
 *                       ascending, count = 1 + #{k : t_(k+1) - t_(k) > tau}
 *                       (single linkage on t; reading R4 in DESIGN.md)
 *   - Readings where the paper is silent:
 *       closed triangle (edge / vertex hits count), closed t in [0,1],
 *       det == 0 exactly -> no hit, ties of nearest -> lowest triangle id,
 *       barycentric u weights v[t_j2], v weights v[t_j3].
 *   - Per-ray ambiguity flags (north_star: "rays the oracle flags as within
 *     1e-6 (relative) of a triangle edge or vertex ... are counted and
 *     reported"), bits:
 *       RSI_ORACLE_FLAG_E  1  near edge/vertex
 *       RSI_ORACLE_FLAG_T  2  endpoint touch (t near 0 or 1)
 *       RSI_ORACLE_FLAG_P  4  near-parallel and near the triangle
 *       RSI_ORACLE_FLAG_B  8  nearest-hit tie within delta
 *       RSI_ORACLE_FLAG_D 16  dedup ambiguity (0.1 tau < |t_a - t_b| <= 10 tau)
 *
 * Pins (tests/test_oracle.py, all -m "not gpu"): the Fig. 3 worked example
 * (P:194-200), exact-rational plane-clip referee on tiny random
 * meshes, closed-form unit-cube clipping, closed-mesh parity, canopy counts.
 * PARITY UNPINNED: the dedup threshold tau of intercept_count itself (the
 * paper never defines "unique intersections"; reading R4) --
 * the single-linkage rule is pinned (layer counts, shared-edge merges), the
 * value 1e-6 is a convention.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RSI_ORACLE_FLAG_E 1u
#define RSI_ORACLE_FLAG_T 2u
#define RSI_ORACLE_FLAG_P 4u
#define RSI_ORACLE_FLAG_B 8u
#define RSI_ORACLE_FLAG_D 16u

/* ---- vector helpers: the SURVEY 8(c) operation order, nothing else ---- */

static void vsub(const double a[3], const double b[3], double r[3])
{
    r[0] = a[0] - b[0];
    r[1] = a[1] - b[1];
    r[2] = a[2] - b[2];
}

/* cross(x,y) = (x.y*y.z - x.z*y.y, x.z*y.x - x.x*y.z, x.x*y.y - x.y*y.x) */
static void vcross(const double x[3], const double y[3], double r[3])
{
    r[0] = x[1] * y[2] - x[2] * y[1];
    r[1] = x[2] * y[0] - x[0] * y[2];
    r[2] = x[0] * y[1] - x[1] * y[0];
}

/* dot(x,y) = (x.x*y.x + x.y*y.y) + x.z*y.z */
static double vdot(const double x[3], const double y[3])
{
    return (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2];
}

/*
 * Moller-Trumbore segment-triangle test in double.
 * Inputs are the fp32 values promoted exactly to double.
 * Returns 1 on hit and writes out[0..3] = (t, u, v, det_signed); 0 on miss.
 * On miss out[] still receives (nt/det, nu/det, nv/det, det) when det != 0
 * (used only for flags), or det = 0.
 */
int rsi_oracle_mt(const double O[3], const double E[3], const double A[3],
                  const double B[3], const double C[3], double out[4])
{
    double d[3], e1[3], e2[3], s[3], p[3], q[3];
    vsub(E, O, d);
    vsub(B, A, e1);
    vsub(C, A, e2);
    vsub(O, A, s);
    vcross(d, e2, p);
    double det = vdot(e1, p);
    vcross(s, e1, q);
    double nu = vdot(s, p);
    double nv = vdot(d, q);
    double nt = vdot(e2, q);
    out[3] = det;
    if (det == 0.0) {
        out[0] = out[1] = out[2] = 0.0;
        return 0;
    }
    out[0] = nt / det;
    out[1] = nu / det;
    out[2] = nv / det;
    if (det < 0.0) {
        det = -det;
        nu = -nu;
        nv = -nv;
        nt = -nt;
    }
    return (nu >= 0.0) && (nv >= 0.0) && ((nu + nv) <= det) && (nt >= 0.0) && (nt <= det);
}

/* ---- ambiguity flags (reporting only; never used to excuse a result) ---- */

static double vnorm(const double x[3]) { return sqrt(vdot(x, x)); }

static unsigned pair_flags(const double O[3], const double E[3], const double A[3],
                           const double B[3], const double C[3], const double mt[4],
                           double delta)
{
    double d[3], e1[3], e2[3], n[3];
    vsub(E, O, d);
    vsub(B, A, e1);
    vsub(C, A, e2);
    vcross(e1, e2, n);
    double dn = vnorm(d), nn = vnorm(n);
    if (dn == 0.0) return 0u; /* zero-length segment: det == 0, never hits */
    double sin_theta = (nn > 0.0) ? fabs(mt[3]) / (dn * nn) : 0.0;
    if (sin_theta > delta) {
        double t = mt[0], u = mt[1], v = mt[2], w = 1.0 - u - v;
        double mn = fmin(u, fmin(v, w));
        unsigned f = 0u;
        if (mn >= -delta && t >= -delta && t <= 1.0 + delta) {
            if (mn <= delta) f |= RSI_ORACLE_FLAG_E;
            if (fabs(t) <= delta || fabs(1.0 - t) <= delta) f |= RSI_ORACLE_FLAG_T;
        }
        return f;
    }
    /* near-parallel (or degenerate triangle): flag when the segment comes
     * within tol of the triangle's plane and AABBs overlap within tol */
    double e3[3];
    vsub(C, B, e3);
    double diam = fmax(vnorm(e1), fmax(vnorm(e2), vnorm(e3)));
    double tol = delta * fmax(dn, diam);
    if (nn > 0.0) {
        double sO[3], sE[3];
        vsub(O, A, sO);
        vsub(E, A, sE);
        double a = vdot(n, sO) / nn, b = vdot(n, sE) / nn;
        double dist = (a * b <= 0.0) ? 0.0 : fmin(fabs(a), fabs(b));
        if (dist > tol) return 0u;
    }
    for (int k = 0; k < 3; ++k) {
        double slo = fmin(O[k], E[k]), shi = fmax(O[k], E[k]);
        double tlo = fmin(A[k], fmin(B[k], C[k])) - tol;
        double thi = fmax(A[k], fmax(B[k], C[k])) + tol;
        if (shi < tlo || slo > thi) return 0u;
    }
    return RSI_ORACLE_FLAG_P;
}

static int cmp_double(const void* a, const void* b)
{
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/*
 * Validation (SPEC S:31-41 readings): every index in [0, N_v).
 * Returns 0 on success, -1 on a bad index.
 */
static int check_indices(const int32_t* T, int64_t nt, int64_t nv)
{
    for (int64_t j = 0; j < 3 * nt; ++j)
        if (T[j] < 0 || (int64_t)T[j] >= nv) return -1;
    return 0;
}

/*
 * Exhaustive oracle, all three modes at once.
 *   V [nv,3] f32, T [nt,3] i32, S/E [nr,3] f32 segment start/end.
 *   tau: dedup tolerance in t units (intercept_count), delta: flag band.
 *   Outputs (any may be NULL):
 *     hit[nr] u8, count[nr] i32, tri[nr] i32 (-1 = miss),
 *     t[nr], dist[nr] f64, point[nr*3] f64 (NaN on miss), flags[nr] u8,
 *     nhits_raw[nr] i32 (number of (ray, triangle) hits before dedup).
 * Returns 0, or -1 for an out-of-range triangle index.
 */
int rsi_oracle_run(const float* V, int64_t nv, const int32_t* T, int64_t nt,
                   const float* S, const float* E, int64_t nr,
                   double tau, double delta, int nthreads,
                   uint8_t* hit, int32_t* count, int32_t* tri, double* t_out,
                   double* dist_out, double* point_out, uint8_t* flags,
                   int32_t* nhits_raw)
{
    if (check_indices(T, nt, nv) != 0) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        int64_t cap = 64;
        double* ts = (double*)malloc((size_t)cap * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < nr; ++i) {
            double O[3] = {S[3 * i], S[3 * i + 1], S[3 * i + 2]};
            double Ee[3] = {E[3 * i], E[3 * i + 1], E[3 * i + 2]};
            int64_t nh = 0;
            int64_t best_j = -1;
            double best_t = 0.0;
            unsigned f = 0u;
            /* reading R12: a segment with a NaN/Inf coordinate is a miss */
            int finite = isfinite(O[0]) && isfinite(O[1]) && isfinite(O[2]) &&
                         isfinite(Ee[0]) && isfinite(Ee[1]) && isfinite(Ee[2]);
            for (int64_t j = 0; finite && j < nt; ++j) {
                const int32_t* tj = T + 3 * j;
                double A[3] = {V[3 * tj[0]], V[3 * tj[0] + 1], V[3 * tj[0] + 2]};
                double B[3] = {V[3 * tj[1]], V[3 * tj[1] + 1], V[3 * tj[1] + 2]};
                double C[3] = {V[3 * tj[2]], V[3 * tj[2] + 1], V[3 * tj[2] + 2]};
                double mt[4];
                int h = rsi_oracle_mt(O, Ee, A, B, C, mt);
                if (flags) f |= pair_flags(O, Ee, A, B, C, mt, delta);
                if (!h) continue;
                if (nh == cap) {
                    cap *= 2;
                    ts = (double*)realloc(ts, (size_t)cap * sizeof(double));
                }
                ts[nh++] = mt[0];
                /* lexicographic min of (t, j); j ascends so only strict < replaces */
                if (best_j < 0 || mt[0] < best_t) {
                    best_j = j;
                    best_t = mt[0];
                }
            }
            if (hit) hit[i] = (uint8_t)(nh > 0);
            if (nhits_raw) nhits_raw[i] = (int32_t)nh;
            double d[3];
            vsub(Ee, O, d);
            if (tri) tri[i] = (int32_t)best_j;
            if (best_j >= 0) {
                if (t_out) t_out[i] = best_t;
                if (dist_out) dist_out[i] = best_t * sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
                if (point_out)
                    for (int k = 0; k < 3; ++k) point_out[3 * i + k] = O[k] + best_t * d[k];
            } else {
                if (t_out) t_out[i] = NAN;
                if (dist_out) dist_out[i] = NAN;
                if (point_out)
                    for (int k = 0; k < 3; ++k) point_out[3 * i + k] = NAN;
            }
            if (nh > 1) qsort(ts, (size_t)nh, sizeof(double), cmp_double);
            int32_t c = 0;
            if (nh > 0) {
                c = 1;
                for (int64_t k = 0; k + 1 < nh; ++k)
                    if (ts[k + 1] - ts[k] > tau) ++c;
            }
            if (count) count[i] = c;
            if (flags) {
                /* B: another hit within delta of the nearest one */
                int nearest_seen = 0;
                for (int64_t k = 0; k < nh; ++k) {
                    if (ts[k] == best_t && !nearest_seen) {
                        nearest_seen = 1;
                        continue;
                    }
                    if (ts[k] - best_t <= delta) f |= RSI_ORACLE_FLAG_B;
                }
                /* D: a pair of hits whose gap is within a decade of tau */
                for (int64_t a = 0; a < nh; ++a)
                    for (int64_t b = a + 1; b < nh && ts[b] - ts[a] <= 10.0 * tau; ++b)
                        if (ts[b] - ts[a] > 0.1 * tau) f |= RSI_ORACLE_FLAG_D;
                flags[i] = (uint8_t)f;
            }
        }
        free(ts);
    }
    return 0;
}

/* Number of OpenMP threads a parallel region would use (for reporting). */
int rsi_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
