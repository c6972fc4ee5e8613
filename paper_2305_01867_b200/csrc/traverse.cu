// traverse.cu -- per-ray BVH traversal + Moller-Trumbore on sm_100a
// (SURVEY 8(a) rows A8 and A9).
//
// One thread per segment, persistent grid.  The default walk visits the
// 4-wide view of the binary tree (k_quads records: a greedy 4-cut of each
// node's subtree, 8-bit quantized boxes on a power-of-two grid, 64 B); every visit
// slab-tests its children conservatively, orders the hit ones near-first,
// keeps the next on a branch-free local stack (<= 288 entries: depth <= 95)
// and queues leaves for a warp-wide Moller-Trumbore phase.  The binary
// child-pair walk (RSI_*_QUAD=0) remains a build switch; the exact
// intercept_count re-pass (k_count_repass) walks the 4-wide records.
//
// Exactness.  Every discrete decision -- hit / miss,
// nearest-hit order, dedup merge -- is taken in fp32 only when a forward error
// bound certifies it; otherwise it is re-made by an fp64 "mirror" that repeats
// the oracle's operation order with correctly rounded
// __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn and no contraction, so it returns the
// oracle's exact double results.  This is the paper's
// USE_DOUBLE_PRECISION_MOLLER idea applied only where fp32 is unsure.
#include <cstdio>
#include <type_traits>

#include "rsi_internal.cuh"

namespace {

constexpr float kU = 5.9604644775390625e-08f;    // 2^-24, fp32 unit roundoff
constexpr float kFilt = 16.0f * kU;              // K = 16
constexpr float kTerr = 12.0f * kU;              // t forward-error constant
constexpr float kSlack = 4.76837158203125e-07f;  // 2^-21: slab-test slack factor
constexpr float kTiny = 1e-30f;                  // absolute floor (underflow)
constexpr float kOutTol = 4e-6f;                 // max certified |t error| for fp32 outputs
// Per-mode traversal configuration.  Measured on B200 (round 1, same box A/B):
// all three modes walk the compressed 4-wide cut records (64 B, 8-bit
// quantized boxes: half the L1 wavefronts of the binary child-pair walk, which
// was L1-data-pipe bound at 87 %) with a branch-free lane stack; once the quad
// visit was cheap, intercept_count also gained (-12 % sphere, -18 % terrain vs
// the binary walk with speculation).  The binary walk stays a build option.
#ifndef RSI_BOOL_QUAD
#define RSI_BOOL_QUAD 1
#endif
#ifndef RSI_BARY_QUAD
#define RSI_BARY_QUAD 1
#endif
#ifndef RSI_COUNT_QUAD
#define RSI_COUNT_QUAD 1
#endif
#ifndef RSI_BOOL_SMEM
#define RSI_BOOL_SMEM 0
#endif
#ifndef RSI_BARY_SMEM
#define RSI_BARY_SMEM 0
#endif
#ifndef RSI_COUNT_SMEM
#define RSI_COUNT_SMEM 0
#endif
constexpr bool kQuadCount = RSI_COUNT_QUAD;
// speculative walk on the 4-wide records (a lane with a pending leaf keeps
// walking): measured -2..-4 % barycentric, +3..5 % boolean with grandchild
// records; with greedy cuts barycentric +5 % sphere / -1 % terrain: off everywhere
#ifndef RSI_QSPEC_BOOL
#define RSI_QSPEC_BOOL 0
#endif
#ifndef RSI_QSPEC_COUNT
#define RSI_QSPEC_COUNT 0
#endif
#ifndef RSI_QSPEC_BARY
#define RSI_QSPEC_BARY 0
#endif
#ifndef RSI_BF_SMEM
#define RSI_BF_SMEM 0
#endif
// quad visits per traversal-phase iteration (the warp votes on leaving the
// phase every kVisits visits): measured per mode on the sphere and
// paper-terrain workloads -- 3 with min_trav 16 / 12 for boolean / barycentric
// (-1..-6 %), 1 for intercept_count (3: +9 %)
#ifndef RSI_VISITS_BOOL
#define RSI_VISITS_BOOL 4  // re-measured with the SAH subtrees: 3 -> 4 sphere -2.3 %, terrain -0.5 %; 6: +2.5 %
#endif
#ifndef RSI_VISITS_BARY
#define RSI_VISITS_BARY 4  // 3 -> 4: sphere -1.5 %, terrain 0; 6: +2 %
#endif
#ifndef RSI_VISITS_COUNT
#define RSI_VISITS_COUNT 1
#endif
#ifndef RSI_QC_SMEM
#define RSI_QC_SMEM 1  // barycentric only: -1.5 % (intercept_count +2 %, boolean neutral)
#endif
#ifndef RSI_SORT_ALL
#define RSI_SORT_ALL 1
#endif
constexpr int kNoRef = (int)0x80000000;  // "no child" (never a valid ref: ~slot > INT_MIN)
// tree depth <= 95: a root-to-leaf path has strictly increasing common-prefix
// lengths of the index-augmented key (<= 63 code bits under RSI_OPT_APETREI,
// 30 otherwise, + <= 31 levels of index bits for duplicate codes).  Binary
// walk: one entry per level; quad walk: <= 48 visits x 3 pushes (grandchild
// records) or <= 95 x 3 (greedy cuts: a member may be one level down).  Entries
// beyond the depth a ray reaches are never touched (no traffic).
constexpr int kStackBinary = 96;
constexpr int kStackQuad = RSI_QUAD_GREEDY ? 288 : 144;
// intercept_count hits held per ray before the exact re-pass: 4 (measured: a
// 6 KB instead of 12 KB shared-memory list per CTA and a shorter certification
// loop; with 7 CTAs per SM -8 % sphere, -16 % folded terrain vs 8 at 6 CTAs;
// 0.13 % of the sphere's segments take the re-pass)
#ifndef RSI_COUNT_CAP
#define RSI_COUNT_CAP 4
#endif
constexpr int kCountCap = RSI_COUNT_CAP;
#ifndef RSI_BOOL_MINB
#define RSI_BOOL_MINB 8
#endif
// resident 128-thread CTAs per SM (register budget: 8 -> 64, 6 -> 80 registers);
// measured: barycentric -8 % at 8 vs 6, intercept_count +4 % at 8 vs 6
#ifndef RSI_BARY_MINB
#define RSI_BARY_MINB 8
#endif
#ifndef RSI_COUNT_MINB
#define RSI_COUNT_MINB 7  // 72 registers; round 2: 8 CTAs +6..13 %, 6 CTAs +7..8 %
#endif
// k_trace block size: with the top-of-tree cache, one CTA per SM shares the
// image (1024 threads at <= 64 registers for boolean, 768 at <= 80 otherwise)
template <int MODE>
__host__ __device__ constexpr int trace_threads() {
    return 128;
}
#ifndef RSI_CHUNK
#define RSI_CHUNK 64
#endif
constexpr int kChunk = RSI_CHUNK;  // rays a warp takes from the global dispenser at once

enum { MT_MISS = 0, MT_HIT = 1, MT_UNSURE = 2 };

struct Ray {
    float ox, oy, oz;  // start (r^start)
    float ex, ey, ez;  // end (r^end), kept exactly for the fp64 mirror
    float dx, dy, dz;  // d = end - start (fp32)
    float ix, iy, iz;  // slab: 1/d per axis (0 on degenerate axes)
    float lx, ly, lz;  // slab offsets applied to the box's lo plane
    float hx, hy, hz;  // slab offsets applied to the box's hi plane
    uint32_t mx, my, mz;  // 4-wide walk: 0xffffffff where inv < 0 (picks the near-plane bytes)
};

// Per-axis slab setup.  t = fma(plane, inv, -off) approximates (plane - o)/d;
// the slack (2^-21 * (1 + |o/d|)) exceeds the fp32 error of that expression
// for |t| <= ~1, and is applied so the computed entry t is never later and the
// exit t never earlier than the exact ones: the test never rejects a box the
// exact segment touches.  |d| < 1e-30 (incl. 0): the axis imposes no constraint.
// inv is MUFU.RCP (rcp.approx.ftz, relative error e <= 2^-23 -- measured max
// 2^-23.28 over 1.2e9 random normal inputs on a B200; one instruction
// instead of the ~24 of an IEEE division): every plane term is multiplied by
// the same inv, so the computed t is t_exact (1 + e) plus the roundings below;
// |t| e + 2^-24 |t| <= 1.5 * 2^-23 for |t| <= 1, inside the 2^-21 of slack.
// A result flushed to zero (|d| >= 2^126) leaves the axis unconstrained.
// The 4-wide walk evaluates t as fma(q', s*inv, fma(pm, inv, -off)) (see the
// visit in k_trace); its extra rounding, <= 2^-24 |pm * inv - off|, is covered
// by `qext` * |inv| in the slack (qext = Pmax / 4 with Pmax >= every |pm|,
// since 2^-21 / 4 = 2 * 2^-24), and axes whose |inv| falls outside
// [lim_lo, lim_hi] are left unconstrained (conservative) so that s * inv stays
// an exact normal float and no term can overflow.
#ifndef RSI_SLAB_BF
#define RSI_SLAB_BF 1  // branch-free ray setup (selects instead of the nested branches): sphere 1e7
                       // boolean -0.7 %, intercept_count -2.5 %, barycentric 0; paper terrain +-1 %
#endif
__device__ __forceinline__ void slab_axis(float o, float d, float& inv, float& offlo, float& offhi,
                                          float qext = 0.0f, float lim_lo = 0.0f, float lim_hi = INFINITY) {
    if (RSI_SLAB_BF) {  // the same values as the branches below, computed unconditionally
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
        const float ai = fabsf(r);
        const float oinv = o * r;
        const float slack = kSlack * fmaf(qext, ai, 1.0f + fabsf(oinv));
        const float sg = r > 0.0f ? slack : -slack;
        const float a = oinv + sg, b = oinv - sg;
        const bool ok = fabsf(d) >= 1e-30f && ai >= lim_lo && ai <= lim_hi && ai > 0.0f && isfinite(a) && isfinite(b);
        inv = ok ? r : 0.0f;
        offlo = ok ? a : INFINITY;
        offhi = ok ? b : -INFINITY;
        return;
    }
    if (fabsf(d) >= 1e-30f) {
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(d));
        const float ai = fabsf(inv);
        if (ai >= lim_lo && ai <= lim_hi && ai > 0.0f) {
            float oinv = o * inv;
            float slack = kSlack * fmaf(qext, ai, 1.0f + fabsf(oinv));
            float sg = inv > 0.0f ? slack : -slack;
            offlo = oinv + sg;
            offhi = oinv - sg;
            if (isfinite(offlo) && isfinite(offhi)) return;
        }
    }
    inv = 0.0f;
    offlo = INFINITY;
    offhi = -INFINITY;
}

__device__ __forceinline__ float ld_stream(const float* p) {
#if RSI_STREAM_NOALLOC
    float v;
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

// Returns false for rays that cannot hit: zero length or a non-finite coordinate
// (reading R12).  `nonfinite` is set for the latter.
// kNearFar: lx/hx become the offsets of each axis's NEAR / FAR plane (lo / hi
// for inv >= 0, hi / lo for inv < 0) for the octant-selected quad slab test.
// Ray setup from r.ox .. r.ez (already loaded); see load_ray.
template <bool kNearFar = false>
__device__ __forceinline__ bool setup_ray(Ray& r, bool& nonfinite, float qext = 0.0f, float lim_lo = 0.0f,
                                          float lim_hi = INFINITY) {
    nonfinite = !(isfinite(r.ox) && isfinite(r.oy) && isfinite(r.oz) && isfinite(r.ex) && isfinite(r.ey) &&
                  isfinite(r.ez));
    r.dx = r.ex - r.ox;
    r.dy = r.ey - r.oy;
    r.dz = r.ez - r.oz;
    slab_axis(r.ox, r.dx, r.ix, r.lx, r.hx, qext, lim_lo, lim_hi);
    slab_axis(r.oy, r.dy, r.iy, r.ly, r.hy, qext, lim_lo, lim_hi);
    slab_axis(r.oz, r.dz, r.iz, r.lz, r.hz, qext, lim_lo, lim_hi);
    if (kNearFar) {
        r.mx = (uint32_t)(__float_as_int(r.ix) >> 31);
        r.my = (uint32_t)(__float_as_int(r.iy) >> 31);
        r.mz = (uint32_t)(__float_as_int(r.iz) >> 31);
        if (r.ix < 0.0f) { const float t = r.lx; r.lx = r.hx; r.hx = t; }
        if (r.iy < 0.0f) { const float t = r.ly; r.ly = r.hy; r.hy = t; }
        if (r.iz < 0.0f) { const float t = r.lz; r.lz = r.hz; r.hz = t; }
    }
    return !nonfinite && !(r.dx == 0.0f && r.dy == 0.0f && r.dz == 0.0f);
}

// Returns false for rays that cannot hit: zero length or a non-finite coordinate
// (reading R12).  `nonfinite` is set for the latter.
// kNearFar: lx/hx become the offsets of each axis's NEAR / FAR plane (lo / hi
// for inv >= 0, hi / lo for inv < 0) for the octant-selected quad slab test.
template <bool kNearFar = false>
__device__ __forceinline__ bool load_ray(Ray& r, const float* __restrict__ S, const float* __restrict__ E,
                                         int64_t i, bool& nonfinite, float qext = 0.0f, float lim_lo = 0.0f,
                                         float lim_hi = INFINITY) {
    // the segment stream is read once: do not let it displace tree nodes in L1
    r.ox = ld_stream(S + 3 * i);
    r.oy = ld_stream(S + 3 * i + 1);
    r.oz = ld_stream(S + 3 * i + 2);
    r.ex = ld_stream(E + 3 * i);
    r.ey = ld_stream(E + 3 * i + 1);
    r.ez = ld_stream(E + 3 * i + 2);
    return setup_ray<kNearFar>(r, nonfinite, qext, lim_lo, lim_hi);
}

// Next-segment prefetch (RSI_RAY_PREFETCH): a lane claims the id of its NEXT
// segment when it starts the current one and copies that segment's six floats
// into its shared-memory column with cp.async (no registers held), so the
// refill that starts it reads shared memory instead of waiting for HBM.
// Measured and rejected (1e7 segments, query): sphere boolean 1.315 -> 1.347 ms,
// barycentric 2.07 -> 2.20, intercept_count 3.31 -> 3.55; paper terrain
// +6 / +9 / +11 % -- the 3 KB per CTA of columns come out of the L1 the
// records live in, and the claim/commit logic adds spills (ray setup's HBM
// wait, 7 % of the stall samples, is hidden by the other warps anyway).
#ifndef RSI_RAY_PF_L1
#define RSI_RAY_PF_L1 1  // intercept_count: L1 prefetch of the chunk's next segments at each refill
                         // (sphere -2 %, terrain -1 %; boolean +1 %, barycentric +2 %: count only)
#endif
#ifndef RSI_RAY_PREFETCH
#define RSI_RAY_PREFETCH 0
#endif
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

// Conservative segment/box overlap on [0, tclip]; tnear is the (lowered) entry t.
__device__ __forceinline__ bool slab(const Ray& r, float lox, float hix, float loy, float hiy, float loz, float hiz,
                                     float tclip, float& tnear) {
    float tx1 = fmaf(lox, r.ix, -r.lx), tx2 = fmaf(hix, r.ix, -r.hx);
    float ty1 = fmaf(loy, r.iy, -r.ly), ty2 = fmaf(hiy, r.iy, -r.hy);
    float tz1 = fmaf(loz, r.iz, -r.lz), tz2 = fmaf(hiz, r.iz, -r.hz);
    tnear = fmaxf(fmaxf(fminf(tx1, tx2), fminf(ty1, ty2)), fmaxf(fminf(tz1, tz2), 0.0f));
    float tfar = fminf(fminf(fmaxf(tx1, tx2), fmaxf(ty1, ty2)), fminf(fmaxf(tz1, tz2), tclip));
    return tnear <= tfar;
}

// ---------------------------------------------------------------- fp32 MT + error filter
// Same algebra as the oracle (p = d x e2, det = e1.p, q = s x e1, nu = s.p,
// nv = d.q, nt = e2.q).  Each quantity X has a "shadow" M_X (the same
// expression on absolute values with + for -): |fl(X) - X| <= ~10u M_X, so a
// sign test on X is certain when |X| > 16u M_X (+ an underflow floor).
// Returns MT_MISS / MT_HIT (with t and a bound et on |t - t_exact|) / MT_UNSURE.
#ifndef RSI_MT_RCP
#define RSI_MT_RCP 1
#endif
#ifndef RSI_LEAF_SEL
#define RSI_LEAF_SEL 1  // boolean: leaf-phase outcome by selects instead of a branch chain (sphere -1.5 %,
                        // terrain -0.7 %; barycentric +1.5 %, intercept_count +2.5 %: boolean only)
#endif
#ifndef RSI_FAST_NORM
#define RSI_FAST_NORM 1  // |d| by one sqrt unless |d|^2 leaves [1e-30, 1e30] (then norm3df's scaling)
#endif
__device__ __forceinline__ int mt32(const Ray& r, const float4& A, const float4& B, const float4& C, float& t,
                                    float& et) {
    const float e1x = B.x - A.x, e1y = B.y - A.y, e1z = B.z - A.z;
    const float e2x = C.x - A.x, e2y = C.y - A.y, e2z = C.z - A.z;
    const float px = r.dy * e2z - r.dz * e2y, py = r.dz * e2x - r.dx * e2z, pz = r.dx * e2y - r.dy * e2x;
    const float adx = fabsf(r.dx), ady = fabsf(r.dy), adz = fabsf(r.dz);
    const float Px = ady * fabsf(e2z) + adz * fabsf(e2y), Py = adz * fabsf(e2x) + adx * fabsf(e2z),
                Pz = adx * fabsf(e2y) + ady * fabsf(e2x);
    const float det = e1x * px + e1y * py + e1z * pz;
    const float Mdet = fabsf(e1x) * Px + fabsf(e1y) * Py + fabsf(e1z) * Pz;
    if (!(fabsf(det) > fmaf(kFilt, Mdet, kTiny))) return MT_UNSURE;  // near-parallel / NaN
    const float sg = det < 0.0f ? -1.0f : 1.0f;
    const float sx = r.ox - A.x, sy = r.oy - A.y, sz = r.oz - A.z;
    const float asx = fabsf(sx), asy = fabsf(sy), asz = fabsf(sz);
    const float nu = sg * (sx * px + sy * py + sz * pz);
    const float Mu = asx * Px + asy * Py + asz * Pz;
    const float bu = fmaf(kFilt, Mu, kTiny);
    if (nu < -bu) return MT_MISS;
    const float qx = sy * e1z - sz * e1y, qy = sz * e1x - sx * e1z, qz = sx * e1y - sy * e1x;
    const float Qx = asy * fabsf(e1z) + asz * fabsf(e1y), Qy = asz * fabsf(e1x) + asx * fabsf(e1z),
                Qz = asx * fabsf(e1y) + asy * fabsf(e1x);
    const float nv = sg * (r.dx * qx + r.dy * qy + r.dz * qz);
    const float Mv = adx * Qx + ady * Qy + adz * Qz;
    const float bv = fmaf(kFilt, Mv, kTiny);
    if (nv < -bv) return MT_MISS;
    const float adet = fabsf(det);
    const float w = adet - nu - nv;
    const float bw = fmaf(kFilt, Mdet + Mu + Mv, kTiny);
    if (w < -bw) return MT_MISS;
    const float nt = sg * (e2x * qx + e2y * qy + e2z * qz);
    const float Mt = fabsf(e2x) * Qx + fabsf(e2y) * Qy + fabsf(e2z) * Qz;
    const float bt = fmaf(kFilt, Mt, kTiny);
    if (nt < -bt) return MT_MISS;
    const float z = adet - nt;
    const float bz = fmaf(kFilt, Mdet + Mt, kTiny);
    if (z < -bz) return MT_MISS;
    if (nu > bu && nv > bv && w > bw && nt > bt && z > bz) {
#if RSI_MT_RCP
        // one approximate reciprocal instead of two IEEE divisions: rcp.approx
        // (relative error <= 2^-23, see slab_axis) times nt adds <= 2.5u |t| <=
        // 2.5u (a certified hit has 0 <= t <= 1) to t, covered by the constant
        // term (3u -> 6u); the bound's own roundings (< 4u relative of a 12u
        // term) by kTerr 12u -> 13u.  adet > 1e-30 here: a normal float.
        float ra;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(adet));
        t = nt * ra;
        et = fmaf(kTerr + kU, (Mt + Mdet) * ra, 6.0f * kU);
#else
        t = __fdiv_rn(nt, adet);
        et = kTerr * (Mt + Mdet) / adet + 3.0f * kU;
#endif
        return MT_HIT;
    }
    return MT_UNSURE;
}

// ---------------------------------------------------------------- fp64 mirror
// Exactly the oracle's operation order (oracle/rsi_oracle.c rsi_oracle_mt,
// SURVEY 8(c)); each * and +/- is a separately rounded IEEE double op.
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

__device__ __noinline__ int mt64(const Ray& r, const float4 A, const float4 B, const float4 C, double* t_out) {
    const double Ox = r.ox, Oy = r.oy, Oz = r.oz;
    const double dx = ds((double)r.ex, Ox), dy = ds((double)r.ey, Oy), dz = ds((double)r.ez, Oz);
    const double Ax = A.x, Ay = A.y, Az = A.z;
    const double e1x = ds(B.x, Ax), e1y = ds(B.y, Ay), e1z = ds(B.z, Az);
    const double e2x = ds(C.x, Ax), e2y = ds(C.y, Ay), e2z = ds(C.z, Az);
    const double sx = ds(Ox, Ax), sy = ds(Oy, Ay), sz = ds(Oz, Az);
    const double px = ds(dm(dy, e2z), dm(dz, e2y));
    const double py = ds(dm(dz, e2x), dm(dx, e2z));
    const double pz = ds(dm(dx, e2y), dm(dy, e2x));
    double det = da(da(dm(e1x, px), dm(e1y, py)), dm(e1z, pz));
    const double qx = ds(dm(sy, e1z), dm(sz, e1y));
    const double qy = ds(dm(sz, e1x), dm(sx, e1z));
    const double qz = ds(dm(sx, e1y), dm(sy, e1x));
    double nu = da(da(dm(sx, px), dm(sy, py)), dm(sz, pz));
    double nv = da(da(dm(dx, qx), dm(dy, qy)), dm(dz, qz));
    double nt = da(da(dm(e2x, qx), dm(e2y, qy)), dm(e2z, qz));
    if (det == 0.0) return 0;
    if (t_out) *t_out = __ddiv_rn(nt, det);
    if (det < 0.0) {
        det = -det;
        nu = -nu;
        nv = -nv;
        nt = -nt;
    }
    return (nu >= 0.0) && (nv >= 0.0) && (da(nu, nv) <= det) && (nt >= 0.0) && (nt <= det);
}

#ifndef RSI_SPEC
#define RSI_SPEC 1
#endif
#ifndef RSI_LDG256
#define RSI_LDG256 1
#endif
// 256-bit read-only global load (sm_100: LDG.E.ENL2.256): one L1 wavefront per
// lane-line instead of two for a pair of 128-bit loads.
__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
#if RSI_LDG256
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
#else
    a = __ldg(p);
    b = __ldg(p + 1);
#endif
}

// L1 eviction priority of the triangle / 4-wide record fetches (RSI_TRI_L1,
// RSI_Q_L1): 0 default, 1 L1::no_allocate, 2 L1::evict_first, 3 L1::evict_last
#ifndef RSI_TRI_L1
#define RSI_TRI_L1 1  // L1::no_allocate: sphere -1 %, terrain -0.5 % (records keep L1)
#endif
#ifndef RSI_Q_L1
#define RSI_Q_L1 0
#endif
#define RSI_LDG256_HINT(hint)                                                                  \
    asm("ld.global.nc" hint ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                          \
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) \
        : "l"(p))
template <int kHint>
__device__ __forceinline__ void ldg256h(const float4* p, float4& a, float4& b) {
    if constexpr (kHint == 1) RSI_LDG256_HINT(".L1::no_allocate");
    else if constexpr (kHint == 2) RSI_LDG256_HINT(".L1::evict_first");
    else if constexpr (kHint == 3) RSI_LDG256_HINT(".L1::evict_last");
    else ldg256(p, a, b);
}
#undef RSI_LDG256_HINT

// triangle slot k: 64 B (4 x float4, the last one padding) for two 256-bit loads
__device__ __forceinline__ void load_tri(const float4* __restrict__ tris, int k, float4& A, float4& B, float4& C) {
    if (kTriF4 == 3) {
        const float4* t = tris + 3 * (int64_t)k;
        A = __ldg(t);
        B = __ldg(t + 1);
        C = __ldg(t + 2);
    } else {
        float4 pad;
        ldg256h<RSI_TRI_L1>(tris + 4 * k, A, B);
        ldg256h<RSI_TRI_L1>(tris + 4 * k + 2, C, pad);
    }
}

// Per-thread counters of rare events, reduced per warp at kernel end.
struct Stats {
    unsigned c[ST_WORDS] = {};
    __device__ __forceinline__ void add(int k, unsigned v = 1) { c[k] += v; }
    unsigned boxes = 0, mts = 0;  // RSI_OPT_COUNTERS only
};

// Decide one (ray, leaf) pair: MT_MISS, or MT_HIT with either (t32, et) or an
// exact t64 (is64 = true).
template <bool kFP64>
__device__ __forceinline__ int decide(const Ray& r, const float4& A, const float4& B,
                                      const float4& C, float& t32, float& et, double& t64, bool& is64, Stats& st) {
    if (!kFP64) {
        int s = mt32(r, A, B, C, t32, et);
        if (s != MT_UNSURE) {
            is64 = false;
            return s;
        }
        st.add(ST_FP64_PAIRS);
    }
    is64 = true;
    return mt64(r, A, B, C, &t64) ? MT_HIT : MT_MISS;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// L2 cache policy for the barycentric output stores (RSI_OUT_HINT: 1 evict_last,
// 2 evict_unchanged, 3 evict_first, 0 none).  Measured (sphere, 1e7): DRAM
// bytes per launch 975 / 820 / 944 / 847 MB for none / 1 / 2 / 3; time
// 2.358 / 2.332 / 2.332 / 2.336 ms.
#ifndef RSI_OUT_HINT
#define RSI_OUT_HINT 1
#endif
__device__ __forceinline__ uint64_t out_policy() {
    uint64_t pol = 0;
#if RSI_OUT_HINT == 1
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#elif RSI_OUT_HINT == 2
    asm("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
#elif RSI_OUT_HINT == 3
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}
__device__ __forceinline__ void st_hint(float* ptr, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(v), "l"(pol) : "memory");
}

// ---------------------------------------------------------------- per-mode ray state
// Each mode keeps its per-ray result state; leaf() returns true when the ray
// can stop (boolean any-hit, intercept_count register overflow).
enum { MODE_BOOL = 0, MODE_BARY = 1, MODE_COUNT = 2 };

struct TraceParams {
    const float4* nodes;
    const float4* quads;
    const float4* top;   // top-of-tree image of the 4-wide records [4 * kQTop] (count: scratch[SCR_NTOP])
    const float4* tris;
    const float* S;
    const float* E;
    int64_t n;
    uint8_t* hit;
    int32_t* tri;
    float* t;
    float* dist;
    float* point;
    int32_t* count;
    double tau;
    int32_t* ovf_list;
    uint32_t* scratch;
    unsigned long long* stats;
    unsigned long long* counter;  // persistent-grid ray dispenser
    int min_trav;           // leave the traversal phase when fewer lanes still search
    uint32_t magic;         // 0x47000000 (float 2^15)
};

template <int MODE>
struct ModeState;

template <>
struct ModeState<MODE_BOOL> {
    bool found;
    __device__ __forceinline__ void init() { found = false; }
    template <bool kFP64>
    __device__ __forceinline__ bool leaf(const TraceParams& p, const Ray& r, int k, float& tclip,
                                         Stats& st) {
        float4 A, B, C;
        load_tri(p.tris, k, A, B, C);
        float t32, et;
        double t64;
        bool is64;
        found = decide<kFP64>(r, A, B, C, t32, et, t64, is64, st) == MT_HIT;
        return found;  // any-hit early exit
    }
    __device__ __forceinline__ void finish(const TraceParams& p, const Ray&, int64_t i, Stats&) {
        p.hit[i] = found ? 1 : 0;
    }
};

// Barycentric: lexicographic min of (t, original id) (reading R5).  A hit is
// held as an interval [t32 - et, t32 + et] or an exact fp64 value; overlapping
// intervals are resolved by recomputing both in the fp64 mirror.  Compact
// state (register pressure): the best's leaf slot (-1: none; bit 30 set when
// its t is exact) and ONE 64-bit word holding either the fp64 t or the fp32
// pair (t32, et); the best's original id is re-read from its triangle record
// only when an exact tie has to be broken.
constexpr int kExactBit = 1 << 30;  // slots < 2^30 (N_t <= 2^30)

template <>
struct ModeState<MODE_BARY> {
    int slot;            // -1, else leaf slot | (kExactBit if w holds an exact fp64 t)
    unsigned long long w;  // fp64 t bits, or (t32 bits) | (et bits) << 32
    __device__ __forceinline__ void init() {
        slot = -1;
        w = 0ull;
    }
    __device__ __forceinline__ bool exact() const { return (slot & kExactBit) != 0; }
    __device__ __forceinline__ int leaf_slot() const { return slot & ~kExactBit; }
    __device__ __forceinline__ double t64() const { return __longlong_as_double((long long)w); }
    __device__ __forceinline__ float t32() const { return __uint_as_float((uint32_t)w); }
    __device__ __forceinline__ float e32() const { return __uint_as_float((uint32_t)(w >> 32)); }
    template <bool kFP64>
    __device__ __forceinline__ bool leaf(const TraceParams& p, const Ray& r, int k, float& tclip,
                                         Stats& st) {
        float4 A, B, C;
        load_tri(p.tris, k, A, B, C);
        float t32c, et;
        double c64;
        bool c_is64;
        if (decide<kFP64>(r, A, B, C, t32c, et, c64, c_is64, st) != MT_HIT) return false;
        bool take;
        if (slot < 0) {
            take = true;
        } else {
            const bool bx = exact();
            const double clo = c_is64 ? c64 : (double)t32c - (double)et, chi = c_is64 ? c64 : (double)t32c + (double)et;
            const double blo = bx ? t64() : (double)t32() - (double)e32(), bhi = bx ? t64() : (double)t32() + (double)e32();
            if (chi < blo) {
                take = true;
            } else if (clo > bhi) {
                take = false;
            } else {  // order not certified: settle both in the fp64 mirror
                st.add(ST_FP64_RAYS);
                if (!c_is64) {
                    mt64(r, A, B, C, &c64);
                    c_is64 = true;
                }
                float4 bA, bB, bC;
                load_tri(p.tris, leaf_slot(), bA, bB, bC);
                double b64 = 0.0;
                if (bx) {
                    b64 = t64();
                } else {
                    mt64(r, bA, bB, bC, &b64);
                    slot |= kExactBit;
                    w = (unsigned long long)__double_as_longlong(b64);
                }
                take = (c64 < b64) || (c64 == b64 && __float_as_int(A.w) < __float_as_int(bA.w));
            }
        }
        if (take) {
            if (c_is64) {
                slot = k | kExactBit;
                w = (unsigned long long)__double_as_longlong(c64);
                tclip = fminf(tclip, __double2float_ru(c64));
            } else {
                slot = k;
                w = (unsigned long long)__float_as_uint(t32c) | ((unsigned long long)__float_as_uint(et) << 32);
                tclip = fminf(tclip, __fadd_ru(t32c, et));
            }
        }
        return false;
    }
    // the ray's outputs (tri id, t, dist = t |d|, point = O + t d; 3b/3d,
    // P:166-168) into tri[0], t[0], dist[0], point[0..2] -- the caller's arrays
    // at the ray's row, or its warp's shared-memory staging rows
    // (RSI_BARY_STAGE); t / dist / point may be null
    __device__ __forceinline__ void emit(const TraceParams& p, const Ray& r, Stats& st, int32_t* tri, float* t,
                                         float* dist, float* point) {
        if (slot >= 0) {
            const int k = leaf_slot();
            // the original id: one word of the triangle record (the whole record only for the fp64 recompute)
            const int id = __ldg(reinterpret_cast<const int*>(p.tris + kTriF4 * (int64_t)k) + 3);
            float tt;
            if (exact()) {
                tt = (float)t64();
            } else if (e32() <= kOutTol) {
                tt = t32();
            } else {  // fp32 value not certified to the output tolerance
                float4 bA, bB, bC;
                load_tri(p.tris, k, bA, bB, bC);
                double v = 0.0;
                mt64(r, bA, bB, bC, &v);
                tt = (float)v;
                st.add(ST_FP64_RAYS);
            }
            tri[0] = id;
            if (t) t[0] = tt;
            if (dist) {
#if RSI_FAST_NORM
                const float d2 = fmaf(r.dx, r.dx, fmaf(r.dy, r.dy, r.dz * r.dz));
                const float nd = (d2 >= 1e-30f && d2 <= 1e30f) ? sqrtf(d2) : norm3df(r.dx, r.dy, r.dz);
                dist[0] = tt * nd;
#else
                dist[0] = tt * norm3df(r.dx, r.dy, r.dz);  // no overflow / underflow of |d|^2
#endif
            }
            if (point) {
                point[0] = fmaf(tt, r.dx, r.ox);
                point[1] = fmaf(tt, r.dy, r.oy);
                point[2] = fmaf(tt, r.dz, r.oz);
            }
        } else {
            tri[0] = -1;
            if (t) t[0] = NAN;
            if (dist) dist[0] = NAN;
            if (point) {
                point[0] = NAN;
                point[1] = NAN;
                point[2] = NAN;
            }
        }
    }
    __device__ __forceinline__ void finish(const TraceParams& p, const Ray& r, int64_t i, Stats& st) {
#if RSI_OUT_HINT
        // direct stores with an L2 eviction-priority hint: the rows of a 32-byte
        // sector arrive from different lanes at different times
        int32_t tri;
        float tt, dd, pt[3];
        emit(p, r, st, &tri, &tt, &dd, pt);
        const uint64_t pol = out_policy();
        st_hint(reinterpret_cast<float*>(p.tri + i), __int_as_float(tri), pol);
        if (p.t) st_hint(p.t + i, tt, pol);
        if (p.dist) st_hint(p.dist + i, dd, pol);
        if (p.point) {
            st_hint(p.point + 3 * i, pt[0], pol);
            st_hint(p.point + 3 * i + 1, pt[1], pol);
            st_hint(p.point + 3 * i + 2, pt[2], pol);
        }
#else
        emit(p, r, st, p.tri + i, p.t ? p.t + i : nullptr, p.dist ? p.dist + i : nullptr,
             p.point ? p.point + 3 * i : nullptr);
#endif
    }
};

// Barycentric output staging (RSI_BARY_STAGE).  Finished segments leave the
// persistent refill in random order, so per-segment stores of 4-12 bytes
// would hit each 32-byte sector of tri / t / dist / point many times apart
// (ncu, round 1: 1.88x the algorithmic DRAM bytes, read-modify-write of
// partial sectors).  Each warp instead stages the outputs of its two most
// recent kChunk-segment chunks in shared memory (slot = chunk index & 1) and
// writes a slot out with full coalesced lines when the slot is taken by a
// newer chunk (and at the end).  A segment still running then -- a straggler
// whose chunk already left the slot -- stores directly; rows not yet written
// hold the sentinel tri = kUnset and are skipped by the flush.
// Measured (sphere, 1e7 segments, B200): DRAM bytes per launch 975 -> 607 MB,
// but the launch is 9 % SLOWER (2.34 -> 2.57 ms; 6 KB per CTA without points:
// +9 %, 32-segment chunks: +5 %): the staging memory comes out of the L1
// carveout the tree fetches live in.  Off; the default stores directly with
// an L2 evict_last hint (RSI_OUT_HINT), which keeps partially written output
// sectors in L2 longer: 975 -> 820 MB and -1 %.
#ifndef RSI_BARY_STAGE
#define RSI_BARY_STAGE 0
#endif
#ifndef RSI_STAGE_POINT
#define RSI_STAGE_POINT 1  // 0: points are stored directly (half the staging memory)
#endif
constexpr int kStageWords = (RSI_STAGE_POINT ? 6 : 3) * kChunk;  // per slot: tri, t, dist [kChunk] (+ point [3 kChunk])
constexpr int kUnset = (int)0x80000001;                            // staged row not written

__device__ __forceinline__ void stage_flush(const TraceParams& p, float* sb, int b, int len, int lane) {
    for (int k = lane; k < len; k += 32) {
        const int tri = __float_as_int(sb[k]);
        if (tri != kUnset) {
            p.tri[b + k] = tri;
            if (p.t) p.t[b + k] = sb[kChunk + k];
            if (p.dist) p.dist[b + k] = sb[2 * kChunk + k];
        }
    }
    if (RSI_STAGE_POINT && p.point) {
        for (int f = lane; f < 3 * len; f += 32)
            if (__float_as_int(sb[f / 3]) != kUnset) p.point[3 * (int64_t)b + f] = sb[3 * kChunk + f];
    }
    __syncwarp();
    for (int k = lane; k < kChunk; k += 32) sb[k] = __int_as_float(kUnset);
    __syncwarp();
}

// intercept_count: count = number of single-linkage clusters of hit t with
// threshold tau (reading R4): 1 + #{sorted gaps > tau}.  The fp32 path is used
// only when every pairwise |t_a - t_b| vs tau decision is certified; otherwise
// all hit t are recomputed in the fp64 mirror and counted exactly as the
// oracle does.  More than kCountCap hits -> the exact re-pass.  The hit list
// lives in shared memory (column per thread) to keep registers for occupancy.
__device__ __forceinline__ void sort_small(double* v, int n) {
    for (int a = 1; a < n; ++a) {
        double x = v[a];
        int b = a - 1;
        while (b >= 0 && v[b] > x) {
            v[b + 1] = v[b];
            --b;
        }
        v[b + 1] = x;
    }
}

template <>
struct ModeState<MODE_COUNT> {
    int stride;  // threads per block: entry x of this lane at te[x * stride]
    float2* te;  // shared: te[x * stride] = (t, err) of hit x
    int* kk;     // shared: leaf slot of hit x
    int nh;
    bool overflow;
    __device__ __forceinline__ void init() {
        nh = 0;
        overflow = false;
    }
    template <bool kFP64>
    __device__ __forceinline__ bool leaf(const TraceParams& p, const Ray& r, int k, float& tclip,
                                         Stats& st) {
        float4 A, B, C;
        load_tri(p.tris, k, A, B, C);
        float t32, et;
        double t64;
        bool is64;
        if (decide<kFP64>(r, A, B, C, t32, et, t64, is64, st) != MT_HIT) return false;
        if (nh == kCountCap) {
            overflow = true;
            return true;
        }
        if (is64) {
            t32 = (float)t64;
            et = fmaf(kU, fabsf(t32), kTiny);
        }
        te[nh * stride] = make_float2(t32, et);
        kk[nh * stride] = k;
        ++nh;
        return false;
    }
    __device__ __forceinline__ void finish(const TraceParams& p, const Ray& r, int64_t i, Stats& st) {
        if (overflow) {
            uint32_t pos = atomicAdd(&p.scratch[SCR_OVF_COUNT], 1u);
            p.ovf_list[pos] = (int32_t)i;
            p.count[i] = -1;
            return;
        }
        if (nh <= 1) {
            p.count[i] = nh;
            return;
        }
        const float ftau = (float)p.tau;
        float lt[kCountCap], le[kCountCap];
#pragma unroll
        for (int x = 0; x < kCountCap; ++x)
            if (x < nh) {
                const float2 v = te[x * stride];
                lt[x] = v.x;
                le[x] = v.y;
            }
        bool sure = true;
#pragma unroll
        for (int a = 0; a < kCountCap; ++a)
#pragma unroll
            for (int c = a + 1; c < kCountCap; ++c)
                if (c < nh) {
                    float g = fabsf(lt[a] - lt[c]);
                    float tol = le[a] + le[c] + fmaf(2.0f * kU, g + ftau, kTiny);
                    if (fabsf(g - ftau) <= tol) sure = false;
                }
        int cnt = 1;
        if (sure) {
#pragma unroll
            for (int a = 1; a < kCountCap; ++a)
#pragma unroll
                for (int c = a; c > 0; --c)
                    if (c < nh && lt[c - 1] > lt[c]) {
                        float x = lt[c];
                        lt[c] = lt[c - 1];
                        lt[c - 1] = x;
                    }
#pragma unroll
            for (int a = 0; a + 1 < kCountCap; ++a)
                if (a + 1 < nh && lt[a + 1] - lt[a] > ftau) ++cnt;
        } else {
            st.add(ST_FP64_RAYS);
            double v[kCountCap];
            for (int a = 0; a < nh; ++a) {
                float4 A, B, C;
                load_tri(p.tris, kk[a * stride], A, B, C);
                mt64(r, A, B, C, &v[a]);
            }
            sort_small(v, nh);
            for (int a = 0; a + 1 < nh; ++a)
                if (da(v[a + 1], -v[a]) > p.tau) ++cnt;
        }
        p.count[i] = cnt;
    }
};

// ---------------------------------------------------------------- the traversal kernel
// Persistent warps with per-lane ray refill and postponed leaves (after Aila &
// Laine's while-while traversal, adapted to segments and child-pair nodes):
//   1. refill: lanes without a ray take the next ray ids from the warp's chunk
//      (one atomicAdd per kChunk rays per warp), so lanes never idle while rays remain;
//   2. traversal phase: a lane walks internal nodes until it holds a pending
//      leaf (a leaf child whose box the segment enters; both children when
//      both are leaves); the phase ends when no lane (or fewer than min_trav
//      lanes, while others wait with leaves) is still searching;
//   3. leaf phase: all lanes with pending leaves run Moller-Trumbore together;
//   4. finished rays write their outputs and free the lane.
template <int kStack, int kSmemStack, int kT>
struct LaneStack {
    int* s;  // this lane's shared-memory column: entry k at s[k * kT]
    int local[kStack - kSmemStack];
    __device__ __forceinline__ void push(int& sp, int x) {
        if (sp < kSmemStack)
            s[sp * kT] = x;
        else
            local[sp - kSmemStack] = x;
        ++sp;
    }
    __device__ __forceinline__ int pop(int& sp) {
        --sp;
        return sp < kSmemStack ? s[sp * kT] : local[sp - kSmemStack];
    }
};

// Local-memory stack whose top entry lives in a register: a pop returns the
// register at once and starts the load of the next entry, whose latency is
// hidden until the next pop (the popped node id no longer waits on an LDL).
template <int kStack, int kT>
struct LaneStack<kStack, 0, kT> {
    int* s;
    int top;
    int local[kStack];
    __device__ __forceinline__ void push(int& sp, int x) {
        if (sp > 0) local[sp - 1] = top;
        top = x;
        ++sp;
    }
    __device__ __forceinline__ int pop(int& sp) {
        const int x = top;
        --sp;
        if (sp > 0) top = local[sp - 1];
        return x;
    }
};

// Branch-free stack for the 4-wide walk: the top entry in a
// register, the entries below it at slots 1 .. sp-1 (slot 0 is scratch), slots
// < kSm in a shared-memory column (one bank per lane at any depth), the rest in
// local memory.  push_if always stores (the old top goes to slot sp, which is
// either claimed by the push or dead), so a visit's up-to-3 pushes are
// straight-line code with no divergent branches.
template <int kStack, int kSm, int kT>
struct BFStack {
    int* s;
    int top;
    int local[kStack + 1 - kSm];
    // (unsigned indices: the compiler then knows a store cannot alias `top`)
    __device__ __forceinline__ void put(int k, int x) {
        if (kSm > 0 && k < kSm)
            s[k * kT] = x;
        else
            local[(unsigned)(k - kSm)] = x;
    }
    __device__ __forceinline__ int get(int k) const {
        return (kSm > 0 && k < kSm) ? s[k * kT] : local[(unsigned)(k - kSm)];
    }
    __device__ __forceinline__ void push_if(int& sp, bool v, int x) {
        put(sp, top);
        top = v ? x : top;
        sp += v ? 1 : 0;
    }
    __device__ __forceinline__ void push(int& sp, int x) { push_if(sp, true, x); }
    __device__ __forceinline__ int pop(int& sp) {
        const int x = top;
        --sp;
        top = get(sp);
        return x;
    }
    // keyed interface (keys ignored): see BFKStack
    __device__ __forceinline__ void push_if(int& sp, bool v, int x, float) { push_if(sp, v, x); }
    __device__ __forceinline__ int pop_live(int& sp, float) { return sp > 0 ? pop(sp) : kNoRef; }
};

// BFStack whose entries carry the entry distance tn of their box
// (RSI_BARY_KEYSTACK, barycentric): a pop skips entries with tn > tclip -- the
// nearest hit found since the push lies before the box, so none of its
// members can pass their own (tn <= tclip) test.  tn is the conservative
// slab bound of the quantized member box, <= the entry into the exact box.
template <int kStack, int kT>
struct BFKStack {
    int* s;  // (no shared-memory part)
    int top;
    float ktop;
    int2 local[kStack + 1];
    __device__ __forceinline__ void push_if(int& sp, bool v, int x, float k) {
        local[(unsigned)sp] = make_int2(top, __float_as_int(ktop));
        top = v ? x : top;
        ktop = v ? k : ktop;
        sp += v ? 1 : 0;
    }
    __device__ __forceinline__ void push(int& sp, int x) { push_if(sp, true, x, -INFINITY); }
    __device__ __forceinline__ int pop(int& sp) {
        const int x = top;
        --sp;
        const int2 e = local[(unsigned)sp];
        top = e.x;
        ktop = __int_as_float(e.y);
        return x;
    }
    __device__ __forceinline__ int pop_live(int& sp, float tclip) {
        while (sp > 0) {
            const bool live = ktop <= tclip;
            const int x = pop(sp);
            if (live) return x;
        }
        return kNoRef;
    }
};

// M + byte j of w, as a float (exact; M = kQuadBias).  Default: one PRMT with an
// immediate selector places the byte in mantissa bits 8..15 of `magic` =
// 0x47000000 (2^15), which the caller holds in a register (kept loop-invariant).
// RSI_HALF_DECODE: the PRMT builds the f16 0x64qq = 1024 + q, widened exactly.
__device__ __forceinline__ float half_lo_f32(uint32_t h) {
    float f;
    asm("{.reg .b16 a, b; mov.b32 {a, b}, %1; cvt.f32.f16 %0, a;}" : "=f"(f) : "r"(h));
    return f;
}
__device__ __forceinline__ float half_hi_f32(uint32_t h) {
    float f;
    asm("{.reg .b16 a, b; mov.b32 {a, b}, %1; cvt.f32.f16 %0, b;}" : "=f"(f) : "r"(h));
    return f;
}
__device__ __forceinline__ float byte_to_2p15(uint32_t w, int j, uint32_t magic) {
    uint32_t r;
#if RSI_HALF_DECODE
    switch (j) {
        case 0: asm("prmt.b32 %0, %1, %2, 0x4440;" : "=r"(r) : "r"(w), "r"(magic)); break;
        case 1: asm("prmt.b32 %0, %1, %2, 0x4441;" : "=r"(r) : "r"(w), "r"(magic)); break;
        case 2: asm("prmt.b32 %0, %1, %2, 0x4442;" : "=r"(r) : "r"(w), "r"(magic)); break;
        default: asm("prmt.b32 %0, %1, %2, 0x4443;" : "=r"(r) : "r"(w), "r"(magic)); break;
    }
    return half_lo_f32(r);
#else
    switch (j) {
        case 0: asm("prmt.b32 %0, %1, %2, 0x7604;" : "=r"(r) : "r"(w), "r"(magic)); break;
        case 1: asm("prmt.b32 %0, %1, %2, 0x7614;" : "=r"(r) : "r"(w), "r"(magic)); break;
        case 2: asm("prmt.b32 %0, %1, %2, 0x7624;" : "=r"(r) : "r"(w), "r"(magic)); break;
        default: asm("prmt.b32 %0, %1, %2, 0x7634;" : "=r"(r) : "r"(w), "r"(magic)); break;
    }
    return __uint_as_float(r);
#endif
}
// RSI_HALF_DECODE: bytes 2k, 2k+1 of w as the f16 pair (1024 + q_2k, 1024 + q_2k+1)
__device__ __forceinline__ uint32_t byte_pair_f16(uint32_t w, int k, uint32_t magic) {
    uint32_t r;
    if (k == 0)
        asm("prmt.b32 %0, %1, %2, 0x4140;" : "=r"(r) : "r"(w), "r"(magic));
    else
        asm("prmt.b32 %0, %1, %2, 0x4342;" : "=r"(r) : "r"(w), "r"(magic));
    return r;
}

// RSI_FHFMA: the visit's plane t = (1024 + q) s*inv + b as ONE fma.rn.f32.f16 with
// both factors in f16 -- the record byte's f16 pair (exact) and s*inv rounded
// to f16 in the conservative direction -- instead of widening the f16 to f32
// (HADD2.F32) and an FFMA: 24 instead of 48 instructions per visit.
#ifndef RSI_FHFMA
#define RSI_FHFMA 0  // measured neutral: boolean -0.6 %, barycentric +1.1 %, count +1.5 % (box tests +1.2 %)
#endif

#if RSI_FHFMA
// fma.rn.f32.f16 (sm_100 FHFMA): f32 result of an f16 x f16 product (exact: 11 x 11
// significant bits) plus an f32 addend, one rounding.  qhi / shi pick the half of
// each packed operand (compile-time constants after inlining).
__device__ __forceinline__ float fhfma(uint32_t qpair, bool qhi, uint32_t spair, bool shi, float c) {
    float d;
    if (!qhi && !shi)
        asm("{.reg .b16 a0, a1, b0, b1; mov.b32 {a0, a1}, %1; mov.b32 {b0, b1}, %2; fma.rn.f32.f16 %0, a0, b0, %3;}"
            : "=f"(d) : "r"(qpair), "r"(spair), "f"(c));
    else if (!qhi)
        asm("{.reg .b16 a0, a1, b0, b1; mov.b32 {a0, a1}, %1; mov.b32 {b0, b1}, %2; fma.rn.f32.f16 %0, a0, b1, %3;}"
            : "=f"(d) : "r"(qpair), "r"(spair), "f"(c));
    else if (!shi)
        asm("{.reg .b16 a0, a1, b0, b1; mov.b32 {a0, a1}, %1; mov.b32 {b0, b1}, %2; fma.rn.f32.f16 %0, a1, b0, %3;}"
            : "=f"(d) : "r"(qpair), "r"(spair), "f"(c));
    else
        asm("{.reg .b16 a0, a1, b0, b1; mov.b32 {a0, a1}, %1; mov.b32 {b0, b1}, %2; fma.rn.f32.f16 %0, a1, b1, %3;}"
            : "=f"(d) : "r"(qpair), "r"(spair), "f"(c));
    return d;
}
#endif
#ifndef RSI_BARY_FULLSORT
#define RSI_BARY_FULLSORT 0  // barycentric: all hit children near-first (0: only the nearest first)
#endif
#ifndef RSI_BOOL_SAT
#define RSI_BOOL_SAT 1  // boolean + intercept_count (tclip == 1): planes clamped to [0, 1] in their FFMA, strict box test
#endif
#ifndef RSI_BARY_SAT
#define RSI_BARY_SAT 0  // barycentric: clamped planes, strict box test + tn <= tclip
#endif
#ifndef RSI_BOOL_FRONT
#define RSI_BOOL_FRONT 0  // boolean: any hit child first by selects (no nearest-first order)
#endif
#ifndef RSI_BARY_KEYSTACK
#define RSI_BARY_KEYSTACK 0  // barycentric: stack entries carry their entry distance (pop skips tn > tclip)
#endif
#ifndef RSI_COUNT_FRONT
#define RSI_COUNT_FRONT 1    // intercept_count: any hit child first by selects instead of the key network
#endif
// compare-and-swap of (key, ref) pairs: ascending keys
__device__ __forceinline__ void cas(float& ka, int& ca, float& kb, int& cb) {
    const bool sw = kb < ka;
    const float tk = sw ? kb : ka;
    kb = sw ? ka : kb;
    ka = tk;
    const int tc = sw ? cb : ca;
    cb = sw ? ca : cb;
    ca = tc;
}

template <int MODE, bool kFP64, bool kCounters>
__global__ void __launch_bounds__(trace_threads<MODE>(), (MODE == MODE_BOOL ? RSI_BOOL_MINB : (MODE == MODE_BARY ? RSI_BARY_MINB : RSI_COUNT_MINB))) k_trace(const TraceParams p) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    // near-first child order: needed for nearest-hit culling, helps any-hit exit; useless for counts
    constexpr bool kSort = (MODE == MODE_BARY) || (MODE == MODE_BOOL && RSI_SORT_ALL) ||
                           (MODE == MODE_COUNT && kQuadCount);  // (4-wide: puts a hit child first)
    constexpr bool kQuad = MODE == MODE_BOOL ? RSI_BOOL_QUAD : (MODE == MODE_BARY ? RSI_BARY_QUAD : RSI_COUNT_QUAD);
    constexpr int kSmemStack = MODE == MODE_BOOL ? RSI_BOOL_SMEM : (MODE == MODE_BARY ? RSI_BARY_SMEM : RSI_COUNT_SMEM);
    constexpr int kStack = kQuad ? kStackQuad : kStackBinary;
    constexpr int kT = trace_threads<MODE>();
    // dynamic shared memory: [top-of-tree image: kQTop x 64 B (4-wide walk)][intercept_count hit lists]
    constexpr int kImg = kQuad ? kQTop : 0;
    extern __shared__ float4 s_dyn[];
    float4* s_top = s_dyn;
    float2* s_te = reinterpret_cast<float2*>(s_dyn + 4 * kImg);
    int* s_k = reinterpret_cast<int*>(s_te + kCountCap * kT);
    // top-of-tree image, loaded once per CTA
    const int n_top = kImg > 0 ? (int)p.scratch[SCR_NTOP] : 0;  // written by the build (k_qtop)
    for (int i = threadIdx.x; i < 4 * n_top; i += kT) s_top[i] = p.top[i];
    __syncthreads();
    Stats st;

    // 32-bit ray indices (rsi_intersect limits n_rays to 2^31 - 1): registers matter
    const int n32 = (int)p.n;
    int cnext = 0, cend = 0;      // warp-uniform chunk [cnext, cend)
    bool exhausted = false;       // warp-uniform
    int ray = -1;
    Ray r;
    int node = -1, sp = 0, l0 = -1, l1 = -1, l2 = -1;  // pending (postponed) leaf slots
    // per-lane traversal stack: the first kSmemStack entries in a shared-memory
    // column (one bank per lane: conflict-free at any depth), the rest local
    constexpr bool kQSpec = MODE == MODE_BOOL ? RSI_QSPEC_BOOL : (MODE == MODE_BARY ? RSI_QSPEC_BARY : RSI_QSPEC_COUNT);
    constexpr bool kBF = kQuad;  // branch-free stack on the 4-wide walk (-11 % boolean, -5 % barycentric)
    constexpr int kSmWords = kBF ? RSI_BF_SMEM : kSmemStack;
    constexpr bool kKeyed = kBF && MODE == MODE_BARY && RSI_BARY_KEYSTACK;
    typename std::conditional<kKeyed, BFKStack<kStack, kT>,
        typename std::conditional<kBF, BFStack<kStack, RSI_BF_SMEM, kT>, LaneStack<kStack, kSmemStack, kT>>::type>::type stk;
    __shared__ int s_stack[kSmWords > 0 ? kSmWords * kT : 1];
    stk.s = s_stack + threadIdx.x;
    float tclip = 1.0f;
    ModeState<MODE> ms;
    constexpr bool kStage = MODE == MODE_BARY && RSI_BARY_STAGE;
    __shared__ float s_stage[kStage ? (kT / 32) * 2 * kStageWords : 1];
    __shared__ int s_own[kStage ? kT / 32 : 1][2];  // chunk base held by each slot (-1: none)
    float* stg = s_stage + (kStage ? (threadIdx.x >> 5) * 2 * kStageWords : 0);
    int* own = s_own[kStage ? threadIdx.x >> 5 : 0];
    if (kStage) {
        for (int k = lane; k < 2 * kChunk; k += 32) stg[(k / kChunk) * kStageWords + k % kChunk] = __int_as_float(kUnset);
        if (lane < 2) own[lane] = -1;
        __syncwarp();
    }
    if constexpr (MODE == MODE_COUNT) {
        ms.stride = kT;
        ms.te = s_te + threadIdx.x;
        ms.kk = s_k + threadIdx.x;
    }
    // root node: 0 for the Karras numbering, the top split under RSI_OPT_APETREI
    // (-1 when a fault-injected build never reached it: every ray misses)
    const int root = n_top > 0 ? (int)kSmemRef : (int)p.scratch[kQuad ? SCR_QROOT : SCR_ROOT_NODE];
    // kQuadMagic (float 2^15, or the f16 exponent byte) from a kernel parameter: an opaque register, so the
    // quad decode's PRMTs keep their byte selectors as immediates
    const uint32_t magic = p.magic;
    // 4-wide walk: slack term Pmax / 4 and the |inv| range that keeps s * inv an
    // exact normal float and every term of the folded decode far from overflow
    // (slab_axis), from the build's scratch words -- read here on the device, so
    // rsi_intersect needs no host read-back of the build
    // (qext, qlim_lo, qlim_hi): read at ray setup, not held in registers (barycentric)
    constexpr bool kQcSmem = RSI_QC_SMEM && MODE == MODE_BARY;
    __shared__ float s_qc[3];
    float qext = 0.0f, qlim_lo = 0.0f, qlim_hi = INFINITY;
    if constexpr (kQuad) {
        const float pmax = __uint_as_float(p.scratch[SCR_QPMAX]);
        const int emin = (int)p.scratch[SCR_QEMIN] - 128, emax = (int)p.scratch[SCR_QEMAX] - 128;
        qext = 0.25f * pmax;
        qlim_lo = scalbnf(1.0f, -124 - emin);
        qlim_hi = scalbnf(1.0f, 100) / (pmax + scalbnf(65536.0f, emax));
        if (kQcSmem) {
            if (threadIdx.x == 0) {
                s_qc[0] = qext;
                s_qc[1] = qlim_lo;
                s_qc[2] = qlim_hi;
            }
            __syncthreads();
        }
    }
    // lanes without a segment take the next ids from the warp's chunk and set up
    // ---- 1. refill: lanes without a segment take the next ids from the warp's
    // chunk (one atomicAdd per kChunk segments per warp) and set them up
    constexpr bool kPf = RSI_RAY_PREFETCH && kQuad && !kStage;
    __shared__ float s_nr[kPf ? 6 * kT : 1];
    float* nr = s_nr + (kPf ? threadIdx.x : 0);  // this lane's column: S.xyz, E.xyz at stride kT
    int nxt = -1;                                // kPf: the claimed next segment (data in flight to nr)
    // lanes with no claimed segment take the next ids from the warp's chunk (one
    // atomicAdd per kChunk segments per warp): kPf -- lanes without a next
    // segment claim one and start its copy; else lanes without a segment
    auto claim = [&](bool& fresh) {
        unsigned want = __ballot_sync(FULL, kPf ? nxt < 0 : ray < 0);
        while (want && !exhausted) {
            if (cnext >= cend) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(p.counter, (unsigned long long)kChunk);
                base = __shfl_sync(FULL, base, 0);
                if ((int64_t)base >= p.n) {
                    exhausted = true;
                    break;
                }
                cnext = (int)base;
                cend = min(cnext + kChunk, n32);
                if (kStage) {  // the chunk's staging slot: write out the older chunk it held
                    const int sl = (cnext / kChunk) & 1;
                    const int ob = own[sl];
                    if (ob >= 0) stage_flush(p, stg + sl * kStageWords, ob, min(kChunk, n32 - ob), lane);
                    if (lane == 0) own[sl] = cnext;
                    __syncwarp();
                }
            }
            const int take = min(__popc(want), cend - cnext);
            const bool mine = (want >> lane) & 1u;
            const int rank = __popc(want & lt);
            const bool got = mine && rank < take;
            if (got) {
                if (kPf) {
                    nxt = cnext + rank;
                    const float* sp3 = p.S + 3 * (int64_t)nxt;
                    const float* ep3 = p.E + 3 * (int64_t)nxt;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        cp_async4(nr + c * kT, sp3 + c);
                        cp_async4(nr + (3 + c) * kT, ep3 + c);
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                } else {
                    ray = cnext + rank;
                    fresh = true;
                }
            }
            want &= ~__ballot_sync(FULL, got);
            cnext += take;
        }
    };
    // ---- 1. refill: lanes without a segment start their claimed next one
    // (kPf) or take the next ids from the warp's chunk, and set them up
    auto refill = [&]() {
        bool fresh = false;
        if (kPf && ray < 0 && nxt >= 0) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            r.ox = nr[0];
            r.oy = nr[kT];
            r.oz = nr[2 * kT];
            r.ex = nr[3 * kT];
            r.ey = nr[4 * kT];
            r.ez = nr[5 * kT];
            ray = nxt;
            nxt = -1;
            fresh = true;
        }
        claim(fresh);
        if (RSI_RAY_PF_L1 && MODE == MODE_COUNT && !kPf && !exhausted && cnext < cend) {
            // L1 prefetch of the 128-byte lines holding the chunk's next 32
            // segments (start and end arrays): the refill that hands them out
            // then finds them in L1.  Lanes 0..3 cover start, 4..7 end.
            const int j1 = min(cnext + 32, cend);
            const int a = lane & 3;
            const float* base = lane < 4 ? p.S : p.E;
            const uint64_t b0 = (reinterpret_cast<uint64_t>(base + 3 * (int64_t)cnext) & ~(uint64_t)127) + 128u * a;
            const uint64_t b1 = reinterpret_cast<uint64_t>(base + 3 * (int64_t)j1);
            if (lane < 8 && b0 < b1) asm volatile("prefetch.global.L1 [%0];" ::"l"(b0));
        }
        if (fresh) {
            bool nonfinite;
            if (kQuad && kQcSmem) {
                qext = s_qc[0];
                qlim_lo = s_qc[1];
                qlim_hi = s_qc[2];
            }
            const bool ok = kPf ? setup_ray<true>(r, nonfinite, qext, qlim_lo, qlim_hi)
                          : kQuad ? load_ray<true>(r, p.S, p.E, ray, nonfinite, qext, qlim_lo, qlim_hi)
                                  : load_ray<false>(r, p.S, p.E, ray, nonfinite);
            if (nonfinite) st.add(ST_NONFINITE);
            ms.init();
            tclip = 1.0f;
            sp = 0;
            l0 = l1 = l2 = -1;
            node = ok ? root : -1;
        }
    };
    if (kPf) {  // prologue: every lane claims its first segment
        bool unused = false;
        claim(unused);
    }
    while (true) {
        refill();
        if (__ballot_sync(FULL, ray >= 0) == 0) break;  // no rays left for this warp

        if constexpr (kQuad) {
        // ---- 2. traversal phase (4-wide view: a visit tests the up-to-4
        // cut members of a binary node; a hit child goes first
        // (kSort) or by slot, the first becomes the next visit and the rest go
        // on the stack; a leaf (ref < 0) becomes the lane's pending leaf)
        while (true) {
            const bool trav = node >= 0 && l0 < 0;
            const unsigned tm = __ballot_sync(FULL, trav);
            if (tm == 0) break;
            if (kCounters && lane == 0) {
                const unsigned pm = __popc(__ballot_sync(FULL, l0 >= 0));
                st.c[ST_IT_SEARCH] += __popc(tm);
                st.c[ST_IT_PEND] += pm;
                st.c[ST_IT_IDLE] += 32u - __popc(tm) - pm;
                st.c[ST_ITERS] += 1;
            } else if (kCounters) {
                __ballot_sync(FULL, l0 >= 0);
            }
            if (__popc(tm) < p.min_trav && __ballot_sync(FULL, l0 >= 0)) break;
            constexpr int kVisits = MODE == MODE_BOOL ? RSI_VISITS_BOOL : (MODE == MODE_BARY ? RSI_VISITS_BARY : RSI_VISITS_COUNT);
#pragma unroll 1
            for (int u = 0; u < kVisits; ++u) {
            // kQSpec: a lane holding one pending leaf keeps walking (its next
            // leaf goes to l1) in slots it would otherwise idle in
            if ((node >= 0 && l0 < 0) || (kQSpec && node >= 0 && l1 < 0)) {
                float4 qa, qb, qc, qd;
                if (kImg > 0 && node >= (int)kSmemRef) {  // the top of the tree, from shared memory
                    const float4* q = s_top + 4 * (node - (int)kSmemRef);
                    qa = q[0];
                    qb = q[1];
                    qc = q[2];
                    qd = q[3];
                } else {
                    const float4* q = p.quads + 4 * node;
                    ldg256h<RSI_Q_L1>(q, qa, qb);
                    ldg256h<RSI_Q_L1>(q + 2, qc, qd);
                }
                // Per axis: grid step s = 2^e and the decode offset pm = p - 2^15 s
                // (stored; exact).  A child plane is p + q s = (2^15 + q) s + pm, so its
                // t = (plane - o) / d is fma(2^15 + q, s*inv, fma(pm, inv, -off)): s*inv
                // is exact (a power of two times inv, kept normal by qlim_lo/qlim_hi),
                // 2^15 + q comes from one PRMT, and the rounding of the inner fma is
                // covered by the slack (slab_axis, qext).  The ray octant picks which
                // byte array holds the near planes (lo for inv >= 0), so each child needs
                // no per-axis min/max.
                float sa[3], bn[3], bf[3];
                uint32_t wn[3], wf[3];
                const float pp[3] = {qa.x, qa.y, qa.z};
                const uint32_t wq[6] = {__float_as_uint(qb.x), __float_as_uint(qb.y), __float_as_uint(qb.z),
                                        __float_as_uint(qb.w), __float_as_uint(qc.x), __float_as_uint(qc.y)};
                const float inv3[3] = {r.ix, r.iy, r.iz};
                const float scv[3] = {qa.w, qd.z, qd.w};  // grid steps s = 2^e
                // octant masks: kept per ray, except for intercept_count (register
                // pressure at 72 registers: derived from the sign of inv per visit)
                const uint32_t msk[3] = {
                    MODE == MODE_COUNT ? (uint32_t)(__float_as_int(r.ix) >> 31) : r.mx,
                    MODE == MODE_COUNT ? (uint32_t)(__float_as_int(r.iy) >> 31) : r.my,
                    MODE == MODE_COUNT ? (uint32_t)(__float_as_int(r.iz) >> 31) : r.mz};
                const float nof[3] = {r.lx, r.ly, r.lz};
                const float fof[3] = {r.hx, r.hy, r.hz};
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    sa[a] = scv[a] * inv3[a];
                    bn[a] = fmaf(pp[a], inv3[a], -nof[a]);
                    bf[a] = fmaf(pp[a], inv3[a], -fof[a]);
                    wn[a] = (wq[2 * a] & ~msk[a]) | (wq[2 * a + 1] & msk[a]);
                    wf[a] = (wq[2 * a + 1] & ~msk[a]) | (wq[2 * a] & msk[a]);
                }
                const int4 q6 = make_int4(__float_as_int(qc.z), __float_as_int(qc.w), __float_as_int(qd.x),
                                          __float_as_int(qd.y));
#if RSI_HALF_DECODE
                uint32_t hn[3][2], hf[3][2];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    hn[a][0] = byte_pair_f16(wn[a], 0, magic);
                    hn[a][1] = byte_pair_f16(wn[a], 1, magic);
                    hf[a][0] = byte_pair_f16(wf[a], 0, magic);
                    hf[a][1] = byte_pair_f16(wf[a], 1, magic);
                }
                auto dq = [](const uint32_t (&h)[2], int j) {
                    return (j & 1) ? half_hi_f32(h[j >> 1]) : half_lo_f32(h[j >> 1]);
                };
#define RSI_DQN(a, j) dq(hn[a], j)
#define RSI_DQF(a, j) dq(hf[a], j)
#else
#define RSI_DQN(a, j) byte_to_2p15(wn[a], j, magic)
#define RSI_DQF(a, j) byte_to_2p15(wf[a], j, magic)
#endif
#if RSI_FHFMA && RSI_HALF_DECODE
                // s*inv per axis as two f16 copies: Z rounded toward zero (|Z| <= |s inv|)
                // and A = Z + 1 ulp (|A| >= |s inv|; the largest finite Z becomes +-inf).
                // A plane's t = (1024 + q) x + b grows with x (1024 + q > 0), so the NEAR
                // planes take the copy <= s inv (Z where s inv >= 0, A where < 0: the
                // octant mask) and the FAR planes the copy >= s inv: the computed entry t
                // is never later, the exit t never earlier, than with s inv itself (the
                // product is exact in f32, the addition rounds once as before), so the
                // slab test stays conservative with the same slack.  Unconstrained axes
                // (inv = 0, b = -+inf) stay unconstrained.
                uint32_t z01, z2;
                asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(z01) : "f"(sa[1]), "f"(sa[0]));
                asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(z2) : "f"(0.0f), "f"(sa[2]));
                const uint32_t a01 = z01 + 0x00010001u, a2 = z2 + 0x00000001u;
                const uint32_t m01 = (msk[0] & 0x0000ffffu) | (msk[1] & 0xffff0000u), m2 = msk[2];
                const uint32_t sn01 = (z01 & ~m01) | (a01 & m01), sf01 = (a01 & ~m01) | (z01 & m01);
                const uint32_t sn2 = (z2 & ~m2) | (a2 & m2), sf2 = (a2 & ~m2) | (z2 & m2);
                auto child = [&](int j, float& tn) {
                    const bool qh = (j & 1) != 0;
                    const float nx = fhfma(hn[0][j >> 1], qh, sn01, false, bn[0]);
                    const float ny = fhfma(hn[1][j >> 1], qh, sn01, true, bn[1]);
                    const float nz = fhfma(hn[2][j >> 1], qh, sn2, false, bn[2]);
                    const float fx = fhfma(hf[0][j >> 1], qh, sf01, false, bf[0]);
                    const float fy = fhfma(hf[1][j >> 1], qh, sf01, true, bf[1]);
                    const float fz = fhfma(hf[2][j >> 1], qh, sf2, false, bf[2]);
#else
                auto child = [&](int j, float& tn) {
                    const float nx = fmaf(RSI_DQN(0, j), sa[0], bn[0]);
                    const float ny = fmaf(RSI_DQN(1, j), sa[1], bn[1]);
                    const float nz = fmaf(RSI_DQN(2, j), sa[2], bn[2]);
                    const float fx = fmaf(RSI_DQF(0, j), sa[0], bf[0]);
                    const float fy = fmaf(RSI_DQF(1, j), sa[1], bf[1]);
                    const float fz = fmaf(RSI_DQF(2, j), sa[2], bf[2]);
#endif
                    if constexpr (MODE != MODE_BARY && RSI_BOOL_SAT) {  // tclip stays 1
                        // [0, 1] clamp of every plane in its FFMA (.SAT) and a strict
                        // test: a box the segment truly crosses has computed
                        // tn < exact entry <= exact exit < computed tf (slack > 0),
                        // so tn' < tf' after clamping; a box wholly beyond an end
                        // clamps to tn' = tf' (0 or 1) and fails
                        tn = fmaxf(fmaxf(__saturatef(nx), __saturatef(ny)), __saturatef(nz));
                        const float tf = fminf(fminf(__saturatef(fx), __saturatef(fy)), __saturatef(fz));
                        return tn < tf;
                    } else if constexpr (MODE == MODE_BARY && RSI_BARY_SAT) {
                        // clamped planes as above; the strict test rejects boxes wholly
                        // beyond an end, the second (<=) keeps boxes entered exactly at
                        // the current nearest t (ties resolve by triangle id)
                        tn = fmaxf(fmaxf(__saturatef(nx), __saturatef(ny)), __saturatef(nz));
                        const float tf = fminf(fminf(__saturatef(fx), __saturatef(fy)), __saturatef(fz));
                        return tn < tf && tn <= tclip;
                    } else {
                        tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
                        const float tf = fminf(fminf(fx, fy), fminf(fz, tclip));
                        return tn <= tf;  // a missing child has an empty box and ref kNoRef
                    }
                };
#undef RSI_DQN
#undef RSI_DQF
                float k0, k1, k2, k3;
                const bool h0 = child(0, k0), h1 = child(1, k1), h2 = child(2, k2), h3 = child(3, k3);
                if (kCounters) st.boxes += 4;
                int c0 = h0 ? q6.x : kNoRef, c1 = h1 ? q6.y : kNoRef, c2 = h2 ? q6.z : kNoRef, c3 = h3 ? q6.w : kNoRef;
                if ((MODE == MODE_COUNT && RSI_COUNT_FRONT) || (MODE == MODE_BOOL && RSI_BOOL_FRONT)) {
                    // counts need no order: bring a hit child to slot 0 (so the walk
                    // continues without a stack round trip)
                    bool m0 = c0 == kNoRef;
                    int t = m0 ? c1 : c0; c1 = m0 ? c0 : c1; c0 = t; m0 = c0 == kNoRef;
                    t = m0 ? c2 : c0; c2 = m0 ? c0 : c2; c0 = t; m0 = c0 == kNoRef;
                    t = m0 ? c3 : c0; c3 = m0 ? c0 : c3; c0 = t;
                } else if (kSort) {
                    k0 = h0 ? k0 : INFINITY;
                    k1 = h1 ? k1 : INFINITY;
                    k2 = h2 ? k2 : INFINITY;
                    k3 = h3 ? k3 : INFINITY;
                    if (MODE == MODE_BARY && RSI_BARY_FULLSORT) {  // full near-first order (nearest-hit culling)
                        cas(k0, c0, k1, c1);
                        cas(k2, c2, k3, c3);
                        cas(k0, c0, k2, c2);
                        cas(k1, c1, k3, c3);
                        cas(k1, c1, k2, c2);
                    } else {  // any hit: only the nearest child goes first
                        cas(k0, c0, k1, c1);
                        cas(k2, c2, k3, c3);
                        cas(k0, c0, k2, c2);
                    }
                }
                // c0 is the nearest hit child (kSort) -- kNoRef only when none hit
                if constexpr (kKeyed) {
                    stk.push_if(sp, c3 != kNoRef, c3, k3);
                    stk.push_if(sp, c2 != kNoRef, c2, k2);
                    stk.push_if(sp, c1 != kNoRef, c1, k1);
                } else {
                    stk.push_if(sp, c3 != kNoRef, c3);
                    stk.push_if(sp, c2 != kNoRef, c2);
                    stk.push_if(sp, c1 != kNoRef, c1);
                }
                int first = c0;
                if (first == kNoRef) first = kKeyed ? stk.pop_live(sp, tclip) : (sp > 0 ? stk.pop(sp) : kNoRef);
                if (first != kNoRef && first < 0) {  // a leaf
                    if (l0 < 0) {
                        l0 = ~first;
                        // kQSpec: keep walking from the next stack entry while
                        // the warp is still in the traversal phase
                        first = !kQSpec ? kNoRef : (kKeyed ? stk.pop_live(sp, tclip) : (sp > 0 ? stk.pop(sp) : kNoRef));
                        if (first != kNoRef && first < 0) {
                            l1 = ~first;
                            first = kNoRef;
                        }
                    } else {
                        l1 = ~first;
                        first = kNoRef;
                    }
                }
                node = first >= 0 ? first : -1;
            }
            if (kVisits > 1 && !((node >= 0 && l0 < 0) || (kQSpec && node >= 0 && l1 < 0))) break;
            }
        }

        // ---- 3. leaf phase: the pending leaf (and the speculative one), then
        // one more in a row if the next stack entry is a leaf
        if (kCounters) {
            const unsigned lm = __popc(__ballot_sync(FULL, l0 >= 0));
            if (lane == 0 && lm) {
                st.c[ST_LEAF_LANES] += lm;
                st.c[ST_LEAF_PHASES] += 1;
            }
        }
        if (l0 >= 0) {
            if (kCounters) st.mts += 1 + (l1 >= 0);
            bool done = ms.template leaf<kFP64>(p, r, l0, tclip, st);
            if (!done && l1 >= 0) done = ms.template leaf<kFP64>(p, r, l1, tclip, st);
            l0 = l1 = -1;
            int nxt = (done || node >= 0) ? kNoRef : (kKeyed ? stk.pop_live(sp, tclip) : (sp > 0 ? stk.pop(sp) : kNoRef));
            if (nxt != kNoRef && nxt < 0) {
                if (kCounters) st.mts += 1;
                done = ms.template leaf<kFP64>(p, r, ~nxt, tclip, st);
                nxt = done ? kNoRef : (kKeyed ? stk.pop_live(sp, tclip) : (sp > 0 ? stk.pop(sp) : kNoRef));
            }
            if (MODE == MODE_BOOL && RSI_LEAF_SEL) {
            // the same outcome by selects (the leaf phase runs at ~6 active lanes):
            // done -> finished; a speculative position stays; else the popped
            // entry is the next visit (>= 0), the next pending leaf (< 0), or none
            const bool keep = !done && node >= 0;
            const bool has = !done && node < 0 && nxt != kNoRef;
            l0 = (has && nxt < 0) ? ~nxt : -1;
            node = keep ? node : ((has && nxt >= 0) ? nxt : -1);
            sp = done ? 0 : sp;
            } else if (done) {
                node = -1;
                sp = 0;
            } else if (node >= 0) {
                // the speculative walk's position stays the next visit
            } else if (nxt == kNoRef) {
                node = -1;
            } else if (nxt >= 0) {
                node = nxt;
            } else {
                l0 = ~nxt;
                node = -1;
            }
        }

        } else {
        // ---- 2. traversal phase
        // a lane walks internal nodes until it holds a pending leaf (l0, and l1
        // when both children of the visited node are leaves)
        while (true) {
            const bool trav = node >= 0 && l0 < 0;
            const unsigned tm = __ballot_sync(FULL, trav);
            if (tm == 0) break;
            if (kCounters && lane == 0) {
                const unsigned pm = __popc(__ballot_sync(FULL, l0 >= 0));
                st.c[ST_IT_SEARCH] += __popc(tm);
                st.c[ST_IT_PEND] += pm;
                st.c[ST_IT_IDLE] += 32u - __popc(tm) - pm;
                st.c[ST_ITERS] += 1;
            } else if (kCounters) {
                __ballot_sync(FULL, l0 >= 0);
            }
            if (__popc(tm) < p.min_trav && __ballot_sync(FULL, l0 >= 0)) break;
            // RSI_SPEC: a lane holding one pending leaf keeps walking in slots it
            // would otherwise idle in (its new leaves queue in l1, l2)
            if (trav || (RSI_SPEC && node >= 0 && l1 < 0)) {
                float4 n0, n1, n2, n3f;
                {
                    const float4* nd = p.nodes + 4 * node;
                    ldg256(nd, n0, n1);
                    ldg256(nd + 2, n2, n3f);
                }
                const int4 n3 = make_int4(__float_as_int(n3f.x), __float_as_int(n3f.y), 0, 0);
                float nearL, nearR;
                bool hL = slab(r, n0.x, n0.y, n0.z, n0.w, n2.x, n2.y, tclip, nearL);
                bool hR = slab(r, n1.x, n1.y, n1.z, n1.w, n2.z, n2.w, tclip, nearR);
                if (kCounters) st.boxes += 2;
                if (hL && n3.x < 0) {
                    if (l0 < 0)
                        l0 = ~n3.x;
                    else
                        l1 = ~n3.x;
                    hL = false;
                }
                if (hR && n3.y < 0) {
                    if (l0 < 0)
                        l0 = ~n3.y;
                    else if (l1 < 0)
                        l1 = ~n3.y;
                    else
                        l2 = ~n3.y;
                    hR = false;
                }
                if (hL && hR) {
                    const bool rfirst = nearR < nearL;
                    stk.push(sp, rfirst ? n3.x : n3.y);
                    node = rfirst ? n3.y : n3.x;
                } else if (hL) {
                    node = n3.x;
                } else if (hR) {
                    node = n3.y;
                } else {
                    node = sp > 0 ? stk.pop(sp) : -1;
                }
            }
        }

        // ---- 3. leaf phase
        if (kCounters) {
            const unsigned lm = __popc(__ballot_sync(FULL, l0 >= 0));
            if (lane == 0 && lm) {
                st.c[ST_LEAF_LANES] += lm;
                st.c[ST_LEAF_PHASES] += 1;
            }
        }
        if (l0 >= 0) {
            if (kCounters) st.mts += 1 + (l1 >= 0) + (l2 >= 0);
            bool done = ms.template leaf<kFP64>(p, r, l0, tclip, st);
            if (!done && l1 >= 0) done = ms.template leaf<kFP64>(p, r, l1, tclip, st);
            if (!done && l2 >= 0) done = ms.template leaf<kFP64>(p, r, l2, tclip, st);
            l0 = l1 = l2 = -1;
            if (done) node = -1;
        }
        }

        // ---- 4. finish
        if (ray >= 0 && node < 0 && l0 < 0) {
            if constexpr (kStage) {
                const int sl = (ray / kChunk) & 1, k = ray % kChunk;
                if (own[sl] == ray - k) {  // staged (else a straggler: direct stores)
                    float* sb = stg + sl * kStageWords;
                    ms.emit(p, r, st, reinterpret_cast<int32_t*>(sb + k), sb + kChunk + k, sb + 2 * kChunk + k,
                            RSI_STAGE_POINT ? sb + 3 * kChunk + 3 * k
                                            : (p.point ? p.point + 3 * (int64_t)ray : nullptr));
                } else {
                    ms.finish(p, r, ray, st);
                }
            } else {
                ms.finish(p, r, ray, st);
            }
            ray = -1;
        }
    }
    if (kStage) {  // every segment is done: write out what is left staged
        __syncwarp();
        for (int sl = 0; sl < 2; ++sl)
            if (own[sl] >= 0) stage_flush(p, stg + sl * kStageWords, own[sl], min(kChunk, n32 - own[sl]), lane);
    }
    if (kCounters) {
        st.add(ST_BOX_TESTS, st.boxes);
        st.add(ST_MT_TESTS, st.mts);
    }
#pragma unroll
    for (int k = 1; k < ST_WORDS; ++k) {
        unsigned v = st.c[k];
        if (__any_sync(FULL, v)) {
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
            if (lane == 0 && v) atomicAdd(p.stats + k, (unsigned long long)v);
        }
    }
}

// ---------------------------------------------------------------- exact re-pass for overflowed rays
// intercept_count rays whose hits do not fit k_trace's kCountCap-entry list are
// counted here, exactly and WITHOUT any host round trip (the overflow count is
// read on the device).  One warp per overflowed segment (persistent warps):
//
//  * walk: the lanes share a stack in shared memory and each iteration pops up
//    to 32 4-wide records at once (the long grazing segments that overflow
//    are walked 32 nodes at a time); every leaf the segment enters is decided
//    exactly (mt32 drops certain misses, the fp64 mirror settles the rest and
//    gives the oracle's t);
//  * windows: hits are keyed (t, leaf slot) -- a total order, ties in t broken
//    by slot -- and a walk keeps the kRpKeep smallest keys above the previous
//    window's last key in a per-warp shared-memory buffer (when the buffer
//    fills it is sorted, cut to the kRpKeep smallest, and only smaller keys
//    are accepted from then on).  A walk that never had to cut holds every
//    remaining hit and is the last; otherwise its kRpKeep smallest are counted
//    and the next walk starts above them.  So the count is exact for any
//    number of hits (<= N_t), with no capacity-dependent result (unlike the
//    paper's fixed CollisionList / InterceptDistances buffers);
//  * count (reading R4, the oracle's single linkage): sorted by a bitonic
//    network over the buffer, count = [nh > 0] + popc of the ballots of
//    "gap to the previous key > tau" with the oracle's correctly rounded gap
//    __dadd_rn(t_i, -t_(i-1)); the last t of a window carries to the next.
//  * boxes: a record member is visited only if its conservative [tn, tf]
//    (clamped to [0, 1]) meets [lo_t, thr_t] of the current window, rounded
//    outward to fp32.
//  * stack: pops are narrowed as the stack fills so that it never overflows:
//    while top <= kRpStack - 3 * 32 - kStackQuad a pop of `take` records can
//    push at most 3 * take more; above that, pops of 1 record continue a
//    depth-first walk whose growth is bounded by kStackQuad (the lane-stack
//    bound of the 4-wide walk).
constexpr int kRpWarps = 4;     // warps per block
constexpr int kRpStack = 1024;  // shared stack entries per warp (4 KB)
constexpr int kRpBuf = 512;     // hit keys buffered per warp (6 KB)
constexpr int kRpKeep = 256;    // keys kept when the buffer is cut
static_assert(kRpStack >= kStackQuad + 3 * 32 + 32, "re-pass stack bound");

__device__ __forceinline__ bool key_less(double ta, int sa, double tb, int sb) {
    return ta < tb || (ta == tb && sa < sb);
}

// ascending bitonic sort of the first n keys of (t, s) (warp-cooperative;
// entries [n, P) are padded with +inf / INT_MAX, P = pow2 >= max(n, 32))
__device__ void warp_sort_keys(double* t, int* s, int n, int lane) {
    int P = 32;
    while (P < n) P <<= 1;
    for (int i = n + lane; i < P; i += 32) {
        t[i] = INFINITY;
        s[i] = 0x7fffffff;
    }
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int x = lane; x < P / 2; x += 32) {
                const int i = 2 * j * (x / j) + (x % j), q = i + j;
                const bool up = (i & k) == 0;
                const double ti = t[i], tq = t[q];
                const int si = s[i], sq = s[q];
                if (key_less(tq, sq, ti, si) == up) {
                    t[i] = tq; s[i] = sq;
                    t[q] = ti; s[q] = si;
                }
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(32 * kRpWarps) k_count_repass(
    const float4* __restrict__ quads, const float4* __restrict__ tris, const float* __restrict__ S,
    const float* __restrict__ E, const int32_t* __restrict__ list, uint32_t* scratch, double tau,
    int32_t* __restrict__ count_out, unsigned long long* stats, uint32_t magic) {
    __shared__ int s_stack[kRpWarps][kRpStack];
    __shared__ double s_t[kRpWarps][kRpBuf];
    __shared__ int s_s[kRpWarps][kRpBuf];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned ltm = lanemask_lt();
    const int n_ovf = (int)*(volatile uint32_t*)&scratch[SCR_OVF_COUNT];
    if (blockIdx.x == 0 && threadIdx.x == 0 && n_ovf > 0) atomicAdd(stats + ST_OVERFLOW, (unsigned long long)n_ovf);
    const int root = (int)scratch[SCR_QROOT];
    const float pmax = __uint_as_float(scratch[SCR_QPMAX]);
    const int emin = (int)scratch[SCR_QEMIN] - 128, emax = (int)scratch[SCR_QEMAX] - 128;
    int* stk = s_stack[w];
    double* bt = s_t[w];
    int* bs = s_s[w];
    constexpr int kWide = kRpStack - kStackQuad - 3 * 32;  // above this top, pops of 1
    while (true) {  // dynamic: each warp takes the next overflowed segment (long ones vary widely)
        int j = 0;
        if (lane == 0) j = (int)atomicAdd(&scratch[SCR_OVF_NEXT], 1u);
        j = __shfl_sync(FULL, j, 0);
        if (j >= n_ovf) break;
        const int ray = list[j];
        Ray r;
        bool nonfinite;
        load_ray<true>(r, S, E, ray, nonfinite, 0.25f * pmax, scalbnf(1.0f, -124 - emin),
                       scalbnf(1.0f, 100) / (pmax + scalbnf(65536.0f, emax)));
        const float inv3[3] = {r.ix, r.iy, r.iz};
        const uint32_t msk[3] = {r.mx, r.my, r.mz};
        const float nof[3] = {r.lx, r.ly, r.lz};
        const float fof[3] = {r.hx, r.hy, r.hz};
        double lo_t = -INFINITY;  // window: keys > (lo_t, lo_s)
        int lo_s = -1;
        bool has_prev = false;    // a hit was counted in an earlier window
        double prev_t = 0.0;
        int cnt = 0;
        bool more = root >= 0;
        while (more) {  // one walk per window
            double thr_t = INFINITY;  // keys < (thr_t, thr_s) once the buffer was cut
            int thr_s = 0x7fffffff;
            bool cut = false;
            int nbuf = 0, top = 0;
            if (lane == 0) stk[0] = root;
            top = 1;
            __syncwarp();
            const float lo_f = lo_t == -INFINITY ? -INFINITY : __double2float_rd(lo_t);
            while (top > 0) {
                float thr_f = thr_t == INFINITY ? INFINITY : __double2float_ru(thr_t);
                int take = top < 32 ? top : 32;
                if (top > kWide) take = 1;
                else if (take > (kWide - top) / 3 + 1) take = (kWide - top) / 3 + 1;
                const int node = lane < take ? stk[top - 1 - lane] : -1;
                top -= take;
                __syncwarp();
                int push[4] = {kNoRef, kNoRef, kNoRef, kNoRef};
                int leafs[4] = {kNoRef, kNoRef, kNoRef, kNoRef};
                if (node >= 0) {
                    const float4* q = quads + 4 * node;
                    float4 qa, qb, qc, qd;
                    ldg256(q, qa, qb);
                    ldg256(q + 2, qc, qd);
                    const float pp[3] = {qa.x, qa.y, qa.z};
                    const uint32_t wq[6] = {__float_as_uint(qb.x), __float_as_uint(qb.y), __float_as_uint(qb.z),
                                            __float_as_uint(qb.w), __float_as_uint(qc.x), __float_as_uint(qc.y)};
                    const float scv[3] = {qa.w, qd.z, qd.w};
                    float sa[3], bn[3], bf[3];
                    uint32_t wn[3], wf[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        sa[a] = scv[a] * inv3[a];
                        bn[a] = fmaf(pp[a], inv3[a], -nof[a]);
                        bf[a] = fmaf(pp[a], inv3[a], -fof[a]);
                        wn[a] = (wq[2 * a] & ~msk[a]) | (wq[2 * a + 1] & msk[a]);
                        wf[a] = (wq[2 * a + 1] & ~msk[a]) | (wq[2 * a] & msk[a]);
                    }
                    const int ref[4] = {__float_as_int(qc.z), __float_as_int(qc.w), __float_as_int(qd.x),
                                        __float_as_int(qd.y)};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float tn = fmaxf(fmaxf(fmaf(byte_to_2p15(wn[0], c, magic), sa[0], bn[0]),
                                                     fmaf(byte_to_2p15(wn[1], c, magic), sa[1], bn[1])),
                                               fmaxf(fmaf(byte_to_2p15(wn[2], c, magic), sa[2], bn[2]), 0.0f));
                        const float tf = fminf(fminf(fmaf(byte_to_2p15(wf[0], c, magic), sa[0], bf[0]),
                                                     fmaf(byte_to_2p15(wf[1], c, magic), sa[1], bf[1])),
                                               fminf(fmaf(byte_to_2p15(wf[2], c, magic), sa[2], bf[2]), 1.0f));
                        if (tn <= tf && tf >= lo_f && tn <= thr_f && ref[c] != kNoRef) {
                            if (ref[c] < 0)
                                leafs[c] = ~ref[c];
                            else
                                push[c] = ref[c];
                        }
                    }
                }
                // leaves: exact decision, key (t, slot) into the window buffer
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    bool acc = false;
                    double t64 = 0.0;
                    if (leafs[c] != kNoRef) {
                        float4 A, B, C;
                        load_tri(tris, leafs[c], A, B, C);
                        float t32, et;
                        if (mt32(r, A, B, C, t32, et) != MT_MISS && mt64(r, A, B, C, &t64))
                            acc = key_less(lo_t, lo_s, t64, leafs[c]) && key_less(t64, leafs[c], thr_t, thr_s);
                    }
                    const unsigned am = __ballot_sync(FULL, acc);
                    if (am == 0) continue;
                    if (nbuf + __popc(am) > kRpBuf) {  // cut: keep the kRpKeep smallest keys
                        warp_sort_keys(bt, bs, nbuf, lane);
                        nbuf = kRpKeep;
                        thr_t = bt[kRpKeep - 1];
                        thr_s = bs[kRpKeep - 1];
                        cut = true;
                        __syncwarp();
                        acc = acc && key_less(t64, leafs[c], thr_t, thr_s);
                    }
                    const unsigned am2 = __ballot_sync(FULL, acc);
                    if (acc) {
                        const int pos = nbuf + __popc(am2 & ltm);
                        bt[pos] = t64;
                        bs[pos] = leafs[c];
                    }
                    nbuf += __popc(am2);
                    __syncwarp();
                }
                // pushes: warp prefix sum of each lane's internal members
                int np = 0;
#pragma unroll
                for (int c = 0; c < 4; ++c) np += push[c] != kNoRef;
                int incl = np;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                int pos = top + incl - np;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (push[c] != kNoRef) stk[pos++] = push[c];
                top += __shfl_sync(FULL, incl, 31);
                __syncwarp();
            }
            const int m = cut ? kRpKeep : nbuf;
            if (m <= 32) {  // the common case: one key per lane, shuffle bitonic sort in registers
                double tk = lane < m ? bt[lane] : INFINITY;
                int sk = lane < m ? bs[lane] : 0x7fffffff;
                for (int k = 2; k <= 32; k <<= 1)
                    for (int jj = k >> 1; jj > 0; jj >>= 1) {
                        const double to = __shfl_xor_sync(FULL, tk, jj);
                        const int so = __shfl_xor_sync(FULL, sk, jj);
                        const bool lower = (lane & jj) == 0, up = (lane & k) == 0;
                        // keep the smaller key on the lower lane of an ascending block
                        const bool take = (lower == up) ? key_less(to, so, tk, sk) : key_less(tk, sk, to, so);
                        if (take) {
                            tk = to;
                            sk = so;
                        }
                    }
                const double tp = __shfl_up_sync(FULL, tk, 1);
                bool gap = false;
                if (lane < m) gap = lane > 0 ? da(tk, -tp) > tau : (!has_prev || da(tk, -prev_t) > tau);
                cnt += __popc(__ballot_sync(FULL, gap));
                if (m > 0) {
                    has_prev = true;
                    prev_t = __shfl_sync(FULL, tk, m - 1);
                }
                more = false;  // m <= 32 < kRpKeep: this walk never cut
                __syncwarp();
                continue;
            }
            // the window's keys, ascending; a walk that never cut holds them all
            warp_sort_keys(bt, bs, nbuf, lane);
            for (int base = 0; base < m; base += 32) {
                const int i = base + lane;
                bool gap = false;
                if (i < m) {
                    const double ti = bt[i];
                    if (i > 0) gap = da(ti, -bt[i - 1]) > tau;
                    else gap = !has_prev || da(ti, -prev_t) > tau;  // first hit overall starts a cluster
                }
                cnt += __popc(__ballot_sync(FULL, gap));
            }
            if (m > 0) {
                has_prev = true;
                prev_t = bt[m - 1];
                lo_t = bt[m - 1];
                lo_s = bs[m - 1];
            }
            more = cut;
            __syncwarp();
        }
        if (lane == 0) count_out[ray] = cnt;
    }
}

// ---------------------------------------------------------------- ordered compaction (3a)
constexpr int kCompactTile = 4096;

__global__ void __launch_bounds__(256) k_compact_count(const int32_t* __restrict__ tri, int64_t n,
                                                       uint32_t* __restrict__ blk) {
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    int64_t beg = (int64_t)blockIdx.x * kCompactTile;
    uint32_t mine = 0;
    for (int64_t i = beg + threadIdx.x; i < beg + kCompactTile && i < n; i += blockDim.x) mine += tri[i] >= 0;
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&c, mine);
    __syncthreads();
    if (threadIdx.x == 0) blk[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) k_compact_scan(uint32_t* blk, int m, int32_t* d_n) {
    // single CTA exclusive scan (m is small: n / 4096)
    __shared__ uint32_t carry;
    __shared__ uint32_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < m; base += 1024) {
        int i = base + threadIdx.x;
        uint32_t v = i < m ? blk[i] : 0u, inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (w == 0) {
            uint32_t s = wsum[lane], si = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
                if (lane >= o) si += y;
            }
            wsum[lane] = si - s;
        }
        __syncthreads();
        if (i < m) blk[i] = carry + wsum[w] + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += wsum[31] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) *d_n = (int32_t)carry;
}

__global__ void __launch_bounds__(256) k_compact_write(const int32_t* __restrict__ tri, int64_t n,
                                                       const uint32_t* __restrict__ blk, int32_t* __restrict__ ids) {
    // each warp handles a contiguous chunk of the tile in order
    __shared__ uint32_t wtot[8];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t beg = (int64_t)blockIdx.x * kCompactTile + (int64_t)w * (kCompactTile / 8);
    const int64_t end = beg + kCompactTile / 8;
    uint32_t cnt = 0;
    for (int64_t i = beg + lane; i < end; i += 32) cnt += (i < n && tri[i] >= 0);
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) wtot[w] = cnt;
    __syncthreads();
    uint32_t base = blk[blockIdx.x];
    for (int x = 0; x < w; ++x) base += wtot[x];
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int64_t i0 = beg; i0 < end; i0 += 32) {
        int64_t i = i0 + lane;
        bool h = i < n && tri[i] >= 0;
        uint32_t bal = __ballot_sync(0xffffffffu, h);
        if (h) ids[base + __popc(bal & lt)] = (int32_t)i;
        base += __popc(bal);
    }
}

// Sparse barycentric return: the values of the compacted hit rays,
// in ascending ray order (grid-stride over the device-side hit count).
__global__ void __launch_bounds__(256) k_gather_hits(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_hits,
                                                     const int32_t* __restrict__ tri, const float* __restrict__ dist,
                                                     const float* __restrict__ point, int32_t* __restrict__ out_tri,
                                                     float* __restrict__ out_dist, float* __restrict__ out_point) {
    const int m = *n_hits;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const int i = ids[j];
        out_tri[j] = tri[i];
        if (dist) out_dist[j] = dist[i];
        if (point) {
            out_point[3 * j] = point[3 * (int64_t)i];
            out_point[3 * j + 1] = point[3 * (int64_t)i + 1];
            out_point[3 * j + 2] = point[3 * (int64_t)i + 2];
        }
    }
}

}  // namespace

rsi_status_t rsi_gather_hits_device(const int32_t* ids, const int32_t* n_hits, int64_t n_max, const int32_t* tri,
                                    const float* dist, const float* point, int32_t* out_tri, float* out_dist,
                                    float* out_point, cudaStream_t s) {
    if (n_max <= 0) return RSI_OK;
    int blocks = rsi_ceil_div(n_max, 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    rsi_note_launch(), k_gather_hits<<<blocks, 256, 0, s>>>(ids, n_hits, tri, dist, point, out_tri, out_dist, out_point);
    return rsi_cuda_check(cudaGetLastError(), "gather launch");
}

// ---------------------------------------------------------------- host side
template <int MODE, bool kFP64, bool kCounters>
static void launch_trace(const TraceParams& p, cudaStream_t s) {
    constexpr int kT = trace_threads<MODE>();
    constexpr bool kQuadM = MODE == MODE_BOOL ? RSI_BOOL_QUAD : (MODE == MODE_BARY ? RSI_BARY_QUAD : RSI_COUNT_QUAD);
    constexpr int kDyn = (kQuadM ? kQTop : 0) * 4 * (int)sizeof(float4) + (MODE == MODE_COUNT ? kCountCap * kT * 12 : 0);
    const size_t dyn = kDyn;
    static int grid = 0;  // persistent grid: resident blocks per SM x SMs (per instantiation)
    if (grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_trace<MODE, kFP64, kCounters>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDyn);
#if RSI_PREFER_L1
        if (kDyn == 0) cudaFuncSetAttribute(k_trace<MODE, kFP64, kCounters>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
#endif
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trace<MODE, kFP64, kCounters>, kT, kDyn);
        grid = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
    }
    const int64_t need = (p.n + kT - 1) / kT;
    const int g = (int)(need < grid ? need : grid);
    rsi_note_launch(), k_trace<MODE, kFP64, kCounters><<<g, kT, dyn, s>>>(p);
}

template <bool kFP64, bool kCounters>
static void launch_mode(int32_t mode, const TraceParams& p, cudaStream_t s) {
    if (mode == RSI_MODE_BOOLEAN)
        launch_trace<MODE_BOOL, kFP64, kCounters>(p, s);
    else if (mode == RSI_MODE_BARYCENTRIC)
        launch_trace<MODE_BARY, kFP64, kCounters>(p, s);
    else
        launch_trace<MODE_COUNT, kFP64, kCounters>(p, s);
}

rsi_status_t rsi_intersect_device(rsi_bvh* h, const float* S, const float* E, int64_t n, int32_t mode,
                                  const rsi_outputs_t* out, cudaStream_t s) {
    if (n == 0) return RSI_OK;
    if (n > ((int64_t)1 << 31) - 1)
        return rsi_set_error(RSI_E_INVALID_ARG, "n_rays %lld exceeds 2^31-1", (long long)n);
    rsi_status_t st;
    if (mode == RSI_MODE_INTERCEPT_COUNT && h->ovf_cap < n) {
        if (h->ovf_list) cudaFreeAsync(h->ovf_list, s);
        h->ovf_list = nullptr;
        h->ovf_cap = 0;
        st = rsi_cuda_check(cudaMallocAsync((void**)&h->ovf_list, (size_t)n * sizeof(int32_t), s), "overflow list");
        if (st != RSI_OK) return RSI_E_OOM;
        h->ovf_cap = n;
    }
    // zero the overflow counters and the ray dispenser (scratch words 16..19)
    st = rsi_cuda_check(cudaMemsetAsync(h->scratch + SCR_OVF_COUNT, 0, 4 * sizeof(uint32_t), s), "memset");
    if (st != RSI_OK) return st;
    TraceParams p{};
    p.nodes = h->nodes;
    p.quads = h->quads;
    p.top = h->top;
    p.tris = h->tris;
    p.S = S;
    p.E = E;
    p.n = n;
    p.hit = out->hit;
    p.tri = out->tri;
    p.t = out->t;
    p.dist = out->dist;
    p.point = out->point;
    p.count = out->count;
    p.tau = h->opt.dedup_tau;
    p.magic = kQuadMagic;
    p.ovf_list = h->ovf_list;
    p.scratch = h->scratch;
    p.stats = h->stats;
    p.counter = reinterpret_cast<unsigned long long*>(h->scratch + SCR_DISPENSER);
    // traversal-phase exit threshold, measured per mode (env RSI_MIN_TRAV overrides)
    // measured per mode on the sphere / paper-terrain workloads
    p.min_trav = h->min_trav >= 0 ? h->min_trav
                                  : (mode == RSI_MODE_BOOLEAN ? 16 : (mode == RSI_MODE_BARYCENTRIC ? 12 : 12));
    const bool fp64 = (h->opt.flags & RSI_OPT_FP64_MOLLER) != 0, ctr = (h->opt.flags & RSI_OPT_COUNTERS) != 0;
    if (fp64)
        ctr ? launch_mode<true, true>(mode, p, s) : launch_mode<true, false>(mode, p, s);
    else
        ctr ? launch_mode<false, true>(mode, p, s) : launch_mode<false, false>(mode, p, s);
    st = rsi_cuda_check(cudaGetLastError(), "traversal launch");
    if (st != RSI_OK) return st;
    if (mode != RSI_MODE_INTERCEPT_COUNT) return RSI_OK;

    // intercept_count: the exact re-pass for rays that overflowed the register
    // list.  Always launched (a persistent grid; every warp reads the overflow
    // count on the device and exits at once when it is 0): no host read-back.
    static int rp_grid = 0;
    if (rp_grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_count_repass, 32 * kRpWarps, 0);
        rp_grid = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
    }
    rsi_note_launch(), k_count_repass<<<rp_grid, 32 * kRpWarps, 0, s>>>(h->quads, h->tris, S, E, h->ovf_list,
                                                                       h->scratch, h->opt.dedup_tau, out->count,
                                                                       h->stats, kQuadMagic);
    return rsi_cuda_check(cudaGetLastError(), "count re-pass launch");
}

bool rsi_uses_quads() { return true; }  // the intercept_count re-pass walks the 4-wide records

rsi_status_t rsi_compact_device(const int32_t* tri, int64_t n, int32_t* ids, int32_t* d_n, cudaStream_t s) {
    if (n == 0) return rsi_cuda_check(cudaMemsetAsync(d_n, 0, sizeof(int32_t), s), "memset");
    const int nb = rsi_ceil_div(n, kCompactTile);
    uint32_t* blk = nullptr;
    rsi_status_t st = rsi_cuda_check(cudaMallocAsync((void**)&blk, (size_t)nb * sizeof(uint32_t), s), "compact");
    if (st != RSI_OK) return RSI_E_OOM;
    rsi_note_launch(), k_compact_count<<<nb, 256, 0, s>>>(tri, n, blk);
    rsi_note_launch(), k_compact_scan<<<1, 1024, 0, s>>>(blk, nb, d_n);
    rsi_note_launch(), k_compact_write<<<nb, 256, 0, s>>>(tri, n, blk, ids);
    st = rsi_cuda_check(cudaGetLastError(), "compaction launch");
    cudaFreeAsync(blk, s);
    return st;
}
