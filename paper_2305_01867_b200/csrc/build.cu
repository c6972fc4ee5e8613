// build.cu -- LBVH construction on sm_100a.
//
//   A1+A2  k_extent_validate  index range + finite check, surface AABB
//   A3     k_morton           30-bit z-major Morton code of each centroid
//   A4     k_sort_rank        stable rank sort, N_t <= 16384 (one launch)
//          k_sort_hist/rowscan/scatter  hand-written stable 8-bit LSD radix sort
//   A5     k_karras           Karras binary radix tree topology
//   A6+A7  k_refit            leaf init + atomic bottom-up AABB refit written
//                             straight into the 64 B child-pair layout (P:255-270,
//                             P:442), triangles packed in Morton order;
//                             optional local SAH rotations (RSI_OPT_ROTATE)
//   A7     k_quads            64 B 4-wide quantized records for the traversal
//   NEXT-1 k_morton63, k_pass2_*, k_apetrei  63-bit codes + the paper's
//                             agglomerative build (RSI_OPT_APETREI)
//   NEXT-2 k_validate_*       GPU integrity validator
//
// Every grid is derived from the element count it covers (the case-study-2
// lesson: never size one kernel's grid from another's count).
#include <cstdio>

#include <cstring>
#include <new>
#include <vector>

#include "rsi_internal.cuh"

namespace {

constexpr int kBlock = 256;

__global__ void k_build_init(uint32_t* scratch, uint32_t root_init) {
    int i = threadIdx.x;
    if (i == 1) scratch[SCR_ROOT_NODE] = root_init;
    if (i < 3) {
        scratch[SCR_EXT_MIN + i] = 0xffffffffu;
        scratch[SCR_EXT_MAX + i] = 0u;
    }
    if (i == 0) {
        scratch[SCR_STATUS] = 0u;
        scratch[SCR_ROOT_SET] = 0u;
        scratch[SCR_QPMAX] = 0u;
        scratch[SCR_QEMIN] = 0xffffffffu;
        scratch[SCR_QEMAX] = 0u;
    }
    if (i < 32) scratch[SCR_SORT_DONE + i] = 0u;
    if (i == 2) scratch[SCR_SAH_COUNT] = 0u;
}

__device__ __forceinline__ float warp_min(float v) {
    for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// A1 + A2: surface extent of ALL vertices (exact fp32 min/max) and validation.
__global__ void __launch_bounds__(kBlock) k_extent_validate(const float* __restrict__ V, int64_t nv,
                                                            const int32_t* __restrict__ T, int64_t nt,
                                                            uint32_t* scratch) {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    uint32_t bad = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float x = V[3 * i + k];
            if (!isfinite(x)) bad |= STATUS_NONFINITE;
            mn[k] = fminf(mn[k], x);
            mx[k] = fmaxf(mx[k], x);
        }
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * nt; i += stride) {
        int32_t a = T[i];
        if (a < 0 || (int64_t)a >= nv) bad |= STATUS_INDEX;
    }
    __shared__ float smn[3][kBlock / 32], smx[3][kBlock / 32];
    __shared__ uint32_t sbad;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float a = warp_min(mn[k]), b = warp_max(mx[k]);
        if (lane == 0) {
            smn[k][w] = a;
            smx[k][w] = b;
        }
    }
    if (bad) atomicOr(&sbad, bad);
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float a = lane < kBlock / 32 ? smn[k][lane] : INFINITY;
            float b = lane < kBlock / 32 ? smx[k][lane] : -INFINITY;
            a = warp_min(a);
            b = warp_max(b);
            if (lane == 0 && a <= b) {
                atomicMin(&scratch[SCR_EXT_MIN + k], rsi_f2ord(a));
                atomicMax(&scratch[SCR_EXT_MAX + k], rsi_f2ord(b));
            }
        }
        if (lane == 0 && sbad) atomicOr(&scratch[SCR_STATUS], sbad);
    }
}

// Spread the low 10 bits of x so bit k lands at bit 3k.
__device__ __forceinline__ uint32_t expand10(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

// Per-axis quantization (reading R8) with each axis's extent floored at 1/64
// of the largest extent (wmax / 64 is exact): compact meshes keep the paper's
// per-axis codes (the Fig. 3 tree), while a flat terrain's thin
// axis no longer takes the top Morton bits and splits the map by height.
__device__ __forceinline__ uint32_t quantize10(float c, float lo, float hi, float wmax) {
    float w = fmaxf(hi - lo, wmax * 0.015625f);
    if (!(w > 0.0f)) return 0u;  // zero-extent mesh -> 0
    float q = floorf((c - lo) / w * 1024.0f);
    q = fminf(fmaxf(q, 0.0f), 1023.0f);  // NaN -> 0 via fmaxf
    return (uint32_t)q;
}

__device__ __forceinline__ int32_t safe_index(int32_t a, int64_t nv) {
    return (a < 0 || (int64_t)a >= nv) ? 0 : a;  // invalid meshes are rejected by status
}

// A3: code = expand(qx) | expand(qy) << 1 | expand(qz) << 2 (z-major, reading R8).
// Also zeroes the refit arrival counters.
__global__ void __launch_bounds__(kBlock) k_morton(const float* __restrict__ V, int64_t nv,
                                                   const int32_t* __restrict__ T, int n,
                                                   const uint32_t* __restrict__ scratch,
                                                   uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                                   uint32_t* __restrict__ arrivals, int n_nodes,
                                                   uint32_t* __restrict__ rank) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    if (j < n_nodes) arrivals[j] = 0u;
    if (rank) rank[j] = 0u;  // rank-sort accumulators (N_t <= kRankSortMax)
    float lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = rsi_ord2f(scratch[SCR_EXT_MIN + k]);
        hi[k] = rsi_ord2f(scratch[SCR_EXT_MAX + k]);
    }
    int32_t a = safe_index(T[3 * j], nv), b = safe_index(T[3 * j + 1], nv), c = safe_index(T[3 * j + 2], nv);
    const float wmax = fmaxf(hi[0] - lo[0], fmaxf(hi[1] - lo[1], hi[2] - lo[2]));
    uint32_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float cen = (V[3 * a + k] + V[3 * b + k] + V[3 * c + k]) / 3.0f;
        q[k] = quantize10(cen, lo[k], hi[k], wmax);
    }
    keys[j] = expand10(q[0]) | (expand10(q[1]) << 1) | (expand10(q[2]) << 2);
    vals[j] = j;
}

// A3 + A4 fused for small meshes (N_t <= kSortSmallMax, RSI_SORT_SMALL): ONE
// CTA computes every code (exactly k_morton's arithmetic) into shared memory
// and sorts (code, index) there by a stable LSD radix sort, 8-bit digits, four
// passes (codes are 30-bit), then writes the sorted codes to `keys` and the
// triangle indices to `vals` -- the same result as the stable rank sort
// (ties by index), in one launch and without the O(N^2) compares.  Each pass:
// warp w owns the contiguous segment [w*seg, (w+1)*seg) of the current order
// and walks it 32 keys at a time in lane order; equal digits of a step are
// grouped by __match_any_sync (the lowest peer writes), so per-warp digit
// counts need no atomics; an exclusive scan in (digit, warp) order turns them
// into offsets; the second walk places key j at offset + its rank among
// earlier equal digits (popc of lower peers).  Order within a digit is (warp,
// position) = the current order: stable.
// Measured and rejected: sphere N_t = 1e4 rebuild 0.107 -> 0.166 ms, 16384
// random triangles 0.146 -> 0.234 ms (one SM: the code phase's gathers and
// the four passes are latency chains; the rank sort spreads over every SM).
#ifndef RSI_SORT_SMALL
#define RSI_SORT_SMALL 0
#endif
constexpr int kSortSmallMax = 16384;
constexpr int kSortSmallT = 1024, kSortSmallW = kSortSmallT / 32;
__host__ __device__ constexpr size_t sort_small_smem(int n) {
    return (size_t)2 * ((n + 3) & ~3) * sizeof(uint32_t) + (size_t)2 * ((n + 7) & ~7) * sizeof(uint16_t) +
           (size_t)kSortSmallW * 256 * sizeof(uint16_t) + 64 * sizeof(uint32_t);
}

__global__ void __launch_bounds__(kSortSmallT, 1) k_morton_sort_small(const float* __restrict__ V, int64_t nv,
                                                                      const int32_t* __restrict__ T, int n,
                                                                      const uint32_t* __restrict__ scratch,
                                                                      uint32_t* __restrict__ keys,
                                                                      int32_t* __restrict__ vals,
                                                                      uint32_t* __restrict__ arrivals, int n_nodes) {
    extern __shared__ uint4 s_ms4[];
    const int n4 = (n + 3) & ~3, n8 = (n + 7) & ~7;
    uint32_t* ka = reinterpret_cast<uint32_t*>(s_ms4);
    uint32_t* kb = ka + n4;
    uint16_t* ia = reinterpret_cast<uint16_t*>(kb + n4);
    uint16_t* ib = ia + n8;
    uint16_t* cnt = ib + n8;                                       // [warp][256]
    uint32_t* s_part = reinterpret_cast<uint32_t*>(cnt + kSortSmallW * 256);  // [32] warp totals of the scan
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int j = tid; j < n_nodes; j += kSortSmallT) arrivals[j] = 0u;
    float lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = rsi_ord2f(scratch[SCR_EXT_MIN + k]);
        hi[k] = rsi_ord2f(scratch[SCR_EXT_MAX + k]);
    }
    const float wmax = fmaxf(hi[0] - lo[0], fmaxf(hi[1] - lo[1], hi[2] - lo[2]));
    for (int j = tid; j < n; j += kSortSmallT) {  // A3: the codes, as k_morton
        const int32_t a = safe_index(T[3 * j], nv), b = safe_index(T[3 * j + 1], nv), c = safe_index(T[3 * j + 2], nv);
        uint32_t q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float cen = (V[3 * a + k] + V[3 * b + k] + V[3 * c + k]) / 3.0f;
            q[k] = quantize10(cen, lo[k], hi[k], wmax);
        }
        ka[j] = expand10(q[0]) | (expand10(q[1]) << 1) | (expand10(q[2]) << 2);
        ia[j] = (uint16_t)j;
    }
    const int seg = (n + kSortSmallW - 1) / kSortSmallW;
    const int s0 = min(w * seg, n), s1 = min(s0 + seg, n);
    uint16_t* my = cnt + w * 256;
    for (int shift = 0; shift < 32; shift += 8) {
        for (int k = tid; k < kSortSmallW * 256; k += kSortSmallT) cnt[k] = 0;
        __syncthreads();
        // (a) per-warp digit counts
        for (int j0 = s0; j0 < s1; j0 += 32) {
            const int j = j0 + lane;
            const unsigned act = __ballot_sync(0xffffffffu, j < s1);
            if (j < s1) {
                const uint32_t d = (ka[j] >> shift) & 255u;
                const unsigned peers = __match_any_sync(act, d);
                if ((peers & lt) == 0u) my[d] = (uint16_t)(my[d] + __popc(peers));
            }
            __syncwarp();
        }
        __syncthreads();
        // (b) exclusive scan in (digit, warp) order: thread t holds digit t / 4,
        // warps (t % 4) * 8 .. + 8
        {
            const int d = tid >> 2, wb = (tid & 3) * 8;
            uint32_t v[8], sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[i] = cnt[(wb + i) * 256 + d];
                sum += v[i];
            }
            uint32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_part[w] = inc;
            __syncthreads();
            if (w == 0) {
                uint32_t x = s_part[lane], xi = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
                    if (lane >= o) xi += y;
                }
                s_part[lane] = xi - x;  // exclusive warp offsets
            }
            __syncthreads();
            uint32_t run = s_part[w] + inc - sum;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[(wb + i) * 256 + d] = (uint16_t)run;
                run += v[i];
            }
        }
        __syncthreads();
        // (c) scatter in the same walk order
        for (int j0 = s0; j0 < s1; j0 += 32) {
            const int j = j0 + lane;
            const unsigned act = __ballot_sync(0xffffffffu, j < s1);
            if (j < s1) {
                const uint32_t key = ka[j];
                const uint32_t d = (key >> shift) & 255u;
                const unsigned peers = __match_any_sync(act, d);
                const int pos = my[d] + __popc(peers & lt);
                kb[pos] = key;
                ib[pos] = ia[j];
                __syncwarp(act);
                if ((peers & lt) == 0u) my[d] = (uint16_t)(my[d] + __popc(peers));
            }
            __syncwarp();
        }
        __syncthreads();
        uint32_t* tk = ka; ka = kb; kb = tk;
        uint16_t* ti = ia; ia = ib; ib = ti;
    }
    for (int j = tid; j < n; j += kSortSmallT) {
        keys[j] = ka[j];
        vals[j] = (int32_t)ia[j];
    }
}

// ------------------------------------------------------------------ A4: radix sort
// N_t <= 16384: the one-launch rank sort (k_sort_rank below).  Larger: stable
// LSD radix sort, 8-bit digits, 4 passes (histogram / scan / scatter per pass).
// Stability of each pass comes from warp-ordered ranking: a warp walks its
// contiguous segment 32 keys at a time, lanes in index order, and ranks equal
// digits with ballots (digit_peers); per-warp digit counts are scanned over
// warps, then over blocks per digit (k_sort_rowscan), then over digits.
constexpr int kDigits = 256;
constexpr int kPasses = 4;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exclusive scan of s[0..255] in place by one warp; returns the total.
__device__ uint32_t warp_scan256(uint32_t* s) {
    int lane = threadIdx.x & 31;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        v[j] = s[lane * 8 + j];
        sum += v[j];
    }
    uint32_t inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        s[lane * 8 + j] = run;
        run += v[j];
    }
    return __shfl_sync(0xffffffffu, inc, 31);
}

// Lanes of the warp holding the same 8-bit digit as this lane (valid lanes
// only): AND over the digit's bits of ballot(bit) or ~ballot(bit) -- cheaper
// than __match_any_sync.
__device__ __forceinline__ uint32_t digit_peers(bool valid, uint32_t d) {
    uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bb : ~bb;
    }
    return valid ? m : 0u;
}

// Count digits of this warp's segment [beg, end) into wcnt (warp-private row).
__device__ __forceinline__ void warp_count(const uint32_t* __restrict__ ks, int beg, int end, int shift,
                                           uint32_t* wcnt) {
    int lane = threadIdx.x & 31;
    for (int base = beg; base < end; base += 32) {
        int i = base + lane;
        bool valid = i < end;
        const uint32_t d = valid ? (ks[i] >> shift) & 255u : 0u;
        const uint32_t peers = digit_peers(valid, d);
        if (valid && lane == __ffs(peers) - 1) wcnt[d] += __popc(peers);
        __syncwarp();
    }
}

// Scatter this warp's segment; wcnt[d] holds the warp's running offset within digit d.
__device__ __forceinline__ void warp_scatter(const uint32_t* __restrict__ ks, const int32_t* __restrict__ vs,
                                             uint32_t* __restrict__ kd, int32_t* __restrict__ vd, int beg,
                                             int end, int shift, uint32_t* wcnt, const uint32_t* dbase) {
    int lane = threadIdx.x & 31;
    uint32_t lt = lanemask_lt();
    for (int base = beg; base < end; base += 32) {
        int i = base + lane;
        bool valid = i < end;
        uint32_t key = valid ? ks[i] : 0u;
        int32_t val = valid ? vs[i] : 0;
        const uint32_t d = valid ? (key >> shift) & 255u : 0u;
        const uint32_t peers = digit_peers(valid, d);
        if (valid) {
            uint32_t pos = dbase[d] + wcnt[d] + __popc(peers & lt);
            kd[pos] = key;
            vd[pos] = val;
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wcnt[d] += __popc(peers);
        __syncwarp();
    }
}

constexpr int kTileThreads = 512;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kTile = 4096;  // keys per block (256 per warp)

__global__ void __launch_bounds__(kTileThreads) k_sort_hist(const uint32_t* __restrict__ ks, int n, int shift,
                                                            uint32_t* __restrict__ hist) {
    __shared__ uint32_t cnt[kDigits];
    for (int i = threadIdx.x; i < kDigits; i += blockDim.x) cnt[i] = 0u;
    __syncthreads();
    int beg = blockIdx.x * kTile, end = min(beg + kTile, n);
    for (int i = beg + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&cnt[(ks[i] >> shift) & 255u], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < kDigits; d += blockDim.x) hist[(size_t)d * gridDim.x + blockIdx.x] = cnt[d];
}

// Exclusive scan of each digit's row hist[d][0..nb) in place, one CTA per
// digit; the row totals go to rows[d] (the scatter scans those 256 itself).
// Each thread owns a contiguous run of ceil(nb / 256) counters: one at
// N_t <= 1 Mi (a single CTA looping over all 256 x nb counters with a carried
// dependence took 50-60 us per pass at N_t = 1e6).
__global__ void __launch_bounds__(kDigits) k_sort_rowscan(uint32_t* __restrict__ hist, int nb,
                                                          uint32_t* __restrict__ rows) {
    __shared__ uint32_t wsum[kDigits / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* row = hist + (size_t)blockIdx.x * nb;
    const int per = (nb + kDigits - 1) / kDigits;
    const int beg = min((int)threadIdx.x * per, nb), end = min(beg + per, nb);
    uint32_t sum = 0;
    for (int i = beg; i < end; ++i) sum += row[i];
    uint32_t inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t base = 0, total = 0;
    for (int x = 0; x < kDigits / 32; ++x) {
        base += x < w ? wsum[x] : 0u;
        total += wsum[x];
    }
    uint32_t run = base + inc - sum;
    for (int i = beg; i < end; ++i) {
        const uint32_t v = row[i];
        row[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) rows[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kTileThreads) k_sort_scatter(const uint32_t* __restrict__ ks,
                                                               const int32_t* __restrict__ vs,
                                                               uint32_t* __restrict__ kd, int32_t* __restrict__ vd,
                                                               int n, int shift, const uint32_t* __restrict__ hist,
                                                               const uint32_t* __restrict__ rows) {
    __shared__ uint32_t wcnt[kTileWarps][kDigits + 1];
    __shared__ uint32_t dbase[kDigits];
    __shared__ uint32_t s_rows[kDigits];
    if (threadIdx.x < kDigits) s_rows[threadIdx.x] = rows[threadIdx.x];
    const int w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kTileWarps * (kDigits + 1); i += blockDim.x) (&wcnt[0][0])[i] = 0u;
    __syncthreads();
    const int tbeg = blockIdx.x * kTile;
    const int beg = min(tbeg + w * (kTile / kTileWarps), n);
    const int end = min(beg + kTile / kTileWarps, n);
    warp_count(ks, beg, end, shift, wcnt[w]);
    __syncthreads();
    if (w == 0) warp_scan256(s_rows);  // digit bases: exclusive scan of the row totals
    __syncthreads();
    if (threadIdx.x < kDigits) {
        uint32_t s = 0;
        for (int x = 0; x < kTileWarps; ++x) {
            uint32_t c = wcnt[x][threadIdx.x];
            wcnt[x][threadIdx.x] = s;
            s += c;
        }
        dbase[threadIdx.x] = s_rows[threadIdx.x] + hist[(size_t)threadIdx.x * gridDim.x + blockIdx.x];
    }
    __syncthreads();
    warp_scatter(ks, vs, kd, vd, beg, end, shift, wcnt[w], dbase);
}

// ------------------------------------------------------------------ A5: Karras topology
// delta(i, j): common-prefix length of the sorted codes; equal codes fall back
// to 32 + clz(i ^ j) (index augmentation); -1 out of range.
__device__ __forceinline__ int kdelta(const uint32_t* __restrict__ k, int n, int i, uint32_t ki, int j) {
    if (j < 0 || j >= n) return -1;
    uint32_t kj = k[j];
    return (ki == kj) ? 32 + __clz(i ^ j) : __clz(ki ^ kj);
}

__device__ __forceinline__ void set_ref(float4* nodes, int node, int side, int32_t ref) {
    reinterpret_cast<int32_t*>(nodes + 4 * node + 3)[side] = ref;
}

// One thread per internal node i in [0, n-2]: range direction, range end by
// exponential + binary search, split position gamma, children and parents.
__global__ void __launch_bounds__(kBlock) k_karras(const uint32_t* __restrict__ keys, int n,
                                                   float4* __restrict__ nodes, int32_t* __restrict__ parent,
                                                   uint32_t* __restrict__ arrivals, int32_t* sah_list,
                                                   uint32_t* scratch, int sah_max) {
    const int n_nodes = n > 1 ? n - 1 : 1;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (n == 1) {  // single triangle: root holds leaf 0 on the left, an unhittable point at +inf on the right
        if (i == 0) {
            float4* nd = nodes;
            nd[1] = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
            nd[2].z = INFINITY;
            nd[2].w = INFINITY;
            nd[3] = make_float4(__int_as_float(~0), __int_as_float(~0), 0.f, 0.f);
            parent[0] = -1;
            parent[n_nodes + 0] = 0;
            arrivals[0] = 2u;
        }
        return;
    }
    if (i >= n - 1) return;
    const uint32_t ki = keys[i];
    const int dir = (kdelta(keys, n, i, ki, i + 1) - kdelta(keys, n, i, ki, i - 1)) > 0 ? 1 : -1;
    const int dmin = kdelta(keys, n, i, ki, i - dir);
    int lmax = 2;
    while (kdelta(keys, n, i, ki, i + lmax * dir) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (kdelta(keys, n, i, ki, i + (l + t) * dir) > dmin) l += t;
    const int j = i + l * dir;
    const int dnode = kdelta(keys, n, i, ki, j);
    int s = 0, step = l;
    do {
        step = (step + 1) >> 1;
        int ns = s + step;
        if (ns < l && kdelta(keys, n, i, ki, i + ns * dir) > dnode) s = ns;
    } while (step > 1);
    const int gamma = i + s * dir + min(dir, 0);
    const int lo = min(i, j), hi = max(i, j);
    int32_t left = (lo == gamma) ? ~gamma : gamma;
    int32_t right = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    set_ref(nodes, i, 0, left);
    set_ref(nodes, i, 1, right);
    // leaf range of node i in the (otherwise unused) last two words: the refit
    // uses it to keep ascents inside a CTA's leaf window in shared memory
    reinterpret_cast<int32_t*>(nodes + 4 * i + 3)[2] = lo;
    reinterpret_cast<int32_t*>(nodes + 4 * i + 3)[3] = hi;
    parent[left >= 0 ? left : n_nodes + ~left] = (i << 1) | 0;
    parent[right >= 0 ? right : n_nodes + ~right] = (i << 1) | 1;
    if (i == 0) parent[0] = -1;
    if (sah_list) {  // the SAH subtree roots (k_sah_sub): maximal nodes of 3 .. sah_max leaves
        const int sz = hi - lo + 1, szl = gamma - lo + 1, szr = hi - gamma;
        if (i == 0 && sz <= sah_max) sah_list[atomicAdd(scratch + SCR_SAH_COUNT, 1u)] = 0;
        if (sz > sah_max) {  // (children of 1 or 2 leaves too: k_sah_sub packs and refits from every item)
            if (szl <= sah_max) sah_list[atomicAdd(scratch + SCR_SAH_COUNT, 1u)] = left;
            if (szr <= sah_max) sah_list[atomicAdd(scratch + SCR_SAH_COUNT, 1u)] = right;
        }
    }
}

// ------------------------------------------------------------------ A6 + A7: refit + pack
__device__ __forceinline__ void write_slot(float4* nodes, int node, int side, const float lo[3], const float hi[3]) {
    float* f = reinterpret_cast<float*>(nodes + 4 * node);
    int o = side ? 4 : 0;
    f[o + 0] = lo[0];
    f[o + 1] = hi[0];
    f[o + 2] = lo[1];
    f[o + 3] = hi[1];
    f[8 + 2 * side] = lo[2];
    f[9 + 2 * side] = hi[2];
}

// RSI_OPT_ROTATE: one local tree rotation at a node whose subtree is complete
// (Kensler-style, surface-area heuristic): swap one child with a grandchild on
// the other side when that shrinks the surface area of the rebuilt child box.
// The node's own leaf set and box are unchanged, so its ancestors are not
// affected; the moved subtrees get new parent links and the rebuilt child's
// slot box is the exact union of its new slots (the validator's invariants
// hold).  Reads use L2-coherent loads: children completed by other threads are
// ordered before us by the refit's barrier / acq_rel protocol.
__device__ __forceinline__ float box_area(const float lo[3], const float hi[3]) {
    const float dx = fmaxf(hi[0] - lo[0], 0.f), dy = fmaxf(hi[1] - lo[1], 0.f), dz = fmaxf(hi[2] - lo[2], 0.f);
    return dx * dy + dy * dz + dz * dx;
}
__device__ __forceinline__ void read_slot(const float4* nodes, int node, int side, float lo[3], float hi[3],
                                          int32_t& ref) {
    const float4* nd = nodes + 4 * node;
    const float4 a = __ldcg(nd + side), z = __ldcg(nd + 2), r = __ldcg(nd + 3);
    lo[0] = a.x; hi[0] = a.y; lo[1] = a.z; hi[1] = a.w;
    lo[2] = side ? z.z : z.x;
    hi[2] = side ? z.w : z.y;
    ref = __float_as_int(side ? r.y : r.x);
}
__device__ __forceinline__ void set_parent(int32_t* parent, int n_nodes, int32_t ref, int node, int side) {
    parent[ref >= 0 ? ref : n_nodes + ~ref] = (node << 1) | side;
}
__device__ void rotate_node(float4* nodes, int32_t* parent, int n_nodes, int node) {
    float Llo[3], Lhi[3], Rlo[3], Rhi[3];
    int32_t rL, rR;
    read_slot(nodes, node, 0, Llo, Lhi, rL);
    read_slot(nodes, node, 1, Rlo, Rhi, rR);
    float best = 0.f;
    int choice = -1;  // 0: L<->R0, 1: L<->R1, 2: R<->L0, 3: R<->L1
    float ulo[3], uhi[3];
    auto uni = [&](const float* alo, const float* ahi, const float* blo, const float* bhi) {
        for (int x = 0; x < 3; ++x) {
            ulo[x] = fminf(alo[x], blo[x]);
            uhi[x] = fmaxf(ahi[x], bhi[x]);
        }
        return box_area(ulo, uhi);
    };
    float R0lo[3], R0hi[3], R1lo[3], R1hi[3], L0lo[3], L0hi[3], L1lo[3], L1hi[3];
    int32_t rR0 = 0, rR1 = 0, rL0 = 0, rL1 = 0;
    if (rR >= 0) {
        read_slot(nodes, rR, 0, R0lo, R0hi, rR0);
        read_slot(nodes, rR, 1, R1lo, R1hi, rR1);
        const float cur = box_area(Rlo, Rhi);
        const float a = cur - uni(Llo, Lhi, R1lo, R1hi), b = cur - uni(R0lo, R0hi, Llo, Lhi);
        if (a > best) { best = a; choice = 0; }
        if (b > best) { best = b; choice = 1; }
    }
    if (rL >= 0) {
        read_slot(nodes, rL, 0, L0lo, L0hi, rL0);
        read_slot(nodes, rL, 1, L1lo, L1hi, rL1);
        const float cur = box_area(Llo, Lhi);
        const float c = cur - uni(Rlo, Rhi, L1lo, L1hi), d = cur - uni(L0lo, L0hi, Rlo, Rhi);
        if (c > best) { best = c; choice = 2; }
        if (d > best) { best = d; choice = 3; }
    }
    if (choice < 0) return;
    if (choice == 0) {  // node = (R0, R' = (L, R1))
        uni(Llo, Lhi, R1lo, R1hi);
        write_slot(nodes, node, 0, R0lo, R0hi);
        set_ref(nodes, node, 0, rR0);
        write_slot(nodes, node, 1, ulo, uhi);
        write_slot(nodes, rR, 0, Llo, Lhi);
        set_ref(nodes, rR, 0, rL);
        set_parent(parent, n_nodes, rR0, node, 0);
        set_parent(parent, n_nodes, rL, rR, 0);
    } else if (choice == 1) {  // node = (R1, R' = (R0, L))
        uni(R0lo, R0hi, Llo, Lhi);
        write_slot(nodes, node, 0, R1lo, R1hi);
        set_ref(nodes, node, 0, rR1);
        write_slot(nodes, node, 1, ulo, uhi);
        write_slot(nodes, rR, 1, Llo, Lhi);
        set_ref(nodes, rR, 1, rL);
        set_parent(parent, n_nodes, rR1, node, 0);
        set_parent(parent, n_nodes, rL, rR, 1);
    } else if (choice == 2) {  // node = (L' = (R, L1), L0)
        uni(Rlo, Rhi, L1lo, L1hi);
        write_slot(nodes, node, 1, L0lo, L0hi);
        set_ref(nodes, node, 1, rL0);
        write_slot(nodes, node, 0, ulo, uhi);
        write_slot(nodes, rL, 0, Rlo, Rhi);
        set_ref(nodes, rL, 0, rR);
        set_parent(parent, n_nodes, rL0, node, 1);
        set_parent(parent, n_nodes, rR, rL, 0);
    } else {  // node = (L' = (L0, R), L1)
        uni(L0lo, L0hi, Rlo, Rhi);
        write_slot(nodes, node, 1, L1lo, L1hi);
        set_ref(nodes, node, 1, rL1);
        write_slot(nodes, node, 0, ulo, uhi);
        write_slot(nodes, rL, 1, Rlo, Rhi);
        set_ref(nodes, rL, 1, rR);
        set_parent(parent, n_nodes, rL1, node, 1);
        set_parent(parent, n_nodes, rR, rL, 1);
    }
}

// ------------------------------------------------------------------ treelet restructuring (NEXT-4 tree quality)
// Karras & Aila's treelet restructuring (HPG 2013), fused into the refit's
// bottom-up climb inside each CTA window: when a window node n completes
// (second arrival), its treelet -- n's two children, then repeatedly the
// member with the largest surface area expanded into its two children, up to
// kTL members -- is rebuilt as the binary tree over those members that
// minimises the surface-area cost
//   C(node) = kCi A(node) + C(left) + C(right),  C(triangle) = kCt A(triangle)
// by exact dynamic programming over the member subsets.  The thread that
// completed n does it alone, on the window's shared-memory mirror of its
// nodes, with the DP fully unrolled in registers (kTL = 5: 31 subsets, 90
// partitions).  Only n's subtree changes: n keeps its box and leaf set, the
// rebuilt internal nodes reuse the treelet's node ids, every slot box is the
// exact fp32 union of its members' boxes, and parent links are rewritten --
// so the validator's invariants hold and traversal results are unchanged
// (the BVH only prunes).  Nodes above the windows keep the Karras topology:
// measured, their treelets cost as much rebuild time as all the windows'
// (a serial chain through global memory) and removed 0.5 % of the box tests.
// Measured (sphere N_t = 1e4, 1.25e7 segments): box tests per segment
// 34.7 -> 33.4, query -3.5 % (boolean) .. -3 % (count), rebuild +50 us before
// the shared-memory mirror.  The Karras topology itself (the
// paper's Fig. 3 structure) is kept with RSI_OPT_PLAIN_TREE.
#ifndef RSI_TREELET
#define RSI_TREELET 5  // treelet members (0: off; 3..5)
#endif
constexpr int kTL = RSI_TREELET;
// meshes up to this many triangles: there the rebuild is a latency chain and the
// treelets add ~35 us for -3.5 % traversal (sphere N_t = 1e4, 1.25e7 segments);
// at N_t = 1e6 they are throughput work over 4000 windows (+1.16 ms rebuild for
// -2.3 % traversal), so large meshes keep the Karras topology
#ifndef RSI_TREELET_MAX_TRI
#define RSI_TREELET_MAX_TRI 65536
#endif
constexpr int kTreeletMaxTri = RSI_TREELET_MAX_TRI;
#ifndef RSI_TREELET_MIN
#define RSI_TREELET_MIN 3  // smallest treelet rebuilt (members)
#endif
static_assert(kTL == 0 || (kTL >= 3 && kTL <= 5), "RSI_TREELET");
constexpr int kTLm = kTL > 0 ? kTL : 3;
constexpr float kCi = 1.2f, kCt = 1.0f;  // SAH constants (node visit vs triangle)

// The refit window's view of its nodes (every node a window treelet touches
// lies in the window): slot boxes, child refs and subtree costs mirrored in
// shared memory -- a treelet reads only shared memory -- while every rebuilt
// slot is written through to the global records and parent links.
struct WindowTree {
    float4* nodes;
    int32_t* parent;
    int n_nodes, c0;
    float (*box)[2][6];  // s_box: slot boxes (lo xyz, hi xyz) of window node c0 + i
    int32_t (*ref)[2];   // s_ref: its child refs
    float* cost;         // s_cost: its subtree cost
    __device__ __forceinline__ void read(int node, int side, float lo[3], float hi[3], int32_t& r) const {
        const float* b = box[node - c0][side];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            lo[x] = b[x];
            hi[x] = b[3 + x];
        }
        r = ref[node - c0][side];
    }
    __device__ __forceinline__ float member_cost(int32_t r, const float lo[3], const float hi[3]) const {
        return r < 0 ? kCt * box_area(lo, hi) : cost[r - c0];
    }
    __device__ __forceinline__ void write(int node, int side, const float lo[3], const float hi[3], int32_t r) const {
        write_slot(nodes, node, side, lo, hi);
        set_ref(nodes, node, side, r);
        set_parent(parent, n_nodes, r, node, side);
        float* b = box[node - c0][side];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            b[x] = lo[x];
            b[3 + x] = hi[x];
        }
        ref[node - c0][side] = r;
    }
    __device__ __forceinline__ void set_cost(int node, float c) const { cost[node - c0] = c; }
};

// Optimal binary tree over K members (K compile-time: the loops unroll, the
// subset / partition masks become constants and every array index is static,
// so the DP runs in registers): returns the least cost of the full set and
// leaves, for every subset s, its left part (the part holding s's lowest
// member) in popt[s] -- one shared-memory row per thread, read back by the
// reconstruction.
template <int K>
__device__ __forceinline__ float treelet_dp(const float (&lo)[kTLm][3], const float (&hi)[kTLm][3],
                                            const float (&lc)[kTLm], unsigned char* row_popt) {
    constexpr int F = (1 << K) - 1;
    float copt[F + 1];
#pragma unroll
    for (int s = 1; s <= F; ++s) {
        if ((s & (s - 1)) == 0) {
            copt[s] = lc[__ffs(s) - 1];
            continue;
        }
        float blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < K; ++i)
            if ((s >> i) & 1)
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    blo[x] = fminf(blo[x], lo[i][x]);
                    bhi[x] = fmaxf(bhi[x], hi[i][x]);
                }
        float best = INFINITY;
        int bp = s & -s;
#pragma unroll
        for (int p = 1; p < s; ++p) {
            if ((p & s) != p || !(p & (s & -s))) continue;
            const float v = copt[p] + copt[s ^ p];
            bp = v < best ? p : bp;
            best = fminf(best, v);
        }
        copt[s] = kCi * box_area(blo, bhi) + best;
        row_popt[s] = (unsigned char)bp;
    }
    return copt[F];
}

// The thread that completed node n restructures n's treelet.  Member arrays
// are indexed statically (unrolled loops with selects) so they stay in
// registers; the DP's partition table lives in this thread's shared-memory row.
template <class Tree>
__device__ void treelet_opt(const Tree& tr, int n, unsigned char* row_popt) {
    float lo[kTLm][3], hi[kTLm][3], lc[kTLm];
    int32_t ref[kTLm], ids[kTLm];
    tr.read(n, 0, lo[0], hi[0], ref[0]);
    tr.read(n, 1, lo[1], hi[1], ref[1]);
    float nlo[3], nhi[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
        nlo[x] = fminf(lo[0][x], lo[1][x]);
        nhi[x] = fmaxf(hi[0][x], hi[1][x]);
    }
    const float cur = kCi * box_area(nlo, nhi) + tr.member_cost(ref[0], lo[0], hi[0]) + tr.member_cost(ref[1], lo[1], hi[1]);
    int k = 2;
    ids[0] = n;
#pragma unroll
    for (int e = 0; e < kTL - 2; ++e) {  // expansion e: the internal member with the largest area -> members bi, 2 + e
        int bi = -1;
        float ba = -1.0f;
#pragma unroll
        for (int i = 0; i < 2 + e; ++i)
            if (ref[i] >= 0) {
                const float a = box_area(lo[i], hi[i]);
                if (a > ba) {
                    ba = a;
                    bi = i;
                }
            }
        if (bi < 0) break;
        int m = 0;
#pragma unroll
        for (int i = 0; i < 2 + e; ++i) m = i == bi ? ref[i] : m;
        ids[1 + e] = m;
        float l0[3], h0[3];
        int32_t r0;
        tr.read(m, 0, l0, h0, r0);
        tr.read(m, 1, lo[2 + e], hi[2 + e], ref[2 + e]);
#pragma unroll
        for (int i = 0; i < 2 + e; ++i)
            if (i == bi) {
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    lo[i][x] = l0[x];
                    hi[i][x] = h0[x];
                }
                ref[i] = r0;
            }
        k = 3 + e;
    }
    if (k < (RSI_TREELET_MIN > 3 ? RSI_TREELET_MIN : 3)) {  // two members: one topology
        tr.set_cost(n, cur);
        return;
    }
#pragma unroll
    for (int i = 0; i < kTLm; ++i)
        if (i < k) lc[i] = tr.member_cost(ref[i], lo[i], hi[i]);
    float best;
    if (kTL >= 5 && k == 5)
        best = treelet_dp<(kTL >= 5 ? 5 : 3)>(lo, hi, lc, row_popt);
    else if (kTL >= 4 && k == 4)
        best = treelet_dp<(kTL >= 4 ? 4 : 3)>(lo, hi, lc, row_popt);
    else
        best = treelet_dp<3>(lo, hi, lc, row_popt);
    if (!(best < cur * (1.0f - 1e-5f))) {
        tr.set_cost(n, cur);
        return;
    }
    // rebuild n's subtree from the optimal partitions (breadth-first; internal
    // nodes reuse ids[] in order, n first)
    unsigned q_s[kTLm - 1];
    int q_id[kTLm - 1];
    q_s[0] = (1u << k) - 1u;
    q_id[0] = n;
    int qn = 1;
#pragma unroll
    for (int it = 0; it < kTLm - 1; ++it) {
        if (it >= qn) break;
        const unsigned s = q_s[it];
        const int id = q_id[it];
        const unsigned ps = row_popt[s];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const unsigned c = side ? s ^ ps : ps;
            float blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
            int32_t r = 0;
#pragma unroll
            for (int i = 0; i < kTLm; ++i)
                if ((c >> i) & 1u) {
                    r = ref[i];
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        blo[x] = fminf(blo[x], lo[i][x]);
                        bhi[x] = fmaxf(bhi[x], hi[i][x]);
                    }
                }
            if (c & (c - 1u)) {  // an internal node: the next id, queued
#pragma unroll
                for (int j = 1; j < kTLm; ++j) r = j == qn ? ids[j] : r;
#pragma unroll
                for (int j = 1; j < kTLm - 1; ++j)
                    if (j == qn) {
                        q_s[j] = c;
                        q_id[j] = r;
                    }
                ++qn;
            }
            tr.write(id, side, blo, bhi, r);
        }
    }
    // subtree costs of the rebuilt nodes, children (later in the queue) first
    float q_c[kTLm - 1];
#pragma unroll
    for (int it = kTLm - 2; it >= 0; --it) {
        if (it >= qn) continue;
        const unsigned s = q_s[it], ps = row_popt[s];
        float blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < kTLm; ++i)
            if ((s >> i) & 1u)
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    blo[x] = fminf(blo[x], lo[i][x]);
                    bhi[x] = fmaxf(bhi[x], hi[i][x]);
                }
        float c = kCi * box_area(blo, bhi);
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const unsigned ch = side ? s ^ ps : ps;
            float cc = 0.0f;
            if (ch & (ch - 1u)) {
#pragma unroll
                for (int j = it + 1; j < kTLm - 1; ++j) cc = (j < qn && q_s[j] == ch) ? q_c[j] : cc;
            } else {
#pragma unroll
                for (int i = 0; i < kTLm; ++i) cc = ch == (1u << i) ? lc[i] : cc;
            }
            c += cc;
        }
        q_c[it] = c;
        tr.set_cost(q_id[it], c);
    }
}

// ------------------------------------------------------------------ NEXT-4 tree quality: SAH subtrees
// RSI_SAH_SUB (default for N_t <= kSahMaxTri; off under RSI_OPT_PLAIN_TREE /
// ROTATE / APETREI): every maximal Karras subtree with <= kSahSub leaves (a
// node of <= kSahSub leaves whose parent has more) is rebuilt top-down by
// binned SAH over its triangles' centroids, between k_karras and k_refit.  The
// Karras topology stays above these subtrees (A5 is still the tree's top), and
// every node still covers a CONTIGUOUS range of leaf slots (a top-down
// partition of the subtree's slot range, the triangles permuted inside it),
// numbered the Karras way: an internal left child takes the last slot of its
// range, a right child the first.  For any such tree over a range that
// numbering is a bijection onto the node ids the Karras subtree used (ids
// [a+1, b] when its root is a left child, else [a, b-1]; the root keeps its id
// and parent link), so k_refit's windows, parent links and leaf ranges work
// unchanged.  One CTA (kSahWarps warps) per subtree: the nodes of a level one
// per warp -- centroid bounds by REDUX, kSahBins bins per axis filled with
// shared-memory atomics (boxes as order-preserving uint32 keys), every plane of
// every axis scanned at once (one lane per (axis, bin)), a warp-ordered stable
// partition -- and every node of <= kSahSmall triangles by ONE thread with the
// exact SAH-optimal topology (treelet_dp).
// Measured (sphere N_t = 1e4, 1e7 segments): box tests per
// segment -4 % (boolean) .. -6 % (intercept_count), query -3.4 / -4.7 / -5.6 %
// (boolean / barycentric / intercept_count), paper terrain -6.8 / -12 / -16 %;
// rebuild 0.126 -> 0.130 ms with the refit's treelets switched off (they add
// nothing on top: same query time).  Host-built trees walked by the same
// kernels (tools/tree_upload.py) bound what SAH quality can give: full binned
// SAH -8 .. -11 %.  At N_t = 1e6 the rebuild grows 0.74 -> 1.9 ms, hence the gate.
#ifndef RSI_SAH_SUB
#define RSI_SAH_SUB 256  // leaves per rebuilt subtree (0: off); 128 / 512: rebuild -11 / +27 us, query +0.2 / -0.7 %
#endif
#ifndef RSI_SAH_MAX_TRI
#define RSI_SAH_MAX_TRI 32768
#endif
constexpr int64_t kSahMaxTri = RSI_SAH_MAX_TRI;
constexpr int64_t kSahMinTri = 64;  // smaller meshes: the launch is not worth it
constexpr int kSahSub = RSI_SAH_SUB > 0 ? RSI_SAH_SUB : 4;
#ifndef RSI_SAH_BINS
#define RSI_SAH_BINS 10  // bins per axis (3 x 10 <= 32 lanes: every plane of every axis in one warp pass)
#endif
constexpr int kSahWarps = 32;
constexpr int kSahBins = RSI_SAH_BINS;
constexpr int kSahGrid = 148;  // persistent CTAs (one per SM) over the subtree list
static_assert(kSahSub <= 65535 && (kSahSub & (kSahSub - 1)) == 0, "RSI_SAH_SUB");

__device__ __forceinline__ uint32_t fkey(float f) {  // order-preserving float -> uint32
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fdekey(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Shared memory of k_sah_sub (dynamic): the subtree's boxes and 3 x centroids,
// triangle ids, the permutation (double-buffered), the level task lists and
// one bin array per warp.
constexpr int kSahBinSlots = 3 * kSahBins;  // (axis, bin) pairs: one lane each in the SAH scan
static_assert(kSahBinSlots <= 32, "RSI_SAH_BINS");
constexpr int kSahSmall = kTLm;  // nodes of <= kSahSmall triangles: one THREAD each, exact SAH over every
                                 // topology (treelet_dp) instead of a warp's binned split per level
constexpr size_t kSahSmem = (size_t)18 * kSahSub * sizeof(float) + (size_t)kSahSub * sizeof(int32_t) +
                            (size_t)2 * kSahSub * sizeof(uint16_t) + (size_t)3 * (kSahSub / 2) * 3 * sizeof(int) +
                            (size_t)kSahWarps * kSahBinSlots * 7 * sizeof(uint32_t) +
                            (size_t)32 * kSahWarps * 32 + 4 * sizeof(int) + 8 * sizeof(float);

// The global refit protocol of k_refit (state 3) from a completed subtree whose
// box is (lo, hi) and whose parent link is p: the box goes into the parent's
// child slot, an acq_rel arrival on the parent's counter (first arrival stops),
// the second merges the sibling's slot (L2-coherent loads) and climbs on; the
// arrival at the root writes the scene box.
__device__ void refit_climb(float4* nodes, const int32_t* parent, uint32_t* arrivals, uint32_t* scratch, int32_t p,
                            float lo[3], float hi[3]) {
    if (p >= 0) {
        write_slot(nodes, p >> 1, p & 1, lo, hi);
        while (true) {
            const int node = p >> 1, side = p & 1;
            const int32_t p_next = node > 0 ? __ldg(parent + node) : -1;
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(arrivals + node) : "memory");
            if (old == 0u) return;
            const float* f = reinterpret_cast<const float*>(nodes + 4 * node);
            const int o = side ? 0 : 4;  // sibling slot
            lo[0] = fminf(lo[0], __ldcg(f + o + 0));
            hi[0] = fmaxf(hi[0], __ldcg(f + o + 1));
            lo[1] = fminf(lo[1], __ldcg(f + o + 2));
            hi[1] = fmaxf(hi[1], __ldcg(f + o + 3));
            lo[2] = fminf(lo[2], __ldcg(f + 8 + 2 * (1 - side)));
            hi[2] = fmaxf(hi[2], __ldcg(f + 9 + 2 * (1 - side)));
            if (node == 0) break;
            p = p_next;
            write_slot(nodes, p >> 1, p & 1, lo, hi);
        }
    }
    float* root = reinterpret_cast<float*>(scratch + SCR_ROOT);
    for (int x = 0; x < 3; ++x) {
        root[x] = lo[x];
        root[3 + x] = hi[x];
    }
    scratch[SCR_ROOT_SET] = 1u;
}

// A node of k <= kSahSmall triangles (slots [a + s, a + e), node id nid): the
// SAH-optimal binary tree over them (treelet_dp: every topology), written with
// its leaves in depth-first order and the Karras numbering.
__device__ void sah_small(int a, int s, int e, int nid, const float* s_lo, const float* s_hi, uint16_t* pm,
                          float4* nodes, int32_t* parent, uint32_t* arrivals, int n_nodes, unsigned char* row_popt,
                          float* set_box, int box_id) {
    const int k = e - s;
    float lo[kTLm][3], hi[kTLm][3], lc[kTLm];
    int q[kTLm];
#pragma unroll
    for (int i = 0; i < kTLm; ++i) {
        q[i] = i < k ? pm[s + i] : 0;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            lo[i][x] = i < k ? s_lo[x * kSahSub + q[i]] : 0.0f;
            hi[i][x] = i < k ? s_hi[x * kSahSub + q[i]] : 0.0f;
        }
        lc[i] = kCt * box_area(lo[i], hi[i]);
    }
    if (k == 2) {
        row_popt[3] = 1;
    } else if (kTLm >= 5 && k == 5) {
        treelet_dp<(kTLm >= 5 ? 5 : 3)>(lo, hi, lc, row_popt);
    } else if (kTLm >= 4 && k == 4) {
        treelet_dp<(kTLm >= 4 ? 4 : 3)>(lo, hi, lc, row_popt);
    } else {
        treelet_dp<3>(lo, hi, lc, row_popt);
    }
    // depth-first: (member set, first slot, node id); the left part holds the lowest member
    int st_set[kTLm], st_lo[kTLm], st_id[kTLm], sp = 0;
    uint16_t out[kTLm];
    st_set[0] = (1 << k) - 1;
    st_lo[0] = a + s;
    st_id[0] = nid;
    sp = 1;
    while (sp > 0) {
        --sp;
        const int set = st_set[sp], l0 = st_lo[sp], id = st_id[sp];
        const int pl = row_popt[set], pr = set ^ pl;
        const int nl = __popc(pl), nr = __popc(pr);
        const int32_t left = nl == 1 ? ~l0 : l0 + nl - 1;
        const int32_t right = nr == 1 ? ~(l0 + nl) : l0 + nl;
        *reinterpret_cast<int4*>(nodes + 4 * id + 3) = make_int4(left, right, l0, l0 + nl + nr - 1);
        parent[left >= 0 ? left : n_nodes + ~left] = (id << 1) | 0;
        parent[right >= 0 ? right : n_nodes + ~right] = (id << 1) | 1;
        {  // the two child boxes (exact unions of the members' boxes); the node is complete
            float bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
            float cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < kTLm; ++i)
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    if ((pl >> i) & 1) { bl[x] = fminf(bl[x], lo[i][x]); bh[x] = fmaxf(bh[x], hi[i][x]); }
                    if ((pr >> i) & 1) { cl[x] = fminf(cl[x], lo[i][x]); ch[x] = fmaxf(ch[x], hi[i][x]); }
                }
            write_slot(nodes, id, 0, bl, bh);
            write_slot(nodes, id, 1, cl, ch);
            arrivals[id] = 2u;
            if (set_box && id == box_id)  // the subtree's root: its box starts the refit above
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    set_box[x] = fminf(bl[x], cl[x]);
                    set_box[3 + x] = fmaxf(bh[x], ch[x]);
                }
        }
        if (nl == 1) out[l0 - (a + s)] = (uint16_t)q[__ffs(pl) - 1];
        if (nr == 1) out[l0 + nl - (a + s)] = (uint16_t)q[__ffs(pr) - 1];
        // right first on the stack so the left subtree is expanded next (slots are explicit anyway)
        if (nr >= 2) {
            st_set[sp] = pr;
            st_lo[sp] = l0 + nl;
            st_id[sp] = right;
            ++sp;
        }
        if (nl >= 2) {
            st_set[sp] = pl;
            st_lo[sp] = l0;
            st_id[sp] = left;
            ++sp;
        }
    }
    for (int i = 0; i < k; ++i) pm[s + i] = out[i];
}

__global__ void __launch_bounds__(32 * kSahWarps, 1) k_sah_sub(const float* __restrict__ V, int64_t nv,
                                                               const int32_t* __restrict__ T, int32_t* vals,
                                                               float4* nodes, float4* __restrict__ tris, int32_t* parent,
                                                               uint32_t* arrivals, int n_nodes,
                                                               const int32_t* __restrict__ list, uint32_t* scratch) {
    extern __shared__ uint4 s_sah_dyn[];
    float* s_f = reinterpret_cast<float*>(s_sah_dyn);
    float* s_lo = s_f;                   // [3][kSahSub]
    float* s_hi = s_f + 3 * kSahSub;     // [3][kSahSub]
    float* s_c = s_f + 6 * kSahSub;      // [3][kSahSub]  (3 x centroid)
    float* s_v = s_f + 9 * kSahSub;      // [9][kSahSub]  the vertices (the triangle records are packed here)
    int32_t* s_id = reinterpret_cast<int32_t*>(s_f + 18 * kSahSub);
    uint16_t* s_perm = reinterpret_cast<uint16_t*>(s_id + kSahSub);  // [2][kSahSub]
    int* s_task = reinterpret_cast<int*>(s_perm + 2 * kSahSub);      // [2][kSahSub / 2][3]
    int* s_small = s_task + 2 * (kSahSub / 2) * 3;                                   // [kSahSub / 2][3]
    uint32_t* s_bins = reinterpret_cast<uint32_t*>(s_small + (kSahSub / 2) * 3);     // [warps][slots][7]
    unsigned char* s_popt = reinterpret_cast<unsigned char*>(s_bins + kSahWarps * kSahBinSlots * 7);  // [threads][32]
    int* s_ntask = reinterpret_cast<int*>(s_popt + 32 * kSahWarps * 32);             // [2], then the small count
    float* s_rbox = reinterpret_cast<float*>(s_ntask + 4);                           // [6] the subtree's box
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int n_sub = (int)scratch[SCR_SAH_COUNT];
    uint32_t* bins = s_bins + warp * kSahBinSlots * 7;
    // this lane's (axis, bin) pair in the SAH scan
    const int my_ax = lane / kSahBins, my_b = lane % kSahBins;
    const bool my_in = lane < kSahBinSlots;
    for (int si = blockIdx.x; si < n_sub; si += gridDim.x) {
        const int root = list[si];
        // ---- a leaf, or a node of two leaves, under a Karras node of more than
        // kSahSub leaves: pack its triangle(s) and refit upwards from it (one thread)
        const int4 rr = root >= 0 ? *reinterpret_cast<const int4*>(nodes + 4 * root + 3) : make_int4(0, 0, 0, 0);
        if (root < 0 || rr.w - rr.z + 1 <= 2) {
            if (threadIdx.x == 0) {
                const int k0 = root < 0 ? ~root : rr.z, kn = root < 0 ? 1 : 2;
                float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
                for (int j = 0; j < kn; ++j) {
                    const int k = k0 + j;
                    const int32_t id = vals[k];
                    const int32_t i0 = safe_index(T[3 * id], nv), i1 = safe_index(T[3 * id + 1], nv),
                                  i2 = safe_index(T[3 * id + 2], nv);
                    float a3[3], b3[3], c3[3], l[3], h[3];
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        a3[x] = V[3 * i0 + x];
                        b3[x] = V[3 * i1 + x];
                        c3[x] = V[3 * i2 + x];
                        l[x] = fminf(a3[x], fminf(b3[x], c3[x]));
                        h[x] = fmaxf(a3[x], fmaxf(b3[x], c3[x]));
                        lo[x] = fminf(lo[x], l[x]);
                        hi[x] = fmaxf(hi[x], h[x]);
                    }
                    tris[kTriF4 * k + 0] = make_float4(a3[0], a3[1], a3[2], __int_as_float(id));
                    tris[kTriF4 * k + 1] = make_float4(b3[0], b3[1], b3[2], 0.f);
                    tris[kTriF4 * k + 2] = make_float4(c3[0], c3[1], c3[2], 0.f);
                    if (kTriF4 == 4) tris[4 * k + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (kn == 2) write_slot(nodes, root, j, l, h);
                }
                if (kn == 2) arrivals[root] = 2u;
                refit_climb(nodes, parent, arrivals, scratch, root < 0 ? parent[n_nodes + ~root] : parent[root], lo, hi);
            }
            continue;
        }
        const int a = rr.z, m = rr.w - rr.z + 1;
        // the subtree's triangles: vertices, exact fp32 boxes and centroids (x 3)
        for (int t = threadIdx.x; t < m; t += blockDim.x) {
            const int32_t id = vals[a + t];
            const int32_t i0 = safe_index(T[3 * id], nv), i1 = safe_index(T[3 * id + 1], nv),
                          i2 = safe_index(T[3 * id + 2], nv);
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                const float p0 = V[3 * i0 + x], p1 = V[3 * i1 + x], p2 = V[3 * i2 + x];
                s_lo[x * kSahSub + t] = fminf(p0, fminf(p1, p2));
                s_hi[x * kSahSub + t] = fmaxf(p0, fmaxf(p1, p2));
                s_c[x * kSahSub + t] = (p0 + p1) + p2;
                s_v[x * kSahSub + t] = p0;
                s_v[(3 + x) * kSahSub + t] = p1;
                s_v[(6 + x) * kSahSub + t] = p2;
            }
            s_id[t] = id;
            s_perm[t] = (uint16_t)t;
        }
        if (threadIdx.x == 0) {
            const bool small = m <= kSahSmall;
            int* t0 = small ? s_small : s_task;
            t0[0] = 0;
            t0[1] = m;
            t0[2] = root;
            s_ntask[0] = small ? 0 : 1;
            s_ntask[1] = 0;
            s_ntask[2] = small ? 1 : 0;
        }
        __syncthreads();
        int cur = 0;
        while (true) {
            const int nt = s_ntask[cur];
            if (nt == 0) break;
            const int* tl = s_task + cur * (kSahSub / 2) * 3;
            for (int ti = warp; ti < nt; ti += kSahWarps) {
                const int s = tl[3 * ti], e = tl[3 * ti + 1], nid = tl[3 * ti + 2];
                const int k = e - s;
                uint16_t* pm = s_perm;
                uint16_t* pt = s_perm + kSahSub;
                int nl = k >> 1;  // fallback: median of the current order
                int best_ax = -1, best_b = 0;
                float cmin[3] = {0.0f, 0.0f, 0.0f}, scale[3] = {0.0f, 0.0f, 0.0f};
                if (k > 2) {
                    // centroid bounds: order-preserving keys, one REDUX per bound
                    uint32_t kmin[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, kmax[3] = {0u, 0u, 0u};
#pragma unroll 4
                    for (int j = s + lane; j < e; j += 32) {
                        const int q = pm[j];
#pragma unroll
                        for (int x = 0; x < 3; ++x) {
                            const uint32_t kc = fkey(s_c[x * kSahSub + q]);
                            kmin[x] = min(kmin[x], kc);
                            kmax[x] = max(kmax[x], kc);
                        }
                    }
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        cmin[x] = fdekey(__reduce_min_sync(FULL, kmin[x]));
                        const float w = fdekey(__reduce_max_sync(FULL, kmax[x])) - cmin[x];
                        const float sv = __fdividef((float)kSahBins, w);  // any value: binning and partition share it
                        scale[x] = (w > 0.0f && sv < 1e30f) ? sv : 0.0f;  // degenerate / non-finite axis: not split
                    }
                }
                if (k > 2 && (scale[0] > 0.0f || scale[1] > 0.0f || scale[2] > 0.0f)) {
                    for (int w = lane; w < kSahBinSlots * 7; w += 32) {
                        const int f = w % 7;
                        bins[w] = f == 0 ? 0u : (f <= 3 ? 0xffffffffu : 0u);
                    }
                    __syncwarp();
#pragma unroll 4
                    for (int j = s + lane; j < e; j += 32) {
                        const int q = pm[j];
                        const uint32_t l0 = fkey(s_lo[q]), l1 = fkey(s_lo[kSahSub + q]), l2 = fkey(s_lo[2 * kSahSub + q]);
                        const uint32_t h0 = fkey(s_hi[q]), h1 = fkey(s_hi[kSahSub + q]), h2 = fkey(s_hi[2 * kSahSub + q]);
#pragma unroll
                        for (int x = 0; x < 3; ++x) {
                            if (scale[x] == 0.0f) continue;
                            const int b = max(0, min(kSahBins - 1, (int)((s_c[x * kSahSub + q] - cmin[x]) * scale[x])));
                            uint32_t* bb = bins + (x * kSahBins + b) * 7;
                            atomicAdd(bb, 1u);
                            atomicMin(bb + 1, l0);
                            atomicMin(bb + 2, l1);
                            atomicMin(bb + 3, l2);
                            atomicMax(bb + 4, h0);
                            atomicMax(bb + 5, h1);
                            atomicMax(bb + 6, h2);
                        }
                    }
                    __syncwarp();
                    // SAH over every (axis, plane) at once: lane = axis * kSahBins + bin;
                    // inclusive prefix / suffix over the axis's bins by segmented shuffles
                    const uint32_t* bb = bins + (my_in ? lane : 0) * 7;
                    const float sc_ax = my_ax == 0 ? scale[0] : (my_ax == 1 ? scale[1] : scale[2]);
                    const bool act = my_in && sc_ax > 0.0f;
                    const uint32_t cnt = act ? bb[0] : 0u;
                    float plo[3], phi[3], slo[3], shi[3];
#pragma unroll
                    for (int y = 0; y < 3; ++y) {
                        plo[y] = slo[y] = cnt ? fdekey(bb[1 + y]) : INFINITY;
                        phi[y] = shi[y] = cnt ? fdekey(bb[4 + y]) : -INFINITY;
                    }
                    uint32_t pc = cnt, scn = cnt;
#pragma unroll
                    for (int o = 1; o < kSahBins; o <<= 1) {
                        const uint32_t uc = __shfl_up_sync(FULL, pc, o), dc = __shfl_down_sync(FULL, scn, o);
                        const bool up = my_b >= o, dn = my_b + o < kSahBins;
                        pc += up ? uc : 0u;
                        scn += dn ? dc : 0u;
#pragma unroll
                        for (int y = 0; y < 3; ++y) {
                            const float ul = __shfl_up_sync(FULL, plo[y], o), uh = __shfl_up_sync(FULL, phi[y], o);
                            const float dl = __shfl_down_sync(FULL, slo[y], o), dh = __shfl_down_sync(FULL, shi[y], o);
                            if (up) { plo[y] = fminf(plo[y], ul); phi[y] = fmaxf(phi[y], uh); }
                            if (dn) { slo[y] = fminf(slo[y], dl); shi[y] = fmaxf(shi[y], dh); }
                        }
                    }
                    // plane after bin b: left = prefix(b), right = suffix(b + 1)
                    const uint32_t rc = __shfl_down_sync(FULL, scn, 1);
                    float rlo[3], rhi[3];
#pragma unroll
                    for (int y = 0; y < 3; ++y) {
                        rlo[y] = __shfl_down_sync(FULL, slo[y], 1);
                        rhi[y] = __shfl_down_sync(FULL, shi[y], 1);
                    }
                    float cost = INFINITY;
                    if (act && my_b < kSahBins - 1 && pc > 0u && rc > 0u) {
                        const float lx = phi[0] - plo[0], ly = phi[1] - plo[1], lz = phi[2] - plo[2];
                        const float rx = rhi[0] - rlo[0], ry = rhi[1] - rlo[1], rz = rhi[2] - rlo[2];
                        cost = (lx * ly + ly * lz + lz * lx) * (float)pc + (rx * ry + ry * rz + rz * rx) * (float)rc;
                    }
                    // warp argmin (ties: lowest lane), as one 64-bit key: cost bits (>= 0) | lane
                    const unsigned long long key =
                        ((unsigned long long)__float_as_uint(cost) << 32) | (unsigned)lane;
                    unsigned long long bk = key;
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const unsigned long long ok = __shfl_xor_sync(FULL, bk, o);
                        bk = ok < bk ? ok : bk;
                    }
                    const int bl = (int)(bk & 31u);
                    const int ncl = __shfl_sync(FULL, (int)pc, bl);
                    if (__uint_as_float((uint32_t)(bk >> 32)) < INFINITY) {
                        best_ax = bl / kSahBins;
                        best_b = bl % kSahBins;
                        nl = ncl;
                        // the children's boxes are the best plane's prefix / suffix bin unions
                        if (lane == bl) {
                            write_slot(nodes, nid, 0, plo, phi);
                            write_slot(nodes, nid, 1, rlo, rhi);
                            if (nid == root)
#pragma unroll
                                for (int y = 0; y < 3; ++y) {
                                    s_rbox[y] = fminf(plo[y], rlo[y]);
                                    s_rbox[3 + y] = fmaxf(phi[y], rhi[y]);
                                }
                        }
                    }
                }
                if (best_ax < 0) {  // median split: the children's boxes by warp reductions
                    float bl3[3] = {INFINITY, INFINITY, INFINITY}, bh3[3] = {-INFINITY, -INFINITY, -INFINITY};
                    float cl3[3] = {INFINITY, INFINITY, INFINITY}, ch3[3] = {-INFINITY, -INFINITY, -INFINITY};
                    for (int j = s + lane; j < e; j += 32) {
                        const int q = pm[j];
                        const bool lft = j < s + nl;
#pragma unroll
                        for (int y = 0; y < 3; ++y) {
                            const float l = s_lo[y * kSahSub + q], h = s_hi[y * kSahSub + q];
                            if (lft) { bl3[y] = fminf(bl3[y], l); bh3[y] = fmaxf(bh3[y], h); }
                            else { cl3[y] = fminf(cl3[y], l); ch3[y] = fmaxf(ch3[y], h); }
                        }
                    }
#pragma unroll
                    for (int y = 0; y < 3; ++y) {
                        bl3[y] = fdekey(__reduce_min_sync(FULL, fkey(bl3[y])));
                        bh3[y] = fdekey(__reduce_max_sync(FULL, fkey(bh3[y])));
                        cl3[y] = fdekey(__reduce_min_sync(FULL, fkey(cl3[y])));
                        ch3[y] = fdekey(__reduce_max_sync(FULL, fkey(ch3[y])));
                    }
                    if (lane == 0) {
                        write_slot(nodes, nid, 0, bl3, bh3);
                        write_slot(nodes, nid, 1, cl3, ch3);
                        if (nid == root)
#pragma unroll
                            for (int y = 0; y < 3; ++y) {
                                s_rbox[y] = fminf(bl3[y], cl3[y]);
                                s_rbox[3 + y] = fmaxf(bh3[y], ch3[y]);
                            }
                    }
                }
                // partition the node's slice of the permutation (warp-ordered, stable)
                {
                    const float cm = best_ax == 0 ? cmin[0] : (best_ax == 1 ? cmin[1] : cmin[2]);
                    const float sc = best_ax == 0 ? scale[0] : (best_ax == 1 ? scale[1] : scale[2]);
                    const float* cax = s_c + (best_ax > 0 ? best_ax : 0) * kSahSub;
                    int base_l = s, base_r = s + nl;
#pragma unroll 4
                    for (int j0 = s; j0 < e; j0 += 32) {
                        const int j = j0 + lane;
                        const bool v = j < e;
                        const int q = v ? pm[j] : 0;
                        const bool left = best_ax >= 0
                                              ? max(0, min(kSahBins - 1, (int)((cax[q] - cm) * sc))) <= best_b
                                              : j < s + nl;
                        const unsigned bl = __ballot_sync(FULL, v && left), br = __ballot_sync(FULL, v && !left);
                        if (v) pt[left ? base_l + __popc(bl & lt) : base_r + __popc(br & lt)] = (uint16_t)q;
                        base_l += __popc(bl);
                        base_r += __popc(br);
                    }
                    __syncwarp();
#pragma unroll 4
                    for (int j = s + lane; j < e; j += 32) pm[j] = pt[j];
                    __syncwarp();
                }
                // node nid: children [s, s + nl) and [s + nl, e), Karras numbering
                if (lane == 0) {
                    const int ls = a + s, rs = a + s + nl;
                    const int32_t left = nl == 1 ? ~ls : rs - 1;
                    const int32_t right = e - (s + nl) == 1 ? ~rs : rs;
                    *reinterpret_cast<int4*>(nodes + 4 * nid + 3) = make_int4(left, right, a + s, a + e - 1);
                    parent[left >= 0 ? left : n_nodes + ~left] = (nid << 1) | 0;
                    parent[right >= 0 ? right : n_nodes + ~right] = (nid << 1) | 1;
                    arrivals[nid] = 2u;  // complete (the validator's "atomic: 2")
                    const int nxt = cur ^ 1;
                    int* tn = s_task + nxt * (kSahSub / 2) * 3;
                    // children of > kSahSmall triangles: the next level's warp tasks; smaller: one thread each
                    if (nl >= 2) {
                        const bool sm = nl <= kSahSmall;
                        const int w = atomicAdd(sm ? &s_ntask[2] : &s_ntask[nxt], 1);
                        int* d = sm ? s_small : tn;
                        d[3 * w] = s;
                        d[3 * w + 1] = s + nl;
                        d[3 * w + 2] = left;
                    }
                    if (k - nl >= 2) {
                        const bool sm = k - nl <= kSahSmall;
                        const int w = atomicAdd(sm ? &s_ntask[2] : &s_ntask[nxt], 1);
                        int* d = sm ? s_small : tn;
                        d[3 * w] = s + nl;
                        d[3 * w + 1] = e;
                        d[3 * w + 2] = right;
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_ntask[cur] = 0;
            cur ^= 1;
            __syncthreads();
        }
        // the small nodes, one thread each (disjoint slices of the permutation)
        const int ns = s_ntask[2];
        for (int t = threadIdx.x; t < ns; t += blockDim.x)
            sah_small(a, s_small[3 * t], s_small[3 * t + 1], s_small[3 * t + 2], s_lo, s_hi, s_perm, nodes, parent,
                      arrivals, n_nodes, s_popt + 32 * threadIdx.x, s_rbox, root);
        __syncthreads();
        // the leaf slots' triangles in the new order, packed (A7): (v0, id), (v1, 0), (v2, 0), pad
        for (int t = threadIdx.x; t < m; t += blockDim.x) {
            const int q = s_perm[t];
            const int32_t id = s_id[q];
            const int k = a + t;
            vals[k] = id;
            tris[kTriF4 * k + 0] = make_float4(s_v[q], s_v[kSahSub + q], s_v[2 * kSahSub + q], __int_as_float(id));
            tris[kTriF4 * k + 1] = make_float4(s_v[3 * kSahSub + q], s_v[4 * kSahSub + q], s_v[5 * kSahSub + q], 0.f);
            tris[kTriF4 * k + 2] = make_float4(s_v[6 * kSahSub + q], s_v[7 * kSahSub + q], s_v[8 * kSahSub + q], 0.f);
            if (kTriF4 == 4) tris[4 * k + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // the subtree is complete: refit upwards from its root (the Karras nodes above)
        if (threadIdx.x == 0) {
            float lo[3] = {s_rbox[0], s_rbox[1], s_rbox[2]}, hi[3] = {s_rbox[3], s_rbox[4], s_rbox[5]};
            refit_climb(nodes, parent, arrivals, scratch, root == 0 ? -1 : parent[root], lo, hi);
        }
        __syncthreads();
    }
}

// One thread per leaf slot k: pack triangle k (Morton order), compute its AABB
// and ascend.  A CTA owns the leaf window [c0, c0 + kRefitLeaves): an
// internal node whose leaf range (stored by k_karras) lies inside the window
// has all its descendants in this CTA, so its two arrivals meet in SHARED
// memory, in barrier-separated rounds: in a round every climbing thread puts
// its box into its slot of the parent and counts its arrival with a
// shared-memory atomic; after the barrier the second arrival reads the
// sibling's slot, merges and climbs on (tens of cycles per level instead of a
// global atomic round trip; the window's parent links and node ranges are
// bulk-loaded first).  A climb that reaches a node crossing the window leaves
// the rounds and continues with the global protocol: box into the node slot,
// acq_rel atomicAdd on the arrival counter (first arrival stops),
// sibling box by L2-coherent loads.  Every arrival also counts in arrivals[]
// (a fire-and-forget reduction in the rounds) for the validator's "atomic: 2"
// check, and every level writes the child's box into the global
// node slot the traversal reads.
#ifndef RSI_REFIT_LEAVES
#define RSI_REFIT_LEAVES 256  // leaves per CTA window (256: -3 % rebuild vs 512; 1024 exceeds static smem)
#endif
constexpr int kRefitLeaves = RSI_REFIT_LEAVES;

// kT: the treelet restructuring is compiled in (its shared memory -- DP rows,
// refs, costs: 11 KB per CTA -- and registers would cost the other builds
// occupancy: N_t = 1e6 refit 467 -> see DESIGN.md 7).
template <bool kT>
__global__ void __launch_bounds__(kRefitLeaves) k_refit(const float* __restrict__ V, int64_t nv,
                                                        const int32_t* __restrict__ T,
                                                        const int32_t* __restrict__ vals, int n_leaves, int n,
                                                        float4* nodes, float4* __restrict__ tris,
                                                        int32_t* parent, uint32_t* arrivals,
                                                        uint32_t* scratch, int rotate, int treelet) {
    __shared__ uint32_t s_arr[kRefitLeaves];
    __shared__ float s_box[kRefitLeaves][2][6];
    __shared__ int32_t s_par[kRefitLeaves];  // parent links of the window's internal nodes
    __shared__ int2 s_rng[kRefitLeaves];     // their leaf ranges
    const int c0 = blockIdx.x * kRefitLeaves;
    const int n_nodes = n > 1 ? n - 1 : 1;
    // the thread that completed a window node restructures its treelet
    constexpr bool kTr = kT && kTL > 0;
    __shared__ unsigned char s_popt[kTr ? kRefitLeaves : 1][1 << kTLm];  // DP partition table, a row per thread
    __shared__ int32_t s_ref[kTr ? kRefitLeaves : 1][2];
    __shared__ float s_cost[kTr ? kRefitLeaves : 1];
    {
        // the window's slice of the tree, in bulk: one coalesced round trip
        // instead of a dependent L2 load per level of every ascent
        const int i = c0 + threadIdx.x;
        s_arr[threadIdx.x] = 0u;
        const bool own = n > 1 && i < n_nodes;
        const int4 r3 = own ? __ldg(reinterpret_cast<const int4*>(nodes + 4 * i + 3)) : make_int4(0, 0, -1, -1);
        s_rng[threadIdx.x] = make_int2(r3.z, r3.w);
        if (kTr) {
            s_ref[kTr ? threadIdx.x : 0][0] = r3.x;
            s_ref[kTr ? threadIdx.x : 0][1] = r3.y;
        }
        s_par[threadIdx.x] = own ? __ldg(parent + i) : -1;
    }
    const int k = c0 + threadIdx.x;
    const bool leaf = k < n_leaves;
    float lo[3], hi[3];
    int32_t p = -1;
    if (leaf) {
        const int32_t id = vals[k];
        const int32_t ia = safe_index(T[3 * id], nv), ib = safe_index(T[3 * id + 1], nv),
                      ic = safe_index(T[3 * id + 2], nv);
        float a[3], b[3], c[3];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            a[x] = V[3 * ia + x];
            b[x] = V[3 * ib + x];
            c[x] = V[3 * ic + x];
            lo[x] = fminf(a[x], fminf(b[x], c[x]));
            hi[x] = fmaxf(a[x], fmaxf(b[x], c[x]));
        }
        tris[kTriF4 * k + 0] = make_float4(a[0], a[1], a[2], __int_as_float(id));
        tris[kTriF4 * k + 1] = make_float4(b[0], b[1], b[2], 0.f);
        tris[kTriF4 * k + 2] = make_float4(c[0], c[1], c[2], 0.f);
        if (kTriF4 == 4) tris[4 * k + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
        p = parent[n_nodes + k];
    }
    __syncthreads();
    // ---- rounds inside the window (state: 0 done, 1 climbing in the window,
    // 2 waiting to merge after the barrier, 3 continue with the global protocol)
    int state = leaf ? 1 : 0;
    int wi = -1, side = 0;
    if (n == 1 && leaf) {  // single triangle: the root's left slot, no arrivals
        write_slot(nodes, 0, 0, lo, hi);
        state = 0;
    }
    while (__syncthreads_or(state == 1)) {
        int done_node = -1;  // the node this thread completed in this round (treelet root)
        if (state == 1) {
            const int node = p >> 1;
            side = p & 1;
            wi = node - c0;
            write_slot(nodes, node, side, lo, hi);
            if (wi >= 0 && wi < kRefitLeaves && s_rng[wi].x >= c0 && s_rng[wi].y < c0 + kRefitLeaves) {
                float* sb = s_box[wi][side];
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    sb[x] = lo[x];
                    sb[3 + x] = hi[x];
                }
                atomicAdd(arrivals + node, 1u);  // count only (result unused: a reduction)
                state = atomicAdd(&s_arr[wi], 1u) == 0u ? 0 : 2;
            } else {
                state = 3;  // the node crosses the window (its box slot is already written)
            }
        }
        __syncthreads();
        if (state == 2) {  // the sibling's slot was written before the barrier
            const float* ob = s_box[wi][1 - side];
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                lo[x] = fminf(lo[x], ob[x]);
                hi[x] = fmaxf(hi[x], ob[3 + x]);
            }
            const int node = wi + c0;
            if (rotate) rotate_node(nodes, parent, n_nodes, node);
            done_node = node;
            if (node == 0) {
                state = 4;  // merged at the root inside the window
            } else {
                p = s_par[wi];
                state = 1;
            }
        }
        if (kTr && treelet && done_node >= 0) {
            const WindowTree tr{nodes, parent, n_nodes, c0, s_box, s_ref, s_cost};
            treelet_opt(tr, done_node, s_popt[threadIdx.x]);
        }
    }
    if (state == 3) {
        // global protocol from node p >> 1 (whose slot this thread already wrote)
        while (true) {
            const int node = p >> 1;
            side = p & 1;
            // the next parent link is not rewritten (treelets stay inside windows): fetch it before the arrival
            const int32_t p_next = node > 0 ? __ldg(parent + node) : -1;
            // acq_rel arrival: releases this child's box, acquires the sibling's
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(arrivals + node) : "memory");
            if (old == 0u) return;
            // sibling box: L2-coherent loads (ld.global.cg), ordered after the atomic
            const float* f = reinterpret_cast<const float*>(nodes + 4 * node);
            const int o = side ? 0 : 4;  // sibling slot
            lo[0] = fminf(lo[0], __ldcg(f + o + 0));
            hi[0] = fmaxf(hi[0], __ldcg(f + o + 1));
            lo[1] = fminf(lo[1], __ldcg(f + o + 2));
            hi[1] = fmaxf(hi[1], __ldcg(f + o + 3));
            lo[2] = fminf(lo[2], __ldcg(f + 8 + 2 * (1 - side)));
            hi[2] = fmaxf(hi[2], __ldcg(f + 9 + 2 * (1 - side)));
            if (rotate) rotate_node(nodes, parent, n_nodes, node);
            if (node == 0) break;
            p = p_next;
            write_slot(nodes, p >> 1, p & 1, lo, hi);
        }
    } else if (state != 4 && !(n == 1 && leaf)) {
        return;
    }
    // root box (scene AABB) for rsi_bvh_info
    float* root = reinterpret_cast<float*>(scratch + SCR_ROOT);
    for (int x = 0; x < 3; ++x) {
        root[x] = lo[x];
        root[3 + x] = hi[x];
    }
    scratch[SCR_ROOT_SET] = 1u;
}

// Small meshes (N_t <= kRankSortMax): the sorted position of key i is its rank
//   r(i) = #{ j : k_j < k_i  or  (k_j == k_i and j < i) }
// (a stable sort by construction), counted directly: CTA (bx, by) compares its
// kRankI keys against key slice `by` held in shared memory and adds the partial
// counts to rank[i] with atomics; the last slice CTA of block bx (a per-block
// counter, after a fence) scatters keys and indices.  O(N^2) compares spread
// over the whole GPU (~1e8 at N = 1e4: a few microseconds) instead of four
// dependent radix passes on one SM.  For a slice wholly below block bx's keys
// "j < i" holds for every pair, so the test is k_j < k_i + 1; wholly above, k_j < k_i.
constexpr int kRankSortMax = 16384;
constexpr int kRankT = 256, kRankPer = 2, kRankI = kRankT * kRankPer;

__global__ void __launch_bounds__(kRankT) k_sort_rank(const uint32_t* __restrict__ keys, int n, int slice,
                                                      uint32_t* rank, uint32_t* __restrict__ out_keys,
                                                      int32_t* __restrict__ out_vals, uint32_t* done) {
    extern __shared__ uint4 s_k4[];
    uint32_t* s_k = reinterpret_cast<uint32_t*>(s_k4);
    const int tid = threadIdx.x;
    const int j0 = blockIdx.y * slice, j1 = min(j0 + slice, n);
    const int nj = j1 > j0 ? j1 - j0 : 0;
    const int nj4 = (nj + 3) >> 2;
    for (int j = tid; j < 4 * nj4; j += kRankT) s_k[j] = j < nj ? keys[j0 + j] : 0xffffffffu;  // pad: > every key
    __syncthreads();
    const int i_lo = blockIdx.x * kRankI, i_hi = min(i_lo + kRankI, n);
    int idx[kRankPer];
    uint32_t ki[kRankPer], cnt[kRankPer];
#pragma unroll
    for (int a = 0; a < kRankPer; ++a) {
        idx[a] = i_lo + tid + a * kRankT;
        ki[a] = idx[a] < n ? keys[idx[a]] : 0u;
        cnt[a] = 0u;
    }
    if (j1 <= i_lo || j0 >= i_hi) {  // slice wholly below / above this block's keys
        const uint32_t add = j1 <= i_lo ? 1u : 0u;
        uint32_t thr[kRankPer];
#pragma unroll
        for (int a = 0; a < kRankPer; ++a) thr[a] = ki[a] + add;
        for (int q = 0; q < nj4; ++q) {
            const uint4 k4 = s_k4[q];
#pragma unroll
            for (int a = 0; a < kRankPer; ++a)
                cnt[a] += (k4.x < thr[a]) + (k4.y < thr[a]) + (k4.z < thr[a]) + (k4.w < thr[a]);
        }
        // a key of 0xffffffff (possible in the 63-bit path's full low words):
        // k_i + 1 wrapped to 0 -- every key of a slice below counts
#pragma unroll
        for (int a = 0; a < kRankPer; ++a)
            if (add && ki[a] == 0xffffffffu) cnt[a] = (uint32_t)nj;
    } else {  // overlapping (diagonal) slice: per-pair index test
        for (int j = 0; j < nj; ++j) {
            const uint32_t kj = s_k[j];
#pragma unroll
            for (int a = 0; a < kRankPer; ++a) cnt[a] += (kj < ki[a] + (j0 + j < idx[a] ? 1u : 0u));
        }
#pragma unroll
        for (int a = 0; a < kRankPer; ++a)
            if (ki[a] == 0xffffffffu) {  // the +1 wrapped: recount exactly (rare)
                cnt[a] = 0u;
                for (int j = 0; j < nj; ++j) cnt[a] += (s_k[j] != 0xffffffffu) || (j0 + j < idx[a]);
            }
    }
#pragma unroll
    for (int a = 0; a < kRankPer; ++a)
        if (idx[a] < n && cnt[a]) atomicAdd(rank + idx[a], cnt[a]);
    __threadfence();
    __syncthreads();
    __shared__ bool s_last;
    if (tid == 0) s_last = atomicAdd(done + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int a = 0; a < kRankPer; ++a) {
        if (idx[a] < n) {
            const uint32_t r = __ldcg(rank + idx[a]);
            out_keys[r] = ki[a];
            out_vals[r] = idx[a];
        }
    }
}

// ------------------------------------------------------------------ NEXT-1: 63-bit codes + Apetrei build
// RSI_OPT_APETREI: the paper's construction.  Codes are
// 63-bit ("64-bit Morton codes"): 21 bits per axis with the same
// quantization rule as the 30-bit path (reading R8) scaled by 2^21 instead of
// 2^10 -- an exact power-of-two rescale, so the top 30 bits of the 63-bit code
// ARE the 30-bit code.  They are sorted by two stable 32-bit LSD sorts (low
// word, then high word) and the tree is built bottom-up in one pass (Apetrei
// 2014, cited at P:504; the paper's construct kernel).

// Spread the low 21 bits of x so bit k lands at bit 3k.
__device__ __forceinline__ unsigned long long expand21(uint32_t v) {
    unsigned long long x = v & 0x1fffffu;
    x = (x | (x << 32)) & 0x1f00000000ffffull;
    x = (x | (x << 16)) & 0x1f0000ff0000ffull;
    x = (x | (x << 8)) & 0x100f00f00f00f00full;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__device__ __forceinline__ uint32_t quantize21(float c, float lo, float hi, float wmax) {
    float w = fmaxf(hi - lo, wmax * 0.015625f);
    if (!(w > 0.0f)) return 0u;
    float q = floorf((c - lo) / w * 2097152.0f);  // 2^21
    q = fminf(fmaxf(q, 0.0f), 2097151.0f);
    return (uint32_t)q;
}

// A3 (63-bit): code = e(qx) | e(qy) << 1 | e(qz) << 2 (z-major); low word into
// keys (sort pass 1) and k_lo, high word into k_hi; zeroes the arrival words.
__global__ void __launch_bounds__(kBlock) k_morton63(const float* __restrict__ V, int64_t nv,
                                                     const int32_t* __restrict__ T, int n,
                                                     const uint32_t* __restrict__ scratch,
                                                     uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                                     uint32_t* __restrict__ k_lo, uint32_t* __restrict__ k_hi,
                                                     unsigned long long* __restrict__ other,
                                                     uint32_t* __restrict__ rank) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    other[j] = 0ull;
    if (rank) rank[j] = 0u;
    float lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = rsi_ord2f(scratch[SCR_EXT_MIN + k]);
        hi[k] = rsi_ord2f(scratch[SCR_EXT_MAX + k]);
    }
    int32_t a = safe_index(T[3 * j], nv), b = safe_index(T[3 * j + 1], nv), c = safe_index(T[3 * j + 2], nv);
    const float wmax = fmaxf(hi[0] - lo[0], fmaxf(hi[1] - lo[1], hi[2] - lo[2]));
    uint32_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float cen = (V[3 * a + k] + V[3 * b + k] + V[3 * c + k]) / 3.0f;
        q[k] = quantize21(cen, lo[k], hi[k], wmax);
    }
    const unsigned long long code = expand21(q[0]) | (expand21(q[1]) << 1) | (expand21(q[2]) << 2);
    keys[j] = (uint32_t)code;
    k_lo[j] = (uint32_t)code;
    k_hi[j] = (uint32_t)(code >> 32);
    vals[j] = j;
}

// Between the two sorts: the high words in pass-1 (low-word) order become the
// keys, the pass-1 order is saved, values restart as positions, and the rank
// sort's accumulators and slice counters are cleared.
__global__ void __launch_bounds__(kBlock) k_pass2_prep(uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                                       const uint32_t* __restrict__ k_hi, int32_t* __restrict__ ids1,
                                                       int n, uint32_t* __restrict__ rank, uint32_t* scratch) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < 32) scratch[SCR_SORT_DONE + j] = 0u;
    if (j >= n) return;
    const int32_t id = vals[j];
    ids1[j] = id;
    keys[j] = k_hi[id];
    vals[j] = j;
    if (rank) rank[j] = 0u;
}

// After the second sort: vals[j] = position in pass-1 order -> triangle id;
// sorted low words gathered beside the sorted high words (keys).
__global__ void __launch_bounds__(kBlock) k_pass2_finish(int32_t* __restrict__ vals, const int32_t* __restrict__ ids1,
                                                         const uint32_t* __restrict__ k_lo,
                                                         uint32_t* __restrict__ lo_sorted, int n) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int32_t id = ids1[vals[j]];
    vals[j] = id;
    lo_sorted[j] = k_lo[id];
}

// Common-prefix length of sorted keys i and i+1 (larger = more similar); equal
// codes fall back to the sorted positions (index augmentation, as k_karras).
__device__ __forceinline__ int cpl63(const uint32_t* __restrict__ khi, const uint32_t* __restrict__ klo, int i) {
    const unsigned long long a = ((unsigned long long)khi[i] << 32) | klo[i];
    const unsigned long long b = ((unsigned long long)khi[i + 1] << 32) | klo[i + 1];
    const unsigned long long x = a ^ b;
    return x ? __clzll(x) : 64 + __clz(i ^ (i + 1));
}

// One thread per leaf slot k (grid = ceil(N_t / block): the case-study-2 rule,
// P:467-494).  The thread holds the leaf range [l, r] of its current subtree.
// Its parent is the node on the side of the more similar neighbour: node r
// (this subtree is its LEFT child) when l == 0 or cpl(r) > cpl(l-1), else node
// l-1 (RIGHT child); internal node i is thus the split between sorted leaves
// i and i+1.  The child writes its box and ref into its slot of the parent,
// then adds (1 << 32 | its far bound) to the parent's 64-bit word with
// acq_rel: the first arrival (old == 0) stops; the second learns the parent's
// full range from the old word, merges the sibling's box and climbs on.  The
// range [0, N_t-1] is the root; the sentinel N_t-1 only points at it.
__global__ void __launch_bounds__(kBlock) k_apetrei(const float* __restrict__ V, int64_t nv,
                                                    const int32_t* __restrict__ T, const int32_t* __restrict__ vals,
                                                    const uint32_t* __restrict__ khi, const uint32_t* __restrict__ klo,
                                                    int n_leaves, int n, float4* nodes, float4* __restrict__ tris,
                                                    int32_t* __restrict__ parent, unsigned long long* other,
                                                    uint32_t* scratch) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_leaves) return;
    const int n_nodes = n - 1;  // n >= 2 on this path
    const int32_t id = vals[k];
    const int32_t ia = safe_index(T[3 * id], nv), ib = safe_index(T[3 * id + 1], nv),
                  ic = safe_index(T[3 * id + 2], nv);
    float a[3], b[3], c[3], lo[3], hi[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
        a[x] = V[3 * ia + x];
        b[x] = V[3 * ib + x];
        c[x] = V[3 * ic + x];
        lo[x] = fminf(a[x], fminf(b[x], c[x]));
        hi[x] = fmaxf(a[x], fmaxf(b[x], c[x]));
    }
    tris[kTriF4 * k + 0] = make_float4(a[0], a[1], a[2], __int_as_float(id));
    tris[kTriF4 * k + 1] = make_float4(b[0], b[1], b[2], 0.f);
    tris[kTriF4 * k + 2] = make_float4(c[0], c[1], c[2], 0.f);
    if (kTriF4 == 4) tris[4 * k + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
    int l = k, r = k;
    int32_t ref = ~k;
    while (true) {
        if (l == 0 && r == n - 1) {  // the root: the sentinel's only child
            scratch[SCR_ROOT_NODE] = (uint32_t)ref;
            parent[ref] = -1;
            float* root = reinterpret_cast<float*>(scratch + SCR_ROOT);
            for (int x = 0; x < 3; ++x) {
                root[x] = lo[x];
                root[3 + x] = hi[x];
            }
            scratch[SCR_ROOT_SET] = 1u;
            return;
        }
        const bool up_right = (l == 0) || (r != n - 1 && cpl63(khi, klo, r) > cpl63(khi, klo, l - 1));
        const int p = up_right ? r : l - 1, side = up_right ? 0 : 1;
        write_slot(nodes, p, side, lo, hi);
        set_ref(nodes, p, side, ref);
        parent[ref >= 0 ? ref : n_nodes + ~ref] = (p << 1) | side;
        const unsigned long long add = (1ull << 32) | (uint32_t)(up_right ? l : r);
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(other + p), "l"(add) : "memory");
        if (old == 0ull) return;  // first arrival: the sibling finishes the node
        const int bound = (int)(uint32_t)old;
        if (up_right) r = bound; else l = bound;
        const float* f = reinterpret_cast<const float*>(nodes + 4 * p);
        const int o = side ? 0 : 4;  // sibling slot
        lo[0] = fminf(lo[0], __ldcg(f + o + 0));
        hi[0] = fmaxf(hi[0], __ldcg(f + o + 1));
        lo[1] = fminf(lo[1], __ldcg(f + o + 2));
        hi[1] = fmaxf(hi[1], __ldcg(f + o + 3));
        lo[2] = fminf(lo[2], __ldcg(f + 8 + 2 * (1 - side)));
        hi[2] = fmaxf(hi[2], __ldcg(f + 9 + 2 * (1 - side)));
        ref = p;
    }
}

// ------------------------------------------------------------------ top-of-tree image (shared-memory cache)
// north_star: "the top tree levels staged in shared memory".  The first
// kQTop 4-wide records the walk meets -- breadth-first from the root, the
// last level possibly in part -- are copied into a separate image in which a
// member that is itself cached points at its image slot (kSmemRef + slot);
// every other ref is unchanged, so a walk leaves the image for the global
// records exactly where the image ends.  k_trace loads the image into shared
// memory once per CTA.  One CTA, level-synchronous (a level is <= 4x the
// previous one, and kQTop <= 256 = blockDim).
__device__ int block_exclusive_scan(int v, int* s_warp, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int x = lane < nw ? s_warp[lane] : 0;
        int xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < nw) s_warp[lane] = xi - x;
        if (lane == 31) s_warp[32] = xi;
    }
    __syncthreads();
    const int r = s_warp[w] + inc - v;
    total = s_warp[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) k_qtop(const float4* __restrict__ quads, float4* __restrict__ image,
                                              uint32_t* scratch) {
    __shared__ int old_of[kQTop > 0 ? kQTop : 1];
    __shared__ int child_slot[kQTop > 0 ? kQTop : 1][4];
    __shared__ int s_warp[33];
    const int tid = threadIdx.x;
    const int root = (int)scratch[SCR_QROOT];
    if (kQTop == 0 || root < 0) {  // (no root: a fault-injected build) -- no image
        if (tid == 0) scratch[SCR_NTOP] = 0;
        return;
    }
    if (tid == 0) old_of[0] = root;
    for (int i = tid; i < kQTop; i += blockDim.x)
        for (int c = 0; c < 4; ++c) child_slot[i][c] = -1;
    __syncthreads();
    int a = 0, b = 1;  // current level = slots [a, b)
    while (b < kQTop) {
        const int sl = a + tid;
        int ref[4] = {kNoRefB, kNoRefB, kNoRefB, kNoRefB}, cnt = 0;
        if (sl < b) {
            const int4 r = *reinterpret_cast<const int4*>(quads + 4 * old_of[sl] + 2);   // refs 0, 1 in .z, .w
            const int4 r2 = *reinterpret_cast<const int4*>(quads + 4 * old_of[sl] + 3);  // refs 2, 3 in .x, .y
            ref[0] = r.z; ref[1] = r.w; ref[2] = r2.x; ref[3] = r2.y;
            for (int c = 0; c < 4; ++c) cnt += ref[c] >= 0;
        }
        int total;
        const int off = block_exclusive_scan(cnt, s_warp, total);
        if (total == 0) break;
        if (sl < b) {
            int k = b + off;
            for (int c = 0; c < 4; ++c)
                if (ref[c] >= 0) {
                    if (k < kQTop) {
                        old_of[k] = ref[c];
                        child_slot[sl][c] = k;
                    }
                    ++k;
                }
        }
        __syncthreads();
        a = b;
        b = min(b + total, kQTop);
    }
    // image: the records with cached members' refs translated to image slots
    for (int sl = tid; sl < b; sl += blockDim.x) {
        const float4* q = quads + 4 * old_of[sl];
        float4* im = image + 4 * sl;
        im[0] = q[0];
        im[1] = q[1];
        float4 qc = q[2], qd = q[3];
        int* rc = reinterpret_cast<int*>(&qc);
        int* rd = reinterpret_cast<int*>(&qd);
        if (child_slot[sl][0] >= 0) rc[2] = (int)kSmemRef + child_slot[sl][0];
        if (child_slot[sl][1] >= 0) rc[3] = (int)kSmemRef + child_slot[sl][1];
        if (child_slot[sl][2] >= 0) rd[0] = (int)kSmemRef + child_slot[sl][2];
        if (child_slot[sl][3] >= 0) rd[1] = (int)kSmemRef + child_slot[sl][3];
        im[2] = qc;
        im[3] = qd;
    }
    if (tid == 0) scratch[SCR_NTOP] = (uint32_t)b;
}

// ------------------------------------------------------------------ 4-wide record compaction
// k_quads writes a record for EVERY internal node, but the walk only reaches
// the records of the collapsed tree -- the root and the internal members of
// reached records, about a third of them (~3.9 members per record) -- so
// two thirds of every 128-byte line of the node-indexed array is dead weight
// in L1.  This pass keeps the live records only, breadth-first from the root
// (index 0; a record's members sit next to each other), with member refs
// rewritten to the new indices (leaf refs and kNoRef unchanged).  One CTA,
// level-synchronous (a level's live records are the previous level's
// internal members, ranked by a block scan).
__global__ void __launch_bounds__(1024) k_qcompact(const float4* __restrict__ full, float4* __restrict__ out,
                                                   int32_t* order, int32_t* map, uint32_t* scratch) {
    __shared__ int s_warp[33];
    const int tid = threadIdx.x;
    const int root = (int)scratch[SCR_ROOT_NODE];
    if (root < 0) {  // (a fault-injected build never reached the root): no records
        if (tid == 0) scratch[SCR_QROOT] = 0xffffffffu;
        return;
    }
    if (tid == 0) {
        order[0] = root;
        map[root] = 0;
    }
    __syncthreads();
    int a = 0, b = 1;  // current level = live records [a, b)
    while (a < b) {
        int next = b;
        for (int base = a; base < b; base += blockDim.x) {
            const int i = base + tid;
            int ref[4] = {kNoRefB, kNoRefB, kNoRefB, kNoRefB}, cnt = 0;
            if (i < b) {
                const int o = order[i];
                const int4 r2 = *reinterpret_cast<const int4*>(full + 4 * o + 2);  // refs 0, 1 in .z, .w
                const int4 r3 = *reinterpret_cast<const int4*>(full + 4 * o + 3);  // refs 2, 3 in .x, .y
                ref[0] = r2.z; ref[1] = r2.w; ref[2] = r3.x; ref[3] = r3.y;
                for (int c = 0; c < 4; ++c) cnt += ref[c] >= 0;
            }
            int total;
            const int off = block_exclusive_scan(cnt, s_warp, total);
            int k = next + off;
            for (int c = 0; c < 4; ++c)
                if (ref[c] >= 0) {
                    order[k] = ref[c];
                    map[ref[c]] = k;
                    ++k;
                }
            next += total;
            __syncthreads();
        }
        a = b;
        b = next;
    }
    for (int i = tid; i < b; i += blockDim.x) {
        const float4* q = full + 4 * order[i];
        float4* d = out + 4 * i;
        d[0] = q[0];
        d[1] = q[1];
        float4 qc = q[2], qd = q[3];
        int* rc = reinterpret_cast<int*>(&qc);
        int* rd = reinterpret_cast<int*>(&qd);
        if (rc[2] >= 0) rc[2] = map[rc[2]];
        if (rc[3] >= 0) rc[3] = map[rc[3]];
        if (rd[0] >= 0) rd[0] = map[rd[0]];
        if (rd[1] >= 0) rd[1] = map[rd[1]];
        d[2] = qc;
        d[3] = qd;
    }
    if (tid == 0) scratch[SCR_QROOT] = 0u;
}

// records indexed by node id (meshes above kQCompactMax internal nodes)

// ------------------------------------------------------------------ 4-wide view (cut records)
// One thread per internal node n: the up-to-4 members of n's cut (grandchildren, or the greedy cut under RSI_QUAD_GREEDY; a leaf child
// stands for itself), their AABBs quantized to 8 bits on a per-axis
// power-of-two grid anchored at an origin p that is itself a multiple of the
// grid step s = 2^e:  lo' = p + qlo*s <= lo,  hi' = p + qhi*s >= hi  (exact:
// computed in double; |p/s| < 2^24 keeps p + q*s exactly representable, so the
// traversal's decode is exact, and directed rounding keeps it conservative
// otherwise).  64 B per record = two 256-bit loads.
//   w0..w2  pm = p - 2^15 s per axis (float, the traversal's decode offset)
//   w3, w14, w15  s_x, s_y, s_z (float 2^e)
//   w4..w9  qlo.x, qhi.x, qlo.y, qhi.y, qlo.z, qhi.z   (byte j = child j)
//   w10..w13 ref[0..3]  (kNoRef = 0x80000000 for the missing children of a
//            node with fewer than 4)
constexpr int kQuadEMin = -126, kQuadEMax = 104;  // s and s*2^23 stay normal floats

__device__ __forceinline__ void quant_axis(const float* lo, const float* hi, int cnt, uint32_t& wlo, uint32_t& whi,
                                           float& p_out, int& e_out, bool& ok) {
    float nlo = INFINITY, nhi = -INFINITY;
    for (int j = 0; j < cnt; ++j) {
        nlo = fminf(nlo, lo[j]);
        nhi = fmaxf(nhi, hi[j]);
    }
    const double ext = (double)nhi - (double)nlo;
    int e = kQuadEMin;
    if (ext > 0.0) {
        int ex;
        frexp(ext / 255.0, &ex);  // ext/255 < 2^ex
        e = ex - 1;
        if (e < kQuadEMin) e = kQuadEMin;
    }
    double sc, isc, p;  // s = 2^e and 1/s (exact), so x * isc == x / s exactly
    while (true) {
        sc = ldexp(1.0, e);
        isc = ldexp(1.0, -e);
        p = floor((double)nlo * isc) * sc;  // multiple of s, p <= nlo
        // covers the node, and p = k*s with |k| < 2^23 so p and p - 2^15 s are exact floats
        if (((double)nhi - p <= 255.0 * sc && fabs(p * isc) < 8388608.0) || e >= kQuadEMax) break;
        ++e;
    }
    wlo = 0u;
    whi = 0u;
    for (int j = 0; j < cnt; ++j) {
        double ql = floor(((double)lo[j] - p) * isc), qh = ceil(((double)hi[j] - p) * isc);
        ql = fmin(fmax(ql, 0.0), 255.0);
        qh = fmin(fmax(qh, 0.0), 255.0);
        wlo |= (uint32_t)ql << (8 * j);
        whi |= (uint32_t)qh << (8 * j);
    }
    for (int j = cnt; j < 4; ++j) wlo |= 255u << (8 * j);  // missing child: empty box (lo > hi)
    p_out = (float)(p - kQuadBias * sc);  // the decode offset p - M s: exact (|p/s - 2^15| < 2^24)
    e_out = e;
    ok = ((double)nhi - p <= 255.0 * sc) && fabs(p * isc) < 8388608.0 && (double)p_out == p - kQuadBias * sc;
}

__global__ void __launch_bounds__(kBlock) k_quads(const float4* __restrict__ nodes, int n_nodes,
                                                  float4* __restrict__ quads, uint32_t* scratch) {
    int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= n_nodes) return;
    // the walks' root record = the root node (k_qcompact, when it runs, renumbers it 0 afterwards)
    if (n == 0) scratch[SCR_QROOT] = scratch[SCR_ROOT_NODE];
    // (one spare slot: a greedy expansion appends both children before moving one)
    float lo[3][5], hi[3][5];
    int ref[5] = {(int)0x80000000, (int)0x80000000, (int)0x80000000, (int)0x80000000,
                  (int)0x80000000};  // kNoRef: no child
    int k = 0;
#if RSI_QUAD_GREEDY
    // greedy 4-cut: start from n's two children and twice replace the internal
    // member with the largest surface area (the likeliest to be entered by a
    // random segment) by its two children (a 2-leaf or leaf-heavy subtree
    // leaves fewer than 4 members)
    auto add_pair = [&](int node, int skip_empty) {
        const float4* nd = nodes + 4 * node;
        const float4 a0 = nd[0], a1 = nd[1], a2 = nd[2];
        const int4 a3 = *reinterpret_cast<const int4*>(nd + 3);
        const float4 cb[2] = {a0, a1};
        const float cz[2][2] = {{a2.x, a2.y}, {a2.z, a2.w}};
        const int cr[2] = {a3.x, a3.y};
        for (int side = 0; side < 2; ++side) {
            if (skip_empty && cr[side] < 0 && cb[side].x == INFINITY) continue;  // 1-triangle tree
            lo[0][k] = cb[side].x; hi[0][k] = cb[side].y; lo[1][k] = cb[side].z; hi[1][k] = cb[side].w;
            lo[2][k] = cz[side][0]; hi[2][k] = cz[side][1];
            ref[k] = cr[side];
            ++k;
        }
    };
    add_pair(n, 1);
    for (int step = 0; step < 2; ++step) {
        int best = -1;
        float best_area = -1.0f;
        for (int j = 0; j < k; ++j) {
            if (ref[j] < 0) continue;
            const float ax = hi[0][j] - lo[0][j], ay = hi[1][j] - lo[1][j], az = hi[2][j] - lo[2][j];
            const float area = ax * ay + ay * az + az * ax;
            if (area > best_area) {
                best_area = area;
                best = j;
            }
        }
        if (best < 0) break;
        // the expanded member's slot takes its right child, its left goes last
        const int node = ref[best];
        const int k0 = k;
        add_pair(node, 0);  // appends 2 members at k0, k0 + 1
        for (int a = 0; a < 3; ++a) {
            lo[a][best] = lo[a][k0 + 1];
            hi[a][best] = hi[a][k0 + 1];
        }
        ref[best] = ref[k0 + 1];
        k = k0 + 1;
    }
#else
    const float4* nd = nodes + 4 * n;
    const float4 n0 = nd[0], n1 = nd[1], n2 = nd[2];
    const int4 n3 = *reinterpret_cast<const int4*>(nd + 3);
    const float4 cb[2] = {n0, n1};
    const float cz[2][2] = {{n2.x, n2.y}, {n2.z, n2.w}};
    const int cr[2] = {n3.x, n3.y};
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const int c = cr[side];
        if (c < 0) {  // leaf child stands for itself
            if (cb[side].x == INFINITY) continue;  // the empty right slot of a 1-triangle tree
            lo[0][k] = cb[side].x; hi[0][k] = cb[side].y; lo[1][k] = cb[side].z; hi[1][k] = cb[side].w;
            lo[2][k] = cz[side][0]; hi[2][k] = cz[side][1];
            ref[k] = c;
            ++k;
        } else {
            const float4* cd = nodes + 4 * c;
            const float4 c0 = cd[0], c1 = cd[1], c2 = cd[2];
            const int4 c3 = *reinterpret_cast<const int4*>(cd + 3);
            lo[0][k] = c0.x; hi[0][k] = c0.y; lo[1][k] = c0.z; hi[1][k] = c0.w; lo[2][k] = c2.x; hi[2][k] = c2.y;
            ref[k] = c3.x;
            ++k;
            lo[0][k] = c1.x; hi[0][k] = c1.y; lo[1][k] = c1.z; hi[1][k] = c1.w; lo[2][k] = c2.z; hi[2][k] = c2.w;
            ref[k] = c3.y;
            ++k;
        }
    }
#endif
    uint32_t w[16];
    float px[3];
    int ex[3];
    bool ok = true;
    for (int a = 0; a < 3; ++a) {
        bool oka;
        quant_axis(lo[a], hi[a], k, w[4 + 2 * a], w[5 + 2 * a], px[a], ex[a], oka);
        ok = ok && oka;
    }
    if (!ok) atomicOr(&scratch[SCR_STATUS], STATUS_RANGE);  // coordinates beyond ~1e33
    // max |decode offset| (non-negative float bits order like uint32): bounds the
    // rounding of the traversal's per-node slab term fma(pm, inv, -off)
    const float pmax = fmaxf(fabsf(px[0]), fmaxf(fabsf(px[1]), fabsf(px[2])));
    atomicMax(&scratch[SCR_QPMAX], __float_as_uint(pmax));
    atomicMin(&scratch[SCR_QEMIN], (uint32_t)(min(ex[0], min(ex[1], ex[2])) + 128));
    atomicMax(&scratch[SCR_QEMAX], (uint32_t)(max(ex[0], max(ex[1], ex[2])) + 128));
    w[0] = __float_as_uint(px[0]);
    w[1] = __float_as_uint(px[1]);
    w[2] = __float_as_uint(px[2]);
    // grid steps as floats (2^e, exact): the traversal multiplies them by 1/d directly
    w[3] = __float_as_uint(ldexpf(1.0f, ex[0]));
    for (int j = 0; j < 4; ++j) w[10 + j] = (uint32_t)ref[j];
    w[14] = __float_as_uint(ldexpf(1.0f, ex[1]));
    w[15] = __float_as_uint(ldexpf(1.0f, ex[2]));
    uint4* q = reinterpret_cast<uint4*>(quads + 4 * n);
    q[0] = make_uint4(w[0], w[1], w[2], w[3]);
    q[1] = make_uint4(w[4], w[5], w[6], w[7]);
    q[2] = make_uint4(w[8], w[9], w[10], w[11]);
    q[3] = make_uint4(w[12], w[13], w[14], w[15]);
}

// ------------------------------------------------------------------ NEXT-2: integrity validator
// One thread per internal node: arrival count, parent links of both children,
// and exact box union of each internal child.  One thread per leaf: triangle-id
// histogram and a parent walk to the root (<= 64 steps: depth <= 62).
enum { V_HALF = 0, V_UNTOUCHED, V_LEAFIDS, V_LINKS, V_BOXES, V_UNREACH, V_WORDS };

__device__ __forceinline__ void node_box(const float4* nodes, int node, int side, float lo[3], float hi[3]) {
    const float* f = reinterpret_cast<const float*>(nodes + 4 * node);
    const int o = side ? 4 : 0;
    lo[0] = f[o + 0];
    hi[0] = f[o + 1];
    lo[1] = f[o + 2];
    hi[1] = f[o + 3];
    lo[2] = f[8 + 2 * side];
    hi[2] = f[9 + 2 * side];
}

__global__ void __launch_bounds__(kBlock) k_validate_nodes(const float4* __restrict__ nodes, int n, int n_nodes,
                                                           const int32_t* __restrict__ parent,
                                                           const uint32_t* __restrict__ arrivals,
                                                           const unsigned long long* __restrict__ other,
                                                           unsigned long long* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_nodes || n == 1) return;
    // arrival count: the refit counter, or the high word of the Apetrei node word
    const uint32_t a = other ? (uint32_t)(other[i] >> 32) : arrivals[i];
    if (a == 1u) atomicAdd(out + V_HALF, 1ull);
    if (a == 0u) atomicAdd(out + V_UNTOUCHED, 1ull);
    const int4 r = *reinterpret_cast<const int4*>(nodes + 4 * i + 3);
    const int ch[2] = {r.x, r.y};
    for (int side = 0; side < 2; ++side) {
        const int c = ch[side];
        const int64_t pi = c >= 0 ? c : (int64_t)n_nodes + ~c;
        if ((c >= 0 && c >= n_nodes) || (c < 0 && ~c >= n) || parent[pi] != ((i << 1) | side)) {
            atomicAdd(out + V_LINKS, 1ull);
            continue;
        }
        if (c >= 0) {  // the slot box of an internal child = union of that child's two slots
            float lo[3], hi[3], l0[3], h0[3], l1[3], h1[3];
            node_box(nodes, i, side, lo, hi);
            node_box(nodes, c, 0, l0, h0);
            node_box(nodes, c, 1, l1, h1);
            bool ok = true;
            for (int x = 0; x < 3; ++x)
                ok = ok && lo[x] == fminf(l0[x], l1[x]) && hi[x] == fmaxf(h0[x], h1[x]);
            if (!ok) atomicAdd(out + V_BOXES, 1ull);
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_validate_leaves(const float4* __restrict__ tris, int n, int n_nodes,
                                                            const uint32_t* __restrict__ scratch,
                                                            const int32_t* __restrict__ parent,
                                                            uint32_t* __restrict__ seen,
                                                            unsigned long long* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int id = __float_as_int(tris[kTriF4 * k].w);
    if (id < 0 || id >= n) atomicAdd(out + V_LEAFIDS, 1ull);
    else atomicAdd(seen + id, 1u);
    const int root = (int)scratch[SCR_ROOT_NODE];
    // parent walk: must end at the root (parent -1) within the depth bound
    // (<= 95 levels for the 63-bit code + 32-bit index key)
    int p = parent[n_nodes + k], last = -1, steps = 0;
    bool ok = true;
    while (p != -1) {
        const int node = p >> 1;
        if (p < 0 || node >= n_nodes || ++steps > 128) {
            ok = false;
            break;
        }
        last = node;
        p = parent[node];
    }
    if (!ok || last != root) atomicAdd(out + V_UNREACH, 1ull);
}

__global__ void __launch_bounds__(kBlock) k_validate_ids(const uint32_t* __restrict__ seen, int n,
                                                         unsigned long long* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n && seen[j] != 1u) atomicAdd(out + V_LEAFIDS, 1ull);
}

}  // namespace

// ------------------------------------------------------------------ host side
static rsi_status_t ensure_capacity(rsi_bvh* h, int64_t n, cudaStream_t s) {
    int nb = rsi_ceil_div(n, kTile);
    if (n <= h->cap_tri && nb <= h->sort_blocks_cap) return RSI_OK;
    void* old[] = {h->nodes, h->top, h->quads, h->tris, h->keys, h->vals, h->keys_tmp, h->vals_tmp, h->parent, h->arrivals, h->hist,
                   h->qfull, h->qorder, h->qmap};
    for (void* p : old)
        if (p) cudaFreeAsync(p, s);
    h->qfull = nullptr;
    h->qorder = nullptr;
    h->qmap = nullptr;
    int64_t nn = n > 1 ? n - 1 : 1;
    cudaError_t e = cudaSuccess;
#define RSI_ALLOC(ptr, bytes) \
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&(ptr), (size_t)(bytes), s);
    RSI_ALLOC(h->nodes, nn * 4 * sizeof(float4));
    RSI_ALLOC(h->top, (size_t)(kQTop > 0 ? kQTop : 1) * 4 * sizeof(float4));
    RSI_ALLOC(h->quads, nn * 4 * sizeof(float4));
    if (nn <= kQCompactMax) {
        RSI_ALLOC(h->qfull, nn * 4 * sizeof(float4));
        RSI_ALLOC(h->qorder, nn * sizeof(int32_t));
        RSI_ALLOC(h->qmap, nn * sizeof(int32_t));
    }
    RSI_ALLOC(h->tris, n * kTriF4 * sizeof(float4));
    RSI_ALLOC(h->keys, n * sizeof(uint32_t));
    RSI_ALLOC(h->vals, n * sizeof(int32_t));
    RSI_ALLOC(h->keys_tmp, n * sizeof(uint32_t));
    RSI_ALLOC(h->vals_tmp, n * sizeof(int32_t));
    RSI_ALLOC(h->parent, (nn + n) * sizeof(int32_t));
    RSI_ALLOC(h->arrivals, nn * sizeof(uint32_t));
    RSI_ALLOC(h->hist, (size_t)kDigits * (nb + 1) * sizeof(uint32_t));  // + the 256 row totals
#undef RSI_ALLOC
    if (e != cudaSuccess) {
        h->cap_tri = 0;
        h->sort_blocks_cap = 0;
        (void)cudaGetLastError();
        return rsi_set_error(RSI_E_OOM, "device allocation for %lld triangles failed: %s", (long long)n,
                             cudaGetErrorString(e));
    }
    h->cap_tri = n;
    h->sort_blocks_cap = nb;
    return RSI_OK;
}

// RSI_OPT_APETREI workspace: 4 words per triangle + one 64-bit node word
static rsi_status_t ensure_k63(rsi_bvh* h, int64_t n, cudaStream_t s) {
    if (n <= h->k63_cap) return RSI_OK;
    if (h->k63) cudaFreeAsync(h->k63, s);
    if (h->other) cudaFreeAsync(h->other, s);
    h->k63 = nullptr;
    h->other = nullptr;
    h->k63_cap = 0;
    cudaError_t e = cudaMallocAsync((void**)&h->k63, (size_t)n * 4 * sizeof(uint32_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&h->other, (size_t)n * sizeof(unsigned long long), s);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return rsi_set_error(RSI_E_OOM, "device allocation for the 63-bit build of %lld triangles failed: %s",
                             (long long)n, cudaGetErrorString(e));
    }
    h->k63_cap = n;
    return RSI_OK;
}

static void launch_sort(rsi_bvh* h, int n, cudaStream_t s) {
    if (n <= kRankSortMax) {
        // rank sort: keys -> keys_tmp (then swapped into h->keys), indices -> vals
        const int bx = rsi_ceil_div(n, kRankI);
        int sy = rsi_ceil_div(148 * 3, bx);
        if (sy > 64) sy = 64;
        int slice = (rsi_ceil_div(n, sy) + 3) & ~3;
        sy = rsi_ceil_div(n, slice);
        rsi_note_launch(), k_sort_rank<<<dim3(bx, sy), kRankT, (size_t)slice * 4, s>>>(
            h->keys, n, slice, reinterpret_cast<uint32_t*>(h->vals_tmp), h->keys_tmp, h->vals,
            h->scratch + SCR_SORT_DONE);
        uint32_t* t = h->keys;
        h->keys = h->keys_tmp;
        h->keys_tmp = t;
        return;
    }
    int nb = rsi_ceil_div(n, kTile);
    for (int p = 0; p < kPasses; ++p) {
        uint32_t* ks = (p & 1) ? h->keys_tmp : h->keys;
        int32_t* vs = (p & 1) ? h->vals_tmp : h->vals;
        uint32_t* kd = (p & 1) ? h->keys : h->keys_tmp;
        int32_t* vd = (p & 1) ? h->vals : h->vals_tmp;
        rsi_note_launch(), k_sort_hist<<<nb, kTileThreads, 0, s>>>(ks, n, 8 * p, h->hist);
        rsi_note_launch(), k_sort_rowscan<<<kDigits, kDigits, 0, s>>>(h->hist, nb, h->hist + (size_t)kDigits * nb);
        rsi_note_launch(), k_sort_scatter<<<nb, kTileThreads, 0, s>>>(ks, vs, kd, vd, n, 8 * p, h->hist,
                                                                      h->hist + (size_t)kDigits * nb);
    }
}

rsi_status_t rsi_build_device(rsi_bvh* h, const float* V, int64_t nv, const int32_t* T, int64_t nt,
                              cudaStream_t s) {
    h->n_tri = 0;
    h->n_nodes = 0;
    if (nt > (int64_t)1 << 30)
        return rsi_set_error(RSI_E_INVALID_ARG, "n_triangles %lld exceeds 2^30", (long long)nt);
    rsi_status_t st = ensure_capacity(h, nt, s);
    if (st != RSI_OK) return st;
    const int n = (int)nt;
    const int n_nodes = n > 1 ? n - 1 : 1;
    const bool apetrei = (h->opt.flags & RSI_OPT_APETREI) && n > 1;
    if (apetrei) {
        st = ensure_k63(h, nt, s);
        if (st != RSI_OK) return st;
    }
    h->apetrei = apetrei;
    rsi_note_launch(), k_build_init<<<1, 32, 0, s>>>(h->scratch, apetrei ? 0xffffffffu : 0u);
    int64_t work = nv > 3 * nt ? nv : 3 * nt;
    int eb = rsi_ceil_div(work, kBlock);
    if (eb > 148 * 8) eb = 148 * 8;
    rsi_note_launch(), k_extent_validate<<<eb, kBlock, 0, s>>>(V, nv, T, nt, h->scratch);
    // the construction grid covers every leaf (case study 2: never size it from
    // another count) -- except under the test-only fault injection option
    const int refit_leaves = (h->opt.debug_refit_leaves > 0 && h->opt.debug_refit_leaves < n)
                                 ? (int)h->opt.debug_refit_leaves : n;
    uint32_t* rank = n <= kRankSortMax ? reinterpret_cast<uint32_t*>(h->vals_tmp) : nullptr;
    if (refit_leaves < n)  // fault injection: untouched nodes hold empty (zero) boxes, not stale memory
        cudaMemsetAsync(h->nodes, 0, (size_t)n_nodes * 4 * sizeof(float4), s);
    if (apetrei) {
        uint32_t* k_lo = h->k63;
        uint32_t* k_hi = h->k63 + nt;
        int32_t* ids1 = reinterpret_cast<int32_t*>(h->k63 + 2 * nt);
        uint32_t* lo_sorted = h->k63 + 3 * nt;
        rsi_note_launch(), k_morton63<<<rsi_ceil_div(n, kBlock), kBlock, 0, s>>>(V, nv, T, n, h->scratch, h->keys, h->vals,
                                                                                k_lo, k_hi, h->other, rank);
        launch_sort(h, n, s);  // stable by the low words
        rsi_note_launch(), k_pass2_prep<<<rsi_ceil_div(n > 32 ? n : 32, kBlock), kBlock, 0, s>>>(
            h->keys, h->vals, k_hi, ids1, n, n <= kRankSortMax ? reinterpret_cast<uint32_t*>(h->vals_tmp) : nullptr,
            h->scratch);
        launch_sort(h, n, s);  // stable by the high words: (hi, lo, index) order
        rsi_note_launch(), k_pass2_finish<<<rsi_ceil_div(n, kBlock), kBlock, 0, s>>>(h->vals, ids1, k_lo, lo_sorted, n);
        if (refit_leaves < n)  // fault injection: stale links read as broken, not as valid
            cudaMemsetAsync(h->parent, 0xfe, (size_t)(n_nodes + n) * sizeof(int32_t), s);
        rsi_note_launch(), k_apetrei<<<rsi_ceil_div(refit_leaves, kBlock), kBlock, 0, s>>>(
            V, nv, T, h->vals, h->keys, lo_sorted, refit_leaves, n, h->nodes, h->tris, h->parent, h->other, h->scratch);
    } else {
        if (RSI_SORT_SMALL && n <= kSortSmallMax) {  // A3 + A4 in one CTA
            static bool attr_ms = false;
            if (!attr_ms) {
                cudaFuncSetAttribute(k_morton_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sort_small_smem(kSortSmallMax));
                attr_ms = true;
            }
            rsi_note_launch(), k_morton_sort_small<<<1, kSortSmallT, sort_small_smem(n), s>>>(
                V, nv, T, n, h->scratch, h->keys, h->vals, h->arrivals, n_nodes);
        } else {
            rsi_note_launch(), k_morton<<<rsi_ceil_div(n, kBlock), kBlock, 0, s>>>(V, nv, T, n, h->scratch, h->keys,
                                                                                  h->vals, h->arrivals, n_nodes, rank);
            launch_sort(h, n, s);
        }
        const bool sah_sub = RSI_SAH_SUB > 0 && !(h->opt.flags & (RSI_OPT_PLAIN_TREE | RSI_OPT_ROTATE)) &&
                             refit_leaves == n && n >= kSahMinTri && n <= kSahMaxTri;
        int32_t* list = sah_sub ? reinterpret_cast<int32_t*>(h->keys_tmp) : nullptr;  // (free after the sort)
        rsi_note_launch(), k_karras<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(h->keys, n, h->nodes, h->parent,
                                                                                   h->arrivals, list, h->scratch, kSahSub);
        if (sah_sub) {
            const int g = rsi_ceil_div(n, 3) < kSahGrid ? rsi_ceil_div(n, 3) : kSahGrid;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_sah_sub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSahSmem);
                attr = true;
            }
            rsi_note_launch(), k_sah_sub<<<g, 32 * kSahWarps, kSahSmem, s>>>(V, nv, T, h->vals, h->nodes, h->tris, h->parent,
                                                                     h->arrivals, n_nodes, list, h->scratch);
        }
        // (with the SAH subtrees, k_sah_sub packs the triangles, writes every box
        // inside the subtrees and refits the Karras nodes above them: no k_refit)
        const int treelet = (h->opt.flags & (RSI_OPT_PLAIN_TREE | RSI_OPT_ROTATE)) || refit_leaves < n ||
                                    n > kTreeletMaxTri ? 0 : 1;
        const int rotate = (h->opt.flags & RSI_OPT_ROTATE) ? 1 : 0;
        if (sah_sub) {
        } else if (treelet)
            rsi_note_launch(), k_refit<true><<<rsi_ceil_div(refit_leaves, kRefitLeaves), kRefitLeaves, 0, s>>>(
                V, nv, T, h->vals, refit_leaves, n, h->nodes, h->tris, h->parent, h->arrivals, h->scratch, rotate, 1);
        else
            rsi_note_launch(), k_refit<false><<<rsi_ceil_div(refit_leaves, kRefitLeaves), kRefitLeaves, 0, s>>>(
                V, nv, T, h->vals, refit_leaves, n, h->nodes, h->tris, h->parent, h->arrivals, h->scratch, rotate, 0);
    }
    if (n_nodes <= kQCompactMax && h->qfull) {  // records of every node, then the live ones, breadth-first
        rsi_note_launch(), k_quads<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(h->nodes, n_nodes, h->qfull, h->scratch);
        rsi_note_launch(), k_qcompact<<<1, 1024, 0, s>>>(h->qfull, h->quads, h->qorder, h->qmap, h->scratch);
    } else {
        rsi_note_launch(), k_quads<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(h->nodes, n_nodes, h->quads, h->scratch);
    }
    if (kQTop > 0) rsi_note_launch(), k_qtop<<<1, 256, 0, s>>>(h->quads, h->top, h->scratch);
    st = rsi_cuda_check(cudaGetLastError(), "build kernel launch");
    if (st != RSI_OK) return st;
    h->n_tri = nt;
    h->n_nodes = n_nodes;
    h->stream = s;
    h->pending_nv = nv;
    h->status_pending = true;
    if (h->opt.flags & RSI_OPT_DEFERRED_STATUS) return RSI_OK;  // checked by rsi_build_status
    return rsi_finish_build(h, s);
}

// Read back the build's scratch words (status bits, scene box) and report the
// device-side input checks; an invalid mesh leaves the handle without a mesh.
rsi_status_t rsi_finish_build(rsi_bvh* h, cudaStream_t s) {
    if (!h->status_pending) return h->n_tri > 0 ? RSI_OK : rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh");
    h->status_pending = false;
    rsi_status_t st = rsi_cuda_check(cudaMemcpyAsync(h->h_words, h->scratch, SCR_WORDS * sizeof(uint32_t),
                                                     cudaMemcpyDeviceToHost, s),
                                     "status read");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "build");
    const uint32_t status = st == RSI_OK ? h->h_words[SCR_STATUS] : 0u;
    if (st == RSI_OK && (status & STATUS_INDEX))
        st = rsi_set_error(RSI_E_INDEX_RANGE, "a triangle index is outside [0, %lld)", (long long)h->pending_nv);
    else if (st == RSI_OK && (status & STATUS_NONFINITE))
        st = rsi_set_error(RSI_E_NONFINITE, "a vertex coordinate is NaN or Inf");
    else if (st == RSI_OK && (status & STATUS_RANGE))
        st = rsi_set_error(RSI_E_INVALID_ARG, "mesh extent too large for the quantized BVH (|coordinates| > ~1e33)");
    if (st != RSI_OK) {
        h->n_tri = 0;
        h->n_nodes = 0;
        return st;
    }
    const float* root = reinterpret_cast<const float*>(h->h_words + SCR_ROOT);
    for (int x = 0; x < 3; ++x) {
        h->scene_lo[x] = root[x];
        h->scene_hi[x] = root[3 + x];
    }
    h->root_node = h->h_words[SCR_ROOT_NODE] == 0xffffffffu ? -1 : (int64_t)h->h_words[SCR_ROOT_NODE];
    return RSI_OK;
}

rsi_status_t rsi_validate_device(rsi_bvh* h, rsi_integrity_t* report, cudaStream_t s) {
    const int n = (int)h->n_tri, n_nodes = (int)h->n_nodes;
    unsigned long long* out = nullptr;
    uint32_t* seen = nullptr;
    rsi_status_t st = rsi_cuda_check(cudaMallocAsync((void**)&out, V_WORDS * sizeof(unsigned long long), s), "validate");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMallocAsync((void**)&seen, (size_t)n * sizeof(uint32_t), s), "validate");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemsetAsync(out, 0, V_WORDS * sizeof(unsigned long long), s), "memset");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemsetAsync(seen, 0, (size_t)n * sizeof(uint32_t), s), "memset");
    if (st == RSI_OK) {
        rsi_note_launch(), k_validate_nodes<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(
            h->nodes, n, n_nodes, h->parent, h->arrivals, h->apetrei ? h->other : nullptr, out);
        rsi_note_launch(), k_validate_leaves<<<rsi_ceil_div(n, kBlock), kBlock, 0, s>>>(h->tris, n, n_nodes, h->scratch,
                                                                                      h->parent, seen, out);
        rsi_note_launch(), k_validate_ids<<<rsi_ceil_div(n, kBlock), kBlock, 0, s>>>(seen, n, out);
        st = rsi_cuda_check(cudaGetLastError(), "validate launch");
    }
    unsigned long long v[V_WORDS] = {0};
    uint32_t root_set = 0;
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(v, out, sizeof(v), cudaMemcpyDeviceToHost, s), "validate");
    if (st == RSI_OK)
        st = rsi_cuda_check(cudaMemcpyAsync(&root_set, h->scratch + SCR_ROOT_SET, 4, cudaMemcpyDeviceToHost, s), "validate");
    if (out) cudaFreeAsync(out, s);
    if (seen) cudaFreeAsync(seen, s);
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "validate");
    if (st != RSI_OK) return st;
    report->n_internal = n_nodes;
    report->half_filled = (int64_t)v[V_HALF];
    report->untouched = (int64_t)v[V_UNTOUCHED];
    report->bad_leaf_ids = (int64_t)v[V_LEAFIDS];
    report->bad_links = (int64_t)v[V_LINKS];
    report->bad_boxes = (int64_t)v[V_BOXES];
    report->unreachable_leaves = (int64_t)v[V_UNREACH];
    report->root_ok = root_set ? 1 : 0;
    return RSI_OK;
}

// rsi_bvh_upload: replace the handle's binary tree by a caller-given topology
// over the same mesh (the inverse of rsi_bvh_download; a debugging and
// tree-quality experiment hook: the walk is exact for ANY valid tree, since a
// BVH only prunes).  Host inputs: child refs / child boxes in the download
// layout, the triangle at each leaf slot, the root node.  The triangle records
// are permuted into the new slot order, then the 4-wide records are rebuilt
// from the uploaded nodes exactly as after a build.
rsi_status_t rsi_bvh_upload_device(rsi_bvh* h, const int32_t* h_child, const float* h_box,
                                   const int32_t* h_leaf_tri, int64_t root, cudaStream_t s) {
    const int64_t nn = h->n_nodes, nt = h->n_tri;
    if (nt < 2 || root < 0 || root >= nn)
        return rsi_set_error(RSI_E_INVALID_ARG, "upload needs N_t >= 2 and a root in [0, n_nodes)");
    float4* tris = new (std::nothrow) float4[kTriF4 * nt];
    float4* ntris = new (std::nothrow) float4[kTriF4 * nt];
    float4* nodes = new (std::nothrow) float4[4 * nn];
    int64_t* slot_of = new (std::nothrow) int64_t[nt];
    rsi_status_t st = (tris && ntris && nodes && slot_of) ? RSI_OK : rsi_set_error(RSI_E_OOM, "host allocation failed");
    if (st == RSI_OK)
        st = rsi_cuda_check(cudaMemcpyAsync(tris, h->tris, nt * kTriF4 * sizeof(float4), cudaMemcpyDeviceToHost, s), "tris");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "tris");
    if (st == RSI_OK) {
        for (int64_t i = 0; i < nt; ++i) slot_of[i] = -1;
        for (int64_t k = 0; k < nt; ++k) {
            int32_t id;
            std::memcpy(&id, &tris[kTriF4 * k].w, 4);
            if (id >= 0 && id < nt) slot_of[id] = k;
        }
        for (int64_t k = 0; k < nt && st == RSI_OK; ++k) {
            const int32_t id = h_leaf_tri[k];
            if (id < 0 || id >= nt || slot_of[id] < 0) {  // (a used id is marked -1: not a permutation)
                st = rsi_set_error(RSI_E_INVALID_ARG, "leaf slot %lld: triangle %d (leaf_tri must be a permutation)",
                                   (long long)k, id);
                break;
            }
            for (int f = 0; f < kTriF4; ++f) ntris[kTriF4 * k + f] = tris[kTriF4 * slot_of[id] + f];
            slot_of[id] = -1;
        }
    }
    if (st == RSI_OK) {  // topology: every internal node and leaf slot reached exactly once from root
        std::vector<unsigned char> seen((size_t)(nn + nt), 0);
        std::vector<int64_t> todo(1, root);
        seen[root] = 1;
        int64_t reached = 1;
        while (!todo.empty() && st == RSI_OK) {
            const int64_t i = todo.back();
            todo.pop_back();
            for (int side = 0; side < 2; ++side) {
                const int32_t c = h_child[2 * i + side];
                const int64_t at = c >= 0 ? (int64_t)c : nn + (int64_t)~c;
                if ((c >= 0 && c >= nn) || (c < 0 && (int64_t)~c >= nt) || seen[at]) {
                    st = rsi_set_error(RSI_E_INVALID_ARG, "node %lld child %d: ref %d out of range or reached twice",
                                       (long long)i, side, c);
                    break;
                }
                seen[at] = 1;
                ++reached;
                if (c >= 0) todo.push_back(c);
            }
        }
        if (st == RSI_OK && reached != nn + nt)
            st = rsi_set_error(RSI_E_INVALID_ARG, "the tree reaches %lld of %lld nodes and leaves", (long long)reached,
                               (long long)(nn + nt));
    }
    if (st == RSI_OK) {
        for (int64_t i = 0; i < nn; ++i) {
            const float* b = h_box + 12 * i;  // [2][6]: lo xyz, hi xyz per side
            nodes[4 * i + 0] = make_float4(b[0], b[3], b[1], b[4]);
            nodes[4 * i + 1] = make_float4(b[6], b[9], b[7], b[10]);
            nodes[4 * i + 2] = make_float4(b[2], b[5], b[8], b[11]);
            float4 r;
            std::memcpy(&r.x, &h_child[2 * i], 4);
            std::memcpy(&r.y, &h_child[2 * i + 1], 4);
            r.z = r.w = 0.0f;
            nodes[4 * i + 3] = r;
        }
        st = rsi_cuda_check(cudaMemcpyAsync(h->nodes, nodes, nn * 4 * sizeof(float4), cudaMemcpyHostToDevice, s), "nodes");
    }
    if (st == RSI_OK)
        st = rsi_cuda_check(cudaMemcpyAsync(h->tris, ntris, nt * kTriF4 * sizeof(float4), cudaMemcpyHostToDevice, s), "tris");
    // parent links and arrival counts of the uploaded tree (what the validator and
    // the download report), the scene box for rsi_bvh_info
    std::vector<int32_t> par((size_t)(nn + nt), -1);
    std::vector<uint32_t> arr((size_t)nn, 2u);
    float scene[6];
    uint32_t one = 1u;
    if (st == RSI_OK) {
        for (int64_t i = 0; i < nn; ++i)
            for (int side = 0; side < 2; ++side) {
                const int32_t c = h_child[2 * i + side];
                par[c >= 0 ? (size_t)c : (size_t)(nn + ~c)] = (int32_t)((i << 1) | side);
            }
        for (int x = 0; x < 3; ++x) {
            scene[x] = fminf(h_box[12 * root + x], h_box[12 * root + 6 + x]);
            scene[3 + x] = fmaxf(h_box[12 * root + 3 + x], h_box[12 * root + 9 + x]);
        }
        st = rsi_cuda_check(cudaMemcpyAsync(h->parent, par.data(), (nn + nt) * sizeof(int32_t), cudaMemcpyHostToDevice, s),
                            "parents");
    }
    if (st == RSI_OK)
        st = rsi_cuda_check(cudaMemcpyAsync(h->arrivals, arr.data(), nn * sizeof(uint32_t), cudaMemcpyHostToDevice, s),
                            "arrivals");
    if (st == RSI_OK) {
        const int n_nodes = (int)nn;
        rsi_note_launch(), k_build_init<<<1, 32, 0, s>>>(h->scratch, (uint32_t)root);
        cudaMemcpyAsync(h->scratch + SCR_ROOT, scene, sizeof(scene), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(h->scratch + SCR_ROOT_SET, &one, sizeof(one), cudaMemcpyHostToDevice, s);
        if (n_nodes <= kQCompactMax && h->qfull) {
            rsi_note_launch(), k_quads<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(h->nodes, n_nodes, h->qfull, h->scratch);
            rsi_note_launch(), k_qcompact<<<1, 1024, 0, s>>>(h->qfull, h->quads, h->qorder, h->qmap, h->scratch);
        } else {
            rsi_note_launch(), k_quads<<<rsi_ceil_div(n_nodes, kBlock), kBlock, 0, s>>>(h->nodes, n_nodes, h->quads, h->scratch);
        }
        if (kQTop > 0) rsi_note_launch(), k_qtop<<<1, 256, 0, s>>>(h->quads, h->top, h->scratch);
        st = rsi_cuda_check(cudaGetLastError(), "upload kernels");
    }
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "upload");
    if (st == RSI_OK) {
        h->apetrei = false;
        h->root_node = root;
    }
    delete[] tris;
    delete[] ntris;
    delete[] nodes;
    delete[] slot_of;
    return st;
}
