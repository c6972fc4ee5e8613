// rsi_internal.cuh -- shared internals of the sm_100a CUDA path (not part of the ABI).
//
// Layouts:
//   node  (64 B, 4 x float4) -- a "child pair": both children's AABBs + refs
//     n0 = (L.lo.x, L.hi.x, L.lo.y, L.hi.y)
//     n1 = (R.lo.x, R.hi.x, R.lo.y, R.hi.y)
//     n2 = (L.lo.z, L.hi.z, R.lo.z, R.hi.z)
//     n3 = (ref L, ref R, 0, 0) as int bits; ref >= 0 internal node, < 0 leaf ~slot
//   quad  (64 B, 4 x float4) -- for every internal node n, its up-to-4
//         cut members (a leaf child stands for itself) with 8-bit quantized
//         AABBs on a power-of-two grid (see k_quads in build.cu); traversing
//         quads visits every other level of the binary tree.
//   tri   (64 B, 4 x float4) in Morton order: (v0, id bits), (v1, 0), (v2, 0), pad
//         (64 B so a triangle is two 256-bit loads)
//   The vertices are stored exactly (not e1/e2) so the fp64 mirror can
//   recompute the oracle's operation order bit-for-bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rsi.h"

#define RSI_VERSION_STRING "rsi-b200 0.1.0 sm_100a"

// scratch words (uint32) in rsi_bvh::scratch
enum {
    SCR_EXT_MIN = 0,   // 3 words: order-preserving encoded min x,y,z
    SCR_EXT_MAX = 3,   // 3 words: encoded max
    SCR_STATUS = 6,    // bit 0 index out of range, bit 1 non-finite vertex
    SCR_ROOT = 9,      // 6 words: root (scene) AABB as float bits
    SCR_OVF_COUNT = 16, // intercept_count overflow list length
    SCR_OVF_NEXT = 17,  // intercept_count re-pass: next overflowed segment (work counter)
    SCR_DISPENSER = 18, // 2 words: 64-bit ray dispenser of the persistent traversal grid
    SCR_NTOP = 20,      // records in the top-of-tree shared-memory image (k_qtop)
    SCR_ROOT_SET = 21,  // 1 once the refit wrote the root box
    SCR_QPMAX = 22,     // max |decode offset| over the quad records (float bits, >= 0)
    SCR_QEMIN = 23,     // min / max grid exponent + 128 over the quad records
    SCR_QEMAX = 24,
    SCR_ROOT_NODE = 25, // root internal node (0 Karras; Apetrei: top split; 0xffffffff unset)
    SCR_QROOT = 26,     // root of the 4-wide records the walks read (0 after compaction; 0xffffffff unset)
    SCR_SAH_COUNT = 27, // SAH-rebuilt subtrees in this build (k_sah_roots)
    SCR_SORT_DONE = 32, // 32 words: per-block slice counters of the rank sort
    SCR_WORDS = 64
};
enum { STATUS_INDEX = 1u, STATUS_NONFINITE = 2u, STATUS_RANGE = 4u };

// stats counters (unsigned long long) in rsi_bvh::stats
enum {
    ST_RAYS = 0, ST_FP64_PAIRS, ST_FP64_RAYS, ST_OVERFLOW, ST_NONFINITE, ST_BOX_TESTS, ST_MT_TESTS,
    // SIMT-efficiency diagnostics (RSI_OPT_COUNTERS): lane-iterations by state
    ST_IT_SEARCH, ST_IT_PEND, ST_IT_IDLE, ST_ITERS, ST_LEAF_LANES, ST_LEAF_PHASES,
    ST_WORDS
};

struct rsi_bvh {
    int device = 0;
    cudaStream_t stream = nullptr;  // build stream (frees are ordered on it)
    rsi_options_t opt{};
    int64_t n_tri = 0, n_nodes = 0;  // current mesh
    int64_t cap_tri = 0;             // allocated capacity (triangles)
    int64_t sort_blocks_cap = 0;
    float4* nodes = nullptr;         // [4 * n_nodes]
    float4* quads = nullptr;         // [4 * n_nodes] compressed 4-wide cut records the walks read: the live
                                     // records only, breadth-first from index 0 (k_qcompact), or indexed
                                     // by binary node id above kQCompactMax nodes
    float4* qfull = nullptr;         // [4 * n_nodes] k_quads output (one record per internal node)
    int32_t* qorder = nullptr;       // [n_nodes] compaction: live record i's binary node
    int32_t* qmap = nullptr;         // [n_nodes] compaction: binary node -> live record index
    float4* top = nullptr;           // [4 * kQTop] top-of-tree image of the 4-wide records
                                     // (refs >= kSmemRef are image slots; record count in SCR_NTOP)
    float4* tris = nullptr;          // [4 * n_tri]
    uint32_t* keys = nullptr;        // sorted Morton codes [n_tri]
    int32_t* vals = nullptr;         // sorted triangle ids [n_tri]
    uint32_t* keys_tmp = nullptr;
    int32_t* vals_tmp = nullptr;
    int32_t* parent = nullptr;       // [n_nodes + n_tri]
    uint32_t* arrivals = nullptr;    // [n_nodes]
    // RSI_OPT_APETREI (63-bit codes + agglomerative build): [4 * cap] words --
    // code lo / hi words in triangle order, pass-1 ids, sorted lo words -- and
    // the per-node 64-bit (arrivals << 32 | first bound) words [cap]
    uint32_t* k63 = nullptr;
    unsigned long long* other = nullptr;
    int64_t k63_cap = 0;
    bool apetrei = false;            // the current tree was built by the Apetrei path
    int64_t root_node = 0;           // host copy of SCR_ROOT_NODE (valid after the status read)
    uint32_t* hist = nullptr;        // sort: [256 * blocks]
    uint32_t* scratch = nullptr;     // [SCR_WORDS]
    unsigned long long* stats = nullptr;  // [ST_WORDS]
    uint32_t h_words[64] = {};       // host words for status reads (small synchronous copies;
                                     // no cudaMallocHost per handle -- it costs ~ms)
    // intercept_count overflow workspace
    int32_t* ovf_list = nullptr;     // ray ids
    int64_t ovf_cap = 0;
    float scene_lo[3] = {0, 0, 0}, scene_hi[3] = {0, 0, 0};
    bool status_pending = false;     // build checks not yet read back (RSI_OPT_DEFERRED_STATUS)
    int64_t pending_nv = 0;          // n_vertices of that build (error message)
    uint64_t host_rays = 0;  // rays counted on the host
    int min_trav = -1;  // traversal-phase exit threshold (-1: per-mode default); env RSI_MIN_TRAV
    // stream ordering across calls (the handle's scratch -- ray dispenser,
    // overflow counters -- is reset by every call): each call records
    // `order_ev` on its stream; a call on a DIFFERENT stream first waits on it
    cudaEvent_t order_ev = nullptr;
    cudaStream_t last_stream = nullptr;
    bool order_valid = false;
};

// ---------------------------------------------------------------- host helpers (api.cu)
rsi_status_t rsi_set_error(rsi_status_t s, const char* fmt, ...);
rsi_status_t rsi_cuda_check(cudaError_t e, const char* what);
void rsi_keep_pool_cached();

// build.cu
rsi_status_t rsi_build_device(rsi_bvh* h, const float* d_vertices, int64_t n_vertices,
                              const int32_t* d_triangles, int64_t n_triangles,
                              cudaStream_t stream);
rsi_status_t rsi_bvh_upload_device(rsi_bvh* h, const int32_t* h_child, const float* h_box,
                                   const int32_t* h_leaf_tri, int64_t root, cudaStream_t stream);
// traverse.cu
rsi_status_t rsi_intersect_device(rsi_bvh* h, const float* d_start, const float* d_end,
                                  int64_t n_rays, int32_t mode, const rsi_outputs_t* out,
                                  cudaStream_t stream);
bool rsi_uses_quads();  // traverse.cu: does any mode walk the 4-wide records
// process-wide count of kernels this library launched (rsi_launch_count)
void rsi_note_launch();
rsi_status_t rsi_finish_build(rsi_bvh* h, cudaStream_t stream);  // build.cu: read back + check
rsi_status_t rsi_validate_device(rsi_bvh* h, rsi_integrity_t* report, cudaStream_t stream);  // build.cu
rsi_status_t rsi_compact_device(const int32_t* d_tri, int64_t n_rays, int32_t* d_ids,
                                int32_t* d_n, cudaStream_t stream);
// traverse.cu: values of the compacted hit rays (sparse barycentric return)
rsi_status_t rsi_gather_hits_device(const int32_t* ids, const int32_t* n_hits, int64_t n_max, const int32_t* tri,
                                    const float* dist, const float* point, int32_t* out_tri, float* out_dist,
                                    float* out_point, cudaStream_t s);

// ---------------------------------------------------------------- device helpers

// Order-preserving float <-> uint32 map (monotone over all non-NaN floats), so
// that float min/max can use integer atomics.
__host__ __device__ inline uint32_t rsi_f2ord(float f) {
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(f);
#else
    uint32_t u;
    __builtin_memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float rsi_ord2f(uint32_t u) {
    uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}

// triangle record: 4 float4 (64 B: two 256-bit loads, the default) or, with
// RSI_TRI48, 3 float4 (48 B: three 128-bit loads, a smaller working set)
#ifndef RSI_TRI48
#define RSI_TRI48 0
#endif
constexpr int kTriF4 = RSI_TRI48 ? 3 : 4;

// 4-wide record decode bias M: a child plane is (M + q) s + pm with pm = p - M s
// stored.  M = 2^15 (default): M + q is one PRMT into the float 2^15's mantissa;
// RSI_HALF_DECODE: M = 1024, one PRMT places two bytes into two f16 1024 + q
// (0x64qq) and HADD2.F32 (FMA pipe) widens each -- half the PRMTs on the ALU pipe
#ifndef RSI_HALF_DECODE
#define RSI_HALF_DECODE 1
#endif
constexpr double kQuadBias = RSI_HALF_DECODE ? 1024.0 : 32768.0;
constexpr uint32_t kQuadMagic = RSI_HALF_DECODE ? 0x00000064u : 0x47000000u;

// 4-wide records hold a greedy largest-area 4-cut of each node's subtree
// (RSI_QUAD_GREEDY) instead of its grandchildren: a member may sit 1 .. 3
// levels below the node, so the walk's stack bound is 3 entries per level
#ifndef RSI_QUAD_GREEDY
#define RSI_QUAD_GREEDY 1
#endif

// top-of-tree shared-memory image of the 4-wide records (build.cu k_qtop,
// traverse.cu): the first RSI_QTOP records of the walk, breadth-first
#ifndef RSI_QTOP
#define RSI_QTOP 0  // measured slower on the 4-wide walk (21..256 records: +4..6 %), DESIGN.md 7
#endif
constexpr int kQTop = RSI_QTOP;               // <= 256 (k_qtop: one slot per thread of a level)
static_assert(kQTop >= 0 && kQTop <= 256, "RSI_QTOP");
// 4-wide record compaction (build.cu k_qcompact, one CTA): meshes up to this
// many internal nodes; larger ones keep the records indexed by node id
#ifndef RSI_QCOMPACT_MAX
#define RSI_QCOMPACT_MAX 0  // measured: query -0.3 %, rebuild +44 us (N_t = 1e4): off
#endif
constexpr int kQCompactMax = RSI_QCOMPACT_MAX;
constexpr uint32_t kSmemRef = 0x40000000u;    // member ref >= kSmemRef: slot in the image
constexpr int kNoRefB = (int)0x80000000;      // "no member" (the walk's kNoRef)

static inline int rsi_ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
