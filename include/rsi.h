/*
 * rsi.h -- C-ABI of the B200-native segment x triangle-mesh intersection
 * library (arXiv 2305.01867 and its CUDA predecessor arXiv 2209.02878).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY 8(b).
 *
 * Problem (section 1 "Background"): N_r line segments ("rays")
 * l_i = (r_i^start, r_i^end) are tested against a surface of N_t triangles
 * t_j = [t_j1, t_j2, t_j3] indexing vertices {v_n}.  A linear BVH built from
 * Morton codes of the triangles and a binary radix tree prunes the candidate
 * triangles; each candidate is tested with Moller-Trumbore.
 * Three modes: boolean, barycentric (nearest intersecting triangle,
 * distance and point), intercept_count (number of unique intersections).
 *
 * Conventions for every entry point
 *   - Pointers prefixed d_ are DEVICE pointers on the current CUDA device;
 *     h_ are HOST pointers.  Arrays are dense, C-order, little-endian.
 *   - Points are float32 [n][3] (x, y, z); triangle indices are int32 [n][3]
 *     (the int32-everywhere lesson of case study 1, P:272-299, P:498 -- a
 *     64-bit index array passed here is a caller bug the Python binding
 *     rejects rather than casting).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device work is stream-ordered; calls return when work is ENQUEUED unless
 *     stated otherwise.
 *   - Every call returns rsi_status_t.  On failure rsi_last_error() returns a
 *     thread-local message; CUDA errors are never swallowed.
 *   - The library is thread-compatible: a handle may be used by one thread at a
 *     time; distinct handles are independent.
 *   - Calls on one handle execute on the device in CALL order, whatever streams
 *     they are given: every rsi_rebuild / rsi_intersect records an event on its
 *     stream, and a call on a different stream than the previous one first
 *     waits on that event (device-side).  This orders the handle's per-call
 *     scratch (ray dispenser, overflow counters), which every call resets.
 *     rsi_free frees after the last call.  Work on distinct handles is not
 *     ordered.
 *   - Pipelining (what bench.py does): a caller that rebuilds and queries every
 *     step can alternate two handles (built with RSI_OPT_DEFERRED_STATUS) on
 *     two streams, so that step k+1's rebuild runs in the SM slots step k's
 *     traversal frees at its end; each handle's own calls stay in call order,
 *     and rsi_build_status reports each handle's input checks afterwards.
 */
#ifndef RSI_H_
#define RSI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RSI_OK = 0,
    RSI_E_INVALID_ARG = 1, /* null pointer, negative size, bad mode, bad options       */
    RSI_E_EMPTY = 2,       /* N_t == 0 or N_v == 0 ("empty mesh")                 */
    RSI_E_INDEX_RANGE = 3, /* a triangle index outside [0, N_v)                 */
    RSI_E_NONFINITE = 4,   /* a NaN / Inf vertex coordinate                   */
    RSI_E_CUDA = 5,        /* a CUDA runtime error; message has cudaGetErrorString      */
    RSI_E_OOM = 6,         /* device allocation failed                                  */
    RSI_E_INTEGRITY = 7    /* BVH validator found a violation               */
} rsi_status_t;

/* Modes. */
typedef enum {
    RSI_MODE_BOOLEAN = 0,        /* P:26 "(N_r,1) boolean array"                        */
    RSI_MODE_BARYCENTRIC = 1,    /* P:27 nearest triangle, distance and point           */
    RSI_MODE_INTERCEPT_COUNT = 2 /* P:28 "number of unique intersections"               */
} rsi_mode_t;

/* Option bits (rsi_options_t.flags). */
#define RSI_OPT_FP64_MOLLER 1u /* every Moller-Trumbore test in double precision: the
                                  paper's USE_DOUBLE_PRECISION_MOLLER.  Results
                                  are identical either way; only speed differs. */
#define RSI_OPT_COUNTERS 2u    /* count box tests and Moller-Trumbore tests in rsi_stats_t
                                  (instrumented kernels; for roofline accounting, slower). */
#define RSI_OPT_DEFERRED_STATUS 4u /* rsi_build / rsi_rebuild only enqueue the build and
                                  return RSI_OK without waiting for the device; the
                                  device-side input checks (index range, non-finite
                                  vertex, extent) are reported by rsi_build_status, which
                                  synchronizes.  Until it returns RSI_OK the outputs of an
                                  rsi_intersect on an invalid mesh are unspecified (no
                                  out-of-bounds access either way).  For pipelines that
                                  rebuild and query every step with no host round trip. */
#define RSI_OPT_ROTATE 16u     /* one bottom-up pass of local tree rotations fused into the
                                  refit (default Karras path): at each completed node swap a
                                  child with a grandchild on the other side when that shrinks
                                  the rebuilt child's surface area (SAH-style, after Kensler).
                                  Fewer box tests per segment; the leaf order (Morton) is
                                  kept, so the paper's node numbering is not.
                                  Same results. */
#define RSI_OPT_PLAIN_TREE 32u /* keep the Karras topology exactly as built (the paper's Fig. 3
                                  structure and node numbering).  By default the
                                  tree's quality is raised after k_karras, same leaves, same
                                  results (the BVH only prunes): for meshes of up to 32768
                                  triangles every maximal Karras subtree of <= 256 leaves is
                                  rebuilt top-down by binned SAH (its leaves permuted within
                                  its slot range, the Karras tree above it kept); for 32769 ..
                                  65536 triangles the refit's bottom-up climb rebuilds the
                                  treelet of every node completed inside a CTA's 256-leaf
                                  window (up to 5 largest-area descendants, Karras & Aila
                                  2013) as the binary tree of least surface-area cost.  Also
                                  off under RSI_OPT_ROTATE and ignored under RSI_OPT_APETREI. */
#define RSI_OPT_APETREI 8u     /* the paper's construction instead of
                                  Karras + refit -- 63-bit Morton codes (21 bits per axis,
                                  z-major; "64-bit Morton codes") sorted as
                                  two stable 32-bit LSD passes, then Apetrei's single-pass
                                  agglomerative build: one thread per leaf
                                  climbs, choosing its parent by comparing the common
                                  prefix with its left and right neighbours, and the
                                  second arrival at a node (a 64-bit atomic that also
                                  counts arrivals) merges the boxes.  Internal node i is
                                  the split between sorted leaves i and i+1, so the root
                                  is not node 0 (rsi_bvh_root) and the sentinel N_t - 1
                                  "only holds a pointer to the root".
                                  Same results; only the tree differs.  N_t == 1 uses the
                                  default path. */

typedef struct {
    uint32_t struct_size; /* sizeof(rsi_options_t); 0 or a NULL options pointer = defaults   */
    uint32_t flags;       /* RSI_OPT_* bits (default 0)                                      */
    double dedup_tau;     /* intercept_count: hits whose t differ by <= tau merge (single
                             linkage on t, reading R4).  Default 1e-6 (t units).   */
    int64_t debug_refit_leaves; /* FAULT INJECTION (tests only): > 0 runs the bottom-up refit
                             over only the first k leaves -- case study 2's under-sized grid
                              -- leaving half-filled / untouched nodes and no root
                             box for rsi_validate to report.  0 (default) = all leaves.      */
} rsi_options_t;

/* BVH integrity report (rsi_validate), the invariants whose violation the
 * paper diagnosed by dumping the tree (case study 1; case study 2,
 * P:407-464).  All counts are 0 for a valid tree. */
typedef struct {
    int64_t n_internal;        /* internal nodes checked (max(N_t - 1, 1))                   */
    int64_t half_filled;       /* internal nodes with refit arrival count 1 ("atomic: 1")   */
    int64_t untouched;         /* internal nodes never reached by the refit ("atomic: 0")   */
    int64_t bad_leaf_ids;      /* triangle ids missing or repeated among the leaves */
    int64_t bad_links;         /* child -> parent -> child links that do not agree           */
    int64_t bad_boxes;         /* child boxes not equal to the union of their children       */
    int64_t unreachable_leaves;/* leaves whose parent chain does not reach the root          */
    int32_t root_ok;           /* 1 when the root box was written by the refit  */
} rsi_integrity_t;

/* Opaque BVH handle: owns the packed triangles and the BVH on the device
 * where it was built.  Created by rsi_build, destroyed by rsi_free. */
typedef struct rsi_bvh* rsi_handle_t;

/*
 * Caller-owned per-ray outputs for rsi_intersect (device pointers) and
 * rsi_test (host pointers).  Which fields are written depends on the mode;
 * fields of other modes are ignored and may be NULL.
 *   BOOLEAN:          hit[n]   uint8 0/1
 *   INTERCEPT_COUNT:  count[n] int32 >= 0
 *   BARYCENTRIC:      tri[n]   int32 original triangle index, -1 on a miss
 *                     t[n]     float32 parametric position in [0,1]       (optional)
 *                     dist[n]  float32 t * |end - start|   (3b)     (optional)
 *                     point[n][3] float32 start + t*(end - start) (3d) (optional)
 *                     t/dist/point are NaN on a miss.
 */
typedef struct {
    uint8_t* hit;
    int32_t* count;
    int32_t* tri;
    float* t;
    float* dist;
    float* point;
} rsi_outputs_t;

/* Cumulative per-handle counters (reporting; SURVEY 5 "stats struct"). */
typedef struct {
    uint64_t rays;           /* rays processed by rsi_intersect                         */
    uint64_t fp64_pairs;     /* (ray, triangle) pairs whose hit decision the fp32 error
                                filter could not certify, re-decided in fp64      */
    uint64_t fp64_rays;      /* rays whose nearest-hit / dedup / output value needed fp64 */
    uint64_t overflow_rays;  /* intercept_count rays that overflowed the register hit
                                list and went through the exact re-pass                  */
    uint64_t nonfinite_rays; /* rays with a NaN/Inf coordinate (reported as misses)       */
    uint64_t box_tests;      /* child-box slab tests (RSI_OPT_COUNTERS only, else 0)      */
    uint64_t mt_tests;       /* Moller-Trumbore tests (RSI_OPT_COUNTERS only, else 0)     */
    /* SIMT-efficiency diagnostics (RSI_OPT_COUNTERS only): summed over traversal
       iterations of every warp, the lanes searching / holding a pending leaf /
       idle (no ray or finished), the iteration count, and for leaf phases the
       lanes testing a leaf and the number of phases. */
    uint64_t it_search, it_pending, it_idle, iterations, leaf_lanes, leaf_phases;
} rsi_stats_t;

/* Library version string, e.g. "rsi-b200 0.1.0 sm_100a". */
const char* rsi_version(void);

/* Number of CUDA kernels this library has launched in this process, all
 * threads and devices (a monotonically increasing host-side counter, bumped
 * at every <<<>>> site; bench.py differences it around the timed region to
 * report gpu_launches).  Never fails. */
uint64_t rsi_launch_count(void);

/* Thread-local message for the most recent failing call on this thread. */
const char* rsi_last_error(void);

/*
 * rsi_build -- build the linear BVH over a triangle mesh (Fig. 1 P:17-24;
 * SURVEY 8(a) A1..A7): validate, surface extent, 30-bit Morton codes of
 * centroids, radix sort, Karras binary radix tree,
 * leaf init + atomic bottom-up AABB refit, packing.
 *   d_vertices  [n_vertices][3] float32, device.  Borrowed during the call only.
 *   d_triangles [n_triangles][3] int32, device.    Borrowed during the call only.
 *   options     may be NULL (defaults).
 *   out         receives the new handle (set to NULL on failure).
 * The handle keeps its own packed copy of the triangles, so the inputs may be
 * freed or overwritten once this call returns.  Validation (indices in range,
 * finite vertices) makes this call SYNCHRONOUS on `stream` at its end (one
 * 4-byte device->host status read).
 * Errors: RSI_E_INVALID_ARG, RSI_E_EMPTY, RSI_E_INDEX_RANGE, RSI_E_NONFINITE,
 *         RSI_E_OOM, RSI_E_CUDA.
 */
rsi_status_t rsi_build(const float* d_vertices, int64_t n_vertices,
                       const int32_t* d_triangles, int64_t n_triangles,
                       const rsi_options_t* options, void* stream, rsi_handle_t* out);

/*
 * rsi_rebuild -- rebuild `h` in place for a new mesh (same semantics as
 * rsi_build).  Device memory is reused when the new mesh fits; on failure the
 * handle is left empty (n_triangles 0) but valid for rsi_free / rsi_rebuild.
 */
rsi_status_t rsi_rebuild(rsi_handle_t h, const float* d_vertices, int64_t n_vertices,
                         const int32_t* d_triangles, int64_t n_triangles, void* stream);

/*
 * rsi_intersect -- test n_rays segments against the mesh of `h` (
 * SURVEY 8(a) A8..A9): per-ray short-stack BVH traversal + Moller-Trumbore.
 *   d_start, d_end  [n_rays][3] float32 segment end points, device.
 *   mode            an rsi_mode_t.
 *   out             device output pointers for `mode` (see rsi_outputs_t).
 * Results equal the exhaustive double-precision definition.
 * Asynchronous in every mode (returns once the work is enqueued; the host
 * never reads device state).  INTERCEPT_COUNT enqueues a second kernel, the
 * exact re-pass for rays whose hits overflow the traversal's register list;
 * it reads the overflow count on the device and has no capacity limit.
 * n_rays == 0 is a no-op.  Errors: RSI_E_INVALID_ARG, RSI_E_OOM, RSI_E_CUDA.
 */
rsi_status_t rsi_intersect(rsi_handle_t h, const float* d_start, const float* d_end,
                           int64_t n_rays, int32_t mode, const rsi_outputs_t* out,
                           void* stream);

/*
 * rsi_test -- the paper's end-to-end call `PyCudaRSI.test(vertices, triangles,
 * raysFrom, raysTo, cfg)` on HOST buffers: host->device copies,
 * rsi_build, rsi_intersect, device->host copies of the mode's outputs, and a
 * final synchronize of `stream`.  Host inputs should be pinned for full copy
 * bandwidth (pageable memory works but is slower).  h_out fields are HOST
 * pointers.  Rays stream through the GPU in 1 Mi-segment chunks so host->device
 * copies, traversal and device->host copies overlap.  The device workspace
 * (BVH, mesh and chunk buffers, events) is cached per calling thread and device
 * and reused by later calls; rsi_release_cache() frees it.
 * Errors: as rsi_build and rsi_intersect.
 */
rsi_status_t rsi_test(const float* h_vertices, int64_t n_vertices,
                      const int32_t* h_triangles, int64_t n_triangles,
                      const float* h_start, const float* h_end, int64_t n_rays,
                      int32_t mode, const rsi_options_t* options,
                      const rsi_outputs_t* h_out, void* stream);

/*
 * rsi_test_sparse -- the paper's barycentric return shape end to end (P:101:
 * `(intersecting_rays, distances, hit_triangles, hit_points) = rsi.test(...)`)
 * on HOST buffers: rays stream to the device in 1 Mi-segment chunks overlapped
 * with the build and the per-chunk traversal; step 3a (compaction of the hit
 * rays) and the gather of their values run on the device; only the hits
 * come back.  Outputs (HOST, capacity n_rays each; the first *h_n_hits entries
 * are written, in ascending ray order):
 *   h_ray_ids [n] int32 ray index; h_dist [n] float32 t*|end-start| (3b);
 *   h_tri [n] int32 original triangle index; h_point [n][3] float32 (3d).
 * h_dist, h_tri, h_point may be NULL.  Synchronizes `stream`.  Workspace cached
 * per thread and device (rsi_release_cache frees it).
 * Errors: as rsi_test; RSI_E_INVALID_ARG for n_rays > 2^31 - 1.
 */
rsi_status_t rsi_test_sparse(const float* h_vertices, int64_t n_vertices,
                             const int32_t* h_triangles, int64_t n_triangles,
                             const float* h_start, const float* h_end, int64_t n_rays,
                             const rsi_options_t* options, int32_t* h_ray_ids, float* h_dist,
                             int32_t* h_tri, float* h_point, int64_t* h_n_hits, void* stream);

/* Free the calling thread's cached rsi_test / rsi_test_sparse workspaces on every device. */
void rsi_release_cache(void);

/*
 * rsi_compact_hits -- step 3a "identify intersecting rays" on the
 * device: writes the ray indices i with d_tri[i] >= 0 in ASCENDING order to
 * d_ray_ids (capacity n_rays) and their number to *d_n_hits (device int32).
 * Together with the dense barycentric outputs this yields the paper's sparse
 * return (intersecting_rays, distances, hit_triangles, hit_points).
 * Asynchronous.  Errors: RSI_E_INVALID_ARG, RSI_E_OOM, RSI_E_CUDA.
 */
rsi_status_t rsi_compact_hits(const int32_t* d_tri, int64_t n_rays, int32_t* d_ray_ids,
                              int32_t* d_n_hits, void* stream);

/*
 * rsi_gather_hits -- the values of the compacted hit rays (the rest of the
 * paper's sparse barycentric return, after step 3a): for j < *d_n_hits,
 *   d_out_tri[j] = d_tri[d_ray_ids[j]], d_out_dist[j] = d_dist[d_ray_ids[j]],
 *   d_out_point[j][0..2] = d_point[d_ray_ids[j]][0..2]
 * (all DEVICE pointers; d_ray_ids / d_n_hits as written by rsi_compact_hits;
 * n_max = the capacity of the outputs, >= *d_n_hits; d_dist/d_out_dist and
 * d_point/d_out_point may be NULL together).  Asynchronous: the hit count is
 * read on the device, never by the host.
 * Errors: RSI_E_INVALID_ARG (null required pointer, n_max < 0), RSI_E_CUDA.
 */
rsi_status_t rsi_gather_hits(const int32_t* d_ray_ids, const int32_t* d_n_hits, int64_t n_max,
                             const int32_t* d_tri, const float* d_dist, const float* d_point,
                             int32_t* d_out_tri, float* d_out_dist, float* d_out_point, void* stream);

/* Release the handle and its device memory (stream-ordered on the build
 * stream, after the handle's last call on any stream). */
rsi_status_t rsi_free(rsi_handle_t h);

/*
 * rsi_validate -- GPU integrity check of the BVH of `h` (the
 * checks the paper performed by hand on decoded dumps).
 * Fills *report (host) and synchronizes `stream`.  Returns RSI_OK for a valid
 * tree, RSI_E_INTEGRITY when any count is non-zero or the root is unset.
 */
rsi_status_t rsi_validate(rsi_handle_t h, rsi_integrity_t* report, void* stream);

/* Result of the device-side input checks of the last rsi_build / rsi_rebuild
 * of `h` (the status rsi_build itself returns without RSI_OPT_DEFERRED_STATUS):
 * RSI_OK, RSI_E_INDEX_RANGE, RSI_E_NONFINITE or RSI_E_INVALID_ARG (extent).
 * Synchronizes `stream` when the result is still pending; an error leaves `h`
 * without a mesh (like a failed rsi_rebuild). */
rsi_status_t rsi_build_status(rsi_handle_t h, void* stream);

/* Read the cumulative counters of `h`; synchronizes `stream`. */
rsi_status_t rsi_get_stats(rsi_handle_t h, rsi_stats_t* out, void* stream);

/* Zero the counters of `h` (stream-ordered). */
rsi_status_t rsi_reset_stats(rsi_handle_t h, void* stream);

/*
 * Diagnostics (the paper's BVH debugging strategy: copy the tree
 * from device to host and decode it).
 * rsi_bvh_info: sizes and the scene AABB (root box) of `h` (host outputs);
 *   n_nodes = max(N_t - 1, 1) internal child-pair nodes.
 * rsi_bvh_download: copies the tree to HOST buffers (any may be NULL) and
 *   synchronizes `stream`:
 *     h_child   [n_nodes][2] int32  child refs: >= 0 internal node, < 0 leaf ~slot
 *     h_box     [n_nodes][2][6] float32 child AABBs (xlo, ylo, zlo, xhi, yhi, zhi)
 *     h_leaf_tri[N_t] int32  original triangle index stored at each leaf slot
 *     h_morton  [N_t] uint32 sorted 30-bit Morton codes (z-major interleave)
 *     h_parent  [n_nodes + N_t] int32 parent of internal nodes then of leaves,
 *               encoded (parent << 1) | side (side 0 = left); -1 for the root
 *               (node 0, or rsi_bvh_root's node under RSI_OPT_APETREI)
 *     h_arrivals[n_nodes] uint32 refit arrival counters ("atomic"); under
 *               RSI_OPT_APETREI the arrival counts of the agglomerative build
 */
rsi_status_t rsi_bvh_info(rsi_handle_t h, int64_t* n_triangles, int64_t* n_nodes,
                          float* scene_lo3, float* scene_hi3);
rsi_status_t rsi_bvh_download(rsi_handle_t h, int32_t* h_child, float* h_box,
                              int32_t* h_leaf_tri, uint32_t* h_morton, int32_t* h_parent,
                              uint32_t* h_arrivals, void* stream);

/*
 * rsi_bvh_upload: the inverse of rsi_bvh_download -- replaces the binary tree of
 *   `h` (built over the same mesh) by a caller-given one and rebuilds the 4-wide
 *   records from it (the paper's BVH debugging strategy, run the
 *   other way: a tree inspected or modified on the host -- or built by another
 *   method, e.g. a SAH builder, for tree-quality experiments -- is traversed by
 *   the same kernels).  Results of rsi_intersect do not depend on the tree (a
 *   BVH only prunes); a tree whose boxes do not contain their subtrees gives
 *   wrong results (the caller's responsibility; rsi_validate checks it).
 *     h_child   [n_nodes][2] int32 child refs (>= 0 internal node, < 0 leaf ~slot),
 *               every internal node and leaf slot reachable from `root` once
 *     h_box     [n_nodes][2][6] float32 child AABBs as in rsi_bvh_download
 *     h_leaf_tri[N_t] int32 triangle index at each leaf slot (a permutation)
 *     root      the root internal node
 *   Host buffers, read before return; synchronizes `stream`.  The parent links,
 *   arrival counts (2 per node) and scene box are set from the uploaded tree,
 *   so rsi_validate / rsi_bvh_download / rsi_bvh_info report it.  The next
 *   rsi_rebuild replaces the uploaded tree.
 * Errors: RSI_E_INVALID_ARG (null / N_t < 2 / root out of range / leaf_tri not
 *   a permutation / a child ref out of range or a node or leaf not reached exactly once
 *   from root), RSI_E_OOM, RSI_E_CUDA.
 */
rsi_status_t rsi_bvh_upload(rsi_handle_t h, const int32_t* h_child, const float* h_box,
                            const int32_t* h_leaf_tri, int64_t root, void* stream);

/*
 * rsi_bvh_root: the root internal node of `h` and the sorted Morton codes at
 * full width (host outputs; h_morton63 may be NULL; synchronizes `stream`).
 *   *root        0 for the default (Karras) numbering; under RSI_OPT_APETREI the
 *                split position of the top node (the fixture tree: 1),
 *                -1 if the construction never reached the root (fault injection).
 *   *sentinel    N_t - 1 under RSI_OPT_APETREI (the node that "only holds a
 *                pointer to the root"), else -1.
 *   h_morton63   [N_t] uint64 sorted codes: 63-bit under RSI_OPT_APETREI, else the
 *                30-bit codes widened.  (rsi_bvh_download's 30-bit h_morton is
 *                the top 30 bits of the 63-bit code: the same quantization.)
 * Errors: RSI_E_INVALID_ARG (null handle / root), RSI_E_CUDA.
 */
rsi_status_t rsi_bvh_root(rsi_handle_t h, int64_t* root, int64_t* sentinel, uint64_t* h_morton63,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RSI_H_ */
