// api.cu -- the extern "C" boundary declared in include/rsi.h.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <atomic>
#include <new>

#include "rsi_internal.cuh"

static thread_local char g_err[512] = "";

rsi_status_t rsi_set_error(rsi_status_t s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

rsi_status_t rsi_cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return RSI_OK;
    (void)cudaGetLastError();
    if (e == cudaErrorMemoryAllocation)
        return rsi_set_error(RSI_E_OOM, "%s: %s", what, cudaGetErrorString(e));
    return rsi_set_error(RSI_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static rsi_status_t read_options(const rsi_options_t* in, rsi_options_t* out) {
    out->struct_size = sizeof(rsi_options_t);
    out->flags = 0;
    out->dedup_tau = 1e-6;
    out->debug_refit_leaves = 0;
    if (!in || in->struct_size == 0) return RSI_OK;
    if (in->struct_size != sizeof(rsi_options_t))
        return rsi_set_error(RSI_E_INVALID_ARG, "rsi_options_t.struct_size %u != %zu", in->struct_size,
                             sizeof(rsi_options_t));
    if (in->flags & ~(RSI_OPT_FP64_MOLLER | RSI_OPT_COUNTERS | RSI_OPT_DEFERRED_STATUS | RSI_OPT_APETREI | RSI_OPT_ROTATE | RSI_OPT_PLAIN_TREE)) return rsi_set_error(RSI_E_INVALID_ARG, "unknown option flags 0x%x", in->flags);
    if (!(in->dedup_tau >= 0.0)) return rsi_set_error(RSI_E_INVALID_ARG, "dedup_tau must be >= 0");
    if (in->debug_refit_leaves < 0) return rsi_set_error(RSI_E_INVALID_ARG, "debug_refit_leaves must be >= 0");
    *out = *in;
    return RSI_OK;
}

static rsi_status_t check_mesh_args(const float* V, int64_t nv, const int32_t* T, int64_t nt) {
    if (nv < 0 || nt < 0) return rsi_set_error(RSI_E_INVALID_ARG, "negative mesh size");
    if (nv == 0 || nt == 0) return rsi_set_error(RSI_E_EMPTY, "empty mesh (n_vertices=%lld, n_triangles=%lld)",
                                                 (long long)nv, (long long)nt);
    if (!V || !T) return rsi_set_error(RSI_E_INVALID_ARG, "null vertices/triangles pointer");
    return RSI_OK;
}

// Two non-blocking copy streams per (thread, device) for rsi_test's pipeline,
// created once (stream creation is not free) and reused by later calls.
static rsi_status_t side_streams(cudaStream_t& sh, cudaStream_t& sd) {
    struct Pair { int dev = -1; cudaStream_t h = nullptr, d = nullptr; };
    static thread_local Pair cache[16];
    int dev = 0;
    rsi_status_t st = rsi_cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (st != RSI_OK) return st;
    Pair& p = cache[dev & 15];
    if (p.dev != dev) {
        st = rsi_cuda_check(cudaStreamCreateWithFlags(&p.h, cudaStreamNonBlocking), "stream");
        if (st == RSI_OK) st = rsi_cuda_check(cudaStreamCreateWithFlags(&p.d, cudaStreamNonBlocking), "stream");
        if (st != RSI_OK) return st;
        p.dev = dev;
    }
    sh = p.h;
    sd = p.d;
    return RSI_OK;
}

// Keep freed stream-ordered allocations cached in the device's default pool, so
// per-call cudaMallocAsync / cudaFreeAsync (rsi_test, overflow pass) do not
// return memory to the OS between calls.
void rsi_keep_pool_cached() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    (void)cudaGetLastError();
}

static std::atomic<uint64_t> g_launches{0};

void rsi_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Calls on one handle run in the order they were made even when the caller
// switches streams: a call on a stream other than the previous call's waits
// for the previous call's event first (device-side; the host never blocks).
static rsi_status_t order_enter(rsi_bvh* h, cudaStream_t s) {
    if (h->order_valid && h->last_stream != s)
        return rsi_cuda_check(cudaStreamWaitEvent(s, h->order_ev, 0), "stream order wait");
    return RSI_OK;
}
static rsi_status_t order_leave(rsi_bvh* h, cudaStream_t s) {
    if (!h->order_ev) {
        rsi_status_t st = rsi_cuda_check(cudaEventCreateWithFlags(&h->order_ev, cudaEventDisableTiming), "event");
        if (st != RSI_OK) return st;
    }
    rsi_status_t st = rsi_cuda_check(cudaEventRecord(h->order_ev, s), "stream order record");
    h->last_stream = s;
    h->order_valid = st == RSI_OK;
    return st;
}

extern "C" {

const char* rsi_version(void) { return RSI_VERSION_STRING; }

uint64_t rsi_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* rsi_last_error(void) { return g_err; }

rsi_status_t rsi_build(const float* d_vertices, int64_t n_vertices, const int32_t* d_triangles,
                       int64_t n_triangles, const rsi_options_t* options, void* stream, rsi_handle_t* out) {
    if (!out) return rsi_set_error(RSI_E_INVALID_ARG, "null output handle pointer");
    *out = nullptr;
    rsi_options_t opt;
    rsi_status_t st = read_options(options, &opt);
    if (st != RSI_OK) return st;
    st = check_mesh_args(d_vertices, n_vertices, d_triangles, n_triangles);
    if (st != RSI_OK) return st;
    rsi_bvh* h = new (std::nothrow) rsi_bvh();
    if (!h) return rsi_set_error(RSI_E_OOM, "host allocation failed");
    h->opt = opt;
    rsi_keep_pool_cached();
    if (const char* e = getenv("RSI_MIN_TRAV")) h->min_trav = atoi(e);  // tuning knobs
    cudaStream_t s = (cudaStream_t)stream;
    h->stream = s;
    st = rsi_cuda_check(cudaGetDevice(&h->device), "cudaGetDevice");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMallocAsync((void**)&h->scratch, SCR_WORDS * sizeof(uint32_t), s), "scratch");
    if (st == RSI_OK)
        st = rsi_cuda_check(cudaMallocAsync((void**)&h->stats, ST_WORDS * sizeof(unsigned long long), s), "stats");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemsetAsync(h->stats, 0, ST_WORDS * sizeof(unsigned long long), s), "stats");
    if (st == RSI_OK) st = rsi_build_device(h, d_vertices, n_vertices, d_triangles, n_triangles, s);
    if (st == RSI_OK) st = order_leave(h, s);
    if (st != RSI_OK) {
        char saved[512];
        memcpy(saved, g_err, sizeof(saved));
        rsi_free(h);
        memcpy(g_err, saved, sizeof(saved));
        return st;
    }
    *out = h;
    return RSI_OK;
}

rsi_status_t rsi_rebuild(rsi_handle_t h, const float* d_vertices, int64_t n_vertices, const int32_t* d_triangles,
                         int64_t n_triangles, void* stream) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != h->device)  // the handle's buffers live on its own device
        return rsi_set_error(RSI_E_INVALID_ARG, "handle built on device %d, current device is %d", h->device, dev);
    h->n_tri = 0;
    h->n_nodes = 0;
    rsi_status_t st = check_mesh_args(d_vertices, n_vertices, d_triangles, n_triangles);
    if (st != RSI_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    st = order_enter(h, s);
    if (st == RSI_OK) st = rsi_build_device(h, d_vertices, n_vertices, d_triangles, n_triangles, s);
    const rsi_status_t st2 = order_leave(h, s);
    return st != RSI_OK ? st : st2;
}

rsi_status_t rsi_intersect(rsi_handle_t h, const float* d_start, const float* d_end, int64_t n_rays, int32_t mode,
                           const rsi_outputs_t* out, void* stream) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    if (h->n_tri <= 0) return rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh (a failed rebuild?)");
    if (n_rays < 0) return rsi_set_error(RSI_E_INVALID_ARG, "negative n_rays");
    if (!out) return rsi_set_error(RSI_E_INVALID_ARG, "null outputs");
    if (mode != RSI_MODE_BOOLEAN && mode != RSI_MODE_BARYCENTRIC && mode != RSI_MODE_INTERCEPT_COUNT)
        return rsi_set_error(RSI_E_INVALID_ARG, "bad mode %d", mode);
    if (n_rays == 0) return RSI_OK;
    if (!d_start || !d_end) return rsi_set_error(RSI_E_INVALID_ARG, "null ray pointer");
    if (mode == RSI_MODE_BOOLEAN && !out->hit) return rsi_set_error(RSI_E_INVALID_ARG, "boolean mode needs out->hit");
    if (mode == RSI_MODE_BARYCENTRIC && !out->tri)
        return rsi_set_error(RSI_E_INVALID_ARG, "barycentric mode needs out->tri");
    if (mode == RSI_MODE_INTERCEPT_COUNT && !out->count)
        return rsi_set_error(RSI_E_INVALID_ARG, "intercept_count mode needs out->count");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != h->device)
        return rsi_set_error(RSI_E_INVALID_ARG, "handle built on device %d, current device is %d", h->device, dev);
    cudaStream_t s = (cudaStream_t)stream;
    rsi_status_t st = order_enter(h, s);
    if (st == RSI_OK) st = rsi_intersect_device(h, d_start, d_end, n_rays, mode, out, s);
    if (st == RSI_OK) h->host_rays += (uint64_t)n_rays;
    const rsi_status_t st2 = order_leave(h, s);
    return st != RSI_OK ? st : st2;
}

rsi_status_t rsi_compact_hits(const int32_t* d_tri, int64_t n_rays, int32_t* d_ray_ids, int32_t* d_n_hits,
                              void* stream) {
    if (n_rays < 0 || (n_rays > 0 && (!d_tri || !d_ray_ids)) || !d_n_hits)
        return rsi_set_error(RSI_E_INVALID_ARG, "bad compaction arguments");
    if (n_rays > ((int64_t)1 << 31) - 1) return rsi_set_error(RSI_E_INVALID_ARG, "n_rays exceeds 2^31-1");
    return rsi_compact_device(d_tri, n_rays, d_ray_ids, d_n_hits, (cudaStream_t)stream);
}

rsi_status_t rsi_gather_hits(const int32_t* d_ray_ids, const int32_t* d_n_hits, int64_t n_max, const int32_t* d_tri,
                             const float* d_dist, const float* d_point, int32_t* d_out_tri, float* d_out_dist,
                             float* d_out_point, void* stream) {
    if (n_max < 0 || (n_max > 0 && (!d_ray_ids || !d_n_hits || !d_tri || !d_out_tri)) ||
        (!d_dist) != (!d_out_dist) || (!d_point) != (!d_out_point))
        return rsi_set_error(RSI_E_INVALID_ARG, "bad gather arguments");
    if (n_max > ((int64_t)1 << 31) - 1) return rsi_set_error(RSI_E_INVALID_ARG, "n_max exceeds 2^31-1");
    return rsi_gather_hits_device(d_ray_ids, d_n_hits, n_max, d_tri, d_dist, d_point, d_out_tri, d_out_dist,
                                  d_out_point, (cudaStream_t)stream);
}

// Per-(thread, device) workspace of rsi_test, reused across calls: the BVH
// handle (rebuilt in place), the mesh and ray-chunk device buffers and the
// pipeline events.  Released by rsi_release_cache() or at thread exit.
struct TestCtx {
    int dev = -1;
    rsi_handle_t h = nullptr;
    char* buf = nullptr;
    size_t buf_bytes = 0;
    cudaEvent_t* ev = nullptr;
    int64_t n_ev = 0;
    cudaStream_t alloc_stream = nullptr;
    void release() {
        if (h) rsi_free(h);
        h = nullptr;
        if (buf) cudaFree(buf);
        buf = nullptr;
        buf_bytes = 0;
        for (int64_t k = 0; k < n_ev; ++k) cudaEventDestroy(ev[k]);
        delete[] ev;
        ev = nullptr;
        n_ev = 0;
        dev = -1;
    }
    ~TestCtx() { release(); }
};
static thread_local TestCtx g_test_ctx[16];

rsi_status_t rsi_test(const float* h_vertices, int64_t n_vertices, const int32_t* h_triangles, int64_t n_triangles,
                      const float* h_start, const float* h_end, int64_t n_rays, int32_t mode,
                      const rsi_options_t* options, const rsi_outputs_t* h_out, void* stream) {
    if (!h_out || n_rays < 0 || (n_rays > 0 && (!h_start || !h_end)))
        return rsi_set_error(RSI_E_INVALID_ARG, "bad rsi_test arguments");
    if (mode != RSI_MODE_BOOLEAN && mode != RSI_MODE_BARYCENTRIC && mode != RSI_MODE_INTERCEPT_COUNT)
        return rsi_set_error(RSI_E_INVALID_ARG, "bad mode %d", mode);
    rsi_status_t st = check_mesh_args(h_vertices, n_vertices, h_triangles, n_triangles);
    if (st != RSI_OK) return st;
    rsi_options_t opt;
    st = read_options(options, &opt);
    if (st != RSI_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    st = rsi_cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (st != RSI_OK) return st;
    TestCtx& ctx = g_test_ctx[dev & 15];
    if (ctx.dev != dev) {
        ctx.release();
        ctx.dev = dev;
    }
    rsi_keep_pool_cached();

    // workspace: [mesh V][mesh T][2 ray slots: start, end, outputs]
    // chunk schedule: kChunkRays-segment chunks; with RSI_TEST_TAIL > 0 they
    // halve down to kTailRays at the end (a shorter un-overlapped tail;
    // measured neutral, so off by default)
    int64_t kChunkRays = (int64_t)1 << 20, kTailRays = 0;
    if (const char* e = getenv("RSI_TEST_CHUNK")) kChunkRays = atoll(e) > 0 ? atoll(e) : kChunkRays;  // tuning
    if (const char* e = getenv("RSI_TEST_TAIL")) kTailRays = atoll(e) >= 0 ? atoll(e) : kTailRays;    // tuning
    int64_t n_sched = 0;
    auto chunk_len = [&](int64_t rem) {
        if (kTailRays <= 0 || rem <= kTailRays) return rem < kChunkRays ? rem : kChunkRays;
        int64_t h = rem / 2;
        h = h > kTailRays ? h : kTailRays;
        return h < kChunkRays ? h : kChunkRays;
    };
    for (int64_t r = 0; r < n_rays; r += chunk_len(n_rays - r)) ++n_sched;
    const int64_t nchunk = n_sched;
    const int64_t crays = n_rays < kChunkRays ? n_rays : kChunkRays;
    // chunk c covers [c0(c), c0(c + 1)): recomputed by walking the schedule
    // (nchunk is tens at most)
    auto c0 = [&](int64_t c) {
        int64_t r = 0;
        for (int64_t k = 0; k < c && r < n_rays; ++k) r += chunk_len(n_rays - r);
        return r < n_rays ? r : n_rays;
    };
    const size_t out_b = mode == RSI_MODE_BOOLEAN ? 1 : (mode == RSI_MODE_INTERCEPT_COUNT ? 4 : 24);
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t bv = (size_t)n_vertices * 3 * sizeof(float), bt = (size_t)n_triangles * 3 * sizeof(int32_t);
    const size_t slot_b = 2 * up((size_t)crays * 12) + up((size_t)crays * out_b);
    const size_t need = up(bv) + up(bt) + 2 * slot_b;
    if (ctx.buf_bytes < need) {
        if (ctx.buf) {
            cudaStreamSynchronize(s);
            cudaFree(ctx.buf);
            ctx.buf = nullptr;
            ctx.buf_bytes = 0;
        }
        st = rsi_cuda_check(cudaMalloc((void**)&ctx.buf, need), "rsi_test workspace");
        if (st != RSI_OK) return st;
        ctx.buf_bytes = need;
    }
    if (ctx.n_ev < 3 * nchunk) {
        for (int64_t k = 0; k < ctx.n_ev; ++k) cudaEventDestroy(ctx.ev[k]);
        delete[] ctx.ev;
        ctx.n_ev = 0;
        ctx.ev = new (std::nothrow) cudaEvent_t[3 * nchunk]();
        if (!ctx.ev) return rsi_set_error(RSI_E_OOM, "host allocation failed");
        for (int64_t k = 0; k < 3 * nchunk; ++k) {
            st = rsi_cuda_check(cudaEventCreateWithFlags(&ctx.ev[k], cudaEventDisableTiming), "event");
            if (st != RSI_OK) return st;
            ctx.n_ev = k + 1;
        }
    }
    cudaEvent_t* ev = ctx.ev;  // per chunk: h2d done, kernel done, d2h done
    float* dV = (float*)ctx.buf;
    int32_t* dT = (int32_t*)(ctx.buf + up(bv));
    char* slots = ctx.buf + up(bv) + up(bt);
    cudaStream_t sh = nullptr, sd = nullptr;
    if (nchunk > 0) {
        st = side_streams(sh, sd);
        if (st != RSI_OK) return st;
        // side streams start after everything previously enqueued on `s`
        // (the workspace's last users)
        st = rsi_cuda_check(cudaEventRecord(ev[0], s), "event");
        if (st == RSI_OK) st = rsi_cuda_check(cudaStreamWaitEvent(sh, ev[0], 0), "wait");
        if (st == RSI_OK) st = rsi_cuda_check(cudaStreamWaitEvent(sd, ev[0], 0), "wait");
        if (st != RSI_OK) return st;
    }
    auto slot = [&](int64_t c) { return slots + (c & 1) * slot_b; };
    auto h2d = [&](int64_t c) {
        const int64_t r0 = c0(c), nr = c0(c + 1) - r0;
        char* b = slot(c);
        if (c >= 2) st = rsi_cuda_check(cudaStreamWaitEvent(sh, ev[3 * (c - 2) + 1], 0), "wait");
        if (st == RSI_OK)
            st = rsi_cuda_check(cudaMemcpyAsync(b, h_start + 3 * r0, (size_t)nr * 12, cudaMemcpyHostToDevice, sh),
                                "H2D start");
        if (st == RSI_OK)
            st = rsi_cuda_check(cudaMemcpyAsync(b + up((size_t)crays * 12), h_end + 3 * r0, (size_t)nr * 12,
                                                cudaMemcpyHostToDevice, sh), "H2D end");
        if (st == RSI_OK) st = rsi_cuda_check(cudaEventRecord(ev[3 * c], sh), "event");
    };

    // 1. mesh upload first (so it is not queued behind ray chunks on the copy
    //    engine), then the first two ray chunks on `sh`, then the build on `s`
    //    (synchronizes once for validation) while those chunks copy
    st = rsi_cuda_check(cudaMemcpyAsync(dV, h_vertices, bv, cudaMemcpyHostToDevice, s), "H2D vertices");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(dT, h_triangles, bt, cudaMemcpyHostToDevice, s), "H2D triangles");
    int64_t issued = 0;
    while (st == RSI_OK && issued < nchunk && issued < 2) h2d(issued++);
    if (st == RSI_OK) {
        if (ctx.h) {
            ctx.h->opt = opt;
            st = rsi_rebuild(ctx.h, dV, n_vertices, dT, n_triangles, stream);
        } else {
            st = rsi_build(dV, n_vertices, dT, n_triangles, &opt, stream, &ctx.h);
        }
    }

    // 2. chunk loop: H2D(c+1) and D2H(c-1) overlap the traversal of chunk c
    for (int64_t c = 0; st == RSI_OK && c < nchunk; ++c) {
        while (st == RSI_OK && issued < nchunk && issued <= c + 1) h2d(issued++);
        if (st != RSI_OK) break;
        const int64_t r0 = c0(c), nr = c0(c + 1) - r0;
        char* b = slot(c);
        char* o = b + 2 * up((size_t)crays * 12);
        st = rsi_cuda_check(cudaStreamWaitEvent(s, ev[3 * c], 0), "wait");
        if (st == RSI_OK && c >= 2) st = rsi_cuda_check(cudaStreamWaitEvent(s, ev[3 * (c - 2) + 2], 0), "wait");
        rsi_outputs_t d_out{};
        if (mode == RSI_MODE_BOOLEAN) d_out.hit = (uint8_t*)o;
        if (mode == RSI_MODE_INTERCEPT_COUNT) d_out.count = (int32_t*)o;
        if (mode == RSI_MODE_BARYCENTRIC) {
            d_out.tri = (int32_t*)o;
            d_out.t = h_out->t ? (float*)(o + 4 * (size_t)crays) : nullptr;
            d_out.dist = h_out->dist ? (float*)(o + 8 * (size_t)crays) : nullptr;
            d_out.point = h_out->point ? (float*)(o + 12 * (size_t)crays) : nullptr;
        }
        if (st == RSI_OK)
            st = rsi_intersect(ctx.h, (const float*)b, (const float*)(b + up((size_t)crays * 12)), nr, mode, &d_out,
                               stream);
        if (st == RSI_OK) st = rsi_cuda_check(cudaEventRecord(ev[3 * c + 1], s), "event");
        if (st == RSI_OK) st = rsi_cuda_check(cudaStreamWaitEvent(sd, ev[3 * c + 1], 0), "wait");
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
            if (dst && st == RSI_OK)
                st = rsi_cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, sd), "D2H");
        };
        if (mode == RSI_MODE_BOOLEAN) d2h(h_out->hit ? h_out->hit + r0 : nullptr, d_out.hit, (size_t)nr);
        if (mode == RSI_MODE_INTERCEPT_COUNT) d2h(h_out->count ? h_out->count + r0 : nullptr, d_out.count, 4 * (size_t)nr);
        if (mode == RSI_MODE_BARYCENTRIC) {
            d2h(h_out->tri ? h_out->tri + r0 : nullptr, d_out.tri, 4 * (size_t)nr);
            d2h(h_out->t ? h_out->t + r0 : nullptr, d_out.t, 4 * (size_t)nr);
            d2h(h_out->dist ? h_out->dist + r0 : nullptr, d_out.dist, 4 * (size_t)nr);
            d2h(h_out->point ? h_out->point + 3 * r0 : nullptr, d_out.point, 12 * (size_t)nr);
        }
        if (st == RSI_OK) st = rsi_cuda_check(cudaEventRecord(ev[3 * c + 2], sd), "event");
    }

    // 3. join the side streams into `s` (also on error paths) and synchronize
    for (cudaStream_t side : {sh, sd}) {
        if (!side) continue;
        cudaEvent_t fin;
        if (cudaEventCreateWithFlags(&fin, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(fin, side);
            cudaStreamWaitEvent(s, fin, 0);
            cudaEventDestroy(fin);
        }
    }
    rsi_status_t st2 = rsi_cuda_check(cudaStreamSynchronize(s), "rsi_test");
    if (st != RSI_OK) {  // a failed build leaves the cached handle empty; start fresh next time
        char saved[512];
        memcpy(saved, g_err, sizeof(saved));
        ctx.release();
        memcpy(g_err, saved, sizeof(saved));
    }
    return st != RSI_OK ? st : st2;
}

// Per-(thread, device) workspace of rsi_test_sparse (its own handle, so the
// two entry points do not rebuild each other's cached BVH).
static thread_local TestCtx g_sparse_ctx[16];

rsi_status_t rsi_test_sparse(const float* h_vertices, int64_t n_vertices, const int32_t* h_triangles,
                             int64_t n_triangles, const float* h_start, const float* h_end, int64_t n_rays,
                             const rsi_options_t* options, int32_t* h_ray_ids, float* h_dist, int32_t* h_tri,
                             float* h_point, int64_t* h_n_hits, void* stream) {
    if (!h_n_hits || !h_ray_ids || n_rays < 0 || (n_rays > 0 && (!h_start || !h_end)))
        return rsi_set_error(RSI_E_INVALID_ARG, "bad rsi_test_sparse arguments");
    if (n_rays > ((int64_t)1 << 31) - 1) return rsi_set_error(RSI_E_INVALID_ARG, "n_rays exceeds 2^31-1");
    rsi_status_t st = check_mesh_args(h_vertices, n_vertices, h_triangles, n_triangles);
    if (st != RSI_OK) return st;
    rsi_options_t opt;
    st = read_options(options, &opt);
    if (st != RSI_OK) return st;
    *h_n_hits = 0;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    st = rsi_cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (st != RSI_OK) return st;
    TestCtx& ctx = g_sparse_ctx[dev & 15];
    if (ctx.dev != dev) {
        ctx.release();
        ctx.dev = dev;
    }
    rsi_keep_pool_cached();
    // workspace: mesh | start | end | dense tri, dist, point | ids, n_hits | sparse tri, dist, point
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t n = (size_t)n_rays;
    const size_t bv = up((size_t)n_vertices * 12), bt = up((size_t)n_triangles * 12);
    const size_t b12 = up(n * 12), b4 = up(n * 4);
    const size_t need = bv + bt + 2 * b12 + (2 * b4 + b12) + (b4 + 256) + (2 * b4 + b12);
    if (ctx.buf_bytes < need) {
        if (ctx.buf) {
            cudaStreamSynchronize(s);
            cudaFree(ctx.buf);
            ctx.buf = nullptr;
            ctx.buf_bytes = 0;
        }
        st = rsi_cuda_check(cudaMalloc((void**)&ctx.buf, need), "rsi_test_sparse workspace");
        if (st != RSI_OK) return st;
        ctx.buf_bytes = need;
    }
    char* q = ctx.buf;
    float* dV = (float*)q; q += bv;
    int32_t* dT = (int32_t*)q; q += bt;
    float* dS = (float*)q; q += b12;
    float* dE = (float*)q; q += b12;
    int32_t* tri = (int32_t*)q; q += b4;
    float* dist = (float*)q; q += b4;
    float* point = (float*)q; q += b12;
    int32_t* ids = (int32_t*)q; q += b4;
    int32_t* d_n = (int32_t*)q; q += 256;
    int32_t* stri = (int32_t*)q; q += b4;
    float* sdist = (float*)q; q += b4;
    float* spoint = (float*)q;
    // rays stream in 1 Mi-segment chunks on a copy stream; each chunk's
    // traversal starts as soon as its copy lands (and the BVH is built)
    const int64_t kChunkRays = (int64_t)1 << 20;
    const int64_t nchunk = (n_rays + kChunkRays - 1) / kChunkRays;
    if (ctx.n_ev < nchunk + 1) {
        for (int64_t k = 0; k < ctx.n_ev; ++k) cudaEventDestroy(ctx.ev[k]);
        delete[] ctx.ev;
        ctx.n_ev = 0;
        ctx.ev = new (std::nothrow) cudaEvent_t[nchunk + 1]();
        if (!ctx.ev) return rsi_set_error(RSI_E_OOM, "host allocation failed");
        for (int64_t k = 0; k < nchunk + 1; ++k) {
            st = rsi_cuda_check(cudaEventCreateWithFlags(&ctx.ev[k], cudaEventDisableTiming), "event");
            if (st != RSI_OK) return st;
            ctx.n_ev = k + 1;
        }
    }
    cudaStream_t sh = nullptr, sd = nullptr;
    st = side_streams(sh, sd);
    if (st == RSI_OK) st = rsi_cuda_check(cudaEventRecord(ctx.ev[nchunk], s), "event");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamWaitEvent(sh, ctx.ev[nchunk], 0), "wait");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(dV, h_vertices, (size_t)n_vertices * 12, cudaMemcpyHostToDevice, s), "H2D vertices");
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(dT, h_triangles, (size_t)n_triangles * 12, cudaMemcpyHostToDevice, s), "H2D triangles");
    for (int64_t c = 0; st == RSI_OK && c < nchunk; ++c) {
        const int64_t r0 = c * kChunkRays, nr = (n_rays - r0) < kChunkRays ? (n_rays - r0) : kChunkRays;
        st = rsi_cuda_check(cudaMemcpyAsync(dS + 3 * r0, h_start + 3 * r0, (size_t)nr * 12, cudaMemcpyHostToDevice, sh), "H2D start");
        if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(dE + 3 * r0, h_end + 3 * r0, (size_t)nr * 12, cudaMemcpyHostToDevice, sh), "H2D end");
        if (st == RSI_OK) st = rsi_cuda_check(cudaEventRecord(ctx.ev[c], sh), "event");
    }
    if (st == RSI_OK) {
        if (ctx.h) {
            ctx.h->opt = opt;
            st = rsi_rebuild(ctx.h, dV, n_vertices, dT, n_triangles, stream);
        } else {
            st = rsi_build(dV, n_vertices, dT, n_triangles, &opt, stream, &ctx.h);
        }
    }
    for (int64_t c = 0; st == RSI_OK && c < nchunk; ++c) {
        const int64_t r0 = c * kChunkRays, nr = (n_rays - r0) < kChunkRays ? (n_rays - r0) : kChunkRays;
        st = rsi_cuda_check(cudaStreamWaitEvent(s, ctx.ev[c], 0), "wait");
        rsi_outputs_t o{};
        o.tri = tri + r0;
        o.dist = dist + r0;
        o.point = point + 3 * r0;
        if (st == RSI_OK) st = rsi_intersect(ctx.h, dS + 3 * r0, dE + 3 * r0, nr, RSI_MODE_BARYCENTRIC, &o, stream);
    }
    // 3a on the device, then the values of the hit rays only
    if (st == RSI_OK) st = rsi_compact_device(tri, n_rays, ids, d_n, s);
    if (st == RSI_OK) st = rsi_gather_hits_device(ids, d_n, n_rays, tri, dist, point, stri, sdist, spoint, s);
    int32_t nh = 0;
    if (st == RSI_OK) st = rsi_cuda_check(cudaMemcpyAsync(&nh, d_n, 4, cudaMemcpyDeviceToHost, s), "D2H hit count");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "rsi_test_sparse");
    if (st == RSI_OK && nh > 0) {
        st = rsi_cuda_check(cudaMemcpyAsync(h_ray_ids, ids, (size_t)nh * 4, cudaMemcpyDeviceToHost, s), "D2H ids");
        if (st == RSI_OK && h_tri) st = rsi_cuda_check(cudaMemcpyAsync(h_tri, stri, (size_t)nh * 4, cudaMemcpyDeviceToHost, s), "D2H tri");
        if (st == RSI_OK && h_dist) st = rsi_cuda_check(cudaMemcpyAsync(h_dist, sdist, (size_t)nh * 4, cudaMemcpyDeviceToHost, s), "D2H dist");
        if (st == RSI_OK && h_point) st = rsi_cuda_check(cudaMemcpyAsync(h_point, spoint, (size_t)nh * 12, cudaMemcpyDeviceToHost, s), "D2H point");
    }
    // join the copy stream (also on error paths) and synchronize
    cudaEvent_t fin;
    if (sh && cudaEventCreateWithFlags(&fin, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(fin, sh);
        cudaStreamWaitEvent(s, fin, 0);
        cudaEventDestroy(fin);
    }
    const rsi_status_t st2 = rsi_cuda_check(cudaStreamSynchronize(s), "rsi_test_sparse");
    if (st != RSI_OK) {
        char saved[512];
        memcpy(saved, g_err, sizeof(saved));
        ctx.release();
        memcpy(g_err, saved, sizeof(saved));
        return st;
    }
    if (st2 == RSI_OK) *h_n_hits = nh;
    return st2;
}

void rsi_release_cache(void) {
    int dev = 0;
    cudaGetDevice(&dev);
    for (auto& c : g_test_ctx) c.release();
    for (auto& c : g_sparse_ctx) c.release();
    cudaSetDevice(dev);
}

rsi_status_t rsi_free(rsi_handle_t h) {
    if (!h) return RSI_OK;
    cudaStream_t s = h->stream;
    order_enter(h, s);  // the frees follow the handle's last use on any stream
    void* bufs[] = {h->nodes, h->top, h->quads, h->tris, h->keys, h->vals, h->keys_tmp, h->vals_tmp, h->parent,
                    h->arrivals, h->hist, h->scratch, h->stats, h->ovf_list, h->k63, h->other, h->qfull, h->qorder, h->qmap};
    rsi_status_t st = RSI_OK;
    for (void* p : bufs)
        if (p) {
            rsi_status_t e = rsi_cuda_check(cudaFreeAsync(p, s), "cudaFreeAsync");
            if (st == RSI_OK) st = e;
        }
    if (h->order_ev) cudaEventDestroy(h->order_ev);
    delete h;
    return st;
}

rsi_status_t rsi_validate(rsi_handle_t h, rsi_integrity_t* report, void* stream) {
    if (!h || !report) return rsi_set_error(RSI_E_INVALID_ARG, "null argument");
    if (h->status_pending) {
        const rsi_status_t st0 = rsi_finish_build(h, (cudaStream_t)stream);
        if (st0 != RSI_OK) return st0;
    }
    if (h->n_tri <= 0) return rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh");
    rsi_status_t st = rsi_validate_device(h, report, (cudaStream_t)stream);
    if (st != RSI_OK) return st;
    if (report->half_filled || report->untouched || report->bad_leaf_ids || report->bad_links || report->bad_boxes ||
        report->unreachable_leaves || !report->root_ok)
        return rsi_set_error(RSI_E_INTEGRITY,
                             "BVH integrity: half_filled=%lld untouched=%lld bad_leaf_ids=%lld bad_links=%lld "
                             "bad_boxes=%lld unreachable_leaves=%lld root_ok=%d",
                             (long long)report->half_filled, (long long)report->untouched,
                             (long long)report->bad_leaf_ids, (long long)report->bad_links,
                             (long long)report->bad_boxes, (long long)report->unreachable_leaves, report->root_ok);
    return RSI_OK;
}

rsi_status_t rsi_get_stats(rsi_handle_t h, rsi_stats_t* out, void* stream) {
    if (!h || !out) return rsi_set_error(RSI_E_INVALID_ARG, "null argument");
    unsigned long long v[ST_WORDS] = {0};
    cudaStream_t s = (cudaStream_t)stream;
    rsi_status_t st = rsi_cuda_check(cudaMemcpyAsync(v, h->stats, sizeof(v), cudaMemcpyDeviceToHost, s), "stats");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "stats");
    if (st != RSI_OK) return st;
    out->rays = h->host_rays;
    out->fp64_pairs = v[ST_FP64_PAIRS];
    out->fp64_rays = v[ST_FP64_RAYS];
    out->overflow_rays = v[ST_OVERFLOW];
    out->nonfinite_rays = v[ST_NONFINITE];
    out->box_tests = v[ST_BOX_TESTS];
    out->mt_tests = v[ST_MT_TESTS];
    out->it_search = v[ST_IT_SEARCH];
    out->it_pending = v[ST_IT_PEND];
    out->it_idle = v[ST_IT_IDLE];
    out->iterations = v[ST_ITERS];
    out->leaf_lanes = v[ST_LEAF_LANES];
    out->leaf_phases = v[ST_LEAF_PHASES];
    return RSI_OK;
}

rsi_status_t rsi_reset_stats(rsi_handle_t h, void* stream) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    h->host_rays = 0;
    return rsi_cuda_check(cudaMemsetAsync(h->stats, 0, ST_WORDS * sizeof(unsigned long long), (cudaStream_t)stream),
                          "reset stats");
}

rsi_status_t rsi_build_status(rsi_handle_t h, void* stream) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    return rsi_finish_build(h, (cudaStream_t)stream);
}

rsi_status_t rsi_bvh_info(rsi_handle_t h, int64_t* n_triangles, int64_t* n_nodes, float* lo3, float* hi3) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    if (h->status_pending) {  // deferred build: the scene box is read back now
        const rsi_status_t st = rsi_finish_build(h, h->stream);
        if (st != RSI_OK) return st;
    }
    if (n_triangles) *n_triangles = h->n_tri;
    if (n_nodes) *n_nodes = h->n_nodes;
    for (int k = 0; k < 3; ++k) {
        if (lo3) lo3[k] = h->scene_lo[k];
        if (hi3) hi3[k] = h->scene_hi[k];
    }
    return RSI_OK;
}

rsi_status_t rsi_bvh_upload(rsi_handle_t h, const int32_t* h_child, const float* h_box, const int32_t* h_leaf_tri,
                            int64_t root, void* stream) {
    if (!h || !h_child || !h_box || !h_leaf_tri) return rsi_set_error(RSI_E_INVALID_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    if (h->status_pending) {
        const rsi_status_t st0 = rsi_finish_build(h, s);
        if (st0 != RSI_OK) return st0;
    }
    if (h->n_tri <= 0) return rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != h->device)
        return rsi_set_error(RSI_E_INVALID_ARG, "handle built on device %d, current device is %d", h->device, dev);
    return rsi_bvh_upload_device(h, h_child, h_box, h_leaf_tri, root, s);
}

rsi_status_t rsi_bvh_download(rsi_handle_t h, int32_t* h_child, float* h_box, int32_t* h_leaf_tri,
                              uint32_t* h_morton, int32_t* h_parent, uint32_t* h_arrivals, void* stream) {
    if (!h) return rsi_set_error(RSI_E_INVALID_ARG, "null handle");
    cudaStream_t s = (cudaStream_t)stream;
    if (h->status_pending) {
        const rsi_status_t st0 = rsi_finish_build(h, s);
        if (st0 != RSI_OK) return st0;
    }
    if (h->n_tri <= 0) return rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh");
    const int64_t nn = h->n_nodes, nt = h->n_tri;
    rsi_status_t st = RSI_OK;
    float4* nodes = nullptr;
    if (h_child || h_box) {
        nodes = new (std::nothrow) float4[4 * nn];
        if (!nodes) return rsi_set_error(RSI_E_OOM, "host allocation failed");
        st = rsi_cuda_check(cudaMemcpyAsync(nodes, h->nodes, nn * 4 * sizeof(float4), cudaMemcpyDeviceToHost, s), "nodes");
    }
    float4* tris = nullptr;
    if (st == RSI_OK && h_leaf_tri) {
        tris = new (std::nothrow) float4[kTriF4 * nt];
        if (!tris) st = rsi_set_error(RSI_E_OOM, "host allocation failed");
        else st = rsi_cuda_check(cudaMemcpyAsync(tris, h->tris, nt * kTriF4 * sizeof(float4), cudaMemcpyDeviceToHost, s), "tris");
    }
    // Apetrei builds: codes are 63-bit (the top 30 bits are the 30-bit code) and
    // arrival counts live in the high words of the 64-bit node words
    uint32_t* khi = nullptr;  // [2 * nt]: sorted high words, then sorted low words
    unsigned long long* other = nullptr;
    if (st == RSI_OK && h_morton) {
        if (h->apetrei) {
            khi = new (std::nothrow) uint32_t[2 * nt];
            if (!khi) st = rsi_set_error(RSI_E_OOM, "host allocation failed");
            else st = rsi_cuda_check(cudaMemcpyAsync(khi, h->keys, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s), "keys");
            if (st == RSI_OK)
                st = rsi_cuda_check(cudaMemcpyAsync(khi + nt, h->k63 + 3 * nt, nt * sizeof(uint32_t),
                                                    cudaMemcpyDeviceToHost, s), "keys");
        } else {
            st = rsi_cuda_check(cudaMemcpyAsync(h_morton, h->keys, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s), "keys");
        }
    }
    if (st == RSI_OK && h_parent)
        st = rsi_cuda_check(cudaMemcpyAsync(h_parent, h->parent, (nn + nt) * sizeof(int32_t), cudaMemcpyDeviceToHost, s),
                            "parent");
    if (st == RSI_OK && h_arrivals) {
        if (h->apetrei) {
            other = new (std::nothrow) unsigned long long[nn];
            if (!other) st = rsi_set_error(RSI_E_OOM, "host allocation failed");
            else st = rsi_cuda_check(cudaMemcpyAsync(other, h->other, nn * sizeof(unsigned long long),
                                                     cudaMemcpyDeviceToHost, s), "arrivals");
        } else {
            st = rsi_cuda_check(cudaMemcpyAsync(h_arrivals, h->arrivals, nn * sizeof(uint32_t), cudaMemcpyDeviceToHost, s),
                                "arrivals");
        }
    }
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "download");
    if (st == RSI_OK && khi)
        for (int64_t k = 0; k < nt; ++k)
            h_morton[k] = (uint32_t)((((unsigned long long)khi[k] << 32) | khi[nt + k]) >> 33);
    if (st == RSI_OK && other)
        for (int64_t i = 0; i < nn; ++i) h_arrivals[i] = (uint32_t)(other[i] >> 32);
    delete[] khi;
    delete[] other;
    if (st == RSI_OK) {
        for (int64_t i = 0; i < nn; ++i) {
            const float* f = reinterpret_cast<const float*>(nodes ? nodes + 4 * i : nullptr);
            if (h_child) {
                int32_t refs[2];
                memcpy(refs, f + 12, 8);
                h_child[2 * i] = refs[0];
                h_child[2 * i + 1] = refs[1];
            }
            if (h_box) {
                float* b = h_box + 12 * i;
                // left: xlo ylo zlo xhi yhi zhi
                b[0] = f[0]; b[1] = f[2]; b[2] = f[8]; b[3] = f[1]; b[4] = f[3]; b[5] = f[9];
                b[6] = f[4]; b[7] = f[6]; b[8] = f[10]; b[9] = f[5]; b[10] = f[7]; b[11] = f[11];
            }
        }
        if (h_leaf_tri)
            for (int64_t k = 0; k < nt; ++k) {
                int32_t id;
                memcpy(&id, &tris[kTriF4 * k].w, 4);
                h_leaf_tri[k] = id;
            }
    }
    delete[] nodes;
    delete[] tris;
    return st;
}

rsi_status_t rsi_bvh_root(rsi_handle_t h, int64_t* root, int64_t* sentinel, uint64_t* h_morton63, void* stream) {
    if (!h || !root) return rsi_set_error(RSI_E_INVALID_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    if (h->status_pending) {
        const rsi_status_t st0 = rsi_finish_build(h, s);
        if (st0 != RSI_OK) return st0;
    }
    if (h->n_tri <= 0) return rsi_set_error(RSI_E_INVALID_ARG, "handle holds no mesh");
    *root = h->root_node;
    if (sentinel) *sentinel = h->apetrei ? h->n_tri - 1 : -1;
    if (!h_morton63) return RSI_OK;
    const int64_t nt = h->n_tri;
    uint32_t* w = new (std::nothrow) uint32_t[2 * nt];
    if (!w) return rsi_set_error(RSI_E_OOM, "host allocation failed");
    rsi_status_t st = rsi_cuda_check(cudaMemcpyAsync(w, h->keys, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s), "keys");
    if (st == RSI_OK && h->apetrei)
        st = rsi_cuda_check(cudaMemcpyAsync(w + nt, h->k63 + 3 * nt, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s),
                            "keys");
    if (st == RSI_OK) st = rsi_cuda_check(cudaStreamSynchronize(s), "keys");
    if (st == RSI_OK)
        for (int64_t k = 0; k < nt; ++k)
            h_morton63[k] = h->apetrei ? (((uint64_t)w[k] << 32) | w[nt + k]) : (uint64_t)w[k];
    delete[] w;
    return st;
}

}  // extern "C"
