// abi.cu -- the C ABI of librici.so (include/rici.h): argument validation, host/device
// staging, workspace, launch sequencing and error reporting.  No compute happens here.
#include <atomic>
#include <cstdarg>
#include <new>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "rici.h"
#include "rici_internal.cuh"

struct rici_mesh_s {
    rici::DeviceMesh m;
    // staging (sort, kd refinement, chunk layout) finishes asynchronously on the creation stream:
    // `ready` is recorded after it, and a use on another stream waits for it first
    cudaStream_t created_on = nullptr;
    cudaEvent_t ready = nullptr;
    void wait_ready(cudaStream_t s) {
        if (ready && s != created_on) cudaStreamWaitEvent(s, ready, 0);
    }
    // one event per stream the mesh was read on, recorded after each use: rici_destroy_mesh
    // orders the frees after every recorded use, whatever the streams' flags
    std::mutex mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
    void note_use(cudaStream_t s) {
        std::lock_guard<std::mutex> lock(mu);
        cudaEvent_t ev = nullptr;
        for (auto &u : uses)
            if (u.first == s) ev = u.second;
        if (!ev) {
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { cudaGetLastError(); return; }
            uses.emplace_back(s, ev);
        }
        cudaEventRecord(ev, s);
    }
};

namespace rici {
static std::atomic<unsigned long long> g_launches{0};
void note_launches(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }

// ---- per-kernel timing: event pairs recorded around one API call's launches of a timed kernel
// (KernelTimer), drained by rici_kernel_time_ms.  The begin event travels with the caller's
// timer, so calls on several threads / streams never mix their events.
static std::atomic<int> g_timing{0};
static std::mutex g_timing_mu;
struct TimedLaunch { cudaEvent_t a, b; };
static std::vector<TimedLaunch> g_timed[2];          // per kernel id: recorded pairs (one per call)
static std::vector<cudaEvent_t> g_event_pool;
static cudaEvent_t take_event() {
    cudaEvent_t e = nullptr;
    if (!g_event_pool.empty()) { e = g_event_pool.back(); g_event_pool.pop_back(); }
    else if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); e = nullptr; }
    return e;
}
cudaEvent_t timing_begin(int kernel, cudaStream_t s) {
    (void)kernel;
    if (!g_timing.load(std::memory_order_relaxed)) return nullptr;
    std::lock_guard<std::mutex> lock(g_timing_mu);
    cudaEvent_t e = take_event();
    if (e && cudaEventRecord(e, s) != cudaSuccess) { cudaGetLastError(); g_event_pool.push_back(e); e = nullptr; }
    return e;
}
void timing_end(int kernel, cudaStream_t s, cudaEvent_t begin) {
    if (!begin) return;
    std::lock_guard<std::mutex> lock(g_timing_mu);
    cudaEvent_t e = take_event();
    if (e && cudaEventRecord(e, s) == cudaSuccess) {
        g_timed[kernel].push_back({begin, e});
    } else {
        cudaGetLastError();
        g_event_pool.push_back(begin);
        if (e) g_event_pool.push_back(e);
    }
}
void timing_release(cudaEvent_t begin) {
    if (!begin) return;
    std::lock_guard<std::mutex> lock(g_timing_mu);
    g_event_pool.push_back(begin);
}
cudaError_t ensure_smem(const void *kernel, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(kernel, dev);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[key] = bytes;
    return e;
}
bool use_mma_path(int N) {
    static const int mode = [] {           // 1 = tensor cores where applicable, 0 = SIMT only
        const char *v = getenv("RICI_CRSS_PATH");
        return (v && strcmp(v, "simt") == 0) ? 0 : 1;
    }();                                   // thread-safe initialisation (magic static)
    return mode == 1 && N == 64;
}
int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}
double env_double(const char *name, double dflt) {
    const char *v = getenv(name);
    return v ? atof(v) : dflt;
}
}  // namespace rici

namespace {

thread_local std::string g_err;

rici_status fail(rici_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
rici_status fail(rici_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

rici_status cuda_fail(cudaError_t e, const char *what) {
    cudaGetLastError();   // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation)
        return fail(RICI_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(RICI_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// sm_100 only (the kernels are compiled for sm_100a and nothing else).  Per-device result and
// pool setting are cached under a mutex (the ABI may be called from several host threads).
rici_status check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static std::mutex mu;
    static std::map<int, bool> ok_dev;
    bool ok;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = ok_dev.find(dev);
        if (it == ok_dev.end()) {
            int major = 0, minor = 0;
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
            ok = (major == 10 && minor == 0);
            if (ok) {                          // keep freed workspace in the stream-ordered pool
                cudaMemPool_t pool;
                if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                    uint64_t thr = ~0ull;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                }
            }
            ok_dev[dev] = ok;
        } else {
            ok = it->second;
        }
    }
    if (!ok) return fail(RICI_ERR_UNSUPPORTED, "device %d is not sm_100; this build is sm_100a only", dev);
    return RICI_OK;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Collects stream-ordered temporaries and host write-backs for one call.
struct Staging {
    cudaStream_t s;
    std::vector<void *> temps;
    struct Back { void *host; const void *dev; size_t bytes; };
    std::vector<Back> backs;
    explicit Staging(cudaStream_t st) : s(st) {}
    ~Staging() { for (void *t : temps) cudaFreeAsync(t, s); }

    cudaError_t in(const void *p, size_t bytes, const void **dev) {
        if (p == nullptr || bytes == 0 || is_device_ptr(p)) { *dev = p; return cudaSuccess; }
        void *d = nullptr;
        cudaError_t e = cudaMallocAsync(&d, bytes, s);
        if (e != cudaSuccess) return e;
        temps.push_back(d);
        *dev = d;
        return cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s);
    }
    cudaError_t out(void *p, size_t bytes, void **dev) {
        if (p == nullptr || bytes == 0 || is_device_ptr(p)) { *dev = p; return cudaSuccess; }
        void *d = nullptr;
        cudaError_t e = cudaMallocAsync(&d, bytes, s);
        if (e != cudaSuccess) return e;
        temps.push_back(d);
        backs.push_back({p, d, bytes});
        *dev = d;
        return cudaSuccess;
    }
    cudaError_t finish() {
        if (backs.empty()) return cudaSuccess;
        for (auto &b : backs) {
            cudaError_t e = cudaMemcpyAsync(b.host, b.dev, b.bytes, cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return e;
        }
        return cudaStreamSynchronize(s);
    }
};

bool valid_bins(int32_t n_bins) { return n_bins >= 2 && n_bins <= 128; }

// a9-a12 counts: tensor-core path for N = 64 (exact, with SIMT fallback inside), else SIMT.
// thr_from_pairs: `thr` is an output, t_i = CRSS(n_i, h_i) (a10) -- the tensor path computes it
// inside its feature pass, the SIMT path with the pair kernel first.
cudaError_t count_below(const void *dn, int64_t nn, const void *dh, int64_t nh, int N, uint64_t *thr,
                        bool thr_from_pairs, bool rank_mode, uint32_t *counts, cudaStream_t s) {
    // the tensor path streams 16-byte vectors of both image arrays
    const bool aligned = ((reinterpret_cast<uintptr_t>(dn) | reinterpret_cast<uintptr_t>(dh)) & 15) == 0;
    if (aligned && rici::use_mma_path(N)) {
        cudaError_t e = rici::launch_crss_count_mma((const uint16_t *)dn, nn, (const uint16_t *)dh, nh, thr,
                                                    thr_from_pairs, rank_mode, counts, s);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if (thr_from_pairs) {
        cudaError_t e = rici::launch_crss_pairs((const uint16_t *)dn, nn, (const uint16_t *)dh, nh, N, nullptr, nn,
                                                thr, s);
        if (e != cudaSuccess) return e;
    }
    return rici::launch_crss_search_tiles((const uint16_t *)dn, nn, (const uint16_t *)dh, nh, N, thr, counts,
                                          nullptr, s, rank_mode);
}

rici_status check_images(const void *p, int64_t n, const char *name) {
    if (n < 0) return fail(RICI_ERR_INVALID_ARGUMENT, "%s: negative count %lld", name, (long long)n);
    if (n > 0 && p == nullptr) return fail(RICI_ERR_INVALID_ARGUMENT, "%s: null pointer", name);
    return RICI_OK;
}

}  // namespace

extern "C" {

const char *rici_last_error(void) { return g_err.c_str(); }

uint64_t rici_launch_count(void) { return rici::g_launches.load(); }

rici_status rici_set_kernel_timing(int32_t enable) {
    g_err.clear();
    rici::g_timing.store(enable ? 1 : 0);
    return RICI_OK;
}

rici_status rici_kernel_time_ms(int32_t kernel, float *out_mean_ms, int64_t *out_launches) {
    g_err.clear();
    if (kernel != RICI_KERNEL_GENERATE && kernel != RICI_KERNEL_CRSS_MMA)
        return fail(RICI_ERR_INVALID_ARGUMENT, "unknown kernel id %d", (int)kernel);
    if (!out_mean_ms || !out_launches) return fail(RICI_ERR_INVALID_ARGUMENT, "null output");
    std::lock_guard<std::mutex> lock(rici::g_timing_mu);
    double sum = 0.0;
    int64_t cnt = 0;
    cudaError_t err = cudaSuccess;
    for (auto &t : rici::g_timed[kernel]) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(t.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, t.a, t.b);
        if (e == cudaSuccess) { sum += ms; ++cnt; } else if (err == cudaSuccess) err = e;
        rici::g_event_pool.push_back(t.a);
        rici::g_event_pool.push_back(t.b);
    }
    rici::g_timed[kernel].clear();
    *out_mean_ms = cnt ? (float)(sum / (double)cnt) : 0.f;    // one pair per API call
    *out_launches = cnt;
    if (err != cudaSuccess) return cuda_fail(err, "rici_kernel_time_ms");
    return RICI_OK;
}

rici_status rici_crss_guard_stats(int64_t out[5], int32_t reset) {
    g_err.clear();
    if (!out) return fail(RICI_ERR_INVALID_ARGUMENT, "null out");
    if (rici_status st = check_device()) return st;
    unsigned long long v[5] = {0, 0, 0, 0, 0};
    cudaError_t e = rici::read_guard_stats(v, reset != 0);
    if (e != cudaSuccess) return cuda_fail(e, "rici_crss_guard_stats");
    for (int k = 0; k < 5; ++k) out[k] = (int64_t)v[k];
    return RICI_OK;
}

const char *rici_version(void) { return "rici-b200 0.2.0 sm_100a"; }

int64_t rici_mesh_num_triangles(rici_mesh mesh) { return mesh ? mesh->m.nt : -1; }

rici_status rici_create_mesh(const float *vertices, int64_t n_vertices, const int32_t *indices,
                             int64_t n_triangles, rici_stream_t stream, rici_mesh *out_mesh) {
    g_err.clear();
    if (!out_mesh) return fail(RICI_ERR_INVALID_ARGUMENT, "out_mesh is null");
    if (n_vertices < 0 || n_triangles < 0)
        return fail(RICI_ERR_INVALID_ARGUMENT, "negative vertex/triangle count");
    if (n_triangles > 0 && (!vertices || !indices))
        return fail(RICI_ERR_INVALID_ARGUMENT, "null vertices/indices");
    if (n_triangles > 0 && n_vertices == 0)
        return fail(RICI_ERR_INVALID_ARGUMENT, "triangles given but no vertices");
    if (n_triangles > rici::kMaxTriangles)
        return fail(RICI_ERR_INVALID_ARGUMENT, "at most %lld triangles per mesh", (long long)rici::kMaxTriangles);
    if (rici_status st = check_device()) return st;
    cudaStream_t s = (cudaStream_t)stream;
    rici_mesh_s *mesh = new (std::nothrow) rici_mesh_s();
    if (!mesh) return fail(RICI_ERR_OUT_OF_MEMORY, "host allocation failed");
    cudaGetDevice(&mesh->m.device);
    int64_t n_chunks = (n_triangles + rici::kChunk - 1) / rici::kChunk;
    cudaError_t e = cudaSuccess;
    if (n_chunks > 0) {
        // stream-ordered pool allocations: no device-wide synchronisation on create/destroy
        e = cudaMallocAsync((void **)&mesh->m.tri, sizeof(float) * rici::kTriFloatsPerChunk * (size_t)n_chunks, s);
        if (e == cudaSuccess) e = cudaMallocAsync((void **)&mesh->m.sphere, sizeof(float4) * (size_t)n_chunks, s);
        if (e == cudaSuccess)
            e = cudaMallocAsync((void **)&mesh->m.super_sphere,
                                sizeof(float4) * (size_t)((n_chunks + rici::kSuper - 1) / rici::kSuper), s);
        if (e != cudaSuccess) { rici_destroy_mesh(mesh); return cuda_fail(e, "mesh allocation"); }
        Staging st(s);
        const void *dv = nullptr, *di = nullptr;
        int *d_bad = nullptr;
        if ((e = st.in(vertices, sizeof(float) * 3 * (size_t)n_vertices, &dv)) == cudaSuccess &&
            (e = st.in(indices, sizeof(int32_t) * 3 * (size_t)n_triangles, &di)) == cudaSuccess &&
            (e = cudaMallocAsync((void **)&d_bad, sizeof(int), s)) == cudaSuccess) {
            st.temps.push_back(d_bad);
            // the index check is synchronous, but waits only for the validating first pass: the
            // sort and staging kernels are enqueued after it and run while the caller continues
            float *centroid = nullptr;
            if ((e = cudaMemsetAsync(d_bad, 0, sizeof(int), s)) == cudaSuccess)
                e = rici::launch_mesh_stage_begin((const float *)dv, n_vertices, (const int32_t *)di,
                                                  n_triangles, &mesh->m, d_bad, &centroid, s);
            if (centroid) st.temps.push_back(centroid);           // freed stream-ordered on any exit
            int bad = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e == cudaSuccess && bad) {
                rici_destroy_mesh(mesh);
                return fail(RICI_ERR_INVALID_ARGUMENT, "triangle index out of range [0, %lld)",
                            (long long)n_vertices);
            }
            if (e == cudaSuccess)
                e = rici::launch_mesh_stage_end((const float *)dv, n_vertices, (const int32_t *)di,
                                                n_triangles, &mesh->m, centroid, s);
            if (e == cudaSuccess) {
                mesh->created_on = s;
                e = cudaEventCreateWithFlags(&mesh->ready, cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventRecord(mesh->ready, s);
                mesh->note_use(s);                 // a destroy before any use waits for staging
            }
        }
        if (e != cudaSuccess) { rici_destroy_mesh(mesh); return cuda_fail(e, "rici_create_mesh"); }
    } else {
        mesh->m.nt = 0;
        mesh->m.n_chunks = 0;
    }
    *out_mesh = mesh;
    return RICI_OK;
}

rici_status rici_destroy_mesh(rici_mesh mesh) {
    g_err.clear();
    if (!mesh) return RICI_OK;
    // stream-ordered frees on the legacy default stream, made to wait for the last recorded use
    // on every stream the mesh was read on (non-blocking streams included); no host wait
    for (auto &u : mesh->uses) {
        cudaStreamWaitEvent(0, u.second, 0);
        cudaEventDestroy(u.second);
    }
    if (mesh->m.tri) cudaFreeAsync(mesh->m.tri, 0);
    if (mesh->m.sphere) cudaFreeAsync(mesh->m.sphere, 0);
    if (mesh->m.super_sphere) cudaFreeAsync(mesh->m.super_sphere, 0);
    if (mesh->m.order) cudaFreeAsync(mesh->m.order, 0);
    if (mesh->ready) cudaEventDestroy(mesh->ready);
    delete mesh;
    return RICI_OK;
}

rici_status rici_generate(rici_mesh mesh, const float *origins, int64_t n, float support_radius,
                          int32_t n_bins, uint16_t *out, rici_stream_t stream) {
    g_err.clear();
    if (!mesh) return fail(RICI_ERR_INVALID_ARGUMENT, "mesh is null");
    if (n < 0) return fail(RICI_ERR_INVALID_ARGUMENT, "negative image count");
    if (n > 0 && (!origins || !out)) return fail(RICI_ERR_INVALID_ARGUMENT, "null origins/out");
    if (!(support_radius > 0.f) || !std::isfinite(support_radius))
        return fail(RICI_ERR_INVALID_ARGUMENT, "support_radius must be finite and > 0");
    if (!valid_bins(n_bins)) return fail(RICI_ERR_INVALID_ARGUMENT, "n_bins must be in [2,128]");
    if (rici_status st = check_device()) return st;
    if (n == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Staging st(s);
    const void *dorig = nullptr;
    void *dout = nullptr;
    size_t out_bytes = sizeof(uint16_t) * (size_t)n * n_bins * n_bins;
    cudaError_t e = st.in(origins, sizeof(float) * 6 * (size_t)n, &dorig);
    if (e == cudaSuccess) e = st.out(out, out_bytes, &dout);
    mesh->wait_ready(s);
    if (e == cudaSuccess)
        e = rici::launch_generate(mesh->m, (const float *)dorig, n, support_radius, n_bins,
                                  (uint16_t *)dout, s);
    if (e == cudaSuccess) mesh->note_use(s);
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_generate");
    return RICI_OK;
}

rici_status rici_clutter_fraction(rici_mesh mesh, const uint8_t *object_tag, const float *origins, int64_t n,
                                  float support_radius, int32_t quadrature_q, float *out_fraction,
                                  float *out_area_all, rici_stream_t stream) {
    g_err.clear();
    if (!mesh) return fail(RICI_ERR_INVALID_ARGUMENT, "mesh is null");
    if (n < 0) return fail(RICI_ERR_INVALID_ARGUMENT, "negative count");
    if (n > 0 && (!origins || !out_fraction)) return fail(RICI_ERR_INVALID_ARGUMENT, "null origins/out_fraction");
    if (mesh->m.nt > 0 && !object_tag) return fail(RICI_ERR_INVALID_ARGUMENT, "null object_tag");
    if (!(support_radius > 0.f) || !std::isfinite(support_radius))
        return fail(RICI_ERR_INVALID_ARGUMENT, "support_radius must be finite and > 0");
    if (quadrature_q < 1 || quadrature_q > 16) return fail(RICI_ERR_INVALID_ARGUMENT, "quadrature_q must be in [1,16]");
    if (rici_status st = check_device()) return st;
    if (n == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Staging st(s);
    const void *dt = nullptr, *dorig = nullptr;
    void *df = nullptr, *da = nullptr;
    cudaError_t e = st.in(object_tag, (size_t)mesh->m.nt, &dt);
    if (e == cudaSuccess) e = st.in(origins, sizeof(float) * 6 * (size_t)n, &dorig);
    if (e == cudaSuccess) e = st.out(out_fraction, sizeof(float) * (size_t)n, &df);
    if (e == cudaSuccess && out_area_all) e = st.out(out_area_all, sizeof(float) * (size_t)n, &da);
    mesh->wait_ready(s);
    if (e == cudaSuccess)
        e = rici::launch_clutter_fraction(mesh->m, (const unsigned char *)dt, (const float *)dorig, n, support_radius,
                                          quadrature_q, (float *)df, (float *)da, s);
    if (e == cudaSuccess) mesh->note_use(s);
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_clutter_fraction");
    return RICI_OK;
}

rici_status rici_crss_pairs(const uint16_t *needles, int64_t n_needles, const uint16_t *haystack,
                            int64_t n_haystack, int32_t n_bins, const int64_t *pairs, int64_t m,
                            uint64_t *out, rici_stream_t stream) {
    g_err.clear();
    if (!valid_bins(n_bins)) return fail(RICI_ERR_INVALID_ARGUMENT, "n_bins must be in [2,128]");
    if (rici_status st = check_images(needles, n_needles, "needles")) return st;
    if (rici_status st = check_images(haystack, n_haystack, "haystack")) return st;
    if (m < 0) return fail(RICI_ERR_INVALID_ARGUMENT, "negative pair count");
    if (m > 0 && (!pairs || !out)) return fail(RICI_ERR_INVALID_ARGUMENT, "null pairs/out");
    if (rici_status st = check_device()) return st;
    if (m == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (!is_device_ptr(pairs)) {
        for (int64_t k = 0; k < m; ++k)
            if (pairs[2 * k] < 0 || pairs[2 * k] >= n_needles || pairs[2 * k + 1] < 0 ||
                pairs[2 * k + 1] >= n_haystack)
                return fail(RICI_ERR_INVALID_ARGUMENT, "pair %lld out of range", (long long)k);
    }
    const size_t P = (size_t)n_bins * n_bins;
    Staging st(s);
    const void *dn = nullptr, *dh = nullptr, *dp = nullptr;
    void *dout = nullptr;
    cudaError_t e = st.in(needles, sizeof(uint16_t) * P * n_needles, &dn);
    if (e == cudaSuccess) e = st.in(haystack, sizeof(uint16_t) * P * n_haystack, &dh);
    if (e == cudaSuccess) e = st.in(pairs, sizeof(int64_t) * 2 * (size_t)m, &dp);
    if (e == cudaSuccess) e = st.out(out, sizeof(uint64_t) * (size_t)m, &dout);
    if (e == cudaSuccess)
        e = rici::launch_crss_pairs((const uint16_t *)dn, n_needles, (const uint16_t *)dh, n_haystack,
                                    n_bins, (const int64_t *)dp, m, (uint64_t *)dout, s);
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_crss_pairs");
    return RICI_OK;
}

rici_status rici_crss_count_below(const uint16_t *needles, int64_t n_needles,
                                  const uint16_t *haystack, int64_t n_haystack, int32_t n_bins,
                                  const uint64_t *thresholds, uint32_t *out_counts,
                                  rici_stream_t stream) {
    g_err.clear();
    if (!valid_bins(n_bins)) return fail(RICI_ERR_INVALID_ARGUMENT, "n_bins must be in [2,128]");
    if (rici_status st = check_images(needles, n_needles, "needles")) return st;
    if (rici_status st = check_images(haystack, n_haystack, "haystack")) return st;
    if (n_needles > 0 && (!thresholds || !out_counts))
        return fail(RICI_ERR_INVALID_ARGUMENT, "null thresholds/out_counts");
    if (rici_status st = check_device()) return st;
    if (n_needles == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)n_bins * n_bins;
    Staging st(s);
    const void *dn = nullptr, *dh = nullptr, *dt = nullptr;
    void *dc = nullptr;
    cudaError_t e = st.in(needles, sizeof(uint16_t) * P * n_needles, &dn);
    if (e == cudaSuccess) e = st.in(haystack, sizeof(uint16_t) * P * n_haystack, &dh);
    if (e == cudaSuccess) e = st.in(thresholds, sizeof(uint64_t) * (size_t)n_needles, &dt);
    if (e == cudaSuccess) e = st.out(out_counts, sizeof(uint32_t) * (size_t)n_needles, &dc);
    if (e == cudaSuccess) e = count_below(dn, n_needles, dh, n_haystack, n_bins, (uint64_t *)const_cast<void *>(dt),
                                          false, false, (uint32_t *)dc, s);
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_crss_count_below");
    return RICI_OK;
}

rici_status rici_crss_distances(const uint16_t *needles, int64_t n_needles,
                                const uint16_t *haystack, int64_t n_haystack, int32_t n_bins,
                                uint64_t *out, rici_stream_t stream) {
    g_err.clear();
    if (!valid_bins(n_bins)) return fail(RICI_ERR_INVALID_ARGUMENT, "n_bins must be in [2,128]");
    if (rici_status st = check_images(needles, n_needles, "needles")) return st;
    if (rici_status st = check_images(haystack, n_haystack, "haystack")) return st;
    if (n_needles > 0 && n_haystack > 0 && !out) return fail(RICI_ERR_INVALID_ARGUMENT, "null out");
    if (rici_status st = check_device()) return st;
    if (n_needles == 0 || n_haystack == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)n_bins * n_bins;
    Staging st(s);
    const void *dn = nullptr, *dh = nullptr;
    void *dout = nullptr;
    cudaError_t e = st.in(needles, sizeof(uint16_t) * P * n_needles, &dn);
    if (e == cudaSuccess) e = st.in(haystack, sizeof(uint16_t) * P * n_haystack, &dh);
    if (e == cudaSuccess) e = st.out(out, sizeof(uint64_t) * (size_t)n_needles * n_haystack, &dout);
    if (e == cudaSuccess)
        e = rici::launch_crss_search_tiles((const uint16_t *)dn, n_needles, (const uint16_t *)dh,
                                           n_haystack, n_bins, nullptr, nullptr, (uint64_t *)dout, s);
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_crss_distances");
    return RICI_OK;
}

rici_status rici_crss_search_ex(const uint16_t *needles, int64_t n_needles, const uint16_t *haystack,
                                int64_t n_haystack, int32_t n_bins, uint32_t flags, uint32_t *out_ranks,
                                rici_stream_t stream) {
    g_err.clear();
    if (!valid_bins(n_bins)) return fail(RICI_ERR_INVALID_ARGUMENT, "n_bins must be in [2,128]");
    if (rici_status st = check_images(needles, n_needles, "needles")) return st;
    if (rici_status st = check_images(haystack, n_haystack, "haystack")) return st;
    if (n_haystack < n_needles)
        return fail(RICI_ERR_INVALID_ARGUMENT, "n_haystack (%lld) < n_needles (%lld): needle i "
                    "corresponds to haystack i", (long long)n_haystack, (long long)n_needles);
    if (n_needles > 0 && !out_ranks) return fail(RICI_ERR_INVALID_ARGUMENT, "null out_ranks");
    if (flags & ~(RICI_CRSS_SIMT | RICI_CRSS_EARLY_EXIT)) return fail(RICI_ERR_INVALID_ARGUMENT, "unknown flags");
    if (rici_status st = check_device()) return st;
    if (n_needles == 0) return RICI_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)n_bins * n_bins;
    Staging st(s);
    const void *dn = nullptr, *dh = nullptr;
    void *dr = nullptr;
    uint64_t *thr = nullptr;
    cudaError_t e = st.in(needles, sizeof(uint16_t) * P * n_needles, &dn);
    if (e == cudaSuccess) e = st.in(haystack, sizeof(uint16_t) * P * n_haystack, &dh);
    if (e == cudaSuccess) e = st.out(out_ranks, sizeof(uint32_t) * (size_t)n_needles, &dr);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&thr, sizeof(uint64_t) * (size_t)n_needles, s);
    if (e == cudaSuccess) st.temps.push_back(thr);
    // a10: t_i = CRSS(n_i, h_i) ("this threshold can be trivially precomputed") -- by
    // the pair kernel for the SIMT path, inside count_below's feature pass otherwise.
    // RICI_CRSS_EARLY_EXIT alone: rank mode on the best path (tensor tiles pruned by a K-prefix
    // bound at N = 64); with RICI_CRSS_SIMT: the SIMT kernel's per-pair early exit.
    if (e == cudaSuccess) {
        if (flags & RICI_CRSS_SIMT) {
            e = rici::launch_crss_pairs((const uint16_t *)dn, n_needles, (const uint16_t *)dh, n_haystack,
                                        n_bins, nullptr, n_needles, thr, s);
            if (e == cudaSuccess)
                e = rici::launch_crss_search_tiles((const uint16_t *)dn, n_needles, (const uint16_t *)dh, n_haystack,
                                                   n_bins, thr, (uint32_t *)dr, nullptr, s,
                                                   (flags & RICI_CRSS_EARLY_EXIT) != 0);
        } else {
            e = count_below(dn, n_needles, dh, n_haystack, n_bins, thr, true, (flags & RICI_CRSS_EARLY_EXIT) != 0,
                            (uint32_t *)dr, s);
        }
    }
    if (e == cudaSuccess) e = st.finish();
    if (e != cudaSuccess) return cuda_fail(e, "rici_crss_search");
    return RICI_OK;
}

rici_status rici_crss_search(const uint16_t *needles, int64_t n_needles, const uint16_t *haystack,
                             int64_t n_haystack, int32_t n_bins, uint32_t *out_ranks,
                             rici_stream_t stream) {
    return rici_crss_search_ex(needles, n_needles, haystack, n_haystack, n_bins, 0u, out_ranks, stream);
}

}  // extern "C"
