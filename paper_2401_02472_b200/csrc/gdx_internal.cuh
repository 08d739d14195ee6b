// gdx_internal.cuh -- shared internals of libgdx.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gdx.h"

namespace gdx {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, gdx_status at the boundary.
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    gdx_status code;
    Error(gdx_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(gdx_status c, const std::string& msg) { throw Error(c, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    gdx_status code = e == cudaErrorMemoryAllocation ? GDX_ERR_OUT_OF_MEMORY : GDX_ERR_CUDA;
    fail(code, std::string("CudaError: ") + what + " -> " + cudaGetErrorString(e) + " (" + file +
                   ":" + std::to_string(line) + ")");
}
#define GDX_CUDA(x) ::gdx::cuda_check((x), #x, __FILE__, __LINE__)
#define GDX_LAUNCH_CHECK() ::gdx::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Sets the calling thread's device for the scope.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) GDX_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Device memory pool (api.cu): freed blocks are kept per device and handed
// back to allocations of similar size, so repeated graph create/destroy
// cycles (the C-ABI e2e path) do not pay cudaMalloc/cudaFree.  Inside a
// StreamScope (every entry point that holds a graph opens one) a release is
// stream-ordered: it records an event on the scope's stream and the block's
// next user waits for it on its own stream; outside any scope a release
// synchronises the device (cudaFree's guarantee).  An allocation that fails
// releases the cache and retries.
struct StreamScope {
    cudaStream_t prev;
    bool prev_set;
    explicit StreamScope(cudaStream_t s);
    ~StreamScope();
    StreamScope(const StreamScope&) = delete;
    StreamScope& operator=(const StreamScope&) = delete;
};
void* pool_alloc(size_t bytes, size_t* got);
void pool_free(void* p, size_t bytes);
size_t pool_trim();
size_t pool_cached();  // bytes held free by the pool (all devices)
void* pinned_alloc();
void pinned_free(void* p);

// Owning device buffer.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    size_t cap = 0;  // bytes of the underlying block
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) { o.p = nullptr, o.n = 0, o.cap = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n, cap = o.cap;
            o.p = nullptr, o.n = 0, o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) count = 1;
        // +64 B tail: vector loads round segment ends up to 16 B.
        p = static_cast<T*>(pool_alloc(count * sizeof(T) + 64, &cap));
        n = count;
    }
    // Grow-only allocation (workspaces cached on the graph handle).
    void ensure(size_t count) {
        if (count > n || p == nullptr) alloc(count);
    }
    void release() {
        if (p) pool_free(p, cap);
        p = nullptr;
        n = 0;
        cap = 0;
    }
    T* get() const { return p; }
    size_t bytes() const { return n * sizeof(T); }
};

// Per-kernel CUDA-event timing (gdx_profile_*): events recorded on the
// launching stream around every launch while enabled.
struct Profiler {
    bool enabled = false;
    struct Rec {
        std::string name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<double, int64_t>> totals;

    cudaEvent_t take() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        GDX_CUDA(cudaEventCreate(&e));
        return e;
    }
    void drain() {  // fold completed pairs into totals (synchronises on them)
        for (auto& r : pending) {
            GDX_CUDA(cudaEventSynchronize(r.b));
            float ms = 0.f;
            GDX_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            auto& t = totals[r.name];
            t.first += ms;
            t.second += 1;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    ~Profiler() {
        for (auto& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

struct PrPlan;
struct PrP2P;
struct SsspWork;
struct SsspP2P;
struct TcPlan;
struct BcWork;
struct Relabel;

}  // namespace gdx

// The opaque handle behind gdx_graph*.
struct gdx_graph {
    int device = 0;
    int32_t n = 0, m = 0;
    bool directed = true;
    bool weighted = false;     // false => every weight is 1
    int32_t max_weight = 1;
    int32_t max_degree = -1;   // max out- (and, directed, in-) degree; lazily computed
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;

    gdx::DevBuf<int32_t> offsets, dests, weights, rev_offsets, rev_srcs, rev_eid;
    // The reverse CSR.  An undirected graph is stored symmetrically with sorted
    // rows, so its reverse CSR *is* the forward one: unless the caller uploaded
    // reverse arrays, these return the forward arrays (no copy, no memory);
    // rev_eid is then built on demand (gdx_graph_download).
    const int32_t* in_offsets() const {
        return rev_offsets.get() ? rev_offsets.get() : directed ? nullptr : offsets.get();
    }
    const int32_t* in_srcs() const {
        return rev_srcs.get() ? rev_srcs.get() : directed ? nullptr : dests.get();
    }

    gdx::Profiler prof;
    std::unique_ptr<gdx::PrPlan> pr;
    std::unique_ptr<gdx::PrPlan> pr_shard;  // gdx_pr_shard_* (one rank's vertex range)
    std::unique_ptr<gdx::PrP2P> pr_p2p;     // gdx_pr_p2p_* (peer-memory exchange)
    std::unique_ptr<gdx::SsspWork> sssp;
    std::unique_ptr<gdx::SsspP2P> sssp_p2p;  // gdx_sssp_p2p_* (peer-memory partitions)
    std::unique_ptr<gdx::TcPlan> tc;
    std::unique_ptr<gdx::BcWork> bc;
    std::unique_ptr<gdx::Relabel> relabel;  // degree-ordered renumbering (relabel.cu)
    int32_t relabel_calls = 0;              // PR / SSSP calls that could have used it
    bool relabel_failed = false;            // its build ran out of device memory: never again

    // scratch for small device->host reads
    int64_t* pinned = nullptr;  // 4 KB pinned host scratch

    ~gdx_graph();
};

namespace gdx {

// The device and stream scope of an entry point working on graph g: sets the
// thread's device and makes pool releases stream-ordered on g's stream.
struct GraphScope {
    DeviceGuard dev;
    StreamScope str;
    explicit GraphScope(gdx_graph* g) : dev(g->device), str(g->stream) {}
};

// Launch helper: brackets a kernel launch with profiler events.
template <class F>
inline void timed_launch(gdx_graph* g, const char* name, F&& launch) {
    if (!g->prof.enabled) {
        launch();
        GDX_LAUNCH_CHECK();
        return;
    }
    cudaEvent_t a = g->prof.take(), b = g->prof.take();
    GDX_CUDA(cudaEventRecord(a, g->stream));
    launch();
    GDX_LAUNCH_CHECK();
    GDX_CUDA(cudaEventRecord(b, g->stream));
    g->prof.pending.push_back({name, a, b});
}

// Copy with unified addressing (host pageable/pinned or device pointers).
inline void copy_out(gdx_graph* g, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    GDX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, g->stream));
}

// Shared-memory carveout (percent of the unified L1 / shared capacity) of a
// gather kernel that uses no shared memory, so the L1 holding its gathered
// lines is as large as it gets; GDX_CARVEOUT = percent overrides, -1 leaves
// the driver's choice.  Set once per kernel and device.
inline void prefer_l1(const void* fn, int dflt) {
    static const int env = [] {
        const char* e = std::getenv("GDX_CARVEOUT");
        return e ? std::atoi(e) : -2;
    }();
    const int pct = env == -2 ? dflt : env;
    if (pct < 0) return;
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    GDX_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (auto& d : done)
        if (d.first == fn && d.second == dev) return;
    GDX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    done.emplace_back(fn, dev);
}

inline int blocks_for(int64_t items, int threads, int cap) {
    int64_t b = (items + threads - 1) / threads;
    if (b < 1) b = 1;
    return static_cast<int>(b < cap ? b : cap);
}

// Max out-degree (and in-degree for directed graphs), computed once per handle
// (api.cu); the kernels pick hub-aware or latency-oriented variants from it.
int32_t graph_max_degree(gdx_graph* g);

// relabel.cu: the degree-ordered renumbering cached on a handle
bool relabel_wanted(gdx_graph* g);
Relabel& relabel_ensure(gdx_graph* g, bool need_fwd, bool need_rev);
// relabel_ensure, or nullptr when its build runs out of device memory (the
// call then runs on the caller's numbering, and the handle stops trying)
Relabel* relabel_try(gdx_graph* g, bool need_fwd, bool need_rev);
void relabel_leave(gdx_graph* g);  // the hidden graph's profile records to g
void relabel_unpermute_f64(gdx_graph* g, const double* in, double* out);
int32_t relabel_vertex(gdx_graph* g, int32_t v);  // newid[v] (host read)

// Builds the reverse CSR (csr.cpp:77-94 semantics) on the device.
void build_reverse_device(gdx_graph* g);
void build_rev_eid_symmetric(gdx_graph* g);
// Upload / finish a graph whose forward arrays are resident.
void finalize_graph(gdx_graph* g);

// Counter-based RNG: splitmix64 finaliser keyed
// by (seed, stream).  Identical on host and device.
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed + stream * 0xD1B54A32D192ED03ULL);
}
__host__ __device__ inline uint64_t ctr_hash(uint64_t key, uint64_t ctr) {
    return mix64(key ^ mix64(ctr));
}
__host__ __device__ inline double ctr_unit(uint64_t h) {
    return static_cast<double>(h >> 11) * 0x1.0p-53;
}
__device__ inline uint32_t ctr_bounded(uint64_t h, uint32_t n) {
    return static_cast<uint32_t>(__umul64hi(h, static_cast<uint64_t>(n)));
}
enum : uint64_t { kStreamRmat = 1, kStreamUniform = 2, kStreamGrid = 3, kStreamWeight = 4 };

}  // namespace gdx
