// api.cu -- C-ABI plumbing: error reporting, graph handle lifetime, upload,
// download, streams and per-kernel profiling.  Algorithm entry points live in
// sssp.cu / pagerank.cu / tc.cu / bc.cu; construction in build.cu.
#include <cstring>

#include <map>
#include <mutex>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace {
thread_local std::string g_last_error;
}

gdx_graph::~gdx_graph() {
    // Plans hold device buffers; release them before the stream goes away.
    relabel.reset();
    pr_p2p.reset();
    sssp_p2p.reset();
    pr.reset();
    pr_shard.reset();
    sssp.reset();
    tc.reset();
    bc.reset();
    // the CSR goes back to the pool while the stream its release is ordered on
    // still exists
    for (auto* b : {&offsets, &dests, &weights, &rev_offsets, &rev_srcs, &rev_eid}) b->release();
    if (pinned) gdx::pinned_free(pinned);
    if (own_stream) cudaStreamDestroy(own_stream);
}

namespace gdx {

// ---- device memory pool ------------------------------------------------------
// Stream-ordered caching: a block released inside a GraphScope records an event
// on that handle's stream instead of synchronising the device; the next user
// of the block makes its own stream wait for that event (or, outside any
// scope, waits on the host).  Distinct handles on distinct streams therefore
// never stall each other through the pool.
namespace {
struct Block {
    int device;
    void* ptr;
    cudaEvent_t ready;  // released-at point on the releasing stream (or null)
};
struct Pool {
    std::mutex mu;
    std::multimap<size_t, Block> free;  // bytes -> block
    std::multimap<int, cudaEvent_t> events;  // device -> spare event
    size_t cached = 0;
};
Pool& pool() {
    static Pool* p = new Pool;  // leaked on purpose: outlives static destructors
    return *p;
}
constexpr size_t kPoolCap = size_t(48) << 30;  // cached bytes kept per process
thread_local cudaStream_t t_stream = nullptr;
thread_local bool t_stream_set = false;
}  // namespace

StreamScope::StreamScope(cudaStream_t s) : prev(t_stream), prev_set(t_stream_set) {
    t_stream = s;
    t_stream_set = true;
}
StreamScope::~StreamScope() {
    t_stream = prev;
    t_stream_set = prev_set;
}

void* pool_alloc(size_t bytes, size_t* got) {
    int dev = 0;
    GDX_CUDA(cudaGetDevice(&dev));
    auto& P = pool();
    Block hit{-1, nullptr, nullptr};
    {
        std::lock_guard<std::mutex> lk(P.mu);
        const size_t hi = bytes + bytes / 4 + (size_t(2) << 20);
        for (auto it = P.free.lower_bound(bytes); it != P.free.end() && it->first <= hi; ++it)
            if (it->second.device == dev) {
                hit = it->second;
                *got = it->first;
                P.cached -= it->first;
                P.free.erase(it);
                break;
            }
    }
    if (hit.ptr) {
        if (hit.ready) {
            if (t_stream_set)
                GDX_CUDA(cudaStreamWaitEvent(t_stream, hit.ready, 0));
            else
                GDX_CUDA(cudaEventSynchronize(hit.ready));
            std::lock_guard<std::mutex> lk(P.mu);
            P.events.emplace(dev, hit.ready);
        }
        return hit.ptr;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        pool_trim();
        e = cudaMalloc(&p, bytes);
    }
    GDX_CUDA(e);
    *got = bytes;
    return p;
}

void pool_free(void* p, size_t bytes) {
    if (!p) return;
    int dev = 0;
    cudaGetDevice(&dev);
    auto& P = pool();
    cudaEvent_t ev = nullptr;
    if (t_stream_set) {
        {
            std::lock_guard<std::mutex> lk(P.mu);
            auto it = P.events.find(dev);
            if (it != P.events.end()) {
                ev = it->second;
                P.events.erase(it);
            }
        }
        if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) ev = nullptr;
        if (ev && cudaEventRecord(ev, t_stream) != cudaSuccess) {
            cudaEventDestroy(ev);
            ev = nullptr;
        }
    }
    if (!ev) cudaDeviceSynchronize();  // outside any scope: cudaFree's guarantee
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.cached + bytes > kPoolCap) {
        cudaFree(p);  // synchronises
        if (ev) P.events.emplace(dev, ev);
        return;
    }
    P.free.emplace(bytes, Block{dev, p, ev});
    P.cached += bytes;
}

// 4 KB pinned host scratch blocks of graph handles (cudaFreeHost would
// synchronise the device on every graph destroy).
namespace {
std::mutex g_pinned_mu;
std::vector<void*>& pinned_free_list() {
    static auto* v = new std::vector<void*>;
    return *v;
}
}  // namespace

void* pinned_alloc() {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        auto& v = pinned_free_list();
        if (!v.empty()) {
            void* p = v.back();
            v.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    GDX_CUDA(cudaMallocHost(&p, 4096));
    return p;
}

void pinned_free(void* p) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    pinned_free_list().push_back(p);
}

size_t pool_cached() {
    auto& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    return P.cached;
}

size_t pool_trim() {
    auto& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    size_t n = P.cached;
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : P.free) {
        cudaSetDevice(kv.second.device);
        cudaFree(kv.second.ptr);
        if (kv.second.ready) cudaEventDestroy(kv.second.ready);
    }
    for (auto& kv : P.events) {
        cudaSetDevice(kv.first);
        cudaEventDestroy(kv.second);
    }
    cudaSetDevice(cur);
    P.free.clear();
    P.events.clear();
    P.cached = 0;
    return n;
}

__global__ void k_max_degree(int32_t n, const int32_t* __restrict__ off, int32_t* out) {
    int32_t m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        m = max(m, off[v + 1] - off[v]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

int32_t graph_max_degree(gdx_graph* g) {
    if (g->max_degree >= 0) return g->max_degree;
    int32_t best = 0;
    for (const int32_t* off : {static_cast<const int32_t*>(g->offsets.get()), g->directed ? g->in_offsets() : nullptr}) {
        if (!off || g->n == 0) continue;
        DevBuf<int32_t> d(1);
        GDX_CUDA(cudaMemsetAsync(d.get(), 0, 4, g->stream));
        k_max_degree<<<blocks_for(g->n, 256, g->num_sms * 4), 256, 0, g->stream>>>(g->n, off,
                                                                                  d.get());
        GDX_LAUNCH_CHECK();
        int32_t h = 0;
        GDX_CUDA(cudaMemcpyAsync(&h, d.get(), 4, cudaMemcpyDeviceToHost, g->stream));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        best = std::max(best, h);
    }
    g->max_degree = best;
    return best;
}

int guard_impl(const std::function<void()>& f) {
    try {
        f();
        return GDX_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "OutOfMemory: host allocation failed";
        return GDX_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_last_error = std::string("RuntimeError: ") + e.what();
        return GDX_ERR_RUNTIME;
    }
}

static void new_handle(gdx_graph* g, int device) {
    int ndev = 0;
    GDX_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: device " + std::to_string(device) +
                                           " out of range [0, " + std::to_string(ndev) + ")");
    g->device = device;
    GDX_CUDA(cudaSetDevice(device));
    GDX_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
    GDX_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
    g->stream = g->own_stream;
    g->pinned = static_cast<int64_t*>(pinned_alloc());
}

gdx_graph* make_graph(int device) {
    auto* g = new gdx_graph;
    try {
        new_handle(g, device);
    } catch (...) {
        delete g;
        throw;
    }
    return g;
}

__global__ void k_max_weight(const int32_t* __restrict__ w, int64_t m, int32_t* out,
                             int32_t* neg) {
    int32_t local = 0;
    int32_t bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = w[i];
        local = max(local, x);
        bad |= x < 0;
    }
    for (int o = 16; o; o >>= 1) {
        local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, local);
        if (bad) atomicOr(neg, 1);
    }
}

// An undirected CsrGraph stores every edge both ways (csr.cpp:42-45) and the
// handle reads its forward arrays as the reverse CSR; a view that claims
// directed = 0 with asymmetric rows is rejected.  One warp per vertex u, lanes
// over N(u), a binary search for u in N(v).
__global__ void k_check_symmetric(int32_t n, const int32_t* __restrict__ off,
                                  const int32_t* __restrict__ dst, int64_t* bad) {
    const int lane = threadIdx.x & 31;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t b = off[u], e = off[u + 1];
        for (int32_t i = b + lane; i < e; i += 32) {
            const int32_t v = dst[i];
            bool found = false;
            if (v >= 0 && v < n) {
                int32_t lo = off[v], hi = off[v + 1];
                while (lo < hi) {
                    const int32_t mid = lo + ((hi - lo) >> 1);
                    const int32_t x = dst[mid];
                    if (x == int32_t(u)) { found = true; break; }
                    if (x < int32_t(u)) lo = mid + 1; else hi = mid;
                }
            }
            if (!found) atomicCAS(reinterpret_cast<unsigned long long*>(bad), ~0ull,
                                  (unsigned long long)(int64_t(u) << 32 | uint32_t(v)));
        }
    }
}

static void check_symmetric(gdx_graph* g) {
    if (g->directed || g->m == 0 || !g->dests.get()) return;
    DevBuf<int64_t> bad(1);
    GDX_CUDA(cudaMemsetAsync(bad.get(), 0xff, 8, g->stream));
    k_check_symmetric<<<blocks_for(int64_t(g->n) * 32, 256, g->num_sms * 16), 256, 0, g->stream>>>(
        g->n, g->offsets.get(), g->dests.get(), bad.get());
    GDX_LAUNCH_CHECK();
    int64_t h = -1;
    GDX_CUDA(cudaMemcpyAsync(&h, bad.get(), 8, cudaMemcpyDeviceToHost, g->stream));
    GDX_CUDA(cudaStreamSynchronize(g->stream));
    if (h != -1)
        fail(GDX_ERR_INVALID_ARGUMENT,
             "InvalidArgument: undirected graph is not stored symmetrically (edge " +
                 std::to_string(h >> 32) + " -> " + std::to_string(int32_t(h & 0xffffffff)) +
                 " has no mirror)");
}

// Computes max_weight (SSSP chooses 32- or 64-bit distances from it) and
// rejects negative weights (csr.cpp:36-39 NegativeWeight).
void finalize_graph(gdx_graph* g) {
    g->relabel.reset();  // the renumbered copy holds the old weights
    g->max_weight = 1;
    if (g->weighted && g->m > 0) {
        DevBuf<int32_t> tmp(2);
        GDX_CUDA(cudaMemsetAsync(tmp.get(), 0, 2 * sizeof(int32_t), g->stream));
        k_max_weight<<<blocks_for(g->m, 256, g->num_sms * 8), 256, 0, g->stream>>>(
            g->weights.get(), g->m, tmp.get(), tmp.get() + 1);
        GDX_LAUNCH_CHECK();
        int32_t h[2];
        GDX_CUDA(cudaMemcpyAsync(h, tmp.get(), sizeof(h), cudaMemcpyDeviceToHost, g->stream));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        if (h[1]) fail(GDX_ERR_INVALID_ARGUMENT, "NegativeWeight: graph has a negative weight");
        g->max_weight = h[0];
    }
}

}  // namespace gdx

using namespace gdx;

extern "C" {

const char* gdx_last_error(void) { return g_last_error.c_str(); }
int gdx_abi_version(void) { return GDX_ABI_VERSION; }

int gdx_device_count(int* count) {
    return guard_impl([&] { GDX_CUDA(cudaGetDeviceCount(count)); });
}

int gdx_graph_create(const gdx_csr_view* v, int device, gdx_graph** out) {
    return guard_impl([&] {
        if (!v || !out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null view/out");
        if (v->n < 0 || v->m < 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: negative size");
        if (!v->offsets) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: offsets required");
        bool has_rev = v->rev_offsets && v->rev_srcs;
        if (!v->dests && !has_rev)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: dests or rev_offsets/rev_srcs required");
        std::unique_ptr<gdx_graph> g(make_graph(device));
        GraphScope dg(g.get());
        g->n = v->n;
        g->m = v->m;
        g->directed = v->directed != 0;
        g->weighted = v->weights != nullptr;
        cudaStream_t s = g->stream;
        const size_t nb = (size_t(v->n) + 1) * sizeof(int32_t), mb = size_t(v->m) * sizeof(int32_t);
        g->offsets.alloc(size_t(v->n) + 1);
        GDX_CUDA(cudaMemcpyAsync(g->offsets.get(), v->offsets, nb, cudaMemcpyDefault, s));
        if (v->dests) {
            g->dests.alloc(v->m);
            GDX_CUDA(cudaMemcpyAsync(g->dests.get(), v->dests, mb, cudaMemcpyDefault, s));
        }
        if (v->weights) {
            g->weights.alloc(v->m);
            GDX_CUDA(cudaMemcpyAsync(g->weights.get(), v->weights, mb, cudaMemcpyDefault, s));
        }
        if (has_rev) {
            g->rev_offsets.alloc(size_t(v->n) + 1);
            g->rev_srcs.alloc(v->m);
            GDX_CUDA(cudaMemcpyAsync(g->rev_offsets.get(), v->rev_offsets, nb, cudaMemcpyDefault, s));
            GDX_CUDA(cudaMemcpyAsync(g->rev_srcs.get(), v->rev_srcs, mb, cudaMemcpyDefault, s));
            if (v->rev_eid) {
                g->rev_eid.alloc(v->m);
                GDX_CUDA(cudaMemcpyAsync(g->rev_eid.get(), v->rev_eid, mb, cudaMemcpyDefault, s));
            }
        } else if (g->directed) {
            build_reverse_device(g.get());
        }
        check_symmetric(g.get());
        finalize_graph(g.get());
        GDX_CUDA(cudaStreamSynchronize(s));
        *out = g.release();
    });
}

int gdx_pool_trim(int64_t* released_bytes) {
    return guard_impl([&] {
        const size_t n = pool_trim();
        if (released_bytes) *released_bytes = int64_t(n);
    });
}

int gdx_graph_destroy(gdx_graph* g) {
    return guard_impl([&] {
        if (!g) return;
        GraphScope dg(g);
        cudaStreamSynchronize(g->stream);
        delete g;
    });
}

int gdx_graph_info(const gdx_graph* g, int32_t* n, int32_t* m, int32_t* directed) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        if (n) *n = g->n;
        if (m) *m = g->m;
        if (directed) *directed = g->directed;
    });
}

int gdx_graph_download(gdx_graph* g, int32_t* offsets, int32_t* dests, int32_t* weights,
                       int32_t* rev_offsets, int32_t* rev_srcs, int32_t* rev_eid) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope dg(g);
        const size_t nb = (size_t(g->n) + 1) * 4, mb = size_t(g->m) * 4;
        auto need = [&](void* dst, const DevBuf<int32_t>& b, size_t bytes, const char* what) {
            if (!dst) return;
            if (!b.get() && bytes)
                fail(GDX_ERR_UNSUPPORTED, std::string("Unsupported: graph has no ") + what);
            copy_out(g, dst, b.get(), bytes);
        };
        need(offsets, g->offsets, nb, "offsets");
        need(dests, g->dests, mb, "dests");
        if (weights) {
            if (g->weighted)
                copy_out(g, weights, g->weights.get(), mb);
            else {  // unweighted: every weight is 1 (host or device destination)
                std::vector<int32_t> ones(size_t(g->m), 1);
                GDX_CUDA(cudaMemcpyAsync(weights, ones.data(), mb, cudaMemcpyDefault, g->stream));
                GDX_CUDA(cudaStreamSynchronize(g->stream));
            }
        }
        auto need_ptr = [&](void* dst, const int32_t* src, size_t bytes, const char* what) {
            if (!dst) return;
            if (!src && bytes) fail(GDX_ERR_UNSUPPORTED, std::string("Unsupported: graph has no ") + what);
            copy_out(g, dst, src, bytes);
        };
        need_ptr(rev_offsets, g->in_offsets(), nb, "rev_offsets");
        need_ptr(rev_srcs, g->in_srcs(), mb, "rev_srcs");
        if (rev_eid && !g->rev_eid.get()) build_rev_eid_symmetric(g);  // undirected: on demand
        need(rev_eid, g->rev_eid, mb, "rev_eid");
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int gdx_graph_set_stream(gdx_graph* g, void* stream) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope dg(g);
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        g->stream = stream ? static_cast<cudaStream_t>(stream) : g->own_stream;
    });
}

int gdx_graph_get_stream(gdx_graph* g, void** stream) {
    return guard_impl([&] {
        if (!g || !stream) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        *stream = g->stream;
    });
}

int gdx_profile_enable(gdx_graph* g, int enable) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        g->prof.enabled = enable != 0;
        if (g->relabel) g->relabel->h->prof.enabled = enable != 0;
    });
}

int gdx_profile_reset(gdx_graph* g) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope dg(g);
        relabel_leave(g);  // the renumbered graph's launches count as g's
        g->prof.drain();
        g->prof.totals.clear();
    });
}

int gdx_profile_read(gdx_graph* g, char* names, double* ms, int64_t* launches, int32_t cap,
                     int32_t* count) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope dg(g);
        relabel_leave(g);
        g->prof.drain();
        int32_t i = 0;
        for (auto& kv : g->prof.totals) {
            if (i < cap) {
                if (names) {
                    std::strncpy(names + 64 * i, kv.first.c_str(), 63);
                    names[64 * i + 63] = 0;
                }
                if (ms) ms[i] = kv.second.first;
                if (launches) launches[i] = kv.second.second;
            }
            ++i;
        }
        if (count) *count = i;
    });
}

}  // extern "C"

// The degree-ordered renumbering kept on g (relabel.cu), for callers that run
// the multi-GPU partitions on it (distributed.py): the renumbered graph, owned
// by g, or NULL when g is not renumbered for this algorithm.
extern "C" int gdx_graph_renumbered(gdx_graph* g, int32_t algo, gdx_graph** h_out, int32_t* newid_out) {
    return guard_impl([&] {
        if (!g || !h_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (algo != 0 && algo != 1) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: algo is 0 (PR) or 1 (SSSP)");
        *h_out = nullptr;
        GraphScope dg(g);
        const bool want = algo == 0 ? g->in_offsets() && g->in_srcs() && relabel_wanted(g)
                                    : g->dests.get() && graph_max_degree(g) > 64 &&
                                          relabel_wanted(g);
        Relabel* RP = want ? relabel_try(g, algo == 1, algo == 0) : nullptr;
        if (!RP) return;
        Relabel& R = *RP;
        if (newid_out)
            copy_out(g, newid_out, R.newid.get(), size_t(g->n) * sizeof(int32_t));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        *h_out = R.h;
    });
}

