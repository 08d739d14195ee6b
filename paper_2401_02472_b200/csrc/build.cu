// build.cu -- CSR construction on the GPU and the counter-based generators.
//
// gdx_graph_build_from_edges reproduces CsrGraph::buildFromEdges +
// buildReverse (reference core/src/csr.cpp:28-94) bit-for-bit:
//   * validation in input order: the first offending edge decides between
//     InvalidEdge (endpoint range, csr.cpp:31-35) and NegativeWeight (:36-39);
//   * undirected inputs are stored both ways, self loops once (:41-43);
//   * sort by (u, v); a duplicate (u, v) run keeps its minimum weight (:46-56);
//   * offsets by counting (:62-69); reverse CSR sorted by source within each
//     destination with rev_eid = forward edge index (:77-94).
// The sort is a CUB radix sort over packed (u << b | v) keys, b = bits(n-1).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

static int key_bits(int32_t n) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) < n) ++b;
    return b;
}

__global__ void k_validate(int64_t E, int32_t n, const int32_t* __restrict__ u,
                           const int32_t* __restrict__ v, const int32_t* __restrict__ w,
                           unsigned long long* first_bad /* [2]: range, weight */) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t a = u[i], b = v[i];
        if (a < 0 || a >= n || b < 0 || b >= n) atomicMin(&first_bad[0], (unsigned long long)i);
        if (w && w[i] < 0) atomicMin(&first_bad[1], (unsigned long long)i);
    }
}

// Writes packed keys (and weights); undirected graphs emit the mirror at
// E + i, self-loop mirrors become the sentinel 1 << (2b) which sorts last.
__global__ void k_emit_keys(int64_t E, bool directed, int b, const int32_t* __restrict__ u,
                            const int32_t* __restrict__ v, const int32_t* __restrict__ w,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const uint64_t sentinel = uint64_t(1) << (2 * b);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t a = uint32_t(u[i]), c = uint32_t(v[i]);
        int32_t wt = w ? w[i] : 1;
        keys[i] = (a << b) | c;
        if (vals) vals[i] = wt;
        if (!directed) {
            keys[E + i] = a == c ? sentinel : ((c << b) | a);
            if (vals) vals[E + i] = wt;
        }
    }
}

// Run heads of the sorted key array (excluding sentinels); for weighted
// graphs the head also takes the minimum weight of its run.
__global__ void k_heads(int64_t E2, uint64_t sentinel, const uint64_t* __restrict__ keys,
                        int32_t* __restrict__ vals, uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E2;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        bool head = k != sentinel && (i == 0 || keys[i - 1] != k);
        flag[i] = head;
        if (head && vals) {
            int32_t best = vals[i];
            for (int64_t j = i + 1; j < E2 && keys[j] == k; ++j) best = min(best, vals[j]);
            vals[i] = best;
        }
    }
}

// offsets[x] = first index whose row >= x (rows = keys >> b); x in [0, n].
__global__ void k_offsets_from_keys(int64_t m, int32_t n, int b, const uint64_t* __restrict__ keys,
                                    int32_t* __restrict__ offsets) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = i < m ? int64_t(keys[i] >> b) : int64_t(n);
        int64_t prev = i == 0 ? -1 : int64_t(keys[i - 1] >> b);
        for (int64_t x = prev + 1; x <= row; ++x) offsets[x] = int32_t(i);
    }
}

__global__ void k_low_bits(int64_t m, int b, const uint64_t* __restrict__ keys,
                           int32_t* __restrict__ out) {
    const uint64_t mask = (uint64_t(1) << b) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = int32_t(keys[i] & mask);
}

// Source vertex of every forward edge (binary search over offsets).
__device__ inline int32_t edge_source(const int32_t* __restrict__ offsets, int32_t n, int64_t e) {
    int32_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int32_t mid = lo + ((hi - lo + 1) >> 1);
        if (offsets[mid] <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

__global__ void k_reverse_keys(int64_t m, int32_t n, int b, const int32_t* __restrict__ offsets,
                               const int32_t* __restrict__ dests, uint64_t* __restrict__ keys,
                               int32_t* __restrict__ eid) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t src = uint32_t(edge_source(offsets, n, e));
        keys[e] = (uint64_t(uint32_t(dests[e])) << b) | src;
        eid[e] = int32_t(e);
    }
}

__global__ void k_hash_weights(int64_t m, int32_t n, bool directed, int32_t lo, uint32_t span,
                               uint64_t key, const int32_t* __restrict__ offsets,
                               const int32_t* __restrict__ dests, int32_t* __restrict__ w) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t p = uint32_t(edge_source(offsets, n, e)), q = uint32_t(dests[e]);
        if (!directed && q < p) {
            uint64_t t = p;
            p = q;
            q = t;
        }
        w[e] = lo + int32_t(ctr_bounded(ctr_hash(key, (p << 32) | q), span));
    }
}

struct CubTemp {
    DevBuf<uint8_t> buf;
    void* get(size_t bytes) {
        buf.ensure(bytes);
        return buf.get();
    }
};

template <class K, class V>
static void radix_sort_pairs(cudaStream_t s, CubTemp& tmp, K* kin, K* kout, V* vin, V* vout,
                             int64_t count, int end_bit) {
    size_t bytes = 0;
    GDX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, count, 0,
                                             end_bit, s));
    GDX_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, kin, kout, vin, vout, count,
                                             0, end_bit, s));
}

template <class K>
static void radix_sort_keys(cudaStream_t s, CubTemp& tmp, K* kin, K* kout, int64_t count,
                            int end_bit) {
    size_t bytes = 0;
    GDX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kin, kout, count, 0, end_bit, s));
    GDX_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(bytes), bytes, kin, kout, count, 0, end_bit, s));
}

static int grid_for(gdx_graph* g, int64_t items) { return blocks_for(items, 256, g->num_sms * 16); }

// Undirected graphs are stored symmetrically with sorted rows, so the reverse
// CSR equals the forward one; rev_eid[e] (row v, entry u) is the forward id of
// (u, v): offsets[u] + position of v in N(u).  One warp per row.
__global__ void k_rev_eid_symmetric(int32_t n, const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ dests, int32_t* rev_eid) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        for (int32_t e = offsets[v] + lane; e < offsets[v + 1]; e += 32) {
            const int32_t u = dests[e];
            int32_t lo = offsets[u], hi = offsets[u + 1];
            while (lo < hi) {
                const int32_t mid = lo + ((hi - lo) >> 1);
                if (dests[mid] < int32_t(v))
                    lo = mid + 1;
                else
                    hi = mid;
            }
            rev_eid[e] = lo;
        }
    }
}

// Reverse CSR: sort (dest << b | src) with the forward edge id as payload
// (directed graphs); undirected graphs copy the forward arrays.
void build_reverse_device(gdx_graph* g) {
    const int32_t n = g->n;
    const int64_t m = g->m;
    cudaStream_t s = g->stream;
    // undirected: the reverse CSR is the forward one (gdx_graph::in_offsets /
    // in_srcs); the mirror ids are built on demand (build_rev_eid_symmetric)
    if (!g->directed) return;
    g->rev_offsets.alloc(size_t(n) + 1);
    g->rev_srcs.alloc(m);
    g->rev_eid.alloc(m);
    if (m == 0) {
        GDX_CUDA(cudaMemsetAsync(g->rev_offsets.get(), 0, (size_t(n) + 1) * 4, s));
        return;
    }
    if (!g->dests.get()) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no forward adjacency");
    const int b = key_bits(n);
    DevBuf<uint64_t> k0(m), k1(m);
    DevBuf<int32_t> e0(m);
    CubTemp tmp;
    k_reverse_keys<<<grid_for(g, m), 256, 0, s>>>(m, n, b, g->offsets.get(), g->dests.get(),
                                                  k0.get(), e0.get());
    GDX_LAUNCH_CHECK();
    radix_sort_pairs(s, tmp, k0.get(), k1.get(), e0.get(), g->rev_eid.get(), m, 2 * b);
    k_offsets_from_keys<<<grid_for(g, m + 1), 256, 0, s>>>(m, n, b, k1.get(), g->rev_offsets.get());
    GDX_LAUNCH_CHECK();
    k_low_bits<<<grid_for(g, m), 256, 0, s>>>(m, b, k1.get(), g->rev_srcs.get());
    GDX_LAUNCH_CHECK();
    GDX_CUDA(cudaStreamSynchronize(s));  // temporaries die at scope exit
}

// rev_eid of an undirected graph (mirror edge ids), on demand.
void build_rev_eid_symmetric(gdx_graph* g) {
    if (g->directed || g->rev_eid.get()) return;
    g->rev_eid.alloc(size_t(g->m));
    if (g->m == 0) return;
    if (!g->dests.get()) fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
    k_rev_eid_symmetric<<<grid_for(g, int64_t(g->n) * 32), 256, 0, g->stream>>>(
        g->n, g->offsets.get(), g->dests.get(), g->rev_eid.get());
    GDX_LAUNCH_CHECK();
}

// Core builder from device-resident edge arrays.
static void build_from_device_edges(gdx_graph* g, int32_t n, int64_t E, const int32_t* du,
                                    const int32_t* dv, const int32_t* dw, bool directed,
                                    const int32_t* hu, const int32_t* hv, const int32_t* hw) {
    cudaStream_t s = g->stream;
    g->n = n;
    g->directed = directed;
    g->weighted = dw != nullptr;
    // Validation in input order (csr.cpp:29-40).
    if (E > 0) {
        DevBuf<unsigned long long> bad(2);
        GDX_CUDA(cudaMemsetAsync(bad.get(), 0xff, 2 * sizeof(unsigned long long), s));
        k_validate<<<grid_for(g, E), 256, 0, s>>>(E, n, du, dv, dw, bad.get());
        GDX_LAUNCH_CHECK();
        unsigned long long h[2];
        GDX_CUDA(cudaMemcpyAsync(h, bad.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        if (h[0] != ~0ull || h[1] != ~0ull) {
            unsigned long long i = h[0] < h[1] ? h[0] : h[1];
            int32_t ev[3] = {0, 0, 1};
            const int32_t* src[3] = {hu ? hu + i : du + i, hv ? hv + i : dv + i,
                                     dw ? (hw ? hw + i : dw + i) : nullptr};
            for (int k = 0; k < 3; ++k)
                if (src[k]) GDX_CUDA(cudaMemcpy(&ev[k], src[k], 4, cudaMemcpyDefault));
            if (h[0] <= h[1])
                fail(GDX_ERR_INVALID_ARGUMENT,
                     "InvalidEdge: endpoint (" + std::to_string(ev[0]) + ", " +
                         std::to_string(ev[1]) + ") out of range [0, " + std::to_string(n) + ")");
            fail(GDX_ERR_INVALID_ARGUMENT, "NegativeWeight: edge (" + std::to_string(ev[0]) + ", " +
                                               std::to_string(ev[1]) + ") has weight " +
                                               std::to_string(ev[2]));
        }
    }
    const int b = key_bits(n);
    const int64_t E2 = directed ? E : 2 * E;
    const uint64_t sentinel = uint64_t(1) << (2 * b);
    CubTemp tmp;
    int64_t m = 0;
    DevBuf<uint64_t> ka(E2), kb(E2);
    DevBuf<int32_t> va, vb;
    if (dw) {
        va.alloc(E2);
        vb.alloc(E2);
    }
    if (E2 > 0) {
        k_emit_keys<<<grid_for(g, E), 256, 0, s>>>(E, directed, b, du, dv, dw, ka.get(), va.get());
        GDX_LAUNCH_CHECK();
        if (dw)
            radix_sort_pairs(s, tmp, ka.get(), kb.get(), va.get(), vb.get(), E2, 2 * b + 1);
        else
            radix_sort_keys(s, tmp, ka.get(), kb.get(), E2, 2 * b + 1);
        DevBuf<uint8_t> flag(E2);
        k_heads<<<grid_for(g, E2), 256, 0, s>>>(E2, sentinel, kb.get(), dw ? vb.get() : nullptr,
                                               flag.get());
        GDX_LAUNCH_CHECK();
        DevBuf<int64_t> nsel(1);
        size_t bytes = 0;
        GDX_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, kb.get(), flag.get(), ka.get(),
                                            nsel.get(), E2, s));
        GDX_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, kb.get(), flag.get(), ka.get(),
                                            nsel.get(), E2, s));
        if (dw) {
            GDX_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, vb.get(), flag.get(), va.get(),
                                                nsel.get(), E2, s));
            GDX_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, vb.get(), flag.get(),
                                                va.get(), nsel.get(), E2, s));
        }
        GDX_CUDA(cudaMemcpyAsync(&m, nsel.get(), sizeof(m), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
    }
    if (m > INT32_MAX)
        fail(GDX_ERR_UNSUPPORTED, "Unsupported: " + std::to_string(m) +
                                      " stored edges exceed the int32 CsrGraph limit");
    g->m = int32_t(m);
    g->offsets.alloc(size_t(n) + 1);
    g->dests.alloc(m);
    if (dw) g->weights.alloc(m);
    if (m == 0) {
        GDX_CUDA(cudaMemsetAsync(g->offsets.get(), 0, (size_t(n) + 1) * 4, s));
    } else {
        k_offsets_from_keys<<<grid_for(g, m + 1), 256, 0, s>>>(m, n, b, ka.get(), g->offsets.get());
        GDX_LAUNCH_CHECK();
        k_low_bits<<<grid_for(g, m), 256, 0, s>>>(m, b, ka.get(), g->dests.get());
        GDX_LAUNCH_CHECK();
        if (dw) GDX_CUDA(cudaMemcpyAsync(g->weights.get(), va.get(), m * 4, cudaMemcpyDeviceToDevice, s));
    }
    // free the big temporaries before the reverse sort allocates its own
    GDX_CUDA(cudaStreamSynchronize(s));
    ka.release();
    kb.release();
    va.release();
    vb.release();
    tmp.buf.release();
    build_reverse_device(g);
    finalize_graph(g);
}

// ---- counter-based generators ---------------------------------------------

__global__ void k_gen_rmat(int64_t E, int32_t nodes, int levels, uint64_t key, double t1,
                           double t2, double t3, int32_t* __restrict__ u, int32_t* __restrict__ v,
                           int32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = 0, y = 0;
        bool ok = false;
        for (uint64_t att = 0; att < 1024 && !ok; ++att) {
            x = 0;
            y = 0;
            for (int l = 0; l < levels; ++l) {
                uint64_t ctr = (uint64_t(i) << 16) | (att << 6) | uint64_t(l);
                double r = ctr_unit(ctr_hash(key, ctr));
                int32_t half = 1 << (levels - 1 - l);
                if (r < t1) {
                } else if (r < t2) {
                    y += half;
                } else if (r < t3) {
                    x += half;
                } else {
                    x += half;
                    y += half;
                }
            }
            ok = x < nodes && y < nodes;
        }
        if (!ok) *bad = 1;
        u[i] = x;
        v[i] = y;
    }
}

__global__ void k_gen_uniform(int64_t E, uint32_t nodes, uint64_t key, int32_t* __restrict__ u,
                              int32_t* __restrict__ v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        u[i] = int32_t(ctr_bounded(ctr_hash(key, 2 * uint64_t(i)), nodes));
        v[i] = int32_t(ctr_bounded(ctr_hash(key, 2 * uint64_t(i) + 1), nodes));
    }
}

__global__ void k_grid_flags(int64_t total, uint64_t key, double keep, uint8_t* __restrict__ f) {
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
         id += (int64_t)gridDim.x * blockDim.x)
        f[id] = ctr_unit(ctr_hash(key, uint64_t(id))) < keep;
}

__global__ void k_grid_edges(int64_t k, int64_t S, const int64_t* __restrict__ ids,
                             int32_t* __restrict__ u, int32_t* __restrict__ v) {
    const int64_t H = S * (S - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t id = ids[i], a, b;
        if (id < H) {
            a = (id / (S - 1)) * S + id % (S - 1);
            b = a + 1;
        } else {
            int64_t j = id - H;
            a = (j / S) * S + j % S;
            b = a + S;
        }
        u[i] = int32_t(a);
        v[i] = int32_t(b);
    }
}

static void set_hash_weights(gdx_graph* g, int32_t lo, int32_t hi, uint64_t seed) {
    if (lo > hi) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: weight range is empty");
    if (lo < 0) fail(GDX_ERR_INVALID_ARGUMENT, "NegativeWeight: weight range below zero");
    g->weights.alloc(g->m);
    g->weighted = true;
    if (g->m > 0) {
        uint32_t span = uint32_t(int64_t(hi) - lo + 1);
        k_hash_weights<<<grid_for(g, g->m), 256, 0, g->stream>>>(
            g->m, g->n, g->directed, lo, span, stream_key(seed, kStreamWeight),
            g->offsets.get(), g->dests.get(), g->weights.get());
        GDX_LAUNCH_CHECK();
    }
    // The reverse arrays carry no weights; max_weight drives SSSP's dist width.
    finalize_graph(g);
}

}  // namespace gdx

using namespace gdx;

extern "C" {

int gdx_graph_build_from_edges(int32_t n, int64_t nedges, const int32_t* u, const int32_t* v,
                               const int32_t* w, int directed, int device, gdx_graph** out) {
    return guard_impl([&] {
        if (!out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null out");
        if (n < 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: negative node count");
        if (nedges < 0 || (nedges > 0 && (!u || !v)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad edge arrays");
        std::unique_ptr<gdx_graph> g(make_graph(device));
        GraphScope dg(g.get());
        cudaStream_t s = g->stream;
        // Stage host inputs on the device (device inputs are used in place).
        auto on_device = [](const void* p) {
            cudaPointerAttributes a;
            if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
        };
        DevBuf<int32_t> su, sv, sw;
        const int32_t *du = u, *dv = v, *dw = w;
        const int32_t *hu = nullptr, *hv = nullptr, *hw = nullptr;
        if (nedges > 0 && !on_device(u)) {
            su.alloc(nedges);
            sv.alloc(nedges);
            GDX_CUDA(cudaMemcpyAsync(su.get(), u, nedges * 4, cudaMemcpyDefault, s));
            GDX_CUDA(cudaMemcpyAsync(sv.get(), v, nedges * 4, cudaMemcpyDefault, s));
            du = su.get();
            dv = sv.get();
            hu = u;
            hv = v;
        }
        if (w && nedges > 0 && !on_device(w)) {
            sw.alloc(nedges);
            GDX_CUDA(cudaMemcpyAsync(sw.get(), w, nedges * 4, cudaMemcpyDefault, s));
            dw = sw.get();
            hw = w;
        }
        if (nedges == 0) dw = w ? dw : nullptr;
        build_from_device_edges(g.get(), n, nedges, du, dv, w ? dw : nullptr, directed != 0, hu, hv,
                                hw);
        if (w && nedges == 0) g->weighted = true;
        GDX_CUDA(cudaStreamSynchronize(s));
        *out = g.release();
    });
}

int gdx_graph_generate(const gdx_gen_params* p, int device, gdx_graph** out) {
    return guard_impl([&] {
        if (!p || !out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        std::unique_ptr<gdx_graph> g(make_graph(device));
        GraphScope dg(g.get());
        cudaStream_t s = g->stream;
        DevBuf<int32_t> u, v;
        int64_t E = 0;
        int32_t n = 0;
        if (p->kind == 0 || p->kind == 1) {
            if (p->nodes <= 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: node count must be positive");
            if (p->edges < 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: negative edge count");
            n = p->nodes;
            E = p->edges;
            u.alloc(E);
            v.alloc(E);
            if (p->kind == 0) {
                int levels = 0;
                while ((int64_t(1) << levels) < n) ++levels;
                if (levels == 0) levels = 1;
                DevBuf<int32_t> bad(1);
                GDX_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
                k_gen_rmat<<<grid_for(g.get(), E), 256, 0, s>>>(
                    E, n, levels, stream_key(p->seed, kStreamRmat), p->a, p->a + p->b,
                    p->a + p->b + p->c, u.get(), v.get(), bad.get());
                GDX_LAUNCH_CHECK();
                int32_t hb = 0;
                GDX_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
                GDX_CUDA(cudaStreamSynchronize(s));
                if (hb) fail(GDX_ERR_RUNTIME, "RuntimeError: rmat resampling exhausted");
            } else {
                k_gen_uniform<<<grid_for(g.get(), E), 256, 0, s>>>(
                    E, uint32_t(n), stream_key(p->seed, kStreamUniform), u.get(), v.get());
                GDX_LAUNCH_CHECK();
            }
        } else if (p->kind == 2) {
            const int64_t S = p->nodes;
            if (S <= 1 || S * S > INT32_MAX)
                fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: grid side out of range");
            n = int32_t(S * S);
            const int64_t total = 2 * S * (S - 1);
            DevBuf<uint8_t> f(total);
            k_grid_flags<<<grid_for(g.get(), total), 256, 0, s>>>(
                total, stream_key(p->seed, kStreamGrid), p->keep, f.get());
            GDX_LAUNCH_CHECK();
            DevBuf<int64_t> ids(total), nsel(1);
            CubTemp tmp;
            size_t bytes = 0;
            thrust::counting_iterator<int64_t> it(0);
            GDX_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, f.get(), ids.get(), nsel.get(),
                                                total, s));
            GDX_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, it, f.get(), ids.get(),
                                                nsel.get(), total, s));
            GDX_CUDA(cudaMemcpyAsync(&E, nsel.get(), 8, cudaMemcpyDeviceToHost, s));
            GDX_CUDA(cudaStreamSynchronize(s));
            u.alloc(E);
            v.alloc(E);
            if (E > 0) {
                k_grid_edges<<<grid_for(g.get(), E), 256, 0, s>>>(E, S, ids.get(), u.get(), v.get());
                GDX_LAUNCH_CHECK();
            }
        } else {
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: unknown generator kind");
        }
        build_from_device_edges(g.get(), n, E, u.get(), v.get(), nullptr, p->directed != 0,
                                nullptr, nullptr, nullptr);
        u.release();
        v.release();
        if (p->whi >= p->wlo) set_hash_weights(g.get(), p->wlo, p->whi, p->seed);
        GDX_CUDA(cudaStreamSynchronize(s));
        *out = g.release();
    });
}

int gdx_graph_set_hash_weights(gdx_graph* g, int32_t lo, int32_t hi, uint64_t seed) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        GraphScope dg(g);
        set_hash_weights(g, lo, hi, seed);
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    });
}

}  // extern "C"
