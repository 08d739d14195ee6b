// refstream.cu -- the reference's sequential random streams, on the host side
// of libgdx.
//
// The reference defines its generated graphs and weights by one std::mt19937_64
// stream consumed in a fixed order (graphgen.cpp:8-56, csr.cpp:172-195,
// graphdsl.cpp:265-296).  That order is inherently sequential, so it cannot be
// reproduced by a parallel generator; libgdx keeps it here (compiled with the
// same libstdc++ distributions as the reference) so that a caller can feed
// exactly the reference's inputs to the device path: the parity configs (C1:
// genRmatEdges(2^18, 2^22) + withRandomWeights(1, 100)) and `graphdsl run
// --weight-min/--weight-max/--weight-seed`.  Bench-scale graphs above
// scale 22 use the counter-based device generators (build.cu) instead.
//
// Nothing here is on the compute path of the four algorithms.
#include <random>
#include <string>
#include <vector>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {
namespace {

// withRandomWeights (csr.cpp:172-195): directed graphs draw one weight per
// stored edge in CSR order; undirected graphs draw one per unordered pair,
// visiting (u, v) with u <= v in CSR order, and copy it to the mirror (v, u)
// found by binary search in the sorted row of v (CsrGraph::edgeIndex,
// csr.cpp:150-158).
void random_weights_host(int32_t n, int32_t m, bool directed, const int32_t* off,
                         const int32_t* dst, int32_t lo, int32_t hi, uint64_t seed, int32_t* w) {
    if (lo > hi) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: weight range is empty");
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int32_t> draw(lo, hi);
    if (directed) {
        for (int32_t e = 0; e < m; ++e) w[e] = draw(rng);
        return;
    }
    for (int32_t u = 0; u < n; ++u) {
        for (int32_t e = off[u]; e < off[u + 1]; ++e) {
            const int32_t v = dst[e];
            if (v < u) continue;
            const int32_t x = draw(rng);
            w[e] = x;
            if (v == u) continue;
            int32_t a = off[v], b = off[v + 1];  // first entry >= u in N(v)
            while (a < b) {
                const int32_t mid = a + (b - a) / 2;
                if (dst[mid] < u) a = mid + 1; else b = mid;
            }
            if (a < off[v + 1] && dst[a] == u) w[a] = x;
        }
    }
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" {

int gdx_gen_uniform_edges_ref(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u,
                              int32_t* v) {
    return guard_impl([&] {
        // graphgen.cpp:8-16
        if (nodes <= 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: node count must be positive");
        if (edges < 0 || (edges > 0 && (!u || !v)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad edge arrays");
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<int32_t> pick(0, nodes - 1);
        for (int64_t i = 0; i < edges; ++i) {
            u[i] = pick(rng);  // the reference's braced initialiser draws u, then v
            v[i] = pick(rng);
        }
    });
}

int gdx_gen_rmat_edges_ref(int32_t nodes, int64_t edges, uint64_t seed, double a, double b,
                           double c, double d, int32_t* u, int32_t* v) {
    return guard_impl([&] {
        // graphgen.cpp:18-56: one uniform draw per level picks a quadrant;
        // endpoints outside [0, nodes) are dropped and redrawn.
        if (nodes <= 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: node count must be positive");
        const double total = a + b + c + d;
        if (total <= 0)
            fail(GDX_ERR_INVALID_ARGUMENT,
                 "InvalidArgument: RMAT parameters must sum to a positive value");
        if (edges < 0 || (edges > 0 && (!u || !v)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad edge arrays");
        int levels = 0;
        while ((int64_t(1) << levels) < nodes) ++levels;
        if (levels == 0) levels = 1;
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        const double pa = a / total, pb = b / total, pc = c / total;
        int64_t k = 0;
        while (k < edges) {
            int32_t x = 0, y = 0;
            for (int l = 0; l < levels; ++l) {
                const double r = unit(rng);
                const int32_t half = int32_t(1) << (levels - 1 - l);
                if (r < pa) {
                } else if (r < pa + pb) {
                    y += half;
                } else if (r < pa + pb + pc) {
                    x += half;
                } else {
                    x += half;
                    y += half;
                }
            }
            if (x >= nodes || y >= nodes) continue;
            u[k] = x;
            v[k] = y;
            ++k;
        }
    });
}

int gdx_gen_edge_weights_ref(int64_t count, uint64_t seed, int32_t wmin, int32_t wmax,
                             int32_t* weights_out) {
    return guard_impl([&] {
        // graphdsl.cpp:281-287: gen-graph's per-edge weight column
        if (count < 0 || (count > 0 && !weights_out))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad weight array");
        if (wmin > wmax) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: weight range is empty");
        std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
        std::uniform_int_distribution<int> weight(wmin, wmax);
        for (int64_t i = 0; i < count; ++i) weights_out[i] = weight(rng);
    });
}

int gdx_random_weights_host(int32_t n, int32_t m, int32_t directed, const int32_t* offsets,
                            const int32_t* dests, int32_t lo, int32_t hi, uint64_t seed,
                            int32_t* weights_out) {
    return guard_impl([&] {
        if (n < 0 || m < 0 || !offsets || (m > 0 && (!dests || !weights_out)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad CSR arrays");
        random_weights_host(n, m, directed != 0, offsets, dests, lo, hi, seed, weights_out);
    });
}

int gdx_graph_set_random_weights(gdx_graph* g, int32_t lo, int32_t hi, uint64_t seed) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        if (lo > hi) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: weight range is empty");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        GraphScope sc(g);
        std::vector<int32_t> off(size_t(g->n) + 1), dst(size_t(g->m)), w(size_t(g->m));
        GDX_CUDA(cudaMemcpyAsync(off.data(), g->offsets.get(), off.size() * 4,
                                 cudaMemcpyDeviceToHost, g->stream));
        if (g->m)
            GDX_CUDA(cudaMemcpyAsync(dst.data(), g->dests.get(), dst.size() * 4,
                                     cudaMemcpyDeviceToHost, g->stream));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        random_weights_host(g->n, g->m, g->directed, off.data(), dst.data(), lo, hi, seed,
                            w.data());
        g->weights.ensure(size_t(g->m));
        if (g->m)
            GDX_CUDA(cudaMemcpyAsync(g->weights.get(), w.data(), w.size() * 4,
                                     cudaMemcpyHostToDevice, g->stream));
        g->weighted = true;
        finalize_graph(g);  // max weight (32/64-bit SSSP distances), negativity
    });
}

}  // extern "C"
