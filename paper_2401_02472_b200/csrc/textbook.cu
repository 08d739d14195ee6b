// textbook.cu -- the reference's textbook algorithms (core/src/oracles.cpp) as
// plain topology-driven device kernels, for `graphdsl check`
// (tools/graphdsl.cpp:175-256: run, then the oracle, then PASS/FAIL at the
// corpus tolerance).  They share nothing with the fast paths: one thread per
// vertex per round or level, a host round trip per round, no worklists, no
// plans -- an independent second computation of each result on the device,
// sized for check-size graphs.
//
//   oracles::sssp  (oracles.cpp:10-31)   gdx_textbook_sssp: Bellman-Ford rounds
//                                        (the same unique distances Dijkstra gives)
//   oracles::bc    (oracles.cpp:33-71)   gdx_textbook_bc: level-synchronous Brandes
//                                        per source, children summed in adjacency order
//   oracles::pr    (oracles.cpp:73-92)   gdx_textbook_pr: maxIter Jacobi iterations,
//                                        stop when max |delta| < eps
//   oracles::tc    (oracles.cpp:94-111)  gdx_textbook_tc: u < v < w with (v,u), (v,w),
//                                        (u,w) edges -- by binary search, so without
//                                        the oracle's n <= 256 cubic-memory guard
#include <cstring>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {
namespace {

constexpr int64_t kInf64 = INT64_MAX / 2;

__device__ bool has_edge(const int32_t* off, const int32_t* dst, int32_t a, int32_t b) {
    int32_t lo = off[a], hi = off[a + 1];
    while (lo < hi) {
        const int32_t mid = lo + ((hi - lo) >> 1);
        const int32_t x = dst[mid];
        if (x == b) return true;
        if (x < b) lo = mid + 1; else hi = mid;
    }
    return false;
}

__global__ void k_tb_sssp_init(int32_t n, int32_t src, long long* d) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        d[v] = v == src ? 0 : kInf64;
}

__global__ void k_tb_sssp_round(int32_t n, const int32_t* off, const int32_t* dst, const int32_t* w,
                                long long* d, int* changed) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const long long du = d[u];
        if (du >= kInf64) continue;
        for (int32_t e = off[u]; e < off[u + 1]; ++e) {
            const long long c = du + (w ? w[e] : 1);
            if (c < d[dst[e]] && c < atomicMin(&d[dst[e]], c)) *changed = 1;
        }
    }
}

__global__ void k_tb_tc(int32_t n, const int32_t* off, const int32_t* dst, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        for (int32_t i = off[v]; i < off[v + 1]; ++i) {
            const int32_t u = dst[i];
            if (u >= v) break;
            for (int32_t j = off[v + 1] - 1; j >= off[v]; --j) {
                const int32_t x = dst[j];
                if (x <= v) break;
                if (has_edge(off, dst, u, x)) ++c;
            }
        }
    if (c) atomicAdd(cnt, c);
}

__global__ void k_tb_pr_dangling(int32_t n, const int32_t* off, const double* rank, double* out) {
    double s = 0.0;  // one thread, ascending order (oracles.cpp:77-79)
    for (int32_t v = 0; v < n; ++v)
        if (off[v + 1] == off[v]) s += rank[v];
    *out = s;
}

__global__ void k_tb_pr_round(int32_t n, double damping, const int32_t* off, const int32_t* roff,
                              const int32_t* rsrc, const double* dangling, const double* rank,
                              double* next, unsigned long long* max_delta) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double sum = *dangling / n;
        for (int32_t e = roff[v]; e < roff[v + 1]; ++e) {
            const int32_t u = rsrc[e];
            sum += rank[u] / double(off[u + 1] - off[u]);
        }
        next[v] = (1.0 - damping) / n + damping * sum;
        const double dlt = fabs(next[v] - rank[v]);
        atomicMax(max_delta, (unsigned long long)__double_as_longlong(dlt));  // >= 0: ordered as bits
    }
}

__global__ void k_tb_bc_init(int32_t n, int32_t s, int32_t* level, double* sigma, double* delta) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        level[v] = v == s ? 0 : -1;
        sigma[v] = v == s ? 1.0 : 0.0;
        delta[v] = 0.0;
    }
}

// Level L -> L+1: claim undiscovered neighbours of level-L vertices.
__global__ void k_tb_bc_claim(int32_t n, int32_t L, const int32_t* off, const int32_t* dst,
                              int32_t* level, int* found) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        if (level[v] != L) continue;
        for (int32_t e = off[v]; e < off[v + 1]; ++e)
            if (atomicCAS(&level[dst[e]], -1, L + 1) == -1) *found = 1;
    }
}

// sigma(w) for level L+1: the level-L in-neighbours' sigma, in-adjacency order.
__global__ void k_tb_bc_sigma(int32_t n, int32_t L, const int32_t* off, const int32_t* dst,
                              const int32_t* level, double* sigma) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
         w += (int64_t)gridDim.x * blockDim.x) {
        if (level[w] != L + 1) continue;
        double s = 0.0;
        for (int32_t e = off[w]; e < off[w + 1]; ++e)
            if (level[dst[e]] == L) s += sigma[dst[e]];
        sigma[w] = s;
    }
}

// delta(w) for level L (oracles.cpp:60-67), then score(w) += delta(w), w != s.
__global__ void k_tb_bc_back(int32_t n, int32_t L, int32_t s, const int32_t* off, const int32_t* dst,
                             const int32_t* level, const double* sigma, double* delta, double* score) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
         w += (int64_t)gridDim.x * blockDim.x) {
        if (level[w] != L) continue;
        double d = 0.0;
        for (int32_t e = off[w]; e < off[w + 1]; ++e) {
            const int32_t x = dst[e];
            if (level[x] == L + 1 && sigma[x] > 0.0) d += (sigma[w] / sigma[x]) * (1.0 + delta[x]);
        }
        delta[w] = d;
        if (w != s) score[w] += d;
    }
}

int grid_of(const gdx_graph* g) { return blocks_for(g->n, 256, g->num_sms * 8); }

void host_flag(gdx_graph* g, int* dflag, int* out) {
    GDX_CUDA(cudaMemcpyAsync(out, dflag, sizeof(int), cudaMemcpyDeviceToHost, g->stream));
    GDX_CUDA(cudaStreamSynchronize(g->stream));
}

void need_forward(const gdx_graph* g) {
    if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
    if (!g->dests.get() && g->m > 0)
        fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
}

}  // namespace
}  // namespace gdx

using namespace gdx;

extern "C" {

int gdx_textbook_sssp(gdx_graph* g, int32_t src, int64_t* dist_out) {
    return guard_impl([&] {
        need_forward(g);
        if (!dist_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (src < 0 || src >= g->n) fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: sssp: source out of range");
        GraphScope sc(g);
        cudaStream_t s = g->stream;
        DevBuf<long long> d(size_t(g->n));
        DevBuf<int> changed(1);
        k_tb_sssp_init<<<grid_of(g), 256, 0, s>>>(g->n, src, d.get());
        for (int h = 1; h;) {
            GDX_CUDA(cudaMemsetAsync(changed.get(), 0, sizeof(int), s));
            k_tb_sssp_round<<<grid_of(g), 256, 0, s>>>(g->n, g->offsets.get(), g->dests.get(),
                                                        g->weighted ? g->weights.get() : nullptr,
                                                        d.get(), changed.get());
            GDX_LAUNCH_CHECK();
            host_flag(g, changed.get(), &h);
        }
        copy_out(g, dist_out, d.get(), size_t(g->n) * 8);
        GDX_CUDA(cudaStreamSynchronize(s));
    });
}

int gdx_textbook_pr(gdx_graph* g, double damping, double eps, int32_t max_iter, double* rank_out) {
    return guard_impl([&] {
        if (!g || !rank_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (!g->in_offsets() || !g->in_srcs())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        if (g->n == 0) return;
        GraphScope sc(g);
        cudaStream_t s = g->stream;
        const size_t n = size_t(g->n);
        std::vector<double> init(n, 1.0 / double(g->n));
        DevBuf<double> rank(n), next(n), dang(1);
        DevBuf<unsigned long long> md(1);
        GDX_CUDA(cudaMemcpyAsync(rank.get(), init.data(), n * 8, cudaMemcpyHostToDevice, s));
        for (int32_t it = 0; it < max_iter; ++it) {
            k_tb_pr_dangling<<<1, 1, 0, s>>>(g->n, g->offsets.get(), rank.get(), dang.get());
            GDX_CUDA(cudaMemsetAsync(md.get(), 0, 8, s));
            k_tb_pr_round<<<grid_of(g), 256, 0, s>>>(g->n, damping, g->offsets.get(),
                                                      g->in_offsets(), g->in_srcs(), dang.get(),
                                                      rank.get(), next.get(), md.get());
            GDX_LAUNCH_CHECK();
            std::swap(rank, next);
            unsigned long long h = 0;
            GDX_CUDA(cudaMemcpyAsync(&h, md.get(), 8, cudaMemcpyDeviceToHost, s));
            GDX_CUDA(cudaStreamSynchronize(s));
            double delta;
            std::memcpy(&delta, &h, 8);
            if (delta < eps) break;
        }
        copy_out(g, rank_out, rank.get(), n * 8);
        GDX_CUDA(cudaStreamSynchronize(s));
    });
}

int gdx_textbook_tc(gdx_graph* g, int64_t* count_out) {
    return guard_impl([&] {
        need_forward(g);
        if (!count_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        GraphScope sc(g);
        cudaStream_t s = g->stream;
        DevBuf<unsigned long long> c(1);
        GDX_CUDA(cudaMemsetAsync(c.get(), 0, 8, s));
        if (g->n > 0)
            k_tb_tc<<<grid_of(g), 256, 0, s>>>(g->n, g->offsets.get(), g->dests.get(), c.get());
        GDX_LAUNCH_CHECK();
        unsigned long long h = 0;
        GDX_CUDA(cudaMemcpyAsync(&h, c.get(), 8, cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        *count_out = int64_t(h);
    });
}

int gdx_textbook_bc(gdx_graph* g, const int32_t* sources, int32_t nsrc, double* bc_out) {
    return guard_impl([&] {
        need_forward(g);
        if (!bc_out || nsrc < 0 || (nsrc > 0 && !sources))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        for (int32_t i = 0; i < nsrc; ++i)
            if (sources[i] < 0 || sources[i] >= g->n)
                fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: bc: source out of range");
        if (g->n == 0) return;
        if (!g->in_offsets() || !g->in_srcs())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        GraphScope sc(g);
        cudaStream_t s = g->stream;
        const size_t n = size_t(g->n);
        DevBuf<int32_t> level(n);
        DevBuf<double> sigma(n), delta(n), score(n);
        DevBuf<int> found(1);
        GDX_CUDA(cudaMemsetAsync(score.get(), 0, n * 8, s));
        const int32_t *off = g->offsets.get(), *dst = g->dests.get();
        for (int32_t i = 0; i < nsrc; ++i) {  // sources in set order (oracles.cpp:36)
            const int32_t src = sources[i];
            k_tb_bc_init<<<grid_of(g), 256, 0, s>>>(g->n, src, level.get(), sigma.get(), delta.get());
            int32_t depth = 0;
            for (int h = 1; h; ++depth) {
                GDX_CUDA(cudaMemsetAsync(found.get(), 0, sizeof(int), s));
                k_tb_bc_claim<<<grid_of(g), 256, 0, s>>>(g->n, depth, off, dst, level.get(),
                                                          found.get());
                k_tb_bc_sigma<<<grid_of(g), 256, 0, s>>>(g->n, depth, g->in_offsets(),
                                                          g->in_srcs(), level.get(), sigma.get());
                GDX_LAUNCH_CHECK();
                host_flag(g, found.get(), &h);
            }
            for (int32_t L = depth; L >= 0; --L)
                k_tb_bc_back<<<grid_of(g), 256, 0, s>>>(g->n, L, src, off, dst, level.get(),
                                                         sigma.get(), delta.get(), score.get());
            GDX_LAUNCH_CHECK();
        }
        copy_out(g, bc_out, score.get(), n * 8);
        GDX_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
