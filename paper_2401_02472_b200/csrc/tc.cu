// tc.cu -- ComputeTC (reference corpus/tc.sp:6-18) on sm_100a.
//
// tc.sp counts, for every middle vertex v, the pairs u < v < w with u, w in
// N(v) and is_an_edge(u, w).  The reference GPU twin runs one thread per v
// doing d_lo x d_hi binary searches and one atomicAdd per triangle
// (tests/golden/tc/cuda/tc_cuda.cu:117-142).
//
// Here the work unit is the oriented edge (v, u), u < v, and the inner
// d_hi loop becomes one sorted-set intersection
//     |{w in N(v) : w > v}  ∩  {w in N(u) : w > v}|
// (identical count, directed or undirected, because adjacency lists are sorted
// and deduplicated, csr.hpp:24-26).  Warps take 32 consecutive middle vertices
// and split their concatenated edge lists across lanes (edge-balanced within
// the warp); each lane intersects with a linear merge, or with galloping
// binary searches when the two lists are very unequal (hub lists).  Counts are
// warp-reduced and added with one 64-bit atomic per warp.
#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

constexpr int kTcBlock = 256;

// first index in [lo, hi) with a[i] > x
__device__ inline int32_t upper_bound_dev(const int32_t* __restrict__ a, int32_t lo, int32_t hi,
                                          int32_t x) {
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (a[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// first index in [lo, hi) with a[i] >= x
__device__ inline int32_t lower_bound_dev(const int32_t* __restrict__ a, int32_t lo, int32_t hi,
                                          int32_t x) {
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (a[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ inline unsigned long long intersect(const int32_t* __restrict__ d, int32_t a, int32_t ae,
                                               int32_t b, int32_t be) {
    unsigned long long c = 0;
    int32_t la = ae - a, lb = be - b;
    if (la <= 0 || lb <= 0) return 0;
    if (la > 16 * lb || lb > 16 * la) {
        // iterate the short list, gallop in the long one
        if (la > lb) {
            int32_t t = a, te = ae;
            a = b, ae = be;
            b = t, be = te;
        }
        for (int32_t i = a; i < ae && b < be; ++i) {
            const int32_t x = d[i];
            b = lower_bound_dev(d, b, be, x);
            if (b < be && d[b] == x) {
                ++c;
                ++b;
            }
        }
        return c;
    }
    int32_t x = d[a], y = d[b];
    while (true) {
        if (x < y) {
            if (++a >= ae) break;
            x = d[a];
        } else if (y < x) {
            if (++b >= be) break;
            y = d[b];
        } else {
            ++c;
            if (++a >= ae || ++b >= be) break;
            x = d[a];
            y = d[b];
        }
    }
    return c;
}

__global__ void __launch_bounds__(kTcBlock) k_tc(int32_t v_begin, int32_t v_end,
                                                 const int32_t* __restrict__ offsets,
                                                 const int32_t* __restrict__ dests,
                                                 unsigned long long* acc) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (blockIdx.x * (int64_t)kTcBlock + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * (kTcBlock / 32);
    unsigned long long count = 0, scanned = 0;
    for (int64_t v0 = v_begin + gwarp * 32; v0 < v_end; v0 += nwarps * 32) {
        const int32_t v = int32_t(v0) + lane;
        const bool valid = v < v_end;
        const int32_t vb = valid ? offsets[v] : 0;
        const int32_t ve = valid ? offsets[v + 1] : 0;
        const int32_t len = ve - vb;
        const int32_t hs = valid ? upper_bound_dev(dests, vb, ve, v) : 0;  // first w > v
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(full, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(full, incl, 31);
        const int excl = incl - len;
        for (int j0 = 0; j0 < total; j0 += 32) {
            const int j = j0 + lane;
            int k = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                int c = k + step;
                int ex = __shfl_sync(full, excl, c & 31);
                if (c < 32 && ex <= j) k = c;
            }
            const int32_t ovb = __shfl_sync(full, vb, k);
            const int32_t ove = __shfl_sync(full, ve, k);
            const int32_t ohs = __shfl_sync(full, hs, k);
            const int32_t oex = __shfl_sync(full, excl, k);
            if (j < total) {
                const int32_t mid = int32_t(v0) + k;
                const int32_t e = ovb + (j - oex);
                const int32_t u = dests[e];
                if (u < mid && ohs < ove) {
                    const int32_t ub = offsets[u], ue = offsets[u + 1];
                    const int32_t bs = upper_bound_dev(dests, ub, ue, mid);
                    scanned += (ove - ohs) + (ue - bs);
                    count += intersect(dests, ohs, ove, bs, ue);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        count += __shfl_xor_sync(full, count, o);
        scanned += __shfl_xor_sync(full, scanned, o);
    }
    if (lane == 0) {
        if (count) atomicAdd(&acc[0], count);
        if (scanned) atomicAdd(&acc[1], scanned);
    }
}

static void run_tc(gdx_graph* g, int32_t v_begin, int32_t v_end, int64_t* count_out,
                   gdx_stats* stats) {
    if (!g->dests.get() && g->m > 0)
        fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
    DeviceGuard dg(g->device);
    cudaStream_t s = g->stream;
    if (!g->tc) g->tc = std::make_unique<TcPlan>();
    auto& P = *g->tc;
    P.acc.ensure(2);
    GDX_CUDA(cudaMemsetAsync(P.acc.get(), 0, 2 * sizeof(unsigned long long), s));
    v_begin = std::max(v_begin, 0);
    v_end = std::min(v_end, g->n);
    if (v_end > v_begin) {
        const int64_t groups = (int64_t(v_end) - v_begin + 31) / 32;
        const int grid = blocks_for(groups * 32, kTcBlock, g->num_sms * 16);
        timed_launch(g, "tc", [&] {
            k_tc<<<grid, kTcBlock, 0, s>>>(v_begin, v_end, g->offsets.get(), g->dests.get(),
                                           P.acc.get());
        });
    }
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, P.acc.get(), 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    *count_out = int64_t(h[0]);
    if (stats) {
        stats->rounds = 1;
        stats->launches = v_end > v_begin ? 1 : 0;
        stats->vertices_visited = int64_t(v_end) - v_begin;
        stats->edges_visited = int64_t(h[1]);
        stats->updates = int64_t(h[0]);
        // offsets 4(n+1) + adjacency scan 4m + 4 per
        // element of every intersected list.
        const double frac = g->n ? double(int64_t(v_end) - v_begin) / g->n : 0.0;
        stats->algorithmic_bytes = frac * (4.0 * (g->n + 1) + 4.0 * g->m) + 4.0 * double(h[1]);
    }
}

}  // namespace gdx

using namespace gdx;

extern "C" {

int gdx_tc(gdx_graph* g, int64_t* count_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !count_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        run_tc(g, 0, g->n, count_out, stats);
    });
}

int gdx_tc_range(gdx_graph* g, int32_t v_begin, int32_t v_end, int64_t* count_out,
                 gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !count_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        run_tc(g, v_begin, v_end, count_out, stats);
    });
}

}  // extern "C"
