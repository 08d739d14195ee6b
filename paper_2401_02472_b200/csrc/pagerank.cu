// pagerank.cu -- ComputePR (reference corpus/pr.sp:5-33) on sm_100a.
//
// The reference's GPU twin does three launches, three device syncs and four
// small copies per round: a single-address atomicAdd(double) for the dangling
// mass, a thread-per-vertex pull that re-reads the source's out-degree per
// in-edge, and a copy-back kernel (tests/golden/pr/cuda/pr_cuda.cu:117-212).
//
// Here one round is one merge-path gather over the reverse CSR:
//   * the (rows + in-edges) merge path is cut into fixed tiles of kTile items
//     (perfect load balance regardless of in-degree skew);
//   * a tile's rev_srcs are read coalesced and the precomputed
//     contrib[u] = rank[u] / outdeg(u) values gathered into shared memory with
//     kItems independent loads per thread;
//   * each thread reduces its merge-path segment; a block-wide reduce-by-key
//     scan stitches rows that cross threads; rows that cross tiles are summed
//     through a compact per-row slot array and finished by a tiny fixup
//     kernel;
//   * the epilogue is fused: new rank, |change| >= threshold vote, next
//     contrib, and the next round's dangling mass (one atomic per block);
//   * rounds are enqueued in batches without host syncs; a round whose
//     predecessor voted "settled" exits immediately on the device.
// Term-wise arithmetic matches pr.sp (contrib is the same f64 quotient the
// interpreter computes per in-edge); only the summation order differs.
#include <cub/cub.cuh>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

constexpr int kPrBlock = 256;
constexpr int kItems = 8;
constexpr int kTile = kPrBlock * kItems;  // merge-path items per tile

struct PrArgs {
    int32_t n;
    int32_t ntiles;
    int32_t nslots;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ rev_offsets;
    const int32_t* __restrict__ rev_srcs;
    const int32_t* __restrict__ tile_row;
    const int32_t* __restrict__ tile_edge;
    const int32_t* __restrict__ tile_first_slot;
    const int32_t* __restrict__ tile_carry_slot;
    const int32_t* __restrict__ slot_row;
    double* slot_acc;
    double* rank0;
    double* rank1;
    double* contrib0;
    double* contrib1;
    double* dangling;  // [3]
    int32_t* flags;
    double damping, threshold, base, nd;
    int32_t max_iter;
};

struct KV {
    int32_t key;
    double val;
};
struct KVOp {
    __device__ KV operator()(const KV& a, const KV& b) const {
        return b.key == a.key ? KV{b.key, a.val + b.val} : b;
    }
};

__device__ inline bool round_skipped(const PrArgs& a, int round) {
    return round > 0 && *reinterpret_cast<const volatile int32_t*>(&a.flags[round - 1]) == 0;
}

// pr.sp:17-30 for one vertex, given sum = sum over in-neighbours of contrib.
__device__ inline void pr_epilogue(const PrArgs& a, int round, int32_t v, double sum,
                                   double dang_in, const double* __restrict__ rank_in,
                                   double* __restrict__ rank_out, double* __restrict__ contrib_out,
                                   double& dang_local, int& unsettled) {
    const double total = dang_in / a.nd + sum;
    const double nr = a.base + a.damping * total;
    double change = nr - rank_in[v];
    if (change < 0.0) change = 0.0 - change;
    if (change >= a.threshold && round < a.max_iter) unsettled = 1;
    rank_out[v] = nr;
    const int32_t od = a.offsets[v + 1] - a.offsets[v];
    contrib_out[v] = od > 0 ? nr / double(od) : 0.0;
    if (od == 0) dang_local += nr;
}

__device__ inline void block_flush(const PrArgs& a, int round, double dang_local, int unsettled) {
    typedef cub::BlockReduce<double, kPrBlock> R;
    __shared__ typename R::TempStorage tmp;
    double tot = R(tmp).Sum(dang_local);
    int any = __syncthreads_or(unsettled);
    if (threadIdx.x == 0) {
        if (tot != 0.0) atomicAdd(&a.dangling[(round + 1) % 3], tot);
        if (any) atomicOr(&a.flags[round], 1);
    }
}

__global__ void __launch_bounds__(kPrBlock) k_pr_tiles(PrArgs a, int round) {
    if (round_skipped(a, round)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.dangling[(round + 2) % 3] = 0.0;
    const double dang_in = *reinterpret_cast<const volatile double*>(&a.dangling[round % 3]);
    const double* __restrict__ contrib = (round & 1) ? a.contrib1 : a.contrib0;
    const double* __restrict__ rank_in = (round & 1) ? a.rank1 : a.rank0;
    double* __restrict__ rank_out = (round & 1) ? a.rank0 : a.rank1;
    double* __restrict__ contrib_out = (round & 1) ? a.contrib0 : a.contrib1;

    __shared__ int32_t s_end[kTile + 1];
    __shared__ double s_val[kTile];
    __shared__ double s_sum[kTile];
    typedef cub::BlockScan<KV, kPrBlock> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;

    const int tid = threadIdx.x;
    double dang_local = 0.0;
    int unsettled = 0;
    for (int32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const int32_t row0 = a.tile_row[t], e0 = a.tile_edge[t];
        const int32_t nrows = a.tile_row[t + 1] - row0, nedges = a.tile_edge[t + 1] - e0;
        for (int i = tid; i <= nrows; i += kPrBlock) {
            const int32_t r = row0 + i;
            s_end[i] = r < a.n ? a.rev_offsets[r + 1] - e0 : INT32_MAX;
        }
        int32_t src[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int i = tid + k * kPrBlock;
            src[k] = i < nedges ? a.rev_srcs[e0 + i] : -1;
        }
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int i = tid + k * kPrBlock;
            if (src[k] >= 0) s_val[i] = __ldg(&contrib[src[k]]);
        }
        __syncthreads();

        // merge-path coordinate of this thread's first item
        const int tile_items = nrows + nedges;
        const int diag = min(tid * kItems, tile_items);
        const int diag_end = min(diag + kItems, tile_items);
        int lo = max(diag - nedges, 0), hi = min(diag, nrows);
        while (lo < hi) {
            const int p = (lo + hi) >> 1;
            if (s_end[p] <= diag - p - 1)
                lo = p + 1;
            else
                hi = p;
        }
        int x = lo, y = diag - lo;
        const int start_row = x;
        bool completed = false;
        double run = 0.0;
        for (int it = diag; it < diag_end; ++it) {
            if (y < s_end[x]) {
                run += s_val[y];
                ++y;
            } else {
                s_sum[x] = run;
                run = 0.0;
                ++x;
                completed = true;
            }
        }
        KV carry{x, run}, prefix, agg;
        Scan(scan_tmp).ExclusiveScan(carry, prefix, KVOp(), agg);
        if (tid > 0 && completed && prefix.key == start_row) s_sum[start_row] += prefix.val;
        __syncthreads();

        const int32_t fslot = a.tile_first_slot[t];
        for (int i = tid; i < nrows; i += kPrBlock) {
            const double sum = s_sum[i];
            if (i == 0 && fslot >= 0) {
                atomicAdd(&a.slot_acc[fslot], sum);  // row began in an earlier tile
                continue;
            }
            pr_epilogue(a, round, row0 + i, sum, dang_in, rank_in, rank_out, contrib_out,
                        dang_local, unsettled);
        }
        if (tid == 0) {
            const int32_t cs = a.tile_carry_slot[t];
            if (cs >= 0) atomicAdd(&a.slot_acc[cs], agg.val);  // row continues in the next tile
        }
        __syncthreads();
    }
    block_flush(a, round, dang_local, unsettled);
}

// Rows that cross a tile boundary: their partial sums arrived via slot_acc.
__global__ void __launch_bounds__(kPrBlock) k_pr_fixup(PrArgs a, int round) {
    if (round_skipped(a, round)) return;
    const double dang_in = *reinterpret_cast<const volatile double*>(&a.dangling[round % 3]);
    const double* __restrict__ rank_in = (round & 1) ? a.rank1 : a.rank0;
    double* __restrict__ rank_out = (round & 1) ? a.rank0 : a.rank1;
    double* __restrict__ contrib_out = (round & 1) ? a.contrib0 : a.contrib1;
    double dang_local = 0.0;
    int unsettled = 0;
    for (int32_t s = blockIdx.x * kPrBlock + threadIdx.x; s < a.nslots; s += gridDim.x * kPrBlock) {
        const double sum = a.slot_acc[s];
        a.slot_acc[s] = 0.0;
        pr_epilogue(a, round, a.slot_row[s], sum, dang_in, rank_in, rank_out, contrib_out,
                    dang_local, unsettled);
    }
    block_flush(a, round, dang_local, unsettled);
}

// pr.sp:9 -- rank = 1/numNodes; contrib and the round-0 dangling mass.
__global__ void __launch_bounds__(kPrBlock) k_pr_init(PrArgs a) {
    double dang_local = 0.0;
    const double r0 = 1.0 / a.nd;
    for (int64_t v = blockIdx.x * (int64_t)kPrBlock + threadIdx.x; v < a.n;
         v += (int64_t)gridDim.x * kPrBlock) {
        a.rank0[v] = r0;
        const int32_t od = a.offsets[v + 1] - a.offsets[v];
        a.contrib0[v] = od > 0 ? r0 / double(od) : 0.0;
        if (od == 0) dang_local += r0;
    }
    typedef cub::BlockReduce<double, kPrBlock> R;
    __shared__ typename R::TempStorage tmp;
    double tot = R(tmp).Sum(dang_local);
    if (threadIdx.x == 0 && tot != 0.0) atomicAdd(&a.dangling[0], tot);
}

// Merge-path coordinates of every tile boundary over (row ends, edge ids).
__global__ void k_pr_tile_coords(int32_t n, int32_t m, int32_t ntiles,
                                 const int32_t* __restrict__ rev_offsets, int32_t* tile_row,
                                 int32_t* tile_edge, uint8_t* spanning) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t total = int64_t(n) + m;
        const int64_t diag = t * kTile < total ? t * kTile : total;
        int64_t lo = diag - m > 0 ? diag - m : 0, hi = diag < n ? diag : n;
        while (lo < hi) {
            const int64_t p = (lo + hi) >> 1;
            if (rev_offsets[p + 1] <= diag - p - 1)
                lo = p + 1;
            else
                hi = p;
        }
        tile_row[t] = int32_t(lo);
        tile_edge[t] = int32_t(diag - lo);
        spanning[t] = t > 0 && t < ntiles && lo < n && (diag - lo) > rev_offsets[lo];
    }
}

static void build_plan(gdx_graph* g) {
    auto& P = *g->pr;
    cudaStream_t s = g->stream;
    const int32_t n = g->n, m = g->m;
    const int64_t total = int64_t(n) + m;
    const int64_t nt = (total + kTile - 1) / kTile;
    if (nt > INT32_MAX) fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph too large for one plan");
    P.ntiles = int32_t(nt);
    P.tile_row.alloc(nt + 1);
    P.tile_edge.alloc(nt + 1);
    DevBuf<uint8_t> span(nt + 1);
    k_pr_tile_coords<<<blocks_for(nt + 1, 256, g->num_sms * 8), 256, 0, s>>>(
        n, m, P.ntiles, g->rev_offsets.get(), P.tile_row.get(), P.tile_edge.get(), span.get());
    GDX_LAUNCH_CHECK();
    std::vector<int32_t> row(nt + 1);
    std::vector<uint8_t> sp(nt + 1);
    GDX_CUDA(cudaMemcpyAsync(row.data(), P.tile_row.get(), (nt + 1) * 4, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemcpyAsync(sp.data(), span.get(), nt + 1, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    // One slot per distinct row crossing >= 1 tile boundary.
    std::vector<int32_t> first(nt + 1, -1), carry(nt, -1), slot_row;
    int32_t last_row = -1;
    for (int64_t t = 0; t <= nt; ++t) {
        if (!sp[t]) continue;
        if (row[t] != last_row) {
            slot_row.push_back(row[t]);
            last_row = row[t];
        }
        first[t] = int32_t(slot_row.size()) - 1;
    }
    for (int64_t t = 0; t < nt; ++t) carry[t] = first[t + 1];
    P.nslots = int32_t(slot_row.size());
    P.tile_first_slot.alloc(nt + 1);
    P.tile_carry_slot.alloc(nt);
    P.slot_row.alloc(slot_row.size());
    P.slot_acc.alloc(slot_row.size());
    GDX_CUDA(cudaMemcpyAsync(P.tile_first_slot.get(), first.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, s));
    GDX_CUDA(cudaMemcpyAsync(P.tile_carry_slot.get(), carry.data(), nt * 4, cudaMemcpyHostToDevice, s));
    if (!slot_row.empty())
        GDX_CUDA(cudaMemcpyAsync(P.slot_row.get(), slot_row.data(), slot_row.size() * 4,
                                 cudaMemcpyHostToDevice, s));
    GDX_CUDA(cudaMemsetAsync(P.slot_acc.get(), 0, P.slot_acc.bytes(), s));
    for (int i = 0; i < 2; ++i) {
        P.rank[i].alloc(n);
        P.contrib[i].alloc(n);
    }
    P.dangling.alloc(3);
    int per_sm = 0;
    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_tiles, kPrBlock, 0));
    P.grid = std::max(1, per_sm) * g->num_sms;
    GDX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gdx

using namespace gdx;

extern "C" int gdx_pagerank(gdx_graph* g, double damping, double threshold, int32_t max_iter,
                            double* rank_out, int32_t* rounds_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !rank_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        // pr.sp:9 evaluates 1.0 / numNodes (interpreter.cpp:454-456 raises on 0).
        if (g->n == 0) fail(GDX_ERR_RUNTIME, "RuntimeError: division by zero");
        if (!g->rev_offsets.get() || !g->rev_srcs.get())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        DeviceGuard dg(g->device);
        cudaStream_t s = g->stream;
        if (!g->pr) {
            g->pr = std::make_unique<PrPlan>();
            build_plan(g);
        }
        auto& P = *g->pr;
        // fixedPoint rounds: at most max_iter+1 (pr.sp:25) and at most the
        // interpreter's cap 10n+100 (interpreter.cpp:977-986).
        const int64_t cap = 10 * int64_t(g->n) + 100;
        const int64_t want = max_iter >= 0 ? int64_t(max_iter) + 1 : 1;
        const int64_t limit = std::min(want, cap);
        if (P.flags_cap < limit) {
            P.flags.alloc(size_t(limit));
            P.flags_cap = int32_t(limit);
        }
        PrArgs a;
        a.n = g->n;
        a.ntiles = P.ntiles;
        a.nslots = P.nslots;
        a.offsets = g->offsets.get();
        a.rev_offsets = g->rev_offsets.get();
        a.rev_srcs = g->rev_srcs.get();
        a.tile_row = P.tile_row.get();
        a.tile_edge = P.tile_edge.get();
        a.tile_first_slot = P.tile_first_slot.get();
        a.tile_carry_slot = P.tile_carry_slot.get();
        a.slot_row = P.slot_row.get();
        a.slot_acc = P.slot_acc.get();
        a.rank0 = P.rank[0].get();
        a.rank1 = P.rank[1].get();
        a.contrib0 = P.contrib[0].get();
        a.contrib1 = P.contrib[1].get();
        a.dangling = P.dangling.get();
        a.flags = P.flags.get();
        a.damping = damping;
        a.threshold = threshold;
        a.nd = double(g->n);
        a.base = (1.0 - damping) / a.nd;
        a.max_iter = max_iter;

        GDX_CUDA(cudaMemsetAsync(P.flags.get(), 0, size_t(limit) * 4, s));
        GDX_CUDA(cudaMemsetAsync(P.dangling.get(), 0, 3 * sizeof(double), s));
        int launches = 0;
        timed_launch(g, "pr_init", [&] {
            k_pr_init<<<blocks_for(g->n, kPrBlock, g->num_sms * 8), kPrBlock, 0, s>>>(a);
        });
        ++launches;
        const int fix_grid = blocks_for(std::max(P.nslots, 1), kPrBlock, g->num_sms * 4);
        int32_t* hflags = reinterpret_cast<int32_t*>(g->pinned);
        int64_t r = 0, rounds = -1, batch = 4;
        while (rounds < 0) {
            const int64_t lim = std::min(r + batch, limit);
            for (int64_t rr = r; rr < lim; ++rr) {
                timed_launch(g, "pr_tiles", [&] {
                    k_pr_tiles<<<P.grid, kPrBlock, 0, s>>>(a, int(rr));
                });
                if (P.nslots > 0)
                    timed_launch(g, "pr_fixup", [&] {
                        k_pr_fixup<<<fix_grid, kPrBlock, 0, s>>>(a, int(rr));
                    });
                launches += 1 + (P.nslots > 0);
            }
            const int64_t cnt = lim - r;
            GDX_CUDA(cudaMemcpyAsync(hflags, P.flags.get() + r, cnt * 4, cudaMemcpyDeviceToHost, s));
            GDX_CUDA(cudaStreamSynchronize(s));
            for (int64_t i = 0; i < cnt; ++i)
                if (hflags[i] == 0) {
                    rounds = r + i + 1;
                    break;
                }
            if (rounds < 0 && lim >= limit) {
                if (limit < want)
                    fail(GDX_ERR_NON_TERMINATION, "NonTermination: fixedPoint exceeded " +
                                                      std::to_string(cap) +
                                                      " iterations without converging");
                rounds = limit;  // unreachable: round max_iter never votes
            }
            r = lim;
            batch = std::min<int64_t>(batch * 2, 32);
        }
        copy_out(g, rank_out, P.rank[rounds & 1].get(), size_t(g->n) * sizeof(double));
        GDX_CUDA(cudaStreamSynchronize(s));
        if (rounds_out) *rounds_out = int32_t(rounds);
        if (stats) {
            stats->rounds = int32_t(rounds);
            stats->launches = launches;
            stats->vertices_visited = int64_t(g->n) * rounds;
            stats->edges_visited = int64_t(g->m) * rounds;
            stats->updates = 0;
            // per round rev_srcs 4m + contrib gather 8m +
            // rev_offsets 4n + offsets 4n + rank in 8n + rank out 8n + contrib out 8n.
            stats->algorithmic_bytes = double(rounds) * (12.0 * g->m + 32.0 * g->n);
        }
    });
}
