// pagerank.cu -- ComputePR (reference corpus/pr.sp:5-33) on sm_100a.
//
// The reference's GPU twin does three launches, three device syncs and four
// small copies per round: a single-address atomicAdd(double) for the dangling
// mass, a thread-per-vertex pull that re-reads the source's out-degree per
// in-edge, and a copy-back kernel (tests/golden/pr/cuda/pr_cuda.cu:117-212).
//
// Here one round is one merge-path gather over the reverse CSR (k_pr_gather):
//   * the (rows + in-edges) merge path is cut into fixed tiles of BLOCK * ITEMS
//     items -- perfect load balance regardless of the in-degree skew
//     (RMAT-24: 56% of rows empty, max in-degree 238,735);
//   * per tile the row ends and rev_srcs are staged in shared memory with
//     coalesced loads; each thread gathers the precomputed
//     contrib[u] = rank[u] / outdeg(u) of its own segment into registers
//     (ITEMS independent loads) and reduces it row by row;
//   * a reduce-by-key scan carries partial sums across threads, the fused
//     epilogue finishes the tile's rows in order (new rank, |change| >=
//     threshold vote, next contrib, next round's dangling mass), and rows
//     crossing tiles are summed through a compact slot array and finished by
//     k_pr_fixup;
//   * rounds are enqueued in batches without host syncs; a round whose
//     predecessor voted "settled" exits immediately on the device.
// Term-wise arithmetic matches pr.sp (contrib is the same f64 quotient the
// interpreter computes per in-edge); only the summation order differs.
#include <cub/cub.cuh>

#include <cstdlib>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

constexpr int kPrBlock = 256;

struct PrArgs {
    int32_t n;
    int32_t ntiles;
    int32_t nslots;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ rev_offsets;
    const int32_t* __restrict__ rev_srcs;
    const int2* __restrict__ tile_coord;  // (row, edge) merge-path coordinate per tile boundary
    const int2* __restrict__ tile_slots;  // (first-row slot, carry slot) per tile, -1 = none
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

template <int BLOCK = kPrBlock>
__device__ inline void block_flush(const PrArgs& a, int round, double dang_local, int unsettled) {
    typedef cub::BlockReduce<double, BLOCK> R;
    __shared__ typename R::TempStorage tmp;
    double tot = R(tmp).Sum(dang_local);
    int any = __syncthreads_or(unsettled);
    if (threadIdx.x == 0) {
        if (tot != 0.0) atomicAdd(&a.dangling[(round + 1) % 3], tot);
        if (any) atomicOr(&a.flags[round], 1);
    }
}

struct KV {
    int32_t key;
    double val;
};
struct KVOp {
    __device__ KV operator()(const KV& a, const KV& b) const {
        return b.key == a.key ? KV{b.key, a.val + b.val} : b;
    }
};

// One PageRank round over tiles of BLOCK * ITEMS merge-path items.  Per tile:
// row ends and rev_srcs are staged in shared memory (coalesced); each thread
// locates its merge-path segment, gathers exactly the contrib values of its
// segment's in-edges into registers (ITEMS independent loads) and reduces them
// row by row into shared row sums; a block scan carries partial sums across
// threads; the epilogue then finishes the tile's rows in order (coalesced).
// Rows crossing tile boundaries go through slot_acc and k_pr_fixup.  Measured
// on B200 (RMAT-24): one-warp blocks with 6 items/thread are fastest -- the
// kernel is latency bound and small blocks never wait on a slow warp.
template <int BLOCK, int ITEMS, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_pr_gather(PrArgs a, int round) {
    constexpr int TILE = BLOCK * ITEMS;
    typedef cub::BlockScan<KV, BLOCK, cub::BLOCK_SCAN_RAKING> Scan;
    if (round_skipped(a, round)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.dangling[(round + 2) % 3] = 0.0;
    const double dang_in = *reinterpret_cast<const volatile double*>(&a.dangling[round % 3]);
    const double* __restrict__ contrib = (round & 1) ? a.contrib1 : a.contrib0;
    const double* __restrict__ rank_in = (round & 1) ? a.rank1 : a.rank0;
    double* __restrict__ rank_out = (round & 1) ? a.rank0 : a.rank1;
    double* __restrict__ contrib_out = (round & 1) ? a.contrib0 : a.contrib1;

    __shared__ int32_t s_end[TILE + 1];
    __shared__ int32_t s_src[TILE];
    __shared__ double s_sum[TILE];
    __shared__ typename Scan::TempStorage scan_tmp;
    const int tid = threadIdx.x;
    double dang_local = 0.0;
    int unsettled = 0;
    int32_t t = blockIdx.x;
    int2 c0 = make_int2(0, 0), c1 = c0, n0 = c0, n1 = c0;
    if (t < a.ntiles) {
        c0 = a.tile_coord[t];
        c1 = a.tile_coord[t + 1];
    }
    for (; t < a.ntiles; t += gridDim.x) {
        const int32_t tn = t + gridDim.x;
        if (tn < a.ntiles) {  // prefetch the next tile's coordinates
            n0 = a.tile_coord[tn];
            n1 = a.tile_coord[tn + 1];
        }
        const int2 slots = a.tile_slots[t];
        const int32_t row0 = c0.x, e0 = c0.y;
        const int nrows = c1.x - row0, nedges = c1.y - e0;
        for (int i = tid; i <= nrows; i += BLOCK) {
            const int32_t r = row0 + i;
            s_end[i] = r < a.n ? a.rev_offsets[r + 1] - e0 : INT32_MAX;
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int i = tid + k * BLOCK;
            if (i < nedges) s_src[i] = a.rev_srcs[e0 + i];
        }
        __syncthreads();
        const int tile_items = nrows + nedges;
        auto search = [&](int diag) {
            int lo = max(diag - nedges, 0), hi = min(diag, nrows);
            while (lo < hi) {
                const int p = (lo + hi) >> 1;
                if (s_end[p] <= diag - p - 1)
                    lo = p + 1;
                else
                    hi = p;
            }
            return lo;
        };
        const int diag = min(tid * ITEMS, tile_items);
        const int diag_end = min(diag + ITEMS, tile_items);
        const int xs = search(diag), xe = search(diag_end);
        const int ys = diag - xs, ye = diag_end - xe;
        double v[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
            v[k] = ys + k < ye ? __ldg(&contrib[s_src[ys + k]]) : 0.0;
        int x = xs;
        int cur_end = s_end[x];
        bool completed = false;
        double run = 0.0;
        auto complete = [&]() {
            s_sum[x] = run;
            completed = true;
            run = 0.0;
            ++x;
            cur_end = s_end[x];
        };
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (ys + k < ye) {
                while (cur_end <= ys + k) complete();
                run += v[k];
            }
        }
        while (x < xe) complete();
        KV carry{x, run}, prefix, agg;
        Scan(scan_tmp).ExclusiveScan(carry, prefix, KVOp(), agg);
        if (completed && tid > 0 && prefix.key == xs) s_sum[xs] += prefix.val;
        __syncthreads();
        // coalesced epilogue over the tile's completed rows
        for (int i = tid; i < nrows; i += BLOCK) {
            const double sum = s_sum[i];
            if (i == 0 && slots.x >= 0)
                atomicAdd(&a.slot_acc[slots.x], sum);  // row began in an earlier tile
            else
                pr_epilogue(a, round, row0 + i, sum, dang_in, rank_in, rank_out, contrib_out,
                            dang_local, unsettled);
        }
        if (tid == 0 && slots.y >= 0) atomicAdd(&a.slot_acc[slots.y], agg.val);
        c0 = n0;
        c1 = n1;
        __syncthreads();
    }
    block_flush<BLOCK>(a, round, dang_local, unsettled);
}

// Tile shapes (block threads x items per thread); GDX_PR_VARIANT selects one
// for A/B runs (tools/pr_variants.py), 40 is the default.
struct PrVariant {
    int id, block, items;
    void* fn;
};
static const PrVariant kPrVariants[] = {
    {40, 32, 6, (void*)k_pr_gather<32, 6, 32>},  // default: one warp per block, 192-item tiles
    {41, 32, 8, (void*)k_pr_gather<32, 8, 32>},
    {43, 32, 4, (void*)k_pr_gather<32, 4, 32>},
    {44, 128, 6, (void*)k_pr_gather<128, 6, 8>},
};
static const PrVariant& pr_variant(int id) {
    for (const auto& v : kPrVariants)
        if (v.id == id) return v;
    return kPrVariants[0];
}
static int pr_variant_tile(int id) {
    const PrVariant& v = pr_variant(id);
    return v.block * v.items;
}
static void k_pr_dispatch(int id, int grid, int block, cudaStream_t s, PrArgs& a, int round) {
    void* args[] = {&a, &round};
    GDX_CUDA(cudaLaunchKernel(pr_variant(id).fn, dim3(grid), dim3(block), args, 0, s));
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
__global__ void k_pr_tile_coords(int32_t n, int32_t m, int32_t ntiles, int32_t tile,
                                 const int32_t* __restrict__ rev_offsets, int2* coord,
                                 uint8_t* spanning) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t total = int64_t(n) + m;
        const int64_t diag = t * tile < total ? t * tile : total;
        int64_t lo = diag - m > 0 ? diag - m : 0, hi = diag < n ? diag : n;
        while (lo < hi) {
            const int64_t p = (lo + hi) >> 1;
            if (rev_offsets[p + 1] <= diag - p - 1)
                lo = p + 1;
            else
                hi = p;
        }
        coord[t] = make_int2(int32_t(lo), int32_t(diag - lo));
        spanning[t] = t > 0 && t < ntiles && lo < n && (diag - lo) > rev_offsets[lo];
    }
}

static void build_plan(gdx_graph* g) {
    auto& P = *g->pr;
    cudaStream_t s = g->stream;
    const int32_t n = g->n, m = g->m;
    const int64_t total = int64_t(n) + m;
    const char* var = std::getenv("GDX_PR_VARIANT");
    P.variant = var ? std::atoi(var) : 40;  // see kPrVariants
    P.tile = pr_variant_tile(P.variant);
    const int64_t nt = (total + P.tile - 1) / P.tile;
    if (nt > INT32_MAX) fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph too large for one plan");
    P.ntiles = int32_t(nt);
    P.tile_coord.alloc(nt + 1);
    DevBuf<uint8_t> span(nt + 1);
    k_pr_tile_coords<<<blocks_for(nt + 1, 256, g->num_sms * 8), 256, 0, s>>>(
        n, m, P.ntiles, P.tile, g->rev_offsets.get(), P.tile_coord.get(), span.get());
    GDX_LAUNCH_CHECK();
    std::vector<int2> coord(nt + 1);
    std::vector<uint8_t> sp(nt + 1);
    GDX_CUDA(cudaMemcpyAsync(coord.data(), P.tile_coord.get(), (nt + 1) * sizeof(int2),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemcpyAsync(sp.data(), span.get(), nt + 1, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    // One slot per distinct row crossing >= 1 tile boundary.  Tile t adds its
    // first row's partial to slot .x when that row began in an earlier tile,
    // and its trailing partial row to slot .y when the row continues.
    std::vector<int32_t> first(nt + 1, -1), slot_row;
    int32_t last_row = -1;
    for (int64_t t = 0; t <= nt; ++t) {
        if (!sp[t]) continue;
        if (coord[t].x != last_row) {
            slot_row.push_back(coord[t].x);
            last_row = coord[t].x;
        }
        first[t] = int32_t(slot_row.size()) - 1;
    }
    std::vector<int2> slots(nt);
    for (int64_t t = 0; t < nt; ++t) slots[t] = make_int2(first[t], first[t + 1]);
    P.nslots = int32_t(slot_row.size());
    P.tile_slots.alloc(nt);
    P.slot_row.alloc(slot_row.size());
    P.slot_acc.alloc(slot_row.size());
    GDX_CUDA(cudaMemcpyAsync(P.tile_slots.get(), slots.data(), nt * sizeof(int2),
                             cudaMemcpyHostToDevice, s));
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
    const PrVariant& V = pr_variant(P.variant);
    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, V.fn, V.block, 0));
    P.block = V.block;
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
        a.tile_coord = P.tile_coord.get();
        a.tile_slots = P.tile_slots.get();
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
                    k_pr_dispatch(P.variant, P.grid, P.block, s, a, int(rr));
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
