// sssp.cu -- ComputeSSSP (reference corpus/sssp.sp:6-20) on sm_100a.
//
// The reference runs a topology-driven fixedPoint: every round scans all V
// vertices, relaxes the out-edges of `modified` ones with atomicMin and does a
// host round trip for the `finished` flag (tests/golden/sssp/cuda/
// sssp_cuda.cu:117-199; interpreter.cpp:968-1000).
//
// Default execution (gdx_sssp): frontier-scan rounds, looped on the device by
// a CUDA graph with a conditional WHILE node (no host round trip per round):
//   * k_sssp_scan_frontier: vertices whose distance dropped since they were
//     last expanded (dist < prev; prev := dist) emit relaxation items of <= 64
//     out-edges (hubs are split), one global atomic per 2048-vertex chunk;
//   * k_sssp_scan_relax: 16 lanes per item, each lane's 4 edges loaded
//     together (dests/weights, then the dist[u] gathers, then the atomicMin of
//     the improving ones);
//   * k_sssp_graph_finish: counts the round, clears the counters and keeps
//     the loop going while the scan produced work.
// The same kernels serve the multi-GPU shards (gdx_sssp_shard_*, int64
// replicas).  The earlier persistent cooperative kernel (k_sssp_rounds:
// worklist + grid.sync per round) and a host-driven loop remain selectable
// with GDX_SSSP_MODE=persistent|scan for A/B runs.
// Distances are 32-bit; a relaxation that would overflow them sets a flag and
// the call reruns with 64-bit distances (exact either way); the result is
// widened to int64 with INF = INT64_MAX/2 (oracles.hpp:12).  Any correct
// relaxation order yields the unique shortest-path distances, so the output is
// bit-identical to oracles::sssp and to interp::run.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace cg = cooperative_groups;

namespace gdx {

constexpr int kSsspBlock = 256;
constexpr int kChunk = 32;  // max edges per work item
constexpr int kSsspQueue = 2048;  // block-local next-frontier staging (int2 items)

// Counter layout in SsspWork::ctrs.
enum { kQ = 0, kWork = 3, kRounds = 6, kVvis = 7, kEvis = 8, kUpd = 9, kOvf = 10, kCtrs = 16 };
constexpr int kWarpChunk = 256;  // queue items a warp reserves once its block's staging is full

template <class D>
struct SsspArgs {
    int32_t n;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ dests;
    const int32_t* __restrict__ weights;  // nullptr => 1
    D* dist;
    int32_t* stamp;
    int2* q0;
    int2* q1;
    unsigned long long* ctr;
    unsigned long long* trace;  // optional per-round (queue size, globaltimer ns)
    int stage_cap;              // block staging capacity (<= kSsspQueue; 0 in tests)
};

__device__ inline unsigned long long ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

template <class D>
__global__ void k_sssp_init(SsspArgs<D> a, int32_t src, D inf) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        a.dist[i] = i == src ? D(0) : inf;
        a.stamp[i] = 0;
    }
    if (blockIdx.x == 0) {
        int32_t b = a.offsets[src], e = a.offsets[src + 1];
        int32_t items = (e - b + kChunk - 1) / kChunk;
        for (int32_t t = threadIdx.x; t < items; t += blockDim.x) a.q0[t] = make_int2(src, b + t * kChunk);
        if (threadIdx.x == 0) a.ctr[kQ + 0] = items;
    }
}

template <class D, int kIlp, bool kPre>
__global__ void __launch_bounds__(kSsspBlock) k_sssp_rounds(SsspArgs<D> a) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const long long nwarps = (long long)gridDim.x * (kSsspBlock / 32);
    const long long gwarp = ((long long)blockIdx.x * kSsspBlock + threadIdx.x) >> 5;
    __shared__ int2 s_q[kSsspQueue];
    __shared__ int s_qn;
    __shared__ unsigned long long s_gpos;
    unsigned long long vvis = 0, evis = 0, upd = 0;
    unsigned long long wq_base = 0;  // this warp's overflow chunk in the next queue
    int wq_left = 0;
    int r = 0;
    for (;; ++r) {
        const int cur = r % 3, nxt = (r + 1) % 3, clr = (r + 2) % 3;
        const int2* Q = (r & 1) ? a.q1 : a.q0;
        int2* QN = (r & 1) ? a.q0 : a.q1;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.ctr[kQ + clr] = 0;
            a.ctr[kWork + clr] = 0;
        }
        const unsigned long long qn = ld_volatile(&a.ctr[kQ + cur]);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && r < 256) {
            unsigned long long t;
            t = clock64();
            a.trace[2 * r] = qn;
            a.trace[2 * r + 1] = t;
        }
        // Static split of the worklist over warps (no shared work counter: a
        // single contended atomic per grab serialises at one L2 address).
        const unsigned long long per = (qn + nwarps - 1) / nwarps;
        const unsigned long long w0 = gwarp * per, w1 = min(qn, w0 + per);
        if (threadIdx.x == 0) s_qn = 0;
        __syncthreads();
        for (unsigned long long base = w0; base < w1; base += 32) {
            const int cnt = int(min(32ull, w1 - base));
            int v = 0, b = 0, len = 0;
            D dv = 0;
            if (lane < cnt) {
                int2 it = Q[base + lane];
                v = it.x;
                b = it.y;
                if (v >= 0) {  // v < 0: padding of a partly used warp chunk
                    int32_t vb = a.offsets[v], ve = a.offsets[v + 1];
                    int32_t e = min(b + kChunk, ve);
                    len = e - b;
                    dv = a.dist[v];
                    vvis += (b == vb);
                }
            }
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(full, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(full, incl, 31);
            const int excl = incl - len;
            evis += len;
            for (int j0 = 0; j0 < total; j0 += 32 * kIlp) {
                // kIlp edges per lane, every load of the group issued together
                int nbr[kIlp];
                D cand[kIlp], cur_d[kIlp];
#pragma unroll
                for (int k = 0; k < kIlp; ++k) {
                    const int j = j0 + 32 * k + lane;
                    int o = 0;  // owner = largest lane with excl <= j
#pragma unroll
                    for (int step = 16; step; step >>= 1) {
                        int c = o + step;
                        int ex = __shfl_sync(full, excl, c & 31);
                        if (c < 32 && ex <= j) o = c;
                    }
                    const int ob = __shfl_sync(full, b, o);
                    const int oex = __shfl_sync(full, excl, o);
                    const D od = __shfl_sync(full, dv, o);
                    const int e = ob + (j - oex);
                    nbr[k] = j < total ? a.dests[e] : -1;
                    const D wt = j < total ? (a.weights ? D(a.weights[e]) : D(1)) : D(0);
                    cand[k] = od + wt;
                    if (sizeof(D) == 4 && j < total && od > D(0xFFFFFFFEu) - wt) {
                        // 32-bit distances would overflow: flag it (the host
                        // reruns with 64-bit distances) and drop the edge
                        a.ctr[kOvf] = 1;
                        nbr[k] = -1;
                    }
                }
#pragma unroll
                for (int k = 0; k < kIlp; ++k) cur_d[k] = kPre && nbr[k] >= 0 ? a.dist[nbr[k]] : D(0);
                bool imp[kIlp];
#pragma unroll
                for (int k = 0; k < kIlp; ++k) {
                    imp[k] = false;
                    if (nbr[k] >= 0 && (!kPre || cand[k] < cur_d[k]))
                        imp[k] = cand[k] < atomicMin(&a.dist[nbr[k]], cand[k]);
                }
                bool fresh[kIlp];
#pragma unroll
                for (int k = 0; k < kIlp; ++k) {
                    upd += imp[k];
                    fresh[k] = imp[k] && atomicExch(&a.stamp[nbr[k]], r + 1) != r + 1;
                }
                int deg[kIlp], mine = 0;
#pragma unroll
                for (int k = 0; k < kIlp; ++k) {
                    deg[k] = fresh[k] ? a.offsets[nbr[k] + 1] - a.offsets[nbr[k]] : 0;
                    mine += (deg[k] + kChunk - 1) / kChunk;
                }
                // warp-aggregated enqueue into the block's shared-memory queue
                // (one global atomic per block per round; overflow goes direct)
                int pincl = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int t = __shfl_up_sync(full, pincl, o);
                    if (lane >= o) pincl += t;
                }
                const int ptotal = __shfl_sync(full, pincl, 31);
                if (ptotal) {
                    int sb = 0;
                    if (lane == 31) sb = atomicAdd(&s_qn, ptotal);
                    sb = __shfl_sync(full, sb, 31);
                    // positions >= kSsspQueue overflow into this warp's chunk of
                    // the global queue (one global atomic per kWarpChunk items)
                    const int lo = max(sb, a.stage_cap);
                    const int over = max(0, sb + ptotal - lo);
                    if (over > wq_left) {
                        // pad the rest of the old chunk, reserve a new one
                        for (int t = lane; t < wq_left; t += 32) QN[wq_base + t] = make_int2(-1, 0);
                        const int want = max(over, kWarpChunk);
                        unsigned long long gb = 0;
                        if (lane == 0) gb = atomicAdd(&a.ctr[kQ + nxt], (unsigned long long)want);
                        wq_base = __shfl_sync(full, gb, 0);
                        wq_left = want;
                    }
                    int p = sb + (pincl - mine);
#pragma unroll
                    for (int k = 0; k < kIlp; ++k) {
                        if (deg[k] > 0) {
                            const int32_t first = a.offsets[nbr[k]];
                            const int items = (deg[k] + kChunk - 1) / kChunk;
                            for (int t = 0; t < items; ++t, ++p) {
                                const int2 it = make_int2(nbr[k], first + t * kChunk);
                                if (p < a.stage_cap)
                                    s_q[p] = it;
                                else
                                    QN[wq_base + (p - lo)] = it;
                            }
                        }
                    }
                    wq_base += over;
                    wq_left -= over;
                }
            }
        }
        // pad this warp's partly used chunk
        for (int t = lane; t < wq_left; t += 32) QN[wq_base + t] = make_int2(-1, 0);
        wq_left = 0;
        // flush the block queue (s_qn may exceed the capacity: those went direct)
        __syncthreads();
        const int qb = min(s_qn, a.stage_cap);
        if (threadIdx.x == 0 && qb > 0)
            s_gpos = atomicAdd(&a.ctr[kQ + nxt], (unsigned long long)qb);
        __syncthreads();
        for (int i = threadIdx.x; i < qb; i += kSsspBlock) QN[s_gpos + i] = s_q[i];
        grid.sync();
        if (ld_volatile(&a.ctr[kQ + nxt]) == 0) break;
    }
    // statistics
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        vvis += __shfl_xor_sync(full, vvis, o);
        evis += __shfl_xor_sync(full, evis, o);
        upd += __shfl_xor_sync(full, upd, o);
    }
    if (lane == 0) {
        atomicAdd(&a.ctr[kVvis], vvis);
        atomicAdd(&a.ctr[kEvis], evis);
        atomicAdd(&a.ctr[kUpd], upd);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctr[kRounds] = r + 1;
}

// SURVEY 8(d)'s U counter: every lane adds its own count with one relaxed
// atomic into one of kUpdSlots counters at the end of the kernel.  Same-box
// A/B on C5 (relaxation without any counter: 20.8 ms): one global counter hit
// by every warp 23.0 ms, a block-wide __syncthreads reduction 22.3 ms, a warp
// __reduce_add_sync (its reconvergence region spans the whole item loop)
// 22.9 ms, per-lane atomics 21.0 ms.  The slots are zeroed by the call's init
// kernel and summed by its widen kernel (sum_slots).
constexpr int kUpdSlots = 1024;
__device__ inline void warp_count(unsigned int v, unsigned long long* slots) {
    if (v) atomicAdd(&slots[(blockIdx.x * blockDim.x + threadIdx.x) & (kUpdSlots - 1)],
                     (unsigned long long)v);
}

// One warp: *out = sum of the kUpdSlots slots.
__device__ inline void sum_slots(const unsigned long long* slots, unsigned long long* out) {
    unsigned long long v = 0;
    for (int i = threadIdx.x; i < kUpdSlots; i += 32) v += slots[i];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *out = v;
}

template <class D>
__global__ void k_sssp_widen(int32_t n, const D* __restrict__ dist, D inf, int64_t* __restrict__ out,
                             const unsigned long long* slots = nullptr,
                             unsigned long long* slots_sum = nullptr,
                             const int32_t* __restrict__ perm = nullptr) {
    if (slots && blockIdx.x == 0 && threadIdx.x < 32) sum_slots(slots, slots_sum);
    // perm: the distances of a renumbered graph, written in the caller's ids
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        D d = dist[perm ? perm[i] : i];
        out[i] = d == inf ? (INT64_MAX / 2) : int64_t(d);
    }
}

// Returns true when 32-bit distances overflowed (the caller reruns with 64).
template <class D>
static bool run_sssp(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats) {
    auto& w = *g->sssp;
    cudaStream_t s = g->stream;
    SsspArgs<D> a;
    a.n = g->n;
    a.offsets = g->offsets.get();
    a.dests = g->dests.get();
    a.weights = g->weighted ? g->weights.get() : nullptr;
    a.dist = reinterpret_cast<D*>(w.dist.get());
    a.stamp = w.stamp.get();
    a.q0 = w.queue[0].get();
    a.q1 = w.queue[1].get();
    a.ctr = w.ctrs.get();
    static const bool trace = std::getenv("GDX_SSSP_TRACE") != nullptr;
    a.trace = nullptr;
    if (trace) {
        w.trace.ensure(512);
        a.trace = w.trace.get();
    }
    // GDX_SSSP_STAGE (tests): block staging capacity, 0 = every push takes
    // the warp-chunk path of large frontiers
    const char* stage = std::getenv("GDX_SSSP_STAGE");
    a.stage_cap = stage ? std::max(0, std::min(kSsspQueue, std::atoi(stage))) : kSsspQueue;
    const D inf = ~D(0);
    const char* var = std::getenv("GDX_SSSP_VARIANT");
    const int vsel = var ? std::atoi(var) : 0;
    void* kfn = vsel == 1 ? (void*)k_sssp_rounds<D, 8, true>
              : vsel == 2 ? (void*)k_sssp_rounds<D, 4, false>
              : vsel == 3 ? (void*)k_sssp_rounds<D, 8, false>
                          : (void*)k_sssp_rounds<D, 4, true>;
    if (w.grid == 0) {
        int per_sm = 0;
        GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kSsspBlock, 0));
        if (per_sm < 1) fail(GDX_ERR_CUDA, "CudaError: sssp kernel cannot be resident");
        w.grid = per_sm * g->num_sms;
    }
    GDX_CUDA(cudaMemsetAsync(w.ctrs.get(), 0, kCtrs * sizeof(unsigned long long), s));
    timed_launch(g, "sssp_init", [&] {
        k_sssp_init<D><<<blocks_for(g->n, 256, g->num_sms * 8), 256, 0, s>>>(a, src, inf);
    });
    timed_launch(g, "sssp_rounds", [&] {
        void* args[] = {&a};
        GDX_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(w.grid), dim3(kSsspBlock),
                                             args, 0, s));
    });
    // Widen into the caller's buffer (host or device).  Device output: write in
    // place; host output: widen into a device staging buffer, then copy.
    cudaPointerAttributes pa;
    bool dev_out = cudaPointerGetAttributes(&pa, dist_out) == cudaSuccess &&
                   pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    int64_t* target = dev_out ? dist_out : reinterpret_cast<int64_t*>(w.queue[1].get());
    timed_launch(g, "sssp_widen", [&] {
        k_sssp_widen<D><<<blocks_for(g->n, 256, g->num_sms * 8), 256, 0, s>>>(g->n, a.dist, inf, target);
    });
    if (!dev_out) copy_out(g, dist_out, target, size_t(g->n) * sizeof(int64_t));
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, w.ctrs.get(), kCtrs * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    if (trace) {
        std::vector<unsigned long long> t(512);
        GDX_CUDA(cudaMemcpy(t.data(), a.trace, 512 * 8, cudaMemcpyDeviceToHost));
        for (unsigned long long r = 0; r < h[kRounds] && r < 256; ++r)
            fprintf(stderr, "sssp round %llu: queue %llu items, %.1f kcycles\n", r, t[2 * r],
                    r + 1 < h[kRounds] ? double(t[2 * r + 3] - t[2 * r + 1]) * 1e-3 : 0.0);
    }
    if (stats) {
        stats->rounds = int32_t(h[kRounds]);
        stats->launches = 3;
        stats->vertices_visited = int64_t(h[kVvis]);
        stats->edges_visited = int64_t(h[kEvis]);
        stats->updates = int64_t(h[kUpd]);
        // 16 V_vis + 12 E_vis + 8 U
        stats->algorithmic_bytes = 16.0 * h[kVvis] + 12.0 * h[kEvis] + 8.0 * h[kUpd];
    }
    return h[kOvf] != 0;
}

// ---------------------------------------------------------------------------
// Sharded SSSP (gdx_sssp_shard_*): one rank of a vertex-range partition.
// Every rank keeps a full int64 replica of dist; a round relaxes the out-edges
// of the rank's own vertices that improved since they were last expanded
// (dist < prev), into the local replica, and the caller merges the replicas
// with an element-wise MIN all-reduce (distributed.py sharded_sssp).
// ---------------------------------------------------------------------------
constexpr int kSplitItems = 8;   // vertices with more items are emitted warp-cooperatively
#ifndef GDX_SSSP_CHUNK
#define GDX_SSSP_CHUNK 64
#endif
constexpr int kUpdSlot = 6;  // shard_ctr slot counting issued relaxations (U)
constexpr int kShardChunk = GDX_SSSP_CHUNK;
// atomicMin over any distance width: 16-bit distances (the narrow first
// attempt of large graphs) take a CAS loop on their aligned 32-bit word.
__device__ __forceinline__ unsigned short dist_atomic_min(unsigned short* p, unsigned short v) {
    unsigned int* w = reinterpret_cast<unsigned int*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
    const int sh = (reinterpret_cast<uintptr_t>(p) & 2) ? 16 : 0;
    unsigned int old = *w, assumed;
    do {
        assumed = old;
        const unsigned short cur = (unsigned short)(assumed >> sh);
        if (cur <= v) return cur;
        old = atomicCAS(w, assumed, (assumed & ~(0xFFFFu << sh)) | (unsigned(v) << sh));
    } while (old != assumed);
    return (unsigned short)(assumed >> sh);
}
template <class D>
__device__ __forceinline__ D dist_atomic_min(D* p, D v) { return atomicMin(p, v); }

  // edges per relaxation item (same-box C5: 21.0 ms vs 22.2 at 32, 24.4 at 128)
// every relaxation kernel splits an item over LPI in {8, 16, 32} lanes
static_assert(kShardChunk % 32 == 0 && kShardChunk >= 32, "GDX_SSSP_CHUNK must be a multiple of 32");

// Frontier scan: queue relaxation items of the vertices in [v0, v1) whose
// distance dropped since they were last expanded (dist < prev; prev := dist).
// One global atomic per block-chunk of kFBlock * 8 vertices.
#ifndef GDX_SSSP_FBLOCK
#define GDX_SSSP_FBLOCK 256
#endif
constexpr int kFBlock = GDX_SSSP_FBLOCK;
#ifndef GDX_SSSP_FPER
#define GDX_SSSP_FPER 8
#endif
constexpr int kFPer = GDX_SSSP_FPER;  // vertices per thread per scan chunk
// graphs below 2^22 vertices scan 4 vertices per thread (more, shorter chunks:
// same-box C1 0.279 -> 0.250 ms per call; C5 keeps 8: 19.1 vs 19.4 ms)
constexpr int kFPerSmall = 4;
constexpr int32_t kSmallScan = 1 << 22;
// SPLIT (the single-GPU round loop): vertices with at most kSmallDeg out-edges
// go to a second queue of one-item vertices, relaxed 2 lanes per item (lane
// utilisation: a 3-edge vertex no longer occupies a 16-lane group); their
// count is ctr[kSmallCtr].
#ifndef GDX_SSSP_SMALLDEG
#define GDX_SSSP_SMALLDEG 8
#endif
constexpr int kSmallDeg = GDX_SSSP_SMALLDEG;
constexpr int kSmallLpi = kSmallDeg / 4;  // 4 edges per lane
constexpr int kSmallCtr = 7;
template <class D, int PER = kFPer, bool SPLIT = false>
__global__ void __launch_bounds__(kFBlock) k_sssp_scan_frontier(int32_t v0, int32_t v1,
                                                           const int32_t* __restrict__ offsets,
                                                           const D* __restrict__ dist, D* prev,
                                                           int2* queue,
                                                           unsigned long long* ctr,
                                                           int2* squeue = nullptr) {
    constexpr int kPer = PER;  // vertices per thread per chunk
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ unsigned long long s_warp[kFBlock / 32];  // (small << 32) | large item counts
    __shared__ unsigned long long s_base, s_sbase;
    // statistics (improved sinks, frontier vertices, their edges) accumulate in
    // registers across the block's chunks and reach the counters with one
    // atomic per block at the end: per-warp atomics on three single addresses
    // serialise in L2 (262K of them per C5 round)
    unsigned long long t_vis = 0, t_edg = 0, t_sinks = 0;
    for (int64_t c0 = v0 + int64_t(blockIdx.x) * kFBlock * kPer; c0 < v1;
         c0 += int64_t(gridDim.x) * kFBlock * kPer) {
        // all loads of the chunk are issued before any is consumed: the prev
        // stores would otherwise order each vertex's loads after the previous
        // vertex's (possible aliasing), one DRAM round trip per vertex
        D dk[kPer], pk[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t v = c0 + int64_t(k) * kFBlock + threadIdx.x;
            dk[k] = v < v1 ? dist[v] : D(0);
            pk[k] = v < v1 ? prev[v] : D(0);
        }
        int items[kPer], first[kPer], last[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t v = c0 + int64_t(k) * kFBlock + threadIdx.x;
            const bool f = dk[k] < pk[k];  // false past v1 (both 0)
            first[k] = f ? offsets[v] : 0;
            last[k] = f ? offsets[v + 1] : -1;
        }
        unsigned long long mine = 0;  // (small items << 32) | large items
        int sinks = 0;
        unsigned long long vis = 0, edg = 0;
        bool small[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t v = c0 + int64_t(k) * kFBlock + threadIdx.x;
            items[k] = 0;
            small[k] = false;
            if (last[k] >= 0) {
                prev[v] = dk[k];
                const int32_t deg = last[k] - first[k];
                small[k] = SPLIT && deg > 0 && deg <= kSmallDeg;
                items[k] = small[k] ? 0 : (deg + kShardChunk - 1) / kShardChunk;
                sinks += deg == 0;
                ++vis;
                edg += deg;
            }
            mine += (unsigned long long)items[k] + (small[k] ? (1ull << 32) : 0ull);
        }
        t_sinks += sinks;
        t_vis += vis;
        t_edg += edg;
        unsigned long long incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(full, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < kFBlock / 32; ++w) {
                const unsigned long long x = s_warp[w];
                s_warp[w] = tot;
                tot += x;
            }
            const unsigned long long tl = tot & 0xffffffffull, ts = tot >> 32;
            s_base = tl ? atomicAdd(&ctr[0], tl) : 0;
            if (SPLIT) s_sbase = ts ? atomicAdd(&ctr[kSmallCtr], ts) : 0;
        }
        __syncthreads();
        const unsigned long long ex = s_warp[warp] + incl - mine;
        unsigned long long pos = s_base + (ex & 0xffffffffull);
        unsigned long long spos = SPLIT ? s_sbase + (ex >> 32) : 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int32_t v = int32_t(c0 + int64_t(k) * kFBlock + threadIdx.x);
            // a hub's items (a degree-10^6 vertex has ~10^4) are written by the
            // whole warp, not serially by its own lane
            const bool big = items[k] > kSplitItems;
            if (SPLIT && small[k]) squeue[spos++] = make_int2(v, first[k]);
            if (!big)
                for (int t = 0; t < items[k]; ++t) queue[pos + t] = make_int2(v, first[k] + t * kShardChunk);
            unsigned hubs = __ballot_sync(full, big);
            while (hubs) {
                const int l = __ffs(hubs) - 1;
                hubs &= hubs - 1;
                const unsigned long long hb = __shfl_sync(full, pos, l);
                const int hc = __shfl_sync(full, items[k], l);
                const int32_t hv = __shfl_sync(full, v, l), hf = __shfl_sync(full, first[k], l);
                for (int t = lane; t < hc; t += 32) queue[hb + t] = make_int2(hv, hf + t * kShardChunk);
            }
            pos += items[k];
        }
        __syncthreads();
    }
    {
        __shared__ unsigned long long s_red[3][kFBlock / 32];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t_vis += __shfl_xor_sync(full, t_vis, o);
            t_edg += __shfl_xor_sync(full, t_edg, o);
            t_sinks += __shfl_xor_sync(full, t_sinks, o);
        }
        if (lane == 0) {
            s_red[0][warp] = t_vis;
            s_red[1][warp] = t_edg;
            s_red[2][warp] = t_sinks;
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            unsigned long long x = 0;
            for (int w = 0; w < kFBlock / 32; ++w) x += s_red[threadIdx.x][w];
            if (x) atomicAdd(&ctr[threadIdx.x == 0 ? 3 : threadIdx.x == 1 ? 4 : 1], x);
        }
    }
}

// Frontier-scan grid: up to 64 blocks per SM (a few chunks each; same-box C5:
// 21.0 vs 21.35 ms with one resident wave of ~44-chunk blocks);
// GDX_SSSP_FGRID = blocks per SM overrides.
template <class D>
static int frontier_grid(const gdx_graph* g, int64_t cnt, int per = kFPer) {
    static const int per_sm = [] {
        const char* e = std::getenv("GDX_SSSP_FGRID");
        return e ? std::max(1, std::atoi(e)) : 64;
    }();
    return blocks_for(cnt, kFBlock * per, g->num_sms * per_sm);
}

// The single-GPU round loop's scan: per-thread chunk by graph size.
// (The partitions of the multi-GPU rounds scan their range [v0, v1) with the
// variant the whole graph's size selects, so every partition runs the same.)
template <class D>
static void launch_scan(const gdx_graph* g, cudaStream_t st, int32_t v0, int32_t v1, D* dist,
                        D* prev, int2* queue, unsigned long long* ctr, int2* squeue) {
    const int64_t cnt = int64_t(v1) - v0;
    const bool small = g->n < kSmallScan;
    if (squeue) {
        if (small)
            k_sssp_scan_frontier<D, kFPerSmall, true>
                <<<frontier_grid<D>(g, cnt, kFPerSmall), kFBlock, 0, st>>>(
                    v0, v1, g->offsets.get(), dist, prev, queue, ctr, squeue);
        else
            k_sssp_scan_frontier<D, kFPer, true><<<frontier_grid<D>(g, cnt), kFBlock, 0, st>>>(
                v0, v1, g->offsets.get(), dist, prev, queue, ctr, squeue);
    } else if (small) {
        k_sssp_scan_frontier<D, kFPerSmall><<<frontier_grid<D>(g, cnt, kFPerSmall), kFBlock, 0, st>>>(
            v0, v1, g->offsets.get(), dist, prev, queue, ctr);
    } else {
        k_sssp_scan_frontier<D><<<frontier_grid<D>(g, cnt), kFBlock, 0, st>>>(
            v0, v1, g->offsets.get(), dist, prev, queue, ctr);
    }
}


// Relaxation: one warp per item (<= kShardChunk out-edges of one vertex), lanes
// over the edges; 32-bit distances flag an overflow (ctr[2]) instead of
// wrapping -- the caller then reruns with 64-bit distances.
// Delta mode (sharded SSSP, gdx_sssp_shard_relax32_delta): every vertex whose
// distance this relaxation lowered is listed once per round (mark = round).
struct SsspDelta {
    int32_t* mark;
    int32_t* changed;
    unsigned long long* count;
    int32_t round;
};

template <class D, int LPI, bool DELTA = false, int CH = kShardChunk>
__global__ void __launch_bounds__(256) k_sssp_scan_relax(const int2* __restrict__ queue,
                                                        const unsigned long long* __restrict__ ctr,
                                                        const int32_t* __restrict__ offsets,
                                                        const int32_t* __restrict__ dests,
                                                        const int32_t* __restrict__ weights,
                                                        D* dist, unsigned long long* ovf,
                                                        SsspDelta dl = {},
                                                        unsigned long long* upd = nullptr) {
    // LPI lanes per item: lane groups of LPI take one item each
    const int sub = threadIdx.x & (LPI - 1);
    unsigned int issued = 0;  // relaxations that issued an atomicMin
    constexpr int kU = CH / LPI;  // edges per lane per item, all loads issued together
    static_assert(CH % LPI == 0, "an item's edges split evenly over its lanes");
    const unsigned long long nq = ctr[0];
    for (unsigned long long i = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) / LPI;
         i < nq; i += ((unsigned long long)gridDim.x * blockDim.x) / LPI) {
        const int2 it = queue[i];
        const D dv = dist[it.x];
        // int64: it.y + CH passes INT32_MAX on the last items of m ~ 2^31 graphs
        const int32_t e1 = int32_t(min(int64_t(it.y) + CH, int64_t(offsets[it.x + 1])));
        int32_t u[kU];
        D c[kU], du[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const int32_t e = it.y + sub + k * LPI;
            u[k] = e < e1 ? dests[e] : -1;
            const D w = e < e1 ? (weights ? D(weights[e]) : D(1)) : D(0);
            c[k] = dv + w;
            if (sizeof(D) < 8 && u[k] >= 0 &&
                uint64_t(dv) + uint64_t(w) >= uint64_t(std::numeric_limits<D>::max())) {
                *ovf = 1;
                u[k] = -1;
            }
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) du[k] = u[k] >= 0 ? dist[u[k]] : D(0);
#pragma unroll
        for (int k = 0; k < kU; ++k)
            if (u[k] >= 0 && c[k] < du[k]) {
                ++issued;
                if (DELTA) {
                    if (c[k] < dist_atomic_min(&dist[u[k]], c[k]) &&
                        atomicMax(&dl.mark[u[k]], dl.round) < dl.round)
                        dl.changed[atomicAdd(dl.count, 1ull)] = u[k];
                } else {
                    dist_atomic_min(&dist[u[k]], c[k]);
                }
            }
    }
    if (upd) warp_count(issued, upd);
}

constexpr int kRelaxCarveout = -1;  // relaxation's shared-memory carveout (prefer_l1)

// The round's relaxations: the <= 64-edge items (LPI lanes each) and, with the
// split queue, the small vertices' one items (2 lanes, <= kSmallDeg edges).
template <class D>
static void launch_relax(const gdx_graph* g, cudaStream_t st, int lpi, int grid, const int2* queue,
                         const unsigned long long* ctr, const int2* squeue, D* dist,
                         unsigned long long* ovf, unsigned long long* upd) {
    const int32_t* w = g->weighted ? g->weights.get() : nullptr;
    auto fn = lpi == 8 ? k_sssp_scan_relax<D, 8>
            : lpi == 16 ? k_sssp_scan_relax<D, 16> : k_sssp_scan_relax<D, 32>;
    fn<<<grid, 256, 0, st>>>(queue, ctr, g->offsets.get(), g->dests.get(), w, dist, ovf,
                             SsspDelta{}, upd);
    if (squeue)
        k_sssp_scan_relax<D, kSmallLpi, false, kSmallDeg><<<grid, 256, 0, st>>>(
            squeue, ctr + kSmallCtr, g->offsets.get(), g->dests.get(), w, dist, ovf, SsspDelta{},
            upd);
}

// (id, value) pairs of the vertices listed by a delta relaxation.
template <class D>
__global__ void k_sssp_delta_values(const int32_t* __restrict__ changed,
                                    const unsigned long long* __restrict__ count,
                                    const D* __restrict__ dist, D* vals) {
    const unsigned long long c = *count;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < c;
         i += (unsigned long long)gridDim.x * blockDim.x)
        vals[i] = dist[changed[i]];
}

// Element-wise MIN of received (id, value) pairs into the replica (id < 0: padding).
template <class D>
__global__ void k_sssp_delta_apply(const int32_t* __restrict__ ids, const D* __restrict__ vals,
                                   int64_t count, D* dist) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        if (v >= 0 && vals[i] < dist[v]) atomicMin(&dist[v], vals[i]);
    }
}

template <class D>
__global__ void k_sssp_scan_init(int32_t n, int32_t src, D inf, D* dist, D* prev,
                                 unsigned long long* z0, int nz0, unsigned long long* z1, int nz1,
                                 unsigned long long* slots) {
    // also zeroes the call's counters (z0[0, nz0), z1[0, nz1), the U slots): no memsets
    if (blockIdx.x == 0 && threadIdx.x < nz0) z0[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x < nz1) z1[threadIdx.x] = 0;
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < kUpdSlots; i += blockDim.x) slots[i] = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        dist[i] = i == src ? D(0) : inf;
        prev[i] = inf;
    }
}

// Device-side loop (CUDA graph with a conditional WHILE node): the body is
// frontier scan -> relaxation -> k_sssp_graph_finish, which counts the round,
// clears the counters and continues while the scan produced work -- no host
// round trip per round.
__global__ void k_sssp_graph_finish(unsigned long long* ctr, unsigned long long* acc,
                                    cudaGraphConditionalHandle h) {
    const unsigned long long items = ctr[0] + ctr[kSmallCtr];
    if (items) acc[0] += 1;
    acc[1] += ctr[3];
    acc[2] += ctr[4];
    for (int i = 0; i < 5; ++i) ctr[i] = 0;
    ctr[kSmallCtr] = 0;
    // a narrow-width overflow ends the loop at once (the call reruns wider)
    cudaGraphSetConditional(h, items && !acc[3] ? 1u : 0u);
}

template <class D>
static cudaGraphExec_t build_sssp_graph(gdx_graph* g, D* dist, D* prev, unsigned long long* ovf,
                                        int lpi, int relax_grid, int2* squeue) {
    auto& w = *g->sssp;
    cudaGraph_t graph;
    GDX_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    GDX_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    GDX_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t cs;
    GDX_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    GDX_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    const int32_t n = g->n;
    unsigned long long* ctr = w.shard_ctr.get();
    launch_scan<D>(g, cs, 0, n, dist, prev, w.shard_queue.get(), ctr, squeue);
    launch_relax<D>(g, cs, lpi, relax_grid, w.shard_queue.get(), ctr, squeue, dist, ovf,
                    w.upd_slots.get());
    k_sssp_graph_finish<<<1, 1, 0, cs>>>(ctr, w.graph_acc.get(), h);
    cudaGraph_t captured;
    GDX_CUDA(cudaStreamEndCapture(cs, &captured));
    GDX_CUDA(cudaStreamDestroy(cs));
    cudaGraphExec_t exec;
    GDX_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    GDX_CUDA(cudaGraphDestroy(graph));
    return exec;
}

// Large graphs: rounds of (frontier scan, relaxation) with one host read of
// the item count per round (the round count is ~ the weighted BFS depth, so
// the host round trips are negligible next to the ~ms rounds).  Returns true
// when 32-bit distances overflowed.
template <class D>
static bool run_sssp_scan(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats,
                          bool use_graph = false) {
    auto& w = *g->sssp;
    cudaStream_t s = g->stream;
    const int32_t n = g->n;
    D* dist = reinterpret_cast<D*>(w.dist.get());
    D* prev = reinterpret_cast<D*>(w.prev.get());
    const D inf = sizeof(D) < 8 ? std::numeric_limits<D>::max() : D(INT64_MAX / 2);
    const size_t items_cap = size_t(n) + size_t(g->m) / kShardChunk + 1;
    w.shard_queue.ensure(items_cap);
    w.shard_ctr.ensure(kSmallCtr + 1);
    w.upd_slots.ensure(kUpdSlots);
    unsigned long long* ctr = w.shard_ctr.get();
    // large graphs: small vertices in their own queue (one more launch per
    // round: same-box C5 19.18 -> 18.65 ms, C1 0.226 -> 0.246 ms, so graphs
    // below 2^22 vertices keep one queue; GDX_SSSP_SPLIT=0/1 overrides)
    const char* spl = std::getenv("GDX_SSSP_SPLIT");
    const bool split = spl ? std::atoi(spl) != 0 : n >= kSmallScan;
    if (split) w.small_queue.ensure(size_t(n));
    int2* squeue = split ? w.small_queue.get() : nullptr;
    // graph path: round counters, [rounds, vertices, edges, overflow] in
    // graph_acc; host loop: its own overflow flag
    w.graph_acc.ensure(4);
    DevBuf<unsigned long long> ovf(1);
    unsigned long long* ovf_flag = use_graph ? w.graph_acc.get() + 3 : ovf.get();
    timed_launch(g, "sssp_init", [&] {
        k_sssp_scan_init<D><<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(
            n, src, inf, dist, prev, ctr, kSmallCtr + 1, use_graph ? w.graph_acc.get() : ovf.get(),
            use_graph ? 4 : 1, w.upd_slots.get());
    });
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    unsigned long long vvis = 0, evis = 0;
    int rounds = 0, launches = 1;
    const char* lv = std::getenv("GDX_SSSP_LPI");
    const int lpi = lv ? std::atoi(lv) : 16;  // lanes per relaxation item
    const char* rc = std::getenv("GDX_SSSP_RELAX_CAP");  // blocks per SM (A/B)
    // 8 blocks/SM for small graphs -- one resident wave of 256-thread blocks
    // (same-box C1 0.222 vs 0.227 ms at 16, 0.238 at 4) -- 128 for large ones
    // (same-box C5: 21.3 vs 21.9 ms at 64, 22.9 at 32; on the renumbered graph
    // 256: 16.61-16.66 vs 16.86 ms at 128, 16.78-16.85 at 512)
    const int relax_grid =
        (rc ? std::max(1, std::atoi(rc)) : (g->m < (int64_t(1) << 26) ? 8 : 256)) * g->num_sms;
    prefer_l1(reinterpret_cast<const void*>(&k_sssp_scan_relax<D, 16>), kRelaxCarveout);
    prefer_l1(reinterpret_cast<const void*>(&k_sssp_scan_relax<D, kSmallLpi, false, kSmallDeg>),
              kRelaxCarveout);
    if (use_graph) {
        const int di = sizeof(D) == 2 ? 2 : sizeof(D) == 4 ? 0 : 1;
        // the instantiated graph bakes in these buffers and the CSR arrays
        // (gdx_graph_set_hash_weights reallocates / enables the weights)
        void* key[SsspWork::kKey] = {dist, prev, w.shard_queue.get(), ctr, w.graph_acc.get(),
                                     g->offsets.get(), g->dests.get(),
                                     g->weighted ? g->weights.get() : nullptr,
                                     reinterpret_cast<void*>(intptr_t(lpi * 65536 + relax_grid) |
                                                             (intptr_t(split) << 40)),
                                     w.upd_slots.get()};
        bool same = w.gexec[di] != nullptr;
        for (int i = 0; i < SsspWork::kKey; ++i) same = same && w.gkey[di][i] == key[i];
        if (!same) {
            if (w.gexec[di]) cudaGraphExecDestroy(w.gexec[di]);
            w.gexec[di] = build_sssp_graph<D>(g, dist, prev, ovf_flag, lpi, relax_grid, squeue);
            for (int i = 0; i < SsspWork::kKey; ++i) w.gkey[di][i] = key[i];
        }
        timed_launch(g, "sssp_graph", [&] { GDX_CUDA(cudaGraphLaunch(w.gexec[di], s)); });
    }
    for (; !use_graph; ++rounds) {
        GDX_CUDA(cudaMemsetAsync(ctr, 0, 5 * sizeof(unsigned long long), s));
        GDX_CUDA(cudaMemsetAsync(ctr + kSmallCtr, 0, sizeof(unsigned long long), s));
        timed_launch(g, "sssp_frontier", [&] {
            launch_scan<D>(g, s, 0, n, dist, prev, w.shard_queue.get(), ctr, squeue);
        });
        GDX_CUDA(cudaMemcpyAsync(h, ctr, (kSmallCtr + 1) * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        ++launches;
        vvis += h[3];
        evis += h[4];
        if (h[0] + h[kSmallCtr] == 0) break;
        timed_launch(g, "sssp_relax", [&] {
            launch_relax<D>(g, s, lpi, relax_grid, w.shard_queue.get(), ctr, squeue, dist,
                            ovf.get(), w.upd_slots.get());
        });
        launches += split ? 2 : 1;
    }
    cudaPointerAttributes pa;
    bool dev_out = cudaPointerGetAttributes(&pa, dist_out) == cudaSuccess &&
                   pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    if (!dev_out) w.queue[1].ensure(size_t(n));
    int64_t* target = dev_out ? dist_out : reinterpret_cast<int64_t*>(w.queue[1].get());
    timed_launch(g, "sssp_widen", [&] {
        k_sssp_widen<D><<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(
            n, dist, inf, target, w.upd_slots.get(), ctr + kUpdSlot, w.out_perm);
    });
    if (!dev_out) copy_out(g, dist_out, target, size_t(n) * sizeof(int64_t));
    // one host read per call: the graph path's counters and the overflow flag
    GDX_CUDA(cudaMemcpyAsync(h, use_graph ? w.graph_acc.get() : ovf.get(),
                             (use_graph ? 4 : 1) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemcpyAsync(h + 4, ctr + kUpdSlot, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    const unsigned long long upd = h[4];
    const bool overflow = (use_graph ? h[3] : h[0]) != 0;
    if (use_graph) {
        rounds = int(h[0]);
        vvis = h[1];
        evis = h[2];
        launches += (split ? 4 : 3) * (rounds + 1);
    }
    if (stats) {
        stats->rounds = rounds;
        stats->launches = launches + 1;
        stats->vertices_visited = int64_t(vvis);
        stats->edges_visited = int64_t(evis);
        stats->updates = int64_t(upd);
        // 16 V_vis + 12 E_vis + 8 U (offsets pair 8 + dist[v] 4 +
        // queue entry 4 per frontier vertex; dest 4 + weight 4 + dist[nbr] 4 per
        // edge; atomicMin 4 + push 4 per relaxation that issued an atomicMin).
        // The frontier scan's full-V read (2 sizeof(D) n per round) is work the
        // formula does not count; bench.py reports it beside the roofline.
        stats->algorithmic_bytes = 16.0 * vvis + 12.0 * evis + 8.0 * upd;
    }
    return overflow;
}

}  // namespace gdx

using namespace gdx;

extern "C" int gdx_sssp_shard_setup(gdx_graph* g, int32_t v_begin, int32_t v_end) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (v_begin < 0 || v_end > g->n || v_begin > v_end)
            fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: vertex range out of bounds");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        GraphScope dg(g);
        if (!g->sssp) g->sssp = std::make_unique<SsspWork>();
        auto& w = *g->sssp;
        int32_t eb[2] = {0, 0};
        GDX_CUDA(cudaMemcpy(&eb[0], g->offsets.get() + v_begin, 4, cudaMemcpyDeviceToHost));
        GDX_CUDA(cudaMemcpy(&eb[1], g->offsets.get() + v_end, 4, cudaMemcpyDeviceToHost));
        w.shard_v0 = v_begin;
        w.shard_v1 = v_end;
        w.shard_edges = int64_t(eb[1]) - eb[0];
        w.shard_queue.ensure(size_t(v_end - v_begin) + size_t(eb[1] - eb[0]) / kShardChunk + 1);
        w.shard_ctr.ensure(kUpdSlot + 1);
        w.shard_ready = true;
    });
}

// D = unsigned long long (int64 replicas, INF = INT64_MAX/2) or int (int32
// replicas, INF = INT32_MAX; a relaxation that would reach INF raises the
// overflow flag reported by the next frontier call).
template <class D>
static void shard_frontier(gdx_graph* g, D* dist, D* prev, int64_t* out, int nout) {
    if (!g || !g->sssp || !g->sssp->shard_ready)
        fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
    auto& w = *g->sssp;
    const int32_t cnt = w.shard_v1 - w.shard_v0;
    if (!out || (g->n > 0 && (!dist || !prev)))
        fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
    GraphScope dg(g);
    cudaStream_t s = g->stream;
    // counters 0,1 (items, improved sinks) and 3,4 (stats) restart every round;
    // 2 (overflow) accumulates over the relaxations since the previous call
    GDX_CUDA(cudaMemsetAsync(w.shard_ctr.get(), 0, 2 * sizeof(unsigned long long), s));
    GDX_CUDA(cudaMemsetAsync(w.shard_ctr.get() + 3, 0, 2 * sizeof(unsigned long long), s));
    if (cnt > 0)
        timed_launch(g, "sssp_shard_frontier", [&] {
            k_sssp_scan_frontier<D><<<frontier_grid<D>(g, cnt), kFBlock, 0, s>>>(
                w.shard_v0, w.shard_v1, g->offsets.get(), dist, prev, w.shard_queue.get(),
                w.shard_ctr.get());
        });
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, w.shard_ctr.get(), 3 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemsetAsync(w.shard_ctr.get() + 2, 0, sizeof(unsigned long long), s));
    GDX_CUDA(cudaStreamSynchronize(s));
    // out (device or host): queued items + improved sinks of this rank [, overflow]
    const int64_t c[2] = {int64_t(h[0] + h[1]), int64_t(h[2] != 0)};
    GDX_CUDA(cudaMemcpy(out, c, size_t(nout) * sizeof(int64_t), cudaMemcpyDefault));
}

template <class D>
static void shard_relax(gdx_graph* g, D* dist) {
    if (!g || !g->sssp || !g->sssp->shard_ready)
        fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
    if (g->n > 0 && !dist) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
    GraphScope dg(g);
    auto& w = *g->sssp;
    cudaStream_t s = g->stream;
    // the single-GPU rule (gdx_sssp): deeper grids for large relaxation sets
    const int blocks = (w.shard_edges < (int64_t(1) << 26) ? 16 : 128) * g->num_sms;
    timed_launch(g, "sssp_shard_relax", [&] {
        k_sssp_scan_relax<D, 16><<<blocks, 256, 0, s>>>(
            w.shard_queue.get(), w.shard_ctr.get(), g->offsets.get(), g->dests.get(),
            g->weighted ? g->weights.get() : nullptr, dist, w.shard_ctr.get() + 2);
    });
}

extern "C" int gdx_sssp_shard_frontier(gdx_graph* g, int64_t* dist, int64_t* prev,
                                       int64_t* count_out) {
    return guard_impl([&] {
        shard_frontier(g, reinterpret_cast<unsigned long long*>(dist),
                       reinterpret_cast<unsigned long long*>(prev), count_out, 1);
    });
}

extern "C" int gdx_sssp_shard_relax(gdx_graph* g, int64_t* dist) {
    return guard_impl([&] { shard_relax(g, reinterpret_cast<unsigned long long*>(dist)); });
}

extern "C" int gdx_sssp_shard_frontier32(gdx_graph* g, int32_t* dist, int32_t* prev,
                                         int64_t* out2) {
    return guard_impl([&] { shard_frontier(g, dist, prev, out2, 2); });
}

extern "C" int gdx_sssp_shard_relax32(gdx_graph* g, int32_t* dist) {
    return guard_impl([&] { shard_relax(g, dist); });
}

extern "C" int gdx_sssp_shard_relax32_delta(gdx_graph* g, int32_t* dist, int32_t* changed_ids,
                                            int32_t* changed_dist, int64_t* count_out) {
    return guard_impl([&] {
        if (!g || !g->sssp || !g->sssp->shard_ready)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
        if (!count_out || (g->n > 0 && (!dist || !changed_ids || !changed_dist)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        GraphScope dg(g);
        auto& w = *g->sssp;
        cudaStream_t s = g->stream;
        if (!w.shard_mark.get() || w.shard_mark.bytes() < size_t(g->n) * 4 ||
            w.shard_round == INT32_MAX) {
            w.shard_mark.ensure(size_t(g->n));
            GDX_CUDA(cudaMemsetAsync(w.shard_mark.get(), 0xff, size_t(g->n) * 4, s));  // -1
            w.shard_round = 0;
        }
        SsspDelta dl{w.shard_mark.get(), changed_ids, w.shard_ctr.get() + 5, ++w.shard_round};
        GDX_CUDA(cudaMemsetAsync(dl.count, 0, sizeof(unsigned long long), s));
        const int blocks = (w.shard_edges < (int64_t(1) << 26) ? 16 : 128) * g->num_sms;
        timed_launch(g, "sssp_shard_relax", [&] {
            k_sssp_scan_relax<int, 16, true><<<blocks, 256, 0, s>>>(
                w.shard_queue.get(), w.shard_ctr.get(), g->offsets.get(), g->dests.get(),
                g->weighted ? g->weights.get() : nullptr, dist,
                w.shard_ctr.get() + 2, dl);
        });
        timed_launch(g, "sssp_shard_delta", [&] {
            k_sssp_delta_values<int><<<g->num_sms * 4, 256, 0, s>>>(changed_ids, dl.count, dist,
                                                                   changed_dist);
        });
        unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
        GDX_CUDA(cudaMemcpyAsync(h, dl.count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        const int64_t c = int64_t(h[0]);
        GDX_CUDA(cudaMemcpy(count_out, &c, sizeof(c), cudaMemcpyDefault));
    });
}

extern "C" int gdx_sssp_shard_apply32(gdx_graph* g, int32_t* dist, const int32_t* ids,
                                      const int32_t* vals, int64_t count) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        if (count < 0 || (count > 0 && (!dist || !ids || !vals)))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (count == 0) return;
        GraphScope dg(g);
        cudaStream_t s = g->stream;
        timed_launch(g, "sssp_shard_apply", [&] {
            k_sssp_delta_apply<int><<<blocks_for(count, 256, g->num_sms * 8), 256, 0, s>>>(
                ids, vals, count, dist);
        });
    });
}

// The call on g (validated; the caller's GraphScope is active).
static void sssp_run(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats) {
    if (!g->sssp) g->sssp = std::make_unique<SsspWork>();
    auto& w = *g->sssp;
    // every vertex enters a round's queue at most once: <= n + m/kChunk
    // items; warp overflow chunks at most double that, plus the padding of
    // the last chunk of every warp
    const size_t qcap = 2 * (size_t(g->n) + size_t(g->m) / kChunk + 1) +
                        size_t(kWarpChunk) * 64 * size_t(g->num_sms);
    w.dist.ensure(size_t(g->n));
    // 32-bit distances unless a relaxation overflows them (then 64-bit):
    // the result is exact either way.  Large graphs use frontier-scan
    // rounds (bandwidth-bound), small ones the persistent kernel
    // (latency-bound); GDX_SSSP_MODE=scan|persistent overrides.
    // Default: frontier-scan rounds driven on the device by a CUDA graph
    // with a conditional WHILE node (C1: 0.36 ms vs 0.44 ms for the
    // persistent kernel and 0.56 ms with a host round trip per round).
    // GDX_SSSP_MODE=persistent|scan|graph selects one for A/B runs.
    // Low-degree graphs (max degree <= 64: road-like, high diameter, thousands
    // of small rounds) take the persistent kernel instead: its queue touches
    // only the frontier while a scan reads all n per round (2000^2 grid:
    // 27 ms vs 76 ms).
    const char* mode = std::getenv("GDX_SSSP_MODE");
    const std::string md = mode ? mode : graph_max_degree(g) <= 64 ? "persistent" : "graph";
    const bool graph = md == "graph";
    const bool scan = md == "scan" || graph;
    if (scan) {
        w.prev.ensure(size_t(g->n));
        // widths: 16-bit first on large graphs (half the footprint of the
        // gathered distance array in L2; GDX_SSSP_NARROW=0/1 overrides),
        // unless a 16-bit attempt on this handle already overflowed; then
        // 32-bit, then 64-bit -- each rerun exact
        const char* ne = std::getenv("GDX_SSSP_NARROW");
        const int narrow_env = ne ? std::atoi(ne) : -1;
        const bool narrow = narrow_env >= 0 ? narrow_env > 0
                                            : (g->n >= (1 << 22) && !w.narrow_overflowed);
        bool ovf = true;
        if (narrow) {
            ovf = run_sssp_scan<unsigned short>(g, src, dist_out, stats, graph);
            if (ovf) w.narrow_overflowed = true;
        }
        if (ovf && run_sssp_scan<unsigned int>(g, src, dist_out, stats, graph))
            run_sssp_scan<unsigned long long>(g, src, dist_out, stats, graph);
    } else {
        // the persistent kernel's queues exist only in this mode (C5 in the
        // default graph mode would otherwise hold 2 x ~2 GB of unused items);
        // queue[1] doubles as the int64 staging buffer for host outputs
        w.stamp.ensure(size_t(g->n));
        w.queue[0].ensure(qcap);
        w.queue[1].ensure(qcap > size_t(g->n) ? qcap : size_t(g->n));
        w.ctrs.ensure(kCtrs);
        const bool overflow = run_sssp<unsigned int>(g, src, dist_out, stats);
        if (overflow) run_sssp<unsigned long long>(g, src, dist_out, stats);
    }
}

extern "C" int gdx_sssp(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !dist_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        // interpreter.cpp:1131-1135 -- the node argument must be a valid id.
        if (src < 0 || src >= g->n)
            fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: node id " + std::to_string(src) +
                                           " out of range [0, " + std::to_string(g->n) + ")");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        GraphScope dg(g);
        const char* mode = std::getenv("GDX_SSSP_MODE");
        Relabel* RP = graph_max_degree(g) > 64 && !(mode && std::string(mode) == "persistent") &&
                              relabel_wanted(g)
                          ? relabel_try(g, true, false)
                          : nullptr;
        if (RP) {
            // frontier-scan rounds on the degree-ordered renumbering
            // (relabel.cu); the widening writes the distances in the caller's ids
            Relabel& R = *RP;
            gdx_graph* h = R.h;
            if (!h->sssp) h->sssp = std::make_unique<SsspWork>();
            h->sssp->out_perm = R.newid.get();
            sssp_run(h, relabel_vertex(g, src), dist_out, stats);
            h->sssp->out_perm = nullptr;
            relabel_leave(g);
        } else {
            sssp_run(g, src, dist_out, stats);
        }
    });
}

// ---------------------------------------------------------------------------
// Multi-GPU SSSP in one process (gdx_sssp_multi, multi.cu): owner-computes
// with the exchange fused into the relaxation.  Device d owns the vertex range
// [bound[d], bound[d+1]) and keeps a full distance replica whose owned entries
// are authoritative and whose other entries are hints (never below the
// owner's value).  Its relaxation sends every improving candidate straight to
// the owner's replica with a peer atomicMin over NVLink (and to its own hint),
// so there is no all-gather / all-reduce of distance vectors at all.  Rounds
// run on each device in a CUDA-graph WHILE loop; two device-side barriers per
// round (arrival counters bumped with system-scope atomics in every device's
// memory) separate the scan from the relaxation and the relaxation from the
// next scan, and the scan's item counts are summed across devices at the
// first barrier so every device leaves the loop in the same round.
// ---------------------------------------------------------------------------
namespace gdx {

constexpr int kMaxMultiDev = 16;

struct MultiSync {              // one per device, in that device's memory
    unsigned long long bar;       // barrier arrivals from all devices (monotonic)
    unsigned long long cum;       // frontier items published by all devices (monotonic)
    unsigned long long phase;     // barriers this device has passed
    unsigned long long prev_cum;  // cum at the previous snapshot
    unsigned long long total;     // this round's frontier items over all devices
    unsigned long long err;       // a wait timed out
    unsigned long long ovf;       // OR of every part's 32-bit overflow flag (this call)
    unsigned long long pad;
};

struct SsspOwners {
    void* dist[kMaxMultiDev];     // every device's replica (D*)
    int32_t bound[kMaxMultiDev + 1];
    int32_t nd, self;
};

__global__ void k_multi_arrive(const unsigned long long* items, MultiSync* const* peers, int nd,
                               int split = 0) {
    if (items) {  // the scan's item count (both queues)
        const unsigned long long v = items[0] + (split ? items[kSmallCtr] : 0ull);
        for (int q = 0; q < nd; ++q) atomicAdd_system(&peers[q]->cum, v);
    }
    __threadfence_system();
    for (int q = 0; q < nd; ++q) atomicAdd_system(&peers[q]->bar, 1ull);
}

__global__ void k_multi_wait(MultiSync* me, int nd, int snapshot) {
    const unsigned long long target = (me->phase + 1) * (unsigned long long)nd;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*reinterpret_cast<volatile unsigned long long*>(&me->bar) < target) {
        __nanosleep(128);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {  // 20 s: a device died; fail instead of hanging
            me->err = 1;
            break;
        }
    }
    me->phase += 1;
    __threadfence_system();
    if (snapshot) {
        const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(&me->cum);
        me->total = me->err ? 0 : c - me->prev_cum;
        me->prev_cum = c;
    }
}

__global__ void k_multi_finish(unsigned long long* ctr, unsigned long long* acc, const MultiSync* me,
                               cudaGraphConditionalHandle h) {
    const unsigned long long total = me->total;
    if (total) acc[0] += 1;
    acc[1] += ctr[3];
    acc[2] += ctr[4];
    for (int i = 0; i < 5; ++i) ctr[i] = 0;
    ctr[kSmallCtr] = 0;
    cudaGraphSetConditional(h, total ? 1u : 0u);
}

template <class D>
__global__ void k_multi_init(int32_t n, int32_t src, D inf, D* dist, D* prev,
                             unsigned long long* ctr, int nctr, unsigned long long* acc, int nacc,
                             unsigned long long* slots) {
    if (blockIdx.x == 0 && threadIdx.x < nctr) ctr[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x < nacc) acc[threadIdx.x] = 0;
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < kUpdSlots; i += blockDim.x) slots[i] = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        dist[i] = i == src ? D(0) : inf;
        prev[i] = inf;
    }
}

// The relaxation of k_sssp_scan_relax with the owner routing: an improving
// candidate for u goes to the owner's replica (peer atomicMin) and to the
// local hint.  Hints never drop below the owner's value, so the filter
// c < dist[u] (local) never drops a candidate the owner needs.
template <class D, int LPI, int CH = kShardChunk>
__global__ void __launch_bounds__(256) k_sssp_multi_relax(const int2* __restrict__ queue,
                                                          const unsigned long long* __restrict__ ctr,
                                                          const int32_t* __restrict__ offsets,
                                                          const int32_t* __restrict__ dests,
                                                          const int32_t* __restrict__ weights,
                                                          D* dist, unsigned long long* ovf,
                                                          unsigned long long* upd, SsspOwners own) {
    const int sub = threadIdx.x & (LPI - 1);
    constexpr int kU = CH / LPI;
    static_assert(CH % LPI == 0, "an item's edges split evenly over its lanes");
    unsigned int issued = 0;
    const unsigned long long nq = ctr[0];
    for (unsigned long long i = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) / LPI;
         i < nq; i += ((unsigned long long)gridDim.x * blockDim.x) / LPI) {
        const int2 it = queue[i];
        const D dv = dist[it.x];
        const int32_t e1 = int32_t(min(int64_t(it.y) + CH, int64_t(offsets[it.x + 1])));
        int32_t u[kU];
        D c[kU], du[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const int32_t e = it.y + sub + k * LPI;
            u[k] = e < e1 ? dests[e] : -1;
            const D w = e < e1 ? (weights ? D(weights[e]) : D(1)) : D(0);
            c[k] = dv + w;
            if (sizeof(D) < 8 && u[k] >= 0 &&
                uint64_t(dv) + uint64_t(w) >= uint64_t(std::numeric_limits<D>::max())) {
                *ovf = 1;
                u[k] = -1;
            }
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) du[k] = u[k] >= 0 ? dist[u[k]] : D(0);
#pragma unroll
        for (int k = 0; k < kU; ++k)
            if (u[k] >= 0 && c[k] < du[k]) {
                ++issued;
                int q = 0;
                while (q + 1 < own.nd && u[k] >= own.bound[q + 1]) ++q;
                if (q != own.self) dist_atomic_min(static_cast<D*>(own.dist[q]) + u[k], c[k]);
                dist_atomic_min(&dist[u[k]], c[k]);
            }
    }
    warp_count(issued, upd);
}

template <class D>
static cudaGraphExec_t build_multi_graph(gdx_graph* g, D* dist, D* prev, int32_t v0, int32_t v1,
                                         MultiSync* me, MultiSync* const* peers, int nd,
                                         const SsspOwners& own, int relax_grid, int2* squeue) {
    auto& w = *g->sssp;
    cudaGraph_t graph;
    GDX_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    GDX_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    GDX_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t cs;
    GDX_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    GDX_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    unsigned long long* ctr = w.shard_ctr.get();
    launch_scan<D>(g, cs, v0, v1, dist, prev, w.shard_queue.get(), ctr, squeue);
    k_multi_arrive<<<1, 1, 0, cs>>>(ctr, peers, nd, squeue ? 1 : 0);
    k_multi_wait<<<1, 1, 0, cs>>>(me, nd, 1);
    const int32_t* wts = g->weighted ? g->weights.get() : nullptr;
    k_sssp_multi_relax<D, 16><<<relax_grid, 256, 0, cs>>>(
        w.shard_queue.get(), ctr, g->offsets.get(), g->dests.get(), wts, dist,
        w.graph_acc.get() + 3, w.upd_slots.get(), own);
    if (squeue)  // the small vertices' one items, 2 lanes each (as launch_relax)
        k_sssp_multi_relax<D, kSmallLpi, kSmallDeg><<<relax_grid, 256, 0, cs>>>(
            squeue, ctr + kSmallCtr, g->offsets.get(), g->dests.get(), wts, dist,
            w.graph_acc.get() + 3, w.upd_slots.get(), own);
    k_multi_arrive<<<1, 1, 0, cs>>>(nullptr, peers, nd);
    k_multi_wait<<<1, 1, 0, cs>>>(me, nd, 0);
    k_multi_finish<<<1, 1, 0, cs>>>(ctr, w.graph_acc.get(), me, h);
    cudaGraph_t captured;
    GDX_CUDA(cudaStreamEndCapture(cs, &captured));
    GDX_CUDA(cudaStreamDestroy(cs));
    cudaGraphExec_t exec;
    GDX_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    GDX_CUDA(cudaGraphDestroy(graph));
    return exec;
}

// After the loop: every part ORs its 32-bit overflow flag into every part's
// MultiSync, so all parts take the same 32 -> 64-bit rerun decision.
__global__ void k_multi_flag(const unsigned long long* ovf, MultiSync* const* peers, int nd) {
    const unsigned long long f = *ovf ? 1ull : 0ull;
    if (f)
        for (int q = 0; q < nd; ++q) atomicOr_system(&peers[q]->ovf, f);
    __threadfence_system();
}

__global__ void k_multi_reset(MultiSync* me) { me->ovf = 0; }

// Full distance vector from the owners' replicas (peer loads over NVLink):
// every range is final once the loop has ended on every part.
template <class D>
__global__ void k_multi_gather(int32_t n, SsspOwners own, D inf, int64_t* __restrict__ out,
                               const unsigned long long* slots, unsigned long long* slots_sum) {
    if (blockIdx.x == 0 && threadIdx.x < 32) sum_slots(slots, slots_sum);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int q = 0;
        while (q + 1 < own.nd && i >= own.bound[q + 1]) ++q;
        const D d = static_cast<const volatile D*>(own.dist[q])[i];
        out[i] = d == inf ? (INT64_MAX / 2) : int64_t(d);
    }
}

// The partitions' round loop follows gdx_sssp's choices from the whole
// graph's size, so every partition (and every rank) decides alike: the small
// vertices' queue on graphs of >= 2^22 vertices (GDX_SSSP_SPLIT overrides),
// and 16-bit distances first there (GDX_SSSP_NARROW overrides) unless a 16-bit
// multi-GPU attempt on the handle already overflowed.
static bool multi_split(const gdx_graph* g) {
    const char* e = std::getenv("GDX_SSSP_SPLIT");
    return e ? std::atoi(e) != 0 : g->n >= kSmallScan;
}
static bool multi_narrow(const gdx_graph* g) {
    const char* e = std::getenv("GDX_SSSP_NARROW");
    return e ? std::atoi(e) > 0 : g->n >= (1 << 22) && !g->sssp->multi_narrow_overflowed;
}

// With lazy module loading (the CUDA 12 default) a kernel's first launch
// loads its module, which waits for the work running on the device: a
// partition whose first launch comes while another partition of the same GPU
// spins in a barrier would deadlock until the barrier times out.  Every
// kernel of the multi-GPU rounds is loaded up front.
template <class D>
static void preload_multi_kernels() {
    cudaFuncAttributes fa;
    const void* fns[] = {
        reinterpret_cast<const void*>(&k_multi_init<D>),
        reinterpret_cast<const void*>(&k_sssp_scan_frontier<D>),
        reinterpret_cast<const void*>(&k_sssp_scan_frontier<D, kFPerSmall>),
        reinterpret_cast<const void*>(&k_sssp_scan_frontier<D, kFPer, true>),
        reinterpret_cast<const void*>(&k_sssp_scan_frontier<D, kFPerSmall, true>),
        reinterpret_cast<const void*>(&k_sssp_multi_relax<D, 16>),
        reinterpret_cast<const void*>(&k_sssp_multi_relax<D, kSmallLpi, kSmallDeg>),
        reinterpret_cast<const void*>(&k_sssp_widen<D>),
        reinterpret_cast<const void*>(&k_multi_gather<D>),
        reinterpret_cast<const void*>(&k_multi_arrive),
        reinterpret_cast<const void*>(&k_multi_wait),
        reinterpret_cast<const void*>(&k_multi_finish),
        reinterpret_cast<const void*>(&k_multi_flag),
        reinterpret_cast<const void*>(&k_multi_reset)};
    for (const void* f : fns) GDX_CUDA(cudaFuncGetAttributes(&fa, f));
}

// One partition of a multi-GPU SSSP: its handle and vertex range, its
// distance replica and barrier state, and this partition's view (device
// tables) of every partition's barrier state.
struct MultiPart {
    gdx_graph* g;
    int32_t v0, v1;
    void* dist;               // 8 B per vertex, read as D
    MultiSync* me;
    MultiSync* const* peers;  // device table [nd]
};

// Every kernel loaded and every loop instantiated, before anything of any
// partition is enqueued (both would wait for another partition's spinning
// barrier on the same GPU).
template <class D>
static void multi_prepare(MultiPart& p, SsspOwners own, int nd, int self) {
    gdx_graph* g = p.g;
    GraphScope sc(g);
    preload_multi_kernels<D>();
    auto& w = *g->sssp;
    const int di = sizeof(D) == 2 ? 2 : sizeof(D) == 4 ? 0 : 1;
    own.self = self;
    int2* squeue = multi_split(g) ? w.small_queue.get() : nullptr;
    D* dist = static_cast<D*>(p.dist);
    D* prev = reinterpret_cast<D*>(w.prev.get());
    const int relax_grid = (g->m < (int64_t(1) << 26) ? 16 : 256) * g->num_sms;  // as gdx_sssp
    // the instantiated loop bakes in this partition's buffers, its range and
    // every partition's replica
    std::vector<void*> key = {dist, prev, w.shard_queue.get(), w.shard_ctr.get(), w.graph_acc.get(),
                              p.me, const_cast<MultiSync**>(p.peers), w.upd_slots.get(),
                              g->offsets.get(), g->dests.get(),
                              g->weighted ? g->weights.get() : nullptr,
                              reinterpret_cast<void*>(intptr_t(p.v0)),
                              reinterpret_cast<void*>(intptr_t(p.v1)), squeue};
    for (int q = 0; q < nd; ++q) key.push_back(own.dist[q]);
    if (!w.mexec[di] || w.mkey[di] != key) {
        if (w.mexec[di]) cudaGraphExecDestroy(w.mexec[di]);
        w.mexec[di] = build_multi_graph<D>(g, dist, prev, p.v0, p.v1, p.me, p.peers, nd, own,
                                           relax_grid, squeue);
        w.mkey[di] = key;
    }
}

// A partition's whole call, enqueued without waiting: init, a barrier (no
// relaxation lands in a replica before it is initialised), the round loop,
// the overflow vote and a barrier, then either its own slice widened into
// out_dev (full = false) or the whole vector gathered from the owners
// followed by a last barrier (nobody re-initialises a replica being read).
template <class D>
static void multi_enqueue(MultiPart& p, SsspOwners own, int nd, int32_t src, bool full,
                          int64_t* out_dev) {
    gdx_graph* g = p.g;
    GraphScope sc(g);
    auto& w = *g->sssp;
    cudaStream_t s = g->stream;
    const int di = sizeof(D) == 2 ? 2 : sizeof(D) == 4 ? 0 : 1;
    const D inf = sizeof(D) < 8 ? std::numeric_limits<D>::max() : D(INT64_MAX / 2);
    const int32_t n = g->n;
    D* dist = static_cast<D*>(p.dist);
    D* prev = reinterpret_cast<D*>(w.prev.get());
    k_multi_reset<<<1, 1, 0, s>>>(p.me);
    timed_launch(g, "sssp_multi_init", [&] {
        k_multi_init<D><<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(
            n, src, inf, dist, prev, w.shard_ctr.get(), kSmallCtr + 1, w.graph_acc.get(), 4,
            w.upd_slots.get());
    });
    k_multi_arrive<<<1, 1, 0, s>>>(nullptr, p.peers, nd);
    k_multi_wait<<<1, 1, 0, s>>>(p.me, nd, 0);
    GDX_LAUNCH_CHECK();
    timed_launch(g, "sssp_multi_graph", [&] { GDX_CUDA(cudaGraphLaunch(w.mexec[di], s)); });
    k_multi_flag<<<1, 1, 0, s>>>(w.graph_acc.get() + 3, p.peers, nd);
    k_multi_arrive<<<1, 1, 0, s>>>(nullptr, p.peers, nd);
    k_multi_wait<<<1, 1, 0, s>>>(p.me, nd, 0);
    GDX_LAUNCH_CHECK();
    if (full) {
        timed_launch(g, "sssp_widen", [&] {
            k_multi_gather<D><<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(
                n, own, inf, out_dev, w.upd_slots.get(), w.shard_ctr.get() + kUpdSlot);
        });
        k_multi_arrive<<<1, 1, 0, s>>>(nullptr, p.peers, nd);
        k_multi_wait<<<1, 1, 0, s>>>(p.me, nd, 0);
    } else {
        timed_launch(g, "sssp_widen", [&] {
            k_sssp_widen<D><<<blocks_for(p.v1 - p.v0, 256, g->num_sms * 8), 256, 0, s>>>(
                p.v1 - p.v0, dist + p.v0, inf, out_dev, w.upd_slots.get(),
                w.shard_ctr.get() + kUpdSlot);
        });
    }
    GDX_LAUNCH_CHECK();
}

struct MultiResult {
    bool overflow = false;
    unsigned long long rounds = 0, vvis = 0, evis = 0, upd = 0;
};

// Waits for a partition's call; its counters, the global overflow vote, and
// a barrier timeout as an error.
static void multi_collect(MultiPart& p, MultiResult& r) {
    gdx_graph* g = p.g;
    GraphScope sc(g);
    auto& w = *g->sssp;
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, w.graph_acc.get(), 4 * 8, cudaMemcpyDeviceToHost, g->stream));
    GDX_CUDA(cudaMemcpyAsync(h + 4, w.shard_ctr.get() + kUpdSlot, 8, cudaMemcpyDeviceToHost,
                             g->stream));
    GDX_CUDA(cudaMemcpyAsync(h + 5, &p.me->err, 8, cudaMemcpyDeviceToHost, g->stream));
    GDX_CUDA(cudaMemcpyAsync(h + 6, &p.me->ovf, 8, cudaMemcpyDeviceToHost, g->stream));
    GDX_CUDA(cudaStreamSynchronize(g->stream));
    if (h[5]) fail(GDX_ERR_CUDA, "CudaError: multi-GPU SSSP barrier timed out");
    r.overflow |= h[6] != 0;
    r.rounds = std::max(r.rounds, h[0]);
    r.vvis += h[1];
    r.evis += h[2];
    r.upd += h[4];
}

static void multi_stats(const MultiResult& r, int nd, gdx_stats* stats, bool split) {
    if (!stats) return;
    stats->rounds = int32_t(r.rounds);
    stats->launches = int32_t(nd * (8 + (split ? 7 : 6) * (r.rounds + 1)));
    stats->vertices_visited = int64_t(r.vvis);
    stats->edges_visited = int64_t(r.evis);
    stats->updates = int64_t(r.upd);
    stats->algorithmic_bytes = 16.0 * r.vvis + 12.0 * r.evis + 8.0 * r.upd;
}

// The workspaces of one partition (everything the loop bakes in).
static void multi_workspace(gdx_graph* g, int32_t v0, int32_t v1) {
    GraphScope sc(g);
    if (!g->sssp) g->sssp = std::make_unique<SsspWork>();
    auto& w = *g->sssp;
    w.prev.ensure(size_t(g->n));
    std::vector<int32_t> off(2, 0);
    if (v1 > v0) {
        GDX_CUDA(cudaMemcpy(&off[0], g->offsets.get() + v0, 4, cudaMemcpyDeviceToHost));
        GDX_CUDA(cudaMemcpy(&off[1], g->offsets.get() + v1, 4, cudaMemcpyDeviceToHost));
    }
    w.shard_queue.ensure(size_t(v1 - v0) + size_t(int64_t(off[1]) - off[0]) / kShardChunk + 1);
    if (multi_split(g)) w.small_queue.ensure(size_t(std::max(v1 - v0, 1)));
    w.shard_ctr.ensure(kSmallCtr + 1);
    w.upd_slots.ensure(kUpdSlots);
    w.graph_acc.ensure(4);
    w.queue[1].ensure(size_t(std::max(v1 - v0, 1)));
}

void sssp_multi(const std::vector<gdx_graph*>& gs, const std::vector<int32_t>& bound, int32_t src,
                int64_t* dist_out, gdx_stats* stats) {
    const int nd = int(gs.size());
    if (nd < 1 || nd > kMaxMultiDev) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: device count");
    std::vector<MultiPart> parts(nd);
    for (int d = 0; d < nd; ++d) {  // workspaces first: every replica's address is needed
        gdx_graph* g = gs[d];
        multi_workspace(g, bound[d], bound[d + 1]);
        GraphScope sc(g);
        auto& w = *g->sssp;
        w.dist.ensure(size_t(g->n));
        if (!w.msync.get()) {
            w.msync.alloc(sizeof(MultiSync) / 8);
            GDX_CUDA(cudaMemset(w.msync.get(), 0, sizeof(MultiSync)));
        }
        parts[d] = MultiPart{g, bound[d], bound[d + 1], w.dist.get(),
                             reinterpret_cast<MultiSync*>(w.msync.get()), nullptr};
    }
    std::vector<MultiSync*> syncs(nd);
    SsspOwners own{};
    own.nd = nd;
    for (int d = 0; d < nd; ++d) {
        syncs[d] = parts[d].me;
        own.dist[d] = parts[d].dist;
    }
    for (int q = 0; q <= nd; ++q) own.bound[q] = bound[q];
    for (int d = 0; d < nd; ++d) {
        GraphScope sc(gs[d]);
        auto& w = *gs[d]->sssp;
        w.mpeers.ensure(nd);
        GDX_CUDA(cudaMemcpy(w.mpeers.get(), syncs.data(), nd * sizeof(void*), cudaMemcpyHostToDevice));
        parts[d].peers = reinterpret_cast<MultiSync* const*>(w.mpeers.get());
    }
    auto width = [&](auto tag) {
        using D = decltype(tag);
        for (int d = 0; d < nd; ++d) multi_prepare<D>(parts[d], own, nd, d);
        for (int d = 0; d < nd; ++d)
            multi_enqueue<D>(parts[d], own, nd, src, false,
                             reinterpret_cast<int64_t*>(gs[d]->sssp->queue[1].get()));
        MultiResult r;
        for (int d = 0; d < nd; ++d) multi_collect(parts[d], r);
        if (!r.overflow) multi_stats(r, nd, stats, multi_split(gs[0]));
        return r.overflow;
    };
    // widths as gdx_sssp: 16-bit first on large graphs, then 32, then 64 (every
    // partition takes the same decision: the overflow vote is global)
    bool ovf = true;
    if (multi_narrow(gs[0])) {
        ovf = width((unsigned short)0);
        if (ovf)
            for (auto* g : gs) g->sssp->multi_narrow_overflowed = true;
    }
    if (ovf && width((unsigned int)0) && width((unsigned long long)0))
        fail(GDX_ERR_RUNTIME, "RuntimeError: distances overflow 64 bits");
    for (int d = 0; d < nd; ++d) {
        gdx_graph* g = gs[d];
        GraphScope sc(g);
        copy_out(g, dist_out + bound[d], g->sssp->queue[1].get(),
                 size_t(bound[d + 1] - bound[d]) * sizeof(int64_t));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    }
}

}  // namespace gdx

// ---------------------------------------------------------------------------
// The same partitioned SSSP with one process per GPU (the
// exchange fused into the relaxation over NVLink peer memory, no NCCL per
// round): every rank exports {replica | barrier state} through CUDA IPC,
// opens every other rank's, and runs its partition of each call with the
// device-side barriers of sssp_multi; the result is gathered from the owners'
// replicas by peer loads.
// ---------------------------------------------------------------------------
using namespace gdx;

static_assert(sizeof(MultiSync) == 64, "barrier state block");

extern "C" int gdx_sssp_p2p_setup(gdx_graph* g, int32_t world, int32_t rank,
                                  const int32_t* bounds, void* handle_out) {
    return guard_impl([&] {
        if (!g || !bounds || !handle_out || world < 1 || world > kMaxMultiDev || rank < 0 ||
            rank >= world)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad sssp p2p setup");
        for (int q = 0; q < world; ++q)
            if (bounds[q] > bounds[q + 1] || bounds[0] != 0 || bounds[world] != g->n)
                fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: vertex ranges must partition [0, n)");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        GraphScope sc(g);
        multi_workspace(g, bounds[rank], bounds[rank + 1]);
        auto X = std::make_unique<SsspP2P>();
        X->world = world;
        X->rank = rank;
        X->n = g->n;
        X->bounds.assign(bounds, bounds + world + 1);
        GDX_CUDA(cudaMalloc(&X->block, X->bytes()));
        GDX_CUDA(cudaMemset(X->block, 0, X->bytes()));
        cudaIpcMemHandle_t h;
        GDX_CUDA(cudaIpcGetMemHandle(&h, X->block));
        std::memcpy(handle_out, &h, sizeof(h));
        g->sssp_p2p = std::move(X);
    });
}

extern "C" int gdx_sssp_p2p_open(gdx_graph* g, const void* handles) {
    return guard_impl([&] {
        if (!g || !g->sssp_p2p || !handles)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no sssp p2p setup");
        GraphScope sc(g);
        auto& X = *g->sssp_p2p;
        X.bases.assign(X.world, nullptr);
        std::vector<void*> syncs(X.world);
        for (int q = 0; q < X.world; ++q) {
            if (q == X.rank) {
                X.bases[q] = X.block;
            } else {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, static_cast<const char*>(handles) + 64 * q, sizeof(h));
                void* p = nullptr;
                GDX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
                X.bases[q] = static_cast<char*>(p);
            }
            syncs[q] = X.bases[q] + size_t(X.n) * 8;
        }
        X.peer_sync.alloc(X.world);
        GDX_CUDA(cudaMemcpy(X.peer_sync.get(), syncs.data(), X.world * sizeof(void*),
                            cudaMemcpyHostToDevice));
    });
}

extern "C" int gdx_sssp_p2p_run(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !g->sssp_p2p || g->sssp_p2p->bases.empty() || !dist_out)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no sssp p2p plan");
        if (src < 0 || src >= g->n)
            fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: node id " + std::to_string(src) +
                                           " out of range [0, " + std::to_string(g->n) + ")");
        GraphScope sc(g);
        auto& X = *g->sssp_p2p;
        const int nd = X.world;
        MultiPart part{g, X.bounds[X.rank], X.bounds[X.rank + 1], X.block,
                       reinterpret_cast<MultiSync*>(X.block + size_t(X.n) * 8),
                       reinterpret_cast<MultiSync* const*>(X.peer_sync.get())};
        SsspOwners own{};
        own.nd = nd;
        for (int q = 0; q < nd; ++q) own.dist[q] = X.bases[q];
        for (int q = 0; q <= nd; ++q) own.bound[q] = X.bounds[q];
        cudaPointerAttributes pa;
        const bool dev_out = cudaPointerGetAttributes(&pa, dist_out) == cudaSuccess &&
                             pa.type == cudaMemoryTypeDevice;
        cudaGetLastError();
        auto& w = *g->sssp;
        if (!dev_out) w.queue[1].ensure(size_t(std::max(g->n, 1)));
        int64_t* target = dev_out ? dist_out : reinterpret_cast<int64_t*>(w.queue[1].get());
        auto width = [&](auto tag) {
            using D = decltype(tag);
            multi_prepare<D>(part, own, nd, X.rank);
            multi_enqueue<D>(part, own, nd, src, true, target);
            MultiResult r;
            multi_collect(part, r);
            if (!r.overflow) multi_stats(r, 1, stats, multi_split(g));
            return r.overflow;
        };
        bool ovf = true;
        if (multi_narrow(g)) {  // every rank takes the same decision (global overflow vote)
            ovf = width((unsigned short)0);
            if (ovf) w.multi_narrow_overflowed = true;
        }
        if (ovf && width((unsigned int)0) && width((unsigned long long)0))
            fail(GDX_ERR_RUNTIME, "RuntimeError: distances overflow 64 bits");
        if (!dev_out) copy_out(g, dist_out, target, size_t(g->n) * sizeof(int64_t));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    });
}

extern "C" int gdx_sssp_p2p_close(gdx_graph* g) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope sc(g);
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        g->sssp_p2p.reset();
    });
}
