// pagerank.cu -- ComputePR (reference corpus/pr.sp:5-33) on sm_100a.
//
// The reference's GPU twin does three launches, three device syncs and four
// small copies per round: a single-address atomicAdd(double) for the dangling
// mass, a thread-per-vertex pull that re-reads the source's out-degree per
// in-edge, and a copy-back kernel (tests/golden/pr/cuda/pr_cuda.cu:117-212).
//
// Here one round is two launches:
//   * k_pr_edges: the reverse-CSR in-edges are cut into aligned groups of 8;
//     a lane loads its group's rev_srcs with two 16 B vector loads and issues
//     its 8 contrib[u] = rank[u] / outdeg(u) gathers back to back.  The row
//     of the group's first edge comes from a precomputed index into the list
//     of non-empty rows (RMAT-24: 56% of rows are empty), so there is no
//     merge-path search and no shared memory; rows finish inside a lane, via a
//     segmented warp-shuffle scan, or -- rows crossing a warp's 256-edge
//     chunk -- as per-chunk head / tail partials that pass B adds in chunk
//     order (no floating-point atomics: results are run-to-run identical).
//     Measured on B200 the gather is limited by the L1->L2 miss-request rate
//     (ncu: l1tex__m_l1tex2xbar_req_cycles_active 87%), so the design keeps
//     every other L1 request to ~1 per 8 edges;
//   * k_pr_vertices: pr.sp:17-30 for every vertex with 16 B vector loads and
//     stores (new rank, |change| >= threshold vote, next contrib, next
//     round's dangling mass), at HBM speed;
//   * rounds are enqueued in batches without host syncs; a round whose
//     predecessor voted "settled" exits immediately on the device.
// Term-wise arithmetic matches pr.sp (contrib is the same f64 quotient the
// interpreter computes per in-edge); only the summation order differs.
#include <cub/cub.cuh>

#include <cstdlib>
#include <cstring>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

constexpr int kPrBlock = 256;
constexpr int kPrCarveout = -1;  // pass A's shared-memory carveout (prefer_l1; -1: the driver's)
constexpr int32_t kFlagRing = 256;  // per-round vote slots (a ring; see clear_flags)
__host__ __device__ inline int32_t flag_slot(int32_t round) { return round & (kFlagRing - 1); }

struct PrArgs {
    int32_t n;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ rev_offsets;
    const int32_t* __restrict__ rev_srcs;
    double* rank0;
    double* rank1;
    double* contrib0;
    double* contrib1;
    double* dangling;  // [3]
    int32_t* flags;
    double damping, threshold, base, nd;
    int32_t max_iter;
    // edge-aligned two-pass plan (k_pr_edges + k_pr_vertices)
    int32_t m, nnz;
    const int2* __restrict__ nz;          // k-th row with in-edges: (vertex, rev_offsets[vertex + 1])
    const int2* __restrict__ grp;         // per 8-edge group: (nz index of its first row, that row's end)
    double* row_sum;                      // per vertex: every non-empty row's sum is stored
                                          // once per round (plain stores, no accumulation),
                                          // empty rows stay 0 from the plan's memset
    // rows crossing a warp chunk (256 in-edges) are summed in pass B from the
    // chunks' partials, in chunk order (deterministic: no atomics)
    double* head_part;                    // per chunk: the row that began in an earlier chunk
    double* tail_part;                    // per chunk: the row that continues into the next
    const int4* __restrict__ cross;       // rows crossing chunks: (row, first chunk, last chunk)
    const int4* __restrict__ cross_long;  // ... spanning more than kCrossShort chunks
    int32_t ncross, nlong;
    double* dang_part;                    // per block of a grid-wide dangling sum
    unsigned int* dang_ctr;               // blocks done (the last one sums dang_part)
    // row range [v_begin, v_end) and its in-edges [e_begin, e_end) (the whole
    // graph on one GPU; one rank's slice when sharded, gdx_pr_shard_*)
    int32_t v_begin, v_end;
    int64_t e_begin, e_end, e_base;       // e_base = e_begin rounded down to 8
    int32_t shard;                        // 1: rounds never skip (the host decides)
    double* contrib_slice;                // shard: contrib_out written at [v - v_begin]
    // peer-memory exchange (gdx_pr_p2p_*): every rank's contrib buffer of the
    // next publish, written directly over NVLink instead of an all-gather
    double* const* peers;
    int32_t npeers;
};


__device__ inline bool round_skipped(const PrArgs& a, int round) {
    return !a.shard && round > 0 &&
           *reinterpret_cast<const volatile int32_t*>(&a.flags[flag_slot(round - 1)]) == 0;
}

// Deterministic grid-wide sum of per-block values: every block stores its
// value in slots[blockIdx.x]; the last block to finish sums the slots in a
// fixed order and writes *out (replaces a float atomicAdd per block, whose
// order -- and so the last bits of the dangling mass -- varied run to run).
template <int BLOCK>
__device__ inline void grid_sum_ordered(double v, double* slots, unsigned int* ctr, double* out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        slots[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += BLOCK) s += __ldcg(&slots[i]);
    typedef cub::BlockReduce<double, BLOCK> R;
    __shared__ typename R::TempStorage tmp;
    const double tot = R(tmp).Sum(s);
    if (threadIdx.x == 0) {
        *out = tot;
        *ctr = 0;  // ready for the next grid
    }
}

template <int BLOCK = kPrBlock>
__device__ inline void block_flush(const PrArgs& a, int round, double dang_local, int unsettled) {
    typedef cub::BlockReduce<double, BLOCK> R;
    __shared__ typename R::TempStorage tmp;
    double tot = R(tmp).Sum(dang_local);
    int any = __syncthreads_or(unsettled);
    if (threadIdx.x == 0 && any) atomicOr(&a.flags[flag_slot(round)], 1);
    grid_sum_ordered<BLOCK>(tot, a.dang_part, a.dang_ctr, &a.dangling[(round + 1) % 3]);
}

// ---------------------------------------------------------------------------
// Edge-aligned two-pass round.
//
// Pass A (k_pr_edges): the in-edge array is cut into aligned groups of 8; a
// lane owns one group, loads its 8 rev_srcs with two 16 B vector loads and
// issues its 8 contrib gathers back to back.  The row of the group's first
// edge comes from a precomputed per-group index into the list of non-empty
// rows, so there is no merge-path search and no shared memory at all: the
// only L1 traffic besides the random gathers is ~1 wavefront per 8 edges.
// Rows finish inside a lane (plain store of the row sum), across lanes of a
// warp (segmented shuffle scan), or across warps (per-chunk partials summed
// in chunk order by pass B).
// Pass B (k_pr_vertices) applies pr.sp:17-30 to every vertex with coalesced
// loads (row_sum needs no clearing: pass A / k_pr_cross store every
// non-empty row's sum exactly once per round).
// ---------------------------------------------------------------------------

constexpr int kEdgeGroup = 8;

// One lane's 8-edge group g (all 32 lanes of the warp call this together
// for 32 consecutive groups).
// R = true: a row range [v_begin, v_end) (sharded); false: the whole graph
// (compile-time zero bases -- keeps the single-GPU kernel at 32 registers).
template <bool R>
__device__ __forceinline__ void pr_edge_group(const PrArgs& a, const double* __restrict__ contrib,
                                              int64_t g) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t e_base = R ? a.e_base : 0, e_begin = R ? a.e_begin : 0;
    const int64_t e_end = R ? a.e_end : int64_t(a.m);
    const int64_t e0 = e_base + g * kEdgeGroup;
    // valid slots k in [klo, khi): edges inside [e_begin, e_end)
    const int64_t dlo = e_begin - e0, dhi = e_end - e0;
    const int klo = dlo <= 0 ? 0 : dlo >= kEdgeGroup ? kEdgeGroup : int(dlo);
    const int khi = dhi <= 0 ? 0 : dhi >= kEdgeGroup ? kEdgeGroup : int(dhi);
    const bool any = khi > klo;
    double v[kEdgeGroup];
    {
        const int4* p = reinterpret_cast<const int4*>(a.rev_srcs + (any ? e0 : 0));
        const int4 q0 = __ldcs(p), q1 = __ldcs(p + 1);
        const int32_t s[kEdgeGroup] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int k = 0; k < kEdgeGroup; ++k)
            v[k] = k >= klo && k < khi ? __ldg(&contrib[s[k]]) : 0.0;
    }
    // grp[g] = (first non-empty row of the group, that row's end): one load
    const int2 gk = any ? a.grp[g] : make_int2(INT32_MAX, 0);
    int32_t key = gk.x;
    const int32_t first = key;
    double run = 0.0, first_val = 0.0;
    bool first_done = false;
    if (any) {
        int32_t end = gk.y, row = -1;  // row of `key` once loaded from nz (not needed for `first`)
#pragma unroll
        for (int k = 0; k < kEdgeGroup; ++k) {
            if (k >= klo && k < khi) {
                while (end <= e0 + k) {  // row `key` ended before edge e0+k
                    if (key == first) {
                        first_val = run;
                        first_done = true;
                    } else {
                        a.row_sum[row] = run;
                    }
                    run = 0.0;
                    const int2 nk = a.nz[++key];  // (row, end) of the next non-empty row
                    row = nk.x;
                    end = nk.y;
                }
                run += v[k];
            }
        }
        if (end <= e0 + khi) {  // the last row ends exactly at the group's end
            if (key == first) {
                first_val = run;
                first_done = true;
            } else {
                a.row_sum[row] = run;
            }
            run = 0.0;
            ++key;
        }
    }
    // segmented inclusive scan of (row, trailing partial) across the warp
    double val = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t k2 = __shfl_up_sync(full, key, o);
        const double v2 = __shfl_up_sync(full, val, o);
        if (lane >= o && k2 == key) val += v2;
    }
    const int32_t pkey = __shfl_up_sync(full, key, 1);
    const double pval = __shfl_up_sync(full, val, 1);
    const int64_t chunk = g >> 5;  // this warp's 256 edges
    if (first_done) {
        const double tot = first_val + (lane > 0 && pkey == first ? pval : 0.0);
        const int64_t warp_e0 = e_base + (g & ~int64_t(31)) * kEdgeGroup;
        const int64_t start = first > 0 ? a.nz[first - 1].y : e_begin;
        if (start < warp_e0)  // the row began in an earlier chunk: k_pr_cross sums it
            a.head_part[chunk] = tot;
        else
            a.row_sum[a.nz[first].x] = tot;
    }
    // the chunk's trailing row continues into the next chunk (written even when
    // zero: pass B reads it for every row crossing the chunk's end)
    if (lane == 31 && key < a.nnz) a.tail_part[chunk] = val;
}


template <bool R>
__global__ void __launch_bounds__(256) k_pr_edges(PrArgs a, int round) {
    if (round_skipped(a, round)) return;
    const double* __restrict__ contrib = (round & 1) ? a.contrib1 : a.contrib0;
    // grid-stride over 256-group block chunks; the grid is capped at 64
    // blocks per SM (measured on B200: 1.05 ms vs 1.13 ms for one chunk per
    // block at RMAT-24); chunks stay warp aligned
    const int64_t ngroups = R ? (a.e_end - a.e_base + kEdgeGroup - 1) / kEdgeGroup
                              : (int64_t(a.m) + kEdgeGroup - 1) / kEdgeGroup;
    for (int64_t g0 = int64_t(blockIdx.x) * blockDim.x; g0 < ngroups;
         g0 += int64_t(gridDim.x) * blockDim.x)
        pr_edge_group<R>(a, contrib, g0 + threadIdx.x);
}

// Rows crossing chunks (between pass A and pass B): a row's sum is tail_part
// of every chunk it leaves plus head_part of the chunk it ends in, added in
// chunk order.  Rows spanning few chunks take a thread each (their loads
// issued together); hub rows (more than kCrossShort chunks) take a warp,
// lanes summing fixed strided subsets combined by a fixed shuffle tree.
// Both orders are fixed, so the sums are run-to-run identical.
constexpr int kCrossShort = 8;
__global__ void __launch_bounds__(256) k_pr_cross(PrArgs a, int round) {
    if (round_skipped(a, round)) return;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < a.ncross; i += nthreads) {
        const int4 c = a.cross[i];  // (row, first chunk, last chunk)
        double t[kCrossShort];
#pragma unroll
        for (int k = 0; k < kCrossShort; ++k) t[k] = c.y + k < c.z ? a.tail_part[c.y + k] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < kCrossShort; ++k) s += t[k];
        a.row_sum[c.x] = s + a.head_part[c.z];
    }
    const int lane = threadIdx.x & 31;
    for (int64_t i = tid >> 5; i < a.nlong; i += nthreads >> 5) {
        const int4 c = a.cross_long[i];
        double s = 0.0;
        for (int64_t k = c.y + lane; k < c.z; k += 32) s += a.tail_part[k];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) a.row_sum[c.x] = s + a.head_part[c.z];
    }
}

// Pass B: two vertices per thread (16 B vector loads/stores), two pairs in
// flight per iteration.  Pairs start at an even vertex; a pair that straddles
// the range bounds (or the array end) takes the scalar path.
__device__ inline void pr_vertex_one(const PrArgs& a, int round, int64_t v, double dang_term,
                                     const double* __restrict__ rank_in,
                                     double* __restrict__ rank_out,
                                     double* __restrict__ contrib_out, double& dang_local,
                                     int& unsettled) {
    const double sum = a.row_sum[v];  // stored this round (or 0: no in-edges)
    const double nr = a.base + a.damping * (dang_term + sum);
    double c = nr - rank_in[v];
    if (c < 0.0) c = 0.0 - c;
    if (c >= a.threshold && round < a.max_iter) unsettled = 1;
    rank_out[v] = nr;
    const int32_t d = a.offsets[v + 1] - a.offsets[v];
    const double cv = d > 0 ? nr / double(d) : 0.0;
    if (a.npeers > 0) {
        // P2P stores over NVLink; a vertex without out-edges is never gathered
        // (no in-edge has it as source), so its contrib is not sent (56% of
        // RMAT-24's vertices: that much less NVLink traffic per round)
        if (d > 0)
            for (int q = 0; q < a.npeers; ++q) a.peers[q][v] = cv;
    } else {
        contrib_out[v] = cv;
    }
    if (d == 0) dang_local += nr;
}

template <bool R>
__device__ inline void pr_vertex_pair(const PrArgs& a, int round, int64_t v, double dang_term,
                                      const double* __restrict__ rank_in,
                                      double* __restrict__ rank_out,
                                      double* __restrict__ contrib_out, double& dang_local,
                                      int& unsettled) {
    const int64_t vb = R ? a.v_begin : 0, ve = R ? a.v_end : a.n;
    // a pair inside the range takes the vector path; a shard's contrib slice
    // is 16 B aligned at the pair only when v_begin is even (peer buffers are
    // whole-graph arrays, always aligned at an even v)
    const bool vec = R ? v >= vb && v + 1 < ve && (a.npeers > 0 || (a.v_begin & 1) == 0)
                       : v + 1 < ve;
    if (vec) {
        const double2 sum = *reinterpret_cast<const double2*>(a.row_sum + v);
        const double2 ri = *reinterpret_cast<const double2*>(rank_in + v);
        const int32_t o0 = a.offsets[v], o1 = a.offsets[v + 1], o2 = a.offsets[v + 2];
        const double nr0 = a.base + a.damping * (dang_term + sum.x);
        const double nr1 = a.base + a.damping * (dang_term + sum.y);
        double c0 = nr0 - ri.x, c1 = nr1 - ri.y;
        if (c0 < 0.0) c0 = 0.0 - c0;
        if (c1 < 0.0) c1 = 0.0 - c1;
        if ((c0 >= a.threshold || c1 >= a.threshold) && round < a.max_iter) unsettled = 1;
        *reinterpret_cast<double2*>(rank_out + v) = make_double2(nr0, nr1);
        const int32_t d0 = o1 - o0, d1 = o2 - o1;
        const double2 cc =
            make_double2(d0 > 0 ? nr0 / double(d0) : 0.0, d1 > 0 ? nr1 / double(d1) : 0.0);
        if (R && a.npeers > 0) {
            // P2P stores over NVLink; a pair without out-edges is never
            // gathered, so it is not sent
            if (d0 > 0 || d1 > 0)
                for (int q = 0; q < a.npeers; ++q) __stcg(reinterpret_cast<double2*>(a.peers[q] + v), cc);
        } else {
            *reinterpret_cast<double2*>(contrib_out + v) = cc;
        }
        if (d0 == 0) dang_local += nr0;
        if (d1 == 0) dang_local += nr1;
    } else {
        for (int64_t x = v; x < v + 2; ++x)
            if (x >= vb && x < ve)
                pr_vertex_one(a, round, x, dang_term, rank_in, rank_out, contrib_out, dang_local,
                              unsettled);
    }
}

template <bool R>
__device__ __forceinline__ void pr_vertices_body(const PrArgs& a, int round) {
    if (round_skipped(a, round)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.dangling[(round + 2) % 3] = 0.0;
    const double dang_in = *reinterpret_cast<const volatile double*>(&a.dangling[round % 3]);
    const double dang_term = dang_in / a.nd;
    const double* __restrict__ rank_in = (round & 1) ? a.rank1 : a.rank0;
    double* __restrict__ rank_out = (round & 1) ? a.rank0 : a.rank1;
    double* __restrict__ contrib_out =
        R ? a.contrib_slice - a.v_begin : ((round & 1) ? a.contrib0 : a.contrib1);
    double dang_local = 0.0;
    int unsettled = 0;
    const int64_t v_al = R ? a.v_begin & ~int64_t(1) : 0;
    const int64_t ve = R ? a.v_end : a.n;
    const int64_t stride = (int64_t)gridDim.x * kPrBlock * 2;
    for (int64_t v = v_al + (blockIdx.x * (int64_t)kPrBlock + threadIdx.x) * 2; v < ve;
         v += 2 * stride) {
        pr_vertex_pair<R>(a, round, v, dang_term, rank_in, rank_out, contrib_out, dang_local,
                          unsettled);
        if (v + stride < ve)
            pr_vertex_pair<R>(a, round, v + stride, dang_term, rank_in, rank_out, contrib_out,
                              dang_local, unsettled);
    }
    block_flush(a, round, dang_local, unsettled);
}

template <bool R>
__global__ void __launch_bounds__(kPrBlock) k_pr_vertices(PrArgs a, int round) {
    pr_vertices_body<R>(a, round);
    if (R && a.npeers > 0) __threadfence_system();  // P2P stores performed before the publish
}

// Non-empty rows of the reverse CSR and the row of every 8-edge group.
__global__ void k_pr_nz_flags(int32_t v0, int32_t cnt, const int32_t* __restrict__ rev_offsets,
                              int32_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = rev_offsets[v0 + i + 1] > rev_offsets[v0 + i];
}
__global__ void k_pr_nz_fill(int32_t v0, int32_t cnt, const int32_t* __restrict__ rev_offsets,
                             const int32_t* __restrict__ pos, int2* nz) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = v0 + i;
        if (rev_offsets[v + 1] > rev_offsets[v]) {
            nz[pos[i]] = make_int2(int32_t(v), rev_offsets[v + 1]);
        }
    }
}
__global__ void k_pr_grp_rows(int64_t ngroups, int64_t e_base, int64_t e_begin, int32_t nnz,
                              const int2* __restrict__ nz, int2* grp) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = max(e_base + g * kEdgeGroup, e_begin);
        int32_t lo = 0, hi = nnz;  // first k whose row ends after edge e
        while (lo < hi) {
            const int32_t mid = lo + ((hi - lo) >> 1);
            if (nz[mid].y <= e)
                lo = mid + 1;
            else
                hi = mid;
        }
        grp[g] = make_int2(lo, lo < nnz ? nz[lo].y : 0);
    }
}

// The same index filled from the rows: row k owns the groups whose first edge
// lies in [start_k, end_k) -- no binary search.  A lane takes a row; rows with
// more than 32 groups (hubs) are written by the whole warp.
__global__ void k_pr_grp_fill(int64_t ngroups, int64_t e_base, int64_t e_begin, int32_t nnz,
                              const int2* __restrict__ nz, int2* grp) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; k0 < nnz;
         k0 += nw * 32) {
        const int64_t k = k0 + lane;
        int64_t g0 = 0, g1 = 0;
        int32_t end = 0;
        if (k < nnz) {
            const int64_t start = k > 0 ? nz[k - 1].y : e_begin;
            end = nz[k].y;
            // group g's first edge: e_begin for g = 0, e_base + 8 g after
            g0 = k == 0 ? 0 : (start - e_base + kEdgeGroup - 1) / kEdgeGroup;
            g1 = min((int64_t(end) - e_base + kEdgeGroup - 1) / kEdgeGroup, ngroups);
        }
        const bool big = g1 - g0 > 32;
        if (!big)
            for (int64_t g = g0; g < g1; ++g) grp[g] = make_int2(int32_t(k), end);
        unsigned hubs = __ballot_sync(full, big);
        while (hubs) {
            const int l = __ffs(hubs) - 1;
            hubs &= hubs - 1;
            const int64_t h0 = __shfl_sync(full, g0, l), h1 = __shfl_sync(full, g1, l);
            const int32_t hk = int32_t(__shfl_sync(full, k, l)), he = __shfl_sync(full, end, l);
            for (int64_t g = h0 + lane; g < h1; g += 32) grp[g] = make_int2(hk, he);
        }
    }
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
    grid_sum_ordered<kPrBlock>(tot, a.dang_part, a.dang_ctr, &a.dangling[0]);
}

// The rows whose in-edges cross a 256-edge chunk boundary (k_pr_cross).
__global__ void k_pr_cross_list(int32_t nnz, const int2* __restrict__ nz, int64_t e_begin,
                                int64_t e_base, int4* cross, int4* cross_long, int32_t* count) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t start = k > 0 ? nz[k - 1].y : e_begin, end = nz[k].y;
        const int32_t c0 = int32_t((start - e_base) >> 8), c1 = int32_t((end - 1 - e_base) >> 8);
        if (c1 - c0 > kCrossShort)
            cross_long[atomicAdd(count + 1, 1)] = make_int4(nz[k].x, c0, c1, 0);
        else if (c0 != c1)
            cross[atomicAdd(count, 1)] = make_int4(nz[k].x, c0, c1, 0);
    }
}

// Edge-aligned plan for the rows [v_begin, v_end) (the whole graph, or one
// rank's slice under gdx_pr_shard_setup).
static void build_edge_plan(gdx_graph* g, PrPlan& P, int32_t v_begin, int32_t v_end) {
    cudaStream_t s = g->stream;
    const int32_t n = g->n;
    const int32_t cnt = v_end - v_begin;
    int32_t eb[2] = {0, 0};
    GDX_CUDA(cudaMemcpyAsync(&eb[0], g->in_offsets() + v_begin, 4, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemcpyAsync(&eb[1], g->in_offsets() + v_end, 4, cudaMemcpyDeviceToHost, s));
    const int grid = blocks_for(std::max(cnt, 1), 256, g->num_sms * 16);
    DevBuf<int32_t> flag(std::max(cnt, 1)), pos(std::max(cnt, 1));
    int32_t last[2] = {0, 0};
    if (cnt > 0) {
        k_pr_nz_flags<<<grid, 256, 0, s>>>(v_begin, cnt, g->in_offsets(), flag.get());
        GDX_LAUNCH_CHECK();
        size_t bytes = 0;
        GDX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag.get(), pos.get(), cnt, s));
        DevBuf<uint8_t> tmp(bytes);
        GDX_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, flag.get(), pos.get(), cnt, s));
        GDX_CUDA(cudaMemcpyAsync(&last[0], pos.get() + cnt - 1, 4, cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaMemcpyAsync(&last[1], flag.get() + cnt - 1, 4, cudaMemcpyDeviceToHost, s));
    }
    GDX_CUDA(cudaStreamSynchronize(s));
    P.v_begin = v_begin;
    P.v_end = v_end;
    P.e_begin = eb[0];
    P.e_end = eb[1];
    P.e_base = P.e_begin & ~int64_t(kEdgeGroup - 1);
    P.nnz = last[0] + last[1];
    P.nz.alloc(size_t(P.nnz) + 1);
    if (cnt > 0) {
        k_pr_nz_fill<<<grid, 256, 0, s>>>(v_begin, cnt, g->in_offsets(), pos.get(),
                                          P.nz.get());
        GDX_LAUNCH_CHECK();
    }
    P.ngroups = (P.e_end - P.e_base + kEdgeGroup - 1) / kEdgeGroup;
    P.grp.alloc(size_t(P.ngroups) + 1);
    if (P.ngroups > 0) {
        if (std::getenv("GDX_PR_GRP_SEARCH"))  // A/B: one binary search per group
            k_pr_grp_rows<<<blocks_for(P.ngroups, 256, g->num_sms * 16), 256, 0, s>>>(
                P.ngroups, P.e_base, P.e_begin, P.nnz, P.nz.get(), P.grp.get());
        else
            k_pr_grp_fill<<<blocks_for(int64_t(P.nnz), 256, g->num_sms * 16), 256, 0, s>>>(
                P.ngroups, P.e_base, P.e_begin, P.nnz, P.nz.get(), P.grp.get());
        GDX_LAUNCH_CHECK();
    }
    P.row_sum.alloc(n);
    GDX_CUDA(cudaMemsetAsync(P.row_sum.get(), 0, P.row_sum.bytes(), s));
    const int64_t chunks = (P.ngroups + 31) / 32 + 1;
    P.head_part.alloc(size_t(chunks));
    P.tail_part.alloc(size_t(chunks));
    // rows crossing a 256-edge chunk: at most one ends in each chunk
    P.cross.alloc(size_t(chunks));
    P.cross_long.alloc(size_t(chunks));
    {
        DevBuf<int32_t> nc(2);
        GDX_CUDA(cudaMemsetAsync(nc.get(), 0, 8, s));
        if (P.nnz > 0) {
            k_pr_cross_list<<<blocks_for(P.nnz, 256, g->num_sms * 16), 256, 0, s>>>(
                P.nnz, P.nz.get(), P.e_begin, P.e_base, P.cross.get(), P.cross_long.get(),
                nc.get());
            GDX_LAUNCH_CHECK();
        }
        int32_t h[2] = {0, 0};
        GDX_CUDA(cudaMemcpyAsync(h, nc.get(), 8, cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        P.ncross = h[0];
        P.nlong = h[1];
    }

    P.dang_part.alloc(size_t(g->num_sms) * 8 + 8);  // >= every pass-B / init grid
    P.dang_ctr.alloc(1);
    GDX_CUDA(cudaMemsetAsync(P.dang_ctr.get(), 0, 4, s));
    for (int i = 0; i < 2; ++i) {
        P.rank[i].alloc(n);
        P.contrib[i].alloc(n);
    }
    P.dangling.alloc(3);
    P.block = 256;
    const char* cap = std::getenv("GDX_PR_GRID_CAP");  // blocks per SM of pass A (A/B)
    P.grid = blocks_for(std::max<int64_t>(P.ngroups, 1), 256,
                        (cap ? std::max(1, std::atoi(cap)) : 64) * g->num_sms);
    GDX_CUDA(cudaStreamSynchronize(s));
}

static void build_plan(gdx_graph* g) { build_edge_plan(g, *g->pr, 0, g->n); }

// The crossing rows' sums of a round (between pass A and pass B); 1 if launched.
static int launch_cross(gdx_graph* g, PrPlan& P, const PrArgs& a, int round) {
    if (P.ncross == 0 && P.nlong == 0) return 0;
    const int64_t work = std::max<int64_t>(P.ncross, int64_t(P.nlong) * 32);
    timed_launch(g, "pr_cross", [&] {
        k_pr_cross<<<blocks_for(work, 256, g->num_sms * 32), 256, 0, g->stream>>>(a, round);
    });
    return 1;
}


// The per-round "unsettled" votes live in a ring of kFlagRing slots (a round
// reads only its predecessor's slot; the host reads a batch of at most
// kFlagRing / 2 rounds after it completes), so maxIter does not size memory.
static void clear_flags(PrPlan& P, int64_t first, int64_t count, cudaStream_t s) {
    P.flags.ensure(kFlagRing);
    while (count > 0) {
        const int32_t slot = flag_slot(int32_t(first));
        const int64_t run = std::min<int64_t>(count, kFlagRing - slot);
        GDX_CUDA(cudaMemsetAsync(P.flags.get() + slot, 0, size_t(run) * 4, s));
        first += run;
        count -= run;
    }
}

static PrArgs make_args(gdx_graph* g, PrPlan& P, double damping, double threshold,
                        int32_t max_iter) {
    P.flags.ensure(kFlagRing);
    PrArgs a;
    a.n = g->n;
    a.offsets = g->offsets.get();
    a.rev_offsets = g->in_offsets();
    a.rev_srcs = g->in_srcs();
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
    a.m = g->m;
    a.nnz = P.nnz;
    a.nz = P.nz.get();
    a.grp = P.grp.get();
    a.row_sum = P.row_sum.get();
    a.head_part = P.head_part.get();
    a.tail_part = P.tail_part.get();
    a.cross = P.cross.get();
    a.cross_long = P.cross_long.get();
    a.ncross = P.ncross;
    a.nlong = P.nlong;
    a.dang_part = P.dang_part.get();
    a.dang_ctr = P.dang_ctr.get();
    a.v_begin = P.shard ? P.v_begin : 0;
    a.v_end = P.shard ? P.v_end : g->n;
    a.e_begin = P.e_begin;
    a.e_end = P.e_end;
    a.e_base = P.e_base;
    a.shard = P.shard ? 1 : 0;
    a.contrib_slice = nullptr;
    a.peers = nullptr;
    a.npeers = 0;
    return a;
}

// Sharded rounds (gdx_pr_shard_*): rank = 1/n, contrib and the dangling mass
// of the slice [v_begin, v_end).
__global__ void __launch_bounds__(kPrBlock) k_pr_shard_init(PrArgs a, double* partials) {
    double dang_local = 0.0;
    const double r0 = 1.0 / a.nd;
    for (int64_t v = a.v_begin + blockIdx.x * (int64_t)kPrBlock + threadIdx.x; v < a.v_end;
         v += (int64_t)gridDim.x * kPrBlock) {
        a.rank0[v] = r0;
        const int32_t od = a.offsets[v + 1] - a.offsets[v];
        const double cv = od > 0 ? r0 / double(od) : 0.0;
        if (a.npeers > 0)
            for (int q = 0; q < a.npeers; ++q) a.peers[q][v] = cv;
        else
            a.contrib_slice[v - a.v_begin] = cv;
        if (od == 0) dang_local += r0;
    }
    typedef cub::BlockReduce<double, kPrBlock> R;
    __shared__ typename R::TempStorage tmp;
    double tot = R(tmp).Sum(dang_local);
    grid_sum_ordered<kPrBlock>(tot, a.dang_part, a.dang_ctr, &partials[0]);
    if (a.npeers > 0) __threadfence_system();
}

__global__ void k_pr_shard_partials(const double* dangling, const int32_t* flags, int round,
                                    double* partials) {
    partials[0] = dangling[(round + 1) % 3];
    partials[1] = flags[flag_slot(round)] ? 1.0 : 0.0;
}

}  // namespace gdx

using namespace gdx;

// The fixedPoint rounds on g; returns the device rank vector of the last
// round (the plan's buffer) and the round count.
static const double* pagerank_run(gdx_graph* g, double damping, double threshold,
                                  int32_t max_iter, int32_t* rounds_out, gdx_stats* stats) {
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
    PrArgs a = make_args(g, P, damping, threshold, max_iter);
    prefer_l1(reinterpret_cast<const void*>(&k_pr_edges<false>), kPrCarveout);

    GDX_CUDA(cudaMemsetAsync(P.dangling.get(), 0, 3 * sizeof(double), s));
    int launches = 0;
    timed_launch(g, "pr_init", [&] {
        k_pr_init<<<blocks_for(g->n, kPrBlock, g->num_sms * 8), kPrBlock, 0, s>>>(a);
    });
    ++launches;
    int32_t* hflags = reinterpret_cast<int32_t*>(g->pinned);
    int64_t r = 0, rounds = -1, batch = 4;
    while (rounds < 0) {
        const int64_t lim = std::min(r + batch, limit);
        clear_flags(P, r, lim - r, s);
        for (int64_t rr = r; rr < lim; ++rr) {
            if (P.ngroups > 0)
                timed_launch(g, "pr_edges", [&] {
                    k_pr_edges<false><<<P.grid, P.block, 0, s>>>(a, int(rr));
                });
            launches += launch_cross(g, P, a, int(rr));
            timed_launch(g, "pr_vertices", [&] {
                k_pr_vertices<false><<<blocks_for(g->n, kPrBlock, g->num_sms * 8), kPrBlock,
                                       0, s>>>(a, int(rr));
            });
            launches += 1 + (P.ngroups > 0);
        }
        const int64_t cnt = lim - r;
        GDX_CUDA(cudaMemcpyAsync(hflags, P.flags.get(), kFlagRing * 4, cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < cnt; ++i)
            if (hflags[flag_slot(int32_t(r + i))] == 0) {
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
    if (rounds_out) *rounds_out = int32_t(rounds);
    if (stats) {
        stats->rounds = int32_t(rounds);
        stats->launches = launches;
        stats->vertices_visited = int64_t(g->n) * rounds;
        stats->edges_visited = int64_t(g->m) * rounds;
        stats->updates = 0;
        // SURVEY.md 8(d), per round 12 m + 24 n: rev_srcs 4m + contrib
        // gather 8m; rev_offsets 4n + rank read 8n + new rank / contrib
        // write 8n + out-degree 4n.
        stats->algorithmic_bytes = double(rounds) * (12.0 * g->m + 24.0 * g->n);
    }
    return P.rank[rounds & 1].get();
}

extern "C" int gdx_pagerank(gdx_graph* g, double damping, double threshold, int32_t max_iter,
                            double* rank_out, int32_t* rounds_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || !rank_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        // pr.sp:9 evaluates 1.0 / numNodes (interpreter.cpp:454-456 raises on 0).
        if (g->n == 0) fail(GDX_ERR_RUNTIME, "RuntimeError: division by zero");
        if (!g->in_offsets() || !g->in_srcs())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        GraphScope dg(g);
        const size_t bytes = size_t(g->n) * sizeof(double);
        Relabel* RP = relabel_wanted(g) ? relabel_try(g, false, true) : nullptr;
        if (RP) {
            // the rounds on the degree-ordered renumbering (relabel.cu), the
            // ranks mapped back: rank_out[v] = rank'[newid[v]]
            Relabel& R = *RP;
            const double* r = pagerank_run(R.h, damping, threshold, max_iter, rounds_out, stats);
            relabel_leave(g);
            cudaPointerAttributes pa;
            const bool dev_out = cudaPointerGetAttributes(&pa, rank_out) == cudaSuccess &&
                                 pa.type == cudaMemoryTypeDevice;
            cudaGetLastError();
            if (!dev_out) R.staging.ensure(size_t(g->n));
            double* tgt = dev_out ? rank_out : R.staging.get();
            timed_launch(g, "pr_unpermute", [&] { relabel_unpermute_f64(g, r, tgt); });
            if (!dev_out) copy_out(g, rank_out, tgt, bytes);
            if (stats) stats->launches += 1;
        } else {
            copy_out(g, rank_out, pagerank_run(g, damping, threshold, max_iter, rounds_out, stats),
                     bytes);
        }
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    });
}

// ---------------------------------------------------------------------------
// Sharded PageRank: one rank of a destination-vertex-range partition
// (SURVEY.md §8(e)); the caller owns the exchange (all-gather of the contrib
// slices, all-reduce of the partials) -- see distributed.py sharded_pr.
// ---------------------------------------------------------------------------
extern "C" int gdx_pr_shard_setup(gdx_graph* g, int32_t v_begin, int32_t v_end) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (v_begin < 0 || v_end > g->n || v_begin > v_end)
            fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: vertex range out of bounds");
        if (!g->in_offsets() || !g->in_srcs())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        GraphScope dg(g);
        g->pr_shard = std::make_unique<PrPlan>();
        g->pr_shard->shard = true;
        build_edge_plan(g, *g->pr_shard, v_begin, v_end);
        g->pr_shard->partials.alloc(2);
    });
}

extern "C" int gdx_pr_shard_init(gdx_graph* g, double* contrib_slice, double* partials) {
    return guard_impl([&] {
        if (!g || !g->pr_shard) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
        if (g->n == 0) fail(GDX_ERR_RUNTIME, "RuntimeError: division by zero");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        cudaStream_t s = g->stream;
        PrArgs a = make_args(g, P, 0.85, 0.0, 0);
        a.contrib_slice = contrib_slice;
        GDX_CUDA(cudaMemsetAsync(partials, 0, 2 * sizeof(double), s));
        GDX_CUDA(cudaMemsetAsync(P.dangling.get(), 0, 3 * sizeof(double), s));
        if (P.v_end > P.v_begin)
            timed_launch(g, "pr_init", [&] {
                k_pr_shard_init<<<blocks_for(P.v_end - P.v_begin, kPrBlock, g->num_sms * 8),
                                  kPrBlock, 0, s>>>(a, partials);
            });
        GDX_CUDA(cudaStreamSynchronize(s));
    });
}

extern "C" int gdx_pr_shard_round(gdx_graph* g, int32_t round, double damping, double threshold,
                                  int32_t max_iter, const double* dangling_in,
                                  const double* contrib_in, double* contrib_slice,
                                  double* partials) {
    return guard_impl([&] {
        if (!g || !g->pr_shard) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
        if (round < 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: negative round");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        cudaStream_t s = g->stream;
        PrArgs a = make_args(g, P, damping, threshold, max_iter);
        a.contrib0 = a.contrib1 = const_cast<double*>(contrib_in);
        a.contrib_slice = contrib_slice;
        GDX_CUDA(cudaMemcpyAsync(P.dangling.get() + round % 3, dangling_in, sizeof(double),
                                 cudaMemcpyDefault, s));
        clear_flags(P, round, 1, s);
        if (P.ngroups > 0)
            timed_launch(g, "pr_edges", [&] {
                k_pr_edges<true><<<P.grid, P.block, 0, s>>>(a, round);
            });
        launch_cross(g, P, a, round);
        timed_launch(g, "pr_vertices", [&] {
            k_pr_vertices<true><<<blocks_for(std::max(P.v_end - P.v_begin, 1), 2 * kPrBlock,
                                       g->num_sms * 8),
                            kPrBlock, 0, s>>>(a, round);
        });
        k_pr_shard_partials<<<1, 1, 0, s>>>(P.dangling.get(), P.flags.get(), round, partials);
        GDX_LAUNCH_CHECK();
    });
}

extern "C" int gdx_pr_shard_rank(gdx_graph* g, int32_t rounds, double* rank_slice) {
    return guard_impl([&] {
        if (!g || !g->pr_shard || !rank_slice)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        copy_out(g, rank_slice, P.rank[rounds & 1].get() + P.v_begin,
                 size_t(P.v_end - P.v_begin) * sizeof(double));
        GDX_CUDA(cudaStreamSynchronize(g->stream));
    });
}

// ---------------------------------------------------------------------------
// Sharded PageRank with the exchange fused into the kernels over peer memory
// (one process per GPU, NVLink P2P through CUDA IPC).  Every rank exports one
// device block {contrib[2][n] | partials[2][world][2] | counter}; pass B stores
// each new contrib value straight into every rank's block (no all-gather), a
// one-thread publish kernel writes the rank's (dangling, unsettled) partials
// into every rank's slot and bumps every rank's counter with a system-scope
// atomic, and the next round's first kernel waits on the local counter.
// Publish j uses contrib/partial parity j & 1: a rank can be at most one
// publish ahead of any other (each wait needs all ranks' previous publish),
// so a parity is never rewritten while a slower rank still reads it.
// ---------------------------------------------------------------------------
namespace gdx {

// Spins until the local counter reaches `target`; gives up after ~20 s (a
// rank died or the peer writes never land) and flags *err instead of hanging.
__global__ void k_p2p_wait(const unsigned long long* ctr, unsigned long long target, int* err) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*reinterpret_cast<const volatile unsigned long long*>(ctr) < target) {
        __nanosleep(256);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {
            *err = 1;
            break;
        }
    }
    __threadfence_system();
}

__global__ void k_p2p_publish(const double* dang, const int32_t* unsettled, double* const* slots,
                              unsigned long long* const* ctrs, int world) {
    const double d = dang ? *dang : 0.0;
    const double u = unsettled && *unsettled ? 1.0 : 0.0;
    for (int q = 0; q < world; ++q) {
        slots[q][0] = d;
        slots[q][1] = u;
    }
    __threadfence_system();
    for (int q = 0; q < world; ++q) atomicAdd_system(ctrs[q], 1ull);
}

// Device-side end of a peer-memory round (gdx_pr_p2p_rounds): wait until
// every rank's publish `target / world - 1` has landed, then sum the published
// (dangling, unsettled) slots in rank order -- identical on every rank -- into
// the next round's dangling mass and this round's global vote, which the next
// round's kernels read to exit early once the ranks have settled.
__global__ void k_p2p_combine(const unsigned long long* ctr, unsigned long long target, int* err,
                              const double* slots, int world, double* dangling_next,
                              int32_t* vote) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*reinterpret_cast<const volatile unsigned long long*>(ctr) < target) {
        __nanosleep(256);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {
            *err = 1;
            break;
        }
    }
    __threadfence_system();
    const volatile double* vs = slots;
    double d = 0.0, u = 0.0;
    for (int q = 0; q < world; ++q) {
        d += vs[2 * q];
        u += vs[2 * q + 1];
    }
    *dangling_next = d;
    *vote = u != 0.0 ? 1 : 0;
}

}  // namespace gdx

using namespace gdx;

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");

// Device tables of every rank's contrib buffers / partial slots / counters.
static void p2p_tables(PrP2P& X) {
    std::vector<double*> pc(2 * X.world), ps(2 * X.world);
    std::vector<unsigned long long*> pk(X.world);
    for (int q = 0; q < X.world; ++q) {
        double* b = X.bases[q];
        for (int par = 0; par < 2; ++par) {
            pc[par * X.world + q] = b + par * X.n;
            ps[par * X.world + q] = b + 2 * X.n + (par * X.world + X.rank) * 2;
        }
        pk[q] = reinterpret_cast<unsigned long long*>(b + 2 * X.n + 4 * X.world);
    }
    X.peer_contrib.alloc(pc.size());
    X.peer_slot.alloc(ps.size());
    X.peer_ctr.alloc(pk.size());
    GDX_CUDA(cudaMemcpy(X.peer_contrib.get(), pc.data(), pc.size() * sizeof(double*), cudaMemcpyHostToDevice));
    GDX_CUDA(cudaMemcpy(X.peer_slot.get(), ps.data(), ps.size() * sizeof(double*), cudaMemcpyHostToDevice));
    GDX_CUDA(cudaMemcpy(X.peer_ctr.get(), pk.data(), pk.size() * sizeof(void*), cudaMemcpyHostToDevice));
    X.err.alloc(1);
    GDX_CUDA(cudaMemset(X.err.get(), 0, sizeof(int)));
}

extern "C" int gdx_pr_p2p_setup(gdx_graph* g, int32_t world, int32_t rank, void* handle_out) {
    return guard_impl([&] {
        if (!g || !g->pr_shard || !handle_out || world < 1 || rank < 0 || rank >= world)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad p2p setup (call gdx_pr_shard_setup first)");
        GraphScope dg(g);
        auto X = std::make_unique<PrP2P>();
        X->world = world;
        X->rank = rank;
        X->n = g->n;
        GDX_CUDA(cudaMalloc(&X->block, X->bytes()));  // IPC export needs a plain cudaMalloc block
        GDX_CUDA(cudaMemset(X->block, 0, X->bytes()));
        cudaIpcMemHandle_t h;
        GDX_CUDA(cudaIpcGetMemHandle(&h, X->block));
        std::memcpy(handle_out, &h, sizeof(h));
        g->pr_p2p = std::move(X);
    });
}

extern "C" int gdx_pr_p2p_open(gdx_graph* g, const void* handles) {
    return guard_impl([&] {
        if (!g || !g->pr_p2p || !handles) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no p2p setup");
        GraphScope dg(g);
        auto& X = *g->pr_p2p;
        X.bases.assign(X.world, nullptr);
        for (int q = 0; q < X.world; ++q) {
            if (q == X.rank) {
                X.bases[q] = X.block;
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + 64 * q, sizeof(h));
            void* p = nullptr;
            GDX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            X.bases[q] = static_cast<double*>(p);
        }
        p2p_tables(X);
    });
}

namespace gdx {
// In-process peers (gdx_pagerank_multi): the exchange blocks of the other
// devices of a context are plain device pointers (peer access enabled), not
// IPC mappings.  Same protocol and kernels as the one-process-per-GPU path.
void pr_p2p_local_setup(gdx_graph* g, int32_t world, int32_t rank) {
    GraphScope dg(g);
    if (!g->pr_shard) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no shard plan");
    auto X = std::make_unique<PrP2P>();
    X->world = world;
    X->rank = rank;
    X->n = g->n;
    X->ipc = false;
    // everything the rounds allocate, allocated now: when several partitions
    // share one GPU, an allocation made while another partition's wait kernel
    // spins would serialise behind it (implicit synchronisation)
    g->pr_shard->flags.ensure(kFlagRing);
    // and every kernel of the rounds loaded (lazy module loading would wait
    // for a spinning wait kernel of another partition of the same GPU)
    {
        cudaFuncAttributes fa;
        const void* fns[] = {reinterpret_cast<const void*>(&k_pr_shard_init),
                             reinterpret_cast<const void*>(&k_pr_edges<true>),
                             reinterpret_cast<const void*>(&k_pr_cross),
                             reinterpret_cast<const void*>(&k_pr_vertices<true>),
                             reinterpret_cast<const void*>(&k_p2p_wait),
                             reinterpret_cast<const void*>(&k_p2p_publish),
                             reinterpret_cast<const void*>(&k_p2p_combine)};
        for (const void* f : fns) GDX_CUDA(cudaFuncGetAttributes(&fa, f));
    }
    GDX_CUDA(cudaMalloc(&X->block, X->bytes()));
    GDX_CUDA(cudaMemset(X->block, 0, X->bytes()));
    g->pr_p2p = std::move(X);
}

double* pr_p2p_block(gdx_graph* g) { return g->pr_p2p ? g->pr_p2p->block : nullptr; }

void pr_p2p_local_open(gdx_graph* g, const std::vector<double*>& blocks) {
    GraphScope dg(g);
    auto& X = *g->pr_p2p;
    X.bases = blocks;
    p2p_tables(X);
}
}  // namespace gdx

// Waits for every rank's publish `j`, then sums the partial slots of parity j & 1.
static void p2p_gather_partials(gdx_graph* g, PrP2P& X, int64_t j, double* out2) {
    cudaStream_t s = g->stream;
    k_p2p_wait<<<1, 1, 0, s>>>(X.own_ctr(), (unsigned long long)(j + 1) * X.world, X.err.get());
    GDX_LAUNCH_CHECK();
    std::vector<double> h(2 * X.world);
    int herr = 0;
    GDX_CUDA(cudaMemcpyAsync(h.data(), X.own_partials(int(j & 1)), h.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaMemcpyAsync(&herr, X.err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    if (herr)
        fail(GDX_ERR_CUDA, "CudaError: peer-memory exchange timed out (publish " +
                               std::to_string(j) + ")");
    out2[0] = out2[1] = 0.0;
    for (int q = 0; q < X.world; ++q) {  // rank order: identical sums on every rank
        out2[0] += h[2 * q];
        out2[1] += h[2 * q + 1];
    }
}

extern "C" int gdx_pr_p2p_init(gdx_graph* g, double* partials_out) {
    return guard_impl([&] {
        if (!g || !g->pr_shard || !g->pr_p2p || g->pr_p2p->bases.empty() || !partials_out)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no p2p plan");
        if (g->n == 0) fail(GDX_ERR_RUNTIME, "RuntimeError: division by zero");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        auto& X = *g->pr_p2p;
        cudaStream_t s = g->stream;
        const int64_t j = X.publishes;
        const int par = int(j & 1);
        PrArgs a = make_args(g, P, 0.85, 0.0, 0);
        a.peers = X.peer_contrib.get() + par * X.world;
        a.npeers = X.world;
        if (!P.partials.get()) P.partials.alloc(2);
        GDX_CUDA(cudaMemsetAsync(P.partials.get(), 0, 2 * sizeof(double), s));
        GDX_CUDA(cudaMemsetAsync(P.dangling.get(), 0, 3 * sizeof(double), s));
        if (j > 0)  // the previous publish must have landed everywhere before parity j&1 is reused
            k_p2p_wait<<<1, 1, 0, s>>>(X.own_ctr(), (unsigned long long)j * X.world, X.err.get());
        if (P.v_end > P.v_begin)
            timed_launch(g, "pr_init", [&] {
                k_pr_shard_init<<<blocks_for(P.v_end - P.v_begin, kPrBlock, g->num_sms * 8),
                                  kPrBlock, 0, s>>>(a, P.partials.get());
            });
        k_p2p_publish<<<1, 1, 0, s>>>(P.partials.get(), nullptr, X.peer_slot.get() + par * X.world,
                                      X.peer_ctr.get(), X.world);
        GDX_LAUNCH_CHECK();
        X.publishes = j + 1;
        p2p_gather_partials(g, X, j, partials_out);
    });
}

extern "C" int gdx_pr_p2p_round(gdx_graph* g, int32_t round, double damping, double threshold,
                                int32_t max_iter, double dangling_in, double* partials_out) {
    return guard_impl([&] {
        if (!g || !g->pr_shard || !g->pr_p2p || g->pr_p2p->bases.empty() || !partials_out)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no p2p plan");
        if (round < 0) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: negative round");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        auto& X = *g->pr_p2p;
        cudaStream_t s = g->stream;
        const int64_t j = X.publishes;  // this round's publish; it reads publish j-1
        PrArgs a = make_args(g, P, damping, threshold, max_iter);
        a.contrib0 = a.contrib1 = X.own_contrib(int((j - 1) & 1));
        a.peers = X.peer_contrib.get() + (j & 1) * X.world;
        a.npeers = X.world;
        GDX_CUDA(cudaMemcpyAsync(P.dangling.get() + round % 3, &dangling_in, sizeof(double),
                                 cudaMemcpyHostToDevice, s));
        clear_flags(P, round, 1, s);
        k_p2p_wait<<<1, 1, 0, s>>>(X.own_ctr(), (unsigned long long)j * X.world, X.err.get());
        GDX_LAUNCH_CHECK();
        if (P.ngroups > 0)
            timed_launch(g, "pr_edges", [&] { k_pr_edges<true><<<P.grid, P.block, 0, s>>>(a, round); });
        launch_cross(g, P, a, round);
        timed_launch(g, "pr_vertices", [&] {
            k_pr_vertices<true><<<blocks_for(std::max(P.v_end - P.v_begin, 1), 2 * kPrBlock,
                                             g->num_sms * 8),
                                  kPrBlock, 0, s>>>(a, round);
        });
        k_p2p_publish<<<1, 1, 0, s>>>(P.dangling.get() + (round + 1) % 3, P.flags.get() + flag_slot(round),
                                      X.peer_slot.get() + (j & 1) * X.world, X.peer_ctr.get(),
                                      X.world);
        GDX_LAUNCH_CHECK();
        X.publishes = j + 1;
        p2p_gather_partials(g, X, j, partials_out);
    });
}

extern "C" int gdx_pr_p2p_rounds(gdx_graph* g, int32_t first, int32_t count, double damping,
                                 double threshold, int32_t max_iter, double dangling_in,
                                 int32_t* settled_out) {
    return guard_impl([&] {
        if (!g || !g->pr_shard || !g->pr_p2p || g->pr_p2p->bases.empty() || !settled_out)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: no p2p plan");
        if (first < 0 || count < 1) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: bad round range");
        GraphScope dg(g);
        auto& P = *g->pr_shard;
        auto& X = *g->pr_p2p;
        cudaStream_t s = g->stream;
        const int32_t last = first + count;
        if (count > kFlagRing / 2)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: at most " +
                                               std::to_string(kFlagRing / 2) + " rounds per call");
        if (first == 0) {  // round 0's dangling mass comes from gdx_pr_p2p_init
            GDX_CUDA(cudaMemcpyAsync(P.dangling.get(), &dangling_in, sizeof(double),
                                     cudaMemcpyHostToDevice, s));
        }
        clear_flags(P, first, count, s);
        prefer_l1(reinterpret_cast<const void*>(&k_pr_edges<true>), kPrCarveout);
        for (int32_t round = first; round < last; ++round) {
            const int64_t j = X.publishes;
            PrArgs a = make_args(g, P, damping, threshold, max_iter);
            a.shard = 0;  // a round after a settled one exits on the device
            a.contrib0 = a.contrib1 = X.own_contrib(int((j - 1) & 1));
            a.peers = X.peer_contrib.get() + (j & 1) * X.world;
            a.npeers = X.world;
            if (P.ngroups > 0)
                timed_launch(g, "pr_edges", [&] { k_pr_edges<true><<<P.grid, P.block, 0, s>>>(a, round); });
            launch_cross(g, P, a, round);
            timed_launch(g, "pr_vertices", [&] {
                k_pr_vertices<true><<<blocks_for(std::max(P.v_end - P.v_begin, 1), 2 * kPrBlock,
                                                 g->num_sms * 8),
                                      kPrBlock, 0, s>>>(a, round);
            });
            k_p2p_publish<<<1, 1, 0, s>>>(P.dangling.get() + (round + 1) % 3, P.flags.get() + flag_slot(round),
                                          X.peer_slot.get() + (j & 1) * X.world, X.peer_ctr.get(),
                                          X.world);
            GDX_LAUNCH_CHECK();
            k_p2p_combine<<<1, 1, 0, s>>>(X.own_ctr(), (unsigned long long)(j + 1) * X.world,
                                          X.err.get(), X.own_partials(int(j & 1)), X.world,
                                          P.dangling.get() + (round + 1) % 3, P.flags.get() + flag_slot(round));
            GDX_LAUNCH_CHECK();
            X.publishes = j + 1;
        }
        std::vector<int32_t> ring(kFlagRing);
        int herr = 0;
        GDX_CUDA(cudaMemcpyAsync(ring.data(), P.flags.get(), kFlagRing * 4,
                                 cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaMemcpyAsync(&herr, X.err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        GDX_CUDA(cudaStreamSynchronize(s));
        if (herr) fail(GDX_ERR_CUDA, "CudaError: peer-memory exchange timed out");
        *settled_out = -1;
        for (int32_t i = 0; i < count; ++i)
            if (ring[size_t(flag_slot(first + i))] == 0) {
                *settled_out = first + i;
                break;
            }
    });
}

extern "C" int gdx_pr_p2p_close(gdx_graph* g) {
    return guard_impl([&] {
        if (!g) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null graph");
        GraphScope dg(g);
        GDX_CUDA(cudaStreamSynchronize(g->stream));
        g->pr_p2p.reset();
    });
}
