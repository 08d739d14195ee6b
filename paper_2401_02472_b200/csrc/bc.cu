// bc.cu -- ComputeBC (reference corpus/bc.sp:6-25) on sm_100a.
//
// The reference runs one source at a time; every BFS level is a full-V
// topology-driven launch plus a host round trip, then a second full-V launch
// per level for the reverse pass (tests/golden/bc/cuda/bc_cuda.cu:117-219;
// interpreter.cpp:1002-1087).
//
// Here a batch of S sources is processed together, level-synchronously, in
// two persistent cooperative kernels (forward / backward) with one grid.sync
// per level:
//   * all (source, vertex) pairs discovered at level L form one contiguous
//     segment of a device log, so each level is a dense work list for every
//     source at once and the reverse pass replays the segments backwards;
//   * forward (iterateInBFS): a level-L item pulls sigma from its level L-1
//     parents (no atomics on sigma) and claims undiscovered neighbours with
//     atomicCAS on level; claims are staged in shared memory and appended
//     with one atomicAdd per block;
//   * backward (iterateInReverse): delta(v) = sum over DAG children w in
//     ascending id order of (sigma(v)/sigma(w)) * (1 + delta(w)) -- the exact
//     expression and order of bc.sp:19-21 / oracles.cpp:60-67 -- then
//     bc[v] += delta(v) for v != source;
//   * sigma is carried as (mantissa, exponent) so path counts never overflow
//     (the reference's double sigma overflows on large grids).
//     Where the reference's sigma is finite the quotients are identical.
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>

#include <cstdio>
#include <cstdlib>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace cg = cooperative_groups;

namespace gdx {

// Block size is a template parameter: fewer, fatter blocks make the per-level
// grid barrier cheaper (BC on high-diameter graphs is barrier-latency bound).

enum { kTail = 0, kLevels = 1, kReached = 2, kFwdScan = 3, kBwdScan = 4, kDag = 5, kBcCtrs = 8 };

struct BcArgs {
    int32_t n;
    int32_t S;
    bool undirected;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ dests;
    const int32_t* __restrict__ in_offsets;
    const int32_t* __restrict__ in_srcs;
    const int32_t* __restrict__ sources;
    int32_t* level;
    double2* sig;  // x = mantissa in [1,2) (or 0), y = binary exponent
    double* delta;
    uint64_t* log;
    long long* lvl_cnt;
    double* bc;
    unsigned long long* ctr;
};

__device__ inline double2 xf_add(double2 a, double2 b) {
    if (a.x == 0.0) return b;
    if (b.x == 0.0) return a;
    if (a.y == b.y) {  // common case: same binade exponent, exact renormalisation
        const double s = a.x + b.x;
        return s < 2.0 ? make_double2(s, a.y) : make_double2(s * 0.5, a.y + 1.0);
    }
    const double e = fmax(a.y, b.y);
    const double s = ldexp(a.x, int(a.y - e)) + ldexp(b.x, int(b.y - e));
    const int k = ilogb(s);
    return make_double2(ldexp(s, -k), e + k);
}

__device__ inline double xf_ratio(double2 a, double2 b) {
    const double q = a.x / b.x;
    return a.y == b.y ? q : ldexp(q, int(a.y - b.y));
}

// Neighbour lists are walked in chunks of kNb with every load of a chunk issued
// before any is consumed (dests -> levels -> sigma/delta), so the per-item
// critical path is a few dependent memory steps instead of one per neighbour.
constexpr int kNb = 4;
static_assert(kNb == 4, "the CTA kernel sums and records exactly kNb = 4 neighbour slots");

// Items whose adjacency exceeds kHeavy edges are deferred to a warp-cooperative
// pass at the end of the block's chunk (lanes stride over the edges, partial
// sums combined with warp shuffles): on skewed graphs a hub's 10^5 neighbours
// would otherwise serialise one thread for the whole level.
constexpr int kHeavy = 64;

__device__ inline double2 xf_warp_sum(double2 a) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double2 b;
        b.x = __shfl_xor_sync(0xffffffffu, a.x, o);
        b.y = __shfl_xor_sync(0xffffffffu, a.y, o);
        a = xf_add(a, b);
    }
    return a;
}

__device__ inline double warp_sum(double d) {
#pragma unroll
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    return d;
}

__device__ inline long long ld_volatile_ll(const long long* p) {
    return *reinterpret_cast<const volatile long long*>(p);
}

__global__ void k_bc_seed(BcArgs a) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < a.S; s += gridDim.x * blockDim.x) {
        const int32_t src = a.sources[s];
        a.level[int64_t(s) * a.n + src] = 0;
        a.log[s] = (uint64_t(s) << 32) | uint32_t(src);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.lvl_cnt[0] = a.S;
}

template <int kBcBlock>
__global__ void __launch_bounds__(kBcBlock) k_bc_forward(BcArgs a) {
    constexpr int kBcQueue = 4 * kBcBlock;
    cg::grid_group grid = cg::this_grid();
    __shared__ uint64_t s_q[kBcQueue];
    __shared__ int s_qn, s_hn;
    __shared__ long long s_h[kBcBlock];  // deferred heavy items (log indices)
    __shared__ long long s_gpos;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long fscan = 0, dag = 0;
    long long beg = 0, end = a.S;
    int L = 0;
    for (;; ++L) {
        for (long long base = beg + (long long)blockIdx.x * kBcBlock; base < end;
             base += (long long)gridDim.x * kBcBlock) {
            if (tid == 0) s_qn = s_hn = 0;
            __syncthreads();
            auto push = [&](int32_t s, int32_t w) {
                const uint64_t x = (uint64_t(s) << 32) | uint32_t(w);
                const int pos = atomicAdd(&s_qn, 1);
                if (pos < kBcQueue) {
                    s_q[pos] = x;
                } else {
                    const long long p = atomicAdd((unsigned long long*)&a.lvl_cnt[L + 1], 1ull);
                    a.log[end + p] = x;
                }
            };
            const long long idx = base + tid;
            if (idx < end) {
                const uint64_t item = a.log[idx];
                const int32_t s = int32_t(item >> 32), v = int32_t(item & 0xffffffffu);
                const int64_t sb = int64_t(s) * a.n;
                int32_t* lev = a.level + sb;
                double2 acc = make_double2(L == 0 ? 1.0 : 0.0, 0.0);
                const int32_t ob = a.offsets[v], oe = a.offsets[v + 1];
                const bool heavy = oe - ob > kHeavy ||
                                   (!a.undirected && L > 0 &&
                                    a.in_offsets[v + 1] - a.in_offsets[v] > kHeavy);
                if (heavy) s_h[atomicAdd(&s_hn, 1)] = idx;
                const int32_t oend = heavy ? ob : oe;  // heavy: no light pass
                fscan += oend - ob;
                for (int32_t e = ob; e < oend; e += kNb) {
                    int32_t w[kNb], lw[kNb];
#pragma unroll
                    for (int k = 0; k < kNb; ++k) w[k] = e + k < oe ? a.dests[e + k] : -1;
#pragma unroll
                    for (int k = 0; k < kNb; ++k) lw[k] = w[k] >= 0 ? lev[w[k]] : -2;
                    double2 sg[kNb];
                    bool par[kNb], got[kNb];
#pragma unroll
                    for (int k = 0; k < kNb; ++k) {
                        par[k] = a.undirected && L > 0 && lw[k] == L - 1;
                        sg[k] = par[k] ? a.sig[sb + w[k]] : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int k = 0; k < kNb; ++k)
                        got[k] = lw[k] == -1 && atomicCAS(&lev[w[k]], -1, L + 1) == -1;
#pragma unroll
                    for (int k = 0; k < kNb; ++k) {
                        if (par[k]) {  // ascending parent order
                            acc = xf_add(acc, sg[k]);
                            ++dag;
                        }
                        if (got[k]) push(s, w[k]);
                    }
                }
                if (!heavy && !a.undirected && L > 0) {
                    const int32_t ib = a.in_offsets[v], ie = a.in_offsets[v + 1];
                    fscan += ie - ib;
                    for (int32_t e = ib; e < ie; e += kNb) {
                        int32_t p[kNb];
                        bool par[kNb];
                        double2 sg[kNb];
#pragma unroll
                        for (int k = 0; k < kNb; ++k) p[k] = e + k < ie ? a.in_srcs[e + k] : -1;
#pragma unroll
                        for (int k = 0; k < kNb; ++k) par[k] = p[k] >= 0 && lev[p[k]] == L - 1;
#pragma unroll
                        for (int k = 0; k < kNb; ++k)
                            sg[k] = par[k] ? a.sig[sb + p[k]] : make_double2(0.0, 0.0);
#pragma unroll
                        for (int k = 0; k < kNb; ++k)
                            if (par[k]) {
                                acc = xf_add(acc, sg[k]);
                                ++dag;
                            }
                    }
                }
                if (!heavy) a.sig[sb + v] = acc;
            }
            __syncthreads();
            // heavy items: one warp each, lanes stride over the adjacency
            for (int h = tid >> 5; h < s_hn; h += kBcBlock / 32) {
                const uint64_t item = a.log[s_h[h]];
                const int32_t s = int32_t(item >> 32), v = int32_t(item & 0xffffffffu);
                const int64_t sb = int64_t(s) * a.n;
                int32_t* lev = a.level + sb;
                double2 acc = make_double2(L == 0 && lane == 0 ? 1.0 : 0.0, 0.0);
                const int32_t ob = a.offsets[v], oe = a.offsets[v + 1];
                if (lane == 0) fscan += oe - ob;
                for (int32_t e = ob + lane; e < oe; e += 32) {
                    const int32_t w = a.dests[e];
                    const int32_t lw = lev[w];
                    if (a.undirected && L > 0 && lw == L - 1) {
                        acc = xf_add(acc, a.sig[sb + w]);
                        ++dag;
                    }
                    if (lw == -1 && atomicCAS(&lev[w], -1, L + 1) == -1) push(s, w);
                }
                if (!a.undirected && L > 0) {
                    const int32_t ib = a.in_offsets[v], ie = a.in_offsets[v + 1];
                    if (lane == 0) fscan += ie - ib;
                    for (int32_t e = ib + lane; e < ie; e += 32) {
                        const int32_t p = a.in_srcs[e];
                        if (lev[p] == L - 1) {
                            acc = xf_add(acc, a.sig[sb + p]);
                            ++dag;
                        }
                    }
                }
                acc = xf_warp_sum(acc);
                if (lane == 0) a.sig[sb + v] = acc;
            }
            __syncthreads();
            const int qn = min(s_qn, kBcQueue);
            if (tid == 0 && qn > 0)
                s_gpos = (long long)atomicAdd((unsigned long long*)&a.lvl_cnt[L + 1], (unsigned long long)qn);
            __syncthreads();
            for (int i = tid; i < qn; i += kBcBlock) a.log[end + s_gpos + i] = s_q[i];
            __syncthreads();
        }
        grid.sync();
        const long long next = ld_volatile_ll(&a.lvl_cnt[L + 1]);
        if (next == 0) break;
        beg = end;
        end += next;
    }
    if (blockIdx.x == 0 && tid == 0) {
        a.ctr[kTail] = (unsigned long long)end;
        a.ctr[kLevels] = (unsigned long long)(L + 1);
    }
    for (int o = 16; o; o >>= 1) {
        fscan += __shfl_xor_sync(0xffffffffu, fscan, o);
        dag += __shfl_xor_sync(0xffffffffu, dag, o);
    }
    if ((tid & 31) == 0) {
        atomicAdd(&a.ctr[kFwdScan], fscan);
        atomicAdd(&a.ctr[kDag], dag);
    }
}

template <int kBcBlock>
__global__ void __launch_bounds__(kBcBlock) k_bc_backward(BcArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_hn;
    __shared__ long long s_h[kBcBlock];  // deferred heavy items (log indices)
    const int tid = threadIdx.x, lane = tid & 31;
    const long long total = (long long)a.ctr[kTail];
    const int levels = int(a.ctr[kLevels]);
    unsigned long long bscan = 0, dag = 0;
    long long end = total;
    for (int L = levels - 1; L >= 0; --L) {
        const long long beg = end - a.lvl_cnt[L];
        for (long long base = beg + (long long)blockIdx.x * kBcBlock; base < end;
             base += (long long)gridDim.x * kBcBlock) {
          if (tid == 0) s_hn = 0;
          __syncthreads();
          const long long idx = base + tid;
          if (idx < end) {
            const uint64_t item = a.log[idx];
            const int32_t s = int32_t(item >> 32), v = int32_t(item & 0xffffffffu);
            const int64_t sb = int64_t(s) * a.n;
            const int32_t* lev = a.level + sb;
            const int32_t ob = a.offsets[v], oe = a.offsets[v + 1];
            const bool heavy = oe - ob > kHeavy;
            if (heavy) s_h[atomicAdd(&s_hn, 1)] = idx;
            const int32_t oend = heavy ? ob : oe;
            const double2 sv = a.sig[sb + v];
            double d = 0.0;
            bscan += oend - ob;
            for (int32_t e = ob; e < oend; e += kNb) {
                int32_t w[kNb];
                bool ch[kNb];
                double2 sw[kNb];
                double dw[kNb];
#pragma unroll
                for (int k = 0; k < kNb; ++k) w[k] = e + k < oe ? a.dests[e + k] : -1;
#pragma unroll
                for (int k = 0; k < kNb; ++k) ch[k] = w[k] >= 0 && lev[w[k]] == L + 1;
#pragma unroll
                for (int k = 0; k < kNb; ++k) {
                    sw[k] = ch[k] ? a.sig[sb + w[k]] : make_double2(1.0, 0.0);
                    dw[k] = ch[k] ? a.delta[sb + w[k]] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < kNb; ++k)
                    if (ch[k] && sw[k].x > 0.0) {  // ascending child order (oracles.cpp:60-67)
                        d += xf_ratio(sv, sw[k]) * (1.0 + dw[k]);
                    }
            }
            if (!heavy) a.delta[sb + v] = d;
          }
          __syncthreads();
          for (int h = tid >> 5; h < s_hn; h += kBcBlock / 32) {
            const uint64_t item = a.log[s_h[h]];
            const int32_t s = int32_t(item >> 32), v = int32_t(item & 0xffffffffu);
            const int64_t sb = int64_t(s) * a.n;
            const int32_t* lev = a.level + sb;
            const int32_t ob = a.offsets[v], oe = a.offsets[v + 1];
            const double2 sv = a.sig[sb + v];
            double d = 0.0;
            if (lane == 0) bscan += oe - ob;
            for (int32_t e = ob + lane; e < oe; e += 32) {
                const int32_t w = a.dests[e];
                if (lev[w] == L + 1) {
                    const double2 sw = a.sig[sb + w];
                    if (sw.x > 0.0) {
                        d += xf_ratio(sv, sw) * (1.0 + a.delta[sb + w]);
                    }
                }
            }
            d = warp_sum(d);
            if (lane == 0) a.delta[sb + v] = d;
          }
          __syncthreads();
        }
        end = beg;
        grid.sync();
    }
    for (int o = 16; o; o >>= 1) {
        bscan += __shfl_xor_sync(0xffffffffu, bscan, o);
        dag += __shfl_xor_sync(0xffffffffu, dag, o);
    }
    if ((tid & 31) == 0) {
        atomicAdd(&a.ctr[kBwdScan], bscan);
        atomicAdd(&a.ctr[kDag], dag);
    }
}


// bc[v] += delta_s(v) over the batch's sources in source order (v reached by
// s, v != s): a fixed summation order, so results are reproducible run to run.
__global__ void k_bc_batch_sum(BcArgs a) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double acc = a.bc[v];
        for (int s = 0; s < a.S; ++s)
            if (a.level[int64_t(s) * a.n + v] >= 0 && a.sources[s] != v)
                acc += a.delta[int64_t(s) * a.n + v];
        a.bc[v] = acc;
    }
}

// ---------------------------------------------------------------------------
// CTA-per-source mode (high-diameter graphs, many sources).  A road-like grid
// has ~10^4 BFS levels of a few thousand vertices: the grid-wide kernels above
// spend ~25 us per level in grid.sync and cross-CTA queue atomics.  Here one
// CTA (or a cluster of CTAs) runs a whole source (forward and backward) with
// the (cluster) barrier as the level barrier and a shared-memory queue tail;
// the clusters of the grid take different sources, so up to #SM sources run
// concurrently with no grid-wide synchronisation at all.  Same arithmetic and
// summation orders as the grid kernels.
// CTA size: 896 threads leave 72 registers per thread (1024 leave 64 and the
// kernel spills ~100 B): same-box C4 166.5 ms vs 173.7 at 1024, 170.8 at 800,
// 171.9 at 928 (64 registers again).
// ---------------------------------------------------------------------------
#ifndef GDX_BC_CTA
#define GDX_BC_CTA 896
#endif
constexpr int kBcCta = GDX_BC_CTA;

// Per-(slot, vertex) state of the CTA kernel: one 16 B record {level tag,
// exponent, mantissa} holding sigma(v) after the forward pass and, once the
// backward pass has visited v, q(v) = (1 + delta(v)) / sigma(v) -- the only
// value v's parents need: delta(p) = sigma(p) * sum over children w of q(w).
// Level tags: a slot's successive sources use disjoint, increasing tag ranges
// (source k's level L is tag base_k + L, base_{k+1} = base_k + levels_k + 1),
// so a record whose tag is below the current base is undiscovered -- no
// per-source restore pass; the slot's base persists on the handle and the
// records are cleared only when the tags would pass INT32_MAX.
struct __align__(16) BcRec {
    int32_t level;  // tag (< base: undiscovered in the current source)
    int32_t sexp;
    double smant;
};

// slot stride of the partial scores: 64 B-aligned slots (16 B vector sums)
__host__ __device__ inline int64_t bcs_stride(int64_t n) { return (n + 7) & ~int64_t(7); }

struct BcCtaArgs {
    int32_t n;
    int32_t nsrc;
    bool undirected;
    const int32_t* __restrict__ offsets;
    const int32_t* __restrict__ dests;
    const int32_t* __restrict__ in_offsets;
    const int32_t* __restrict__ in_srcs;
    const int32_t* __restrict__ sources;
    BcRec* rec;        // [grid][n]
    int32_t* base;     // [grid] level tag base of the slot's next source
    bool any_heavy;    // some vertex has more than kHeavy out- (or in-) edges
    int32_t* log;      // [grid][n] int4 (v, out-begin, out-end, 0): discovery order, levels contiguous
    int32_t* loff;     // [grid][n+2] level boundaries in log
    bool kids;         // record each item's children in its own log entry (low-degree graphs)
    double* bcs;       // [grid][n] the slot's partial scores (its sources in order), 0 between calls
    double* bc;
    unsigned long long* ctr;
    unsigned long long* trace;  // optional: slot 0's (globaltimer ns, items) per level step
    int32_t trace_cap;
};

__device__ inline void bc_trace(const BcCtaArgs& a, int64_t slot, int tid, int& k, int items) {
    if (a.trace && slot == 0 && tid == 0 && k < a.trace_cap) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[2 * k] = t;
        a.trace[2 * k + 1] = (unsigned long long)(unsigned)items;
    }
    ++k;
}

// The CTA kernel carries sigma as {mantissa, int exponent} (3 registers, no
// int<->double conversions); same values as the double2 form above.
struct XF {
    double m;  // in [1, 2), or 0
    int e;
};

__device__ inline XF xf_add(XF a, XF b) {
    if (a.m == 0.0) return b;
    if (b.m == 0.0) return a;
    if (a.e == b.e) {  // common case: same binade exponent, exact renormalisation
        const double s = a.m + b.m;
        return s < 2.0 ? XF{s, a.e} : XF{s * 0.5, a.e + 1};
    }
    // big + small * 2^d (d < 0): the sum is in [1, 3), so at most one halving;
    // 2^d is built from its bits (the same values as ldexp / ilogb)
    const XF big = a.e > b.e ? a : b, small = a.e > b.e ? b : a;
    const int d = small.e - big.e;
    if (d < -60) return big;  // below half an ulp of big: the sum rounds to big
    const double s = big.m + small.m * __longlong_as_double((long long)(d + 1023) << 52);
    return s < 2.0 ? XF{s, big.e} : XF{s * 0.5, big.e + 1};
}

__device__ inline double xf_ratio(XF a, XF b) {
    const double q = a.m / b.m;
    return a.e == b.e ? q : ldexp(q, a.e - b.e);
}

__device__ inline XF xf_warp_sum(XF a) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        XF b;
        b.m = __shfl_xor_sync(0xffffffffu, a.m, o);
        b.e = __shfl_xor_sync(0xffffffffu, a.e, o);
        a = xf_add(a, b);
    }
    return a;
}

__device__ inline void rec_level_sigma(const BcRec* r, int32_t& level, XF& sig) {
    const int4 q = *reinterpret_cast<const int4*>(r);
    level = q.x;
    sig = XF{__hiloint2double(q.w, q.z), q.y};
}
// delta(v) = sigma(v) * S (S = sum of the children's q) and the record's new
// value q(v) = (1 + delta(v)) / sigma(v)
__device__ inline double xf_mul_double(XF a, XF b) {
    if (a.m == 0.0 || b.m == 0.0) return 0.0;
    const int e = a.e + b.e;  // the product of the mantissas is in [1, 4)
    if (e > -1020 && e < 1020)  // 2^e is a normal double: one exact multiply
        return a.m * b.m * __longlong_as_double((long long)(e + 1023) << 52);
    return ldexp(a.m * b.m, e);
}
__device__ inline XF xf_q(double delta, XF sig) {
    const double q = (1.0 + delta) / sig.m;  // finite, normal, in (0.5, n + 1]
    const long long bits = __double_as_longlong(q);
    const int k = int((bits >> 52) & 0x7ff) - 1023;
    return XF{__longlong_as_double((bits & 0x800fffffffffffffll) | (1023ll << 52)), k - sig.e};
}
__device__ inline void rec_store_sigma(BcRec* r, int32_t level, XF sig) {
    *reinterpret_cast<int4*>(r) =
        make_int4(level, sig.e, __double2loint(sig.m), __double2hiint(sig.m));
}

// Backward-pass pipelining (GDX_BC_PIPE, graphs with recorded children): while
// a thread works on one item of a level, its next item's log entry and
// children list, then its own and its children's records, are copied into the
// thread's shared-memory slot with cp.async -- no registers held across the
// current item, so its next item starts with its data on chip.
#ifndef GDX_BC_PIPE
#define GDX_BC_PIPE 1
#endif
constexpr bool kBcPipe = GDX_BC_PIPE != 0;
struct __align__(16) BcPf {
    int4 log, own, ch[3];
};
__device__ inline void cp16(void* sdst, const void* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ inline void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ inline void cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// stage 2: the item's own record and its recorded children's (slot's log entry ready)
__device__ inline void bc_pf_records(BcPf* pf, const BcRec* rec) {
    const int4 it = pf->log;
    if (it.x < 0 && it.y < 0) {  // a leaf: nothing to load (its q is final)
    } else if (it.x < 0) {  // (~v, children): see the forward pass
        cp16(&pf->own, rec + ~it.x);
        if (it.y >= 0) cp16(&pf->ch[0], rec + it.y);
        if (it.z >= 0) cp16(&pf->ch[1], rec + it.z);
        if (it.w >= 0) cp16(&pf->ch[2], rec + it.w);
    } else {
        cp16(&pf->own, rec + it.x);
    }
    cp_commit();
}

// CS CTAs (a thread-block cluster) share one source: the level barrier is a
// cluster barrier and the queue tail lives in CTA 0's shared memory (DSMEM
// atomics), so a source's levels are spread over CS * kBcCta threads.
// Heavy items of the CTA kernel (one warp each, lanes stride over the
// adjacency).  Out of line so their registers do not weigh on the light path.
__device__ __forceinline__ void bc_cta_heavy_forward(const BcCtaArgs& a, BcRec* rec, int4* log,
                                                  const int* s_h, int hn, int L, int end,
                                                  int* s_next, int* const* s_copy, int ncopy,
                                                  int32_t base, unsigned& fscan,
                                                  unsigned& dag) {
    const int ltid = threadIdx.x, lane = ltid & 31;
    for (int h = ltid >> 5; h < hn; h += kBcCta / 32) {
        const int4 it = log[s_h[h]];
        const int32_t v = it.x, ob = it.y, oe = it.z;
        XF acc{L == 0 && lane == 0 ? 1.0 : 0.0, 0};
        if (lane == 0) fscan += oe - ob;
        for (int32_t e = ob + lane; e < oe; e += 32) {
            const int32_t w = a.dests[e];
            int32_t lw;
            XF sg;
            rec_level_sigma(rec + w, lw, sg);
            if (a.undirected && L > 0 && lw == base + L - 1) {
                acc = xf_add(acc, sg);
                ++dag;
            }
            if (lw < base) {
                const int32_t w0 = a.offsets[w], w1 = a.offsets[w + 1];
                if (atomicCAS(&rec[w].level, lw, base + L + 1) == lw) {
                    log[end + atomicAdd(&s_next[L % 3], 1)] = make_int4(w, w0, w1, 0);
                    for (int q = 0; q < ncopy; ++q) atomicAdd(&s_copy[q][L % 3], 1);
                }
            }
        }
        if (!a.undirected && L > 0) {
            const int32_t ib = a.in_offsets[v], ie = a.in_offsets[v + 1];
            if (lane == 0) fscan += ie - ib;
            for (int32_t e = ib + lane; e < ie; e += 32) {
                int32_t lp;
                XF sg;
                rec_level_sigma(rec + a.in_srcs[e], lp, sg);
                if (lp == base + L - 1) {
                    acc = xf_add(acc, sg);
                    ++dag;
                }
            }
        }
        acc = xf_warp_sum(acc);
        if (lane == 0) rec_store_sigma(rec + v, base + L, acc);
    }
}

__device__ __forceinline__ void bc_cta_heavy_backward(const BcCtaArgs& a, BcRec* rec, const int4* log,
                                                   const int* s_h, int hn, int Lb, int32_t src,
                                                   int32_t base, double* bcs) {
    const int ltid = threadIdx.x, lane = ltid & 31;
    for (int h = ltid >> 5; h < hn; h += kBcCta / 32) {
        const int4 it = log[s_h[h]];
        const int32_t v = it.x, ob = it.y, oe = it.z;
        int32_t lv;
        XF sv;
        rec_level_sigma(rec + v, lv, sv);
        XF sum{0.0, 0};
        for (int32_t e = ob + lane; e < oe; e += 32) {
            int32_t lw;
            XF qw;
            rec_level_sigma(rec + a.dests[e], lw, qw);
            if (lw == base + Lb + 1) {
                sum = xf_add(sum, qw);
            }
        }
        sum = xf_warp_sum(sum);
        if (lane == 0) {
            const double d = xf_mul_double(sv, sum);
            rec_store_sigma(rec + v, lv, xf_q(d, sv));
            if (v != src && d != 0.0) bcs[v] += d;  // leaves add nothing
        }
    }
}

// HEAVY = false compiles the kernel without the heavy-item paths (graphs whose
// maximum degree is at most kHeavy, e.g. road-like grids): no extra barrier and
// no register pressure from code that never runs.
template <int CS, bool HEAVY>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(kBcCta) k_bc_cta(BcCtaArgs a) {
    __shared__ int s_next_local[3];
    __shared__ int s_hn;
    __shared__ int s_h[kBcCta];  // this CTA's deferred heavy items (log indices) of a level
    extern __shared__ BcPf s_pf[];  // GDX_BC_PIPE: one slot per thread (dynamic)
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = int(cluster.block_rank());
    int* s_next = cluster.map_shared_rank(s_next_local, 0);
    // every other CTA keeps a copy of the tails (count-only reds from all
    // CTAs), so after the barrier each thread reads its own shared memory
    int* s_copy[CS > 1 ? CS - 1 : 1];
#pragma unroll
    for (int q = 1; q < CS; ++q) s_copy[q - 1] = cluster.map_shared_rank(s_next_local, q);
    const int tid = crank * kBcCta + int(threadIdx.x);
    const int ltid = threadIdx.x;
    if (ltid == 0) s_hn = 0;
    constexpr int kStride = CS * kBcCta;
    const int64_t slot = blockIdx.x / CS;
    const int32_t nslots = gridDim.x / CS;
    BcRec* rec = a.rec + slot * a.n;
    int4* log = reinterpret_cast<int4*>(a.log) + slot * a.n;  // (v, out-begin, out-end, 0)
    int32_t* loff = a.loff + slot * (int64_t(a.n) + 2);
    // children recorded in the log entries: after the forward pass processed
    // item i (vertex v), log[i] = (~v, c0, c1, c2) -- v's children (neighbours
    // claimed at the next level, by v or not) in ascending order, -1 padded --
    // when v has at most 3; otherwise it stays (v, out-begin, out-end) and the
    // backward pass scans the adjacency.  (A vertex below the source has a
    // parent, so on graphs of maximum degree 4 only the source can have 4.)
    const bool kids = !HEAVY && a.kids;
    double* bcs = a.bcs + slot * bcs_stride(a.n);
    // per-source 32-bit counters (registers are the kernel's limit), flushed
    // to the 64-bit totals after every source
    unsigned fscan = 0, dag = 0;
    int tk = 0;
    int32_t base = a.base[slot];  // tag of the next source's level 0
    for (int32_t si = int32_t(slot); si < a.nsrc; si += nslots) {
        const int32_t src = a.sources[si];
        const bool first_src = si == int32_t(slot);
        if (int64_t(base) + a.n + 2 > INT32_MAX) {  // tags exhausted: clear the slot
            for (int i = tid; i < a.n; i += kStride) rec[i].level = 0;
            base = 1;
            cluster.sync();
        }
        if (tid == 0) {
            rec[src].level = base;
            log[0] = make_int4(src, a.offsets[src], a.offsets[src + 1], 0);
            loff[0] = 0;
            s_next[0] = s_next[1] = s_next[2] = 0;
        }
        if (ltid == 0) s_next_local[0] = s_next_local[1] = s_next_local[2] = 0;
        cluster.sync();
        bool leaf = false;  // the current forward item has no children (recorded lists)
        // one chunk of <= kNb neighbours of item i (level L): parents' sigma,
        // claims (CAS) of undiscovered neighbours, the children list, the claims'
        // log positions (one DSMEM atomic per converged lane group) and entries.
        auto fwd_chunk = [&](int i, int32_t v, int L, int end, int deg, const int32_t (&w)[kNb],
                             const int32_t (&lw)[kNb], const XF (&sg)[kNb], XF& acc) {
            bool par[kNb], got[kNb];
            int32_t w0[kNb], w1[kNb], lnew[kNb];
#pragma unroll
            for (int k = 0; k < kNb; ++k) {
                par[k] = a.undirected && L > 0 && lw[k] == base + L - 1;
                const bool cand = w[k] >= 0 && lw[k] < base;
                w0[k] = cand ? a.offsets[w[k]] : 0;  // issued with the CAS
                w1[k] = cand ? a.offsets[w[k] + 1] : 0;
                lnew[k] = cand ? atomicCAS(&rec[w[k]].level, lw[k], base + L + 1) : lw[k];
                got[k] = cand && lnew[k] == lw[k];
            }
            if (kids && deg <= kNb) {
                // the children of v: neighbours claimed at this level, by v or
                // not (a failed CAS returns the claimer's level) -- the
                // backward pass reads them here instead of the adjacency
                int32_t c0 = -1, c1 = -1, c2 = -1;
                int nc = 0;
#pragma unroll
                for (int k = 0; k < kNb; ++k)
                    if (w[k] >= 0 && (got[k] || lnew[k] == base + L + 1)) {
                        if (nc == 0) c0 = w[k];
                        else if (nc == 1) c1 = w[k];
                        else if (nc == 2) c2 = w[k];
                        ++nc;
                    }
                if (nc <= 3) log[i] = make_int4(~v, c0, c1, c2);
                leaf = nc == 0;
            }
            // log positions: one DSMEM atomic per group of converged lanes
            // (scan of the claim counts) instead of one per claim
            {
                cg::coalesced_group act = cg::coalesced_threads();
                const int cnt = int(got[0]) + int(got[1]) + int(got[2]) + int(got[3]);
                const int excl = cg::exclusive_scan(act, cnt);
                const int last = int(act.size()) - 1;
                const int tot = act.shfl(excl + cnt, last);
                int qb = 0;
                if (int(act.thread_rank()) == last && tot) {
                    qb = atomicAdd(&s_next[L % 3], tot);
#pragma unroll
                    for (int q = 0; q < CS - 1; ++q) atomicAdd(&s_copy[q][L % 3], tot);
                }
                int pos = end + act.shfl(qb, last) + excl;
#pragma unroll
                for (int k = 0; k < kNb; ++k) {
                    if (par[k]) {  // ascending parent order
                        acc = xf_add(acc, sg[k]);
                        ++dag;
                    }
                    if (got[k]) log[pos++] = make_int4(w[k], w0[k], w1[k], 0);
                }
            }
        };
        // ---- forward: iterateInBFS ----
        int beg = 0, end = 1, L = 0;
        for (;; ++L) {
            int deferred = 0;
            for (int i = beg + tid; i < end; i += kStride) {
                // the log entry carries v's out-edge range (one dependent load fewer)
                const int4 it = log[i];
                const int32_t v = it.x, ob = it.y, oe = it.z;
                bool heavy = HEAVY && (oe - ob > kHeavy ||
                                       (!a.undirected && L > 0 &&
                                        a.in_offsets[v + 1] - a.in_offsets[v] > kHeavy));
                if (heavy) {
                    const int hp = atomicAdd(&s_hn, 1);
                    if (hp < kBcCta) {
                        s_h[hp] = i;
                        deferred = 1;
                        continue;
                    }
                    heavy = false;  // list full: this item runs on its own thread
                }
                XF acc{L == 0 ? 1.0 : 0.0, 0};
                fscan += oe - ob;
                leaf = kids && oe == ob;  // fwd_chunk sets it from the children it records
                for (int32_t e = ob; e < oe; e += kNb) {
                    int32_t w[kNb], lw[kNb];
                    XF sg[kNb];
#pragma unroll
                    for (int k = 0; k < kNb; ++k) w[k] = e + k < oe ? a.dests[e + k] : -1;
#pragma unroll
                    for (int k = 0; k < kNb; ++k) {  // level and sigma in one 16 B load
                        lw[k] = -2;  // below every tag, but never a candidate (w < 0)
                        sg[k] = XF{0.0, 0};
                        if (w[k] >= 0) rec_level_sigma(rec + w[k], lw[k], sg[k]);
                    }
                    fwd_chunk(i, v, L, end, oe - ob, w, lw, sg, acc);
                }
                if (!a.undirected && L > 0) {
                    const int32_t ib = a.in_offsets[v], ie = a.in_offsets[v + 1];
                    fscan += ie - ib;
                    for (int32_t e = ib; e < ie; e += kNb) {
                        int32_t p[kNb], lp[kNb];
                        XF sg[kNb];
#pragma unroll
                        for (int k = 0; k < kNb; ++k) p[k] = e + k < ie ? a.in_srcs[e + k] : -1;
#pragma unroll
                        for (int k = 0; k < kNb; ++k) {
                            lp[k] = -2;
                            sg[k] = XF{0.0, 0};
                            if (p[k] >= 0) rec_level_sigma(rec + p[k], lp[k], sg[k]);
                        }
#pragma unroll
                        for (int k = 0; k < kNb; ++k)
                            if (p[k] >= 0 && lp[k] == base + L - 1) {
                                acc = xf_add(acc, sg[k]);
                                ++dag;
                            }
                    }
                }
                if (kids && oe == ob) log[i] = make_int4(~v, -1, -1, -1);  // no children
                // a leaf's sigma has no reader in the forward pass (a reader would
                // be a child), so its record gets its final q = 1 / sigma now and
                // the backward pass skips it
                rec_store_sigma(rec + v, base + L, leaf ? xf_q(0.0, acc) : acc);
            }
            // heavy items of this CTA: one warp each, lanes stride over the adjacency
            // (graphs without a vertex above kHeavy skip the extra barrier)
            if (HEAVY && __syncthreads_count(deferred) > 0) {
                bc_cta_heavy_forward(a, rec, log, s_h, min(s_hn, kBcCta), L, end, s_next, s_copy,
                                     CS - 1, base, fscan, dag);
                __syncthreads();
                if (ltid == 0) s_hn = 0;
            }
            // one barrier per level: level L pushes to tail L % 3; the tail of
            // level L+2 (last read right after the previous barrier) is reset now
            cluster.sync();
            const int next = s_next_local[L % 3];  // this CTA's copy (CTA 0: the tail itself)
            bc_trace(a, slot, tid, tk, end - beg);
            if (ltid == 0) s_next_local[(L + 2) % 3] = 0;
            if (tid == 0) loff[L + 1] = end;
            if (next == 0) break;
            beg = end;
            end += next;
        }
        cluster.sync();  // loff[levels] (written by thread 0 above) before the backward pass
        const int levels = L + 1;  // loff[0..levels] bound the levels in log
        if (tid == 0) {
            atomicAdd(&a.ctr[kReached], (unsigned long long)end);
            atomicMax(&a.ctr[kLevels], (unsigned long long)levels);
        }
        // ---- backward: iterateInReverse ----
        if (!HEAVY && kBcPipe && kids) {
            BcPf* pf = s_pf + ltid;
            for (int Lb = levels - 1; Lb >= 0; --Lb) {
                const int b0 = loff[Lb], b1 = loff[Lb + 1];
                int i = b0 + tid;
                if (i < b1) {  // the first item: both stages now
                    cp16(&pf->log, log + i);
                    cp_commit();
                    cp_wait();
                    bc_pf_records(pf, rec);
                }
                for (; i < b1; i += kStride) {
                    cp_wait();
                    const int4 it = pf->log, ow = pf->own;
                    const bool kf = it.x < 0;  // (~v, children) or (v, out-begin, out-end)
                    const bool lf = kf && it.y < 0;  // a leaf: final q stored by the forward pass
                    const int32_t v = kf ? ~it.x : it.x, ob = it.y, oe = it.z;
                    const int32_t lv = ow.x;
                    const XF sv{__hiloint2double(ow.w, ow.z), ow.y};
                    XF sum{0.0, 0};
                    const int in = i + kStride;
                    if (kf) {  // the recorded children, ascending
                        const int32_t w[3] = {it.y, it.z, it.w};
                        int4 r[3];
#pragma unroll
                        for (int k = 0; k < 3; ++k) r[k] = w[k] >= 0 ? pf->ch[k] : make_int4(0, 0, 0, 0);
                        if (in < b1) {  // stage 1 of the next item
                            cp16(&pf->log, log + in);
                            cp_commit();
                        }
#pragma unroll
                        for (int k = 0; k < 3; ++k)
                            if (w[k] >= 0) sum = xf_add(sum, XF{__hiloint2double(r[k].w, r[k].z), r[k].y});
                    } else {
                        if (in < b1) {
                            cp16(&pf->log, log + in);
                            cp_commit();
                        }
                        for (int32_t e = ob; e < oe; e += kNb) {
                            int32_t w[kNb], lw[kNb];
                            XF qw[kNb];
#pragma unroll
                            for (int k = 0; k < kNb; ++k) w[k] = e + k < oe ? a.dests[e + k] : -1;
#pragma unroll
                            for (int k = 0; k < kNb; ++k) {
                                lw[k] = -2;
                                qw[k] = XF{0.0, 0};
                                if (w[k] >= 0) rec_level_sigma(rec + w[k], lw[k], qw[k]);
                            }
#pragma unroll
                            for (int k = 0; k < kNb; ++k)
                                if (w[k] >= 0 && lw[k] == base + Lb + 1) sum = xf_add(sum, qw[k]);
                        }
                    }
                    if (in < b1) {  // stage 2 of the next item
                        cp_wait();
                        bc_pf_records(pf, rec);
                    }
                    if (!lf) {
                        const double d = xf_mul_double(sv, sum);  // delta(v)
                        rec_store_sigma(rec + v, lv, xf_q(d, sv));
                        if (v != src && d != 0.0) bcs[v] = first_src ? d : bcs[v] + d;
                    }
                }
                cluster.sync();
                bc_trace(a, slot, tid, tk, b0 - b1);  // negative: backward
            }
        } else
        for (int Lb = levels - 1; Lb >= 0; --Lb) {
            const int b0 = loff[Lb], b1 = loff[Lb + 1];
            int deferred = 0;
            for (int i = b0 + tid; i < b1; i += kStride) {
                const int4 it = log[i];
                const bool kf = kids && it.x < 0;  // (~v, children) or (v, out-begin, out-end)
                if (kf && it.y < 0) continue;      // a leaf: its q is final (forward pass)
                const int32_t v = kf ? ~it.x : it.x, ob = it.y, oe = it.z;
                if (HEAVY && oe - ob > kHeavy) {
                    const int hp = atomicAdd(&s_hn, 1);
                    if (hp < kBcCta) {
                        s_h[hp] = i;
                        deferred = 1;
                        continue;
                    }
                }
                int32_t lv;
                XF sv;
                rec_level_sigma(rec + v, lv, sv);
                // S = sum of the children's q(w) = (1 + delta(w)) / sigma(w), ascending
                XF sum{0.0, 0};
                if (kf) {  // the recorded children, ascending
                    const int32_t w[3] = {it.y, it.z, it.w};
                    int32_t lw[3];
                    XF qw[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        qw[k] = XF{0.0, 0};
                        if (w[k] >= 0) rec_level_sigma(rec + w[k], lw[k], qw[k]);
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        if (w[k] >= 0) sum = xf_add(sum, qw[k]);
                } else {
                    for (int32_t e = ob; e < oe; e += kNb) {
                        int32_t w[kNb], lw[kNb];
                        XF qw[kNb];
#pragma unroll
                        for (int k = 0; k < kNb; ++k) w[k] = e + k < oe ? a.dests[e + k] : -1;
#pragma unroll
                        for (int k = 0; k < kNb; ++k) {  // level and q in one 16 B load
                            lw[k] = -2;
                            qw[k] = XF{0.0, 0};
                            if (w[k] >= 0) rec_level_sigma(rec + w[k], lw[k], qw[k]);
                        }
#pragma unroll
                        for (int k = 0; k < kNb; ++k)
                            if (w[k] >= 0 && lw[k] == base + Lb + 1) {  // ascending child order
                                sum = xf_add(sum, qw[k]);
                            }
                    }
                }
                const double d = xf_mul_double(sv, sum);  // delta(v)
                rec_store_sigma(rec + v, lv, xf_q(d, sv));
                // leaves add nothing (one thread per v); the slot's first source of
                // the call stores (its partials were cleared by the last sum)
                if (v != src && d != 0.0) bcs[v] = first_src ? d : bcs[v] + d;
            }
            if (HEAVY && __syncthreads_count(deferred) > 0) {
                bc_cta_heavy_backward(a, rec, log, s_h, min(s_hn, kBcCta), Lb, src, base, bcs);
                __syncthreads();
                if (ltid == 0) s_hn = 0;
            }
            cluster.sync();
            bc_trace(a, slot, tid, tk, b0 - b1);  // negative: backward
        }
        {
            unsigned long long f = fscan, d = dag;
            for (int o = 16; o; o >>= 1) {
                f += __shfl_xor_sync(0xffffffffu, f, o);
                d += __shfl_xor_sync(0xffffffffu, d, o);
            }
            if ((ltid & 31) == 0) {
                atomicAdd(&a.ctr[kFwdScan], f);
                atomicAdd(&a.ctr[kDag], d);
            }
            fscan = dag = 0;
        }
        // the next source's tags start above every tag this one wrote
        base += levels + 1;
    }
    if (tid == 0) a.base[slot] = base;
}

// bc[v] = sum of the slots' partials in slot order (each slot's own sources
// in order): reproducible; the partials are cleared for the next call.
// Two vertices per thread (16 B loads / stores; slot stride a multiple of 8).
__global__ void k_bc_slot_sum(int32_t n, int64_t stride, int32_t slots, double* __restrict__ bcs,
                              double* __restrict__ bc) {
    for (int64_t v = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); v < n;
         v += 2 * (int64_t)gridDim.x * blockDim.x) {
        double2 acc = make_double2(bc[v], v + 1 < n ? bc[v + 1] : 0.0);
        for (int q = 0; q < slots; ++q) {
            double2* p = reinterpret_cast<double2*>(bcs + q * stride + v);
            const double2 x = *p;
            if (x.x != 0.0 || x.y != 0.0) {
                acc.x += x.x;
                acc.y += x.y;
                *p = make_double2(0.0, 0.0);
            }
        }
        bc[v] = acc.x;
        if (v + 1 < n) bc[v + 1] = acc.y;
    }
}

static void run_bc_cta(gdx_graph* g, const std::vector<int32_t>& hsrc,
                       unsigned long long* totals, int& launches, int& max_levels,
                       bool& used_kids) {
    auto& W = *g->bc;
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    const int32_t nsrc = int32_t(hsrc.size());
    // cluster size: spread each source over CS SMs while there are SMs to spare
    const char* csv = std::getenv("GDX_BC_CLUSTER");
    int CS = 1;
    if (csv)
        CS = std::atoi(csv);
    else
        while (CS < 4 && int64_t(2 * CS) * std::min<int32_t>(nsrc, g->num_sms) <= g->num_sms) CS *= 2;
    if (CS != 1 && CS != 2 && CS != 4) CS = 1;
    int slots = std::max(1, std::min<int32_t>(nsrc, g->num_sms / CS));
    // graphs without heavy vertices record each log entry's children (16 B,
    // the backward pass then skips the adjacency); GDX_BC_KIDS=0 disables
    const bool any_heavy = graph_max_degree(g) > kHeavy;
    const char* kv = std::getenv("GDX_BC_KIDS");
    const bool a_kids = !any_heavy && !(kv && std::string(kv) == "0");
    // a slot holds 44 B per vertex (record, log entry -- later the children --,
    // level bound, partial score): fewer
    // slots (each then runs several sources) when they would not fit (queried
    // only when the slots have to grow)
    if (W.cta_grid < slots) {
        size_t free_b = 0, tot_b = 0;
        GDX_CUDA(cudaMemGetInfo(&free_b, &tot_b));
        const size_t per_slot = size_t(n) * 44 + 8;
        const size_t held = W.cta_rec.bytes() + W.cta_log.bytes() + W.cta_loff.bytes() +
                            W.cta_bcs.bytes() +
                            pool_cached();
        const int64_t fit = int64_t(double(free_b + held) * 0.85 / double(per_slot));
        if (fit < 1)
            fail(GDX_ERR_OUT_OF_MEMORY, "OutOfMemory: BC needs " + std::to_string(per_slot) +
                                            " bytes of device memory per source slot");
        slots = int(std::min<int64_t>(slots, fit));
    }
    const int grid = slots * CS;
    if (W.cta_grid < slots) {
        W.level.release();
        W.sig.release();
        W.delta.release();
        W.log.release();
        W.cta_log.release();
        W.cta_loff.release();
        W.batch = 0;
        W.cta_rec.alloc(size_t(slots) * n * 2);  // 16 B BcRec per (slot, vertex)
        W.cta_log.alloc(size_t(slots) * n * 4);  // int4 entries
        W.cta_loff.alloc(size_t(slots) * (n + 2));
        W.cta_grid = slots;
        // every tag 0 lies below the slots' first base (1)
        GDX_CUDA(cudaMemsetAsync(W.cta_rec.get(), 0, W.cta_rec.bytes(), s));
        W.cta_base.alloc(size_t(slots));
        W.cta_bcs.alloc(size_t(slots) * bcs_stride(n));
        GDX_CUDA(cudaMemsetAsync(W.cta_bcs.get(), 0, W.cta_bcs.bytes(), s));
        // GDX_BC_TAG_START (tests): first base of new slots, e.g. close to
        // INT32_MAX to exercise the slot clearing when the tags run out
        const char* ts = std::getenv("GDX_BC_TAG_START");
        std::vector<int32_t> ones(size_t(slots), ts ? std::max(1, std::atoi(ts)) : 1);
        GDX_CUDA(cudaMemcpyAsync(W.cta_base.get(), ones.data(), ones.size() * 4,
                                 cudaMemcpyHostToDevice, s));
        GDX_CUDA(cudaStreamSynchronize(s));  // `ones` is pageable and local
    }
    W.sources.ensure(size_t(nsrc));
    GDX_CUDA(cudaMemcpyAsync(W.sources.get(), hsrc.data(), size_t(nsrc) * 4,
                             cudaMemcpyHostToDevice, s));
    GDX_CUDA(cudaMemsetAsync(W.ctrs.get(), 0, kBcCtrs * 8, s));
    BcCtaArgs a;
    a.n = g->n;
    a.nsrc = nsrc;
    a.undirected = !g->directed;
    a.offsets = g->offsets.get();
    a.dests = g->dests.get();
    a.in_offsets = g->in_offsets();
    a.in_srcs = g->in_srcs();
    a.sources = W.sources.get();
    a.rec = reinterpret_cast<BcRec*>(W.cta_rec.get());
    a.base = W.cta_base.get();
    a.any_heavy = any_heavy;
    a.kids = a_kids;
    used_kids = a_kids;
    a.log = W.cta_log.get();
    a.loff = W.cta_loff.get();
    a.bc = W.bc.get();
    a.bcs = W.cta_bcs.get();
    a.ctr = W.ctrs.get();
    // GDX_BC_TRACE=<file>: slot 0's per-level-step (ns since the previous step, items)
    const char* trace = std::getenv("GDX_BC_TRACE");
    a.trace = nullptr;
    a.trace_cap = 1 << 16;
    DevBuf<unsigned long long> tbuf;
    if (trace) {
        tbuf.alloc(size_t(2) * a.trace_cap);
        GDX_CUDA(cudaMemsetAsync(tbuf.get(), 0, tbuf.bytes(), s));
        a.trace = tbuf.get();
    }
    if (g->directed && (!a.in_offsets || !a.in_srcs))
        fail(GDX_ERR_UNSUPPORTED, "Unsupported: directed BC needs the reverse CSR");
    // the slot partials are cleared by the sum kernel; a call that stopped
    // between the two (an error) leaves them dirty: clear them before reuse
    if (W.cta_dirty) GDX_CUDA(cudaMemsetAsync(W.cta_bcs.get(), 0, W.cta_bcs.bytes(), s));
    W.cta_dirty = true;
    timed_launch(g, "bc_cta", [&] {
        if (a.any_heavy) {
            if (CS == 4)
                k_bc_cta<4, true><<<grid, kBcCta, 0, s>>>(a);
            else if (CS == 2)
                k_bc_cta<2, true><<<grid, kBcCta, 0, s>>>(a);
            else
                k_bc_cta<1, true><<<grid, kBcCta, 0, s>>>(a);
        } else {
            const int dyn = kBcPipe ? int(kBcCta * sizeof(BcPf)) : 0;
            static bool attr_set = false;
            if (dyn && !attr_set) {
                GDX_CUDA(cudaFuncSetAttribute(k_bc_cta<4, false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
                GDX_CUDA(cudaFuncSetAttribute(k_bc_cta<2, false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
                GDX_CUDA(cudaFuncSetAttribute(k_bc_cta<1, false>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
                attr_set = true;
            }
            if (CS == 4)
                k_bc_cta<4, false><<<grid, kBcCta, dyn, s>>>(a);
            else if (CS == 2)
                k_bc_cta<2, false><<<grid, kBcCta, dyn, s>>>(a);
            else
                k_bc_cta<1, false><<<grid, kBcCta, dyn, s>>>(a);
        }
    });
    timed_launch(g, "bc_sum", [&] {
        k_bc_slot_sum<<<blocks_for((n + 1) / 2, 256, g->num_sms * 8), 256, 0, s>>>(
            int32_t(n), bcs_stride(n), slots, a.bcs, a.bc);
    });
    W.cta_dirty = false;
    launches += 2;
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, W.ctrs.get(), kBcCtrs * 8, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    totals[kReached] += h[kReached];
    totals[kFwdScan] += h[kFwdScan];
    totals[kBwdScan] += h[kBwdScan];
    totals[kDag] += h[kDag];
    max_levels = std::max<int>(max_levels, int(h[kLevels]));
    if (trace) {
        std::vector<unsigned long long> t(size_t(2) * a.trace_cap);
        GDX_CUDA(cudaMemcpy(t.data(), a.trace, t.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(trace, "w")) {
            for (int k = 1; k < a.trace_cap && t[2 * k]; ++k)
                std::fprintf(f, "%llu %lld\n", t[2 * k] - t[2 * k - 2], (long long)int(t[2 * k + 1]));
            std::fclose(f);
        }
    }
}

}  // namespace gdx

using namespace gdx;

extern "C" int gdx_bc(gdx_graph* g, const int32_t* sources, int32_t nsrc, double* bc_out,
                      gdx_stats* stats) {
    return guard_impl([&] {
        if (!g || (!bc_out && g->n > 0) || (nsrc > 0 && !sources) || nsrc < 0)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        // interpreter.cpp:1115-1118 -- every node of the set must be in range.
        std::vector<int32_t> hsrc(sources, sources + nsrc);
        for (int32_t x : hsrc)
            if (x < 0 || x >= g->n)
                fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: node id " + std::to_string(x) +
                                               " out of range [0, " + std::to_string(g->n) + ")");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        if (g->n == 0) return;
        GraphScope dg(g);
        cudaStream_t s = g->stream;
        if (!g->bc) g->bc = std::make_unique<BcWork>();
        auto& W = *g->bc;
        const int64_t n = g->n;
        W.bc.ensure(n);
        W.ctrs.ensure(kBcCtrs);
        GDX_CUDA(cudaMemsetAsync(W.bc.get(), 0, n * sizeof(double), s));
        unsigned long long totals[kBcCtrs] = {};
        int launches = 0, max_levels = 0;
        bool used_kids = false;
        // CTA-cluster-per-source mode when there are enough sources to fill
        // the GPU with independent BFS trees, or when no vertex has more than
        // kHeavy edges (low-degree, typically high-diameter graphs: barrier
        // latency dominates, measured 2x faster even for one source); the
        // grid-wide kernels otherwise (few sources on skewed graphs, whose
        // wide levels want every SM).  GDX_BC_MODE=grid|cta overrides.
        const char* mode = std::getenv("GDX_BC_MODE");
        const bool cta_mode = mode ? std::string(mode) == "cta"
                                   : nsrc >= std::max(16, g->num_sms / 4) ||
                                         (nsrc > 0 && graph_max_degree(g) <= kHeavy);
        if (nsrc > 0 && cta_mode) {
            run_bc_cta(g, hsrc, totals, launches, max_levels, used_kids);
        } else if (nsrc > 0) {
            if (W.cta_grid > 0) {  // switch back from CTA mode: release its buffers
                W.cta_rec.release();
                W.cta_base.release();
                W.cta_bcs.release();
                W.cta_log.release();
                W.cta_loff.release();
                        W.cta_grid = 0;
                W.batch = 0;
            }
            // batch size: 36 bytes per (source, vertex) of state + log
            size_t free_b = 0, tot_b = 0;
            GDX_CUDA(cudaMemGetInfo(&free_b, &tot_b));
            const size_t per_src = size_t(n) * 36;
            const size_t have = W.level.bytes() + W.sig.bytes() + W.delta.bytes() + W.log.bytes();
            int64_t S = int64_t(double(free_b + have - std::min(free_b + have, (size_t(n) + 2) * 8)) *
                                0.75 / double(per_src));
            S = std::max<int64_t>(1, std::min<int64_t>({S, nsrc, 4096}));
            if (W.batch < S) {
                W.level.release();
                W.sig.release();
                W.delta.release();
                W.log.release();
                W.level.alloc(size_t(S) * n);
                W.sig.alloc(size_t(S) * n * 2);
                W.delta.alloc(size_t(S) * n);
                W.log.alloc(size_t(S) * n);
                W.batch = int32_t(S);
            }
            W.lvl_start.ensure(size_t(n) + 2);
            W.sources.ensure(size_t(W.batch));
            if (W.grid == 0) {
                int a1 = 0, a2 = 0;
                const char* bs = std::getenv("GDX_BC_BLOCK");
                W.block = bs ? std::atoi(bs) : 256;
                if (W.block != 512 && W.block != 1024) W.block = 256;
                if (W.block == 256) {
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, k_bc_forward<256>, 256, 0));
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a2, k_bc_backward<256>, 256, 0));
                } else if (W.block == 512) {
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, k_bc_forward<512>, 512, 0));
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a2, k_bc_backward<512>, 512, 0));
                } else {
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, k_bc_forward<1024>, 1024, 0));
                    GDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a2, k_bc_backward<1024>, 1024, 0));
                }
                const int per_sm = std::min(a1, a2);
                if (per_sm < 1) fail(GDX_ERR_CUDA, "CudaError: bc kernels cannot be resident");
                W.grid = per_sm * g->num_sms;
            }
            BcArgs a;
            a.n = g->n;
            a.undirected = !g->directed;
            a.offsets = g->offsets.get();
            a.dests = g->dests.get();
            a.in_offsets = g->in_offsets();
            a.in_srcs = g->in_srcs();
            a.sources = W.sources.get();
            a.level = W.level.get();
            a.sig = reinterpret_cast<double2*>(W.sig.get());
            a.delta = W.delta.get();
            a.log = W.log.get();
            a.lvl_cnt = W.lvl_start.get();
            a.bc = W.bc.get();
            a.ctr = W.ctrs.get();
            if (g->directed && (!a.in_offsets || !a.in_srcs))
                fail(GDX_ERR_UNSUPPORTED, "Unsupported: directed BC needs the reverse CSR");
            unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
            for (int32_t b0 = 0; b0 < nsrc; b0 += W.batch) {
                const int32_t cnt = std::min<int32_t>(W.batch, nsrc - b0);
                a.S = cnt;
                GDX_CUDA(cudaMemcpyAsync(W.sources.get(), hsrc.data() + b0, cnt * 4,
                                         cudaMemcpyHostToDevice, s));
                GDX_CUDA(cudaMemsetAsync(W.level.get(), 0xff, size_t(cnt) * n * 4, s));
                GDX_CUDA(cudaMemsetAsync(W.lvl_start.get(), 0, (size_t(n) + 2) * 8, s));
                GDX_CUDA(cudaMemsetAsync(W.ctrs.get(), 0, kBcCtrs * 8, s));
                timed_launch(g, "bc_seed", [&] { k_bc_seed<<<blocks_for(cnt, 256, 1024), 256, 0, s>>>(a); });
                void* args[] = {&a};
                timed_launch(g, "bc_forward", [&] {
                    void* fn = W.block == 256 ? (void*)k_bc_forward<256>
                               : W.block == 512 ? (void*)k_bc_forward<512> : (void*)k_bc_forward<1024>;
                    GDX_CUDA(cudaLaunchCooperativeKernel(fn, dim3(W.grid), dim3(W.block), args, 0, s));
                });
                timed_launch(g, "bc_backward", [&] {
                    void* fn = W.block == 256 ? (void*)k_bc_backward<256>
                               : W.block == 512 ? (void*)k_bc_backward<512> : (void*)k_bc_backward<1024>;
                    GDX_CUDA(cudaLaunchCooperativeKernel(fn, dim3(W.grid), dim3(W.block), args, 0, s));
                });
                timed_launch(g, "bc_sum", [&] {
                    k_bc_batch_sum<<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(a);
                });
                launches += 4;
                GDX_CUDA(cudaMemcpyAsync(h, W.ctrs.get(), kBcCtrs * 8, cudaMemcpyDeviceToHost, s));
                GDX_CUDA(cudaStreamSynchronize(s));
                totals[kReached] += h[kTail];
                totals[kFwdScan] += h[kFwdScan];
                totals[kBwdScan] += h[kBwdScan];
                totals[kDag] += h[kDag];
                max_levels = std::max<int>(max_levels, int(h[kLevels]));
            }
        }
        copy_out(g, bc_out, W.bc.get(), size_t(n) * sizeof(double));
        GDX_CUDA(cudaStreamSynchronize(s));
        if (stats) {
            stats->rounds = max_levels;
            stats->launches = launches;
            stats->vertices_visited = int64_t(totals[kReached]);
            // m_scanned (the forward pass's scanned edges; the backward pass
            // reads the same adjacency or the recorded children) and the DAG
            // edges (counted once, as parents in the forward pass)
            stats->edges_visited = int64_t(totals[kFwdScan]);
            stats->updates = int64_t(totals[kDag]);
            // SURVEY.md 8(d), per source: 48 n_reached + 16 m_scanned + 24 m_dag.
            // Per reached vertex: offsets, level, sigma, delta, bc read-modify-
            // write; per scanned edge (m_scanned = edges the forward pass
            // scanned): dest + level in each direction; per DAG edge: the sigma
            // atomic forward, sigma / delta reads backward.  Charged the same
            // whether or not the backward pass reads recorded children instead
            // of rescanning the adjacency (an implementation choice).
            (void)used_kids;
            stats->algorithmic_bytes = 48.0 * totals[kReached] + 16.0 * totals[kFwdScan] +
                                       24.0 * totals[kDag];
        }
    });
}
