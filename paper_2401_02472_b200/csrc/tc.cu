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
#include <cub/cub.cuh>

#include <cstdlib>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

#ifndef GDX_TC_BLOCK
#define GDX_TC_BLOCK 128  // same-box C3: 4.80 vs 4.86 ms at 256, 4.99 at 512
#endif
constexpr int kTcBlock = GDX_TC_BLOCK;
// degree binning: a vertex with more (oriented) neighbours than this has its
// pairs spread over the whole grid (k_tc_heavy / k_tc_heavy_mid)
constexpr int kTcHeavy = 256;
// acc layout: [count, work, work slots...] (the slots are summed on the host)
constexpr int kTcSlots = 256;

// first index in [lo, hi) with a[i] > x
__device__ inline int32_t upper_bound_dev(const int32_t* __restrict__ a, int32_t lo, int32_t hi,
                                          int32_t x) {
    while (lo < hi) {
        int32_t mid = lo + ((hi - lo) >> 1);
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
        int32_t mid = lo + ((hi - lo) >> 1);
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
        const int32_t len = ve - vb > kTcHeavy ? 0 : ve - vb;  // heavy: k_tc_heavy_mid
        const int32_t hs = valid && len ? upper_bound_dev(dests, vb, ve, v) : 0;  // first w > v
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

// ---------------------------------------------------------------------------
// Undirected graphs: oriented counting.  On a symmetric graph tc.sp's count
// (u < v < w, v the middle vertex) is the number of triangles, which is also
//     sum over v, sum over u in N+(v):  |N+(v) ∩ N+(u)|,   N+(x) = N(x) ∩ (x, inf)
// (each triangle a < b < c is found once, at v = a, u = b, w = c).  This needs
// no binary search in the random list N+(u) and only half the adjacency.
//
// k_tc_orient_count / k_tc_orient_fill build the oriented CSR (off+, adj+)
// inside the call.  k_tc_oriented: a warp owns 32 consecutive vertices; their
// N+ lists are one contiguous range of adj+, staged into the warp's shared
// memory with coalesced loads.  The (v, u) pairs of the 32 lists are spread
// over the lanes; a lane loads N+(u) with 16 B vector loads (one L1 wavefront
// per 4 elements -- the gather is the kernel's bound) and merges it against
// the tail of N+(v) after u in shared memory.  One 64-bit atomic per warp.
// ---------------------------------------------------------------------------
__global__ void k_tc_orient_count(int32_t n, const int32_t* __restrict__ offsets,
                                  const int32_t* __restrict__ dests, int32_t* cnt,
                                  int32_t* hs) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = offsets[v], e = offsets[v + 1];
        const int32_t h = upper_bound_dev(dests, b, e, int32_t(v));
        hs[v] = h;
        cnt[v] = e - h;
    }
}

__global__ void k_tc_orient_fill(int32_t n, const int32_t* __restrict__ dests,
                                 const int32_t* __restrict__ hs,
                                 const int32_t* __restrict__ off_plus, int32_t* adj_plus) {
    // A warp fills the contiguous adj+ range of 32 consecutive vertices with
    // coalesced stores; the source row of each output slot is found by a
    // shuffle binary search over the 32 list starts.
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v0 = w * 32; v0 < n; v0 += nw * 32) {
        const int64_t v = v0 + lane;
        const int32_t src = v < n ? hs[v] : 0;
        const int32_t dst = v < n ? off_plus[v] : INT32_MAX;
        const int32_t d0 = __shfl_sync(full, dst, 0);
        const int32_t d1 = v0 + 32 <= n ? off_plus[v0 + 32] : off_plus[n];
        for (int32_t d = d0 + lane; d - lane < d1; d += 32) {
            int k = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int c = k + step;
                const int32_t st = __shfl_sync(full, dst, c & 31);
                if (c < 32 && st <= d) k = c;
            }
            const int32_t ks = __shfl_sync(full, src, k);
            const int32_t kd = __shfl_sync(full, dst, k);
            if (d < d1) adj_plus[d] = dests[ks + (d - kd)];
        }
    }
}

// Pair filter (GDX_TC_SIG): every vertex x has a 64-bit signature -- one bit
// per element w of N+(x), bit = hash(w) -- and sigp[i] = signature of adj+[i]
// sits beside each entry of adj+, so the v side of a pair streams it in order.
// A pair (v, u) whose short tail of N+(v) after u shares no signature bit with
// N+(u) has no common element: it is skipped without touching N+(u) or its
// off+ range -- the random DRAM access that bounds the kernel.  Exact: a
// common element would set the same bit on both sides.
#ifndef GDX_TC_SIG
#define GDX_TC_SIG 1
#endif
constexpr bool kTcSig = GDX_TC_SIG != 0;
#ifndef GDX_TC_SIGTAIL
#define GDX_TC_SIGTAIL 16
#endif
constexpr int kSigTail = GDX_TC_SIGTAIL;  // longer tails are not filtered (hashing them costs more)
#ifndef GDX_TC_SIGW
#define GDX_TC_SIGW 2  // signature words of 64 bits (same-box C3: 3.37 ms at 2, 3.46 at 1)
#endif
constexpr int kSigW = GDX_TC_SIGW;
struct Sig {
    unsigned long long w[kSigW];
};
__device__ __forceinline__ void sig_add(Sig& s, int32_t x) {
    const uint32_t h = uint32_t(x) * 0x9E3779B1u;
    if (kSigW == 1) {
        s.w[0] |= 1ull << (h >> 26);
    } else {
#pragma unroll
        for (int q = 0; q < kSigW; ++q) s.w[q] |= (h >> 31) == uint32_t(q & 1) ? 1ull << ((h >> 25) & 63) : 0ull;
    }
}
// the same bit from its precomputed 7-bit index (h >> 25)
__device__ __forceinline__ void sig_add_bit(Sig& s, unsigned b) {
    if (kSigW == 1) {
        s.w[0] |= 1ull << (b >> 1);
    } else {
#pragma unroll
        for (int q = 0; q < kSigW; ++q) s.w[q] |= (b >> 6) == unsigned(q & 1) ? 1ull << (b & 63) : 0ull;
    }
}
__device__ __forceinline__ bool sig_meet(const Sig& a, const Sig& b) {
    unsigned long long x = 0;
#pragma unroll
    for (int q = 0; q < kSigW; ++q) x |= a.w[q] & b.w[q];
    return x != 0;
}
__global__ void k_tc_sig(int32_t n, const int32_t* __restrict__ off_plus,
                         const int32_t* __restrict__ adj, Sig* __restrict__ sig) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        Sig b{};
        for (int32_t i = off_plus[v], e = off_plus[v + 1]; i < e; ++i) sig_add(b, adj[i]);
        sig[v] = b;
    }
}
__global__ void k_tc_sigp(int64_t cnt, const int32_t* __restrict__ adj,
                          const Sig* __restrict__ sig, Sig* __restrict__ sigp) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        sigp[i] = sig[adj[i]];
}

#ifndef GDX_TC_STAGE
#define GDX_TC_STAGE 512
#endif
constexpr int kTcStage = GDX_TC_STAGE;  // ints of staged N+ lists per warp

#ifndef GDX_TC_THREADS_SM
#define GDX_TC_THREADS_SM 1536  // resident threads per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(kTcBlock, GDX_TC_THREADS_SM / kTcBlock) k_tc_oriented(int32_t v_begin, int32_t v_end,
                                                          const int32_t* __restrict__ off_plus,
                                                          const int32_t* __restrict__ adj,
                                                          unsigned long long* acc,
                                                          const Sig* __restrict__ sigp = nullptr) {
    const unsigned full = 0xffffffffu;
    __shared__ int32_t stage[kTcBlock / 32][kTcStage];
    __shared__ uint16_t s_list[kTcBlock / 32][kTcStage];  // the warp's pairs that pass the filter
    __shared__ uint8_t s_bit[kTcBlock / 32][kTcStage];    // signature bit of each staged element
    const int lane = threadIdx.x & 31;
    int32_t* sA = stage[threadIdx.x >> 5];
    uint16_t* sL = s_list[threadIdx.x >> 5];
    const int64_t gwarp = (blockIdx.x * (int64_t)kTcBlock + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * (kTcBlock / 32);
    const int4* adj4 = reinterpret_cast<const int4*>(adj);
    unsigned long long count = 0, scanned = 0;
    for (int64_t v0 = v_begin + gwarp * 32; v0 < v_end; v0 += nwarps * 32) {
        const int32_t v = int32_t(v0) + lane;
        const bool valid = v < v_end;
        const int32_t ob = valid ? off_plus[v] : 0;
        const int32_t oe = valid ? off_plus[v + 1] : 0;
        const int32_t r0 = __shfl_sync(full, ob, 0);
        int32_t last_end = oe;
#pragma unroll
        for (int o = 16; o; o >>= 1) last_end = max(last_end, __shfl_xor_sync(full, last_end, o));
        const int32_t rlen = last_end - r0;
        // stage the warp's lists (one contiguous range of adj+) when they fit
        const bool staged = rlen <= kTcStage;
        if (staged)
            for (int32_t i = lane; i < rlen; i += 32) {
                const int32_t x = adj[r0 + i];
                sA[i] = x;
                if (kTcSig && sigp) s_bit[threadIdx.x >> 5][i] = uint8_t((uint32_t(x) * 0x9E3779B1u) >> 25);
            }
        __syncwarp();
        const int32_t* A = staged ? sA - r0 : adj;  // A[x] for x in [r0, last_end)
        // The pair filter, computed here for every staged entry (its pair is
        // (owner vertex, entry)) in one coalesced pass: the pairs that pass are
        // listed in shared memory and only they are spread over the lanes --
        // a filtered pair costs neither its random N+(u) fetch nor a lane slot.
        const bool filt = kTcSig && sigp && staged;
        int ntp = 0;  // pairs that pass
        if (filt) {
            for (int32_t i0 = 0; i0 < rlen; i0 += 32) {
                const int32_t q = r0 + i0 + lane;
                int k = 0;  // the warp's vertex lane whose list holds entry q
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int c = k + step;
                    const int32_t st = __shfl_sync(full, valid ? ob : INT32_MAX, c & 31);
                    if (c < 32 && st <= q) k = c;
                }
                const int32_t kend = __shfl_sync(full, oe, k);
                const int32_t kbeg = __shfl_sync(full, ob, k);
                bool pass = i0 + lane < rlen && q < kend - 1 && kend - kbeg <= kTcHeavy;
                if (pass && kend - q - 1 <= kSigTail) {
                    Sig ts{};
                    const uint8_t* sb = s_bit[threadIdx.x >> 5] - r0;
                    for (int32_t x = q + 1; x < kend; ++x) sig_add_bit(ts, sb[x]);
                    pass = sig_meet(ts, sigp[q]);
                }
                const unsigned m = __ballot_sync(full, pass);
                if (pass) sL[ntp + __popc(m & ((1u << lane) - 1))] = uint16_t(q - r0);
                ntp += __popc(m);
            }
            __syncwarp();
        }
        // pairs (v, i): u = N+(v)[i] for i < len-1 (the last u has no tail)
        // heavy vertices (|N+(v)| > kTcHeavy) are left to k_tc_heavy, which
        // spreads their pairs over the whole grid instead of one warp
        const int32_t np = oe - ob > kTcHeavy ? 0 : max(oe - ob - 1, 0);
        int incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(full, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(full, incl, 31);
        const int excl = incl - np;
        // The off+ range of the next pair's u is loaded while the current
        // pair merges; the current pair's first three 16 B words of N+(u)
        // are issued together (one L1 wavefront per 4 elements).
        auto locate = [&](int j, int32_t& pu, int32_t& koe) {
            int k = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int c = k + step;
                const int ex = __shfl_sync(full, excl, c & 31);
                if (c < 32 && ex <= j) k = c;
            }
            const int32_t kob = __shfl_sync(full, ob, k);
            koe = __shfl_sync(full, oe, k);
            pu = kob + (j - __shfl_sync(full, excl, k));
        };
        // filtered warps walk their listed pairs: entry -> owner list's end
        auto locate_f = [&](int j, int32_t& pu_, int32_t& koe_) {
            pu_ = r0 + (j < ntp ? int32_t(sL[j]) : 0);
            int k = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int c = k + step;
                const int32_t st = __shfl_sync(full, valid ? ob : INT32_MAX, c & 31);
                if (c < 32 && st <= pu_) k = c;
            }
            koe_ = __shfl_sync(full, oe, k);
        };
        const int npairs = filt ? ntp : total;
        int32_t pu = 0, koe = 0, bb = 0, be = 0;
        if (filt) locate_f(lane, pu, koe); else locate(lane, pu, koe);
        if (lane < npairs) {
            const int32_t u = A[pu];
            bb = off_plus[u];
            be = off_plus[u + 1];
        }
        for (int j0 = 0; j0 < npairs; j0 += 32) {
            const bool have = j0 + lane < npairs;
            const int32_t cpu = pu, ckoe = koe, cbb = bb, cbe = be;
            if (filt) locate_f(j0 + 32 + lane, pu, koe); else locate(j0 + 32 + lane, pu, koe);
            if (j0 + 32 + lane < npairs) {
                const int32_t u = A[pu];
                bb = off_plus[u];
                be = off_plus[u + 1];
            }
            if (!have || cbb >= cbe) continue;
            const int32_t q0 = cbb & ~3;
            int4 w[3];
#pragma unroll
            for (int t = 0; t < 3; ++t)
                w[t] = q0 + 4 * t < cbe ? adj4[(q0 >> 2) + t]
                                        : make_int4(INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX);
            int32_t p = cpu + 1;  // tail of N+(v) after u: A[p .. ckoe)
            scanned += (ckoe - p) + (cbe - cbb) + 2;
            const int32_t la = ckoe - p, lb = cbe - cbb;
            if (la > 16 * lb + 16 || lb > 16 * la + 16) {
                // very unequal lists (hubs of skewed graphs): walk the short one,
                // binary-search the long one (O(short * log long), not O(long))
                unsigned long long c = 0;
                if (la <= lb) {
                    int32_t lo = cbb;
                    for (int32_t i = p; i < ckoe && lo < cbe; ++i) {
                        const int32_t x = A[i];
                        int32_t hi = cbe;
                        while (lo < hi) {
                            const int32_t mid = lo + ((hi - lo) >> 1);
                            if (adj[mid] < x) lo = mid + 1; else hi = mid;
                        }
                        if (lo < cbe && adj[lo] == x) ++c;
                    }
                } else {
                    int32_t lo = p;
                    for (int32_t i = cbb; i < cbe && lo < ckoe; ++i) {
                        const int32_t x = adj[i];
                        int32_t hi = ckoe;
                        while (lo < hi) {
                            const int32_t mid = lo + ((hi - lo) >> 1);
                            if (A[mid] < x) lo = mid + 1; else hi = mid;
                        }
                        if (lo < ckoe && A[lo] == x) ++c;
                    }
                }
                count += c;
                continue;
            }
            int32_t ap = A[p];
            const int32_t a_last = A[ckoe - 1];
            unsigned long long c = 0;
            bool done = false;
#pragma unroll
            for (int t = 0; t < 12; ++t) {
                const int32_t idx = q0 + t;
                const int32_t xv = (&w[t >> 2].x)[t & 3];
                if (!done && idx >= cbb && idx < cbe) {
                    while (ap < xv && ++p < ckoe) ap = A[p];
                    if (p >= ckoe || xv > a_last)
                        done = true;
                    else if (ap == xv)
                        ++c;
                }
            }
            for (int32_t q = q0 + 12; !done && q < cbe; q += 4) {  // long lists
                const int4 w4 = adj4[q >> 2];
                const int32_t x[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (!done && q + t < cbe) {
                        const int32_t xv = x[t];
                        while (ap < xv && ++p < ckoe) ap = A[p];
                        if (p >= ckoe || xv > a_last)
                            done = true;
                        else if (ap == xv)
                            ++c;
                    }
                }
            }
            count += c;
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        count += __shfl_xor_sync(full, count, o);
        scanned += __shfl_xor_sync(full, scanned, o);
    }
    if (lane == 0) {
        if (count) atomicAdd(&acc[0], count);
        // the work counter is spread over kTcSlots addresses: ~300K warps
        // adding to one address serialise in L2
        if (scanned) atomicAdd(&acc[2 + (blockIdx.x & (kTcSlots - 1))], scanned);
    }
}

// |N+(a) tail ∩ N+(u)| for one pair: merge, or walk the shorter list and
// binary-search the longer one when their lengths differ by > 16x.
__device__ inline unsigned long long tc_intersect(const int32_t* __restrict__ adj, int32_t p,
                                                  int32_t ae, int32_t bb, int32_t be) {
    const int32_t la = ae - p, lb = be - bb;
    if (la <= 0 || lb <= 0) return 0;
    unsigned long long c = 0;
    if (la > 16 * lb || lb > 16 * la) {
        const int32_t s0 = la <= lb ? p : bb, s1 = la <= lb ? ae : be;
        int32_t lo = la <= lb ? bb : p;
        const int32_t hi0 = la <= lb ? be : ae;
        for (int32_t i = s0; i < s1 && lo < hi0; ++i) {
            const int32_t x = adj[i];
            int32_t hi = hi0;
            while (lo < hi) {
                const int32_t mid = lo + ((hi - lo) >> 1);
                if (adj[mid] < x) lo = mid + 1; else hi = mid;
            }
            if (lo < hi0 && adj[lo] == x) ++c;
        }
        return c;
    }
    int32_t x = adj[p], y = adj[bb];
    while (true) {
        if (x < y) {
            if (++p >= ae) break;
            x = adj[p];
        } else if (y < x) {
            if (++bb >= be) break;
            y = adj[bb];
        } else {
            ++c;
            if (++p >= ae || ++bb >= be) break;
            x = adj[p];
            y = adj[bb];
        }
    }
    return c;
}

// Degree binning: vertices with more than kTcHeavy oriented neighbours.
__global__ void k_tc_heavy_list(int32_t v_begin, int32_t v_end, const int32_t* __restrict__ off_plus,
                                int32_t* heavy, int32_t* cnt) {
    for (int64_t v = v_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < v_end;
         v += (int64_t)gridDim.x * blockDim.x)
        if (off_plus[v + 1] - off_plus[v] > kTcHeavy) heavy[atomicAdd(cnt, 1)] = int32_t(v);
}

__global__ void k_tc_heavy_sizes(int32_t nh, const int32_t* __restrict__ heavy,
                                 const int32_t* __restrict__ off, int32_t drop, long long* sizes) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += gridDim.x * blockDim.x) {
        const int32_t v = heavy[h];
        sizes[h] = max(off[v + 1] - off[v] - drop, 0);
    }
}

// Directed graphs (tc.sp's middle vertex): the edges (v, u), u < v, of the
// heavy middle vertices, one per thread over the whole grid.
__global__ void __launch_bounds__(256) k_tc_heavy_mid(int32_t nh, const int32_t* __restrict__ heavy,
                                                      const long long* __restrict__ pre,
                                                      const int32_t* __restrict__ offsets,
                                                      const int32_t* __restrict__ dests,
                                                      unsigned long long* acc) {
    unsigned long long count = 0, scanned = 0;
    const long long total = pre[nh];
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total;
         j += (long long)gridDim.x * blockDim.x) {
        int32_t lo = 0, hi = nh;  // last h with pre[h] <= j
        while (hi - lo > 1) {
            const int32_t mid = lo + ((hi - lo) >> 1);
            if (pre[mid] <= j) lo = mid; else hi = mid;
        }
        const int32_t v = heavy[lo];
        const int32_t vb = offsets[v], ve = offsets[v + 1];
        const int32_t u = dests[vb + int32_t(j - pre[lo])];
        if (u >= v) continue;
        const int32_t hs = upper_bound_dev(dests, vb, ve, v);  // N(v) ∩ (v, inf)
        const int32_t ub = offsets[u], ue = offsets[u + 1];
        const int32_t bs = upper_bound_dev(dests, ub, ue, v);  // N(u) ∩ (v, inf)
        scanned += (ve - hs) + (ue - bs);
        count += tc_intersect(dests, hs, ve, bs, ue);
    }
    for (int o = 16; o; o >>= 1) {
        count += __shfl_xor_sync(0xffffffffu, count, o);
        scanned += __shfl_xor_sync(0xffffffffu, scanned, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (count) atomicAdd(&acc[0], count);
        if (scanned) atomicAdd(&acc[1], scanned);
    }
}

// Lists the vertices of [v_begin, v_end) with more than kTcHeavy entries in
// `off` and the prefix of their pair counts (deg - drop); returns their count.
static int32_t tc_heavy_plan(gdx_graph* g, TcPlan& P, int32_t v_begin, int32_t v_end,
                             const int32_t* off, int32_t drop, long long* total_pairs) {
    cudaStream_t s = g->stream;
    *total_pairs = 0;
    if (v_end <= v_begin) return 0;
    P.heavy.ensure(size_t(v_end - v_begin) + 1);
    P.heavy_cnt.ensure(1);
    GDX_CUDA(cudaMemsetAsync(P.heavy_cnt.get(), 0, 4, s));
    k_tc_heavy_list<<<blocks_for(v_end - v_begin, 256, g->num_sms * 8), 256, 0, s>>>(
        v_begin, v_end, off, P.heavy.get(), P.heavy_cnt.get());
    GDX_LAUNCH_CHECK();
    int32_t nh = 0;
    GDX_CUDA(cudaMemcpyAsync(&nh, P.heavy_cnt.get(), 4, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    if (nh == 0) return 0;
    P.heavy_pre.ensure(size_t(nh) + 1);
    k_tc_heavy_sizes<<<blocks_for(nh, 256, 1024), 256, 0, s>>>(nh, P.heavy.get(), off, drop,
                                                              P.heavy_pre.get() + 1);
    GDX_LAUNCH_CHECK();
    GDX_CUDA(cudaMemsetAsync(P.heavy_pre.get(), 0, 8, s));
    size_t tb = 0;
    GDX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, P.heavy_pre.get() + 1,
                                           P.heavy_pre.get() + 1, nh, s));
    P.scan_tmp.ensure(tb);
    GDX_CUDA(cub::DeviceScan::InclusiveSum(P.scan_tmp.get(), tb, P.heavy_pre.get() + 1,
                                           P.heavy_pre.get() + 1, nh, s));
    GDX_CUDA(cudaMemcpyAsync(total_pairs, P.heavy_pre.get() + nh, 8, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    return nh;
}

// The heavy vertices' pairs (v, i), i < |N+(v)| - 1, one per thread over the
// whole grid (pre[h] = first pair of heavy vertex h).
__global__ void __launch_bounds__(256) k_tc_heavy(int32_t nh, const int32_t* __restrict__ heavy,
                                                  const long long* __restrict__ pre,
                                                  const int32_t* __restrict__ off_plus,
                                                  const int32_t* __restrict__ adj,
                                                  unsigned long long* acc) {
    unsigned long long count = 0, scanned = 0;
    const long long total = pre[nh];
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total;
         j += (long long)gridDim.x * blockDim.x) {
        int32_t lo = 0, hi = nh;  // last h with pre[h] <= j
        while (hi - lo > 1) {
            const int32_t mid = lo + ((hi - lo) >> 1);
            if (pre[mid] <= j) lo = mid; else hi = mid;
        }
        const int32_t v = heavy[lo];
        const int32_t ob = off_plus[v], oe = off_plus[v + 1];
        const int32_t pu = ob + int32_t(j - pre[lo]);
        const int32_t u = adj[pu];
        const int32_t bb = off_plus[u], be = off_plus[u + 1];
        scanned += (oe - pu - 1) + (be - bb) + 2;
        count += tc_intersect(adj, pu + 1, oe, bb, be);
    }
    for (int o = 16; o; o >>= 1) {
        count += __shfl_xor_sync(0xffffffffu, count, o);
        scanned += __shfl_xor_sync(0xffffffffu, scanned, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (count) atomicAdd(&acc[0], count);
        if (scanned) atomicAdd(&acc[1], scanned);
    }
}

// SURVEY.md 8(d) TC work measure: sum over oriented edges v->u of
// d+(u) + d+(v) (= sum_v d+(v)^2 + sum_v sum_{u in N+(v)} d+(u)).
__global__ void k_tc_survey_pairs(int32_t n, const int32_t* __restrict__ off_plus,
                                  const int32_t* __restrict__ adj, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = off_plus[v], e = off_plus[v + 1];
        acc += (unsigned long long)(e - b) * (unsigned long long)(e - b);
        for (int32_t i = b; i < e; ++i) {
            const int32_t u = adj[i];
            acc += (unsigned long long)(off_plus[u + 1] - off_plus[u]);
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// The oriented CSR (off+, adj+) is a derived index of the immutable graph:
// built by the first TC call on a handle and kept with it (like the PageRank
// plan), sized from the scanned total -- not from m/2 + n, which only holds
// for symmetric rows.
static void build_oriented(gdx_graph* g, TcPlan& P) {
    cudaStream_t s = g->stream;
    const int32_t n = g->n;
    P.off_plus.ensure(size_t(n) + 1);
    P.hi_start.ensure(size_t(n) + 1);
    static const int orient_per_sm = [] {  // blocks per SM of the orientation passes
        const char* e = std::getenv("GDX_TC_ORIENT_GRID");
        return e ? std::max(1, std::atoi(e)) : 64;  // same-box C3: count 0.204 vs 0.227 ms at 16
    }();
    const int grid_v = blocks_for(n, 256, g->num_sms * orient_per_sm);
    timed_launch(g, "tc_orient", [&] {
        k_tc_orient_count<<<grid_v, 256, 0, s>>>(n, g->offsets.get(), g->dests.get(),
                                                 P.off_plus.get(), P.hi_start.get());
    });
    size_t bytes = 0;
    GDX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, P.off_plus.get(), P.off_plus.get(),
                                           n + 1, s));
    P.scan_tmp.ensure(bytes);
    // exclusive scan over n+1 entries: off_plus[n] = total (the count slot n is zeroed)
    GDX_CUDA(cudaMemsetAsync(P.off_plus.get() + n, 0, 4, s));
    GDX_CUDA(cub::DeviceScan::ExclusiveSum(P.scan_tmp.get(), bytes, P.off_plus.get(),
                                           P.off_plus.get(), n + 1, s));
    int32_t* h = reinterpret_cast<int32_t*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h, P.off_plus.get() + n, 4, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    const int64_t total = h[0];  // oriented entries
    P.adj_plus.ensure(size_t(total) + 8);
    timed_launch(g, "tc_orient_fill", [&] {
        k_tc_orient_fill<<<grid_v, 256, 0, s>>>(n, g->dests.get(), P.hi_start.get(),
                                                P.off_plus.get(), P.adj_plus.get());
    });
    DevBuf<unsigned long long> sp(1);
    GDX_CUDA(cudaMemsetAsync(sp.get(), 0, 8, s));
    k_tc_survey_pairs<<<blocks_for(n, 256, g->num_sms * 8), 256, 0, s>>>(n, P.off_plus.get(),
                                                                         P.adj_plus.get(), sp.get());
    GDX_LAUNCH_CHECK();
    unsigned long long* h64 = reinterpret_cast<unsigned long long*>(g->pinned);
    GDX_CUDA(cudaMemcpyAsync(h64, sp.get(), 8, cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    P.survey_pairs = double(h64[0]);
    if (kTcSig && total > 0) {  // the pair filter's signatures: sig per vertex, sigp per entry
        DevBuf<unsigned long long> sig{size_t(n) * kSigW};
        P.sigp.ensure(size_t(total) * kSigW);
        timed_launch(g, "tc_sig", [&] {
            k_tc_sig<<<grid_v, 256, 0, s>>>(n, P.off_plus.get(), P.adj_plus.get(),
                                            reinterpret_cast<Sig*>(sig.get()));
            k_tc_sigp<<<blocks_for(total, 256, g->num_sms * 16), 256, 0, s>>>(
                total, P.adj_plus.get(), reinterpret_cast<const Sig*>(sig.get()),
                reinterpret_cast<Sig*>(P.sigp.get()));
        });
    }
    P.oriented = true;
}

static void run_tc_oriented(gdx_graph* g, int32_t v_begin, int32_t v_end, gdx_stats* stats) {
    cudaStream_t s = g->stream;
    auto& P = *g->tc;
    const bool built_now = !P.oriented;
    if (built_now) build_oriented(g, P);
    if (v_end > v_begin) {
        const int64_t groups = (int64_t(v_end) - v_begin + 31) / 32;
        const char* cap = std::getenv("GDX_TC_GRID_CAP");  // blocks per SM (A/B)
        const int grid = blocks_for(groups * 32, kTcBlock,
                                    (cap ? std::max(1, std::atoi(cap)) : 512) * g->num_sms);
        timed_launch(g, "tc", [&] {
            k_tc_oriented<<<grid, kTcBlock, 0, s>>>(v_begin, v_end, P.off_plus.get(),
                                                    P.adj_plus.get(), P.acc.get(),
                                                    kTcSig ? reinterpret_cast<const Sig*>(P.sigp.get())
                                                           : nullptr);
        });
    }
    // degree binning: the heavy vertices' pairs over the whole grid
    int heavy_launches = 0;
    long long pairs = 0;
    const int32_t nh = tc_heavy_plan(g, P, v_begin, v_end, P.off_plus.get(), 1, &pairs);
    if (nh > 0 && pairs > 0) {
        const int grid = blocks_for(pairs, 256, g->num_sms * 16);
        timed_launch(g, "tc_heavy", [&] {
            k_tc_heavy<<<grid, 256, 0, s>>>(nh, P.heavy.get(), P.heavy_pre.get(), P.off_plus.get(),
                                            P.adj_plus.get(), P.acc.get());
        });
        heavy_launches = 1;
    }
    if (stats) stats->launches = (built_now ? 3 : 0) + (v_end > v_begin) + heavy_launches;
}

static void run_tc(gdx_graph* g, int32_t v_begin, int32_t v_end, int64_t* count_out,
                   gdx_stats* stats) {
    if (!g->dests.get() && g->m > 0)
        fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
    GraphScope dg(g);
    cudaStream_t s = g->stream;
    if (!g->tc) g->tc = std::make_unique<TcPlan>();
    auto& P = *g->tc;
    P.acc.ensure(2 + kTcSlots);
    GDX_CUDA(cudaMemsetAsync(P.acc.get(), 0, (2 + kTcSlots) * sizeof(unsigned long long), s));
    v_begin = std::max(v_begin, 0);
    v_end = std::min(v_end, g->n);
    const bool oriented = !g->directed && std::getenv("GDX_TC_MIDDLE") == nullptr;
    if (oriented) {
        run_tc_oriented(g, v_begin, v_end, stats);
    } else if (v_end > v_begin) {
        const int64_t groups = (int64_t(v_end) - v_begin + 31) / 32;
        const int grid = blocks_for(groups * 32, kTcBlock, g->num_sms * 16);
        timed_launch(g, "tc", [&] {
            k_tc<<<grid, kTcBlock, 0, s>>>(v_begin, v_end, g->offsets.get(), g->dests.get(),
                                           P.acc.get());
        });
        long long pairs = 0;
        const int32_t nh = tc_heavy_plan(g, P, v_begin, v_end, g->offsets.get(), 0, &pairs);
        if (nh > 0 && pairs > 0)
            timed_launch(g, "tc_heavy", [&] {
                k_tc_heavy_mid<<<blocks_for(pairs, 256, g->num_sms * 16), 256, 0, s>>>(
                    nh, P.heavy.get(), P.heavy_pre.get(), g->offsets.get(), g->dests.get(),
                    P.acc.get());
            });
    }
    unsigned long long* h = reinterpret_cast<unsigned long long*>(g->pinned);
    static_assert((2 + kTcSlots) * sizeof(unsigned long long) <= 4096, "pinned staging page");
    GDX_CUDA(cudaMemcpyAsync(h, P.acc.get(), (2 + kTcSlots) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
    GDX_CUDA(cudaStreamSynchronize(s));
    *count_out = int64_t(h[0]);
    for (int q = 0; q < kTcSlots; ++q) h[1] += h[2 + q];
    if (stats) {
        stats->rounds = 1;
        if (!oriented) stats->launches = v_end > v_begin ? 1 : 0;
        stats->vertices_visited = int64_t(v_end) - v_begin;
        stats->edges_visited = int64_t(h[1]);
        stats->updates = int64_t(h[0]);
        // DESIGN.md "TC bytes".  Middle-vertex kernel: offsets 4(n+1) +
        // adjacency scan 4m + 4 per element of every intersected list.
        // Oriented kernel: orientation (offsets 4(n+1) read, dests 4m read,
        // adj+ 2m + off+ 4(n+1) written) + N+ staging 2m + per pair the off+
        // pair of u (8) and 4 per element of both merged lists.
        // Oriented kernel over the whole graph: SURVEY.md 8(d) exactly,
        // 4(n+1) + 4m + 4 * sum over oriented edges of (d+(u) + d+(v)).
        const double frac = g->n ? double(int64_t(v_end) - v_begin) / g->n : 0.0;
        if (oriented && v_begin == 0 && v_end == g->n)
            stats->algorithmic_bytes = 4.0 * (g->n + 1) + 4.0 * g->m + 4.0 * P.survey_pairs;
        else if (oriented)
            stats->algorithmic_bytes = frac * (4.0 * (g->n + 1) + 4.0 * g->m) + 4.0 * double(h[1]);
        else
            stats->algorithmic_bytes =
                frac * (4.0 * (g->n + 1) + 4.0 * g->m) + 4.0 * double(h[1]);
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
