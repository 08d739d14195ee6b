// gdx_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see gdx_oracle.h).
//
// CPU restatement of the reference hot path.  Each function cites the
// reference file:line it restates (paths relative to /root/reference/proj).
// Pinned against the reference itself (oracle/_ref) and tests/golden/.
#include "gdx_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <functional>
#include <limits>
#include <queue>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(const std::string& msg) {
    g_err = msg;
    return 1;
}

constexpr int64_t kInf = INT64_MAX / 2;  // oracles.hpp:12

int clamp_threads(int t) {
    if (t <= 0) t = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, t);
}

// Dynamic-chunk parallel for over [0, n).
void parallel_for(int64_t n, int nthreads, int64_t chunk,
                  const std::function<void(int, int64_t, int64_t)>& body) {
    nthreads = clamp_threads(nthreads);
    if (nthreads == 1 || n <= chunk) {
        body(0, 0, n);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] {
            while (true) {
                int64_t b = next.fetch_add(chunk);
                if (b >= n) break;
                body(t, b, std::min(n, b + chunk));
            }
        });
    for (auto& th : pool) th.join();
}

struct View {
    const orc_csr* g;
    int32_t outdeg(int32_t v) const { return g->offsets[v + 1] - g->offsets[v]; }
    int32_t w(int64_t e) const { return g->weights ? g->weights[e] : 1; }
};

// Counter-based RNG shared (by specification, not by code) with the product's
// GPU generators: splitmix64 finaliser keyed by (seed, stream).
inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed + stream * 0xD1B54A32D192ED03ULL);
}
inline uint64_t ctr_hash(uint64_t key, uint64_t ctr) { return mix64(key ^ mix64(ctr)); }
inline double ctr_unit(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }
inline uint32_t ctr_bounded(uint64_t h, uint32_t n) {
    return static_cast<uint32_t>((static_cast<unsigned __int128>(h) * n) >> 64);
}
enum : uint64_t { kStreamRmat = 1, kStreamUniform = 2, kStreamGrid = 3, kStreamWeight = 4 };

// Extended-exponent path count: value = m * 2^e, m in [1,2) (or m == 0).
// Addition/division reproduce IEEE double results bit-for-bit whenever the
// plain-double computation stays finite.
struct XF {
    double m = 0.0;
    int32_t e = 0;
};
inline XF xf_norm(double s, int32_t e) {
    if (s == 0.0) return {0.0, 0};
    int k = std::ilogb(s);
    return {std::ldexp(s, -k), e + k};
}
inline XF xf_add(XF a, XF b) {
    if (a.m == 0.0) return b;
    if (b.m == 0.0) return a;
    int32_t e = std::max(a.e, b.e);
    double s = std::ldexp(a.m, a.e - e) + std::ldexp(b.m, b.e - e);
    return xf_norm(s, e);
}
inline double xf_ratio(XF a, XF b) {  // a / b as a plain double
    return std::ldexp(a.m / b.m, a.e - b.e);
}

}  // namespace

struct orc_graph {
    int32_t n = 0, m = 0;
    bool directed = true;
    std::vector<int32_t> offsets, dests, weights, rev_offsets, rev_srcs, rev_eid;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// csr.cpp:77-94 -- stable counting transpose; each reverse range comes out
// sorted by source because forward edges are visited in (u, v) order.
static void build_reverse(orc_graph* g) {
    g->rev_offsets.assign(g->n + 1, 0);
    g->rev_srcs.resize(g->m);
    g->rev_eid.resize(g->m);
    for (int32_t e = 0; e < g->m; ++e) g->rev_offsets[g->dests[e] + 1]++;
    for (int32_t i = 0; i < g->n; ++i) g->rev_offsets[i + 1] += g->rev_offsets[i];
    std::vector<int32_t> cur(g->rev_offsets.begin(), g->rev_offsets.end() - 1);
    for (int32_t u = 0; u < g->n; ++u)
        for (int32_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e) {
            int32_t s = cur[g->dests[e]]++;
            g->rev_srcs[s] = u;
            g->rev_eid[s] = e;
        }
}

// csr.cpp:28-75 -- validate, double undirected edges (self loops once), sort
// by (u, v, w), keep the first (= minimum weight) of each (u, v) run.
int orc_build_from_edges(int32_t n, int64_t nedges, const int32_t* u, const int32_t* v,
                         const int32_t* w, int directed, orc_graph** out) {
    if (n < 0) return fail("negative node count");
    struct Raw {
        int32_t u, v, w;
    };
    std::vector<Raw> raw;
    raw.reserve(static_cast<size_t>(nedges) * (directed ? 1 : 2));
    for (int64_t i = 0; i < nedges; ++i) {
        if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n)
            return fail("InvalidEdge: endpoint (" + std::to_string(u[i]) + ", " +
                        std::to_string(v[i]) + ") out of range [0, " + std::to_string(n) + ")");
        int32_t wi = w ? w[i] : 1;
        if (wi < 0)
            return fail("NegativeWeight: edge (" + std::to_string(u[i]) + ", " +
                        std::to_string(v[i]) + ") has weight " + std::to_string(wi));
        raw.push_back({u[i], v[i], wi});
        if (!directed && u[i] != v[i]) raw.push_back({v[i], u[i], wi});
    }
    std::sort(raw.begin(), raw.end(), [](const Raw& a, const Raw& b) {
        if (a.u != b.u) return a.u < b.u;
        if (a.v != b.v) return a.v < b.v;
        return a.w < b.w;
    });
    auto* g = new orc_graph;
    g->n = n;
    g->directed = directed != 0;
    g->offsets.assign(n + 1, 0);
    for (size_t i = 0; i < raw.size(); ++i) {
        if (i > 0 && raw[i].u == raw[i - 1].u && raw[i].v == raw[i - 1].v) continue;
        g->dests.push_back(raw[i].v);
        g->weights.push_back(raw[i].w);
        g->offsets[raw[i].u + 1]++;
    }
    if (g->dests.size() > static_cast<size_t>(INT32_MAX)) {
        delete g;
        return fail("edge count exceeds int32");
    }
    g->m = static_cast<int32_t>(g->dests.size());
    for (int32_t i = 0; i < n; ++i) g->offsets[i + 1] += g->offsets[i];
    build_reverse(g);
    *out = g;
    return 0;
}

// csr.cpp:172-195 -- one mt19937_64 draw per unordered pair in canonical
// (u <= v) CSR order; the mirror slot gets the same weight.
int orc_with_random_weights(orc_graph* g, int32_t lo, int32_t hi, uint64_t seed) {
    if (lo > hi) return fail("weight range is empty");
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int32_t> dist(lo, hi);
    if (g->directed) {
        for (int32_t e = 0; e < g->m; ++e) g->weights[e] = dist(rng);
        return 0;
    }
    for (int32_t a = 0; a < g->n; ++a)
        for (int32_t e = g->offsets[a]; e < g->offsets[a + 1]; ++e) {
            int32_t b = g->dests[e];
            if (b < a) continue;
            int32_t wt = dist(rng);
            g->weights[e] = wt;
            if (b != a) {
                auto first = g->dests.begin() + g->offsets[b];
                auto last = g->dests.begin() + g->offsets[b + 1];
                auto it = std::lower_bound(first, last, a);
                if (it != last && *it == a) g->weights[it - g->dests.begin()] = wt;
            }
        }
    return 0;
}

int orc_graph_from_csr(const orc_csr* c, orc_graph** out) {
    auto* g = new orc_graph;
    g->n = c->n;
    g->m = c->m;
    g->directed = c->directed != 0;
    g->offsets.assign(c->offsets, c->offsets + c->n + 1);
    g->dests.assign(c->dests, c->dests + c->m);
    if (c->weights)
        g->weights.assign(c->weights, c->weights + c->m);
    else
        g->weights.assign(c->m, 1);
    if (c->rev_offsets && c->rev_srcs && c->rev_eid) {
        g->rev_offsets.assign(c->rev_offsets, c->rev_offsets + c->n + 1);
        g->rev_srcs.assign(c->rev_srcs, c->rev_srcs + c->m);
        g->rev_eid.assign(c->rev_eid, c->rev_eid + c->m);
    } else {
        build_reverse(g);
    }
    *out = g;
    return 0;
}

void orc_graph_view(const orc_graph* g, orc_csr* view) {
    view->n = g->n;
    view->m = g->m;
    view->directed = g->directed;
    view->offsets = g->offsets.data();
    view->dests = g->dests.data();
    view->weights = g->weights.data();
    view->rev_offsets = g->rev_offsets.data();
    view->rev_srcs = g->rev_srcs.data();
    view->rev_eid = g->rev_eid.data();
}

void orc_graph_free(orc_graph* g) { delete g; }

// graphgen.cpp:8-16
int orc_gen_uniform_edges(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u, int32_t* v) {
    if (nodes <= 0) return fail("node count must be positive");
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int32_t> pick(0, nodes - 1);
    for (int64_t i = 0; i < edges; ++i) {
        // Two draws per edge, u first (the braced initialiser fixes the order).
        int32_t a = pick(rng);
        int32_t b = pick(rng);
        u[i] = a;
        v[i] = b;
    }
    return 0;
}

// graphgen.cpp:18-56 -- recursive quadrant descent; out-of-range endpoints
// are resampled.
int orc_gen_rmat_edges(int32_t nodes, int64_t edges, uint64_t seed, double a, double b, double c,
                       double d, int32_t* u, int32_t* v) {
    if (nodes <= 0) return fail("node count must be positive");
    double total = a + b + c + d;
    if (total <= 0) return fail("RMAT parameters must sum to a positive value");
    int levels = 0;
    while ((1 << levels) < nodes) ++levels;
    if (levels == 0) levels = 1;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    const double pa = a / total, pb = b / total, pc = c / total;
    int64_t k = 0;
    while (k < edges) {
        int32_t x = 0, y = 0;
        for (int l = 0; l < levels; ++l) {
            double r = unit(rng);
            int32_t half = 1 << (levels - 1 - l);
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
    return 0;
}

// ---- counter-based generators (twin of csrc/generate.cu) ----------------

int orc_gen_rmat_ctr(int32_t nodes, int64_t edges, uint64_t seed, double a, double b, double c,
                     int32_t* u, int32_t* v, int nthreads) {
    if (nodes <= 0) return fail("node count must be positive");
    int levels = 0;
    while ((1LL << levels) < nodes) ++levels;
    if (levels == 0) levels = 1;
    const double t1 = a, t2 = a + b, t3 = a + b + c;
    const uint64_t key = stream_key(seed, kStreamRmat);
    std::atomic<int> bad{0};
    parallel_for(edges, nthreads, 1 << 16, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            int32_t x = 0, y = 0;
            bool ok = false;
            for (uint64_t att = 0; att < 1024 && !ok; ++att) {
                x = 0;
                y = 0;
                for (int l = 0; l < levels; ++l) {
                    uint64_t ctr = (static_cast<uint64_t>(i) << 16) | (att << 6) | l;
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
            if (!ok) bad.store(1);
            u[i] = x;
            v[i] = y;
        }
    });
    return bad.load() ? fail("rmat_ctr: resampling exhausted") : 0;
}

int orc_gen_uniform_ctr(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u, int32_t* v,
                        int nthreads) {
    if (nodes <= 0) return fail("node count must be positive");
    const uint64_t key = stream_key(seed, kStreamUniform);
    parallel_for(edges, nthreads, 1 << 16, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            u[i] = static_cast<int32_t>(ctr_bounded(ctr_hash(key, 2 * i), nodes));
            v[i] = static_cast<int32_t>(ctr_bounded(ctr_hash(key, 2 * i + 1), nodes));
        }
    });
    return 0;
}

int64_t orc_gen_grid_ctr(int32_t side, double keep, uint64_t seed, int32_t* u, int32_t* v) {
    const uint64_t key = stream_key(seed, kStreamGrid);
    const int64_t S = side;
    const int64_t H = S * (S - 1);  // horizontal edges first, then vertical
    int64_t k = 0;
    for (int64_t id = 0; id < 2 * H; ++id) {
        if (!(ctr_unit(ctr_hash(key, id)) < keep)) continue;
        int64_t a, b;
        if (id < H) {
            int64_t r = id / (S - 1), c = id % (S - 1);
            a = r * S + c;
            b = a + 1;
        } else {
            int64_t j = id - H;
            int64_t r = j / S, c = j % S;
            a = r * S + c;
            b = a + S;
        }
        if (u) {
            u[k] = static_cast<int32_t>(a);
            v[k] = static_cast<int32_t>(b);
        }
        ++k;
    }
    return k;
}

void orc_hash_weights(const orc_csr* g, int32_t lo, int32_t hi, uint64_t seed, int32_t* w_out,
                      int nthreads) {
    const uint64_t key = stream_key(seed, kStreamWeight);
    const uint32_t span = static_cast<uint32_t>(static_cast<int64_t>(hi) - lo + 1);
    parallel_for(g->n, nthreads, 4096, [&](int, int64_t b, int64_t e) {
        for (int64_t x = b; x < e; ++x)
            for (int32_t k = g->offsets[x]; k < g->offsets[x + 1]; ++k) {
                uint64_t p = static_cast<uint64_t>(x), q = static_cast<uint64_t>(g->dests[k]);
                if (!g->directed && q < p) std::swap(p, q);
                w_out[k] = lo + static_cast<int32_t>(ctr_bounded(ctr_hash(key, (p << 32) | q), span));
            }
    });
}

// ---- algorithms -----------------------------------------------------------

// oracles.cpp:10-31 -- binary-heap Dijkstra.
int orc_sssp(const orc_csr* g, int32_t src, int64_t* dist) {
    View G{g};
    const int32_t n = g->n;
    if (src < 0 || src >= n) return fail("sssp: source out of range");
    std::fill(dist, dist + n, kInf);
    dist[src] = 0;
    using Item = std::pair<int64_t, int32_t>;
    std::priority_queue<Item, std::vector<Item>, std::greater<>> heap;
    heap.push({0, src});
    while (!heap.empty()) {
        auto [d, x] = heap.top();
        heap.pop();
        if (d != dist[x]) continue;
        for (int32_t e = g->offsets[x]; e < g->offsets[x + 1]; ++e) {
            int64_t cand = d + G.w(e);
            int32_t y = g->dests[e];
            if (cand < dist[y]) {
                dist[y] = cand;
                heap.push({cand, y});
            }
        }
    }
    return 0;
}

// One Jacobi round of pr.sp:12-31.  Returns whether any node voted
// "not settled" (|change| >= threshold && iter < maxIter).
static bool pr_round(const orc_csr* g, double damping, double threshold, int64_t iter,
                     int64_t max_iter, const std::vector<double>& rank, std::vector<double>& next,
                     int nthreads) {
    View G{g};
    const int32_t n = g->n;
    const double numNodes = static_cast<double>(n);
    // pr.sp:13-16 -- dangling mass from the current ranks, ascending order.
    double dangling = 0.0;
    for (int32_t x = 0; x < n; ++x)
        if (G.outdeg(x) == 0) dangling += rank[x];
    std::atomic<bool> unsettled{false};
    parallel_for(n, nthreads, 8192, [&](int, int64_t b, int64_t e) {
        bool local = false;
        for (int64_t x = b; x < e; ++x) {
            double total = dangling / numNodes;  // pr.sp:18
            for (int32_t s = g->rev_offsets[x]; s < g->rev_offsets[x + 1]; ++s) {
                int32_t y = g->rev_srcs[s];
                total += rank[y] / static_cast<double>(G.outdeg(y));  // pr.sp:20
            }
            double newRank = (1.0 - damping) / numNodes + damping * total;  // pr.sp:22
            double change = newRank - rank[x];
            if (change < 0.0) change = 0.0 - change;
            if (change >= threshold && iter < max_iter) local = true;  // pr.sp:25
            next[x] = newRank;
        }
        if (local) unsettled.store(true, std::memory_order_relaxed);
    });
    return unsettled.load();
}

int orc_pr(const orc_csr* g, double damping, double threshold, int32_t max_iter, double* rank_out,
           int32_t* rounds_out, int nthreads) {
    const int32_t n = g->n;
    // pr.sp:9 evaluates 1.0 / numNodes; the interpreter raises on a zero divisor
    // (interpreter.cpp:454-456).
    if (n == 0) return fail("RuntimeError: division by zero");
    std::vector<double> rank(n, 1.0 / static_cast<double>(n)), next(n, 0.0);
    // fixedPoint cap, interpreter.cpp:977-986.
    const int64_t cap = 10 * static_cast<int64_t>(n) + 100;
    int64_t iter = 0, rounds = 0;
    while (true) {
        if (++rounds > cap) return fail("NonTermination: fixedPoint exceeded cap");
        bool unsettled = pr_round(g, damping, threshold, iter, max_iter, rank, next, nthreads);
        rank.swap(next);
        iter += 1;
        if (!unsettled) break;
    }
    std::copy(rank.begin(), rank.end(), rank_out);
    if (rounds_out) *rounds_out = static_cast<int32_t>(rounds);
    return 0;
}

int orc_pr_rounds(const orc_csr* g, double damping, int32_t rounds, double* rank_out,
                  int nthreads) {
    const int32_t n = g->n;
    if (n == 0) return fail("RuntimeError: division by zero");
    std::vector<double> rank(n, 1.0 / static_cast<double>(n)), next(n, 0.0);
    for (int32_t r = 0; r < rounds; ++r) {
        pr_round(g, damping, 0.0, r, INT64_MAX, rank, next, nthreads);
        rank.swap(next);
    }
    std::copy(rank.begin(), rank.end(), rank_out);
    return 0;
}

// tc.sp:6-18 -- for each middle v: u in N(v), u < v; w in N(v), w > v;
// count is_an_edge(u, w).  |N(v)_{>v} ∩ N(u)| by a sorted merge.
int orc_tc_range(const orc_csr* g, int32_t v_begin, int32_t v_end, int64_t* count,
                 int nthreads) {
    v_begin = std::max(v_begin, 0);
    v_end = std::min(v_end, g->n);
    int T = clamp_threads(nthreads);
    std::vector<int64_t> part(T, 0);
    const int32_t* off = g->offsets;
    const int32_t* dst = g->dests;
    parallel_for(std::max<int64_t>(0, v_end - v_begin), T, 2048, [&](int t, int64_t b, int64_t e) {
        int64_t local = 0;
        for (int64_t i = b; i < e; ++i) {
            int32_t x = static_cast<int32_t>(v_begin + i);
            const int32_t* nb = dst + off[x];
            const int32_t* ne = dst + off[x + 1];
            const int32_t* hi = std::upper_bound(nb, ne, x);  // first w > v
            for (const int32_t* p = nb; p < ne && *p < x; ++p) {
                int32_t y = *p;  // u < v
                const int32_t* a = hi;
                const int32_t* b2 = std::upper_bound(dst + off[y], dst + off[y + 1], x);
                const int32_t* be = dst + off[y + 1];
                while (a < ne && b2 < be) {
                    if (*a < *b2)
                        ++a;
                    else if (*b2 < *a)
                        ++b2;
                    else {
                        ++local;
                        ++a;
                        ++b2;
                    }
                }
            }
        }
        part[t] += local;
    });
    int64_t s = 0;
    for (int64_t p : part) s += p;
    *count = s;
    return 0;
}

int orc_tc(const orc_csr* g, int64_t* count, int nthreads) {
    return orc_tc_range(g, 0, g->n, count, nthreads);
}

// The partial-count contract of gdx_tc_range (include/gdx.h): directed graphs
// keep tc.sp's middle vertex as the owner (orc_tc_range); on undirected graphs
// a triangle a < b < c is owned by its smallest vertex a, counted as
// |N+(a) ∩ N+(b)| with N+(x) = N(x) ∩ (x, inf) -- the GPU's oriented kernel.
// Over [0, n) both equal orc_tc.
int orc_tc_range_owner(const orc_csr* g, int32_t v_begin, int32_t v_end, int64_t* count,
                       int nthreads) {
    if (g->directed) return orc_tc_range(g, v_begin, v_end, count, nthreads);
    v_begin = std::max(v_begin, 0);
    v_end = std::min(v_end, g->n);
    int T = clamp_threads(nthreads);
    std::vector<int64_t> part(T, 0);
    const int32_t* off = g->offsets;
    const int32_t* dst = g->dests;
    parallel_for(std::max<int64_t>(0, v_end - v_begin), T, 2048, [&](int t, int64_t b, int64_t e) {
        int64_t local = 0;
        for (int64_t i = b; i < e; ++i) {
            const int32_t a = static_cast<int32_t>(v_begin + i);
            const int32_t* ae = dst + off[a + 1];
            for (const int32_t* p = std::upper_bound(dst + off[a], ae, a); p < ae; ++p) {
                const int32_t bv = *p;  // a < bv
                const int32_t* x = p + 1;
                const int32_t* be = dst + off[bv + 1];
                const int32_t* y = std::upper_bound(dst + off[bv], be, bv);
                while (x < ae && y < be) {
                    if (*x < *y)
                        ++x;
                    else if (*y < *x)
                        ++y;
                    else {
                        ++local;
                        ++x;
                        ++y;
                    }
                }
            }
        }
        part[t] += local;
    });
    int64_t s = 0;
    for (int64_t p : part) s += p;
    *count = s;
    return 0;
}

// oracles.cpp:33-71 -- per source: BFS with path counting in queue order, then
// dependency accumulation in reverse BFS order over children in ascending id
// order.  Sources run concurrently; their dependency vectors are added into
// the score in source order, so the sum is identical to the sequential oracle.
int orc_bc(const orc_csr* g, const int32_t* sources, int32_t nsrc, double* bc, int nthreads) {
    const int32_t n = g->n;
    for (int32_t i = 0; i < nsrc; ++i)
        if (sources[i] < 0 || sources[i] >= n) return fail("bc: source out of range");
    std::fill(bc, bc + n, 0.0);
    int T = std::min<int>(clamp_threads(nthreads), std::max<int32_t>(nsrc, 1));
    const int32_t* off = g->offsets;
    const int32_t* dst = g->dests;
    for (int32_t base = 0; base < nsrc; base += T) {
        int32_t cnt = std::min<int32_t>(T, nsrc - base);
        std::vector<std::vector<double>> deltas(cnt);
        std::vector<std::vector<int32_t>> orders(cnt);
        std::vector<std::thread> pool;
        for (int32_t k = 0; k < cnt; ++k)
            pool.emplace_back([&, k] {
                int32_t s = sources[base + k];
                std::vector<int32_t> level(n, -1);
                std::vector<XF> sigma(n);
                std::vector<double>& delta = deltas[k];
                delta.assign(n, 0.0);
                std::vector<int32_t>& order = orders[k];
                level[s] = 0;
                sigma[s] = {1.0, 0};
                std::deque<int32_t> q{s};
                while (!q.empty()) {
                    int32_t x = q.front();
                    q.pop_front();
                    order.push_back(x);
                    for (int32_t e = off[x]; e < off[x + 1]; ++e) {
                        int32_t y = dst[e];
                        if (level[y] < 0) {
                            level[y] = level[x] + 1;
                            q.push_back(y);
                        }
                        if (level[y] == level[x] + 1) sigma[y] = xf_add(sigma[y], sigma[x]);
                    }
                }
                for (auto it = order.rbegin(); it != order.rend(); ++it) {
                    int32_t y = *it;
                    for (int32_t e = off[y]; e < off[y + 1]; ++e) {
                        int32_t z = dst[e];
                        if (level[z] == level[y] + 1 && sigma[z].m > 0.0)
                            delta[y] += xf_ratio(sigma[y], sigma[z]) * (1.0 + delta[z]);
                    }
                }
            });
        for (auto& th : pool) th.join();
        for (int32_t k = 0; k < cnt; ++k) {
            int32_t s = sources[base + k];
            for (int32_t y : orders[k])
                if (y != s) bc[y] += deltas[k][y];
        }
    }
    return 0;
}

// oracles.cpp:113-129
int orc_bfs_levels(const orc_csr* g, int32_t root, int32_t* level) {
    const int32_t n = g->n;
    if (root < 0 || root >= n) return fail("bfs: root out of range");
    std::fill(level, level + n, -1);
    level[root] = 0;
    std::deque<int32_t> q{root};
    while (!q.empty()) {
        int32_t x = q.front();
        q.pop_front();
        for (int32_t e = g->offsets[x]; e < g->offsets[x + 1]; ++e)
            if (level[g->dests[e]] < 0) {
                level[g->dests[e]] = level[x] + 1;
                q.push_back(g->dests[e]);
            }
    }
    return 0;
}

}  // extern "C"
