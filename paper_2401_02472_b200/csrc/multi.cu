// multi.cu -- several GPUs driven from one process.
//
// A gdx_context owns a device list, the peer access between every pair of
// them and (for distinct devices) one NCCL communicator per device.  A
// gdx_multi_graph is a replica of one CsrGraph on every device of a context;
// the *_multi entry points partition the work as SURVEY.md 8(e) says:
//
//   SSSP  vertex ranges balanced by out-edges; the relaxation sends improving
//         candidates to the owner's distance replica with peer atomicMin and
//         the round loop runs on the devices with device-side barriers
//         (sssp.cu sssp_multi) -- no dist all-gather at all
//   PR    destination-vertex ranges balanced by in-edges; pass B stores every
//         new contrib value straight into every device's contrib buffer and
//         the (dangling, unsettled) partials are published through peer
//         memory (pagerank.cu, the gdx_pr_p2p_* protocol with in-process
//         peers) -- no all-gather / all-reduce per round
//   TC    owner-vertex ranges balanced by ~deg^2 over the replicated graph;
//         the per-device counts are summed in device order
//   BC    contiguous source blocks over the replicated graph; one ncclAllReduce
//         (sum) of the n-vector of scores, or a peer-memory sum in device order
//         when the context has no NCCL communicators (a device listed twice)
//
// This is what a C++ caller of interp::run (interpreter.hpp:64-88) needs for
// an ExecMode::Device with a device list.  NCCL is resolved
// at run time (dlopen "libnccl.so.2": torch's bundled copy when torch is
// loaded, else the system one), so libgdx has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "gdx_internal.cuh"
#include "plans.cuh"

namespace gdx {

void sssp_multi(const std::vector<gdx_graph*>& gs, const std::vector<int32_t>& bound, int32_t src,
                int64_t* dist_out, gdx_stats* stats);
void pr_p2p_local_setup(gdx_graph* g, int32_t world, int32_t rank);
double* pr_p2p_block(gdx_graph* g);
void pr_p2p_local_open(gdx_graph* g, const std::vector<double*>& blocks);
void relabel_unpermute_i64(gdx_graph* g, const int64_t* in, int64_t* out);

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl* N = [] {
        auto* n = new Nccl;
        // GDX_NCCL_LIB names the library to use (the Python layer points it at
        // torch's bundled NCCL: loading another libnccl.so.2 first would shadow
        // the one torch links against)
        const char* env = std::getenv("GDX_NCCL_LIB");
        void* h = env && *env ? dlopen(env, RTLD_NOW | RTLD_GLOBAL) : nullptr;
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n->why = "libnccl.so.2 not found";
            return n;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
        n->comm_init_all = reinterpret_cast<decltype(n->comm_init_all)>(sym("ncclCommInitAll"));
        n->comm_destroy = reinterpret_cast<decltype(n->comm_destroy)>(sym("ncclCommDestroy"));
        n->all_reduce = reinterpret_cast<decltype(n->all_reduce)>(sym("ncclAllReduce"));
        n->group_start = reinterpret_cast<decltype(n->group_start)>(sym("ncclGroupStart"));
        n->group_end = reinterpret_cast<decltype(n->group_end)>(sym("ncclGroupEnd"));
        n->error_string = reinterpret_cast<decltype(n->error_string)>(sym("ncclGetErrorString"));
        n->ok = n->comm_init_all && n->comm_destroy && n->all_reduce && n->group_start &&
                n->group_end && n->error_string;
        if (!n->ok) n->why = "libnccl.so.2 lacks an entry point";
        return n;
    }();
    return *N;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(GDX_ERR_NCCL, std::string("NcclError: ") + what + " -> " + nccl().error_string(r));
}

// Runs fn(d) for every device on its own host thread (the devices' work
// waits on each other through peer memory, so no single thread may block on
// one device before the others have enqueued theirs); rethrows the first
// failure in the calling thread.
void on_devices(int nd, const std::function<void(int)>& fn) {
    if (nd == 1) {
        fn(0);
        return;
    }
    std::mutex mu;
    gdx_status code = GDX_OK;
    std::string msg;
    std::vector<std::thread> ts;
    for (int d = 0; d < nd; ++d)
        ts.emplace_back([&, d] {
            try {
                fn(d);
            } catch (const Error& e) {
                std::lock_guard<std::mutex> lk(mu);
                if (code == GDX_OK) code = e.code, msg = e.what();
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> lk(mu);
                if (code == GDX_OK) code = GDX_ERR_RUNTIME, msg = std::string("RuntimeError: ") + e.what();
            }
        });
    for (auto& t : ts) t.join();
    if (code != GDX_OK) fail(code, msg);
}

// A C-ABI call made from inside the library: failures become exceptions.
void call(int rc) {
    if (rc != GDX_OK) fail(gdx_status(rc), gdx_last_error());
}

// balanced_ranges of distributed.py: contiguous ranges of ~equal total weight.
std::vector<int32_t> balanced_bounds(const std::vector<double>& w, int parts) {
    const int32_t n = int32_t(w.size());
    std::vector<double> csum(size_t(n) + 1, 0.0);
    for (int32_t i = 0; i < n; ++i) csum[i + 1] = csum[i] + w[i];
    std::vector<int32_t> b(parts + 1, 0);
    for (int p = 1; p < parts; ++p) {
        const double t = csum[n] * p / parts;
        b[p] = int32_t(std::lower_bound(csum.begin(), csum.end(), t) - csum.begin());
        b[p] = std::min(std::max(b[p], b[p - 1]), n);
    }
    b[parts] = n;
    return b;
}

__global__ void k_sum_peers(double* out, const double* const* peers, int np, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = out[i];
        for (int q = 0; q < np; ++q) s += peers[q][i];  // device order
        out[i] = s;
    }
}

}  // namespace
}  // namespace gdx

struct gdx_context {
    std::vector<int> devices;
    bool distinct = true;
    bool peer_all = true;
    std::vector<ncclComm_t> comms;  // empty: no NCCL (device listed twice, or no libnccl)
    std::string nccl_why;
    ~gdx_context() {
        for (auto c : comms)
            if (c) gdx::nccl().comm_destroy(c);
    }
};

struct gdx_multi_graph {
    gdx_context* ctx = nullptr;
    std::vector<gdx_graph*> gs;  // one replica per device of the context
    int32_t n = 0, m = 0;
    bool directed = true;
    std::vector<int32_t> offsets, in_offsets;  // host copies, for the partitions
    std::vector<int32_t> pr_bound;             // ranges of the prepared PR exchange
    std::vector<gdx::DevBuf<double>> bc_buf;   // per-device BC accumulators
    // the replicas' degree-ordered renumbering (relabel.cu), once they have one:
    // its host offsets per side for the partitions, and the PR exchange over it
    gdx_graph* ren_h0 = nullptr;               // device 0's renumbered handle they belong to
    std::vector<int32_t> ren_offsets, ren_in_offsets, ren_pr_bound;
    ~gdx_multi_graph() {
        for (size_t d = 0; d < bc_buf.size() && d < gs.size(); ++d) {  // on its own device
            gdx::GraphScope sc(gs[d]);
            bc_buf[d].release();
        }
        for (auto* g : gs)
            if (g) gdx_graph_destroy(g);
    }
};

using namespace gdx;

namespace {

std::vector<double> degree_weights(const std::vector<int32_t>& off, bool squared) {
    const size_t n = off.empty() ? 0 : off.size() - 1;
    std::vector<double> w(n);
    for (size_t v = 0; v < n; ++v) {
        const double d = double(off[v + 1]) - double(off[v]);
        w[v] = squared ? d * d / 2.0 + d + 1.0 : d + 1.0;
    }
    return w;
}

// The replicas' renumbered handles for this call (algo 0 PR, 1 SSSP), or an
// empty vector: every replica takes gdx_pagerank / gdx_sssp's decision
// (relabel_wanted counts the calls per handle, so they agree), and the host
// offsets of the renumbered graph are cached for the partitions.
std::vector<gdx_graph*> multi_renumbered(gdx_multi_graph* mg, int algo) {
    std::vector<gdx_graph*> hs;
    const int nd = int(mg->gs.size());
    for (int d = 0; d < nd; ++d) {
        gdx_graph* g = mg->gs[d];
        GraphScope sc(g);
        const bool want = algo == 0 ? relabel_wanted(g)
                                    : graph_max_degree(g) > 64 && relabel_wanted(g);
        if (!want) {
            if (d > 0) fail(GDX_ERR_RUNTIME, "RuntimeError: replicas disagree on the renumbering");
            return {};
        }
        Relabel* R = relabel_try(g, algo == 1, algo == 0);
        if (!R) {  // out of memory on one replica: every replica keeps its numbering
            for (auto* r : mg->gs) {
                GraphScope s2(r);
                r->relabel.reset();
                r->relabel_failed = true;
            }
            mg->ren_h0 = nullptr;
            return {};
        }
        hs.push_back(R->h);
    }
    if (mg->ren_h0 != hs[0]) {  // a new renumbering (first use, or the weights changed)
        mg->ren_h0 = hs[0];
        mg->ren_offsets.clear();
        mg->ren_in_offsets.clear();
        mg->ren_pr_bound.clear();
    }
    gdx_graph* h = hs[0];
    GraphScope sc(mg->gs[0]);
    if (mg->ren_offsets.empty()) {
        mg->ren_offsets.resize(size_t(mg->n) + 1);
        GDX_CUDA(cudaMemcpyAsync(mg->ren_offsets.data(), h->offsets.get(), mg->ren_offsets.size() * 4,
                                 cudaMemcpyDeviceToHost, h->stream));
    }
    if (algo == 0 && mg->ren_in_offsets.empty()) {
        mg->ren_in_offsets.resize(size_t(mg->n) + 1);
        GDX_CUDA(cudaMemcpyAsync(mg->ren_in_offsets.data(), h->in_offsets(),
                                 mg->ren_in_offsets.size() * 4, cudaMemcpyDeviceToHost, h->stream));
    }
    GDX_CUDA(cudaStreamSynchronize(h->stream));
    return hs;
}

// out[v] = in[newid[v]] on device 0, into dst (host or device).
void multi_unpermute(gdx_multi_graph* mg, const int64_t* in, int64_t* dst) {
    gdx_graph* g = mg->gs[0];
    GraphScope sc(g);
    DevBuf<int64_t> tmp(size_t(std::max(mg->n, 1)));
    relabel_unpermute_i64(g, in, tmp.get());
    copy_out(g, dst, tmp.get(), size_t(mg->n) * sizeof(int64_t));
    GDX_CUDA(cudaStreamSynchronize(g->stream));
}

void merge_stats(gdx_stats* into, const gdx_stats& s) {
    into->rounds = std::max(into->rounds, s.rounds);
    into->launches += s.launches;
    into->vertices_visited += s.vertices_visited;
    into->edges_visited += s.edges_visited;
    into->updates += s.updates;
    into->algorithmic_bytes += s.algorithmic_bytes;
}

}  // namespace

extern "C" {

int gdx_context_create(int ndev, const int* devices, gdx_context** out) {
    return guard_impl([&] {
        if (ndev < 1 || !devices || !out)
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: need a device list");
        int have = 0;
        GDX_CUDA(cudaGetDeviceCount(&have));
        auto ctx = std::make_unique<gdx_context>();
        ctx->devices.assign(devices, devices + ndev);
        for (int d : ctx->devices)
            if (d < 0 || d >= have)
                fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: device " + std::to_string(d) +
                                                   " out of range [0, " + std::to_string(have) + ")");
        std::vector<int> sorted = ctx->devices;
        std::sort(sorted.begin(), sorted.end());
        ctx->distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
        // peer access between every pair of distinct devices (NVLink / NVSwitch)
        for (int a : ctx->devices)
            for (int b : ctx->devices) {
                if (a == b) continue;
                int can = 0;
                GDX_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
                if (!can) {
                    ctx->peer_all = false;
                    continue;
                }
                DeviceGuard dg(a);
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else
                    GDX_CUDA(e);
            }
        if (!ctx->peer_all)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: the devices of a context need peer access");
        if (!ctx->distinct) {
            ctx->nccl_why = "a device is listed twice (NCCL needs one rank per GPU)";
        } else if (!nccl().ok) {
            ctx->nccl_why = nccl().why;
        } else {
            ctx->comms.assign(ndev, nullptr);
            nccl_check(nccl().comm_init_all(ctx->comms.data(), ndev, ctx->devices.data()),
                       "ncclCommInitAll");
        }
        *out = ctx.release();
    });
}

int gdx_context_destroy(gdx_context* ctx) {
    return guard_impl([&] { delete ctx; });
}

int gdx_context_info(const gdx_context* ctx, int32_t* ndev, int32_t* nccl_comms,
                     int32_t* peer_access) {
    return guard_impl([&] {
        if (!ctx) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null context");
        if (ndev) *ndev = int32_t(ctx->devices.size());
        if (nccl_comms) *nccl_comms = int32_t(ctx->comms.size());
        if (peer_access) *peer_access = ctx->peer_all ? 1 : 0;
    });
}

int gdx_multi_graph_create(gdx_context* ctx, const gdx_csr_view* view, gdx_multi_graph** out) {
    return guard_impl([&] {
        if (!ctx || !view || !out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        auto mg = std::make_unique<gdx_multi_graph>();
        mg->ctx = ctx;
        for (int d : ctx->devices) {
            gdx_graph* g = nullptr;
            call(gdx_graph_create(view, d, &g));
            mg->gs.push_back(g);
        }
        gdx_graph* g0 = mg->gs[0];
        mg->n = g0->n;
        mg->m = g0->m;
        mg->directed = g0->directed;
        mg->offsets.resize(size_t(mg->n) + 1);
        mg->in_offsets.resize(size_t(mg->n) + 1);
        call(gdx_graph_download(g0, mg->offsets.data(), nullptr, nullptr,
                                g0->in_offsets() ? mg->in_offsets.data() : nullptr, nullptr,
                                nullptr));
        if (!g0->in_offsets()) mg->in_offsets.clear();
        *out = mg.release();
    });
}

int gdx_multi_graph_destroy(gdx_multi_graph* g) {
    return guard_impl([&] { delete g; });
}

int gdx_sssp_multi(gdx_multi_graph* mg, int32_t src, int64_t* dist_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!mg || !dist_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (src < 0 || src >= mg->n)
            fail(GDX_ERR_OUT_OF_RANGE, "RuntimeError: node id " + std::to_string(src) +
                                           " out of range [0, " + std::to_string(mg->n) + ")");
        const int nd = int(mg->gs.size());
        gdx_stats st{};
        const auto hs = multi_renumbered(mg, 1);
        if (!hs.empty()) {
            // the partitions of the renumbered graph gdx_sssp runs on, the
            // distances mapped back (device 0 gathers them)
            gdx_graph* g0 = mg->gs[0];
            const int32_t s = relabel_vertex(g0, src);
            DevBuf<int64_t> tmp;
            {
                GraphScope sc(g0);
                tmp.alloc(size_t(std::max(mg->n, 1)));
            }
            sssp_multi(hs, balanced_bounds(degree_weights(mg->ren_offsets, false), nd), s,
                       tmp.get(), &st);
            multi_unpermute(mg, tmp.get(), dist_out);
            GraphScope sc(g0);
            tmp.release();
        } else {
            sssp_multi(mg->gs, balanced_bounds(degree_weights(mg->offsets, false), nd), src,
                       dist_out, &st);
        }
        if (stats) *stats = st;
    });
}

int gdx_pagerank_multi(gdx_multi_graph* mg, double damping, double threshold, int32_t max_iter,
                       double* rank_out, int32_t* rounds_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!mg || !rank_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (mg->n == 0) fail(GDX_ERR_RUNTIME, "RuntimeError: division by zero");  // pr.sp:9
        if (mg->in_offsets.empty())
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no reverse adjacency");
        const int nd = int(mg->gs.size());
        // the replicas, or their renumbering (the graph gdx_pagerank runs on)
        const auto hs = multi_renumbered(mg, 0);
        const bool ren = !hs.empty();
        const std::vector<gdx_graph*>& gs = ren ? hs : mg->gs;
        std::vector<int32_t>& bound = ren ? mg->ren_pr_bound : mg->pr_bound;
        if (bound.empty()) {  // shard plans and the peer-memory exchange, once
            const auto b = balanced_bounds(
                degree_weights(ren ? mg->ren_in_offsets : mg->in_offsets, false), nd);
            std::vector<double*> blocks(nd);
            for (int d = 0; d < nd; ++d) {
                call(gdx_pr_shard_setup(gs[d], b[d], b[d + 1]));
                pr_p2p_local_setup(gs[d], nd, d);
                blocks[d] = pr_p2p_block(gs[d]);
            }
            for (int d = 0; d < nd; ++d) pr_p2p_local_open(gs[d], blocks);
            bound = b;
        }
        const auto& b = bound;
        DevBuf<int64_t> tmp;  // renumbered: the ranks in the new ids, on device 0
        if (ren) {
            GraphScope sc(mg->gs[0]);
            tmp.alloc(size_t(mg->n));
        }
        double* out = ren ? reinterpret_cast<double*>(tmp.get()) : rank_out;
        // fixedPoint rounds: at most max_iter+1 (pr.sp:25) and the
        // interpreter's cap 10n+100 (interpreter.cpp:977-986)
        const int64_t cap = 10 * int64_t(mg->n) + 100;
        const int64_t want = max_iter >= 0 ? int64_t(max_iter) + 1 : 1;
        const int64_t limit = std::min(want, cap);
        std::vector<int64_t> rounds(nd, -1);
        std::vector<char> settled_seen(nd, 0);
        on_devices(nd, [&](int d) {
            gdx_graph* g = gs[d];
            double part[2];
            call(gdx_pr_p2p_init(g, part));
            const double dangling = part[0];
            int64_t r = 0, batch = 4, done = limit;
            while (r < limit) {  // the same batches on every device
                const int32_t cnt = int32_t(std::min<int64_t>(batch, limit - r));
                int32_t settled = -1;
                call(gdx_pr_p2p_rounds(g, int32_t(r), cnt, damping, threshold, max_iter, dangling,
                                       &settled));
                if (settled >= 0) {
                    done = settled + 1;
                    settled_seen[d] = 1;
                    break;
                }
                r += cnt;
                batch = std::min<int64_t>(2 * batch, 64);
            }
            rounds[d] = done;
            call(gdx_pr_shard_rank(g, int32_t(done), out + b[d]));
        });
        if (ren) {  // the f64 bit patterns move like int64
            multi_unpermute(mg, tmp.get(), reinterpret_cast<int64_t*>(rank_out));
            GraphScope sc(mg->gs[0]);
            tmp.release();
        }
        const int64_t done = rounds[0];
        if (!settled_seen[0] && limit < want) {
            // every round voted "unsettled" up to the cap
            fail(GDX_ERR_NON_TERMINATION, "NonTermination: fixedPoint exceeded " +
                                              std::to_string(cap) + " iterations without converging");
        }
        if (rounds_out) *rounds_out = int32_t(done);
        if (stats) {
            *stats = gdx_stats{};
            stats->rounds = int32_t(done);
            stats->vertices_visited = int64_t(mg->n) * done;
            stats->edges_visited = int64_t(mg->m) * done;
            stats->algorithmic_bytes = double(done) * (12.0 * mg->m + 24.0 * mg->n);
        }
    });
}

int gdx_tc_multi(gdx_multi_graph* mg, int64_t* count_out, gdx_stats* stats) {
    return guard_impl([&] {
        if (!mg || !count_out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        const int nd = int(mg->gs.size());
        const auto b = balanced_bounds(degree_weights(mg->offsets, true), nd);
        std::vector<int64_t> cnt(nd, 0);
        std::vector<gdx_stats> st(nd);
        on_devices(nd, [&](int d) {
            call(gdx_tc_range(mg->gs[d], b[d], b[d + 1], &cnt[d], &st[d]));
        });
        int64_t total = 0;
        gdx_stats all{};
        for (int d = 0; d < nd; ++d) {
            total += cnt[d];
            merge_stats(&all, st[d]);
        }
        *count_out = total;
        if (stats) *stats = all;
    });
}

int gdx_bc_multi(gdx_multi_graph* mg, const int32_t* sources, int32_t nsrc, double* bc_out,
                 gdx_stats* stats) {
    return guard_impl([&] {
        if (!mg || !bc_out || nsrc < 0 || (nsrc > 0 && !sources))
            fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        const int nd = int(mg->gs.size());
        const int64_t n = mg->n;
        mg->bc_buf.resize(nd);
        for (int d = 0; d < nd; ++d) {
            GraphScope sc(mg->gs[d]);
            mg->bc_buf[d].ensure(size_t(std::max<int64_t>(n, 1)));
        }
        // contiguous source blocks (order kept), sizes differ by <= 1
        std::vector<int32_t> sb(nd + 1, 0);
        for (int d = 0; d < nd; ++d) sb[d + 1] = sb[d] + nsrc / nd + (d < nsrc % nd ? 1 : 0);
        std::vector<gdx_stats> st(nd);
        on_devices(nd, [&](int d) {
            call(gdx_bc(mg->gs[d], sources + sb[d], sb[d + 1] - sb[d], mg->bc_buf[d].get(), &st[d]));
        });
        gdx_context* ctx = mg->ctx;
        if (nd > 1 && !ctx->comms.empty()) {
            nccl_check(nccl().group_start(), "ncclGroupStart");
            for (int d = 0; d < nd; ++d) {
                DeviceGuard dg(mg->gs[d]->device);
                nccl_check(nccl().all_reduce(mg->bc_buf[d].get(), mg->bc_buf[d].get(), size_t(n),
                                             ncclDouble, ncclSum, ctx->comms[d], mg->gs[d]->stream),
                           "ncclAllReduce");
            }
            nccl_check(nccl().group_end(), "ncclGroupEnd");
            for (int d = 0; d < nd; ++d) {
                DeviceGuard dg(mg->gs[d]->device);
                GDX_CUDA(cudaStreamSynchronize(mg->gs[d]->stream));
            }
        } else if (nd > 1) {  // peer-memory sum into device 0, device order
            gdx_graph* g0 = mg->gs[0];
            GraphScope sc(g0);
            std::vector<const double*> peers;
            for (int d = 1; d < nd; ++d) peers.push_back(mg->bc_buf[d].get());
            DevBuf<const double*> tab(peers.size());
            GDX_CUDA(cudaMemcpyAsync(tab.get(), peers.data(), peers.size() * sizeof(void*),
                                     cudaMemcpyHostToDevice, g0->stream));
            timed_launch(g0, "bc_multi_sum", [&] {
                k_sum_peers<<<blocks_for(n, 256, g0->num_sms * 8), 256, 0, g0->stream>>>(
                    mg->bc_buf[0].get(), tab.get(), int(peers.size()), n);
            });
            GDX_CUDA(cudaStreamSynchronize(g0->stream));
        }
        gdx_graph* g0 = mg->gs[0];
        GraphScope sc(g0);
        copy_out(g0, bc_out, mg->bc_buf[0].get(), size_t(n) * sizeof(double));
        GDX_CUDA(cudaStreamSynchronize(g0->stream));
        if (stats) {
            gdx_stats all{};
            for (int d = 0; d < nd; ++d) merge_stats(&all, st[d]);
            *stats = all;
        }
    });
}

}  // extern "C"
