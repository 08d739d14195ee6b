// plans.cuh -- per-graph cached plans / workspaces of the four algorithms.
// They live on the gdx_graph handle so repeated calls reuse device memory
// (no cudaMalloc inside a steady-state call).
#pragma once

#include <functional>

#include "gdx_internal.cuh"

namespace gdx {

int guard_impl(const std::function<void()>& f);
gdx_graph* make_graph(int device);

// PageRank merge-path plan (pagerank.cu).
struct PrPlan {
    DevBuf<double> rank[2], contrib[2];
    DevBuf<double> dangling;              // 3 rotating accumulators
    DevBuf<int32_t> flags;                // per-round "unsettled" votes (ring, pagerank.cu)
    // edge-aligned two-pass plan
    int32_t nnz = 0;
    DevBuf<int2> nz;                      // non-empty rows of the reverse CSR: (vertex, end)
    DevBuf<int2> grp;                     // per 8-edge group: (nz index of its first row, its end)
    DevBuf<double> row_sum;               // per-vertex gather sums (zero between rounds)
    DevBuf<double> head_part, tail_part;  // per 256-edge chunk: partials of rows crossing chunks
    DevBuf<int4> cross, cross_long;       // crossing rows (row, first chunk, last chunk): short, hub
    int32_t ncross = 0, nlong = 0;
    DevBuf<double> dang_part;             // per-block dangling partials (ordered grid sum)
    DevBuf<unsigned int> dang_ctr;
    int32_t v_begin = 0, v_end = 0;       // row range of the plan
    int64_t e_begin = 0, e_end = 0, e_base = 0, ngroups = 0;
    bool shard = false;                   // built by gdx_pr_shard_setup
    DevBuf<double> partials;              // shard: [dangling partial, unsettled]
    int grid = 0;
    int block = 256;
};

// Degree-ordered renumbering of a graph (relabel.cu): the renumbered graph as
// a hidden handle on the owner's stream, and the permutation both ways.
struct Relabel {
    gdx_graph* h = nullptr;    // owned
    DevBuf<int32_t> newid;     // old id -> new id
    DevBuf<int32_t> order;     // new id -> old id
    bool fwd_off = false, fwd_adj = false, rev = false;  // arrays of h built so far
    DevBuf<double> staging;    // a call's output in the old numbering (host outputs)
    Relabel() = default;
    Relabel(const Relabel&) = delete;
    Relabel& operator=(const Relabel&) = delete;
    ~Relabel();
};

// Peer-memory exchange state of the sharded PageRank (pagerank.cu gdx_pr_p2p_*).
struct PrP2P {
    int32_t world = 0, rank = 0;
    int64_t n = 0;
    double* block = nullptr;            // own IPC-exported block (cudaMalloc)
    std::vector<double*> bases;         // every rank's block (own + opened peers)
    DevBuf<double*> peer_contrib;       // [2][world]: contrib buffer of each parity
    DevBuf<double*> peer_slot;          // [2][world]: this rank's partial slot in every block
    DevBuf<unsigned long long*> peer_ctr;  // [world]
    DevBuf<int> err;                    // set by a timed-out wait
    int64_t publishes = 0;              // publishes so far (identical on every rank)
    bool ipc = true;                    // peers opened through CUDA IPC (else in-process pointers)
    double* own_contrib(int par) const { return block + par * n; }
    double* own_partials(int par) const { return block + 2 * n + par * world * 2; }
    unsigned long long* own_ctr() const {
        return reinterpret_cast<unsigned long long*>(block + 2 * n + 4 * world);
    }
    size_t bytes() const { return (2 * size_t(n) + 4 * size_t(world) + 1) * sizeof(double); }
    ~PrP2P() {
        if (ipc)
            for (int q = 0; q < int(bases.size()); ++q)
                if (q != rank && bases[q]) cudaIpcCloseMemHandle(bases[q]);
        if (block) cudaFree(block);
    }
};

// SSSP frontier workspace (sssp.cu).
struct SsspWork {
    DevBuf<uint64_t> dist;   // 32- or 64-bit distances (reinterpreted)
    DevBuf<uint64_t> prev;   // frontier-scan mode: distance at the last expansion
    DevBuf<int32_t> stamp;   // round at which a vertex was last enqueued
    DevBuf<int2> queue[2];   // work items (vertex, first edge)
    DevBuf<unsigned long long> ctrs;  // rotating counters + stats
    DevBuf<unsigned long long> trace; // optional per-round trace (GDX_SSSP_TRACE)
    size_t qcap = 0;
    int grid = 0;
    // gdx_sssp_shard_*: this rank's vertex range and relaxation items
    bool shard_ready = false;
    int32_t shard_v0 = 0, shard_v1 = 0;
    int64_t shard_edges = 0;
    DevBuf<int2> shard_queue;
    DevBuf<int2> small_queue;  // single-GPU rounds: vertices of <= 8 out-edges (one item each)
    DevBuf<unsigned long long> shard_ctr;  // [items, improved sinks, overflow, vertices, edges, changed]
    DevBuf<int32_t> shard_mark;  // delta mode: round in which a vertex was last listed as changed
    int32_t shard_round = 0;
    // device-side round loop (CUDA graph with a conditional WHILE node), per distance width
    static constexpr int kKey = 10;
    cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};  // u32, u64, u16 distances
    void* gkey[3][kKey] = {};
    bool narrow_overflowed = false;  // a 16-bit attempt on this handle overflowed
    const int32_t* out_perm = nullptr;  // renumbered graph (relabel.cu): out[v] = dist[out_perm[v]]
    DevBuf<unsigned long long> graph_acc;  // [rounds, vertices, edges, overflow]
    DevBuf<unsigned long long> upd_slots;  // U counter slots (sssp.cu block_count)
    // in-process multi-GPU rounds (gdx_sssp_multi): barrier state and the
    // instantiated round loop per distance width
    DevBuf<unsigned long long> msync;
    DevBuf<void*> mpeers;
    cudaGraphExec_t mexec[3] = {nullptr, nullptr, nullptr};  // u32, u64, u16 distances
    std::vector<void*> mkey[3];
    bool multi_narrow_overflowed = false;  // a 16-bit multi-GPU attempt overflowed
    ~SsspWork() {
        for (auto& e : gexec)
            if (e) cudaGraphExecDestroy(e);
        for (auto& e : mexec)
            if (e) cudaGraphExecDestroy(e);
    }
};

// Multi-process SSSP partitions over peer memory (sssp.cu gdx_sssp_p2p_*):
// this rank's exported block {distance replica (8 B per vertex) | barrier
// state (64 B)} and every rank's block opened through CUDA IPC.
struct SsspP2P {
    int32_t world = 0, rank = 0;
    std::vector<int32_t> bounds;        // world + 1 vertex-range bounds
    int64_t n = 0;
    char* block = nullptr;              // own block (plain cudaMalloc: IPC export)
    std::vector<char*> bases;           // every rank's block (own + opened peers)
    DevBuf<void*> peer_sync;            // [world] every rank's barrier state
    size_t bytes() const { return size_t(n) * 8 + 64; }
    ~SsspP2P() {
        for (int q = 0; q < int(bases.size()); ++q)
            if (q != rank && bases[q]) cudaIpcCloseMemHandle(bases[q]);
        if (block) cudaFree(block);
    }
};

// Triangle-counting workspace (tc.cu).
struct TcPlan {
    DevBuf<unsigned long long> acc;
    DevBuf<int32_t> hi_start;  // first index of N(v) with dest > v
    DevBuf<int32_t> heavy, heavy_cnt;  // degree binning: vertices with |N+(v)| > kTcHeavy
    DevBuf<long long> heavy_pre;       // their pair prefix
    DevBuf<int32_t> off_plus;  // oriented CSR (undirected graphs): N+(v) = N(v) ∩ (v, inf)
    DevBuf<int32_t> adj_plus;
    DevBuf<unsigned long long> sigp;  // per adj+ entry: signature of that vertex's N+ (pair filter)
    DevBuf<uint8_t> scan_tmp;
    bool oriented = false;     // off+/adj+ built (once per handle: the graph is immutable)
    double survey_pairs = 0;   // sum over oriented edges of d+(u) + d+(v)
};

// BC batched Brandes workspace (bc.cu).
struct BcWork {
    int32_t batch = 0;
    DevBuf<int32_t> level;      // [batch][n]
    DevBuf<double> sig;         // [batch][n] x (mantissa, exponent)
    DevBuf<double> delta;       // [batch][n]
    DevBuf<uint64_t> log;       // (source slot << 32 | vertex), all levels
    DevBuf<long long> lvl_start;
    DevBuf<int32_t> sources;
    DevBuf<double> bc;
    DevBuf<unsigned long long> ctrs;
    size_t log_cap = 0;
    int grid = 0;
    int block = 0;
    // CTA-per-source mode (k_bc_cta): one state slot per CTA
    int32_t cta_grid = 0;
    DevBuf<double> cta_rec;     // [cta_grid][n] x 16 B (level tag, exponent, mantissa)
    DevBuf<int32_t> cta_base;   // [cta_grid] level tag base of each slot's next source
    DevBuf<double> cta_bcs;     // [cta_grid][n] per-slot partial scores (summed in slot order)
    bool cta_dirty = false;     // partials written but not yet summed (and cleared)
    DevBuf<int32_t> cta_log;    // [cta_grid][n] int4
    DevBuf<int32_t> cta_loff;   // [cta_grid][n+2]
};

}  // namespace gdx
