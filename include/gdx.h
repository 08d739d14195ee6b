/*
 * gdx.h -- C ABI of the B200 graph-analytics backend (libgdx.so).
 *
 * Drop-in for the execution of the four corpus entry points of the reference
 * (arxiv/paper_2401_02472, /root/reference/proj):
 *
 *   reference interface                                   replaced by
 *   ----------------------------------------------------  -----------------------------
 *   CsrGraph spans (core/include/graphdsl/csr.hpp:39-44)  gdx_graph_create (gdx_csr_view)
 *   CsrGraph::buildFromEdges (core/src/csr.cpp:28-94)     gdx_graph_build_from_edges
 *   ComputeSSSP via interp::run (corpus/sssp.sp:6-20,     gdx_sssp
 *     interpreter.hpp:87-88); golden computesssp
 *     (tests/golden/sssp/cuda/sssp_cuda.cu:136)
 *   ComputePR  (corpus/pr.sp:5-33); computepr             gdx_pagerank
 *     (tests/golden/pr/cuda/pr_cuda.cu:150)
 *   ComputeTC  (corpus/tc.sp:6-18); computetc             gdx_tc
 *     (tests/golden/tc/cuda/tc_cuda.cu:144)
 *   ComputeBC  (corpus/bc.sp:6-25); computebc             gdx_bc
 *     (tests/golden/bc/cuda/bc_cuda.cu:149)
 *   CompileError kinds (diagnostics.hpp:31-57)            gdx_status + gdx_last_error()
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross this boundary.  Every
 *    function returns a gdx_status; on failure gdx_last_error() (thread-local)
 *    holds "<Kind>: <message>" where Kind mirrors the reference's CompileError
 *    kinds (RuntimeError, NonTermination, InvalidEdge, ...).
 *  - Output pointers may be host memory (pageable or pinned) or device memory
 *    on the graph's device (unified addressing decides; cudaMemcpyDefault).
 *  - A graph handle owns its device memory and one CUDA stream; it must be used
 *    by one host thread at a time.  Distinct handles may run concurrently.
 *  - Results are bit-exact with the reference for SSSP distances and triangle
 *    counts and within 1e-6 relative for PageRank and BC.
 */
#ifndef GDX_H
#define GDX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDX_ABI_VERSION 1

typedef enum {
    GDX_OK = 0,
    GDX_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument / InvalidEdge / NegativeWeight */
    GDX_ERR_OUT_OF_RANGE = 2,     /* node id out of range (RuntimeError in interp::run) */
    GDX_ERR_RUNTIME = 3,          /* other RuntimeError (e.g. division by zero) */
    GDX_ERR_NON_TERMINATION = 4,  /* fixedPoint cap exceeded (interpreter.cpp:977-986) */
    GDX_ERR_CUDA = 5,
    GDX_ERR_OUT_OF_MEMORY = 6,
    GDX_ERR_UNSUPPORTED = 7,
    GDX_ERR_NCCL = 8
} gdx_status;

typedef struct gdx_graph gdx_graph;

/* Exactly the reference's GraphCsr (sssp_cuda.cu:8-17) plus `directed`.
 * weights may be NULL (all 1).  rev_* may be NULL: the reverse CSR is then
 * rebuilt on the device with csr.cpp:77-94 semantics (a sort for directed
 * graphs; undirected graphs are stored symmetrically by CsrGraph, csr.cpp:42-45,
 * so their reverse arrays equal the forward ones: the handle reads the forward
 * arrays and builds the mirror edge ids only when gdx_graph_download asks for
 * rev_eid).  dests may be NULL only when rev_offsets/rev_srcs are given
 * (PageRank-only graphs). */
typedef struct {
    int32_t n;
    int32_t m;
    int32_t directed;
    const int32_t* offsets;     /* n+1 */
    const int32_t* dests;       /* m   */
    const int32_t* weights;     /* m   */
    const int32_t* rev_offsets; /* n+1 */
    const int32_t* rev_srcs;    /* m   */
    const int32_t* rev_eid;     /* m   */
} gdx_csr_view;

/* Per-call statistics (algorithmic work, used for GTEPS / roofline). */
typedef struct {
    int32_t rounds;           /* fixedPoint rounds / BFS levels / tiles */
    int32_t launches;         /* kernels launched by the call */
    int64_t vertices_visited; /* SSSP: sum of frontier sizes; BC: reached (s,v) pairs */
    int64_t edges_visited;    /* edges scanned */
    int64_t updates;          /* SSSP successful relaxations; BC DAG edges */
    double algorithmic_bytes; /* SURVEY.md 8(d) formula for this call */
} gdx_stats;

const char* gdx_last_error(void);
int gdx_abi_version(void);
int gdx_device_count(int* count);

/* ---- graph lifetime ------------------------------------------------------ */
int gdx_graph_create(const gdx_csr_view* view, int device, gdx_graph** out);
int gdx_graph_destroy(gdx_graph* g);
/* Device memory of destroyed graphs and released workspaces is cached by the
 * library (size-matched reuse, like a caching allocator; capped at 48 GiB) so
 * create/destroy cycles avoid cudaMalloc/cudaFree.  Returns it to the driver. */
int gdx_pool_trim(int64_t* released_bytes);
int gdx_graph_info(const gdx_graph* g, int32_t* n, int32_t* m, int32_t* directed);
/* Copies the device CSR back; any pointer may be NULL to skip that array. */
int gdx_graph_download(gdx_graph* g, int32_t* offsets, int32_t* dests, int32_t* weights,
                       int32_t* rev_offsets, int32_t* rev_srcs, int32_t* rev_eid);
/* The CUDA stream (cudaStream_t) all kernels of this handle run on.  Setting
 * it to a caller stream (e.g. torch.cuda.current_stream()) orders the calls
 * with the caller's work; NULL restores the handle's own (non-blocking)
 * stream; cudaStreamLegacy ((void*)1) selects the legacy default stream. */
int gdx_graph_set_stream(gdx_graph* g, void* stream);
int gdx_graph_get_stream(gdx_graph* g, void** stream);

/* ---- device graph construction (csr.cpp:28-94 on the GPU) ----------------
 * u/v/w are host or device arrays of nedges input edges (w may be NULL).
 * Semantics are exactly CsrGraph::buildFromEdges: validation errors
 * (InvalidEdge / NegativeWeight), undirected doubling with self loops stored
 * once, sort by (u,v), duplicates keep the minimum weight, stable reverse CSR. */
int gdx_graph_build_from_edges(int32_t n, int64_t nedges, const int32_t* u, const int32_t* v,
                               const int32_t* w, int directed, int device, gdx_graph** out);

/* Edge-list files.  Load = CsrGraph::loadEdgeList (csr.cpp:96-130): "u v [w]"
 * lines, '#' comments, node count inferred as max id + 1 when node_count < 0;
 * errors "ParseError: malformed edge line in <path>" etc.; built on the GPU.
 * Write = writeEdgeList (csr.cpp:211-223): "# nodes N stored-edges M" header,
 * one line per stored edge (directed) or per u <= v pair (undirected). */
int gdx_graph_load_edge_list(const char* path, int directed, int32_t node_count, int device,
                             gdx_graph** out);
int gdx_graph_write_edge_list(gdx_graph* g, const char* path, int with_weights);

/* Counter-based synthetic generators on the GPU.
 * kind: 0 = RMAT (a,b,c; d = 1-a-b-c), 1 = uniform, 2 = 2-D grid (side x side,
 * each lattice edge kept with probability keep).  The edge list is built into
 * a CSR with buildFromEdges semantics.  Weights (if whi >= wlo >= 0) are
 * counter-hashed per unordered pair (symmetric on undirected graphs). */
typedef struct {
    int32_t kind;
    int32_t nodes;    /* RMAT/uniform: vertex count; grid: side */
    int64_t edges;    /* RMAT/uniform: edges drawn (before dedup) */
    uint64_t seed;
    double a, b, c;   /* RMAT */
    double keep;      /* grid */
    int32_t directed;
    int32_t wlo, whi; /* weights; whi < wlo => unweighted (all 1) */
} gdx_gen_params;
int gdx_graph_generate(const gdx_gen_params* p, int device, gdx_graph** out);
/* Counter-hash weights in [lo, hi] (symmetric for undirected graphs). */
int gdx_graph_set_hash_weights(gdx_graph* g, int32_t lo, int32_t hi, uint64_t seed);

/* ---- the reference's sequential streams (host side; refstream.cu) -----------
 * Exactly the reference's std::mt19937_64 streams, for feeding the device path
 * the reference's own inputs (parity configs, `graphdsl run --weight-*`):
 *   genUniformEdges (core/src/graphgen.cpp:8-16)   gdx_gen_uniform_edges_ref
 *   genRmatEdges    (core/src/graphgen.cpp:18-56)  gdx_gen_rmat_edges_ref
 *   gen-graph weight column (tools/graphdsl.cpp:281-287)
 *                                      gdx_gen_edge_weights_ref
 *   CsrGraph::withRandomWeights (core/src/csr.cpp:172-195)
 *                                      gdx_random_weights_host (host CSR arrays)
 *                                      gdx_graph_set_random_weights (a handle)
 * u, v, weights_out are host arrays of the given lengths.  Errors mirror the
 * reference's std::invalid_argument messages ("node count must be positive",
 * "weight range is empty", ...). */
int gdx_gen_uniform_edges_ref(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u, int32_t* v);
int gdx_gen_rmat_edges_ref(int32_t nodes, int64_t edges, uint64_t seed, double a, double b,
                           double c, double d, int32_t* u, int32_t* v);
/* gen-graph's weight column (tools/graphdsl.cpp:281-287): count draws of
 * uniform_int<int>(wmin, wmax) from mt19937_64(seed ^ 0x9e3779b97f4a7c15). */
int gdx_gen_edge_weights_ref(int64_t count, uint64_t seed, int32_t wmin, int32_t wmax,
                             int32_t* weights_out);
int gdx_random_weights_host(int32_t n, int32_t m, int32_t directed, const int32_t* offsets,
                            const int32_t* dests, int32_t lo, int32_t hi, uint64_t seed,
                            int32_t* weights_out);
int gdx_graph_set_random_weights(gdx_graph* g, int32_t lo, int32_t hi, uint64_t seed);

/* ---- the four entry points -------------------------------------------------
 * ComputeSSSP: dist_out[n] int64, unreachable = INT64_MAX/2 (oracles.hpp:12).
 * The corpus postconditions hold on return: `modified` is all false and
 * `finished` is true (test_interpreter.cpp:34-44). */
int gdx_sssp(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats);

/* ComputePR: rank_out[n] f64; *rounds_out = fixedPoint rounds executed
 * (== the interpreter's final `iter`), at most max_iter+1 (pr.sp:25). */
int gdx_pagerank(gdx_graph* g, double damping, double threshold, int32_t max_iter,
                 double* rank_out, int32_t* rounds_out, gdx_stats* stats);

/* ComputeTC: the tc.sp count (== its return value). */
int gdx_tc(gdx_graph* g, int64_t* count_out, gdx_stats* stats);
/* Partial count for sharding: the triangles whose owner vertex lies in
 * [v_begin, v_end).  The owner is tc.sp's middle vertex on directed graphs and
 * the smallest vertex on undirected ones (the oriented kernel, tc.cu); ranges
 * that partition [0, n) sum to gdx_tc either way. */
int gdx_tc_range(gdx_graph* g, int32_t v_begin, int32_t v_end, int64_t* count_out,
                 gdx_stats* stats);

/* ComputeBC: bc_out[n] f64, unnormalised, sources excluded (bc.sp:6-25).
 * Sigma never overflows (mantissa + exponent); the per-source dependencies are
 * summed in a fixed order (no floating-point atomics), so repeated calls on a
 * handle return bit-identical scores; within 1e-6 relative of the reference. */
int gdx_bc(gdx_graph* g, const int32_t* sources, int32_t nsrc, double* bc_out, gdx_stats* stats);

/* ---- multi-GPU shards (one process per GPU) ----------------
 * The caller owns the exchange (torch.distributed / NCCL in distributed.py);
 * all buffer pointers below may be device or host memory unless noted.
 *
 * PageRank, destination-vertex ranges: the rank computes rows [v_begin, v_end)
 * from the full contrib vector.  A round writes the slice's next contrib
 * (contrib_slice[v - v_begin]) and partials[2] = {dangling mass of the slice's
 * new ranks, unsettled vote 0/1}; the caller all-gathers the slices and
 * all-reduces the partials (dangling_in of the next round = the summed
 * dangling mass; the fixedPoint ends when no rank is unsettled).  Same
 * arithmetic as gdx_pagerank (pr.sp:5-33) -- replaces the single-address
 * dangling atomic and full-V launches of pr_cuda.cu:117-212. */
int gdx_pr_shard_setup(gdx_graph* g, int32_t v_begin, int32_t v_end);
int gdx_pr_shard_init(gdx_graph* g, double* contrib_slice, double* partials /* device [2] */);
int gdx_pr_shard_round(gdx_graph* g, int32_t round, double damping, double threshold,
                       int32_t max_iter, const double* dangling_in /* device [1] */,
                       const double* contrib_in /* device [n] */,
                       double* contrib_slice /* device */, double* partials /* device [2] */);
int gdx_pr_shard_rank(gdx_graph* g, int32_t rounds, double* rank_slice);

/* PageRank with the exchange fused into the kernels over peer memory (NVLink
 * P2P through CUDA IPC; one process per GPU).  After gdx_pr_shard_setup:
 * gdx_pr_p2p_setup exports this rank's exchange block (handle_out: 64 bytes,
 * a cudaIpcMemHandle_t); the caller all-gathers the handles (rank order) and
 * passes them to gdx_pr_p2p_open.  gdx_pr_p2p_init / _round then write every
 * new contrib value of the rank's rows straight into every rank's block from
 * the vertex kernel, publish (dangling mass, unsettled vote) with system-scope
 * atomics, and return the partials summed over all ranks in rank order
 * (partials_out: host [2]) -- no separate all-gather or all-reduce.  The final
 * ranks come from gdx_pr_shard_rank.  Same arithmetic as gdx_pagerank. */
int gdx_pr_p2p_setup(gdx_graph* g, int32_t world, int32_t rank, void* handle_out);
int gdx_pr_p2p_open(gdx_graph* g, const void* handles /* world * 64 bytes */);
int gdx_pr_p2p_init(gdx_graph* g, double* partials_out);
int gdx_pr_p2p_round(gdx_graph* g, int32_t round, double damping, double threshold,
                     int32_t max_iter, double dangling_in, double* partials_out);
/* Rounds [first, first + count) enqueued without host round trips: each ends
 * with a device-side wait for every rank's publish and the rank-ordered sum of
 * the published partials (next round's dangling mass, global vote); a round
 * after a settled one exits on the device.  dangling_in is used for round 0
 * only (from gdx_pr_p2p_init).  *settled_out = the first round in the range
 * whose global vote is "settled", or -1.  Every rank must issue the same ranges. */
int gdx_pr_p2p_rounds(gdx_graph* g, int32_t first, int32_t count, double damping,
                      double threshold, int32_t max_iter, double dangling_in,
                      int32_t* settled_out);
int gdx_pr_p2p_close(gdx_graph* g);

/* SSSP, vertex ranges: every rank keeps a full int64 replica of dist (device
 * [n], INF = INT64_MAX/2) and prev (device [n], the value each own vertex had
 * when last expanded).  frontier: queue the rank's vertices with dist < prev
 * (prev := dist) and report how many improved (*count_out, host or device);
 * relax: relax their out-edges into the local replica with atomicMin.  The
 * caller MIN-all-reduces dist between rounds and stops when no rank reports
 * an improvement (sssp.sp's fixedPoint; sssp_cuda.cu:117-199). */
int gdx_sssp_shard_setup(gdx_graph* g, int32_t v_begin, int32_t v_end);
int gdx_sssp_shard_frontier(gdx_graph* g, int64_t* dist, int64_t* prev, int64_t* count_out);
int gdx_sssp_shard_relax(gdx_graph* g, int64_t* dist);
/* The same rounds over int32 replicas (INF = INT32_MAX): half the gather and
 * collective bytes.  out2 = {improved count, overflow}: overflow is 1 when a
 * relaxation since the previous frontier call would have reached INT32_MAX;
 * the caller then reruns with the int64 entry points (distributed.py
 * sharded_sssp), so the result is exact either way. */
int gdx_sssp_shard_frontier32(gdx_graph* g, int32_t* dist, int32_t* prev, int64_t* out2);
int gdx_sssp_shard_relax32(gdx_graph* g, int32_t* dist);
/* Delta exchange: the int32 relaxation that also lists, once,
 * every vertex whose replica distance it lowered -- changed_ids / changed_dist
 * (device, capacity n) receive the ids and their values after the round,
 * *count_out (host or device) their number.  The caller all-gathers the lists
 * and applies every rank's pairs with gdx_sssp_shard_apply32 (element-wise MIN;
 * ids < 0 are padding) instead of MIN-all-reducing the whole replica. */
int gdx_sssp_shard_relax32_delta(gdx_graph* g, int32_t* dist, int32_t* changed_ids,
                                 int32_t* changed_dist, int64_t* count_out);
int gdx_sssp_shard_apply32(gdx_graph* g, int32_t* dist, const int32_t* ids, const int32_t* vals,
                           int64_t count);

/* ---- textbook kernels for `graphdsl check` (textbook.cu) -------------------
 * The reference's oracles (core/src/oracles.cpp:10-111) as plain topology-
 * driven device kernels -- one thread per vertex per round / level, a host
 * round trip per round, nothing shared with the fast paths -- so that `check`
 * (tools/graphdsl.cpp:175-256) compares two independent device computations:
 *   oracles::sssp -> gdx_textbook_sssp (Bellman-Ford rounds; same distances)
 *   oracles::pr   -> gdx_textbook_pr   (<= max_iter iterations, stop when
 *                                       max |delta| < eps, oracles.cpp:73-92)
 *   oracles::tc   -> gdx_textbook_tc   (tc.sp's u < v < w by binary search;
 *                                       no n <= 256 guard)
 *   oracles::bc   -> gdx_textbook_bc   (level-synchronous Brandes per source)
 * Sized for check-size graphs, not for the benchmark configurations. */
int gdx_textbook_sssp(gdx_graph* g, int32_t src, int64_t* dist_out);
int gdx_textbook_pr(gdx_graph* g, double damping, double eps, int32_t max_iter, double* rank_out);
int gdx_textbook_tc(gdx_graph* g, int64_t* count_out);
int gdx_textbook_bc(gdx_graph* g, const int32_t* sources, int32_t nsrc, double* bc_out);

/* ---- several GPUs from one process (multi.cu) --------
 * For a C++ caller of interp::run (interpreter.hpp:64-88) that wants an
 * ExecMode::Device over a device list.  gdx_context_create enables peer access
 * between every pair of the listed devices (required: NVLink / NVSwitch) and,
 * when every device is distinct, creates one NCCL communicator per device
 * (ncclCommInitAll; NCCL is dlopen'ed, *nccl_comms reports how many).  A
 * device may be listed more than once (several partitions on one GPU: the
 * same protocol, no NCCL).  gdx_multi_graph_create uploads a replica of the
 * graph to every device of the context.  The *_multi entry points have the
 * single-GPU semantics and outputs (host pointers, or memory on the first
 * device) and partition the work per SURVEY.md 8(e):
 *   SSSP  vertex ranges by out-edges; improving candidates go straight to the
 *         owner's distance replica by peer atomicMin; the round loop and its
 *         barriers run on the devices (no dist all-gather)
 *   PR    destination ranges by in-edges; new contrib values and the
 *         (dangling, unsettled) partials are written into every device's
 *         buffers over peer memory (no per-round collective)
 *   TC    owner-vertex ranges by ~deg^2; counts summed in device order
 *   BC    contiguous source blocks; one ncclAllReduce (sum) of the scores, or
 *         a peer-memory sum in device order without NCCL
 * Results: SSSP distances and TC counts identical to the single-GPU calls;
 * PR ranks identical (same arithmetic, rank-ordered partial sums); BC within
 * 1e-6 relative (the cross-device sum order differs from source order). */
typedef struct gdx_context gdx_context;
typedef struct gdx_multi_graph gdx_multi_graph;
int gdx_context_create(int ndev, const int* devices, gdx_context** out);
int gdx_context_destroy(gdx_context* ctx);
int gdx_context_info(const gdx_context* ctx, int32_t* ndev, int32_t* nccl_comms,
                     int32_t* peer_access);
int gdx_multi_graph_create(gdx_context* ctx, const gdx_csr_view* view, gdx_multi_graph** out);
int gdx_multi_graph_destroy(gdx_multi_graph* g);
int gdx_sssp_multi(gdx_multi_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats);
int gdx_pagerank_multi(gdx_multi_graph* g, double damping, double threshold, int32_t max_iter,
                       double* rank_out, int32_t* rounds_out, gdx_stats* stats);
int gdx_tc_multi(gdx_multi_graph* g, int64_t* count_out, gdx_stats* stats);
int gdx_bc_multi(gdx_multi_graph* g, const int32_t* sources, int32_t nsrc, double* bc_out,
                 gdx_stats* stats);

/* SSSP partitions with one process per GPU over peer memory (the multi-
 * process form of gdx_sssp_multi; distributed.py sharded_sssp_p2p).  bounds:
 * world+1 vertex-range bounds partitioning [0, n).  gdx_sssp_p2p_setup
 * exports this rank's block {distance replica | barrier state}
 * (handle_out: 64 bytes, a cudaIpcMemHandle_t); the caller all-gathers the
 * handles in rank order and passes them to gdx_sssp_p2p_open.  Every rank then
 * calls gdx_sssp_p2p_run with the same source: its partition's relaxations
 * send improving candidates to the owners' replicas by peer atomicMin, the
 * rounds and their barriers run on the devices (no per-round collective, no
 * host round trip), and dist_out (n, host or device) receives the whole
 * vector read from the owners' replicas.  Bit-exact like gdx_sssp. */
int gdx_sssp_p2p_setup(gdx_graph* g, int32_t world, int32_t rank, const int32_t* bounds,
                       void* handle_out);
int gdx_sssp_p2p_open(gdx_graph* g, const void* handles /* world * 64 bytes */);
int gdx_sssp_p2p_run(gdx_graph* g, int32_t src, int64_t* dist_out, gdx_stats* stats);
int gdx_sssp_p2p_close(gdx_graph* g);

/* The degree-ordered renumbering gdx_pagerank / gdx_sssp run skewed graphs of
 * >= 2^22 vertices on (csrc/relabel.cu; GDX_RELABEL=0/1 overrides): new id i
 * is the i-th vertex by descending out-degree.  No reference counterpart --
 * it lets the partitioned paths above (distributed.py) run on the same
 * renumbered graph as the single-GPU calls.  algo: 0 PageRank (reverse CSR),
 * 1 SSSP (forward CSR).  *h_out = the renumbered graph, owned by g (valid
 * until g is destroyed or its weights change; never destroy it), or NULL when
 * g is not renumbered for that algorithm; newid_out (n int32, host or device,
 * may be NULL) receives newid[v] for every vertex v of g. */
int gdx_graph_renumbered(gdx_graph* g, int32_t algo, gdx_graph** h_out, int32_t* newid_out);

/* ---- measurement ------------------------------------------------------------
 * When enabled, the library brackets every kernel launch of this handle with
 * CUDA events on the launching stream.  gdx_profile_read reports, per kernel
 * name, the summed device time (ms) and launch count since the last reset. */
int gdx_profile_enable(gdx_graph* g, int enable);
int gdx_profile_reset(gdx_graph* g);
/* Writes up to cap entries; *count = number of distinct kernels. */
int gdx_profile_read(gdx_graph* g, char* names /* cap*64 bytes */, double* ms, int64_t* launches,
                     int32_t cap, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* GDX_H */
