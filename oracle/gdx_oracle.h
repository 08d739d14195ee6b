/*
 * gdx_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement ("port") of the reference's hot path (arxiv/paper_2401_02472,
 * /root/reference/proj/core) used as the parity checker for the B200 kernels.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product library
 * (paper_2401_02472_b200/lib/libgdx.so) never links or calls it.
 *
 * Parity pinning: every function here is checked against the reference itself
 * (oracle/_ref/libgraphdsl_ref.so, compiled from the reference's own sources by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 */
#ifndef GDX_ORACLE_H
#define GDX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A CSR graph laid out exactly like graphdsl::CsrGraph (csr.hpp:73-81). */
typedef struct orc_graph orc_graph;

typedef struct {
    int32_t n, m, directed;
    const int32_t* offsets;     /* n+1 */
    const int32_t* dests;       /* m   */
    const int32_t* weights;     /* m, NULL = all 1 */
    const int32_t* rev_offsets; /* n+1 */
    const int32_t* rev_srcs;    /* m   */
    const int32_t* rev_eid;     /* m   */
} orc_csr;

const char* orc_last_error(void);

/* ---- graph construction: csr.cpp:28-94, :172-195 ---------------------- */
/* Returns 0 on success, nonzero (see orc_last_error) on invalid input. */
int orc_build_from_edges(int32_t n, int64_t nedges, const int32_t* u, const int32_t* v,
                         const int32_t* w /* nullable */, int directed, orc_graph** out);
/* Copy stored CSR arrays into an owned graph (weights NULL -> all 1). */
int orc_graph_from_csr(const orc_csr* view, orc_graph** out);
int orc_with_random_weights(orc_graph* g, int32_t lo, int32_t hi, uint64_t seed);
void orc_graph_view(const orc_graph* g, orc_csr* view);
void orc_graph_free(orc_graph* g);

/* ---- reference generators (mt19937_64 stream): graphgen.cpp:8-56 -------- */
int orc_gen_uniform_edges(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u, int32_t* v);
int orc_gen_rmat_edges(int32_t nodes, int64_t edges, uint64_t seed, double a, double b, double c,
                       double d, int32_t* u, int32_t* v);

/* ---- counter-based generators: CPU twin of the product's GPU generators --
 * (paper_2401_02472_b200/csrc/generate.cu).  Not reference code: they let the
 * tests rebuild the bench-size graphs on the CPU to check the GPU builder. */
int orc_gen_rmat_ctr(int32_t scale_nodes, int64_t edges, uint64_t seed, double a, double b,
                     double c, int32_t* u, int32_t* v, int nthreads);
int orc_gen_uniform_ctr(int32_t nodes, int64_t edges, uint64_t seed, int32_t* u, int32_t* v,
                        int nthreads);
/* Grid: side x side lattice, each of the 2*side*(side-1) edges kept with
 * probability keep.  Returns the number of kept edges; u/v may be NULL to count. */
int64_t orc_gen_grid_ctr(int32_t side, double keep, uint64_t seed, int32_t* u, int32_t* v);
/* Counter-based weights in [lo, hi], symmetric for undirected graphs. */
void orc_hash_weights(const orc_csr* g, int32_t lo, int32_t hi, uint64_t seed, int32_t* w_out,
                      int nthreads);

/* ---- the four algorithms ------------------------------------------------- */
/* Dijkstra, oracles.cpp:10-31.  dist: int64, INF = INT64_MAX/2. */
int orc_sssp(const orc_csr* g, int32_t src, int64_t* dist);
/* ComputePR semantics (pr.sp:5-33; interpreter fixedPoint :968-1000): up to
 * maxIter+1 rounds, per-node |change| >= threshold vote.  Each node's gather
 * is sequential in ascending in-neighbour order and the dangling sum ascends,
 * so the result is bit-identical to oracles::pr(g, d, thr, rounds)
 * (oracles.cpp:73-92) and to the sequential interpreter. */
int orc_pr(const orc_csr* g, double damping, double threshold, int32_t max_iter, double* rank,
           int32_t* rounds, int nthreads);
/* Run exactly `rounds` PR rounds (for bounded CPU-baseline samples). */
int orc_pr_rounds(const orc_csr* g, double damping, int32_t rounds, double* rank, int nthreads);
/* ComputeTC semantics (tc.sp:6-18): sum over v of |{(u,w): u<v<w, u,w in N(v), (u,w) in E}|.
 * Scalable restatement (oracles::tc is O(n^3), guarded to n<=256). */
int orc_tc(const orc_csr* g, int64_t* count, int nthreads);
/* Middle vertices restricted to [v_begin, v_end) -- for sharded checks. */
int orc_tc_range(const orc_csr* g, int32_t v_begin, int32_t v_end, int64_t* count, int nthreads);
int orc_tc_range_owner(const orc_csr* g, int32_t v_begin, int32_t v_end, int64_t* count,
                       int nthreads);
/* Brandes over a source set, oracles.cpp:33-71, with sigma carried as
 * (double mantissa, int exponent) so it never overflows.  Bit-identical to
 * oracles::bc wherever the reference's double sigma stays finite. */
int orc_bc(const orc_csr* g, const int32_t* sources, int32_t nsrc, double* bc, int nthreads);
/* Queue BFS levels, oracles.cpp:113-129. */
int orc_bfs_levels(const orc_csr* g, int32_t root, int32_t* level);

#ifdef __cplusplus
}
#endif
#endif
