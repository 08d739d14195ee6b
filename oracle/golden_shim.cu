// oracle/golden_shim.cu -- TEST / MEASUREMENT INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the reference's own generated CUDA units
// (proj/tests/golden/{sssp,pr,tc,bc}/cuda/*.cu, compiled unchanged from where
// they lie by `make -C oracle golden` into oracle/_ref/libgolden.so): the
// reference's GPU realisation of the corpus, timed beside ours on the same
// B200 by tools/golden_gpu.py.  Each golden unit does its own cudaMalloc,
// upload, per-iteration host round trips and download per call
// (e.g. pr_cuda.cu:150-224); nothing here changes that.
#include <cstdint>

typedef struct GraphCsr {  // layout of the golden units' GraphCsr (pr_cuda.cu:8-17)
    int n;
    int m;
    int* offsets;
    int* dests;
    int* weights;
    int* rev_offsets;
    int* rev_srcs;
    int* rev_eid;
} GraphCsr;

void computesssp(const GraphCsr& g, int* dist, const int* weight, int src);
void computepr(const GraphCsr& g, double damping, double threshold, int maxIter, double* rank);
long long computetc(const GraphCsr& g);
void computebc(const GraphCsr& g, double* bc, const int* sourceSet, int sourceSet_count);

static GraphCsr view(int n, int m, int* off, int* dst, int* w, int* roff, int* rsrc, int* reid) {
    GraphCsr g;
    g.n = n;
    g.m = m;
    g.offsets = off;
    g.dests = dst;
    g.weights = w;
    g.rev_offsets = roff;
    g.rev_srcs = rsrc;
    g.rev_eid = reid;
    return g;
}

extern "C" {
void golden_sssp(int n, int m, int* off, int* dst, int* w, int* roff, int* rsrc, int* reid,
                 int src, int* dist) {
    computesssp(view(n, m, off, dst, w, roff, rsrc, reid), dist, w, src);
}
void golden_pr(int n, int m, int* off, int* dst, int* w, int* roff, int* rsrc, int* reid,
               double damping, double threshold, int max_iter, double* rank) {
    computepr(view(n, m, off, dst, w, roff, rsrc, reid), damping, threshold, max_iter, rank);
}
long long golden_tc(int n, int m, int* off, int* dst, int* w, int* roff, int* rsrc, int* reid) {
    return computetc(view(n, m, off, dst, w, roff, rsrc, reid));
}
void golden_bc(int n, int m, int* off, int* dst, int* w, int* roff, int* rsrc, int* reid,
               const int* sources, int nsrc, double* bc) {
    computebc(view(n, m, off, dst, w, roff, rsrc, reid), bc, sources, nsrc);
}
}
