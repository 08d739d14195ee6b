// unit_main.cpp -- the emitted units' command-line contract over libgdx.
//
// The reference's code generator gives every generated unit a main()
// (core/src/codegen_runtime.cpp:174-296; e.g. tests/golden/sssp/cuda/
// sssp_cuda.cu:201-218):
//
//   <unit> <graph> <directed 0|1> <scalar args / comma-separated node set>
//
// prints `return<TAB>value` for a returned scalar, then `name<TAB>i<TAB>value`
// for every node property (%.17g for floating point), and exits 2 with a
// usage line when fewer than two arguments are given.  This file builds the
// same four executables (bin/{sssp,pr,tc,bc}_b200) on the B200 path: the
// edge list goes through gdx_graph_load_edge_list (csr.cpp:96-130 semantics,
// which match the emitted loader: n = max id + 1, duplicates keep the minimum
// weight, undirected edges stored both ways) and the entry point through the
// C ABI.  One deliberate difference: the generated SSSP unit keeps int
// distances, so an unreachable vertex prints INT_MAX / 2 -- printed the same
// here -- while a reachable distance above INT_MAX / 2 prints its exact int64
// value instead of the generated unit's overflowed int.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/gdx.h"

static int die(const char* what) {
    std::fprintf(stderr, "%s: %s\n", what, gdx_last_error());
    return 1;
}

int main(int argc, char** argv) {
#if defined(GDX_UNIT_SSSP)
    const char* usage = "<graph> <directed 0|1> <src>";
#elif defined(GDX_UNIT_PR)
    const char* usage = "<graph> <directed 0|1> <damping> <threshold> <maxIter>";
#elif defined(GDX_UNIT_TC)
    const char* usage = "<graph> <directed 0|1>";
#else
    const char* usage = "<graph> <directed 0|1> <sourceSet>";
#endif
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s %s\n", argv[0], usage);
        return 2;
    }
    const char* dev_env = std::getenv("GDX_DEVICE");
    const int device = dev_env ? std::atoi(dev_env) : 0;
    gdx_graph* g = nullptr;
    if (gdx_graph_load_edge_list(argv[1], std::atoi(argv[2]), -1, device, &g) != GDX_OK)
        return die("load");
    int32_t n = 0;
    gdx_graph_info(g, &n, nullptr, nullptr);
#if defined(GDX_UNIT_SSSP)
    const int32_t src = argc > 3 ? int32_t(std::atoll(argv[3])) : 0;
    std::vector<int64_t> dist(size_t(n) + 1);
    if (gdx_sssp(g, src, dist.data(), nullptr) != GDX_OK) return die("sssp");
    for (int32_t i = 0; i < n; ++i) {
        const long long d = dist[i] >= INT64_MAX / 2 ? INT_MAX / 2 : (long long)dist[i];
        std::printf("dist\t%d\t%lld\n", i, d);
    }
#elif defined(GDX_UNIT_PR)
    const double damping = argc > 3 ? std::atof(argv[3]) : 0.0;
    const double threshold = argc > 4 ? std::atof(argv[4]) : 0.0;
    const int32_t max_iter = argc > 5 ? int32_t(std::atoll(argv[5])) : 0;
    std::vector<double> rank(size_t(n) + 1);
    if (gdx_pagerank(g, damping, threshold, max_iter, rank.data(), nullptr, nullptr) != GDX_OK)
        return die("pagerank");
    for (int32_t i = 0; i < n; ++i) std::printf("rank\t%d\t%.17g\n", i, rank[i]);
#elif defined(GDX_UNIT_TC)
    int64_t count = 0;
    if (gdx_tc(g, &count, nullptr) != GDX_OK) return die("tc");
    std::printf("return\t%lld\n", (long long)count);
#else
    std::vector<int32_t> sources;
    if (argc > 3) {
        std::vector<char> list(argv[3], argv[3] + std::strlen(argv[3]) + 1);
        for (char* tok = std::strtok(list.data(), ","); tok; tok = std::strtok(nullptr, ","))
            sources.push_back(std::atoi(tok));
    }
    std::vector<double> bc(size_t(n) + 1);
    if (gdx_bc(g, sources.data(), int32_t(sources.size()), bc.data(), nullptr) != GDX_OK)
        return die("bc");
    for (int32_t i = 0; i < n; ++i) std::printf("bc\t%d\t%.17g\n", i, bc[i]);
#endif
    gdx_graph_destroy(g);
    return 0;
}
