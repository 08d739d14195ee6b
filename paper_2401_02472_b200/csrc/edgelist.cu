// edgelist.cu -- edge-list file I/O for device graphs (host code).
//
// gdx_graph_load_edge_list follows CsrGraph::loadEdgeList (reference
// core/src/csr.cpp:96-130): one "u v [w]" edge per line, blank lines and lines
// starting with '#' skipped, iostream extraction semantics (a non-numeric third
// token leaves the edge unweighted; a fourth token is an error), the node count
// inferred as max id + 1 unless given; errors carry the reference's messages
// (ParseError with the line number, "cannot open graph file").  The edges are
// then built on the GPU with buildFromEdges semantics (build.cu).
// gdx_graph_write_edge_list follows writeEdgeList (csr.cpp:211-223).
#include <algorithm>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "gdx_internal.cuh"
#include "plans.cuh"

using namespace gdx;

extern "C" {

int gdx_graph_load_edge_list(const char* path, int directed, int32_t node_count, int device,
                             gdx_graph** out) {
    std::vector<int32_t> u, v, w;
    bool any_weight = false;
    int rc = guard_impl([&] {
        if (!path || !out) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        std::ifstream in(path);
        if (!in) fail(GDX_ERR_RUNTIME, std::string("RuntimeError: cannot open graph file: ") + path);
        std::string line;
        int64_t line_no = 0;  // the reference reports it in the CompileError span
        int32_t max_id = -1;
        auto parse_error = [&](const std::string& msg) {
            fail(GDX_ERR_INVALID_ARGUMENT,
                 "ParseError: " + msg + " in " + path);
        };
        while (std::getline(in, line)) {
            ++line_no;
            (void)line_no;
            const size_t first = line.find_first_not_of(" \t\r");
            if (first == std::string::npos || line[first] == '#') continue;
            std::istringstream ls(line);
            long long a, b;
            if (!(ls >> a >> b)) parse_error("malformed edge line");
            long long wt = 1;
            bool has_w = false;
            if (ls >> wt) has_w = true;
            std::string rest;
            if (ls >> rest) parse_error("trailing characters on edge line");
            if (a < 0 || b < 0 || a > INT32_MAX || b > INT32_MAX) parse_error("node id out of range");
            u.push_back(int32_t(a));
            v.push_back(int32_t(b));
            w.push_back(has_w ? int32_t(wt) : 1);
            any_weight |= has_w;
            max_id = std::max(max_id, int32_t(std::max(a, b)));
        }
        const int32_t n = node_count >= 0 ? node_count : max_id + 1;
        *out = nullptr;
        const int brc = gdx_graph_build_from_edges(n, int64_t(u.size()), u.data(), v.data(),
                                                   any_weight ? w.data() : nullptr, directed,
                                                   device, out);
        if (brc != GDX_OK) throw Error(gdx_status(brc), gdx_last_error());
    });
    return rc;
}

int gdx_graph_write_edge_list(gdx_graph* g, const char* path, int with_weights) {
    return guard_impl([&] {
        if (!g || !path) fail(GDX_ERR_INVALID_ARGUMENT, "InvalidArgument: null argument");
        if (!g->dests.get() && g->m > 0)
            fail(GDX_ERR_UNSUPPORTED, "Unsupported: graph has no forward adjacency");
        std::vector<int32_t> off(size_t(g->n) + 1), dst(g->m), wt(g->m);
        const int rc = gdx_graph_download(g, off.data(), dst.data(), wt.data(), nullptr, nullptr,
                                          nullptr);
        if (rc != GDX_OK) throw Error(gdx_status(rc), gdx_last_error());
        std::ofstream out(path);
        if (!out) fail(GDX_ERR_RUNTIME, std::string("RuntimeError: cannot open output file: ") + path);
        out << "# nodes " << g->n << " stored-edges " << g->m << "\n";
        for (int32_t a = 0; a < g->n; ++a)
            for (int32_t e = off[a]; e < off[a + 1]; ++e) {
                if (!g->directed && dst[e] < a) continue;
                out << a << " " << dst[e];
                if (with_weights) out << " " << wt[e];
                out << "\n";
            }
        if (!out) fail(GDX_ERR_RUNTIME, std::string("RuntimeError: write failed: ") + path);
    });
}

}  // extern "C"
