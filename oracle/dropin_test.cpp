// dropin_test.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A reference-side C++ caller exercising the drop-in: it builds graphs and
// programs with the reference's own API (CsrGraph, genRmatEdges, parseSource,
// typeCheck), runs each corpus program through interp::run (the reference) and
// through gdx_graphdsl::run (include/gdx_graphdsl.hpp -> libgdx.so on the B200),
// and compares the RunResults with the corpus tolerances.  Built by
// `make -C oracle ref` into oracle/_ref/gdx_dropin_test (needs the reference
// headers, so it is compiled here and run on the GPU box).  Exit 0 = all PASS.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "graphdsl/csr.hpp"
#include "graphdsl/diagnostics.hpp"
#include "graphdsl/graphgen.hpp"
#include "graphdsl/interpreter.hpp"
#include "graphdsl/parser.hpp"
#include "graphdsl/sema.hpp"
#include "gdx_graphdsl.hpp"

using namespace graphdsl;

extern const char* gdx_ref_corpus_source(const char* name);

static int failures = 0;

static void report(const std::string& what, bool ok, const std::string& note = "") {
    std::printf("%s [%s]%s%s\n", what.c_str(), ok ? "PASS" : "FAIL", note.empty() ? "" : " - ",
                note.c_str());
    if (!ok) ++failures;
}

static double relerr(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return 1e300;
    double e = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        double s = std::max({std::fabs(a[i]), std::fabs(b[i]), 1e-12});
        e = std::max(e, std::fabs(a[i] - b[i]) / s);
    }
    return e;
}

int main() {
    auto load = [](const char* name) {
        return sema::typeCheck(parseSource(gdx_ref_corpus_source(name)), name);
    };
    auto sssp = load("sssp"), pr = load("pr"), tc = load("tc"), bc = load("bc");
    interp::RunOptions par{interp::ExecMode::Parallel, 8};
    for (uint64_t seed : {1ull, 2ull, 3ull}) {
        const int32_t n = 1 << 12;
        auto edges = genRmatEdges(n, 16 * n, seed);
        CsrGraph und = CsrGraph::buildFromEdges(n, edges, false).withRandomWeights(1, 100, seed);
        CsrGraph dir = CsrGraph::buildFromEdges(n, edges, true);
        gdx_graphdsl::DeviceGraph du(und), dd(dir);
        std::string tag = " seed " + std::to_string(seed);

        auto a = interp::run(sssp, und, {{"src", int64_t(seed)}}, par);
        auto b = gdx_graphdsl::run(sssp, du, {{"src", int64_t(seed)}});
        report("ComputeSSSP dist" + tag,
               a.property(sssp.symbols, "dist")->ints == b.property(sssp.symbols, "dist")->ints);
        report("ComputeSSSP modified/finished" + tag,
               a.property(sssp.symbols, "modified")->bools == b.property(sssp.symbols, "modified")->bools &&
                   b.scalar(sssp.symbols, "finished")->asBool());

        interp::ArgMap prArgs{{"damping", 0.85}, {"threshold", 1e-9}, {"maxIter", int64_t(110)}};
        a = interp::run(pr, dir, prArgs, par);
        b = gdx_graphdsl::run(pr, dd, prArgs);
        double e = relerr(a.property(pr.symbols, "rank")->floats, b.property(pr.symbols, "rank")->floats);
        report("ComputePR rank" + tag, e < 1e-9, "max rel " + std::to_string(e));
        report("ComputePR iter" + tag,
               a.scalar(pr.symbols, "iter")->asInt() == b.scalar(pr.symbols, "iter")->asInt());

        a = interp::run(tc, und, {}, par);
        b = gdx_graphdsl::run(tc, du, {});
        report("ComputeTC" + tag,
               a.scalar(tc.symbols, "triangleCount")->asInt() ==
                       b.scalar(tc.symbols, "triangleCount")->asInt() &&
                   a.returnValue->asInt() == b.returnValue->asInt());

        std::vector<int32_t> srcs{0, 1, 2, 3, 100, 4095};
        a = interp::run(bc, und, {{"sourceSet", srcs}}, par);
        b = gdx_graphdsl::run(bc, du, {{"sourceSet", srcs}});
        e = relerr(a.property(bc.symbols, "bc")->floats, b.property(bc.symbols, "bc")->floats);
        report("ComputeBC" + tag, e < 1e-9, "max rel " + std::to_string(e));
    }
    // ExecMode::Device over a device list (gdx_context / gdx_*_multi): one GPU,
    // and device 0 listed twice (two partitions of the same protocol)
    for (const std::vector<int>& devs : {std::vector<int>{0}, std::vector<int>{0, 0}}) {
        const int32_t n = 1 << 12;
        auto edges = genRmatEdges(n, 16 * n, 7);
        CsrGraph und = CsrGraph::buildFromEdges(n, edges, false).withRandomWeights(1, 100, 7);
        CsrGraph dir = CsrGraph::buildFromEdges(n, edges, true);
        gdx_graphdsl::MultiDevice ctx(devs);
        gdx_graphdsl::MultiGraph mu(ctx, und), md(ctx, dir);
        std::string tag = " devices x" + std::to_string(devs.size());
        auto a = interp::run(sssp, und, {{"src", int64_t(7)}}, par);
        auto b = gdx_graphdsl::run(sssp, mu, {{"src", int64_t(7)}});
        report("multi ComputeSSSP dist" + tag,
               a.property(sssp.symbols, "dist")->ints == b.property(sssp.symbols, "dist")->ints);
        interp::ArgMap prArgs{{"damping", 0.85}, {"threshold", 1e-9}, {"maxIter", int64_t(110)}};
        a = interp::run(pr, dir, prArgs, par);
        b = gdx_graphdsl::run(pr, md, prArgs);
        double e = relerr(a.property(pr.symbols, "rank")->floats, b.property(pr.symbols, "rank")->floats);
        report("multi ComputePR" + tag,
               e < 1e-9 && a.scalar(pr.symbols, "iter")->asInt() == b.scalar(pr.symbols, "iter")->asInt(),
               "max rel " + std::to_string(e));
        a = interp::run(tc, und, {}, par);
        b = gdx_graphdsl::run(tc, mu, {});
        report("multi ComputeTC" + tag, a.returnValue->asInt() == b.returnValue->asInt());
        std::vector<int32_t> srcs{0, 1, 2, 3, 100, 4095};
        a = interp::run(bc, und, {{"sourceSet", srcs}}, par);
        b = gdx_graphdsl::run(bc, mu, {{"sourceSet", srcs}});
        e = relerr(a.property(bc.symbols, "bc")->floats, b.property(bc.symbols, "bc")->floats);
        report("multi ComputeBC" + tag, e < 1e-9, "max rel " + std::to_string(e));
    }
    // interp::run-shaped overload (uploads per call) and error kinds
    CsrGraph tri = CsrGraph::buildFromEdges(3, {{0, 1, 5}, {1, 2, 1}, {0, 2, 7}}, false);
    auto r = gdx_graphdsl::run(sssp, tri, {{"src", int64_t(0)}});
    report("weighted triangle [0,5,6]",
           r.property(sssp.symbols, "dist")->ints == std::vector<int64_t>{0, 5, 6});
    auto kind_of = [&](auto&& fn) -> std::string {
        try {
            fn();
        } catch (const CompileError& e) {
            return e.kind() + ": " + e.what();
        }
        return "";
    };
    std::string k1 = kind_of([&] { gdx_graphdsl::run(sssp, tri, {{"src", int64_t(99)}}); });
    std::string k2 = kind_of([&] { interp::run(sssp, tri, {{"src", int64_t(99)}}); });
    report("out-of-range source kind", k1.rfind("RuntimeError", 0) == 0 && k2.rfind("RuntimeError", 0) == 0,
           k1 + " | " + k2);
    std::string k3 = kind_of([&] { gdx_graphdsl::run(bc, tri, {}); });
    report("missing node-set argument", k3.find("missing node-set argument 'sourceSet'") != std::string::npos, k3);
    CsrGraph cyc = CsrGraph::buildFromEdges(2, {{0, 1, {}}, {1, 0, {}}}, true);
    std::string k4 = kind_of([&] {
        gdx_graphdsl::run(pr, cyc, {{"damping", 0.85}, {"threshold", -1.0}, {"maxIter", int64_t(1000)}});
    });
    interp::RunOptions capped;
    std::string k5 = kind_of([&] {
        interp::run(pr, cyc, {{"damping", 0.85}, {"threshold", -1.0}, {"maxIter", int64_t(1000)}}, capped);
    });
    report("NonTermination kind", k4.rfind("NonTermination", 0) == 0 && k5.rfind("NonTermination", 0) == 0,
           k4 + " | " + k5);
    std::printf("%s\n", failures ? "DROPIN FAIL" : "DROPIN PASS");
    return failures ? 1 : 0;
}
