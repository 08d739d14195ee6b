// gdx_graphdsl.hpp -- header-only C++ drop-in for graphdsl::interp::run on the
// four corpus programs, executing on the B200 through the C ABI in gdx.h.
//
// Include it after the reference's own headers; it speaks the reference's types:
//
//   #include "graphdsl/interpreter.hpp"      // reference: core/include/graphdsl/
//   #include "gdx_graphdsl.hpp"
//   auto r = gdx_graphdsl::run(program, graph, args);   // same shape as interp::run
//   r.property(program.symbols, "dist")->ints ...
//
// Replaces interp::run (reference core/include/graphdsl/interpreter.hpp:87-88) for
// programs whose entry is ComputeSSSP / ComputePR / ComputeTC / ComputeBC
// (core/src/corpus.cpp:57-106); anything else raises
// CompileError("UnsupportedConstruct").  Argument binding and its errors follow
// Machine::executeImpl (core/src/interpreter.cpp:1099-1140); the result holds the
// symbols the interpreter leaves for each program:
//   ComputeSSSP: dist (Int), modified (Bool, all false), finished = true
//   ComputePR:   rank, rankNext (Float), settled (Bool, all true), iter, converged, numNodes
//   ComputeTC:   triangleCount; returnValue
//   ComputeBC:   bc (Float)
// Library failures are rethrown as graphdsl::CompileError with the kind carried
// by gdx_last_error() ("RuntimeError", "NonTermination", ...).
#pragma once

#include <cstdint>
#include <limits>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "gdx.h"

namespace gdx_graphdsl {

namespace detail {

inline void check(int rc) {
    if (rc == GDX_OK) return;
    std::string msg = gdx_last_error();
    std::string kind = "RuntimeError";
    auto colon = msg.find(':');
    if (colon != std::string::npos) kind = msg.substr(0, colon);
    throw graphdsl::CompileError(kind, graphdsl::SourceSpan{}, msg);
}

[[noreturn]] inline void rt(const std::string& msg) {
    throw graphdsl::CompileError("RuntimeError", graphdsl::SourceSpan{}, msg);
}

// Value::asInt / asFloat of an ArgValue bound into a scalar cell.
inline int64_t as_int(const graphdsl::interp::ArgValue& v) {
    if (std::holds_alternative<int64_t>(v)) return std::get<int64_t>(v);
    if (std::holds_alternative<double>(v)) return static_cast<int64_t>(std::get<double>(v));
    return 0;
}
inline double as_float(const graphdsl::interp::ArgValue& v) {
    if (std::holds_alternative<int64_t>(v)) return static_cast<double>(std::get<int64_t>(v));
    if (std::holds_alternative<double>(v)) return std::get<double>(v);
    return 0.0;
}

inline const graphdsl::interp::ArgValue& scalar_arg(const graphdsl::interp::ArgMap& args,
                                                    const std::string& name) {
    auto it = args.find(name);
    if (it == args.end()) rt("missing argument '" + name + "'");
    if (std::holds_alternative<std::vector<int32_t>>(it->second))
        rt("argument '" + name + "' has the wrong shape");
    return it->second;
}

inline int32_t node_arg(int64_t v, int32_t n) {
    if (v < 0 || v >= n)
        rt("node id " + std::to_string(v) + " out of range [0, " + std::to_string(n) + ")");
    return static_cast<int32_t>(v);
}

inline int sym(const graphdsl::sema::AnnotatedProgram& p, const char* name) {
    const auto* s = p.symbols.findByName(name);
    return s ? s->id : -1;
}

}  // namespace detail

// A CsrGraph resident in HBM.  Construct once, reuse across calls (the
// reference keeps its CsrGraph immutable and shared the same way).
class DeviceGraph {
public:
    template <class Csr>
    explicit DeviceGraph(const Csr& g, int device = 0) {
        gdx_csr_view v{};
        v.n = g.nodeCount();
        v.m = g.edgeCount();
        v.directed = g.directed() ? 1 : 0;
        v.offsets = g.offsets().data();
        v.dests = g.dests().data();
        v.weights = g.weights().data();
        v.rev_offsets = g.revOffsets().data();
        v.rev_srcs = g.revSrcs().data();
        v.rev_eid = g.revEid().data();
        detail::check(gdx_graph_create(&v, device, &h_));
    }
    ~DeviceGraph() {
        if (h_) gdx_graph_destroy(h_);
    }
    DeviceGraph(const DeviceGraph&) = delete;
    DeviceGraph& operator=(const DeviceGraph&) = delete;
    DeviceGraph(DeviceGraph&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

    gdx_graph* get() const { return h_; }
    int32_t nodeCount() const {
        int32_t n = 0;
        detail::check(gdx_graph_info(h_, &n, nullptr, nullptr));
        return n;
    }
    int sssp(int32_t src, int64_t* out) const { return gdx_sssp(h_, src, out, nullptr); }
    int pagerank(double d, double t, int32_t mi, double* out, int32_t* rounds) const {
        return gdx_pagerank(h_, d, t, mi, out, rounds, nullptr);
    }
    int tc(int64_t* out) const { return gdx_tc(h_, out, nullptr); }
    int bc(const int32_t* s, int32_t k, double* out) const { return gdx_bc(h_, s, k, out, nullptr); }

private:
    gdx_graph* h_ = nullptr;
};

namespace detail {
// The binding and result symbols of interp::run for the four entries, over a
// backend E: one GPU (DeviceGraph) or a device list (MultiGraph).
template <class E>
graphdsl::interp::RunResult run_entries(const graphdsl::sema::AnnotatedProgram& program,
                                        const E& graph, const graphdsl::interp::ArgMap& args) {
    using namespace graphdsl;
    using interp::PropArray;
    using interp::ScalarCell;
    interp::RunResult res;
    const std::string& entry = program.entry().name;
    const int32_t n = graph.nodeCount();
    auto put_prop = [&](const char* name, ast::TypeKind kind, auto&& fill) {
        const int id = sym(program, name);
        if (id < 0) return;
        PropArray a;
        a.elem = kind;
        fill(a);
        res.properties[id] = std::move(a);
    };
    auto put_scalar = [&](const char* name, ast::TypeKind kind, int64_t i, double f, uint8_t b) {
        const int id = sym(program, name);
        if (id < 0) return;
        ScalarCell c;
        c.type = kind;
        c.i = i;
        c.f = f;
        c.b = b;
        res.scalars[id] = c;
    };
    if (entry == "ComputeSSSP") {
        const int32_t src = node_arg(as_int(scalar_arg(args, "src")), n);
        std::vector<int64_t> dist(n);
        check(graph.sssp(src, dist.data()));
        put_prop("dist", ast::TypeKind::Int, [&](PropArray& a) { a.ints = std::move(dist); });
        put_prop("modified", ast::TypeKind::Bool, [&](PropArray& a) { a.bools.assign(n, 0); });
        put_scalar("finished", ast::TypeKind::Bool, 0, 0.0, 1);
    } else if (entry == "ComputePR") {
        const double damping = as_float(scalar_arg(args, "damping"));
        const double threshold = as_float(scalar_arg(args, "threshold"));
        int64_t mi = as_int(scalar_arg(args, "maxIter"));
        mi = std::min<int64_t>(std::max<int64_t>(mi, std::numeric_limits<int32_t>::min()),
                               std::numeric_limits<int32_t>::max());
        std::vector<double> rank(n);
        int32_t rounds = 0;
        check(graph.pagerank(damping, threshold, static_cast<int32_t>(mi), rank.data(), &rounds));
        put_prop("rankNext", ast::TypeKind::Float, [&](PropArray& a) { a.floats = rank; });
        put_prop("rank", ast::TypeKind::Float, [&](PropArray& a) { a.floats = std::move(rank); });
        put_prop("settled", ast::TypeKind::Bool, [&](PropArray& a) { a.bools.assign(n, 1); });
        put_scalar("iter", ast::TypeKind::Int, rounds, 0.0, 0);
        put_scalar("converged", ast::TypeKind::Bool, 0, 0.0, 1);
        put_scalar("numNodes", ast::TypeKind::Float, 0, static_cast<double>(n), 0);
    } else if (entry == "ComputeTC") {
        int64_t count = 0;
        check(graph.tc(&count));
        put_scalar("triangleCount", ast::TypeKind::Long, count, 0.0, 0);
        res.returnValue = interp::Value::ofInt(count);
    } else if (entry == "ComputeBC") {
        auto it = args.find("sourceSet");
        if (it == args.end() || !std::holds_alternative<std::vector<int32_t>>(it->second))
            rt("missing node-set argument 'sourceSet' (pass --arg sourceSet=v0,v1,...)");
        const auto& src = std::get<std::vector<int32_t>>(it->second);
        for (int32_t v : src) node_arg(v, n);
        std::vector<double> bc(n);
        check(graph.bc(src.data(), static_cast<int32_t>(src.size()), bc.data()));
        put_prop("bc", ast::TypeKind::Float, [&](PropArray& a) { a.floats = std::move(bc); });
    } else {
        throw CompileError("UnsupportedConstruct", program.entry().span,
                           "entry '" + entry + "' is not a B200 corpus entry point");
    }
    return res;
}
}  // namespace detail

inline graphdsl::interp::RunResult run(const graphdsl::sema::AnnotatedProgram& program,
                                       const DeviceGraph& graph,
                                       const graphdsl::interp::ArgMap& args) {
    return detail::run_entries(program, graph, args);
}

// Several GPUs from this process (gdx_context; SURVEY.md 8(e) partitions):
// peer access between every pair and one NCCL communicator per distinct
// device.  An ExecMode::Device with a device list.
class MultiDevice {
public:
    explicit MultiDevice(const std::vector<int>& devices) {
        detail::check(gdx_context_create(static_cast<int>(devices.size()), devices.data(), &c_));
    }
    ~MultiDevice() {
        if (c_) gdx_context_destroy(c_);
    }
    MultiDevice(const MultiDevice&) = delete;
    MultiDevice& operator=(const MultiDevice&) = delete;
    gdx_context* get() const { return c_; }

private:
    gdx_context* c_ = nullptr;
};

// A CsrGraph replicated on every device of a MultiDevice.
class MultiGraph {
public:
    template <class Csr>
    MultiGraph(const MultiDevice& ctx, const Csr& g) : n_(g.nodeCount()) {
        gdx_csr_view v{};
        v.n = g.nodeCount();
        v.m = g.edgeCount();
        v.directed = g.directed() ? 1 : 0;
        v.offsets = g.offsets().data();
        v.dests = g.dests().data();
        v.weights = g.weights().data();
        v.rev_offsets = g.revOffsets().data();
        v.rev_srcs = g.revSrcs().data();
        v.rev_eid = g.revEid().data();
        detail::check(gdx_multi_graph_create(ctx.get(), &v, &h_));
    }
    ~MultiGraph() {
        if (h_) gdx_multi_graph_destroy(h_);
    }
    MultiGraph(const MultiGraph&) = delete;
    MultiGraph& operator=(const MultiGraph&) = delete;
    int32_t nodeCount() const { return n_; }
    int sssp(int32_t src, int64_t* out) const { return gdx_sssp_multi(h_, src, out, nullptr); }
    int pagerank(double d, double t, int32_t mi, double* out, int32_t* rounds) const {
        return gdx_pagerank_multi(h_, d, t, mi, out, rounds, nullptr);
    }
    int tc(int64_t* out) const { return gdx_tc_multi(h_, out, nullptr); }
    int bc(const int32_t* s, int32_t k, double* out) const {
        return gdx_bc_multi(h_, s, k, out, nullptr);
    }

private:
    gdx_multi_graph* h_ = nullptr;
    int32_t n_ = 0;
};

inline graphdsl::interp::RunResult run(const graphdsl::sema::AnnotatedProgram& program,
                                       const MultiGraph& graph,
                                       const graphdsl::interp::ArgMap& args) {
    return detail::run_entries(program, graph, args);
}

// interp::run-shaped overload: uploads the graph for this call.
template <class Csr>
graphdsl::interp::RunResult run(const graphdsl::sema::AnnotatedProgram& program, const Csr& graph,
                                const graphdsl::interp::ArgMap& args, int device = 0) {
    DeviceGraph dg(graph, device);
    return run(program, dg, args);
}

// interp::run-shaped overload over a device list (uploads a replica per device).
template <class Csr>
graphdsl::interp::RunResult run(const graphdsl::sema::AnnotatedProgram& program, const Csr& graph,
                                const graphdsl::interp::ArgMap& args,
                                const std::vector<int>& devices) {
    MultiDevice ctx(devices);
    MultiGraph mg(ctx, graph);
    return run(program, mg, args);
}

}  // namespace gdx_graphdsl
