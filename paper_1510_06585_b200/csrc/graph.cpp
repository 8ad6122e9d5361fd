// graph.cpp — CUDA-graph capture and replay of built trees (P:124-126:
// a built SCT receives repeated execution requests): mw_graph_capture[_many],
// with only the data dependencies between captured runs kept (independent
// runs of a scratch-free chain on parallel lanes).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"

using namespace mwx;

extern "C" {

// ------------------------------------------------------------ graphs
struct mw_graph {
    mw_ctx* ctx = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    mw_future f;          // result slot of the captured run
    int64_t kernels = 0;  // library kernels per replay
    std::vector<void*> bufs;   // ctx scratch the graph writes (kept alive while it lives)
    int lanes = 1;             // parallel capture lanes (independent runs)
};

// Runs of `root` on the nsets argument sets may execute concurrently when the
// tree is one fused Map/Pipeline chain that touches no ctx scratch and no set
// writes a byte another set reads or writes (data dependencies are the only
// order a replay must keep).
static bool sets_independent(const Node* root, const mw_arg* args, int nargs, int nsets) {
    mw_status st;
    const mw::NodeCache* nc = mw::plan_cached(root, &st);
    if (!nc || nc->prog.size() != 1) return false;
    const Step& s0 = nc->prog[0];
    if (s0.kind == StepKind::Saxpy) {
        if (saxpy_groups(s0.ops).size() != 1) return false;
    } else if (s0.kind == StepKind::Rgba) {
        if (rgba_groups(s0.ops).size() != 1) return false;
    } else if (s0.kind == StepKind::U8) {
        if (u8_groups(s0.ops).size() != 1) return false;
    } else {
        return false;
    }
    if (nargs != 2) return false;
    struct Range {
        uintptr_t a, b;
        bool w;
    };
    std::vector<std::vector<Range>> rs(nsets);
    for (int k = 0; k < nsets; ++k)
        for (int i = 0; i < nargs; ++i) {
            const mw_arg& x = args[(size_t)k * nargs + i];
            if (x.location != MW_LOC_DEVICE) return false;
            const uintptr_t a = reinterpret_cast<uintptr_t>(x.ptr);
            rs[k].push_back({a, a + (uintptr_t)(x.local_rows * row_bytes(x)), i == 1});
        }
    for (int j = 0; j < nsets; ++j)
        for (int k = j + 1; k < nsets; ++k)
            for (const Range& u : rs[j])
                for (const Range& v : rs[k])
                    if ((u.w || v.w) && u.a < v.b && v.a < u.b) return false;
    return true;
}

mw_status mw_graph_capture_many(mw_ctx* c, const mw_node* root, const mw_arg* args,
                                int32_t nargs, int32_t nsets, void* stream, mw_graph** out) {
    if (!c || !root || !out || (nargs > 0 && !args) || nsets < 1)
        return fail(MW_E_INVALID_SPEC, "NULL argument or nsets < 1");
    if (!stream) return fail(MW_E_INVALID_SPEC, "graph capture needs a non-default stream");
    if (c->destroyed) return fail(MW_E_STATE, "ctx was destroyed");
    CUDA_OK(cudaSetDevice(c->device));
    (void)cudaGetLastError();   // see mw_run
    std::unique_ptr<mw_graph> g(new mw_graph);
    g->ctx = c;
    g->f.ctx = c;
    MW_OK_OR_RETURN(fifo_enter(c, static_cast<cudaStream_t>(stream)));   // before capture begins
    CUDA_OK(cudaHostAlloc(&g->f.res, 32, cudaHostAllocDefault));
    memset(g->f.res, 0, 32);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned long long l0 = mwk::launch_count();
    CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    c->capturing = true;
    std::vector<void*> used;
    c->capture_bufs = &used;
    mw_status st = MW_OK;
    try {
        // independent runs: round-robin over `lanes` streams forked from and
        // joined back into the capture stream
        int lanes = std::min<int>(c->tune[mwk::TUNE_GRAPH_LANES], nsets);
        if (lanes > 1 && !sets_independent(reinterpret_cast<const Node*>(root), args, nargs, nsets)) lanes = 1;
        cudaStream_t ls[4] = {s, nullptr, nullptr, nullptr};
        for (int l = 1; l < lanes && st == MW_OK; ++l) {
            if (!c->lane_s[l - 1] &&
                cudaStreamCreateWithFlags(&c->lane_s[l - 1], cudaStreamNonBlocking) != cudaSuccess)
                st = fail(MW_E_CUDA, "lane stream");
            ls[l] = c->lane_s[l - 1];
        }
        for (int l = 0; l < lanes && st == MW_OK; ++l)
            if (!c->lane_ev[l] && cudaEventCreateWithFlags(&c->lane_ev[l], cudaEventDisableTiming) != cudaSuccess)
                st = fail(MW_E_CUDA, "lane event");
        if (lanes > 1 && st == MW_OK) {
            cudaEventRecord(c->lane_ev[0], s);
            for (int l = 1; l < lanes; ++l) cudaStreamWaitEvent(ls[l], c->lane_ev[0], 0);
        }
        for (int32_t k = 0; k < nsets && st == MW_OK; ++k) {
            g->f.has_reduce = false;
            g->f.plane_loop = false;
            st = run(c, reinterpret_cast<const Node*>(root), args + (size_t)k * nargs, nargs, ls[k % lanes],
                     &g->f);
        }
        if (lanes > 1)
            for (int l = 1; l < lanes; ++l) {
                cudaEventRecord(c->lane_ev[l], ls[l]);
                cudaStreamWaitEvent(s, c->lane_ev[l], 0);
            }
        g->lanes = lanes;
    } catch (...) {
        st = fail(MW_E_INVALID_SPEC, "internal error");
    }
    c->capturing = false;
    c->capture_bufs = nullptr;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (st != MW_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaFreeHost(g->f.res);
        if (st != MW_OK) return st;
        return fail(MW_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    }
    g->graph = graph;
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        cudaFreeHost(g->f.res);
        return fail(MW_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
    g->kernels = (int64_t)(mwk::launch_count() - l0);
    std::sort(used.begin(), used.end());
    used.erase(std::unique(used.begin(), used.end()), used.end());
    for (void* p : used) ++c->graph_refs[p];
    g->bufs = std::move(used);
    ctx_retain(c);
    *out = g.release();
    return MW_OK;
}

mw_status mw_graph_capture(mw_ctx* c, const mw_node* root, const mw_arg* args, int32_t nargs,
                           void* stream, mw_graph** out) {
    return mw_graph_capture_many(c, root, args, nargs, 1, stream, out);
}

mw_status mw_graph_launch(mw_graph* g, void* stream) {
    if (!g || !g->exec) return fail(MW_E_STATE, "invalid graph");
    CUDA_OK(cudaSetDevice(g->ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MW_OK_OR_RETURN(fifo_enter(g->ctx, s));
    CUDA_OK(cudaGraphLaunch(g->exec, s));
    fifo_exit(g->ctx, s);
    return MW_OK;
}

mw_status mw_graph_result(mw_graph* g, double* out, int32_t n) {
    if (!g || !out) return fail(MW_E_STATE, "invalid graph");
    g->f.waited = true;   // the caller synchronised the launch stream
    return mw_future_result(&g->f, out, n);
}

mw_status mw_graph_kernels(const mw_graph* g, int64_t* out) {
    if (!g || !out) return fail(MW_E_STATE, "invalid graph");
    *out = g->kernels;
    return MW_OK;
}

mw_status mw_graph_destroy(mw_graph* g) {
    if (!g) return fail(MW_E_STATE, "NULL graph");
    cudaSetDevice(g->ctx->device);
    cudaDeviceSynchronize();
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->f.res) cudaFreeHost(g->f.res);
    mw_ctx* c = g->ctx;
    for (void* p : g->bufs) {
        auto it = c->graph_refs.find(p);
        if (it == c->graph_refs.end() || --it->second > 0) continue;
        c->graph_refs.erase(it);
        auto o = std::find(c->orphans.begin(), c->orphans.end(), p);
        if (o != c->orphans.end()) {   // replaced while the graph lived: free it now
            c->orphans.erase(o);
            ctx_free(c, p);
        }
    }
    delete g;
    ctx_release(c);
    return MW_OK;
}

}  // extern "C"
