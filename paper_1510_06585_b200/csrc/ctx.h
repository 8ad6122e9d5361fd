// ctx.h — the context and future objects of libmarrow and the executor
// helpers shared by exec.cpp (runs, futures, monitoring), graph.cpp (CUDA
// graph capture / replay) and profile.cpp (Alg. 1 profile building, the
// Fig. 5 managed runs, device classes).  Internal; the ABI is marrow.h.
#pragma once
#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "comm.h"
#include "marrow.h"
#include "mw_kernels.h"
#include "sct.h"

namespace mw {
const char* last_error_cstr();
}

#define CUDA_OK(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? MW_E_OOM : MW_E_CUDA,         \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    } while (0)
#define MW_OK_OR_RETURN(expr)          \
    do {                               \
        mw_status s_ = (expr);         \
        if (s_ != MW_OK) return s_;    \
    } while (0)

namespace mwx {

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

constexpr int kStageSlots = 3;

}  // namespace mwx

struct mw_ctx {
    int device = 0, rank = 0, nranks = 1, ppr = 1, P = 1;
    std::unique_ptr<mwc::Comm> comm;   // NCCL, or the test-only loopback (comm.h)
    mw_alloc_fns alloc{};
    bool has_alloc = false;
    std::vector<double> dist;
    std::map<std::string, mwx::Buf> scratch;
    // one-partition plane loop: the (S0, S1, K, flags, rows, wp) whose zero halo
    // rows and loop flags are in place (the loop kernel leaves flags ready for
    // the next run), so a repeated run enqueues no memsets
    std::vector<uintptr_t> planes_prep;
    std::vector<uintptr_t> planes_multi_prep;   // the same for the fused multi-partition loop
    // Scratch pointers baked into live CUDA graphs (refcount per pointer): a
    // buffer replaced by a larger one while a graph references it is parked in
    // `orphans` and freed with the last such graph (or at teardown).
    std::map<void*, int> graph_refs;
    std::vector<void*> orphans;
    std::vector<void*>* capture_bufs = nullptr;   // collects scratch used while capturing
    // FIFO of runs across streams: every run waits for the previous run's end
    // (a no-op on one stream) and records it (ctx scratch is shared by runs).
    cudaEvent_t last_run = nullptr;
    cudaStream_t last_stream = nullptr;
    bool have_last_run = false;
    // run pipelining (mw_ctx_set_run_pipelining): the byte ranges the previous
    // run read and wrote, to launch an independent next run without the
    // programmatic-dependent-launch wait
    bool pipelining = false;
    struct Ranges {
        std::vector<std::pair<uintptr_t, uintptr_t>> rd, wr;
        bool valid = false;
    } prev_io;
    bool staging_overlap = false;   // mw_ctx_set_staging_overlap
    // cross-rank fused hysteresis: this rank's barrier block (cudaMalloc:
    // IPC-exportable), peers' buffers opened through CUDA IPC (NCCL ranks)
    int* xblock = nullptr;
    std::map<std::string, void*> ipc_open;
    bool xr_broken = false;         // a cross-rank barrier timed out: per-pass path from now on
    cudaStream_t lane_s[3]{};       // extra capture lanes of mw_graph_capture_many
    cudaEvent_t lane_ev[4]{};
    // pinned host memory
    int32_t* h_flag = nullptr;   // 16 ints: [0] byte-stencil flag, [4..7] plane-pass ring
    cudaEvent_t lag_ev[4]{};
    std::vector<double*> res_free;
    std::vector<double*> res_pages;
    // monitoring
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Rec {
        int part;
        int cls;
        cudaEvent_t a, b;
        int64_t launches;
    };
    std::vector<Rec> recs;      // last run (mw_last_timings)
    bool stats_on = false;
    std::vector<Rec> stats;     // every run since mw_stats_enable (mw_kernel_stats)
    cudaEvent_t wall_a = nullptr, wall_b = nullptr;
    std::vector<int64_t> last_len;
    bool have_run = false;
    mw_balance_state bstate{};
    std::vector<float> slow;
    // device classes (NEXT-4 heterogeneous devices): class id and
    // relative performance per partition
    std::vector<int> cls;
    std::vector<double> relperf;
    // managed runs (Fig. 5): the (SCT, workload) of the previous
    // managed run, and its result still to be persisted in the KB
    std::string mkey;
    bool m_pending = false;
    const mw_node* m_root = nullptr;
    std::vector<int64_t> m_dims;
    int m_prov = MW_PROV_DERIVED;
    mw_kb* m_kb = nullptr;
    unsigned long long launches0 = 0;
    // host staging (NEXT-1 overlap)
    cudaStream_t copy_in = nullptr, copy_out = nullptr, aux = nullptr;
    cudaEvent_t st_in[mwx::kStageSlots]{}, st_comp[mwx::kStageSlots]{}, st_out[mwx::kStageSlots]{};
    cudaEvent_t st_start = nullptr;
    bool st_valid[mwx::kStageSlots]{};   // slot has a recorded st_out (possibly from an earlier run)
    bool capturing = false;     // inside mw_graph_capture: no timing events, no host syncs
    bool monitor = true;        // per-partition timing events (mw_ctx_set_monitoring)
    int refs = 1;               // the user's handle + outstanding futures and graphs
    bool destroyed = false;     // mw_ctx_destroy called; teardown at the last release
    // futures released while their run was still in flight: reclaimed once
    // their event completed (next mw_run) or at mw_ctx_destroy — releasing a
    // future never blocks the host, so a loop that drops each future keeps
    // the device fed
    std::deque<mw_future*> retired;    // in release order
    std::vector<cudaEvent_t> fut_ev;   // completion events of released futures, reused
    int tune[mwk::TUNE_COUNT];  // tuning knobs (mw_ctx_set_tuning)
};

struct mw_future {
    mw_ctx* ctx = nullptr;
    cudaEvent_t done = nullptr;
    double* res = nullptr;     // pinned slot (4 x 8 B): [0] reduced, [1] plane-loop {E, converged} int32
    bool has_reduce = false;
    bool plane_loop = false;
    int64_t plane_m = 1, plane_nb = 0;   // steps per body execution, max body executions
    bool plane_xr = false;               // cross-rank fused loop: state[3] < 0 = aborted
    bool plane_count = true;             // the plane state counts executions (a while-loop)
    double executions = 0.0;
    double converged = 1.0;
    bool waited = false;
    bool completed = false;    // a query or wait saw the run complete
    // MapReduce with a non-ADD merging function: per-partition partials (pinned)
    double* parts = nullptr;
    std::vector<char> part_active;
    int32_t merge_op = 0;
    mw_merge_fn merge_fn = nullptr;
    void* merge_user = nullptr;
};

namespace mwx {
using mw::fail;
using mw::Node;
using mw::Step;
using mw::StepKind;

// device memory of the ctx allocator (PyTorch's caching allocator in the
// binding); named scratch buffers grow on demand (kept while a live graph
// references them)
mw_status ctx_alloc(mw_ctx* c, size_t bytes, cudaStream_t s, void** out);
void ctx_free(mw_ctx* c, void* p);
mw_status scratch(mw_ctx* c, const std::string& name, size_t bytes, cudaStream_t s, void** out);
int64_t row_bytes(const mw_arg& a);
std::vector<mwk::RgbaProg> rgba_groups(const std::vector<mw::ChainOp>& ops);
std::vector<mwk::U8Prog> u8_groups(const std::vector<mw::ChainOp>& ops);
std::vector<mwk::SaxpyProg> saxpy_groups(const std::vector<mw::ChainOp>& ops);
// enqueue one execution of a tree (the body of mw_run)
mw_status run(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s, mw_future* f);
// runs of a ctx are FIFO across streams (lazy last-run event)
mw_status fifo_enter(mw_ctx* c, cudaStream_t s);
void fifo_exit(mw_ctx* c, cudaStream_t s);
// futures and graphs hold a reference on their ctx
void ctx_retain(mw_ctx* c);
void ctx_release(mw_ctx* c);
}  // namespace mwx
