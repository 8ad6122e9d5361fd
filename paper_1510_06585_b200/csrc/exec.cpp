// exec.cpp — contexts, the partitioned executor, futures, monitoring and the
// NCCL plumbing of libmarrow.
//
// The executor realises the paper's SPMD locality-aware decomposition
// (P:296-338): the domain is cut into P partitions by the distribution vector
// (R13), every partition runs the whole fused plan on
// its slice, intermediates stay on the device, and the only data that moves
// between partitions is what a skeleton requires: hysteresis halo rows
// (Loop "global synchronization"), MapReduce chunk partials (merge
// "+"), N-body COPY re-replication and the loop
// condition.  Inside a rank those are device copies; between ranks
// they are NCCL collectives over NVLink.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>


#include "ctx.h"

using namespace mwx;

#define NCCL_OK(expr)                                                                   \
    do {                                                                                \
        ncclResult_t r_ = (expr);                                                       \
        if (r_ != ncclSuccess)                                                          \
            return fail(MW_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)

namespace mwx {

// ------------------------------------------------------------ memory
mw_status ctx_alloc(mw_ctx* c, size_t bytes, cudaStream_t s, void** out) {
    void* p = nullptr;
    if (bytes == 0) bytes = 256;
    if (c->has_alloc) {
        p = c->alloc.alloc(bytes, (void*)s, c->alloc.user);
        if (!p) return fail(MW_E_OOM, "allocator callback returned NULL for " + std::to_string(bytes) + " bytes");
    } else {
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess)
            return fail(MW_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    *out = p;
    return MW_OK;
}
void ctx_free(mw_ctx* c, void* p) {
    if (!p) return;
    if (c->has_alloc)
        c->alloc.free(p, c->alloc.user);
    else
        cudaFree(p);
}
mw_status scratch(mw_ctx* c, const std::string& name, size_t bytes, cudaStream_t s, void** out) {
    Buf& b = c->scratch[name];
    if (b.bytes < bytes) {
        if (b.p) {
            auto it = c->graph_refs.find(b.p);
            if (it != c->graph_refs.end() && it->second > 0) {
                c->orphans.push_back(b.p);   // a live graph still writes it
            } else if (c->capturing) {
                c->orphans.push_back(b.p);   // freeing is not capturable; freed at teardown
            } else {
                // every stream of the ctx may still use it (copy streams,
                // timings): drain them before the caching allocator may
                // hand the block to someone else
                for (cudaStream_t q : {s, c->copy_in, c->copy_out, c->aux})
                    if (q) cudaStreamSynchronize(q);
                ctx_free(c, b.p);
            }
        }
        b.p = nullptr;
        b.bytes = 0;
        // under capture the allocator must not touch the capturing stream
        MW_OK_OR_RETURN(ctx_alloc(c, bytes, c->capturing ? nullptr : s, &b.p));
        b.bytes = bytes;
    }
    if (c->capture_bufs) c->capture_bufs->push_back(b.p);
    *out = b.p;
    return MW_OK;
}

// ------------------------------------------------------------ timing
cudaEvent_t next_event(mw_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}
// Brackets one partition's kernels of one class with CUDA events on the
// launching stream (monitoring).
// `shared`: a further partition of a launch already timed by another
// PartTimer (several partitions in one launch): it feeds mw_last_timings but
// not the per-kernel-class statistics, which count each launch once.
struct PartTimer {
    mw_ctx* c;
    cudaStream_t s;
    int part, cls;
    bool shared;
    cudaEvent_t a;
    unsigned long long l0;
    PartTimer(mw_ctx* c_, cudaStream_t s_, int p, int cl, bool sh = false)
        : c(c_), s(s_), part(p), cls(cl), shared(sh) {
        a = nullptr;
        l0 = mwk::launch_count();
        if (c->capturing || !c->monitor) return;
        a = next_event(c);
        cudaEventRecord(a, s);
    }
    ~PartTimer() {
        if (c->capturing || !c->monitor) return;
        cudaEvent_t b = next_event(c);
        cudaEventRecord(b, s);
        mw_ctx::Rec r{part, cls, a, b, shared ? 0 : (int64_t)(mwk::launch_count() - l0)};
        c->recs.push_back(r);
        if (c->stats_on && !shared) c->stats.push_back(r);
    }
};
mwk::Launch launch_for(mw_ctx* c, cudaStream_t s, int part) {
    mwk::Launch L;
    L.stream = s;
    L.slow = c->slow[part];
    L.tune = c->tune;
    return L;
}
mw_status kerr(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        return fail(MW_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return MW_OK;
}

// ------------------------------------------------------------ argument binding
struct Bound {
    const mw_arg* a;
    int64_t row_bytes;  // bytes per outer unit
};
int64_t dt_size(int32_t dt) {
    switch (dt) {
        case MW_DT_U8: return 1;
        case MW_DT_F32: return 4;
        case MW_DT_F64: return 8;
        case MW_DT_I64: return 8;
    }
    return 0;
}
mw_status check_arg(const mw_arg& a, int idx, int32_t dtype, int ndim_min, int ndim_max,
                    int32_t mode, int64_t last_dim /* -1 any */) {
    std::string pre = "arg " + std::to_string(idx) + ": ";
    // a rank may hold no rows of a PARTITION argument (zero share): NULL is fine then
    if (!a.ptr && (a.mode == MW_COPY ? a.shape[0] : a.local_rows) != 0)
        return fail(MW_E_SHAPE_MISMATCH, pre + "NULL pointer");
    if (a.dtype != dtype) return fail(MW_E_SHAPE_MISMATCH, pre + "wrong dtype");
    if (a.ndim < ndim_min || a.ndim > ndim_max || a.ndim > 4)
        return fail(MW_E_SHAPE_MISMATCH, pre + "wrong number of dimensions");
    for (int d = 0; d < a.ndim; ++d)
        if (a.shape[d] < 0) return fail(MW_E_SHAPE_MISMATCH, pre + "negative extent");
    if (a.mode != mode)
        return fail(MW_E_SHAPE_MISMATCH, pre + (mode == MW_COPY ? "must be COPY (P:686-688)"
                                                                : "must be PARTITION"));
    if (last_dim >= 0 && a.shape[a.ndim - 1] != last_dim)
        return fail(MW_E_SHAPE_MISMATCH, pre + "wrong innermost extent");
    if (a.location != MW_LOC_DEVICE && a.location != MW_LOC_HOST)
        return fail(MW_E_SHAPE_MISMATCH, pre + "bad location");
    return MW_OK;
}
int64_t row_bytes(const mw_arg& a) {
    int64_t b = dt_size(a.dtype);
    for (int d = 1; d < a.ndim; ++d) b *= a.shape[d];
    return b;
}
bool same_shape(const mw_arg& a, const mw_arg& b) {
    if (a.ndim != b.ndim) return false;
    for (int d = 0; d < a.ndim; ++d)
        if (a.shape[d] != b.shape[d]) return false;
    return true;
}
// pointer to global outer row `row` of a PARTITION arg
template <typename T>
T* at_row(const mw_arg& a, int64_t row) {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(a.ptr) + (row - a.local_offset) * row_bytes(a));
}

// ------------------------------------------------------------ plan helpers
std::vector<mwk::RgbaProg> rgba_groups(const std::vector<mw::ChainOp>& ops) {
    // split into launches of <= kMaxOps pointwise ops; mirrors fold into the
    // source-column parity of their group and the key parity of earlier ops.
    std::vector<std::vector<mw::ChainOp>> groups(1);
    int cnt = 0;
    for (const auto& o : ops) {
        if (o.kind != mw::LeafKind::Mirror) {
            if (cnt == mwk::kMaxOps) {
                groups.emplace_back();
                cnt = 0;
            }
            ++cnt;
        }
        groups.back().push_back(o);
    }
    std::vector<mwk::RgbaProg> out;
    for (const auto& g : groups) {
        mwk::RgbaProg p{};
        int mirrors_after = 0;
        for (const auto& o : g)
            if (o.kind == mw::LeafKind::Mirror) ++mirrors_after;
        p.mirror = mirrors_after & 1;
        for (const auto& o : g) {
            if (o.kind == mw::LeafKind::Mirror) {
                --mirrors_after;
                continue;
            }
            int k = p.n++;
            if (o.kind == mw::LeafKind::GaussNoise) {
                // R1: K = lowbias32(seed ^ 0x9E3779B9)
                uint32_t v = (uint32_t)o.ia ^ 0x9E3779B9u;
                v ^= v >> 16; v *= 0x7feb352du; v ^= v >> 15; v *= 0x846ca68bu; v ^= v >> 16;
                p.kind[k] = mwk::RGBA_NOISE;
                p.key[k] = v;
                p.param[k] = (int32_t)o.ib;
            } else {
                p.kind[k] = mwk::RGBA_SOLARIZE;
                p.param[k] = (int32_t)o.ia;
            }
            p.key_mirror[k] = mirrors_after & 1;
        }
        out.push_back(p);
    }
    return out;
}
std::vector<mwk::U8Prog> u8_groups(const std::vector<mw::ChainOp>& ops) {
    std::vector<mwk::U8Prog> out(1);
    out[0] = mwk::U8Prog{};
    for (const auto& o : ops) {
        if (out.back().n == mwk::kMaxOps) out.push_back(mwk::U8Prog{});
        mwk::U8Prog& p = out.back();
        int k = p.n++;
        if (o.kind == mw::LeafKind::Segment) {
            p.kind[k] = mwk::U8_SEGMENT;
            p.lo[k] = (int32_t)o.ia;
            p.hi[k] = (int32_t)o.ib;
        } else {
            p.kind[k] = mwk::U8_FINALIZE;
        }
    }
    return out;
}
std::vector<mwk::SaxpyProg> saxpy_groups(const std::vector<mw::ChainOp>& ops) {
    std::vector<mwk::SaxpyProg> out(1);
    out[0] = mwk::SaxpyProg{};
    for (const auto& o : ops) {
        if (out.back().n == mwk::kMaxOps) out.push_back(mwk::SaxpyProg{});
        out.back().a[out.back().n++] = o.fa;
    }
    return out;
}

// A while-loop runs in steps (m per body execution, at most nb bodies); the
// body changed iff one of its steps did.  From the step count E_steps (the
// last changing step + 2 when a step changed nothing, else m x nb): the body
// executions the oracle's LoopWhileChanged reports, and whether it converged.
void body_execs(int64_t e_steps, bool step_conv, int64_t m, int64_t nb, double* E, bool* conv) {
    if (m <= 1) {
        *E = (double)e_steps;
        *conv = step_conv;
        return;
    }
    if (step_conv) {
        const int64_t last = e_steps - 2;   // -1: nothing ever changed
        const int64_t eb = (last < 0 ? -1 : last / m) + 2;
        if (eb <= nb) {
            *E = (double)eb;
            *conv = true;
            return;
        }
    }
    *E = (double)nb;
    *conv = false;
}

// ------------------------------------------------------------ run state
struct RunCtx {
    mw_ctx* c;
    cudaStream_t s;
    std::vector<int64_t> off, len;  // all P partitions
    int first;                      // this rank's first partition
    bool indep = false;             // the next launch may read ahead of the PDL wait (pipelining)
    int owner(int part) const { return part / c->ppr; }
    bool local(int part) const { return owner(part) == c->rank; }
};

// Launch a chain of RGBA groups over rows [r0, r0+n): src -> ... -> dst.
mw_status run_rgba(RunCtx& R, int part, const std::vector<mwk::RgbaProg>& progs,
                   const uint8_t* src, uint8_t* dst, int64_t rows, int64_t W, int64_t row0,
                   uint8_t* tmp0, uint8_t* tmp1, bool dep_wait = true) {
    mwk::Launch L = launch_for(R.c, R.s, part);
    L.slow = 1.0f;   // slowdown is applied by repetition (caller)
    L.dep_wait = dep_wait || progs.size() != 1;
    const uint8_t* in = src;
    for (size_t g = 0; g < progs.size(); ++g) {
        uint8_t* out = (g + 1 == progs.size()) ? dst : ((g & 1) ? tmp1 : tmp0);
        MW_OK_OR_RETURN(kerr(mwk::rgba_chain(progs[g], in, out, rows, W, row0, L), "rgba_chain"));
        in = out;
    }
    return MW_OK;
}

// ------------------------------------------------------------ exchange helpers
struct Halo {
    uint8_t* buf[2];  // two ping-pong buffers of (len+2) x pitch, halo row at 0
};

// Exchange `hr` boundary rows of `rb` bytes between neighbouring active
// partitions.  bufs[q] (local partition q) holds hr halo rows, len interior
// rows, hr halo rows; every active partition has len >= hr.
mw_status exchange_rows(RunCtx& R, const std::vector<uint8_t*>& bufs, int64_t hr, int64_t rb) {
    mw_ctx* c = R.c;
    const int P = c->P;
    std::vector<int> act;
    for (int p = 0; p < P; ++p)
        if (R.len[p] > 0) act.push_back(p);
    const int64_t n = hr * rb;
    bool group = false;
    mwk::CopyBatch cb;
    cb.n = 0;
    for (size_t i = 0; i + 1 < act.size(); ++i) {
        int a = act[i], b = act[i + 1];
        bool la = R.local(a), lb = R.local(b);
        if (!la && !lb) continue;
        uint8_t* abuf = la ? bufs[a - R.first] : nullptr;
        uint8_t* bbuf = lb ? bufs[b - R.first] : nullptr;
        uint8_t* a_last = la ? abuf + R.len[a] * rb : nullptr;        // a's last hr rows
        uint8_t* a_bhalo = la ? abuf + (R.len[a] + hr) * rb : nullptr;
        uint8_t* b_first = lb ? bbuf + n : nullptr;                    // b's first hr rows
        uint8_t* b_thalo = bbuf;
        if (la && lb) {
            for (int k = 0; k < 2; ++k) {
                if (cb.n == 32) {
                    MW_OK_OR_RETURN(kerr(mwk::copy_batch(cb, R.s), "copy_batch"));
                    cb.n = 0;
                }
                cb.src[cb.n] = k ? b_first : a_last;
                cb.dst[cb.n] = k ? a_bhalo : b_thalo;
                cb.bytes[cb.n++] = n;
            }
            continue;
        }
        if (!c->comm) return fail(MW_E_STATE, "cross-rank halo without a communicator");
        if (!group) {
            MW_OK_OR_RETURN(c->comm->group_start());
            group = true;
        }
        if (la) {
            int peer = R.owner(b);
            MW_OK_OR_RETURN(c->comm->send(a_last, n, peer, R.s));
            MW_OK_OR_RETURN(c->comm->recv(a_bhalo, n, peer, R.s));
        } else {
            int peer = R.owner(a);
            MW_OK_OR_RETURN(c->comm->send(b_first, n, peer, R.s));
            MW_OK_OR_RETURN(c->comm->recv(b_thalo, n, peer, R.s));
        }
    }
    if (group) MW_OK_OR_RETURN(c->comm->group_end());
    if (cb.n) MW_OK_OR_RETURN(kerr(mwk::copy_batch(cb, R.s), "copy_batch"));
    return MW_OK;
}

mw_status exchange_halos(RunCtx& R, std::vector<Halo>& H, int which, int64_t pitch) {
    std::vector<uint8_t*> bufs(H.size());
    for (size_t q = 0; q < H.size(); ++q) bufs[q] = H[q].buf[which];
    return exchange_rows(R, bufs, 1, pitch);
}

// ------------------------------------------------------------ cross-rank fused loop setup
// A device pointer as another rank can open it: the raw address (ranks in
// one process) and a CUDA IPC handle of its allocation + the offset in it.
struct XPtr {
    uint64_t raw, off;
    uint8_t h[64];
};
struct XRec {   // what a rank publishes before a cross-rank fused loop
    int32_t ok, nact;
    int64_t first_rows, last_rows;
    XPtr fs[2], ls[2], blk;   // first / last active partition's S0, S1; the barrier block
};
bool ipc_export(const void* p, XPtr* out) {
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<GetRange>(f);
    }();
    out->raw = reinterpret_cast<uint64_t>(p);
    CUdeviceptr base = 0;
    size_t size = 0;
    cudaIpcMemHandle_t h;
    if (!fn || fn(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS ||
        cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(out->h, &h, 64);
    out->off = reinterpret_cast<uint64_t>(p) - (uint64_t)base;
    return true;
}
void* ipc_import(mw_ctx* c, const XPtr& x) {
    const std::string key(reinterpret_cast<const char*>(x.h), 64);
    auto it = c->ipc_open.find(key);
    if (it == c->ipc_open.end()) {
        cudaIpcMemHandle_t h;
        memcpy(&h, x.h, 64);
        void* base = nullptr;
        if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            (void)cudaGetLastError();
            return nullptr;
        }
        it = c->ipc_open.emplace(key, base).first;
    }
    return static_cast<uint8_t*>(it->second) + x.off;
}

// Every rank publishes its boundary partitions' planes and its barrier block;
// the fused loop runs only when every rank can (no injected slowdown, <= 8
// active partitions, pointers reachable): *xr tells.  Collective.
mw_status xrank_setup(RunCtx& R, const std::vector<int>& act, const std::vector<uint8_t*> (&S)[2],
                      bool slowed, mwk::PlaneMultiHost* hm, bool* xr) {
    mw_ctx* c = R.c;
    *xr = false;
    const int n = c->nranks;
    const bool same = c->comm->same_process();
    if (!c->xblock) {   // nothing device-synchronising here: a peer's kernel may be spinning
        if (cudaMalloc(&c->xblock, mwk::kXBlockInts * sizeof(int)) != cudaSuccess) {
            (void)cudaGetLastError();
            c->xblock = nullptr;
        } else {
            CUDA_OK(cudaMemsetAsync(c->xblock, 0, mwk::kXBlockInts * sizeof(int), R.s));
        }
    }
    XRec me{};
    me.ok = !slowed && (int)act.size() <= mwk::kPlaneMaxParts && n <= mwk::kXRanks && c->xblock != nullptr;
    me.nact = (int)act.size();
    auto exp = [&](const void* p, XPtr* o) {
        if (same) {
            o->raw = reinterpret_cast<uint64_t>(p);
            return true;
        }
        return ipc_export(p, o);
    };
    if (me.ok && !act.empty()) {
        const int qf = act.front(), ql = act.back();
        me.first_rows = R.len[R.first + qf];
        me.last_rows = R.len[R.first + ql];
        for (int b = 0; b < 2; ++b) {
            me.ok &= exp(S[b][qf], &me.fs[b]);
            me.ok &= exp(S[b][ql], &me.ls[b]);
        }
    }
    if (me.ok) me.ok &= exp(c->xblock, &me.blk);
    void* d;
    MW_OK_OR_RETURN(scratch(c, "xrank_recs", (size_t)n * sizeof(XRec) + sizeof(int), R.s, &d));
    XRec* drec = static_cast<XRec*>(d);
    std::vector<XRec> all(n);
    CUDA_OK(cudaMemcpyAsync(drec + c->rank, &me, sizeof me, cudaMemcpyHostToDevice, R.s));
    MW_OK_OR_RETURN(c->comm->allgather(drec + c->rank, drec, sizeof(XRec), R.s));
    CUDA_OK(cudaMemcpyAsync(all.data(), drec, (size_t)n * sizeof(XRec), cudaMemcpyDeviceToHost, R.s));
    CUDA_OK(cudaStreamSynchronize(R.s));
    bool all_ok = true;
    for (const XRec& r : all) all_ok &= r.ok != 0;
    if (!all_ok) return MW_OK;
    // open the peers' pointers; every rank must succeed (second agreement)
    auto imp = [&](int r, const XPtr& x) -> void* {
        if (same || r == c->rank) return reinterpret_cast<void*>(x.raw);
        return ipc_import(c, x);
    };
    int ok2 = 1;
    int prev = -1, next = -1;
    for (int r = c->rank - 1; r >= 0 && prev < 0; --r)
        if (all[r].nact > 0) prev = r;
    for (int r = c->rank + 1; r < n && next < 0; ++r)
        if (all[r].nact > 0) next = r;
    for (int r = 0; r < n; ++r) {
        hm->xbar[r] = static_cast<int*>(imp(r, all[r].blk));
        ok2 &= hm->xbar[r] != nullptr;
    }
    if (!act.empty() && prev >= 0) {
        hm->remote_prev = true;
        hm->rprev_rows = all[prev].last_rows;
        for (int b = 0; b < 2; ++b) {
            hm->rprev_S[b] = static_cast<uint32_t*>(imp(prev, all[prev].ls[b]));
            ok2 &= hm->rprev_S[b] != nullptr;
        }
    }
    if (!act.empty() && next >= 0) {
        hm->remote_next = true;
        for (int b = 0; b < 2; ++b) {
            hm->rnext_S[b] = static_cast<uint32_t*>(imp(next, all[next].fs[b]));
            ok2 &= hm->rnext_S[b] != nullptr;
        }
    }
    int* dok = reinterpret_cast<int*>(drec + n);
    CUDA_OK(cudaMemcpyAsync(dok, &ok2, sizeof ok2, cudaMemcpyHostToDevice, R.s));
    MW_OK_OR_RETURN(c->comm->allreduce(dok, 1, mwc::DType::I32, mwc::ROp::Min, R.s));
    CUDA_OK(cudaMemcpyAsync(&ok2, dok, sizeof ok2, cudaMemcpyDeviceToHost, R.s));
    CUDA_OK(cudaStreamSynchronize(R.s));
    if (!ok2) return MW_OK;
    hm->rank = c->rank;
    hm->nranks = n;
    hm->grid_div = same ? n : 1;   // loopback ranks share the GPU
    *xr = true;
    return MW_OK;
}

// ------------------------------------------------------------ bit planes, several partitions
// [u8 chain ending with the threshold] -> stencil loop -> [u8 chain] over P
// partitions (this rank's ppr of them).  Each partition's planes carry T halo
// rows; a pass of T executions runs per partition (one launch each), then T
// plane rows are exchanged with the neighbours (device copies on this rank,
// NCCL send/recv across ranks) and, for a while-loop, the last changing
// execution is reduced (atomicMax on the device, NCCL max across ranks) and
// read on the host: the loop stops after the first pass whose final execution
// changed nothing, with E = last + 2 exactly as in the one-partition kernel.
mw_status run_planes_multi(RunCtx& R, const std::vector<Step>& prog, const mw_arg& src,
                           const mw_arg& dst, mw_future* f) {
    mw_ctx* c = R.c;
    const int ppr = c->ppr;
    const int64_t W = row_bytes(src);
    const int64_t wp = mwk::plane_words(W);
    const int64_t rb = wp * 4;
    const Step& st = prog[1];
    const bool is_while = st.kind == StepKind::StencilWhile;
    int64_t min_len = INT64_MAX;
    for (int p = 0; p < c->P; ++p)
        if (R.len[p] > 0) min_len = std::min(min_len, R.len[p]);
    const int T = mwk::planes_pass_depth(c->tune[mwk::TUNE_HYST_T], min_len);
    auto pre = u8_groups(prog[0].ops);
    if (pre.size() != 1) return fail(MW_E_UNSUPPORTED, "chain before the loop > 16 ops");
    mwk::U8Prog post{};
    if (prog.size() == 3) {
        auto g = u8_groups(prog[2].ops);
        if (g.size() != 1) return fail(MW_E_UNSUPPORTED, "chain after the loop > 16 ops");
        post = g[0];
    }
    std::vector<uint8_t*> S[2], K;
    std::vector<uint8_t*> fl(ppr, nullptr);
    std::vector<int> top(ppr, 0), bot(ppr, 0);
    for (int b = 0; b < 2; ++b) S[b].assign(ppr, nullptr);
    K.assign(ppr, nullptr);
    void* lp;
    MW_OK_OR_RETURN(scratch(c, "planes_last", 64, R.s, &lp));
    int* d_last = static_cast<int*>(lp);
    // (buffers, lengths, T, W) of the partitions: when equal to the last FUSED
    // run's, the image-edge halo rows are still zero and the fused loop left
    // its flags ready, so the run enqueues no memsets
    std::vector<uintptr_t> key = {(uintptr_t)d_last, (uintptr_t)T, (uintptr_t)W};
    const bool fused_path = (c->nranks == 1 && c->tune[mwk::TUNE_HYST_FUSED] != 0) ||
                            (c->nranks > 1 && c->comm && c->tune[mwk::TUNE_HYST_FUSED] != 0 && !c->xr_broken &&
                             !c->capturing);
    bool prepared = false;
    for (int pass2 = 0; pass2 < 2; ++pass2) {   // pass 0: buffers -> key; pass 1: memsets if needed
    if (pass2 == 1) {
        prepared = fused_path && c->planes_multi_prep == key;
        c->planes_multi_prep.clear();
        if (!prepared) CUDA_OK(cudaMemsetAsync(d_last, 0, 64, R.s));   // d_last[4..6]: unpack state (buffer 0)
    }
    for (int q = 0; q < ppr; ++q) {
        const int p = R.first + q;
        const int64_t len = R.len[p];
        if (len == 0) continue;
        const size_t pb = (size_t)(len + 2 * T) * rb;
        void* v;
        const std::string sq = std::to_string(q);
        MW_OK_OR_RETURN(scratch(c, "mplane_s0_" + sq, pb, R.s, &v));
        S[0][q] = static_cast<uint8_t*>(v);
        MW_OK_OR_RETURN(scratch(c, "mplane_s1_" + sq, pb, R.s, &v));
        S[1][q] = static_cast<uint8_t*>(v);
        MW_OK_OR_RETURN(scratch(c, "mplane_k_" + sq, pb, R.s, &v));
        K[q] = static_cast<uint8_t*>(v);
        MW_OK_OR_RETURN(scratch(c, "mplane_tf_" + sq, (size_t)(2 * mwk::planes_tiles(len, W)), R.s, &v));
        fl[q] = static_cast<uint8_t*>(v);
        top[q] = bot[q] = 0;
        for (int a = 0; a < p; ++a) top[q] |= R.len[a] > 0;
        for (int a = p + 1; a < c->P; ++a) bot[q] |= R.len[a] > 0;
        if (pass2 == 0) {
            for (uint8_t* b : {S[0][q], S[1][q], K[q]}) key.push_back((uintptr_t)b);
            key.insert(key.end(), {(uintptr_t)q, (uintptr_t)len, (uintptr_t)top[q], (uintptr_t)bot[q]});
            continue;
        }
        // halo rows outside the image stay 0; the others are filled by the
        // exchanges (K, S0 below; S1 by the first pass) before they are read
        if (!prepared)
            for (uint8_t* b : {S[0][q], S[1][q], K[q]}) {
                if (!top[q]) CUDA_OK(cudaMemsetAsync(b, 0, T * rb, R.s));
                if (!bot[q]) CUDA_OK(cudaMemsetAsync(b + (len + T) * rb, 0, T * rb, R.s));
            }
    }
    }
    std::vector<int> act;
    bool slowed = false;
    for (int q = 0; q < ppr; ++q) {
        if (R.len[R.first + q] > 0) act.push_back(q);
        slowed |= c->slow[R.first + q] > 1.0f;
    }
    // Without an injected slowdown the packs (unpacks) of all local partitions
    // are one launch (blockIdx.y = partition); the launch is every active
    // partition's compute time (they run concurrently inside it).
    const bool batched = !slowed && !act.empty() && (int)act.size() <= mwk::kPlaneMaxParts;
    auto timers_all = [&](int cls) {
        std::vector<std::unique_ptr<PartTimer>> t;
        for (int q : act) t.emplace_back(new PartTimer(c, R.s, R.first + q, cls, !t.empty()));
        return t;
    };
    auto close_timers = [](std::vector<std::unique_ptr<PartTimer>>& t) {
        while (!t.empty()) t.pop_back();   // closing events in reverse order
    };
    auto io_of = [&]() {
        mwk::PlaneIO io{};
        io.np = (int)act.size();
        io.sp = W;
        for (int i = 0; i < io.np; ++i) {
            const int q = act[i], p = R.first + q;
            io.src[i] = at_row<const uint8_t>(src, R.off[p]);
            io.dst[i] = at_row<uint8_t>(dst, R.off[p]);
            io.S0[i] = reinterpret_cast<uint32_t*>(S[0][q]);
            io.S1[i] = reinterpret_cast<uint32_t*>(S[1][q]);
            io.K[i] = reinterpret_cast<uint32_t*>(K[q]);
            io.rows[i] = R.len[p];
        }
        return io;
    };
    if (batched) {
        auto t = timers_all(MW_KC_U8);
        MW_OK_OR_RETURN(kerr(mwk::planes_pack_io(pre[0], io_of(), W, launch_for(c, R.s, R.first), T),
                             "planes_pack"));
        close_timers(t);
    } else {
        for (int q : act) {
            const int p = R.first + q;
            PartTimer t(c, R.s, p, MW_KC_U8);
            MW_OK_OR_RETURN(kerr(mwk::planes_pack(pre[0], at_row<const uint8_t>(src, R.off[p]), W, R.len[p],
                                                  W, reinterpret_cast<uint32_t*>(S[0][q]),
                                                  reinterpret_cast<uint32_t*>(K[q]), launch_for(c, R.s, p), T),
                                 "planes_pack"));
        }
    }
    MW_OK_OR_RETURN(exchange_rows(R, K, T, rb));
    MW_OK_OR_RETURN(exchange_rows(R, S[0], T, rb));
    // One rank, <= kPlaneMaxParts active partitions, no injected slowdown:
    // the whole loop is one cooperative kernel over all partitions, halos
    // exchanged inside it (stores into the neighbours' halo rows) and the loop
    // condition decided on the device — no per-pass launches, copies or host
    // reads.
    // Several ranks: the same kernel on every rank, its halo stores going
    // straight into the neighbouring ranks' planes (NVLink peer memory / the
    // same device for loopback ranks) and a rank barrier per pass that also
    // all-reduces the loop condition — one launch per rank for the whole
    // loop, no per-pass transport calls or host reads.
    mwk::PlaneMultiHost hm{};
    bool xr = false;
    if (c->nranks > 1 && c->comm && c->tune[mwk::TUNE_HYST_FUSED] != 0 && !c->xr_broken && !c->capturing)
        MW_OK_OR_RETURN(xrank_setup(R, act, S, slowed, &hm, &xr));
    if (xr || (c->nranks == 1 && batched && c->tune[mwk::TUNE_HYST_FUSED] != 0)) {
        hm.np = (int)act.size();
        hm.wp = wp;
        for (int i = 0; i < hm.np; ++i) {
            const int q = act[i];
            hm.S0[i] = reinterpret_cast<uint32_t*>(S[0][q]);
            hm.S1[i] = reinterpret_cast<uint32_t*>(S[1][q]);
            hm.K[i] = reinterpret_cast<const uint32_t*>(K[q]);
            hm.fl[i] = fl[q];
            hm.fl_bytes[i] = 2 * mwk::planes_tiles(R.len[R.first + q], W);
            hm.rows[i] = R.len[R.first + q];
        }
        {
            int64_t words = 1;
            for (int i = 0; i < hm.np; ++i) words += mwk::planes_tiles(hm.rows[i], W);
            void* av;
            MW_OK_OR_RETURN(scratch(c, "mplane_act", (size_t)words * 4, R.s, &av));
            hm.act = static_cast<uint32_t*>(av);
            hm.act_words = words;
        }
        int* state = d_last + 4;   // {E, converged, final buffer, abort}: read by the unpack
        int* pflags = d_last + 8;
        if (!prepared) CUDA_OK(cudaMemsetAsync(pflags, 0xFF, 3 * sizeof(int), R.s));
        {
            auto t = timers_all(MW_KC_STENCIL);
            mwk::Launch L = launch_for(c, R.s, R.first);
            if (xr) L.slow = 1.0f;   // every rank's grid is sized for co-residency
            MW_OK_OR_RETURN(kerr(mwk::planes_multi(hm, T, st.n, pflags, state, L), "planes_multi"));
            close_timers(t);
        }
        if (xr) MW_OK_OR_RETURN(c->comm->launch_barrier());
        if (!act.empty()) {
            auto t = timers_all(MW_KC_U8);
            MW_OK_OR_RETURN(kerr(mwk::planes_unpack_io(post, io_of(), state, W, W, launch_for(c, R.s, R.first), T),
                                 "planes_unpack"));
            close_timers(t);
        }
        c->planes_multi_prep = key;
        if (is_while || xr) {
            CUDA_OK(cudaMemcpyAsync(f->res + 1, state, 16, cudaMemcpyDeviceToHost, R.s));
            f->plane_loop = true;
            f->plane_xr = xr;
            f->plane_m = st.m;
            f->plane_nb = st.n / st.m;
            f->plane_count = is_while;
        }
        return MW_OK;
    }
    if (prepared) CUDA_OK(cudaMemsetAsync(d_last, 0, 64, R.s));   // skipped above for a fused run
    if (is_while && c->capturing)
        return fail(MW_E_UNSUPPORTED,
                    "this while-loop evaluates its condition on the host (several ranks or "
                    "partitions) and cannot be captured in a graph");
    // The host reads the (running-max) last changing execution LAG passes
    // behind the device, so the GPU never waits for it; passes queued after
    // the fixed point change nothing, so they cost only their boundary tiles.
    constexpr int LAG = 2, SLOTS = 4;
    const int64_t max_it = st.n;
    int cur = 0, pass = 0, slot = 0;
    int64_t k0 = 0, E = max_it;
    bool converged = false;
    struct Pending {
        int slot;
        int64_t end;
    };
    std::deque<Pending> inflight;
    if (is_while) {
        CUDA_OK(cudaMemsetAsync(d_last, 0xFF, sizeof(int), R.s));
        for (int i = 0; i < SLOTS; ++i)
            if (!c->lag_ev[i]) CUDA_OK(cudaEventCreateWithFlags(&c->lag_ev[i], cudaEventDisableTiming));
    }
    auto settled = [&](const Pending& x) {   // after cudaEventSynchronize(lag_ev[x.slot])
        const int64_t last = c->h_flag[4 + x.slot];
        if (last < x.end - 1) {   // that pass ended with an execution that changed nothing
            converged = true;
            E = last + 2;
        }
        return converged;
    };
    while (k0 < max_it) {
        const int steps = (int)std::min<int64_t>(T, max_it - k0);
        for (int q = 0; q < ppr; ++q) {
            const int p = R.first + q;
            if (R.len[p] == 0) continue;
            const int64_t nt = mwk::planes_tiles(R.len[p], W);
            PartTimer t(c, R.s, p, MW_KC_STENCIL);
            MW_OK_OR_RETURN(kerr(mwk::planes_pass(reinterpret_cast<const uint32_t*>(S[cur][q]),
                                                  reinterpret_cast<uint32_t*>(S[1 - cur][q]),
                                                  reinterpret_cast<const uint32_t*>(K[q]), R.len[p], W, T,
                                                  steps, k0, fl[q] + ((pass + 1) & 1) * nt,
                                                  fl[q] + (pass & 1) * nt, pass == 0, top[q], bot[q],
                                                  d_last, launch_for(c, R.s, p)),
                                 "planes_pass"));
        }
        cur = 1 - cur;
        ++pass;
        MW_OK_OR_RETURN(exchange_rows(R, S[cur], T, rb));
        k0 += steps;
        if (!is_while) continue;
        if (c->comm) MW_OK_OR_RETURN(c->comm->allreduce(d_last, 1, mwc::DType::I32, mwc::ROp::Max, R.s));
        CUDA_OK(cudaMemcpyAsync(c->h_flag + 4 + slot, d_last, sizeof(int32_t), cudaMemcpyDeviceToHost, R.s));
        CUDA_OK(cudaEventRecord(c->lag_ev[slot], R.s));
        inflight.push_back({slot, k0});
        slot = (slot + 1) % SLOTS;
        if ((int)inflight.size() > LAG) {
            const Pending x = inflight.front();
            inflight.pop_front();
            CUDA_OK(cudaEventSynchronize(c->lag_ev[x.slot]));
            if (settled(x)) break;
        }
    }
    while (is_while && !converged && !inflight.empty()) {
        const Pending x = inflight.front();
        inflight.pop_front();
        CUDA_OK(cudaEventSynchronize(c->lag_ev[x.slot]));
        settled(x);
    }
    if (is_while) {
        double eb;
        bool cv;
        body_execs(E, converged, st.m, st.n / st.m, &eb, &cv);
        f->executions += eb;
        if (!cv) f->converged = 0.0;
    }
    if (batched) {   // d_last[4..6] = 0: the unpack reads S0, here set to the final buffer
        mwk::PlaneIO io = io_of();
        for (int i = 0; i < io.np; ++i) io.S0[i] = reinterpret_cast<uint32_t*>(S[cur][act[i]]);
        auto t = timers_all(MW_KC_U8);
        MW_OK_OR_RETURN(kerr(mwk::planes_unpack_io(post, io, d_last + 4, W, W, launch_for(c, R.s, R.first), T),
                             "planes_unpack"));
        close_timers(t);
        return MW_OK;
    }
    for (int q = 0; q < ppr; ++q) {
        const int p = R.first + q;
        if (R.len[p] == 0) continue;
        const uint32_t* fin = reinterpret_cast<const uint32_t*>(S[cur][q]);
        PartTimer t(c, R.s, p, MW_KC_U8);
        MW_OK_OR_RETURN(kerr(mwk::planes_unpack(post, fin, fin, reinterpret_cast<const uint32_t*>(K[q]),
                                                d_last + 4, at_row<uint8_t>(dst, R.off[p]), W, R.len[p],
                                                W, launch_for(c, R.s, p), T),
                             "planes_unpack"));
    }
    return MW_OK;
}

// ------------------------------------------------------------ U8 programs (chains + stencils)
mw_status run_u8(RunCtx& R, const std::vector<Step>& prog, const mw_arg& src, const mw_arg& dst,
                 mw_future* f) {
    mw_ctx* c = R.c;
    const int ppr = c->ppr;
    const int64_t inner = row_bytes(src);  // bytes per outer row
    const bool has_stencil = std::any_of(prog.begin(), prog.end(), [](const Step& s) {
        return s.kind == StepKind::StencilFor || s.kind == StepKind::StencilWhile;
    });
    const int64_t W = inner;               // 2-D when a stencil is present (validated)
    const int64_t pitch = (W + 15) / 16 * 16;
    // ---- bit-plane path: one partition on this device, pattern
    //      [u8 chain ending with the threshold] -> stencil loop -> [u8 chain]
    {
        int sidx = -1, nst = 0;
        for (size_t i = 0; i < prog.size(); ++i)
            if (prog[i].kind == StepKind::StencilFor || prog[i].kind == StepKind::StencilWhile) {
                sidx = (int)i;
                ++nst;
            }
        const bool planes_on = c->tune[mwk::TUNE_HYST_PLANES] != 0;
        const int p0 = R.first;
        const bool pattern = planes_on && nst == 1 && sidx == 1 &&
                             prog[0].kind == StepKind::U8 && !prog[0].ops.empty() &&
                             prog[0].ops.back().kind == mw::LeafKind::Segment &&
                             (int)prog.size() <= 3 &&
                             (prog.size() == 2 || prog[2].kind == StepKind::U8);
        const bool eligible = pattern && c->nranks == 1 && ppr == 1 && R.len[p0] > 0;
        const bool any = std::any_of(R.len.begin(), R.len.end(), [](int64_t l) { return l > 0; });
        if (pattern && any && (c->nranks > 1 || ppr > 1))
            return run_planes_multi(R, prog, src, dst, f);
        if (eligible) {
            const int64_t rows = R.len[p0];
            const int64_t wp = mwk::plane_words(W);
            const size_t pb = (size_t)(rows + 2) * wp * 4;
            void *s0, *s1, *kk, *fl;
            MW_OK_OR_RETURN(scratch(c, "plane_s0", pb, R.s, &s0));
            MW_OK_OR_RETURN(scratch(c, "plane_s1", pb, R.s, &s1));
            MW_OK_OR_RETURN(scratch(c, "plane_k", pb, R.s, &kk));
            MW_OK_OR_RETURN(scratch(c, "plane_flags", 64, R.s, &fl));
            void* tf;
            MW_OK_OR_RETURN(scratch(c, "plane_act", (size_t)(4 * (mwk::planes_tiles(rows, W) + 1)), R.s, &tf));
            uint32_t* S0 = static_cast<uint32_t*>(s0);
            uint32_t* S1 = static_cast<uint32_t*>(s1);
            uint32_t* K = static_cast<uint32_t*>(kk);
            int* flags = static_cast<int*>(fl);
            int* state = flags + 4;
            const std::vector<uintptr_t> key = {(uintptr_t)S0, (uintptr_t)S1, (uintptr_t)K, (uintptr_t)flags,
                                                (uintptr_t)rows, (uintptr_t)wp};
            if (c->planes_prep != key) {
                // no kernel writes the halo rows, and the loop leaves its flags
                // at -1 for the next run: both are set up once per buffer set
                c->planes_prep.clear();
                for (uint32_t* b : {S0, S1, K}) {   // zero halo rows (outside the image = 0)
                    CUDA_OK(cudaMemsetAsync(b, 0, wp * 4, R.s));
                    CUDA_OK(cudaMemsetAsync(b + (rows + 1) * wp, 0, wp * 4, R.s));
                }
                CUDA_OK(cudaMemsetAsync(flags, 0xFF, 64, R.s));   // pass flags start at -1
            }
            auto pre = u8_groups(prog[0].ops);
            if (pre.size() != 1) return fail(MW_E_UNSUPPORTED, "chain before the loop > 16 ops");
            mwk::U8Prog post{};
            if (prog.size() == 3) {
                auto g = u8_groups(prog[2].ops);
                if (g.size() != 1) return fail(MW_E_UNSUPPORTED, "chain after the loop > 16 ops");
                post = g[0];
            }
            const mwk::Launch L = launch_for(c, R.s, p0);
            {
                PartTimer t(c, R.s, p0, MW_KC_U8);
                MW_OK_OR_RETURN(kerr(mwk::planes_pack(pre[0], at_row<const uint8_t>(src, R.off[p0]), inner,
                                                      rows, W, S0, K, L), "planes_pack"));
            }
            {
                PartTimer t(c, R.s, p0, MW_KC_STENCIL);
                MW_OK_OR_RETURN(kerr(mwk::planes_loop(S0, S1, K, rows, W, prog[1].n, flags, state,
                                                      static_cast<uint32_t*>(tf), L),
                                     "planes_loop"));
            }
            {
                PartTimer t(c, R.s, p0, MW_KC_U8);
                MW_OK_OR_RETURN(kerr(mwk::planes_unpack(post, S0, S1, K, state,
                                                        at_row<uint8_t>(dst, R.off[p0]), inner, rows, W, L),
                                     "planes_unpack"));
            }
            c->planes_prep = key;
            if (prog[1].kind == StepKind::StencilWhile) {
                CUDA_OK(cudaMemcpyAsync(f->res + 1, state, 8, cudaMemcpyDeviceToHost, R.s));
                f->plane_loop = true;
                f->plane_xr = false;
                f->plane_count = true;
                f->plane_m = prog[1].m;
                f->plane_nb = prog[1].n / prog[1].m;
            }
            return MW_OK;
        }
    }
    std::vector<Halo> H(ppr);
    if (has_stencil) {
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            for (int b = 0; b < 2; ++b) {
                void* ptr;
                MW_OK_OR_RETURN(scratch(c, "halo" + std::to_string(b) + "_" + std::to_string(q),
                                        (size_t)(R.len[p] + 2) * pitch, R.s, &ptr));
                H[q].buf[b] = static_cast<uint8_t*>(ptr);
                // zero halo rows and pad columns (out-of-image neighbours are 0, R11)
                CUDA_OK(cudaMemsetAsync(H[q].buf[b], 0, pitch, R.s));
                CUDA_OK(cudaMemsetAsync(H[q].buf[b] + (R.len[p] + 1) * pitch, 0, pitch, R.s));
                if (pitch > W)
                    CUDA_OK(cudaMemset2DAsync(H[q].buf[b] + pitch + W, pitch, 0, pitch - W,
                                              R.len[p], R.s));
            }
        }
    }
    // current location of the value, per local partition
    struct Loc {
        const uint8_t* p;
        int64_t pitch;
        int hb;  // -1: not a halo buffer, else which halo buffer holds it
    };
    std::vector<Loc> cur(ppr);
    for (int q = 0; q < ppr; ++q) {
        int p = R.first + q;
        cur[q] = {at_row<const uint8_t>(src, R.off[p]), inner, -1};
    }
    int32_t* d_last = nullptr;
    for (size_t si = 0; si < prog.size(); ++si) {
        const Step& st = prog[si];
        const bool last = si + 1 == prog.size();
        if (st.kind == StepKind::U8) {
            auto groups = u8_groups(st.ops);
            const bool next_stencil = !last && (prog[si + 1].kind == StepKind::StencilFor ||
                                                prog[si + 1].kind == StepKind::StencilWhile);
            for (int q = 0; q < ppr; ++q) {
                int p = R.first + q;
                if (R.len[p] == 0) continue;
                uint8_t* out;
                int64_t opitch;
                int hb = -1;
                if (last) {
                    out = at_row<uint8_t>(dst, R.off[p]);
                    opitch = inner;
                } else if (next_stencil) {
                    hb = cur[q].hb == 0 ? 1 : 0;
                    out = H[q].buf[hb] + pitch;
                    opitch = pitch;
                } else {
                    return fail(MW_E_UNSUPPORTED, "u8 chain followed by a non-stencil step");
                }
                PartTimer t(c, R.s, p, MW_KC_U8);
                mwk::Launch L = launch_for(c, R.s, p);
                // a one-step chain: the first launch may read ahead (pipelining), a
                // later partition's follows one that wrote other rows of dst only
                L.dep_wait = !(R.indep && prog.size() == 1 && groups.size() == 1 && !c->monitor);
                R.indep = prog.size() == 1 && groups.size() == 1;
                const uint8_t* in = cur[q].p;
                int64_t ipitch = cur[q].pitch;
                for (size_t g = 0; g < groups.size(); ++g) {
                    // multi-group chains (> 16 ops) run in place on the output rows
                    MW_OK_OR_RETURN(kerr(mwk::u8_chain(groups[g], in, ipitch, out, opitch, R.len[p], W, L),
                                         "u8_chain"));
                    in = out;
                    ipitch = opitch;
                }
                cur[q] = {out, opitch, hb};
            }
            continue;
        }
        // stencil loop
        const bool is_while = st.kind == StepKind::StencilWhile;
        if (!d_last) {
            void* ptr;
            MW_OK_OR_RETURN(scratch(c, "last_changed", sizeof(int32_t), R.s, &ptr));
            d_last = static_cast<int32_t*>(ptr);
        }
        int hb = 0;
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            if (cur[q].hb < 0)
                CUDA_OK(cudaMemcpy2DAsync(H[q].buf[0] + pitch, pitch, cur[q].p, cur[q].pitch, W,
                                          R.len[p], cudaMemcpyDeviceToDevice, R.s));
            else
                hb = cur[q].hb;
        }
        MW_OK_OR_RETURN(exchange_halos(R, H, hb, pitch));
        CUDA_OK(cudaMemsetAsync(d_last, 0xFF, sizeof(int32_t), R.s));  // -1
        // per-tile change flags (two generations) and neighbour presence
        std::vector<uint8_t*> flags(ppr, nullptr);
        std::vector<int> top_nbr(ppr, 0), bot_nbr(ppr, 0);
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            void* fp;
            int64_t nt = mwk::hyst_tiles(R.len[p], pitch);
            MW_OK_OR_RETURN(scratch(c, "hflags_" + std::to_string(q), (size_t)(2 * nt), R.s, &fp));
            flags[q] = static_cast<uint8_t*>(fp);
            for (int a = 0; a < p; ++a) top_nbr[q] |= R.len[a] > 0;
            for (int a = p + 1; a < c->P; ++a) bot_nbr[q] |= R.len[a] > 0;
        }
        const int64_t max_it = st.n;
        const int64_t ce = is_while ? std::max<int64_t>(1, st.check_every) * st.m : max_it;
        int64_t it = 0;
        bool converged = !is_while;
        int64_t E = 0;
        while (it < max_it) {
            const int64_t blk = std::min(ce, max_it - it);
            for (int64_t b = 0; b < blk; ++b, ++it) {
                for (int q = 0; q < ppr; ++q) {
                    int p = R.first + q;
                    if (R.len[p] == 0) continue;
                    const int64_t nt = mwk::hyst_tiles(R.len[p], pitch);
                    uint8_t* fcur = flags[q] + (it & 1) * nt;
                    const uint8_t* fprev = it == 0 ? nullptr : flags[q] + ((it + 1) & 1) * nt;
                    PartTimer t(c, R.s, p, MW_KC_STENCIL);
                    MW_OK_OR_RETURN(kerr(mwk::hyst_step(H[q].buf[hb], H[q].buf[1 - hb], R.len[p], pitch,
                                                        (int)it, d_last, fprev, fcur, top_nbr[q],
                                                        bot_nbr[q], launch_for(c, R.s, p)),
                                         "hyst_step"));
                }
                hb = 1 - hb;
                MW_OK_OR_RETURN(exchange_halos(R, H, hb, pitch));
            }
            if (!is_while) continue;
            if (c->capturing)
                return fail(MW_E_UNSUPPORTED,
                            "this while-loop evaluates its condition on the host (multi-partition "
                            "byte stencil) and cannot be captured in a graph");
            // loop condition (P:376 stage 1), reduced over ranks on the device
            if (c->comm)
                MW_OK_OR_RETURN(c->comm->allreduce(d_last, 1, mwc::DType::I32, mwc::ROp::Max, R.s));
            CUDA_OK(cudaMemcpyAsync(c->h_flag, d_last, sizeof(int32_t), cudaMemcpyDeviceToHost, R.s));
            CUDA_OK(cudaStreamSynchronize(R.s));
            const int64_t lastc = *c->h_flag;
            if (lastc < it - 1) {  // iteration it-1 changed nothing: fixed point reached
                converged = true;
                E = lastc + 2;
                break;
            }
        }
        if (is_while) {
            if (!converged) E = max_it;
            double eb;
            bool cv;
            body_execs(E, converged, st.m, st.n / st.m, &eb, &cv);
            f->executions += eb;
            if (!cv) f->converged = 0.0;
        }
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            cur[q] = {H[q].buf[hb] + pitch, pitch, hb};
        }
        if (last) {
            for (int q = 0; q < ppr; ++q) {
                int p = R.first + q;
                if (R.len[p] == 0) continue;
                CUDA_OK(cudaMemcpy2DAsync(at_row<uint8_t>(dst, R.off[p]), inner, cur[q].p, pitch, W,
                                          R.len[p], cudaMemcpyDeviceToDevice, R.s));
            }
        }
    }
    if (prog.empty()) {
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            CUDA_OK(cudaMemcpyAsync(at_row<uint8_t>(dst, R.off[p]), cur[q].p, R.len[p] * inner,
                                    cudaMemcpyDeviceToDevice, R.s));
        }
    }
    return MW_OK;
}

// ------------------------------------------------------------ N-body
mw_status allgather_slices(RunCtx& R, float4* buf) {
    mw_ctx* c = R.c;
    if (c->nranks == 1) return MW_OK;
    MW_OK_OR_RETURN(c->comm->group_start());
    for (int r = 0; r < c->nranks; ++r) {
        int p0 = r * c->ppr, p1 = p0 + c->ppr - 1;
        int64_t o = R.off[p0], n = R.off[p1] + R.len[p1] - o;
        if (n == 0) continue;
        // allgather-v: one broadcast per root over its contiguous slice (in place)
        MW_OK_OR_RETURN(c->comm->broadcast(buf + o, (size_t)n * sizeof(float4), r, R.s));
    }
    MW_OK_OR_RETURN(c->comm->group_end());
    return MW_OK;
}

mw_status run_nbody(RunCtx& R, const Step& st, const mw_arg& pos, const mw_arg& vel) {
    mw_ctx* c = R.c;
    const int64_t N = pos.shape[0];
    void *p2, *v2;
    MW_OK_OR_RETURN(scratch(c, "nbody_pos", (size_t)N * 16, R.s, &p2));
    MW_OK_OR_RETURN(scratch(c, "nbody_vel", (size_t)N * 16, R.s, &v2));
    float4* P[2] = {static_cast<float4*>(pos.ptr), static_cast<float4*>(p2)};
    float4* V[2] = {static_cast<float4*>(vel.ptr), static_cast<float4*>(v2)};
    int cur = 0;
    for (int64_t it = 0; it < st.n; ++it) {
        for (int q = 0; q < c->ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            PartTimer t(c, R.s, p, MW_KC_NBODY);
            // The step kernel is idempotent (reads state k, writes state k+1), so the
            // slowdown injector repeats it `factor` times: time grows exactly by the
            // factor, as on a device that is that much slower (the grid clamp used for
            // the other kernels is not proportional once a partition no longer fills
            // the GPU).  Results are unchanged.
            mwk::Launch L = launch_for(c, R.s, p);
            const int reps = L.slow > 1.0f ? (int)std::lround(L.slow) : 1;
            L.slow = 1.0f;
            void* pp;
            MW_OK_OR_RETURN(scratch(c, "nbody_part", (size_t)mwk::nbody_part_doubles(R.len[p]) * 8, R.s, &pp));
            for (int rep = 0; rep < reps; ++rep)
                MW_OK_OR_RETURN(kerr(mwk::nbody(P[cur], V[cur], P[1 - cur], V[1 - cur], nullptr,
                                                R.off[p], R.len[p], N, st.eps2, st.dt, 0,
                                                static_cast<double*>(pp), L),
                                     "nbody"));
        }
        // Loop state update with global sync: re-replicate
        MW_OK_OR_RETURN(allgather_slices(R, P[1 - cur]));
        MW_OK_OR_RETURN(allgather_slices(R, V[1 - cur]));
        cur = 1 - cur;
    }
    if (cur == 1) {
        CUDA_OK(cudaMemcpyAsync(P[0], P[1], (size_t)N * 16, cudaMemcpyDeviceToDevice, R.s));
        CUDA_OK(cudaMemcpyAsync(V[0], V[1], (size_t)N * 16, cudaMemcpyDeviceToDevice, R.s));
    }
    return MW_OK;
}

// FFT chains (NEXT-3): groups of <= 32 stages per fft_chain call, the first
// reading src, later ones in place on dst.
mw_status run_fft_chain(mw_ctx* c, const std::vector<mw::ChainOp>& ops, const float* src, float* dst,
                        int64_t nfft, int log2n, mwk::Launch L) {
    if (const size_t wb = mwk::fft_work_bytes(nfft, log2n)) {
        MW_OK_OR_RETURN(scratch(c, "fft_work", wb, L.stream, &L.work));
        L.work_bytes = wb;
    }
    for (size_t g = 0; g < ops.size(); g += 32) {
        const int n = (int)std::min<size_t>(32, ops.size() - g);
        uint32_t inv = 0;
        for (int i = 0; i < n; ++i)
            if (ops[g + i].ib) inv |= 1u << i;
        MW_OK_OR_RETURN(kerr(mwk::fft_chain(g == 0 ? src : dst, dst, nfft, log2n, inv, n, L), "fft_chain"));
    }
    return MW_OK;
}

// ------------------------------------------------------------ host-staged chains (NEXT-1)
mw_status run_staged(RunCtx& R, const Step& st, int in_kind, const mw_arg* args) {
    mw_ctx* c = R.c;
    const mw_arg& a0 = args[0];
    const mw_arg& a1 = args[1];
    const int64_t rb = row_bytes(a0);
    if (!c->copy_in) {
        CUDA_OK(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
        for (int i = 0; i < kStageSlots; ++i) {
            CUDA_OK(cudaEventCreateWithFlags(&c->st_in[i], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&c->st_comp[i], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&c->st_out[i], cudaEventDisableTiming));
        }
        CUDA_OK(cudaEventCreateWithFlags(&c->st_start, cudaEventDisableTiming));
    }
    static const int64_t stage_bytes = [] {
        const char* v = getenv("MW_STAGE_MB");   // staging chunk (MiB); 32 measured best
        const int64_t mb = v ? atoll(v) : 32;
        return (mb > 0 ? mb : 32) << 20;
    }();
    const int64_t chunk_rows = std::max<int64_t>(1, stage_bytes / std::max<int64_t>(1, rb));
    void* slot_in[kStageSlots];
    void* slot_out[kStageSlots];
    for (int i = 0; i < kStageSlots; ++i) {
        MW_OK_OR_RETURN(scratch(c, "stage_in" + std::to_string(i), (size_t)(chunk_rows * rb), R.s, &slot_in[i]));
        MW_OK_OR_RETURN(scratch(c, "stage_out" + std::to_string(i), (size_t)(chunk_rows * rb), R.s, &slot_out[i]));
    }
    const bool a0_host = a0.location == MW_LOC_HOST, a1_host = a1.location == MW_LOC_HOST;
    // Uploads start after the work enqueued on the run's stream before this
    // call (a pinned host input may be filled by an asynchronous D2H on that
    // stream).  With staging overlap on (mw_ctx_set_staging_overlap: host
    // inputs are complete when mw_run is called) there is no start barrier:
    // the copy streams only wait for the previous use of each staging slot
    // (possibly by the previous run), so this run's first uploads overlap the
    // previous run's last downloads.  Device arguments and kernels stay
    // ordered on the run's stream.
    if (!c->staging_overlap) {
        CUDA_OK(cudaEventRecord(c->st_start, R.s));
        CUDA_OK(cudaStreamWaitEvent(c->copy_in, c->st_start, 0));
    }
    auto rgba = st.kind == StepKind::Rgba ? rgba_groups(st.ops) : std::vector<mwk::RgbaProg>{};
    auto u8 = st.kind == StepKind::U8 ? u8_groups(st.ops) : std::vector<mwk::U8Prog>{};
    auto sx = st.kind == StepKind::Saxpy ? saxpy_groups(st.ops) : std::vector<mwk::SaxpyProg>{};
    if (st.kind == StepKind::Rgba && rgba.size() > 1)
        return fail(MW_E_UNSUPPORTED, "host-staged RGBA chains are limited to 16 pointwise ops");
    int64_t chunk = 0;
    bool used[kStageSlots] = {false, false, false};   // by this run
    for (int q = 0; q < c->ppr; ++q) {
        int p = R.first + q;
        for (int64_t r0 = R.off[p]; r0 < R.off[p] + R.len[p]; r0 += chunk_rows, ++chunk) {
            const int64_t n = std::min(chunk_rows, R.off[p] + R.len[p] - r0);
            const int sl = (int)(chunk % kStageSlots);
            if (used[sl] || c->st_valid[sl]) CUDA_OK(cudaStreamWaitEvent(c->copy_in, c->st_out[sl], 0));
            used[sl] = true;
            uint8_t* din = static_cast<uint8_t*>(slot_in[sl]);
            uint8_t* dout = static_cast<uint8_t*>(slot_out[sl]);
            // inputs
            const uint8_t* h0 = at_row<const uint8_t>(a0, r0);
            const uint8_t* d0 = h0;
            if (a0_host) {
                CUDA_OK(cudaMemcpyAsync(din, h0, n * rb, cudaMemcpyHostToDevice, c->copy_in));
                d0 = din;
            }
            uint8_t* d1 = at_row<uint8_t>(a1, r0);
            if (a1_host) {
                d1 = dout;
                if (in_kind == MW_VK_SAXPY)  // y is read and written
                    CUDA_OK(cudaMemcpyAsync(dout, at_row<const uint8_t>(a1, r0), n * rb,
                                            cudaMemcpyHostToDevice, c->copy_in));
            }
            CUDA_OK(cudaEventRecord(c->st_in[sl], c->copy_in));
            CUDA_OK(cudaStreamWaitEvent(R.s, c->st_in[sl], 0));
            {
                PartTimer t(c, R.s, p,
                            st.kind == StepKind::Rgba ? MW_KC_RGBA
                            : st.kind == StepKind::U8 ? MW_KC_U8
                            : st.kind == StepKind::Fft ? MW_KC_FFT
                                                       : MW_KC_SAXPY);
                mwk::Launch L = launch_for(c, R.s, p);
                if (st.kind == StepKind::Fft) {
                    MW_OK_OR_RETURN(run_fft_chain(c, st.ops, reinterpret_cast<const float*>(d0),
                                                  reinterpret_cast<float*>(d1), n, (int)st.ops[0].ia, L));
                } else if (st.kind == StepKind::Rgba) {
                    MW_OK_OR_RETURN(kerr(mwk::rgba_chain(rgba[0], d0, d1, n, a0.shape[1], r0, L), "rgba_chain"));
                } else if (st.kind == StepKind::U8) {
                    const uint8_t* in = d0;
                    for (auto& g : u8) {
                        MW_OK_OR_RETURN(kerr(mwk::u8_chain(g, in, rb, d1, rb, n, rb, L), "u8_chain"));
                        in = d1;
                    }
                } else {
                    for (auto& g : sx)
                        MW_OK_OR_RETURN(kerr(mwk::saxpy_chain(g, reinterpret_cast<const float*>(d0),
                                                              reinterpret_cast<float*>(d1), n, L),
                                             "saxpy_chain"));
                }
            }
            CUDA_OK(cudaEventRecord(c->st_comp[sl], R.s));
            CUDA_OK(cudaStreamWaitEvent(c->copy_out, c->st_comp[sl], 0));
            if (a1_host)
                CUDA_OK(cudaMemcpyAsync(at_row<uint8_t>(a1, r0), d1, n * rb, cudaMemcpyDeviceToHost,
                                        c->copy_out));
            CUDA_OK(cudaEventRecord(c->st_out[sl], c->copy_out));
            c->st_valid[sl] = true;
        }
    }
    for (int i = 0; i < kStageSlots; ++i)
        if (used[i]) CUDA_OK(cudaStreamWaitEvent(R.s, c->st_out[i], 0));
    return MW_OK;
}

// ------------------------------------------------------------ run pipelining
// Byte ranges of a run's device arguments: [0] read, [1] written for the
// src -> dst chains; every argument counts as read and written otherwise.
mw_ctx::Ranges run_ranges(const mw_arg* args, int nargs, bool chain) {
    mw_ctx::Ranges r;
    for (int i = 0; i < nargs; ++i) {
        const mw_arg& a = args[i];
        if (a.location != MW_LOC_DEVICE || !a.ptr) continue;
        const int64_t n = a.mode == MW_COPY ? a.shape[0] : a.local_rows;
        const uintptr_t b = reinterpret_cast<uintptr_t>(a.ptr);
        const std::pair<uintptr_t, uintptr_t> rg{b, b + (uintptr_t)(n * row_bytes(a))};
        if (!chain || i == 0) r.rd.push_back(rg);
        if (!chain || i == 1) r.wr.push_back(rg);
    }
    r.valid = true;
    return r;
}
bool overlaps(const std::vector<std::pair<uintptr_t, uintptr_t>>& a,
              const std::vector<std::pair<uintptr_t, uintptr_t>>& b) {
    for (auto& x : a)
        for (auto& y : b)
            if (x.first < y.second && y.first < x.second) return true;
    return false;
}
// The run's first kernel may start reading before the previous run's last
// kernel completed: the ctx promised pipelining, the previous run was on this
// stream, and this run (a src -> dst chain) reads nothing that run wrote.
// (Its stores still wait for the predecessor, so write hazards cannot arise.)
bool run_independent(const mw_ctx* c, const mw_arg* args, int nargs) {
    if (!c->pipelining || !c->prev_io.valid || c->capturing) return false;
    const mw_ctx::Ranges cur = run_ranges(args, nargs, true);
    return !overlaps(cur.rd, c->prev_io.wr);
}

// ------------------------------------------------------------ the run
mw_status run_loop_host(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s,
                        mw_future* f);

mw_status run_split_host(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s,
                         mw_future* f, int h);

// index of the host-condition loop among a pipeline root's stages (-1: none)
int host_stage(const Node* root) {
    if (root->type != mw::NodeType::Pipeline) return -1;
    for (size_t i = 0; i < root->kids.size(); ++i)
        if (root->kids[i]->type == mw::NodeType::LoopHost) return (int)i;
    return -1;
}

mw_status run(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s,
              mw_future* f) {
    while (root->type == mw::NodeType::Map) root = root->kids[0];   // Map(t) runs t
    if (root->type == mw::NodeType::LoopHost) return run_loop_host(c, root, args, nargs, s, f);
    if (const int h = host_stage(root); h >= 0) return run_split_host(c, root, args, nargs, s, f, h);
    mw_status pst;
    const mw::NodeCache* nc = mw::plan_cached(root, &pst);
    if (!nc) return pst;
    const std::vector<Step>& prog = nc->prog;
    const int ik = root->in_kind, ok = root->out_kind;
    // ---- interface (marrow.h, mw_run)
    int need = (ik == MW_VK_VEC1 || ik == MW_VK_TRAITS) ? 1 : 2;
    if (nargs != need)
        return fail(MW_E_SHAPE_MISMATCH, "root expects " + std::to_string(need) + " args, got " +
                                             std::to_string(nargs));
    switch (ik) {
        case MW_VK_SAXPY:
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_F32, 1, 1, MW_PARTITION, -1));
            MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_F32, 1, 1, MW_PARTITION, -1));
            break;
        case MW_VK_RGBA:
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_U8, 3, 3, MW_PARTITION, 4));
            MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_U8, 3, 3, MW_PARTITION, 4));
            break;
        case MW_VK_U8:
        case MW_VK_U8_2D: {
            int lo = ik == MW_VK_U8_2D ? 2 : 1, hi = ik == MW_VK_U8_2D ? 2 : 4;
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_U8, lo, hi, MW_PARTITION, -1));
            MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_U8, lo, hi, MW_PARTITION, -1));
            break;
        }
        case MW_VK_NBODY:
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_F32, 2, 2, MW_COPY, 4));
            if (ok == MW_VK_ACCEL)
                MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_F32, 2, 2, MW_PARTITION, 4));
            else
                MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_F32, 2, 2, MW_COPY, 4));
            break;
        case MW_VK_VEC1:
        case MW_VK_VEC2:
            for (int i = 0; i < nargs; ++i)
                MW_OK_OR_RETURN(check_arg(args[i], i, MW_DT_F32, 1, 1, MW_PARTITION, -1));
            break;
        case MW_VK_TRAITS:
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_I64, 2, 2, MW_PARTITION, 2));
            break;
        case MW_VK_CPLX:
            MW_OK_OR_RETURN(check_arg(args[0], 0, MW_DT_F32, 3, 3, MW_PARTITION, 2));
            MW_OK_OR_RETURN(check_arg(args[1], 1, MW_DT_F32, 3, 3, MW_PARTITION, 2));
            for (const Step& stp : prog)
                for (const mw::ChainOp& o : stp.ops)
                    if (args[0].shape[1] != (int64_t{1} << o.ia))
                        return fail(MW_E_SHAPE_MISMATCH,
                                    "fft leaf of N = 2^" + std::to_string(o.ia) + " on rows of " +
                                        std::to_string(args[0].shape[1]) + " points");
            break;
        default: return fail(MW_E_UNSUPPORTED, "root value kind cannot be run");
    }
    if (nargs == 2 && !same_shape(args[0], args[1]))
        return fail(MW_E_SHAPE_MISMATCH, "args 0 and 1 must have the same global shape");
    const int64_t L = args[0].shape[0];
    // ---- partition (identical on every rank)
    if (nc->gst) {   // re-derive the granule error message for this call
        mw_status st;
        mw::granule_of(root, &st);
        return st;
    }
    const int64_t g = nc->granule;
    RunCtx R{c, s, std::vector<int64_t>(c->P), std::vector<int64_t>(c->P), c->rank * c->ppr};
    MW_OK_OR_RETURN(mw::partition_plan(L, g, c->dist.data(), c->P, nc->strict, R.off.data(),
                                       R.len.data()));
    const int plast = R.first + c->ppr - 1;
    const int64_t s0 = R.off[R.first], s1 = R.off[plast] + R.len[plast];
    bool host = false;
    for (int i = 0; i < nargs; ++i) {
        const mw_arg& a = args[i];
        host |= a.location == MW_LOC_HOST;
        if (a.mode == MW_PARTITION && s1 > s0 &&
            (a.local_offset > s0 || a.local_offset + a.local_rows < s1 || a.local_rows < 0))
            return fail(MW_E_SHAPE_MISMATCH,
                        "arg " + std::to_string(i) + " holds rows [" + std::to_string(a.local_offset) +
                            "," + std::to_string(a.local_offset + a.local_rows) +
                            ") but this rank's partitions need [" + std::to_string(s0) + "," +
                            std::to_string(s1) + ")");
    }
    if (nargs == 2 && ik != MW_VK_SAXPY && ik != MW_VK_VEC2 && args[0].ptr == args[1].ptr &&
        args[0].ptr && L > 0 && args[0].location == args[1].location)
        return fail(MW_E_SHAPE_MISMATCH, "src and dst must not alias");
    // ---- execute
    c->recs.clear();
    if (!c->stats_on) c->ev_used = 0;   // events of accumulated stats stay live
    if (!c->capturing && c->monitor) CUDA_OK(cudaEventRecord(c->wall_a, s));
    const int ppr = c->ppr;
    if (host && c->capturing)
        return fail(MW_E_UNSUPPORTED, "host-resident arguments cannot be captured in a graph");
    if (host) {
        if (prog.size() != 1 || (prog[0].kind != StepKind::Saxpy && prog[0].kind != StepKind::Rgba &&
                                 prog[0].kind != StepKind::U8 && prog[0].kind != StepKind::Fft) ||
            (prog[0].kind == StepKind::Fft && prog[0].ops.empty()))
            return fail(MW_E_UNSUPPORTED,
                        "host-resident arguments are supported for single fused Map/Pipeline "
                        "chains (NEXT-1)");
        MW_OK_OR_RETURN(run_staged(R, prog[0], ik, args));
    } else if (ik == MW_VK_SAXPY && !(prog.size() == 1 && prog[0].kind == StepKind::Reduce)) {
        auto groups = prog.empty() ? std::vector<mwk::SaxpyProg>{} : saxpy_groups(prog[0].ops);
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            PartTimer t(c, s, p, MW_KC_SAXPY);
            for (auto& gp : groups)
                MW_OK_OR_RETURN(kerr(mwk::saxpy_chain(gp, at_row<const float>(args[0], R.off[p]),
                                                      at_row<float>(args[1], R.off[p]), R.len[p],
                                                      launch_for(c, s, p)),
                                     "saxpy_chain"));
        }
    } else if (ik == MW_VK_RGBA) {
        auto groups = rgba_groups(prog.empty() ? std::vector<mw::ChainOp>{} : prog[0].ops);
        const int64_t W = args[0].shape[1];
        uint8_t *t0 = nullptr, *t1 = nullptr;
        if (groups.size() > 1) {
            int64_t mx = 0;
            for (int q = 0; q < ppr; ++q) mx = std::max(mx, R.len[R.first + q]);
            void *a, *b;
            MW_OK_OR_RETURN(scratch(c, "rgba_tmp0", (size_t)(mx * W * 4), s, &a));
            MW_OK_OR_RETURN(scratch(c, "rgba_tmp1", (size_t)(mx * W * 4), s, &b));
            t0 = static_cast<uint8_t*>(a);
            t1 = static_cast<uint8_t*>(b);
        }
        // The first launch may read ahead of the dependent-launch wait when the
        // previous run wrote nothing it reads (pipelining contract); a later
        // partition's launch follows the previous partition's, which wrote
        // other rows of dst only (src and dst never alias).
        bool indep = run_independent(c, args, nargs);
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            PartTimer t(c, s, p, MW_KC_RGBA);
            // src -> dst chains are idempotent: the slowdown injector repeats them
            // (time exactly proportional to the factor; results unchanged)
            const int reps = c->slow[p] > 1.0f ? (int)std::lround(c->slow[p]) : 1;
            for (int rep = 0; rep < reps; ++rep) {
                MW_OK_OR_RETURN(run_rgba(R, p, groups, at_row<const uint8_t>(args[0], R.off[p]),
                                         at_row<uint8_t>(args[1], R.off[p]), R.len[p], W, R.off[p],
                                         t0, t1, !indep || rep > 0 || c->monitor));
                indep = true;
            }
        }
    } else if (ik == MW_VK_U8 || ik == MW_VK_U8_2D) {
        R.indep = run_independent(c, args, nargs);
        MW_OK_OR_RETURN(run_u8(R, prog, args[0], args[1], f));
    } else if (ik == MW_VK_NBODY && ok == MW_VK_NBODY) {
        if (L > 0 && args[0].ptr == args[1].ptr) return fail(MW_E_SHAPE_MISMATCH, "pos and vel alias");
        for (const Step& stp : prog) MW_OK_OR_RETURN(run_nbody(R, stp, args[0], args[1]));
    } else if (ik == MW_VK_NBODY) {
        const Step& stp = prog[0];
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            void* pp;
            MW_OK_OR_RETURN(scratch(c, "nbody_part", (size_t)mwk::nbody_part_doubles(R.len[p]) * 8, s, &pp));
            PartTimer t(c, s, p, MW_KC_NBODY);
            MW_OK_OR_RETURN(kerr(mwk::nbody(static_cast<const float4*>(args[0].ptr), nullptr, nullptr,
                                            nullptr, at_row<float4>(args[1], R.off[p]), R.off[p],
                                            R.len[p], L, stp.eps2, 0.f, 1, static_cast<double*>(pp),
                                            launch_for(c, s, p)),
                                 "nbody_accel"));
        }
    } else if (ik == MW_VK_VEC1 || ik == MW_VK_VEC2 || ik == MW_VK_SAXPY) {   // MapReduce
        const int64_t CH = 1ll << mwk::kChunkLog2;
        const int64_t nch = (L + CH - 1) / CH;
        void *pp, *rp;
        MW_OK_OR_RETURN(scratch(c, "partials", (size_t)std::max<int64_t>(1, nch) * 8, s, &pp));
        MW_OK_OR_RETURN(scratch(c, "result", 8, s, &rp));
        double* partials = static_cast<double*>(pp);
        // device reduction stage (MW_REDUCE_*; SUM for mw_map_reduce): chunk
        // partials start at the operator's identity
        const int rop = prog[0].reduce_op;
        MW_OK_OR_RETURN(kerr(mwk::reduce_fill_identity(partials, std::max<int64_t>(1, nch), s, rop),
                             "reduce_fill"));
        const bool dot = prog[0].dot;
        mwk::SaxpyProg pre{};   // saxpy chain fused into the map stage (sct.cpp plan)
        for (const mw::ChainOp& o : prog[0].pre) pre.a[pre.n++] = o.fa;
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            PartTimer t(c, s, p, MW_KC_REDUCE);
            MW_OK_OR_RETURN(kerr(mwk::reduce_chunks(at_row<const float>(args[0], R.off[p]),
                                                    dot ? at_row<const float>(args[1], R.off[p]) : nullptr,
                                                    R.off[p], R.off[p], R.len[p], L, partials,
                                                    launch_for(c, s, p), rop, pre.n ? &pre : nullptr,
                                                    prog[0].term_map),
                                 "reduce_chunks"));
        }
        // merge "+" across ranks: each chunk partial has exactly
        // one non-zero contributor, so the sum is exact and order-free.
        // (max / min: one contributor per chunk, the others hold the identity)
        if (c->comm && nch > 0)
            MW_OK_OR_RETURN(c->comm->allreduce(partials, (size_t)nch, mwc::DType::F64,
                                               rop == MW_REDUCE_MAX   ? mwc::ROp::Max
                                               : rop == MW_REDUCE_MIN ? mwc::ROp::Min
                                                                      : mwc::ROp::Sum,
                                               s));
        if (prog[0].merge_op == MW_MERGE_ADD) {
            mwk::ScalarPost post{};
            if (prog[0].post.size() > 8) return fail(MW_E_UNSUPPORTED, "more than 8 scalar maps");
            for (const auto& pm : prog[0].post) {
                post.kind[post.n] = pm.first;
                post.c[post.n++] = pm.second;
            }
            MW_OK_OR_RETURN(kerr(mwk::reduce_combine(partials, nch, static_cast<double*>(rp), s, rop, &post),
                                 "reduce_combine"));
            CUDA_OK(cudaMemcpyAsync(f->res, rp, 8, cudaMemcpyDeviceToHost, s));
        } else {
            // NEXT-4 merging functions: every rank holds every chunk partial after
            // the all-reduce, so each forms all P partition partials (same fixed
            // tree as the canonical combine, over the partition's chunk range)
            if (c->capturing)
                return fail(MW_E_UNSUPPORTED, "MapReduce with a non-ADD merge is merged on the host "
                                              "and cannot be captured in a graph");
            void* dp;
            MW_OK_OR_RETURN(scratch(c, "part_partials", (size_t)c->P * 8, s, &dp));
            double* dparts = static_cast<double*>(dp);
            f->part_active.assign(c->P, 0);
            for (int p = 0; p < c->P; ++p) {
                if (R.len[p] == 0) continue;
                const int64_t c0 = R.off[p] / CH, c1 = (R.off[p] + R.len[p] + CH - 1) / CH;
                MW_OK_OR_RETURN(kerr(mwk::reduce_combine(partials + c0, c1 - c0, dparts + p, s), "reduce_combine"));
                f->part_active[p] = 1;
            }
            CUDA_OK(cudaHostAlloc(&f->parts, (size_t)c->P * 8, cudaHostAllocDefault));
            CUDA_OK(cudaMemcpyAsync(f->parts, dparts, (size_t)c->P * 8, cudaMemcpyDeviceToHost, s));
            f->merge_op = prog[0].merge_op;
            f->merge_fn = reinterpret_cast<mw_merge_fn>(prog[0].fn);
            f->merge_user = prog[0].user;
        }
        f->has_reduce = true;
    } else if (ik == MW_VK_CPLX) {
        const std::vector<mw::ChainOp> none;
        const std::vector<mw::ChainOp>& ops = prog.empty() ? none : prog[0].ops;
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            if (ops.empty()) {   // e.g. loop_for(fft, 0): identity
                CUDA_OK(cudaMemcpyAsync(at_row<float>(args[1], R.off[p]), at_row<const float>(args[0], R.off[p]),
                                        R.len[p] * row_bytes(args[0]), cudaMemcpyDeviceToDevice, s));
                continue;
            }
            PartTimer t(c, s, p, MW_KC_FFT);
            MW_OK_OR_RETURN(run_fft_chain(c, ops, at_row<const float>(args[0], R.off[p]),
                                          at_row<float>(args[1], R.off[p]), R.len[p], (int)ops[0].ia,
                                          launch_for(c, s, p)));
        }
    } else if (ik == MW_VK_TRAITS) {
        for (int q = 0; q < ppr; ++q) {
            int p = R.first + q;
            if (R.len[p] == 0) continue;
            PartTimer t(c, s, p, MW_KC_TRAITS);
            MW_OK_OR_RETURN(kerr(mwk::fill_traits(at_row<int64_t>(args[0], R.off[p]), R.len[p], R.len[p],
                                                  R.off[p], launch_for(c, s, p)),
                                 "fill_traits"));
        }
    }
    if (!c->capturing) {
        if (c->monitor) CUDA_OK(cudaEventRecord(c->wall_b, s));
        c->last_len = R.len;
        c->have_run = c->monitor;
        c->prev_io = run_ranges(args, nargs, ik == MW_VK_RGBA || ik == MW_VK_U8 || ik == MW_VK_U8_2D);
        c->prev_io.valid = !host && prog.size() <= 1;
    }
    return MW_OK;
}

// Loop with a host-side condition (NEXT-4, reading R27): stage 1
// (the condition) and stage 3 (state update) run on the host between body
// executions; stage 2 (the body) runs through run().  Value kinds with a
// separate output ping-pong through a scratch copy of this rank's rows.
mw_status run_loop_host(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s,
                        mw_future* f) {
    if (c->capturing)
        return fail(MW_E_UNSUPPORTED, "a host-condition loop evaluates its condition on the host "
                                      "and cannot be captured in a graph");
    for (int i = 0; i < nargs; ++i)
        if (args[i].location == MW_LOC_HOST)
            return fail(MW_E_UNSUPPORTED, "host-condition loops take device-resident arguments");
    const Node* body = root->kids[0];
    auto cond = reinterpret_cast<mw_loop_cond_fn>(root->fn);
    const int ik = body->in_kind;
    const bool two = nargs == 2 && (ik == MW_VK_RGBA || ik == MW_VK_U8 || ik == MW_VK_U8_2D ||
                                    ik == MW_VK_CPLX);
    std::vector<mw_arg> cur(args, args + nargs);
    void* tmp = nullptr;
    size_t tbytes = 0;
    if (two) {
        tbytes = (size_t)(args[1].local_rows * row_bytes(args[1]));
        MW_OK_OR_RETURN(scratch(c, "loop_host_tmp", std::max<size_t>(tbytes, 16), s, &tmp));
    }
    int64_t E = 0;
    bool stopped = false;
    for (int64_t it = 0; it < root->n; ++it) {
        CUDA_OK(cudaStreamSynchronize(s));   // stage 3 of the previous iteration is visible
        if (!cond(it, root->user)) {
            stopped = true;
            break;
        }
        if (two && it > 0) {   // input of iteration it = output of it - 1
            CUDA_OK(cudaMemcpyAsync(tmp, args[1].ptr, tbytes, cudaMemcpyDeviceToDevice, s));
            cur[0] = args[1];
            cur[0].ptr = tmp;
        }
        MW_OK_OR_RETURN(run(c, body, cur.data(), nargs, s, f));
        ++E;
    }
    if (two && E == 0 && args[0].ptr != args[1].ptr)   // no iteration: the loop is the identity
        CUDA_OK(cudaMemcpyAsync(args[1].ptr, static_cast<const uint8_t*>(args[0].ptr) +
                                                 (args[1].local_offset - args[0].local_offset) * row_bytes(args[0]),
                                tbytes, cudaMemcpyDeviceToDevice, s));
    f->executions += (double)E;
    if (!stopped) f->converged = 0.0;
    return MW_OK;
}

// A pipeline with a host-condition loop among its stages (NEXT-4, the Fig. 1
// shape with the paper's host-side loop stages P:374-378): the stages before
// the loop run as one fused sub-pipeline into an intermediate buffer, the
// loop ping-pongs on the device with its condition on the host, the stages
// after it run from its output into the destination.  In-place value kinds
// (saxpy, N-body) run every part on the arguments themselves.
mw_status run_split_host(mw_ctx* c, const Node* root, const mw_arg* args, int nargs, cudaStream_t s,
                         mw_future* f, int h) {
    if (c->capturing)
        return fail(MW_E_UNSUPPORTED, "a host-condition loop evaluates its condition on the host "
                                      "and cannot be captured in a graph");
    const std::vector<Node*>& kids = root->kids;
    for (size_t i = 0; i < kids.size(); ++i)
        if ((int)i != h && host_stage(kids[i]) >= 0)
            return fail(MW_E_UNSUPPORTED, "one host-condition loop per pipeline");
    // the stages before / after the loop as nodes (a transient pipeline when
    // there are several: the tree itself stays immutable)
    auto part = [&](size_t b, size_t e, mw_node** out) -> mw_status {
        *out = nullptr;
        if (e <= b) return MW_OK;
        if (e - b == 1) {
            *out = reinterpret_cast<mw_node*>(kids[b]);
            mw_node_retain(*out);
            return MW_OK;
        }
        std::vector<mw_node*> st;
        for (size_t i = b; i < e; ++i) st.push_back(reinterpret_cast<mw_node*>(kids[i]));
        return mw_pipeline(st.data(), (int32_t)st.size(), out);
    };
    mw_node *pre = nullptr, *post = nullptr;
    MW_OK_OR_RETURN(part(0, (size_t)h, &pre));
    mw_status st = part((size_t)h + 1, kids.size(), &post);
    if (st != MW_OK) {
        if (pre) mw_node_release(pre);
        return st;
    }
    struct Rel {
        mw_node* n;
        ~Rel() {
            if (n) mw_node_release(n);
        }
    } rp{pre}, rq{post};
    const Node* loop = kids[h];
    const int ik = root->in_kind;
    const bool two = nargs == 2 && (ik == MW_VK_RGBA || ik == MW_VK_U8 || ik == MW_VK_U8_2D || ik == MW_VK_CPLX);
    if (!two) {   // in place: every part on the same arguments, in order
        if (pre) MW_OK_OR_RETURN(run(c, reinterpret_cast<const Node*>(pre), args, nargs, s, f));
        MW_OK_OR_RETURN(run_loop_host(c, loop, args, nargs, s, f));
        if (post) MW_OK_OR_RETURN(run(c, reinterpret_cast<const Node*>(post), args, nargs, s, f));
        return MW_OK;
    }
    // intermediates: this rank's rows, the destination's shape
    const size_t bytes = (size_t)std::max<int64_t>(16, args[1].local_rows * row_bytes(args[1]));
    auto tmp_arg = [&](const char* name, mw_arg* out) -> mw_status {
        void* p;
        MW_OK_OR_RETURN(scratch(c, name, bytes, s, &p));
        *out = args[1];
        out->ptr = p;
        out->location = MW_LOC_DEVICE;
        return MW_OK;
    };
    mw_arg a_in = args[0], a_mid, a_out;
    if (pre) {
        MW_OK_OR_RETURN(tmp_arg("split_pre", &a_mid));
        const mw_arg pa[2] = {args[0], a_mid};
        MW_OK_OR_RETURN(run(c, reinterpret_cast<const Node*>(pre), pa, 2, s, f));
        a_in = a_mid;
    }
    if (post) MW_OK_OR_RETURN(tmp_arg("split_post", &a_out));
    else a_out = args[1];
    const mw_arg la[2] = {a_in, a_out};
    MW_OK_OR_RETURN(run_loop_host(c, loop, la, 2, s, f));
    if (post) {
        const mw_arg qa[2] = {a_out, args[1]};
        MW_OK_OR_RETURN(run(c, reinterpret_cast<const Node*>(post), qa, 2, s, f));
    }
    return MW_OK;
}

// Runs of one ctx execute in call order even on different streams (they
// share the ctx scratch): a run's stream first waits for the previous run's
// end, which each run records.  On one stream the wait is a no-op.
// The event is recorded lazily, only when the stream changes: consecutive
// runs on one stream keep no event operations between their kernels (which
// would stand between programmatically dependent launches).
mw_status fifo_enter(mw_ctx* c, cudaStream_t s) {
    if (c->capturing || !c->have_last_run || s == c->last_stream) return MW_OK;
    if (cudaEventRecord(c->last_run, c->last_stream) != cudaSuccess) {
        (void)cudaGetLastError();   // the previous stream is gone: drain the device instead
        CUDA_OK(cudaDeviceSynchronize());
    } else {
        CUDA_OK(cudaStreamWaitEvent(s, c->last_run, 0));
    }
    c->prev_io.valid = false;   // another stream: no programmatic overlap
    return MW_OK;
}
void fifo_exit(mw_ctx* c, cudaStream_t s) {
    if (c->capturing) return;
    c->last_stream = s;
    c->have_last_run = true;
}

static void ctx_teardown(mw_ctx* c) {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& kv : c->scratch) ctx_free(c, kv.second.p);
    c->comm.reset();
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : c->fut_ev) cudaEventDestroy(e);
    if (c->wall_a) cudaEventDestroy(c->wall_a);
    if (c->wall_b) cudaEventDestroy(c->wall_b);
    for (int i = 0; i < kStageSlots; ++i) {
        if (c->st_in[i]) cudaEventDestroy(c->st_in[i]);
        if (c->st_comp[i]) cudaEventDestroy(c->st_comp[i]);
        if (c->st_out[i]) cudaEventDestroy(c->st_out[i]);
    }
    if (c->st_start) cudaEventDestroy(c->st_start);
    if (c->last_run) cudaEventDestroy(c->last_run);
    for (void* p : c->orphans) ctx_free(c, p);
    for (auto& kv : c->ipc_open) cudaIpcCloseMemHandle(kv.second);
    if (c->xblock) cudaFree(c->xblock);
    if (c->m_root) mw_node_release(const_cast<mw_node*>(c->m_root));
    if (c->copy_in) cudaStreamDestroy(c->copy_in);
    if (c->copy_out) cudaStreamDestroy(c->copy_out);
    if (c->aux) cudaStreamDestroy(c->aux);
    for (cudaStream_t q : c->lane_s)
        if (q) cudaStreamDestroy(q);
    for (cudaEvent_t e : c->lane_ev)
        if (e) cudaEventDestroy(e);
    if (c->h_flag) cudaFreeHost(c->h_flag);
    for (cudaEvent_t e : c->lag_ev)
        if (e) cudaEventDestroy(e);
    for (double* p : c->res_pages) cudaFreeHost(p);
    (void)cudaGetLastError();   // leave no stale error behind for the host application
    delete c;
}
void ctx_retain(mw_ctx* c) { ++c->refs; }
void ctx_release(mw_ctx* c) {
    if (--c->refs == 0) ctx_teardown(c);
}

}  // namespace mwx

// ============================================================ C-ABI
extern "C" {

const char* mw_last_error(const mw_ctx*) { return mw::last_error_cstr(); }

mw_status mw_nccl_unique_id(uint8_t out[128]) {
    if (!out) return fail(MW_E_INVALID_SPEC, "NULL output");
    ncclUniqueId id;
    NCCL_OK(ncclGetUniqueId(&id));
    static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
    memcpy(out, id.internal, 128);
    return MW_OK;
}

mw_status mw_ctx_create(int32_t device, int32_t rank, int32_t nranks, int32_t parts_per_rank,
                        const uint8_t* nccl_id, int32_t transport, const mw_alloc_fns* alloc,
                        mw_ctx** out) {
    if (!out) return fail(MW_E_INVALID_SPEC, "out is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks || parts_per_rank < 1)
        return fail(MW_E_INVALID_SPEC, "need 0 <= rank < nranks and parts_per_rank >= 1");
    if (transport < MW_TRANSPORT_AUTO || transport > MW_TRANSPORT_LOOPBACK)
        return fail(MW_E_INVALID_SPEC, "unknown transport");
    const bool use_comm = nranks > 1 || transport != MW_TRANSPORT_AUTO;
    if (use_comm && !nccl_id) return fail(MW_E_INVALID_SPEC, "group id required");
    if (alloc && (!alloc->alloc || !alloc->free))
        return fail(MW_E_INVALID_SPEC, "allocator needs both alloc and free");
    CUDA_OK(cudaSetDevice(device));
    std::unique_ptr<mw_ctx> c(new mw_ctx);
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    c->ppr = parts_per_rank;
    c->P = nranks * parts_per_rank;
    c->dist.assign(c->P, 1.0 / c->P);
    c->slow.assign(c->P, 1.0f);
    c->cls.assign(c->P, 0);
    c->relperf.assign(c->P, 1.0);
    mwk::tune_defaults(c->tune);
    if (alloc) {
        c->alloc = *alloc;
        c->has_alloc = true;
    }
    CUDA_OK(cudaHostAlloc(&c->h_flag, 64, cudaHostAllocDefault));
    CUDA_OK(cudaEventCreate(&c->wall_a));
    CUDA_OK(cudaEventCreate(&c->wall_b));
    CUDA_OK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->last_run, cudaEventDisableTiming));
    CUDA_OK(mwk::fft_prepare(c->aux));   // before any capture can start
    CUDA_OK(cudaStreamSynchronize(c->aux));
    c->launches0 = mwk::launch_count();
    c->bstate = mw_balance_state{};
    if (use_comm) {
        if (transport == MW_TRANSPORT_LOOPBACK)
            MW_OK_OR_RETURN(mwc::make_loopback(device, rank, nranks, nccl_id, &c->comm));
        else
            MW_OK_OR_RETURN(mwc::make_nccl(rank, nranks, nccl_id, &c->comm));
    }
    *out = c.release();
    return MW_OK;
}

static void reap_retired(mw_ctx* c, bool sync);

// Futures and graphs hold a reference: a ctx destroyed while they are alive
// is torn down when the last of them is released.
mw_status mw_ctx_destroy(mw_ctx* c) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (c->destroyed) return fail(MW_E_STATE, "ctx already destroyed");
    c->destroyed = true;
    reap_retired(c, true);   // the retired futures' references (the user's handle remains)
    ctx_release(c);
    return MW_OK;
}

mw_status mw_ctx_info(const mw_ctx* c, int32_t* n_parts, int32_t* first_part, int32_t* ppr,
                      int32_t* rank, int32_t* nranks) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (n_parts) *n_parts = c->P;
    if (first_part) *first_part = c->rank * c->ppr;
    if (ppr) *ppr = c->ppr;
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->nranks;
    return MW_OK;
}

mw_status mw_set_distribution(mw_ctx* c, const double* fractions, int32_t n) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (n != c->P) return fail(MW_E_INVALID_SPEC, "distribution needs one fraction per partition");
    MW_OK_OR_RETURN(mw::check_distribution(fractions, n));
    c->dist.assign(fractions, fractions + n);
    return MW_OK;
}

mw_status mw_get_distribution(const mw_ctx* c, double* out, int32_t n) {
    if (!c || !out) return fail(MW_E_STATE, "NULL argument");
    if (n < c->P) return fail(MW_E_INVALID_SPEC, "output too small");
    for (int i = 0; i < c->P; ++i) out[i] = c->dist[i];
    return MW_OK;
}

mw_status mw_partition(const mw_ctx* c, const mw_node* root, int64_t L, int64_t* offsets,
                       int64_t* lengths) {
    if (!c || !root || !offsets || !lengths) return fail(MW_E_INVALID_SPEC, "NULL argument");
    mw_status st;
    const Node* r = reinterpret_cast<const Node*>(root);
    int64_t g = mw::granule_of(r, &st);
    if (st) return st;
    std::vector<int64_t> o(c->P), l(c->P);
    MW_OK_OR_RETURN(mw::partition_plan(L, g, c->dist.data(), c->P, mw::strict_of(r), o.data(), l.data()));
    for (int i = 0; i < c->P; ++i) {
        offsets[i] = o[i];
        lengths[i] = l[i];
    }
    return MW_OK;
}

mw_status mw_run(mw_ctx* c, const mw_node* root, const mw_arg* args, int32_t nargs, void* stream,
                 mw_future** out) {
    if (!c || !root || !out || (nargs > 0 && !args)) return fail(MW_E_INVALID_SPEC, "NULL argument");
    if (c->destroyed) return fail(MW_E_STATE, "ctx was destroyed");
    CUDA_OK(cudaSetDevice(c->device));
    reap_retired(c, false);
    // Consume a stale non-sticky error left in the runtime's last-error slot by
    // an unrelated earlier call (ours or the host application's), so that the
    // post-launch checks below report only this run's launches.  Sticky
    // (asynchronous) faults are still returned by every subsequent call.
    (void)cudaGetLastError();
    std::unique_ptr<mw_future> f(new mw_future);
    f->ctx = c;
    if (c->res_free.empty()) {
        double* page;
        CUDA_OK(cudaHostAlloc(&page, 4096, cudaHostAllocDefault));
        c->res_pages.push_back(page);
        for (int i = 0; i < 128; ++i) c->res_free.push_back(page + 4 * i);
    }
    f->res = c->res_free.back();
    c->res_free.pop_back();
    *f->res = 0.0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MW_OK_OR_RETURN(fifo_enter(c, s));
    mw_status st;
    try {
        st = run(c, reinterpret_cast<const Node*>(root), args, nargs, s, f.get());
    } catch (const std::bad_alloc&) {
        st = fail(MW_E_OOM, "host allocation failed");
    } catch (...) {
        st = fail(MW_E_INVALID_SPEC, "internal error");
    }
    if (st != MW_OK) {
        // copies into the result slot (or the partials) may already be queued
        // (e.g. a host-condition loop failing on a later iteration): drain
        // them before the slot can serve another future
        cudaStreamSynchronize(s);
        (void)cudaGetLastError();
        c->res_free.push_back(f->res);
        if (f->parts) cudaFreeHost(f->parts);
        f->parts = nullptr;
        return st;
    }
    fifo_exit(c, s);
    cudaError_t e = cudaSuccess;
    if (!c->fut_ev.empty()) {
        f->done = c->fut_ev.back();
        c->fut_ev.pop_back();
    } else {
        e = cudaEventCreateWithFlags(&f->done, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventRecord(f->done, s);
    if (e != cudaSuccess) {
        c->res_free.push_back(f->res);
        if (f->done) cudaEventDestroy(f->done);
        return fail(MW_E_CUDA, std::string("future event: ") + cudaGetErrorString(e));
    }
    ctx_retain(c);
    *out = f.release();
    return MW_OK;
}

mw_status mw_future_wait(mw_future* f) {
    if (!f || !f->done) return fail(MW_E_STATE, "invalid future");
    cudaError_t e = cudaEventSynchronize(f->done);
    if (e != cudaSuccess) return fail(MW_E_CUDA, std::string("run failed: ") + cudaGetErrorString(e));
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MW_E_CUDA, std::string("run failed: ") + cudaGetErrorString(e));
    if (f->ctx->comm) MW_OK_OR_RETURN(f->ctx->comm->async_error());
    f->waited = true;
    return MW_OK;
}

mw_status mw_future_query(mw_future* f, int32_t* done) {
    if (!f || !f->done || !done) return fail(MW_E_STATE, "invalid future");
    cudaError_t e = cudaEventQuery(f->done);
    if (e == cudaErrorNotReady) {
        *done = 0;
        return MW_OK;
    }
    if (e != cudaSuccess) return fail(MW_E_CUDA, std::string("run failed: ") + cudaGetErrorString(e));
    *done = 1;
    f->completed = true;
    return MW_OK;
}

mw_status mw_future_result(mw_future* f, double* out, int32_t n) {
    if (!f || !out) return fail(MW_E_STATE, "invalid future");
    if (!f->waited) MW_OK_OR_RETURN(mw_future_wait(f));
    double ex = f->executions, conv = f->converged;
    if (f->plane_loop) {
        const int32_t* st = reinterpret_cast<const int32_t*>(f->res + 1);
        if (f->plane_xr && st[3] < 0) {
            f->ctx->xr_broken = true;
            return fail(MW_E_NCCL, "cross-rank hysteresis: a rank did not reach the pass barrier "
                                   "within 10 s (the run aborted; later runs use the per-pass exchange)");
        }
        if (f->plane_count) {
            double eb;
            bool cv;
            body_execs(st[0], st[1] != 0, f->plane_m, f->plane_nb, &eb, &cv);
            ex += eb;
            if (!cv) conv = 0.0;
        }
    }
    double red = f->has_reduce ? *f->res : 0.0;
    if (f->parts) {   // merging function over the partitions with work, in global order
        bool first = true;
        red = 0.0;
        for (size_t p = 0; p < f->part_active.size(); ++p) {
            if (!f->part_active[p]) continue;
            const double r = f->parts[p];
            if (first) {
                red = r;
                first = false;
                continue;
            }
            switch (f->merge_op) {
                case MW_MERGE_SUB: red = red - r; break;
                case MW_MERGE_MUL: red = red * r; break;
                case MW_MERGE_DIV: red = red / r; break;
                default: red = f->merge_fn(red, r, f->merge_user); break;
            }
        }
    }
    double v[4] = {red, (double)(float)red, ex, conv};
    for (int i = 0; i < n && i < 4; ++i) out[i] = v[i];
    return MW_OK;
}

static void future_free(mw_future* f);

// reclaim retired futures whose run completed (sync: wait for all of them)
static void reap_retired(mw_ctx* c, bool sync) {
    // oldest first; stop at the first run still in flight (later releases are
    // usually later runs), so a call costs O(reclaimed + 1) event queries
    while (!c->retired.empty()) {
        mw_future* f = c->retired.front();
        if (!sync && cudaEventQuery(f->done) == cudaErrorNotReady) {
            (void)cudaGetLastError();   // a NotReady query is not an error of the next call
            break;
        }
        c->retired.pop_front();
        future_free(f);
    }
}

void mw_future_release(mw_future* f) {
    if (!f) return;
    if (f->done && !f->ctx->destroyed && !f->completed && !f->waited) {   // reclaimed later
        f->ctx->retired.push_back(f);
        return;
    }
    future_free(f);
}

static void future_free(mw_future* f) {
    if (f->done) {
        cudaEventSynchronize(f->done);
        if (f->ctx->fut_ev.size() < 256) f->ctx->fut_ev.push_back(f->done);
        else cudaEventDestroy(f->done);
    }
    if (f->res) f->ctx->res_free.push_back(f->res);
    if (f->parts) cudaFreeHost(f->parts);
    mw_ctx* c = f->ctx;
    delete f;
    ctx_release(c);
}

mw_status mw_last_timings(mw_ctx* c, float* per_part_ms, int32_t n, float* wall_ms) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (!c->have_run)
        return fail(MW_E_STATE, c->monitor ? "no run yet" : "monitoring is disabled (mw_ctx_set_monitoring)");
    if (per_part_ms && n < c->P) return fail(MW_E_INVALID_SPEC, "output too small");
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaEventSynchronize(c->wall_b));
    std::vector<float> local(c->ppr, 0.0f);
    for (auto& r : c->recs) {
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, r.a, r.b));
        local[r.part - c->rank * c->ppr] += ms;
    }
    std::vector<float> all(c->P, 0.0f);
    if (c->nranks > 1) {
        void* d;
        MW_OK_OR_RETURN(scratch(c, "timings", (size_t)c->P * 4, c->aux, &d));
        float* df = static_cast<float*>(d);
        CUDA_OK(cudaMemcpyAsync(df + c->rank * c->ppr, local.data(), c->ppr * 4, cudaMemcpyHostToDevice, c->aux));
        MW_OK_OR_RETURN(c->comm->allgather(df + c->rank * c->ppr, df, (size_t)c->ppr * 4, c->aux));
        CUDA_OK(cudaMemcpyAsync(all.data(), df, c->P * 4, cudaMemcpyDeviceToHost, c->aux));
        CUDA_OK(cudaStreamSynchronize(c->aux));
    } else {
        all = local;
    }
    if (per_part_ms)
        for (int i = 0; i < c->P; ++i) per_part_ms[i] = all[i];
    if (wall_ms) CUDA_OK(cudaEventElapsedTime(wall_ms, c->wall_a, c->wall_b));
    return MW_OK;
}

mw_status mw_stats_enable(mw_ctx* c, int32_t on) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaDeviceSynchronize());
    c->stats.clear();
    c->recs.clear();
    c->have_run = false;
    c->ev_used = 0;
    c->stats_on = on != 0;
    return MW_OK;
}

mw_status mw_kernel_stats(mw_ctx* c, int32_t kernel_class, double* total_ms, int64_t* launches) {
    if (!c || !total_ms || !launches) return fail(MW_E_INVALID_SPEC, "NULL argument");
    if (kernel_class < 0 || kernel_class >= MW_KC_COUNT) return fail(MW_E_INVALID_SPEC, "bad kernel class");
    CUDA_OK(cudaSetDevice(c->device));
    double tot = 0.0;
    int64_t n = 0;
    for (auto& r : c->stats) {
        if (r.cls != kernel_class) continue;
        CUDA_OK(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, r.a, r.b));
        tot += ms;
        n += r.launches;
    }
    *total_ms = tot;
    *launches = n;
    return MW_OK;
}

mw_status mw_last_lengths(const mw_ctx* c, int64_t* per_part_len, int32_t n) {
    if (!c || !per_part_len) return fail(MW_E_STATE, "NULL argument");
    if (!c->have_run)
        return fail(MW_E_STATE, c->monitor ? "no run yet" : "monitoring is disabled (mw_ctx_set_monitoring)");
    if (n < c->P) return fail(MW_E_INVALID_SPEC, "output too small");
    for (int i = 0; i < c->P; ++i) per_part_len[i] = c->last_len[i];
    return MW_OK;
}

mw_status mw_rebalance(mw_ctx* c, const mw_balance_params* p, int32_t* triggered) {
    if (!c || !p) return fail(MW_E_INVALID_SPEC, "NULL argument");
    std::vector<float> ms(c->P);
    MW_OK_OR_RETURN(mw_last_timings(c, ms.data(), c->P, nullptr));
    std::vector<double> next(c->P);
    int trig = 0;
    MW_OK_OR_RETURN(mw::balance_step(*p, c->bstate, ms.data(), c->last_len.data(), c->dist.data(), c->P,
                                     next.data(), &trig));
    if (trig) MW_OK_OR_RETURN(mw_set_distribution(c, next.data(), c->P));
    if (triggered) *triggered = trig;
    return MW_OK;
}

mw_status mw_get_balance_state(const mw_ctx* c, mw_balance_state* out) {
    if (!c || !out) return fail(MW_E_INVALID_SPEC, "NULL argument");
    *out = c->bstate;
    return MW_OK;
}

mw_status mw_ctx_set_slowdown(mw_ctx* c, int32_t part, float factor) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (part < 0 || part >= c->P || !(factor >= 1.0f))
        return fail(MW_E_INVALID_SPEC, "bad partition or factor < 1");
    c->slow[part] = factor;
    return MW_OK;
}

mw_status mw_ctx_set_run_pipelining(mw_ctx* c, int32_t on) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    c->pipelining = on != 0;
    c->prev_io.valid = false;
    return MW_OK;
}

mw_status mw_ctx_set_staging_overlap(mw_ctx* c, int32_t on) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    c->staging_overlap = on != 0;
    return MW_OK;
}

mw_status mw_ctx_set_monitoring(mw_ctx* c, int32_t on) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    c->monitor = on != 0;
    if (!c->monitor) c->have_run = false;
    return MW_OK;
}

mw_status mw_ctx_set_tuning(mw_ctx* c, int32_t knob, int32_t value) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (knob < 0 || knob >= MW_TUNE_COUNT) return fail(MW_E_INVALID_SPEC, "unknown tuning knob");
    if (!mwk::tune_valid(knob, value))
        return fail(MW_E_INVALID_SPEC, "tuning value not supported for knob " + std::to_string(knob));
    if (knob == MW_TUNE_HYST_T || knob == MW_TUNE_HYST_ROWS) {   // (T, ROWS) must be a built pair
        int T = knob == MW_TUNE_HYST_T ? value : c->tune[MW_TUNE_HYST_T];
        int Rw = knob == MW_TUNE_HYST_ROWS ? value : c->tune[MW_TUNE_HYST_ROWS];
        const bool ok = (Rw == 32 && (T == 4 || T == 6 || T == 8)) || (Rw == 40 && (T == 8 || T == 12)) ||
                        (Rw == 48 && (T == 6 || T == 8));
        if (!ok)
            return fail(MW_E_INVALID_SPEC,
                        "(hyst T, rows) pair not built: use (4|6|8, 32), (8|12, 40) or (6|8, 48)");
    }
    c->tune[knob] = value;
    return MW_OK;
}

mw_status mw_ctx_get_tuning(const mw_ctx* c, int32_t knob, int32_t* value) {
    if (!c || !value) return fail(MW_E_INVALID_SPEC, "NULL argument");
    if (knob < 0 || knob >= MW_TUNE_COUNT) return fail(MW_E_INVALID_SPEC, "unknown tuning knob");
    *value = c->tune[knob];
    return MW_OK;
}

mw_status mw_ctx_launch_count(const mw_ctx* c, int64_t* out) {
    if (!c || !out) return fail(MW_E_INVALID_SPEC, "NULL argument");
    *out = (int64_t)(mwk::launch_count() - c->launches0);
    return MW_OK;
}


}  // extern "C"
