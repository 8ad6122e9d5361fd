// comm.cpp — NCCL and loopback transports behind comm.h.
#include "comm.h"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "mw_kernels.h"
#include "sct.h"

using mw::fail;

#define MW_OK_OR_RETURN_LB(expr)    \
    do {                            \
        mw_status s_ = (expr);      \
        if (s_ != MW_OK) return s_; \
    } while (0)

namespace mwc {
namespace {

// ------------------------------------------------------------ NCCL
ncclDataType_t nccl_dt(DType d) {
    switch (d) {
        case DType::I32: return ncclInt32;
        case DType::F32: return ncclFloat32;
        default: return ncclFloat64;
    }
}
ncclRedOp_t nccl_op(ROp o) {
    switch (o) {
        case ROp::Max: return ncclMax;
        case ROp::Min: return ncclMin;
        default: return ncclSum;
    }
}

#define NCCL_CALL(expr)                                                                     \
    do {                                                                                    \
        ncclResult_t r_ = (expr);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return fail(MW_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));     \
    } while (0)

class NcclComm final : public Comm {
public:
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) ncclCommDestroy(comm);
    }
    const char* transport() const override { return "nccl"; }
    mw_status group_start() override {
        NCCL_CALL(ncclGroupStart());
        return MW_OK;
    }
    mw_status group_end() override {
        NCCL_CALL(ncclGroupEnd());
        return MW_OK;
    }
    mw_status send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
        NCCL_CALL(ncclSend(buf, bytes, ncclUint8, peer, comm, s));
        return MW_OK;
    }
    mw_status recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
        NCCL_CALL(ncclRecv(buf, bytes, ncclUint8, peer, comm, s));
        return MW_OK;
    }
    mw_status allreduce(void* buf, size_t count, DType dt, ROp op, cudaStream_t s) override {
        NCCL_CALL(ncclAllReduce(buf, buf, count, nccl_dt(dt), nccl_op(op), comm, s));
        return MW_OK;
    }
    mw_status broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
        NCCL_CALL(ncclBroadcast(buf, buf, bytes, ncclUint8, root, comm, s));
        return MW_OK;
    }
    mw_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        NCCL_CALL(ncclAllGather(send, recv, bytes, ncclUint8, comm, s));
        return MW_OK;
    }
    bool same_process() const override { return false; }
    mw_status launch_barrier() override { return MW_OK; }
    mw_status async_error() override {
        ncclResult_t r = ncclSuccess;
        ncclCommGetAsyncError(comm, &r);
        if (r != ncclSuccess) return fail(MW_E_NCCL, std::string("NCCL: ") + ncclGetErrorString(r));
        return MW_OK;
    }
};

// ------------------------------------------------------------ loopback
enum OpKind : int { SEND = 0, RECV = 1, BCAST = 2, ALLREDUCE = 3, ALLGATHER = 4 };
struct LbOp {
    int kind;
    const void* src;   // SEND / BCAST (root) / ALLREDUCE / ALLGATHER: the rank's buffer
    void* dst;         // RECV / BCAST / ALLREDUCE / ALLGATHER
    size_t bytes;      // ALLREDUCE: count elements
    int peer;          // SEND / RECV: peer; BCAST: root
    DType dt;
    ROp op;
};

constexpr auto kTimeout = std::chrono::seconds(120);

// A rank's message to one peer for the current round between them: stage 1 =
// its operations are posted and its `ready` event recorded after the work
// that produced its buffers; stage 2 = it finished reading its peers' buffers
// (`consumed` recorded); stage 3 = it enqueued its waits on its peers'
// `consumed`, so both events may be recorded again.
struct Msg {
    uint64_t seq = 0;
    int stage = 0;
    std::vector<LbOp> ops;
    cudaEvent_t ready = nullptr, consumed = nullptr;
};

struct Hub {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    bool broken = false;
    std::vector<Msg> msg;              // [from * nranks + to]
    std::vector<uint64_t> pairseq;     // [i * nranks + j]: rounds rank i had with j
    std::vector<cudaEvent_t> ready, consumed;   // owned by their rank
    std::vector<int> joined;
    int arrived = 0;
    uint64_t gen = 0;

    // all ranks (join)
    mw_status barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return MW_OK;
        }
        if (!cv.wait_for(lk, kTimeout, [&] { return gen != g || broken; }) || broken) {
            broken = true;
            cv.notify_all();
            return fail(MW_E_NCCL, "loopback: not every rank joined the group");
        }
        return MW_OK;
    }
};

std::mutex g_reg_mu;
std::map<std::string, std::weak_ptr<Hub>> g_reg;

size_t dsize(DType d) { return d == DType::F64 ? 8 : 4; }

class Loopback final : public Comm {
public:
    std::shared_ptr<Hub> h;
    int me = 0, device = 0;
    bool grouped = false;
    std::vector<LbOp> pend;
    cudaStream_t gstream = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaStream_t tmp_stream = nullptr;

    ~Loopback() override {
        if (tmp) cudaFreeAsync(tmp, tmp_stream);
        if (h) {
            if (h->ready[me]) cudaEventDestroy(h->ready[me]);
            if (h->consumed[me]) cudaEventDestroy(h->consumed[me]);
        }
    }
    const char* transport() const override { return "loopback"; }

    mw_status add(const LbOp& o, cudaStream_t s) {
        if (grouped) {
            if (!pend.empty() && gstream != s)
                return fail(MW_E_NCCL, "loopback: a group's operations must share one stream");
            gstream = s;
            pend.push_back(o);
            return MW_OK;
        }
        pend.assign(1, o);
        return round(s);
    }
    mw_status group_start() override {
        if (grouped) return fail(MW_E_NCCL, "loopback: nested group");
        grouped = true;
        pend.clear();
        return MW_OK;
    }
    mw_status group_end() override {
        if (!grouped) return fail(MW_E_NCCL, "loopback: group_end without group_start");
        grouped = false;
        if (pend.empty()) return MW_OK;   // an empty group is a no-op
        return round(gstream);
    }
    mw_status send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
        return add({SEND, buf, nullptr, bytes, peer, DType::I32, ROp::Sum}, s);
    }
    mw_status recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
        return add({RECV, nullptr, buf, bytes, peer, DType::I32, ROp::Sum}, s);
    }
    mw_status allreduce(void* buf, size_t count, DType dt, ROp op, cudaStream_t s) override {
        return add({ALLREDUCE, buf, buf, count, -1, dt, op}, s);
    }
    mw_status broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
        return add({BCAST, buf, buf, bytes, root, DType::I32, ROp::Sum}, s);
    }
    mw_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        return add({ALLGATHER, send, recv, bytes, -1, DType::I32, ROp::Sum}, s);
    }
    mw_status async_error() override { return MW_OK; }
    bool same_process() const override { return true; }
    mw_status launch_barrier() override { return h->barrier(); }

    // post stage `st` to every peer, then wait until every peer reached it
    mw_status stage(const std::vector<int>& peers, const std::vector<uint64_t>& seq, int st) {
        const int n = h->nranks;
        std::unique_lock<std::mutex> lk(h->mu);
        for (size_t i = 0; i < peers.size(); ++i) {
            Msg& m = h->msg[(size_t)me * n + peers[i]];
            m.seq = seq[i];
            m.stage = st;
            if (st == 1) {
                m.ops = pend;
                m.ready = h->ready[me];
                m.consumed = h->consumed[me];
            }
        }
        h->cv.notify_all();
        auto reached = [&] {
            if (h->broken) return true;
            for (size_t i = 0; i < peers.size(); ++i) {
                const Msg& m = h->msg[(size_t)peers[i] * n + me];
                if (!(m.seq > seq[i] || (m.seq == seq[i] && m.stage >= st))) return false;
            }
            return true;
        };
        if (!h->cv.wait_for(lk, kTimeout, reached) || h->broken) {
            h->broken = true;
            h->cv.notify_all();
            return fail(MW_E_NCCL, "loopback: timed out waiting for a peer (ranks issued different "
                                   "exchanges)");
        }
        return MW_OK;
    }

    // One exchange among the ranks it involves (the peers of its send/recv,
    // or every rank for a collective): stage 1 publishes the operations and
    // the buffers' `ready` events; each rank then reads what it needs from its
    // peers' buffers on its own stream and records `consumed` (stage 2); it
    // waits for its peers' `consumed` (nobody reads its buffers any more)
    // before writing its in-place results; stage 3 makes event reuse safe.
    mw_status round(cudaStream_t s) {
        const int n = h->nranks;
        bool coll = false;
        std::vector<char> inv(n, 0);
        for (const LbOp& o : pend) {
            if (o.kind == SEND || o.kind == RECV) {
                if (o.peer < 0 || o.peer >= n || o.peer == me)
                    return fail(MW_E_NCCL, "loopback: bad peer " + std::to_string(o.peer));
                inv[o.peer] = 1;
            } else {
                coll = true;
            }
        }
        std::vector<int> peers;
        for (int r = 0; r < n; ++r)
            if (r != me && (coll || inv[r])) peers.push_back(r);
        std::vector<uint64_t> seq(peers.size());
        {
            std::lock_guard<std::mutex> g(h->mu);
            for (size_t i = 0; i < peers.size(); ++i) seq[i] = ++h->pairseq[(size_t)me * n + peers[i]];
        }
        size_t need = 0;
        for (const LbOp& o : pend)
            if (o.kind == ALLREDUCE) need += (o.bytes * dsize(o.dt) + 255) / 256 * 256;
        mw_status err = MW_OK;
        if (need > tmp_bytes) {
            // stream-ordered: a device-wide synchronisation here could wait for
            // another rank's kernel that is waiting for this rank
            if (tmp) cudaFreeAsync(tmp, s);
            tmp = nullptr;
            tmp_bytes = 0;
            if (cudaMallocAsync(&tmp, need, s) != cudaSuccess)
                err = fail(MW_E_OOM, "loopback: scratch allocation failed");
            else
                tmp_bytes = need;
            tmp_stream = s;
        }
        cudaEventRecord(h->ready[me], s);
        MW_OK_OR_RETURN_LB(stage(peers, seq, 1));
        // the peers' operations and events (stable until they pass stage 2)
        std::vector<std::vector<LbOp>> pops(n);
        std::vector<cudaEvent_t> pready(n, nullptr), pcons(n, nullptr);
        {
            std::lock_guard<std::mutex> g(h->mu);
            for (int r : peers) {
                const Msg& m = h->msg[(size_t)r * n + me];
                pops[r] = m.ops;
                pready[r] = m.ready;
                pcons[r] = m.consumed;
            }
        }
        pops[me] = pend;
        auto nth = [&](int r, int k, auto pred) -> const LbOp* {
            for (const LbOp& o : pops[r])
                if (pred(o) && k-- == 0) return &o;
            return nullptr;
        };
        std::vector<char> waited(n, 0);
        auto wait_for = [&](int r) {
            if (r != me && !waited[r]) {
                cudaStreamWaitEvent(s, pready[r], 0);
                waited[r] = 1;
            }
        };
        std::map<int, int> recv_k, bcast_k;
        int ar_k = 0, ag_k = 0;
        size_t toff = 0;
        struct Write {
            void* dst;
            const void* src;
            size_t bytes;
        };
        std::vector<Write> phase2;
        for (const LbOp& o : pend) {
            if (err != MW_OK) break;
            if (o.kind == SEND) continue;
            if (o.kind == RECV) {
                const int k = recv_k[o.peer]++;
                const LbOp* m = nth(o.peer, k, [&](const LbOp& x) { return x.kind == SEND && x.peer == me; });
                if (!m || m->bytes != o.bytes) {
                    err = fail(MW_E_NCCL, "loopback: recv from rank " + std::to_string(o.peer) +
                                              " has no matching send of the same size");
                    break;
                }
                wait_for(o.peer);
                if (o.bytes) cudaMemcpyAsync(o.dst, m->src, o.bytes, cudaMemcpyDeviceToDevice, s);
            } else if (o.kind == BCAST) {
                const int k = bcast_k[o.peer]++;
                if (o.peer == me) continue;
                const LbOp* m = o.peer >= 0 && o.peer < n
                                    ? nth(o.peer, k, [&](const LbOp& x) { return x.kind == BCAST && x.peer == o.peer; })
                                    : nullptr;
                if (!m || m->bytes != o.bytes) {
                    err = fail(MW_E_NCCL, "loopback: broadcast mismatch with root " + std::to_string(o.peer));
                    break;
                }
                wait_for(o.peer);
                if (o.bytes) cudaMemcpyAsync(o.dst, m->src, o.bytes, cudaMemcpyDeviceToDevice, s);
            } else if (o.kind == ALLREDUCE) {
                const int k = ar_k++;
                std::vector<const void*> srcs(n);
                for (int r = 0; r < n && err == MW_OK; ++r) {
                    const LbOp* m = nth(r, k, [](const LbOp& x) { return x.kind == ALLREDUCE; });
                    if (!m || m->bytes != o.bytes || m->dt != o.dt || m->op != o.op)
                        err = fail(MW_E_NCCL, "loopback: all-reduce mismatch with rank " + std::to_string(r));
                    else
                        srcs[r] = m->src;
                    wait_for(r);
                }
                if (err != MW_OK) break;
                void* t = static_cast<char*>(tmp) + toff;
                toff += (o.bytes * dsize(o.dt) + 255) / 256 * 256;
                if (o.bytes) {
                    cudaError_t e = mwk::reduce_ranks(srcs.data(), n, t, o.bytes, (int)o.dt, (int)o.op, s);
                    if (e != cudaSuccess) {
                        err = fail(MW_E_CUDA, std::string("loopback reduce: ") + cudaGetErrorString(e));
                        break;
                    }
                    phase2.push_back({o.dst, t, o.bytes * dsize(o.dt)});
                }
            } else if (o.kind == ALLGATHER) {
                const int k = ag_k++;
                for (int r = 0; r < n && err == MW_OK; ++r) {
                    const LbOp* m = nth(r, k, [](const LbOp& x) { return x.kind == ALLGATHER; });
                    if (!m || m->bytes != o.bytes) {
                        err = fail(MW_E_NCCL, "loopback: all-gather mismatch with rank " + std::to_string(r));
                        break;
                    }
                    void* d = static_cast<char*>(o.dst) + (size_t)r * o.bytes;
                    wait_for(r);
                    if (o.bytes && d != m->src)
                        cudaMemcpyAsync(d, m->src, o.bytes, cudaMemcpyDeviceToDevice, s);
                }
            }
        }
        cudaEventRecord(h->consumed[me], s);
        MW_OK_OR_RETURN_LB(stage(peers, seq, 2));
        for (int r : peers) cudaStreamWaitEvent(s, pcons[r], 0);
        MW_OK_OR_RETURN_LB(stage(peers, seq, 3));
        for (const Write& w : phase2) cudaMemcpyAsync(w.dst, w.src, w.bytes, cudaMemcpyDeviceToDevice, s);
        pend.clear();
        if (err == MW_OK) {
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) err = fail(MW_E_CUDA, std::string("loopback: ") + cudaGetErrorString(e));
        }
        return err;
    }
};

}  // namespace

mw_status make_nccl(int rank, int nranks, const uint8_t id[128], std::unique_ptr<Comm>* out) {
    std::unique_ptr<NcclComm> c(new NcclComm);
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "NCCL unique id size");
    memcpy(uid.internal, id, 128);
    NCCL_CALL(ncclCommInitRank(&c->comm, nranks, uid, rank));
    *out = std::move(c);
    return MW_OK;
}

mw_status make_loopback(int device, int rank, int nranks, const uint8_t id[128],
                        std::unique_ptr<Comm>* out) {
    const std::string key(reinterpret_cast<const char*>(id), 128);
    std::shared_ptr<Hub> h;
    {
        std::lock_guard<std::mutex> g(g_reg_mu);
        auto it = g_reg.find(key);
        if (it != g_reg.end()) h = it->second.lock();
        if (!h) {
            h = std::make_shared<Hub>();
            h->nranks = nranks;
            h->msg.resize((size_t)nranks * nranks);
            h->pairseq.assign((size_t)nranks * nranks, 0);
            h->ready.assign(nranks, nullptr);
            h->consumed.assign(nranks, nullptr);
            h->joined.assign(nranks, 0);
            g_reg[key] = h;
        }
        if (h->nranks != nranks) return fail(MW_E_INVALID_SPEC, "loopback: ranks disagree on nranks");
        if (h->joined[rank]) return fail(MW_E_INVALID_SPEC, "loopback: rank joined twice");
        h->joined[rank] = 1;
    }
    std::unique_ptr<Loopback> c(new Loopback);
    c->h = h;
    c->me = rank;
    c->device = device;
    {
        std::lock_guard<std::mutex> g(h->mu);
        if (cudaEventCreateWithFlags(&h->ready[rank], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->consumed[rank], cudaEventDisableTiming) != cudaSuccess)
            return fail(MW_E_CUDA, "loopback: event creation failed");
    }
    MW_OK_OR_RETURN_LB(h->barrier());   // every rank joined (collective, like ncclCommInitRank)
    if (rank == 0) {
        std::lock_guard<std::mutex> g(g_reg_mu);
        auto it = g_reg.find(key);
        if (it != g_reg.end() && it->second.lock() == h) g_reg.erase(it);
    }
    *out = std::move(c);
    return MW_OK;
}

}  // namespace mwc
