// comm.h — the exchange API every cross-partition step of the executor goes
// through (internal; the ABI is marrow.h).
//
// The paper's inter-partition data movement is four operations: the Loop's
// "global synchronization" between iterations (halo rows), the
// MapReduce merge "+" of partition partials, the re-replication of
// COPY vectors a Loop body updates and the loop condition reduced
// over partitions.  Between ranks they map onto point-to-point
// send/recv, an in-place all-reduce, an in-place broadcast per root (grouped:
// allgather-v) and an all-gather.  Two transports implement the same calls:
//   * NCCL (the product path across GPUs, NVLink / NVSwitch);
//   * loopback (test-only, MW_TRANSPORT_LOOPBACK): ranks are threads of ONE
//     process sharing a device; every operation is device copies between the
//     ranks' buffers ordered by CUDA events and two host barriers, with NCCL's
//     completion semantics (an operation has completed on a rank's stream only
//     once every rank has finished reading that rank's buffers).  It lets the
//     cross-rank branches of the executor run — and be compared with the
//     oracle — on a one-GPU box.
// All calls are stream-ordered and must be made by every rank of the group
// in the same order (marrow.h "collective rule").
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>

#include <cuda_runtime.h>

#include "marrow.h"

namespace mwc {

enum class DType : int { I32 = 0, F32 = 1, F64 = 2 };
enum class ROp : int { Sum = 0, Max = 1, Min = 2 };

class Comm {
public:
    virtual ~Comm() = default;
    virtual const char* transport() const = 0;
    // Point-to-point calls between group_start/group_end are matched per
    // peer in call order and progress together (no deadlock on send+recv).
    virtual mw_status group_start() = 0;
    virtual mw_status group_end() = 0;
    virtual mw_status send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual mw_status recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    // in place: buf[i] = op over ranks of buf[i]
    virtual mw_status allreduce(void* buf, size_t count, DType dt, ROp op, cudaStream_t s) = 0;
    // in place: every rank's buf = root's buf (inside a group: allgather-v)
    virtual mw_status broadcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
    // recv[r * bytes, (r+1) * bytes) = rank r's send (send may alias its slot)
    virtual mw_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    // asynchronous transport faults (NCCL async errors); MW_OK if none
    virtual mw_status async_error() = 0;
    // the ranks are threads of one process sharing a device (loopback):
    // device pointers are valid on every rank as they are
    virtual bool same_process() const = 0;
    // host barrier among all ranks (loopback: after every rank launched its
    // kernel of a cross-rank fused loop, so that no rank's first launch of
    // another kernel — a lazy module load, which waits for the context's
    // running kernels — can delay a peer's launch; NCCL ranks own their
    // devices: no-op)
    virtual mw_status launch_barrier() = 0;
};

// NCCL communicator from a 128-byte ncclUniqueId (collective over the group).
mw_status make_nccl(int rank, int nranks, const uint8_t id[128], std::unique_ptr<Comm>* out);
// Loopback group keyed by `id` (any 128 bytes shared by the group's threads);
// the call blocks until all nranks ranks joined (or a 120 s timeout).
mw_status make_loopback(int device, int rank, int nranks, const uint8_t id[128],
                        std::unique_ptr<Comm>* out);

}  // namespace mwc
