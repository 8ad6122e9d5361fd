// kcommon.cuh — helpers shared by the kernel translation units (chains.cu,
// planes.cu, nbody.cu, reduce.cu, kernels.cu): streaming loads/stores, exact
// fast division, the lowbias32 hash, launch sizing, programmatic dependent
// launch and the mbarrier / bulk-copy (TMA) primitives.  Everything is in an
// anonymous namespace (one copy per translation unit) except the launch
// counter, defined once in kernels.cu.
#pragma once
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cooperative_groups.h>
#include <math_constants.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "mw_kernels.h"

namespace cg = cooperative_groups;

namespace mwk {
extern thread_local unsigned long long g_launches;   // per host thread (one ctx per thread)
namespace {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// Exact floor(n / d) for n < 2^31 (Granlund-Montgomery: m = ceil(2^(31+s)/d),
// s = ceil(log2 d)).
struct FastDiv {
    uint32_t d;
    uint32_t shift;  // 31 + s
    uint64_t m;
};
inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    FastDiv f;
    f.d = d;
    f.shift = 31 + s;
    f.m = ((1ull << (31 + s)) + d - 1) / d;
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (uint32_t)(((uint64_t)n * f.m) >> f.shift);
}

// lowbias32 (R1): v^=v>>16; v*=0x7feb352d; v^=v>>15; v*=0x846ca68b; v^=v>>16
__device__ __forceinline__ uint32_t lowbias32(uint32_t v) {
    v ^= v >> 16;
    v *= 0x7feb352du;
    v ^= v >> 15;
    v *= 0x846ca68bu;
    v ^= v >> 16;
    return v;
}

// Tuning knobs (block shape / elements per thread): defaults are the
// measured best on B200; MW_* environment variables override them for
// sweeps (the profile-building knobs of NEXT-2).
inline int tuning_knob(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <typename K>
int resident_ctas(K kernel, int threads, size_t smem = 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess ||
        n < 1)
        n = 1;
    return n;
}

inline unsigned grid_for(int64_t tiles, int per_sm, const Launch& L) {
    int64_t g = (int64_t)sm_count() * per_sm;
    if (tiles < g) g = tiles;
    if (L.slow > 1.0f) g = (int64_t)ceil((double)g / (double)L.slow);
    return g < 1 ? 1u : (unsigned)g;
}

// Programmatic dependent launch: launched with programmatic stream
// serialization, the kernel may be scheduled while its predecessor drains;
// griddepcontrol.wait (before any global access) blocks until the
// predecessor grid has completed and its memory is visible, so ordering is
// unchanged — only the launch latency is hidden (a 2^20 saxpy is ~2 us of HBM
// time, comparable to the launch gap between graph nodes).
__device__ __forceinline__ void pdl_wait_and_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier / bulk-copy (TMA) primitives
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace
}  // namespace mwk
