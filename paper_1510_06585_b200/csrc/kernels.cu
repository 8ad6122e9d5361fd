// kernels.cu — hand-written sm_100a kernels of the Marrow hot path.
//
// Every kernel is a grid-stride ("persistent-style") loop over tiles so the
// host can size the grid to SMs x resident CTAs (and clamp it for the
// slowdown injector) without changing results.  None of these stages is a
// dense contraction, so there are no tensor cores here: the fused Map chains,
// the stencil and the reduction are HBM-bound streams (128-bit coalesced
// accesses, SWAR / DPX byte arithmetic), N-body is FP32-pipe bound.
//
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
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
namespace {

// ------------------------------------------------------------ helpers
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
FastDiv make_fastdiv(uint32_t d) {
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

int g_sms = 0;

// Tuning knobs (block shape / elements per thread): defaults are the
// measured best on B200; MW_* environment variables override them for
// sweeps (the profile-building knobs of NEXT-2).
int tuning_knob(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}
thread_local unsigned long long g_launches = 0;   // per host thread (one ctx per thread)

template <typename K>
int resident_ctas(K kernel, int threads, size_t smem = 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess ||
        n < 1)
        n = 1;
    return n;
}

unsigned grid_for(int64_t tiles, int per_sm, const Launch& L) {
    int64_t g = (int64_t)sm_count() * per_sm;
    if (tiles < g) g = tiles;
    if (L.slow > 1.0f) g = (int64_t)ceil((double)g / (double)L.slow);
    return g < 1 ? 1u : (unsigned)g;
}

// ------------------------------------------------------------ saxpy chain
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


// y_i <- fma(a_k, x_i, y_i), k = 0..n-1 (R8 single rounding).
__global__ void __launch_bounds__(256) k_saxpy_vec(const __grid_constant__ SaxpyProg p, const float4* __restrict__ x,
                                                   float4* __restrict__ y, int64_t nvec) {
    pdl_wait_and_release();
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * 256) {
        uint4 xr = ld_stream(reinterpret_cast<const uint4*>(x + i));
        float4 yv = y[i];
        float4 xv = make_float4(__uint_as_float(xr.x), __uint_as_float(xr.y),
                                __uint_as_float(xr.z), __uint_as_float(xr.w));
        for (int k = 0; k < p.n; ++k) {
            float a = p.a[k];
            yv.x = __fmaf_rn(a, xv.x, yv.x);
            yv.y = __fmaf_rn(a, xv.y, yv.y);
            yv.z = __fmaf_rn(a, xv.z, yv.z);
            yv.w = __fmaf_rn(a, xv.w, yv.w);
        }
        y[i] = yv;
    }
}
__global__ void k_saxpy_scalar(const __grid_constant__ SaxpyProg p, const float* __restrict__ x, float* __restrict__ y,
                               int64_t n) {
    pdl_wait_and_release();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float yv = y[i], xv = x[i];
        for (int k = 0; k < p.n; ++k) yv = __fmaf_rn(p.a[k], xv, yv);
        y[i] = yv;
    }
}

// ------------------------------------------------------------ RGBA chain
// Pixels are kept as two 16x2 SIMD words: rb = (R, B), ga = (G, A).
struct Px2 {
    uint32_t rb, ga;
};
__device__ __forceinline__ Px2 unpack(uint32_t w) {
    Px2 q;
    q.rb = __byte_perm(w, 0, 0x4240);
    q.ga = __byte_perm(w, 0, 0x4341);
    return q;
}
__device__ __forceinline__ uint32_t pack(const Px2& q) { return __byte_perm(q.rb, q.ga, 0x6240); }

// Gaussian noise (R1): n_c = (popc(field_c) - 5) * S; out = clamp(in + n, 0, 255).
// The add is done biased (+ popc*S, then -5S) so every lane stays >= 0 until
// VIADDMNMX.S16x2 applies "-5S then max 0" and VIMNMX.S16x2 "min 255".
__device__ __forceinline__ void noise_px(Px2& q, uint32_t h, uint32_t S, uint32_t m5s_rb,
                                         uint32_t m5s_g) {
    uint32_t pr = __popc(h & 0x3FFu), pg = __popc(h & 0xFFC00u), pb = __popc(h & 0x3FF00000u);
    q.rb += pr * S + ((pb * S) << 16);
    q.ga += pg * S;
    q.rb = __vimin_s16x2_relu(__viaddmax_s16x2(q.rb, m5s_rb, 0u), 0x00FF00FFu);
    q.ga = __vimin_s16x2_relu(__viaddmax_s16x2(q.ga, m5s_g, 0u), 0x00FF00FFu);
}
// Solarize (R2): c >= T ? 255 - c : c on R,G,B (lane bit 15 of c + 0x8000 - T).
__device__ __forceinline__ void solarize_px(Px2& q, uint32_t cT2, uint32_t cT1) {
    uint32_t mrb = ((q.rb + cT2) >> 15) & 0x00010001u;
    uint32_t mga = ((q.ga + cT1) >> 15) & 0x00000001u;
    q.rb ^= mrb * 0xFFu;
    q.ga ^= mga * 0xFFu;
}

struct RgbaConst {
    uint32_t S[kMaxOps], m5s_rb[kMaxOps], m5s_g[kMaxOps], cT2[kMaxOps], cT1[kMaxOps];
};

__device__ __forceinline__ void apply_rgba(const RgbaProg& p, const RgbaConst& c, uint32_t* w,
                                           uint32_t base, uint32_t x0, uint32_t W) {
    Px2 q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) q[e] = unpack(w[e]);
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == RGBA_NOISE) {
            const uint32_t K = p.key[k];
            const bool km = p.key_mirror[k];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t x = x0 + e;
                uint32_t idx = base + (km ? (W - 1u - x) : x);
                noise_px(q[e], lowbias32(idx ^ K), c.S[k], c.m5s_rb[k], c.m5s_g[k]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) solarize_px(q[e], c.cT2[k], c.cT1[k]);
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = pack(q[e]);
}

// 16 B (4 px) per vector; tile = 256 threads x U vectors, grid-stride.
template <int U>
__global__ void __launch_bounds__(256) k_rgba_vec(const __grid_constant__ RgbaProg p,
                                                  const __grid_constant__ RgbaConst c,
                                                  const uint4* __restrict__ src,
                                                  uint4* __restrict__ dst, uint32_t total,
                                                  FastDiv V, uint32_t W, uint32_t row0W) {
    for (uint32_t t0 = blockIdx.x * (256u * U); t0 < total; t0 += gridDim.x * (256u * U)) {
        uint4 v[U];
        uint32_t row[U], col[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                uint32_t r = fdiv(n, V);
                uint32_t cc = n - r * V.d;
                row[u] = r;
                col[u] = cc;
                v[u] = ld_stream(src + (p.mirror ? r * V.d + (V.d - 1u - cc) : n));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                if (p.mirror) {
                    uint32_t t = w[0];
                    w[0] = w[3];
                    w[3] = t;
                    t = w[1];
                    w[1] = w[2];
                    w[2] = t;
                }
                apply_rgba(p, c, w, row0W + row[u] * W, 4u * col[u], W);
                st_stream(dst + n, make_uint4(w[0], w[1], w[2], w[3]));
            }
        }
    }
}

// ---- specialised fused chain: noise -> solarize (any mirror placement).
// The fusion planner's most common RGBA program (the Filter Pipeline,
// P:725-728) gets a straight-line kernel: no per-op dispatch, the mirror and
// the noise key parity are template parameters, the hash's first xor-shift
// is folded with the key (K1 = K ^ K>>16), the three field popcounts are
// taken on left-shifted copies of h (the shifts run on the FMA pipe as
// IMAD.SHL) with the field differences folded into the noise IMADs, and for
// T = 128 solarize is min(c, 255 - c) in 16x2 SIMD lanes.
struct NsConst {
    uint32_t K1;       // K ^ (K >> 16)
    uint32_t S;        // noise scale
    uint32_t S16;      // S << 16
    uint32_t m5s_rb;   // (-5S) in both 16-bit lanes
    uint32_t m5s_g;    // (-5S) in the low lane
    uint32_t cT2, cT1; // general-T solarize constants
};

template <bool T128>
__device__ __forceinline__ uint32_t noise_solarize(uint32_t w, uint32_t idx, const NsConst& c) {
    uint32_t v = idx ^ (idx >> 16) ^ c.K1;
    v *= 0x7feb352du;
    v ^= v >> 15;
    v *= 0x846ca68bu;
    v ^= v >> 16;
    const uint32_t p10 = __popc(v << 22);          // bits 0..9   (R)
    const uint32_t p20 = __popc(v << 12);          // bits 0..19
    const uint32_t p30 = __popc(v << 2);           // bits 0..29
    uint32_t rb = w & 0x00FF00FFu;
    uint32_t ga = __byte_perm(w, 0, 0x4341);
    rb += p10 * c.S + p30 * c.S16 - p20 * c.S16;   // + pR*S, + pB*S in the high lane
    ga += p20 * c.S - p10 * c.S;                   // + pG*S
    // clamp(lane - 5S, 0, 255) in one VIADDMNMX.S16x2.RELU: relu(min(lane - 5S, 255))
    rb = __viaddmin_s16x2_relu(rb, c.m5s_rb, 0x00FF00FFu);
    ga = __viaddmin_s16x2_relu(ga, c.m5s_g, 0x00FF00FFu);
    uint32_t o = rb + ga * 256u;
    if (T128) {
        // c >= 128 -> 255 - c == c ^ 0xFF on R, G, B (alpha byte untouched)
        // byte mask 0xFF where bit 7 is set (R,G,B), 0 for alpha: one PRMT in
        // sign-replicate mode (selector nibbles 8,9,A = sign of bytes 0,1,2)
        uint32_t m;
        asm("prmt.b32 %0, %1, 0, 0x4A98;" : "=r"(m) : "r"(o));
        o ^= m;
    } else {
        uint32_t mrb = ((rb + c.cT2) >> 15) & 0x00010001u;
        uint32_t mga = ((ga + c.cT1) >> 15) & 0x00000001u;
        o ^= (mrb + mga * 256u) * 0xFFu;
    }
    return o;
}

template <int U, bool MIRROR, bool KM, bool T128>
__global__ void __launch_bounds__(256) k_rgba_ns(const __grid_constant__ NsConst c,
                                                 const uint4* __restrict__ src,
                                                 uint4* __restrict__ dst, uint32_t total,
                                                 FastDiv V, uint32_t W, uint32_t row0W) {
    for (uint32_t t0 = blockIdx.x * (256u * U); t0 < total; t0 += gridDim.x * (256u * U)) {
        uint4 v[U];
        uint32_t ib[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                const uint32_t r = fdiv(n, V);
                const uint32_t cc = n - r * V.d;
                // global noise index of the output vector's first pixel
                ib[u] = row0W + r * W + (KM ? (W - 1u - 4u * cc) : 4u * cc);
                v[u] = ld_stream(src + (MIRROR ? r * V.d + (V.d - 1u - cc) : n));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                uint32_t w0 = v[u].x, w1 = v[u].y, w2 = v[u].z, w3 = v[u].w;
                if (MIRROR) {
                    uint32_t t = w0; w0 = w3; w3 = t;
                    t = w1; w1 = w2; w2 = t;
                }
                const uint32_t i0 = ib[u];
                uint4 o;
                o.x = noise_solarize<T128>(w0, KM ? i0 : i0, c);
                o.y = noise_solarize<T128>(w1, KM ? i0 - 1u : i0 + 1u, c);
                o.z = noise_solarize<T128>(w2, KM ? i0 - 2u : i0 + 2u, c);
                o.w = noise_solarize<T128>(w3, KM ? i0 - 3u : i0 + 3u, c);
                st_stream(dst + n, o);
            }
        }
    }
}

// ---- TMA (bulk-copy) variant of the same chain.  Persistent CTAs (one per
// SM slot) stream row chunks of CH bytes through an NS-stage shared-memory
// ring: one thread issues cp.async.bulk global->smem loads completing on an
// mbarrier (expect_tx), all 256 threads run the chain smem->smem, and the
// same thread writes the result back with cp.async.bulk smem->global
// (bulk_group).  The mirror is a contiguous source segment read backwards.
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

template <int kTmaChunk, int kTmaStages, bool MIRROR, bool KM, bool T128>
__global__ void __launch_bounds__(256) k_rgba_ns_tma(const __grid_constant__ NsConst c,
                                                     const uint8_t* __restrict__ src,
                                                     uint8_t* __restrict__ dst, int64_t rows,
                                                     uint32_t W, uint32_t row0, int dep) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint4* sin = reinterpret_cast<uint4*>(smem);                                   // NS x CH
    uint4* sout = reinterpret_cast<uint4*>(smem + kTmaStages * kTmaChunk);         // NS x CH
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * kTmaStages * kTmaChunk);
    const uint32_t rowb = W * 4u;
    const uint32_t cpr = rowb / kTmaChunk;                 // chunks per row
    const int64_t n_items = rows * cpr;
    constexpr uint32_t VPC = kTmaChunk / 16;                // vectors per chunk
    constexpr uint32_t PPC = kTmaChunk / 4;                 // pixels per chunk
    auto src_of = [&](int64_t item) {                      // global source of an item
        const int64_t r = item / cpr;
        const uint32_t ch = (uint32_t)(item - r * cpr);
        const uint32_t sc = MIRROR ? (cpr - 1u - ch) : ch;   // mirrored chunk of the row
        return src + r * (int64_t)rowb + (int64_t)sc * kTmaChunk;
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // launched with programmatic stream serialization: the CTA may start
        // while the previous kernel drains; thread 0 is the only thread that
        // touches global memory (bulk copies), so it waits here for the
        // predecessor grid, then lets the next run's grid be scheduled.
        // dep == 0 (Launch::dep_wait false: the predecessor wrote nothing this
        // run reads) issues the first loads BEFORE the wait, overlapping the
        // predecessor's drain; every store still follows the wait, so each
        // grid completes after its predecessor and the stream order holds.
        if (dep) pdl_wait_and_release();
        for (int s = 0; s < kTmaStages; ++s) {
            const int64_t item = blockIdx.x + (int64_t)s * gridDim.x;
            if (item < n_items) {
                mbar_expect_tx(&bar[s], kTmaChunk);
                bulk_load(sin + s * VPC, src_of(item), kTmaChunk, &bar[s]);
            }
        }
        if (!dep) pdl_wait_and_release();
    }
    __syncthreads();
    int it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int stage = it % kTmaStages;
        const uint32_t phase = (uint32_t)(it / kTmaStages) & 1u;
        mbar_wait(&bar[stage], phase);
        if (threadIdx.x == 0) bulk_wait_read<kTmaStages - 1>();   // out[stage] free again
        __syncthreads();
        const int64_t r = item / cpr;
        const uint32_t ch = (uint32_t)(item - r * cpr);
        const uint32_t x0 = ch * PPC;                            // first output pixel
        const uint32_t rowbase = (row0 + (uint32_t)r) * W;
        const uint4* in = sin + stage * VPC;
        uint4* out = sout + stage * VPC;
#pragma unroll
        for (int k = 0; k < (int)(VPC / 256); ++k) {
            const uint32_t v = k * 256u + threadIdx.x;            // output vector in chunk
            uint4 q = in[MIRROR ? (VPC - 1u - v) : v];
            uint32_t w0 = q.x, w1 = q.y, w2 = q.z, w3 = q.w;
            if (MIRROR) {
                uint32_t t = w0; w0 = w3; w3 = t;
                t = w1; w1 = w2; w2 = t;
            }
            const uint32_t xo = x0 + 4u * v;                      // output column
            const uint32_t i0 = rowbase + (KM ? (W - 1u - xo) : xo);
            uint4 o;
            o.x = noise_solarize<T128>(w0, i0, c);
            o.y = noise_solarize<T128>(w1, KM ? i0 - 1u : i0 + 1u, c);
            o.z = noise_solarize<T128>(w2, KM ? i0 - 2u : i0 + 2u, c);
            o.w = noise_solarize<T128>(w3, KM ? i0 - 3u : i0 + 3u, c);
            out[v] = o;
        }
        fence_proxy_async();   // make the generic-proxy smem writes visible to the bulk copy
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_store(dst + r * (int64_t)rowb + (int64_t)ch * kTmaChunk, out, kTmaChunk);
            const int64_t nxt = item + (int64_t)kTmaStages * gridDim.x;
            if (nxt < n_items) {                                 // in[stage] fully consumed
                mbar_expect_tx(&bar[stage], kTmaChunk);
                bulk_load(sin + stage * VPC, src_of(nxt), kTmaChunk, &bar[stage]);
            }
        }
    }
    if (threadIdx.x == 0) bulk_wait_read<0>();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- warp-granular TMA variant: every warp owns an NS-stage ring of CH-byte
// chunks and issues its own bulk loads/stores (lane 0), synchronising only
// with __syncwarp and its own mbarriers — no CTA-wide barrier, so warps of a
// CTA stream independently.
template <int CH, int NS, int WARPS, bool MIRROR, bool KM, bool T128>
__global__ void __launch_bounds__(32 * WARPS) k_rgba_ns_tmaw(const __grid_constant__ NsConst c,
                                                             const uint8_t* __restrict__ src,
                                                             uint8_t* __restrict__ dst,
                                                             int64_t rows, uint32_t W,
                                                             uint32_t row0) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr uint32_t VPC = CH / 16, PPC = CH / 4;
    uint4* sin = reinterpret_cast<uint4*>(smem + (size_t)wid * 2 * NS * CH);
    uint4* sout = sin + NS * VPC;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * 2 * NS * CH) + wid * NS;
    const uint32_t rowb = W * 4u;
    const uint32_t cpr = rowb / CH;
    const int64_t n_items = rows * cpr;
    const int64_t gw = (int64_t)blockIdx.x * WARPS + wid, nw = (int64_t)gridDim.x * WARPS;
    auto src_of = [&](int64_t item) {
        const int64_t r = item / cpr;
        const uint32_t ch = (uint32_t)(item - r * cpr);
        const uint32_t sc = MIRROR ? (cpr - 1u - ch) : ch;
        return src + r * (int64_t)rowb + (int64_t)sc * CH;
    };
    if (lane == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < NS; ++st) {
            const int64_t item = gw + (int64_t)st * nw;
            if (item < n_items) {
                mbar_expect_tx(&bar[st], CH);
                bulk_load(sin + st * VPC, src_of(item), CH, &bar[st]);
            }
        }
    }
    __syncwarp();
    int it = 0;
    for (int64_t item = gw; item < n_items; item += nw, ++it) {
        const int stage = it % NS;
        mbar_wait(&bar[stage], (uint32_t)(it / NS) & 1u);
        if (lane == 0) bulk_wait_read<NS - 1>();   // out[stage] of NS items ago was read
        __syncwarp();
        const int64_t r = item / cpr;
        const uint32_t ch = (uint32_t)(item - r * cpr);
        const uint32_t x0 = ch * PPC;
        const uint32_t rowbase = (row0 + (uint32_t)r) * W;
        const uint4* in = sin + stage * VPC;
        uint4* out = sout + stage * VPC;
#pragma unroll
        for (int k = 0; k < (int)(VPC / 32); ++k) {
            const uint32_t v = k * 32u + lane;
            uint4 q = in[MIRROR ? (VPC - 1u - v) : v];
            uint32_t w0 = q.x, w1 = q.y, w2 = q.z, w3 = q.w;
            if (MIRROR) {
                uint32_t t = w0; w0 = w3; w3 = t;
                t = w1; w1 = w2; w2 = t;
            }
            const uint32_t xo = x0 + 4u * v;
            const uint32_t i0 = rowbase + (KM ? (W - 1u - xo) : xo);
            uint4 o;
            o.x = noise_solarize<T128>(w0, i0, c);
            o.y = noise_solarize<T128>(w1, KM ? i0 - 1u : i0 + 1u, c);
            o.z = noise_solarize<T128>(w2, KM ? i0 - 2u : i0 + 2u, c);
            o.w = noise_solarize<T128>(w3, KM ? i0 - 3u : i0 + 3u, c);
            out[v] = o;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            bulk_store(dst + r * (int64_t)rowb + (int64_t)ch * CH, out, CH);
            const int64_t nxt = item + (int64_t)NS * nw;
            if (nxt < n_items) {
                mbar_expect_tx(&bar[stage], CH);
                bulk_load(sin + stage * VPC, src_of(nxt), CH, &bar[stage]);
            }
        }
    }
    if (lane == 0) {
        bulk_wait_read<0>();
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// Any width / alignment: one pixel per element.
__global__ void __launch_bounds__(256) k_rgba_scalar(const __grid_constant__ RgbaProg p,
                                                     const __grid_constant__ RgbaConst c,
                                                     const uint32_t* __restrict__ src,
                                                     uint32_t* __restrict__ dst, uint32_t total,
                                                     FastDiv Wd, uint32_t row0W) {
    const uint32_t W = Wd.d;
    for (uint32_t n = blockIdx.x * 256u + threadIdx.x; n < total; n += gridDim.x * 256u) {
        uint32_t r = fdiv(n, Wd), x = n - r * W;
        uint32_t w = src[p.mirror ? r * W + (W - 1u - x) : n];
        Px2 q = unpack(w);
        for (int k = 0; k < p.n; ++k) {
            if (p.kind[k] == RGBA_NOISE) {
                uint32_t idx = row0W + r * W + (p.key_mirror[k] ? (W - 1u - x) : x);
                noise_px(q, lowbias32(idx ^ p.key[k]), c.S[k], c.m5s_rb[k], c.m5s_g[k]);
            } else {
                solarize_px(q, c.cT2[k], c.cT1[k]);
            }
        }
        dst[n] = pack(q);
    }
}

// ------------------------------------------------------------ u8 chain (SWAR)
// Per-byte unsigned v >= c as bit 7 (c broadcast in every byte, 0 <= c <= 255).
__device__ __forceinline__ uint32_t ge_bytes(uint32_t x, uint32_t c7, bool c_hi) {
    // d bit7 = (x & 0x7f) >= (c & 0x7f); no inter-byte borrow since each byte of
    // (x | 0x80) - (c & 0x7f) is >= 1.
    uint32_t d = (x | 0x80808080u) - c7;
    return c_hi ? (x & d & 0x80808080u) : ((x | d) & 0x80808080u);
}
// threshold t in [0, 256]: mode 0 = every byte >= t (t <= 0), 1 = none (t >= 256),
// 2 = compare with t >= 128, 3 = compare with t < 128.
__device__ __forceinline__ uint32_t ge_t(uint32_t x, uint32_t c7, int mode) {
    return mode == 0 ? 0x80808080u : (mode == 1 ? 0u : ge_bytes(x, c7, mode == 2));
}
struct U8Const {
    uint32_t lo7[kMaxOps], hi7[kMaxOps];
    int32_t lo_mode[kMaxOps], hi_mode[kMaxOps];
};
__device__ __forceinline__ uint8_t apply_u8_byte(const U8Prog& p, uint8_t v) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT)
            v = v < p.lo[k] ? 0 : (v < p.hi[k] ? 128 : 255);
        else
            v = v == 128 ? 0 : v;
    }
    return v;
}

// Apply one SEGMENT op to N words with its threshold modes fixed at compile
// time (the per-op dispatch is hoisted out of the word loop).
template <int LM, int HM, int N>
__device__ __forceinline__ void seg_words(uint32_t* w, uint32_t lo7, uint32_t hi7) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t x = w[i];
        const uint32_t flo = ge_t(x, lo7, LM), fhi = ge_t(x, hi7, HM);
        w[i] = flo | (fhi - (fhi >> 7));
    }
}
template <int N>
__device__ __forceinline__ void seg_dispatch(uint32_t* w, int lm, int hm, uint32_t lo7,
                                             uint32_t hi7) {
    switch (lm * 4 + hm) {
#define MW_SEG_CASE(A, B) \
    case A * 4 + B: seg_words<A, B, N>(w, lo7, hi7); break;
        MW_SEG_CASE(0, 0) MW_SEG_CASE(0, 1) MW_SEG_CASE(0, 2) MW_SEG_CASE(0, 3)
        MW_SEG_CASE(1, 1) MW_SEG_CASE(2, 1) MW_SEG_CASE(2, 2) MW_SEG_CASE(3, 1)
        MW_SEG_CASE(3, 2) MW_SEG_CASE(3, 3)
#undef MW_SEG_CASE
        default: break;   // unreachable for lo <= hi
    }
}

template <int N>
__device__ __forceinline__ void u8_apply_words(const U8Prog& p, const U8Const& c, uint32_t* w) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT) {
            seg_dispatch<N>(w, c.lo_mode[k], c.hi_mode[k], c.lo7[k], c.hi7[k]);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                // R11 finalize: byte == 128 -> 0 (exact zero-byte test on x ^ 0x80)
                const uint32_t x = w[i];
                const uint32_t z = ~((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
                w[i] = x & ~((z >> 7) * 0xFFu);
            }
        }
    }
}

template <int U>
__global__ void __launch_bounds__(256) k_u8_vec(const __grid_constant__ U8Prog p,
                                                const __grid_constant__ U8Const c,
                                                const uint8_t* __restrict__ src, int64_t sp,
                                                uint8_t* __restrict__ dst, int64_t dp,
                                                uint32_t total, FastDiv V) {
    for (uint32_t t0 = blockIdx.x * (256u * U); t0 < total; t0 += gridDim.x * (256u * U)) {
        uint32_t w[4 * U];
        uint32_t row[U], col[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t n = t0 + u * 256u + threadIdx.x;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (n < total) {
                const uint32_t r = fdiv(n, V);
                row[u] = r;
                col[u] = n - r * V.d;
                v = ld_stream(reinterpret_cast<const uint4*>(src + r * sp) + col[u]);
            }
            w[4 * u] = v.x;
            w[4 * u + 1] = v.y;
            w[4 * u + 2] = v.z;
            w[4 * u + 3] = v.w;
        }
        u8_apply_words<4 * U>(p, c, w);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total)
                st_stream(reinterpret_cast<uint4*>(dst + row[u] * dp) + col[u],
                          make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]));
        }
    }
}
// ---- TMA (bulk-copy) streaming variant of the u8 chain for contiguous rows
// (segmentation volumes): same ring as k_rgba_ns_tma, flat byte stream.
template <int CH, int NS>
__global__ void __launch_bounds__(256) k_u8_tma(const __grid_constant__ U8Prog p,
                                                const __grid_constant__ U8Const c,
                                                const uint8_t* __restrict__ src,
                                                uint8_t* __restrict__ dst, int64_t nbytes, int dep) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint4* sin = reinterpret_cast<uint4*>(smem);
    uint4* sout = reinterpret_cast<uint4*>(smem + NS * CH);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * NS * CH);
    const int64_t n_items = (nbytes + CH - 1) / CH;
    constexpr uint32_t VPC = CH / 16;
    auto len_of = [&](int64_t item) { return (uint32_t)min((int64_t)CH, nbytes - item * CH); };
    if (threadIdx.x == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // programmatic dependent launch, as k_rgba_ns_tma: thread 0 alone
        // touches global memory; dep == 0 reads ahead of the wait
        if (dep) pdl_wait_and_release();
        for (int st = 0; st < NS; ++st) {
            const int64_t item = blockIdx.x + (int64_t)st * gridDim.x;
            if (item < n_items) {
                mbar_expect_tx(&bar[st], len_of(item));
                bulk_load(sin + st * VPC, src + item * CH, len_of(item), &bar[st]);
            }
        }
        if (!dep) pdl_wait_and_release();
    }
    __syncthreads();
    int it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int stage = it % NS;
        mbar_wait(&bar[stage], (uint32_t)(it / NS) & 1u);
        if (threadIdx.x == 0) bulk_wait_read<NS - 1>();
        __syncthreads();
        const uint32_t nv = len_of(item) / 16;
        const uint4* in = sin + stage * VPC;
        uint4* out = sout + stage * VPC;
        constexpr int PER = VPC / 256;
        uint32_t w[4 * PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t v = k * 256u + threadIdx.x;
            const uint4 q = v < nv ? in[v] : make_uint4(0, 0, 0, 0);
            w[4 * k] = q.x; w[4 * k + 1] = q.y; w[4 * k + 2] = q.z; w[4 * k + 3] = q.w;
        }
        u8_apply_words<4 * PER>(p, c, w);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t v = k * 256u + threadIdx.x;
            if (v < nv) out[v] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        }
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_store(dst + item * CH, out, len_of(item));
            const int64_t nxt = item + (int64_t)NS * gridDim.x;
            if (nxt < n_items) {
                mbar_expect_tx(&bar[stage], len_of(nxt));
                bulk_load(sin + stage * VPC, src + nxt * CH, len_of(nxt), &bar[stage]);
            }
        }
    }
    if (threadIdx.x == 0) bulk_wait_read<0>();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_u8_scalar(const __grid_constant__ U8Prog p, const uint8_t* __restrict__ src, int64_t sp,
                            uint8_t* __restrict__ dst, int64_t dp, int64_t rows, int64_t W) {
    int64_t total = rows * W;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < total;
         n += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = n / W, x = n - r * W;
        dst[r * dp + x] = apply_u8_byte(p, src[r * sp + x]);
    }
}

// ------------------------------------------------------------ hysteresis step
// R11: L'(p) = 255 if L(p) = 128 and an 8-neighbour inside the image is 255.
// Thread = 16-byte column segment x R rows; a warp covers 512 contiguous bytes
// of a row.  Rows slide through registers (prev/cur/next horizontal strong
// masks), so each input row is loaded once per strip (+2 halo rows / strip).
// Per-byte exact equality tests (SWAR): bit 7 of each byte.
__device__ __forceinline__ uint32_t is255(uint32_t x) {
    return ~((~x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
}
__device__ __forceinline__ uint32_t is128(uint32_t x) {
    return ~((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
}

constexpr int kStencilRows = 32;
constexpr int kStencilThreads = 128;

struct Row4 {
    uint32_t w[4];
};

// strong mask of a row segment, OR-ed horizontally with its left/right bytes
__device__ __forceinline__ Row4 hmask(const uint4& v, uint32_t left_word, uint32_t right_word,
                                      int lane, bool lane_lo_edge, bool lane_hi_edge) {
    uint32_t s0 = is255(v.x), s1 = is255(v.y), s2 = is255(v.z), s3 = is255(v.w);
    // neighbouring words' strong masks across thread boundaries
    uint32_t up = __shfl_up_sync(0xffffffffu, s3, 1);     // lane-1's last word
    uint32_t dn = __shfl_down_sync(0xffffffffu, s0, 1);   // lane+1's first word
    if (lane == 0) up = is255(left_word);
    if (lane == 31) dn = is255(right_word);
    if (lane_lo_edge) up = 0;
    if (lane_hi_edge) dn = 0;
    Row4 h;
    h.w[0] = s0 | __funnelshift_l(up, s0, 8) | __funnelshift_r(s0, s1, 8);
    h.w[1] = s1 | __funnelshift_l(s0, s1, 8) | __funnelshift_r(s1, s2, 8);
    h.w[2] = s2 | __funnelshift_l(s1, s2, 8) | __funnelshift_r(s2, s3, 8);
    h.w[3] = s3 | __funnelshift_l(s2, s3, 8) | __funnelshift_r(s3, dn, 8);
    return h;
}

// Active-tile Jacobi: a tile whose 3x3 tile neighbourhood changed nothing
// in the previous execution is already at the next state in the output
// buffer (state_{k-1} == state_k == state_{k+1} there), so it is skipped —
// the iterates, the fixed point and E are exactly those of dense Jacobi.
// prev_flags == nullptr: every tile is active (first execution).
__global__ void __launch_bounds__(kStencilThreads) k_hyst_step(
    const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t rows, int64_t pitch,
    int iter, int* last_changed, int64_t n_strips, int64_t n_colblk,
    const uint8_t* __restrict__ prev_flags, uint8_t* __restrict__ cur_flags, int top_nbr,
    int bot_nbr) {
    const int lane = threadIdx.x & 31;
    const int64_t segs = pitch >> 4;  // 16-byte segments per row
    const int64_t n_tiles = n_strips * n_colblk;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t strip = t / n_colblk, cb = t - strip * n_colblk;
        bool active = prev_flags == nullptr || (top_nbr && strip == 0) ||
                      (bot_nbr && strip == n_strips - 1);
        if (!active) {
            for (int64_t ds = -1; ds <= 1 && !active; ++ds)
                for (int64_t dc = -1; dc <= 1; ++dc) {
                    const int64_t s2 = strip + ds, c2 = cb + dc;
                    if (s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_colblk &&
                        prev_flags[s2 * n_colblk + c2]) {
                        active = true;
                        break;
                    }
                }
        }
        if (!active) {   // uniform over the CTA
            if (threadIdx.x == 0) cur_flags[t] = 0;
            continue;
        }
        uint32_t changed = 0;
        const int64_t seg = cb * kStencilThreads + threadIdx.x;
        const bool valid = seg < segs;
        const int64_t y0 = strip * kStencilRows;                 // first interior row
        const int64_t y1 = min(rows, y0 + (int64_t)kStencilRows);
        const bool lo_edge = seg == 0, hi_edge = seg == segs - 1;
        // row pointer for interior row y (halo rows are y = -1 and y = rows)
        auto rowp = [&](int64_t y) { return in + (y + 1) * pitch; };
        auto load = [&](int64_t y, uint32_t& lw, uint32_t& rw) {
            const uint8_t* r = rowp(y);
            uint4 v = valid ? *reinterpret_cast<const uint4*>(r + seg * 16) : make_uint4(0, 0, 0, 0);
            lw = (lane == 0 && valid && !lo_edge) ? *reinterpret_cast<const uint32_t*>(r + seg * 16 - 4) : 0u;
            rw = (lane == 31 && valid && !hi_edge) ? *reinterpret_cast<const uint32_t*>(r + seg * 16 + 16) : 0u;
            return v;
        };
        uint32_t lw, rw;
        uint4 vprev = load(y0 - 1, lw, rw);
        Row4 hprev = hmask(vprev, lw, rw, lane, lo_edge, hi_edge);
        uint4 vcur = load(y0, lw, rw);
        Row4 hcur = hmask(vcur, lw, rw, lane, lo_edge, hi_edge);
        for (int64_t y = y0; y < y1; ++y) {
            uint4 vnext = load(y + 1, lw, rw);
            Row4 hnext = hmask(vnext, lw, rw, lane, lo_edge, hi_edge);
            uint32_t c[4] = {vcur.x, vcur.y, vcur.z, vcur.w};
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t prom = is128(c[k]) & (hprev.w[k] | hcur.w[k] | hnext.w[k]);
                changed |= prom;
                o[k] = c[k] + (prom >> 7) * 0x7Fu;   // 0x80 -> 0xFF where promoted
            }
            if (valid)
                *reinterpret_cast<uint4*>(out + (y + 1) * pitch + seg * 16) =
                    make_uint4(o[0], o[1], o[2], o[3]);
            vcur = vnext;
            hprev = hcur;
            hcur = hnext;
        }
        const int tile_changed = __syncthreads_or(changed != 0);
        if (threadIdx.x == 0) {
            cur_flags[t] = (uint8_t)tile_changed;
            if (tile_changed) atomicMax(last_changed, iter);
        }
    }
}

// ------------------------------------------------------------ hysteresis on bit planes
// When the labels entering the loop are known to be 3-valued (the stage
// before the loop ends with the threshold), the loop state is held as two
// bit planes: S (== 255) and K (== 128, constant).  One Jacobi execution is
//     S' = S | (K & dilate8(S))
// on 32 pixels per 32-bit word — the same iterates as the byte stencil, at
// 1/16 of the bytes (the 16384^2 planes are 32 MiB each and stay in L2).
// The whole while-loop runs in ONE cooperative kernel: the loop condition is
// evaluated on the device after a grid-wide barrier every execution (exact,
// no extra executions, no host round trip).  Plane layout: (rows + 2) x wp
// words, rows 0 and rows+1 zero halos; bit b of word w is pixel x = 32w + b.

__device__ __forceinline__ uint32_t nib_of(uint32_t flags80) {   // bits 7,15,23,31 -> 4 bits
    return ((flags80 >> 7) * 0x10204080u) >> 28;
}
__device__ __forceinline__ uint32_t expand_nib(uint32_t n) {      // 4 bits -> 0x00/0xFF bytes
    return ((n * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// SEG >= 0: the chain is exactly one threshold with compile-time compare modes
// (lo mode = SEG / 4, hi mode = SEG % 4); SEG < 0: any chain ending with it.
// blockIdx.y = partition (PlaneIO table: several partitions in one launch)
template <int SEG>
__global__ void __launch_bounds__(256) k_planes_pack(const __grid_constant__ U8Prog p,
                                                     const __grid_constant__ U8Const c,
                                                     const __grid_constant__ PlaneIO io, int64_t W,
                                                     int64_t wp, FastDiv WP, int hd) {
    const int q = blockIdx.y;
    const uint8_t* __restrict__ src = io.src[q];
    const int64_t sp = io.sp;
    uint32_t* __restrict__ S = io.S0[q];
    uint32_t* __restrict__ K = io.K[q];
    const uint32_t total = (uint32_t)(io.rows[q] * wp);
    uint32_t one;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(one));
    one = one > 0u ? 1u : 0u;
    for (uint32_t n = blockIdx.x * 256u + threadIdx.x; n < total; n += gridDim.x * 256u) {
        const uint32_t y = fdiv(n, WP), w = n - y * WP.d;
        const int64_t x0 = 32ll * w;
        const uint8_t* r = src + y * sp + x0;
        uint32_t v[8];
        if (x0 + 32 <= W && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
            const uint4 a = ld_stream(reinterpret_cast<const uint4*>(r));
            const uint4 b = ld_stream(reinterpret_cast<const uint4*>(r) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t x = 0;
                for (int e = 0; e < 4; ++e) {
                    const int64_t xx = x0 + 4 * i + e;
                    if (xx < W) x |= (uint32_t)r[4 * i + e] << (8 * e);
                }
                v[i] = x;
            }
        }
        uint32_t sb = 0, kb = 0;
        if constexpr (SEG >= 0) {
            // the chain is exactly the threshold: strong = v >= hi, weak = lo <= v < hi.
            // The byte msbs 7,15,23,31 land on product bits 28..31 of f * 0x00204081
            // (partial products at distinct bits: no carries), then move to 4i.
            // The nibble lands at bit 4i through a multiply-add by 2^(4i) (FMA
            // pipe; the nibbles are disjoint) — `one` is opaque to ptxas
            // (%nsmid >= 1) so it stays an IMAD instead of a shift + OR.
            // lo <= hi, so the strong flags are a subset of the v >= lo flags:
            // weak = (v >= lo) - strong, bitwise and as whole planes.
            const uint32_t l7 = c.lo7[0], h7 = c.hi7[0];
            uint32_t lb = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t fhi = ge_t(v[i], h7, SEG % 4), flo = ge_t(v[i], l7, SEG / 4);
                const uint32_t pw = one << (4 * i);
                sb = ((fhi * 0x00204081u) >> 28) * pw + sb;
                lb = ((flo * 0x00204081u) >> 28) * pw + lb;
            }
            kb = lb - sb;
        } else {
            u8_apply_words<8>(p, c, v);   // the chain before the loop (ends with the threshold)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                sb |= nib_of(is255(v[i])) << (4 * i);
                kb |= nib_of(is128(v[i])) << (4 * i);
            }
        }
        const int64_t rem = W - x0;   // bits beyond the image width stay 0
        if (rem < 32) {   // (pad words past the image: rem <= 0)
            const uint32_t keep = rem <= 0 ? 0u : (1u << rem) - 1u;
            sb &= keep;
            kb &= keep;
        }
        S[(y + hd) * wp + w] = sb;
        K[(y + hd) * wp + w] = kb;
    }
}

// Unpack when the chain after the loop is exactly finalize and a row has a
// multiple of 4096 pixels: a warp owns 4 KiB of output (128 plane words);
// lane l writes 16-byte chunk l of every 512 B, so each STG.128 of the warp
// covers 512 contiguous bytes, and the 8 plane-word loads per lane (2 lanes
// share a word) are issued before any store.  (The per-word variant below
// left every thread with one dependent L2 load per 32 bytes of output.)
__global__ void __launch_bounds__(256) k_planes_unpack_fin_w(const __grid_constant__ PlaneIO io,
                                                             const int* __restrict__ state,
                                                             int64_t dp, int64_t wp, FastDiv UPR,
                                                             int hd) {
    const int q = blockIdx.y;
    const uint32_t* S = state[2] ? io.S1[q] : io.S0[q];
    uint8_t* __restrict__ dst = io.dst[q];
    const int lane = threadIdx.x & 31;
    const uint32_t total = (uint32_t)(io.rows[q] * (wp / 128));
    for (uint32_t u = blockIdx.x * 8u + (threadIdx.x >> 5); u < total; u += gridDim.x * 8u) {
        const uint32_t y = fdiv(u, UPR), q = u - y * UPR.d;
        const uint32_t* srow = S + ((int64_t)y + hd) * wp + 128ll * q;
        uint8_t* drow = dst + (int64_t)y * dp + 4096ll * q + 16 * lane;
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = srow[(lane >> 1) + 16 * k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t h = w[k] >> (16 * (lane & 1));   // this lane's 16 pixels
            uint32_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t m = ((h >> (4 * i)) & 15u) * 0x10204080u;
                asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(v[i]) : "r"(m));
            }
            st_stream(reinterpret_cast<uint4*>(drow + 512 * k), make_uint4(v[0], v[1], v[2], v[3]));
        }
    }
}

template <bool FIN_ONLY>
__global__ void __launch_bounds__(256) k_planes_unpack(const __grid_constant__ U8Prog p,
                                                       const __grid_constant__ U8Const c,
                                                       const __grid_constant__ PlaneIO io,
                                                       const int* __restrict__ state, int64_t dp,
                                                       int64_t W, int64_t wp, FastDiv WP, int hd) {
    const int q = blockIdx.y;
    const uint32_t* S = state[2] ? io.S1[q] : io.S0[q];
    const uint32_t* __restrict__ K = io.K[q];
    uint8_t* __restrict__ dst = io.dst[q];
    const uint32_t total = (uint32_t)(io.rows[q] * wp);
    for (uint32_t n = blockIdx.x * 256u + threadIdx.x; n < total; n += gridDim.x * 256u) {
        const uint32_t y = fdiv(n, WP), w = n - y * WP.d;
        const uint32_t sb = S[(y + hd) * wp + w];
        uint32_t v[8];
        if (FIN_ONLY) {
            // the chain is exactly finalize (128 -> 0): strong pixels 255, all else 0;
            // nibble bits to byte msbs with one IMAD, then a sign-replicating PRMT
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t m = ((sb >> (4 * i)) & 15u) * 0x10204080u;
                asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(v[i]) : "r"(m));
            }
        } else {
            const uint32_t kb = K[(y + hd) * wp + w];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t bs = expand_nib((sb >> (4 * i)) & 15u);
                const uint32_t bk = expand_nib((kb >> (4 * i)) & 15u);
                v[i] = bs | (bk & 0x80808080u);   // 255 / 128 / 0 labels
            }
            u8_apply_words<8>(p, c, v);           // the chain after the loop
        }
        const int64_t x0 = 32ll * w;
        uint8_t* r = dst + y * dp + x0;
        if (x0 + 32 <= W && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
            st_stream(reinterpret_cast<uint4*>(r), make_uint4(v[0], v[1], v[2], v[3]));
            st_stream(reinterpret_cast<uint4*>(r) + 1, make_uint4(v[4], v[5], v[6], v[7]));
        } else {
            for (int e = 0; e < 32 && x0 + e < W; ++e) r[e] = (uint8_t)(v[e >> 2] >> (8 * (e & 3)));
        }
    }
}

// Temporal blocking: one pass advances the state by T Jacobi executions.  A
// warp tile holds kTbRows rows x 32 words in registers: lanes 1..30 and rows
// T..kTbRows-T-1 are owned (written back), lanes 0/31 and T rows above and
// below are halo recomputed from the neighbours (validity shrinks by one
// pixel per execution, so T <= 31 bits / T <= kTbRows/2 rows stay exact).
// Every execution inside a pass is one global Jacobi step; the device keeps
// the last execution index that changed an owned pixel, so E is exact and a
// pass that ends without change has reached the fixed point (extra in-pass
// executions past it are no-ops).  Tiles whose 3x3 tile neighbourhood did not
// change in the previous pass are skipped.  One cooperative kernel runs all
// passes; flags[pass % 3] = last changed execution of the pass (-1: none).

// One warp tile: T Jacobi executions (steps <= T) on register rows
// [strip*R - T, strip*R + R + T) x lanes, owned rows/lanes written to `out`.
// Buffers hold rows [-hd, rows + hd) at buffer row y + hd (halo rows: zero at
// the image boundary, the neighbour partition's rows otherwise); rows outside
// are zero.  Returns the last execution (0-based) that changed an owned bit.
// (Measured on B200: keeping the weak plane in registers with 256-thread CTAs
// and a rolled execution loop beats smem-resident K and a fully unrolled
// shrinking-window loop, whose code no longer fits the instruction cache.)
// One execution on register rows [LO, HI] (rows outside keep their values
// and only serve as neighbours).  Returns bit 0: an owned row [T, ROWS - T)
// of an owned lane changed; bit 1: a bit of the window inside `vm` changed.
// vm masks off the bits of lanes 0/31 whose value is no longer exact (their
// missing outer neighbour: one bit per execution from the far end).
template <int T, int ROWS, int LO, int HI>
__device__ __forceinline__ int plane_exec(uint32_t (&sv)[ROWS], const uint32_t (&kv)[ROWS],
                                          bool own_lane, uint32_t vm) {
    auto hrow = [&](uint32_t sx) {
        // lanes 0/31 take their own word as the outer neighbour: the error
        // enters at their far bits and moves one bit per execution, never
        // reaching the owned lanes (T <= 16)
        const uint32_t l = __shfl_up_sync(0xffffffffu, sx, 1);
        const uint32_t r = __shfl_down_sync(0xffffffffu, sx, 1);
        return sx | __funnelshift_l(l, sx, 1) | __funnelshift_r(sx, r, 1);
    };
    uint32_t hp = hrow(sv[LO - 1]), hc = hrow(sv[LO]);
    uint32_t ch = 0, ca = 0;
#pragma unroll
    for (int i = LO; i <= HI; ++i) {
        const uint32_t hn = hrow(sv[i + 1]);     // old row i+1 (not yet updated)
        const uint32_t s2 = sv[i] | (kv[i] & (hp | hc | hn));
        if (i >= T && i < ROWS - T) ch |= s2 ^ sv[i];
        else ca |= s2 ^ sv[i];
        sv[i] = s2;
        hp = hc;
        hc = hn;
    }
    const bool any = ((ch | ca) & vm) != 0;
    return (__any_sync(0xffffffffu, own_lane && ch != 0) ? 1 : 0) | (__any_sync(0xffffffffu, any) ? 2 : 0);
}

// T executions on a register tile (rows [ybase, ybase + ROWS) x lanes).
// Row r is exact after execution st when st < r < ROWS - 1 - st (validity
// shrinks by a row per execution at each end), so a full pass computes rows
// [1, ROWS-2] in its first T/2 executions and only [T/2 + 1, ROWS - 2 - T/2]
// in the rest (a superset of what each later execution needs); executions
// run in pairs so the updated rows alternate between two register sets
// instead of being moved back every execution.
// Early stop: the positions still exact after execution j+1 shrink by the
// stencil radius per execution (V_{j+1} within V_j), and their values depend
// only on V_j.  When execution j+1 changes nothing on (a superset of) V_{j+1},
// the true iterates j and j+1 agree there, hence by induction every later
// iterate agrees with iterate j on the smaller V_m, which contains the owned
// region: the remaining executions of the pass cannot change an owned bit,
// and the registers already hold the pass's result there.
// Returns the last execution (0-based) that changed an owned bit.
template <int T, int ROWS>
__device__ __forceinline__ int plane_steps(uint32_t (&sv)[ROWS], const uint32_t (&kv)[ROWS],
                                           int steps, bool own_lane, int lane, int* nexec = nullptr) {
    int tile_last = -1;
    int ne = 0;
    struct Cnt {   // executions run (diagnostics: MW_HYST_PROF)
        int* p; int& n;
        __device__ ~Cnt() { if (p) *p = n; }
    } cnt{nexec, ne};
    // exact bits of this lane after the next execution (lanes 0/31 lose one
    // bit per execution at their far end)
    const int shl = lane == 0, shr = lane == 31;
    uint32_t vm = ~0u;
    if (T % 4 == 0 && steps == T) {
        constexpr int H = T / 2;
#pragma unroll 1
        for (int st = 0; st < H; st += 2) {
            vm = (vm << shl) >> shr;
            ++ne;
            int r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st;
            if (!(r & 2)) return tile_last;
            vm = (vm << shl) >> shr;
            ++ne;
            r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st + 1;
            if (!(r & 2)) return tile_last;
        }
#pragma unroll 1
        for (int st = H; st < T; st += 2) {
            vm = (vm << shl) >> shr;
            ++ne;
            int r = plane_exec<T, ROWS, H + 1, ROWS - 2 - H>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st;
            if (!(r & 2)) return tile_last;
            vm = (vm << shl) >> shr;
            ++ne;
            r = plane_exec<T, ROWS, H + 1, ROWS - 2 - H>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st + 1;
            if (!(r & 2)) return tile_last;
        }
        return tile_last;
    }
#pragma unroll 1
    for (int st = 0; st < steps; ++st) {
        vm = (vm << shl) >> shr;
        ++ne;
        const int r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
        if (r & 1) tile_last = st;
        if (!(r & 2)) break;
    }
    return tile_last;
}

template <int T, int ROWS>
__device__ __forceinline__ void plane_store(const uint32_t (&sv)[ROWS], uint32_t* __restrict__ out,
                                            int64_t rows, int64_t wp, int hd, int64_t ybase,
                                            int64_t w, bool own_lane, bool wv) {
    constexpr int R = ROWS - 2 * T;
    if (!own_lane || !wv) return;
    uint32_t* o = out + (ybase + T + hd) * wp + w;    // owned row 0
    const uint32_t pw = (uint32_t)wp;
    if (ybase + T + R <= rows) {                       // every owned row inside the image
#pragma unroll
        for (int i = 0; i < R; ++i) o[i * pw] = sv[T + i];
    } else {
        const int n = (int)(rows - (ybase + T));
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (i < n) o[i * pw] = sv[T + i];
    }
}

// is tile t active: some tile of its 3x3 neighbourhood changed in the last
// execution of the previous pass (flag bit 0), the tile itself changed at any
// execution of it (bit 1: its newest state must reach this pass's output
// buffer), or it touches a partition boundary whose halo may have changed.
// A front that stopped before the last execution of a pass changes nothing
// later, and one alive at it moves at most T pixels in the next pass, which
// stays inside the 3x3 tile neighbourhood (T <= R rows, T <= 30 words).
__device__ __forceinline__ bool plane_tile_active(const uint8_t* fprev, int64_t strip, int64_t cb,
                                                  int64_t n_strips, int64_t n_cb, bool first,
                                                  int top_nbr, int bot_nbr, int lane) {
    bool act = first || (top_nbr && strip == 0) || (bot_nbr && strip == n_strips - 1);
    if (!act) {
        bool a = false;
        if (lane < 9) {
            const int64_t s2 = strip + lane / 3 - 1, c2 = cb + lane % 3 - 1;
            a = s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_cb &&
                (fprev[s2 * n_cb + c2] & (lane == 4 ? 3 : 1));
        }
        act = __any_sync(0xffffffffu, a);
    }
    return act;
}

// Whole loop, one partition per device: one cooperative kernel, all passes.
// Every warp prefetches its next active tile (S and K boxes of ROWS x 36
// words from the 16-byte-aligned column at or left of the tile's first word
// — TMA box origins are 16-byte aligned; lane l reads word o + l of a box
// row — 2-D TMA with out-of-bounds zero fill = the image-boundary rule)
// into its shared-memory slot while it computes the current one; the L2
// latency of the tile load (~2.4 us per tile measured with plain loads,
// 28 % of the loop) is hidden behind the T executions.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// One pass of a warp over its tiles (t = gw, gw + nwarps, ...): prefetch the
// next active tile into the warp's slot (sb: S box, kb: K box, bar, phase)
// while the current one runs its executions; returns the last execution
// (0-based) in which one of the warp's tiles changed an owned bit.  Buffers
// hold rows [-hd, rows + hd) at buffer row y + hd; tensor maps cover them.
template <int T, int ROWS>
__device__ __forceinline__ int plane_pass_warp(const CUtensorMap* tin, const CUtensorMap* tk,
                                               uint32_t* __restrict__ out, int64_t rows,
                                               int64_t wp, int hd, int steps,
                                               const uint8_t* __restrict__ fprev,
                                               uint8_t* __restrict__ fcur, bool all_active,
                                               int top_nbr, int bot_nbr, int64_t gw,
                                               int64_t nwarps, int lane, uint32_t* sb,
                                               uint32_t* kb, uint64_t* bar, uint32_t& phase,
                                               bool last_bit = false,
                                               unsigned long long* pstat = nullptr) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;                          // box width (words)
    constexpr uint32_t kBox = ROWS * BW * 4;        // bytes per plane box
    const int64_t n_strips = (rows + R - 1) / R;
    const int64_t n_cb = (wp + OW - 1) / OW;
    const int64_t n_tiles = n_strips * n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    // the next active tile of this warp at or after t (inactive ones are
    // marked unchanged on the way)
    auto next_active = [&](int64_t t) {
        for (; t < n_tiles; t += nwarps) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            if (plane_tile_active(fprev, strip, cb, n_strips, n_cb, all_active, top_nbr, bot_nbr, lane))
                break;
            if (lane == 0) fcur[t] = 0;
        }
        return t;
    };
    auto issue = [&](int64_t t) {
        if (lane == 0) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R - T + hd);
            mbar_expect_tx(bar, 2 * kBox);
            tma_load_2d(sb, tin, x, y, bar);
            tma_load_2d(kb, tk, x, y, bar);
        }
    };
    int my_last = -1;
    int64_t t = next_active(gw);
    if (t < n_tiles) issue(t);
    while (t < n_tiles) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        const int o = (int)((t % n_cb) * OW - 1) & 3;   // tile's first word in the box
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                               // slot free: prefetch the next tile
        const int64_t tn = next_active(t + nwarps);
        if (tn < n_tiles) issue(tn);
        const int64_t strip = t / n_cb, cb = t - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        int ne = 0;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane, pstat ? &ne : nullptr);
        if (pstat && lane == 0) {
            atomicAdd(pstat, (unsigned long long)ne);
            atomicAdd(pstat + 32, 1ull);
        }
        // bit 0: changed in the last execution of the pass (fronts still alive);
        // bit 1: changed at all.  last_bit = false: bit 0 = bit 1 (the looser
        // any-change rule; both kernels use the tight one — boundary strips of
        // a partition with a neighbour are active every pass regardless).
        const uint8_t fl = tl < 0 ? 0 : (tl == steps - 1 || !last_bit ? 3 : 2);
        my_last = max(my_last, tl);
        plane_store<T, ROWS>(sv, out, rows, wp, hd, strip * R - T, w, own_lane, w >= 0 && w < wp);
        if (lane == 0) fcur[t] = fl;
        t = tn;
    }
    return my_last;
}

// The per-warp slots of shared memory: [8][2][ROWS][36] words, then 8 mbarriers.
template <int ROWS>
constexpr size_t plane_smem_bytes() { return 8 * 2 * ROWS * 36 * 4 + 8 * 8; }
// The one-partition loop keeps TWO slots per warp: [8][2 slots][2][ROWS][36]
// words, then 16 mbarriers (221 KiB at ROWS = 48).
template <int ROWS>
constexpr size_t plane_loop_smem_bytes() { return 8 * 2 * 2 * ROWS * 36 * 4 + 16 * 8; }

// One pass of the one-partition loop for one warp.  Activity is PUSHED: a
// tile that changed an owned bit stamps itself for the next pass (its newest
// state must reach the other buffer), and one still changing in the last
// execution (a live front, which moves at most T <= R rows / 30 words in the
// next pass) stamps its 3x3 tile neighbourhood.  act[t] == stamp: t is
// active in this pass (stamps are unique per pass and run, so nothing is ever
// cleared; a stale equal value could only add work, never change a result:
// a processed tile computes the same iterates from the buffer).  The warp
// reads the stamps of its tiles (gw + i nwarps) 32 at a time, so the active
// list is known up front (no per-tile flag scan on the critical path), and
// keeps two tiles in flight in its two slots — in the sparse late passes a
// tile runs 1-2 executions, too few to hide a tile load behind.  (Measured:
// a global queue of the pass's active tiles claimed with atomics — dynamic
// balance — made every pass ~2x slower: one hot counter for ~10^4 claims.)
template <int T, int ROWS>
__device__ __forceinline__ int plane_loop_pass_warp(const CUtensorMap* tin, const CUtensorMap* tk,
                                                    uint32_t* __restrict__ out, int64_t rows,
                                                    int64_t wp, int steps, uint32_t* __restrict__ act,
                                                    uint32_t stamp, bool all_active, int64_t gw,
                                                    int64_t nwarps, int lane, uint32_t* slots,
                                                    uint64_t* bars, uint32_t& phases,
                                                    unsigned long long* pstat) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;
    constexpr uint32_t kBox = ROWS * BW * 4;
    const int64_t n_strips = (rows + R - 1) / R;
    const int64_t n_cb = (wp + OW - 1) / OW;
    const int64_t n_tiles = n_strips * n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    const int64_t n_my = gw < n_tiles ? (n_tiles - gw + nwarps - 1) / nwarps : 0;
    // active-tile generator over the warp's tiles, 32 stamps per load
    int64_t chunk = -1;
    uint32_t mask = 0;
    auto next_tile = [&]() -> int64_t {
        while (mask == 0) {
            ++chunk;
            if (chunk * 32 >= n_my) return -1;
            const int64_t i = chunk * 32 + lane;
            bool a = false;
            if (i < n_my) a = all_active || __ldcg(act + gw + i * nwarps) == stamp;
            mask = __ballot_sync(0xffffffffu, a);
        }
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        return gw + (chunk * 32 + b) * nwarps;
    };
    auto issue = [&](int64_t t, int s) {
        if (lane == 0) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R - T + 1);   // hd = 1
            uint32_t* sb = slots + s * (2 * ROWS * BW);
            mbar_expect_tx(&bars[s], 2 * kBox);
            tma_load_2d(sb, tin, x, y, &bars[s]);
            tma_load_2d(sb + ROWS * BW, tk, x, y, &bars[s]);
        }
    };
    int my_last = -1;
    int64_t cur = next_tile();
    if (cur >= 0) issue(cur, 0);
    int64_t nxt = cur >= 0 ? next_tile() : -1;
    if (nxt >= 0) issue(nxt, 1);
    int s = 0;
    while (cur >= 0) {
        mbar_wait(&bars[s], (phases >> s) & 1u);
        phases ^= 1u << s;
        const uint32_t* sb = slots + s * (2 * ROWS * BW);
        const uint32_t* kb = sb + ROWS * BW;
        const int o = (int)((cur % n_cb) * OW - 1) & 3;
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                                  // slot s free: refill it
        const int64_t n2 = nxt >= 0 ? next_tile() : -1;
        if (n2 >= 0) issue(n2, s);
        const int64_t strip = cur / n_cb, cb = cur - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        int ne = 0;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane, pstat ? &ne : nullptr);
        if (pstat && lane == 0) {
            atomicAdd(pstat, (unsigned long long)ne);
            atomicAdd(pstat + 32, 1ull);
        }
        my_last = max(my_last, tl);
        plane_store<T, ROWS>(sv, out, rows, wp, 1, strip * R - T, w, own_lane, w >= 0 && w < wp);
        if (tl >= 0) {
            const int64_t s2 = strip + lane / 3 - 1, c2 = cb + lane % 3 - 1;
            const bool nb = tl == steps - 1 ? lane < 9 : lane == 4;
            if (nb && s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_cb) act[s2 * n_cb + c2] = stamp + 1;
        }
        cur = nxt;
        nxt = n2;
        s ^= 1;
    }
    return my_last;
}

template <int T, int ROWS>
__global__ void __launch_bounds__(256) k_planes_loop(const __grid_constant__ CUtensorMap tm_s0,
                                                     const __grid_constant__ CUtensorMap tm_s1,
                                                     const __grid_constant__ CUtensorMap tm_k,
                                                     uint32_t* __restrict__ S0,
                                                     uint32_t* __restrict__ S1, int64_t rows,
                                                     int64_t wp, int64_t max_iters,
                                                     int* __restrict__ flags,
                                                     int* __restrict__ state,
                                                     uint32_t* __restrict__ act,
                                                     unsigned long long* __restrict__ prof) {
    constexpr int R = ROWS - 2 * T;
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];   // 8 x 2 warp slots, then 16 mbarriers
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * 2 * ROWS * BW);
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* slots = psm + wid * (2 * 2 * ROWS * BW);
    uint64_t* bar = &bars[2 * wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const int64_t n_tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    // act[n_tiles] = this run's stamp base (pass p is active at base + p);
    // the leader advances it past the run's stamps after the last barrier
    const uint32_t base = *((volatile uint32_t*)&act[n_tiles]);
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    if (prof && leader) prof[0] = gtime();
    uint32_t phases = 0;
    int64_t k0 = 0;
    int pass = 0;
    while (k0 < max_iters) {
        const int steps = (int)min((int64_t)T, max_iters - k0);
        if (leader) flags[(pass + 1) % 3] = -1;   // last read two barriers ago
        const int my_last = plane_loop_pass_warp<T, ROWS>(
            (pass & 1) ? &tm_s1 : &tm_s0, &tm_k, (pass & 1) ? S0 : S1, rows, wp, steps, act,
            base + (uint32_t)pass, pass == 0, gw, nwarps, lane, slots, bar, phases,
            prof && pass < 30 ? prof + 32 + pass : nullptr);
        if (lane == 0 && my_last >= 0) atomicMax(&flags[pass % 3], (int)(k0 + my_last));
        // the next pass reads `out` through the async (TMA) proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        grid.sync();
        if (prof && leader) prof[1 + pass] = gtime();
        const int last = *((volatile int*)&flags[pass % 3]);
        if (last < k0 + steps - 1) {   // the pass ended with an execution that changed nothing
            if (leader) {
                const int64_t last_global = last >= 0 ? last : k0 - 1;
                state[0] = (int)(last_global + 2);
                state[1] = 1;
                state[2] = (pass & 1) ? 0 : 1;
                act[n_tiles] = base + (uint32_t)pass + 2;
                // ready for the next run (every thread has read the flags
                // and decided to leave: -1 only confirms that decision)
                flags[0] = -1;
            }
            return;
        }
        k0 += steps;
        ++pass;
    }
    if (leader) {
        state[0] = (int)max_iters;
        state[1] = 0;
        state[2] = pass == 0 ? 0 : (((pass - 1) & 1) ? 0 : 1);
        act[n_tiles] = base + (uint32_t)pass + 2;
        flags[0] = -1;
    }
}

// One pass over one partition of several (halo depth T, host loop between
// passes exchanges T plane rows with the neighbours and reduces `last`);
// the same TMA-prefetched warp tiles as the one-partition loop.
template <int T, int ROWS>
__global__ void __launch_bounds__(256) k_planes_pass(const __grid_constant__ CUtensorMap tm_in,
                                                     const __grid_constant__ CUtensorMap tm_k,
                                                     uint32_t* __restrict__ out, int64_t rows,
                                                     int64_t wp, int steps, int64_t k0,
                                                     const uint8_t* __restrict__ fprev,
                                                     uint8_t* __restrict__ fcur, int first,
                                                     int top_nbr, int bot_nbr,
                                                     int* __restrict__ last) {
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * ROWS * BW);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* sb = psm + wid * (2 * ROWS * BW);
    uint32_t* kb = sb + ROWS * BW;
    uint64_t* bar = &bars[wid];
    if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;
    const int my_last = plane_pass_warp<T, ROWS>(
        &tm_in, &tm_k, out, rows, wp, T, steps, fprev, fcur, first != 0, top_nbr, bot_nbr,
        (int64_t)blockIdx.x * 8 + wid, (int64_t)gridDim.x * 8, lane, sb, kb, bar, phase, true);
    if (lane == 0 && my_last >= 0) atomicMax(last, (int)(k0 + my_last));
}

// Whole loop over SEVERAL partitions of one rank in one cooperative kernel.
// The partitions keep their own plane buffers with T halo rows (the layout
// of the per-pass protocol); the global tile list is the concatenation of the
// partitions' tiles.  The halo exchange between neighbouring partitions is
// folded into the store: a tile writing owned rows y < T (y >= rows - T) of
// partition q also writes them into the bottom (top) halo rows of the previous
// (next) active partition's output buffer — a pointer table, no extra pass
// and no extra barrier; the next pass reads them through TMA after the grid
// barrier.  Loop condition and exact E as in k_planes_loop.
template <int T, int ROWS>
__device__ __forceinline__ void plane_store_fwd(const uint32_t (&sv)[ROWS], const PlaneMultiArgs& a,
                                                int q, int cur, int64_t strip, int64_t w, bool own_lane,
                                                bool wv) {
    constexpr int R = ROWS - 2 * T;
    if (!own_lane || !wv) return;
    const PlanePartDesc& d = a.p[q];
    const int64_t y0 = strip * R;                      // owned row 0 of the tile
    const int64_t wp = a.wp;
    if (d.prev != -1 && y0 < T) {                      // top rows -> prev's bottom halo
        // prev == -2: the previous active rank's last partition (peer memory)
        uint32_t* base = d.prev >= 0 ? a.p[d.prev].S[cur ^ 1] : a.rprev_S[cur ^ 1];
        const int64_t prows = d.prev >= 0 ? a.p[d.prev].rows : a.rprev_rows;
        uint32_t* o = base + (prows + T + y0) * wp + w;
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (y0 + i < T && y0 + i < d.rows) o[i * wp] = sv[T + i];
    }
    if (d.next != -1 && y0 + R > d.rows - T) {         // bottom rows -> next's top halo
        uint32_t* o = (d.next >= 0 ? a.p[d.next].S[cur ^ 1] : a.rnext_S[cur ^ 1]) + w;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t y = y0 + i;
            if (y >= d.rows - T && y < d.rows) o[(y - d.rows + T) * wp] = sv[T + i];
        }
    }
}

// One pass of the multi-partition loop for one warp: the push-model activity
// and two-slot ring of plane_loop_pass_warp over the concatenated tile list.
// A live front also stamps across partition boundaries: a tile in a
// partition's first strip stamps the previous partition's last strip (and the
// one before it when that last strip has fewer than T rows — a front crosses
// it within one pass), a tile in the last strip (or in the second-to-last one
// when the last is short) the next partition's first strip.  Boundary strips
// whose neighbour is on another rank run every pass (its flags are not read).
template <int T, int ROWS>
__device__ __forceinline__ int plane_multi_pass_warp(const PlaneMultiArgs& a, int cur, int steps,
                                                     bool first, uint32_t stamp, int64_t gw,
                                                     int64_t nwarps, int lane, uint32_t* slots,
                                                     uint64_t* bars, uint32_t& phases) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;
    constexpr uint32_t kBox = ROWS * BW * 4;
    const int64_t n_cb = a.n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    if (a.total == 0) return -1;   // a rank without active partitions only joins the barriers
    uint32_t* __restrict__ act = a.act;
    const int64_t n_my = gw < a.total ? (a.total - gw + nwarps - 1) / nwarps : 0;
    auto part_of = [&](int64_t t) {
        int q = 0;
        while (q + 1 < a.np && t >= a.p[q + 1].tile0) ++q;
        return q;
    };
    auto short_last = [&](const PlanePartDesc& d) { return d.rows - (d.n_strips - 1) * R < T; };
    int64_t chunk = -1;
    uint32_t mask = 0;
    auto next_tile = [&]() -> int64_t {
        while (mask == 0) {
            ++chunk;
            if (chunk * 32 >= n_my) return -1;
            const int64_t i = chunk * 32 + lane;
            bool on = false;
            if (i < n_my) {
                const int64_t t = gw + i * nwarps;
                on = first || __ldcg(act + t) == stamp;
                if (!on) {
                    const PlanePartDesc& d = a.p[part_of(t)];
                    const int64_t strip = (t - d.tile0) / n_cb;
                    on = (d.prev == -2 && strip == 0) ||
                         (d.next == -2 && (strip == d.n_strips - 1 || (short_last(d) && strip == d.n_strips - 2)));
                }
            }
            mask = __ballot_sync(0xffffffffu, on);
        }
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        return gw + (chunk * 32 + b) * nwarps;
    };
    auto issue = [&](int64_t t, int s) {
        if (lane == 0) {
            const int q = part_of(t);
            const int64_t lt = t - a.p[q].tile0;
            const int64_t strip = lt / n_cb, cb = lt - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R);   // buffer row (hd = T)
            uint32_t* sb = slots + s * (2 * ROWS * BW);
            mbar_expect_tx(&bars[s], 2 * kBox);
            tma_load_2d(sb, &a.ts[q][cur], x, y, &bars[s]);
            tma_load_2d(sb + ROWS * BW, &a.tk[q], x, y, &bars[s]);
        }
    };
    int my_last = -1;
    int64_t t = next_tile();
    if (t >= 0) issue(t, 0);
    int64_t nxt = t >= 0 ? next_tile() : -1;
    if (nxt >= 0) issue(nxt, 1);
    int s = 0;
    while (t >= 0) {
        mbar_wait(&bars[s], (phases >> s) & 1u);
        phases ^= 1u << s;
        const int q = part_of(t);
        const PlanePartDesc& d = a.p[q];
        const int64_t lt = t - d.tile0;
        const uint32_t* sb = slots + s * (2 * ROWS * BW);
        const uint32_t* kb = sb + ROWS * BW;
        const int o = (int)((lt % n_cb) * OW - 1) & 3;
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                                  // slot s free: refill it
        const int64_t n2 = nxt >= 0 ? next_tile() : -1;
        if (n2 >= 0) issue(n2, s);
        const int64_t strip = lt / n_cb, cb = lt - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane);
        my_last = max(my_last, tl);
        const bool wv = w >= 0 && w < a.wp;
        plane_store<T, ROWS>(sv, d.S[cur ^ 1], d.rows, a.wp, T, strip * R - T, w, own_lane, wv);
        plane_store_fwd<T, ROWS>(sv, a, q, cur, strip, w, own_lane, wv);
        if (tl >= 0) {
            const bool live = tl == steps - 1;
            int64_t target = -1;
            const int64_t c2 = cb + lane % 3 - 1;
            if (lane < 9) {   // the partition's own 3x3 neighbourhood (lane 4: the tile)
                const int64_t s2 = strip + lane / 3 - 1;
                if ((live || lane == 4) && s2 >= 0 && s2 < d.n_strips && c2 >= 0 && c2 < n_cb)
                    target = d.tile0 + s2 * n_cb + c2;
            } else if (live && lane < 18 && c2 >= 0 && c2 < n_cb) {
                if (lane < 15) {   // previous partition: last strip, and the one before a short one
                    if (strip == 0 && d.prev >= 0) {
                        const PlanePartDesc& pd = a.p[d.prev];
                        if (lane < 12) target = pd.tile0 + (pd.n_strips - 1) * n_cb + c2;
                        else if (short_last(pd) && pd.n_strips >= 2) target = pd.tile0 + (pd.n_strips - 2) * n_cb + c2;
                    }
                } else if (d.next >= 0 && (strip == d.n_strips - 1 || (short_last(d) && strip == d.n_strips - 2))) {
                    target = a.p[d.next].tile0 + c2;   // next partition: first strip
                }
            }
            if (target >= 0) act[target] = stamp + 1;
        }
        t = nxt;
        nxt = n2;
        s ^= 1;
    }
    return my_last;
}

template <int T, int ROWS>
__global__ void __launch_bounds__(256, 1) k_planes_multi(const __grid_constant__ PlaneMultiArgs a,
                                                      int64_t max_iters, int* __restrict__ flags,
                                                      int* __restrict__ state,
                                                      unsigned long long* __restrict__ prof) {
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];   // 8 x 2 warp slots, then 16 mbarriers
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * 2 * ROWS * BW);
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* slots = psm + wid * (2 * 2 * ROWS * BW);
    uint64_t* bar = &bars[2 * wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    const bool xr = a.nranks > 1;
    int* own = xr ? a.xbar[a.rank] : nullptr;
    // arrivals of earlier runs (every rank ran the same passes: equal on all)
    const int epoch0 = xr && leader ? *((volatile int*)&own[1]) : 0;
    // act[total] = this run's stamp base (as in k_planes_loop)
    const uint32_t base = *((volatile uint32_t*)&a.act[a.total]);
    if (prof && leader) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        prof[0] = t;
    }
    uint32_t phases = 0;
    int64_t k0 = 0;
    int pass = 0;
    while (k0 < max_iters) {
        const int steps = (int)min((int64_t)T, max_iters - k0);
        if (leader) flags[(pass + 1) % 3] = -1;
        const int my_last = plane_multi_pass_warp<T, ROWS>(a, pass & 1, steps, pass == 0, base + (uint32_t)pass,
                                                           gw, nwarps, lane, slots, bar, phases);
        if (lane == 0 && my_last >= 0) atomicMax(&flags[pass % 3], (int)(k0 + my_last));
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xr) __threadfence_system();   // halo stores into peers before the rank barrier
        grid.sync();
        if (prof && leader && pass < 30) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[1 + pass] = t;
        }
        if (xr) {
            // rank barrier + all-reduce (max) of the last changing execution:
            // each leader publishes its value into every rank's slot, then
            // arrives on every rank's counter (release at system scope) and
            // waits for all arrivals of this pass on its own (acquire)
            if (leader) {
                const int slot = 4 + (pass % 3) * kXRanks;
                const int lv = *((volatile int*)&flags[pass % 3]);
                for (int r = 0; r < a.nranks; ++r)
                    asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(a.xbar[r] + slot + a.rank), "r"(lv)
                                 : "memory");
                __threadfence_system();
                for (int r = 0; r < a.nranks; ++r)
                    asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(a.xbar[r]) : "memory");
                const int target = epoch0 + (pass + 1) * a.nranks;
                unsigned long long t0;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                bool ok = true;
                for (;;) {
                    int cnt;
                    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(cnt) : "l"(own) : "memory");
                    if (cnt >= target) break;
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t - t0 > 10000000000ull) {   // 10 s: a rank is not running; abort
                        ok = false;
                        break;
                    }
                    __nanosleep(64);
                }
                int g = -1;
                for (int r = 0; r < a.nranks && ok; ++r) g = max(g, *((volatile int*)&own[slot + r]));
                flags[pass % 3] = ok ? g : INT_MIN;
            }
            grid.sync();
            asm volatile("fence.proxy.async.global;" ::: "memory");   // peers' halo rows, read by TMA
        }
        const int last = *((volatile int*)&flags[pass % 3]);
        if (last == INT_MIN) {   // cross-rank barrier timed out
            if (leader) {
                state[0] = (int)k0;
                state[1] = 0;
                state[2] = (pass & 1) ? 0 : 1;
                state[3] = -1;
                a.act[a.total] = base + (uint32_t)pass + 2;
                flags[0] = -1;   // ready for the next run (see k_planes_loop)
            }
            return;
        }
        if (last < k0 + steps - 1) {
            if (leader) {
                const int64_t last_global = last >= 0 ? last : k0 - 1;
                state[0] = (int)(last_global + 2);
                state[1] = 1;
                state[2] = (pass & 1) ? 0 : 1;
                state[3] = 0;
                if (xr) own[1] = epoch0 + (pass + 1) * a.nranks;
                a.act[a.total] = base + (uint32_t)pass + 2;
                flags[0] = -1;
            }
            return;
        }
        k0 += steps;
        ++pass;
    }
    if (leader) {
        state[0] = (int)max_iters;
        state[1] = 0;
        state[2] = pass == 0 ? 0 : (((pass - 1) & 1) ? 0 : 1);
        state[3] = 0;
        if (xr) own[1] = epoch0 + pass * a.nranks;
        a.act[a.total] = base + (uint32_t)pass + 2;
        flags[0] = -1;
    }
}

// ------------------------------------------------------------ N-body
// a_i = sum_j m_j d_ij (|d_ij|^2 + eps2)^-3/2 (R12): fp32 inside each
// 256-source tile (global tile boundaries, so results do not depend on the
// partitioning), fp64 across tiles.  Four bodies per thread amortise the
// shared-memory broadcast loads; MUFU.RSQ for the inverse square root.
constexpr int kNbTile = 256;
constexpr int kNbPairs = 3;               // body pairs per thread (6 bodies; 2 and 4 measured slower)
constexpr int kNbPer = 2 * kNbPairs;
// The source range is cut into kNbSeg fixed segments (tile-aligned thirds):
// work items are (body block, segment), so 2^20 bodies make 3072 items for
// 444 resident CTAs (6.9 waves, 99 % busy) instead of 1024 (2.3 waves, 77 %).
// Each item writes its fp64 partial; k_nbody_fin sums the segments in order.
// The split depends only on N, so results stay identical for every
// distribution of the bodies.
constexpr int kNbSeg = 3;

// Packed FP32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2): one instruction
// updates a pair of bodies; scalar operands are broadcast by ptxas.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& lo, float& hi) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float rsqrt_mufu(float x) {
    float r;  // MUFU.RSQ; x >= eps2 > 0 is never denormal, so .ftz is exact here
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Per interaction (for each body of a pair, in FP32x2 lanes):
//   d = p_j - p_i;  r2 = dx*dx + (dy*dy + (dz*dz + eps2));  inv = rsqrt(r2)
//   w = (m_j * inv) * (inv * inv);  f += d * w
// = 6 packed ops per coordinate triple + 6 more: 12 FP32x2 + 2 MUFU per pair.
template <bool SPLIT>
__global__ void __launch_bounds__(kNbTile) k_nbody(const float4* __restrict__ pos,
                                                   const float4* __restrict__ vel,
                                                   float4* __restrict__ pos_out,
                                                   float4* __restrict__ vel_out,
                                                   float4* __restrict__ acc_out, int64_t first,
                                                   int64_t count, int64_t N, float eps2, float dt,
                                                   int mode, double* __restrict__ part) {
    __shared__ float4 sp[kNbTile];
    __shared__ float2 bp[3][kNbPairs][kNbTile];
    const int64_t per_blk = (int64_t)kNbTile * kNbPer;
    const int64_t nblk = (count + per_blk - 1) / per_blk;
    const int64_t ntiles = (N + kNbTile - 1) / kNbTile;
    for (int64_t w = blockIdx.x; w < nblk * kNbSeg; w += gridDim.x) {
        const int64_t b = w / kNbSeg;
        const int seg = (int)(w - b * kNbSeg);
        const int64_t j0 = (ntiles * seg / kNbSeg) * kNbTile;
        const int64_t j1e = (ntiles * (seg + 1) / kNbSeg) * kNbTile;
        const int64_t j1 = j1e < N ? j1e : N;
        double ax[kNbPer], ay[kNbPer], az[kNbPer];
        // body positions live only as packed pairs (one aligned register pair each)
        f2_t px[kNbPairs], py[kNbPairs], pz[kNbPairs];
        // stage the pairs through shared memory so each lands in an aligned
        // register pair straight from an LDS.64 (no per-use re-pairing MOVs)
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kNbPairs; ++h) {
            float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f), b4 = a4;
            const int64_t la = b * per_blk + (2 * h) * kNbTile + threadIdx.x;
            const int64_t lb = la + kNbTile;
            if (la < count) a4 = pos[first + la];
            if (lb < count) b4 = pos[first + lb];
            bp[0][h][threadIdx.x] = make_float2(a4.x, b4.x);
            bp[1][h][threadIdx.x] = make_float2(a4.y, b4.y);
            bp[2][h][threadIdx.x] = make_float2(a4.z, b4.z);
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kNbPairs; ++h) {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(px[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[0][h][threadIdx.x])));
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(py[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[1][h][threadIdx.x])));
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(pz[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[2][h][threadIdx.x])));
        }
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) ax[q] = ay[q] = az[q] = 0.0;
        const f2_t e2 = f2_pack(eps2, eps2);
        for (int64_t jt = j0; jt < j1; jt += kNbTile) {
            __syncthreads();
            const int64_t j = jt + threadIdx.x;
            sp[threadIdx.x] = j < N ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass-0 pads
            __syncthreads();
            f2_t fx[kNbPairs], fy[kNbPairs], fz[kNbPairs];   // packed accumulators
            float gx[kNbPer], gy[kNbPer], gz[kNbPer];        // scalar accumulators (SPLIT)
#pragma unroll
            for (int h = 0; h < kNbPairs; ++h) fx[h] = fy[h] = fz[h] = 0ull;
#pragma unroll
            for (int q = 0; q < kNbPer; ++q) gx[q] = gy[q] = gz[q] = 0.f;
#pragma unroll 8
            for (int k = 0; k < kNbTile; ++k) {
                const float4 s4 = sp[k];
                const f2_t sx = f2_pack(s4.x, s4.x), sy = f2_pack(s4.y, s4.y),
                           sz = f2_pack(s4.z, s4.z), sw = f2_pack(s4.w, s4.w);
#pragma unroll
                for (int h = 0; h < kNbPairs; ++h) {
                    const f2_t dx = f2_sub(sx, px[h]), dy = f2_sub(sy, py[h]),
                               dz = f2_sub(sz, pz[h]);
                    const f2_t r2 = f2_fma(dx, dx, f2_fma(dy, dy, f2_fma(dz, dz, e2)));
                    float r0, r1;
                    f2_unpack(r2, r0, r1);
                    const f2_t inv = f2_pack(rsqrt_mufu(r0), rsqrt_mufu(r1));
                    if (SPLIT) {
                        // 8 packed ops on the FMA-heavy pipe, 8 scalar ops free to
                        // issue to the FMA-lite pipe (same roundings as the packed form)
                        const f2_t t = f2_mul(sw, inv), i2 = f2_mul(inv, inv);
                        float t0, t1, q0, q1, x0, x1, y0, y1, z0, z1;
                        f2_unpack(t, t0, t1);
                        f2_unpack(i2, q0, q1);
                        f2_unpack(dx, x0, x1);
                        f2_unpack(dy, y0, y1);
                        f2_unpack(dz, z0, z1);
                        const float w0 = t0 * q0, w1 = t1 * q1;
                        gx[2 * h] = __fmaf_rn(x0, w0, gx[2 * h]);
                        gx[2 * h + 1] = __fmaf_rn(x1, w1, gx[2 * h + 1]);
                        gy[2 * h] = __fmaf_rn(y0, w0, gy[2 * h]);
                        gy[2 * h + 1] = __fmaf_rn(y1, w1, gy[2 * h + 1]);
                        gz[2 * h] = __fmaf_rn(z0, w0, gz[2 * h]);
                        gz[2 * h + 1] = __fmaf_rn(z1, w1, gz[2 * h + 1]);
                    } else {
                        const f2_t w = f2_mul(f2_mul(sw, inv), f2_mul(inv, inv));
                        fx[h] = f2_fma(dx, w, fx[h]);
                        fy[h] = f2_fma(dy, w, fy[h]);
                        fz[h] = f2_fma(dz, w, fz[h]);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < kNbPairs; ++h) {
                float x0, x1, y0, y1, z0, z1;
                f2_unpack(fx[h], x0, x1);
                f2_unpack(fy[h], y0, y1);
                f2_unpack(fz[h], z0, z1);
                if (SPLIT) {
                    x0 = gx[2 * h]; x1 = gx[2 * h + 1];
                    y0 = gy[2 * h]; y1 = gy[2 * h + 1];
                    z0 = gz[2 * h]; z1 = gz[2 * h + 1];
                }
                ax[2 * h] += (double)x0; ax[2 * h + 1] += (double)x1;
                ay[2 * h] += (double)y0; ay[2 * h + 1] += (double)y1;
                az[2 * h] += (double)z0; az[2 * h + 1] += (double)z1;
            }
        }
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) {
            const int64_t l = b * per_blk + q * kNbTile + threadIdx.x;
            if (l >= count) continue;
            double* o = part + (seg * count + l) * 3;
            o[0] = ax[q];
            o[1] = ay[q];
            o[2] = az[q];
        }
    }
}

// Sum the segment partials in order, then the epilogue: mode 1 writes a_i;
// mode 0 the symplectic Euler step (fp64 update, fp32 state).
__global__ void k_nbody_fin(const double* __restrict__ part, const float4* __restrict__ pos,
                            const float4* __restrict__ vel, float4* __restrict__ pos_out,
                            float4* __restrict__ vel_out, float4* __restrict__ acc_out,
                            int64_t first, int64_t count, float dt, int mode) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < count;
         l += (int64_t)gridDim.x * blockDim.x) {
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
        for (int sgi = 0; sgi < kNbSeg; ++sgi) {
            const double* o = part + (sgi * count + l) * 3;
            ax += o[0];
            ay += o[1];
            az += o[2];
        }
        const int64_t i = first + l;
        if (mode == 1) {
            acc_out[l] = make_float4((float)ax, (float)ay, (float)az, 0.f);
        } else {
            const float4 v = vel[i];
            const float4 pq = pos[i];
            const double d = (double)dt;
            const double vx = (double)v.x + ax * d, vy = (double)v.y + ay * d,
                         vz = (double)v.z + az * d;
            vel_out[i] = make_float4((float)vx, (float)vy, (float)vz, v.w);
            pos_out[i] = make_float4((float)((double)pq.x + vx * d),
                                     (float)((double)pq.y + vy * d),
                                     (float)((double)pq.z + vz * d), pq.w);
        }
    }
}

// ------------------------------------------------------------ MapReduce
// One CTA per canonical 2^16-element chunk; thread t folds elements
// (k*256 + t)*4 + e, k = 0..63, into accumulator e = 0..3 in fp64 (each fp32
// converted exactly; products x*y exact in fp64), then a fixed xor-shuffle
// tree and a fixed 8-warp tree.  The order depends only on global chunk
// boundaries, so every distribution vector gives bit-identical partials.
// OP (MW_REDUCE_*): 0 = fp64 sum; 1 / 2 = maxNum / minNum of the exactly
// converted terms (a NaN term is ignored), exact in any order.
constexpr int kRedThreads = 256;

template <int OP>
__device__ __forceinline__ double red_op(double a, double b) {
    if constexpr (OP == 0) return a + b;
    else if constexpr (OP == 1) return fmax(a, b);
    else return fmin(a, b);
}
template <int OP>
__device__ __forceinline__ double red_id() {
    return OP == 0 ? 0.0 : (OP == 1 ? -CUDART_INF : CUDART_INF);
}
// one term into the accumulator: sum folds with an fma for products; TM
// (reduction-stage term map): 0 none, 1 |t|, 2 t*t (fp64) before the fold
template <int OP, bool DOT, int TM = 0>
__device__ __forceinline__ double red_term(double acc, float a, float b) {
    if constexpr (TM == 0) {
        if constexpr (OP == 0) return DOT ? __fma_rn((double)a, (double)b, acc) : acc + (double)a;
        else return red_op<OP>(acc, DOT ? (double)a * (double)b : (double)a);
    } else {
        const double t = DOT ? (double)a * (double)b : (double)a;
        return red_op<OP>(acc, TM == 1 ? fabs(t) : t * t);
    }
}

// PRE: the map stage is pipeline(saxpy chain, map_product) fused into the
// reduction: the second operand is y' = fma(a_k, x, y) (k = 0..pre.n-1, fp32,
// one rounding each, as the saxpy leaf) computed in registers, never stored.
template <bool PRE>
__device__ __forceinline__ float pre_y(const SaxpyProg& pre, float x, float y) {
    if (PRE)
        for (int k = 0; k < pre.n; ++k) y = __fmaf_rn(pre.a[k], x, y);
    return y;
}

template <bool DOT, int OP, bool PRE = false, int TM = 0>
__global__ void __launch_bounds__(kRedThreads) k_reduce_chunks(const float* __restrict__ x,
                                                               const float* __restrict__ y,
                                                               int64_t x0, int64_t first_chunk,
                                                               int64_t n_chunks, int64_t total,
                                                               double* __restrict__ partials,
                                                               const __grid_constant__ SaxpyProg pre) {
    __shared__ double warp_part[kRedThreads / 32];
    const int64_t CH = 1ll << kChunkLog2;
    for (int64_t cc = blockIdx.x; cc < n_chunks; cc += gridDim.x) {
        const int64_t c = first_chunk + cc;
        const int64_t gbase = c * CH;
        const int64_t len = min(CH, total - gbase);
        const int64_t base = gbase - x0;  // local index of the chunk's first element
        // four independent accumulators (element e of each 4-vector), joined
        // as (a0 . a1) . (a2 . a3): a fixed order, so partials stay
        // independent of the partitioning; four chains instead of one
        // dependent chain of 256 fp64 operations per thread
        double acc4[4] = {red_id<OP>(), red_id<OP>(), red_id<OP>(), red_id<OP>()};
        const bool vec = len == CH && ((reinterpret_cast<uintptr_t>(x + base) & 15) == 0) &&
                         (!DOT || ((reinterpret_cast<uintptr_t>(y + base) & 15) == 0));
        if (vec) {
            const uint4* xv = reinterpret_cast<const uint4*>(x + base);
            const uint4* yv = reinterpret_cast<const uint4*>(DOT ? y + base : x + base);
#pragma unroll 8
            for (int k = 0; k < (int)(CH / 4 / kRedThreads); ++k) {
                uint4 a = ld_stream(xv + k * kRedThreads + threadIdx.x);
                uint4 b = a;
                if (DOT) b = ld_stream(yv + k * kRedThreads + threadIdx.x);
                const float ax = __uint_as_float(a.x), ay = __uint_as_float(a.y);
                const float az = __uint_as_float(a.z), aw = __uint_as_float(a.w);
                acc4[0] = red_term<OP, DOT, TM>(acc4[0], ax, pre_y<PRE>(pre, ax, __uint_as_float(b.x)));
                acc4[1] = red_term<OP, DOT, TM>(acc4[1], ay, pre_y<PRE>(pre, ay, __uint_as_float(b.y)));
                acc4[2] = red_term<OP, DOT, TM>(acc4[2], az, pre_y<PRE>(pre, az, __uint_as_float(b.z)));
                acc4[3] = red_term<OP, DOT, TM>(acc4[3], aw, pre_y<PRE>(pre, aw, __uint_as_float(b.w)));
            }
        } else {
            for (int k = 0; k < (int)(CH / 4 / kRedThreads); ++k) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    int64_t i = ((int64_t)k * kRedThreads + threadIdx.x) * 4 + e;
                    if (i < len)
                        acc4[e] = red_term<OP, DOT, TM>(acc4[e], x[base + i],
                                                        DOT ? pre_y<PRE>(pre, x[base + i], y[base + i]) : 0.f);
                }
            }
        }
        double acc = red_op<OP>(red_op<OP>(acc4[0], acc4[1]), red_op<OP>(acc4[2], acc4[3]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = red_op<OP>(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = red_id<OP>();
#pragma unroll
            for (int w = 0; w < kRedThreads / 32; ++w) s = red_op<OP>(s, warp_part[w]);
            partials[c] = s;
        }
        __syncthreads();
    }
}

template <int OP>
__global__ void __launch_bounds__(1024) k_reduce_combine(const double* __restrict__ partials,
                                                         int64_t n, double* __restrict__ result,
                                                         const __grid_constant__ ScalarPost post) {
    __shared__ double wp[32];
    double acc = red_id<OP>();
    for (int64_t i = threadIdx.x; i < n; i += 1024) acc = red_op<OP>(acc, partials[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = red_op<OP>(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double s = wp[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = red_op<OP>(s, __shfl_xor_sync(0xffffffffu, s, o));
        // reduction-stage scalar maps of the reduced value, in order
        for (int k = 0; k < post.n; ++k) s = post.kind[k] == 0 ? sqrt(s) : s * post.c[k];
        if (threadIdx.x == 0) *result = s;
    }
}

template <int OP>
__global__ void k_fill_identity(double* __restrict__ p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = red_id<OP>();
}

__global__ void k_traits(int64_t* out, int64_t count, int64_t size, int64_t offset) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        out[2 * i] = size;
        out[2 * i + 1] = offset;
    }
}

}  // namespace

// ============================================================ launchers
unsigned long long launch_count() { return g_launches; }
void note_launch() { ++g_launches; }

void tune_defaults(int* out) {
    out[TUNE_RGBA_TMA] = tuning_knob("MW_RGBA_TMA", 1);        // 16 KiB x 3 stages
    out[TUNE_RGBA_UNROLL] = tuning_knob("MW_RGBA_UNROLL", 2);
    out[TUNE_HYST_PLANES] = tuning_knob("MW_HYST_PLANES", 1);
    out[TUNE_HYST_T] = tuning_knob("MW_HYST_T", 8);
    out[TUNE_HYST_ROWS] = tuning_knob("MW_HYST_ROWS", 48);   // (8, 48): 0.407 vs 0.44 ms (8, 40)
    out[TUNE_NBODY_SPLIT] = tuning_knob("MW_NBODY_SPLIT", 0);
    out[TUNE_U8_TMA] = tuning_knob("MW_U8_TMA", 1);
    out[TUNE_HYST_FUSED] = tuning_knob("MW_HYST_FUSED", 1);
    out[TUNE_GRAPH_LANES] = tuning_knob("MW_GRAPH_LANES", 4);
    for (int k = 0; k < TUNE_COUNT; ++k)
        if (!tune_valid(k, out[k])) {   // ignore malformed overrides
            const int d[TUNE_COUNT] = {1, 2, 1, 8, 48, 0, 1, 1, 4};
            out[k] = d[k];
        }
}

bool tune_valid(int knob, int v) {
    switch (knob) {
        case TUNE_RGBA_TMA: return v >= 0 && v <= 9;
        case TUNE_RGBA_UNROLL: return v == 2 || v == 4 || v == 8;
        case TUNE_HYST_PLANES: return v == 0 || v == 1;
        case TUNE_HYST_T: return v == 4 || v == 6 || v == 8 || v == 12;
        case TUNE_HYST_ROWS: return v == 32 || v == 40 || v == 48;
        case TUNE_NBODY_SPLIT: return v == 0 || v == 1;
        case TUNE_U8_TMA: return v == 0 || v == 1;
        case TUNE_HYST_FUSED: return v == 0 || v == 1;
        case TUNE_GRAPH_LANES: return v == 1 || v == 2 || v == 4;
    }
    return false;
}

int sm_count() {
    if (g_sms == 0) {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
            n = 148;
        g_sms = n;
    }
    return g_sms;
}

cudaError_t saxpy_chain(const SaxpyProg& p, const float* x, float* y, int64_t n, const Launch& L) {
    if (n <= 0) return cudaSuccess;
    static int occ_v = resident_ctas(k_saxpy_vec, 256), occ_s = resident_ctas(k_saxpy_scalar, 256);
    bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    int64_t nv = al ? n / 4 : 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.stream = L.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (nv > 0) {
        ++g_launches;
        cfg.gridDim = dim3(grid_for((nv + 255) / 256, occ_v, L));
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_saxpy_vec, p, reinterpret_cast<const float4*>(x),
                                           reinterpret_cast<float4*>(y), nv);
        if (e != cudaSuccess) return e;
    }
    int64_t rest = n - nv * 4;
    if (rest > 0) {
        ++g_launches;
        cfg.gridDim = dim3(grid_for((rest + 255) / 256, occ_s, L));
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_saxpy_scalar, p, x + nv * 4, y + nv * 4, rest);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t rgba_chain(const RgbaProg& p, const uint8_t* src, uint8_t* dst, int64_t rows,
                       int64_t W, int64_t row0, const Launch& L) {
    if (rows <= 0 || W <= 0) return cudaSuccess;
    if ((row0 + rows) * W > 0xFFFFFFFFll) return cudaErrorInvalidValue;  // idx is u32 (R1)
    RgbaConst c;
    for (int k = 0; k < p.n; ++k) {
        uint32_t S = (uint32_t)p.param[k];
        c.S[k] = S;
        c.m5s_rb[k] = ((0u - 5u * S) & 0xFFFFu) * 0x10001u;
        c.m5s_g[k] = (0u - 5u * S) & 0xFFFFu;
        uint32_t T = (uint32_t)p.param[k];
        c.cT2[k] = (0x8000u - T) * 0x10001u;
        c.cT1[k] = 0x8000u - T;
    }
    const uint32_t row0W = (uint32_t)(row0 * W);
    const bool vec = (W % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    if (vec && p.n == 2 && p.kind[0] == RGBA_NOISE && p.kind[1] == RGBA_SOLARIZE) {
        NsConst nc;
        const uint32_t K = p.key[0], S = (uint32_t)p.param[0];
        nc.K1 = K ^ (K >> 16);
        nc.S = S;
        nc.S16 = S << 16;
        nc.m5s_rb = c.m5s_rb[0];
        nc.m5s_g = c.m5s_g[0];
        nc.cT2 = c.cT2[1];
        nc.cT1 = c.cT1[1];
        const bool t128 = p.param[1] == 128;
        const uint32_t total = (uint32_t)(rows * W / 4);
        const FastDiv V = make_fastdiv((uint32_t)(W / 4));
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        // TMA path: chunk bytes x stages per CTA (tuning knob MW_RGBA_TMA:
        // 0 = LSU path, 1 = 16 KiB x 3 (measured best), 2 = 8 KiB x 4, 3 = 8 KiB x 3,
        // 4 = 4 KiB x 4, 5 = 32 KiB x 3, 6 = 16 KiB x 6)
        const int tma_cfg = L.tune[TUNE_RGBA_TMA];
        const int chunk = (tma_cfg == 1 || tma_cfg == 6 || tma_cfg == 9) ? 16384
                          : ((tma_cfg == 4 || tma_cfg == 7) ? 4096 : (tma_cfg == 5 ? 32768 : 8192));
        if ((tma_cfg == 7 || tma_cfg == 8) && (W * 4) % chunk == 0 &&
            ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
#define MW_TMAW_LAUNCH(CH, NS, WP, MI, KMI, TI)                                               \
    do {                                                                                       \
        constexpr size_t smem = (size_t)WP * 2 * NS * CH + WP * NS * 8;                        \
        static int occ = [] {                                                                  \
            cudaFuncSetAttribute(k_rgba_ns_tmaw<CH, NS, WP, MI, KMI, TI>,                      \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
            return resident_ctas(k_rgba_ns_tmaw<CH, NS, WP, MI, KMI, TI>, 32 * WP, smem);      \
        }();                                                                                   \
        const int64_t items = rows * (W * 4 / CH);                                             \
        ++g_launches;                                                                          \
        k_rgba_ns_tmaw<CH, NS, WP, MI, KMI, TI>                                                \
            <<<grid_for((items + WP - 1) / WP, occ, L), 32 * WP, smem, L.stream>>>(            \
                nc, src, dst, rows, (uint32_t)W, (uint32_t)row0);                              \
    } while (0)
#define MW_TMAW_CFG(MI, KMI, TI)                                                               \
    do {                                                                                       \
        if (tma_cfg == 7) MW_TMAW_LAUNCH(4096, 3, 8, MI, KMI, TI);                             \
        else MW_TMAW_LAUNCH(8192, 2, 6, MI, KMI, TI);                                          \
    } while (0)
            const int selw = (p.mirror ? 4 : 0) | (p.key_mirror[0] ? 2 : 0) | (t128 ? 1 : 0);
            switch (selw) {
                case 0: MW_TMAW_CFG(false, false, false); break;
                case 1: MW_TMAW_CFG(false, false, true); break;
                case 2: MW_TMAW_CFG(false, true, false); break;
                case 3: MW_TMAW_CFG(false, true, true); break;
                case 4: MW_TMAW_CFG(true, false, false); break;
                case 5: MW_TMAW_CFG(true, false, true); break;
                case 6: MW_TMAW_CFG(true, true, false); break;
                default: MW_TMAW_CFG(true, true, true); break;
            }
#undef MW_TMAW_CFG
#undef MW_TMAW_LAUNCH
            return cudaGetLastError();
        }
        // default (1): 16 KiB x 2 stages (three CTAs per SM) for launches of at
        // least 8 waves of chunks, 16 KiB x 3 (two CTAs per SM, fewer tail
        // rounds) below — measured 89.3 vs 92.7 us at 8192 rows, 25.3 vs
        // 26.3 us at 2048 rows, 17.1 vs 15.1 us at 1024 rows
        const bool big = rows * (W * 4 / 16384) >= 8ll * sm_count() * 3;
        if (tma_cfg > 0 && (W * 4) % chunk == 0 &&
            ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
#define MW_TMA_LAUNCH(CH, NS, MI, KMI, TI)                                                     \
    do {                                                                                       \
        constexpr size_t smem = 2 * NS * CH + 64;                                              \
        static int occ = [] {                                                                  \
            cudaFuncSetAttribute(k_rgba_ns_tma<CH, NS, MI, KMI, TI>,                           \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
            return resident_ctas(k_rgba_ns_tma<CH, NS, MI, KMI, TI>, 256, smem);               \
        }();                                                                                   \
        const int64_t items = rows * (W * 4 / CH);                                             \
        ++g_launches;                                                                          \
        cudaLaunchAttribute at[1];                                                             \
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                         \
        at[0].val.programmaticStreamSerializationAllowed = 1;                                  \
        cudaLaunchConfig_t cfg = {};                                                           \
        cfg.gridDim = dim3(grid_for(items, occ, L));                                           \
        cfg.blockDim = dim3(256);                                                              \
        cfg.dynamicSmemBytes = smem;                                                           \
        cfg.stream = L.stream;                                                                 \
        cfg.attrs = at;                                                                        \
        cfg.numAttrs = 1;                                                                      \
        cudaLaunchKernelEx(&cfg, k_rgba_ns_tma<CH, NS, MI, KMI, TI>, nc, src, dst, rows,       \
                           (uint32_t)W, (uint32_t)row0, (int)L.dep_wait);                      \
    } while (0)
#define MW_TMA_CFG(MI, KMI, TI)                                                                \
    do {                                                                                       \
        if (tma_cfg == 1 && big) MW_TMA_LAUNCH(16384, 2, MI, KMI, TI);                         \
        else if (tma_cfg == 1) MW_TMA_LAUNCH(16384, 3, MI, KMI, TI);                           \
        else if (tma_cfg == 9) MW_TMA_LAUNCH(16384, 2, MI, KMI, TI);                           \
        else if (tma_cfg == 5) MW_TMA_LAUNCH(32768, 3, MI, KMI, TI);                           \
        else if (tma_cfg == 6) MW_TMA_LAUNCH(16384, 6, MI, KMI, TI);                           \
        else if (tma_cfg == 3) MW_TMA_LAUNCH(8192, 3, MI, KMI, TI);                            \
        else if (tma_cfg == 4) MW_TMA_LAUNCH(4096, 4, MI, KMI, TI);                            \
        else MW_TMA_LAUNCH(8192, 4, MI, KMI, TI);                                              \
    } while (0)
            const int sel = (p.mirror ? 4 : 0) | (p.key_mirror[0] ? 2 : 0) | (t128 ? 1 : 0);
            switch (sel) {
                case 0: MW_TMA_CFG(false, false, false); break;
                case 1: MW_TMA_CFG(false, false, true); break;
                case 2: MW_TMA_CFG(false, true, false); break;
                case 3: MW_TMA_CFG(false, true, true); break;
                case 4: MW_TMA_CFG(true, false, false); break;
                case 5: MW_TMA_CFG(true, false, true); break;
                case 6: MW_TMA_CFG(true, true, false); break;
                default: MW_TMA_CFG(true, true, true); break;
            }
#undef MW_TMA_CFG
#undef MW_TMA_LAUNCH
            return cudaGetLastError();
        }
        const int unroll = L.tune[TUNE_RGBA_UNROLL];
#define MW_NS_LAUNCH_U(U, MI, KMI, TI)                                                    \
    do {                                                                                  \
        static int occ = resident_ctas(k_rgba_ns<U, MI, KMI, TI>, 256);                   \
        const int64_t tiles = (total + 256 * U - 1) / (256 * U);                          \
        ++g_launches;                                                                     \
        k_rgba_ns<U, MI, KMI, TI><<<grid_for(tiles, occ, L), 256, 0, L.stream>>>(         \
            nc, s4, d4, total, V, (uint32_t)W, row0W);                                    \
    } while (0)
#define MW_NS_LAUNCH(MI, KMI, TI)                                                         \
    do {                                                                                  \
        if (unroll == 2) MW_NS_LAUNCH_U(2, MI, KMI, TI);                                  \
        else if (unroll == 8) MW_NS_LAUNCH_U(8, MI, KMI, TI);                             \
        else MW_NS_LAUNCH_U(4, MI, KMI, TI);                                              \
    } while (0)
        const int sel = (p.mirror ? 4 : 0) | (p.key_mirror[0] ? 2 : 0) | (t128 ? 1 : 0);
        switch (sel) {
            case 0: MW_NS_LAUNCH(false, false, false); break;
            case 1: MW_NS_LAUNCH(false, false, true); break;
            case 2: MW_NS_LAUNCH(false, true, false); break;
            case 3: MW_NS_LAUNCH(false, true, true); break;
            case 4: MW_NS_LAUNCH(true, false, false); break;
            case 5: MW_NS_LAUNCH(true, false, true); break;
            case 6: MW_NS_LAUNCH(true, true, false); break;
            default: MW_NS_LAUNCH(true, true, true); break;
        }
#undef MW_NS_LAUNCH
#undef MW_NS_LAUNCH_U
        return cudaGetLastError();
    }
    if (vec) {
        constexpr int U = 4;
        static int occ = resident_ctas(k_rgba_vec<U>, 256);
        uint32_t total = (uint32_t)(rows * W / 4);
        FastDiv V = make_fastdiv((uint32_t)(W / 4));
        ++g_launches;
        k_rgba_vec<U><<<grid_for((total + 256 * U - 1) / (256 * U), occ, L), 256, 0, L.stream>>>(
            p, c, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), total, V,
            (uint32_t)W, row0W);
    } else {
        static int occ = resident_ctas(k_rgba_scalar, 256);
        if (rows * W >= (1ll << 31)) return cudaErrorInvalidValue;  // FastDiv range
        uint32_t total = (uint32_t)(rows * W);
        ++g_launches;
        k_rgba_scalar<<<grid_for((total + 255) / 256, occ, L), 256, 0, L.stream>>>(
            p, c, reinterpret_cast<const uint32_t*>(src), reinterpret_cast<uint32_t*>(dst), total,
            make_fastdiv((uint32_t)W), row0W);
    }
    return cudaGetLastError();
}

cudaError_t u8_chain(const U8Prog& p, const uint8_t* src, int64_t sp, uint8_t* dst, int64_t dp,
                     int64_t rows, int64_t W, const Launch& L) {
    if (rows <= 0 || W <= 0) return cudaSuccess;
    U8Const c;
    auto mode = [](int t) { return t <= 0 ? 0 : (t >= 256 ? 1 : (t >= 128 ? 2 : 3)); };
    for (int k = 0; k < p.n; ++k) {
        c.lo_mode[k] = mode(p.lo[k]);
        c.hi_mode[k] = mode(p.hi[k]);
        c.lo7[k] = (uint32_t)(p.lo[k] & 0x7F) * 0x01010101u;
        c.hi7[k] = (uint32_t)(p.hi[k] & 0x7F) * 0x01010101u;
    }
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    if (L.tune[TUNE_U8_TMA] && sp == W && dp == W && aligned && (rows * W) % 16 == 0) {
        // 16 KiB chunks; 2 stages (three CTAs per SM) for launches of at least
        // 8 waves of chunks, else 3 (measured on the 512 MiB volume: 180.8 vs
        // 183.2 us)
        constexpr int CH = 16384;
        const int64_t items = (rows * W + CH - 1) / CH;
        ++g_launches;
#define MW_U8_TMA_LAUNCH(NS)                                                                   \
        {                                                                                      \
            constexpr size_t smem = 2 * NS * CH + 64;                                          \
            static int occ = [] {                                                              \
                cudaFuncSetAttribute(k_u8_tma<CH, NS>,                                         \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
                return resident_ctas(k_u8_tma<CH, NS>, 256, smem);                             \
            }();                                                                               \
            cudaLaunchAttribute at[1];                                                         \
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                     \
            at[0].val.programmaticStreamSerializationAllowed = 1;                              \
            cudaLaunchConfig_t cfg = {};                                                       \
            cfg.gridDim = dim3(grid_for(items, occ, L));                                       \
            cfg.blockDim = dim3(256);                                                          \
            cfg.dynamicSmemBytes = smem;                                                       \
            cfg.stream = L.stream;                                                             \
            cfg.attrs = at;                                                                    \
            cfg.numAttrs = 1;                                                                  \
            cudaLaunchKernelEx(&cfg, k_u8_tma<CH, NS>, p, c, src, dst, rows * W,               \
                               (int)L.dep_wait);                                               \
        }
        if (items >= 8ll * sm_count() * 3) MW_U8_TMA_LAUNCH(2) else MW_U8_TMA_LAUNCH(3)
#undef MW_U8_TMA_LAUNCH
        return cudaGetLastError();
    }
    const bool vec = (W % 16 == 0) && (sp % 16 == 0) && (dp % 16 == 0) && aligned &&
                     rows * (W / 16) < (1ll << 31);
    if (vec) {
        constexpr int U = 4;
        static int occ = resident_ctas(k_u8_vec<U>, 256);
        uint32_t total = (uint32_t)(rows * (W / 16));
        ++g_launches;
        k_u8_vec<U><<<grid_for((total + 256 * U - 1) / (256 * U), occ, L), 256, 0, L.stream>>>(
            p, c, src, sp, dst, dp, total, make_fastdiv((uint32_t)(W / 16)));
    } else {
        static int occ = resident_ctas(k_u8_scalar, 256);
        ++g_launches;
        k_u8_scalar<<<grid_for((rows * W + 255) / 256, occ, L), 256, 0, L.stream>>>(p, src, sp, dst,
                                                                                      dp, rows, W);
    }
    return cudaGetLastError();
}

int64_t hyst_tiles(int64_t rows, int64_t pitch) {
    return ((rows + kStencilRows - 1) / kStencilRows) *
           ((pitch / 16 + kStencilThreads - 1) / kStencilThreads);
}

cudaError_t hyst_step(const uint8_t* in, uint8_t* out, int64_t rows, int64_t pitch, int iter,
                      int* last_changed, const uint8_t* prev_flags, uint8_t* cur_flags,
                      int top_nbr, int bot_nbr, const Launch& L) {
    if (rows <= 0) return cudaSuccess;
    if (pitch % 16 != 0) return cudaErrorInvalidValue;
    static int occ = resident_ctas(k_hyst_step, kStencilThreads);
    int64_t strips = (rows + kStencilRows - 1) / kStencilRows;
    int64_t colblk = (pitch / 16 + kStencilThreads - 1) / kStencilThreads;
    ++g_launches;
    k_hyst_step<<<grid_for(strips * colblk, occ, L), kStencilThreads, 0, L.stream>>>(
        in, out, rows, pitch, iter, last_changed, strips, colblk, prev_flags, cur_flags, top_nbr,
        bot_nbr);
    return cudaGetLastError();
}

static U8Const u8_consts(const U8Prog& p) {
    U8Const c;
    auto mode = [](int t) { return t <= 0 ? 0 : (t >= 256 ? 1 : (t >= 128 ? 2 : 3)); };
    for (int k = 0; k < p.n; ++k) {
        c.lo_mode[k] = mode(p.lo[k]);
        c.hi_mode[k] = mode(p.hi[k]);
        c.lo7[k] = (uint32_t)(p.lo[k] & 0x7F) * 0x01010101u;
        c.hi7[k] = (uint32_t)(p.hi[k] & 0x7F) * 0x01010101u;
    }
    return c;
}

// Batched device copies (halo rows between partitions on one device): one
// launch instead of one cudaMemcpyAsync per boundary; blockIdx.y = entry.
__global__ void __launch_bounds__(256) k_copy_batch(const __grid_constant__ CopyBatch b) {
    const int e = blockIdx.y;
    const int64_t n = b.bytes[e];
    if (((uintptr_t)b.src[e] | (uintptr_t)b.dst[e] | (uintptr_t)n) % 16 == 0) {
        const int4* s = reinterpret_cast<const int4*>(b.src[e]);
        int4* d = reinterpret_cast<int4*>(b.dst[e]);
        for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n / 16; i += (int64_t)gridDim.x * 256)
            d[i] = s[i];
    } else {
        for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
            b.dst[e][i] = b.src[e][i];
    }
}

cudaError_t copy_batch(const CopyBatch& b, cudaStream_t s) {
    if (b.n <= 0) return cudaSuccess;
    int64_t mx = 0;
    for (int i = 0; i < b.n; ++i) mx = std::max(mx, b.bytes[i]);
    const int gx = (int)std::min<int64_t>(64, std::max<int64_t>(1, (mx / 16 + 255) / 256));
    ++g_launches;
    k_copy_batch<<<dim3(gx, b.n), 256, 0, s>>>(b);
    return cudaGetLastError();
}

struct RankPtrs {
    const void* p[16];
};
template <typename T, int OP>
__global__ void __launch_bounds__(256) k_reduce_ranks(const __grid_constant__ RankPtrs src, int n, T* dst,
                                                      int64_t count) {
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256) {
        T acc = static_cast<const T*>(src.p[0])[i];
        for (int r = 1; r < n; ++r) {
            const T v = static_cast<const T*>(src.p[r])[i];
            acc = OP == 0 ? acc + v : (OP == 1 ? (v > acc ? v : acc) : (v < acc ? v : acc));
        }
        dst[i] = acc;
    }
}

cudaError_t reduce_ranks(const void* const* srcs, int n, void* dst, size_t count, int dt, int op,
                         cudaStream_t s) {
    if (n < 1 || n > 16 || dt < 0 || dt > 2 || op < 0 || op > 2) return cudaErrorInvalidValue;
    if (count == 0) return cudaSuccess;
    RankPtrs rp{};
    for (int r = 0; r < n; ++r) rp.p[r] = srcs[r];
    const int g = (int)std::min<int64_t>(1024, ((int64_t)count + 255) / 256);
    ++g_launches;
#define RR_CASE(T, D, O) \
    if (dt == D && op == O) k_reduce_ranks<T, O><<<g, 256, 0, s>>>(rp, n, static_cast<T*>(dst), (int64_t)count);
    RR_CASE(int32_t, 0, 0) RR_CASE(int32_t, 0, 1) RR_CASE(int32_t, 0, 2)
    RR_CASE(float, 1, 0) RR_CASE(float, 1, 1) RR_CASE(float, 1, 2)
    RR_CASE(double, 2, 0) RR_CASE(double, 2, 1) RR_CASE(double, 2, 2)
#undef RR_CASE
    return cudaGetLastError();
}

// rounded up to 4 words: the row pitch of a TMA tensor map is a multiple of 16 B
int64_t plane_words(int64_t W) { return (W + 127) / 128 * 4; }

// grid: x = resident CTAs split over the partitions (y), at least one each
static dim3 io_grid(const PlaneIO& io, int64_t per_row_items, int occ, const Launch& L) {
    int64_t tot = 0;
    for (int q = 0; q < io.np; ++q) tot += io.rows[q] * per_row_items;
    const unsigned gx = grid_for(tot, occ, L);
    return dim3(std::max(1u, gx / (unsigned)io.np), io.np);
}

cudaError_t planes_pack_io(const U8Prog& p, const PlaneIO& io, int64_t W, const Launch& L, int hd) {
    const int64_t wp = plane_words(W);
    if (io.np < 1 || io.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    for (int q = 0; q < io.np; ++q)
        if (io.rows[q] <= 0 || io.rows[q] * wp >= (1ll << 31)) return cudaErrorInvalidValue;
    const U8Const c = u8_consts(p);
    ++g_launches;
    const FastDiv WPd = make_fastdiv((uint32_t)wp);
#define MW_PACK(SEGV)                                                                       \
    {                                                                                       \
        static int occ = resident_ctas(k_planes_pack<SEGV>, 256);                           \
        k_planes_pack<SEGV><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(     \
            p, c, io, W, wp, WPd, hd);                                                      \
        return cudaGetLastError();                                                          \
    }
    if (p.n == 1 && p.kind[0] == U8_SEGMENT) {
        switch (c.lo_mode[0] * 4 + c.hi_mode[0]) {   // modes fixed at compile time
            case 0: MW_PACK(0)
            case 1: MW_PACK(1)
            case 2: MW_PACK(2)
            case 3: MW_PACK(3)
            case 5: MW_PACK(5)
            case 9: MW_PACK(9)
            case 10: MW_PACK(10)
            case 13: MW_PACK(13)
            case 14: MW_PACK(14)
            case 15: MW_PACK(15)
            default: break;
        }
    }
    MW_PACK(-1)
#undef MW_PACK
}

cudaError_t planes_pack(const U8Prog& p, const uint8_t* src, int64_t sp, int64_t rows, int64_t W,
                        uint32_t* S, uint32_t* K, const Launch& L, int hd) {
    if (rows <= 0) return cudaSuccess;
    PlaneIO io{};
    io.np = 1;
    io.sp = sp;
    io.src[0] = src;
    io.S0[0] = S;
    io.K[0] = K;
    io.rows[0] = rows;
    return planes_pack_io(p, io, W, L, hd);
}

cudaError_t planes_unpack_io(const U8Prog& p, const PlaneIO& io, const int* state, int64_t dp,
                             int64_t W, const Launch& L, int hd) {
    const int64_t wp = plane_words(W);
    if (io.np < 1 || io.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    bool dst_aligned = dp % 16 == 0, wide_ok = true;
    for (int q = 0; q < io.np; ++q) {
        if (io.rows[q] <= 0 || io.rows[q] * wp >= (1ll << 31)) return cudaErrorInvalidValue;
        dst_aligned &= (reinterpret_cast<uintptr_t>(io.dst[q]) & 15) == 0;
        wide_ok &= io.rows[q] * (wp / 128) < (1ll << 31);
    }
    const U8Const c = u8_consts(p);
    ++g_launches;
    if (p.n == 1 && p.kind[0] == U8_FINALIZE && wp % 128 == 0 && dst_aligned && wide_ok) {
        static int occ = resident_ctas(k_planes_unpack_fin_w, 256);
        // one warp per 128 plane words of a row
        dim3 g = io_grid(io, 1, occ, L);
        int64_t units = 0;
        for (int q = 0; q < io.np; ++q) units = std::max(units, io.rows[q] * (wp / 128));
        g.x = (unsigned)std::min<int64_t>(g.x, std::max<int64_t>(1, (units + 7) / 8));
        k_planes_unpack_fin_w<<<g, 256, 0, L.stream>>>(io, state, dp, wp,
                                                       make_fastdiv((uint32_t)(wp / 128)), hd);
    } else if (p.n == 1 && p.kind[0] == U8_FINALIZE) {
        static int occ = resident_ctas(k_planes_unpack<true>, 256);
        k_planes_unpack<true><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(
            p, c, io, state, dp, W, wp, make_fastdiv((uint32_t)wp), hd);
    } else {
        static int occ = resident_ctas(k_planes_unpack<false>, 256);
        k_planes_unpack<false><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(
            p, c, io, state, dp, W, wp, make_fastdiv((uint32_t)wp), hd);
    }
    return cudaGetLastError();
}

cudaError_t planes_unpack(const U8Prog& p, const uint32_t* S0, const uint32_t* S1,
                          const uint32_t* K, const int* state, uint8_t* dst, int64_t dp,
                          int64_t rows, int64_t W, const Launch& L, int hd) {
    if (rows <= 0) return cudaSuccess;
    PlaneIO io{};
    io.np = 1;
    io.S0[0] = const_cast<uint32_t*>(S0);
    io.S1[0] = const_cast<uint32_t*>(S1);
    io.K[0] = const_cast<uint32_t*>(K);
    io.dst[0] = dst;
    io.rows[0] = rows;
    return planes_unpack_io(p, io, state, dp, W, L, hd);
}

int64_t planes_tiles(int64_t rows, int64_t W) {   // upper bound over the variants (R >= 8)
    return ((rows + 7) / 8) * ((plane_words(W) + 29) / 30);
}

// 2-D tensor map over a plane buffer of (rows + 2 hd) x wp words, box ROWS x 36
static bool plane_tmap(CUtensorMap* tm, const uint32_t* base, int64_t rows, int64_t wp, int box_rows,
                       int hd = 1) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = []() {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!enc) return false;
    // encoded maps are cached by (buffer, shape): the per-partition pass kernel
    // launches twice per partition and pass on the same scratch planes
    struct Key {
        const void* p;
        int64_t rows, wp;
        int box, hd;
        bool operator==(const Key& o) const {
            return p == o.p && rows == o.rows && wp == o.wp && box == o.box && hd == o.hd;
        }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.p) ^ (size_t)(k.rows * 1000003 + k.wp * 131 + k.box * 7 + k.hd);
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{base, rows, wp, box_rows, hd};
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *tm = it->second;
            return true;
        }
    }
    const cuuint64_t dims[2] = {(cuuint64_t)wp, (cuuint64_t)(rows + 2 * hd)};
    const cuuint64_t strides[1] = {(cuuint64_t)wp * 4};
    const cuuint32_t box[2] = {36, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    if (enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();   // bounded (freed scratch leaves stale keys)
    cache[key] = *tm;
    return true;
}

// MW_HYST_PROF=1: per-pass device timestamps of the loop kernel to stderr
static unsigned long long* hyst_prof_buf() {
    static unsigned long long* p = []() -> unsigned long long* {
        unsigned long long* q = nullptr;
        if (getenv("MW_HYST_PROF") && cudaMalloc(&q, 1024) != cudaSuccess) q = nullptr;
        return q;
    }();
    return p;
}
static void hyst_prof_print(const unsigned long long* prof, unsigned grid, int64_t tiles, cudaStream_t st) {
    unsigned long long h[128];
    cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "MW_HYST_PROF grid=%u tiles=%lld", grid, (long long)tiles);
    for (int i = 1; i < 32 && h[i]; ++i) fprintf(stderr, " %.1f", (h[i] - h[0]) / 1e3);
    fprintf(stderr, " us; tiles run / executions per pass:");
    for (int i = 0; i < 30 && h[64 + i]; ++i) fprintf(stderr, " %llu/%llu", h[64 + i], h[32 + i]);
    fprintf(stderr, "\n");
}

template <int T, int ROWS>
static cudaError_t planes_loop_t(uint32_t* S0, uint32_t* S1, const uint32_t* K, int64_t rows,
                                 int64_t wp, int64_t max_iters, int* flags, int* state,
                                 uint32_t* act, const Launch& L) {
    constexpr size_t smem = plane_loop_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_loop<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_loop<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    const int64_t tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    // cooperative: every CTA must be co-resident
    unsigned grid = grid_for((tiles + 7) / 8, occ, L);
    CUtensorMap ts0, ts1, tk;
    if (!plane_tmap(&ts0, S0, rows, wp, ROWS) || !plane_tmap(&ts1, S1, rows, wp, ROWS) ||
        !plane_tmap(&tk, K, rows, wp, ROWS))
        return cudaErrorInvalidValue;
    unsigned long long* prof = hyst_prof_buf();
    if (prof) cudaMemsetAsync(prof, 0, 1024, L.stream);
    int64_t r = rows, w = wp, mi = max_iters;
    void* args[] = {&ts0, &ts1, &tk, &S0, &S1, &r, &w, &mi, &flags, &state, &act, &prof};
    ++g_launches;
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_planes_loop<T, ROWS>, dim3(grid),
                                                dim3(256), args, smem, L.stream);
    if (prof && e == cudaSuccess) hyst_prof_print(prof, grid, tiles, L.stream);
    return e;
}

template <int T, int ROWS>
static cudaError_t planes_pass_t(const uint32_t* in, uint32_t* out, const uint32_t* K, int64_t rows,
                                 int64_t wp, int steps, int64_t k0, const uint8_t* fprev,
                                 uint8_t* fcur, int first, int top, int bot, int* last,
                                 const Launch& L) {
    constexpr size_t smem = plane_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_pass<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_pass<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    const int64_t tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    CUtensorMap tin, tk;
    if (!plane_tmap(&tin, in, rows, wp, ROWS, T) || !plane_tmap(&tk, K, rows, wp, ROWS, T))
        return cudaErrorInvalidValue;
    ++g_launches;
    k_planes_pass<T, ROWS><<<grid_for((tiles + 7) / 8, occ, L), 256, smem, L.stream>>>(
        tin, tk, out, rows, wp, steps, k0, fprev, fcur, first, top, bot, last);
    return cudaGetLastError();
}

int planes_pass_depth(int T_pref, int64_t min_rows) {
    const int ts[] = {12, 8, 6, 4, 2, 1};
    for (int t : ts)
        if (t <= T_pref && t <= min_rows) return t;
    return 1;
}

cudaError_t planes_pass(const uint32_t* in, uint32_t* out, const uint32_t* K, int64_t rows,
                        int64_t W, int T, int steps, int64_t k0, const uint8_t* fprev,
                        uint8_t* fcur, int first, int top, int bot, int* last, const Launch& L) {
    const int64_t wp = plane_words(W);
    if (rows <= 0) return cudaSuccess;
    switch (T) {
        case 12: return planes_pass_t<12, 40>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 8: return planes_pass_t<8, 48>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 6: return planes_pass_t<6, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 4: return planes_pass_t<4, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 2: return planes_pass_t<2, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        default: return planes_pass_t<1, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
    }
}

cudaError_t planes_loop(uint32_t* S0, uint32_t* S1, const uint32_t* K, int64_t rows, int64_t W,
                        int64_t max_iters, int* flags, int* state, uint32_t* act,
                        const Launch& L) {
    const int64_t wp = plane_words(W);
    const int T = L.tune[TUNE_HYST_T];
    const int ROWS = L.tune[TUNE_HYST_ROWS];
#define MW_PL(TT, RR) \
    if (T == TT && ROWS == RR) return planes_loop_t<TT, RR>(S0, S1, K, rows, wp, max_iters, flags, state, act, L)
    MW_PL(4, 32);
    MW_PL(6, 32);
    MW_PL(8, 32);
    MW_PL(8, 40);
    MW_PL(12, 40);
    MW_PL(8, 48);
    MW_PL(6, 48);
#undef MW_PL
    return planes_loop_t<8, 48>(S0, S1, K, rows, wp, max_iters, flags, state, act, L);
}

template <int T, int ROWS>
static cudaError_t planes_multi_t(const PlaneMultiHost& h, int64_t max_iters, int* flags, int* state,
                                  const Launch& L) {
    constexpr size_t smem = plane_loop_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_multi<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_multi<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    static PlaneMultiArgs a;   // host staging of the (large) parameter block
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    a = PlaneMultiArgs{};
    a.np = h.np;
    a.wp = h.wp;
    a.n_cb = (h.wp + 29) / 30;
    a.rank = h.rank;
    a.nranks = h.nranks;
    if (h.nranks < 1 || h.nranks > kXRanks) return cudaErrorInvalidValue;
    for (int r = 0; r < h.nranks && h.nranks > 1; ++r) {
        if (!h.xbar[r]) return cudaErrorInvalidValue;
        a.xbar[r] = h.xbar[r];
    }
    a.rprev_S[0] = h.rprev_S[0];
    a.rprev_S[1] = h.rprev_S[1];
    a.rprev_rows = h.rprev_rows;
    a.rnext_S[0] = h.rnext_S[0];
    a.rnext_S[1] = h.rnext_S[1];
    int64_t tiles = 0;
    for (int q = 0; q < h.np; ++q) {
        PlanePartDesc& d = a.p[q];
        d.S[0] = h.S0[q];
        d.S[1] = h.S1[q];
        d.fl = h.fl[q];
        d.rows = h.rows[q];
        d.n_strips = (d.rows + R - 1) / R;
        d.nt = d.n_strips * a.n_cb;
        d.tile0 = tiles;
        tiles += d.nt;
        d.prev = q > 0 ? q - 1 : (h.remote_prev ? -2 : -1);
        d.next = q + 1 < h.np ? q + 1 : (h.remote_next ? -2 : -1);
        if (d.rows < T || 2 * d.nt > h.fl_bytes[q]) return cudaErrorInvalidValue;
        if (!plane_tmap(&a.ts[q][0], h.S0[q], d.rows, h.wp, ROWS, T) ||
            !plane_tmap(&a.ts[q][1], h.S1[q], d.rows, h.wp, ROWS, T) ||
            !plane_tmap(&a.tk[q], h.K[q], d.rows, h.wp, ROWS, T))
            return cudaErrorInvalidValue;
    }
    a.total = tiles;
    if (!h.act || h.act_words < tiles + 1) return cudaErrorInvalidValue;
    a.act = h.act;
    // loopback ranks share the GPU: each rank's cooperative grid takes its
    // share of the SMs so every rank's kernel is resident at the barriers
    const unsigned grid = std::max(1u, std::min(grid_for(std::max<int64_t>(1, (tiles + 7) / 8), occ, L),
                                                (unsigned)(sm_count() * occ / std::max(1, h.grid_div))));
    int64_t mi = max_iters;
    unsigned long long* prof = hyst_prof_buf();
    if (prof) cudaMemsetAsync(prof, 0, 1024, L.stream);
    void* args[] = {&a, &mi, &flags, &state, &prof};
    ++g_launches;
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_planes_multi<T, ROWS>, dim3(grid), dim3(256),
                                                args, smem, L.stream);
    if (prof && e == cudaSuccess) hyst_prof_print(prof, grid, tiles, L.stream);
    return e;
}

cudaError_t planes_multi(const PlaneMultiHost& h, int T, int64_t max_iters, int* flags, int* state,
                         const Launch& L) {
    if (h.np < (h.nranks > 1 ? 0 : 1) || h.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    switch (T) {
        case 12: return planes_multi_t<12, 40>(h, max_iters, flags, state, L);
        case 8: return planes_multi_t<8, 48>(h, max_iters, flags, state, L);
        case 6: return planes_multi_t<6, 32>(h, max_iters, flags, state, L);
        case 4: return planes_multi_t<4, 32>(h, max_iters, flags, state, L);
        case 2: return planes_multi_t<2, 32>(h, max_iters, flags, state, L);
        default: return planes_multi_t<1, 32>(h, max_iters, flags, state, L);
    }
}

int64_t nbody_part_doubles(int64_t count) { return (int64_t)kNbSeg * count * 3; }

cudaError_t nbody(const float4* pos, const float4* vel, float4* pos_out, float4* vel_out,
                  float4* acc, int64_t first, int64_t count, int64_t N, float eps2, float dt,
                  int mode, double* part, const Launch& L) {
    if (count <= 0) return cudaSuccess;
    // MW_NBODY_SPLIT: 1 = packed FP32x2 + scalar split across the FMA pipes (measured
    // slower on B200: 537 vs 519 ms per 2^20 step, so off by default)
    const int split = L.tune[TUNE_NBODY_SPLIT];
    const int64_t items = (count + kNbTile * kNbPer - 1) / (kNbTile * kNbPer) * kNbSeg;
    ++g_launches;
    if (split) {
        static int occ = resident_ctas(k_nbody<true>, kNbTile);
        k_nbody<true><<<grid_for(items, occ, L), kNbTile, 0, L.stream>>>(
            pos, vel, pos_out, vel_out, acc, first, count, N, eps2, dt, mode, part);
    } else {
        static int occ = resident_ctas(k_nbody<false>, kNbTile);
        k_nbody<false><<<grid_for(items, occ, L), kNbTile, 0, L.stream>>>(
            pos, vel, pos_out, vel_out, acc, first, count, N, eps2, dt, mode, part);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_nbody_fin<<<grid_for((count + 255) / 256, 8, L), 256, 0, L.stream>>>(
        part, pos, vel, pos_out, vel_out, acc, first, count, dt, mode);
    return cudaGetLastError();
}

template <bool DOT, int OP, bool PRE, int TM>
static void reduce_chunks_t(const float* x, const float* y, int64_t x0, int64_t c0, int64_t nc,
                            int64_t total, double* partials, const Launch& L, const SaxpyProg& pre) {
    static int occ = resident_ctas(k_reduce_chunks<DOT, OP, PRE, TM>, kRedThreads);
    ++g_launches;
    k_reduce_chunks<DOT, OP, PRE, TM><<<grid_for(nc, occ, L), kRedThreads, 0, L.stream>>>(
        x, y, x0, c0, nc, total, partials, pre);
}
template <bool DOT, int OP>
static void reduce_chunks_tm(const float* x, const float* y, int64_t x0, int64_t c0, int64_t nc,
                             int64_t total, double* partials, const Launch& L, const SaxpyProg* pre,
                             int tm) {
    if (DOT && pre && pre->n > 0) {   // fused saxpy map stage: no term map combination needed
        if (tm == 0) reduce_chunks_t<DOT, OP, true, 0>(x, y, x0, c0, nc, total, partials, L, *pre);
        else if (tm == 1) reduce_chunks_t<DOT, OP, true, 1>(x, y, x0, c0, nc, total, partials, L, *pre);
        else reduce_chunks_t<DOT, OP, true, 2>(x, y, x0, c0, nc, total, partials, L, *pre);
        return;
    }
    const SaxpyProg none{};
    if (tm == 0) reduce_chunks_t<DOT, OP, false, 0>(x, y, x0, c0, nc, total, partials, L, none);
    else if (tm == 1) reduce_chunks_t<DOT, OP, false, 1>(x, y, x0, c0, nc, total, partials, L, none);
    else reduce_chunks_t<DOT, OP, false, 2>(x, y, x0, c0, nc, total, partials, L, none);
}

cudaError_t reduce_chunks(const float* x, const float* y, int64_t x0, int64_t first,
                          int64_t count, int64_t total, double* partials, const Launch& L,
                          int op, const SaxpyProg* pre, int term_map) {
    if (count <= 0) return cudaSuccess;
    const int64_t CH = 1ll << kChunkLog2;
    if (first % CH != 0 || op < 0 || op > 2 || term_map < -1 || term_map > 1 ||
        (pre && pre->n > 0 && !y))
        return cudaErrorInvalidValue;
    const int tm = term_map + 1;
    int64_t c0 = first / CH, nc = (count + CH - 1) / CH;
    switch (op * 2 + (y ? 1 : 0)) {
        case 0: reduce_chunks_tm<false, 0>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
        case 1: reduce_chunks_tm<true, 0>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
        case 2: reduce_chunks_tm<false, 1>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
        case 3: reduce_chunks_tm<true, 1>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
        case 4: reduce_chunks_tm<false, 2>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
        default: reduce_chunks_tm<true, 2>(x, y, x0, c0, nc, total, partials, L, pre, tm); break;
    }
    return cudaGetLastError();
}

cudaError_t reduce_combine(const double* partials, int64_t nchunks, double* result,
                           cudaStream_t s, int op, const ScalarPost* post) {
    ++g_launches;
    const ScalarPost none{};
    const ScalarPost& ps = post ? *post : none;
    if (op == 1) k_reduce_combine<1><<<1, 1024, 0, s>>>(partials, nchunks, result, ps);
    else if (op == 2) k_reduce_combine<2><<<1, 1024, 0, s>>>(partials, nchunks, result, ps);
    else k_reduce_combine<0><<<1, 1024, 0, s>>>(partials, nchunks, result, ps);
    return cudaGetLastError();
}

cudaError_t reduce_fill_identity(double* partials, int64_t n, cudaStream_t s, int op) {
    if (n <= 0) return cudaSuccess;
    if (op == 0) return cudaMemsetAsync(partials, 0, (size_t)n * 8, s);
    ++g_launches;
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 1024);
    if (op == 1) k_fill_identity<1><<<g, 256, 0, s>>>(partials, n);
    else k_fill_identity<2><<<g, 256, 0, s>>>(partials, n);
    return cudaGetLastError();
}

cudaError_t fill_traits(int64_t* out, int64_t count, int64_t size, int64_t offset,
                        const Launch& L) {
    if (count <= 0) return cudaSuccess;
    ++g_launches;
    k_traits<<<grid_for((count + 255) / 256, 8, L), 256, 0, L.stream>>>(out, count, size, offset);
    return cudaGetLastError();
}

}  // namespace mwk
