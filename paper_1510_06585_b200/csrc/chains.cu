// chains.cu — the fused Map / Pipeline chains: saxpy, the RGBA
// Filter Pipeline noise -> solarize -> mirror (LSU and TMA-ring
// variants) and the u8 chain (segmentation / threshold / finalize).  Every
// kernel is a grid-stride ("persistent-style") loop over tiles so the host can
// size the grid to SMs x resident CTAs (and clamp it for the slowdown
// injector) without changing results.  HBM-bound streams: 128-bit coalesced
// accesses or bulk copies, SWAR / 16x2 SIMD byte arithmetic.
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
#include "kcommon.cuh"
#include "ku8.cuh"

namespace mwk {
namespace {

// ------------------------------------------------------------ saxpy chain
// Programmatic dependent launch: launched with programmatic stream
// serialization, the kernel may be scheduled while its predecessor drains;
// griddepcontrol.wait (before any global access) blocks until the
// predecessor grid has completed and its memory is visible, so ordering is
// unchanged — only the launch latency is hidden (a 2^20 saxpy is ~2 us of HBM
// time, comparable to the launch gap between graph nodes).


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


}  // namespace

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


}  // namespace mwk
