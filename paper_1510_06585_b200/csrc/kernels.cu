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
#include <cstdint>
#include <cuda_runtime.h>

#include "mw_kernels.h"

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
unsigned long long g_launches = 0;

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
// y_i <- fma(a_k, x_i, y_i), k = 0..n-1 (R8 single rounding).
__global__ void __launch_bounds__(256) k_saxpy_vec(SaxpyProg p, const float4* __restrict__ x,
                                                   float4* __restrict__ y, int64_t nvec) {
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
__global__ void k_saxpy_scalar(SaxpyProg p, const float* __restrict__ x, float* __restrict__ y,
                               int64_t n) {
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
__global__ void __launch_bounds__(256) k_rgba_vec(RgbaProg p, RgbaConst c,
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

// Any width / alignment: one pixel per element.
__global__ void __launch_bounds__(256) k_rgba_scalar(RgbaProg p, RgbaConst c,
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
__device__ __forceinline__ uint32_t apply_u8(const U8Prog& p, const U8Const& c, uint32_t x) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT) {
            // R6: v < lo -> 0; lo <= v < hi -> 128; v >= hi -> 255 (lo <= hi)
            uint32_t flo = ge_t(x, c.lo7[k], c.lo_mode[k]);
            uint32_t fhi = ge_t(x, c.hi7[k], c.hi_mode[k]);
            x = flo | (fhi - (fhi >> 7));
        } else {
            // R11 finalize: byte == 128 -> 0 (exact zero-byte test on x ^ 0x80)
            uint32_t z = ~((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
            x &= ~((z >> 7) * 0xFFu);
        }
    }
    return x;
}
__device__ __forceinline__ uint8_t apply_u8_byte(const U8Prog& p, uint8_t v) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT)
            v = v < p.lo[k] ? 0 : (v < p.hi[k] ? 128 : 255);
        else
            v = v == 128 ? 0 : v;
    }
    return v;
}

template <int U>
__global__ void __launch_bounds__(256) k_u8_vec(U8Prog p, U8Const c, const uint8_t* __restrict__ src,
                                                int64_t sp, uint8_t* __restrict__ dst, int64_t dp,
                                                uint32_t total, FastDiv V) {
    for (uint32_t t0 = blockIdx.x * (256u * U); t0 < total; t0 += gridDim.x * (256u * U)) {
        uint4 v[U];
        uint32_t row[U], col[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                uint32_t r = fdiv(n, V);
                row[u] = r;
                col[u] = n - r * V.d;
                v[u] = ld_stream(reinterpret_cast<const uint4*>(src + r * sp) + col[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t n = t0 + u * 256u + threadIdx.x;
            if (n < total) {
                uint4 o = make_uint4(apply_u8(p, c, v[u].x), apply_u8(p, c, v[u].y),
                                     apply_u8(p, c, v[u].z), apply_u8(p, c, v[u].w));
                st_stream(reinterpret_cast<uint4*>(dst + row[u] * dp) + col[u], o);
            }
        }
    }
}
__global__ void k_u8_scalar(U8Prog p, const uint8_t* __restrict__ src, int64_t sp,
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

__global__ void __launch_bounds__(kStencilThreads) k_hyst_step(const uint8_t* __restrict__ in,
                                                               uint8_t* __restrict__ out,
                                                               int64_t rows, int64_t pitch,
                                                               int iter, int* last_changed,
                                                               int64_t n_strips, int64_t n_colblk) {
    const int lane = threadIdx.x & 31;
    const int64_t segs = pitch >> 4;  // 16-byte segments per row
    const int64_t n_tiles = n_strips * n_colblk;
    uint32_t changed = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t strip = t / n_colblk, cb = t - strip * n_colblk;
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
    }
    if (__any_sync(0xffffffffu, changed != 0) && lane == 0) atomicMax(last_changed, iter);
}

// ------------------------------------------------------------ N-body
// a_i = sum_j m_j d_ij (|d_ij|^2 + eps2)^-3/2 (R12): fp32 inside each
// 256-source tile (global tile boundaries, so results do not depend on the
// partitioning), fp64 across tiles.  Two bodies per thread amortise the
// shared-memory broadcast loads; MUFU.RSQ for the inverse square root.
constexpr int kNbTile = 256;
constexpr int kNbPer = 2;

__global__ void __launch_bounds__(kNbTile) k_nbody(const float4* __restrict__ pos,
                                                   const float4* __restrict__ vel,
                                                   float4* __restrict__ pos_out,
                                                   float4* __restrict__ vel_out,
                                                   float4* __restrict__ acc_out, int64_t first,
                                                   int64_t count, int64_t N, float eps2, float dt,
                                                   int mode) {
    __shared__ float4 sp[kNbTile];
    const int64_t per_blk = (int64_t)kNbTile * kNbPer;
    const int64_t nblk = (count + per_blk - 1) / per_blk;
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        float4 pi[kNbPer];
        int64_t idx[kNbPer];
        double ax[kNbPer], ay[kNbPer], az[kNbPer];
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) {
            int64_t l = b * per_blk + q * kNbTile + threadIdx.x;
            idx[q] = first + l;
            pi[q] = l < count ? pos[first + l] : make_float4(0.f, 0.f, 0.f, 0.f);
            ax[q] = ay[q] = az[q] = 0.0;
        }
        for (int64_t jt = 0; jt < N; jt += kNbTile) {
            __syncthreads();
            int64_t j = jt + threadIdx.x;
            sp[threadIdx.x] = j < N ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass 0 pads
            __syncthreads();
            float fx[kNbPer], fy[kNbPer], fz[kNbPer];
#pragma unroll
            for (int q = 0; q < kNbPer; ++q) fx[q] = fy[q] = fz[q] = 0.f;
#pragma unroll 8
            for (int k = 0; k < kNbTile; ++k) {
                float4 s = sp[k];
#pragma unroll
                for (int q = 0; q < kNbPer; ++q) {
                    float dx = s.x - pi[q].x, dy = s.y - pi[q].y, dz = s.z - pi[q].z;
                    float r2 = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmaf_rn(dz, dz, eps2)));
                    float inv = rsqrtf(r2);
                    float w = s.w * inv * inv * inv;
                    fx[q] = __fmaf_rn(dx, w, fx[q]);
                    fy[q] = __fmaf_rn(dy, w, fy[q]);
                    fz[q] = __fmaf_rn(dz, w, fz[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < kNbPer; ++q) {
                ax[q] += (double)fx[q];
                ay[q] += (double)fy[q];
                az[q] += (double)fz[q];
            }
        }
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) {
            int64_t l = idx[q] - first;
            if (l >= count) continue;
            int64_t i = idx[q];
            if (mode == 1) {
                acc_out[l] = make_float4((float)ax[q], (float)ay[q], (float)az[q], 0.f);
            } else {
                float4 v = vel[i];
                double d = (double)dt;
                double vx = (double)v.x + ax[q] * d, vy = (double)v.y + ay[q] * d,
                       vz = (double)v.z + az[q] * d;
                vel_out[i] = make_float4((float)vx, (float)vy, (float)vz, v.w);
                pos_out[i] = make_float4((float)((double)pi[q].x + vx * d),
                                         (float)((double)pi[q].y + vy * d),
                                         (float)((double)pi[q].z + vz * d), pi[q].w);
            }
        }
    }
}

// ------------------------------------------------------------ MapReduce
// One CTA per canonical 2^16-element chunk; thread t folds elements
// (k*256 + t)*4 + e, k = 0..63, e = 0..3, in that order in fp64 (each fp32
// converted exactly; products x*y exact in fp64), then a fixed xor-shuffle
// tree and a fixed 8-warp tree.  The order depends only on global chunk
// boundaries, so every distribution vector gives bit-identical partials.
constexpr int kRedThreads = 256;

template <bool DOT>
__global__ void __launch_bounds__(kRedThreads) k_reduce_chunks(const float* __restrict__ x,
                                                               const float* __restrict__ y,
                                                               int64_t x0, int64_t first_chunk,
                                                               int64_t n_chunks, int64_t total,
                                                               double* __restrict__ partials) {
    __shared__ double warp_part[kRedThreads / 32];
    const int64_t CH = 1ll << kChunkLog2;
    for (int64_t cc = blockIdx.x; cc < n_chunks; cc += gridDim.x) {
        const int64_t c = first_chunk + cc;
        const int64_t gbase = c * CH;
        const int64_t len = min(CH, total - gbase);
        const int64_t base = gbase - x0;  // local index of the chunk's first element
        double acc = 0.0;
        const bool vec = len == CH && ((reinterpret_cast<uintptr_t>(x + base) & 15) == 0) &&
                         (!DOT || ((reinterpret_cast<uintptr_t>(y + base) & 15) == 0));
        if (vec) {
            const uint4* xv = reinterpret_cast<const uint4*>(x + base);
            const uint4* yv = reinterpret_cast<const uint4*>(DOT ? y + base : x + base);
#pragma unroll 8
            for (int k = 0; k < (int)(CH / 4 / kRedThreads); ++k) {
                uint4 a = ld_stream(xv + k * kRedThreads + threadIdx.x);
                if (DOT) {
                    uint4 b = ld_stream(yv + k * kRedThreads + threadIdx.x);
                    acc = __fma_rn((double)__uint_as_float(a.x), (double)__uint_as_float(b.x), acc);
                    acc = __fma_rn((double)__uint_as_float(a.y), (double)__uint_as_float(b.y), acc);
                    acc = __fma_rn((double)__uint_as_float(a.z), (double)__uint_as_float(b.z), acc);
                    acc = __fma_rn((double)__uint_as_float(a.w), (double)__uint_as_float(b.w), acc);
                } else {
                    acc += (double)__uint_as_float(a.x);
                    acc += (double)__uint_as_float(a.y);
                    acc += (double)__uint_as_float(a.z);
                    acc += (double)__uint_as_float(a.w);
                }
            }
        } else {
            for (int k = 0; k < (int)(CH / 4 / kRedThreads); ++k) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    int64_t i = ((int64_t)k * kRedThreads + threadIdx.x) * 4 + e;
                    if (i < len) {
                        if (DOT)
                            acc = __fma_rn((double)x[base + i], (double)y[base + i], acc);
                        else
                            acc += (double)x[base + i];
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kRedThreads / 32; ++w) s += warp_part[w];
            partials[c] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_reduce_combine(const double* __restrict__ partials,
                                                         int64_t n, double* __restrict__ result) {
    __shared__ double wp[32];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 1024) acc += partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double s = wp[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *result = s;
    }
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
    if (nv > 0)
        ++g_launches;
        k_saxpy_vec<<<grid_for((nv + 255) / 256, occ_v, L), 256, 0, L.stream>>>(
            p, reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), nv);
    int64_t rest = n - nv * 4;
    if (rest > 0)
        ++g_launches;
        k_saxpy_scalar<<<grid_for((rest + 255) / 256, occ_s, L), 256, 0, L.stream>>>(
            p, x + nv * 4, y + nv * 4, rest);
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
    const bool vec = (W % 16 == 0) && (sp % 16 == 0) && (dp % 16 == 0) &&
                     ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
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

cudaError_t hyst_step(const uint8_t* in, uint8_t* out, int64_t rows, int64_t pitch, int iter,
                      int* last_changed, const Launch& L) {
    if (rows <= 0) return cudaSuccess;
    if (pitch % 16 != 0) return cudaErrorInvalidValue;
    static int occ = resident_ctas(k_hyst_step, kStencilThreads);
    int64_t strips = (rows + kStencilRows - 1) / kStencilRows;
    int64_t colblk = (pitch / 16 + kStencilThreads - 1) / kStencilThreads;
    ++g_launches;
    k_hyst_step<<<grid_for(strips * colblk, occ, L), kStencilThreads, 0, L.stream>>>(
        in, out, rows, pitch, iter, last_changed, strips, colblk);
    return cudaGetLastError();
}

cudaError_t nbody(const float4* pos, const float4* vel, float4* pos_out, float4* vel_out,
                  float4* acc, int64_t first, int64_t count, int64_t N, float eps2, float dt,
                  int mode, const Launch& L) {
    if (count <= 0) return cudaSuccess;
    static int occ = resident_ctas(k_nbody, kNbTile);
    int64_t blocks = (count + kNbTile * kNbPer - 1) / (kNbTile * kNbPer);
    ++g_launches;
    k_nbody<<<grid_for(blocks, occ, L), kNbTile, 0, L.stream>>>(pos, vel, pos_out, vel_out, acc,
                                                                first, count, N, eps2, dt, mode);
    return cudaGetLastError();
}

cudaError_t reduce_chunks(const float* x, const float* y, int64_t x0, int64_t first,
                          int64_t count, int64_t total, double* partials, const Launch& L) {
    if (count <= 0) return cudaSuccess;
    const int64_t CH = 1ll << kChunkLog2;
    if (first % CH != 0) return cudaErrorInvalidValue;
    int64_t c0 = first / CH, nc = (count + CH - 1) / CH;
    if (y) {
        static int occ = resident_ctas(k_reduce_chunks<true>, kRedThreads);
        ++g_launches;
        k_reduce_chunks<true><<<grid_for(nc, occ, L), kRedThreads, 0, L.stream>>>(x, y, x0, c0, nc, total, partials);
    } else {
        static int occ = resident_ctas(k_reduce_chunks<false>, kRedThreads);
        ++g_launches;
        k_reduce_chunks<false><<<grid_for(nc, occ, L), kRedThreads, 0, L.stream>>>(x, y, x0, c0, nc, total, partials);
    }
    return cudaGetLastError();
}

cudaError_t reduce_combine(const double* partials, int64_t nchunks, double* result,
                           cudaStream_t s) {
    ++g_launches;
    k_reduce_combine<<<1, 1024, 0, s>>>(partials, nchunks, result);
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
