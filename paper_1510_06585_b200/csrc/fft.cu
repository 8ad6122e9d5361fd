// fft.cu — the FFT workload (NEXT-3): batched FFT / inverse FFT chains.
//
// PAPER.md P:729-732 (§4): "FFT is a set of Fast-Fourier Transformations
// adapted from the SHOC Benchmark Suite, where FFT is pipelined with its
// inversion.  The elementary partitioning unit is the size of each FFT which
// is 512 KBytes."  Readings R23-R25: N = 65536 complex64 points
// per FFT (2^13..2^16 accepted), forward e^{-2 pi i nk/N}, inverse with 1/N.
//
// B200 design.  The fused pipeline(fft, ifft) at N = 65536 (the benchmark)
// runs as a 16 x 4096 four-step FFT by default (k_fft16_*, below: three
// launches, the column passes HBM-bound register DFT-16s, the row pass one
// 4096-point row per CTA with forward and inverse fused); a 256 x 256
// four-step form (k_fft4_*, three launches or one dataflow launch) and the
// cluster kernel are kept as tuning alternatives.  Every other chain:
// one FFT is held on chip by a thread-block CLUSTER of
// C = N / 8192 CTAs (C in {1,2,4,8}); each CTA keeps 8192 points (64 KiB,
// padded) in shared memory and the CTAs exchange data through distributed
// shared memory, so one FFT moves through HBM exactly once per launch — and a
// fused pipeline(fft, ifft) (the planner fuses consecutive FFT leaves) reads
// the input once and writes the output once, with no intermediate in HBM.
// Decomposition N = C * N2 (N2 = 8192), n = N2 n1 + n2, k = k1 + C k2:
//   X[k1 + C k2] = sum_n2 W_N2^{n2 k2} W_N^{n2 k1} sum_n1 x[N2 n1 + n2] W_C^{n1 k1}
// forward: radix-C DFT across the cluster (each CTA owns a slice of n2 and
// pushes y[k1][n2] into CTA k1's shared memory), then a local 8192-point
// Stockham FFT (radix 32, 16, 16) leaves X[k1 + C k2] at position k2 of CTA
// k1 ("T layout").  The inverse runs the mirror image: local inverse FFT on
// the T layout, then the twiddled radix-C inverse DFT gathered across the
// cluster lands in natural order — fft followed by ifft needs no exchange in
// the middle.  Twiddles come from exact-rounded fp64 tables laid out so a
// warp reads them without index arithmetic or quadrant folding: the 512-point
// pass from a [r][k] table in shared memory (k = thread mod 32: one load per
// twiddle serves both butterflies of a thread), the 8192-point pass from a
// [r][k] table in global memory (64 KiB, L1-resident: both CTAs of an SM read
// the same table), the cross-CTA twiddle W_65536^e from two full-circle
// 256-entry tables (e = 256 h + l); so mu <= 4u (R25).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>

#include "mw_kernels.h"

namespace cg = cooperative_groups;

namespace mwk {
namespace {

constexpr int FN2 = 8192;              // points per CTA
constexpr int FT = 256;                // threads per CTA
constexpr int FPAD = FN2 + FN2 / 32;   // one pad element per 32 (conflict-free radix-32 stores)
constexpr int T9 = 16 * 32;            // W_512^(r k) at [r][k], r < 16, k < 32
constexpr int THI = 256, TLO = 256;    // W_65536^(256 h) and W_65536^l, full circle
constexpr size_t kFftSmem = sizeof(float2) * (FPAD + T9 + THI + TLO);

// W_8192^(r k) at [r][k], r < 16, k < 512 (forward sign), filled once per
// device by k_fft_tw13 before the first FFT launch.
__device__ float2 g_tw13[16 * 512];
// The 4-step path's tables: W_256^(l k) at [l][k] (l, k < 16) and the
// full-circle two-level W_65536^e = hi[e >> 8] * lo[e & 255].
__device__ float2 g_w256[256];
__device__ float2 g_w16hi[256];
__device__ float2 g_w16lo[256];
// The 16 x 4096 path's tables, laid out [m][t] so a warp reads consecutive
// entries: W_4096^(m t) and W_65536^(m t), m < 16, t < 256.
__device__ float2 g_w4096t[16 * 256];
__device__ float2 g_w65536t[16 * 256];
__global__ void k_fft_tw13() {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double sn, cs;
    if (i < 16 * 512) {
        const int r = i / 512, k = i % 512;
        sincospi(2.0 * ((r * k) & 8191) / 8192.0, &sn, &cs);
        g_tw13[i] = make_float2((float)cs, (float)-sn);
    } else if (i < 16 * 512 + 3 * 256) {
        const int j = i - 16 * 512, t = j / 256, e = j % 256;
        const double x = t == 0 ? 2.0 * ((e / 16) * (e % 16)) / 256.0
                       : t == 1 ? 2.0 * 256.0 * e / 65536.0 : 2.0 * e / 65536.0;
        sincospi(x, &sn, &cs);
        (t == 0 ? g_w256 : t == 1 ? g_w16hi : g_w16lo)[e] = make_float2((float)cs, (float)-sn);
    } else if (i < 16 * 512 + 3 * 256 + 2 * 4096) {
        const int j = i - (16 * 512 + 3 * 256), q = j / 4096, mt = j % 4096;
        const int m = mt / 256, t = mt % 256;
        const double x = q == 0 ? 2.0 * ((m * t) % 4096) / 4096.0 : 2.0 * (m * t) / 65536.0;
        sincospi(x, &sn, &cs);
        (q == 0 ? g_w4096t : g_w65536t)[mt] = make_float2((float)cs, (float)-sn);
    }
}

__device__ __forceinline__ int fpad(int i) { return i + (i >> 5); }

// complex add / sub as one packed FP32x2 instruction (sm_100a FADD2)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    unsigned long long ua, ub, ur;
    asm("mov.b64 %0, {%1,%2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(ur) : "l"(ua), "l"(ub));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(ur));
    return r;
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    unsigned long long ua, ub, ur;
    asm("mov.b64 %0, {%1,%2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ur) : "l"(ua), "l"(ub));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(ur));
    return r;
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * w (INV: a * conj(w))
template <bool INV>
__device__ __forceinline__ float2 cmulw(float2 a, float2 w) {
    if (INV) return make_float2(fmaf(a.x, w.x, a.y * w.y), fmaf(a.y, w.x, -a.x * w.y));
    return cmul(a, w);
}

// cos(2 pi k / 32), k = 0..8 (fp32, correctly rounded)
__host__ __device__ constexpr float c32(int k) {
    return k == 0 ? 1.0f
         : k == 1 ? 9.807852507e-01f
         : k == 2 ? 9.238795042e-01f
         : k == 3 ? 8.314695954e-01f
         : k == 4 ? 7.071067691e-01f
         : k == 5 ? 5.555702448e-01f
         : k == 6 ? 3.826834261e-01f
         : k == 7 ? 1.950903237e-01f
         : 0.0f;
}

// d * W_32^k (forward W = e^{-2 pi i/32}; INV: conjugate), 0 <= k < 16.  k is
// a constant after unrolling, so the branches and table fold away.
template <bool INV>
__device__ __forceinline__ float2 tw32(float2 d, int k) {
    if (k == 0) return d;
    if (k == 8) return INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);   // +-i
    const float c = k <= 8 ? c32(k) : -c32(16 - k);
    const float s = k <= 8 ? c32(8 - k) : c32(k - 8);
    const float si = INV ? s : -s;
    // d * (c + i si) = d.x (c, si) + d.y (-si, c): FMUL2 + FFMA2 with the
    // scalar d.x / d.y broadcast across the pair
    unsigned long long bx, by, w, iw, t, r;
    asm("mov.b64 %0, {%1,%1};" : "=l"(bx) : "f"(d.x));
    asm("mov.b64 %0, {%1,%1};" : "=l"(by) : "f"(d.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(w) : "f"(c), "f"(si));
    asm("mov.b64 %0, {%1,%2};" : "=l"(iw) : "f"(-si), "f"(c));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(bx), "l"(w));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(by), "l"(iw), "l"(t));
    float2 o;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}

__host__ __device__ constexpr int bitrev(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// In-register R-point DFT (R | 32): radix-2 decimation in frequency (one
// template level per stage, so every index is a compile-time constant), then
// a compile-time bit-reversal renaming to natural output order.
template <int R, int HALF, bool INV>
__device__ __forceinline__ void dif_stage(float2* v) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * HALF) {
#pragma unroll
        for (int j = 0; j < HALF; ++j) {
            const float2 a = v[blk + j], b = v[blk + j + HALF];
            v[blk + j] = cadd(a, b);
            v[blk + j + HALF] = tw32<INV>(csub(a, b), j * (16 / HALF));
        }
    }
    if constexpr (HALF > 1) dif_stage<R, HALF / 2, INV>(v);
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
    if constexpr (R > 1) {
        dif_stage<R, R / 2, INV>(v);
        float2 t[R];
#pragma unroll
        for (int i = 0; i < R; ++i) t[i] = v[bitrev(i, ilog2(R))];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = t[i];
    }
}

// W_65536^e (INV: conjugate), e < 65536, two-level full-circle tables
template <bool INV>
__device__ __forceinline__ float2 tw_cross(const float2* Thi, const float2* Tlo, int e) {
    float2 w = cmul(Thi[e >> 8], Tlo[e & 255]);
    if (INV) w.y = -w.y;
    return w;
}

// One Stockham pass over the CTA's 8192 points (in place: all loads, barrier,
// all stores): v[r] = s[j + r N2/R] * W_{Ns R}^{r k}, R-point DFT, stored at
// (j / Ns) Ns R + k + r Ns, k = j mod Ns.
template <int R, int NS, bool INV>
__device__ __forceinline__ void stockham_pass(float2* s, const float2* T9p) {
    constexpr int NB = FN2 / R, PER = NB / FT;
    int tid = threadIdx.x;
    asm volatile("" : "+r"(tid));   // per pass: no addresses kept live across passes
    float2 v[PER][R];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const int j = tid + p * FT;
        const int k = j & (NS - 1);
        // NB is a multiple of 32: fpad(j + r NB) = fpad(j) + r (NB + NB/32), so
        // every load is one base register plus an immediate offset
        const float2* src = s + fpad(j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[p][r] = src[r * (NB + NB / 32)];
        if constexpr (NS > 1) {
            static_assert(NS * R == 512 || NS * R == 8192, "twiddle tables");
            // k = j mod NS with j = tid + 256 p: the [r][k] tables are read at
            // consecutive k across a warp (no bank conflicts, full sectors)
            const float2* tw = NS * R == 512 ? T9p + k : g_tw13 + k;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const float2 w = NS * R == 512 ? tw[r * NS] : __ldg(tw + r * NS);
                v[p][r] = cmulw<INV>(v[p][r], w);
            }
        }
        dft<R, INV>(v[p]);
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const int j = tid + p * FT;
        const int k = j & (NS - 1);
        const int d = (j / NS) * NS * R + k;
        // NS = 1: d is a multiple of R = 32, so d + r stays in one 32-run;
        // NS >= 32: r NS is a multiple of 32 -> immediate offsets again
        static_assert(NS == 1 ? R == 32 : NS % 32 == 0, "padding plan");
        float2* dst = s + fpad(d);
#pragma unroll
        for (int r = 0; r < R; ++r) dst[NS == 1 ? r : r * (NS + NS / 32)] = v[p][r];
    }
    __syncthreads();
}

// Not inlined: the three passes get their own register allocation instead of
// competing with the cluster-exchange code around them (measured: inlining
// them into the fused forward->inverse kernel spills ~400 B per thread).
template <bool INV>
__device__ __noinline__ void local_fft(float2* s, const float2* T9p) {
    static_assert(FN2 == 32 * 16 * 16, "pass plan");
    stockham_pass<32, 1, INV>(s, T9p);
    stockham_pass<16, 32, INV>(s, T9p);
    stockham_pass<16, 512, INV>(s, T9p);
}

template <int C>
__device__ __forceinline__ void csync() {
    if constexpr (C > 1) cg::this_cluster().sync();
    else __syncthreads();
}
// Split barrier without memory ordering: only protects shared memory that
// peers READ before arriving (their loaded values were consumed before the
// arrive, so the reads are complete) from our next writes.  The arrive is
// issued right after the gather; the output stores and the next transform's
// input loads run before the matching wait.
template <int C>
__device__ __forceinline__ void war_arrive() {
    if constexpr (C > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
template <int C>
__device__ __forceinline__ void war_wait() {
    if constexpr (C > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    else __syncthreads();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float2 ld_nc(const float2* p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs(float2* p, float2 v) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

enum FftMode { FFT_F = 0, FFT_I = 1, FFT_FI = 2 };

// One launch = one of: forward, inverse, or the fused forward -> inverse
// (pipeline(fft, ifft)) over nfft transforms of N = C * 8192 points.  Longer
// chains are split into such launches by the host (in place on the output).
template <int C, int MODE>
__global__ void __launch_bounds__(FT, 2) k_fft(const float2* in, float2* out, int64_t nfft) {
    extern __shared__ float4 fft_smem[];
    float2* S = reinterpret_cast<float2*>(fft_smem);
    float2* T9p = S + FPAD;
    float2* Thi = T9p + T9;
    float2* Tlo = Thi + THI;
    for (int i = threadIdx.x; i < T9 + THI + TLO; i += FT) {
        double x;   // angle / pi
        if (i < T9) {
            const int r = i / 32, k = i % 32;
            x = 2.0 * ((r * k) & 511) / 512.0;
        } else if (i < T9 + THI) {
            x = 2.0 * 256.0 * (i - T9) / 65536.0;
        } else {
            x = 2.0 * (i - T9 - THI) / 65536.0;
        }
        double sn, cs;
        sincospi(x, &sn, &cs);
        T9p[i] = make_float2((float)cs, (float)-sn);   // the three tables are contiguous
    }
    __syncthreads();
    constexpr int NI = 32 / C;             // n2 values per thread (x C values of n1)
    constexpr int N = C * FN2;
    constexpr int STEP = 65536 / N;        // W_N = W_65536^STEP
    const int c = C > 1 ? (int)cg::this_cluster().block_rank() : 0;
    // peer CTA k's shared-memory window (one mapa instruction)
    auto rem = [S](int k) -> float2* {
        float2* p = S;
        asm volatile("" : "+l"(p));   // recompute per use instead of holding C pointers live
        if constexpr (C > 1) return cg::this_cluster().map_shared_rank(p, k);
        else return p;
    };
    const float scale = 1.0f / (float)N;   // exact (power of two)
    war_arrive<C>();
    for (int64_t f = blockIdx.x / C; f < nfft; f += gridDim.x / C) {
        // opaque per iteration: keeps the compiler from hoisting the 32
        // per-element addresses out of the persistent loop (and spilling them)
        int tid = threadIdx.x;
        asm volatile("" : "+r"(tid));
        const float2* x = in + f * N;
        float2* y = out + f * N;
        {   // natural-order input: thread owns n2 = c N2/C + tid + 256 i, all n1
            float2 v[NI][C];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int n2 = c * (FN2 / C) + tid + FT * i;
#pragma unroll
                for (int n1 = 0; n1 < C; ++n1) v[i][n1] = ld_nc(x + n1 * FN2 + n2);
            }
            war_wait<C>();   // every peer is done reading the shared memory we write
            if constexpr (MODE == FFT_I) {
                // T layout directly: X[m] goes to CTA m mod C at position m / C
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int n2 = c * (FN2 / C) + tid + FT * i;
#pragma unroll
                    for (int n1 = 0; n1 < C; ++n1) {
                        const int m = n1 * FN2 + n2;
                        rem(m % C)[fpad(m / C)] = v[i][n1];
                    }
                }
            } else {
                // radix-C forward DFT across the cluster, twiddle W_N^{n2 k1}, push to CTA k1
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int n2 = c * (FN2 / C) + tid + FT * i;
                    dft<C, false>(v[i]);
#pragma unroll
                    for (int k1 = 0; k1 < C; ++k1) {
                        float2 t = v[i][k1];
                        if (k1 > 0) t = cmul(t, tw_cross<false>(Thi, Tlo, (n2 * k1 * STEP) & 65535));
                        rem(k1)[fpad(n2)] = t;
                    }
                }
            }
            csync<C>();
        }
        if constexpr (MODE != FFT_I) local_fft<false>(S, T9p);   // -> X[k1 + C k2] at k2
        if constexpr (MODE != FFT_F) local_fft<true>(S, T9p);    // -> z[k1][n2] at n2
        csync<C>();   // every CTA's local transform is complete
        {
            float2 v[NI][C];
            if constexpr (MODE == FFT_F) {
                // T layout -> natural order
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int n2 = c * (FN2 / C) + tid + FT * i;
#pragma unroll
                    for (int n1 = 0; n1 < C; ++n1) {
                        const int m = n1 * FN2 + n2;
                        v[i][n1] = rem(m % C)[fpad(m / C)];
                    }
                }
            } else {
                // twiddle W_N^{-k1 n2}, radix-C inverse DFT across the cluster, 1/N
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int n2 = c * (FN2 / C) + tid + FT * i;
#pragma unroll
                    for (int k1 = 0; k1 < C; ++k1) {
                        float2 t = rem(k1)[fpad(n2)];
                        if (k1 > 0) t = cmul(t, tw_cross<true>(Thi, Tlo, (n2 * k1 * STEP) & 65535));
                        v[i][k1] = t;
                    }
                    dft<C, true>(v[i]);
#pragma unroll
                    for (int n1 = 0; n1 < C; ++n1) v[i][n1] = make_float2(v[i][n1].x * scale, v[i][n1].y * scale);
                }
            }
            // done reading peers' shared memory: the inverse gather's values were
            // consumed by the DFT above; the plain transpose's by the stores below
            if constexpr (MODE != FFT_F) war_arrive<C>();
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int n2 = c * (FN2 / C) + tid + FT * i;
#pragma unroll
                for (int n1 = 0; n1 < C; ++n1) st_cs(y + n1 * FN2 + n2, v[i][n1]);
            }
            if constexpr (MODE == FFT_F) war_arrive<C>();
        }
    }
    war_wait<C>();   // no CTA leaves while a peer may still read its shared memory
}

// ---- 4-step path for the fused pipeline(fft, ifft) at N = 65536 = 256 x 256.
// n = c + 256 r (c: column, r: row), k = k2 + 256 k1:
//   A (columns):  Y[k2][c] = sum_r x[c + 256 r] W_256^{r k2}, then x W_N^{c k2}
//   B (rows):     X[k2 + 256 k1] = sum_c Y'[k2][c] W_256^{c k1}
// and the inverse mirrored: B^-1 over k1 -> Z'[k2][c], x W_N^{-c k2}, A^-1
// over k2 -> x[c + 256 r] (1/N).  Three launches per chunk of transforms
// (MW_FFT4_CHUNK, default the whole batch) — A, then B with B^-1 fused (the
// spectrum never leaves the registers), then A^-1 — each in place on the
// output buffer, which holds the intermediate (a batch larger than L2
// round-trips it through HBM once per pass; k_fft4_flow keeps it in L2
// instead).  No clusters, no
// distributed shared memory: every 256-point DFT belongs to one half-warp
// (16 points per lane, two radix-16 register DFTs and one shared-memory
// transpose), so each SM keeps many independent DFTs in flight.

// DFT-256 of TWO independent rows by a half-warp (interleaved for ILP): lane
// l holds x[l + 16 j], j < 16, of each and ends with X[l + 16 j] (the same
// layout).  16 x 16: DFT-16 over j, twiddle W_256^{l k1} (the table is
// symmetric, read as [k1][l]: consecutive across the lanes), transpose
// through sc ([16][17] per row: conflict-free both ways), DFT-16 over l.
template <bool INV>
__device__ __forceinline__ void dft256_hw2(float2 (&a)[16], float2 (&b)[16], int l, float2* sa, float2* sb,
                                           const float2* w256) {
    dft<16, INV>(a);
    dft<16, INV>(b);
#pragma unroll
    for (int k = 1; k < 16; ++k) {
        const float2 w = w256[k * 16 + l];
        a[k] = cmulw<INV>(a[k], w);
        b[k] = cmulw<INV>(b[k], w);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        sa[k * 17 + l] = a[k];
        sb[k * 17 + l] = b[k];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        a[j] = sa[l * 17 + j];
        b[j] = sb[l * 17 + j];
    }
    __syncwarp();
    dft<16, INV>(a);
    dft<16, INV>(b);
}
// The same two DFT-256s with the transpose done inside the columns' own
// tile storage (column c at tile[r * pitch + c]): y[l][k1] goes to row
// 16 k1 + ((l + k1) & 15), read back by lane L at rows 16 L + ((j + L) & 15)
// — with an odd pitch both directions are bank-conflict-free, and no scratch
// is needed (more CTAs per SM).
template <bool INV, int PITCH>
__device__ __forceinline__ void dft256_col2(float2 (&a)[16], float2 (&b)[16], int l, float2* tile, int ca,
                                            int cb, const float2* w256) {
    dft<16, INV>(a);
    dft<16, INV>(b);
#pragma unroll
    for (int k = 1; k < 16; ++k) {
        const float2 w = w256[k * 16 + l];
        a[k] = cmulw<INV>(a[k], w);
        b[k] = cmulw<INV>(b[k], w);
    }
    __syncwarp();   // every lane has read its column values
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int r = 16 * k + ((l + k) & 15);
        tile[r * PITCH + ca] = a[k];
        tile[r * PITCH + cb] = b[k];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int r = 16 * l + ((j + l) & 15);
        a[j] = tile[r * PITCH + ca];
        b[j] = tile[r * PITCH + cb];
    }
    __syncwarp();
    dft<16, INV>(a);
    dft<16, INV>(b);
}
__device__ __forceinline__ float2 tw65536(const float2* tb, int e, bool inv) {
    float2 w = cmul(tb[256 + (e >> 8)], tb[512 + (e & 255)]);
    if (inv) w.y = -w.y;
    return w;
}
// the three 256-entry tables (W_256 [l][k], W_65536 hi, lo) into shared memory
__device__ __forceinline__ void f4_tables(float2* tb) {
    for (int i = threadIdx.x; i < 768; i += blockDim.x)
        tb[i] = __ldg(i < 256 ? &g_w256[i] : i < 512 ? &g_w16hi[i - 256] : &g_w16lo[i - 512]);
}



// Column pass over one 256 x 32 tile (columns c0 .. c0 + 31) of transform f:
// INV = false: A + W_N^{c k2}; INV = true: A^-1 and 1/N.  In place on `out`
// (the input `in` on the forward pass).
constexpr int kF4Cols = 16;                 // columns per tile (8 half-warps x 2)
constexpr int kF4Pitch = kF4Cols + 1;       // odd pitch: conflict-free column access
constexpr size_t kF4ColSmem = sizeof(float2) * (256 * kF4Pitch + 768);

// Column pass over one 256 x 16 tile (columns c0 .. c0 + 15) of transform f:
// INV = false: A + W_N^{c k2}; INV = true: A^-1 and 1/N.  In place on `out`
// (the input `in` on the forward pass).  128 threads, ~41 KiB: four CTAs per
// SM overlap one another's load, compute and store phases.  (Measured: a
// persistent version with two tile buffers per CTA — the next tile's copies
// landing during the current one — 0.405 vs 0.335 ms per batch: fewer CTAs
// per SM hide less.)
// One column tile (256 x kF4Cols, columns c0 ..) of transform f by 128
// threads: INV = false: A + W_N^{c k2}; INV = true: A^-1 and 1/N.  Reads
// in + f N, writes out + f N (in place when they alias).  Ends with the
// tile's stores issued; the caller synchronises before reusing `tile`.
template <bool INV>
__device__ __forceinline__ void f4_col_tile(const float2* in, float2* out, int64_t f, int c0, float2* tile,
                                            const float2* tb) {
    const int tid = threadIdx.x;
    const float2* src = in + f * 65536 + c0;
    float2* dst = out + f * 65536 + c0;
    const int cc = tid & (kF4Cols - 1), r0 = tid / kF4Cols;
    constexpr int kRowStep = 128 / kF4Cols;
    // all of this thread's elements in flight at once (asynchronous copies
    // straight into the padded tile: no registers held across the latency)
#pragma unroll
    for (int i = 0; i < 256 / kRowStep; ++i) {
        const int r = r0 + kRowStep * i;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(tile + r * kF4Pitch + cc)),
                     "l"(src + r * 256 + cc)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int hw = tid >> 4, l = tid & 15;
    const int ca = 2 * hw, cb = 2 * hw + 1;   // this half-warp's two columns
    float2 a[16], b[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        a[j] = tile[(l + 16 * j) * kF4Pitch + ca];
        b[j] = tile[(l + 16 * j) * kF4Pitch + cb];
    }
    dft256_col2<INV, kF4Pitch>(a, b, l, tile, ca, cb, tb);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int k = l + 16 * j;
        if (!INV) {
            a[j] = cmul(a[j], tw65536(tb, ((c0 + ca) * k) & 65535, false));
            b[j] = cmul(b[j], tw65536(tb, ((c0 + cb) * k) & 65535, false));
        } else {
            a[j] = make_float2(a[j].x * (1.0f / 65536.0f), a[j].y * (1.0f / 65536.0f));
            b[j] = make_float2(b[j].x * (1.0f / 65536.0f), b[j].y * (1.0f / 65536.0f));
        }
    }
    __syncwarp();   // the transposed values were read by every lane
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int k = l + 16 * j;
        tile[k * kF4Pitch + ca] = a[j];
        tile[k * kF4Pitch + cb] = b[j];
    }
    __syncthreads();
    // the forward pass leaves the intermediate for the row pass (no
    // streaming hint); the inverse pass writes the result (streaming)
#pragma unroll 8
    for (int i = 0; i < 256 / kRowStep; ++i) {
        const int r = r0 + kRowStep * i;
        if (INV) st_cs(dst + r * 256 + cc, tile[r * kF4Pitch + cc]);
        else dst[r * 256 + cc] = tile[r * kF4Pitch + cc];
    }
}

// Column pass over one 256 x 16 tile (columns c0 .. c0 + 15) of transform f:
// INV = false: A + W_N^{c k2}; INV = true: A^-1 and 1/N.  In place on `out`
// (the input `in` on the forward pass).  128 threads, ~41 KiB: four CTAs per
// SM overlap one another's load, compute and store phases.  (Measured: a
// persistent version with two tile buffers per CTA — the next tile's copies
// landing during the current one — 0.405 vs 0.335 ms per batch: fewer CTAs
// per SM hide less; five CTAs per SM at 96 registers: 0.389 ms.)
template <bool INV>
__global__ void __launch_bounds__(128) k_fft4_cols(const float2* in, float2* out, int64_t f0) {
    extern __shared__ float4 f4_smem[];
    float2* tile = reinterpret_cast<float2*>(f4_smem);
    float2* tb = tile + 256 * kF4Pitch;
    f4_tables(tb);
    constexpr int kTiles = 256 / kF4Cols;
    f4_col_tile<INV>(in, out, f0 + blockIdx.x / kTiles, (blockIdx.x % kTiles) * kF4Cols, tile, tb);
}

// Rows k0 .. k0 + blockDim / 8 - 1 of transform f, fused B then B^-1 (then
// W_N^{-c k2}), two rows per half-warp (interleaved), in place; rows go
// straight to registers (coalesced), the transposes through a [16][17]
// scratch per row (scr: 2 * 16 * 17 float2 per half-warp).
__device__ __forceinline__ void f4_row_block(float2* out, int64_t f, int k0, float2* scr, const float2* tb) {
    const int tid = threadIdx.x;
    const int hw = tid >> 4, l = tid & 15;
    const int ka = k0 + 2 * hw, kb = ka + 1;
    float2* ra = out + f * 65536 + (int64_t)ka * 256;
    float2* rb = ra + 256;
    float2 a[16], b[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        a[j] = ra[l + 16 * j];
        b[j] = rb[l + 16 * j];
    }
    float2* sa = scr + (2 * hw) * (16 * 17);
    float2* sb = sa + 16 * 17;
    dft256_hw2<false>(a, b, l, sa, sb, tb);   // X[k2 + 256 k1], k1 = l + 16 j
    dft256_hw2<true>(a, b, l, sa, sb, tb);    // Z'[k2][c], c = l + 16 j
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int c = l + 16 * j;
        ra[c] = cmul(a[j], tw65536(tb, (ka * c) & 65535, true));
        rb[c] = cmul(b[j], tw65536(tb, (kb * c) & 65535, true));
    }
}

// Row pass, 32 rows per CTA of 256 threads.  (Staging the rows through
// shared memory with in-place transposes, as the column pass does, measured
// slower: 0.347 vs 0.335 ms per batch; three CTAs per SM at 80 registers:
// 0.354 ms.)
constexpr size_t kF4RowSmem = sizeof(float2) * (32 * 16 * 17 + 768);
__global__ void __launch_bounds__(256) k_fft4_rows_fi(float2* out, int64_t f0) {
    extern __shared__ float4 f4r_smem[];
    float2* scr = reinterpret_cast<float2*>(f4r_smem);
    float2* tb = scr + 32 * 16 * 17;
    f4_tables(tb);
    __syncthreads();
    f4_row_block(out, f0 + blockIdx.x / 8, (blockIdx.x % 8) * 32, scr, tb);
}

// ---- Dataflow form of the same three passes: ONE persistent launch whose
// CTAs claim work items from an atomic ticket in an order that pipelines the
// transforms through the passes — slot group g holds the 16 column tiles of
// transform g, the 16 row blocks (16 rows each) of transform g - L and the
// 16 inverse column tiles of transform g - 2L.  Without launch boundaries
// the passes of different transforms overlap, so a batch too small to fill
// the SMs in whole waves of each pass (a rank's share of a strong-scaled
// batch) loses no partial-wave tails; a transform's intermediate is consumed
// from L2.  Readiness: ctr[1 + f] counts the finished column tiles (16) then
// row blocks (32) of transform f, released after the item's stores
// (bar.sync, then fence + atomic by one thread), acquired by the consumer's
// first thread before its loads.  An item waits only on items with smaller
// tickets, all claimed by running CTAs, so the kernel cannot deadlock,
// whatever the residency.  Same arithmetic per element as the three
// launches: bit-identical results.
constexpr int kF4FlowTpf = 48;   // items per transform (16 + 16 + 16)
constexpr size_t kF4FlowSmem = sizeof(float2) * (256 * kF4Pitch + 768);   // the row scratch fits the tile
static_assert(16 * 16 * 17 <= 256 * kF4Pitch, "row scratch of 16 rows inside the column tile");

__device__ __forceinline__ int64_t f4_slots_before(int64_t g, int64_t nf, int64_t L) {
    auto cl = [nf](int64_t v) { return v < 0 ? (int64_t)0 : v > nf ? nf : v; };
    return cl(g) + cl(g - L) + cl(g - 2 * L);
}
// the slot group of slot s: the largest g with slots_before(g) <= s.  For
// nf >= 2L, slots_before is linear on [0, L), [L, 2L), [2L, nf), [nf, nf + L)
// and [nf + L, nf + 2L) with slopes 1, 2, 3, 2, 1 — solved directly (checked
// against the binary search for every slot of nf < 1000, L <= 64); a binary
// search otherwise
__device__ __forceinline__ int64_t f4_slot_group(int64_t s, int64_t nf, int64_t L) {
    if (nf >= 2 * L) {
        if (s < L) return s;
        if (s < 3 * L) return (s + L) >> 1;
        if (s < 3 * nf - 3 * L) return (s + 3 * L) / 3;
        if (s < 3 * nf - L) return (s - nf + 3 * L) >> 1;
        return s - 2 * nf + 2 * L;
    }
    int64_t lo = 0, hi = nf + 2 * L - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (f4_slots_before(mid, nf, L) <= s) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(128, 4) k_fft4_flow(const float2* in, float2* out, int64_t nf, int64_t L,
                                                      unsigned* ctr) {
    extern __shared__ float4 f4f_smem[];
    float2* tile = reinterpret_cast<float2*>(f4f_smem);
    float2* tb = tile + 256 * kF4Pitch;
    __shared__ long long s_item[2];
    f4_tables(tb);
    const int64_t total = nf * kF4FlowTpf;
    long long next = 0;
    if (threadIdx.x == 0) next = (long long)atomicAdd(ctr, 1u);
    for (;;) {
        if (threadIdx.x == 0) {
            const long long t = next;
            long long kind = -1, f = 0, sub = 0;
            if (t < total) {
                next = (long long)atomicAdd(ctr, 1u);   // claim the next item early
                const int64_t s = t >> 4;
                sub = t & 15;
                const int64_t lo = f4_slot_group(s, nf, L);
                int64_t j = s - f4_slots_before(lo, nf, L);
                for (int q = 0; q < 3; ++q) {
                    const int64_t g = lo - q * L;
                    if (g < 0 || g >= nf) continue;
                    if (j-- == 0) {
                        kind = q;
                        f = g;
                        break;
                    }
                }
                if (kind > 0) {   // wait for the producing pass of transform f
                    const unsigned need = kind == 1 ? 16u : 32u;
                    const unsigned* p = ctr + 1 + f;
                    while (ld_acquire_u32(p) < need) __nanosleep(256);
                }
            }
            s_item[0] = kind;
            s_item[1] = (f << 4) | sub;
        }
        __syncthreads();
        const long long kind = s_item[0], fs = s_item[1];
        if (kind < 0) break;
        const int64_t f = fs >> 4;
        const int sub = (int)(fs & 15);
        if (kind == 0) f4_col_tile<false>(in, out, f, sub * kF4Cols, tile, tb);
        else if (kind == 1) f4_row_block(out, f, sub * 16, tile, tb);
        else f4_col_tile<true>(out, out, f, sub * kF4Cols, tile, tb);
        __syncthreads();   // every store of the item issued; the tile is free
        // release by the last warp, overlapping thread 0's claim and wait (a
        // release RMW: unlike a fence it does not invalidate the SM's L1)
        if (kind < 2 && threadIdx.x == blockDim.x - 32)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 1 + f) : "memory");
    }
}

// ---- 16 x 4096 four-step path (MW_TUNE_FFT_4STEP = 4) for the fused
// pipeline(fft, ifft) at N = 65536: n = c + 4096 r (c < 4096, r < 16),
// k = k1 + 16 k2:
//   A:     Y[k1][c] = sum_r x[c + 4096 r] W_16^{r k1}, times W_N^{c k1}
//   B:     X[k1 + 16 k2] = sum_c Y'[k1][c] W_4096^{c k2}; B^-1 over k2, then
//          times W_N^{-c k1}
//   A^-1:  x[c + 4096 r] = (1/N) sum_k1 Z'[k1][c] W_16^{-r k1}
// The column passes are one register DFT-16 per thread over 16 loads that
// are coalesced across the warp (consecutive c): no shared memory at all.
// The row pass holds one contiguous 4096-point row per CTA: DFT-4096 =
// 16 x 256 (c = t + 256 j, k2 = m + 16 k'): a DFT-16 over j per thread t,
// twiddle W_4096^{t m}, a transpose through shared memory, a DFT-256 over t
// per half-warp (m = half-warp), then the inverse mirrored (spectrum never
// leaves the registers).  Against the 256 x 256 path this halves the
// shared-memory traffic (the 256-point column DFTs needed staged tiles).
__device__ __forceinline__ float2 tw65536g(int e, bool inv) {
    float2 w = cmul(__ldg(&g_w16hi[e >> 8]), __ldg(&g_w16lo[e & 255]));
    if (inv) w.y = -w.y;
    return w;
}

// pass A (INV = false: DFT-16 over r, times W_N^{c k1}) and pass A^-1
// (INV = true: inverse DFT-16 over k1, times 1/N), one column per thread,
// in place on `out` (reading `in` on the forward pass)
template <bool INV>
__device__ __forceinline__ void f16_col(const float2* in, float2* out, int64_t f, int b) {
    const int c = b * 256 + threadIdx.x;
    const float2* src = in + f * 65536 + c;
    float2* dst = out + f * 65536 + c;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = src[r * 4096];
    dft<16, INV>(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (!INV) {
            if (k > 0) v[k] = cmul(v[k], tw65536g((c * k) & 65535, false));
            dst[k * 4096] = v[k];
        } else {
            st_cs(dst + k * 4096, make_float2(v[k].x * (1.0f / 65536.0f), v[k].y * (1.0f / 65536.0f)));
        }
    }
}
template <bool INV>
__global__ void __launch_bounds__(256) k_fft16_cols(const float2* in, float2* out, int64_t f0) {
    f16_col<INV>(in, out, f0 + blockIdx.x / 16, blockIdx.x % 16);
}

// DFT-256 by a half-warp: lane l holds x[l + 16 j] (j < 16) and ends with
// X[l + 16 j]; sc is the half-warp's [16][17] scratch (dft256_hw2 for one row)
template <bool INV>
__device__ __forceinline__ void dft256_hw1(float2 (&a)[16], int l, float2* sc, const float2* w256) {
    dft<16, INV>(a);
#pragma unroll
    for (int k = 1; k < 16; ++k) a[k] = cmulw<INV>(a[k], w256[k * 16 + l]);
#pragma unroll
    for (int k = 0; k < 16; ++k) sc[k * 17 + l] = a[k];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = sc[l * 17 + j];
    __syncwarp();
    dft<16, INV>(a);
}

// pass B, B^-1 and W_N^{-c k1} on row k1 of transform f (one row per CTA of
// 256 threads), in place
constexpr int kF16Pitch = 272;   // >= 256 points of a row, and >= 16 x 17 scratch
constexpr size_t kF16RowSmem = sizeof(float2) * (16 * kF16Pitch + 768);
// (S: 16 x kF16Pitch float2; tb: the W_256 table, filled and synchronised)
__device__ __forceinline__ void f16_row(float2* out, int64_t f, int k1, float2* S, const float2* tb) {
    float2* row = out + f * 65536 + (int64_t)k1 * 4096;
    const int t = threadIdx.x;
    float2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[t + 256 * j];
    dft<16, false>(v);   // U[t][m]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        if (m > 0) v[m] = cmul(v[m], __ldg(&g_w4096t[m * 256 + t]));
        S[m * kF16Pitch + t] = v[m];
    }
    __syncthreads();
    const int h = t >> 4, l = t & 15;   // half-warp h: m = h
    float2* Sh = S + h * kF16Pitch;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = Sh[l + 16 * i];
    __syncwarp();   // the row is in registers: its storage is the scratch now
    dft256_hw1<false>(v, l, Sh, tb);   // X[m + 16 k'], k' = l + 16 i
    dft256_hw1<true>(v, l, Sh, tb);    // 256 U'[t][m], t = l + 16 i
#pragma unroll
    for (int i = 0; i < 16; ++i) Sh[l + 16 * i] = v[i];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        v[m] = S[m * kF16Pitch + t];
        if (m > 0) v[m] = cmulw<true>(v[m], __ldg(&g_w4096t[m * 256 + t]));
    }
    dft<16, true>(v);   // 4096 Y'[t + 256 j]
    // W_N^{-c k1}, c = t + 256 j: W_N^{t k1} (table [k1][t]) W_256^{j k1}
    const float2 wt = __ldg(&g_w65536t[k1 * 256 + t]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float2 w = j == 0 ? wt : cmul(wt, tb[j * 16 + k1]);   // tb[0..255]: W_256^(a b) at [a][b]
        row[t + 256 * j] = k1 == 0 ? v[j] : cmulw<true>(v[j], w);
    }
}
__global__ void __launch_bounds__(256) k_fft16_rows_fi(float2* out, int64_t f0) {
    extern __shared__ float4 f16_smem[];
    float2* S = reinterpret_cast<float2*>(f16_smem);
    float2* tb = S + 16 * kF16Pitch;
    f4_tables(tb);
    __syncthreads();
    f16_row(out, f0 + blockIdx.x / 16, blockIdx.x % 16, S, tb);
}

// The 16 x 4096 passes as ONE persistent dataflow launch (the scheme of
// k_fft4_flow: tickets, slot groups g = A of g, B of g - L, A^-1 of g - 2L,
// readiness counters per transform; 16 column blocks of 256 columns, 16
// rows, 16 inverse column blocks per transform): the intermediate is
// consumed from L2, so HBM sees the input once and the output once and the
// HBM-bound column passes overlap the SM-bound row pass.  Same arithmetic
// per element as k_fft16_*: bit-identical results.
__global__ void __launch_bounds__(256, 3) k_fft16_flow(const float2* in, float2* out, int64_t nf, int64_t L,
                                                       unsigned* ctr) {
    extern __shared__ float4 f16f_smem[];
    float2* S = reinterpret_cast<float2*>(f16f_smem);
    float2* tb = S + 16 * kF16Pitch;
    __shared__ long long s_item[2];
    f4_tables(tb);
    const int64_t total = nf * kF4FlowTpf;
    long long next = 0;
    if (threadIdx.x == 0) next = (long long)atomicAdd(ctr, 1u);
    for (;;) {
        if (threadIdx.x == 0) {
            const long long t = next;
            long long kind = -1, f = 0, sub = 0;
            if (t < total) {
                next = (long long)atomicAdd(ctr, 1u);   // claim the next item early
                const int64_t s = t >> 4;
                sub = t & 15;
                const int64_t lo = f4_slot_group(s, nf, L);
                int64_t j = s - f4_slots_before(lo, nf, L);
                for (int q = 0; q < 3; ++q) {
                    const int64_t g = lo - q * L;
                    if (g < 0 || g >= nf) continue;
                    if (j-- == 0) {
                        kind = q;
                        f = g;
                        break;
                    }
                }
                if (kind > 0) {   // wait for the producing pass of transform f
                    const unsigned need = kind == 1 ? 16u : 32u;
                    const unsigned* p = ctr + 1 + f;
                    while (ld_acquire_u32(p) < need) __nanosleep(256);
                }
            }
            s_item[0] = kind;
            s_item[1] = (f << 4) | sub;
        }
        __syncthreads();
        const long long kind = s_item[0], fs = s_item[1];
        if (kind < 0) break;
        const int64_t f = fs >> 4;
        const int sub = (int)(fs & 15);
        if (kind == 0) f16_col<false>(in, out, f, sub);
        else if (kind == 1) f16_row(out, f, sub, S, tb);
        else f16_col<true>(out, out, f, sub);
        __syncthreads();   // every store of the item issued; S is free
        // release by the last warp while thread 0 claims and waits for the
        // next item (off the CTA's critical path), as a release RMW: unlike a
        // fence it does not invalidate the SM's L1
        if (kind < 2 && threadIdx.x == blockDim.x - 32)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 1 + f) : "memory");
    }
}

cudaError_t fft16_fi(const float2* in, float2* out, int64_t nfft, const Launch& L) {
    static bool attr = [] {
        cudaFuncSetAttribute(k_fft16_rows_fi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF16RowSmem);
        return true;
    }();
    (void)attr;
    const unsigned grid = (unsigned)(nfft * 16);
    note_launch();
    k_fft16_cols<false><<<grid, 256, 0, L.stream>>>(in, out, 0);
    note_launch();
    k_fft16_rows_fi<<<grid, 256, kF16RowSmem, L.stream>>>(out, 0);
    note_launch();
    k_fft16_cols<true><<<grid, 256, 0, L.stream>>>(out, out, 0);
    return cudaGetLastError();
}

static int64_t tuning_chunk() {
    static const int64_t c = [] {
        const char* v = getenv("MW_FFT4_CHUNK");
        return v ? (int64_t)atoi(v) : (int64_t)512;
    }();
    return c;
}

static int64_t tuning_lag() {
    static const int64_t c = [] {
        const char* v = getenv("MW_FFT4_LAG");
        return v ? (int64_t)atoi(v) : (int64_t)64;
    }();
    return c;
}
// the dataflow launch: L.work holds (1 + nfft) counters, zeroed here
cudaError_t fft4_flow(const float2* in, float2* out, int64_t nfft, const Launch& L) {
    static int per_sm = [] {
        cudaFuncSetAttribute(k_fft4_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4FlowSmem);
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fft4_flow, 128, kF4FlowSmem) != cudaSuccess || n < 1)
            n = 1;
        return n;
    }();
    const size_t need = (size_t)(nfft + 1) * sizeof(unsigned);
    if (!L.work || L.work_bytes < need || nfft * kF4FlowTpf >= (int64_t)UINT32_MAX) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(L.work, 0, need, L.stream);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > nfft * kF4FlowTpf) grid = nfft * kF4FlowTpf;
    note_launch();
    k_fft4_flow<<<(unsigned)grid, 128, kF4FlowSmem, L.stream>>>(in, out, nfft, tuning_lag(),
                                                                 static_cast<unsigned*>(L.work));
    return cudaGetLastError();
}

// The 16 x 4096 dataflow launch: L.work holds (1 + nfft) counters, zeroed
// here.  Measured on the 512-transform batch: 0.258 ms at lag 40 against
// 0.315 ms for the three launches on the same box (lag 24 / 32 / 48: 0.274 /
// 0.262 / 0.2585);
// 256 / 128 / 64 transforms: 146 / 82 / 47 us against 163 / 83 / 48 us.
static int64_t tuning_lag16() {
    static const int64_t c = [] {
        const char* v = getenv("MW_FFT16_LAG");
        return v ? (int64_t)atoi(v) : (int64_t)40;
    }();
    return c;
}
cudaError_t fft16_flow(const float2* in, float2* out, int64_t nfft, const Launch& L) {
    static int per_sm = [] {
        cudaFuncSetAttribute(k_fft16_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF16RowSmem);
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fft16_flow, 256, kF16RowSmem) != cudaSuccess || n < 1)
            n = 1;
        return n;
    }();
    const size_t need = (size_t)(nfft + 1) * sizeof(unsigned);
    if (!L.work || L.work_bytes < need || nfft * kF4FlowTpf >= (int64_t)UINT32_MAX) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(L.work, 0, need, L.stream);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > nfft * kF4FlowTpf) grid = nfft * kF4FlowTpf;
    note_launch();
    k_fft16_flow<<<(unsigned)grid, 256, kF16RowSmem, L.stream>>>(in, out, nfft, tuning_lag16(),
                                                                  static_cast<unsigned*>(L.work));
    return cudaGetLastError();
}

cudaError_t fft4_fi(const float2* in, float2* out, int64_t nfft, const Launch& L) {
    // 16 x 4096 as 1 (one dataflow launch, default) or 4 (three launches);
    // 256 x 256 as 2 (dataflow launch) or 3 (three launches) — the 16 x 4096
    // forms are faster at every batch size measured, its dataflow launch as
    // fast as its three launches from 64 transforms and faster from 256
    const int form = L.tune[TUNE_FFT_4STEP];
    if (form == 1) return fft16_flow(in, out, nfft, L);
    if (form == 4) return fft16_fi(in, out, nfft, L);
    if (form == 2) return fft4_flow(in, out, nfft, L);
    static bool attr = [] {
        cudaFuncSetAttribute(k_fft4_cols<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4ColSmem);
        cudaFuncSetAttribute(k_fft4_cols<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4ColSmem);
        cudaFuncSetAttribute(k_fft4_rows_fi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4RowSmem);
        return true;
    }();
    (void)attr;
    const int64_t chunk = tuning_chunk();   // transforms per launch triple
    for (int64_t f0 = 0; f0 < nfft; f0 += chunk) {
        const int64_t nf = nfft - f0 < chunk ? nfft - f0 : chunk;
        const unsigned cgrid = (unsigned)(nf * (256 / kF4Cols));
        note_launch();
        k_fft4_cols<false><<<cgrid, 128, kF4ColSmem, L.stream>>>(in, out, f0);
        note_launch();
        k_fft4_rows_fi<<<(unsigned)(nf * 8), 256, kF4RowSmem, L.stream>>>(out, f0);
        note_launch();
        k_fft4_cols<true><<<cgrid, 128, kF4ColSmem, L.stream>>>(out, out, f0);
    }
    return cudaGetLastError();
}

template <int C, int MODE>
cudaError_t fft_launch(const float2* in, float2* out, int64_t nfft, const Launch& L) {
    static int max_clusters = -1;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    if (max_clusters < 0) {
        cudaError_t e = cudaFuncSetAttribute(k_fft<C, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kFftSmem);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * 1024);
        cfg.blockDim = dim3(FT);
        cfg.dynamicSmemBytes = kFftSmem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_fft<C, MODE>, &cfg) != cudaSuccess || n < 1) n = 1;
        max_clusters = n;
    }
    int64_t clusters = nfft < max_clusters ? nfft : max_clusters;
    if (L.slow > 1.0f) clusters = (int64_t)((double)clusters / (double)L.slow + 0.999);
    if (clusters < 1) clusters = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * C));
    cfg.blockDim = dim3(FT);
    cfg.dynamicSmemBytes = kFftSmem;
    cfg.stream = L.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    note_launch();
    return cudaLaunchKernelEx(&cfg, k_fft<C, MODE>, in, out, nfft);
}

template <int C>
cudaError_t fft_launch_mode(int mode, const float2* in, float2* out, int64_t nfft, const Launch& L) {
    switch (mode) {
        case FFT_F: return fft_launch<C, FFT_F>(in, out, nfft, L);
        case FFT_I: return fft_launch<C, FFT_I>(in, out, nfft, L);
        default: return fft_launch<C, FFT_FI>(in, out, nfft, L);
    }
}

}  // namespace

bool fft_supported(int log2n) { return log2n >= 13 && log2n <= 16; }

cudaError_t fft_prepare(cudaStream_t s) {
    static std::mutex mu;
    static std::set<int> filled;   // devices whose g_tw13 is written (one module copy per device)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (filled.count(dev)) return cudaSuccess;
    k_fft_tw13<<<(16 * 512 + 3 * 256 + 2 * 4096 + 255) / 256, 256, 0, s>>>();
    e = cudaGetLastError();
    if (e == cudaSuccess) filled.insert(dev);
    return e;
}

size_t fft_work_bytes(int64_t nfft, int log2n) {
    return log2n == 16 ? (size_t)(nfft + 1) * sizeof(unsigned) : 0;
}

cudaError_t fft_chain(const float* in, float* out, int64_t nfft, int log2n, uint32_t inv, int nst,
                      const Launch& L) {
    if (nfft <= 0) return cudaSuccess;
    if (nst > 32 || !fft_supported(log2n)) return cudaErrorInvalidValue;
    {
        cudaError_t e = fft_prepare(L.stream);   // no-op after the context's creation
        if (e != cudaSuccess) return e;
    }
    const float2* src = reinterpret_cast<const float2*>(in);
    float2* o2 = reinterpret_cast<float2*>(out);
    if (nst == 0) {
        if (in != out) return cudaMemcpyAsync(out, in, (size_t)nfft << (log2n + 3), cudaMemcpyDeviceToDevice, L.stream);
        return cudaSuccess;
    }
    // greedy grouping: a forward followed by an inverse is one fused launch
    for (int s = 0; s < nst;) {
        const bool iv = (inv >> s) & 1;
        int mode = iv ? FFT_I : FFT_F;
        int used = 1;
        if (!iv && s + 1 < nst && ((inv >> (s + 1)) & 1)) {
            mode = FFT_FI;
            used = 2;
        }
        cudaError_t e;
        // a four-step path for the fused pair at 2^16 (the slowdown injector's
        // clamped grids stay on the cluster path, whose clusters are persistent)
        if (mode == FFT_FI && log2n == 16 && L.tune[TUNE_FFT_4STEP] && !(L.slow > 1.0f)) {
            e = fft4_fi(src, o2, nfft, L);
            if (e != cudaSuccess) return e;
            src = o2;
            s += used;
            continue;
        }
        switch (log2n) {
            case 13: e = fft_launch_mode<1>(mode, src, o2, nfft, L); break;
            case 14: e = fft_launch_mode<2>(mode, src, o2, nfft, L); break;
            case 15: e = fft_launch_mode<4>(mode, src, o2, nfft, L); break;
            default: e = fft_launch_mode<8>(mode, src, o2, nfft, L); break;
        }
        if (e != cudaSuccess) return e;
        src = o2;   // later launches run in place on the output
        s += used;
    }
    return cudaSuccess;
}

}  // namespace mwk
