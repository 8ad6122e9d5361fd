// reduce.cu — the MapReduce reduction (R9, R28): per-element fp64 terms of
// the map stage (x, x*y, or a fused saxpy chain) folded in canonical 2^16
// chunks into fixed-order partials, the combine, the identity fill for the
// max / min reduction stage, and the partition traits (SIZE / OFFSET).
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
#include "kcommon.cuh"

namespace mwk {
namespace {

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
