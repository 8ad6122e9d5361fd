// kernels.cu — host side shared by the hand-written sm_100a kernel families.
//
// Every kernel is a grid-stride ("persistent-style") loop over tiles so the
// host can size the grid to SMs x resident CTAs (and clamp it for the
// slowdown injector) without changing results.  None of these stages is a
// dense contraction, so there are no tensor cores here: the fused Map chains,
// the stencil and the reduction are HBM-bound streams (128-bit coalesced
// accesses, SWAR / DPX byte arithmetic), N-body is FP32-pipe bound.
//
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
//
// This translation unit holds what the kernel families share on the host: the
// launch counter, tuning defaults / validation, the SM count, the batched
// device copies between partitions and the element-wise rank reduction of
// the loopback transport.  The families: chains.cu (saxpy, RGBA, u8),
// planes.cu (hysteresis), nbody.cu, reduce.cu (MapReduce), fft.cu.
#include "kcommon.cuh"

namespace mwk {
thread_local unsigned long long g_launches = 0;
namespace {
int g_sms = 0;
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
    out[TUNE_FFT_4STEP] = tuning_knob("MW_FFT_4STEP", 1);
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
        case TUNE_FFT_4STEP: return v >= 0 && v <= 4;
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

}  // namespace mwk
