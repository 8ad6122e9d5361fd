// Measured ALU peaks of this B200 for the "alu"-bound roofline rows of
// bench.py (N-body: FP32 FMA pipe; hysteresis: integer ALU pipe).
//
// Each kernel keeps 8 independent dependency chains per thread (latency
// hidden by ILP and 16 warps per SM), a grid of 148 SMs x 4 CTAs x 256
// threads, and runs long enough (~50 ms) to be timed with CUDA events after a
// warm-up launch.  Outputs one JSON object per line:
//   ffma    scalar fp32 FFMA             (2 flop per lane-op)
//   ffma2   packed fp32x2 FFMA (FFMA2)   (4 flop per instruction)
//   lop3    integer LOP3.LUT             (1 op per lane-op)
//   shf     funnel shift SHF             (1 op per lane-op)
//   popc_xor POPC (XU pipe) + LOP3 per step (instructions per second)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = __fmaf_rn(x[c], a, b);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    unsigned long long x[kChains];
    unsigned long long av, bv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        float v = threadIdx.x * 1e-3f + c;
        asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(v));
    }
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(av), "l"(bv));
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= x[c];
    if (s == 12345ull) out[0] = (float)s;
}

template <int OP>
__global__ void k_int(unsigned* out, unsigned a, unsigned b) {
    unsigned x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 2654435761u + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == 0) {   // LOP3: x = (x ^ a) & b | ~x  (one LUT op)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            } else if (OP == 1) {   // SHF (funnel shift)
                asm volatile("shf.l.wrap.b32 %0, %0, %1, 3;" : "+r"(x[c]) : "r"(a));
            } else if (OP == 2) {   // IADD3
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(b));
            } else {   // POPC
                asm volatile("popc.b32 %0, %0;" : "+r"(x[c]));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            }
        }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= x[c];
    if (s == 12345u) out[0] = s;
}

template <typename F>
static double time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();   // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const dim3 grid(sms * 4), block(256);
    const double lanes = (double)grid.x * block.x;
    float* fo;
    unsigned* io;
    cudaMalloc(&fo, 64);
    cudaMalloc(&io, 64);
    auto report = [&](const char* name, double ms, double ops_per_lane_iter, double unit_per_op,
                      const char* unit) {
        const double ops = lanes * kIters * kChains * ops_per_lane_iter;
        printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"value\": %.4f, \"unit\": \"%s\", \"sms\": %d, "
               "\"clock_attr_mhz\": %.0f}\n",
               name, ms, ops * unit_per_op / (ms / 1e3) / 1e12, unit, sms, clk_khz / 1e3);
    };
    report("ffma", time_ms([&] { k_ffma<<<grid, block>>>(fo, 0.999f, 1e-3f); }), 1, 2, "TFLOP/s");
    report("ffma2", time_ms([&] { k_ffma2<<<grid, block>>>(fo, 0.999f, 1e-3f); }), 1, 4, "TFLOP/s");
    report("lop3", time_ms([&] { k_int<0><<<grid, block>>>(io, 0x9E3779B9u, 0x7F4A7C15u); }), 1, 1,
           "Tops/s");
    report("shf", time_ms([&] { k_int<1><<<grid, block>>>(io, 0x9E3779B9u, 0u); }), 1, 1, "Tops/s");
    report("popc_xor", time_ms([&] { k_int<3><<<grid, block>>>(io, 0x9E3779B9u, 0u); }), 2, 1,
           "Tinstr/s");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
