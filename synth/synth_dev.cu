// synth_dev.cu — device twin of synth_host.c (same SplitMix64 streams, same
// recipes; see the header comment there).  Holds no arithmetic of the method.
// C-ABI: every fill writes `count` elements of the stream starting at global
// element `start` into device memory `out`, enqueued on `stream`
// (cudaStream_t passed as void*).  Returns 0 or a cudaError_t code.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t s, uint64_t i) {
    uint64_t z = s + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void synth_gen_f32_um11(uint64_t seed, uint64_t start, uint64_t n, float* out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = (float)(sm64(seed, start + k) >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

__global__ void synth_gen_f32_u01(uint64_t seed, uint64_t start, uint64_t n, float* out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = (float)(sm64(seed, start + k) >> 40) * (1.0f / 16777216.0f);
}

__global__ void synth_gen_u8(uint64_t seed, uint64_t start, uint64_t n, uint8_t* out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = start + k;
        out[k] = (uint8_t)(sm64(seed, v >> 3) >> (8 * (v & 7)));
    }
}

__global__ void synth_gen_rgba(uint64_t seed, uint64_t start, uint64_t n, uint32_t* out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = sm64(seed, start + k);
        out[k] = (uint32_t)(z & 0xFFFFFFull) | 0xFF000000u;
    }
}

__global__ void synth_gen_nbody(uint64_t seed, uint64_t start, uint64_t n, float mass,
                        float4* pos, float4* vel) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b = start + k;
        float4 p;
        p.x = (float)(sm64(seed, 3 * b + 0) >> 40) * (1.0f / 8388608.0f) - 1.0f;
        p.y = (float)(sm64(seed, 3 * b + 1) >> 40) * (1.0f / 8388608.0f) - 1.0f;
        p.z = (float)(sm64(seed, 3 * b + 2) >> 40) * (1.0f / 8388608.0f) - 1.0f;
        p.w = mass;
        pos[k] = p;
        if (vel) vel[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

inline unsigned grid_for(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    if (g > 148ull * 64) g = 148ull * 64;
    return g ? (unsigned)g : 1u;
}

}  // namespace

#define SYNTH_RET(launch)                                   \
    do {                                                    \
        if (count == 0) return 0;                           \
        launch;                                             \
        return (int)cudaGetLastError();                     \
    } while (0)

extern "C" {

int synth_dev_f32_um11(uint64_t seed, uint64_t start, uint64_t count, float* out, void* stream) {
    SYNTH_RET((synth_gen_f32_um11<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(seed, start, count, out)));
}
int synth_dev_f32_u01(uint64_t seed, uint64_t start, uint64_t count, float* out, void* stream) {
    SYNTH_RET((synth_gen_f32_u01<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(seed, start, count, out)));
}
int synth_dev_u8_stream(uint64_t seed, uint64_t start, uint64_t count, uint8_t* out, void* stream) {
    SYNTH_RET((synth_gen_u8<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(seed, start, count, out)));
}
int synth_dev_rgba(uint64_t seed, uint64_t start_px, uint64_t count, uint8_t* out, void* stream) {
    SYNTH_RET((synth_gen_rgba<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(seed, start_px, count,
                                                                         (uint32_t*)out)));
}
int synth_dev_nbody(uint64_t seed, uint64_t start, uint64_t count, float mass, float* pos4,
                    float* vel4, void* stream) {
    SYNTH_RET((synth_gen_nbody<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(
        seed, start, count, mass, (float4*)pos4, (float4*)vel4)));
}

}  // extern "C"
