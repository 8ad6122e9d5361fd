// Two cooperative kernels from two threads: co-resident or serialized,
// depending on the size of the kernel's parameter block?
#include <cstdio>
#include <thread>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
template <int NB>
struct Big { int pad[NB / 4]; };
template <int NB>
__global__ void k(const __grid_constant__ Big<NB> b, int* mine, int* other, int* met) {
    extern __shared__ int sm[];
    cg::grid_group g = cg::this_grid();
    sm[threadIdx.x] = b.pad[threadIdx.x % (NB / 4)];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd_system(mine, 1);
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            int v;
            asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(other) : "memory");
            if (v > 0) { *met = 1; break; }
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 1000000000ull) { *met = 0; break; }
        }
    }
    g.sync();
}
template <int NB>
void run() {
    int *f, *met;
    cudaMalloc(&f, 16);
    cudaMalloc(&met, 16);
    const int smem = 110 * 1024;
    cudaFuncSetAttribute(k<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(f, 0, 16);
    cudaMemset(met, 0xff, 16);
    cudaDeviceSynchronize();
    Big<NB> b{};
    auto launch = [&](int i) {
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        int* a = f + i; int* bb = f + (1 - i); int* m = met + i;
        void* args[] = {&b, &a, &bb, &m};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k<NB>, 1, 256, args, smem, s);
        if (e != cudaSuccess) printf("launch %d: %s\n", i, cudaGetErrorString(e));
        cudaStreamSynchronize(s);
    };
    std::thread t0(launch, 0), t1(launch, 1);
    t0.join();
    t1.join();
    int h[2];
    cudaMemcpy(h, met, 8, cudaMemcpyDeviceToHost);
    printf("param %d B: met = %d %d (%s)\n", NB, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<512>();
    run<3840>();
    run<4096>();
    run<8192>();
    return 0;
}
