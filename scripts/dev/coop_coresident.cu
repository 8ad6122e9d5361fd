// Can two cooperative kernels launched on two streams (from two host
// threads) run at the same time when each CTA takes ~110 KiB of dynamic
// shared memory?  Each kernel's block 0 bumps its own flag and waits
// (bounded) for the other's.
#include <cstdio>
#include <thread>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k(int* mine, int* other, int* met) {
    extern __shared__ int sm[];
    cg::grid_group g = cg::this_grid();
    sm[threadIdx.x] = threadIdx.x;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd_system(mine, 1);
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            int v;
            asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(other) : "memory");
            if (v > 0) { *met = 1; break; }
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 2000000000ull) { *met = 0; break; }
        }
    }
    g.sync();
}
int main() {
    int *f, *met;
    cudaMalloc(&f, 16);
    cudaMalloc(&met, 16);
    const int smem = 110 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 4; ++mode) {
        cudaMemset(f, 0, 16);
        cudaMemset(met, 0xff, 16);
        cudaDeviceSynchronize();
        const bool threads = mode & 1, coop = !(mode & 2);
        auto launch = [&](int i) {
            cudaStream_t s;
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            int* a = f + i; int* b = f + (1 - i); int* m = met + i;
            void* args[] = {&a, &b, &m};
            cudaError_t e = coop ? cudaLaunchCooperativeKernel((void*)k, 1, 256, args, smem, s)
                                 : cudaLaunchKernel((void*)k, 1, 256, args, smem, s);
            if (e != cudaSuccess) printf("launch %d: %s\n", i, cudaGetErrorString(e));
            cudaStreamSynchronize(s);
        };
        if (threads) {
            std::thread t0(launch, 0), t1(launch, 1);
            t0.join();
            t1.join();
        } else {
            std::thread t0(launch, 0);
            launch(1);
            t0.join();
        }
        int h[2];
        cudaMemcpy(h, met, 8, cudaMemcpyDeviceToHost);
        printf("%s %s smem %d: met = %d %d (%s)\n", coop ? "cooperative" : "plain", threads ? "2 threads" : "1+1",
               smem, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
