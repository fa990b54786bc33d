// sync_cost.cu -- microbenchmark: cooperative grid.sync() and cluster barrier cost on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void grid_sync_loop(int iters, long long *out) {
    cg::grid_group grid = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) grid.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}

__global__ void __cluster_dims__(2, 1, 1) cluster_sync_loop(int iters, long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cl.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}

__global__ void block_sync_loop(int iters, long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}

int main() {
    long long *d, h;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bs : {256, 512, 1024}) {
        for (int per : {1, 2}) {
            if (bs * per > 2048) continue;
            int iters = 2000;
            void *args[] = {&iters, &d};
            cudaError_t e = cudaLaunchCooperativeKernel((void *)grid_sync_loop, sms * per, bs, args, 0, 0);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("grid.sync  grid=%d x %d threads: %lld cycles (%s)\n", sms * per, bs, h, cudaGetErrorString(e));
        }
    }
    cluster_sync_loop<<<sms, 1024>>>(2000, d);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster(2).sync 1024 threads: %lld cycles\n", h);
    block_sync_loop<<<sms, 1024>>>(2000, d);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads 1024 threads: %lld cycles\n", h);
    return 0;
}
