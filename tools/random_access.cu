// random_access.cu -- microbenchmark: all-SM random 8/16-byte gathers, RED.MIN.64 and
// CAS.128 throughput over a working set that misses (1-4 GB) or hits (64 MB) L2.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void gather16(const ulonglong2 *a, u64 n, int iters, u64 *sink) {
    unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (int i = 0; i < iters; ++i) {
        unsigned idx = hsh(t * 7919u + i * 104729u) % (unsigned)n;
        ulonglong2 v = __ldcg(&a[idx]);
        acc += v.x ^ v.y;
    }
    if (acc == 42) *sink = acc;
}
__global__ void redmin64(u64 *a, u64 n, int iters) {
    unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        unsigned idx = hsh(t * 7919u + i * 104729u) % (unsigned)n;
        atomicMin(&a[2 * (u64)idx], (u64)(t + i));
    }
}
__global__ void cas128(u64 *a, u64 n, int iters, u64 *sink) {
    unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (int i = 0; i < iters; ++i) {
        unsigned idx = hsh(t * 7919u + i * 104729u) % (unsigned)n;
        u64 *p = a + 2 * (u64)idx;
        u64 elo = ~0ull, ehi = ~0ull, dlo = t, dhi = i, olo, ohi;
        asm volatile("{\n\t.reg .b128 e, d, o;\n\tmov.b128 e, {%2, %3};\n\tmov.b128 d, {%4, %5};\n\t"
                     "atom.relaxed.gpu.global.cas.b128 o, [%6], e, d;\n\tmov.b128 {%0, %1}, o;\n\t}"
                     : "=l"(olo), "=l"(ohi) : "l"(elo), "l"(ehi), "l"(dlo), "l"(dhi), "l"(p) : "memory");
        acc += olo ^ ohi;
    }
    if (acc == 42) *sink = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    u64 *a, *sink; size_t bytes = (size_t)4 << 30;
    cudaMalloc(&a, bytes); cudaMalloc(&sink, 8); cudaMemset(a, 0xff, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (size_t ws : {(size_t)64 << 20, (size_t)1 << 30, (size_t)4 << 30}) {
        u64 n = ws / 16;
        int blocks = sms * 8, threads = 256, iters = 64;
        double ops = (double)blocks * threads * iters;
        float ms;
        gather16<<<blocks, threads>>>((ulonglong2 *)a, n, iters, sink);
        cudaEventRecord(e0); gather16<<<blocks, threads>>>((ulonglong2 *)a, n, iters, sink); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("ws=%5zu MB  random 16B gather : %6.2f G/s\n", ws >> 20, ops / ms / 1e6);
        cudaEventRecord(e0); redmin64<<<blocks, threads>>>(a, n, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("ws=%5zu MB  random RED.MIN.64 : %6.2f G/s\n", ws >> 20, ops / ms / 1e6);
        cudaEventRecord(e0); cas128<<<blocks, threads>>>(a, n, iters, sink); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("ws=%5zu MB  random CAS.128    : %6.2f G/s\n", ws >> 20, ops / ms / 1e6);
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
