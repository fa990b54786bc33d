// mem_latency.cu -- microbenchmark: dependent-chain latency of global loads (L2 hit / DRAM),
// 64- and 128-bit atomic CAS, and shared-memory atomics on B200.  Informs the decoder design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__global__ void chase(const unsigned *next, int steps, unsigned start, long long *cyc, unsigned *sink) {
    unsigned p = start;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) p = __ldcg(&next[p]);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = (t1 - t0) / steps; *sink = p; }
}

__global__ void cas128_chain(u64 *slots, const unsigned *idx, int steps, long long *cyc, u64 *sink) {
    u64 acc = 0;
    unsigned j = 0;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
        u64 *p = slots + 2 * (size_t)idx[(j + i) & 1023];
        u64 elo = 0xFFFFFFFFFFFFFFFFull, ehi = 0xFFFFFFFFFFFFFFFFull, dlo = acc + i, dhi = 0, olo, ohi;
        asm volatile("{\n\t.reg .b128 e, d, o;\n\tmov.b128 e, {%2, %3};\n\tmov.b128 d, {%4, %5};\n\t"
                     "atom.relaxed.gpu.global.cas.b128 o, [%6], e, d;\n\tmov.b128 {%0, %1}, o;\n\t}"
                     : "=l"(olo), "=l"(ohi) : "l"(elo), "l"(ehi), "l"(dlo), "l"(dhi), "l"(p) : "memory");
        acc += olo & 1;
        j += (unsigned)(olo & 7);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = (t1 - t0) / steps; *sink = acc; }
}

__global__ void cas64_chain(u64 *slots, const unsigned *idx, int steps, long long *cyc, u64 *sink) {
    u64 acc = 0;
    unsigned j = 0;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
        u64 *p = slots + 2 * (size_t)idx[(j + i) & 1023];
        u64 o = atomicCAS(p, 0xFFFFFFFFFFFFFFFFull, acc + i);
        acc += o & 1;
        j += (unsigned)(o & 7);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = (t1 - t0) / steps; *sink = acc; }
}

int main() {
    const size_t N_small = 1 << 20, N_big = 1 << 28;  // 4 MB (L2) and 1 GB (DRAM) chains
    unsigned *next; u64 *slots; unsigned *idx; long long *cyc; unsigned *sink; u64 *sink64;
    cudaMalloc(&next, N_big * 4); cudaMalloc(&slots, N_big * 8); cudaMalloc(&idx, 4096 * 4);
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 4); cudaMalloc(&sink64, 8);
    unsigned *h = (unsigned *)malloc(N_big * 4);
    for (size_t n : {N_small, N_big}) {
        // random cyclic permutation with stride to defeat prefetch
        for (size_t i = 0; i < n; ++i) h[i] = (unsigned)((i * 2654435761ull + 12345) % n);
        cudaMemcpy(next, h, n * 4, cudaMemcpyHostToDevice);
        chase<<<1, 1>>>(next, 2000, 1, cyc, sink);  // warm
        chase<<<1, 1>>>(next, 20000, 7, cyc, sink);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("dependent ld.cg chain over %zu MB: %lld cycles/load\n", n * 4 >> 20, c);
    }
    for (int i = 0; i < 4096; ++i) h[i] = (unsigned)((i * 2654435761ull) % (N_big / 2));
    cudaMemcpy(idx, h, 4096 * 4, cudaMemcpyHostToDevice);
    cudaMemset(slots, 0xFF, N_big * 8);
    cas128_chain<<<1, 1>>>(slots, idx, 4000, cyc, sink64);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent CAS.128 (random, mostly DRAM-cold): %lld cycles/op\n", c);
    cas128_chain<<<1, 1>>>(slots, idx, 4000, cyc, sink64);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent CAS.128 (same 1024 lines, L2-warm): %lld cycles/op\n", c);
    cas64_chain<<<1, 1>>>(slots, idx, 4000, cyc, sink64);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent CAS.64 (L2-warm): %lld cycles/op\n", c);
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
