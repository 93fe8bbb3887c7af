// Microbenchmark: throughput of per-target arrival counting in shared memory
// on sm_100a (decides the receive-side accumulation design of
// include/synq/detail/persistent.cuh).  148 CTAs x 1024 threads, each lane
// issues ITERS increments to distinct (conflict-free) smem addresses.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 1024, ITERS = 4096, WORDS = 8192;

template <int MODE>
__global__ void __launch_bounds__(NT, 1) k(unsigned* out, unsigned long long* cyc, unsigned* g) {
    __shared__ unsigned s[WORDS];
    for (int i = threadIdx.x; i < WORDS; i += NT) s[i] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long t0 = clock64();
    unsigned base = warp * 97;
#pragma unroll 8
    for (int i = 0; i < ITERS; ++i) {
        unsigned a = (base + i * 32 + lane) & (WORDS - 1);
        if (MODE == 0) atomicAdd(&s[a], 1u);                       // ATOMS.POPC.INC
        if (MODE == 1) atomicAdd(&s[a], (unsigned)(i & 3) + 1u);   // ATOMS.ADD
        if (MODE == 2) { unsigned w = (warp * 256 + ((i * 32 + lane) & 255)); s[w] += 1; }  // private LDS+STS
        if (MODE == 3) atomicAdd(&g[(blockIdx.x * 65536 + base + i * 32 + lane) & ((1 << 24) - 1)], 1u);  // REDG
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    unsigned acc = 0;
    for (int i = threadIdx.x; i < WORDS; i += NT) acc += s[i];
    if (acc == 12345) out[0] = acc;
}

int main() {
    unsigned *out, *g; unsigned long long* cyc;
    cudaMalloc(&out, 4); cudaMalloc(&g, 4 << 24); cudaMalloc(&cyc, 8 * 148);
    const char* names[] = {"ATOMS.POPC.INC (atomicAdd 1)", "ATOMS.ADD (atomicAdd v)", "LDS+STS private", "REDG.ADD distinct"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148, NT>>>(out, cyc, g);
            if (mode == 1) k<1><<<148, NT>>>(out, cyc, g);
            if (mode == 2) k<2><<<148, NT>>>(out, cyc, g);
            if (mode == 3) k<3><<<148, NT>>>(out, cyc, g);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long c[148]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
            double ops = 148.0 * NT * ITERS;
            if (rep == 2)
                printf("%-30s %8.3f ms  %7.1f Gop/s  %6.2f cycles per warp-op per SM (%llu cyc/CTA)\n", names[mode], ms,
                       ops / ms / 1e6, (double)c[0] / (ITERS * (NT / 32.0)), c[0]);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
