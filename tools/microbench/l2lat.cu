// Microbenchmark: L2 latency / throughput under load for random 16-byte
// loads from an L2-resident buffer (sizes 8 MB .. 4 GB).  148 CTAs x 512
// threads; every thread issues U independent loads per round (addresses
// depend on the previous round's data, so rounds are serial), R rounds.
// Reports ns per round (= loaded latency) and GB/s of 16-byte loads.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__host__ __device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352d;
    x ^= x >> 15;
    x *= 0x846ca68b;
    x ^= x >> 16;
    return x;
}

template <int U, int MODE>
__global__ void __launch_bounds__(512, 1) k(const uint4* a, uint32_t n16, int R, uint32_t* sink) {
    uint32_t x = hash(blockIdx.x * 512 + threadIdx.x);
    for (int r = 0; r < R; ++r) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = hash(x + u * 977u) % n16;
            if (MODE == 0)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(a + i));
            else
                asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(a + i));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x += v[u].x ^ v[u].w;
    }
    if (x == 0x1234567) sink[0] = x;
}

int main() {
    uint4* a;
    uint32_t* sink;
    const size_t maxb = 4ull << 30;
    cudaMalloc(&a, maxb);
    cudaMemset(a, 0, maxb);
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int R = 200;
    for (size_t mb : {8, 32, 96, 4096}) {
        const uint32_t n16 = uint32_t(mb * (1 << 20) / 16);
        for (int U : {1, 4, 8, 16}) {
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (U == 1) k<1, 0><<<148, 512>>>(a, n16, R, sink);
                if (U == 4) k<4, 0><<<148, 512>>>(a, n16, R, sink);
                if (U == 8) k<8, 0><<<148, 512>>>(a, n16, R, sink);
                if (U == 16) k<16, 0><<<148, 512>>>(a, n16, R, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double loads = 148.0 * 512 * U * R;
            printf("buf %5zu MB U=%2d: %7.1f ns/round  %7.1f GB/s  (%.1f G loads/s)\n", mb, U, ms * 1e6 / R,
                   loads * 16 / (ms * 1e-3) / 1e9, loads / (ms * 1e-3) / 1e9);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
