// Useful bandwidth of random contiguous segment reads vs segment length on
// B200: one warp reads one SEG-word segment (random start, 16-B aligned) at a
// time with 16-byte vector loads, U segments in flight per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int U>
__global__ void __launch_bounds__(1024, 1) k(const uint4* a, uint64_t n16, uint32_t seg16, int iters, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31, warp = (blockIdx.x * 1024 + threadIdx.x) >> 5;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t start = (hash(warp * 7919u + it * 131u + u * 17u) * 2654435761ull) % (n16 - seg16);
            v[u] = lane < seg16 ? a[start + lane] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
        // segments longer than 32 x 16 B: the rest sequentially
        for (uint32_t o = 32; o < seg16; o += 32) {
            const uint64_t start = (hash(warp * 7919u + it * 131u) * 2654435761ull) % (n16 - seg16);
            if (lane + o < seg16) acc += a[start + o + lane].y;
        }
    }
    if (acc == 0x12345678) out[0] = acc;
}
int main() {
    const uint64_t bytes = 4ull << 30, n16 = bytes / 16;
    uint4* a; cudaMalloc(&a, bytes); cudaMemset(a, 1, bytes);
    uint32_t* out; cudaMalloc(&out, 4);
    const uint32_t segs[] = {8, 16, 32, 128, 512};  // x16 bytes: 128 B .. 8 KB
    for (uint32_t s16 : segs) {
        const int iters = s16 >= 128 ? 8 : 64;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<4><<<148, 1024>>>(a, n16, s16, iters, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double per_iter = 4.0 * (s16 < 32 ? s16 : 32) * 16 + (s16 > 32 ? (s16 - 32) * 16.0 : 0.0);
            if (rep == 1) printf("segment %6u B: %7.1f GB/s useful\n", s16 * 16, 148.0 * 32 * iters * per_iter / ms / 1e6);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
