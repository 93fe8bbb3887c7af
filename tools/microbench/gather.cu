// Microbenchmark: scattered row-segment gathers as in Receive Spikes.
// Each warp reads SEG consecutive u32 from a random 128-B-aligned row start
// (+ random 4-B offset) of an ARRAY_GB array; U independent segments in
// flight per warp; 148 CTAs x 1024 threads.  Reports useful GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int U, int MODE>
__global__ void __launch_bounds__(1024, 1) k(const uint32_t* a, uint64_t words, uint64_t pitch, int iters, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31, warp = (blockIdx.x * 1024 + threadIdx.x) >> 5;
    const uint64_t rows = words / pitch;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash(warp * 7919u + it * 131u + u * 17u);
            const uint64_t row = h % rows;
            const uint64_t off = row * pitch + ((h >> 7) % (pitch - 40));
            if (MODE == 0) v[u] = __ldcg(a + off + lane);
            else if (MODE == 1) v[u] = __ldg(a + off + lane);
            else { uint32_t r; asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(a + off + lane)); v[u] = r; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    const double gbs[] = {0.25, 4.0};
    for (double gb : gbs) {
        uint64_t words = (uint64_t)(gb * (1ull << 30)) / 4;
        uint32_t* a; cudaMalloc(&a, words * 4); cudaMemset(a, 1, words * 4);
        uint32_t* out; cudaMalloc(&out, 4);
        const uint64_t pitch = 7456;
        const int iters = 64;
        auto run = [&](auto kern, const char* name) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                kern<<<148, 1024>>>(a, words, pitch, iters, out);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 2) printf("%5.2f GB array %-28s %8.3f ms  useful %7.1f GB/s\n", gb, name, ms, name[2] == '1' ? 0.0 : 0.0 + 148.0 * 32 * iters * 128.0 * (name[0] - '0') / ms / 1e6);
            }
        };
        run(k<1, 0>, "1 ldcg"); run(k<4, 0>, "4 ldcg"); run(k<8, 0>, "8 ldcg");
        run(k<4, 1>, "4 ldg"); run(k<4, 2>, "4 nc.no_allocate"); run(k<8, 2>, "8 nc.no_allocate");
        cudaFree(a); cudaFree(out);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
