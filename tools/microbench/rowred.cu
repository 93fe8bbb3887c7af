// Microbenchmark: whole-row delivery with integer global reductions.
// A Brunel-1e9-shaped padded ELL (141,421 rows, pitch 7456, ~7071 sorted
// targets per row in [0, 70710)) is streamed row by row: every spike's FULL
// row is read by one CTA (coalesced 16-byte loads) and each target gets a
// red.global.add.u32 into counts[class][target] (class by source id).
// Variants: 0 = read only (checksum), 1 = read + RED, 2 = read + RED with
// lanes taking 4 consecutive targets (row-contiguous per warp).
// Reports us per frame of 421 spikes (and TB/s of row bytes).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352d;
    x ^= x >> 15;
    x *= 0x846ca68b;
    x ^= x >> 16;
    return x;
}

constexpr uint32_t NROWS = 141421, PITCH = 7456, NTGT = 70710, SENT = 0xffffffffu;

// one CTA per row: Bernoulli(0.1) targets, compacted in order
__global__ void gen(uint32_t* cells, uint32_t* deg) {
    __shared__ uint32_t s_w[32], s_base;
    const uint32_t row = blockIdx.x;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (uint32_t t0 = 0; t0 < NTGT; t0 += blockDim.x) {
        const uint32_t t = t0 + threadIdx.x;
        const bool keep = t < NTGT && (hash(row * 2654435761u ^ (t * 40503u + 7u)) % 1000u) < 100u;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(b);
        __syncthreads();
        uint32_t pre = 0, tot = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
            if (w < (threadIdx.x >> 5)) pre += s_w[w];
            tot += s_w[w];
        }
        const uint32_t base = s_base;
        const uint32_t pos = base + pre + __popc(b & ((1u << (threadIdx.x & 31)) - 1));
        if (keep && pos < PITCH) cells[uint64_t(row) * PITCH + pos] = t;
        __syncthreads();
        if (threadIdx.x == 0) s_base = base + tot;
        __syncthreads();
    }
    for (uint32_t k = s_base + threadIdx.x; k < PITCH; k += blockDim.x) cells[uint64_t(row) * PITCH + k] = SENT;
    if (threadIdx.x == 0) deg[row] = min(s_base, PITCH);
}

__device__ __forceinline__ uint4 ldg4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void red(uint32_t* p) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(512) deliver(const uint32_t* cells, const uint32_t* deg, const uint32_t* spikes,
                                               uint32_t nspk, uint32_t* counts, uint32_t* sink) {
    uint32_t acc = 0;
    for (uint32_t g = blockIdx.x; g < nspk; g += gridDim.x) {
        const uint32_t src = spikes[g];
        const uint32_t d = deg[src];
        const uint32_t cls = src < 56568 ? 0 : (src < 70710 ? 1 : 2);
        uint32_t* cb = counts + cls * NTGT;
        const uint4* row = reinterpret_cast<const uint4*>(cells + uint64_t(src) * PITCH);
        const uint32_t nch = (d + 3) / 4;
        for (uint32_t q = threadIdx.x; q < nch; q += blockDim.x * 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t qq = q + u * blockDim.x;
                v[u] = qq < nch ? ldg4(row + qq) : make_uint4(SENT, SENT, SENT, SENT);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (MODE == 0) {
                    acc += v[u].x + v[u].y + v[u].z + v[u].w;
                } else {
                    if (v[u].x != SENT) red(cb + v[u].x);
                    if (v[u].y != SENT) red(cb + v[u].y);
                    if (v[u].z != SENT) red(cb + v[u].z);
                    if (v[u].w != SENT) red(cb + v[u].w);
                }
            }
        }
    }
    if (acc == 0x1234567) sink[0] = acc;
}

int main() {
    uint32_t *cells, *deg, *spk, *counts, *sink;
    cudaMalloc(&cells, uint64_t(NROWS) * PITCH * 4);
    cudaMalloc(&deg, NROWS * 4);
    cudaMalloc(&counts, 3 * NTGT * 4);
    cudaMalloc(&sink, 4);
    gen<<<NROWS, 256>>>(cells, deg);
    cudaDeviceSynchronize();
    std::vector<uint32_t> d(NROWS);
    cudaMemcpy(d.data(), deg, NROWS * 4, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : d) avg += x;
    printf("avg degree %.1f  (err %s)\n", avg / NROWS, cudaGetErrorString(cudaGetLastError()));
    const uint32_t F = 200, S = 421;
    std::vector<uint32_t> h(F * S);
    for (uint32_t i = 0; i < F * S; ++i) h[i] = (i * 2654435761u + 12345u) % NROWS;
    cudaMalloc(&spk, F * S * 4);
    cudaMemcpy(spk, h.data(), F * S * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = double(S) * avg / NROWS * 4;
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {148, 296, 592}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                for (uint32_t f = 0; f < F; ++f) {
                    if (mode == 0)
                        deliver<0><<<grid, 512>>>(cells, deg, spk + f * S, S, counts, sink);
                    else
                        deliver<1><<<grid, 512>>>(cells, deg, spk + f * S, S, counts, sink);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("mode %d grid %d: %.2f us/frame  %.2f TB/s of rows  %.3f T red/s\n", mode, grid,
                                ms * 1e3 / F, bytes * F / (ms * 1e-3) / 1e12, bytes / 4 * F / (ms * 1e-3) / 1e12);
            }
        }
    // many frames per launch: whole batch in one launch (no launch gaps)
    for (int mode = 0; mode < 2; ++mode) {
        cudaEventRecord(e0);
        if (mode == 0)
            deliver<0><<<592, 512>>>(cells, deg, spk, F * S, counts, sink);
        else
            deliver<1><<<592, 512>>>(cells, deg, spk, F * S, counts, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("batched mode %d: %.2f us/frame  %.2f TB/s  %.3f T red/s\n", mode, ms * 1e3 / F,
               bytes * F / (ms * 1e-3) / 1e12, bytes / 4 * F / (ms * 1e-3) / 1e12);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
