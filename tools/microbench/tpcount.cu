// Microbenchmark: the bitmap delivery's counting loop in isolation (data in
// shared memory).  Per iteration a warp loads one 16-byte window column of
// 32 spikes (LDS.128), transposes the 4 words (32x32 bit transposes, 5 SHFL
// each) and accumulates popcounts.  MODE 0: as in the kernel; MODE 1: same
// ALU work but the 5 SHFL replaced by register ops (isolates SHFL cost);
// MODE 2: bit-sliced accumulation of 8 blocks into 4 planes, then 4
// transposes per word (fewer SHFL).  Reports cycles per 32x128-bit block.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct tpk {
    uint32_t sel16, sel8, rot[3], keep[3];
};
__device__ tpk mk(uint32_t lane) {
    tpk k;
    k.sel16 = (lane & 16) ? 0x3276u : 0x5410u;
    k.sel8 = (lane & 8) ? 0x3715u : 0x6240u;
    for (int s = 0; s < 3; ++s) {
        const uint32_t j = 4u >> s;
        const uint32_t m = s == 0 ? 0x0f0f0f0fu : (s == 1 ? 0x33333333u : 0x55555555u);
        const bool hi = (lane & j) != 0;
        k.rot[s] = hi ? 32 - j : j;
        k.keep[s] = hi ? ~m : m;
    }
    return k;
}
__device__ __forceinline__ uint32_t lop(uint32_t x, uint32_t t, uint32_t keep) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(x), "r"(t), "r"(keep));
    return d;
}
template <bool SH>
__device__ __forceinline__ uint32_t tp(uint32_t x, const tpk& k) {
    uint32_t y = SH ? __shfl_xor_sync(0xffffffffu, x, 16) : (x * 2654435761u);
    x = __byte_perm(x, y, k.sel16);
    y = SH ? __shfl_xor_sync(0xffffffffu, x, 8) : (x * 2654435761u);
    x = __byte_perm(x, y, k.sel8);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        y = SH ? __shfl_xor_sync(0xffffffffu, x, 4 >> s) : (x * 2654435761u);
        x = lop(x, __funnelshift_l(y, y, k.rot[s]), k.keep[s]);
    }
    return x;
}

template <int MODE>
__global__ void k(int iters, uint32_t* out, unsigned long long* cyc) {
    __shared__ uint4 sw[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
        sw[i] = make_uint4(i * 7919u, i * 104729u, i * 1299709u, i * 15485863u);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const tpk K = mk(lane);
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    const long long t0 = clock64();
    if (MODE < 2) {
        for (int it = 0; it < iters; it += 2) {
            uint4 x[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) x[v] = sw[((it + v) * 32 + warp * 97 + lane) & 2047];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                c0 += __popc(tp<MODE == 0>(x[v].x, K));
                c1 += __popc(tp<MODE == 0>(x[v].y, K));
                c2 += __popc(tp<MODE == 0>(x[v].z, K));
                c3 += __popc(tp<MODE == 0>(x[v].w, K));
            }
        }
    } else {
        for (int it = 0; it < iters; it += 8) {
            uint32_t p[4][4] = {};
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                const uint4 x = sw[((it + v) * 32 + warp * 97 + lane) & 2047];
                const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    uint32_t c = w[e];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t t = p[e][q] & c;
                        p[e][q] ^= c;
                        c = t;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                c0 += __popc(tp<true>(p[0][q], K)) << q;
                c1 += __popc(tp<true>(p[1][q], K)) << q;
                c2 += __popc(tp<true>(p[2][q], K)) << q;
                c3 += __popc(tp<true>(p[3][q], K)) << q;
            }
        }
    }
    const long long t1 = clock64();
    if ((c0 ^ c1 ^ c2 ^ c3) == 0x1234567u) out[0] = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    uint32_t* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8 * 148);
    const int iters = 4096;
    const char* names[] = {"transpose (5 SHFL)", "transpose, SHFL->ALU", "bit-sliced 8 blocks + 4 transposes"};
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {8, 16, 32}) {
            if (mode == 0) k<0><<<148, warps * 32>>>(iters, out, cyc);
            if (mode == 1) k<1><<<148, warps * 32>>>(iters, out, cyc);
            if (mode == 2) k<2><<<148, warps * 32>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            unsigned long long c[148];
            cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
            printf("%-36s warps %2d: %6.1f cycles per 32x128-bit block per SM (%.1f per warp-block)\n", names[mode],
                   warps, double(c[0]) / (iters * warps), double(c[0]) / iters);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
