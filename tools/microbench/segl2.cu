// Microbenchmark: does streaming whole rows into L2 first make the
// target-tiled segment reads (148 CTAs x ~190 B of every spike's row) run at
// L2 speed?  Same Brunel-1e9-shaped ELL as rowred.cu.
//   phase A (optional): bring the frame's 421 rows into L2
//       1 = cp.async.bulk.prefetch.L2 of each full row (one thread per row)
//       2 = plain coalesced 16-byte loads of each full row (one CTA per row)
//   phase B: CTA c reads its 1/148 window of every row (16-byte chunks,
//       warp per spike, U spikes in flight per warp) and counts targets in smem.
// Every phase is its own launch, timed with events; frames cycle through 200
// distinct spike sets so nothing is L2-resident from a previous frame.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__host__ __device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352d;
    x ^= x >> 15;
    x *= 0x846ca68b;
    x ^= x >> 16;
    return x;
}
constexpr uint32_t NROWS = 141421, PITCH = 7456, NTGT = 70710, SENT = 0xffffffffu, C = 148;

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

__global__ void pf_bulk(const uint32_t* cells, const uint32_t* deg, const uint32_t* spk, uint32_t S) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= S) return;
    const uint32_t s = spk[g];
    const uint32_t bytes = (deg[s] * 4 + 15) & ~15u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cells + uint64_t(s) * PITCH), "r"(bytes) : "memory");
}
__global__ void pf_load(const uint32_t* cells, const uint32_t* deg, const uint32_t* spk, uint32_t S, uint32_t* sink) {
    uint32_t acc = 0;
    for (uint32_t g = blockIdx.x; g < S; g += gridDim.x) {
        const uint32_t s = spk[g];
        const uint4* row = reinterpret_cast<const uint4*>(cells + uint64_t(s) * PITCH);
        const uint32_t n = (deg[s] + 3) / 4;
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
            uint4 v;
            asm volatile("ld.global.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(row + q));
            acc += v.x;
        }
    }
    if (acc == 0x1234567) sink[0] = acc;
}

// CTA c: window c of every row (equal split of the row positions), warp per
// spike, U spikes in flight per warp, counting in smem
template <int U, bool ATOM = true>
__global__ void __launch_bounds__(512, 1) seg(const uint32_t* cells, const uint32_t* deg, const uint32_t* spk,
                                              uint32_t S, uint32_t* sink) {
    __shared__ uint32_t cnt[NTGT / C * 3 + 1024];
    for (uint32_t j = threadIdx.x; j < NTGT / C * 3 + 1024; j += blockDim.x) cnt[j] = 0;
    __syncthreads();
    const uint32_t c = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NWP = blockDim.x / 32;
    for (uint32_t g0 = warp; g0 < S; g0 += NWP * U) {
        uint4 v[U];
        uint32_t lo[U], hi[U], w0[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t g = g0 + u * NWP;
            lo[u] = hi[u] = w0[u] = 0;
            v[u] = make_uint4(0, 0, 0, 0);
            if (g < S) {
                const uint32_t s = spk[g];
                const uint32_t d = deg[s];
                const uint32_t a = d * c / C, b = d * (c + 1) / C;
                w0[u] = ((a >> 2) + lane) << 2;
                lo[u] = a;
                hi[u] = b;
                if (w0[u] < b) v[u] = ldg4(reinterpret_cast<const uint4*>(cells + uint64_t(s) * PITCH + w0[u]));
            }
        }
        if (!ATOM) {
            uint32_t x = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) x += v[u].x + v[u].y + v[u].z + v[u].w;
            if (x == 0x1234567) sink[1] = x;
            continue;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t base = (u % 3) * (NTGT / C);
            if (w0[u] >= lo[u] && w0[u] < hi[u]) atomicAdd(&cnt[base + v[u].x % (NTGT / C)], 1u);
            if (w0[u] + 1 >= lo[u] && w0[u] + 1 < hi[u]) atomicAdd(&cnt[base + v[u].y % (NTGT / C)], 1u);
            if (w0[u] + 2 >= lo[u] && w0[u] + 2 < hi[u]) atomicAdd(&cnt[base + v[u].z % (NTGT / C)], 1u);
            if (w0[u] + 3 >= lo[u] && w0[u] + 3 < hi[u]) atomicAdd(&cnt[base + v[u].w % (NTGT / C)], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt[5] == 0x1234567) sink[0] = 1;
}

int main() {
    uint32_t *cells, *deg, *spk, *sink;
    cudaMalloc(&cells, uint64_t(NROWS) * PITCH * 4);
    cudaMalloc(&deg, NROWS * 4);
    cudaMalloc(&sink, 4);
    gen<<<NROWS, 256>>>(cells, deg);
    cudaDeviceSynchronize();
    const uint32_t F = 200, S = 421;
    std::vector<uint32_t> h(F * S);
    for (uint32_t f = 0; f < F; ++f) {
        std::vector<uint32_t> fr(S);
        for (uint32_t i = 0; i < S; ++i) fr[i] = hash(f * 1000003u + i) % NROWS;
        std::sort(fr.begin(), fr.end());
        for (uint32_t i = 0; i < S; ++i) h[f * S + i] = fr[i];
    }
    cudaMalloc(&spk, F * S * 4);
    cudaMemcpy(spk, h.data(), F * S * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e[4];
    for (auto& x : e) cudaEventCreate(&x);
    const double bytes = double(S) * 7071 * 4;
    for (int mode = 0; mode < 3; ++mode)
        for (int U : {4, 8}) {
            float ta = 0, tb = 0;
            for (int rep = 0; rep < 2; ++rep) {
                ta = tb = 0;
                for (uint32_t f = 0; f < F; ++f) {
                    const uint32_t* sp = spk + f * S;
                    cudaEventRecord(e[0]);
                    if (mode == 1) pf_bulk<<<(S + 127) / 128, 128>>>(cells, deg, sp, S);
                    if (mode == 2) pf_load<<<296, 512>>>(cells, deg, sp, S, sink);
                    cudaEventRecord(e[1]);
                    if (U == 4)
                        seg<4><<<C, 512>>>(cells, deg, sp, S, sink);
                    else
                        seg<8><<<C, 512>>>(cells, deg, sp, S, sink);
                    cudaEventRecord(e[2]);
                    cudaEventSynchronize(e[2]);
                    float a, b;
                    cudaEventElapsedTime(&a, e[0], e[1]);
                    cudaEventElapsedTime(&b, e[1], e[2]);
                    ta += a;
                    tb += b;
                }
            }
            printf("prefetch mode %d U=%d: phase A %.2f us (%.2f TB/s)  phase B %.2f us (%.2f TB/s of rows)\n", mode, U,
                   ta * 1e3 / F, mode ? bytes / (ta * 1e-3 / F) / 1e12 : 0.0, tb * 1e3 / F, bytes / (tb * 1e-3 / F) / 1e12);
        }
    // hot: the same frame twice in a row (second run entirely L2-resident), with / without atomics
    for (int atom = 0; atom < 2; ++atom) {
        float tb = 0;
        for (uint32_t f = 0; f < F; ++f) {
            const uint32_t* sp = spk + f * S;
            if (atom) seg<8, true><<<C, 512>>>(cells, deg, sp, S, sink); else seg<8, false><<<C, 512>>>(cells, deg, sp, S, sink);
            cudaEventRecord(e[1]);
            if (atom) seg<8, true><<<C, 512>>>(cells, deg, sp, S, sink); else seg<8, false><<<C, 512>>>(cells, deg, sp, S, sink);
            cudaEventRecord(e[2]);
            cudaEventSynchronize(e[2]);
            float b;
            cudaEventElapsedTime(&b, e[1], e[2]);
            tb += b;
        }
        printf("hot L2 rerun atom=%d: phase B %.2f us\n", atom, tb * 1e3 / F);
    }
    // launch overhead reference: empty kernel
    {
        cudaEventRecord(e[1]);
        for (uint32_t f = 0; f < F; ++f) pf_bulk<<<1, 32>>>(cells, deg, spk, 0);
        cudaEventRecord(e[2]);
        cudaEventSynchronize(e[2]);
        float b;
        cudaEventElapsedTime(&b, e[1], e[2]);
        printf("empty launch: %.2f us\n", b * 1e3 / F);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
