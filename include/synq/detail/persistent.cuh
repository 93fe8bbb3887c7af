#pragma once
// Persistent, target-tiled pipeline for population-delivery models
// (vogels / brunel; trait synq::population_delivery<M>).
//
// Reference semantics: engine.hpp:188-218 (step), 308-341 (update),
// 369-409 (receive), lif.hpp:23-49 (LIF update / delta-synapse receive).
//
// Design (one cooperative launch runs a whole batch of steps):
// * CTA c owns a contiguous id tile [lo_c, lo_{c+1}) balanced by
//   (update cost + in-degree).  It updates exactly those neurons and receives
//   exactly the deliveries that target them, so the Receive(t) -> Update(t+1)
//   dependency never leaves the SM and needs no grid barrier.
// * Frame t is published per CTA: the CTA's spikes, compacted in ascending id
//   order, go to its own slice of queue slot t % Q, and one release-store of
//   {t+1, count} to finfo[slot][c] makes them visible.  Concatenating the
//   slices in CTA order gives the sorted frame.  Receive(t) consumes frame
//   t-delay+1, i.e. a frame every CTA finished delay-1 steps earlier: the only
//   cross-CTA wait is an acquire-poll that is normally already satisfied.
//   With Q = 2*delay slots no slot is rewritten while a slower CTA may still
//   read it (a CTA can be at most delay-1 steps ahead of the slowest).
// * Delivery is integer counting: per (target, source class) arrivals are
//   counted with native shared-memory atomics (ATOMS.POPC.INC); the row
//   segment of spike s inside tile c is [split[s][c], split[s][c+1]) of the
//   sorted ELL row.  The update re-adds fl(c*w_k) count_k times in ascending
//   class (= ascending source id) order, which is exactly the float sum the
//   reference's deterministic receive produces.  Bit-exact and order-free.
#include <cuda_runtime.h>

#include <cstdint>

#include "synq/detail/device_refs.cuh"
#include "synq/detail/kernels.cuh"
#include "synq/models/benchmarks.hpp"

namespace synq::dev {

constexpr int kPersistThreads = 1024;
constexpr int kMaxTiles = 1024;
constexpr int kMaxClasses = 4;
constexpr int kUnroll = 8;

template <class M>
struct persist_state {
    using NF = typename M::neuron_fields;
    field_ptrs<NF> nf;
    xorshift* rng;
    const uint32_t* cells;
    const uint32_t* split;    // [n][C+1]
    const uint32_t* tile_lo;  // [C+1]
    const uint32_t* win_lo;   // [C] first receiving id of the tile (count window)
    uint32_t pitch, n, C;
    uint32_t* queue;             // Q slots x n
    unsigned long long* finfo;   // Q x C: (t+1) << 32 | count
    uint32_t Q;
    int K;
    uint32_t bound[kMaxClasses];
    float delta[kMaxClasses];
    float dt;
    uint32_t delay;
    unsigned long long* counters;
    uint32_t* step_spikes;
    uint32_t* step_meas;
    uint32_t meas_lo, meas_hi;
    // ordered frame log (recording / taps): CTA 0 copies every frame it
    // receives with due >= log_from, in CTA (= ascending id) order
    uint32_t* log;
    unsigned long long* log_end;  // out: entries written
    unsigned long long log_cap;
    int64_t log_from;
    uint32_t* flags;
    uint32_t win_cap;      // count-window capacity per class (smem)
    uint32_t spike_chunk;  // spikes staged per receive round (smem)
};

SYNQ_DEV void st_release_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SYNQ_DEV unsigned long long ld_acquire_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <class M>
SYNQ_DEV int source_class(const persist_state<M>& ps, uint32_t src) {
    int k = 0;
#pragma unroll
    for (int q = 0; q < kMaxClasses - 1; ++q)
        if (q < ps.K - 1 && src >= ps.bound[q]) k = q + 1;
    return k;
}

template <class M>
__global__ void __launch_bounds__(kPersistThreads, 1)
    k_persistent(M model, persist_state<M> ps, int64_t t0, int32_t nsteps) {
    using NF = typename M::neuron_fields;
    constexpr size_t ACC = population_delivery<M>::acc_field;
    constexpr int NT = kPersistThreads, NW = NT / 32;

    extern __shared__ uint32_t smem[];
    uint32_t* cnt = smem;                                   // K x win_cap
    uint32_t* s_src = cnt + ps.K * ps.win_cap;              // spike_chunk
    uint32_t* s_beg = s_src + ps.spike_chunk;
    uint32_t* s_len = s_beg + ps.spike_chunk;
    __shared__ uint32_t s_lo[kMaxTiles + 1];
    __shared__ uint32_t s_seg[kMaxTiles + 1];
    __shared__ uint32_t s_warp[NW];
    __shared__ uint32_t s_pass, s_meas;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, C = ps.C;
    for (uint32_t j = tid; j <= C; j += NT) s_lo[j] = ps.tile_lo[j];
    for (uint32_t j = tid; j < ps.K * ps.win_cap; j += NT) cnt[j] = 0;
    if (tid == 0) s_meas = 0;
    __syncthreads();
    const uint32_t lo = s_lo[c], hi = s_lo[c + 1];
    const uint32_t wlo = ps.win_lo[c];
    unsigned long long my_deliv = 0, my_spikes = 0;
    unsigned long long lc = 0;  // CTA 0: log cursor

    for (int32_t s = 0; s < nsteps; ++s) {
        const int64_t t = t0 + s;
        const uint32_t slot = static_cast<uint32_t>(t % ps.Q);
        uint32_t* qseg = ps.queue + static_cast<uint64_t>(slot) * ps.n + lo;

        // ------------------------------------------------ Update(t)
        uint32_t out = 0;
        for (uint32_t base = lo; base < hi; base += NT) {
            const uint32_t i = base + tid;
            bool spk = false;
            if (i < hi) {
                values_t<NF> v;
                load_all(ps.nf, i, v);
                values_t<NF> before = v;
                if (i >= wlo && i - wlo < ps.win_cap) {
                    float acc = detail::pack_get<ACC>::get(v);
                    for (int k = 0; k < ps.K; ++k) {
                        uint32_t* slotp = cnt + k * ps.win_cap + (i - wlo);
                        const uint32_t r = *slotp;
                        if (r) {
                            *slotp = 0;
                            const float d = ps.delta[k];
                            for (uint32_t q = 0; q < r; ++q) acc = acc + d;
                        }
                    }
                    detail::pack_get<ACC>::get(v) = acc;
                }
                xorshift rr;
                bool live = false;
                local_neuron<NF> ref{i, &v, &rr, &live, ps.rng};
                spk = model.update(ref, ps.dt);
                store_changed(ps.nf, i, v, before);
                if constexpr (model_uses_rng<M>())
                    if (live) ps.rng[i] = rr;
            }
            const unsigned ball = __ballot_sync(0xffffffffu, spk);
            const unsigned mball = __ballot_sync(0xffffffffu, spk && i >= ps.meas_lo && i < ps.meas_hi);
            if (lane == 0) {
                s_warp[warp] = __popc(ball);
                if (mball) atomicAdd(&s_meas, __popc(mball));
            }
            __syncthreads();
            if (warp == 0) {
                const uint32_t x = s_warp[lane];
                uint32_t incl = x;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= static_cast<uint32_t>(o)) incl += y;
                }
                s_warp[lane] = incl - x;
                if (lane == 31) s_pass = incl;
            }
            __syncthreads();
            if (spk) qseg[out + s_warp[warp] + __popc(ball & ((1u << lane) - 1u))] = i;
            out += s_pass;
            __syncthreads();
        }
        // publish this CTA's slice of frame t
        if (tid == 0) {
            __threadfence();
            st_release_gpu(&ps.finfo[static_cast<uint64_t>(slot) * C + c],
                           (static_cast<unsigned long long>(t + 1) << 32) | out);
            if (out) atomicAdd(&ps.step_spikes[s], out);
            if (s_meas) atomicAdd(&ps.step_meas[s], s_meas);
            s_meas = 0;
            my_spikes += out;
        }
        __syncthreads();

        // ------------------------------------------------ Receive(t - delay + 1)
        const int64_t due = t - static_cast<int64_t>(ps.delay) + 1;
        if (due < 0) continue;
        const uint32_t dslot = static_cast<uint32_t>(due % ps.Q);
        if (warp == 0) {
            const unsigned long long want = static_cast<unsigned long long>(due + 1);
            uint32_t run = 0;
            for (uint32_t j0 = 0; j0 < C; j0 += 32) {
                const uint32_t j = j0 + lane;
                uint32_t cj = 0;
                if (j < C) {
                    const unsigned long long* p = ps.finfo + static_cast<uint64_t>(dslot) * C + j;
                    unsigned long long v = ld_acquire_gpu(p);
                    while ((v >> 32) != want) {
                        __nanosleep(32);
                        v = ld_acquire_gpu(p);
                    }
                    cj = static_cast<uint32_t>(v);
                }
                uint32_t incl = cj;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= static_cast<uint32_t>(o)) incl += y;
                }
                if (j < C) s_seg[j] = run + incl - cj;
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) s_seg[C] = run;
        }
        __syncthreads();
        const uint32_t S = s_seg[C];
        const uint32_t* dq = ps.queue + static_cast<uint64_t>(dslot) * ps.n;
        const bool logging = ps.log && c == 0 && due >= ps.log_from;
        for (uint32_t c0 = 0; c0 < S; c0 += ps.spike_chunk) {
            const uint32_t m = min(ps.spike_chunk, S - c0);
            // stage ids and this tile's row segments
            for (uint32_t g = tid; g < m; g += NT) {
                const uint32_t gg = c0 + g;
                uint32_t a = 0, b = C;  // last j with s_seg[j] <= gg
                while (b - a > 1) {
                    const uint32_t mid = (a + b) >> 1;
                    if (s_seg[mid] <= gg) a = mid; else b = mid;
                }
                const uint32_t src = __ldcg(dq + s_lo[a] + (gg - s_seg[a]));
                const uint32_t* sp = ps.split + static_cast<uint64_t>(src) * (C + 1) + c;
                const uint32_t sb = __ldg(sp), se = __ldg(sp + 1);
                if (logging && lc + gg < ps.log_cap) ps.log[lc + gg] = src;
                s_src[g] = src;
                s_beg[g] = sb;
                s_len[g] = se - sb;
                my_deliv += se - sb;
            }
            __syncthreads();
            // count arrivals: warp per spike, kUnroll row loads in flight per lane
            uint32_t g = warp, ck = 0;
            while (g < m) {
                uint32_t tg[kUnroll];
                int kc[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    tg[u] = 0xffffffffu;
                    kc[u] = 0;
                    if (g < m) {
                        const uint32_t len = s_len[g];
                        const uint32_t p = ck * 32 + lane;
                        if (p < len) {
                            const uint32_t src = s_src[g];
                            tg[u] = __ldg(ps.cells + static_cast<uint64_t>(src) * ps.pitch + s_beg[g] + p);
                            kc[u] = source_class(ps, src);
                        }
                        ++ck;
                        if (ck * 32 >= len) {
                            ck = 0;
                            g += NW;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    if (tg[u] != 0xffffffffu) atomicAdd(&cnt[kc[u] * ps.win_cap + (tg[u] - wlo)], 1u);
            }
            __syncthreads();
        }
        if (logging) lc += S;
    }
    if (ps.log && c == 0 && tid == 0) {
        *ps.log_end = lc;
        if (lc > ps.log_cap) ps.flags[0] = 1;
    }

    // fold pending arrivals into ACC so host reads and the next launch see them
    for (uint32_t i = lo + tid; i < hi; i += NT) {
        if (i < wlo || i - wlo >= ps.win_cap) continue;
        float acc = ps.nf.template get<ACC>()[i];
        bool any = false;
        for (int k = 0; k < ps.K; ++k) {
            const uint32_t r = cnt[k * ps.win_cap + (i - wlo)];
            any |= r != 0;
            const float d = ps.delta[k];
            for (uint32_t q = 0; q < r; ++q) acc = acc + d;
        }
        if (any) ps.nf.template get<ACC>()[i] = acc;
    }
    for (int o = 16; o; o >>= 1) my_deliv += __shfl_xor_sync(0xffffffffu, my_deliv, o);
    if (lane == 0 && my_deliv) atomicAdd(&ps.counters[C_DELIVERIES], my_deliv);
    if (tid == 0 && my_spikes) atomicAdd(&ps.counters[C_SPIKES], my_spikes);
}

// Copy frames [from, to] (all complete in the ring) into the ordered log;
// used once at the end of run() for the frames not yet consumed by Receive.
template <class M>
__global__ void k_log_drain(persist_state<M> ps, int64_t from, int64_t to) {
    __shared__ uint32_t s_seg[kMaxTiles + 1];
    __shared__ uint32_t s_lo[kMaxTiles + 1];
    const uint32_t C = ps.C;
    for (uint32_t j = threadIdx.x; j <= C; j += blockDim.x) s_lo[j] = ps.tile_lo[j];
    unsigned long long lc = 0;
    for (int64_t f = from; f <= to; ++f) {
        const uint32_t slot = static_cast<uint32_t>(f % ps.Q);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (uint32_t j = 0; j < C; ++j) {
                s_seg[j] = run;
                run += static_cast<uint32_t>(ps.finfo[static_cast<uint64_t>(slot) * C + j]);
            }
            s_seg[C] = run;
        }
        __syncthreads();
        const uint32_t S = s_seg[C];
        for (uint32_t j = 0; j < C; ++j) {
            const uint32_t cnt = s_seg[j + 1] - s_seg[j];
            for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x)
                if (lc + s_seg[j] + k < ps.log_cap)
                    ps.log[lc + s_seg[j] + k] = ps.queue[static_cast<uint64_t>(slot) * ps.n + s_lo[j] + k];
        }
        lc += S;
    }
    if (threadIdx.x == 0) {
        *ps.log_end = lc;
        if (lc > ps.log_cap) ps.flags[0] = 1;
    }
}

}  // namespace synq::dev
