#pragma once
// Single-CTA persistent engine for small population-delivery networks
// (Vogels-Abbott 4000, BASELINE config 1; SURVEY.md 7.1 hard part 1).
//
// Reference semantics are those of k_persistent / k_pipeline
// (engine.hpp:188-218 step, 308-341 update, 369-409 receive): arrivals are
// counted per (target, source class) and re-added in class order by the
// update, so spike trains and state are the reference's deterministic ones.
// What changes is the machine: a network of <= 4096 neurons lives on ONE SM.
// The neuron state is in registers (<= 4 neurons per thread), the frame ring
// and the delivered counts in shared memory, and a step is four CTA
// barriers with no global-memory synchronisation at all (the multi-CTA
// engines pay a gpu-scope release / acquire round trip per frame).  Rows are
// copied into shared memory one step before they are delivered
// (cp.async), so no global latency is on the step's chain either.
//
// Per step t:
//   1. fold the counts of frame t - delay (delivered at step t - 1), update,
//      ballot;                                                    [barrier]
//   2. warp 0: prefix of the spike counts and of the frame's padded row
//      sizes;                                                     [barrier]
//   3. write frame t (ascending ids) to the global queue slot (the format
//      k_log_drain and the host read), to the shared-memory ring and its
//      row offsets; frame word; wait for the rows copied last step; [barrier]
//   4. count frame t - delay + 1 into the counts (rows from shared memory,
//      or straight from global memory for a frame that did not fit), log it
//      (CTA-order = id order), issue the row copies of frame t - delay + 2.
//                                                                  [barrier]
// Frames published by an earlier launch are delivered from global memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "synq/detail/persistent.cuh"
#include "synq/detail/pipeline.cuh"

namespace synq::dev {

constexpr int kSoloThreads = 1024;
constexpr uint32_t kSoloMaxNeurons = 4 * kSoloThreads;
constexpr uint32_t kSoloRing = 4096;    // frame ids held in the ring (+ one row offset each)
constexpr uint32_t kSoloRows = 8192;    // row entries per copy buffer (two buffers)
constexpr uint32_t kSoloMaxDelay = 64;  // frame metadata slots (frame f in slot f % delay)

// shared-memory bytes of the solo kernel's dynamic part
inline size_t solo_smem_bytes(uint32_t K, uint32_t na, uint32_t n) {
    return (size_t(K) * na + 2 * size_t(kSoloRing) + 2 * size_t(kSoloRows) + n) * 4 + 16;
}

template <class M, int NPT>
__global__ void __launch_bounds__(kSoloThreads, 1)
    k_solo(M model, persist_state<M> ps, int64_t t0, int32_t nsteps) {
    using NF = typename M::neuron_fields;
    constexpr size_t ACC = population_delivery<M>::acc_field;
    constexpr int NT = kSoloThreads, NW = NT / 32;
    constexpr uint32_t NONE = 0xffffffffu;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t K = static_cast<uint32_t>(ps.K), delay = ps.delay, n = ps.n;
    const uint32_t pa = ps.cta_piece[0], pb = ps.cta_piece[1];
    const uint32_t alo = ps.piece_lo[pa], na = ps.piece_lo[pa + 1] - alo;  // receiving piece
    const uint32_t blo = ps.piece_lo[pb], nb = ps.piece_lo[pb + 1] - blo;  // update-only piece
    const bool a_first = alo <= blo;                                      // piece (= id) order of the frame
    uint32_t* cnt = sm;                                  // K x na arrival counts
    uint32_t* ring = cnt + K * na;                       // kSoloRing frame ids
    uint32_t* rofs = ring + kSoloRing;                   // kSoloRing: padded row offset of each id
    // 2 x kSoloRows row entries, 16-byte aligned for cp.async (the dynamic
    // segment follows the static one and may start on an 8-byte boundary)
    uint32_t* rows = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(rofs + kSoloRing) + 15) & ~uintptr_t(15));
    uint32_t* sdeg = rows + 2 * kSoloRows;               // n out-degrees
    __shared__ uint32_t fm_cnt[kSoloMaxDelay], fm_ca[kSoloMaxDelay], fm_off[kSoloMaxDelay], fm_rows[kSoloMaxDelay];
    __shared__ uint32_t fm_pf[kSoloMaxDelay];  // rows of the frame are in shared memory (prefetched)
    __shared__ uint32_t s_wa[NPT * NW], s_wb[NPT * NW], s_ra[NPT * NW], s_rb[NPT * NW], s_mw[NW];
    __shared__ uint32_t s_out[6];
    __shared__ uint32_t s_head, s_tail;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t j = tid; j < K * na; j += NT) cnt[j] = 0;
    for (uint32_t j = tid; j < n; j += NT) sdeg[j] = ps.degree[j];
    // frames of earlier launches (t0 - delay + 1 .. t0 - 1) are read from global memory
    for (uint32_t j = tid; j < delay; j += NT) {
        fm_off[j] = NONE;
        fm_rows[j] = NONE;
        fm_cnt[j] = 0;
        fm_ca[j] = 0;
        fm_pf[j] = 0;
    }
    if (tid == 0) {
        s_head = 0;
        s_tail = 0;
    }
    __syncthreads();
    for (uint32_t j = tid; j + 1 < delay; j += NT) {
        const int64_t f = t0 - 1 - j;
        if (f < 0) continue;
        const unsigned long long w = ps.finfo[static_cast<uint64_t>(f % ps.Q) * ps.E];
        fm_cnt[f % delay] = word_a(w) + word_b(w);
        fm_ca[f % delay] = word_a(w);
    }
    __syncthreads();

    // register-resident state: local index j = tid + r * NT, A piece first
    auto id_of = [&](uint32_t j) { return j < na ? alo + j : blo + (j - na); };
    values_t<NF> v[NPT];
    xorshift rr[NPT];
    bool live[NPT];
    unsigned amask[NPT];
    bool inmeas[NPT];
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
        live[r] = false;
        const uint32_t j = tid + r * NT;
        if (j < na + nb) load_all(ps.nf, id_of(j), v[r]);
        const int na_here = static_cast<int>(na) - static_cast<int>(warp * 32 + r * NT);
        amask[r] = na_here >= 32 ? 0xffffffffu : (na_here <= 0 ? 0u : (1u << na_here) - 1u);
        inmeas[r] = j < na + nb && id_of(j) >= ps.meas_lo && id_of(j) < ps.meas_hi;
    }
    const unsigned below = (1u << lane) - 1u;
    unsigned long long my_deliv = 0, my_spikes = 0, lc = 0;
    const bool logging = ps.log != nullptr;

    // count frame f (the frame of ring slot f % delay) into the counts
    auto deliver = [&](int64_t f) {
        const uint32_t sl = static_cast<uint32_t>(f % delay);
        const uint32_t S = fm_cnt[sl], off = fm_off[sl];
        const bool staged = fm_pf[sl] != 0;
        const uint32_t* qs = ps.queue + static_cast<uint64_t>(f % ps.Q) * n;
        const uint32_t ca = fm_ca[sl];
        auto spike_id = [&](uint32_t i) -> uint32_t {
            if (off != NONE) return ring[(off + i) % kSoloRing];
            const bool in_first = a_first ? i < ca : i < S - ca;
            if (a_first) return in_first ? qs[alo + i] : qs[blo + (i - ca)];
            return in_first ? qs[blo + i] : qs[alo + (i - (S - ca))];
        };
        const uint32_t* rb = rows + (f & 1) * kSoloRows;
        for (uint32_t i = warp; i < S; i += NW) {
            const uint32_t src = spike_id(i);
            const uint32_t d = sdeg[src];
            const uint32_t cls = static_cast<uint32_t>(source_class(ps, src));
            uint32_t* cb = cnt + cls * na - alo;
            if (staged) {
                const uint32_t* r0 = rb + rofs[(off + i) % kSoloRing];
                for (uint32_t q = lane; q < d; q += 32) atomicAdd(cb + r0[q], 1u);
            } else {
                const uint32_t* r0 = ps.cells + static_cast<uint64_t>(src) * ps.pitch;
                for (uint32_t q = lane; q < d; q += 32) atomicAdd(cb + __ldg(r0 + q), 1u);
            }
            if (lane == 0) my_deliv += d;
            if (logging && f >= ps.log_from && lane == 0 && lc + i < ps.log_cap) ps.log[lc + i] = src;
        }
        if (logging && f >= ps.log_from) {
            if (tid == 0) ps.log_cnt[f - ps.log_from] = S;
            lc += S;
        }
    };
    // copy the rows of frame g into buffer g & 1 (16-byte chunks; every
    // id's segment starts on a 4-entry boundary)
    auto prefetch = [&](int64_t g) {
        const uint32_t sl = static_cast<uint32_t>(g % delay);
        const uint32_t S = fm_cnt[sl], off = fm_off[sl];
        if (off == NONE || fm_rows[sl] == NONE) return;
        if (tid == 0) fm_pf[sl] = 1;  // read by deliver() after the step's barriers
        uint4* rb = reinterpret_cast<uint4*>(rows + (g & 1) * kSoloRows);
        for (uint32_t i = warp; i < S; i += NW) {
            const uint32_t src = ring[(off + i) % kSoloRing];
            const uint32_t c4 = (sdeg[src] + 3) >> 2, o4 = rofs[(off + i) % kSoloRing] >> 2;
            const uint4* gr = reinterpret_cast<const uint4*>(ps.cells + static_cast<uint64_t>(src) * ps.pitch);
            for (uint32_t q = lane; q < c4; q += 32) cp_async16_cg(rb + o4 + q, gr + q);
        }
    };

    uint32_t slot = static_cast<uint32_t>(t0 % ps.Q);
    for (uint32_t s = 0; s < static_cast<uint32_t>(nsteps); ++s, slot = slot + 1 == ps.Q ? 0u : slot + 1) {
        const int64_t t = t0 + s;
        // ---- 1. fold frame t - delay (counted at step t - 1) and update
        bool spk[NPT];
        unsigned bal[NPT];
        uint32_t rlo[NPT];
        uint32_t mcount = 0;
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            const uint32_t j = tid + r * NT;
            spk[r] = false;
            if (j < na + nb) {
                if (j < na) {
                    uint32_t a[kMaxClasses];
#pragma unroll
                    for (int k = 0; k < kMaxClasses; ++k) {
                        a[k] = static_cast<uint32_t>(k) < K ? cnt[k * na + j] : 0u;
                        if (a[k]) cnt[k * na + j] = 0;
                    }
                    detail::pack_get<ACC>::get(v[r]) = fold_frame(ps, detail::pack_get<ACC>::get(v[r]), a);
                }
                local_neuron<NF> ref{id_of(j), &v[r], &rr[r], &live[r], ps.rng};
                spk[r] = model.update(ref, ps.dt);
            }
            bal[r] = __ballot_sync(0xffffffffu, spk[r]);
            mcount += __popc(__ballot_sync(0xffffffffu, spk[r] && inmeas[r]));
            // padded row sizes of the spikes (4-entry boundaries): lane
            // offset inside the warp's part of its piece, warp totals
            const uint32_t pd = spk[r] ? (sdeg[id_of(j)] + 3) & ~3u : 0u;
            const bool in_a = (amask[r] >> lane) & 1u;
            const uint32_t xa = in_a ? pd : 0u, xb = in_a ? 0u : pd;
            const uint32_t ia = warp_incl_scan(xa), ib = warp_incl_scan(xb);
            rlo[r] = in_a ? ia - xa : ib - xb;
            if (lane == 31) {
                s_ra[r * NW + warp] = ia;
                s_rb[r * NW + warp] = ib;
            }
            if (lane == 0) {
                s_wa[r * NW + warp] = __popc(bal[r] & amask[r]);
                s_wb[r * NW + warp] = __popc(bal[r] & ~amask[r]);
            }
        }
        if (lane == 0) s_mw[warp] = mcount;
        __syncthreads();
        // ---- 2. prefixes in local-index order (A piece, then B piece)
        if (warp == 0) {
            uint32_t runa = 0, runb = 0, rra = 0, rrb = 0;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                const uint32_t xa = s_wa[r * NW + lane], xb = s_wb[r * NW + lane];
                const uint32_t ya = s_ra[r * NW + lane], yb = s_rb[r * NW + lane];
                const uint32_t ia = warp_incl_scan(xa), ib = warp_incl_scan(xb);
                const uint32_t ja = warp_incl_scan(ya), jb = warp_incl_scan(yb);
                s_wa[r * NW + lane] = runa + ia - xa;
                s_wb[r * NW + lane] = runb + ib - xb;
                s_ra[r * NW + lane] = rra + ja - ya;
                s_rb[r * NW + lane] = rrb + jb - yb;
                runa += __shfl_sync(0xffffffffu, ia, 31);
                runb += __shfl_sync(0xffffffffu, ib, 31);
                rra += __shfl_sync(0xffffffffu, ja, 31);
                rrb += __shfl_sync(0xffffffffu, jb, 31);
            }
            uint32_t mm = s_mw[lane];
            for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
            if (lane == 0) {
                const uint32_t S = runa + runb, rtot = rra + rrb;
                const uint32_t sl = static_cast<uint32_t>(t % delay);
                // frame t - delay was delivered at step t - 1: its ring space is free
                if (t - static_cast<int64_t>(delay) >= t0 && fm_off[sl] != NONE) s_tail += fm_cnt[sl];
                const bool fits = s_head + S - s_tail <= kSoloRing;
                s_out[0] = runa;
                s_out[1] = runb;
                s_out[2] = mm;
                s_out[3] = fits ? s_head : NONE;
                s_out[4] = rra;
                s_out[5] = rrb;
                fm_cnt[sl] = S;
                fm_ca[sl] = runa;
                fm_off[sl] = fits ? s_head % kSoloRing : NONE;
                fm_rows[sl] = fits && rtot <= kSoloRows ? rtot : NONE;
                fm_pf[sl] = 0;
                if (fits) s_head += S;
            }
        }
        __syncthreads();
        // ---- 3. frame t: global queue slot, ring, row offsets; frame word
        {
            uint32_t* qslot = ps.queue + static_cast<uint64_t>(slot) * n;
            const uint32_t outa = s_out[0], outb = s_out[1], rbase = s_out[3];
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                if (!spk[r]) continue;
                const uint32_t j = tid + r * NT, id = id_of(j);
                const bool in_a = (amask[r] >> lane) & 1u;
                const unsigned m = in_a ? amask[r] : ~amask[r];
                const uint32_t pos = (in_a ? s_wa[r * NW + warp] : s_wb[r * NW + warp]) + __popc(bal[r] & m & below);
                qslot[(in_a ? alo : blo) + pos] = id;
                if (rbase != NONE) {
                    // merged (id-ordered) frame position and padded row offset
                    const uint32_t mp = in_a ? (a_first ? pos : outb + pos) : (a_first ? outa + pos : pos);
                    const uint32_t rbase_piece = in_a ? (a_first ? 0u : s_out[5]) : (a_first ? s_out[4] : 0u);
                    const uint32_t ro = rbase_piece + (in_a ? s_ra[r * NW + warp] : s_rb[r * NW + warp]) + rlo[r];
                    ring[(rbase + mp) % kSoloRing] = id;
                    rofs[(rbase + mp) % kSoloRing] = ro;
                }
            }
            if (tid == 0) {
                ps.finfo[static_cast<uint64_t>(slot) * ps.E] = frame_word(t, outa, outb);
                ps.step_spikes[s] = outa + outb;
                ps.step_meas[s] = s_out[2];
                my_spikes += outa + outb;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // ---- 4. count frame t - delay + 1, copy the rows of the next due frame
        const int64_t f = t - static_cast<int64_t>(delay) + 1;
        if (f >= 0) deliver(f);
        if (f + 1 >= 0 && f + 1 <= t && s + 1 < static_cast<uint32_t>(nsteps)) prefetch(f + 1);
        __syncthreads();
    }
    cp_async_wait_all();
    // write back the state; fold the counts of the last delivered frame
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
        const uint32_t j = tid + r * NT;
        if (j >= na + nb) continue;
        if (j < na) {
            uint32_t a[kMaxClasses];
#pragma unroll
            for (int k = 0; k < kMaxClasses; ++k) a[k] = static_cast<uint32_t>(k) < K ? cnt[k * na + j] : 0u;
            detail::pack_get<ACC>::get(v[r]) = fold_frame(ps, detail::pack_get<ACC>::get(v[r]), a);
        }
        store_all(ps.nf, id_of(j), v[r]);
        if constexpr (model_uses_rng<M>())
            if (live[r]) ps.rng[id_of(j)] = rr[r];
    }
    for (int o = 16; o; o >>= 1) my_deliv += __shfl_xor_sync(0xffffffffu, my_deliv, o);
    if (lane == 0 && my_deliv) atomicAdd(&ps.counters[C_DELIVERIES], my_deliv);
    if (tid == 0) {
        if (my_spikes) atomicAdd(&ps.counters[C_SPIKES], my_spikes);
        if (logging) {
            *ps.log_end = lc;
            if (lc > ps.log_cap) ps.flags[0] = 1;
        }
    }
}

}  // namespace synq::dev
