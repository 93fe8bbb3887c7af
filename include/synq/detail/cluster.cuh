#pragma once
// Thread-block-cluster engine for small population-delivery networks
// (Vogels-Abbott 4000, BASELINE config 1; SURVEY.md 7.1 hard part 1).
//
// Reference semantics are those of k_persistent / k_pipeline
// (engine.hpp:188-218 step, 308-341 update, 369-409 receive): arrivals are
// counted per (target, source class) and re-added in class order by the
// update, so spike trains and state are the reference's deterministic ones.
//
// The machine: one cluster of CL CTAs (8, or 16 with the non-portable size)
// owns the whole network, each CTA a receiving piece and an update-only
// piece, state in registers.  Frames never touch global memory on the step's
// chain: every CTA writes its spike ids and piece counts straight into every
// peer's shared-memory frame ring (distributed shared memory), and one
// cluster barrier per step (arrive.release / wait.acquire) makes frame t
// complete everywhere.  The multi-CTA engines instead publish through L2
// with a gpu-scope release and poll it.  Each CTA then counts the due frame
// for its own targets from its row segments (cached per source at launch),
// whose rows were copied into shared memory one step earlier.
//
// Ring slots: frame f lives in slot f % (delay + 1).  A CTA writes frame t+1
// only after the barrier of step t, i.e. after every CTA published frame t;
// a slower CTA may still be counting frame t - delay + 1 (slot
// (t - delay + 1) % (delay + 1) != (t + 1) % (delay + 1)) or copying rows of
// frame t - delay + 2 (likewise distinct), so no slot is overwritten early.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "synq/detail/persistent.cuh"
#include "synq/detail/pipeline.cuh"

namespace synq::dev {

constexpr int kClusterThreads = 512;
constexpr uint32_t kClusterMaxNeurons = 16 * 2 * kClusterThreads;  // 16 CTAs x 2 neurons per thread
constexpr uint32_t kClusterMaxDelay = 63;
constexpr uint32_t kClusterRows = 4096;  // row entries per copy buffer (two buffers)

// dynamic shared memory of one CTA: counts K x wcap, ring (delay+1) x n ids,
// piece counts (delay+1) x 2CL, row segments n, two row buffers
inline size_t cluster_smem_bytes(uint32_t K, uint32_t wcap, uint32_t n, uint32_t delay, uint32_t CL) {
    return (size_t(K) * wcap + size_t(delay + 1) * n + size_t(delay + 1) * 2 * CL + n + 2 * size_t(kClusterRows)) * 4 +
           64;
}

template <class M, int NPT>
__global__ void __launch_bounds__(kClusterThreads, 1)
    k_cluster(M model, persist_state<M> ps, int64_t t0, int32_t nsteps) {
    namespace cg = cooperative_groups;
    using NF = typename M::neuron_fields;
    constexpr size_t ACC = population_delivery<M>::acc_field;
    constexpr int NT = kClusterThreads, NW = NT / 32;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t c = cluster.block_rank(), CL = cluster.num_blocks();
    const uint32_t K = static_cast<uint32_t>(ps.K), delay = ps.delay, n = ps.n, P = ps.P, D1 = delay + 1;
    const uint32_t pa = ps.cta_piece[2 * c], pb = ps.cta_piece[2 * c + 1];
    const uint32_t alo = ps.piece_lo[pa], na = ps.piece_lo[pa + 1] - alo;
    const uint32_t blo = ps.piece_lo[pb], nb = ps.piece_lo[pb + 1] - blo;
    const uint32_t wcap = ps.win_cap;
    uint32_t* cnt = sm;                        // K x wcap arrival counts of the own targets
    uint32_t* ring = cnt + K * wcap;           // D1 x n: frame f's piece p at ring[f % D1][piece_lo[p]..]
    uint32_t* pcnt = ring + D1 * n;            // D1 x P piece counts
    uint32_t* seg = pcnt + D1 * P;             // n: own row segment of each source (lo | hi << 16)
    uint32_t* rows = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(seg + n) + 15) & ~uintptr_t(15));
    __shared__ uint32_t s_wa[NPT * NW], s_wb[NPT * NW], s_mw[NW];
    __shared__ uint32_t s_out[3];
    __shared__ uint32_t s_rofs[2][kClusterThreads];  // prefetched rows: offset of each spike's segment
    __shared__ long long s_pff[2];                   // frame whose rows each buffer holds (-1: none)
    __shared__ uint32_t s_tmp[NW + 1];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t j = tid; j < K * wcap; j += NT) cnt[j] = 0;
    for (uint32_t s = tid; s < n; s += NT) {
        const uint32_t* sp = ps.split + static_cast<uint64_t>(s) * (ps.C + 1) + c;
        seg[s] = __ldg(sp) | (__ldg(sp + 1) << 16);
    }
    // frames of earlier launches (t0 - delay + 1 .. t0 - 1) into the ring
    for (uint32_t k = 1; k < delay; ++k) {
        const int64_t f = t0 - static_cast<int64_t>(k);
        if (f < 0) break;
        const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(f % ps.Q) * ps.E;
        const uint32_t* qs = ps.queue + static_cast<uint64_t>(f % ps.Q) * n;
        uint32_t* rs = ring + static_cast<uint32_t>(f % D1) * n;
        for (uint32_t p = warp; p < P; p += NW) {
            const uint32_t src = ps.piece_src[p];
            const uint32_t cp = word_half(fi[src >> 1], src & 1);
            if (lane == 0) pcnt[static_cast<uint32_t>(f % D1) * P + p] = cp;
            for (uint32_t i = lane; i < cp; i += 32) rs[ps.piece_lo[p] + i] = qs[ps.piece_lo[p] + i];
        }
    }
    if (tid < 2) s_pff[tid] = -1;
    __syncthreads();

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
    const bool log_cta = ps.log != nullptr && c == 0;
    // the spikes of frame f in id order: pieces in id order, each a slice
    auto frame_size = [&](int64_t f) {
        const uint32_t* pc = pcnt + static_cast<uint32_t>(f % D1) * P;
        uint32_t S = 0;
        for (uint32_t p = 0; p < P; ++p) S += pc[p];
        return S;
    };

    uint32_t slot = static_cast<uint32_t>(t0 % ps.Q);
    for (uint32_t s = 0; s < static_cast<uint32_t>(nsteps); ++s, slot = slot + 1 == ps.Q ? 0u : slot + 1) {
        const int64_t t = t0 + s;
        // ---- 1. fold frame t - delay (counted at step t - 1), update, ballots
        bool spk[NPT];
        unsigned bal[NPT];
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
                        a[k] = static_cast<uint32_t>(k) < K ? cnt[k * wcap + j] : 0u;
                        if (a[k]) cnt[k * wcap + j] = 0;
                    }
                    detail::pack_get<ACC>::get(v[r]) = fold_frame(ps, detail::pack_get<ACC>::get(v[r]), a);
                }
                local_neuron<NF> ref{id_of(j), &v[r], &rr[r], &live[r], ps.rng};
                spk[r] = model.update(ref, ps.dt);
            }
            bal[r] = __ballot_sync(0xffffffffu, spk[r]);
            mcount += __popc(__ballot_sync(0xffffffffu, spk[r] && inmeas[r]));
            if (lane == 0) {
                s_wa[r * NW + warp] = __popc(bal[r] & amask[r]);
                s_wb[r * NW + warp] = __popc(bal[r] & ~amask[r]);
            }
        }
        if (lane == 0) s_mw[warp] = mcount;
        __syncthreads();
        if (warp == 0) {
            uint32_t runa = 0, runb = 0;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                const uint32_t xa = lane < NW ? s_wa[r * NW + lane] : 0u, xb = lane < NW ? s_wb[r * NW + lane] : 0u;
                const uint32_t ia = warp_incl_scan(xa), ib = warp_incl_scan(xb);
                if (lane < NW) {
                    s_wa[r * NW + lane] = runa + ia - xa;
                    s_wb[r * NW + lane] = runb + ib - xb;
                }
                runa += __shfl_sync(0xffffffffu, ia, 31);
                runb += __shfl_sync(0xffffffffu, ib, 31);
            }
            uint32_t mm = lane < NW ? s_mw[lane] : 0u;
            for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
            if (lane == 0) {
                s_out[0] = runa;
                s_out[1] = runb;
                s_out[2] = mm;
            }
        }
        __syncthreads();
        // ---- 2. frame t: own slices into every CTA's ring (DSMEM), global
        // queue slot and frame word (host / log drain format)
        {
            const uint32_t outa = s_out[0], outb = s_out[1];
            const uint32_t rslot = static_cast<uint32_t>(t % D1);
            uint32_t* qslot = ps.queue + static_cast<uint64_t>(slot) * n;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                if (!spk[r]) continue;
                const uint32_t j = tid + r * NT, id = id_of(j);
                const bool in_a = (amask[r] >> lane) & 1u;
                const unsigned m = in_a ? amask[r] : ~amask[r];
                const uint32_t pos = (in_a ? s_wa[r * NW + warp] : s_wb[r * NW + warp]) + __popc(bal[r] & m & below);
                const uint32_t at = (in_a ? alo : blo) + pos;
                qslot[at] = id;
                for (uint32_t q = 0; q < CL; ++q) cluster.map_shared_rank(ring, q)[rslot * n + at] = id;
            }
            if (tid < CL) {
                uint32_t* pc = cluster.map_shared_rank(pcnt, tid) + rslot * P;
                pc[pa] = outa;
                pc[pb] = outb;
            }
            if (tid == 0) {
                ps.finfo[static_cast<uint64_t>(slot) * ps.E + c] = frame_word(t, outa, outb);
                my_spikes += outa + outb;
            }
            if (tid == 0) atomicAdd(&ps.step_spikes[s], outa + outb);
            if (tid == 0 && s_out[2]) atomicAdd(&ps.step_meas[s], s_out[2]);
        }
        cp_async_wait_all();
        cluster.sync();  // frame t complete in every CTA; rows of the due frame landed
        // ---- 3. count frame f = t - delay + 1 for the own targets
        const int64_t f = t - static_cast<int64_t>(delay) + 1;
        if (f >= 0) {
            const uint32_t fs = static_cast<uint32_t>(f % D1);
            const uint32_t* pc = pcnt + fs * P;
            const uint32_t* rs = ring + fs * n;
            const uint32_t S = frame_size(f);
            const bool staged = s_pff[f & 1] == f;
            const uint32_t* rb = rows + (f & 1) * kClusterRows;
            // spike i of the frame (id order) handled by warp i % NW
            uint32_t p = 0, base = 0;
            for (uint32_t i = warp; i < S; i += NW) {
                while (base + pc[p] <= i) base += pc[p++];
                const uint32_t src = rs[ps.piece_lo[p] + (i - base)];
                const uint32_t sg = seg[src], lo = sg & 0xffffu, hi = sg >> 16;
                const uint32_t cls = static_cast<uint32_t>(source_class(ps, src));
                uint32_t* cb = cnt + cls * wcap - alo;
                if (staged && i < kClusterThreads) {
                    const uint32_t* r0 = rb + s_rofs[f & 1][i];
                    for (uint32_t q = lane; q < hi - lo; q += 32) atomicAdd(cb + r0[q], 1u);
                } else {
                    const uint32_t* r0 = ps.cells + static_cast<uint64_t>(src) * ps.pitch + lo;
                    for (uint32_t q = lane; q < hi - lo; q += 32) atomicAdd(cb + __ldg(r0 + q), 1u);
                }
                if (lane == 0) my_deliv += hi - lo;
                if (log_cta && f >= ps.log_from && lane == 0 && lc + i < ps.log_cap) ps.log[lc + i] = src;
            }
            if (log_cta && f >= ps.log_from) {
                if (tid == 0) ps.log_cnt[f - ps.log_from] = S;
                lc += S;
            }
        }
        // ---- 4. copy the own row segments of the next due frame (f + 1)
        if (f + 1 >= 0 && f + 1 <= t && s + 1 < static_cast<uint32_t>(nsteps)) {
            const int64_t g = f + 1;
            const uint32_t gs = static_cast<uint32_t>(g % D1);
            const uint32_t* pc = pcnt + gs * P;
            const uint32_t* rs = ring + gs * n;
            const uint32_t S = frame_size(g);
            // offsets: exclusive scan of segment sizes over the first <= NT spikes
            uint32_t len = 0, src = 0;
            if (tid < S && tid < kClusterThreads) {
                uint32_t p = 0, base = 0;
                while (base + pc[p] <= tid) base += pc[p++];
                src = rs[ps.piece_lo[p] + (tid - base)];
                const uint32_t sg = seg[src];
                len = (sg >> 16) - (sg & 0xffffu);
            }
            uint32_t tot = 0;
            const uint32_t off = block_exclusive_scan<NT>(len, s_tmp, tot);
            const bool fits = S <= kClusterThreads && tot <= kClusterRows;
            if (fits && tid < S) {
                s_rofs[g & 1][tid] = off;
                const uint32_t lo = seg[src] & 0xffffu;
                const uint32_t* gr = ps.cells + static_cast<uint64_t>(src) * ps.pitch + lo;
                uint32_t* db = rows + (g & 1) * kClusterRows + off;
                for (uint32_t q = 0; q < len; ++q) cp_async4(db + q, gr + q);
            }
            if (tid == 0) s_pff[g & 1] = fits ? g : -1;
        }
        __syncthreads();
    }
    cp_async_wait_all();
    cluster.sync();  // no CTA leaves while a peer may still write into its ring
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
        const uint32_t j = tid + r * NT;
        if (j >= na + nb) continue;
        if (j < na) {
            uint32_t a[kMaxClasses];
#pragma unroll
            for (int k = 0; k < kMaxClasses; ++k) a[k] = static_cast<uint32_t>(k) < K ? cnt[k * wcap + j] : 0u;
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
        if (log_cta) {
            *ps.log_end = lc;
            if (lc > ps.log_cap) ps.flags[0] = 1;
        }
    }
}

}  // namespace synq::dev
