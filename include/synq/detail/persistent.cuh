#pragma once
// Persistent, target-tiled pipeline for population-delivery models
// (vogels / brunel; trait synq::population_delivery<M>).
//
// Reference semantics: engine.hpp:188-218 (step), 308-341 (update),
// 369-409 (receive), lif.hpp:23-49 (LIF update / delta-synapse receive).
//
// Design (one cooperative launch runs a whole batch of steps):
// * Ownership.  The id space is cut into 2C contiguous PIECES; CTA c owns
//   piece A_c (a share of the receiving neurons, balanced by in-degree) and
//   piece B_c (a share of the update-only neurons, e.g. Brunel's Poisson
//   stimulus, balanced by count).  A CTA updates exactly its neurons and
//   receives exactly the deliveries that target A_c, so Receive(t) ->
//   Update(t+1) never leaves the SM and needs no grid barrier.  The neuron
//   state of the CTA lives in registers for the whole launch.
// * Frames.  Each CTA compacts its spikes per piece in ascending id order
//   into the piece's slice of queue slot t % Q and release-stores
//   {t+1, count} into finfo[slot][piece].  Pieces are numbered in id order,
//   so concatenating their slices gives the sorted frame.  Receive(t)
//   consumes frame t-delay+1, finished by every CTA delay-1 steps earlier: the
//   only cross-CTA wait is an acquire-poll that is normally satisfied at once.
//   With Q = 2*delay slots no slot is rewritten while a slower CTA may still
//   read it (a CTA runs at most delay-1 steps ahead of the slowest).
// * Delivery.  The row segment of spike s inside A_c is
//   [split[s][c], split[s][c+1]) of the sorted ELL row.  Segments are staged
//   as 32-target items in shared memory, read with kItemBatch loads in flight
//   per warp, and counted per (target, source class) with native shared-memory
//   atomics.  The update re-adds fl(c*w_k) count_k times in ascending class
//   (= ascending source id) order — exactly the reference's deterministic
//   float sum, independent of delivery order.
// * DRAM efficiency.  One step ahead, the full rows of frame due+1 are
//   streamed into L2 with one cp.async.bulk.prefetch.L2 per spike (spike g by
//   CTA g mod C): HBM sees contiguous ~28 KB row reads instead of C scattered
//   ~200-byte segment reads, and the next step's segment loads hit L2.
#include <cuda_runtime.h>

#include <cstdint>

#include "synq/detail/device_refs.cuh"
#include "synq/detail/kernels.cuh"
#include "synq/models/benchmarks.hpp"

namespace synq::dev {

constexpr int kPersistThreads = 1024;
constexpr int kMaxTiles = 160;             // CTAs (>= 148 SMs)
constexpr int kMaxPieces = 2 * kMaxTiles;  // id-ordered pieces
constexpr int kMaxClasses = 4;
constexpr uint32_t kItemCap = 2048;  // staged 32-target delivery items per pass (static smem)
constexpr int kItemBatch = 4;        // row loads in flight per warp

enum prof_slot : int { P_UPDATE = 0, P_PUBLISH, P_POLL, P_GATHER, P_DELIVER, P_STEPS, P_SLOTS = 8 };

template <class M>
struct persist_state {
    using NF = typename M::neuron_fields;
    field_ptrs<NF> nf;
    xorshift* rng;
    const uint32_t* cells;
    const uint32_t* split;      // [n][C+1]: receive-window boundaries of the CTAs
    const uint32_t* piece_lo;   // [P+1] piece boundaries in id order
    const uint32_t* cta_piece;  // [2C]: (A piece, B piece) of every CTA
    uint32_t pitch, n, C, P;
    uint32_t* queue;            // Q slots x n ids
    unsigned long long* finfo;  // Q x P: (t+1) << 32 | count
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
    // receives with due >= log_from, in piece (= ascending id) order
    uint32_t* log;
    unsigned long long* log_end;  // out: entries written
    unsigned long long log_cap;
    int64_t log_from;
    uint32_t* flags;
    uint32_t win_cap;          // count-window capacity per class (smem), >= max |A_c|
    unsigned long long* prof;  // optional per-CTA phase cycle counters (P_SLOTS each)
};

// streaming read of adjacency cells: read-only, no L1 allocation
SYNQ_DEV uint32_t ldg_stream(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
SYNQ_DEV void st_release_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SYNQ_DEV unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
SYNQ_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <class M>
SYNQ_DEV int source_class(const persist_state<M>& ps, uint32_t src) {
    int k = 0;
#pragma unroll
    for (int q = 0; q < kMaxClasses - 1; ++q)
        if (q < ps.K - 1 && src >= ps.bound[q]) k = q + 1;
    return k;
}

// re-add the per-class increments in ascending class (= ascending source id)
// order: the reference's float summation, one rounding per arrival
SYNQ_DEV float fold_arrivals(float acc, uint32_t n, float d) {
    uint32_t q = 0;
    for (; q + 4 <= n; q += 4) {
        acc = acc + d;
        acc = acc + d;
        acc = acc + d;
        acc = acc + d;
    }
    for (; q < n; ++q) acc = acc + d;
    return acc;
}

// block-wide exclusive scan of one value per thread (all NT threads call it)
template <int NT>
SYNQ_DEV uint32_t block_exclusive_scan(uint32_t x, uint32_t* s_tmp, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (lane == 31) s_tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < NT / 32 ? s_tmp[lane] : 0;
        uint32_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= static_cast<uint32_t>(o)) wi += y;
        }
        if (lane < NT / 32) s_tmp[lane] = wi - w;
        if (lane == 31) s_tmp[NT / 32] = wi;
    }
    __syncthreads();
    total = s_tmp[NT / 32];
    return s_tmp[warp] + incl - x;
}

// Warp-wide: wait until every piece of frame f is published (or, when
// nonblocking, only look), acquire, and write the exclusive piece prefix
// into seg[0..P] (seg[P] = frame size).  Returns false if nonblocking and the
// frame is not complete yet (seg untouched).
template <class M>
SYNQ_DEV bool frame_prefix(const persist_state<M>& ps, int64_t f, uint32_t* seg, bool nonblocking) {
    const uint32_t lane = threadIdx.x & 31, P = ps.P;
    const unsigned long long want = static_cast<unsigned long long>(f + 1);
    const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(f % ps.Q) * P;
    constexpr int kHalf = (kMaxPieces + 63) / 64;  // per lane, in two halves
    uint32_t cnt[2 * kHalf];
    bool ok = true;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        unsigned long long val[kHalf];
#pragma unroll
        for (int q = 0; q < kHalf; ++q) {
            const uint32_t j = (h * kHalf + q) * 32 + lane;
            val[q] = (j < P) ? ld_relaxed_gpu(fi + j) : (want << 32);
        }
#pragma unroll
        for (int q = 0; q < kHalf; ++q) {
            const uint32_t j = (h * kHalf + q) * 32 + lane;
            if (nonblocking) {
                ok &= (val[q] >> 32) == want;
            } else {
                while ((val[q] >> 32) != want) {
                    __nanosleep(20);
                    val[q] = ld_relaxed_gpu(fi + j);
                }
            }
            cnt[h * kHalf + q] = static_cast<uint32_t>(val[q]);
        }
    }
    if (nonblocking && !__all_sync(0xffffffffu, ok)) return false;
    fence_acq_rel_gpu();  // acquire: the slices are visible to this CTA
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < 2 * kHalf; ++q) {
        if (q * 32 >= static_cast<int>(P)) break;
        const uint32_t j = q * 32 + lane;
        const uint32_t cj = j < P ? cnt[q] : 0;
        uint32_t incl = cj;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (j < P) seg[j] = run + incl - cj;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) seg[P] = run;
    return true;
}

// the piece holding frame position g: last j with seg[j] <= g
SYNQ_DEV uint32_t piece_of(const uint32_t* seg, uint32_t P, uint32_t g) {
    uint32_t a = 0, e = P;
    while (e - a > 1) {
        const uint32_t mid = (a + e) >> 1;
        if (seg[mid] <= g)
            a = mid;
        else
            e = mid;
    }
    return a;
}

// NPT: neurons per thread, held in registers for the whole launch
template <class M, int NPT>
__global__ void __launch_bounds__(kPersistThreads, 1)
    k_persistent(M model, persist_state<M> ps, int64_t t0, int32_t nsteps) {
    using NF = typename M::neuron_fields;
    constexpr size_t ACC = population_delivery<M>::acc_field;
    constexpr int NT = kPersistThreads, NW = NT / 32;

    extern __shared__ __align__(16) uint32_t cnt[];       // K x win_cap arrival counters
    __shared__ uint4 s_item[kItemCap + kItemBatch * NW];  // {row lo, row hi, valid lanes, count offset}
    __shared__ uint32_t s_lo[kMaxPieces + 1];
    __shared__ uint32_t s_seg[kMaxPieces + 1];
    __shared__ uint32_t s_seg2[kMaxPieces + 1];  // frame due+1 (L2 row streaming); [P] = 0 if not ready
    __shared__ uint32_t s_wa[NPT * NW], s_wb[NPT * NW];
    __shared__ uint32_t s_tmp[NW + 1];
    __shared__ uint32_t s_mw[NW];
    __shared__ uint32_t s_out[2];
    __shared__ unsigned long long s_prof[P_SLOTS];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, C = ps.C, P = ps.P;
    for (uint32_t j = tid; j <= P; j += NT) s_lo[j] = ps.piece_lo[j];
    for (uint32_t j = tid; j < ps.K * ps.win_cap; j += NT) cnt[j] = 0;
    for (uint32_t j = tid; j < kItemBatch * NW; j += NT) s_item[kItemCap + j] = make_uint4(0, 0, 0, 0);
    if (tid < P_SLOTS) s_prof[tid] = 0;
    __syncthreads();
    const uint32_t pa = ps.cta_piece[2 * c], pb = ps.cta_piece[2 * c + 1];
    const uint32_t alo = s_lo[pa], na = s_lo[pa + 1] - alo;  // receiving piece
    const uint32_t blo = s_lo[pb], nb = s_lo[pb + 1] - blo;  // update-only piece
    unsigned long long my_deliv = 0, my_spikes = 0;
    unsigned long long lc = 0;  // CTA 0: log cursor
    const bool profiling = ps.prof != nullptr && tid == 0;
    long long tp = profiling ? clock64() : 0;
    auto mark = [&](int slot) {
        if (profiling) {
            const long long now = clock64();
            s_prof[slot] += now - tp;
            tp = now;
        }
    };
    // local index j -> neuron id: A piece first, then B piece
    auto id_of = [&](uint32_t j) { return j < na ? alo + j : blo + (j - na); };

    // register-resident neuron state
    values_t<NF> v[NPT];
    xorshift rr[NPT];
    bool live[NPT];
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
        live[r] = false;
        const uint32_t j = tid + r * NT;
        if (j < na + nb) load_all(ps.nf, id_of(j), v[r]);
    }

    for (int32_t s = 0; s < nsteps; ++s) {
        const int64_t t = t0 + s;
        const uint32_t slot = static_cast<uint32_t>(t % ps.Q);
        uint32_t* qslot = ps.queue + static_cast<uint64_t>(slot) * ps.n;

        // ------------------------------------------------ Update(t)
        bool spk[NPT];
        uint32_t mcount = 0;
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            const uint32_t j = tid + r * NT;
            spk[r] = false;
            if (j < na + nb) {
                const uint32_t i = id_of(j);
                if (j < na) {  // receiving neuron: fold the arrivals in class order
                    float acc = detail::pack_get<ACC>::get(v[r]);
                    for (int k = 0; k < ps.K; ++k) {
                        uint32_t* slotp = cnt + k * ps.win_cap + j;
                        const uint32_t a = *slotp;
                        if (a) {
                            *slotp = 0;
                            acc = fold_arrivals(acc, a, ps.delta[k]);
                        }
                    }
                    detail::pack_get<ACC>::get(v[r]) = acc;
                }
                local_neuron<NF> ref{i, &v[r], &rr[r], &live[r], ps.rng};
                spk[r] = model.update(ref, ps.dt);
                mcount += (spk[r] && i >= ps.meas_lo && i < ps.meas_hi) ? 1u : 0u;
            }
            const unsigned ba = __ballot_sync(0xffffffffu, spk[r] && j < na);
            const unsigned bb = __ballot_sync(0xffffffffu, spk[r] && j >= na);
            if (lane == 0) {
                s_wa[r * NW + warp] = __popc(ba);
                s_wb[r * NW + warp] = __popc(bb);
            }
        }
        for (int o = 16; o; o >>= 1) mcount += __shfl_xor_sync(0xffffffffu, mcount, o);
        if (lane == 0) s_mw[warp] = mcount;
        __syncthreads();
        if (warp == 0) {  // exclusive scans of the per-warp counts, ascending local index
            uint32_t runa = 0, runb = 0;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                const uint32_t xa = s_wa[r * NW + lane], xb = s_wb[r * NW + lane];
                uint32_t ia = xa, ib = xb;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
                    const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
                    if (lane >= static_cast<uint32_t>(o)) {
                        ia += ya;
                        ib += yb;
                    }
                }
                s_wa[r * NW + lane] = runa + ia - xa;
                s_wb[r * NW + lane] = runb + ib - xb;
                runa += __shfl_sync(0xffffffffu, ia, 31);
                runb += __shfl_sync(0xffffffffu, ib, 31);
            }
            uint32_t mm = s_mw[lane];
            for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
            if (lane == 0) {
                s_out[0] = runa;
                s_out[1] = runb;
                s_mw[0] = mm;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            const uint32_t j = tid + r * NT;
            const unsigned ba = __ballot_sync(0xffffffffu, spk[r] && j < na);
            const unsigned bb = __ballot_sync(0xffffffffu, spk[r] && j >= na);
            const unsigned below = (1u << lane) - 1u;
            if (spk[r]) {
                if (j < na)
                    qslot[alo + s_wa[r * NW + warp] + __popc(ba & below)] = id_of(j);
                else
                    qslot[blo + s_wb[r * NW + warp] + __popc(bb & below)] = id_of(j);
            }
        }
        const uint32_t outa = s_out[0], outb = s_out[1];
        const uint32_t meas = s_mw[0];
        mark(P_UPDATE);
        __syncthreads();  // piece slices complete
        // publish (the release covers the whole CTA's queue writes, ordered
        // before it by the barrier)
        if (tid == 0) {
            unsigned long long* fi = ps.finfo + static_cast<uint64_t>(slot) * P;
            const unsigned long long tag = static_cast<unsigned long long>(t + 1) << 32;
            st_release_gpu(fi + pa, tag | outa);
            st_release_gpu(fi + pb, tag | outb);
            if (outa + outb) atomicAdd(&ps.step_spikes[s], outa + outb);
            if (meas) atomicAdd(&ps.step_meas[s], meas);
            my_spikes += outa + outb;
        }
        mark(P_PUBLISH);

        // ------------------------------------------------ Receive(t - delay + 1)
        const int64_t due = t - static_cast<int64_t>(ps.delay) + 1;
        if (due < 0) continue;
        const uint32_t* dq = ps.queue + static_cast<uint64_t>(due % ps.Q) * ps.n;
        if (warp == 0) {
            frame_prefix(ps, due, s_seg, false);
        } else if (warp == 1) {
            const bool ready = due + 1 < t && frame_prefix(ps, due + 1, s_seg2, true);
            if (!ready && lane == 0) s_seg2[P] = 0;
        }
        __syncthreads();
        mark(P_POLL);
        // stream the FULL rows of frame due+1 into L2 (spike g by CTA g mod C)
        {
            const uint32_t S2 = s_seg2[P];
            const uint32_t g2 = c + (NT - 1 - tid) * C;
            if (g2 < S2) {
                const uint32_t a = piece_of(s_seg2, P, g2);
                const uint32_t* dq2 = ps.queue + static_cast<uint64_t>((due + 1) % ps.Q) * ps.n;
                const uint32_t src = __ldcg(dq2 + s_lo[a] + (g2 - s_seg2[a]));
                const uint32_t deg = __ldg(ps.split + static_cast<uint64_t>(src) * (C + 1) + C);
                const uint32_t bytes = (deg * 4 + 15) & ~15u;
                if (bytes)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     ps.cells + static_cast<uint64_t>(src) * ps.pitch),
                                 "r"(bytes)
                                 : "memory");
            }
        }
        const uint32_t S = s_seg[P];
        const bool logging = ps.log && c == 0 && due >= ps.log_from;
        for (uint32_t c0 = 0; c0 < S; c0 += NT) {
            // one spike per thread: id, this CTA's row segment, item count
            const uint32_t g = c0 + tid;
            uint32_t len = 0, cofs = 0, nchunk = 0;
            uint64_t row = 0;
            if (g < S) {
                const uint32_t a = piece_of(s_seg, P, g);
                const uint32_t src = __ldcg(dq + s_lo[a] + (g - s_seg[a]));
                if (logging && lc + g < ps.log_cap) ps.log[lc + g] = src;
                const uint32_t* sp = ps.split + static_cast<uint64_t>(src) * (C + 1) + c;
                const uint32_t sb = __ldg(sp), se = __ldg(sp + 1);
                len = se - sb;
                row = static_cast<uint64_t>(src) * ps.pitch + sb;
                cofs = static_cast<uint32_t>(source_class(ps, src)) * ps.win_cap - alo;
                nchunk = (len + 31) >> 5;
                my_deliv += len;
            }
            uint32_t nitems;
            const uint32_t first = block_exclusive_scan<NT>(nchunk, s_tmp, nitems);
            mark(P_GATHER);
            // items in passes of kItemCap (a pass is normally the whole frame)
            for (uint32_t i0 = 0; i0 < nitems; i0 += kItemCap) {
                for (uint32_t q = 0; q < nchunk; ++q) {
                    const uint32_t it = first + q;
                    if (it < i0 || it >= i0 + kItemCap) continue;
                    const uint64_t rq = row + 32ull * q;
                    s_item[it - i0] = make_uint4(static_cast<uint32_t>(rq), static_cast<uint32_t>(rq >> 32),
                                                 min(32u, len - 32 * q), cofs);
                }
                __syncthreads();
                const uint32_t m = min(kItemCap, nitems - i0);
                // kItemBatch items per warp in flight: LDS.128 -> LDG -> ATOMS
                // (items past m read the zero padding: no valid lanes)
                for (uint32_t it = warp; it < m; it += kItemBatch * NW) {
                    uint4 d[kItemBatch];
                    uint32_t tg[kItemBatch];
#pragma unroll
                    for (int u = 0; u < kItemBatch; ++u) {
                        const uint32_t k = it + u * NW;
                        d[u] = s_item[k < m ? k : kItemCap + u * NW + warp];
                    }
#pragma unroll
                    for (int u = 0; u < kItemBatch; ++u) {
                        const uint32_t* rp = ps.cells + ((static_cast<uint64_t>(d[u].y) << 32) | d[u].x);
                        tg[u] = lane < d[u].z ? ldg_stream(rp + lane) : 0xffffffffu;
                    }
#pragma unroll
                    for (int u = 0; u < kItemBatch; ++u)
                        if (tg[u] != 0xffffffffu) atomicAdd(&cnt[d[u].w + tg[u]], 1u);
                }
                __syncthreads();
            }
            mark(P_DELIVER);
        }
        if (logging) lc += S;
    }
    if (ps.log && c == 0 && tid == 0) {
        *ps.log_end = lc;
        if (lc > ps.log_cap) ps.flags[0] = 1;
    }

    // write back the register-resident state; fold pending arrivals into ACC
    // so host reads and the next launch see them
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
        const uint32_t j = tid + r * NT;
        if (j >= na + nb) continue;
        if (j < na) {
            float acc = detail::pack_get<ACC>::get(v[r]);
            for (int k = 0; k < ps.K; ++k) acc = fold_arrivals(acc, cnt[k * ps.win_cap + j], ps.delta[k]);
            detail::pack_get<ACC>::get(v[r]) = acc;
        }
        const uint32_t i = id_of(j);
        store_all(ps.nf, i, v[r]);
        if constexpr (model_uses_rng<M>())
            if (live[r]) ps.rng[i] = rr[r];
    }
    for (int o = 16; o; o >>= 1) my_deliv += __shfl_xor_sync(0xffffffffu, my_deliv, o);
    if (lane == 0 && my_deliv) atomicAdd(&ps.counters[C_DELIVERIES], my_deliv);
    if (tid == 0 && my_spikes) atomicAdd(&ps.counters[C_SPIKES], my_spikes);
    if (profiling) {
        s_prof[P_STEPS] = static_cast<unsigned long long>(nsteps);
        for (int k = 0; k < P_SLOTS; ++k) atomicAdd(&ps.prof[c * P_SLOTS + k], s_prof[k]);
    }
}

// Copy frames [from, to] (all complete in the ring) into the ordered log;
// used once at the end of run() for the frames not yet consumed by Receive.
template <class M>
__global__ void k_log_drain(persist_state<M> ps, int64_t from, int64_t to) {
    __shared__ uint32_t s_seg[kMaxPieces + 1];
    __shared__ uint32_t s_lo[kMaxPieces + 1];
    const uint32_t P = ps.P;
    for (uint32_t j = threadIdx.x; j <= P; j += blockDim.x) s_lo[j] = ps.piece_lo[j];
    unsigned long long lc = 0;
    for (int64_t f = from; f <= to; ++f) {
        const uint32_t slot = static_cast<uint32_t>(f % ps.Q);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (uint32_t j = 0; j < P; ++j) {
                s_seg[j] = run;
                run += static_cast<uint32_t>(ps.finfo[static_cast<uint64_t>(slot) * P + j]);
            }
            s_seg[P] = run;
        }
        __syncthreads();
        const uint32_t S = s_seg[P];
        for (uint32_t j = 0; j < P; ++j) {
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
