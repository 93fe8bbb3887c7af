#pragma once
// Pipelined persistent engine for population-delivery models (vogels /
// brunel; trait synq::population_delivery<M>): the default step kernel.
//
// Reference semantics are those of k_persistent (persistent.cuh):
// engine.hpp:188-218 (step), 308-341 (update), 369-409 (receive),
// lif.hpp:23-49.  Ownership (pieces A_c / B_c), frames (per-piece slices of
// queue slot f % Q + one release-stored word per publisher) and exactness
// (arrivals counted per (target, source class), re-added in class order by
// the update) are the same.  What changes is the schedule.
//
// Receive(t) consumes frame t-delay+1, and its arrivals are first read by
// Update(t+1).  A frame is therefore needed delay steps after it was
// published, and the delivery work of a step is NOT on the update's critical
// path.  k_persistent still runs update -> publish -> poll -> gather ->
// deliver as one serial chain per step (a chain of L2/HBM round trips,
// ~15 us per step at Brunel 1e9).  Here every CTA is warp-specialised:
//
// * Update warps (UW warps, neuron state in registers) run Update(t):
//   fold the arrival counts of frame t-delay from the count ring, call
//   model.update, compact the spikes per piece, publish the frame, and
//   stream the full rows of their spikes into L2
//   (cp.async.bulk.prefetch.L2) for the deliverers of every CTA.
// * Delivery warps stream frames into a ring of R per-frame count windows
//   in shared memory (slot = frame mod R).  Each pass takes EVERY frame that
//   is complete (up to kPipeMaxBatch): the more the deliverers lag, the
//   larger their batches, so latency is amortised over more work.  A
//   delivery pass is: poll (one warp per frame), gather (spike ids, row
//   windows, 16-byte chunk list), then 16-byte row-chunk loads with
//   shared-memory counting atomics (ATOMS.POPC.INC).
//
// Flow control (all shared-memory release/acquire inside the CTA):
// * frame f is delivered once frame f + lag is complete: its publishers
//   streamed its rows into L2 meanwhile, so HBM sees whole-row bulk reads
//   and the deliverers' 16-byte chunk loads hit L2;
// * update(t) waits until frame t - min(lead, delay) is delivered locally.
//   This is needed for t - delay.  The lead bounds how far the update can
//   run ahead, so the rows it prefetched are still in L2 when they are
//   delivered.  The wait never reaches past frame t - delay + R - 1: that
//   frame's ring slot is only freed by update(t) itself;
// * delivering frame f into slot f mod R waits until update(f - R + delay)
//   folded (and zeroed) that slot's previous frame;
// * the queue ring (Q = 2*delay slots) is never overwritten before every CTA
//   delivered the frame: a CTA at update(t) implies every CTA delivered
//   frame >= t - 2*lead >= t - Q.
// Frames are indexed relative to the launch: rel(f) = f - (t0 - delay), so a
// launch of nsteps delivers rel 1 .. nsteps and update step s folds rel s.
#include <cuda_runtime.h>

#include <cstdint>

#include "synq/detail/persistent.cuh"

namespace synq::dev {

constexpr int kPipeThreads = 512;
constexpr int kStreamChunks = 64;  // streamed update: up to 64 x UT neurons per CTA
constexpr int kPipeMaxBatch = 8;  // frames per delivery pass (group ids frame * 4 + class < 32)
constexpr int kEllSpt = 4;        // ELL delivery: spikes per thread per iteration

SYNQ_DEV uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
SYNQ_DEV void st_release_cta(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
SYNQ_DEV uint32_t ld_acquire_cta(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
SYNQ_DEV void named_bar(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// wait until *p >= want (every calling thread acquires)
SYNQ_DEV void wait_at_least(const uint32_t* p, uint32_t want) {
    while (ld_acquire_cta(p) < want) __nanosleep(64);
}

// exclusive scan of one value per thread over a named-barrier group of NTH
// threads starting at warp W0
template <int NTH, int W0, int BAR>
SYNQ_DEV uint32_t group_exclusive_scan(uint32_t x, uint32_t* s_tmp, uint32_t& total) {
    constexpr int NWG = NTH / 32;
    const uint32_t lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - W0;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (lane == 31) s_tmp[warp] = incl;
    named_bar(BAR, NTH);
    if (warp == 0) {
        const uint32_t w = lane < NWG ? s_tmp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= static_cast<uint32_t>(o)) wi += y;
        }
        if (lane < NWG) s_tmp[lane] = wi - w;
        if (lane == 31) s_tmp[NWG] = wi;
    }
    named_bar(BAR, NTH);
    total = s_tmp[NWG];
    const uint32_t r = s_tmp[warp] + incl - x;
    named_bar(BAR, NTH);  // s_tmp may be reused right after
    return r;
}

// Ampere-style asynchronous global->shared copies (LDGSTS): no registers
// are held while the copies are in flight
SYNQ_DEV void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
SYNQ_DEV void cp_async16_cg(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
SYNQ_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 32x32 bit transpose across a warp: lane i holds row i on entry, lane b
// holds column b on exit (bit i = bit b of lane i's entry word).  Stages 16
// and 8 are byte permutes, stages 4 / 2 / 1 a rotate plus one LOP3 merge.
// The per-lane selectors / rotations / merge masks are hoisted (tp_consts).
struct tp_consts {
    uint32_t sel16, sel8, rot[3], keep[3];
};
SYNQ_DEV tp_consts make_tp_consts(uint32_t lane) {
    tp_consts k;
    k.sel16 = (lane & 16) ? 0x3276u : 0x5410u;
    k.sel8 = (lane & 8) ? 0x3715u : 0x6240u;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        const uint32_t j = 4u >> s;
        const uint32_t m = s == 0 ? 0x0f0f0f0fu : (s == 1 ? 0x33333333u : 0x55555555u);
        const bool hi = (lane & j) != 0;
        k.rot[s] = hi ? 32 - j : j;
        k.keep[s] = hi ? ~m : m;
    }
    return k;
}
SYNQ_DEV uint32_t lop3_merge(uint32_t x, uint32_t t, uint32_t keep) {  // (x & keep) | (t & ~keep)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(x), "r"(t), "r"(keep));
    return d;
}
SYNQ_DEV uint32_t transpose32(uint32_t x, const tp_consts& k) {
    uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16);
    x = __byte_perm(x, y, k.sel16);
    y = __shfl_xor_sync(0xffffffffu, x, 8);
    x = __byte_perm(x, y, k.sel8);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        y = __shfl_xor_sync(0xffffffffu, x, 4 >> s);
        x = lop3_merge(x, __funnelshift_l(y, y, k.rot[s]), k.keep[s]);
    }
    return x;
}

// UW update warps (NPT neurons per update thread); the other warps deliver.
// BM: bitmap delivery (receive-window bitmaps + transposed counting), else
// 16-byte ELL row chunks counted with one shared-memory atomic per delivery.
template <class M, int UW, int NPT, bool BM, int NT = kPipeThreads>
__global__ void __launch_bounds__(NT, 1)
    k_pipeline(M model, persist_state<M> ps, int64_t t0, int32_t nsteps) {
    using NF = typename M::neuron_fields;
    constexpr size_t ACC = population_delivery<M>::acc_field;
    constexpr int NW = NT / 32;
    constexpr int UT = UW * 32, DT = NT - UT, DW = NW - UW;
    constexpr uint32_t BAR_U = 1, BAR_D = 2;
    // frames per delivery pass: one polling warp per frame
    constexpr int MB = DW < kPipeMaxBatch ? DW : kPipeMaxBatch;
    static_assert(MB >= 4, "at least 4 delivery warps");
    static_assert(4 * MB <= 32, "bitmap group tables hold 32 (frame, class) groups");

    // dynamic: count ring (R x K x win_cap) | row prefetch windows (pf) | chunk list
    extern __shared__ __align__(16) uint32_t ring[];
    const uint32_t ring_words = (ps.R * ps.K * ps.win_cap + 3) & ~3u;
    uint2* pf = reinterpret_cast<uint2*>(ring + ring_words);
    uint2* chunks = pf + ps.pf_cap;
    __shared__ uint32_t s_lo[kMaxPieces + 1];
    __shared__ uint32_t s_psrc[kMaxPieces];
    __shared__ uint32_t s_seg[MB][kMaxPieces + 1];
    __shared__ unsigned long long s_fval[MB][kMaxTiles];
    __shared__ uint32_t s_ok[MB];
    __shared__ uint32_t s_gbeg[32], s_gend[32];  // bitmap delivery: spike range of group frame * 4 + class
    __shared__ uint32_t s_gcp[33];                // ... exclusive prefix of its 7-block chunks
    __shared__ uint32_t s_qbase[MB];  // queue slot base of frame w of the pass
    __shared__ uint32_t s_cbase[MB];  // count-ring slot base of frame w of the pass
    __shared__ uint32_t s_dtmp[DW + 1];
    __shared__ uint32_t s_wa[(NPT > 0 ? NPT : 1) * UW], s_wb[(NPT > 0 ? NPT : 1) * UW], s_mw[UW], s_out[3];
    // streamed update (NPT == 0): per (chunk, warp) spike counts and ballots
    constexpr int kSE = NPT == 0 ? kStreamChunks * UW : 1;
    __shared__ uint32_t s_sa[kSE], s_sb[kSE], s_spk[kSE];
    // streamed bitmap delivery: frame table + linear work space
    __shared__ uint32_t s_ft_base[MB], s_ft_nb[MB], s_ft_S[MB], s_ft_q[MB], s_ft_cb[MB], s_ft_done[MB];
    __shared__ unsigned long long s_ft_lb[MB];
    __shared__ uint32_t s_work_next, s_work_end, s_work_total;
    __shared__ uint32_t s_delivered;  // frames delivered: rel 0 .. s_delivered
    __shared__ uint32_t s_updated;    // update steps whose fold is done
    __shared__ unsigned long long s_prof[P_SLOTS];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, C = ps.C, P = ps.P;
    for (uint32_t j = tid; j <= P; j += NT) s_lo[j] = ps.piece_lo[j];
    for (uint32_t j = tid; j < P; j += NT) s_psrc[j] = ps.piece_src[j];
    for (uint32_t j = tid; j < ring_words; j += NT) ring[j] = 0;
    if (tid < 32) {
        s_gbeg[tid] = 0;
        s_gend[tid] = 0;
    }
    if (tid < P_SLOTS) s_prof[tid] = 0;
    if (tid == 0) {
        s_delivered = 0;
        s_updated = 0;
        s_work_next = 0;
        s_work_end = 0;
        s_work_total = 0xffffffffu;
    }
    if (tid < MB) {
        s_ft_base[tid] = 0;
        s_ft_nb[tid] = 0;
        s_ft_done[tid] = 0;
        s_ft_S[tid] = 0;
    }
    __syncthreads();
    const uint32_t pa = ps.cta_piece[2 * c], pb = ps.cta_piece[2 * c + 1];
    const uint32_t alo = s_lo[pa], na = s_lo[pa + 1] - alo;  // receiving piece
    const uint32_t blo = s_lo[pb], nb = s_lo[pb + 1] - blo;  // update-only piece
    auto id_of = [&](uint32_t j) { return j < na ? alo + j : blo + (j - na); };
    // this shard's window of every row: [split[s][0], split[s][C])
    if (ps.pf_cap)
        for (uint32_t j = tid; j < na + nb; j += NT) {
            const uint32_t i = id_of(j);
            pf[j] = make_uint2(__ldg(ps.split + static_cast<uint64_t>(i) * (C + 1)) & ~3u,
                               __ldg(ps.split + static_cast<uint64_t>(i) * (C + 1) + C));
        }
    __syncthreads();
    const uint32_t R = ps.R;
    const int64_t fbase = t0 - static_cast<int64_t>(ps.delay);  // frame of rel 0
    const uint32_t nrel = static_cast<uint32_t>(nsteps);
    const bool profiling = ps.prof != nullptr && (tid == 0 || tid == static_cast<uint32_t>(UT));
    long long tp = profiling ? clock64() : 0;
    auto mark = [&](int slot) {
        if (profiling) {
            const long long now = clock64();
            s_prof[slot] += now - tp;
            tp = now;
        }
    };

    if (NPT == 0 && warp < static_cast<uint32_t>(UW)) {
        // ============================================ update warps, streamed
        // NPT == 0: more neurons per CTA than registers hold (up to
        // kStreamChunks * UT).  The state stays in HBM (SoA, coalesced) and is
        // loaded, updated and stored every step in chunks of UT neurons; the
        // spike flags go through a shared-memory bitmask.
        const uint32_t lead = min(ps.lead, ps.delay);
        const uint32_t L = na + nb, MC = (L + UT - 1) / UT;
        unsigned long long my_spikes = 0;
        uint32_t slot = static_cast<uint32_t>(t0 % ps.Q);
        for (uint32_t s = 0; s < nrel; ++s, slot = slot + 1 == ps.Q ? 0u : slot + 1) {
            const int64_t t = t0 + s;
            uint32_t* qslot = ps.queue + static_cast<uint64_t>(slot) * ps.n;
            if (warp == 0) wait_at_least(&s_delivered, min(min(s + ps.delay - lead, s + R - 1), nrel));
            named_bar(BAR_U, UT);
            mark(P_POLL);
            uint32_t* cslot = ring + (s % R) * ps.K * ps.win_cap;
            uint32_t mcount = 0;
            // chunk m + 1's state (and RNG) is loaded before chunk m is
            // updated and stored (distinct neurons), so the loads of the next
            // chunk are in flight while this one computes
            values_t<NF> vn{};
            xorshift rn;
            auto fetch = [&](uint32_t m) {
                const uint32_t j = tid + m * UT;
                if (j < L) {
                    const uint32_t i = id_of(j);
                    load_all(ps.nf, i, vn);
                    if constexpr (model_uses_rng<M>()) rn = ps.rng[i];
                }
            };
            if (MC) fetch(0);
            for (uint32_t m = 0; m < MC; ++m) {
                const uint32_t j = tid + m * UT;
                bool sp = false;
                values_t<NF> vl = vn;
                xorshift rl = rn;
                if (m + 1 < MC) fetch(m + 1);
                if (j < L) {
                    const uint32_t i = id_of(j);
                    if (j < na) {  // receiving neuron: fold frame rel s in class order
                        uint32_t a[kMaxClasses];
#pragma unroll
                        for (int k = 0; k < kMaxClasses; ++k) {
                            a[k] = k < ps.K ? cslot[k * ps.win_cap + j] : 0u;
                            if (a[k]) cslot[k * ps.win_cap + j] = 0;
                        }
                        detail::pack_get<ACC>::get(vl) = fold_frame(ps, detail::pack_get<ACC>::get(vl), a);
                    }
                    const xorshift r0 = rl;
                    bool ll = model_uses_rng<M>();  // prefetched: rng() must not reload it
                    local_neuron<NF> ref{i, &vl, &rl, &ll, ps.rng};
                    sp = model.update(ref, ps.dt);
                    store_all(ps.nf, i, vl);
                    if constexpr (model_uses_rng<M>()) {
                        uint4 a, b;
                        memcpy(&a, &rl, 16);
                        memcpy(&b, &r0, 16);
                        if (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) ps.rng[i] = rl;  // drawn from
                    }
                    if (sp && i >= ps.meas_lo && i < ps.meas_hi) ++mcount;
                }
                const int na_here = static_cast<int>(na) - static_cast<int>(m * UT + warp * 32);
                const unsigned amask = na_here >= 32 ? 0xffffffffu : (na_here <= 0 ? 0u : (1u << na_here) - 1u);
                const unsigned bal = __ballot_sync(0xffffffffu, sp);
                if (lane == 0) {
                    s_sa[m * UW + warp] = __popc(bal & amask);
                    s_sb[m * UW + warp] = __popc(bal & ~amask);
                    s_spk[m * UW + warp] = bal;
                }
            }
            for (int o = 16; o; o >>= 1) mcount += __shfl_xor_sync(0xffffffffu, mcount, o);
            if (lane == 0) s_mw[warp] = mcount;
            mark(P_UPDATE);
            named_bar(BAR_U, UT);  // counts, flags and the slot zeroing are complete
            if (tid == 0) st_release_cta(&s_updated, s + 1);
            if (warp == 0) {  // exclusive scans in ascending local index: (chunk, warp) order
                uint32_t runa = 0, runb = 0;
                for (uint32_t e0 = 0; e0 < MC * UW; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    const uint32_t xa = e < MC * UW ? s_sa[e] : 0u, xb = e < MC * UW ? s_sb[e] : 0u;
                    const uint32_t ia = warp_incl_scan(xa), ib = warp_incl_scan(xb);
                    if (e < MC * UW) {
                        s_sa[e] = runa + ia - xa;
                        s_sb[e] = runb + ib - xb;
                    }
                    runa += __shfl_sync(0xffffffffu, ia, 31);
                    runb += __shfl_sync(0xffffffffu, ib, 31);
                }
                uint32_t mm = lane < UW ? s_mw[lane] : 0;
                for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
                if (lane == 0) {
                    s_out[0] = runa;
                    s_out[1] = runb;
                    s_out[2] = mm;
                }
            }
            named_bar(BAR_U, UT);
            mark(9);
            const unsigned below = (1u << lane) - 1u;
            for (uint32_t m = 0; m < MC; ++m) {
                const uint32_t j = tid + m * UT;
                const unsigned bal = s_spk[m * UW + warp];
                if ((bal >> lane) & 1u) {
                    const int na_here = static_cast<int>(na) - static_cast<int>(m * UT + warp * 32);
                    const unsigned amask = na_here >= 32 ? 0xffffffffu : (na_here <= 0 ? 0u : (1u << na_here) - 1u);
                    if (j < na)
                        qslot[alo + s_sa[m * UW + warp] + __popc(bal & amask & below)] = id_of(j);
                    else
                        qslot[blo + s_sb[m * UW + warp] + __popc(bal & ~amask & below)] = id_of(j);
                }
            }
            const uint32_t outa = s_out[0], outb = s_out[1], meas = s_out[2];
            named_bar(BAR_U, UT);  // piece slices complete (and s_out / s_s* reusable)
            if (tid == 0) {
                st_release_gpu(ps.finfo + static_cast<uint64_t>(slot) * ps.E + c, frame_word(t, outa, outb));
                if (outa + outb) atomicAdd(&ps.step_spikes[s], outa + outb);
                if (meas) atomicAdd(&ps.step_meas[s], meas);
                my_spikes += outa + outb;
            }
            mark(P_PUBLISH);
        }
        named_bar(BAR_U, UT);
        // fold the last delivered frame (rel nsteps) into ACC
        wait_at_least(&s_delivered, nrel);
        const uint32_t* cl = ring + (nrel % R) * ps.K * ps.win_cap;
        for (uint32_t j = tid; j < na; j += UT) {
            uint32_t a[kMaxClasses];
            bool any = false;
            for (int k = 0; k < ps.K; ++k) {
                a[k] = cl[k * ps.win_cap + j];
                any |= a[k] != 0;
            }
            if (any) {
                auto* accp = &ps.nf.template get<ACC>()[alo + j];
                *accp = fold_frame(ps, *accp, a);
            }
        }
        if (tid == 0 && my_spikes) atomicAdd(&ps.counters[C_SPIKES], my_spikes);
        if (profiling) s_prof[P_STEPS] = static_cast<unsigned long long>(nsteps);
    } else if (NPT != 0 && warp < static_cast<uint32_t>(UW)) {
        // ============================================ update warps
        const uint32_t lead = min(ps.lead, ps.delay);
        values_t<NF> v[NPT > 0 ? NPT : 1];
        xorshift rr[NPT > 0 ? NPT : 1];
        bool live[NPT > 0 ? NPT : 1];
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            live[r] = false;
            const uint32_t j = tid + r * UT;
            if (j < na + nb) load_all(ps.nf, id_of(j), v[r]);
        }
        // per register slot: lanes of this (warp, r) in the A piece (a lane
        // prefix), whether this lane's neuron exists / is measured, its id
        unsigned amask[NPT > 0 ? NPT : 1];
        bool inmeas[NPT > 0 ? NPT : 1];
        uint32_t ids[NPT > 0 ? NPT : 1];
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            const int na_here = static_cast<int>(na) - static_cast<int>(warp * 32 + r * UT);
            amask[r] = na_here >= 32 ? 0xffffffffu : (na_here <= 0 ? 0u : (1u << na_here) - 1u);
            const uint32_t j = tid + r * UT;
            ids[r] = j < na + nb ? id_of(j) : 0u;
            inmeas[r] = j < na + nb && ids[r] >= ps.meas_lo && ids[r] < ps.meas_hi;
        }
        const unsigned below = (1u << lane) - 1u;
        unsigned long long my_spikes = 0;
        uint32_t slot = static_cast<uint32_t>(t0 % ps.Q);
        for (uint32_t s = 0; s < nrel; ++s, slot = slot + 1 == ps.Q ? 0u : slot + 1) {
            const int64_t t = t0 + s;
            uint32_t* qslot = ps.queue + static_cast<uint64_t>(slot) * ps.n;
            // frames through rel s (needed) and s + delay - lead (pacing);
            // never beyond rel s + R - 1, whose ring slot this step frees
            // (one warp polls; the others wait on the hardware barrier, which
            // costs no issue slots; the barrier orders the acquire before
            // every update thread's ring reads)
            if (warp == 0) wait_at_least(&s_delivered, min(min(s + ps.delay - lead, s + R - 1), nrel));
            named_bar(BAR_U, UT);
            mark(P_POLL);
            uint32_t* cslot = ring + (s % R) * ps.K * ps.win_cap;
            bool spk[NPT > 0 ? NPT : 1];
            unsigned bal[NPT > 0 ? NPT : 1];
            uint32_t mcount = 0;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                const uint32_t j = tid + r * UT;
                spk[r] = false;
                if (j < na + nb) {
                    const uint32_t i = ids[r];
                    if (j < na) {  // receiving neuron: fold frame rel s in class order
                        uint32_t a[kMaxClasses];
#pragma unroll
                        for (int k = 0; k < kMaxClasses; ++k) {
                            a[k] = k < ps.K ? cslot[k * ps.win_cap + j] : 0u;
                            if (a[k]) cslot[k * ps.win_cap + j] = 0;
                        }
                        detail::pack_get<ACC>::get(v[r]) = fold_frame(ps, detail::pack_get<ACC>::get(v[r]), a);
                    }
                    values_t<NF> vl = v[r];
                    xorshift rl = rr[r];
                    bool ll = live[r];
                    local_neuron<NF> ref{i, &vl, &rl, &ll, ps.rng};
                    spk[r] = model.update(ref, ps.dt);
                    v[r] = vl;
                    rr[r] = rl;
                    live[r] = ll;
                }
                bal[r] = __ballot_sync(0xffffffffu, spk[r]);
                mcount += __popc(__ballot_sync(0xffffffffu, spk[r] && inmeas[r]));
                if (lane == 0) {
                    s_wa[r * UW + warp] = __popc(bal[r] & amask[r]);
                    s_wb[r * UW + warp] = __popc(bal[r] & ~amask[r]);
                }
            }
            if (lane == 0) s_mw[warp] = mcount;
            mark(P_UPDATE);
            named_bar(BAR_U, UT);  // counts and the slot zeroing are complete
            mark(8);
            if (tid == 0) st_release_cta(&s_updated, s + 1);
            if (warp == 0) {  // exclusive scans of the per-warp counts, ascending local index
                uint32_t runa = 0, runb = 0;
#pragma unroll
                for (int r = 0; r < NPT; ++r) {
                    const uint32_t xa = lane < UW ? s_wa[r * UW + lane] : 0;
                    const uint32_t xb = lane < UW ? s_wb[r * UW + lane] : 0;
                    uint32_t ia = xa, ib = xb;
#pragma unroll
                    for (int o = 1; o < UW; o <<= 1) {
                        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
                        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
                        if (lane >= static_cast<uint32_t>(o)) {
                            ia += ya;
                            ib += yb;
                        }
                    }
                    if (lane < UW) {
                        s_wa[r * UW + lane] = runa + ia - xa;
                        s_wb[r * UW + lane] = runb + ib - xb;
                    }
                    runa += __shfl_sync(0xffffffffu, ia, UW - 1);
                    runb += __shfl_sync(0xffffffffu, ib, UW - 1);
                }
                uint32_t mm = lane < UW ? s_mw[lane] : 0;
                for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
                if (lane == 0) {
                    s_out[0] = runa;
                    s_out[1] = runb;
                    s_out[2] = mm;
                }
            }
            named_bar(BAR_U, UT);
            mark(9);
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                if (spk[r]) {
                    if ((amask[r] >> lane) & 1u)
                        qslot[alo + s_wa[r * UW + warp] + __popc(bal[r] & amask[r] & below)] = ids[r];
                    else
                        qslot[blo + s_wb[r * UW + warp] + __popc(bal[r] & ~amask[r] & below)] = ids[r];
                }
            }
            const uint32_t outa = s_out[0], outb = s_out[1], meas = s_out[2];
            named_bar(BAR_U, UT);  // piece slices complete (and s_out / s_w* reusable)
            if (tid == 0) {
                st_release_gpu(ps.finfo + static_cast<uint64_t>(slot) * ps.E + c, frame_word(t, outa, outb));
                if (outa + outb) atomicAdd(&ps.step_spikes[s], outa + outb);
                if (meas) atomicAdd(&ps.step_meas[s], meas);
                my_spikes += outa + outb;
            }
            // stream the rows of this CTA's spikes into L2 for every deliverer
            if (BM && ps.bm_prefetch) {
#pragma unroll
                for (int r = 0; r < NPT; ++r)
                    if (spk[r])
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                         ps.bm + static_cast<uint64_t>(ids[r]) * ps.bm_row4),
                                     "r"(ps.bm_row4 * 16)
                                     : "memory");
            } else if (ps.pf_cap) {
#pragma unroll
                for (int r = 0; r < NPT; ++r) {
                    const uint32_t j = tid + r * UT;
                    if (spk[r]) {
                        const uint2 w = pf[j];
                        const uint32_t bytes = w.y > w.x ? ((w.y - w.x) * 4 + 15) & ~15u : 0;
                        if (bytes)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                             ps.cells + static_cast<uint64_t>(id_of(j)) * ps.pitch + w.x),
                                         "r"(bytes)
                                         : "memory");
                        // ... and its receive windows (split row), read by every deliverer
                        const uint64_t s0 = static_cast<uint64_t>(id_of(j)) * (C + 1) * 4;
                        const uint64_t a0 = s0 & ~15ull, a1 = (s0 + (C + 1) * 4 + 15) & ~15ull;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                         reinterpret_cast<const char*>(ps.split) + a0),
                                     "r"(static_cast<uint32_t>(a1 - a0))
                                     : "memory");
                    }
                }
            }
            mark(P_PUBLISH);
        }
        named_bar(BAR_U, UT);
        // write back the register-resident state; fold the last delivered
        // frame (rel nsteps) into ACC so host reads and the next launch see it
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
            const uint32_t j = tid + r * UT;
            if (j >= na + nb) continue;
            if (j < na) {
                wait_at_least(&s_delivered, nrel);
                const uint32_t* cslot = ring + (nrel % R) * ps.K * ps.win_cap;
                uint32_t a[kMaxClasses];
#pragma unroll
                for (int k = 0; k < kMaxClasses; ++k) a[k] = k < ps.K ? cslot[k * ps.win_cap + j] : 0u;
                detail::pack_get<ACC>::get(v[r]) = fold_frame(ps, detail::pack_get<ACC>::get(v[r]), a);
            }
            const uint32_t i = id_of(j);
            store_all(ps.nf, i, v[r]);
            if constexpr (model_uses_rng<M>())
                if (live[r]) ps.rng[i] = rr[r];
        }
        if (tid == 0 && my_spikes) atomicAdd(&ps.counters[C_SPIKES], my_spikes);
        if (profiling) s_prof[P_STEPS] = static_cast<unsigned long long>(nsteps);
    } else if (BM && ps.stream_mode) {
        // ============================================ delivery warps (bitmap, streamed)
        // No passes and no group barriers.  Warp 0 (poller) claims complete
        // frames in order into a table of FT slots (piece prefix, queue /
        // ring bases) and appends each frame's blocks of 32 spikes to a
        // linear work space; the other warps take work items with one shared
        // atomic and count each block independently: piece search, spike
        // ids, receive windows straight into registers, warp bit-transposes,
        // conflict-free shared atomics.  The poller releases frames in order
        // once all their blocks are counted.
        constexpr uint32_t FT = MB;
        const uint32_t dwarp = warp - UW;
        unsigned long long my_deliv = 0;
        const bool log_cta = ps.log && c == 0;
        const uint32_t WQ = ps.wq;
        const tp_consts tpk = make_tp_consts(lane);
        const uint4* bmw = ps.bm + static_cast<uint64_t>(c) * WQ;
        uint32_t r_first = 1;
        if (fbase + 1 < 0) r_first = static_cast<uint32_t>(min(-1 - fbase, static_cast<int64_t>(nrel))) + 1;
        if (dwarp == 0) {
            // ---------------- poller
            if (r_first > 1 && lane == 0) st_release_cta(&s_delivered, r_first - 1);
            uint32_t r_poll = r_first, r_rel = r_first, wend = 0;
            unsigned long long lc = 0;
            bool total_set = false;
            while (r_rel <= nrel) {
                bool progress = false;
                // release counted frames in order
                while (r_rel < r_poll) {
                    const uint32_t sl = r_rel % FT;
                    if (ld_acquire_cta(&s_ft_done[sl]) != s_ft_nb[sl]) break;
                    if (lane == 0) st_release_cta(&s_delivered, r_rel);
                    ++r_rel;
                    progress = true;
                }
                // claim the next frame when it is complete and its ring slot free
                if (r_poll <= nrel && r_poll < r_rel + FT && r_poll + 1 <= ld_acquire_cta(&s_updated) + R &&
                    (ps.lag == 0 || frame_complete(ps, fbase + r_poll + ps.lag, false, ps.C))) {
                    const uint32_t sl = r_poll % FT;
                    if (frame_prefix(ps, fbase + r_poll, s_seg[sl], s_fval[0], s_psrc, true)) {
                        const uint32_t S = s_seg[sl][P], nb = (S + 31) / 32;
                        const bool logged = log_cta && fbase + r_poll >= ps.log_from;
                        if (lane == 0) {
                            s_ft_base[sl] = wend;
                            s_ft_nb[sl] = nb;
                            s_ft_S[sl] = S;
                            s_ft_q[sl] = static_cast<uint32_t>((fbase + r_poll) % ps.Q) * ps.n;
                            s_ft_cb[sl] = (r_poll % R) * ps.K * ps.win_cap;
                            s_ft_lb[sl] = logged ? lc : ~0ull;
                            s_ft_done[sl] = 0;
                        }
                        if (logged) {
                            if (lane == 0) ps.log_cnt[fbase + r_poll - ps.log_from] = S;
                            lc += S;
                        }
                        wend += nb;
                        __syncwarp();
                        if (lane == 0) st_release_cta(&s_work_end, wend);
                        ++r_poll;
                        progress = true;
                    }
                }
                if (r_poll > nrel && !total_set) {
                    if (lane == 0) st_release_cta(&s_work_total, wend);
                    total_set = true;
                }
                if (!progress) __nanosleep(32);
            }
            if (!total_set && lane == 0) st_release_cta(&s_work_total, wend);
            if (log_cta && lane == 0) {
                *ps.log_end = lc;
                if (lc > ps.log_cap) ps.flags[0] = 1;
            }
        } else {
            // ---------------- workers
            for (;;) {
                uint32_t item = 0;
                if (lane == 0) item = atomicAdd(&s_work_next, 1u);
                item = __shfl_sync(0xffffffffu, item, 0);
                bool done = false;
                for (;;) {  // wait until the item exists (or the launch has no more work)
                    if (item < ld_acquire_cta(&s_work_end)) break;
                    if (item >= ld_acquire_cta(&s_work_total)) {
                        done = true;
                        break;
                    }
                    __nanosleep(64);
                }
                if (done) break;
                uint32_t sl = 0;
#pragma unroll
                for (uint32_t k = 0; k < FT; ++k) {
                    const uint32_t b0 = s_ft_base[k];
                    if (item >= b0 && item < b0 + s_ft_nb[k] && s_ft_done[k] < s_ft_nb[k]) sl = k;
                }
                const uint32_t S = s_ft_S[sl], blk = item - s_ft_base[sl];
                const uint32_t* seg = s_seg[sl];
                const uint32_t g = blk * 32 + lane;
                const bool valid = g < S;
                uint32_t src = 0, cls = 0xffu;
                if (valid) {
                    const uint32_t a = piece_of(seg, P, g);
                    src = __ldcg(ps.queue + s_ft_q[sl] + s_lo[a] + (g - seg[a]));
                    cls = static_cast<uint32_t>(source_class(ps, src));
                    const unsigned long long lb = s_ft_lb[sl];
                    if (lb != ~0ull && lb + g < ps.log_cap) ps.log[lb + g] = src;
                }
                unsigned cm[kMaxClasses];
#pragma unroll
                for (int k = 0; k < kMaxClasses; ++k) cm[k] = __ballot_sync(0xffffffffu, cls == static_cast<uint32_t>(k));
                uint32_t* rb = ring + s_ft_cb[sl] + lane;
                const uint4* row = bmw + static_cast<uint64_t>(src) * ps.bm_row4;
                for (uint32_t q0 = 0; q0 < WQ; q0 += 4) {
                    uint4 x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        x[u] = (valid && q0 + u < WQ) ? ldg_stream4(row + q0 + u) : make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (q0 + u >= WQ) break;
                        const uint32_t wv[4] = {transpose32(x[u].x, tpk), transpose32(x[u].y, tpk),
                                                transpose32(x[u].z, tpk), transpose32(x[u].w, tpk)};
#pragma unroll
                        for (int k = 0; k < kMaxClasses; ++k) {
                            if (!cm[k]) continue;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const uint32_t cnt = __popc(wv[e] & cm[k]);
                                if (cnt) {
                                    atomicAdd(rb + k * ps.win_cap + ((q0 + u) * 4 + e) * 32, cnt);
                                    my_deliv += cnt;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                __threadfence_block();
                if (lane == 0) atomicAdd(&s_ft_done[sl], 1u);
            }
        }
        for (int o = 16; o; o >>= 1) my_deliv += __shfl_xor_sync(0xffffffffu, my_deliv, o);
        if (lane == 0 && my_deliv) atomicAdd(&ps.counters[C_DELIVERIES], my_deliv);
    } else {
        // ============================================ delivery warps
        const uint32_t dtid = tid - UT, dwarp = warp - UW;
        unsigned long long my_deliv = 0;
        unsigned long long lc = 0;  // CTA 0: log cursor
        const bool log_cta = ps.log && c == 0;
        const uint4* cells4 = reinterpret_cast<const uint4*>(ps.cells);
        const uint32_t pitch4 = ps.pitch >> 2;
        const uint32_t cap = ps.stage_items;
        uint32_t r_next = 1;
        // peer exchange: this CTA exports the frames f = c (mod C) published
        // by this launch, each as soon as its local pieces are complete
        const int64_t last_pub = t0 + nrel - 1;
        int64_t next_exp = t0 + static_cast<int64_t>((c + C - static_cast<uint32_t>(t0 % C)) % C);
        auto try_export = [&]() {
            while (next_exp <= last_pub && frame_complete(ps, next_exp, false, C)) {
                fence_acq_rel_gpu();
                peer_export(ps, next_exp);
                next_exp += C;
            }
        };
        // frames before 0 do not exist: nothing to deliver (engine.hpp:371-380)
        if (fbase + 1 < 0) {
            const int64_t last_neg = -1 - fbase;  // rel of frame -1
            r_next = static_cast<uint32_t>(min(last_neg, static_cast<int64_t>(nrel))) + 1;
            if (dtid == 0) st_release_cta(&s_delivered, r_next - 1);
        }
        while (r_next <= nrel) {
            // ---- poll: warp w takes frame rel r_next + w (warp 0 waits)
            // (frame f is taken once frame f + lag is complete: the
            // publishers streamed the rows of f into L2 meanwhile)
            if (dwarp < min(static_cast<uint32_t>(MB), ps.max_pass)) {
                const uint32_t r = r_next + dwarp;
                bool ok = false;
                if (dwarp == 0 && ps.npeers) {
                    // the same waits, spinning: the exports of this CTA's
                    // frames may not wait behind the remote part of frame r
                    for (;;) {
                        if (ps.progress && lane == 0) {
                            volatile uint32_t* w = ps.progress + 8 * c;
                            w[0] = r;
                            w[1] = static_cast<uint32_t>(next_exp - t0);
                            w[2] = ld_acquire_cta(&s_updated);
                            w[3] = ld_acquire_cta(&s_delivered);
                            w[4] = 1;
                        }
                        try_export();
                        if (r >= R && ld_acquire_cta(&s_updated) < r - R + 1) continue;
                        if (ps.lag && !frame_complete(ps, fbase + r + ps.lag, false, ps.C)) continue;
                        if (frame_prefix(ps, fbase + r, s_seg[0], s_fval[0], s_psrc, true)) break;
                    }
                    if (profiling) mark(6);
                    ok = true;
                } else if (dwarp == 0) {
                    // ring slot r % R is free once update step r - R folded it
                    if (r >= R) wait_at_least(&s_updated, r - R + 1);
                    if (ps.lag) frame_complete(ps, fbase + r + ps.lag, true, ps.C);  // local publishers only
                    if (profiling) mark(6);
                    ok = frame_prefix(ps, fbase + r, s_seg[0], s_fval[0], s_psrc, false);
                } else if (r <= nrel && r + 1 <= ld_acquire_cta(&s_updated) + R &&
                           (ps.lag == 0 || frame_complete(ps, fbase + r + ps.lag, false, ps.C))) {
                    ok = frame_prefix(ps, fbase + r, s_seg[dwarp], s_fval[dwarp], s_psrc, true);
                }
                if (lane == 0) {
                    s_ok[dwarp] = ok ? 1u : 0u;
                    s_qbase[dwarp] = static_cast<uint32_t>((fbase + r) % ps.Q) * ps.n;
                    s_cbase[dwarp] = (r % R) * ps.K * ps.win_cap;
                }
            }
            named_bar(BAR_D, DT);
            if (profiling) mark(10);
            uint32_t B = 0;
            uint32_t fpre[MB + 1];
            fpre[0] = 0;
#pragma unroll
            for (int w = 0; w < MB; ++w) {
                const bool take = (static_cast<uint32_t>(w) == B) && s_ok[w] && static_cast<uint32_t>(w) < ps.max_pass;
                if (take) ++B;
                fpre[w + 1] = fpre[w] + (take ? s_seg[w][P] : 0u);
            }
            const uint32_t S = fpre[B];
            // CTA 0 logs the frames >= log_from of this pass, in order
            uint32_t wlog = B;
            if (log_cta) {
                const int64_t d = ps.log_from - (fbase + r_next);
                wlog = d <= 0 ? 0u : static_cast<uint32_t>(min(d, static_cast<int64_t>(B)));
            }
            uint32_t flog = 0;
#pragma unroll
            for (int q = 1; q <= MB; ++q)
                if (static_cast<uint32_t>(q) == wlog) flog = fpre[q];
            const unsigned long long lbase = lc - flog;
            if (log_cta && dtid == 0)
                for (uint32_t w = wlog; w < B; ++w) ps.log_cnt[fbase + r_next + w - ps.log_from] = s_seg[w][P];
            if constexpr (BM) {
                // ---- bitmap delivery: per spike, this CTA's receive window is
                // WQ x 128 bits of the spike's bitmap row.  Stage the windows of
                // the pass in shared memory, then count arrivals per (frame,
                // class, target) with warp bit-transposes + popc: one counting
                // atomic per 32 targets x 32 spikes instead of one per delivery.
                const uint32_t WQ = ps.wq, wq_sh = WQ == 1 ? 0u : (WQ == 2 ? 1u : (WQ == 4 ? 2u : 3u));
                const tp_consts tpk = make_tp_consts(lane);
                uint4* sw = reinterpret_cast<uint4*>(chunks);  // cap x WQ, 16-byte slots swizzled
                uint32_t* s_src = reinterpret_cast<uint32_t*>(sw + cap * WQ);
                uint8_t* s_grp = reinterpret_cast<uint8_t*>(s_src + cap);
                const uint32_t swz_sh = WQ == 2 ? 2u : (WQ == 4 ? 1u : 0u);
                const uint32_t swz_m = WQ == 1 ? 0u : (WQ == 2 ? 1u : (WQ == 4 ? 3u : 7u));
                const uint4* bmw = ps.bm + static_cast<uint64_t>(c) * WQ;
                for (uint32_t g0 = 0; g0 < S; g0 += cap) {
                    const uint32_t n = min(cap, S - g0);
                    // (1)+(2) per warp and 32 pass positions: lane L loads the
                    // spike id of position i0 + L (its frame by the pass
                    // prefix, its piece by binary search over the frame's
                    // piece prefix; L2 loads, the slices were acquired with
                    // the frame words), records its (frame, class) group, and
                    // the warp then issues the spikes' windows (16-byte
                    // cp.async.cg, 32 / WQ spikes x WQ columns per
                    // instruction, ids by shuffle) right away: no wait or
                    // barrier between the id and the window of a spike
                    const uint32_t spi = 32u >> wq_sh;  // spikes per window instruction
                    const bool stage = (ps.dbg & 2) == 0;
                    constexpr int kIdU = 4;  // id loads in flight per lane before their windows
                    for (uint32_t b0 = dwarp * 32; b0 < n; b0 += DW * 32 * kIdU) {
                        uint32_t srcv[kIdU];
#pragma unroll
                        for (int k = 0; k < kIdU; ++k) {
                            const uint32_t i = b0 + k * DW * 32 + lane;
                            srcv[k] = 0;
                            if (i < n) {
                                const uint32_t g = g0 + i;
                                uint32_t w = 0;
#pragma unroll
                                for (int q = 1; q < MB; ++q)
                                    if (static_cast<uint32_t>(q) < B && fpre[q] <= g) w = q;
                                const uint32_t gl = g - fpre[w];
                                const uint32_t* seg = s_seg[w];
                                const uint32_t a = piece_of(seg, P, gl);
                                srcv[k] = __ldcg(ps.queue + s_qbase[w] + s_lo[a] + (gl - seg[a]));
                                s_grp[i] = static_cast<uint8_t>(w);
                            }
                        }
#pragma unroll
                        for (int k = 0; k < kIdU; ++k) {
                            const uint32_t i0 = b0 + k * DW * 32, i = i0 + lane;
                            if (i0 >= n) break;
                            const uint32_t src = srcv[k];
                            if (i < n) {
                                const uint32_t w = s_grp[i];
                                s_src[i] = src;
                                if (w >= wlog && lbase + g0 + i < ps.log_cap) ps.log[lbase + g0 + i] = src;
                                s_grp[i] = static_cast<uint8_t>(w * 4 + static_cast<uint32_t>(source_class(ps, src)));
                            }
                            if (stage) {
                                for (uint32_t j = 0; j < WQ; ++j) {
                                    const uint32_t sl = j * spi + (lane >> wq_sh), q = lane & (WQ - 1);
                                    const uint32_t sid = __shfl_sync(0xffffffffu, src, sl);
                                    const uint32_t gg = i0 + sl;
                                    if (gg < n)
                                        cp_async16_cg(sw + gg * WQ + (q ^ ((gg >> swz_sh) & swz_m)),
                                                      bmw + static_cast<uint64_t>(sid) * ps.bm_row4 + q);
                                }
                            }
                        }
                    }
                    if (profiling) mark(P_GATHER);
                    cp_async_wait_all();
                    named_bar(BAR_D, DT);
                    if (profiling) mark(11);
                    // (3) count.  Unit = (group G = frame * 4 + class, 16-byte
                    // column q): the spikes of one group are contiguous in
                    // the pass, so a unit owns its counters (no atomics),
                    // accumulates popcounts of the transposed 32-spike blocks
                    // in registers and adds them to the ring once.
                    for (uint32_t i = dtid; i < n; i += DT) {  // group boundaries
                        const uint32_t G = s_grp[i];
                        if (i == 0 || s_grp[i - 1] != G) s_gbeg[G] = i;
                        if (i + 1 == n || s_grp[i + 1] != G) s_gend[G] = i + 1;
                    }
                    named_bar(BAR_D, DT);
                    // work items = (chunk of <= 7 blocks of one group, column):
                    // groups differ ~5x in size, equal chunks keep the warps
                    // balanced; chunks of one (group, column) add with
                    // conflict-free shared atomics
                    if (dwarp == 0) {
                        const uint32_t gb = s_gbeg[lane], ge = s_gend[lane];
                        const uint32_t nb = ge > gb ? ((ge + 31) >> 5) - (gb >> 5) : 0u;
                        const uint32_t nc = (nb + 6) / 7;
                        const uint32_t inc = warp_incl_scan(nc);
                        s_gcp[lane] = inc - nc;
                        if (lane == 31) s_gcp[32] = inc;
                    }
                    named_bar(BAR_D, DT);
                    const uint32_t nwork = (ps.dbg & 2) ? 0u : s_gcp[32] << wq_sh;
                    for (uint32_t it = dwarp; it < nwork; it += DW) {
                        const uint32_t q = it & (WQ - 1), ci = it >> wq_sh;
                        uint32_t G = 0;  // last group with s_gcp[G] <= ci
#pragma unroll
                        for (uint32_t step = 16; step; step >>= 1)
                            if (s_gcp[G + step] <= ci) G += step;
                        const uint32_t gb = s_gbeg[G], ge = s_gend[G];
                        const uint32_t blk = (gb >> 5) + 7 * (ci - s_gcp[G]);
                        const uint32_t take = min(7u, ((ge + 31) >> 5) - blk);
                        uint32_t cnt[4] = {0, 0, 0, 0};
                        if (take >= 3) {
                            // bit-sliced sum of the blocks per lane (3 planes),
                            // then one transpose per plane
                            uint32_t p0[4] = {0, 0, 0, 0}, p1[4] = {0, 0, 0, 0}, p2[4] = {0, 0, 0, 0};
                            for (uint32_t v = 0; v < take; ++v) {
                                const uint32_t gs = (blk + v) * 32 + lane;
                                const bool in = gs >= gb && gs < ge;
                                const uint4 x = in ? sw[gs * WQ + (q ^ ((gs >> swz_sh) & swz_m))] : make_uint4(0, 0, 0, 0);
                                const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const uint32_t c0 = p0[e] & wv[e];
                                    p0[e] ^= wv[e];
                                    const uint32_t c1 = p1[e] & c0;
                                    p1[e] ^= c0;
                                    p2[e] ^= c1;  // at most 7 blocks: no carry out of plane 2
                                }
                            }
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                cnt[e] = __popc(transpose32(p0[e], tpk)) + (__popc(transpose32(p1[e], tpk)) << 1) +
                                         (__popc(transpose32(p2[e], tpk)) << 2);
                        } else {
                            for (uint32_t v = 0; v < take; ++v) {
                                const uint32_t gs = (blk + v) * 32 + lane;
                                const bool in = gs >= gb && gs < ge;
                                const uint4 x = in ? sw[gs * WQ + (q ^ ((gs >> swz_sh) & swz_m))] : make_uint4(0, 0, 0, 0);
                                cnt[0] += __popc(transpose32(x.x, tpk));
                                cnt[1] += __popc(transpose32(x.y, tpk));
                                cnt[2] += __popc(transpose32(x.z, tpk));
                                cnt[3] += __popc(transpose32(x.w, tpk));
                            }
                        }
                        uint32_t* cb = ring + s_cbase[G >> 2] + (G & 3u) * ps.win_cap + q * 128 + lane;
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (cnt[e]) atomicAdd(cb + e * 32, cnt[e]);
                        my_deliv += cnt[0] + cnt[1] + cnt[2] + cnt[3];
                    }
                    named_bar(BAR_D, DT);
                    for (uint32_t i = dtid; i < 32; i += DT) {  // reset the group table
                        s_gbeg[i] = 0;
                        s_gend[i] = 0;
                    }
                    named_bar(BAR_D, DT);  // counts complete, staging reusable
                    if (profiling) mark(P_DELIVER);
                }
            } else {
                for (uint32_t g0 = 0; g0 < S; g0 += DT * kEllSpt) {
                    // kEllSpt spikes per thread (loads of all of them in
                    // flight together): id, this CTA's row window, chunks
                    uint32_t nch[kEllSpt], sbv[kEllSpt], sev[kEllSpt], basev[kEllSpt], srcv[kEllSpt];
                    uint32_t nchunk = 0;
#pragma unroll
                    for (int u = 0; u < kEllSpt; ++u) {
                        const uint32_t g = g0 + u * DT + dtid;
                        srcv[u] = 0xffffffffu;
                        basev[u] = 0;
                        if (g < S) {
                            uint32_t w = 0, fw = 0;
#pragma unroll
                            for (int q = 1; q < MB; ++q)
                                if (static_cast<uint32_t>(q) < B && fpre[q] <= g) {
                                    w = q;
                                    fw = fpre[q];
                                }
                            const uint32_t gl = g - fw;
                            const uint32_t* seg = s_seg[w];
                            const uint32_t a = piece_of(seg, P, gl);
                            srcv[u] = __ldcg(ps.queue + s_qbase[w] + s_lo[a] + (gl - seg[a]));
                            basev[u] = s_cbase[w];
                            if (w >= wlog && lbase + g < ps.log_cap) ps.log[lbase + g] = srcv[u];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kEllSpt; ++u) {
                        sbv[u] = sev[u] = 0;
                        if (srcv[u] != 0xffffffffu) {
                            const uint32_t* sp = ps.split + static_cast<uint64_t>(srcv[u]) * (C + 1) + c;
                            sbv[u] = __ldg(sp);
                            sev[u] = __ldg(sp + 1);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kEllSpt; ++u) {
                        nch[u] = sev[u] > sbv[u] ? ((sev[u] + 3) >> 2) - (sbv[u] >> 2) : 0;
                        nchunk += nch[u];
                        my_deliv += sev[u] - sbv[u];
                        if (srcv[u] != 0xffffffffu)
                            basev[u] += static_cast<uint32_t>(source_class(ps, srcv[u])) * ps.win_cap;
                    }
                    uint32_t total;
                    const uint32_t first = group_exclusive_scan<DT, UW, BAR_D>(nchunk, s_dtmp, total);
                    if (profiling) mark(P_GATHER);
                    for (uint32_t i0 = 0; i0 < total; i0 += cap) {
                        // chunk list: {16-byte chunk index, ring base << 5 | hi << 2 | lo}
                        uint32_t off = first;
#pragma unroll
                        for (int u = 0; u < kEllSpt; ++u) {
                            const uint32_t sb = sbv[u], se = sev[u], row4 = srcv[u] * pitch4, base = basev[u];
                            for (uint32_t q = 0; q < nch[u]; ++q) {
                                const uint32_t it = off + q;
                                if (it < i0 || it >= i0 + cap) continue;
                                const uint32_t w0 = ((sb >> 2) + q) << 2;  // first word of the chunk
                                const uint32_t lo = sb > w0 ? sb - w0 : 0;
                                const uint32_t hi = min(4u, se - w0);
                                chunks[it - i0] = make_uint2(row4 + (sb >> 2) + q, (base << 5) | (hi << 2) | lo);
                            }
                            off += nch[u];
                        }
                        named_bar(BAR_D, DT);
                        if (profiling) mark(11);
                        const uint32_t m = min(cap, total - i0);
                        for (uint32_t k0 = dtid; k0 < m; k0 += kChunkBatch * DT) {
                            uint2 d[kChunkBatch];
                            uint4 x[kChunkBatch];
    #pragma unroll
                            for (int u = 0; u < kChunkBatch; ++u) {
                                const uint32_t k = k0 + u * DT;
                                d[u] = k < m ? chunks[k] : make_uint2(0, 0);
                            }
    #pragma unroll
                            for (int u = 0; u < kChunkBatch; ++u)
                                x[u] = d[u].y ? ldg_stream4(cells4 + d[u].x) : make_uint4(0, 0, 0, 0);
    #pragma unroll
                            for (int u = 0; u < kChunkBatch; ++u) {
                                const uint32_t lo = d[u].y & 3u, hi = (d[u].y >> 2) & 7u;
                                uint32_t* cb = ring + (d[u].y >> 5) - alo;
                                if (lo == 0 && hi > 0) atomicAdd(cb + x[u].x, 1u);
                                if (lo <= 1 && hi > 1) atomicAdd(cb + x[u].y, 1u);
                                if (lo <= 2 && hi > 2) atomicAdd(cb + x[u].z, 1u);
                                if (hi > 3) atomicAdd(cb + x[u].w, 1u);
                            }
                        }
                        named_bar(BAR_D, DT);
                    }
                    if (profiling) mark(P_DELIVER);
                }
            }
            if (wlog < B) lc = lbase + S;
            // every counting atomic of the pass precedes the release (barrier)
            if (S == 0) named_bar(BAR_D, DT);
            if (dtid == 0) st_release_cta(&s_delivered, r_next + B - 1);
            if (profiling) s_prof[7] += 1;
            r_next += B;
        }
        if (dwarp == 0 && ps.npeers)  // the rest of this launch's frames (local completion only)
            while (next_exp <= last_pub) {
                if (ps.progress && lane == 0) {
                    ps.progress[8 * c + 1] = static_cast<uint32_t>(next_exp - t0);
                    ps.progress[8 * c + 4] = 2;
                }
                frame_complete(ps, next_exp, true, C);
                fence_acq_rel_gpu();
                peer_export(ps, next_exp);
                next_exp += C;
            }
        for (int o = 16; o; o >>= 1) my_deliv += __shfl_xor_sync(0xffffffffu, my_deliv, o);
        if (lane == 0 && my_deliv) atomicAdd(&ps.counters[C_DELIVERIES], my_deliv);
        if (log_cta && dtid == 0) {
            *ps.log_end = lc;
            if (lc > ps.log_cap) ps.flags[0] = 1;
        }
    }
    __syncthreads();
    if (ps.prof != nullptr && tid < P_SLOTS) atomicAdd(&ps.prof[c * P_SLOTS + tid], s_prof[tid]);
}

}  // namespace synq::dev
