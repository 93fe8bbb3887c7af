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
//   into the piece's slice of queue slot t % Q and release-stores one word
//   {t+1, count of its low piece, count of its high piece} into
//   finfo[slot][cta].  Pieces are numbered in id order,
//   so concatenating their slices gives the sorted frame.  Receive(t)
//   consumes frame t-delay+1, finished by every CTA delay-1 steps earlier: the
//   only cross-CTA wait is an acquire-poll that is normally satisfied at once.
//   With Q = 2*delay slots no slot is rewritten while a slower CTA may still
//   read it (a CTA runs at most delay-1 steps ahead of the slowest).
// * Delivery.  The row segment of spike s inside A_c is
//   [split[s][c], split[s][c+1]) of the sorted ELL row.  Segments are cut
//   into 32-target items, copied global -> shared with cp.async (LDGSTS: no
//   registers held in flight, one latency round per frame) and counted per
//   (target, source class) with native shared-memory atomics.  The update re-adds fl(c*w_k) count_k times in ascending class
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

constexpr int kPersistThreads = 512;
constexpr int kMaxTiles = 160;             // publishers: local CTAs (<= 148 SMs) + remote shards
constexpr int kMaxPieces = 2 * kMaxTiles;  // id-ordered pieces
constexpr int kMaxClasses = 4;
constexpr int kChunkBatch = 8;  // 16-byte row chunks in flight per lane during delivery

enum prof_slot : int { P_UPDATE = 0, P_PUBLISH, P_POLL, P_GATHER, P_DELIVER, P_STEPS, P_SLOTS = 16 };
// pipelined kernel only: 6 delivery wait for frames, 7 delivery passes,
// 8 update first barrier, 9 update scan, 10 delivery frame prefixes,
// NVLink peer exchange (engine_options::shard_peer): the step kernel stores
// this shard's frames straight into every other shard's queue ring and its
// publisher word there (peer-mapped memory), so a sharded run needs no host
// exchange between launches
struct peer_link {
    uint32_t* queue;            // the peer's Q x n queue ring
    unsigned long long* finfo;  // the peer's Q x E frame words
    uint32_t E;                 // the peer's publisher count
    uint32_t entry;             // this shard's publisher entry there
};
constexpr int kMaxPeers = 32;

// 11 delivery chunk list

template <class M>
struct persist_state {
    using NF = typename M::neuron_fields;
    field_ptrs<NF> nf;
    xorshift* rng;
    const uint32_t* cells;
    const uint32_t* degree;     // [n] out-degrees (k_solo)
    const uint32_t* split;      // [n][C+1]: receive-window boundaries of the CTAs
    const uint32_t* piece_lo;   // [P+1] piece boundaries in id order
    const uint32_t* cta_piece;  // [2C]: (A piece, B piece) of every local CTA
    const uint32_t* piece_src;  // [P]: publisher entry << 1 | half (0: bits 16..31 = A, 1: bits 0..15 = B)
    uint32_t pitch, n, C, P, E;  // local CTAs, pieces, publishers (C local CTAs + remote shards)
    uint32_t* queue;            // Q slots x n ids
    unsigned long long* finfo;  // Q x E frame words, see frame_word()
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
    uint32_t* log_cnt;            // out: ids logged per frame, index f - log_from (the
                                  // merged frame of every publisher, remote ranks included)
    unsigned long long log_cap;
    int64_t log_from;
    uint32_t* flags;
    uint32_t win_cap;          // count-window capacity per class (smem), >= max |A_c|
    uint32_t stage_items;      // 32-target items staged in smem per delivery pass
    unsigned long long* prof;  // optional per-CTA phase cycle counters (P_SLOTS each)
    // pipelined engine (pipeline.cuh)
    uint32_t R;       // count-ring slots (frames in flight between delivery and update)
    uint32_t lead;    // update runs at most this many frames ahead of local delivery
    uint32_t pf_cap;  // row-prefetch windows held in smem (0: no L2 row prefetch)
    uint32_t lag;     // frame f is delivered once frame f + lag is complete (its rows are in L2)
    // bitmap delivery: row s = C windows of wq uint4 (bits of targets window_lo + k)
    const uint4* bm;
    uint32_t bm_row4;      // uint4 per bitmap row (= C * wq)
    uint32_t wq;           // uint4 per window (1, 2, 4 or 8)
    uint32_t bm_prefetch;  // stream the bitmap rows of published spikes into L2
    uint32_t stream_mode;  // bitmap delivery: barrier-free work items instead of passes
    uint32_t max_pass;     // frames per delivery pass (<= the polling warps)
    uint32_t dbg;          // timing experiments only (SYNQ_DBG): bit 1 = bitmap passes skip staging + counting
    // peer exchange: every other shard's ring (npeers = 0: none); this
    // shard's A / B id ranges start at a_lo / b_lo
    const peer_link* peers;
    uint32_t npeers;
    uint32_t a_lo, b_lo;
    volatile uint32_t* progress;  // SYNQ_WATCHDOG: 8 words per CTA, host-mapped
    // fold table (k_fold_table): tab[n0 * (T1 + 1) + n1] = fl-sum from +0 of
    // n0 copies of delta[0] then n1 copies of delta[1]; nullptr: no table
    const float* fold_tab;
    uint32_t fold_t0, fold_t1;
};

// streaming 16-byte read of adjacency cells: read-only, no L1 allocation
SYNQ_DEV uint4 ldg_stream4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
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
SYNQ_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
SYNQ_DEV void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SYNQ_DEV void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

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
#pragma unroll 1
    for (; n >= 4; n -= 4) {
        acc = acc + d;
        acc = acc + d;
        acc = acc + d;
        acc = acc + d;
    }
#pragma unroll 1
    for (; n; --n) acc = acc + d;
    return acc;
}

// the fold table: entry (n0, n1) is the reference's sequential float sum
// starting from +0, n0 additions of d0 followed by n1 of d1 (K == 1: t1 = 0).
// Built on the device with the same additions as fold_arrivals.
__global__ void k_fold_table(float d0, float d1, uint32_t t0, uint32_t t1, float* tab) {
    for (uint32_t n0 = blockIdx.x * blockDim.x + threadIdx.x; n0 <= t0; n0 += gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (uint32_t k = 0; k < n0; ++k) acc = acc + d0;
        for (uint32_t n1 = 0; n1 <= t1; ++n1) {
            tab[n0 * (t1 + 1) + n1] = acc;
            acc = acc + d1;
        }
    }
}

// fold one frame's arrival counts a[0..K) into acc in class order.  When acc
// is zero (the LIF models reset it every step) and the table covers them, the
// first two classes are one table read: for d != 0, (+-0) + d == d, so the
// sequence from either zero is the table's (a zero count leaves acc alone).
template <class M>
SYNQ_DEV float fold_frame(const persist_state<M>& ps, float acc, const uint32_t* a) {
    int k0 = 0;
    if (ps.fold_tab && acc == 0.0f && (a[0] | (ps.K > 1 ? a[1] : 0u))) {
        uint32_t n0 = a[0], n1 = ps.K > 1 ? a[1] : 0u;
        if (n0 <= ps.fold_t0) {
            const uint32_t m1 = min(n1, ps.fold_t1);
            acc = __ldg(ps.fold_tab + n0 * (ps.fold_t1 + 1) + m1);
            acc = fold_arrivals(acc, n1 - m1, ps.delta[1 % kMaxClasses]);
            k0 = 2;
        } else {
            acc = __ldg(ps.fold_tab + ps.fold_t0 * (ps.fold_t1 + 1));
            acc = fold_arrivals(acc, n0 - ps.fold_t0, ps.delta[0]);
            k0 = 1;
        }
    }
#pragma unroll
    for (int k = 0; k < kMaxClasses; ++k)
        if (k >= k0 && k < ps.K && a[k]) acc = fold_arrivals(acc, a[k], ps.delta[k]);
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

// A published frame word: the 16-bit tag (f+1) (unambiguous because the
// ring holds Q << 65536 frames) and the publisher's A / B piece spike counts
// in 24 bits each (a remote shard publishes its whole range as one entry).
SYNQ_HD unsigned long long frame_word(int64_t f, uint32_t ca, uint32_t cb) {
    return (static_cast<unsigned long long>(static_cast<uint32_t>(f + 1) & 0xffffu) << 48) |
           (static_cast<unsigned long long>(ca) << 24) | cb;
}
SYNQ_HD uint32_t frame_tag(int64_t f) { return static_cast<uint32_t>(f + 1) & 0xffffu; }
SYNQ_HD uint32_t word_tag(unsigned long long w) { return static_cast<uint32_t>(w >> 48); }
SYNQ_HD uint32_t word_a(unsigned long long w) { return static_cast<uint32_t>(w >> 24) & 0xffffffu; }
SYNQ_HD uint32_t word_b(unsigned long long w) { return static_cast<uint32_t>(w) & 0xffffffu; }
SYNQ_HD uint32_t word_half(unsigned long long w, uint32_t half) { return half ? word_b(w) : word_a(w); }

// Warp-wide: wait until every publisher (local CTA or remote shard) has
// published frame f (or, when nonblocking, only look), acquire, and write the
// exclusive prefix over the P pieces in id order into seg[0..P] (seg[P] =
// frame size).  fval / psrc: shared scratch (publisher counts) and the piece
// table.  Returns false if nonblocking and the frame is not complete yet.
template <class M>
SYNQ_DEV bool frame_prefix(const persist_state<M>& ps, int64_t f, uint32_t* seg, unsigned long long* fval,
                           const uint32_t* psrc, bool nonblocking) {
    const uint32_t lane = threadIdx.x & 31, E = ps.E, P = ps.P;
    const uint32_t want = frame_tag(f);
    const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(f % ps.Q) * E;
    constexpr int kPer = (kMaxTiles + 31) / 32;
    unsigned long long val[kPer];
    bool ok = true;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const uint32_t j = q * 32 + lane;
        val[q] = (j < E) ? ld_relaxed_gpu(fi + j) : frame_word(f, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const uint32_t j = q * 32 + lane;
        if (nonblocking) {
            ok &= word_tag(val[q]) == want;
        } else {
            while (word_tag(val[q]) != want) {
                __nanosleep(20);
                val[q] = ld_relaxed_gpu(fi + j);
            }
        }
    }
    if (nonblocking && !__all_sync(0xffffffffu, ok)) return false;
    // peer entries were released by another GPU at system scope: acquire them
    // at that scope (the words are complete, this re-read synchronises)
    if (ps.npeers)
        for (uint32_t j = ps.C + lane; j < E; j += 32) (void)ld_acquire_sys(fi + j);
    fence_acq_rel_gpu();  // acquire: the slices are visible to this CTA
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const uint32_t j = q * 32 + lane;
        if (j < E) fval[j] = val[q];
    }
    __syncwarp();
    uint32_t run = 0;
    for (uint32_t p0 = 0; p0 < P; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint32_t cj = 0;
        if (p < P) {
            const uint32_t src = psrc[p];
            cj = word_half(fval[src >> 1], src & 1);
        }
        uint32_t incl = cj;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (p < P) seg[p] = run + incl - cj;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) seg[P] = run;
    __syncwarp();
    return true;
}

// Warp-wide: is frame f published by the first E publishers (blocking:
// wait)?  The local CTAs are publishers 0 .. C-1, remote shards follow.
template <class M>
SYNQ_DEV bool frame_complete(const persist_state<M>& ps, int64_t f, bool blocking, uint32_t E) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t want = frame_tag(f);
    const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(f % ps.Q) * ps.E;
    bool ok = true;
    for (uint32_t j = lane; j < E; j += 32) {
        if (blocking) {
            while (word_tag(ld_relaxed_gpu(fi + j)) != want) __nanosleep(20);
        } else {
            ok &= word_tag(ld_relaxed_gpu(fi + j)) == want;
        }
    }
    return __all_sync(0xffffffffu, ok);
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

    extern __shared__ __align__(16) uint32_t cnt[];  // K x win_cap arrival counters | chunk list
    uint4* chunks = reinterpret_cast<uint4*>(cnt + ((ps.K * ps.win_cap + 31) & ~31u));  // stage_items
    __shared__ uint32_t s_lo[kMaxPieces + 1];
    __shared__ uint32_t s_seg[kMaxPieces + 1];
    __shared__ uint32_t s_seg2[kMaxPieces + 1];  // double buffer with s_seg (current / look-ahead frame)
    __shared__ uint32_t s_psrc[kMaxPieces];      // piece table
    __shared__ unsigned long long s_fval[2][kMaxTiles];  // publisher words (poll / look-ahead scratch)
    __shared__ uint32_t s_ahead;
    static_assert(NW <= 32, "one scan warp covers every warp");
    __shared__ uint32_t s_wa[NPT * NW], s_wb[NPT * NW];
    __shared__ uint32_t s_tmp[NW + 1];
    __shared__ uint32_t s_mw[NW];
    __shared__ uint32_t s_out[2];
    __shared__ unsigned long long s_prof[P_SLOTS];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, C = ps.C, P = ps.P;
    for (uint32_t j = tid; j <= P; j += NT) s_lo[j] = ps.piece_lo[j];
    for (uint32_t j = tid; j < P; j += NT) s_psrc[j] = ps.piece_src[j];
    for (uint32_t j = tid; j < ps.K * ps.win_cap; j += NT) cnt[j] = 0;
    if (tid < P_SLOTS) s_prof[tid] = 0;
    __syncthreads();
    const uint32_t pa = ps.cta_piece[2 * c], pb = ps.cta_piece[2 * c + 1];
    const uint32_t alo = s_lo[pa], na = s_lo[pa + 1] - alo;  // receiving piece
    const uint32_t blo = s_lo[pb], nb = s_lo[pb + 1] - blo;  // update-only piece
    unsigned long long my_deliv = 0, my_spikes = 0;
    unsigned long long lc = 0;  // CTA 0: log cursor
    uint32_t* seg_cur = s_seg;
    uint32_t* seg_next = s_seg2;
    bool have_next = false;
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
                // work on scalar copies: no pointer into the register arrays
                // escapes, so the state stays in registers (no local memory)
                values_t<NF> vl = v[r];
                xorshift rl = rr[r];
                bool ll = live[r];
                local_neuron<NF> ref{i, &vl, &rl, &ll, ps.rng};
                spk[r] = model.update(ref, ps.dt);
                v[r] = vl;
                rr[r] = rl;
                live[r] = ll;
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
        if (profiling) {
            const long long now = clock64();
            s_prof[6] += now - tp;  // thread 0's own update work
        }
        __syncthreads();
        if (profiling) {
            const long long now = clock64();
            s_prof[7] += now - tp;  // ... plus waiting for the slowest warp
        }
        if (warp == 0) {  // exclusive scans of the per-warp counts, ascending local index
            uint32_t runa = 0, runb = 0;
#pragma unroll
            for (int r = 0; r < NPT; ++r) {
                const uint32_t xa = lane < NW ? s_wa[r * NW + lane] : 0;
                const uint32_t xb = lane < NW ? s_wb[r * NW + lane] : 0;
                uint32_t ia = xa, ib = xb;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
                    const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
                    if (lane >= static_cast<uint32_t>(o)) {
                        ia += ya;
                        ib += yb;
                    }
                }
                if (lane < NW) {
                    s_wa[r * NW + lane] = runa + ia - xa;
                    s_wb[r * NW + lane] = runb + ib - xb;
                }
                runa += __shfl_sync(0xffffffffu, ia, 31);
                runb += __shfl_sync(0xffffffffu, ib, 31);
            }
            uint32_t mm = lane < NW ? s_mw[lane] : 0;
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
            st_release_gpu(ps.finfo + static_cast<uint64_t>(slot) * ps.E + c, frame_word(t, outa, outb));
            if (outa + outb) atomicAdd(&ps.step_spikes[s], outa + outb);
            if (meas) atomicAdd(&ps.step_meas[s], meas);
            my_spikes += outa + outb;
        }
        mark(P_PUBLISH);

        // ------------------------------------------------ Receive(t - delay + 1)
        const int64_t due = t - static_cast<int64_t>(ps.delay) + 1;
        if (due < 0) continue;
        const uint32_t* dq = ps.queue + static_cast<uint64_t>(due % ps.Q) * ps.n;
        // frame due: prefix from the previous step's look-ahead when it was
        // complete, else poll now; frame due+1: look ahead without waiting
        uint32_t* seg = have_next ? seg_next : seg_cur;
        uint32_t* seg_ahead = have_next ? seg_cur : seg_next;
        if (warp == 0) {
            if (!have_next) frame_prefix(ps, due, seg, s_fval[0], s_psrc, false);
        } else if (warp == 1) {
            const bool ready = due + 1 < t && frame_prefix(ps, due + 1, seg_ahead, s_fval[1], s_psrc, true);
            if (lane == 0) s_ahead = ready ? 1u : 0u;
        }
        __syncthreads();
        have_next = s_ahead != 0;
        seg_next = seg_ahead;
        seg_cur = seg;
        mark(P_POLL);
        // stream the FULL rows of frame due+1 into L2 (spike g by CTA g mod C)
        if (have_next) {
            const uint32_t S2 = seg_next[P];
            const uint32_t g2 = c + (NT - 1 - tid) * C;
            if (g2 < S2) {
                const uint32_t a = piece_of(seg_next, P, g2);
                const uint32_t* dq2 = ps.queue + static_cast<uint64_t>((due + 1) % ps.Q) * ps.n;
                const uint32_t src = __ldcg(dq2 + s_lo[a] + (g2 - seg_next[a]));
                // this shard's receive range of the row: [split[s][0], split[s][C])
                const uint32_t r0 = __ldg(ps.split + static_cast<uint64_t>(src) * (C + 1)) & ~3u;
                const uint32_t r1 = __ldg(ps.split + static_cast<uint64_t>(src) * (C + 1) + C);
                const uint32_t bytes = r1 > r0 ? ((r1 - r0) * 4 + 15) & ~15u : 0;
                if (bytes)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     ps.cells + static_cast<uint64_t>(src) * ps.pitch + r0),
                                 "r"(bytes)
                                 : "memory");
            }
        }
        const uint32_t S = seg_cur[P];
        const bool logging = ps.log && c == 0 && due >= ps.log_from;
        if (logging && tid == 0) ps.log_cnt[due - ps.log_from] = S;
        for (uint32_t c0 = 0; c0 < S; c0 += NT) {
            // one spike per thread: id, this CTA's row segment, item count
            const uint32_t g = c0 + tid;
            uint32_t len = 0, cofs = 0, nchunk = 0, beg = 0;
            uint64_t row = 0;
            if (g < S) {
                const uint32_t a = piece_of(seg_cur, P, g);
                const uint32_t src = __ldcg(dq + s_lo[a] + (g - seg_cur[a]));
                if (logging && lc + g < ps.log_cap) ps.log[lc + g] = src;
                const uint32_t* sp = ps.split + static_cast<uint64_t>(src) * (C + 1) + c;
                const uint32_t sb = __ldg(sp), se = __ldg(sp + 1);
                len = se - sb;
                row = static_cast<uint64_t>(src) * ps.pitch;  // row start (16-B aligned)
                cofs = static_cast<uint32_t>(source_class(ps, src)) * ps.win_cap - alo;
                // aligned 16-B chunks covering [sb, se)
                beg = sb;
                nchunk = len ? (((se + 3) >> 2) - (sb >> 2)) : 0;
                my_deliv += len;
            }
            uint32_t nitems;
            const uint32_t first = block_exclusive_scan<NT>(nchunk, s_tmp, nitems);
            mark(P_GATHER);
            // flattened 16-byte chunk list, in passes (a pass is normally the
            // whole frame): chunk = {row pointer of 4 targets, count offset,
            // valid word range}; every lane loads its own chunk with a 16-byte
            // load (consecutive lanes -> consecutive chunks of one segment,
            // coalesced), kChunkBatch chunks in flight per lane
            const uint32_t cap = ps.stage_items;
            for (uint32_t i0 = 0; i0 < nitems; i0 += cap) {
                for (uint32_t q = 0; q < nchunk; ++q) {
                    const uint32_t it = first + q;
                    if (it < i0 || it >= i0 + cap) continue;
                    const uint32_t w0 = ((beg >> 2) + q) << 2;  // first word of the chunk
                    const uint32_t lo = beg > w0 ? beg - w0 : 0;
                    const uint32_t hi = min(4u, beg + len - w0);
                    const uint64_t a = row + w0;
                    chunks[it - i0] = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32), cofs,
                                                 lo | (hi << 8));
                }
                __syncthreads();
                const uint32_t m = min(cap, nitems - i0);
                for (uint32_t k0 = tid; k0 < m; k0 += kChunkBatch * NT) {
                    uint4 d[kChunkBatch];
                    uint4 w[kChunkBatch];
#pragma unroll
                    for (int u = 0; u < kChunkBatch; ++u) {
                        const uint32_t k = k0 + u * NT;
                        d[u] = k < m ? chunks[k] : make_uint4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < kChunkBatch; ++u) {
                        const uint4* rp = reinterpret_cast<const uint4*>(
                            ps.cells + ((static_cast<uint64_t>(d[u].y) << 32) | d[u].x));
                        w[u] = (d[u].w >> 8) ? ldg_stream4(rp) : make_uint4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < kChunkBatch; ++u) {
                        const uint32_t lo = d[u].w & 0xffu, hi = d[u].w >> 8;
                        if (lo <= 0 && hi > 0) atomicAdd(&cnt[d[u].z + w[u].x], 1u);
                        if (lo <= 1 && hi > 1) atomicAdd(&cnt[d[u].z + w[u].y], 1u);
                        if (lo <= 2 && hi > 2) atomicAdd(&cnt[d[u].z + w[u].z], 1u);
                        if (hi > 3) atomicAdd(&cnt[d[u].z + w[u].w], 1u);
                    }
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
    __shared__ uint32_t s_psrc[kMaxPieces];
    __shared__ unsigned long long s_fval[kMaxTiles];
    const uint32_t P = ps.P;
    for (uint32_t j = threadIdx.x; j <= P; j += blockDim.x) s_lo[j] = ps.piece_lo[j];
    for (uint32_t j = threadIdx.x; j < P; j += blockDim.x) s_psrc[j] = ps.piece_src[j];
    unsigned long long lc = 0;
    for (int64_t f = from; f <= to; ++f) {
        const uint32_t slot = static_cast<uint32_t>(f % ps.Q);
        __syncthreads();
        // every publisher's word of frame f (peer shards publish theirs
        // asynchronously: wait for them), then the piece prefix
        if (threadIdx.x < 32) frame_prefix(ps, f, s_seg, s_fval, s_psrc, false);
        __syncthreads();
        const uint32_t S = s_seg[P];
        if (threadIdx.x == 0) ps.log_cnt[f - from] = S;
        // one thread per frame position (its piece by binary search over the
        // piece prefix): every load and host store of the frame in flight at once
        for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
            const uint32_t a = piece_of(s_seg, P, i);
            if (lc + i < ps.log_cap)
                ps.log[lc + i] = ps.queue[static_cast<uint64_t>(slot) * ps.n + s_lo[a] + (i - s_seg[a])];
        }
        lc += S;
    }
    if (threadIdx.x == 0) {
        *ps.log_end = lc;
        if (lc > ps.log_cap) ps.flags[0] = 1;
    }
}

// ---- shard exchange: frames produced by this shard's CTAs in
// steps [t0, t0+b) are packed as
//   words[0] = b, words[1 + 2k] / [2 + 2k] = A / B spike count of step k,
//   then the ids of every step: A piece ids (CTA order) then B piece ids.
// A and B pieces of one shard are contiguous id ranges, so a remote shard's
// frame slice is two contiguous runs.  One warp per step; the lanes split the
// C publishers (warp scans give every CTA's offset), so the exchange costs a
// few L2 round trips per batch, not one per (step, CTA).

// warp-wide inclusive scan
SYNQ_DEV uint32_t warp_incl_scan(uint32_t x) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    return x;
}

template <class M>
__global__ void k_export(persist_state<M> ps, int64_t t0, uint32_t b, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t C = ps.C;
    if (threadIdx.x == 0) out[0] = b;
    // (1) per-step totals into the header
    for (uint32_t k = warp; k < b; k += nw) {
        const uint64_t* fi = reinterpret_cast<const uint64_t*>(ps.finfo) + static_cast<uint64_t>((t0 + k) % ps.Q) * ps.E;
        uint32_t ta = 0, tb = 0;
        for (uint32_t c = lane; c < C; c += 32) {
            const unsigned long long e = fi[c];
            ta += word_a(e);
            tb += word_b(e);
        }
        for (int o = 16; o; o >>= 1) {
            ta += __shfl_xor_sync(0xffffffffu, ta, o);
            tb += __shfl_xor_sync(0xffffffffu, tb, o);
        }
        if (lane == 0) {
            out[1 + 2 * k] = ta;
            out[2 + 2 * k] = tb;
        }
    }
    __syncthreads();
    // (2) per step: base offset from the header, then every CTA's slices
    for (uint32_t k = warp; k < b; k += nw) {
        uint32_t before = 0;
        for (uint32_t q = lane; q < k; q += 32) before += out[1 + 2 * q] + out[2 + 2 * q];
        for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
        const uint32_t base = 1 + 2 * b + before, ta = out[1 + 2 * k];
        const uint32_t slot = static_cast<uint32_t>((t0 + k) % ps.Q);
        const uint64_t* fi = reinterpret_cast<const uint64_t*>(ps.finfo) + static_cast<uint64_t>(slot) * ps.E;
        const uint32_t* q = ps.queue + static_cast<uint64_t>(slot) * ps.n;
        uint32_t runa = 0, runb = 0;
        for (uint32_t c0 = 0; c0 < C; c0 += 32) {
            const uint32_t c = c0 + lane;
            const unsigned long long e = c < C ? fi[c] : 0ull;
            const uint32_t ca = c < C ? word_a(e) : 0u, cb = c < C ? word_b(e) : 0u;
            const uint32_t ia = warp_incl_scan(ca), ib = warp_incl_scan(cb);
            if (c < C) {
                const uint32_t alo = ps.piece_lo[ps.cta_piece[2 * c]], blo = ps.piece_lo[ps.cta_piece[2 * c + 1]];
                uint32_t* oa = out + base + runa + ia - ca;
                uint32_t* ob = out + base + ta + runb + ib - cb;
                for (uint32_t j = 0; j < ca; ++j) oa[j] = q[alo + j];
                for (uint32_t j = 0; j < cb; ++j) ob[j] = q[blo + j];
            }
            runa += __shfl_sync(0xffffffffu, ia, 31);
            runb += __shfl_sync(0xffffffffu, ib, 31);
        }
    }
}

// unpack a remote shard's frames (b steps from t0) into the ring as publisher
// `entry`; its pieces start at ids alo / blo.  One block per step.
template <class M>
__global__ void k_import(persist_state<M> ps, int64_t t0, uint32_t b, const uint32_t* in, uint32_t entry,
                         uint32_t alo, uint32_t blo) {
    __shared__ uint32_t s_base;
    const uint32_t k = blockIdx.x;
    if (k >= b) return;
    if (threadIdx.x < 32) {
        uint32_t before = 0;
        for (uint32_t q = threadIdx.x; q < k; q += 32) before += in[1 + 2 * q] + in[2 + 2 * q];
        for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
        if (threadIdx.x == 0) {
            s_base = 1 + 2 * b + before;
            if (in[0] != b) ps.flags[2] = 1;  // batch length mismatch between shards
        }
    }
    __syncthreads();
    const uint32_t ca = in[1 + 2 * k], cb = in[2 + 2 * k], base = s_base;
    const uint32_t slot = static_cast<uint32_t>((t0 + k) % ps.Q);
    uint32_t* q = ps.queue + static_cast<uint64_t>(slot) * ps.n;
    for (uint32_t j = threadIdx.x; j < ca; j += blockDim.x) q[alo + j] = in[base + j];
    for (uint32_t j = threadIdx.x; j < cb; j += blockDim.x) q[blo + j] = in[base + ca + j];
    __syncthreads();
    if (threadIdx.x == 0) ps.finfo[static_cast<uint64_t>(slot) * ps.E + entry] = frame_word(t0 + k, ca, cb);
}

// debug_checks for the persistent engine (engine.hpp:440-446): block k
// checks frame t0 + k: every publisher's piece slices are strictly ascending
// and inside their pieces (pieces tile the id space in order, so the merged
// frame is sorted and unique), and the slices add up to the step's spike
// count (step_spikes, this rank's CTAs).  flags[3] |= 1 / 2.
template <class M>
__global__ void k_check_persist(persist_state<M> ps, int64_t t0, uint32_t b) {
    const uint32_t k = blockIdx.x;
    if (k >= b) return;
    const uint32_t slot = static_cast<uint32_t>((t0 + k) % ps.Q);
    const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(slot) * ps.E;
    const uint32_t* q = ps.queue + static_cast<uint64_t>(slot) * ps.n;
    __shared__ unsigned long long s_local;
    if (threadIdx.x == 0) s_local = 0;
    __syncthreads();
    bool bad = false;
    unsigned long long local = 0;
    for (uint32_t p = threadIdx.x; p < ps.P; p += blockDim.x) {
        const uint32_t src = ps.piece_src[p];
        if ((src >> 1) >= ps.C) continue;  // remote ranks' frames are imported after the batch
        const unsigned long long w = fi[src >> 1];
        if (word_tag(w) != frame_tag(t0 + k)) {
            bad = true;
            continue;
        }
        const uint32_t cnt = word_half(w, src & 1), lo = ps.piece_lo[p], hi = ps.piece_lo[p + 1];
        local += cnt;
        if (cnt > hi - lo) {
            bad = true;
            continue;
        }
        for (uint32_t i = 0; i < cnt; ++i) {
            const uint32_t id = q[lo + i];
            bad |= id < lo || id >= hi || (i > 0 && q[lo + i - 1] >= id);
        }
    }
    if (bad) atomicOr(ps.flags + 3, 1u);
    atomicAdd(&s_local, local);
    __syncthreads();
    if (threadIdx.x == 0 && s_local != ps.step_spikes[k]) atomicOr(ps.flags + 3, 2u);
}

// ---- in-engine exchange (NCCL allgather of fixed-size spike bitmasks) ----
// Rank r's send block: words[0] = b, then for step k < b: wa_max + wb_max
// words: bit i of the A part = id a_lo_r + i spiked, bit i of the B part =
// id b_lo_r + i spiked (wa_max / wb_max = the largest A / B range of any
// rank, in words).  Fixed size, so the allgather needs no counts exchange
// and no host synchronisation.
// Warp-wide: copy this shard's part of frame f (its local pieces, complete
// and acquired by the caller) into every peer's ring as one consolidated
// A slice and one B slice in ascending id order, then release the frame's
// publisher word there (system scope: the stores cross NVLink).
template <class M>
SYNQ_DEV void peer_export(const persist_state<M>& ps, int64_t f) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t slot = static_cast<uint64_t>(f % ps.Q);
    const unsigned long long* fi = ps.finfo + slot * ps.E;
    const uint32_t* q = ps.queue + slot * ps.n;
    uint32_t tot[2];
    for (uint32_t half = 0; half < 2; ++half) {
        const uint32_t dlo = half ? ps.b_lo : ps.a_lo;
        uint32_t run = 0;
        for (uint32_t c0 = 0; c0 < ps.C; c0 += 32) {
            const uint32_t cc = c0 + lane;
            const uint32_t cnt = cc < ps.C ? word_half(__ldcg(fi + cc), half) : 0u;
            const uint32_t incl = warp_incl_scan(cnt);
            const uint32_t src = cc < ps.C ? ps.piece_lo[ps.cta_piece[2 * cc + half]] : 0u;
            const uint64_t dst = slot * ps.n + dlo + run + incl - cnt;
            for (uint32_t j = 0; j < cnt; ++j) {
                const uint32_t id = __ldcg(q + src + j);
                for (uint32_t p = 0; p < ps.npeers; ++p) ps.peers[p].queue[dst + j] = id;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        tot[half] = run;
    }
    __syncwarp();
    fence_acq_rel_sys();  // every lane's slice stores before the words
    __syncwarp();
    for (uint32_t p = lane; p < ps.npeers; p += 32) {
        const peer_link L = ps.peers[p];
        st_relaxed_sys(L.finfo + slot * L.E + L.entry, frame_word(f, tot[0], tot[1]));
    }
}

struct xbits_layout {
    uint32_t wa, wb;   // words per step of the A / B part (max over ranks)
    uint32_t steps;    // steps per block (delay - 1)
    uint32_t block;    // words per rank block = 1 + steps * (wa + wb)
};

// one block per step: this shard's frames -> bitmask (built in shared memory)
template <class M>
__global__ void k_export_bits(persist_state<M> ps, int64_t t0, uint32_t b, xbits_layout L, uint32_t a_lo,
                              uint32_t b_lo, uint32_t* out) {
    extern __shared__ uint32_t s_bits[];  // wa + wb words
    const uint32_t k = blockIdx.x;
    if (k == 0 && threadIdx.x == 0) out[0] = b;
    if (k >= b) return;
    const uint32_t W = L.wa + L.wb;
    for (uint32_t j = threadIdx.x; j < W; j += blockDim.x) s_bits[j] = 0;
    __syncthreads();
    const uint32_t slot = static_cast<uint32_t>((t0 + k) % ps.Q);
    const unsigned long long* fi = ps.finfo + static_cast<uint64_t>(slot) * ps.E;
    const uint32_t* q = ps.queue + static_cast<uint64_t>(slot) * ps.n;
    // thread per (local CTA, part): a frame holds a few ids per CTA, so one
    // round of independent load chains (finfo, piece offset, ids) covers all
    for (uint32_t x = threadIdx.x; x < 2 * ps.C; x += blockDim.x) {
        const uint32_t c = x >> 1, part = x & 1;
        const uint32_t lo = ps.piece_lo[ps.cta_piece[2 * c + part]];
        const unsigned long long e = fi[c];
        const uint32_t cnt = part ? word_b(e) : word_a(e);
        const uint32_t base = part ? b_lo : a_lo, woff = part ? L.wa : 0u;
#pragma unroll 4
        for (uint32_t j = 0; j < cnt; ++j) {
            const uint32_t i = q[lo + j] - base;
            atomicOr(&s_bits[woff + (i >> 5)], 1u << (i & 31));
        }
    }
    __syncthreads();
    uint32_t* o = out + 1 + static_cast<uint64_t>(k) * W;
    for (uint32_t j = threadIdx.x; j < W; j += blockDim.x) o[j] = s_bits[j];
}

// block (k, rank slot): a remote rank's bitmask of step k -> ascending ids in
// its pieces' slices of queue slot (t0 + k) % Q, then its frame word
struct xbits_remote {
    uint32_t rank, entry, a_lo, b_lo, na, nb;  // rank id, publisher entry, id ranges
};
template <class M>
__global__ void k_import_bits(persist_state<M> ps, int64_t t0, uint32_t b, xbits_layout L, const uint32_t* in,
                              const xbits_remote* remotes) {
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_cnt[2];
    const uint32_t k = blockIdx.x, rr = blockIdx.y;
    const xbits_remote R = remotes[rr];
    const uint32_t* blk = in + static_cast<uint64_t>(R.rank) * L.block;
    if (k >= b) return;
    if (k == 0 && threadIdx.x == 0 && blk[0] != b) ps.flags[2] = 1;
    const uint32_t W = L.wa + L.wb;
    const uint32_t* bits = blk + 1 + static_cast<uint64_t>(k) * W;
    const uint32_t slot = static_cast<uint32_t>((t0 + k) % ps.Q);
    uint32_t* q = ps.queue + static_cast<uint64_t>(slot) * ps.n;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // two parts: A (ids a_lo + i, i < na) then B (ids b_lo + i, i < nb)
    for (int part = 0; part < 2; ++part) {
        const uint32_t nwords = part == 0 ? (R.na + 31) / 32 : (R.nb + 31) / 32;
        const uint32_t* wbits = bits + (part == 0 ? 0u : L.wa);
        const uint32_t lo = part == 0 ? R.a_lo : R.b_lo;
        // contiguous chunk of words per thread, block-wide exclusive scan of popcounts
        const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
        const uint32_t w0 = threadIdx.x * per, w1 = min(nwords, w0 + per);
        uint32_t mine = 0;
        for (uint32_t w = w0; w < w1; ++w) mine += __popc(wbits[w]);
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (lane == 31) s_scan[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t x = lane < nw ? s_scan[lane] : 0u;
            uint32_t wi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= static_cast<uint32_t>(o)) wi += y;
            }
            if (lane < nw) s_scan[lane] = wi - x;
            if (lane == 31) s_cnt[part] = wi;
        }
        __syncthreads();
        uint32_t pos = s_scan[warp] + incl - mine;
        for (uint32_t w = w0; w < w1; ++w) {
            uint32_t m = wbits[w];
            while (m) {
                const uint32_t bit = __ffs(m) - 1;
                m &= m - 1;
                q[lo + pos++] = lo + w * 32 + bit;
            }
        }
        __syncthreads();  // s_scan reused by the next part
    }
    if (threadIdx.x == 0) {
        __threadfence();
        ps.finfo[static_cast<uint64_t>(slot) * ps.E + R.entry] = frame_word(t0 + k, s_cnt[0], s_cnt[1]);
    }
}

}  // namespace synq::dev
