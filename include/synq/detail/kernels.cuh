#pragma once
// Generic sm_100a kernels of the synq pipeline, templated on the user Model
// (reference stages: proj/include/synq/engine.hpp:308-436).
//
// One simulation step on the generic path is a short kernel sequence on one
// stream (captured into a CUDA graph by the engine):
//
//   k_update        Update Neurons: model.update per neuron; spikers are
//                   compacted into the frame's queue IN ASCENDING ID ORDER by
//                   a single-pass decoupled look-back scan over id tiles; bit
//                   history + expiry (plastic models).
//   k_catchup       Update Synapses (lazy STDP, engine.hpp:343-367, 414-436):
//                   CTA per neuron of frame(due) U expiring; each thread
//                   replays its synapses in registers over [ages, t] against
//                   the neuron-major bit history, stores once.
//   k_receive       Receive Spikes (engine.hpp:369-409): warp per
//                   (spike, 256-target chunk); deliveries through device
//                   atomics (fast mode), or
//   k_det_*         ordered delivery (deterministic mode): count, scan,
//                   scatter, then one thread per target applies its events in
//                   ascending source order with plain stores — the
//                   reference's sequential accumulation order, bit for bit.
//
// The step index lives on the device (t_dev) and advances in the epilogue of
// the step's last kernel, so one captured graph replays for any step.
#include <cuda_runtime.h>

#include <concepts>
#include <cstdint>

#include "synq/detail/device_refs.cuh"
#include "synq/models/benchmarks.hpp"
#include "synq/soa.hpp"

namespace synq::dev {

template <class M, class = void>
struct synapse_fields_of {
    using type = fields<>;
    static constexpr bool present = false;
};
template <class M>
struct synapse_fields_of<M, std::void_t<typename M::synapse_fields>> {
    using type = typename M::synapse_fields;
    static constexpr bool present = true;
};
template <class M>
constexpr bool model_uses_rng() {
    if constexpr (requires { M::uses_rng; })
        return M::uses_rng;
    else
        return false;
}

template <class M>
constexpr bool model_has_plastic() {
    return requires(const M& m, uint32_t a, uint32_t b) { { m.plastic(a, b) } -> std::convertible_to<bool>; };
}
constexpr uint32_t kTraceRing = 128;  // steps of per-neuron trace history (trace-STDP models)

template <class M>
constexpr bool model_trace_stdp() {
    if constexpr (requires { trace_stdp<M>::available; })
        return trace_stdp<M>::available;
    else
        return false;
}

// receive reads only the weight field W (== field 0) and writes no synapse
// field (a trace_stdp trait declaration): stage W once, no write-back
template <class M>
constexpr bool model_receive_weight_only() {
    if constexpr (requires { trace_stdp<M>::receive_reads_weight_only; })
        return trace_stdp<M>::receive_reads_weight_only && trace_stdp<M>::W == 0;
    else
        return false;
}

// a model exposing plastic(src, dst) declares update_synapse a no-op for the
// other synapses (benchmarks.hpp brunel_plus_model): catch-up skips them

enum counter_slot : int { C_SPIKES = 0, C_DELIVERIES = 1, C_SYN_UPDATES = 2, C_EXPIRY = 3, C_COUNT = 8 };

template <class M>
struct engine_state {
    using NF = typename M::neuron_fields;
    using SF = typename synapse_fields_of<M>::type;

    field_ptrs<NF> nf;
    field_ptrs<SF> sf;
    xorshift* rng;
    const uint32_t* cells;
    const uint32_t* degree;
    uint32_t n, pitch, deg_max;

    uint32_t* queue;   // Q frames x n ids
    uint32_t* qcount;  // Q
    uint32_t Q;

    uint64_t* hist;  // neuron-major spike history, hist_words per neuron
    uint32_t hist_words;
    uint32_t* ages;
    uint32_t* expiring;
    uint32_t* expiring_count;
    uint8_t* caught;              // k_catchup1 (mode 0): ages advance to t + 1 in the next k_update
    unsigned long long* split_param;  // split catch-up: [0] = t, [1] = expiring count (written by part 1)
    float* tr_p;                  // trace-STDP models: P_i(u) at [(u & (kTraceRing - 1)) * n + i]
    float* tr_q;                  // ... Q_i(u)
    const uint8_t* row_plastic;   // models with plastic(): row holds a plastic synapse (else nullptr)

    unsigned long long* counters;
    unsigned long long* tile_status;  // decoupled look-back, one word per id tile
    uint32_t* tile_bal;               // k_update<.., false>: spike ballot per (tile, warp)
    uint32_t* tile_ctr;               // [2] dynamic tile ids, by step parity
    uint32_t* done_ctr;               // last-block detection of the step's final kernel

    int64_t* t_dev;
    const int64_t* t0_dev;  // first step of the current batch (per-step arrays index)
    uint32_t* step_spikes;
    uint32_t* step_meas;
    uint32_t meas_lo, meas_hi;
    uint32_t step_cap;

    uint32_t* log;  // frame log (taps / raster), ids of consecutive frames
    unsigned long long* log_cursor;  // [2] by step parity
    unsigned long long log_cap;
    uint32_t* flags;  // [0] log overflow, [1] ordered-delivery overflow

    float dt;
    uint32_t delay, history;
    bool track_bits;

    // ordered (deterministic) delivery scratch
    uint32_t* det_cnt;
    uint32_t* det_off;
    uint32_t* det_fill;
    unsigned long long* det_ev;
    unsigned long long det_cap;
};

// ------------------------------------------------------------- helpers
SYNQ_DEV uint32_t lane_id() { return threadIdx.x & 31; }

// programmatic dependent launch (PDL): the primary lets its dependent grid
// be scheduled early; the dependent waits for the primary's memory before
// touching its outputs (both are no-ops without the launch attribute)
SYNQ_DEV void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
SYNQ_DEV void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <class M>
SYNQ_DEV bool hist_bit(const engine_state<M>& st, uint32_t id, int64_t u) {
    if (u < 0) return false;
    const uint32_t slots = 64u * st.hist_words;
    const uint32_t slot = st.hist_words == 1 ? static_cast<uint32_t>(u & 63) : static_cast<uint32_t>(u % slots);
    return (st.hist[static_cast<uint64_t>(id) * st.hist_words + (slot >> 6)] >> (slot & 63)) & 1ull;
}

SYNQ_DEV bool word_bit(const uint64_t* words, uint32_t nwords, int64_t u) {
    if (u < 0) return false;
    const uint32_t slot = static_cast<uint32_t>(u % (64u * nwords));
    return (words[slot >> 6] >> (slot & 63)) & 1ull;
}

SYNQ_DEV unsigned long long ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
SYNQ_DEV void st_volatile(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// status word: tag(30) | flag(2) | value(32); flag 1 = aggregate, 2 = inclusive prefix
SYNQ_DEV unsigned long long lb_pack(uint32_t tag, uint32_t flag, uint32_t v) {
    return (static_cast<unsigned long long>(tag) << 34) | (static_cast<unsigned long long>(flag) << 32) | v;
}

// warp-cooperative decoupled look-back: returns the exclusive prefix of `tile`
SYNQ_DEV uint32_t lookback(unsigned long long* status, uint32_t tile, uint32_t agg, uint32_t tag) {
    const uint32_t lane = lane_id();
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], lb_pack(tag, 2, agg));
        __syncwarp();
        return 0;
    }
    if (lane == 0) st_volatile(&status[tile], lb_pack(tag, 1, agg));
    uint32_t excl = 0;
    int64_t j = static_cast<int64_t>(tile) - 1;
    while (true) {
        const int64_t idx = j - lane;
        uint32_t flag = 2, val = 0;
        if (idx >= 0) {
            unsigned long long w;
            do {
                w = ld_volatile(&status[idx]);
            } while (static_cast<uint32_t>(w >> 34) != tag || ((w >> 32) & 3u) == 0);
            flag = static_cast<uint32_t>((w >> 32) & 3u);
            val = static_cast<uint32_t>(w);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, flag == 2);
        if (pmask) {
            const int first = __ffs(pmask) - 1;  // nearest predecessor holding a full prefix
            uint32_t v = lane <= static_cast<uint32_t>(first) ? val : 0;
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            excl += v;
            break;
        }
        uint32_t v = val;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        j -= 32;
    }
    if (lane == 0) st_volatile(&status[tile], lb_pack(tag, 2, excl + agg));
    __syncwarp();
    return excl;
}

// end-of-step housekeeping, run once by the last block of the step's final kernel
template <class M>
SYNQ_DEV void step_epilogue(const engine_state<M>& st, int64_t t) {
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(st.done_ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        *st.done_ctr = 0;
        if (st.expiring_count) *st.expiring_count = 0;
        st.tile_ctr[(t + 1) & 1] = 0;
        __threadfence();
        *st.t_dev = t + 1;
    }
}

// ------------------------------------------------------------- init
template <class M>
__global__ void k_init_neurons(M model, engine_state<M> st, uint64_t seed) {
    using NF = typename M::neuron_fields;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += gridDim.x * blockDim.x) {
        values_t<NF> v;
        load_all(st.nf, i, v);
        xorshift r;
        bool live = false;
        if constexpr (model_uses_rng<M>()) {
            r.reseed(derive_seed(seed, (1ull << 32) + i));  // engine.hpp:161-163
            live = true;
        }
        local_neuron<NF> ref{i, &v, &r, &live, st.rng};
        model.init(ref);
        store_all(st.nf, i, v);
        if constexpr (model_uses_rng<M>()) st.rng[i] = r;
    }
}

template <class M>
__global__ void k_init_synapses(M model, engine_state<M> st) {
    using SF = typename synapse_fields_of<M>::type;
    const uint32_t lane = lane_id();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t s = warp; s < st.n; s += nwarps) {
        const uint32_t d = st.degree[s];
        const uint32_t* row = st.cells + static_cast<uint64_t>(s) * st.pitch;
        bool any = false;
        for (uint32_t k = lane; k < d; k += 32) {
            global_synapse<SF> syn{static_cast<uint64_t>(s) * st.deg_max + k, s, row[k], st.sf};
            model.init_synapse(syn);
            if constexpr (model_has_plastic<M>()) any |= model.plastic(s, row[k]);
        }
        if constexpr (model_has_plastic<M>()) {
            any = __any_sync(0xffffffffu, any);
            if (lane == 0 && st.row_plastic) const_cast<uint8_t*>(st.row_plastic)[s] = any ? 1 : 0;
        }
    }
}

// ------------------------------------------------------------- update
// kLookback: compact in the same kernel with a decoupled look-back across
// tiles (large networks); otherwise every tile stores its warps' spike
// ballots (tile_bal) and k_compact places the ids (a look-back over a few
// hundred tiles is a chain of L2 round trips: ~10 us at Brunel+ 1e8)
template <class M, int BLOCK, bool kLookback = true>
__global__ void __launch_bounds__(BLOCK) k_update(M model, engine_state<M> st) {
    using NF = typename M::neuron_fields;
    constexpr bool kSyn = synapse_fields_of<M>::present;
    constexpr int NW = BLOCK / 32;
    __shared__ uint32_t s_tile, s_base;
    __shared__ uint32_t s_warp[NW];
    __shared__ uint32_t s_meas;

    grid_dependency_wait();    // PDL: the previous step's kernels are complete
    grid_launch_dependents();  // the catch-up may be scheduled on the SMs this grid frees
    const int64_t t = *st.t_dev;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_tile = kLookback ? atomicAdd(&st.tile_ctr[t & 1], 1u) : blockIdx.x;
        s_meas = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t i = tile * BLOCK + threadIdx.x;

    bool spk = false;
    unsigned long long n_exp = 0, n_upd = 0;  // expiring neurons, retired non-plastic synapse updates
    bool listed = false;                      // expiring with a plastic row: catch-up list
    if (i < st.n) {
        values_t<NF> v;
        load_all(st.nf, i, v);
        values_t<NF> before = v;
        xorshift r;
        bool live = false;
        local_neuron<NF> ref{i, &v, &r, &live, st.rng};
        spk = model.update(ref, st.dt);
        store_changed(st.nf, i, v, before);
        if constexpr (model_uses_rng<M>())
            if (live) st.rng[i] = r;
        if (st.track_bits) {
            const uint32_t slot = st.hist_words == 1 ? static_cast<uint32_t>(t & 63)
                                                     : static_cast<uint32_t>(t % (64u * st.hist_words));
            uint64_t* w = st.hist + static_cast<uint64_t>(i) * st.hist_words + (slot >> 6);
            *w = (*w & ~(1ull << (slot & 63))) | (static_cast<uint64_t>(spk) << (slot & 63));
        }
        if constexpr (model_trace_stdp<M>()) {
            if (st.tr_p) {  // the per-neuron traces of step t (the stdp_step float sequence)
                const stdp_params& sp = trace_stdp<M>::params(model);
                const uint32_t u = static_cast<uint32_t>(t) & (kTraceRing - 1), um = (u - 1) & (kTraceRing - 1);
                float pt = st.tr_p[static_cast<uint64_t>(um) * st.n + i], qt = st.tr_q[static_cast<uint64_t>(um) * st.n + i];
                pt *= sp.decay_plus;
                qt *= sp.decay_minus;
                if (hist_bit(st, i, t - static_cast<int64_t>(st.delay))) pt += 1.0f;  // pre of this source at t
                if (spk) qt += 1.0f;                                                 // post of this target at t
                st.tr_p[static_cast<uint64_t>(u) * st.n + i] = pt;
                st.tr_q[static_cast<uint64_t>(u) * st.n + i] = qt;
            }
        }
        if constexpr (kSyn) {  // engine.hpp:318-330
            if (st.caught && st.caught[i]) {  // caught up through t - 1 by the last step's k_catchup1
                st.caught[i] = 0;
                st.ages[i] = static_cast<uint32_t>(t);
            }
            const bool transmits = (st.delay == 1) ? spk : hist_bit(st, i, t - st.delay + 1);
            const int64_t a = st.ages[i];
            if (!transmits && a + st.history <= t + st.delay + 1) {
                n_exp = 1;  // expiry_batches (engine.hpp:349), summed per warp below
                if (st.row_plastic && !st.row_plastic[i]) {
                    // no plastic synapse in the row: the catch-up through t is
                    // only its counter and age (no replay, not listed)
                    if (a <= t) {
                        n_upd = static_cast<unsigned long long>(st.degree[i]) * static_cast<unsigned long long>(t - a + 1);
                        st.ages[i] = static_cast<uint32_t>(t + 1);
                    }
                } else {
                    listed = true;
                }
            }
        }
    }

    if constexpr (kSyn) {  // one atomic per warp, not per neuron (one counter word for the whole grid)
        const unsigned lm = __ballot_sync(0xffffffffu, listed);
        if (lm) {  // the expiring list, appended per warp (its order does not matter)
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(st.expiring_count, static_cast<uint32_t>(__popc(lm)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (listed) st.expiring[base + __popc(lm & ((1u << lane) - 1u))] = i;
        }
        for (int o = 16; o; o >>= 1) {
            n_exp += __shfl_xor_sync(0xffffffffu, n_exp, o);
            n_upd += __shfl_xor_sync(0xffffffffu, n_upd, o);
        }
        if (lane == 0 && n_exp) atomicAdd(&st.counters[C_EXPIRY], n_exp);
        if (lane == 0 && n_upd) atomicAdd(&st.counters[C_SYN_UPDATES], n_upd);
    }
    // ordered compaction: warp ballots -> block scan -> look-back across tiles
    const unsigned ball = __ballot_sync(0xffffffffu, spk);
    if (lane == 0) s_warp[warp] = __popc(ball);
    const bool meas = spk && i >= st.meas_lo && i < st.meas_hi;
    const unsigned mball = __ballot_sync(0xffffffffu, meas);
    if (lane == 0 && mball) atomicAdd(&s_meas, __popc(mball));
    if constexpr (!kLookback) {
        if (lane == 0) st.tile_bal[tile * NW + warp] = ball;
        __syncthreads();
        if (threadIdx.x == 0 && s_meas) {
            const int64_t rel = t - *st.t0_dev;
            if (rel < st.step_cap) atomicAdd(&st.step_meas[rel], s_meas);
        }
        return;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t c = lane < NW ? s_warp[lane] : 0;
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane < NW) s_warp[lane] = incl - c;
        const uint32_t tag = static_cast<uint32_t>((t + 1) & 0x3fffffff);
        const uint32_t excl = lookback(st.tile_status, tile, agg, tag);
        if (lane == 0) {
            s_base = excl;
            const int64_t rel = t - *st.t0_dev;
            if (s_meas && rel < st.step_cap) atomicAdd(&st.step_meas[rel], s_meas);
            const uint32_t ntiles = (st.n + BLOCK - 1) / BLOCK;
            if (tile == ntiles - 1) {  // the last tile knows the frame size
                const uint32_t total = excl + agg;
                st.qcount[t % st.Q] = total;
                atomicAdd(&st.counters[C_SPIKES], total);
                if (rel < st.step_cap) st.step_spikes[rel] = total;
                if (st.log) {
                    const unsigned long long base = st.log_cursor[t & 1];
                    st.log_cursor[(t + 1) & 1] = base + total;
                    if (base + total > st.log_cap) st.flags[0] = 1;
                }
            }
        }
    }
    __syncthreads();
    if (spk) {
        const uint32_t pos = s_base + s_warp[warp] + __popc(ball & ((1u << lane) - 1u));
        st.queue[static_cast<uint64_t>(t % st.Q) * st.n + pos] = i;
        if (st.log) {
            const unsigned long long at = st.log_cursor[t & 1] + pos;
            if (at < st.log_cap) st.log[at] = i;
        }
    }
}

// ordered placement of the spikes of step t from the tiles' ballots: tile
// b's base is the spike count of tiles 0..b-1 (summed by the block from the
// ballots), its warps' offsets follow, so frame t is in ascending id order
// (a device function: run by the first ntiles blocks of the calling grid,
// whose block size must be BLOCK)
template <class M, int BLOCK>
SYNQ_DEV void compact_tiles(const engine_state<M>& st, int64_t t) {
    constexpr int NW = BLOCK / 32;
    __shared__ uint32_t s_red[NW], s_warp[NW];
    __shared__ uint32_t s_base;
    const uint32_t ntiles = (st.n + BLOCK - 1) / BLOCK;
    if (blockIdx.x >= ntiles) return;
    const uint32_t tile = blockIdx.x, lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t before = 0;
    for (uint32_t w = threadIdx.x; w < tile * NW; w += BLOCK) before += __popc(st.tile_bal[w]);
    for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if (lane == 0) s_red[warp] = before;
    const unsigned ball = st.tile_bal[tile * NW + warp];
    if (lane == 0) s_warp[warp] = __popc(ball);
    __syncthreads();
    if (warp == 0) {
        uint32_t b = lane < NW ? s_red[lane] : 0u;
        for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        const uint32_t c = lane < NW ? s_warp[lane] : 0u;
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (lane < NW) s_warp[lane] = incl - c;
        const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) {
            s_base = b;
            if (tile == ntiles - 1) {  // the last tile knows the frame size
                const uint32_t total = b + agg;
                const int64_t rel = t - *st.t0_dev;
                st.qcount[t % st.Q] = total;
                atomicAdd(&st.counters[C_SPIKES], total);
                if (rel < st.step_cap) st.step_spikes[rel] = total;
                if (st.log) {
                    const unsigned long long base = st.log_cursor[t & 1];
                    st.log_cursor[(t + 1) & 1] = base + total;
                    if (base + total > st.log_cap) st.flags[0] = 1;
                }
            }
        }
    }
    __syncthreads();
    if ((ball >> lane) & 1u) {
        const uint32_t i = tile * BLOCK + threadIdx.x;
        const uint32_t pos = s_base + s_warp[warp] + __popc(ball & ((1u << lane) - 1u));
        st.queue[static_cast<uint64_t>(t % st.Q) * st.n + pos] = i;
        if (st.log) {
            const unsigned long long at = st.log_cursor[t & 1] + pos;
            if (at < st.log_cap) st.log[at] = i;
        }
    }
}

template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_compact(engine_state<M> st) {
    compact_tiles<M, BLOCK>(st, *st.t_dev);
}

// debug_checks (engine.hpp:440-446 check_frame): frame t of the generic
// engine is strictly ascending (sorted, unique) and, with the bit history,
// its size equals the popcount of the history slot.  flags[3] |= 1 (order)
// or 2 (popcount); the host throws the reference's logic_error messages.
template <class M>
__global__ void k_check_frame(engine_state<M> st) {
    __shared__ unsigned long long s_pop;
    const int64_t t = *st.t_dev;
    const uint32_t cnt = st.qcount[t % st.Q];
    const uint32_t* f = st.queue + static_cast<uint64_t>(t % st.Q) * st.n;
    if (threadIdx.x == 0) s_pop = 0;
    __syncthreads();
    bool bad = false;
    for (uint32_t i = threadIdx.x + 1; i < cnt; i += blockDim.x) bad |= f[i - 1] >= f[i];
    if (bad) atomicOr(st.flags + 3, 1u);
    if (st.track_bits) {
        unsigned long long pop = 0;
        for (uint32_t i = threadIdx.x; i < st.n; i += blockDim.x) pop += hist_bit(st, i, t) ? 1 : 0;
        atomicAdd(&s_pop, pop);
        __syncthreads();
        if (threadIdx.x == 0 && s_pop != cnt) atomicOr(st.flags + 3, 2u);
    }
}

// ------------------------------------------------------------- catch-up
// mode 0: frame(due) U expiring through t;  mode 1 (flush): every neuron through t-1
template <class M>
__global__ void k_catchup(M model, engine_state<M> st, int mode) {
    using SF = typename synapse_fields_of<M>::type;
    const int64_t t = *st.t_dev;
    const int64_t through = mode == 0 ? t : t - 1;
    const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
    uint32_t ntr = 0, total;
    const uint32_t* frame = nullptr;
    if (mode == 0) {
        if (due >= 0) {
            frame = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
            ntr = st.qcount[due % st.Q];
        }
        total = ntr + *st.expiring_count;  // (k_update counts the expiring neurons)
    } else {
        total = st.n;
    }
    // one CTA per neuron (grid-stride): its synapses replay blockDim.x at a
    // time, so the serial replay chains of many synapses overlap
    constexpr uint32_t kMaxWords = 4;
    for (uint32_t k = blockIdx.x; k < total; k += gridDim.x) {
        const uint32_t nid = mode == 1 ? k : (k < ntr ? frame[k] : st.expiring[k - ntr]);
        const int64_t a0 = st.ages[nid];
        if (a0 > through) continue;
        const uint32_t d = st.degree[nid];
        const uint32_t* row = st.cells + static_cast<uint64_t>(nid) * st.pitch;
        const uint64_t base = static_cast<uint64_t>(nid) * st.deg_max;
        uint64_t pre[kMaxWords];
        const uint32_t W = st.hist_words;
#pragma unroll
        for (uint32_t w = 0; w < kMaxWords; ++w)
            pre[w] = w < W ? st.hist[static_cast<uint64_t>(nid) * W + w] : 0;
        for (uint32_t kk = threadIdx.x; kk < d; kk += blockDim.x) {
            const uint32_t dst = row[kk];
            uint64_t post[kMaxWords];
#pragma unroll
            for (uint32_t w = 0; w < kMaxWords; ++w)
                post[w] = w < W ? st.hist[static_cast<uint64_t>(dst) * W + w] : 0;
            synapse_state<SF> s;
            load_syn(st.sf, base + kk, s);
            const synapse_state<SF> s0 = s;
            s.src_ = nid;
            s.dst_ = dst;
            // replay [a0, through]: ring positions advance incrementally (no
            // 64-bit modulo per step); words picked from registers
            const uint32_t HB = 64u * W;
            int64_t upre = a0 - static_cast<int64_t>(st.delay);
            uint32_t sp = static_cast<uint32_t>(a0 % HB);
            uint32_t spre = upre >= 0 ? static_cast<uint32_t>(upre % HB) : 0u;
            auto pick = [](const uint64_t* w, uint32_t slot) {
                const uint32_t q = slot >> 6;
                const uint64_t v = q == 0 ? w[0] : (q == 1 ? w[1] : (q == 2 ? w[2] : w[3]));
                return ((v >> (slot & 63)) & 1ull) != 0;
            };
            for (int64_t u = a0; u <= through; ++u) {
                const bool pb = upre >= 0 && pick(pre, spre);
                model.update_synapse(s, pb, pick(post, sp), st.dt);
                sp = sp + 1 == HB ? 0u : sp + 1;
                if (upre >= 0) spre = spre + 1 == HB ? 0u : spre + 1;
                ++upre;
            }
            store_syn_changed(st.sf, base + kk, s, s0);
        }
        if (threadIdx.x == 0) {
            atomicAdd(&st.counters[C_SYN_UPDATES],
                      static_cast<unsigned long long>(d) * static_cast<unsigned long long>(through - a0 + 1));
            st.ages[nid] = static_cast<uint32_t>(through + 1);
        }
    }
}

// Catch-up for one-word histories (history <= 64 steps, the default 50):
// the replay window [a0, through] is at most 64 steps, so the pre and post
// bits of the whole window are two register words rotated to start at a0;
// between events the model is stepped with (false, false) in a tight loop
// (for STDP: two multiplies per step).  A model exposing
// plastic(src, dst) declares update_synapse a no-op for the other synapses
// (benchmarks.hpp brunel_plus_model), which are skipped.  Same results as
// k_catchup, bit for bit.
SYNQ_DEV uint64_t rotr64(uint64_t x, uint32_t r) { return r ? (x >> r) | (x << (64 - r)) : x; }

// pre bits of a replay window of n <= 64 steps from a0 (source history word
// hw): bit j = the source spiked at a0 + j - delay (< 0: false)
SYNQ_DEV uint64_t catchup_prew(uint64_t hw, int64_t a0, uint32_t delay, uint32_t n) {
    const uint64_t lastn = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    const int64_t p0 = a0 - static_cast<int64_t>(delay);
    uint64_t prew = 0;
    if (n <= 64 && p0 + static_cast<int64_t>(n) > 0) {
        if (p0 >= 0) {
            prew = rotr64(hw, static_cast<uint32_t>(p0 % 64));
        } else {
            const uint32_t neg = static_cast<uint32_t>(-p0);  // leading steps with u - delay < 0
            prew = neg >= 64 ? 0ull : (hw << neg);             // bit j <- slot j - neg = u - delay
        }
    }
    return prew & lastn;
}

// trace-STDP catch-up of one plastic synapse (rs -> rd) over the window from
// a0: the traces are the neurons' P_src / Q_dst (trace_stdp), so only the
// weight moves, at the window's events, with the decayed traces stdp_step
// sees there (lif.hpp:78-89)
template <class M>
SYNQ_DEV float trace_catchup_weight(const engine_state<M>& st, const stdp_params& sp, uint32_t rs, uint32_t rd, int64_t a0,
                                    uint64_t prew, uint64_t postu, float w) {
    const uint64_t rn = st.n;  // step-major rings: [slot * n + neuron]
    for (uint64_t ev = prew | postu; ev; ev &= ev - 1) {
        const uint32_t e = static_cast<uint32_t>(__ffsll(static_cast<long long>(ev))) - 1;
        const uint32_t um = static_cast<uint32_t>(a0 + e - 1) & (kTraceRing - 1);
        if ((prew >> e) & 1ull) {
            const float qt = st.tr_q[um * rn + rd] * sp.decay_minus;
            w = clamp_weight(w - sp.a_minus * qt, sp.w_min, sp.w_max);
        }
        if ((postu >> e) & 1ull) {
            const float pt = st.tr_p[um * rn + rs] * sp.decay_plus;
            w = clamp_weight(w + sp.a_plus * pt, sp.w_min, sp.w_max);
        }
    }
    return w;
}

// the catch-up list of step t: frame(due) U expiring (mode 0), or every
// neuron (mode 1, flush through t - 1)
template <class M>
struct catchup_list {
    const uint32_t* frame = nullptr;
    uint32_t ntr = 0, total = 0;
    int64_t through = 0;
    // part 0: the whole list; 1: frame(due) only; 2: the expiring neurons
    // only, with t and their count from split_param (written by part 1: the
    // expiring part may run beside the receive, whose epilogue advances t);
    // 3: the expiring neurons only (frame(due) is caught up inside k_recv_win)
    int part = 0;
    SYNQ_DEV void load(const engine_state<M>& st, int mode, int64_t t, int part_ = 0) {
        part = part_;
        through = mode == 0 ? t : t - 1;
        if (mode == 0 && (part == 2 || part == 3)) {
            frame = nullptr;
            ntr = 0;
            total = part == 2 ? static_cast<uint32_t>(st.split_param[1]) : *st.expiring_count;
            return;
        }
        if (mode == 0) {
            const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
            if (due >= 0) {
                frame = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
                ntr = st.qcount[due % st.Q];
            }
            total = part == 1 ? ntr : ntr + *st.expiring_count;
        } else {
            total = st.n;
            ntr = 0;
            frame = nullptr;
        }
    }
    SYNQ_DEV uint32_t at(const engine_state<M>& st, int mode, uint32_t k) const {
        if (mode == 1) return k;
        if (part >= 2) return st.expiring[k];
        return k < ntr ? frame[k] : st.expiring[k - ntr];
    }
};

// ages of the caught-up neurons: through + 1 (engine.hpp:434); strided over
// the calling grid (after every catch-up item of the step has run)
template <class M>
SYNQ_DEV void advance_ages(const engine_state<M>& st, const catchup_list<M>& cl, int mode) {
    for (uint32_t kq = blockIdx.x * blockDim.x + threadIdx.x; kq < cl.total; kq += gridDim.x * blockDim.x) {
        const uint32_t nid = cl.at(st, mode, kq);
        if (static_cast<int64_t>(st.ages[nid]) <= cl.through) st.ages[nid] = static_cast<uint32_t>(cl.through + 1);
    }
}

// replay one synapse over n <= 64 steps from pre / post bit windows
template <class M, class SS>
SYNQ_DEV void replay_window(const M& model, SS& sv, uint64_t prew, uint64_t postw, uint32_t n, float dt) {
    uint64_t ev = prew | postw;
    uint32_t j = 0;
    while (j < n) {
        const uint32_t e = ev ? static_cast<uint32_t>(__ffsll(static_cast<long long>(ev))) - 1 : n;
#pragma unroll 4
        for (; j < e; ++j) model.update_synapse(sv, false, false, dt);
        if (e < n) {
            model.update_synapse(sv, ((prew >> e) & 1ull) != 0, ((postw >> e) & 1ull) != 0, dt);
            ev &= ev - 1;
            j = e + 1;
        }
    }
}

// U: synapses per lane (loads batched); MINB: CTAs per SM the registers allow
template <class M, bool kCompact = false, int U = 4, int MINB = 4>
__global__ void __launch_bounds__(256, MINB) k_catchup1(M model, engine_state<M> st, int mode, int part) {
    using SF = typename synapse_fields_of<M>::type;
    grid_launch_dependents();  // k_recv_win may start its prologue on SMs this grid frees
    grid_dependency_wait();    // PDL: k_update (and its ballots) are complete
    const int64_t t = part == 2 ? static_cast<int64_t>(st.split_param[0]) : *st.t_dev;
    if (part == 1 && blockIdx.x == 0 && threadIdx.x == 0) {  // parameters of the expiring part
        st.split_param[0] = static_cast<unsigned long long>(t);
        st.split_param[1] = *st.expiring_count;
    }
    if constexpr (kCompact) compact_tiles<M, 256>(st, t);
    catchup_list<M> cl;
    cl.load(st, mode, t, part);  // (k_update counts the expiring neurons)
    const int64_t through = cl.through;
    // work item = (neuron, chunk of U x 32 synapses), one per warp: many
    // items' load chains in flight per SM; ages advance later
    constexpr uint32_t CH = U * 32;
    const uint32_t lane = lane_id();
    const uint32_t mc = (st.deg_max + CH - 1) / CH;
    const uint64_t items = static_cast<uint64_t>(cl.total) * mc;
    const uint64_t wstride = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += wstride) {
        const uint32_t kq = static_cast<uint32_t>(it / mc), ch = static_cast<uint32_t>(it - uint64_t(kq) * mc);
        const uint32_t nid = cl.at(st, mode, kq);
        // a row without a plastic synapse: every update_synapse is a no-op,
        // only its counter and age move (chunk 0, one lane)
        // one round of independent loads per item: row flags, age, degree,
        // history word, the chunk's row targets (the padded row is readable up
        // to the pitch) and synapse state (up to deg_max); then the targets'
        // history words
        const uint32_t k0 = ch * CH + lane;
        const uint32_t* row = st.cells + static_cast<uint64_t>(nid) * st.pitch;
        const bool plastic_row = !st.row_plastic || st.row_plastic[nid];
        const int64_t a0 = st.ages[nid];
        const uint32_t d = st.degree[nid];
        const uint64_t hw = st.hist[nid];
        uint32_t dst[U];
        synapse_state<SF> sv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t kk = k0 + u * 32;
            dst[u] = kk < st.pitch ? row[kk] : 0xffffffffu;
            if (kk < st.deg_max) {
                const uint64_t si = static_cast<uint64_t>(nid) * st.deg_max + kk;
                if constexpr (model_trace_stdp<M>()) {
                    if (st.tr_p)  // the traces come from the rings: only the weight is read
                        sv[u].template get<trace_stdp<M>::W>() = st.sf.template get<trace_stdp<M>::W>()[si];
                    else
                        load_syn(st.sf, si, sv[u]);
                } else {
                    load_syn(st.sf, si, sv[u]);
                }
            }
        }
        if (!plastic_row && (ch != 0 || lane != 0)) continue;
        if (a0 > through) continue;
        const uint32_t n = static_cast<uint32_t>(through - a0 + 1);  // <= 64 under the expiry rule
        if (ch == 0 && lane == 0) {
            atomicAdd(&st.counters[C_SYN_UPDATES], static_cast<unsigned long long>(d) * n);
            if (mode == 0) st.caught[nid] = 1;
        }
        if (!plastic_row) continue;
        if (k0 >= d) continue;
        const uint64_t lastn = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
        // pre bits: u - delay for u in [a0, through]; u - delay < 0 is false
        const uint64_t prew = catchup_prew(hw, a0, st.delay, n);
        const uint32_t r0 = static_cast<uint32_t>(a0 % 64);
        bool on[U];
        uint64_t postw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            on[u] = k0 + u * 32 < d;
            if constexpr (model_has_plastic<M>()) on[u] = on[u] && model.plastic(nid, dst[u]);
            postw[u] = on[u] ? st.hist[dst[u]] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!on[u]) continue;
            if constexpr (model_has_plastic<M>()) __builtin_assume(model.plastic(nid, dst[u]));
            const synapse_state<SF> s0 = sv[u];
            sv[u].src_ = nid;
            sv[u].dst_ = dst[u];
            if (n > 64) {  // not reached under the expiry rule; replayed step by step if it is
                for (int64_t x = a0; x <= through; ++x)
                    model.update_synapse(sv[u], hist_bit(st, nid, x - static_cast<int64_t>(st.delay)),
                                         hist_bit(st, dst[u], x), st.dt);
            } else if (model_trace_stdp<M>() && st.tr_p) {
                if constexpr (model_trace_stdp<M>()) {
                    using T = trace_stdp<M>;
                    const uint64_t rs = nid, rd = dst[u], rn = st.n;  // step-major rings: [slot * n + neuron]
                    const uint64_t postu = rotr64(postw[u], r0) & lastn;
                    const float w = trace_catchup_weight(st, T::params(model), nid, dst[u], a0, prew, postu,
                                                         sv[u].template get<T::W>());
                    const uint32_t ut = static_cast<uint32_t>(through) & (kTraceRing - 1);
                    sv[u].template get<T::W>() = w;
                    sv[u].template get<T::PT>() = st.tr_p[ut * rn + rs];
                    sv[u].template get<T::QT>() = st.tr_q[ut * rn + rd];
                }
            } else {
                replay_window(model, sv[u], prew, rotr64(postw[u], r0) & lastn, n, st.dt);
            }
            if (model_trace_stdp<M>() && st.tr_p)
                store_syn(st.sf, static_cast<uint64_t>(nid) * st.deg_max + k0 + u * 32, sv[u]);
            else
                store_syn_changed(st.sf, static_cast<uint64_t>(nid) * st.deg_max + k0 + u * 32, sv[u], s0);
        }
    }
}

// pending k_catchup1 ages (caught flags) applied outside a step: before a
// flush and when run() returns (host reads of ages)
template <class M>
__global__ void k_apply_caught(engine_state<M> st) {
    const int64_t t = *st.t_dev;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += gridDim.x * blockDim.x)
        if (st.caught[i]) {
            st.caught[i] = 0;
            st.ages[i] = static_cast<uint32_t>(t);
        }
}

template <class M>
__global__ void k_catchup_ages(engine_state<M> st, int mode) {
    catchup_list<M> cl;
    cl.load(st, mode, *st.t_dev);
    advance_ages(st, cl, mode);
}

// ------------------------------------------------------------- receive
template <class M>
SYNQ_DEV void deliver(const M& model, const engine_state<M>& st, uint32_t src, uint32_t k,
                      uint32_t to_id) {
    using NF = typename M::neuron_fields;
    using SF = typename synapse_fields_of<M>::type;
    global_neuron<NF, true> from{src, st.nf, st.rng};
    global_neuron<NF, true> to{to_id, st.nf, st.rng};
    if constexpr (synapse_fields_of<M>::present) {
        global_synapse<SF> syn{static_cast<uint64_t>(src) * st.deg_max + k, src, to_id, st.sf};
        model.receive(from, to, syn);
    } else {
        model.receive(from, to);
    }
}

constexpr uint32_t kChunk = 256;  // targets per (spike, chunk) work item

template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_receive(M model, engine_state<M> st) {
    const int64_t t = *st.t_dev;
    const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
    unsigned long long mine = 0;
    if (due >= 0) {
        const uint32_t S = st.qcount[due % st.Q];
        const uint32_t* spikes = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
        const uint32_t mc = (st.deg_max + kChunk - 1) / kChunk;
        const uint64_t items = static_cast<uint64_t>(S) * mc;
        const uint32_t lane = lane_id();
        const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(BLOCK) + threadIdx.x) >> 5;
        const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * BLOCK) >> 5;
        for (uint64_t w = warp; w < items; w += nwarps) {
            const uint32_t src = spikes[w / mc];
            const uint32_t c = static_cast<uint32_t>(w % mc);
            const uint32_t d = st.degree[src];
            const uint32_t beg = c * kChunk;
            if (beg >= d) continue;
            const uint32_t end = min(d, beg + kChunk);
            const uint32_t* row = st.cells + static_cast<uint64_t>(src) * st.pitch;
            for (uint32_t k = beg + lane; k < end; k += 32) deliver(model, st, src, k, row[k]);
            if (c == 0 && lane == 0) mine += d;
        }
        for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if (lane == 0 && mine) atomicAdd(&st.counters[C_DELIVERIES], mine);
    }
    step_epilogue(st, t);
}

// ---- ordered windowed delivery (exact, the default for the generic engine)
// CTA c owns the targets [lo[c], lo[c+1]) and keeps their state in registers
// (thread j: targets j, j + BLOCK, ...).  Per chunk of the due frame's spikes
// (ascending ids) it stages the spikes' row segments inside its window
// (split[s][c] .. split[s][c+1], like the persistent engine) together with
// the synapse state they read, buckets the events by target in ascending
// spike order (rank = popcount of the target's spike bitmask below the
// spike: order-free to build), and each thread then applies its targets'
// events in that order through model.receive.  That is the reference's
// sequential accumulation order per target (engine.hpp:384-404), so the
// result is bit-identical to its deterministic mode, with no device atomics
// on neuron state and no sort.
struct recv_win {
    const uint32_t* lo;     // [C + 1] window bounds (lo[C] = n)
    const uint32_t* split;  // [n][C + 1] row position of the first target >= lo[c]
    uint32_t C;
    uint32_t wmax;  // largest window (<= kWinTPT * block)
    uint32_t ecap;  // events staged per chunk
    uint32_t ages;  // advance the ages of the step's k_catchup1 list first
    // trace-STDP models: catch up the due frame's rows inside the receive,
    // window by window (k_catchup1 then takes the expiring neurons only)
    uint32_t catchup;
};
constexpr int kWinTPT = 2;      // targets per thread (1024-thread CTAs)
constexpr int kWinSpikes = 256;  // spikes per chunk (8 mask words per target)

// synapse handle on the staged copy of an event's synapse state
template <class FieldList>
struct staged_synapse {
    uint32_t e_, src_, dst_;
    unsigned char* base_;
    uint32_t ecap_;
    SYNQ_HD uint32_t src() const { return src_; }
    SYNQ_HD uint32_t dst() const { return dst_; }
    template <size_t I>
    SYNQ_HD auto& get() const {
        return reinterpret_cast<field_t<I, FieldList>*>(base_ + staged_offset<I>(ecap_))[e_];
    }
    template <size_t I>
    SYNQ_HD static size_t staged_offset(uint32_t ecap) {
        if constexpr (I == 0)
            return 0;
        else
            return staged_offset<I - 1>(ecap) + ((sizeof(field_t<I - 1, FieldList>) * ecap + 15) & ~size_t(15));
    }
};
// stage synapse i's fields at e (working copy) and e + half (original)
template <class FieldList, size_t I = 0>
SYNQ_DEV void stage_syn(const field_ptrs<FieldList>& f, uint64_t i, unsigned char* base, uint32_t ecap2, uint32_t e,
                        uint32_t half) {
    if constexpr (I < FieldList::count) {
        using T = field_t<I, FieldList>;
        T* a = reinterpret_cast<T*>(base + staged_synapse<FieldList>::template staged_offset<I>(ecap2));
        const T x = f.template get<I>()[i];
        a[e] = x;
        a[e + half] = x;
        stage_syn<FieldList, I + 1>(f, i, base, ecap2, e, half);
    }
}
// staged arrays hold 2 x half entries per field: [0, half) working copies,
// [half, 2 half) the originals
template <class FieldList, size_t I = 0>
SYNQ_DEV void unstage_syn(const field_ptrs<FieldList>& f, uint64_t i, const unsigned char* base, uint32_t ecap2,
                          uint32_t e, uint32_t half) {
    if constexpr (I < FieldList::count) {
        using T = field_t<I, FieldList>;
        const T* a = reinterpret_cast<const T*>(base + staged_synapse<FieldList>::template staged_offset<I>(ecap2));
        if (!same_bits(a[e], a[e + half])) f.template get<I>()[i] = a[e];
        unstage_syn<FieldList, I + 1>(f, i, base, ecap2, e, half);
    }
}

// fused catch-up + weight staging for up to 4 events per thread (events
// e = e_first + u * stride): the synapse of event e is caught up through t
// exactly as k_catchup1 does (trace-STDP: weight moved at the window's events,
// PT / QT = P_src(t) / Q_dst(t) stored; replay beyond 64 steps is not reached
// under the expiry rule and replays step by step if it is), then its weight
// is staged for the receive.  Loads of the four events go out together.
template <class M>
SYNQ_DEV void fused_catchup_stage(const M& model, const engine_state<M>& st, const uint32_t* s_spk, const uint32_t* s_cu_n,
                                  const uint32_t* s_cu_a0, const unsigned long long* s_cu_prew, const float* s_cu_pt,
                                  const uint32_t (&ej)[4], const uint32_t (&ek)[4], const uint32_t (&tg)[4],
                                  uint32_t e_first, uint32_t stride, uint32_t E, int64_t t, uint32_t ut, float* s_w) {
    if constexpr (model_trace_stdp<M>()) {
        using T = trace_stdp<M>;
        using SF = typename synapse_fields_of<M>::type;
        float w[4], qn[4];
        uint64_t post[4];
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t e = e_first + u * stride;
            on[u] = false;
            if (e < E) {
                const uint32_t j = ej[u], src = s_spk[j];
                const uint64_t si = static_cast<uint64_t>(src) * st.deg_max + ek[u];
                w[u] = st.sf.template get<T::W>()[si];
                on[u] = s_cu_n[j] != 0;
                if constexpr (model_has_plastic<M>()) on[u] = on[u] && model.plastic(src, tg[u]);
                if (on[u]) {
                    post[u] = st.hist[tg[u]];
                    qn[u] = st.tr_q[static_cast<uint64_t>(ut) * st.n + tg[u]];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t e = e_first + u * stride;
            if (e >= E) continue;
            if (on[u]) {
                if constexpr (model_has_plastic<M>()) __builtin_assume(model.plastic(s_spk[ej[u]], tg[u]));
                const uint32_t j = ej[u], src = s_spk[j], n = s_cu_n[j];
                const int64_t a0 = s_cu_a0[j];
                const uint64_t si = static_cast<uint64_t>(src) * st.deg_max + ek[u];
                if (n <= 64) {
                    const uint64_t lastn = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
                    const uint64_t postu = rotr64(post[u], static_cast<uint32_t>(a0 % 64)) & lastn;
                    w[u] = trace_catchup_weight(st, T::params(model), src, tg[u], a0, s_cu_prew[j], postu, w[u]);
                    st.sf.template get<T::W>()[si] = w[u];
                    st.sf.template get<T::PT>()[si] = s_cu_pt[j];
                    st.sf.template get<T::QT>()[si] = qn[u];
                } else {
                    synapse_state<SF> sv;
                    load_syn(st.sf, si, sv);
                    sv.src_ = src;
                    sv.dst_ = tg[u];
                    for (int64_t x = a0; x <= t; ++x)
                        model.update_synapse(sv, hist_bit(st, src, x - static_cast<int64_t>(st.delay)),
                                             hist_bit(st, tg[u], x), st.dt);
                    store_syn(st.sf, si, sv);
                    w[u] = sv.template get<T::W>();
                }
            }
            s_w[e] = w[u];
        }
    }
}

template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_recv_win(M model, engine_state<M> st, recv_win rw) {
    using NF = typename M::neuron_fields;
    using SF = typename synapse_fields_of<M>::type;
    constexpr bool kSyn = synapse_fields_of<M>::present;
    constexpr bool kWOnly = kSyn && model_receive_weight_only<M>();
    constexpr bool kFuse = kWOnly && model_trace_stdp<M>();
    constexpr int NW = BLOCK / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_spk[kWinSpikes], s_sb[kWinSpikes], s_off[kWinSpikes + 1];
    // fused catch-up: per spike of the chunk, its replay window (steps, start, pre bits) and P_src(t)
    constexpr int kCu = kFuse ? kWinSpikes : 1;
    __shared__ uint32_t s_cu_n[kCu], s_cu_a0[kCu];
    __shared__ unsigned long long s_cu_prew[kCu];
    __shared__ float s_cu_pt[kCu];
    __shared__ uint32_t s_tmp[NW + 1];
    __shared__ uint32_t s_take;
    const uint32_t wmax = rw.wmax, ecap = rw.ecap;
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem);  // wmax
    uint32_t* s_toff = s_tcnt + wmax;                      // wmax
    uint32_t* s_mask = s_toff + wmax;                      // wmax x 8
    uint32_t* s_ev = s_mask + 8 * wmax;                    // ecap: row position k | spike << 24
    uint32_t* s_et = s_ev + ecap;                          // ecap: local target
    uint32_t* s_ord = s_et + ecap;                         // ecap: events by (target, spike)
    unsigned char* s_syn = reinterpret_cast<unsigned char*>(s_ord + ecap);

    grid_launch_dependents();  // the next step's k_update may be scheduled early (it waits first)
    const int64_t t = *st.t_dev;
    const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, C = rw.C;

    const uint32_t lo = rw.lo[c], wn = rw.lo[c + 1] - lo;
    unsigned long long mine = 0;
    const bool fuse = kFuse && rw.catchup != 0;
    const uint32_t ut = static_cast<uint32_t>(t) & (kTraceRing - 1);
    if constexpr (kFuse) {
        if (fuse && due >= 0) {
            // the due frame's rows are caught up through t below, each window
            // by its CTA; their synapse-update counters and caught flags once
            // per row here (k_catchup1 semantics, engine.hpp:414-436)
            const uint32_t S = st.qcount[due % st.Q];
            const uint32_t* spikes = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
            for (uint32_t k = c * BLOCK + tid; k < S; k += C * BLOCK) {
                const uint32_t sid = spikes[k];
                const int64_t a0 = st.ages[sid];
                if (a0 <= t) {
                    atomicAdd(&st.counters[C_SYN_UPDATES],
                              static_cast<unsigned long long>(st.degree[sid]) * static_cast<unsigned long long>(t - a0 + 1));
                    st.caught[sid] = 1;
                }
            }
        }
    }
    if (due >= 0 && wn > 0) {
        const uint32_t S = st.qcount[due % st.Q];
        const uint32_t* spikes = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
        values_t<NF> v[kWinTPT], v0[kWinTPT];
        xorshift rr[kWinTPT];
        bool live[kWinTPT];
#pragma unroll
        for (int r = 0; r < kWinTPT; ++r) {
            live[r] = false;
            const uint32_t j = tid + r * BLOCK;
            if (j < wn) load_all(st.nf, lo + j, v[r]);
            v0[r] = v[r];
        }
        for (uint32_t g0 = 0; g0 < S;) {
            const uint32_t m = min(static_cast<uint32_t>(kWinSpikes), S - g0);
            // (1) the spikes' segments in this window; exclusive scan of their sizes
            uint32_t cnt = 0;
            if (tid < m) {
                const uint32_t sid = spikes[g0 + tid];
                const uint32_t* sp = rw.split + static_cast<uint64_t>(sid) * (C + 1) + c;
                const uint32_t sb = sp[0];
                cnt = sp[1] - sb;
                s_spk[tid] = sid;
                s_sb[tid] = sb;
                if constexpr (kFuse) {
                    if (fuse) {  // the row's replay window [a0, t] (k_catchup1)
                        const int64_t a0 = st.ages[sid];
                        const bool on = (!st.row_plastic || st.row_plastic[sid]) && a0 <= t;
                        const uint32_t n = on ? static_cast<uint32_t>(t - a0 + 1) : 0u;
                        s_cu_n[tid] = n;
                        s_cu_a0[tid] = static_cast<uint32_t>(a0);
                        s_cu_prew[tid] = on ? catchup_prew(st.hist[sid], a0, st.delay, n) : 0ull;
                        s_cu_pt[tid] = st.tr_p[static_cast<uint64_t>(ut) * st.n + sid];
                    }
                }
            }
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= static_cast<uint32_t>(o)) incl += y;
            }
            if (lane == 31) s_tmp[warp] = incl;
            for (uint32_t x = tid; x < wn; x += BLOCK) s_tcnt[x] = 0;
            for (uint32_t x = tid; x < 8 * wn; x += BLOCK) s_mask[x] = 0;
            __syncthreads();
            if (warp == 0) {
                const uint32_t w = lane < NW ? s_tmp[lane] : 0u;
                uint32_t wi = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= static_cast<uint32_t>(o)) wi += y;
                }
                if (lane < NW) s_tmp[lane] = wi - w;
            }
            __syncthreads();
            if (tid < kWinSpikes) s_off[tid + 1] = s_tmp[warp] + incl;
            if (tid == 0) s_off[0] = 0;
            __syncthreads();
            // take the longest spike prefix whose events fit (at least one spike)
            if (tid < m && s_off[tid] <= ecap && (tid + 1 == m || s_off[tid + 1] > ecap))
                s_take = s_off[tid + 1] <= ecap ? tid + 1 : max(1u, tid);
            __syncthreads();
            const uint32_t mt = s_take, E = s_off[mt];
            // (2) events, one per thread (spike found by binary search over
            // the segment offsets), up to 4 per thread with their loads in
            // flight together; the synapse state is staged twice (working
            // copy + original, so write-back needs no global reads)
            for (uint32_t e0 = 0; e0 < E; e0 += 4 * BLOCK) {
                uint32_t ej[4], ek[4], tg[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * BLOCK + tid;
                    tg[u] = 0;
                    if (e < E) {
                        uint32_t a = 0, z = mt;  // last j with s_off[j] <= e
                        while (z - a > 1) {
                            const uint32_t mid = (a + z) >> 1;
                            if (s_off[mid] <= e)
                                a = mid;
                            else
                                z = mid;
                        }
                        ej[u] = a;
                        ek[u] = s_sb[a] + (e - s_off[a]);
                        tg[u] = st.cells[static_cast<uint64_t>(s_spk[a]) * st.pitch + ek[u]];
                    }
                }
                // the synapse state of the due spikes' rows is the catch-up's
                // output: with programmatic dependent launch this kernel got
                // here while k_catchup1 was still running
                if constexpr (kSyn) {
                    // (fused: the frame's rows are this kernel's own: no wait)
                    if (g0 == 0 && e0 == 0 && !fuse) grid_dependency_wait();
                    if constexpr (kFuse) {
                        if (fuse) {
                            fused_catchup_stage<M>(model, st, s_spk, s_cu_n, s_cu_a0, s_cu_prew, s_cu_pt, ej, ek, tg,
                                                   e0 + tid, BLOCK, E, t, ut,
                                                   reinterpret_cast<field_t<0, SF>*>(s_syn));
                        }
                    }
                    if (!fuse) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t e = e0 + u * BLOCK + tid;
                            if (e < E) {
                                const uint64_t si = static_cast<uint64_t>(s_spk[ej[u]]) * st.deg_max + ek[u];
                                if constexpr (kWOnly)
                                    reinterpret_cast<field_t<0, SF>*>(s_syn)[e] = st.sf.template get<0>()[si];
                                else
                                    stage_syn(st.sf, si, s_syn, 2 * ecap, e, ecap);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * BLOCK + tid;
                    if (e < E) {
                        const uint32_t j = ej[u], tl = tg[u] - lo;
                        s_ev[e] = ek[u] | (j << 24);
                        s_et[e] = tl;
                        atomicAdd(&s_tcnt[tl], 1u);
                        atomicOr(&s_mask[tl * 8 + (j >> 5)], 1u << (j & 31));
                    }
                }
            }
            __syncthreads();
            // (3) target offsets (exclusive scan over the window)
            uint32_t carry = 0;
            for (uint32_t b0 = 0; b0 < wn; b0 += BLOCK) {
                const uint32_t x = b0 + tid < wn ? s_tcnt[b0 + tid] : 0u;
                uint32_t in2 = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, in2, o);
                    if (lane >= static_cast<uint32_t>(o)) in2 += y;
                }
                if (lane == 31) s_tmp[warp] = in2;
                __syncthreads();
                if (warp == 0) {
                    const uint32_t w = lane < NW ? s_tmp[lane] : 0u;
                    uint32_t wi = w;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                        if (lane >= static_cast<uint32_t>(o)) wi += y;
                    }
                    if (lane < NW) s_tmp[lane] = wi - w;
                    if (lane == 31) s_tmp[NW] = wi;
                }
                __syncthreads();
                if (b0 + tid < wn) s_toff[b0 + tid] = carry + s_tmp[warp] + in2 - x;
                carry += s_tmp[NW];
                __syncthreads();
            }
            // (4) stable placement: rank = earlier spikes of this chunk hitting the target
            for (uint32_t e = tid; e < E; e += BLOCK) {
                const uint32_t tl = s_et[e], j = s_ev[e] >> 24;
                const uint32_t* mk = s_mask + tl * 8;
                uint32_t rank = __popc(mk[j >> 5] & ((1u << (j & 31)) - 1u));
                for (uint32_t w = 0; w < (j >> 5); ++w) rank += __popc(mk[w]);
                s_ord[s_toff[tl] + rank] = e;
            }
            __syncthreads();
            // (5) apply, per target in ascending spike order
#pragma unroll
            for (int r = 0; r < kWinTPT; ++r) {
                const uint32_t j = tid + r * BLOCK;
                if (j >= wn) continue;
                const uint32_t b = s_toff[j], ne = s_tcnt[j];
                local_neuron<NF> to{lo + j, &v[r], &rr[r], &live[r], st.rng};
                for (uint32_t x = b; x < b + ne; ++x) {
                    const uint32_t e = s_ord[x], jj = s_ev[e] >> 24;
                    const uint32_t src = s_spk[jj];
                    global_neuron<NF, false> from{src, st.nf, st.rng};
                    if constexpr (kSyn) {
                        staged_synapse<SF> syn{e, src, lo + j, s_syn, 2 * ecap};
                        model.receive(from, to, syn);
                    } else {
                        model.receive(from, to);
                    }
                }
            }
            __syncthreads();
            // (6) synapse state written by receive (if any) goes back
            if constexpr (kSyn && !kWOnly) {
                for (uint32_t e = tid; e < E; e += BLOCK) {
                    const uint32_t j = s_ev[e] >> 24, k = s_ev[e] & 0xffffffu;
                    unstage_syn(st.sf, static_cast<uint64_t>(s_spk[j]) * st.deg_max + k, s_syn, 2 * ecap, e, ecap);
                }
            }
            if (tid == 0) mine += E;
            __syncthreads();
            g0 += mt;
        }
#pragma unroll
        for (int r = 0; r < kWinTPT; ++r) {
            const uint32_t j = tid + r * BLOCK;
            if (j < wn) store_changed(st.nf, lo + j, v[r], v0[r]);
        }
        if (tid == 0 && mine) atomicAdd(&st.counters[C_DELIVERIES], mine);
    }
    grid_dependency_wait();  // the epilogue resets what the catch-up still reads (t, expiring count)
    step_epilogue(st, t);
}

// ---- ordered delivery: count -> (scan) -> scatter -> apply
template <class M, int BLOCK, bool kScatter>
__global__ void __launch_bounds__(BLOCK) k_det_events(engine_state<M> st) {
    const int64_t t = *st.t_dev;
    const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
    if (due < 0) return;
    const uint32_t S = st.qcount[due % st.Q];
    const uint32_t* spikes = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
    const uint32_t mc = (st.deg_max + kChunk - 1) / kChunk;
    const uint64_t items = static_cast<uint64_t>(S) * mc;
    const uint32_t lane = lane_id();
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(BLOCK) + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * BLOCK) >> 5;
    unsigned long long mine = 0;
    for (uint64_t w = warp; w < items; w += nwarps) {
        const uint32_t rank = static_cast<uint32_t>(w / mc);
        const uint32_t src = spikes[rank];
        const uint32_t c = static_cast<uint32_t>(w % mc);
        const uint32_t d = st.degree[src];
        const uint32_t beg = c * kChunk;
        if (beg >= d) continue;
        const uint32_t end = min(d, beg + kChunk);
        const uint32_t* row = st.cells + static_cast<uint64_t>(src) * st.pitch;
        for (uint32_t k = beg + lane; k < end; k += 32) {
            const uint32_t to = row[k];
            if constexpr (!kScatter) {
                atomicAdd(&st.det_cnt[to], 1u);
            } else {
                const unsigned long long pos =
                    static_cast<unsigned long long>(st.det_off[to]) + atomicAdd(&st.det_fill[to], 1u);
                if (pos < st.det_cap)
                    st.det_ev[pos] = (static_cast<unsigned long long>(rank) << 32) | k;
                else
                    st.flags[1] = 1;
            }
        }
        if (!kScatter && c == 0 && lane == 0) mine += d;
    }
    if constexpr (!kScatter) {
        for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if (lane == 0 && mine) atomicAdd(&st.counters[C_DELIVERIES], mine);
    }
}

template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_det_apply(M model, engine_state<M> st) {
    using NF = typename M::neuron_fields;
    using SF = typename synapse_fields_of<M>::type;
    const int64_t t = *st.t_dev;
    const int64_t due = t - static_cast<int64_t>(st.delay) + 1;
    if (due >= 0) {
        const uint32_t* spikes = st.queue + static_cast<uint64_t>(due % st.Q) * st.n;
        for (uint32_t j = blockIdx.x * BLOCK + threadIdx.x; j < st.n; j += gridDim.x * BLOCK) {
            const uint32_t c = st.det_cnt[j];
            if (c == 0) continue;
            unsigned long long* ev = st.det_ev + st.det_off[j];
            const unsigned long long room = st.det_cap - st.det_off[j];
            const uint32_t m = room < c ? static_cast<uint32_t>(room) : c;
            for (uint32_t a = 1; a < m; ++a) {  // insertion sort by (rank, k)
                const unsigned long long x = ev[a];
                uint32_t b = a;
                while (b > 0 && ev[b - 1] > x) {
                    ev[b] = ev[b - 1];
                    --b;
                }
                ev[b] = x;
            }
            global_neuron<NF, false> to{j, st.nf, st.rng};
            for (uint32_t a = 0; a < m; ++a) {
                const uint32_t rank = static_cast<uint32_t>(ev[a] >> 32);
                const uint32_t k = static_cast<uint32_t>(ev[a]);
                const uint32_t src = spikes[rank];
                global_neuron<NF, false> from{src, st.nf, st.rng};
                if constexpr (synapse_fields_of<M>::present) {
                    global_synapse<SF> syn{static_cast<uint64_t>(src) * st.deg_max + k, src, j, st.sf};
                    model.receive(from, to, syn);
                } else {
                    model.receive(from, to);
                }
            }
            st.det_cnt[j] = 0;
            st.det_fill[j] = 0;
        }
    }
    step_epilogue(st, t);
}

// exclusive scan of det_cnt into det_off (single block; each thread owns 16
// consecutive counts per round, so a 45K-neuron network takes 3 rounds, not
// 45; the ordered path is the reference's deterministic mode)
template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_det_scan(engine_state<M> st) {
    const int64_t t = *st.t_dev;
    if (t - static_cast<int64_t>(st.delay) + 1 < 0) return;
    constexpr uint32_t E = 16;  // counts per thread per round
    __shared__ uint32_t s_warp[BLOCK / 32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < st.n; base += BLOCK * E) {
        const uint32_t i0 = base + threadIdx.x * E;
        uint32_t c[E];
        uint32_t sum = 0;
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            c[e] = i0 + e < st.n ? st.det_cnt[i0 + e] : 0u;
            sum += c[e];
        }
        uint32_t incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < BLOCK / 32 ? s_warp[lane] : 0;
            uint32_t wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= static_cast<uint32_t>(o)) wi += y;
            }
            if (lane < BLOCK / 32) s_warp[lane] = wi - w;
        }
        __syncthreads();
        uint32_t run = s_carry + s_warp[warp] + incl - sum;
#pragma unroll
        for (uint32_t e = 0; e < E; ++e) {
            if (i0 + e < st.n) st.det_off[i0 + e] = run;
            run += c[e];
        }
        __syncthreads();
        if (threadIdx.x == BLOCK - 1) s_carry += s_warp[warp] + incl;
        __syncthreads();
    }
}

}  // namespace synq::dev
