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

#include <cstdint>

#include "synq/detail/device_refs.cuh"
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

    unsigned long long* counters;
    unsigned long long* tile_status;  // decoupled look-back, one word per id tile
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

template <class M>
SYNQ_DEV bool hist_bit(const engine_state<M>& st, uint32_t id, int64_t u) {
    if (u < 0) return false;
    const uint32_t slots = 64u * st.hist_words;
    const uint32_t slot = static_cast<uint32_t>(u % slots);
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
        for (uint32_t k = lane; k < d; k += 32) {
            global_synapse<SF> syn{static_cast<uint64_t>(s) * st.deg_max + k, s, row[k], st.sf};
            model.init_synapse(syn);
        }
    }
}

// ------------------------------------------------------------- update
template <class M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_update(M model, engine_state<M> st) {
    using NF = typename M::neuron_fields;
    constexpr bool kSyn = synapse_fields_of<M>::present;
    constexpr int NW = BLOCK / 32;
    __shared__ uint32_t s_tile, s_base;
    __shared__ uint32_t s_warp[NW];
    __shared__ uint32_t s_meas;

    const int64_t t = *st.t_dev;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(&st.tile_ctr[t & 1], 1u);
        s_meas = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t i = tile * BLOCK + threadIdx.x;

    bool spk = false;
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
            const uint32_t slot = static_cast<uint32_t>(t % (64u * st.hist_words));
            uint64_t* w = st.hist + static_cast<uint64_t>(i) * st.hist_words + (slot >> 6);
            *w = (*w & ~(1ull << (slot & 63))) | (static_cast<uint64_t>(spk) << (slot & 63));
        }
        if constexpr (kSyn) {  // engine.hpp:318-330
            const bool transmits = (st.delay == 1) ? spk : hist_bit(st, i, t - st.delay + 1);
            if (!transmits && static_cast<int64_t>(st.ages[i]) + st.history <= t + st.delay + 1) {
                const uint32_t slot = atomicAdd(st.expiring_count, 1u);
                st.expiring[slot] = i;
            }
        }
    }

    // ordered compaction: warp ballots -> block scan -> look-back across tiles
    const unsigned ball = __ballot_sync(0xffffffffu, spk);
    if (lane == 0) s_warp[warp] = __popc(ball);
    const bool meas = spk && i >= st.meas_lo && i < st.meas_hi;
    const unsigned mball = __ballot_sync(0xffffffffu, meas);
    if (lane == 0 && mball) atomicAdd(&s_meas, __popc(mball));
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
        const uint32_t nex = *st.expiring_count;
        total = ntr + nex;
        if (blockIdx.x == 0 && threadIdx.x == 0 && nex) atomicAdd(&st.counters[C_EXPIRY], nex);
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
