#pragma once
// network<Model>: the reference's clock-driven simulator API
// (proj/include/synq/engine.hpp:46-471) backed by B200 device state.
//
// Same constructor, init/step/run/flush, accessors and spike tap.  What runs
// where:
//   construction  host degree plan + device expansion (csrc/construct.cu)
//   init          k_init_neurons / k_init_synapses
//   step / run    population-delivery models (vogels, brunel, and any user
//                 model specialising synq::population_delivery): ONE
//                 cooperative persistent launch per batch of steps
//                 (detail/persistent.cuh), bit-exact with the reference's
//                 deterministic mode.
//                 Every other model: a CUDA graph of per-step kernels
//                 (detail/kernels.cuh); deterministic mode (or threads == 1)
//                 selects ordered delivery, reproducing the reference's
//                 sequential float accumulation order exactly.
//   tap / spans   host mirrors synced lazily; the tap is replayed per batch
//                 from a device frame log, in step order, before run()
//                 returns.
//
// Compile translation units that include this header with nvcc
// (-std=c++20 --expt-relaxed-constexpr -fmad=false -gencode
// arch=compute_100a,code=sm_100a) and link libsynq.so.
#if !defined(__CUDACC__)
#error "synq/engine.hpp launches sm_100a kernels: compile this translation unit with nvcc"
#endif

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "synq/adjacency.hpp"
#include "synq/detail/cuda_util.hpp"
#include "synq/detail/device_graph.hpp"
#include "synq/detail/kernels.cuh"
#include "synq/detail/persistent.cuh"
#include "synq/detail/pipeline.cuh"
#include "synq/detail/solo.cuh"
#include "synq/detail/cluster.cuh"
#include "synq/detail/exchange.hpp"
#include "synq/models/benchmarks.hpp"
#include "synq/network_desc.hpp"
#include "synq/random.hpp"
#include "synq/soa.hpp"

namespace synq {

struct engine_options {
    uint64_t seed = 1;
    unsigned threads = 0;         // reference: CPU workers; here threads == 1 implies ordered delivery
    bool deterministic = false;   // ordered (reference-exact) delivery on the generic path
    uint32_t history_frames = 0;  // 0 = max(delay + 1, 50)
    uint32_t pitch_align = 32;    // 32 u32 = 128-byte rows
    bool debug_checks = false;    // per-batch frame checks (sorted / unique)
    // ---- B200 extensions
    uint32_t batch_steps = 0;  // steps per device batch (0 = auto)
    int persistent = -1;       // -1 auto, 0 never, 1 require (population-delivery models)
    uint32_t tiles = 0;        // persistent CTAs (0 = auto)
    bool profile = false;      // per-phase cycle counters in the persistent kernel
    int pipeline = -1;         // persistent kernel: -1 auto (pipelined when it fits), 0 serial, 1 pipelined
    uint32_t lead = 0;         // pipelined: frames the update may run ahead of delivery (0 = auto)
    // target-partitioned multi-GPU shard: this process owns
    // shard_rank of shard_world; frames are exchanged with export/import
    uint32_t shard_rank = 0;
    uint32_t shard_world = 1;
    // in-engine exchange: every shard passes the same NCCL unique id and the
    // engine allgathers the spike frames itself after every batch
    bool shard_nccl = false;
    std::array<char, 128> nccl_id{};
    // NVLink peer exchange: the step kernel stores this shard's frames
    // straight into every other shard's queue ring (peer-mapped memory), so
    // run() is one persistent launch per batch with no host exchange.
    // Connect with connect_peers (same process) or connect_peers_ipc; with
    // shard_nccl the engine exchanges the IPC handles over NCCL itself.
    bool shard_peer = false;
};

// one shard's peer-exchange buffers (device pointers in the owner's space)
struct peer_endpoint {
    uint32_t* queue = nullptr;
    unsigned long long* finfo = nullptr;
    uint32_t publishers = 0;
    uint32_t reserved = 0;
};
// cudaIpcMemHandle_t of the queue ring and of the frame words + publishers
constexpr size_t kPeerHandleBytes = 2 * 64 + 8;

struct engine_counters {
    uint64_t steps = 0;
    uint64_t spikes = 0;
    uint64_t deliveries = 0;
    uint64_t synapse_updates = 0;
    uint64_t expiry_batches = 0;
    uint64_t frames_consumed = 0;
};

struct phase_seconds {
    double construct = 0.0;
    double init_neurons = 0.0;
    double init_synapses = 0.0;
    double simulate = 0.0;
};

struct engine_memory {
    uint64_t neuron_fields = 0;
    uint64_t neuron_rng = 0;
    uint64_t spike_queues = 0;
    uint64_t spike_bitmasks = 0;
    uint64_t ages = 0;
    uint64_t expirations = 0;
    uint64_t adjacency = 0;
    uint64_t synapse_fields = 0;
    uint64_t total() const {
        return neuron_fields + neuron_rng + spike_queues + spike_bitmasks + ages + expirations +
               adjacency + synapse_fields;
    }
};

inline constexpr uint32_t lazy_history_default = 50;

namespace detail {
template <class M>
constexpr bool model_uses_rng() {
    return dev::model_uses_rng<M>();
}
template <class M, class = void>
struct population_ok : std::false_type {};
template <class M>
struct population_ok<M, std::enable_if_t<population_delivery<M>::available>> : std::true_type {};

template <class FieldList, size_t I = 0>
void alloc_fields(std::vector<dev_array<unsigned char>>& cols, dev::field_ptrs<FieldList>& ptrs,
                  size_t n, cudaStream_t s) {
    if constexpr (I < FieldList::count) {
        using T = field_t<I, FieldList>;
        cols[I].resize(std::max<size_t>(1, n) * sizeof(T));
        cols[I].zero(s);
        ptrs.p[I] = cols[I].get();
        alloc_fields<FieldList, I + 1>(cols, ptrs, n, s);
    }
}
template <class FieldList, size_t I = 0>
uint64_t field_bytes() {
    if constexpr (I < FieldList::count)
        return sizeof(field_t<I, FieldList>) + field_bytes<FieldList, I + 1>();
    else
        return 0;
}
}  // namespace detail

template <class Model>
class network {
public:
    using model_type = Model;
    using neuron_fields = typename Model::neuron_fields;
    using synapse_fields = typename dev::synapse_fields_of<Model>::type;
    static constexpr bool has_synapses = dev::synapse_fields_of<Model>::present;
    static constexpr bool uses_rng = detail::model_uses_rng<Model>();
    static constexpr bool population_model = detail::population_ok<Model>::value;

    using neuron_store = soa_store<neuron_fields>;
    using synapse_store = soa_store<synapse_fields>;
    using tap_fn = std::function<void(int64_t, std::span<const uint32_t>)>;

    network(network_desc desc, Model model, engine_options opt = {})
        : desc_(std::move(desc)), model_(std::move(model)), opt_(opt) {
        validate_or_throw(desc_);
        n_ = desc_.neuron_count();
        dt_ = static_cast<float>(desc_.dt);
        delay_ = desc_.delay;
        SYNQ_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        int dev = 0;
        SYNQ_CUDA(cudaGetDevice(&dev));
        SYNQ_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
        for (auto& e : ev_) SYNQ_CUDA(cudaEventCreate(&e));

        auto t0 = clock::now();
        // a shard of a multi-GPU run stores only the sub-rows of the targets
        // it receives for: ~1/W of the synapses per GPU
        uint32_t tlo = 0, thi = 0xffffffffu;
        if (opt_.shard_world > 1) {
            if (opt_.shard_rank >= opt_.shard_world) throw std::invalid_argument("shard rank out of range");
            cut_ = shard_cut_of(desc_, opt_.shard_world);
            tlo = cut_.ra[opt_.shard_rank];
            thi = cut_.ra[opt_.shard_rank + 1];
        }
        graph_ = build_device_graph(desc_, opt_.seed, opt_.pitch_align, stream_, tlo, thi);
        timings_.construct = since(t0);

        if constexpr (has_synapses) {
            const uint32_t floor = delay_ + 1;
            history_ = opt_.history_frames ? std::max(opt_.history_frames, floor)
                                           : std::max(floor, lazy_history_default);
        }
        exact_ = opt_.deterministic || opt_.threads == 1;
        allocate();
        init();
    }

    ~network() {
        if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
        for (auto& e : ev_)
            if (e) cudaEventDestroy(e);
        for (auto& sl : slots_)
            for (auto& e : sl.ev)
                if (e) cudaEventDestroy(e);
        if (nccl_) {
            if (stream_) cudaStreamSynchronize(stream_);
            detail::nccl_comm_destroy(nccl_);
        }
        for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
        if (side_) {
            cudaStreamSynchronize(side_);
            cudaStreamDestroy(side_);
        }
        if (fork_ev_) cudaEventDestroy(fork_ev_);
        if (join_ev_) cudaEventDestroy(join_ev_);
        if (stream_) {
            cudaStreamSynchronize(stream_);
            cudaStreamDestroy(stream_);
        }
    }
    network(const network&) = delete;
    network& operator=(const network&) = delete;

    // (re)run the Init stage (engine.hpp:154-186)
    void init() {
        push_mirrors();
        t_ = 0;
        counters_ = {};
        host_steps_done_ = 0;
        step_measured_.clear();
        step_spikes_host_.clear();
        expiring_host_.clear();
        logged_upto_ = 0;
        log_pred_ = 0;
        std::fill(imported_upto_.begin(), imported_upto_.end(), 0);
        const int64_t zero = 0;
        SYNQ_CUDA(cudaMemcpyAsync(t_dev_.get(), &zero, sizeof zero, cudaMemcpyHostToDevice, stream_));
        counters_dev_.zero(stream_);
        qcount_.zero(stream_);
        if (hist_) hist_.zero(stream_);
        tile_ctr_.zero(stream_);
        done_ctr_.zero(stream_);
        tile_status_.zero(stream_);
        if (finfo_) finfo_.zero(stream_);
        log_cursor_.zero(stream_);
        if (expiring_count_) expiring_count_.zero(stream_);
        flags_.zero(stream_);
        if (det_cnt_) {
            det_cnt_.zero(stream_);
            det_fill_.zero(stream_);
        }
        SYNQ_CUDA(cudaStreamSynchronize(stream_));

        auto t0 = clock::now();
        const int grid = grid_for(n_, 256);
        dev::k_init_neurons<Model><<<grid, 256, 0, stream_>>>(model_, state(), opt_.seed);
        SYNQ_CUDA(cudaGetLastError());
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        timings_.init_neurons = since(t0);

        if constexpr (has_synapses) {
            t0 = clock::now();
            ages_.zero(stream_);
            caught_.zero(stream_);
            if (tr_p_) {
                tr_p_.zero(stream_);
                tr_q_.zero(stream_);
            }
            for (auto& col : syn_cols_) col.zero(stream_);
            if (graph_.edges)
                dev::k_init_synapses<Model><<<grid_for(uint64_t(n_) * 32, 256), 256, 0, stream_>>>(model_, state());
            SYNQ_CUDA(cudaGetLastError());
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            timings_.init_synapses = since(t0);
        }
        invalidate_mirrors();
    }

    void step() { run(1); }

    void run(int64_t steps) {
        if (steps <= 0) return;
        if (opt_.shard_peer && !peers_connected_) {
            if (!nccl_) throw std::logic_error("peer shard: connect_peers / connect_peers_ipc before run");
            if constexpr (population_model) exchange_ipc_handles();
        }
        if (sharded() && !nccl_ && !opt_.shard_peer) {
            // a shard may only run steps whose due frames are all present:
            // at most delay-1 steps past the frames imported from every rank
            if (steps > int64_t(delay_) - 1)
                throw std::invalid_argument("sharded run: at most delay-1 steps between frame exchanges");
            for (uint32_t q = 0; q < opt_.shard_world; ++q)
                if (q != opt_.shard_rank && imported_upto_[q] < t_ + steps - int64_t(delay_) + 1)
                    throw std::logic_error("sharded run: frames of rank " + std::to_string(q) +
                                           " not imported (export/import after every run)");
            last_batch_t0_ = t_;
            last_batch_b_ = static_cast<uint32_t>(steps);
        }
        push_mirrors();
        auto t0 = clock::now();
        SYNQ_CUDA(cudaEventRecord(ev_[0], stream_));
        if (persistent_) {
            // two batches in flight: batch k+1 is launched before the host
            // emits batch k's frames (logs are written by the kernel straight
            // into pinned host slots), so the GPU never idles on the host
            int slot = 0;
            bool pending = false;
            // in-engine exchange: batches of at most delay-1 steps, each
            // followed by export -> ncclAllGather -> import on this stream
            int64_t cap = nccl_xchg() ? std::min<int64_t>(batch_cap_, int64_t(delay_) - 1) : int64_t(batch_cap_);
            // debug_checks: the frames of a batch are checked after it, so a
            // batch may not outrun the queue ring (Q slots)
            if (opt_.debug_checks) cap = std::min<int64_t>(cap, Q_);
            while (steps > 0) {
                const int64_t b = std::min<int64_t>(steps, cap);
                if constexpr (population_model)
                    if (nccl_xchg()) {
                        last_batch_t0_ = t_;
                        last_batch_b_ = static_cast<uint32_t>(b);
                    }
                launch_persistent(static_cast<uint32_t>(b), slot);
                if constexpr (population_model)
                    if (nccl_xchg()) {
                        enqueue_export_bits(last_batch_t0_, last_batch_b_, xsend_.get());
                        detail::nccl_allgather_u32(nccl_, xsend_.get(), xrecv_.get(), xl_.block, stream_);
                        enqueue_import_bits(last_batch_t0_, last_batch_b_, xrecv_.get());
                    }
                if (pending) finish_persistent(slot ^ 1);
                pending = true;
                slot ^= 1;
                steps -= b;
            }
            if (pending) finish_persistent(slot ^ 1);
            pull_counters();
            if (flags_host_[1]) throw device_error("ordered delivery scratch overflow");
            if (flags_host_[2]) throw device_error("sharded run: imported frames of a different batch length");
            check_debug_flags();
            if (log_on_ && logged_upto_ < t_ && (!sharded() || nccl_ || opt_.shard_peer)) drain_log();
        } else {
            while (steps > 0) {
                const int64_t b = std::min<int64_t>(steps, batch_cap_);
                run_batch(static_cast<uint32_t>(b));
                steps -= b;
            }
            if constexpr (has_synapses)  // the last step's catch-up ages (k_catchup1 leaves them to k_update)
                if (caught_) {
                    dev::k_apply_caught<Model><<<std::max<uint32_t>(1, std::min<uint32_t>((n_ + 255) / 256, sms_)), 256, 0,
                                                 stream_>>>(state());
                    SYNQ_CUDA(cudaGetLastError());
                    launches_ += 1;
                }
        }
        SYNQ_CUDA(cudaEventRecord(ev_[1], stream_));
        SYNQ_CUDA(cudaEventSynchronize(ev_[1]));
        float ms = 0;
        SYNQ_CUDA(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        device_seconds_ += ms * 1e-3;
        timings_.simulate += since(t0);
        invalidate_mirrors();
    }

    // bring every synapse current (engine.hpp:226-234)
    void flush() {
        if constexpr (has_synapses) {
            push_mirrors();
            auto t0 = clock::now();
            enqueue_catchup(1);
            SYNQ_CUDA(cudaGetLastError());
            pull_counters();
            timings_.simulate += since(t0);
            invalidate_mirrors();
        }
    }

    int64_t now() const { return t_; }
    float dt() const { return dt_; }
    uint32_t delay() const { return delay_; }
    uint32_t history_frames() const { return history_; }
    uint32_t neuron_count() const { return n_; }
    uint64_t edge_count() const { return graph_.edges; }
    uint64_t synapse_capacity() const {
        return has_synapses ? static_cast<uint64_t>(n_) * graph_.deg_max : 0;
    }
    // host mirror of the adjacency; a shard holds (and returns) the sub-rows
    // of its own targets [graph_targets()), rebuilt if they were released
    const adjacency_list& graph() const {
        if (!adj_mirror_) {
            if (graph_.cells || graph_.edges == 0) {
                adj_mirror_ = std::make_unique<adjacency_list>(download_graph(graph_, stream_));
            } else {
                const device_graph g = build_device_graph(desc_, opt_.seed, opt_.pitch_align, stream_,
                                                          graph_.target_lo, graph_.target_hi);
                adj_mirror_ = std::make_unique<adjacency_list>(download_graph(g, stream_));
            }
        }
        return *adj_mirror_;
    }
    std::pair<uint32_t, uint32_t> graph_targets() const { return {graph_.target_lo, graph_.target_hi}; }
    const network_desc& desc() const { return desc_; }
    const engine_counters& counters() const { return counters_; }
    const phase_seconds& timings() const { return timings_; }
    uint64_t seed() const { return opt_.seed; }
    bool deterministic() const { return opt_.deterministic; }
    unsigned worker_count() const { return persistent_ ? tiles_ : static_cast<unsigned>(sms_); }
    bool persistent() const { return persistent_; }
    bool pipelined() const { return persistent_ && pipe_; }
    bool solo() const { return persistent_ && solo_; }
    bool cluster() const { return persistent_ && cluster_; }
    bool bitmap_delivery() const { return persistent_ && pipe_ && pipe_bm_; }
    bool exact() const { return exact_ || persistent_ || (win_on_ && !atomic_recv_); }
    uint64_t construction_fixups() const { return graph_.tie_fixups; }
    // device time of all run() calls (CUDA events on the engine stream) and of
    // the dominant kernel alone; kernel launches; host<->device bytes moved
    double device_seconds() const { return device_seconds_; }
    double kernel_seconds() const { return kernel_seconds_; }
    uint64_t kernel_launches() const { return launches_; }
    uint64_t h2d_bytes() const { return h2d_bytes_; }
    uint64_t d2h_bytes() const { return d2h_bytes_; }
    unsigned tiles() const { return tiles_; }

    // ---- multi-GPU shard exchange -------------------------
    // a shard of a multi-GPU run; an in-engine NCCL exchange is a shard even
    // with one rank (then the allgather copies the rank's own block)
    bool sharded() const { return opt_.shard_world > 1 || opt_.shard_nccl || opt_.shard_peer; }
    const engine_options& options() const { return opt_; }
    // frames exchanged by export -> ncclAllGather -> import after every batch
    bool nccl_xchg() const { return nccl_ != nullptr && !opt_.shard_peer; }

    // ---- NVLink peer exchange (engine_options::shard_peer) ---------------
    // this shard's ring and frame words, for the other shards' kernels
    peer_endpoint peer_buffers() const {
        if (!opt_.shard_peer || !persistent_) throw std::logic_error("peer_buffers: not a peer shard");
        return {queue_.get(), finfo_.get(), publishers_, 0};
    }
    // eps[q]: shard q's buffers as this process addresses them (eps[rank]
    // is ignored).  Same-device shards of one process can pass the pointers
    // of peer_buffers() directly; across processes use connect_peers_ipc.
    void connect_peers(const std::vector<peer_endpoint>& eps) {
        const uint32_t W = opt_.shard_world, R = opt_.shard_rank;
        if (!opt_.shard_peer || !persistent_) throw std::logic_error("connect_peers: not a peer shard");
        if (eps.size() != W) throw std::invalid_argument("connect_peers: need one endpoint per rank");
        if (W - 1 > uint32_t(dev::kMaxPeers)) throw std::invalid_argument("connect_peers: too many ranks");
        std::vector<dev::peer_link> links;
        for (uint32_t q = 0; q < W; ++q) {
            if (q == R) continue;
            const peer_endpoint& e = eps[q];
            if (!e.queue || !e.finfo || e.publishers < W) throw std::invalid_argument("connect_peers: bad endpoint");
            const uint32_t Cq = e.publishers - (W - 1);  // the peer's local CTAs come first
            links.push_back({e.queue, e.finfo, e.publishers, Cq + (R < q ? R : R - 1)});
        }
        peers_dev_.resize(std::max<size_t>(1, links.size()));
        if (!links.empty()) peers_dev_.upload(links.data(), links.size(), stream_);
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        npeers_ = static_cast<uint32_t>(links.size());
        peers_connected_ = true;
    }
    // kPeerHandleBytes: IPC handles of this shard's ring and frame words
    void peer_ipc_handle(void* out) const {
        const peer_endpoint e = peer_buffers();
        cudaIpcMemHandle_t hq{}, hf{};
        SYNQ_CUDA(cudaIpcGetMemHandle(&hq, e.queue));
        SYNQ_CUDA(cudaIpcGetMemHandle(&hf, e.finfo));
        auto* b = static_cast<char*>(out);
        std::memset(b, 0, kPeerHandleBytes);
        std::memcpy(b, &hq, sizeof hq);
        std::memcpy(b + 64, &hf, sizeof hf);
        std::memcpy(b + 128, &e.publishers, 4);
    }
    // all: world x kPeerHandleBytes (rank q's handle at q * kPeerHandleBytes)
    void connect_peers_ipc(const void* all) {
        const uint32_t W = opt_.shard_world, R = opt_.shard_rank;
        const auto* b = static_cast<const char*>(all);
        std::vector<peer_endpoint> eps(W);
        for (uint32_t q = 0; q < W; ++q) {
            if (q == R) continue;
            cudaIpcMemHandle_t hq{}, hf{};
            std::memcpy(&hq, b + q * kPeerHandleBytes, sizeof hq);
            std::memcpy(&hf, b + q * kPeerHandleBytes + 64, sizeof hf);
            void *pq = nullptr, *pf = nullptr;
            SYNQ_CUDA(cudaIpcOpenMemHandle(&pq, hq, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened_.push_back(pq);
            SYNQ_CUDA(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened_.push_back(pf);
            eps[q].queue = static_cast<uint32_t*>(pq);
            eps[q].finfo = static_cast<unsigned long long*>(pf);
            std::memcpy(&eps[q].publishers, b + q * kPeerHandleBytes + 128, 4);
        }
        connect_peers(eps);
    }
    bool peers_connected() const { return peers_connected_; }
    // words needed to export the frames of the last run() (upper bound)
    uint64_t export_capacity() const {
        return 1 + 2ull * (delay_ ? delay_ : 1) + uint64_t(delay_) * ((shard_lo_[1] - shard_lo_[0]) + (shard_lo_[3] - shard_lo_[2]));
    }
    // pack this shard's frames of the last run() into dst (device or host
    // memory); returns the words written
    uint64_t export_frames(void* dst, uint64_t cap_words, bool device_dst) {
        if constexpr (population_model) {
            if (!sharded() || !persistent_) throw std::logic_error("export_frames: not a persistent shard");
            const uint64_t need = export_capacity();
            // straight into a device destination that can hold the worst case
            const bool direct = device_dst && cap_words >= need;
            if (!direct && xbuf_.size() < need) xbuf_.resize(need);
            uint32_t* out = direct ? static_cast<uint32_t*>(dst) : xbuf_.get();
            dev::k_export<Model><<<1, 1024, 0, stream_>>>(pstate(), last_batch_t0_, last_batch_b_, out);
            SYNQ_CUDA(cudaGetLastError());
            launches_ += 1;
            uint64_t words = 1 + 2ull * last_batch_b_;
            xcounts_.resize(2 * size_t(last_batch_b_) + 1);
            if (last_batch_b_)
                SYNQ_CUDA(cudaMemcpyAsync(xcounts_.data(), out + 1, 8ull * last_batch_b_, cudaMemcpyDeviceToHost, stream_));
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            for (uint32_t k = 0; k < 2 * last_batch_b_; ++k) words += xcounts_[k];
            if (words > cap_words) throw std::invalid_argument("export_frames: destination too small");
            if (!direct) {
                SYNQ_CUDA(cudaMemcpyAsync(dst, xbuf_.get(), words * 4,
                                          device_dst ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream_));
                SYNQ_CUDA(cudaStreamSynchronize(stream_));
            }
            return words;
        } else {
            throw std::logic_error("export_frames: model has no persistent engine");
        }
    }
    // unpack rank `from`'s exported frames (batch starting at the same step
    // as this shard's last run; every shard runs the same batches).  Stream-
    // ordered, no host synchronisation: a device source must stay valid
    // until the next run() (which synchronises).
    void import_frames(const void* src, uint64_t words, uint32_t from, bool device_src) {
        if constexpr (population_model) {
            if (!sharded() || !persistent_) throw std::logic_error("import_frames: not a persistent shard");
            if (from >= opt_.shard_world || from == opt_.shard_rank) throw std::invalid_argument("import_frames: bad rank");
            const uint32_t b = last_batch_b_;
            if (words < 1 + 2ull * b) throw std::invalid_argument("import_frames: truncated frame words");
            const uint32_t* in = static_cast<const uint32_t*>(src);
            if (!device_src) {
                const size_t slot = from % 2;  // host sources: staged per rank parity (stream-ordered reuse)
                if (ibuf_[slot].size() < words) {
                    SYNQ_CUDA(cudaStreamSynchronize(stream_));
                    ibuf_[slot].resize(words);
                }
                SYNQ_CUDA(cudaMemcpyAsync(ibuf_[slot].get(), src, words * 4, cudaMemcpyHostToDevice, stream_));
                SYNQ_CUDA(cudaStreamSynchronize(stream_));  // the host buffer may be reused by the caller
                in = ibuf_[slot].get();
            }
            const int64_t t0 = imported_upto_[from];
            if (b)
                dev::k_import<Model><<<b, 256, 0, stream_>>>(pstate(), t0, b, in, remote_[from][0], remote_[from][1],
                                                           remote_[from][2]);
            SYNQ_CUDA(cudaGetLastError());
            launches_ += 1;
            imported_upto_[from] = t0 + b;
        } else {
            throw std::logic_error("import_frames: model has no persistent engine");
        }
    }
    // this shard's receiving [lo, hi) and update-only [lo, hi) neuron ids
    std::array<uint32_t, 4> shard_range() const {
        return sharded() ? shard_lo_ : std::array<uint32_t, 4>{0, n_, n_, n_};
    }
    uint32_t shard_rank() const { return opt_.shard_rank; }
    uint32_t shard_world() const { return opt_.shard_world; }
    // persistent-kernel phase profile: average cycles per step per CTA for
    // update, publish, poll, gather, deliver (opt.profile only)
    std::vector<double> phase_cycles() const {
        // [0..4] mean over CTAs, [5..9] the pacing CTA (least time waiting for
        // its staged frame); slots: update, publish, wait, deliver, producer prep
        std::vector<double> out(15, 0.0);
        if (!prof_ || !tiles_) return out;
        std::vector<unsigned long long> h(prof_.size());
        prof_.download(h.data(), h.size(), stream_);
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        uint32_t crit = 0;
        double best = 1e300;
        for (uint32_t c = 0; c < tiles_; ++c) {
            const double steps = std::max<unsigned long long>(1, h[c * dev::P_SLOTS + dev::P_STEPS]);
            for (int k = 0; k < 5; ++k) out[k] += h[c * dev::P_SLOTS + k] / steps / tiles_;
            const double poll = h[c * dev::P_SLOTS + dev::P_POLL] / steps;
            if (poll < best) {
                best = poll;
                crit = c;
            }
        }
        const double steps = std::max<unsigned long long>(1, h[crit * dev::P_SLOTS + dev::P_STEPS]);
        for (int k = 0; k < 5; ++k) out[5 + k] = h[crit * dev::P_SLOTS + k] / steps;
        out[10] = h[crit * dev::P_SLOTS + 6] / steps;
        out[11] = h[crit * dev::P_SLOTS + 7] / steps;
        out[12] = h[crit * dev::P_SLOTS + 8] / steps;
        out[13] = h[crit * dev::P_SLOTS + 9] / steps;
        out[14] = (h[crit * dev::P_SLOTS + 10] + h[crit * dev::P_SLOTS + 11]) / steps;
        return out;
    }

    // On a shard the tap sees the merged frame of every rank.  With the
    // in-engine exchange every frame is emitted before run() returns; on a
    // manually exchanged shard a frame is emitted once it is delivered, i.e.
    // in the run() after the other ranks' frames of it were imported (so the
    // last delay-1 frames trail now()).
    void set_spike_tap(tap_fn fn) {
        tap_ = std::move(fn);
        if (tap_) {
            ensure_log();
            logged_upto_ = t_;  // a new tap observes frames from now on
            log_pred_ = t_;
        } else {
            drop_log();
        }
    }

    // measured-population spike counts per step, kept on the device and
    // returned per batch (the reference's sim_runtime tap, sim_runtime.cpp:33-39)
    void set_measure_range(uint32_t lo, uint32_t hi) {
        meas_lo_ = lo;
        meas_hi_ = hi;
        reset_graph();
    }
    const std::vector<uint32_t>& step_measured() const { return step_measured_; }
    const std::vector<uint32_t>& step_spike_counts() const { return step_spikes_host_; }

    template <size_t I>
    auto neuron_field() {
        using T = field_t<I, neuron_fields>;
        if (!nmirror_valid_[I]) {
            SYNQ_CUDA(cudaMemcpyAsync(host_neurons_.template data<I>(), neuron_cols_[I].get(),
                                      n_ * sizeof(T), cudaMemcpyDeviceToHost, stream_));
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            nmirror_valid_[I] = true;
        }
        ndirty_[I] = true;
        return std::span<T>(host_neurons_.template data<I>(), n_);
    }
    template <size_t I>
    auto synapse_field() {
        static_assert(has_synapses);
        using T = field_t<I, synapse_fields>;
        const size_t cap = synapse_capacity();
        if (!smirror_valid_[I]) {
            SYNQ_CUDA(cudaMemcpyAsync(host_synapses_.template data<I>(), syn_cols_[I].get(),
                                      cap * sizeof(T), cudaMemcpyDeviceToHost, stream_));
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            smirror_valid_[I] = true;
        }
        sdirty_[I] = true;
        return std::span<T>(host_synapses_.template data<I>(), cap);
    }
    std::span<const uint32_t> ages() const {
        if constexpr (has_synapses) {
            ages_host_.resize(n_);
            ages_.download(ages_host_.data(), n_, stream_);
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
        }
        return {ages_host_.data(), ages_host_.size()};
    }
    std::span<const uint32_t> expiring() const {
        if constexpr (has_synapses) return {expiring_host_.data(), expiring_host_.size()};
        return {};
    }
    Model& model() { return model_; }

    engine_memory memory() const {
        engine_memory m;
        m.neuron_fields = detail::field_bytes<neuron_fields>() * n_;
        m.neuron_rng = uses_rng ? uint64_t(n_) * sizeof(xorshift) : 0;
        m.spike_bitmasks = hist_.bytes();
        m.spike_queues = queue_.bytes() + qcount_.bytes() + finfo_.bytes() + xsend_.bytes() + xrecv_.bytes() +
                         step_ctr_dev_.bytes() + step_spikes_dev_.bytes() + step_meas_dev_.bytes();
        m.ages = has_synapses ? uint64_t(n_) * 4 : 0;
        m.expirations = has_synapses ? uint64_t(n_) * 4 : 0;
        m.adjacency = graph_.bytes() + split_.bytes() + bm_.bytes() + win_split_.bytes();  // + receive-window bitmaps
        m.synapse_fields = detail::field_bytes<synapse_fields>() * synapse_capacity();
        return m;
    }

private:
    using clock = std::chrono::steady_clock;
    static double since(clock::time_point t0) {
        return std::chrono::duration<double>(clock::now() - t0).count();
    }
    int grid_for(uint64_t work, int block) const {
        const uint64_t want = (work + block - 1) / block;
        return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, 16ull * sms_)));
    }

    // ------------------------------------------------------------ setup
    void allocate() {
        neuron_cols_.resize(std::max<size_t>(1, neuron_fields::count));
        detail::alloc_fields<neuron_fields>(neuron_cols_, nptrs_, n_, stream_);
        host_neurons_.resize(n_);
        if constexpr (uses_rng) rng_.resize(std::max<uint32_t>(1, n_));
        if constexpr (has_synapses) {
            const size_t cap = synapse_capacity();
            syn_cols_.resize(std::max<size_t>(1, synapse_fields::count));
            detail::alloc_fields<synapse_fields>(syn_cols_, sptrs_, cap, stream_);
            host_synapses_.resize(cap);
            ages_.resize(std::max<uint32_t>(1, n_));
            caught_.resize(std::max<uint32_t>(1, n_));
            if constexpr (dev::model_has_plastic<Model>()) row_plastic_.resize(std::max<uint32_t>(1, n_));
            expiring_.resize(std::max<uint32_t>(1, n_));
            expiring_count_.resize(1);
            hist_words_ = (history_ + 63) / 64;
            if (hist_words_ > 4) throw std::invalid_argument("history_frames above 256 are not supported");
            hist_.resize(std::max<size_t>(1, size_t(n_) * hist_words_));
            // trace-STDP models on the one-word-history catch-up: per-neuron
            // trace rings (SYNQ_TRACE_RINGS=0: replay every synapse step)
            if constexpr (dev::model_trace_stdp<Model>()) {
                const char* e = std::getenv("SYNQ_TRACE_RINGS");
                if (hist_words_ == 1 && (!e || std::atoi(e) != 0)) {
                    tr_p_.resize(size_t(std::max<uint32_t>(1, n_)) * dev::kTraceRing);
                    tr_q_.resize(size_t(std::max<uint32_t>(1, n_)) * dev::kTraceRing);
                }
            }
        }
        if (!has_synapses && opt_.debug_checks) {  // debug_checks tracks spike bits for every model
            history_ = delay_ + 1;
            hist_words_ = (history_ + 63) / 64;
            if (hist_words_ > 4) throw std::invalid_argument("debug_checks: delay above 255 steps is not supported");
            hist_.resize(std::max<size_t>(1, size_t(n_) * hist_words_));
        }
        counters_dev_.resize(dev::C_COUNT);
        tile_ctr_.resize(2);
        done_ctr_.resize(1);
        t_dev_.resize(1);
        t0_dev_.resize(1);
        flags_.resize(4);
        log_cursor_.resize(2);
        ntiles_update_ = std::max<uint32_t>(1, (n_ + kUpdateBlock - 1) / kUpdateBlock);
        tile_status_.resize(ntiles_update_);
        tile_bal_.resize(size_t(ntiles_update_) * (kUpdateBlock / 32));

        if constexpr (population_model) {
            if (opt_.persistent != 0) setup_persistent();
            if (opt_.persistent == 1 && !persistent_)
                throw std::invalid_argument("persistent engine requested but the network does not fit it");
        }
        if (sharded() && !persistent_)
            throw std::invalid_argument("sharding needs the persistent engine (population-delivery model)");
        if (sharded() && delay_ < 2)
            throw std::invalid_argument("sharding needs a delay of at least 2 steps (frames are exchanged every delay-1 steps)");
        if constexpr (population_model)
            if (sharded()) setup_exchange();
        // a shard delivering from window bitmaps never reads its ELL sub-rows
        // again: release them (graph() rebuilds them on demand)
        if (opt_.shard_world > 1 && persistent_ && pipe_ && pipe_bm_) graph_.cells.release();
        Q_ = persistent_ ? 2 * delay_ : delay_;
        queue_.resize(std::max<size_t>(1, size_t(Q_) * n_));
        qcount_.resize(Q_);
        if (!persistent_) setup_recv_win();
        if (!persistent_ && exact_ && !win_on_) {  // scratch of the count/scan/scatter ordered receive
            det_cnt_.resize(std::max<uint32_t>(1, n_));
            det_off_.resize(std::max<uint32_t>(1, n_));
            det_fill_.resize(std::max<uint32_t>(1, n_));
            det_cap_ = std::max<uint64_t>(1, std::min<uint64_t>(graph_.edges, 1ull << 27));
            det_ev_.resize(det_cap_);
        }
        batch_cap_ = opt_.batch_steps ? opt_.batch_steps : 1000;
        step_spikes_dev_.resize(2 * size_t(batch_cap_));
        step_meas_dev_.resize(2 * size_t(batch_cap_));
        step_ctr_dev_.resize(4 * size_t(batch_cap_));
        step_buf_.resize(4 * size_t(batch_cap_));
    }

    // ordered windowed receive for the generic engine (kernels.cuh
    // k_recv_win): target windows balanced by in-degree, at most
    // kWinTPT x kWinBlock targets each, row splits per window.  Off when the
    // split table would be large next to the adjacency (very sparse
    // networks) or SYNQ_WINRECV=0; SYNQ_ATOMIC_RECV=1 keeps the device-atomic
    // k_receive for the fast (non-deterministic) mode.
    void setup_recv_win() {
        if (const char* e = std::getenv("SYNQ_WINRECV"); e && std::atoi(e) == 0) return;
        if (const char* e = std::getenv("SYNQ_ATOMIC_RECV")) atomic_recv_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SYNQ_PDL")) {
            pdl_ = std::atoi(e) != 0;
            pdl_all_ = std::atoi(e) == 2;
        }
        if (const char* e = std::getenv("SYNQ_CATCHUP_U")) catchup_u_ = std::atoi(e);
        if (n_ == 0 || graph_.edges == 0 || graph_.deg_max >= (1u << 24) || !graph_.cells) return;
        const uint32_t cap_t = uint32_t(dev::kWinTPT) * kWinBlock;
        const std::vector<uint32_t> indeg = in_degrees(graph_, stream_);
        std::vector<double> prefix(size_t(n_) + 1, 0.0);
        for (uint32_t k = 0; k < n_; ++k) prefix[k + 1] = prefix[k] + receive_cost(indeg[k]);
        uint32_t C = std::min<uint32_t>(n_, std::max<uint32_t>(uint32_t(sms_), (n_ + cap_t - 1) / cap_t));
        std::vector<uint32_t> lo;
        uint32_t wmax = 0;
        for (;;) {
            lo = cut_by_cost(prefix, 0, 0, n_, C);
            wmax = 0;
            for (uint32_t c = 0; c < C; ++c) wmax = std::max(wmax, lo[c + 1] - lo[c]);
            if (wmax <= cap_t || C >= n_) break;
            C = std::min<uint32_t>(n_, C + C / 4 + 1);
        }
        if (wmax > cap_t) return;
        const uint64_t split_bytes = uint64_t(n_) * (C + 1) * 4;
        if (split_bytes > std::max<uint64_t>(256ull << 20, graph_.bytes() / 4)) return;
        int dev = 0, max_smem = 0;
        SYNQ_CUDA(cudaGetDevice(&dev));
        SYNQ_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        auto fn = dev::k_recv_win<Model, kWinBlock>;
        cudaFuncAttributes fa{};
        SYNQ_CUDA(cudaFuncGetAttributes(&fa, fn));
        const size_t avail = size_t(max_smem) - fa.sharedSizeBytes - 1024;
        const size_t per_target = 10 * 4, per_event = 12 + 2 * detail::field_bytes<synapse_fields>() + 16;
        if (avail <= per_target * wmax) return;
        size_t ecap = std::min<size_t>(8192, (avail - per_target * wmax) / per_event) & ~size_t(31);
        if (ecap < wmax || ecap < 64) return;
        win_smem_ = per_target * wmax + 3 * 4 * ecap + 2 * detail::field_bytes<synapse_fields>() * ecap + 16 * 8;
        SYNQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(win_smem_)));
        win_lo_dev_.resize(C + 1);
        win_lo_dev_.upload(lo.data(), C + 1, stream_);
        build_splits(graph_, lo, win_split_, stream_);
        win_ = dev::recv_win{win_lo_dev_.get(), win_split_.get(), C, wmax, static_cast<uint32_t>(ecap)};
        win_on_ = true;
        if constexpr (has_synapses) {
            // opt-in: at Brunel+ 1e8 the receive's whole-SM CTAs wait for the
            // side stream's CTAs (39.4 vs 35.1 us per step); 1e9: 203.6 vs 207
            bool split = false;
            if (const char* e = std::getenv("SYNQ_SPLIT_CATCHUP")) split = std::atoi(e) != 0;
            if (split && hist_words_ == 1) {
                SYNQ_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
                SYNQ_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
                SYNQ_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
                split_param_.resize(2);
                split_catchup_ = true;
            }
        }
    }

    // ---- partition helpers (setup_persistent; shard construction)
    struct shard_cut {
        uint32_t r0 = 0, r1 = 0, u0 = 0, u1 = 0;  // receiving / update-only regions
        bool u_after = true;                      // update-only region after the receiving one
        std::vector<uint32_t> ra, ub;             // W rank ranges of each (W + 1 bounds)
    };
    static double receive_cost(double indeg) { return 16.0 + 0.003 * indeg; }
    // ids [lo, hi) of a region starting at r0 cut into `parts` ranges of equal
    // prefix cost
    static std::vector<uint32_t> cut_by_cost(const std::vector<double>& prefix, uint32_t r0, uint32_t lo,
                                             uint32_t hi, uint32_t parts) {
        std::vector<uint32_t> b(parts + 1);
        const double c0 = prefix[lo - r0], c1 = prefix[hi - r0];
        for (uint32_t c = 0; c <= parts; ++c) {
            const double target = c0 + (c1 - c0) * c / parts;
            b[c] = r0 + static_cast<uint32_t>(std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin());
            b[c] = std::clamp(b[c], lo, hi);
        }
        b[0] = lo;
        b[parts] = hi;
        for (uint32_t c = 1; c <= parts; ++c) b[c] = std::max(b[c], b[c - 1]);
        return b;
    }
    static std::vector<uint32_t> cut_by_count(uint32_t lo, uint32_t hi, uint32_t parts) {
        std::vector<uint32_t> b(parts + 1);
        for (uint32_t c = 0; c <= parts; ++c) b[c] = lo + static_cast<uint32_t>(uint64_t(hi - lo) * c / parts);
        return b;
    }
    // the receiving region [r0, r1) (neurons outside receive nothing) and the
    // update-only remainder, which must be one range on one side, else the
    // whole id space is the receiving region (B pieces stay empty)
    template <class T>
    static shard_cut region_of(const std::vector<T>& indeg, uint32_t n) {
        shard_cut k;
        uint32_t r0 = 0, r1 = 0;
        while (r0 < n && indeg[r0] == 0) ++r0;
        r1 = n;
        while (r1 > r0 && indeg[r1 - 1] == 0) --r1;
        if (r0 == r1) r0 = r1 = 0;
        k.u0 = r1;
        k.u1 = n;
        if (r0 > 0 && r1 < n) {
            r0 = 0;
            r1 = n;
            k.u0 = k.u1 = n;
        } else if (r0 > 0) {
            k.u0 = 0;
            k.u1 = r0;
            k.u_after = false;
        }
        k.r0 = r0;
        k.r1 = r1;
        return k;
    }
    // rank ranges of a W-way shard from the description alone: the expected
    // in-degree (sum of |src| * p over the connections into a neuron) sets
    // the receiving region and the receive cost, so every rank computes the
    // same cut before (and without) building the whole graph
    static shard_cut shard_cut_of(const network_desc& d, uint32_t W) {
        const uint32_t n = d.neuron_count();
        std::vector<double> e(n, 0.0);
        for (const auto& c : d.connections) {
            auto [sa, sb] = d.id_range(c.src);
            auto [ta, tb] = d.id_range(c.dst);
            if (c.p <= 0.0 || sb == sa) continue;
            for (uint32_t t = ta; t < tb; ++t) e[t] += double(sb - sa) * c.p;
        }
        shard_cut k = region_of(e, n);
        std::vector<double> prefix(size_t(k.r1 - k.r0) + 1, 0.0);
        for (uint32_t j = 0; j < k.r1 - k.r0; ++j) prefix[j + 1] = prefix[j] + receive_cost(e[k.r0 + j]);
        k.ra = cut_by_cost(prefix, k.r0, k.r0, k.r1, W);
        k.ub = cut_by_count(k.u0, k.u1, W);
        return k;
    }

    // Partition for the persistent engine (detail/persistent.cuh): every CTA
    // owns a receiving piece A_c and an update-only piece B_c; pieces tile the
    // id space and are numbered in id order.
    void setup_persistent() requires population_model {
        const std::vector<uint32_t> indeg = in_degrees(graph_, stream_);
        uint32_t bound[dev::kMaxClasses] = {};
        float delta[dev::kMaxClasses] = {};
        const int K = population_delivery<Model>::classes(model_, n_, bound, delta);
        if (K < 1 || K > dev::kMaxClasses || n_ == 0) return;
        // receiving region [r0, r1): everything outside receives nothing.
        // A shard only holds its own sub-rows, so its region and rank ranges
        // come from the description (shard_cut_of, identical on every rank);
        // the CTA cut inside the rank uses the exact local in-degrees.
        const uint32_t W = std::max<uint32_t>(1, opt_.shard_world), R = opt_.shard_rank;
        if (R >= W) throw std::invalid_argument("shard rank out of range");
        shard_cut cut = W > 1 ? cut_ : region_of(indeg, n_);
        const uint32_t r0 = cut.r0, r1 = cut.r1, u0 = cut.u0, u1 = cut.u1;
        const bool u_after = cut.u_after;
        const uint32_t nr = r1 - r0;
        const uint32_t NTH = dev::kPersistThreads;
        // ~90% thread occupancy per CTA keeps one neuron per thread (NPT = 1)
        // about one CTA per 128 neurons, up to one per SM: the pipelined
        // kernel's delivery work per step does not shrink with the neurons a
        // CTA owns, so a shard of a multi-GPU run still uses every SM
        constexpr int64_t kNeuronsPerTile = 128;
        // (small networks: at least min(32, n/32) CTAs, measured best for
        // Vogels 1000 / 4000)
        auto tiles_for = [&](int64_t n) {
            const int64_t want = std::max<int64_t>((n + kNeuronsPerTile - 1) / kNeuronsPerTile, std::min<int64_t>(32, n / 32));
            return static_cast<uint32_t>(std::clamp<int64_t>(want, 1, sms_));
        };
        // SYNQ_SOLO=1: the single-CTA engine (detail/solo.cuh) for networks
        // of <= 4096 neurons.  Opt-in: measured 2.9-5x slower than the
        // multi-CTA pipeline from 1,414 to 4,000 Vogels neurons (one SM
        // issues the whole update)
        bool solo = W == 1 && !opt_.shard_nccl && n_ <= dev::kSoloMaxNeurons && delay_ <= dev::kSoloMaxDelay &&
                    (opt_.tiles == 0 || opt_.tiles == 1) && opt_.pipeline < 0 && !std::getenv("SYNQ_PIPELINE");
        const char* solo_env = std::getenv("SYNQ_SOLO");
        solo = solo && solo_env && std::atoi(solo_env) != 0;
        // SYNQ_CLUSTER=1: one thread-block cluster owns the network
        // (detail/cluster.cuh), frames through distributed shared memory
        bool clus = !solo && W == 1 && !opt_.shard_nccl && n_ <= dev::kClusterMaxNeurons &&
                    delay_ <= dev::kClusterMaxDelay && opt_.tiles == 0 && opt_.pipeline < 0 &&
                    !std::getenv("SYNQ_PIPELINE");
        const char* clus_env = std::getenv("SYNQ_CLUSTER");
        clus = clus && clus_env && std::atoi(clus_env) != 0 && !cluster_failed_;
        uint32_t CLn = 16;
        if (const char* e = std::getenv("SYNQ_CLUSTER_SIZE")) CLn = static_cast<uint32_t>(std::atoi(e));
        if (clus && (CLn < 2 || CLn > 16 || n_ > CLn * 2 * dev::kClusterThreads)) clus = false;
        uint32_t C = solo ? 1u : (clus ? CLn : (opt_.tiles ? opt_.tiles : tiles_for(n_)));
        C = std::min<uint32_t>({C, static_cast<uint32_t>(sms_), static_cast<uint32_t>(dev::kMaxTiles), n_});
        const uint32_t max_local = 4 * NTH;  // register-resident state: <= 4 neurons per thread
        // shards: contiguous rank ranges of the receiving region (by receive
        // cost) and of the update-only region (by count); then this rank's
        // range into C local pieces of each kind
        std::vector<double> prefix(size_t(nr) + 1, 0.0);
        for (uint32_t k = 0; k < nr; ++k) prefix[k + 1] = prefix[k] + receive_cost(indeg[r0 + k]);
        auto cut_cost = [&](uint32_t lo, uint32_t hi, uint32_t parts) { return cut_by_cost(prefix, r0, lo, hi, parts); };
        const std::vector<uint32_t> ra = W > 1 ? cut.ra : std::vector<uint32_t>{r0, r1};
        const std::vector<uint32_t> ub = W > 1 ? cut.ub : std::vector<uint32_t>{u0, u1};
        // the local shard sizes its CTA count by its own neurons
        const uint64_t mine = W > 1 ? uint64_t(ra[R + 1] - ra[R]) + (ub[R + 1] - ub[R]) : uint64_t(n_);
        if (W > 1 && !opt_.tiles) C = tiles_for(static_cast<int64_t>(mine));
        if (!solo && !clus && uint64_t(C) * max_local < mine)
            C = static_cast<uint32_t>(std::min<uint64_t>(sms_, (mine + max_local - 1) / max_local));
        if (C + W - 1 > uint32_t(dev::kMaxTiles)) return;
        if (2ull * delay_ >= (1u << 15)) return;  // 16-bit frame tags need Q << 65536
        const std::vector<uint32_t> alo = cut_cost(ra[R], ra[R + 1], C), blo = cut_by_count(ub[R], ub[R + 1], C);
        uint32_t longest = 0, wcap = 1;
        for (uint32_t c = 0; c < C; ++c) {
            longest = std::max(longest, (alo[c + 1] - alo[c]) + (blo[c + 1] - blo[c]));
            wcap = std::max(wcap, alo[c + 1] - alo[c]);
        }
        const bool pipe_fits = longest <= uint32_t(dev::kStreamChunks) * 256 && uint64_t(n_) * (graph_.pitch / 4) < (1ull << 32);
        if (longest > max_local && !pipe_fits) return;  // cannot hold the state: per-step kernel graph
        npt_ = longest <= NTH ? 1 : (longest <= 2 * NTH ? 2 : 4);
        // pieces in id order; publishers: local CTAs 0..C-1, then remote shards
        const uint32_t E = C + W - 1;
        auto remote_entry = [&](uint32_t q) { return C + (q < R ? q : q - 1); };
        std::vector<uint32_t> piece_lo, piece_src, cta_piece(2 * C);
        remote_.assign(W, {0, 0, 0});
        auto emit_region = [&](int half) {
            for (uint32_t q = 0; q < W; ++q) {
                if (q == R) {
                    for (uint32_t c = 0; c < C; ++c) {
                        cta_piece[2 * c + half] = static_cast<uint32_t>(piece_lo.size());
                        piece_lo.push_back(half ? blo[c] : alo[c]);
                        piece_src.push_back((c << 1) | half);
                    }
                } else {
                    piece_lo.push_back(half ? ub[q] : ra[q]);
                    piece_src.push_back((remote_entry(q) << 1) | half);
                    remote_[q][0] = remote_entry(q);
                    remote_[q][1 + half] = half ? ub[q] : ra[q];
                }
            }
        };
        if (u_after) {
            emit_region(0);
            emit_region(1);
        } else {
            emit_region(1);
            emit_region(0);
        }
        const uint32_t P = static_cast<uint32_t>(piece_lo.size());
        piece_lo.push_back(n_);
        for (uint32_t p = 0; p + 1 < piece_lo.size(); ++p)  // pieces must tile the id space in order
            if (piece_lo[p] > piece_lo[p + 1]) throw device_error("internal: shard pieces out of order");
        int max_smem = 0, dev = 0;
        SYNQ_CUDA(cudaGetDevice(&dev));
        SYNQ_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        size_t smem = 0;
        solo_ = false;
        cluster_ = false;
        if (clus) {
            smem = dev::cluster_smem_bytes(uint32_t(K), wcap, n_, delay_, C);
            if (C != CLn || longest > 2 * uint32_t(dev::kClusterThreads) || smem + 16 * 1024 > size_t(max_smem)) {
                cluster_failed_ = true;  // the multi-CTA engines instead
                return setup_persistent();
            }
            cluster_ = true;
            pipe_ = false;
            pipe_bm_ = false;
            npt_ = longest <= uint32_t(dev::kClusterThreads) ? 1 : 2;
        } else if (solo) {
            if (C != 1) throw device_error("internal: single-CTA engine with several pieces");
            smem = dev::solo_smem_bytes(uint32_t(K), wcap, n_);
            if (smem + 16 * 1024 > size_t(max_smem) || longest > dev::kSoloMaxNeurons) return;
            solo_ = true;
            pipe_ = false;
            pipe_bm_ = false;
            npt_ = longest <= 1024 ? 1 : (longest <= 2048 ? 2 : 4);
        } else if (!setup_pipeline(K, wcap, longest, delay_, size_t(max_smem), smem, alo)) {
            if (longest > max_local) return;
            // dynamic smem: counts only (delivery items are static)
            const size_t static_smem = 3 * (dev::kMaxPieces + 1) * 4 + 8192;
            const size_t counts = ((size_t(K) * wcap + 31) & ~size_t(31)) * 4;
            if (counts + static_smem + 1024 * 16 > size_t(max_smem)) return;
            // the rest of shared memory holds the 16-byte chunk list (16 B per chunk)
            const size_t chunk_cap = std::min<size_t>(16384, (size_t(max_smem) - static_smem - counts) / 16);
            smem = counts + chunk_cap * 16;
            stage_items_ = static_cast<uint32_t>(chunk_cap);
        }
        npt_select_ = npt_;
        const void* fn = kernel_fn();
        {   // the attribute is per kernel, shared by every network in the process:
            // always the maximum, so a smaller network never shrinks a larger one's
            cudaFuncAttributes fa{};
            SYNQ_CUDA(cudaFuncGetAttributes(&fa, fn));
            SYNQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           max_smem - static_cast<int>(fa.sharedSizeBytes)));
        }
        int per_sm = 0;
        SYNQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, static_cast<int>(kernel_threads()), smem));
        if (per_sm < 1) return;
        if (cluster_) {  // the whole cluster must be schedulable (16 CTAs: non-portable size)
            if (C > 8) SYNQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(kernel_threads());
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclus = 0;
            if (cudaOccupancyMaxActiveClusters(&nclus, fn, &cfg) != cudaSuccess || nclus < 1) {
                cudaGetLastError();
                cluster_ = false;
                cluster_failed_ = true;
                return setup_persistent();
            }
        }
        if (opt_.profile) {
            prof_.resize(size_t(C) * dev::P_SLOTS);
            prof_.zero(stream_);
        }

        tiles_ = C;
        pieces_ = P;
        publishers_ = E;
        tile_lo_host_ = piece_lo;
        tile_lo_.resize(P + 1);
        tile_lo_.upload(piece_lo.data(), P + 1, stream_);
        win_lo_.resize(2 * C);
        win_lo_.upload(cta_piece.data(), 2 * C, stream_);
        piece_src_.resize(P);
        piece_src_.upload(piece_src.data(), P, stream_);
        build_splits(graph_, alo, split_, stream_);
        finfo_.resize(size_t(2) * delay_ * E);
        shard_lo_ = {ra[R], ra[R + 1], ub[R], ub[R + 1]};
        all_ra_ = ra;
        all_ub_ = ub;
        imported_upto_.assign(W, 0);
        K_ = K;
        std::copy(bound, bound + dev::kMaxClasses, bound_);
        std::copy(delta, delta + dev::kMaxClasses, delta_);
        win_cap_ = wcap;
        smem_ = smem;
        persistent_ = true;
        // fold table (persistent.cuh fold_frame): the first two classes' sums
        // from zero in one read; SYNQ_FOLD_TABLE=0 disables it
        {
            const char* e = std::getenv("SYNQ_FOLD_TABLE");
            const bool want = !e || std::atoi(e) != 0;
            const bool ok = delta_[0] != 0.0f && std::isfinite(delta_[0]) &&
                            (K == 1 || (delta_[1] != 0.0f && std::isfinite(delta_[1])));
            if (want && ok) {
                fold_t0_ = 63;
                fold_t1_ = K > 1 ? 31 : 0;
                fold_tab_.resize(size_t(fold_t0_ + 1) * (fold_t1_ + 1));
                dev::k_fold_table<<<1, 64, 0, stream_>>>(delta_[0], K > 1 ? delta_[1] : 0.0f, fold_t0_, fold_t1_,
                                                         fold_tab_.get());
                SYNQ_CUDA(cudaGetLastError());
            }
        }
    }

    // fixed-size bitmask exchange (detail/persistent.cuh k_export_bits /
    // k_import_bits); the NCCL communicator only with opt.shard_nccl
    void setup_exchange() requires population_model {
        const uint32_t W = opt_.shard_world, R = opt_.shard_rank;
        if (opt_.shard_peer) {
            // frames go straight into the peers' rings from the pipelined
            // step kernel (pipeline.cuh peer_export)
            if (!pipe_) throw std::invalid_argument("peer shard: needs the pipelined step kernel");
            if (opt_.shard_nccl) nccl_ = detail::nccl_comm_init(R, W, opt_.nccl_id.data());
            return;
        }
        uint32_t wa = 1, wb = 1;
        for (uint32_t q = 0; q < W; ++q) {
            wa = std::max(wa, (all_ra_[q + 1] - all_ra_[q] + 31) / 32);
            wb = std::max(wb, (all_ub_[q + 1] - all_ub_[q] + 31) / 32);
        }
        xl_ = dev::xbits_layout{wa, wb, delay_ - 1, 1 + (delay_ - 1) * (wa + wb)};
        if ((wa + wb) * 4ull > 160 * 1024) throw std::invalid_argument("shard exchange: rank range too large");
        if ((wa + wb) * 4ull > 48 * 1024)
            SYNQ_CUDA(cudaFuncSetAttribute(dev::k_export_bits<Model>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>((wa + wb) * 4)));
        std::vector<dev::xbits_remote> rem;
        for (uint32_t q = 0; q < W; ++q)
            if (q != R)
                rem.push_back({q, remote_[q][0], all_ra_[q], all_ub_[q], all_ra_[q + 1] - all_ra_[q],
                               all_ub_[q + 1] - all_ub_[q]});
        xremotes_.resize(std::max<size_t>(1, rem.size()) * sizeof(dev::xbits_remote) / 4);
        if (!rem.empty()) SYNQ_CUDA(cudaMemcpy(xremotes_.get(), rem.data(), rem.size() * sizeof(rem[0]), cudaMemcpyHostToDevice));
        if (opt_.shard_nccl) {
            xsend_.resize(xl_.block);
            xrecv_.resize(size_t(W) * xl_.block);
            nccl_ = detail::nccl_comm_init(R, W, opt_.nccl_id.data());
        }
    }

    // shard_peer + shard_nccl: allgather the IPC handles over NCCL, map them
    void exchange_ipc_handles() requires population_model {
        const uint32_t W = opt_.shard_world;
        constexpr size_t words = kPeerHandleBytes / 4;
        pinned_array<uint32_t> h(words * W);
        peer_ipc_handle(h.get());
        dev_array<uint32_t> send(words), recv(words * W);
        send.upload(h.get(), words, stream_);
        detail::nccl_allgather_u32(nccl_, send.get(), recv.get(), words, stream_);
        SYNQ_CUDA(cudaMemcpyAsync(h.get(), recv.get(), words * W * 4, cudaMemcpyDeviceToHost, stream_));
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        connect_peers_ipc(h.get());
    }

    // this shard's frames of steps [t0, t0+b) -> its bitmask block at `out`
    void enqueue_export_bits(int64_t t0, uint32_t b, uint32_t* out) requires population_model {
        dev::k_export_bits<Model><<<std::max<uint32_t>(1, b), 1024, (xl_.wa + xl_.wb) * 4, stream_>>>(
            pstate(), t0, b, xl_, shard_lo_[0], shard_lo_[2], out);
        SYNQ_CUDA(cudaGetLastError());
        launches_ += 1;
    }
    // every other rank's block of the gathered buffer -> the ring
    void enqueue_import_bits(int64_t t0, uint32_t b, const uint32_t* all) requires population_model {
        const uint32_t W = opt_.shard_world, R = opt_.shard_rank;
        if (W > 1 && b)
            dev::k_import_bits<Model><<<dim3(b, W - 1), 256, 0, stream_>>>(
                pstate(), t0, b, xl_, all, reinterpret_cast<const dev::xbits_remote*>(xremotes_.get()));
        SYNQ_CUDA(cudaGetLastError());
        launches_ += 1;
        for (uint32_t q = 0; q < W; ++q)
            if (q != R) imported_upto_[q] = t0 + b;
    }

public:
    // words per rank block of the bitmask exchange (0 when not sharded)
    uint64_t exchange_block_words() const { return sharded() ? xl_.block : 0; }
    // manual bitmask exchange (the in-engine NCCL path does the same after
    // every batch): export the last run's frames into dst (device, block
    // words), import every other rank's block of a gathered buffer
    void export_bits(uint32_t* dst) {
        if constexpr (population_model) {
            if (!sharded()) throw std::logic_error("export_bits: not a shard");
            enqueue_export_bits(last_batch_t0_, last_batch_b_, dst);
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
        }
    }
    void import_bits(const uint32_t* all) {
        if constexpr (population_model) {
            if (!sharded()) throw std::logic_error("import_bits: not a shard");
            enqueue_import_bits(last_batch_t0_, last_batch_b_, all);
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
        }
    }

private:
    void reset_graph() {
        if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
    }

    void drop_log() {
        if (!log_on_) return;
        reset_graph();
        log_ids_ = dev_array<uint32_t>();
        log_cap_ = 0;
        log_on_ = false;
    }

    void ensure_log() {
        if (log_on_) return;
        reset_graph();
        log_on_ = true;
        // frames of one batch; the batch shrinks to keep the log bounded
        const uint64_t cap = std::max<uint64_t>(1024, std::min<uint64_t>(uint64_t(batch_cap_ + delay_) * n_, 1ull << 26));
        log_cap_ = cap;
        if (persistent_) {
            // written by the kernel in place (pinned, device-addressable)
            plog_[0].resize(cap);
            plog_[1].resize(cap);
            plog_end_.resize(2);
        } else {
            log_ids_.resize(cap);
            log_host_.resize(cap);
        }
        // a persistent batch logs up to delay-1 frames of the previous batch too
        const uint64_t frames = cap / std::max<uint32_t>(1, n_);
        const uint64_t fit = frames > delay_ ? frames - delay_ : 1;
        batch_cap_ = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(batch_cap_, fit)));
        if (persistent_) {
            // logged ids per frame (a batch logs <= batch_cap_ frames, the drain <= delay)
            plog_cnt_[0].resize(size_t(batch_cap_) + delay_ + 1);
            plog_cnt_[1].resize(size_t(batch_cap_) + delay_ + 1);
        }
    }

    dev::engine_state<Model> state() {
        dev::engine_state<Model> s{};
        s.nf = nptrs_;
        s.sf = sptrs_;
        s.rng = rng_.get();
        s.cells = graph_.cells.get();
        s.degree = graph_.degree.get();
        s.n = n_;
        s.pitch = graph_.pitch;
        s.deg_max = graph_.deg_max;
        s.queue = queue_.get();
        s.qcount = qcount_.get();
        s.Q = Q_;
        s.hist = hist_.get();
        s.hist_words = hist_words_;
        s.ages = ages_.get();
        s.caught = caught_ ? caught_.get() : nullptr;
        s.split_param = split_param_ ? split_param_.get() : nullptr;
        s.tr_p = tr_p_ ? tr_p_.get() : nullptr;
        s.tr_q = tr_q_ ? tr_q_.get() : nullptr;
        s.row_plastic = row_plastic_ ? row_plastic_.get() : nullptr;
        s.expiring = expiring_.get();
        s.expiring_count = expiring_count_.get();
        s.counters = counters_dev_.get();
        s.tile_status = tile_status_.get();
        s.tile_bal = tile_bal_.get();
        s.tile_ctr = tile_ctr_.get();
        s.done_ctr = done_ctr_.get();
        s.t_dev = t_dev_.get();
        s.t0_dev = t0_dev_.get();
        s.step_spikes = step_spikes_dev_.get();
        s.step_meas = step_meas_dev_.get();
        s.meas_lo = meas_lo_;
        s.meas_hi = meas_hi_;
        s.step_cap = batch_cap_;
        s.log = log_ids_.get();
        s.log_cursor = log_cursor_.get();
        s.log_cap = log_cap_;
        s.flags = flags_.get();
        s.dt = dt_;
        s.delay = delay_;
        s.history = history_;
        s.track_bits = has_synapses || (opt_.debug_checks && hist_);
        s.det_cnt = det_cnt_.get();
        s.det_off = det_off_.get();
        s.det_fill = det_fill_.get();
        s.det_ev = det_ev_.get();
        s.det_cap = det_cap_;
        return s;
    }

    // Pipelined kernel (detail/pipeline.cuh) when the options allow it and it
    // fits: UW update warps hold <= 8 neurons per thread in registers; shared
    // memory holds a count ring of R <= delay frames, the row prefetch windows
    // and the chunk list.  Sets pipe_* and stage_items_; false = serial kernel.
    bool setup_pipeline(int K, uint32_t wcap, uint32_t longest, uint32_t delay, size_t max_smem, size_t& smem,
                        const std::vector<uint32_t>& alo) requires population_model {
        pipe_ = false;
        pipe_bm_ = false;
        int mode = opt_.pipeline;
        if (const char* e = std::getenv("SYNQ_PIPELINE")) mode = std::atoi(e);
        if (mode == 0) return false;
        if (uint64_t(n_) * (graph_.pitch / 4) >= (1ull << 32)) return false;  // 32-bit chunk indices
        // bitmap delivery when the receive-window bitmaps are clearly smaller
        // than the ELL rows (dense connectivity, e.g. Brunel p = 0.1)
        const uint32_t C = static_cast<uint32_t>(alo.size()) - 1;
        uint32_t wq = (wcap + 127) / 128;
        wq = wq <= 1 ? 1 : (wq <= 2 ? 2 : (wq <= 4 ? 4 : 8));
        const uint64_t bm_bytes = uint64_t(n_) * C * wq * 16, ell_bytes = uint64_t(n_) * graph_.pitch * 4;
        bool use_bm = wcap <= 1024 && 3 * bm_bytes < 2 * ell_bytes && K <= 4;
        // SYNQ_BITMAP: 0 = never, 1 = when smaller (default), 2 = whenever it fits
        if (const char* e = std::getenv("SYNQ_BITMAP")) {
            const int v = std::atoi(e);
            use_bm = v == 0 ? false : (v == 2 ? (wcap <= 1024 && K <= 4) : use_bm);
        }
        pipe_bm_ = use_bm;
        // update warps: bitmap delivery runs 1024-thread CTAs (16 update + 16
        // delivery warps) whenever a CTA holds <= 1024 neurons (best at B1e9);
        // otherwise 8 once a CTA holds more than 512 neurons (the update's
        // per-thread chain is the critical path), else 4 (more deliverers)
        uint32_t uw_pref = (use_bm && longest <= 1024) ? 16 : (longest > 512 ? 8 : 4);
        if (const char* e = std::getenv("SYNQ_UW")) uw_pref = static_cast<uint32_t>(std::atoi(e));
        pipe_threads_ = dev::kPipeThreads;
        bool force_stream = false;  // SYNQ_STREAM=1: state in HBM even when registers would hold it (tests)
        if (const char* e = std::getenv("SYNQ_STREAM")) force_stream = std::atoi(e) != 0;
        if (force_stream && longest <= uint32_t(dev::kStreamChunks) * 8 * 32) {
            pipe_uw_ = 8;
            pipe_npt_ = 0;
        } else if (uw_pref == 16 && longest <= 16 * 32 * 2) {  // 1024-thread CTAs: 16 update + 16 delivery warps
            pipe_uw_ = 16;
            pipe_npt_ = longest <= 512 ? 1 : 2;
            pipe_threads_ = 1024;
        } else if (uw_pref == 8 && longest <= 8 * 32 * 8) {
            pipe_uw_ = 8;
            pipe_npt_ = longest <= 1024 ? 4 : 8;
        } else if (longest <= 4 * 32 * 8) {
            pipe_uw_ = 4;
            pipe_npt_ = longest <= 128 ? 1 : (longest <= 256 ? 2 : (longest <= 512 ? 4 : 8));
        } else if (longest <= 8 * 32 * 8) {
            pipe_uw_ = 8;
            pipe_npt_ = 8;
        } else if (longest <= uint32_t(dev::kStreamChunks) * 8 * 32) {
            pipe_uw_ = 8;
            pipe_npt_ = 0;  // streamed: the neuron state stays in HBM
        } else {
            return false;
        }
        pipe_ = true;
        cudaFuncAttributes attr{};
        SYNQ_CUDA(cudaFuncGetAttributes(&attr, kernel_fn()));
        const size_t avail = max_smem > attr.sharedSizeBytes ? max_smem - attr.sharedSizeBytes : 0;
        // L2 row prefetch at publish: pays for the ELL delivery once the
        // adjacency outgrows L2; the bitmap windows are read fast enough
        // without it (measured: same step time, fewer update instructions)
        bool prefetch = !use_bm && pipe_npt_ != 0 && graph_.pitch * 4ull * n_ > (64ull << 20);
        if (const char* e = std::getenv("SYNQ_PREFETCH")) prefetch = std::atoi(e) != 0;
        const uint32_t pf_cap = prefetch && !use_bm ? ((longest + 1) & ~1u) : 0;
        const size_t slot_bytes = size_t(K) * wcap * 4;
        // bitmap: staged windows + id + group per spike; ELL: 8-byte chunk descriptors
        const size_t item_bytes = use_bm ? size_t(wq) * 16 + 5 : 8;
        const size_t min_items = use_bm ? 1024 : 2048;
        const size_t fixed = size_t(pf_cap) * 8 + min_items * item_bytes + 16;
        if (avail <= fixed || slot_bytes == 0) {
            pipe_ = false;
            return false;
        }
        uint64_t R = std::min<uint64_t>(delay, (avail - fixed) / slot_bytes);
        while (R > 0 && R * K * wcap >= (1ull << 27)) --R;  // ring offsets are 27-bit in the chunk list
        if (R < 1) {
            pipe_ = false;
            return false;
        }
        // delivery lag (frames) behind publication: rows prefetched at publish
        // reach L2 before they are delivered; lead > lag avoids a deadlock
        uint32_t lag = prefetch ? 1 : 0;
        if (const char* e = std::getenv("SYNQ_LAG")) lag = static_cast<uint32_t>(std::max(0, std::atoi(e)));
        lag = std::min(lag, delay - 1);
        // lead: as far ahead as the queue ring allows (deliverers batch more
        // frames per pass the further the update may run ahead)
        uint32_t lead = opt_.lead ? opt_.lead : delay;
        if (const char* e = std::getenv("SYNQ_LEAD")) lead = static_cast<uint32_t>(std::max(1, std::atoi(e)));
        lead = std::max(lead, lag + 1);
        const size_t ring_bytes = ((R * K * wcap + 3) & ~uint64_t(3)) * 4;
        size_t chunk_cap = std::min<size_t>(use_bm ? 4096 : 16384,
                                            (avail - ring_bytes - size_t(pf_cap) * 8 - 16) / item_bytes);
        if (use_bm) chunk_cap &= ~size_t(15);
        smem = ring_bytes + size_t(pf_cap) * 8 + chunk_cap * item_bytes + 16;
        if (use_bm) {
            std::vector<uint32_t> wlo(alo.begin(), alo.end() - 1), whi(alo.begin() + 1, alo.end());
            build_window_bitmaps(graph_, wlo, whi, wq, bm_, stream_);
            bm_wq_ = wq;
            bm_row4_ = C * wq;
        }
        stage_items_ = static_cast<uint32_t>(chunk_cap);
        ring_R_ = static_cast<uint32_t>(R);
        lead_ = std::max<uint32_t>(1, std::min(lead, delay));
        lag_ = lag;
        pf_cap_ = pf_cap;
        return true;
    }

    template <bool BM>
    static const void* pipeline_fn(uint32_t uw, uint32_t npt) requires population_model {
        if (uw == 16) {
            if (npt <= 1) return reinterpret_cast<const void*>(dev::k_pipeline<Model, 16, 1, BM, 1024>);
            return reinterpret_cast<const void*>(dev::k_pipeline<Model, 16, 2, BM, 1024>);
        }
        if (uw == 8) {
            if (npt == 0) return reinterpret_cast<const void*>(dev::k_pipeline<Model, 8, 0, BM>);
            if (npt <= 4) return reinterpret_cast<const void*>(dev::k_pipeline<Model, 8, 4, BM>);
            return reinterpret_cast<const void*>(dev::k_pipeline<Model, 8, 8, BM>);
        }
        switch (npt) {
            case 1: return reinterpret_cast<const void*>(dev::k_pipeline<Model, 4, 1, BM>);
            case 2: return reinterpret_cast<const void*>(dev::k_pipeline<Model, 4, 2, BM>);
            case 4: return reinterpret_cast<const void*>(dev::k_pipeline<Model, 4, 4, BM>);
            default: return reinterpret_cast<const void*>(dev::k_pipeline<Model, 4, 8, BM>);
        }
    }

    // the persistent step kernel: cooperative launch (all CTAs co-resident),
    // or one thread-block cluster (the cluster engine)
    void launch_step_kernel(void** args) requires population_model {
        if (cluster_) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(tiles_);
            cfg.blockDim = dim3(kernel_threads());
            cfg.dynamicSmemBytes = smem_;
            cfg.stream = stream_;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = tiles_;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            SYNQ_CUDA(cudaLaunchKernelExC(&cfg, kernel_fn(), args));
        } else if (opt_.shard_peer) {
            // one CTA per SM, co-resident by occupancy; a plain launch lets
            // same-device shards of one process run side by side
            SYNQ_CUDA(cudaLaunchKernel(kernel_fn(), dim3(tiles_), dim3(kernel_threads()), args, smem_, stream_));
        } else {
            SYNQ_CUDA(cudaLaunchCooperativeKernel(kernel_fn(), dim3(tiles_), dim3(kernel_threads()), args, smem_,
                                                  stream_));
        }
    }

    uint32_t kernel_threads() const {
        if (cluster_) return static_cast<uint32_t>(dev::kClusterThreads);
        if (solo_) return static_cast<uint32_t>(dev::kSoloThreads);
        return pipe_ ? pipe_threads_ : static_cast<uint32_t>(dev::kPersistThreads);
    }

    const void* kernel_fn() const requires population_model {
        if (cluster_)
            return npt_ == 1 ? reinterpret_cast<const void*>(dev::k_cluster<Model, 1>)
                             : reinterpret_cast<const void*>(dev::k_cluster<Model, 2>);
        if (solo_)
            return npt_ == 1 ? reinterpret_cast<const void*>(dev::k_solo<Model, 1>)
                             : (npt_ == 2 ? reinterpret_cast<const void*>(dev::k_solo<Model, 2>)
                                          : reinterpret_cast<const void*>(dev::k_solo<Model, 4>));
        if (pipe_)
            return pipe_bm_ ? pipeline_fn<true>(pipe_uw_, pipe_npt_) : pipeline_fn<false>(pipe_uw_, pipe_npt_);
        return persistent_fn();
    }

    const void* persistent_fn() const requires population_model {
        switch (npt_) {
            case 1: return reinterpret_cast<const void*>(dev::k_persistent<Model, 1>);
            case 2: return reinterpret_cast<const void*>(dev::k_persistent<Model, 2>);
            default: return reinterpret_cast<const void*>(dev::k_persistent<Model, 4>);
        }
    }

    dev::persist_state<Model> pstate() requires population_model {
        dev::persist_state<Model> p{};
        p.nf = nptrs_;
        p.rng = rng_.get();
        p.cells = graph_.cells.get();
        p.degree = graph_.degree.get();
        p.split = split_.get();
        p.piece_lo = tile_lo_.get();
        p.cta_piece = win_lo_.get();
        p.piece_src = piece_src_.get();
        p.pitch = graph_.pitch;
        p.n = n_;
        p.C = tiles_;
        p.P = pieces_;
        p.E = publishers_;
        p.queue = queue_.get();
        p.finfo = finfo_.get();
        p.peers = npeers_ ? peers_dev_.get() : nullptr;
        p.npeers = npeers_;
        p.a_lo = shard_lo_[0];
        p.b_lo = shard_lo_[2];
        p.Q = Q_;
        p.K = K_;
        std::copy(bound_, bound_ + dev::kMaxClasses, p.bound);
        std::copy(delta_, delta_ + dev::kMaxClasses, p.delta);
        p.fold_tab = fold_tab_ ? fold_tab_.get() : nullptr;
        p.fold_t0 = fold_t0_;
        p.fold_t1 = fold_t1_;
        p.dt = dt_;
        p.delay = delay_;
        p.counters = counters_dev_.get();
        p.step_spikes = step_spikes_dev_.get();
        p.step_meas = step_meas_dev_.get();
        p.meas_lo = meas_lo_;
        p.meas_hi = meas_hi_;
        p.log = log_ids_.get();
        p.log_end = log_end_.get();
        p.log_cap = log_cap_;
        p.log_from = logged_upto_;
        p.flags = flags_.get();
        p.win_cap = win_cap_;
        p.stage_items = stage_items_;
        p.prof = prof_ ? prof_.get() : nullptr;
        p.R = ring_R_;
        p.lead = lead_;
        p.pf_cap = pf_cap_;
        p.lag = lag_;
        p.bm = pipe_bm_ ? bm_.get() : nullptr;
        p.bm_row4 = bm_row4_;
        p.wq = bm_wq_;
        p.bm_prefetch = pipe_bm_ && lag_ > 0 ? 1u : 0u;
        // bitmap: 7 frames per pass measured best at B1e9 with the fused
        // id / window staging (43.30 ms per bio-s; 6: 43.84, 8: 43.4, 4: 47.1)
        p.max_pass = pipe_bm_ ? 7 : 8;
        // NCCL-exchanging shards' launches hold delay-1 steps, all their frames
        // complete at launch: 4 frames per pass (one-rank NCCL shard 91.0 vs
        // 93.4 ms per bio-s at 6); peer shards run full-length launches
        if (pipe_bm_ && sharded() && !opt_.shard_peer) p.max_pass = 4;
        if (const char* e = std::getenv("SYNQ_MAXPASS")) p.max_pass = static_cast<uint32_t>(std::max(1, std::atoi(e)));
        p.stream_mode = 0;
        if (const char* e = std::getenv("SYNQ_WORKQ")) p.stream_mode = std::atoi(e) != 0 ? 1u : 0u;
        if (opt_.shard_peer) p.stream_mode = 0;  // the exports run in the pass-mode poller
        p.dbg = 0;
        p.progress = nullptr;
        if (std::getenv("SYNQ_WATCHDOG")) {
            if (!progress_.get()) {
                progress_.resize(size_t(8) * tiles_);
                std::memset(progress_.get(), 0, size_t(32) * tiles_);
            }
            uint32_t* d = nullptr;
            SYNQ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), progress_.get(), 0));
            p.progress = d;
        }
        if (const char* e = std::getenv("SYNQ_DBG")) p.dbg = static_cast<uint32_t>(std::atoi(e));
        return p;
    }

    // ------------------------------------------------------------ stepping
    static constexpr int kUpdateBlock = 256;
    static constexpr int kReceiveBlock = 256;
    static constexpr uint32_t kGraphSteps = 16;
    static constexpr int kWinBlock = 1024;
    static constexpr uint32_t kCompactTiles = 1024;  // k_update + k_compact up to this many tiles

    // generic step: update -> [compact] -> catch-up -> receive.  Spike
    // compaction (k_compact) is fused into the catch-up launch when the
    // frame it writes is not the one the catch-up reads (delay >= 2), and the
    // catch-up's ages advance at the start of the windowed receive
    template <class... KArgs, class... Args>
    void launch_pdl(void (*kernel)(KArgs...), uint32_t grid, uint32_t block, size_t smem, Args... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream_;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SYNQ_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
    }

    // trace-STDP models on the windowed receive: k_recv_win catches up the
    // due frame's rows itself (window by window, right before receiving them)
    // and k_catchup1 takes the expiring neurons only.  Opt-in
    // (SYNQ_FUSED_CATCHUP=1): bit-exact, but at Brunel+ 1e8 30.7-36.7 us per
    // step against 29.6 for the separate catch-up (the expiring neurons'
    // catch-up, not the frame's, is most of the catch-up time, and the
    // receive's whole-SM CTAs then wait beside it).
    bool fused_recv_catchup() const {
        if constexpr (has_synapses && dev::model_trace_stdp<Model>() && dev::model_receive_weight_only<Model>()) {
            const char* e = std::getenv("SYNQ_FUSED_CATCHUP");
            if (!e || std::atoi(e) == 0) return false;
            return win_on_ && (exact_ || !atomic_recv_) && static_cast<bool>(tr_p_) && hist_words_ == 1 &&
                   !split_catchup_ && !pdl_all_;
        } else {
            return false;
        }
    }

    void enqueue_catchup(int mode, bool fuse_compact = false) {
        if constexpr (has_synapses) {
            if (hist_words_ == 1) {
                // warp items; 4 CTAs of 8 warps per SM (60 registers)
                uint32_t g = static_cast<uint32_t>(sms_) * 4;
                // mode 0 with a side stream: frame(due) here (the receive
                // needs its synapses), the expiring neurons on side_ beside
                // the receive (disjoint rows: expiring = not transmitting);
                // fused: the expiring neurons only (part 3)
                const int part = (mode == 0 && split_catchup_) ? 1 : (mode == 0 && fused_recv_catchup()) ? 3 : 0;
                // SYNQ_CATCHUP_U=2: 2 synapses per lane, 6 CTAs per SM (A/B)
                const bool u2 = catchup_u_ == 2;
                if (u2) g = static_cast<uint32_t>(sms_) * 6;
                if (fuse_compact) {
                    g = std::max(g, ntiles_update_);
                    if (u2)
                        dev::k_catchup1<Model, true, 2, 6><<<g, 256, 0, stream_>>>(model_, state(), mode, part);
                    else if (catchup_pdl_ && mode == 0)
                        launch_pdl(dev::k_catchup1<Model, true>, g, 256, 0, Model(model_), state(), mode, part);
                    else
                        dev::k_catchup1<Model, true><<<g, 256, 0, stream_>>>(model_, state(), mode, part);
                } else {
                    if (u2)
                        dev::k_catchup1<Model, false, 2, 6><<<g, 256, 0, stream_>>>(model_, state(), mode, part);
                    else
                        dev::k_catchup1<Model, false><<<g, 256, 0, stream_>>>(model_, state(), mode, part);
                }
                if (part == 1) {
                    SYNQ_CUDA(cudaEventRecord(fork_ev_, stream_));
                    SYNQ_CUDA(cudaStreamWaitEvent(side_, fork_ev_, 0));
                    dev::k_catchup1<Model, false><<<uint32_t(sms_) * 4, 256, 0, side_>>>(model_, state(), mode, 2);
                    SYNQ_CUDA(cudaEventRecord(join_ev_, side_));
                    join_pending_ = true;
                }
                if (mode == 1)  // (mode 0: the next k_update advances the caught neurons' ages)
                    dev::k_catchup_ages<Model><<<std::max<uint32_t>(1, std::min<uint32_t>((n_ + 255) / 256, sms_)), 256, 0,
                                                 stream_>>>(state(), mode);
            } else {
                const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(n_, uint32_t(sms_) * 8));
                dev::k_catchup<Model><<<grid, 256, 0, stream_>>>(model_, state(), mode);
            }
        }
    }

    void enqueue_generic_step() {
        auto st = state();
        const bool compact = ntiles_update_ <= kCompactTiles;
        const bool win = win_on_ && (exact_ || !atomic_recv_);
        const bool fuse = compact && has_synapses && hist_words_ == 1 && delay_ >= 2 && !opt_.debug_checks;
        // SYNQ_PDL=2: programmatic dependent launches on every edge of the
        // step (update, catch-up, receive); measured slower than the receive
        // edge alone (Brunel+ 1e8: 32.1 vs 31.1 us per step): the early
        // update / catch-up CTAs wait on SMs the predecessor's tail needs
        const bool pdl = win && pdl_all_ && has_synapses && hist_words_ == 1 && delay_ >= 2;
        if (compact) {
            if (pdl)
                launch_pdl(dev::k_update<Model, kUpdateBlock, false>, ntiles_update_, kUpdateBlock, 0, Model(model_), st);
            else
                dev::k_update<Model, kUpdateBlock, false><<<ntiles_update_, kUpdateBlock, 0, stream_>>>(model_, st);
            if (!fuse) dev::k_compact<Model, kUpdateBlock><<<ntiles_update_, kUpdateBlock, 0, stream_>>>(st);
        } else {
            dev::k_update<Model, kUpdateBlock, true><<<ntiles_update_, kUpdateBlock, 0, stream_>>>(model_, st);
        }
        catchup_pdl_ = pdl && fuse;
        if (opt_.debug_checks) dev::k_check_frame<Model><<<1, 1024, 0, stream_>>>(st);
        enqueue_catchup(0, fuse);
        const int rgrid = 8 * sms_;
        if (win) {
            // programmatic dependent launch after k_catchup1 (its frame is an
            // older step's when delay >= 2): the window prologue overlaps
            // the catch-up's tail; SYNQ_PDL=0 launches it plainly
            const bool pdl = has_synapses && hist_words_ == 1 && delay_ >= 2 && pdl_;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(win_.C);
            cfg.blockDim = dim3(kWinBlock);
            cfg.dynamicSmemBytes = win_smem_;
            cfg.stream = stream_;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            Model m = model_;
            dev::recv_win rw = win_;
            rw.catchup = fused_recv_catchup() ? 1u : 0u;
            SYNQ_CUDA(cudaLaunchKernelEx(&cfg, dev::k_recv_win<Model, kWinBlock>, m, st, rw));
        } else if (exact_) {
            dev::k_det_events<Model, kReceiveBlock, false><<<rgrid, kReceiveBlock, 0, stream_>>>(st);
            dev::k_det_scan<Model, 1024><<<1, 1024, 0, stream_>>>(st);
            dev::k_det_events<Model, kReceiveBlock, true><<<rgrid, kReceiveBlock, 0, stream_>>>(st);
            dev::k_det_apply<Model, kReceiveBlock><<<grid_for(n_, kReceiveBlock), kReceiveBlock, 0, stream_>>>(model_, st);
        } else {
            dev::k_receive<Model, kReceiveBlock><<<rgrid, kReceiveBlock, 0, stream_>>>(model_, st);
        }
        if (join_pending_) {  // the next step starts after the side stream's expiring catch-up
            SYNQ_CUDA(cudaStreamWaitEvent(stream_, join_ev_, 0));
            join_pending_ = false;
        }
    }

    void ensure_graph() {
        if (graph_exec_) return;
        cudaGraph_t g = nullptr;
        SYNQ_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        for (uint32_t k = 0; k < kGraphSteps; ++k) enqueue_generic_step();
        SYNQ_CUDA(cudaStreamEndCapture(stream_, &g));
        SYNQ_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
        cudaGraphDestroy(g);
    }

    // one batch of the per-step kernel graph (generic engine), synchronous
    void run_batch(uint32_t b) {
        step_spikes_dev_.zero(stream_);
        step_meas_dev_.zero(stream_);
        const bool logging = log_on_;
        if (logging && !persistent_) {
            const unsigned long long zero2[2] = {0, 0};
            SYNQ_CUDA(cudaMemcpyAsync(log_cursor_.get(), zero2, sizeof zero2, cudaMemcpyHostToDevice, stream_));
            h2d_bytes_ += sizeof zero2;
        }
        SYNQ_CUDA(cudaEventRecord(ev_[2], stream_));
        if (persistent_) {
            if constexpr (population_model) {
                auto ps = pstate();
                int64_t t0 = t_;
                int32_t nsteps = static_cast<int32_t>(b);
                Model m = model_;
                void* args[] = {&m, &ps, &t0, &nsteps};
                launch_step_kernel(args);
                launches_ += 1;
            }
        } else {
            const int64_t t0 = t_;
            SYNQ_CUDA(cudaMemcpyAsync(t0_dev_.get(), &t0, sizeof t0, cudaMemcpyHostToDevice, stream_));
            h2d_bytes_ += sizeof t0;
            uint32_t left = b;
            if (left >= kGraphSteps) {
                ensure_graph();
                while (left >= kGraphSteps) {
                    SYNQ_CUDA(cudaGraphLaunch(graph_exec_, stream_));
                    left -= kGraphSteps;
                }
            }
            while (left--) enqueue_generic_step();
            launches_ += uint64_t(b) * kernels_per_step();
        }
        SYNQ_CUDA(cudaGetLastError());
        SYNQ_CUDA(cudaEventRecord(ev_[3], stream_));
        step_spikes_dev_.download(step_buf_.data(), b, stream_);
        step_meas_dev_.download(step_buf_.data() + b, b, stream_);
        d2h_bytes_ += 8ull * b;
        uint64_t logged = 0;
        if (logging) {
            unsigned long long cur[2] = {0, 0};
            if (persistent_)
                SYNQ_CUDA(cudaMemcpyAsync(cur, log_end_.get(), sizeof(cur[0]), cudaMemcpyDeviceToHost, stream_));
            else
                SYNQ_CUDA(cudaMemcpyAsync(cur, log_cursor_.get(), sizeof cur, cudaMemcpyDeviceToHost, stream_));
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            logged = persistent_ ? cur[0] : cur[(t_ + b) & 1];
            logged = std::min<uint64_t>(logged, log_cap_);
            log_ids_.download(log_host_.data(), logged, stream_);
            d2h_bytes_ += 16 + 4 * logged;
        }
        pull_counters();  // synchronises
        float ms = 0;
        SYNQ_CUDA(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
        kernel_seconds_ += ms * 1e-3;
        if (flags_host_[0]) throw device_error("spike log overflow (batch too large for the frame log)");
        if (flags_host_[1]) throw device_error("ordered delivery scratch overflow");
        check_debug_flags();

        // per-step bookkeeping, frames_consumed (engine.hpp:371-380)
        for (uint32_t k = 0; k < b; ++k) {
            step_spikes_host_.push_back(step_buf_[k]);
            step_measured_.push_back(step_buf_[b + k]);
            if (t_ + k - int64_t(delay_) + 1 >= 0) ++counters_.frames_consumed;
        }
        counters_.steps += b;
        const int64_t t_end = t_ + b;
        if (logging) {
            // generic: frames t_ .. t_end-1; persistent: frames logged_upto_ .. t_end-delay
            const int64_t last = persistent_ ? t_end - int64_t(delay_) : t_end - 1;
            emit_logged(log_host_.data(), logged, last);
        }
        t_ = t_end;
    }

    // persistent engine: enqueue one batch into slot `slot` (kernel, step
    // counts -> pinned host, completion event); t_ advances at launch
    void launch_persistent(uint32_t b, int slot) {
        if constexpr (population_model) {
            auto ps = pstate();
            // one counter block per slot: spikes [0, b), measured [b, 2b), so a
            // batch costs one memset and one copy of 2b words
            ps.step_spikes = step_ctr_dev_.get() + size_t(slot) * 2 * batch_cap_;
            ps.step_meas = ps.step_spikes + b;
            batch_slot& fl = slots_[slot];
            fl.t0 = t_;
            fl.b = b;
            fl.logging = log_on_;
            if (log_on_) {
                ps.log = plog_[slot].get();
                ps.log_end = plog_end_.get() + slot;
                ps.log_cnt = plog_cnt_[slot].get();
                ps.log_cap = log_cap_;
                ps.log_from = log_pred_;
                fl.log_from = log_pred_;
                plog_end_[slot] = 0;
                // frames logged_upto_ .. t_end-delay are emitted when it finishes
                log_pred_ = std::max(log_pred_, t_ + int64_t(b) - int64_t(delay_) + 1);
            } else {
                ps.log = nullptr;
            }
            SYNQ_CUDA(cudaMemsetAsync(ps.step_spikes, 0, sizeof(uint32_t) * 2 * b, stream_));
            if (!fl.ev[0])
                for (auto& e : fl.ev) SYNQ_CUDA(cudaEventCreate(&e));
            SYNQ_CUDA(cudaEventRecord(fl.ev[0], stream_));
            int64_t t0 = t_;
            int32_t nsteps = static_cast<int32_t>(b);
            Model m = model_;
            void* args[] = {&m, &ps, &t0, &nsteps};
            launch_step_kernel(args);
            SYNQ_CUDA(cudaGetLastError());
            launches_ += 1;
            if (opt_.debug_checks) {
                dev::k_check_persist<Model><<<b, 256, 0, stream_>>>(ps, t0, b);
                SYNQ_CUDA(cudaGetLastError());
                launches_ += 1;
            }
            SYNQ_CUDA(cudaEventRecord(fl.ev[1], stream_));
            uint32_t* hb = step_buf_.data() + size_t(slot) * 2 * batch_cap_;
            SYNQ_CUDA(cudaMemcpyAsync(hb, ps.step_spikes, sizeof(uint32_t) * 2 * b, cudaMemcpyDeviceToHost, stream_));
            d2h_bytes_ += 8ull * b;
            SYNQ_CUDA(cudaEventRecord(fl.ev[2], stream_));
            t_ += b;
        }
    }

    // wait for slot `slot`'s batch and do its host bookkeeping / emission
    void finish_persistent(int slot) {
        batch_slot& fl = slots_[slot];
        if (const char* e = std::getenv("SYNQ_WATCHDOG"); e && progress_.get()) {
            // debugging aid: the delivery pollers' progress after a timeout
            const auto t_end = clock::now() + std::chrono::duration<double>(std::atof(e));
            while (cudaEventQuery(fl.ev[2]) == cudaErrorNotReady) {
                if (clock::now() > t_end) {
                    std::fprintf(stderr, "[synq watchdog] rank %u t0 %lld C %u\n", opt_.shard_rank,
                                 static_cast<long long>(fl.t0), tiles_);
                    for (uint32_t c = 0; c < tiles_; ++c) {
                        const volatile uint32_t* w = progress_.get() + 8 * c;
                        std::fprintf(stderr, "  cta %u: r_next %u next_exp-t0 %u updated %u delivered %u where %u\n", c,
                                     w[0], w[1], w[2], w[3], w[4]);
                    }
                    std::fflush(stderr);
                    std::abort();
                }
                std::this_thread::sleep_for(std::chrono::microseconds(50));
            }
        }
        SYNQ_CUDA(cudaEventSynchronize(fl.ev[2]));
        float ms = 0;
        SYNQ_CUDA(cudaEventElapsedTime(&ms, fl.ev[0], fl.ev[1]));
        kernel_seconds_ += ms * 1e-3;
        const uint32_t b = fl.b;
        const uint32_t* hb = step_buf_.data() + size_t(slot) * 2 * batch_cap_;
        // per-step bookkeeping, frames_consumed (engine.hpp:371-380)
        for (uint32_t k = 0; k < b; ++k) {
            step_spikes_host_.push_back(hb[k]);
            step_measured_.push_back(hb[b + k]);
            if (fl.t0 + k - int64_t(delay_) + 1 >= 0) ++counters_.frames_consumed;
        }
        counters_.steps += b;
        if (fl.logging) {
            const uint64_t end = plog_end_[slot];
            if (end > log_cap_) throw device_error("spike log overflow (batch too large for the frame log)");
            d2h_bytes_ += 8 + 4 * end;  // written to host memory by the kernel
            emit_logged(plog_[slot].data(), end, fl.t0 + int64_t(b) - int64_t(delay_), plog_cnt_[slot].data(),
                        fl.log_from);
        }
    }

    uint64_t kernels_per_step() const {
        const bool win = win_on_ && (exact_ || !atomic_recv_);
        const bool compact = ntiles_update_ <= kCompactTiles;
        const bool fuse = compact && has_synapses && hist_words_ == 1 && delay_ >= 2 && !opt_.debug_checks;
        return 2 + (compact && !fuse ? 1 : 0) + (has_synapses ? (split_catchup_ ? 2 : 1) : 0) +
               (!win && exact_ ? 3 : 0) +
               (opt_.debug_checks ? 1 : 0);
    }

    // frames logged_upto_ .. last are the next entries of `log`, in order.
    // cnts[f - cnt_from]: ids logged for frame f by the persistent kernel (the
    // merged frame; on a shard step_spikes_host_ only counts local spikes),
    // else the per-step spike counts of the generic engine
    void emit_logged(const uint32_t* log, uint64_t logged, int64_t last, const uint32_t* cnts = nullptr,
                     int64_t cnt_from = 0) {
        uint64_t off = 0;
        for (int64_t f = logged_upto_; f <= last; ++f) {
            const uint32_t cnt = cnts ? cnts[f - cnt_from] : step_spikes_host_[static_cast<size_t>(f)];
            const uint64_t a = std::min(off, logged), e = std::min(off + cnt, logged);
            off += cnt;
            emit(f, std::span<const uint32_t>(log + a, e - a));
        }
        logged_upto_ = std::max(logged_upto_, last + 1);
        log_pred_ = std::max(log_pred_, logged_upto_);
    }

    void drain_log() {
        if constexpr (population_model) {
            auto ps = pstate();
            ps.log = plog_[0].get();
            ps.log_end = plog_end_.get();
            ps.log_cnt = plog_cnt_[0].get();
            ps.log_cap = log_cap_;
            plog_end_[0] = 0;
            dev::k_log_drain<Model><<<1, 1024, 0, stream_>>>(ps, logged_upto_, t_ - 1);
            SYNQ_CUDA(cudaGetLastError());
            launches_ += 1;
            SYNQ_CUDA(cudaStreamSynchronize(stream_));
            const uint64_t logged = std::min<uint64_t>(plog_end_[0], log_cap_);
            d2h_bytes_ += 8 + 4 * logged;
            emit_logged(plog_[0].data(), logged, t_ - 1, plog_cnt_[0].data(), logged_upto_);
        }
    }

    // device-side check_frame results (k_check_frame / k_check_persist)
    void check_debug_flags() {
        if (!opt_.debug_checks || !flags_host_[3]) return;
        const uint32_t f = flags_host_[3];
        flags_host_[3] = 0;
        const uint32_t zero = 0;
        SYNQ_CUDA(cudaMemcpyAsync(flags_.get() + 3, &zero, sizeof zero, cudaMemcpyHostToDevice, stream_));
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        if (f & 1) throw std::logic_error("spike frame not sorted/unique");
        throw std::logic_error("spike queue and bitmask disagree");
    }

    void emit(int64_t t, std::span<const uint32_t> frame) {
        if (opt_.debug_checks)
            for (size_t i = 1; i < frame.size(); ++i)
                if (frame[i - 1] >= frame[i]) throw std::logic_error("spike frame not sorted/unique");
        if (tap_) tap_(t, frame);
    }

    void pull_counters() {
        unsigned long long c[dev::C_COUNT];
        counters_dev_.download(c, dev::C_COUNT, stream_);
        flags_.download(flags_host_, 4, stream_);
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
        d2h_bytes_ += sizeof c + sizeof flags_host_;
        counters_.spikes = c[dev::C_SPIKES];
        counters_.deliveries = c[dev::C_DELIVERIES];
        counters_.synapse_updates = c[dev::C_SYN_UPDATES];
        counters_.expiry_batches = c[dev::C_EXPIRY];
    }

    // ------------------------------------------------------------ mirrors
    void invalidate_mirrors() {
        std::fill(std::begin(nmirror_valid_), std::end(nmirror_valid_), false);
        std::fill(std::begin(smirror_valid_), std::end(smirror_valid_), false);
    }
    template <size_t I = 0>
    void push_neuron_cols() {
        if constexpr (I < neuron_fields::count) {
            using T = field_t<I, neuron_fields>;
            if (ndirty_[I])
                SYNQ_CUDA(cudaMemcpyAsync(neuron_cols_[I].get(), host_neurons_.template data<I>(),
                                          n_ * sizeof(T), cudaMemcpyHostToDevice, stream_));
            ndirty_[I] = false;
            push_neuron_cols<I + 1>();
        }
    }
    template <size_t I = 0>
    void push_syn_cols() {
        if constexpr (I < synapse_fields::count) {
            using T = field_t<I, synapse_fields>;
            if (sdirty_[I])
                SYNQ_CUDA(cudaMemcpyAsync(syn_cols_[I].get(), host_synapses_.template data<I>(),
                                          synapse_capacity() * sizeof(T), cudaMemcpyHostToDevice, stream_));
            sdirty_[I] = false;
            push_syn_cols<I + 1>();
        }
    }
    void push_mirrors() {
        push_neuron_cols();
        if constexpr (has_synapses) push_syn_cols();
        SYNQ_CUDA(cudaStreamSynchronize(stream_));
    }

    // ------------------------------------------------------------ members
    network_desc desc_;
    Model model_;
    engine_options opt_;
    uint32_t n_ = 0;
    float dt_ = 1.0f;
    uint32_t delay_ = 1;
    uint32_t history_ = 0;
    bool exact_ = false;
    int sms_ = 148;
    cudaStream_t stream_ = nullptr;

    device_graph graph_;
    mutable std::unique_ptr<adjacency_list> adj_mirror_;

    std::vector<dev_array<unsigned char>> neuron_cols_, syn_cols_;
    dev::field_ptrs<neuron_fields> nptrs_{};
    dev::field_ptrs<synapse_fields> sptrs_{};
    dev_array<xorshift> rng_;
    dev_array<uint32_t> ages_, expiring_, expiring_count_;
    dev_array<uint64_t> hist_;
    uint32_t hist_words_ = 1;
    dev_array<uint32_t> queue_, qcount_;
    uint32_t Q_ = 1;
    dev_array<unsigned long long> counters_dev_, tile_status_, log_cursor_;
    dev_array<uint32_t> tile_bal_;
    dev_array<uint8_t> caught_, row_plastic_;
    dev_array<float> tr_p_, tr_q_;  // trace-STDP per-neuron trace rings
    // split catch-up (SYNQ_SPLIT_CATCHUP=1, with the windowed receive)
    dev_array<unsigned long long> split_param_;
    cudaStream_t side_ = nullptr;
    cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
    bool split_catchup_ = false, join_pending_ = false;
    dev_array<uint32_t> tile_ctr_, done_ctr_, flags_;
    uint32_t ntiles_update_ = 1;
    dev_array<int64_t> t_dev_, t0_dev_;
    dev_array<uint32_t> step_spikes_dev_, step_meas_dev_;
    dev_array<uint32_t> step_ctr_dev_;  // persistent engine: 2 slots x {spikes, measured} x batch_cap
    pinned_array<uint32_t> step_buf_;
    dev_array<uint32_t> det_cnt_, det_off_, det_fill_;
    dev_array<unsigned long long> det_ev_;
    uint64_t det_cap_ = 0;
    dev_array<uint32_t> log_ids_;
    dev_array<unsigned long long> log_end_;
    pinned_array<uint32_t> log_host_;
    int64_t logged_upto_ = 0;
    int64_t log_pred_ = 0;  // first frame the next persistent launch logs
    bool log_on_ = false;
    pinned_array<uint32_t> plog_[2];          // persistent engine: frame logs, one per batch slot
    pinned_array<unsigned long long> plog_end_;
    pinned_array<uint32_t> plog_cnt_[2];  // ids logged per frame, one per batch slot
    struct batch_slot {
        int64_t t0 = 0;
        int64_t log_from = 0;
        uint32_t b = 0;
        bool logging = false;
        cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // kernel start, kernel end, copies done
    };
    batch_slot slots_[2];
    cudaEvent_t ev_[4] = {nullptr, nullptr, nullptr, nullptr};
    double device_seconds_ = 0, kernel_seconds_ = 0;
    uint64_t launches_ = 0, h2d_bytes_ = 0, d2h_bytes_ = 0;
    uint64_t log_cap_ = 0;
    uint32_t flags_host_[4] = {0, 0, 0, 0};
    cudaGraphExec_t graph_exec_ = nullptr;
    uint32_t batch_cap_ = 1000;

    // persistent engine
    bool persistent_ = false;
    uint32_t tiles_ = 0;
    std::vector<uint32_t> tile_lo_host_;
    dev_array<uint32_t> tile_lo_, win_lo_, split_;
    dev_array<unsigned long long> finfo_;
    int K_ = 0;
    uint32_t bound_[dev::kMaxClasses] = {};
    float delta_[dev::kMaxClasses] = {};
    dev_array<float> fold_tab_;
    dev::recv_win win_{};  // generic engine: ordered windowed receive
    dev_array<uint32_t> win_lo_dev_, win_split_;
    size_t win_smem_ = 0;
    bool win_on_ = false, atomic_recv_ = false, pdl_ = true;
    int catchup_u_ = 4;
    bool catchup_pdl_ = false, pdl_all_ = false;
    uint32_t fold_t0_ = 0, fold_t1_ = 0;
    uint32_t win_cap_ = 0, pieces_ = 0, publishers_ = 0, stage_items_ = 0;
    dev_array<uint32_t> piece_src_;
    // shard exchange
    std::vector<std::array<uint32_t, 3>> remote_;  // per rank: publisher entry, A lo, B lo
    std::vector<uint32_t> all_ra_, all_ub_;          // every rank's receiving / update-only ranges
    dev::xbits_layout xl_{};
    dev_array<uint32_t> xremotes_, xsend_, xrecv_;
    void* nccl_ = nullptr;  // ncclComm_t of the in-engine exchange
    // peer exchange: links to the other shards' rings, IPC mappings
    dev_array<dev::peer_link> peers_dev_;
    uint32_t npeers_ = 0;
    bool peers_connected_ = false;
    std::vector<void*> ipc_opened_;
    pinned_array<uint32_t> progress_;  // SYNQ_WATCHDOG: per-CTA poller progress (mapped)
    std::array<uint32_t, 4> shard_lo_{};           // this shard: A [lo, hi), B [lo, hi)
    shard_cut cut_;                                // W > 1: rank ranges from the description
    std::vector<int64_t> imported_upto_;            // frames < this imported, per rank
    dev_array<uint32_t> xbuf_;
    dev_array<uint32_t> ibuf_[2];
    std::vector<uint32_t> xcounts_;                      // export / import staging
    int64_t last_batch_t0_ = 0;
    uint32_t last_batch_b_ = 0;
    int npt_select_ = 1;
    bool pipe_ = false;  // pipelined kernel (detail/pipeline.cuh)
    bool pipe_bm_ = false;  // ... with bitmap delivery
    bool solo_ = false;     // single-CTA engine (detail/solo.cuh)
    bool cluster_ = false;  // one-cluster engine (detail/cluster.cuh)
    bool cluster_failed_ = false;
    dev_array<uint4> bm_;
    uint32_t bm_wq_ = 0, bm_row4_ = 0;
    uint32_t pipe_uw_ = 4, pipe_npt_ = 1, ring_R_ = 0, lead_ = 0, lag_ = 0, pf_cap_ = 0;
    uint32_t pipe_threads_ = dev::kPipeThreads;
    size_t smem_ = 0;
    int npt_ = 1;
    dev_array<unsigned long long> prof_;

    // host-visible state
    neuron_store host_neurons_;
    synapse_store host_synapses_;
    bool nmirror_valid_[16] = {}, ndirty_[16] = {};
    bool smirror_valid_[16] = {}, sdirty_[16] = {};
    mutable std::vector<uint32_t> ages_host_;
    std::vector<uint32_t> expiring_host_;
    uint32_t meas_lo_ = 0, meas_hi_ = 0;
    std::vector<uint32_t> step_measured_, step_spikes_host_;
    uint64_t host_steps_done_ = 0;

    int64_t t_ = 0;
    tap_fn tap_;
    engine_counters counters_;
    phase_seconds timings_;
};

}  // namespace synq
