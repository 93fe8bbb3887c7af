// C ABI of the B200 synq engine (declared in include/synq/synq.h).
//
// Mirrors the reference's runtime + C surface (proj/src/sim_runtime.cpp,
// proj/src/capi.cpp): a type-erased simulation over the four shipped models,
// exception -> status mapping, thread-local error text, stats/raster output.
// Differences are confined to where the work runs: every simulation here is a
// synq::network<M> on the B200 (include/synq/engine.hpp).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <thread>
#include <fstream>
#include <functional>
#include <iostream>
#include <memory>
#include <new>
#include <optional>
#include <string>

#include "synq/analysis.hpp"
#include "synq/engine.hpp"
#include "synq/models/benchmarks.hpp"
#include "synq/params.hpp"
#include "synq/synq.h"

namespace synq {
namespace {

// f(a, b) over [0, n) split into contiguous ranges on up to 16 host threads
// (large rasters); f must not throw
template <class F>
void parallel_ranges(size_t n, F&& f) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (size_t(1) << 18) || hw == 1) {
        f(size_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (n + hw - 1) / hw;
    for (unsigned k = 1; k < hw; ++k)
        pool.emplace_back([&f, n, per, k] { f(std::min(n, k * per), std::min(n, (k + 1) * per)); });
    f(size_t(0), std::min(n, per));
    for (auto& th : pool) th.join();
}

struct sim_config {  // sim_runtime.hpp:15-21
    param_set params = builtin_defaults();
    engine_options engine;
    bool record_spikes = false;
    std::optional<double> dt_ms;
    std::optional<uint32_t> delay_steps;
};

class sim_base {  // sim_runtime.hpp:26-61 + B200 extensions
public:
    virtual ~sim_base() = default;
    virtual void step() = 0;
    virtual void run(int64_t steps) = 0;
    virtual void flush() = 0;
    virtual model_kind kind() const = 0;
    virtual uint32_t neurons() const = 0;
    virtual uint64_t synapses() const = 0;
    virtual uint64_t synapse_capacity() const = 0;
    virtual int64_t now() const = 0;
    virtual double dt() const = 0;
    virtual uint32_t delay() const = 0;
    virtual uint64_t seed() const = 0;
    virtual bool deterministic() const = 0;
    virtual unsigned workers() const = 0;
    virtual double scale_c() const = 0;
    virtual const engine_counters& counters() const = 0;
    virtual const phase_seconds& timings() const = 0;
    virtual engine_memory memory_actual() const = 0;
    virtual double measured_rate() const = 0;
    virtual uint64_t measured_spike_count() const = 0;
    virtual uint32_t measured_neurons() const = 0;
    virtual int64_t warmup_steps() const = 0;
    virtual const spike_raster& raster() const = 0;  // materialised on demand (file output)
    virtual uint64_t raster_size() const = 0;
    virtual void raster_copy(int64_t* steps, uint32_t* ids) const = 0;
    virtual bool persistent() const = 0;
    virtual bool pipelined() const = 0;
    virtual bool solo() const = 0;
    virtual bool cluster() const = 0;
    virtual bool bitmap_delivery() const = 0;
    virtual bool exact() const = 0;
    virtual const std::vector<uint32_t>& step_spikes() const = 0;
    virtual void neuron_field_bytes(uint32_t f, void* out, uint64_t bytes) = 0;
    virtual void synapse_field_bytes(uint32_t f, void* out, uint64_t bytes) = 0;
    virtual void ages_copy(uint32_t* out, uint64_t capacity) = 0;
    virtual const adjacency_list& graph() const = 0;
    virtual uint64_t fixups() const = 0;
    virtual void device_time(double out[2]) const = 0;
    virtual uint64_t launches() const = 0;
    virtual void transfers(uint64_t out[2]) const = 0;
    virtual void set_record(bool on) = 0;
    virtual std::vector<double> phase_cycles() const = 0;
    virtual unsigned tiles() const = 0;
    virtual uint64_t shard_capacity() const = 0;
    virtual std::array<uint32_t, 4> shard_range() const = 0;
    virtual uint64_t shard_export(void* dst, uint64_t cap, bool device) = 0;
    virtual void shard_import(const void* src, uint64_t words, uint32_t from, bool device) = 0;
    virtual uint64_t shard_bits_words() const = 0;
    virtual void shard_export_bits(void* dst) = 0;
    virtual void shard_import_bits(const void* all) = 0;
    virtual synq::peer_endpoint peer_endpoint() const = 0;
    virtual void peer_connect(const std::vector<synq::peer_endpoint>& eps) = 0;
    virtual void peer_ipc_handle(void* out) const = 0;
    virtual void peer_connect_ipc(const void* all) = 0;
    virtual uint32_t shard_world() const = 0;

    void write_stats(std::ostream& out) const;
    void write_stats_to(const std::string& path) const;
};

template <class FL, size_t I = 0, class Net>
void copy_neuron_field(Net& net, uint32_t f, void* out, uint64_t bytes) {
    if constexpr (I < FL::count) {
        if (f == I) {
            auto s = net.template neuron_field<I>();
            if (bytes < s.size_bytes()) throw std::invalid_argument("buffer too small for field");
            std::memcpy(out, s.data(), s.size_bytes());
            return;
        }
        copy_neuron_field<FL, I + 1>(net, f, out, bytes);
    } else {
        throw std::out_of_range("neuron field index out of range");
    }
}

template <class FL, size_t I = 0, class Net>
void copy_synapse_field(Net& net, uint32_t f, void* out, uint64_t bytes) {
    if constexpr (I < FL::count) {
        if (f == I) {
            auto s = net.template synapse_field<I>();
            if (bytes < s.size_bytes()) throw std::invalid_argument("buffer too small for field");
            std::memcpy(out, s.data(), s.size_bytes());
            return;
        }
        copy_synapse_field<FL, I + 1>(net, f, out, bytes);
    } else {
        throw std::out_of_range("synapse field index out of range");
    }
}

template <class M>
class sim_impl final : public sim_base {  // sim_runtime.cpp:13-90
public:
    sim_impl(model_kind kind, model_build<M> b, const sim_config& cfg)
        : kind_(kind), mb_(b.measure_begin), me_(b.measure_end), scale_(b.scale_c),
          record_(cfg.record_spikes) {
        if (cfg.dt_ms) b.desc.dt = *cfg.dt_ms;
        if (cfg.delay_steps) b.desc.delay = *cfg.delay_steps;
        warmup_ = static_cast<int64_t>(std::ceil(param(cfg.params, "measure.warmup_ms") / b.desc.dt));
        if (param(cfg.params, "measure.exclude_stimulus") == 0.0) {
            mb_ = 0;
            me_ = b.desc.neuron_count();
        }
        net_ = std::make_unique<network<M>>(b.desc, b.model, cfg.engine);
        net_->set_measure_range(mb_, me_);
        raster_.dt = net_->dt();
        raster_.neurons = net_->neuron_count();
        if (record_) set_record(true);
    }

    std::vector<double> phase_cycles() const override { return net_->phase_cycles(); }
    unsigned tiles() const override { return net_->tiles(); }
    std::array<uint32_t, 4> shard_range() const override { return net_->shard_range(); }
    uint64_t shard_capacity() const override { return net_->sharded() ? net_->export_capacity() : 0; }
    uint64_t shard_export(void* dst, uint64_t cap, bool device) override {
        return net_->export_frames(dst, cap, device);
    }
    void shard_import(const void* src, uint64_t words, uint32_t from, bool device) override {
        net_->import_frames(src, words, from, device);
    }
    uint64_t shard_bits_words() const override { return net_->exchange_block_words(); }
    void shard_export_bits(void* dst) override { net_->export_bits(static_cast<uint32_t*>(dst)); }
    void shard_import_bits(const void* all) override { net_->import_bits(static_cast<const uint32_t*>(all)); }
    synq::peer_endpoint peer_endpoint() const override { return net_->peer_buffers(); }
    void peer_connect(const std::vector<synq::peer_endpoint>& eps) override { net_->connect_peers(eps); }
    void peer_ipc_handle(void* out) const override { net_->peer_ipc_handle(out); }
    void peer_connect_ipc(const void* all) override { net_->connect_peers_ipc(all); }
    uint32_t shard_world() const override { return net_->options().shard_world; }
    void set_record(bool on) override {
        record_ = on;
        // the recorded raster is kept compact: the ids of every frame in
        // order plus one (step, end) run per step with spikes; clear() keeps
        // the capacity, so a recurring recording reuses the pages
        rids_.clear();
        rruns_.clear();
        raster_.records.clear();
        raster_valid_ = true;
        if (on)
            net_->set_spike_tap([this](int64_t t, std::span<const uint32_t> frame) {
                const size_t o = rids_.size(), n = frame.size();
                if (n == 0) return;
                if (rids_.capacity() < o + n) rids_.reserve(std::max<size_t>(2 * rids_.capacity(), o + n + (size_t(1) << 20)));
                rids_.insert(rids_.end(), frame.begin(), frame.end());
                rruns_.push_back({t, o + n});
                raster_valid_ = false;
            });
        else
            net_->set_spike_tap(nullptr);
    }

    void step() override { net_->step(); }
    void run(int64_t steps) override { net_->run(steps); }
    void flush() override { net_->flush(); }
    model_kind kind() const override { return kind_; }
    uint32_t neurons() const override { return net_->neuron_count(); }
    uint64_t synapses() const override { return net_->edge_count(); }
    uint64_t synapse_capacity() const override { return net_->synapse_capacity(); }
    int64_t now() const override { return net_->now(); }
    double dt() const override { return net_->dt(); }
    uint32_t delay() const override { return net_->delay(); }
    uint64_t seed() const override { return net_->seed(); }
    bool deterministic() const override { return net_->deterministic(); }
    unsigned workers() const override { return net_->worker_count(); }
    double scale_c() const override { return scale_; }
    const engine_counters& counters() const override { return net_->counters(); }
    const phase_seconds& timings() const override { return net_->timings(); }
    engine_memory memory_actual() const override { return net_->memory(); }

    double measured_rate() const override {  // sim_runtime.cpp:42-47
        const int64_t steps = now() - warmup_;
        if (steps <= 0 || me_ <= mb_) return 0.0;
        return firing_rate(measured_spike_count(), me_ - mb_, steps);
    }
    uint64_t measured_spike_count() const override {
        const auto& v = net_->step_measured();
        uint64_t total = 0;
        for (size_t i = static_cast<size_t>(std::min<int64_t>(warmup_, now())); i < v.size(); ++i)
            total += v[i];
        return total;
    }
    uint32_t measured_neurons() const override { return me_ - mb_; }
    int64_t warmup_steps() const override { return warmup_; }
    const spike_raster& raster() const override {
        if (!raster_valid_) {
            raster_.records.resize(rids_.size());
            raster_copy_records(raster_.records.data());
            raster_valid_ = true;
        }
        return raster_;
    }
    uint64_t raster_size() const override { return rids_.size(); }
    // (steps, ids) of the recorded raster, split over host threads by record
    // range (each range: its first run by binary search, then fills + copies)
    void raster_copy(int64_t* steps, uint32_t* ids) const override {
        parallel_ranges(rids_.size(), [&](size_t a, size_t b) {
            size_t r = std::upper_bound(rruns_.begin(), rruns_.end(), a,
                                        [](size_t x, const std::pair<int64_t, size_t>& run) { return x < run.second; }) -
                       rruns_.begin();
            for (size_t i = a; i < b; ++r) {
                const size_t e = std::min(b, rruns_[r].second);
                std::fill(steps + i, steps + e, rruns_[r].first);
                std::memcpy(ids + i, rids_.data() + i, (e - i) * sizeof(uint32_t));
                i = e;
            }
        });
    }
    bool persistent() const override { return net_->persistent(); }
    bool pipelined() const override { return net_->pipelined(); }
    bool solo() const override { return net_->solo(); }
    bool cluster() const override { return net_->cluster(); }
    bool bitmap_delivery() const override { return net_->bitmap_delivery(); }
    bool exact() const override { return net_->exact(); }
    const std::vector<uint32_t>& step_spikes() const override { return net_->step_spike_counts(); }
    void neuron_field_bytes(uint32_t f, void* out, uint64_t bytes) override {
        copy_neuron_field<typename M::neuron_fields>(*net_, f, out, bytes);
    }
    void ages_copy(uint32_t* out, uint64_t capacity) override {
        if constexpr (network<M>::has_synapses) {
            auto a = net_->ages();
            if (capacity < a.size()) throw std::invalid_argument("buffer too small for ages");
            std::memcpy(out, a.data(), a.size_bytes());
        } else {
            throw std::invalid_argument("model has no synapse state");
        }
    }
    void synapse_field_bytes(uint32_t f, void* out, uint64_t bytes) override {
        if constexpr (network<M>::has_synapses)
            copy_synapse_field<typename network<M>::synapse_fields>(*net_, f, out, bytes);
        else
            throw std::invalid_argument("model has no synapse state");
    }
    const adjacency_list& graph() const override { return net_->graph(); }
    uint64_t fixups() const override { return net_->construction_fixups(); }
    void device_time(double out[2]) const override {
        out[0] = net_->device_seconds();
        out[1] = net_->kernel_seconds();
    }
    uint64_t launches() const override { return net_->kernel_launches(); }
    void transfers(uint64_t out[2]) const override {
        out[0] = net_->h2d_bytes();
        out[1] = net_->d2h_bytes();
    }

private:
    model_kind kind_;
    uint32_t mb_, me_;
    double scale_;
    bool record_;
    int64_t warmup_ = 0;
    std::unique_ptr<network<M>> net_;
    std::vector<uint32_t> rids_;                       // recorded ids, frame after frame
    std::vector<std::pair<int64_t, size_t>> rruns_;  // (step, end in rids_) per step with spikes
    mutable spike_raster raster_;                      // record form, built for file output
    mutable bool raster_valid_ = true;
    void raster_copy_records(spike_record* out) const {
        parallel_ranges(rids_.size(), [&](size_t a, size_t b) {
            size_t r = std::upper_bound(rruns_.begin(), rruns_.end(), a,
                                        [](size_t x, const std::pair<int64_t, size_t>& run) { return x < run.second; }) -
                       rruns_.begin();
            for (size_t i = a; i < b; ++r) {
                const size_t e = std::min(b, rruns_[r].second);
                for (; i < e; ++i) out[i] = {rruns_[r].first, rids_[i]};
            }
        });
    }
};

// sim_runtime.cpp:98-141 (+ engine line)
void sim_base::write_stats(std::ostream& out) const {
    const auto& c = counters();
    const auto& t = timings();
    const auto mem = memory_actual();
    const double rate = measured_rate();
    out << "model=" << model_name(kind()) << "\n"
        << "neurons=" << neurons() << "\n"
        << "synapses=" << synapses() << "\n"
        << "synapse_capacity=" << synapse_capacity() << "\n"
        << "seed=" << seed() << "\n"
        << "threads=" << workers() << "\n"
        << "deterministic=" << (deterministic() ? 1 : 0) << "\n"
        << "dt_ms=" << dt() << "\n"
        << "delay_steps=" << delay() << "\n"
        << "steps=" << now() << "\n"
        << "scale_c=" << scale_c() << "\n"
        << "construct_s=" << t.construct << "\n"
        << "init_neurons_s=" << t.init_neurons << "\n"
        << "init_synapses_s=" << t.init_synapses << "\n"
        << "setup_s=" << (t.construct + t.init_neurons + t.init_synapses) << "\n"
        << "sim_s=" << t.simulate << "\n"
        << "steps_per_s=" << (t.simulate > 0 ? static_cast<double>(now()) / t.simulate : 0.0) << "\n"
        << "spikes_total=" << c.spikes << "\n"
        << "deliveries=" << c.deliveries << "\n"
        << "synapse_updates=" << c.synapse_updates << "\n"
        << "firing_rate=" << rate << "\n"
        << "firing_rate_hz=" << (dt() > 0 ? rate * 1000.0 / dt() : 0.0) << "\n"
        << "measured_neurons=" << measured_neurons() << "\n"
        << "warmup_steps=" << warmup_steps() << "\n"
        << "mem_actual_bytes=" << mem.total() << "\n";
    try {
        const auto est = memory_estimate(kind());
        out << "mem_est_neuron_b=" << est.neuron_total() << "\n"
            << "mem_est_synapse_b=" << est.synapse_total() << "\n"
            << "mem_est_total_bytes=" << static_cast<uint64_t>(est.total_bytes(neurons(), synapses()))
            << "\n";
    } catch (const std::invalid_argument&) {
    }
    out << "engine="
        << (bitmap_delivery() ? "b200-pipelined-bitmap"
                              : (pipelined() ? "b200-pipelined" : (persistent() ? "b200-persistent" : "b200-graph")))
        << "\n"
        << "exact=" << (exact() ? 1 : 0) << "\n";
    out.flush();
}

void sim_base::write_stats_to(const std::string& path) const {
    if (path.empty() || path == "-") {
        write_stats(std::cout);
        return;
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open stats file for writing: " + path);
    write_stats(out);
    if (!out) throw std::runtime_error("failed writing stats file: " + path);
}

std::unique_ptr<sim_base> make_sim_from_desc(model_kind k, const network_desc& d, const sim_config& cfg) {
    switch (k) {
        case model_kind::pingpong:
            return std::make_unique<sim_impl<pingpong_model>>(k, build_pingpong_from_desc(d, cfg.params), cfg);
        case model_kind::vogels:
            return std::make_unique<sim_impl<vogels_model>>(k, build_vogels_from_desc(d, cfg.params), cfg);
        case model_kind::brunel:
            return std::make_unique<sim_impl<brunel_model>>(k, build_brunel_from_desc(d, cfg.params), cfg);
        case model_kind::brunel_plus:
            return std::make_unique<sim_impl<brunel_plus_model>>(
                k, build_brunel_plus_from_desc(d, cfg.params), cfg);
    }
    throw std::invalid_argument("make_sim_from_desc: bad model kind");
}

std::unique_ptr<sim_base> make_sim(model_kind k, uint32_t neurons, const sim_config& cfg) {
    switch (k) {
        case model_kind::pingpong:
            return std::make_unique<sim_impl<pingpong_model>>(k, build_pingpong(cfg.params), cfg);
        case model_kind::vogels:
            return std::make_unique<sim_impl<vogels_model>>(k, build_vogels(neurons, cfg.params), cfg);
        case model_kind::brunel:
            return std::make_unique<sim_impl<brunel_model>>(k, build_brunel(neurons, cfg.params), cfg);
        case model_kind::brunel_plus:
            return std::make_unique<sim_impl<brunel_plus_model>>(k, build_brunel_plus(neurons, cfg.params), cfg);
    }
    throw std::invalid_argument("make_sim: bad model kind");
}

thread_local std::string g_error;
void set_error(const char* what) { g_error = what ? what : "unknown error"; }

// capi.cpp:19-39: exception class -> status
template <class Fn>
synq_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return SYNQ_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        set_error(e.what());
        return SYNQ_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc& e) {
        set_error("out of memory (host or device)");
        return SYNQ_ERR_NO_MEMORY;
    } catch (const std::runtime_error& e) {
        set_error(e.what());
        return SYNQ_ERR_IO;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SYNQ_ERR_INTERNAL;
    }
}

}  // namespace
}  // namespace synq

using namespace synq;

struct synq_opts {
    sim_config cfg;
};
struct synq_sim {
    std::unique_ptr<sim_base> impl;
};

namespace {

bool parse_kind(const char* model, model_kind& kind) {
    try {
        if (!model) throw std::invalid_argument("model name is null");
        kind = parse_model(model);
        return true;
    } catch (const std::exception& e) {
        set_error(e.what());
        return false;
    }
}

template <class Make>
synq_status make_common(const char* model, const synq_opts* opts, synq_sim** out, Make&& make) {
    if (!out) {
        set_error("output handle is null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    model_kind kind;
    if (!parse_kind(model, kind)) return SYNQ_ERR_UNKNOWN_MODEL;
    static const sim_config defaults;
    const sim_config& cfg = opts ? opts->cfg : defaults;
    return guarded([&] {
        *out = new synq_sim{make(kind, cfg)};
        return SYNQ_OK;
    });
}

#define SYNQ_CHECK_HANDLE(h)              \
    do {                                  \
        if (!(h)) {                       \
            set_error("null handle");     \
            return SYNQ_ERR_INVALID_ARGUMENT; \
        }                                 \
    } while (0)

}  // namespace

extern "C" {

const char* synq_version(void) { return "1.0.0-b200"; }

const char* synq_status_name(synq_status s) {
    switch (s) {
        case SYNQ_OK: return "ok";
        case SYNQ_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SYNQ_ERR_UNKNOWN_MODEL: return "unknown model";
        case SYNQ_ERR_IO: return "io error";
        case SYNQ_ERR_NO_MEMORY: return "out of memory";
        case SYNQ_ERR_INTERNAL: return "internal error";
    }
    return "?";
}

const char* synq_last_error(void) { return g_error.c_str(); }

synq_opts* synq_opts_new(void) {
    try {
        return new synq_opts();
    } catch (...) {
        return nullptr;
    }
}
void synq_opts_free(synq_opts* o) { delete o; }

synq_status synq_opts_seed(synq_opts* o, uint64_t seed) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.seed = seed;
    return SYNQ_OK;
}
synq_status synq_opts_threads(synq_opts* o, uint32_t threads) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.threads = threads;
    return SYNQ_OK;
}
synq_status synq_opts_deterministic(synq_opts* o, int on) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.deterministic = on != 0;
    return SYNQ_OK;
}
synq_status synq_opts_dt(synq_opts* o, double dt_ms) {
    SYNQ_CHECK_HANDLE(o);
    if (!(dt_ms > 0)) {
        set_error("dt must be > 0");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.dt_ms = dt_ms;
    return SYNQ_OK;
}
synq_status synq_opts_delay(synq_opts* o, uint32_t steps) {
    SYNQ_CHECK_HANDLE(o);
    if (steps < 1) {
        set_error("delay must be >= 1 timestep");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.delay_steps = steps;
    return SYNQ_OK;
}
synq_status synq_opts_record(synq_opts* o, int rec) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.record_spikes = rec != 0;
    return SYNQ_OK;
}
synq_status synq_opts_defaults_file(synq_opts* o, const char* path) {
    SYNQ_CHECK_HANDLE(o);
    if (!path) {
        set_error("path is null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        merge_params_file(o->cfg.params, path);
        return SYNQ_OK;
    });
}
synq_status synq_opts_param(synq_opts* o, const char* key, double value) {
    SYNQ_CHECK_HANDLE(o);
    if (!key || !*key) {
        set_error("parameter key is null or empty");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.params[key] = value;
    return SYNQ_OK;
}

synq_status synq_sim_new(const char* model, uint32_t neurons, const synq_opts* opts, synq_sim** out) {
    return make_common(model, opts, out,
                       [&](model_kind k, const sim_config& c) { return make_sim(k, neurons, c); });
}
synq_status synq_sim_new_for_synapses(const char* model, uint64_t synapses, const synq_opts* opts,
                                      synq_sim** out) {
    return make_common(model, opts, out, [&](model_kind k, const sim_config& c) {
        return make_sim(k, solve_neurons(k, synapses, c.params), c);
    });
}
synq_status synq_sim_new_from_file(const char* model, const char* desc_path, const synq_opts* opts,
                                   synq_sim** out) {
    if (!desc_path) {
        set_error("descriptor path is null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    const std::string path = desc_path;
    return make_common(model, opts, out, [&](model_kind k, const sim_config& c) {
        network_desc d = load_desc(path);
        validate_or_throw(d);
        return make_sim_from_desc(k, d, c);
    });
}
void synq_sim_free(synq_sim* s) { delete s; }

synq_status synq_sim_step(synq_sim* s) {
    SYNQ_CHECK_HANDLE(s);
    return guarded([&] {
        s->impl->step();
        return SYNQ_OK;
    });
}
synq_status synq_sim_run(synq_sim* s, int64_t steps) {
    SYNQ_CHECK_HANDLE(s);
    if (steps < 0) {
        set_error("step count must be >= 0");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        s->impl->run(steps);
        return SYNQ_OK;
    });
}
synq_status synq_sim_flush(synq_sim* s) {
    SYNQ_CHECK_HANDLE(s);
    return guarded([&] {
        s->impl->flush();
        return SYNQ_OK;
    });
}

uint32_t synq_sim_neurons(const synq_sim* s) { return s ? s->impl->neurons() : 0; }
uint64_t synq_sim_synapses(const synq_sim* s) { return s ? s->impl->synapses() : 0; }
uint64_t synq_sim_synapse_capacity(const synq_sim* s) { return s ? s->impl->synapse_capacity() : 0; }
int64_t synq_sim_now(const synq_sim* s) { return s ? s->impl->now() : 0; }
double synq_sim_dt(const synq_sim* s) { return s ? s->impl->dt() : 0.0; }
uint32_t synq_sim_delay(const synq_sim* s) { return s ? s->impl->delay() : 0; }
uint64_t synq_sim_seed(const synq_sim* s) { return s ? s->impl->seed() : 0; }
double synq_sim_scaling(const synq_sim* s) { return s ? s->impl->scale_c() : 0.0; }

synq_status synq_sim_firing_rate(const synq_sim* s, double* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    *out = s->impl->measured_rate();
    return SYNQ_OK;
}
synq_status synq_sim_spike_count(const synq_sim* s, uint64_t* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    *out = s->impl->counters().spikes;
    return SYNQ_OK;
}

double synq_sim_seconds(const synq_sim* s, synq_phase phase) {
    if (!s) return 0.0;
    const auto& t = s->impl->timings();
    switch (phase) {
        case SYNQ_PHASE_CONSTRUCT: return t.construct;
        case SYNQ_PHASE_INIT_NEURONS: return t.init_neurons;
        case SYNQ_PHASE_INIT_SYNAPSES: return t.init_synapses;
        case SYNQ_PHASE_SIMULATE: return t.simulate;
    }
    return 0.0;
}

synq_status synq_sim_write_raster(const synq_sim* s, const char* path) {
    SYNQ_CHECK_HANDLE(s);
    if (!path) {
        set_error("raster path is null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        write_raster_file(path, s->impl->raster());
        return SYNQ_OK;
    });
}
synq_status synq_sim_write_stats(const synq_sim* s, const char* path) {
    SYNQ_CHECK_HANDLE(s);
    return guarded([&] {
        s->impl->write_stats_to(path ? path : "");
        return SYNQ_OK;
    });
}

synq_status synq_memory_estimate(const char* model, uint64_t neurons, uint64_t synapses, synq_memory* out) {
    SYNQ_CHECK_HANDLE(out);
    model_kind kind;
    if (!parse_kind(model, kind)) return SYNQ_ERR_UNKNOWN_MODEL;
    return guarded([&] {
        const auto m = memory_estimate(kind);
        out->neuron_fields = m.neuron_fields;
        out->neuron_spikes = m.neuron_spikes;
        out->neuron_bitmasks = m.neuron_bitmasks;
        out->neuron_ages = m.neuron_ages;
        out->neuron_expirations = m.neuron_expirations;
        out->synapse_adjacency = m.synapse_adjacency;
        out->synapse_fields = m.synapse_fields;
        out->neuron_total = m.neuron_total();
        out->synapse_total = m.synapse_total();
        out->total_bytes = m.total_bytes(neurons, synapses);
        return SYNQ_OK;
    });
}

// capi.cpp:334-354: the running allocation on the same per-unit slots
synq_status synq_sim_memory_actual(const synq_sim* s, synq_memory* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    const engine_memory m = s->impl->memory_actual();
    const double n = std::max(1.0, static_cast<double>(s->impl->neurons()));
    const uint64_t cap = s->impl->synapse_capacity();
    const double syn = static_cast<double>(std::max<uint64_t>(1, cap ? cap : s->impl->synapses()));
    out->neuron_fields = (m.neuron_fields + m.neuron_rng) / n;
    out->neuron_spikes = m.spike_queues / n;
    out->neuron_bitmasks = m.spike_bitmasks / n;
    out->neuron_ages = m.ages / n;
    out->neuron_expirations = m.expirations / n;
    out->synapse_adjacency = static_cast<double>(m.adjacency) / syn;
    out->synapse_fields = static_cast<double>(m.synapse_fields) / syn;
    out->neuron_total = out->neuron_fields + out->neuron_spikes + out->neuron_bitmasks +
                        out->neuron_ages + out->neuron_expirations;
    out->synapse_total = out->synapse_adjacency + out->synapse_fields;
    out->total_bytes = static_cast<double>(m.total());
    return SYNQ_OK;
}

synq_status synq_scaling_constant(const char* model, uint64_t neurons, double* out) {
    SYNQ_CHECK_HANDLE(out);
    model_kind kind;
    if (!parse_kind(model, kind)) return SYNQ_ERR_UNKNOWN_MODEL;
    return guarded([&] {
        *out = scaling_constant(kind, neurons);
        return SYNQ_OK;
    });
}

synq_status synq_solve_neurons(const char* model, uint64_t synapses, uint32_t* out) {
    SYNQ_CHECK_HANDLE(out);
    model_kind kind;
    if (!parse_kind(model, kind)) return SYNQ_ERR_UNKNOWN_MODEL;
    return guarded([&] {
        *out = solve_neurons(kind, synapses, builtin_defaults());
        return SYNQ_OK;
    });
}

// ---------------------------------------------------------- B200 extensions
synq_status synq_opts_batch_steps(synq_opts* o, uint32_t steps) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.batch_steps = steps;
    return SYNQ_OK;
}
synq_status synq_opts_persistent(synq_opts* o, int mode) {
    SYNQ_CHECK_HANDLE(o);
    if (mode < -1 || mode > 1) {
        set_error("persistent mode must be -1, 0 or 1");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.engine.persistent = mode;
    return SYNQ_OK;
}
synq_status synq_opts_tiles(synq_opts* o, uint32_t tiles) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.tiles = tiles;
    return SYNQ_OK;
}
synq_status synq_opts_shard(synq_opts* o, uint32_t rank, uint32_t world) {
    SYNQ_CHECK_HANDLE(o);
    if (world < 1 || rank >= world) {
        set_error("shard: need rank < world, world >= 1");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.engine.shard_rank = rank;
    o->cfg.engine.shard_world = world;
    return SYNQ_OK;
}
synq_status synq_sim_shard_range(const synq_sim* s, uint32_t out[4]) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    const auto r = s->impl->shard_range();
    std::copy(r.begin(), r.end(), out);
    return SYNQ_OK;
}
uint64_t synq_sim_shard_capacity(const synq_sim* s) { return s ? s->impl->shard_capacity() : 0; }
synq_status synq_sim_shard_export(synq_sim* s, void* dst, uint64_t capacity, int device, uint64_t* words) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(dst);
    SYNQ_CHECK_HANDLE(words);
    return guarded([&] {
        *words = s->impl->shard_export(dst, capacity, device != 0);
        return SYNQ_OK;
    });
}
synq_status synq_sim_shard_import(synq_sim* s, const void* src, uint64_t words, uint32_t from_rank, int device) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(src);
    return guarded([&] {
        s->impl->shard_import(src, words, from_rank, device != 0);
        return SYNQ_OK;
    });
}
synq_status synq_nccl_unique_id(void* out) {
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        detail::nccl_unique_id(static_cast<char*>(out));
        return SYNQ_OK;
    });
}
synq_status synq_opts_shard_nccl(synq_opts* o, uint32_t rank, uint32_t world, const void* id) {
    SYNQ_CHECK_HANDLE(o);
    SYNQ_CHECK_HANDLE(id);
    if (world < 1 || rank >= world) {
        set_error("shard: need rank < world, world >= 1");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.engine.shard_rank = rank;
    o->cfg.engine.shard_world = world;
    o->cfg.engine.shard_nccl = true;
    std::memcpy(o->cfg.engine.nccl_id.data(), id, o->cfg.engine.nccl_id.size());
    return SYNQ_OK;
}
static_assert(SYNQ_PEER_HANDLE_BYTES == synq::kPeerHandleBytes, "peer handle size");
static_assert(sizeof(synq_peer_endpoint) == sizeof(synq::peer_endpoint), "peer endpoint layout");
synq_status synq_opts_shard_peer(synq_opts* o, int enable) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.shard_peer = enable != 0;
    return SYNQ_OK;
}
synq_status synq_sim_peer_endpoint(const synq_sim* s, synq_peer_endpoint* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        const synq::peer_endpoint e = s->impl->peer_endpoint();
        *out = synq_peer_endpoint{e.queue, e.finfo, e.publishers, 0};
        return SYNQ_OK;
    });
}
synq_status synq_sim_peer_connect(synq_sim* s, const synq_peer_endpoint* eps, uint32_t world) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(eps);
    return guarded([&] {
        if (world != s->impl->shard_world()) throw std::invalid_argument("peer_connect: world differs from the shard's");
        std::vector<synq::peer_endpoint> v(world);
        for (uint32_t q = 0; q < world; ++q)
            v[q] = {static_cast<uint32_t*>(eps[q].queue), static_cast<unsigned long long*>(eps[q].finfo),
                    eps[q].publishers, 0};
        s->impl->peer_connect(v);
        return SYNQ_OK;
    });
}
synq_status synq_sim_peer_ipc_handle(const synq_sim* s, void* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        s->impl->peer_ipc_handle(out);
        return SYNQ_OK;
    });
}
synq_status synq_sim_peer_connect_ipc(synq_sim* s, const void* all, uint32_t world) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(all);
    return guarded([&] {
        if (world != s->impl->shard_world()) throw std::invalid_argument("peer_connect_ipc: world differs from the shard's");
        s->impl->peer_connect_ipc(all);
        return SYNQ_OK;
    });
}
uint64_t synq_sim_shard_bits_words(const synq_sim* s) { return s ? s->impl->shard_bits_words() : 0; }
synq_status synq_sim_shard_export_bits(synq_sim* s, void* dst) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(dst);
    return guarded([&] {
        s->impl->shard_export_bits(dst);
        return SYNQ_OK;
    });
}
synq_status synq_sim_shard_import_bits(synq_sim* s, const void* all) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(all);
    return guarded([&] {
        s->impl->shard_import_bits(all);
        return SYNQ_OK;
    });
}
synq_status synq_opts_pipeline(synq_opts* o, int mode, uint32_t lead) {
    SYNQ_CHECK_HANDLE(o);
    if (mode < -1 || mode > 1) {
        set_error("pipeline mode must be -1, 0 or 1");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    o->cfg.engine.pipeline = mode;
    o->cfg.engine.lead = lead;
    return SYNQ_OK;
}
synq_status synq_opts_profile(synq_opts* o, int on) {
    SYNQ_CHECK_HANDLE(o);
    o->cfg.engine.profile = on != 0;
    return SYNQ_OK;
}
synq_status synq_sim_phase_cycles(const synq_sim* s, double out[15], uint32_t* tiles) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        const auto v = s->impl->phase_cycles();
        for (int k = 0; k < 15; ++k) out[k] = v[k];
        if (tiles) *tiles = s->impl->tiles();
        return SYNQ_OK;
    });
}
int synq_sim_engine(const synq_sim* s) {
    if (!s || !s->impl->persistent()) return 0;
    if (s->impl->solo()) return 4;
    if (s->impl->cluster()) return 5;
    return s->impl->bitmap_delivery() ? 3 : (s->impl->pipelined() ? 2 : 1);
}
int synq_sim_exact(const synq_sim* s) { return s && s->impl->exact() ? 1 : 0; }

synq_status synq_sim_counters(const synq_sim* s, uint64_t out[6]) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    const auto& c = s->impl->counters();
    out[0] = c.steps;
    out[1] = c.spikes;
    out[2] = c.deliveries;
    out[3] = c.synapse_updates;
    out[4] = c.expiry_batches;
    out[5] = c.frames_consumed;
    return SYNQ_OK;
}
synq_status synq_sim_raster_size(const synq_sim* s, uint64_t* out) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    *out = s->impl->raster_size();
    return SYNQ_OK;
}
synq_status synq_sim_raster_copy(const synq_sim* s, int64_t* steps, uint32_t* ids, uint64_t capacity) {
    SYNQ_CHECK_HANDLE(s);
    const uint64_t n = s->impl->raster_size();
    if (capacity < n || (n && (!steps || !ids))) {
        set_error("raster buffers too small or null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    s->impl->raster_copy(steps, ids);
    return SYNQ_OK;
}
synq_status synq_sim_step_spikes(const synq_sim* s, uint32_t* out, uint64_t capacity) {
    SYNQ_CHECK_HANDLE(s);
    const auto& v = s->impl->step_spikes();
    if (capacity < v.size() || (!v.empty() && !out)) {
        set_error("buffer too small or null");
        return SYNQ_ERR_INVALID_ARGUMENT;
    }
    std::copy(v.begin(), v.end(), out);
    return SYNQ_OK;
}
synq_status synq_sim_neuron_field(synq_sim* s, uint32_t field, void* out, uint64_t bytes) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        s->impl->neuron_field_bytes(field, out, bytes);
        return SYNQ_OK;
    });
}
synq_status synq_sim_synapse_field(synq_sim* s, uint32_t field, void* out, uint64_t bytes) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        s->impl->synapse_field_bytes(field, out, bytes);
        return SYNQ_OK;
    });
}
synq_status synq_sim_ages(synq_sim* s, uint32_t* out, uint64_t capacity) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        s->impl->ages_copy(out, capacity);
        return SYNQ_OK;
    });
}
synq_status synq_sim_graph_shape(const synq_sim* s, uint32_t* pitch, uint32_t* deg_max) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(pitch);
    SYNQ_CHECK_HANDLE(deg_max);
    return guarded([&] {
        const auto& g = s->impl->graph();
        *pitch = g.row_pitch();
        *deg_max = g.deg_max();
        return SYNQ_OK;
    });
}
synq_status synq_sim_graph_cells(const synq_sim* s, uint32_t* out, uint64_t capacity) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    return guarded([&] {
        const auto& g = s->impl->graph();
        const uint64_t n = static_cast<uint64_t>(g.neuron_count()) * g.row_pitch();
        if (capacity < n) throw std::invalid_argument("buffer too small for adjacency");
        std::memcpy(out, g.cells(), n * sizeof(uint32_t));
        return SYNQ_OK;
    });
}
uint64_t synq_sim_construction_fixups(const synq_sim* s) { return s ? s->impl->fixups() : 0; }

synq_status synq_sim_device_time(const synq_sim* s, double out[2]) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    s->impl->device_time(out);
    return SYNQ_OK;
}
uint64_t synq_sim_kernel_launches(const synq_sim* s) { return s ? s->impl->launches() : 0; }
synq_status synq_sim_set_record(synq_sim* s, int on) {
    SYNQ_CHECK_HANDLE(s);
    return guarded([&] {
        s->impl->set_record(on != 0);
        return SYNQ_OK;
    });
}
synq_status synq_sim_transfer_bytes(const synq_sim* s, uint64_t out[2]) {
    SYNQ_CHECK_HANDLE(s);
    SYNQ_CHECK_HANDLE(out);
    s->impl->transfers(out);
    return SYNQ_OK;
}

}  // extern "C"
