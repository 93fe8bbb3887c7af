// C++ model-API tests on the B200: user-defined models compiled into the
// device engine through include/synq/engine.hpp, exercising the reference's
// own engine properties (restated from proj/tests/test_engine.cpp and
// test_lazy.cpp; acceptance c5, c6, c10).  Prints one line per case and
// exits non-zero on any failure.  Run by tests/test_gpu_cpp.py.
#include <cstdio>
#include <cstring>
#include <functional>
#include <span>
#include <string>
#include <vector>

#include <chrono>

#include "synq/detail/device_graph.hpp"
#include "synq/engine.hpp"
#include "synq/models/benchmarks.hpp"

using namespace synq;

static int g_failures = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        if (!(cond)) {                                                            \
            std::printf("  CHECK FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++g_failures;                                                         \
        }                                                                         \
    } while (0)

// Spikes on a per-neuron schedule held in device memory (bit s = spike at
// step s); counts deliveries and records the step of the latest one
// (probes.hpp:19-44, with the schedule as a device pointer).
struct probe_model {
    using neuron_fields = fields<uint32_t, uint32_t, uint32_t>;
    enum : size_t { STEP = 0, RECV_COUNT = 1, LAST_RECV = 2 };
    const uint64_t* schedule = nullptr;

    template <class It>
    SYNQ_HD void init(It it) const {
        it.template get<STEP>() = 0;
        it.template get<RECV_COUNT>() = 0;
        it.template get<LAST_RECV>() = 0;
    }
    template <class It>
    SYNQ_HD bool update(It it, float) const {
        const uint32_t s = it.template get<STEP>()++;
        if (s >= 64) return false;
        return (schedule[it.id()] >> s) & 1ull;
    }
    template <class From, class To>
    SYNQ_HD void receive(From, To to) const {
        to.template add<RECV_COUNT>(1u);
        to.template put<LAST_RECV>(to.template get<STEP>());
    }
};

// never spikes; its synapse counts applied steps (test_lazy.cpp:90-111)
struct silent_model {
    using neuron_fields = fields<uint8_t>;
    using synapse_fields = fields<float, float, float>;
    template <class It>
    SYNQ_HD void init(It it) const {
        it.template get<0>() = 0;
    }
    template <class It>
    SYNQ_HD bool update(It, float) const {
        return false;
    }
    template <class F, class T, class S>
    SYNQ_HD void receive(F, T, S) const {}
    template <class S>
    SYNQ_HD void init_synapse(S syn) const {
        syn.template get<0>() = 0.0f;
    }
    template <class S>
    SYNQ_HD void update_synapse(S& syn, bool, bool, float) const {
        syn.template get<0>() += 1.0f;
    }
};

struct meta_rng {  // the reference tests' generator for random networks
    xorshift r;
    explicit meta_rng(uint64_t s) : r(s) {}
    uint32_t operator()() { return r(); }
};

network_desc random_net(meta_rng& meta, uint32_t delay) {
    network_desc d;
    const size_t pops = 1 + meta() % 3;
    for (size_t i = 0; i < pops; ++i) d.populations.push_back({10 + meta() % 60});
    for (uint32_t s = 0; s < pops; ++s)
        for (uint32_t t = 0; t < pops; ++t) d.connections.push_back({s, t, (meta() % 100) / 300.0});
    d.dt = 1.0;
    d.delay = delay;
    return d;
}

struct frame_log {
    std::vector<std::vector<uint32_t>> frames;
    void operator()(int64_t, std::span<const uint32_t> f) { frames.emplace_back(f.begin(), f.end()); }
    bool spiked(int64_t t, uint32_t id) const {
        if (t < 0 || t >= static_cast<int64_t>(frames.size())) return false;
        const auto& f = frames[t];
        return std::binary_search(f.begin(), f.end(), id);
    }
};

// every delivery lands exactly `delay` steps after emission
// (test_engine.cpp:66-109, acceptance c6); both delivery modes
void test_delay_property() {
    std::printf("delay_property\n");
    meta_rng meta(31337);
    int checked = 0;
    for (int trial = 0; trial < 60; ++trial) {
        const uint32_t delay = 1 + meta() % 16;
        const network_desc d = random_net(meta, delay);
        const uint32_t n = d.neuron_count();
        std::vector<uint64_t> sched(n, 0);
        for (uint32_t i = 0; i < n; ++i)
            if (meta() % 4) sched[i] = 1ull << (meta() % 40);
        dev_array<uint64_t> dsched(n);
        dsched.upload(sched.data(), n);
        cudaDeviceSynchronize();
        probe_model m;
        m.schedule = dsched.get();
        engine_options opt;
        opt.seed = meta();
        opt.deterministic = trial % 2 == 0;
        opt.debug_checks = true;
        network<probe_model> net(d, m, opt);
        net.run(40 + delay + 2);
        std::vector<uint32_t> want_count(n, 0), want_last(n, 0);
        for (uint32_t src = 0; src < n; ++src) {
            if (!sched[src]) continue;
            const uint32_t e = static_cast<uint32_t>(__builtin_ctzll(sched[src]));
            for (uint32_t tgt : net.graph().row(src)) {
                want_count[tgt] += 1;
                want_last[tgt] = std::max(want_last[tgt], e + delay);
            }
        }
        auto cnt = net.neuron_field<probe_model::RECV_COUNT>();
        auto last = net.neuron_field<probe_model::LAST_RECV>();
        for (uint32_t i = 0; i < n; ++i) {
            CHECK(cnt[i] == want_count[i]);
            if (want_count[i]) {
                CHECK(last[i] == want_last[i]);
                ++checked;
            }
        }
    }
    CHECK(checked > 500);
}

// pingpong vs a naive flag replay (probes.hpp:48-76, acceptance c10)
void test_pingpong_flag_reference() {
    std::printf("pingpong_flag_reference\n");
    const auto b = build_pingpong(builtin_defaults());
    for (int det = 0; det < 2; ++det) {
        engine_options opt;
        opt.seed = 5;
        opt.deterministic = det != 0;
        network<pingpong_model> net(b.desc, b.model, opt);
        frame_log log;
        net.set_spike_tap(std::ref(log));
        net.run(1000);
        const auto& adj = net.graph();
        const uint32_t n = adj.neuron_count();
        std::vector<uint8_t> flag(n, 0);
        for (uint32_t i = 0; i < b.model.first_pop && i < n; ++i) flag[i] = 1;
        std::vector<std::vector<uint32_t>> want;
        for (int64_t t = 0; t < 1000; ++t) {
            std::vector<uint32_t> now;
            for (uint32_t i = 0; i < n; ++i)
                if (flag[i]) {
                    now.push_back(i);
                    flag[i] = 0;
                }
            want.push_back(now);
            const int64_t due = t - net.delay() + 1;
            if (due >= 0)
                for (uint32_t src : want[due])
                    for (uint32_t tgt : adj.row(src)) flag[tgt] = 1;
        }
        CHECK(log.frames == want);
        bool any = false;
        for (size_t t = 0; t < log.frames.size(); ++t)
            for (uint32_t id : log.frames[t]) {
                any = true;
                CHECK((id < 100) == (t % 2 == 0));
            }
        CHECK(any);
    }
}

// lazy plasticity == eager per-step replay, bit for bit (test_lazy.cpp:33-71,
// acceptance c5), for the default, tight and an odd history size
void check_lazy_equals_eager(uint32_t neurons, int64_t steps, uint32_t history, uint64_t seed) {
    std::printf("lazy_equals_eager N=%u steps=%lld history=%u\n", neurons, (long long)steps, history);
    const auto b = build_brunel_plus(neurons, builtin_defaults());
    engine_options opt;
    opt.seed = seed;
    opt.deterministic = true;
    opt.history_frames = history;
    network<brunel_plus_model> net(b.desc, b.model, opt);
    std::vector<std::vector<float>> init(3);
    {
        auto w = net.synapse_field<0>(), p = net.synapse_field<1>(), q = net.synapse_field<2>();
        init[0].assign(w.begin(), w.end());
        init[1].assign(p.begin(), p.end());
        init[2].assign(q.begin(), q.end());
    }
    frame_log log;
    net.set_spike_tap(std::ref(log));
    net.run(steps);
    net.flush();
    const auto& adj = net.graph();
    auto result = init;
    const float dt = net.dt();
    for (uint32_t src = 0; src < adj.neuron_count(); ++src) {
        const auto row = adj.row(src);
        const uint64_t base = uint64_t(src) * adj.deg_max();
        for (size_t k = 0; k < row.size(); ++k) {
            synapse_state<brunel_plus_model::synapse_fields> st;
            st.src_ = src;
            st.dst_ = row[k];
            st.get<0>() = result[0][base + k];
            st.get<1>() = result[1][base + k];
            st.get<2>() = result[2][base + k];
            for (int64_t u = 0; u < steps; ++u)
                b.model.update_synapse(st, log.spiked(u - net.delay(), src), log.spiked(u, row[k]), dt);
            result[0][base + k] = st.get<0>();
            result[1][base + k] = st.get<1>();
            result[2][base + k] = st.get<2>();
        }
    }
    for (int f = 0; f < 3; ++f) {
        std::span<float> got = f == 0 ? net.synapse_field<0>() : (f == 1 ? net.synapse_field<1>() : net.synapse_field<2>());
        CHECK(got.size() == result[f].size());
        CHECK(std::memcmp(got.data(), result[f].data(), got.size_bytes()) == 0);
    }
    CHECK(net.counters().synapse_updates == net.edge_count() * static_cast<uint64_t>(steps));
}

// a silent neuron is caught up in whole batches when it expires
// (test_lazy.cpp:136-159)
void test_silent_expiry() {
    std::printf("silent_expiry\n");
    network_desc d;
    d.populations = {{1}};
    d.connections = {{0, 0, 1.0}};
    d.delay = 1;
    engine_options opt;
    opt.deterministic = true;
    opt.history_frames = 10;
    network<silent_model> net(d, {}, opt);
    int64_t first_batch = -1;
    for (int64_t t = 0; t < 30; ++t) {
        net.step();
        if (first_batch < 0 && net.counters().expiry_batches > 0) first_batch = net.now();
    }
    CHECK(first_batch > 1);
    CHECK(first_batch <= 10);
    CHECK(net.counters().expiry_batches > 1);
    net.flush();
    CHECK(net.synapse_field<0>()[0] == 30.0f);
}

// ages never outrun the retained history (test_lazy.cpp:115-134)
void test_ages_bound() {
    std::printf("ages_bound\n");
    const auto b = build_brunel_plus(100, builtin_defaults());
    engine_options opt;
    opt.seed = 13;
    opt.deterministic = true;
    network<brunel_plus_model> net(b.desc, b.model, opt);
    const int64_t history = net.history_frames(), delay = net.delay();
    for (int64_t t = 0; t < 150; ++t) {
        net.step();
        for (uint32_t age : net.ages()) {
            CHECK(static_cast<int64_t>(age) >= net.now() - history + delay);
            CHECK(static_cast<int64_t>(age) <= net.now());
        }
    }
}

// re-running init restores the initial state exactly (test_engine.cpp:208-221)
void test_reinit() {
    std::printf("reinit\n");
    const auto b = build_vogels(200, builtin_defaults());
    engine_options opt;
    opt.seed = 31;
    opt.deterministic = true;
    network<vogels_model> net(b.desc, b.model, opt);
    auto v = net.neuron_field<0>();
    std::vector<float> v0(v.begin(), v.end());
    net.run(100);
    net.init();
    auto v1 = net.neuron_field<0>();
    CHECK(std::memcmp(v0.data(), v1.data(), v0.size() * sizeof(float)) == 0);
    CHECK(net.now() == 0);
    CHECK(net.persistent());
}

// debug_checks (engine.hpp:374-378, 440-446): the device-side frame checks
// (sorted / unique, queue size == bitmask popcount, pieces inside their
// ranges) run every step on both engines and pass on real runs; frames and
// state are unchanged by them
template <class M>
void check_debug_run(model_build<M> b, int64_t steps, const char* name) {
    engine_options opt;
    opt.seed = 3;
    opt.deterministic = true;
    opt.debug_checks = true;
    network<M> net(b.desc, b.model, opt);
    frame_log log;
    net.set_spike_tap(std::ref(log));
    bool ok = true;
    try {
        net.run(steps);
    } catch (const std::exception& e) {
        std::printf("  %s: %s\n", name, e.what());
        ok = false;
    }
    CHECK(ok);
    opt.debug_checks = false;
    network<M> ref(b.desc, b.model, opt);
    frame_log rlog;
    ref.set_spike_tap(std::ref(rlog));
    ref.run(steps);
    CHECK(log.frames == rlog.frames);
    size_t spikes = 0;
    for (const auto& f : log.frames) spikes += f.size();
    CHECK(spikes > 0);
    std::printf("  %s: %zu spikes, engine %s\n", name, spikes, net.persistent() ? "persistent" : "graph");
}

void test_debug_checks() {
    std::printf("debug_checks\n");
    check_debug_run(build_vogels(1000, builtin_defaults()), 600, "vogels");
    check_debug_run(build_brunel_plus(400, builtin_defaults()), 300, "brunel+");
    check_debug_run(build_pingpong(builtin_defaults()), 200, "pingpong");
}

// writes through a host span reach the device before the next step
void test_span_writeback() {
    std::printf("span_writeback\n");
    const auto b = build_pingpong(builtin_defaults());
    engine_options opt;
    opt.deterministic = true;
    network<pingpong_model> net(b.desc, b.model, opt);
    frame_log log;
    net.set_spike_tap(std::ref(log));
    auto flags = net.neuron_field<0>();
    for (auto& f : flags) f = 0;
    flags[150] = 1;  // only neuron 150 fires next
    net.step();
    CHECK(log.frames.size() == 1);
    CHECK(log.frames[0].size() == 1 && log.frames[0][0] == 150);
}

// parallel accumulation of many floats into one target ~ sequential
// (test_engine.cpp:153-172): fast (atomic) and ordered modes
struct accum_model {
    using neuron_fields = fields<float, uint32_t>;
    template <class It>
    SYNQ_HD void init(It it) const {
        it.template get<0>() = 0.0f;
        it.template get<1>() = 0;
    }
    template <class It>
    SYNQ_HD bool update(It it, float) const {
        return it.template get<1>()++ == 0 && it.id() < 200;
    }
    template <class From, class To>
    SYNQ_HD void receive(From from, To to) const {
        to.template add<0>(0.001f * (1 + from.id() % 7));
    }
};

void test_accumulation_modes() {
    std::printf("accumulation_modes\n");
    network_desc d;
    d.populations = {{200}, {4}};
    d.connections = {{0, 1, 1.0}};
    d.delay = 1;
    engine_options det;
    det.deterministic = true;
    network<accum_model> a(d, {}, det);
    a.run(3);
    engine_options fast;
    network<accum_model> b(d, {}, fast);
    b.run(3);
    auto va = a.neuron_field<0>();
    auto vb = b.neuron_field<0>();
    float seq = 0.0f;  // the reference's ascending-source sum
    for (uint32_t s = 0; s < 200; ++s) seq += 0.001f * (1 + s % 7);
    for (uint32_t i = 200; i < 204; ++i) {
        CHECK(va[i] == seq);  // ordered mode is bit-exact
        CHECK(std::abs(vb[i] - va[i]) <= 1e-5f * std::abs(va[i]));
    }
}

// The device degree plan (csrc/plan.cu) against the host restatement of
// plan_jobs (adjacency.cpp:29-71): every job, degree and offset identical.
static network_desc make_desc(std::vector<uint32_t> pops, std::vector<connectivity_spec> conns) {
    network_desc d;
    for (uint32_t n : pops) d.populations.push_back(population_spec{n});
    d.connections = std::move(conns);
    d.dt = 0.1;
    d.delay = 2;
    return d;
}

static void check_plan(const network_desc& d, uint64_t seed, const char* name) {
    using clk = std::chrono::steady_clock;
    cudaFree(nullptr);  // context creation is not part of the plan
    const auto t0 = clk::now();
    const construction_plan a = plan_jobs(d, seed, 32);
    const auto t1 = clk::now();
    const construction_plan b = plan_jobs_device(d, seed, 32, nullptr);
    const auto t2 = clk::now();
    CHECK(a.jobs.size() == b.jobs.size());
    size_t bad = 0;
    for (size_t q = 0; q < std::min(a.jobs.size(), b.jobs.size()); ++q) {
        const auto &x = a.jobs[q], &y = b.jobs[q];
        bad += x.n != y.n || x.a != y.a || x.b != y.b || x.o != y.o;
    }
    CHECK(bad == 0);
    CHECK(a.out_degree == b.out_degree);
    CHECK(a.deg_max == b.deg_max);
    CHECK(a.row_pitch == b.row_pitch);
    CHECK(a.total_edges == b.total_edges);
    std::printf("  plan %-10s seed %llu: %zu jobs, %llu edges, host %.3f s, device %.3f s, mismatched jobs %zu\n", name,
                static_cast<unsigned long long>(seed), a.jobs.size(), static_cast<unsigned long long>(a.total_edges),
                std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(), bad);
}

void test_plan() {
    // Vogels 4000 and a small Brunel shape
    check_plan(make_desc({3200, 800}, {{0, 0, 0.02}, {0, 1, 0.02}, {1, 0, 0.02}, {1, 1, 0.02}}), 1, "vogels4k");
    check_plan(make_desc({5657, 1414, 7071}, {{0, 0, 0.1}, {0, 1, 0.1}, {1, 0, 0.1}, {1, 1, 0.1}, {2, 0, 0.1}, {2, 1, 0.1}}),
               7, "brunel1e7");
    // edge cases: p = 0 and p = 1 (no draws), sparse and dense, a one-neuron
    // population, mixed p across connections
    check_plan(make_desc({1, 300000, 2000, 37},
                         {{0, 1, 0.001}, {1, 2, 0.0}, {2, 3, 1.0}, {1, 0, 0.5}, {3, 1, 0.0001}, {2, 2, 0.9}, {3, 3, 0.3}}),
               12345, "edge");
    for (uint64_t seed : {2ull, 3ull}) check_plan(make_desc({20000, 30000}, {{0, 1, 0.05}, {1, 0, 0.2}}), seed, "two-pop");
}

void test_plan_large() {
    // Brunel 1e9 (282,842 jobs, 999,981,220 edges)
    check_plan(make_desc({56568, 14142, 70711}, {{0, 0, 0.1}, {0, 1, 0.1}, {1, 0, 0.1}, {1, 1, 0.1}, {2, 0, 0.1}, {2, 1, 0.1}}),
               1, "brunel1e9");
}

int main(int argc, char** argv) {
    const std::string only = argc > 1 ? argv[1] : "";
    auto run = [&](const char* name, void (*fn)()) {
        if (only.empty() || only == name) fn();
    };
    run("delay_property", test_delay_property);
    run("pingpong_flag_reference", test_pingpong_flag_reference);
    run("silent_expiry", test_silent_expiry);
    run("ages_bound", test_ages_bound);
    run("reinit", test_reinit);
    run("span_writeback", test_span_writeback);
    run("accumulation_modes", test_accumulation_modes);
    run("debug_checks", test_debug_checks);
    run("plan", test_plan);
    if (only == "plan_large") test_plan_large();
    if (only.empty() || only == "lazy") {
        check_lazy_equals_eager(120, 400, 0, 2024);
        check_lazy_equals_eager(80, 200, 1, 7);
        check_lazy_equals_eager(90, 333, 23, 99);
    }
    std::printf("%s: %d failure(s)\n", g_failures ? "FAIL" : "PASS", g_failures);
    return g_failures ? 1 : 0;
}
