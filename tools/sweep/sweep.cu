// Synthetic sweep (BASELINE.json config 4, SURVEY.md 8 "SW"): connectivity
// p x firing rate at a fixed synapse budget S.  The model
// (include/synq/models/sweep.hpp) is user code against the public C++ API
// (synq::network<Model>, include/synq/engine.hpp); it specialises
// population_delivery, so it runs on the persistent pipelined engine (bitmap
// delivery when dense, ELL rows when sparse).
//
//   build/sweep [S] [steps]          one line per (p, rate): engine, events/s,
//                                     ms per bio-second (device-timed)
//   build/sweep dump S P RATE SEED STEPS OUT
//                                     one deterministic run written like
//                                     oracle/_ref/synq_golden sweep (OUT.frames:
//                                     per step u32 n + ids; OUT.state; OUT.counters)
//   build/sweep point S P RATE STEPS  one timed point (same columns)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "synq/engine.hpp"
#include "synq/models/sweep.hpp"

using namespace synq;

namespace {

network_desc sweep_desc(double S, double p, double dt) {
    const uint32_t n = static_cast<uint32_t>(std::llround(std::sqrt(S / p)));
    network_desc desc;
    desc.populations = {population_spec{n}};
    desc.connections = {connectivity_spec{0, 0, p}};
    desc.dt = dt;
    desc.delay = 15;
    return desc;
}

sweep_model sweep_params(double rate, double dt) {
    sweep_model m;
    m.p_spike = static_cast<float>(rate * dt * 1e-3);
    return m;
}

void point(double S, double p, double rate, int steps) {
    const double dt = 0.1;  // ms
    engine_options opt;
    opt.seed = 1;
    opt.deterministic = true;
    const auto t0 = std::chrono::steady_clock::now();
    network<sweep_model> net(sweep_desc(S, p, dt), sweep_params(rate, dt), opt);
    const double setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    net.run(500);
    const double k0 = net.device_seconds();
    const uint64_t e0 = net.counters().deliveries;
    net.run(steps);
    const double secs = net.device_seconds() - k0;
    const uint64_t ev = net.counters().deliveries - e0;
    const char* eng = net.bitmap_delivery() ? "pipelined-bitmap"
                                            : (net.pipelined() ? "pipelined-ell"
                                                               : (net.persistent() ? "persistent" : "graph"));
    std::printf("%-7g %-6g %9u %12llu %-18s %12.3e %12.2f %10.1f\n", p, rate, net.neuron_count(),
                static_cast<unsigned long long>(net.edge_count()), eng, ev / secs, secs / steps * 10000.0 * 1e3,
                setup);
    std::fflush(stdout);
}

int dump(double S, double p, double rate, uint64_t seed, int64_t steps, const std::string& out) {
    const double dt = 0.1;
    engine_options opt;
    opt.seed = seed;
    opt.deterministic = true;
    network<sweep_model> net(sweep_desc(S, p, dt), sweep_params(rate, dt), opt);
    std::vector<uint32_t> buf;
    net.set_spike_tap([&](int64_t, std::span<const uint32_t> f) {
        buf.push_back(static_cast<uint32_t>(f.size()));
        buf.insert(buf.end(), f.begin(), f.end());
    });
    net.run(steps);
    std::ofstream(out + ".frames", std::ios::binary).write(reinterpret_cast<const char*>(buf.data()), buf.size() * 4);
    auto acc = net.neuron_field<0>();
    std::ofstream(out + ".state", std::ios::binary).write(reinterpret_cast<const char*>(acc.data()), acc.size_bytes());
    const auto& c = net.counters();
    std::ofstream o(out + ".counters");
    o << "steps=" << c.steps << "\nspikes=" << c.spikes << "\ndeliveries=" << c.deliveries
      << "\nframes_consumed=" << c.frames_consumed << "\nedges=" << net.edge_count()
      << "\nneurons=" << net.neuron_count() << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "dump") == 0) {
        if (argc < 8) return 2;
        return dump(std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4]), std::strtoull(argv[5], nullptr, 0),
                    std::atoll(argv[6]), argv[7]);
    }
    if (argc > 1 && std::strcmp(argv[1], "point") == 0) {
        if (argc < 6) return 2;
        point(std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4]), std::atoi(argv[5]));
        return 0;
    }
    const double S = argc > 1 ? std::atof(argv[1]) : 1e9;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 2000;
    std::printf("# S=%.3g synapses, %d steps of dt=0.1 ms after 500 warm-up steps\n", S, steps);
    std::printf("%-7s %-6s %9s %12s %-18s %12s %12s %10s\n", "p", "rate", "neurons", "synapses", "engine",
                "events/s", "ms/bio-s", "setup_s");
    for (double p : {0.1, 0.01, 0.001})
        for (double rate : {1.0, 10.0, 100.0}) point(S, p, rate, steps);
    return 0;
}
