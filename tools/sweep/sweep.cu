// Synthetic sweep (BASELINE.json config 4, SURVEY.md 8 "SW"): connectivity
// p x firing rate at a fixed synapse budget S.  One population of
// N = sqrt(S / p) neurons, each a Poisson source at rate r that also
// receives (ACC += w per arrival), connected to itself with probability p.
// The model is user code compiled against the public C++ API
// (synq::network<Model>, include/synq/engine.hpp); it specialises
// population_delivery, so it runs on the persistent pipelined engine
// (bitmap delivery when dense, ELL rows when sparse) or, when a CTA cannot
// hold its neurons, on the per-step kernel graph.
//
//   build/sweep [S] [steps]     -> one line per (p, rate): engine, events/s,
//                                   ms per bio-second (device-timed)
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "synq/engine.hpp"

using namespace synq;

struct sweep_model {
    using neuron_fields = fields<float>;  // ACC
    static constexpr bool uses_rng = true;
    enum : size_t { ACC = 0 };
    float p_spike = 0.0f;  // rate * dt
    float w = 0.01f;

    template <class It>
    SYNQ_HD void init(It it) const {
        it.template get<ACC>() = 0.0f;
    }
    template <class It>
    SYNQ_HD bool update(It it, float) const {
        it.template get<ACC>() = 0.0f;  // consume the input
        return it.rng().uniform01() <= p_spike;
    }
    template <class From, class To>
    SYNQ_HD void receive(From, To to) const {
        to.template add<ACC>(w);
    }
};

namespace synq {
template <>
struct population_delivery<sweep_model> {
    static constexpr bool available = true;
    static constexpr size_t acc_field = sweep_model::ACC;
    static int classes(const sweep_model& m, uint32_t neurons, uint32_t* bound, float* delta) {
        bound[0] = neurons;
        delta[0] = m.w;
        return 1;
    }
};
}  // namespace synq

int main(int argc, char** argv) {
    const double S = argc > 1 ? std::atof(argv[1]) : 1e9;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 2000;
    const double dt = 0.1;  // ms
    std::printf("# S=%.3g synapses, %d steps of dt=%.1f ms after 500 warm-up steps\n", S, steps, dt);
    std::printf("%-7s %-6s %9s %12s %-18s %12s %12s %10s\n", "p", "rate", "neurons", "synapses", "engine",
                "events/s", "ms/bio-s", "setup_s");
    for (double p : {0.1, 0.01, 0.001})
        for (double rate : {1.0, 10.0, 100.0}) {
            const uint32_t n = static_cast<uint32_t>(std::llround(std::sqrt(S / p)));
            network_desc desc;
            desc.populations = {population_spec{n}};
            desc.connections = {connectivity_spec{0, 0, p}};
            desc.dt = dt;
            desc.delay = 15;
            sweep_model m;
            m.p_spike = static_cast<float>(rate * dt * 1e-3);
            engine_options opt;
            opt.seed = 1;
            opt.deterministic = true;
            const auto t0 = std::chrono::steady_clock::now();
            network<sweep_model> net(desc, m, opt);
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
            std::printf("%-7g %-6g %9u %12llu %-18s %12.3e %12.2f %10.1f\n", p, rate, n,
                        static_cast<unsigned long long>(net.edge_count()), eng, ev / secs,
                        secs / steps * 10000.0 * 1e3, setup);
            std::fflush(stdout);
        }
    return 0;
}
