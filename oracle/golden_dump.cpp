// Golden-vector dumper — TEST INFRASTRUCTURE, built by oracle/Makefile into
// oracle/_ref/synq_golden and linked against the UNMODIFIED reference sources
// in /root/reference/proj (it only calls the reference's public C++ API).
//
// It exists so the parity tests can compare the CUDA path with the reference
// itself on identical seeds: raw RNG streams, construction plans, adjacency
// dumps, per-step spike frames and end-of-run state of the benchmark models.
//
//   synq_golden rng SEED COUNT                 -> u32[COUNT]           (stdout, binary)
//   synq_golden uniform SEED COUNT             -> f64[COUNT]
//   synq_golden derive MASTER IDX              -> u64 (text)
//   synq_golden binomial SEED M P COUNT        -> u32[COUNT]
//   synq_golden sorted N A B SEED              -> u32[N]
//   synq_golden fig2                           -> f64 trace rows (8 x 5) + u32[6]
//   synq_golden plan MODEL NEURONS SEED OUT    -> plan file (see write_plan)
//   synq_golden adj MODEL NEURONS SEED OUT     -> adjacency_list::dump format
//   synq_golden run MODEL NEURONS SEED STEPS OUT [HISTORY] [DT DELAY]
//        deterministic run; OUT.frames (per step: u32 n, u32 ids[n]),
//        OUT.state (f32 fields), OUT.syn (brunel+ synapse fields after flush),
//        OUT.counters (text)
//   synq_golden run_desc MODEL DESC SEED STEPS OUT
//   synq_golden sweep S P RATE SEED STEPS OUT
//        the synthetic sweep model (include/synq/models/sweep.hpp, compiled
//        here against the reference headers), N = round(sqrt(S/p)), one
//        population self-connected with probability p, dt 0.1 ms, delay 15;
//        deterministic run dumped like `run` (OUT.state = ACC)
//   synq_golden sweep_time S P RATE SEED WARM STEPS THREADS DET
//        CPU baseline of one sweep point: prints events / sim_s / construct_s
//   synq_golden big MODEL SYNAPSES SEED STEPS OUT
//        network sized like synq_sim_new_for_synapses (solve_neurons,
//        benchmarks.cpp:220-249), deterministic run; OUT.adj
//        (adjacency_list::save_file of the built graph), OUT.frames,
//        OUT.state, OUT.counters as for `run`
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "synq/adjacency.hpp"
#include "synq/analysis.hpp"
#include "synq/engine.hpp"
#include "synq/models/benchmarks.hpp"
#include "synq/network_desc.hpp"
#include "synq/params.hpp"
#include "synq/random.hpp"
// the sweep model is user code against the model concept: this repo's header,
// resolved against the reference's own synq/soa.hpp (include path order)
#include "../include/synq/models/sweep.hpp"

using namespace synq;

namespace {

template <class T>
void out_bin(const T* p, size_t n) {
    fwrite(p, sizeof(T), n, stdout);
}

struct replay {
    std::vector<double> v;
    size_t next = 0;
    double uniform01() { return v.at(next++); }
};

network_desc desc_for(const std::string& model, uint32_t neurons, const param_set& ps,
                      double& dt_out) {
    if (model == "pingpong") return build_pingpong(ps).desc;
    if (model == "vogels") return build_vogels(neurons, ps).desc;
    if (model == "brunel") return build_brunel(neurons, ps).desc;
    if (model == "brunel+") return build_brunel_plus(neurons, ps).desc;
    (void)dt_out;
    throw std::invalid_argument("unknown model " + model);
}

void write_plan(const construction_plan& p, const std::string& path) {
    std::ofstream o(path, std::ios::binary);
    uint32_t hdr[4] = {static_cast<uint32_t>(p.jobs.size()), p.deg_max, p.row_pitch,
                       static_cast<uint32_t>(p.out_degree.size())};
    o.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
    uint64_t te = p.total_edges;
    o.write(reinterpret_cast<const char*>(&te), 8);
    for (const auto& j : p.jobs) {
        uint32_t w[3] = {j.n, j.a, j.b};
        o.write(reinterpret_cast<const char*>(w), 12);
        o.write(reinterpret_cast<const char*>(&j.o), 8);
    }
    o.write(reinterpret_cast<const char*>(p.out_degree.data()), p.out_degree.size() * 4);
}

struct frame_log {
    std::vector<uint32_t> buf;
    void operator()(int64_t, std::span<const uint32_t> f) {
        buf.push_back(static_cast<uint32_t>(f.size()));
        buf.insert(buf.end(), f.begin(), f.end());
    }
};

template <class M>
void dump_run(network<M>& net, int64_t steps, const std::string& out) {
    frame_log log;
    net.set_spike_tap(std::ref(log));
    net.run(steps);
    {
        std::ofstream o(out + ".frames", std::ios::binary);
        o.write(reinterpret_cast<const char*>(log.buf.data()), log.buf.size() * 4);
    }
    {
        std::ofstream o(out + ".state", std::ios::binary);
        constexpr size_t nf = M::neuron_fields::count;
        auto put_field = [&](auto span) {
            o.write(reinterpret_cast<const char*>(span.data()), span.size_bytes());
        };
        put_field(net.template neuron_field<0>());
        if constexpr (nf > 1) put_field(net.template neuron_field<1>());
        if constexpr (nf > 2) put_field(net.template neuron_field<2>());
    }
    if constexpr (network<M>::has_synapses) {
        std::vector<uint32_t> ages(net.ages().begin(), net.ages().end());
        {
            std::ofstream o(out + ".ages", std::ios::binary);
            o.write(reinterpret_cast<const char*>(ages.data()), ages.size() * 4);
        }
        auto c0 = net.counters();
        net.flush();
        std::ofstream o(out + ".syn", std::ios::binary);
        auto put = [&](auto span) {
            o.write(reinterpret_cast<const char*>(span.data()), span.size_bytes());
        };
        put(net.template synapse_field<0>());
        put(net.template synapse_field<1>());
        put(net.template synapse_field<2>());
        std::ofstream c(out + ".preflush");
        c << "synapse_updates=" << c0.synapse_updates << "\n"
          << "expiry_batches=" << c0.expiry_batches << "\n";
    }
    const auto& c = net.counters();
    std::ofstream o(out + ".counters");
    o << "steps=" << c.steps << "\nspikes=" << c.spikes << "\ndeliveries=" << c.deliveries
      << "\nsynapse_updates=" << c.synapse_updates << "\nexpiry_batches=" << c.expiry_batches
      << "\nframes_consumed=" << c.frames_consumed << "\nedges=" << net.edge_count()
      << "\nneurons=" << net.neuron_count() << "\ndeg_max=" << net.graph().deg_max()
      << "\nrow_pitch=" << net.graph().row_pitch() << "\nhistory=" << net.history_frames()
      << "\n";
}

template <class M>
void big_run(model_build<M> b, uint64_t seed, int64_t steps, const std::string& out) {
    engine_options opt;
    opt.seed = seed;
    opt.deterministic = true;
    network<M> net(b.desc, b.model, opt);
    net.graph().save_file(out + ".adj");
    dump_run(net, steps, out);
}

model_build<sweep_model> sweep_build(double S, double p, double rate) {
    const uint32_t n = static_cast<uint32_t>(std::llround(std::sqrt(S / p)));
    model_build<sweep_model> b;
    b.desc.populations = {population_spec{n}};
    b.desc.connections = {connectivity_spec{0, 0, p}};
    b.desc.dt = 0.1;
    b.desc.delay = 15;
    b.model.p_spike = static_cast<float>(rate * 0.1 * 1e-3);
    return b;
}

template <class M>
void run_model(model_build<M> b, uint64_t seed, int64_t steps, const std::string& out,
               uint32_t history) {
    engine_options opt;
    opt.seed = seed;
    opt.deterministic = true;
    opt.history_frames = history;
    network<M> net(b.desc, b.model, opt);
    dump_run(net, steps, out);
}

int run_cmd(const std::string& model, const network_desc* d, uint32_t neurons, uint64_t seed,
            int64_t steps, const std::string& out, uint32_t history, double dt, uint32_t delay) {
    param_set ps = builtin_defaults();
    auto fix = [&](auto b) {
        if (dt > 0) b.desc.dt = dt;
        if (delay > 0) b.desc.delay = delay;
        return b;
    };
    if (model == "pingpong")
        run_model(fix(d ? build_pingpong_from_desc(*d, ps) : build_pingpong(ps)), seed, steps,
                  out, history);
    else if (model == "vogels")
        run_model(fix(d ? build_vogels_from_desc(*d, ps) : build_vogels(neurons, ps)), seed,
                  steps, out, history);
    else if (model == "brunel")
        run_model(fix(d ? build_brunel_from_desc(*d, ps) : build_brunel(neurons, ps)), seed,
                  steps, out, history);
    else if (model == "brunel+")
        run_model(fix(d ? build_brunel_plus_from_desc(*d, ps) : build_brunel_plus(neurons, ps)),
                  seed, steps, out, history);
    else
        return 2;
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::string cmd = argv[1];
    try {
        if (cmd == "rng") {
            xorshift r(std::strtoull(argv[2], nullptr, 0));
            size_t n = std::strtoull(argv[3], nullptr, 0);
            std::vector<uint32_t> v(n);
            for (auto& x : v) x = r();
            out_bin(v.data(), n);
        } else if (cmd == "uniform") {
            xorshift r(std::strtoull(argv[2], nullptr, 0));
            size_t n = std::strtoull(argv[3], nullptr, 0);
            std::vector<double> v(n);
            for (auto& x : v) x = r.uniform01();
            out_bin(v.data(), n);
        } else if (cmd == "derive") {
            std::printf("%llu\n", static_cast<unsigned long long>(derive_seed(
                                      std::strtoull(argv[2], nullptr, 0),
                                      std::strtoull(argv[3], nullptr, 0))));
        } else if (cmd == "binomial") {
            xorshift r(std::strtoull(argv[2], nullptr, 0));
            uint32_t m = std::strtoul(argv[3], nullptr, 0);
            double p = std::strtod(argv[4], nullptr);
            size_t n = std::strtoull(argv[5], nullptr, 0);
            std::vector<uint32_t> v(n);
            for (auto& x : v) x = binomial(m, p, r);
            out_bin(v.data(), n);
        } else if (cmd == "sorted") {
            uint32_t n = std::strtoul(argv[2], nullptr, 0);
            uint32_t a = std::strtoul(argv[3], nullptr, 0);
            uint32_t b = std::strtoul(argv[4], nullptr, 0);
            xorshift r(std::strtoull(argv[5], nullptr, 0));
            std::vector<uint32_t> v(n);
            sorted_random(n, a, b, r, v.data());
            out_bin(v.data(), n);
        } else if (cmd == "fig2") {
            replay src{{0.46, 0.97, 0.22, 0.81, 0.98, 0.38, 0.70, 0.18}};
            std::vector<uint32_t> out(6);
            sorted_random_trace tr;
            sorted_random(6, 0, 100, src, out.data(), &tr);
            for (size_t i = 0; i < 8; ++i) {
                double row[5] = {tr.draws[i], tr.exponentials[i], tr.prefix[i], tr.normalized[i],
                                 static_cast<double>(tr.scaled[i])};
                out_bin(row, 5);
            }
            out_bin(out.data(), 6);
        } else if (cmd == "plan" || cmd == "adj") {
            double dt = 0;
            auto d = desc_for(argv[2], std::strtoul(argv[3], nullptr, 0), builtin_defaults(), dt);
            uint64_t seed = std::strtoull(argv[4], nullptr, 0);
            if (cmd == "plan")
                write_plan(plan_jobs(d, seed), argv[5]);
            else
                build_adjacency(d, seed).save_file(argv[5]);
        } else if (cmd == "run") {
            uint32_t hist = argc > 7 ? std::strtoul(argv[7], nullptr, 0) : 0;
            double dt = argc > 8 ? std::strtod(argv[8], nullptr) : 0;
            uint32_t delay = argc > 9 ? std::strtoul(argv[9], nullptr, 0) : 0;
            return run_cmd(argv[2], nullptr, std::strtoul(argv[3], nullptr, 0),
                           std::strtoull(argv[4], nullptr, 0), std::strtoll(argv[5], nullptr, 0),
                           argv[6], hist, dt, delay);
        } else if (cmd == "sweep") {
            auto b = sweep_build(std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4]));
            run_model(b, std::strtoull(argv[5], nullptr, 0), std::strtoll(argv[6], nullptr, 0), argv[7], 0);
        } else if (cmd == "sweep_time") {
            auto b = sweep_build(std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4]));
            engine_options opt;
            opt.seed = std::strtoull(argv[5], nullptr, 0);
            opt.threads = static_cast<unsigned>(std::strtoul(argv[8], nullptr, 0));
            opt.deterministic = std::atoi(argv[9]) != 0;
            network<sweep_model> net(b.desc, b.model, opt);
            net.run(std::strtoll(argv[6], nullptr, 0));
            const double t0 = net.timings().simulate;
            const uint64_t d0 = net.counters().deliveries;
            net.run(std::strtoll(argv[7], nullptr, 0));
            std::printf("events=%llu\nsim_s=%.9f\nconstruct_s=%.6f\nneurons=%u\nsynapses=%llu\n",
                        static_cast<unsigned long long>(net.counters().deliveries - d0), net.timings().simulate - t0,
                        net.timings().construct, net.neuron_count(),
                        static_cast<unsigned long long>(net.edge_count()));
        } else if (cmd == "big") {
            const std::string model = argv[2];
            param_set ps = builtin_defaults();
            const uint32_t n = solve_neurons(parse_model(model), std::strtoull(argv[3], nullptr, 0), ps);
            const uint64_t seed = std::strtoull(argv[4], nullptr, 0);
            const int64_t steps = std::strtoll(argv[5], nullptr, 0);
            if (model == "brunel")
                big_run(build_brunel(n, ps), seed, steps, argv[6]);
            else if (model == "brunel+")
                big_run(build_brunel_plus(n, ps), seed, steps, argv[6]);
            else if (model == "vogels")
                big_run(build_vogels(n, ps), seed, steps, argv[6]);
            else
                return 2;
        } else if (cmd == "run_desc") {
            network_desc d = load_desc(argv[3]);
            return run_cmd(argv[2], &d, 0, std::strtoull(argv[4], nullptr, 0),
                           std::strtoll(argv[5], nullptr, 0), argv[6], 0, 0, 0);
        } else {
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "synq_golden: %s\n", e.what());
        return 1;
    }
    return 0;
}
