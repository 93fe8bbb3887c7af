// `synq` command line front end for the B200 library.
//
// Same options and behaviour as the reference runner
// (proj/tools/synq.cpp:60-189): build a benchmark network through the C ABI,
// simulate it on the GPU, write the raster and stats, or sweep network
// sizes into a Fig.-3-style CSV (synapses,setup_s,sim_s,bytes).  The option
// parser is a small table instead of CLI11 (not in this image).  Everything
// goes through include/synq/synq.h; nothing here touches the device.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "synq/synq.h"

namespace {

[[noreturn]] void fail(const std::string& what, int code = 1) {
    std::cerr << "synq: error: " << what << "\n";
    std::exit(code);
}

void check(synq_status st, const std::string& what) {
    if (st != SYNQ_OK) fail(what + ": " + synq_status_name(st) + " (" + synq_last_error() + ")");
}

struct opts_deleter {
    void operator()(synq_opts* o) const { synq_opts_free(o); }
};
struct sim_deleter {
    void operator()(synq_sim* s) const { synq_sim_free(s); }
};

// ------------------------------------------------------------ arguments
struct args {
    std::string model;
    uint64_t neurons = 0;
    double synapses = 0;
    double duration_s = 10.0;
    double dt_ms = 0;
    uint64_t delay = 0;
    uint64_t seed = 1;
    uint64_t threads = 0;
    bool deterministic = false;
    std::string raster, stats, net, defaults, sweep, out;
    std::vector<std::string> params;
};

enum class kind { text, count, real, flag, multi };
struct option {
    const char* name;
    kind k;
    const char* help;
    void* dst;
};

std::vector<option> option_table(args& a) {
    return {
        {"--model", kind::text, "pingpong, vogels, brunel or brunel+ (required)", &a.model},
        {"--neurons", kind::count, "network size in neurons", &a.neurons},
        {"--synapses", kind::real, "network size as an expected synapse count", &a.synapses},
        {"--duration", kind::real, "simulated seconds (default 10)", &a.duration_s},
        {"--dt", kind::real, "timestep override, simulated ms", &a.dt_ms},
        {"--delay", kind::count, "synaptic delay override, whole timesteps", &a.delay},
        {"--seed", kind::count, "master seed (default 1)", &a.seed},
        {"--threads", kind::count, "1 = reference-ordered delivery, else parallel (0 = default)", &a.threads},
        {"--deterministic", kind::flag, "reference-ordered (bit-exact) delivery", &a.deterministic},
        {"--raster", kind::text, "write the spike raster to this file", &a.raster},
        {"--stats", kind::text, "write the run summary here (default stdout)", &a.stats},
        {"--param", kind::multi, "model parameter override KEY=VALUE (repeatable)", &a.params},
        {"--defaults", kind::text, "parameter file merged over built-ins", &a.defaults},
        {"--net", kind::text, "network descriptor file (overrides --neurons)", &a.net},
        {"--sweep", kind::text, "comma-separated synapse counts; one CSV row per size", &a.sweep},
        {"--out", kind::text, "sweep CSV destination (default stdout)", &a.out},
    };
}

void usage(const std::vector<option>& table) {
    std::cout << "synq: clock-driven spiking neural network benchmark runner (B200)\n"
                 "usage: synq --model NAME [options]\n\noptions:\n";
    for (const auto& o : table) std::printf("  %-16s %s\n", o.name, o.help);
    std::printf("  %-16s %s\n  %-16s %s\n", "--help", "print this help", "--version", "print the library version");
}

double to_real(const std::string& name, const std::string& v) {
    try {
        size_t used = 0;
        const double x = std::stod(v, &used);
        if (used != v.size()) throw std::invalid_argument(v);
        return x;
    } catch (const std::exception&) {
        fail("option " + name + ": '" + v + "' is not a number", 2);
    }
}

uint64_t to_count(const std::string& name, const std::string& v) {
    if (v.empty() || v[0] == '-') fail("option " + name + ": '" + v + "' is not a non-negative integer", 2);
    try {
        size_t used = 0;
        const unsigned long long x = std::stoull(v, &used);
        if (used != v.size()) throw std::invalid_argument(v);
        return x;
    } catch (const std::exception&) {
        fail("option " + name + ": '" + v + "' is not a non-negative integer", 2);
    }
}

args parse(int argc, char** argv) {
    args a;
    const auto table = option_table(a);
    for (int i = 1; i < argc; ++i) {
        std::string tok = argv[i], val;
        bool has_val = false;
        if (tok == "--help" || tok == "-h") {
            usage(table);
            std::exit(0);
        }
        if (tok == "--version") {
            std::cout << synq_version() << "\n";
            std::exit(0);
        }
        if (const auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = tok.substr(eq + 1);
            tok = tok.substr(0, eq);
            has_val = true;
        }
        const option* o = nullptr;
        for (const auto& c : table)
            if (tok == c.name) o = &c;
        if (!o) fail("unknown option '" + tok + "' (see --help)", 2);
        if (o->k == kind::flag) {
            if (has_val) fail("option " + tok + " takes no value", 2);
            *static_cast<bool*>(o->dst) = true;
            continue;
        }
        if (!has_val) {
            if (i + 1 >= argc) fail("option " + tok + " needs a value", 2);
            val = argv[++i];
        }
        switch (o->k) {
            case kind::text: *static_cast<std::string*>(o->dst) = val; break;
            case kind::count: *static_cast<uint64_t*>(o->dst) = to_count(tok, val); break;
            case kind::real: *static_cast<double*>(o->dst) = to_real(tok, val); break;
            case kind::multi: static_cast<std::vector<std::string>*>(o->dst)->push_back(val); break;
            case kind::flag: break;
        }
    }
    if (a.model.empty()) fail("--model is required (see --help)", 2);
    return a;
}

std::vector<uint64_t> sweep_sizes(const std::string& list) {
    std::vector<uint64_t> sizes;
    std::stringstream ss(list);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        if (tok.empty()) continue;
        const double v = to_real("--sweep", tok);
        if (v < 1) fail("sweep sizes must be >= 1 synapse");
        sizes.push_back(static_cast<uint64_t>(std::llround(v)));
    }
    return sizes;
}

int64_t steps_for(double seconds, synq_sim* sim) {
    return static_cast<int64_t>(std::llround(seconds * 1000.0 / synq_sim_dt(sim)));
}

}  // namespace

int main(int argc, char** argv) {
    const args a = parse(argc, argv);
    const bool sweeping = !a.sweep.empty();
    if (a.neurons && a.synapses) fail("give either --neurons or --synapses, not both");
    if (sweeping && (a.neurons || a.synapses || !a.net.empty() || !a.raster.empty()))
        fail("--sweep cannot be combined with --neurons/--synapses/--net/--raster");
    if (!sweeping && a.model != "pingpong" && !a.neurons && !a.synapses && a.net.empty())
        fail("model '" + a.model + "' needs --neurons, --synapses or --net");
    if (!(a.duration_s > 0)) fail("--duration must be > 0");
    if (a.neurons > 0xffffffffull) fail("--neurons must fit 32 bits");
    if (a.delay > 0xffffffffull) fail("--delay must fit 32 bits");
    if (a.threads > 0xffffffffull) fail("--threads must fit 32 bits");

    std::unique_ptr<synq_opts, opts_deleter> opts(synq_opts_new());
    if (!opts) fail("out of memory");
    check(synq_opts_seed(opts.get(), a.seed), "seed");
    check(synq_opts_threads(opts.get(), static_cast<uint32_t>(a.threads)), "threads");
    check(synq_opts_deterministic(opts.get(), a.deterministic ? 1 : 0), "deterministic");
    if (!a.defaults.empty()) check(synq_opts_defaults_file(opts.get(), a.defaults.c_str()), "defaults file");
    for (const auto& kv : a.params) {
        const auto eq = kv.find('=');
        if (eq == std::string::npos || eq == 0) fail("bad --param '" + kv + "'");
        double v = 0;
        try {
            size_t used = 0;
            v = std::stod(kv.substr(eq + 1), &used);
            if (used != kv.size() - eq - 1) throw std::invalid_argument(kv);
        } catch (const std::exception&) {
            fail("bad --param value in '" + kv + "'");
        }
        check(synq_opts_param(opts.get(), kv.substr(0, eq).c_str(), v), "param");
    }
    if (a.dt_ms > 0) check(synq_opts_dt(opts.get(), a.dt_ms), "dt");
    if (a.delay > 0) check(synq_opts_delay(opts.get(), static_cast<uint32_t>(a.delay)), "delay");
    if (!a.raster.empty()) check(synq_opts_record(opts.get(), 1), "record");

    if (sweeping) {
        const auto sizes = sweep_sizes(a.sweep);
        if (sizes.size() < 2) fail("--sweep needs at least two sizes");
        std::ofstream file;
        std::ostream* out = &std::cout;
        if (!a.out.empty()) {
            file.open(a.out);
            if (!file) fail("cannot open sweep output: " + a.out);
            out = &file;
        }
        *out << "synapses,setup_s,sim_s,bytes\n" << std::flush;
        for (uint64_t size : sizes) {
            synq_sim* raw = nullptr;
            if (synq_sim_new_for_synapses(a.model.c_str(), size, opts.get(), &raw) != SYNQ_OK)
                fail("sweep size " + std::to_string(size) + ": " + synq_last_error());
            std::unique_ptr<synq_sim, sim_deleter> sim(raw);
            if (synq_sim_run(raw, steps_for(a.duration_s, raw)) != SYNQ_OK || synq_sim_flush(raw) != SYNQ_OK)
                fail("sweep size " + std::to_string(size) + ": " + synq_last_error());
            const double setup = synq_sim_seconds(raw, SYNQ_PHASE_CONSTRUCT) +
                                 synq_sim_seconds(raw, SYNQ_PHASE_INIT_NEURONS) +
                                 synq_sim_seconds(raw, SYNQ_PHASE_INIT_SYNAPSES);
            synq_memory mem{};
            check(synq_memory_estimate(a.model.c_str(), synq_sim_neurons(raw), synq_sim_synapses(raw), &mem),
                  "memory estimate");
            *out << synq_sim_synapses(raw) << "," << setup << "," << synq_sim_seconds(raw, SYNQ_PHASE_SIMULATE)
                 << "," << static_cast<uint64_t>(mem.total_bytes) << "\n"
                 << std::flush;
            if (!*out) fail("failed writing sweep output");
        }
        return 0;
    }

    synq_sim* raw = nullptr;
    synq_status st;
    if (!a.net.empty())
        st = synq_sim_new_from_file(a.model.c_str(), a.net.c_str(), opts.get(), &raw);
    else if (a.synapses > 0)
        st = synq_sim_new_for_synapses(a.model.c_str(), static_cast<uint64_t>(std::llround(a.synapses)), opts.get(),
                                       &raw);
    else
        st = synq_sim_new(a.model.c_str(), static_cast<uint32_t>(a.neurons), opts.get(), &raw);
    check(st, "building '" + a.model + "'");
    std::unique_ptr<synq_sim, sim_deleter> sim(raw);
    check(synq_sim_run(raw, steps_for(a.duration_s, raw)), "simulation");
    check(synq_sim_flush(raw), "flush");
    if (!a.raster.empty()) check(synq_sim_write_raster(raw, a.raster.c_str()), "raster");
    check(synq_sim_write_stats(raw, a.stats.empty() ? nullptr : a.stats.c_str()), "stats");
    return 0;
}
