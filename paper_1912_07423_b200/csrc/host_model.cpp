// Host-side model plumbing: descriptors, parameters, analysis helpers and
// the benchmark builders.  Behaviour follows the reference (file:line cited
// per function); none of this is on the device hot path, but the builders
// decide every constant the kernels consume, so they must agree exactly.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <limits>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>

#include "synq/analysis.hpp"
#include "synq/models/benchmarks.hpp"
#include "synq/network_desc.hpp"
#include "synq/params.hpp"

namespace synq {

namespace {
std::string strip(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return {};
    const auto e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}
}  // namespace

// ---------------------------------------------------------- network_desc
// network_desc.cpp:9-22
uint32_t network_desc::neuron_count() const {
    uint64_t n = 0;
    for (const auto& p : populations) n += p.size;
    return static_cast<uint32_t>(n);
}

std::pair<uint32_t, uint32_t> network_desc::id_range(size_t pop) const {
    if (pop >= populations.size()) throw std::out_of_range("population index out of range");
    uint32_t lo = 0;
    for (size_t i = 0; i < pop; ++i) lo += populations[i].size;
    return {lo, lo + populations[pop].size};
}

// network_desc.cpp:26-59: every violated invariant, one message each
std::vector<std::string> validate(const network_desc& d) {
    std::vector<std::string> bad;
    uint64_t total = 0;
    for (size_t i = 0; i < d.populations.size(); ++i) {
        if (d.populations[i].size == 0)
            bad.push_back("population " + std::to_string(i) + " is empty; size must be >= 1");
        total += d.populations[i].size;
    }
    if (total >= std::numeric_limits<uint32_t>::max())
        bad.push_back("total neuron count " + std::to_string(total) +
                      " exceeds the supported id space");
    std::set<std::pair<uint32_t, uint32_t>> pairs;
    for (size_t i = 0; i < d.connections.size(); ++i) {
        const auto& c = d.connections[i];
        const std::string at = "connection " + std::to_string(i);
        if (c.src >= d.populations.size())
            bad.push_back(at + ": source population index " + std::to_string(c.src) +
                          " is dangling");
        if (c.dst >= d.populations.size())
            bad.push_back(at + ": target population index " + std::to_string(c.dst) +
                          " is dangling");
        if (!(c.p >= 0.0 && c.p <= 1.0))
            bad.push_back(at + ": probability " + std::to_string(c.p) + " out of range [0, 1]");
        if (!pairs.insert({c.src, c.dst}).second)
            bad.push_back(at + ": duplicate (src, dst) pair " + std::to_string(c.src) + " -> " +
                          std::to_string(c.dst));
    }
    if (d.delay < 1) bad.push_back("delay must be >= 1 timestep");
    if (!(d.dt > 0.0)) bad.push_back("dt must be > 0");
    return bad;
}

void validate_or_throw(const network_desc& d) {
    const auto bad = validate(d);
    if (bad.empty()) return;
    std::string msg = "invalid network description:";
    for (const auto& b : bad) msg += "\n  - " + b;
    throw std::invalid_argument(msg);
}

// network_desc.cpp:80-125
network_desc parse_desc(std::istream& in) {
    network_desc d;
    bool have_pops = false;
    std::string line;
    for (size_t no = 1; std::getline(in, line); ++no) {
        if (const auto h = line.find('#'); h != std::string::npos) line.erase(h);
        line = strip(line);
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw std::invalid_argument("descriptor line " + std::to_string(no) +
                                        ": expected key = value");
        const std::string key = strip(line.substr(0, eq));
        const std::string val = strip(line.substr(eq + 1));
        if (key == "populations") {
            have_pops = true;
            std::stringstream ss(val);
            for (std::string tok; std::getline(ss, tok, ',');) {
                tok = strip(tok);
                if (!tok.empty()) d.populations.push_back({static_cast<uint32_t>(std::stoul(tok))});
            }
        } else if (key == "connection") {
            std::stringstream ss(val);
            connectivity_spec c;
            if (!(ss >> c.src >> c.dst >> c.p))
                throw std::invalid_argument("descriptor line " + std::to_string(no) +
                                            ": expected 'connection = src dst p'");
            d.connections.push_back(c);
        } else if (key == "dt") {
            d.dt = std::stod(val);
        } else if (key == "delay") {
            d.delay = static_cast<uint32_t>(std::stoul(val));
        } else {
            throw std::invalid_argument("descriptor line " + std::to_string(no) +
                                        ": unknown key '" + key + "'");
        }
    }
    if (!have_pops) throw std::invalid_argument("descriptor: missing 'populations' entry");
    return d;
}

network_desc load_desc(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open descriptor file: " + path);
    return parse_desc(in);
}

void write_desc(std::ostream& out, const network_desc& d) {
    out << "populations = ";
    for (size_t i = 0; i < d.populations.size(); ++i) out << (i ? ", " : "") << d.populations[i].size;
    out << "\n";
    for (const auto& c : d.connections) out << "connection = " << c.src << " " << c.dst << " " << c.p << "\n";
    out << "dt = " << d.dt << "\ndelay = " << d.delay << "\n";
}

// ----------------------------------------------------------------- params
// params.cpp:8-56 == configs/model_defaults.cfg
param_set builtin_defaults() {
    return {
        {"measure.warmup_ms", 500.0},      {"measure.exclude_stimulus", 1.0},
        {"pingpong.population", 100.0},    {"pingpong.p", 0.01},
        {"pingpong.dt_ms", 1.0},           {"pingpong.delay_steps", 1.0},
        {"vogels.dt_ms", 0.1},             {"vogels.delay_steps", 8.0},
        {"vogels.p", 0.02},                {"vogels.exc_fraction", 0.8},
        {"vogels.tau_m_ms", 20.0},         {"vogels.v_rest_mv", -49.0},
        {"vogels.v_reset_mv", -60.0},      {"vogels.v_threshold_mv", -50.0},
        {"vogels.refractory_ms", 5.0},     {"vogels.background_mv_per_ms", 0.0},
        {"vogels.w_exc_mv", 0.4},          {"vogels.w_inh_mv", -2.2},
        {"vogels.v_init_lo_mv", -60.0},    {"vogels.v_init_hi_mv", -50.0},
        {"brunel.dt_ms", 0.1},             {"brunel.delay_steps", 15.0},
        {"brunel.p", 0.1},                 {"brunel.exc_fraction", 0.4},
        {"brunel.inh_fraction", 0.1},      {"brunel.tau_m_ms", 20.0},
        {"brunel.v_rest_mv", 0.0},         {"brunel.v_reset_mv", 10.0},
        {"brunel.v_threshold_mv", 20.0},   {"brunel.refractory_ms", 2.0},
        {"brunel.background_mv_per_ms", 0.0}, {"brunel.j_mv", 0.1},
        {"brunel.g", 5.0},                 {"brunel.eta", 2.0},
        {"stdp.a_plus", 0.01},             {"stdp.a_minus", 0.0105},
        {"stdp.tau_plus_ms", 20.0},        {"stdp.tau_minus_ms", 20.0},
        {"stdp.w_min_mv", 0.0},            {"stdp.w_max_mv", 0.3},
    };
}

// params.cpp:69-93 (file errors are runtime_error -> SYNQ_ERR_IO)
void merge_params_file(param_set& base, const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open parameter file: " + path);
    std::string line;
    for (size_t no = 1; std::getline(in, line); ++no) {
        if (const auto h = line.find('#'); h != std::string::npos) line.erase(h);
        line = strip(line);
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw std::runtime_error(path + ":" + std::to_string(no) + ": expected key = value");
        const std::string key = strip(line.substr(0, eq));
        const std::string val = strip(line.substr(eq + 1));
        try {
            base[key] = std::stod(val);
        } catch (const std::exception&) {
            throw std::runtime_error(path + ":" + std::to_string(no) + ": not a number: '" + val + "'");
        }
    }
}

// params.cpp:95-107
void merge_param_kv(param_set& base, const std::string& kv) {
    const auto eq = kv.find('=');
    if (eq == std::string::npos) throw std::invalid_argument("expected KEY=VALUE, got '" + kv + "'");
    const std::string key = strip(kv.substr(0, eq));
    if (key.empty()) throw std::invalid_argument("empty parameter key in '" + kv + "'");
    try {
        base[key] = std::stod(strip(kv.substr(eq + 1)));
    } catch (const std::exception&) {
        throw std::invalid_argument("parameter value is not a number: '" + kv + "'");
    }
}

double param(const param_set& ps, const std::string& key) {
    const auto it = ps.find(key);
    if (it == ps.end()) throw std::invalid_argument("missing parameter: " + key);
    return it->second;
}

// --------------------------------------------------------------- analysis
// analysis.cpp:9-26
model_kind parse_model(const std::string& name) {
    if (name == "pingpong") return model_kind::pingpong;
    if (name == "vogels") return model_kind::vogels;
    if (name == "brunel") return model_kind::brunel;
    if (name == "brunel+" || name == "brunel_plus") return model_kind::brunel_plus;
    throw std::invalid_argument("unknown model '" + name +
                                "' (expected pingpong, vogels, brunel or brunel+)");
}

const char* model_name(model_kind k) {
    switch (k) {
        case model_kind::pingpong: return "pingpong";
        case model_kind::vogels: return "vogels";
        case model_kind::brunel: return "brunel";
        case model_kind::brunel_plus: return "brunel+";
    }
    return "?";
}

// Eq. 1 (analysis.cpp:28-39): c = 16e6/N^2 for vogels, 2e4/N for brunel(+)
double scaling_constant(model_kind k, uint64_t neurons) {
    if (neurons == 0) throw std::invalid_argument("scaling_constant: neuron count must be > 0");
    const double n = static_cast<double>(neurons);
    if (k == model_kind::vogels) return 16000000.0 / (n * n);
    if (k == model_kind::brunel || k == model_kind::brunel_plus) return 20000.0 / n;
    throw std::invalid_argument(std::string("scaling_constant: no scaling rule for model '") +
                                model_name(k) + "'");
}

double firing_rate(uint64_t spikes, uint64_t neurons, int64_t steps) {
    if (steps <= 0) throw std::invalid_argument("firing_rate: steps must be > 0");
    if (neurons == 0) return 0.0;
    return static_cast<double>(spikes) / (static_cast<double>(neurons) * static_cast<double>(steps));
}

double firing_rate(const spike_raster& r, uint64_t neurons, int64_t steps) {
    return firing_rate(r.records.size(), neurons, steps);
}

bool rate_retention(model_kind k, double at_size, double at_original) {
    double lo = 0, hi = 0;
    if (k == model_kind::vogels) {
        lo = 0.5;
        hi = 2.0;
    } else if (k == model_kind::brunel || k == model_kind::brunel_plus) {
        lo = 0.8;
        hi = 1.25;
    } else {
        throw std::invalid_argument(std::string("rate_retention: no band for model '") +
                                    model_name(k) + "'");
    }
    return at_size >= lo * at_original && at_size <= hi * at_original;
}

// Table 1 of the paper (analysis.cpp:71-102)
memory_breakdown memory_estimate(model_kind k) {
    memory_breakdown m;
    switch (k) {
        case model_kind::vogels:
            m.neuron_fields = 16;
            m.neuron_spikes = 8 * 4;
            m.synapse_adjacency = 4;
            return m;
        case model_kind::brunel:
            m.neuron_fields = 8;
            m.neuron_spikes = 15 * 4;
            m.synapse_adjacency = 4;
            return m;
        case model_kind::brunel_plus:
            m.neuron_fields = 8;
            m.neuron_spikes = 15 * 4;
            m.neuron_bitmasks = 50.0 / 8.0;
            m.neuron_ages = 4;
            m.neuron_expirations = 4;
            m.synapse_adjacency = 4;
            m.synapse_fields = 12;
            return m;
        default:
            break;
    }
    throw std::invalid_argument(std::string("memory_estimate: no accounting for model '") +
                                model_name(k) + "'");
}

void write_raster(std::ostream& out, const spike_raster& r) {
    out << "# dt=" << r.dt << " N=" << r.neurons << "\n";
    for (const auto& rec : r.records) out << rec.step << "\t" << rec.neuron << "\n";
}

void write_raster_file(const std::string& path, const spike_raster& r) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open raster file for writing: " + path);
    write_raster(out, r);
    out.flush();
    if (!out) throw std::runtime_error("failed writing raster file: " + path);
}

spike_raster read_raster(std::istream& in) {
    spike_raster r;
    std::string line;
    if (!std::getline(in, line) || line.rfind("# dt=", 0) != 0)
        throw std::runtime_error("raster: missing '# dt=<ms> N=<count>' header");
    {
        std::stringstream ss(line.substr(5));
        std::string ntok;
        ss >> r.dt >> ntok;
        if (ntok.rfind("N=", 0) != 0) throw std::runtime_error("raster: malformed header");
        r.neurons = static_cast<uint32_t>(std::stoul(ntok.substr(2)));
    }
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::stringstream ss(line);
        spike_record rec{};
        if (!(ss >> rec.step >> rec.neuron)) throw std::runtime_error("raster: malformed record");
        r.records.push_back(rec);
    }
    return r;
}

spike_raster read_raster_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open raster file: " + path);
    return read_raster(in);
}

// -------------------------------------------------------------- builders
namespace {

uint32_t nearest(double x) { return static_cast<uint32_t>(std::llround(x)); }

lif_params lif_of(const param_set& ps, const std::string& pre) {  // benchmarks.cpp:9-21
    lif_params p;
    p.tau_m = static_cast<float>(param(ps, pre + ".tau_m_ms"));
    p.v_rest = static_cast<float>(param(ps, pre + ".v_rest_mv"));
    p.v_reset = static_cast<float>(param(ps, pre + ".v_reset_mv"));
    p.v_threshold = static_cast<float>(param(ps, pre + ".v_threshold_mv"));
    p.refractory = static_cast<float>(param(ps, pre + ".refractory_ms"));
    p.background = static_cast<float>(param(ps, pre + ".background_mv_per_ms"));
    if (!(p.tau_m > 0)) throw std::invalid_argument(pre + ": tau_m must be > 0");
    if (!(p.v_threshold > p.v_reset))
        throw std::invalid_argument(pre + ": v_threshold must exceed v_reset");
    return p;
}

double p_of(const network_desc& d, uint32_t src, uint32_t dst) {
    for (const auto& c : d.connections)
        if (c.src == src && c.dst == dst) return c.p;
    return 0.0;
}

void need_pops(const network_desc& d, size_t n, const char* model) {
    if (d.populations.size() != n)
        throw std::invalid_argument(std::string(model) + ": descriptor must declare " +
                                    std::to_string(n) + " populations, got " +
                                    std::to_string(d.populations.size()));
}

// benchmarks.cpp:105-138: Eq.-1 scaling and the size-invariant stimulus rate
void brunel_common(brunel_model& m, const network_desc& d, const param_set& ps, double& scale) {
    const uint32_t ne = d.populations[0].size, ni = d.populations[1].size,
                   ns = d.populations[2].size;
    m.lif = lif_of(ps, "brunel");
    const double j = param(ps, "brunel.j_mv"), g = param(ps, "brunel.g");
    m.j_exc = static_cast<float>(j);
    m.j_inh = static_cast<float>(-g * j);
    m.n_exc = ne;
    m.n_recurrent = ne + ni;
    m.v_init_hi = m.lif.v_threshold;
    scale = scaling_constant(model_kind::brunel, d.neuron_count());
    m.scale_c = static_cast<float>(scale);
    const double eta = param(ps, "brunel.eta");
    const double c_e = p_of(d, 0, 0) * ne;
    const double c_p = p_of(d, 2, 0) * ns;
    if (c_e <= 0 || c_p <= 0)
        throw std::invalid_argument("brunel: descriptor must connect populations 0->0 and 2->0");
    const double theta = m.lif.v_threshold - m.lif.v_rest;
    const double tau_s = m.lif.tau_m / 1000.0;
    const double rate_thr_hz = theta / (j * scale * c_e * tau_s);
    const double rate_p_hz = eta * rate_thr_hz * c_e / c_p;
    const double p_spike = rate_p_hz / 1000.0 * d.dt;
    if (p_spike > 1.0)
        throw std::invalid_argument("brunel: stimulus rate*dt exceeds 1; lower eta or dt");
    m.p_spike = static_cast<float>(p_spike);
}

network_desc brunel_layout(uint32_t neurons, const param_set& ps) {  // benchmarks.cpp:140-158
    if (neurons < 10) throw std::invalid_argument("brunel: need at least 10 neurons to split");
    const uint32_t ne = nearest(param(ps, "brunel.exc_fraction") * neurons);
    const uint32_t ni = nearest(param(ps, "brunel.inh_fraction") * neurons);
    if (ne == 0 || ni == 0 || ne + ni >= neurons)
        throw std::invalid_argument("brunel: split leaves an empty population");
    const double p = param(ps, "brunel.p");
    network_desc d;
    d.populations = {{ne}, {ni}, {neurons - ne - ni}};
    d.connections = {{0, 0, p}, {0, 1, p}, {1, 0, p}, {1, 1, p}, {2, 0, p}, {2, 1, p}};
    d.dt = param(ps, "brunel.dt_ms");
    d.delay = nearest(param(ps, "brunel.delay_steps"));
    return d;
}

}  // namespace

model_build<pingpong_model> build_pingpong_from_desc(const network_desc& d, const param_set&) {
    need_pops(d, 2, "pingpong");
    model_build<pingpong_model> b;
    b.desc = d;
    b.model.first_pop = d.populations[0].size;
    b.measure_begin = 0;
    b.measure_end = d.neuron_count();
    b.scale_c = 1.0;
    return b;
}

model_build<pingpong_model> build_pingpong(const param_set& ps) {
    const uint32_t pop = nearest(param(ps, "pingpong.population"));
    const double p = param(ps, "pingpong.p");
    network_desc d;
    d.populations = {{pop}, {pop}};
    d.connections = {{0, 1, p}, {1, 0, p}};
    d.dt = param(ps, "pingpong.dt_ms");
    d.delay = nearest(param(ps, "pingpong.delay_steps"));
    return build_pingpong_from_desc(d, ps);
}

model_build<vogels_model> build_vogels_from_desc(const network_desc& d, const param_set& ps) {
    need_pops(d, 2, "vogels");
    const uint32_t n = d.neuron_count();
    model_build<vogels_model> b;
    b.desc = d;
    b.model.lif = lif_of(ps, "vogels");
    b.model.w_exc = static_cast<float>(param(ps, "vogels.w_exc_mv"));
    b.model.w_inh = static_cast<float>(param(ps, "vogels.w_inh_mv"));
    b.model.n_exc = d.populations[0].size;
    b.model.v_init_lo = static_cast<float>(param(ps, "vogels.v_init_lo_mv"));
    b.model.v_init_hi = static_cast<float>(param(ps, "vogels.v_init_hi_mv"));
    b.scale_c = scaling_constant(model_kind::vogels, n);
    b.model.scale_c = static_cast<float>(b.scale_c);
    b.measure_begin = 0;
    b.measure_end = n;
    return b;
}

model_build<vogels_model> build_vogels(uint32_t neurons, const param_set& ps) {
    if (neurons < 10) throw std::invalid_argument("vogels: need at least 10 neurons to split");
    const uint32_t ne = nearest(param(ps, "vogels.exc_fraction") * neurons);
    if (ne == 0 || ne >= neurons)
        throw std::invalid_argument("vogels: excitatory split leaves an empty population");
    const double p = param(ps, "vogels.p");
    network_desc d;
    d.populations = {{ne}, {neurons - ne}};
    d.connections = {{0, 0, p}, {0, 1, p}, {1, 0, p}, {1, 1, p}};
    d.dt = param(ps, "vogels.dt_ms");
    d.delay = nearest(param(ps, "vogels.delay_steps"));
    return build_vogels_from_desc(d, ps);
}

model_build<brunel_model> build_brunel_from_desc(const network_desc& d, const param_set& ps) {
    need_pops(d, 3, "brunel");
    model_build<brunel_model> b;
    b.desc = d;
    brunel_common(b.model, b.desc, ps, b.scale_c);
    b.measure_begin = 0;
    b.measure_end = b.model.n_recurrent;
    return b;
}

model_build<brunel_model> build_brunel(uint32_t neurons, const param_set& ps) {
    return build_brunel_from_desc(brunel_layout(neurons, ps), ps);
}

model_build<brunel_plus_model> build_brunel_plus_from_desc(const network_desc& d,
                                                           const param_set& ps) {
    need_pops(d, 3, "brunel+");
    model_build<brunel_plus_model> b;
    b.desc = d;
    brunel_common(b.model, b.desc, ps, b.scale_c);
    auto& s = b.model.stdp;
    s.a_plus = static_cast<float>(param(ps, "stdp.a_plus"));
    s.a_minus = static_cast<float>(param(ps, "stdp.a_minus"));
    s.tau_plus = static_cast<float>(param(ps, "stdp.tau_plus_ms"));
    s.tau_minus = static_cast<float>(param(ps, "stdp.tau_minus_ms"));
    s.w_min = static_cast<float>(param(ps, "stdp.w_min_mv"));
    s.w_max = static_cast<float>(param(ps, "stdp.w_max_mv"));
    if (!(s.w_min < s.w_max)) throw std::invalid_argument("stdp: need w_min < w_max");
    s.bind(static_cast<float>(b.desc.dt));
    b.measure_begin = 0;
    b.measure_end = b.model.n_recurrent;
    return b;
}

model_build<brunel_plus_model> build_brunel_plus(uint32_t neurons, const param_set& ps) {
    return build_brunel_plus_from_desc(brunel_layout(neurons, ps), ps);
}

// benchmarks.cpp:201-249
double expected_synapses(model_kind k, uint32_t neurons, const param_set& ps) {
    const double n = neurons;
    switch (k) {
        case model_kind::pingpong: {
            const double pop = param(ps, "pingpong.population");
            return 2.0 * param(ps, "pingpong.p") * pop * pop;
        }
        case model_kind::vogels: return param(ps, "vogels.p") * n * n;
        case model_kind::brunel:
        case model_kind::brunel_plus: {
            const double targets =
                param(ps, "brunel.exc_fraction") * n + param(ps, "brunel.inh_fraction") * n;
            return param(ps, "brunel.p") * n * targets;
        }
    }
    return 0.0;
}

uint32_t solve_neurons(model_kind k, uint64_t synapses, const param_set& ps) {
    const double target = static_cast<double>(synapses);
    double guess = 0;
    if (k == model_kind::vogels) {
        guess = std::sqrt(target / param(ps, "vogels.p"));
    } else if (k == model_kind::brunel || k == model_kind::brunel_plus) {
        const double f = param(ps, "brunel.exc_fraction") + param(ps, "brunel.inh_fraction");
        guess = std::sqrt(target / (param(ps, "brunel.p") * f));
    } else {
        throw std::invalid_argument(std::string("solve_neurons: model '") + model_name(k) +
                                    "' has a fixed size");
    }
    uint32_t best = std::max<uint32_t>(10, nearest(guess));
    double best_err = std::abs(expected_synapses(k, best, ps) - target);
    for (int64_t d = -2; d <= 2; ++d) {
        const int64_t cand = static_cast<int64_t>(std::llround(guess)) + d;
        if (cand < 10) continue;
        const double err = std::abs(expected_synapses(k, static_cast<uint32_t>(cand), ps) - target);
        if (err < best_err) {
            best_err = err;
            best = static_cast<uint32_t>(cand);
        }
    }
    return best;
}

}  // namespace synq
