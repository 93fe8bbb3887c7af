#pragma once
// Padded-ELL adjacency and its construction
// (reference: proj/include/synq/adjacency.hpp, proj/src/adjacency.cpp).
//
// B200 design: the degree plan (one sequential binomial stream) is drawn on
// the host exactly as the reference does; expansion of every job into sorted
// random target ids runs on the device (one thread per job, exact double
// arithmetic), writing straight into the final row-sorted position so no
// per-row sort pass is needed.  adjacency_list is the host mirror.
#include <cmath>
#include <cstdint>
#include <iosfwd>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "synq/network_desc.hpp"
#include "synq/random.hpp"

namespace synq {

class thread_pool;  // accepted for signature compatibility; the device does the work

// "write n sorted, uniformly distributed random integers from [a, b) at o"
struct construction_job {
    uint32_t n = 0;
    uint32_t a = 0;
    uint32_t b = 0;
    uint64_t o = 0;
};

struct sorted_random_trace {
    std::vector<double> draws;
    std::vector<double> exponentials;
    std::vector<double> prefix;
    std::vector<double> normalized;
    std::vector<int64_t> scaled;
    std::vector<uint32_t> out;
};

// n strictly increasing integers in [a, b) from exactly n + 2 uniforms
// (adjacency.hpp:112-163): -ln -> exclusive running sum -> / total ->
// * (span - n), round half up -> + rank -> + a.
template <class Rng>
void sorted_random(uint32_t n, uint32_t a, uint32_t b, Rng& rng, uint32_t* out,
                   sorted_random_trace* trace = nullptr) {
    if (b <= a) throw std::invalid_argument("sorted_random: empty interval");
    const uint32_t span = b - a;
    if (n > span) throw std::invalid_argument("sorted_random: n exceeds interval size");
    std::vector<double> acc(n + 2);
    for (uint32_t i = 0; i < n + 2; ++i) acc[i] = rng.uniform01();
    if (trace) {
        trace->draws = acc;
        trace->exponentials.resize(n + 2);
    }
    double running = 0.0;
    for (uint32_t i = 0; i < n + 2; ++i) {
        const double e = -std::log(acc[i]);
        if (trace) trace->exponentials[i] = e;
        acc[i] = running;
        running += e;
    }
    double total = acc[n + 1];
    if (total <= 0.0) total = 1.0;
    const double scale = static_cast<double>(span - n);
    if (trace) {
        trace->prefix = acc;
        trace->normalized.resize(n + 2);
        trace->scaled.resize(n + 2);
        for (uint32_t i = 0; i < n + 2; ++i) {
            trace->normalized[i] = acc[i] / total;
            trace->scaled[i] = static_cast<int64_t>(std::floor(acc[i] / total * scale + 0.5));
        }
    }
    for (uint32_t i = 0; i < n; ++i)
        out[i] = a + static_cast<uint32_t>(std::floor(acc[i + 1] / total * scale + 0.5)) + i;
    if (trace) trace->out.assign(out, out + n);
}

struct construction_plan {
    std::vector<construction_job> jobs;  // source-major, connection order (seed index j+1)
    std::vector<uint32_t> out_degree;
    uint32_t deg_max = 0;
    uint32_t row_pitch = 0;
    uint64_t total_edges = 0;
};

// Host mirror of the device table: rows sorted ascending, padded to
// row_pitch with the sentinel 0xFFFFFFFF.
class adjacency_list {
public:
    static constexpr uint32_t sentinel = 0xffffffffu;

    adjacency_list() = default;
    adjacency_list(uint32_t neurons, uint32_t deg_max, uint32_t row_pitch);
    adjacency_list(uint32_t neurons, uint32_t deg_max, uint32_t row_pitch,
                   std::vector<uint32_t> cells, std::vector<uint32_t> degree);

    uint32_t neuron_count() const { return neurons_; }
    uint32_t deg_max() const { return deg_max_; }
    uint32_t row_pitch() const { return pitch_; }
    uint64_t edge_count() const { return edges_; }
    uint64_t bytes() const { return (cells_.size() + degree_.size()) * sizeof(uint32_t); }
    uint32_t out_degree(uint32_t id) const { return degree_[id]; }

    std::span<const uint32_t> row(uint32_t id) const;      // valid prefix
    std::span<const uint32_t> raw_row(uint32_t id) const;  // incl. sentinel padding

    const uint32_t* cells() const { return cells_.data(); }
    const uint32_t* degrees() const { return degree_.data(); }

    void dump(std::ostream& out) const;
    static adjacency_list load(std::istream& in);
    void save_file(const std::string& path) const;
    static adjacency_list load_file(const std::string& path);

private:
    uint32_t neurons_ = 0;
    uint32_t deg_max_ = 0;
    uint32_t pitch_ = 0;
    uint64_t edges_ = 0;
    std::vector<uint32_t> cells_;
    std::vector<uint32_t> degree_;
};

// sequential degree plan on derive_seed(seed, 0) (adjacency.cpp:29-71)
construction_plan plan_jobs(const network_desc& desc, uint64_t seed, uint32_t pitch_align = 32);

// expansion on the B200, downloaded into a host mirror (adjacency.cpp:73-103)
adjacency_list expand_jobs(const construction_plan& plan, uint32_t neurons, uint64_t seed,
                           thread_pool* pool = nullptr);

adjacency_list build_adjacency(const network_desc& desc, uint64_t seed,
                               uint32_t pitch_align = 32, thread_pool* pool = nullptr);

}  // namespace synq
