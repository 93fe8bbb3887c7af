#pragma once
// Synthetic sweep model (BASELINE.json config 4, SURVEY.md 8 "SW"): one
// population of N = sqrt(S / p) neurons connected to itself with
// probability p; every neuron is a Poisson source at rate r (p_spike = r dt)
// that also receives (ACC += w per arrival, consumed by the next update).
//
// It is user code against the reference's model concept
// (proj/include/synq/engine.hpp:25-42): the same header compiles against the
// reference's own headers (oracle/golden_dump.cpp, the sweep goldens and CPU
// baseline) and against this repo's device engine (tools/sweep/sweep.cu,
// bench.py --workload sweep), where the population-delivery trait below
// selects the persistent engine.
#include <cstddef>
#include <cstdint>

#include "synq/soa.hpp"
#if defined(SYNQ_DEV)  // this repo's headers: the population-delivery trait
#include "synq/models/benchmarks.hpp"
#endif

#ifndef SYNQ_HD
#define SYNQ_HD inline
#endif

namespace synq {

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

#if defined(SYNQ_DEV)  // this repo's device engine (synq/config.hpp)
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
#endif

}  // namespace synq
