#pragma once
// Device-side handles passed to model callbacks inside the sm_100a kernels.
// They expose the reference's iterator surface (soa.hpp:80-171):
//   id(), get<I>(), add<I>(v), put<I>(v), rng()   — neurons
//   src(), dst(), get<I>()                         — synapses
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <type_traits>

#include "synq/random.hpp"
#include "synq/soa.hpp"

namespace synq::dev {

// One HBM array per field, type-erased to keep the state struct POD.
template <class FieldList>
struct field_ptrs {
    void* p[FieldList::count > 0 ? FieldList::count : 1] = {};
    template <size_t I>
    SYNQ_HD field_t<I, FieldList>* get() const {
        return static_cast<field_t<I, FieldList>*>(p[I]);
    }
};

template <class FieldList>
struct values;
template <class... Ts>
struct values<fields<Ts...>> {
    using type = detail::value_pack<Ts...>;
};
template <class FieldList>
using values_t = typename values<FieldList>::type;

// load / store every field of element i between HBM and a register pack
template <class FieldList, size_t I = 0>
SYNQ_DEV void load_all(const field_ptrs<FieldList>& f, uint64_t i, values_t<FieldList>& v) {
    if constexpr (I < FieldList::count) {
        detail::pack_get<I>::get(v) = f.template get<I>()[i];
        load_all<FieldList, I + 1>(f, i, v);
    }
}
template <class FieldList, size_t I = 0>
SYNQ_DEV void store_all(const field_ptrs<FieldList>& f, uint64_t i, const values_t<FieldList>& v) {
    if constexpr (I < FieldList::count) {
        f.template get<I>()[i] = detail::pack_get<I>::get(const_cast<values_t<FieldList>&>(v));
        store_all<FieldList, I + 1>(f, i, v);
    }
}
// bitwise equality (so -0.0 vs 0.0 and NaN payloads count as changes)
template <class T>
SYNQ_DEV bool same_bits(const T& a, const T& b) {
    if constexpr (sizeof(T) == 4) {
        uint32_t x, y;
        memcpy(&x, &a, 4);
        memcpy(&y, &b, 4);
        return x == y;
    } else if constexpr (sizeof(T) == 8) {
        unsigned long long x, y;
        memcpy(&x, &a, 8);
        memcpy(&y, &b, 8);
        return x == y;
    } else {
        return a == b;
    }
}

// store only the fields whose bits changed (keeps the update's write traffic
// to what the model actually modified)
template <class FieldList, size_t I = 0>
SYNQ_DEV void store_changed(const field_ptrs<FieldList>& f, uint64_t i, values_t<FieldList>& now,
                            values_t<FieldList>& before) {
    if constexpr (I < FieldList::count) {
        const auto& a = detail::pack_get<I>::get(now);
        if (!same_bits(a, detail::pack_get<I>::get(before))) f.template get<I>()[i] = a;
        store_changed<FieldList, I + 1>(f, i, now, before);
    }
}

// ---- own-neuron handle for init / update: register copy of the fields,
// lazily loaded random stream (only models that call rng() pay for it)
template <class FieldList>
struct local_neuron {
    uint32_t id_;
    values_t<FieldList>* v_;
    xorshift* rng_local_;
    bool* rng_live_;
    const xorshift* rng_global_;

    SYNQ_HD uint32_t id() const { return id_; }
    template <size_t I>
    SYNQ_HD auto& get() const {
        return detail::pack_get<I>::get(*v_);
    }
    template <size_t I, class V>
    SYNQ_HD void add(V x) const {
        get<I>() += x;
    }
    template <size_t I, class V>
    SYNQ_HD void put(V x) const {
        get<I>() = x;
    }
    SYNQ_HD xorshift& rng() const {
        if (!*rng_live_) {
            *rng_local_ = rng_global_[id_];
            *rng_live_ = true;
        }
        return *rng_local_;
    }
};

// ---- atomic RMW on any field type (sub-word types via a 32-bit CAS)
template <class T>
SYNQ_DEV void atomic_add_any(T* p, T v) {
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double> ||
                  std::is_same_v<T, int> || std::is_same_v<T, unsigned>) {
        atomicAdd(p, v);
    } else if constexpr (sizeof(T) == 8 && std::is_integral_v<T>) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
    } else if constexpr (sizeof(T) < 4) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p);
        unsigned* w = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
        const unsigned shift = static_cast<unsigned>(a & 3) * 8;
        const unsigned mask = ((1u << (8 * sizeof(T))) - 1u) << shift;
        unsigned old = *w, assumed;
        do {
            assumed = old;
            T cur = static_cast<T>((assumed & mask) >> shift);
            cur = static_cast<T>(cur + v);
            const unsigned repl = (assumed & ~mask) | ((static_cast<unsigned>(cur) << shift) & mask);
            old = atomicCAS(w, assumed, repl);
        } while (old != assumed);
    } else {
        static_assert(sizeof(T) == 0, "atomic_add_any: unsupported field type");
    }
}

template <class T>
SYNQ_DEV void store_any(T* p, T v) {
    *reinterpret_cast<volatile T*>(p) = v;
}

// ---- cross-neuron handle used as `from` / `to` during delivery.
// Atomic=true: concurrent deliveries compose through device atomics.
// Atomic=false: the caller owns the target exclusively (ordered delivery).
template <class FieldList, bool Atomic>
struct global_neuron {
    uint32_t id_;
    field_ptrs<FieldList> f_;
    xorshift* rng_;

    SYNQ_HD uint32_t id() const { return id_; }
    template <size_t I>
    SYNQ_HD auto& get() const {
        return f_.template get<I>()[id_];
    }
    template <size_t I, class V>
    SYNQ_HD void add(V x) const {
        using T = field_t<I, FieldList>;
        if constexpr (Atomic)
            atomic_add_any<T>(f_.template get<I>() + id_, static_cast<T>(x));
        else
            f_.template get<I>()[id_] += static_cast<T>(x);
    }
    template <size_t I, class V>
    SYNQ_HD void put(V x) const {
        using T = field_t<I, FieldList>;
        if constexpr (Atomic)
            store_any<T>(f_.template get<I>() + id_, static_cast<T>(x));
        else
            f_.template get<I>()[id_] = static_cast<T>(x);
    }
    SYNQ_HD xorshift& rng() const { return rng_[id_]; }
};

// ---- synapse handle at (src, k): fields live at src * deg_max + k
template <class FieldList>
struct global_synapse {
    uint64_t index_;
    uint32_t src_, dst_;
    field_ptrs<FieldList> f_;

    SYNQ_HD uint32_t src() const { return src_; }
    SYNQ_HD uint32_t dst() const { return dst_; }
    template <size_t I>
    SYNQ_HD auto& get() const {
        return f_.template get<I>()[index_];
    }
};

template <class FieldList, size_t I = 0>
SYNQ_DEV void load_syn(const field_ptrs<FieldList>& f, uint64_t i, synapse_state<FieldList>& s) {
    if constexpr (I < FieldList::count) {
        s.template get<I>() = f.template get<I>()[i];
        load_syn<FieldList, I + 1>(f, i, s);
    }
}
template <class FieldList, size_t I = 0>
SYNQ_DEV void store_syn(const field_ptrs<FieldList>& f, uint64_t i, const synapse_state<FieldList>& s) {
    if constexpr (I < FieldList::count) {
        f.template get<I>()[i] = s.template get<I>();
        store_syn<FieldList, I + 1>(f, i, s);
    }
}
// catch-up write-back: untouched (non-plastic) synapses cost no store
template <class FieldList, size_t I = 0>
SYNQ_DEV void store_syn_changed(const field_ptrs<FieldList>& f, uint64_t i,
                                const synapse_state<FieldList>& s, const synapse_state<FieldList>& s0) {
    if constexpr (I < FieldList::count) {
        if (!same_bits(s.template get<I>(), s0.template get<I>())) f.template get<I>()[i] = s.template get<I>();
        store_syn_changed<FieldList, I + 1>(f, i, s, s0);
    }
}

}  // namespace synq::dev
