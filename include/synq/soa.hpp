#pragma once
// Structure-of-arrays field declarations and access handles
// (reference API: proj/include/synq/soa.hpp:13-171).
//
// Host side: soa_store keeps one std::vector per field (it backs the host
// mirrors the engine exposes through neuron_field<I>() / synapse_field<I>()).
// Device side: the engine keeps one HBM array per field and hands model
// callbacks its own handle types (synq/detail/device_refs.cuh) that expose
// the same id()/get<I>()/add<I>()/put<I>()/rng()/src()/dst() surface.
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "synq/config.hpp"
#include "synq/random.hpp"

namespace synq {

template <class... Ts>
struct fields {
    static constexpr size_t count = sizeof...(Ts);
};

namespace detail {
template <size_t I, class... Ts>
struct nth;
template <class T, class... Ts>
struct nth<0, T, Ts...> {
    using type = T;
};
template <size_t I, class T, class... Ts>
struct nth<I, T, Ts...> {
    using type = typename nth<I - 1, Ts...>::type;
};
template <size_t I, class FieldList>
struct field_at;
template <size_t I, class... Ts>
struct field_at<I, fields<Ts...>> {
    using type = typename nth<I, Ts...>::type;
};
}  // namespace detail

template <size_t I, class FieldList>
using field_t = typename detail::field_at<I, FieldList>::type;

template <class FieldList>
class soa_store;

template <class... Ts>
class soa_store<fields<Ts...>> {
public:
    using field_list = fields<Ts...>;

    void resize(size_t n) {
        std::apply([n](auto&... col) { (col.assign(n, {}), ...); }, cols_);
        n_ = n;
    }
    size_t size() const { return n_; }

    template <size_t I>
    auto* data() {
        return std::get<I>(cols_).data();
    }
    template <size_t I>
    const auto* data() const {
        return std::get<I>(cols_).data();
    }

    uint64_t bytes() const {
        uint64_t total = 0;
        std::apply([&](const auto&... col) { ((total += col.size() * sizeof(col[0])), ...); },
                   cols_);
        return total;
    }

private:
    std::tuple<std::vector<Ts>...> cols_;
    size_t n_ = 0;
};

template <>
class soa_store<fields<>> {
public:
    using field_list = fields<>;
    void resize(size_t n) { n_ = n; }
    size_t size() const { return n_; }
    uint64_t bytes() const { return 0; }

private:
    size_t n_ = 0;
};

// Host handle to one neuron (soa.hpp:80-117).  Atomic selects lock-free
// read-modify-write for add/put, as the reference's parallel mode does.
template <class Store, bool Atomic>
class neuron_ref {
public:
    neuron_ref(Store* s, uint32_t id, xorshift* rng) : s_(s), id_(id), rng_(rng) {}

    uint32_t id() const { return id_; }

    template <size_t I>
    auto& get() const {
        return s_->template data<I>()[id_];
    }

    template <size_t I, class V>
    void add(V v) const {
        auto& slot = s_->template data<I>()[id_];
        using T = std::remove_reference_t<decltype(slot)>;
        if constexpr (Atomic) {
            std::atomic_ref<T> r(slot);
            T cur = r.load(std::memory_order_relaxed);
            while (!r.compare_exchange_weak(cur, static_cast<T>(cur + static_cast<T>(v)),
                                            std::memory_order_relaxed)) {
            }
        } else {
            slot += v;
        }
    }

    template <size_t I, class V>
    void put(V v) const {
        auto& slot = s_->template data<I>()[id_];
        using T = std::remove_reference_t<decltype(slot)>;
        if constexpr (Atomic)
            std::atomic_ref<T>(slot).store(static_cast<T>(v), std::memory_order_relaxed);
        else
            slot = v;
    }

    xorshift& rng() const { return rng_[id_]; }

private:
    Store* s_;
    uint32_t id_;
    xorshift* rng_;
};

// Host handle to one synapse at (row = source, col) with pitch deg_max.
template <class Store>
class synapse_ref {
public:
    synapse_ref(Store* s, uint64_t index, uint32_t src, uint32_t dst)
        : s_(s), index_(index), src_(src), dst_(dst) {}
    uint32_t src() const { return src_; }
    uint32_t dst() const { return dst_; }
    template <size_t I>
    auto& get() const {
        return s_->template data<I>()[index_];
    }

private:
    Store* s_;
    uint64_t index_;
    uint32_t src_, dst_;
};

// Register-resident copy of one synapse used during lazy catch-up
// (soa.hpp:143-171).  Usable on host and device.
template <class FieldList>
struct synapse_state;

namespace detail {
template <class... Ts>
struct value_pack;
template <>
struct value_pack<> {};
template <class T, class... Ts>
struct value_pack<T, Ts...> {
    T head{};
    value_pack<Ts...> tail;
};
template <size_t I>
struct pack_get {
    template <class P>
    SYNQ_HD static auto& get(P& p) {
        return pack_get<I - 1>::get(p.tail);
    }
};
template <>
struct pack_get<0> {
    template <class P>
    SYNQ_HD static auto& get(P& p) {
        return p.head;
    }
};
}  // namespace detail

template <class... Ts>
struct synapse_state<fields<Ts...>> {
    detail::value_pack<Ts...> v;
    uint32_t src_ = 0, dst_ = 0;

    SYNQ_HD uint32_t src() const { return src_; }
    SYNQ_HD uint32_t dst() const { return dst_; }

    template <size_t I>
    SYNQ_HD auto& get() {
        return detail::pack_get<I>::get(v);
    }
    template <size_t I>
    SYNQ_HD const auto& get() const {
        return detail::pack_get<I>::get(v);
    }

    template <class Store>
    void load(Store& s, uint64_t index) {
        load_impl(s, index, std::index_sequence_for<Ts...>{});
    }
    template <class Store>
    void store(Store& s, uint64_t index) const {
        store_impl(s, index, std::index_sequence_for<Ts...>{});
    }

private:
    template <class Store, size_t... Is>
    void load_impl(Store& s, uint64_t index, std::index_sequence<Is...>) {
        ((get<Is>() = s.template data<Is>()[index]), ...);
    }
    template <class Store, size_t... Is>
    void store_impl(Store& s, uint64_t index, std::index_sequence<Is...>) const {
        ((s.template data<Is>()[index] = get<Is>()), ...);
    }
};

}  // namespace synq
