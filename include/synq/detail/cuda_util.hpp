#pragma once
// Minimal CUDA runtime helpers for the synq engine: error mapping onto the
// C ABI status classes (bad_alloc -> SYNQ_ERR_NO_MEMORY, device_error ->
// SYNQ_ERR_INTERNAL) and RAII device / pinned-host buffers.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <exception>
#include <new>
#include <string>
#include <utility>

namespace synq {

// CUDA failures are internal errors, not I/O errors: derive from
// std::exception directly so capi maps them to SYNQ_ERR_INTERNAL.
class device_error : public std::exception {
public:
    explicit device_error(std::string what) : what_(std::move(what)) {}
    const char* what() const noexcept override { return what_.c_str(); }

private:
    std::string what_;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        throw std::bad_alloc();
    }
    throw device_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

#define SYNQ_CUDA(expr) ::synq::cuda_check((expr), #expr)

template <class T>
class dev_array {
public:
    dev_array() = default;
    explicit dev_array(size_t n) { resize(n); }
    ~dev_array() { release(); }
    dev_array(const dev_array&) = delete;
    dev_array& operator=(const dev_array&) = delete;
    dev_array(dev_array&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    dev_array& operator=(dev_array&& o) noexcept {
        if (this != &o) {
            release();
            p_ = std::exchange(o.p_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }

    void resize(size_t n) {
        release();
        if (n) SYNQ_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
        n_ = n;
    }
    void zero(cudaStream_t s = nullptr) {
        if (n_) SYNQ_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    void fill_bytes(int v, cudaStream_t s = nullptr) {
        if (n_) SYNQ_CUDA(cudaMemsetAsync(p_, v, n_ * sizeof(T), s));
    }
    void upload(const T* h, size_t n, cudaStream_t s = nullptr) {
        if (n) SYNQ_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T* h, size_t n, cudaStream_t s = nullptr) const {
        if (n) SYNQ_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }

    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }
    explicit operator bool() const { return p_ != nullptr; }

    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

template <class T>
class pinned_array {
public:
    pinned_array() = default;
    explicit pinned_array(size_t n) { resize(n); }
    ~pinned_array() {
        if (p_) cudaFreeHost(p_);
    }
    pinned_array(const pinned_array&) = delete;
    pinned_array& operator=(const pinned_array&) = delete;
    void resize(size_t n) {
        if (n <= n_) return;
        if (p_) cudaFreeHost(p_);
        p_ = nullptr;
        SYNQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p_), n * sizeof(T)));
        n_ = n;
    }
    T* get() const { return p_; }
    T* data() const { return p_; }
    T& operator[](size_t i) const { return p_[i]; }
    size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace synq
