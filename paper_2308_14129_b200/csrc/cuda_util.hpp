// CUDA plumbing shared by the device translation units: error mapping to the
// C-ABI status convention (CUDA failures are status 3 "CudaError"), a small
// device-buffer RAII type, and the device-selection guard.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "host.hpp"

namespace spd {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        internal_error("CudaError", std::string(what) + ": " + cudaGetErrorString(e));
}
#define SPD_CUDA(x) ::spd::cuda_check((x), #x)

// Fails loudly (status 3) when there is no usable sm_100 device: the product
// path has no CPU fallback.
void require_device(int device);

// Opt a kernel in to `bytes` of dynamic shared memory on the current device
// (the attribute is per device: a process driving several GPUs sets it on
// each); optionally prefer the maximum shared-memory carveout.
template <class K>
void ensure_smem(K kern, std::size_t bytes, bool max_carveout = false) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, std::size_t> done;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    std::size_t& have = done[{reinterpret_cast<const void*>(kern), dev}];
    if (bytes <= have) return;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)),
               "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    if (max_carveout)
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        int(cudaSharedmemCarveoutMaxShared)),
                   "cudaFuncSetAttribute(PreferredSharedMemoryCarveout)");
    have = bytes;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(std::size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(std::exchange(o.p, nullptr)), n(std::exchange(o.n, 0)) {}
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = std::exchange(o.p, nullptr);
            n = std::exchange(o.n, 0);
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(std::size_t count) {
        release();
        n = count;
        if (count) SPD_CUDA(cudaMalloc(&p, sizeof(T) * count));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    std::size_t bytes() const { return sizeof(T) * n; }
    void upload(const T* h, std::size_t count, cudaStream_t s = 0) {
        if (count) SPD_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
    }
    void download(T* h, std::size_t count, cudaStream_t s = 0) const {
        if (count) SPD_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s = 0) {
        if (n) SPD_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SPD_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace spd
