// Shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "host.hpp"

namespace fclsh_b200 {

#define FCLSH_CUDA(call)                                                                     \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::fclsh_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Per-thread count of kernels launched by this library (bench accounting).
uint64_t& launch_counter();

#define FCLSH_LAUNCHED()                                                                     \
    do {                                                                                     \
        ::fclsh_b200::launch_counter()++;                                                    \
        cudaError_t _e = cudaGetLastError();                                                 \
        if (_e != cudaSuccess)                                                               \
            throw ::fclsh_b200::CudaError(std::string("kernel launch (") + __FILE__ + ":" +            \
                                          std::to_string(__LINE__) + "): " + cudaGetErrorString(_e));  \
    } while (0)

constexpr int kNumSMs = 148; // B200

inline int sm_count(int device) {
    static int cache[64] = {};
    if (device >= 0 && device < 64 && cache[device] > 0) return cache[device];
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
        return kNumSMs;
    if (device >= 0 && device < 64) cache[device] = v;
    return v;
}

// Waits for the stream by polling (a blocking cudaStreamSynchronize may
// yield the thread and add tens of microseconds of wake-up to a ~0.3 ms
// query batch).
inline void stream_spin_wait(cudaStream_t s) {
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) FCLSH_CUDA(e);
    }
}

// Resident CTAs per SM of kern at (threads, dynamic smem) on device, raising
// the kernel's dynamic-smem limit first. Cached: the attribute call and the
// occupancy query cost host microseconds on every query batch otherwise.
int resident_ctas_impl(const void* kern, int threads, size_t smem, int device);
template <typename F>
int resident_ctas(F* kern, int threads, size_t smem, int device) {
    return resident_ctas_impl(reinterpret_cast<const void*>(kern), threads, smem, device);
}

// RAII device buffer (grow-only when reused as a workspace).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void* ensure(size_t want) {
        if (want <= bytes && p) return p;
        release();
        if (want == 0) want = 16;
        FCLSH_CUDA(cudaMalloc(&p, want));
        bytes = want;
        return p;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

} // namespace fclsh_b200
