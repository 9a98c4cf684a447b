// Shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#include "host.hpp"

namespace fclsh_b200 {

#define FCLSH_CUDA(call)                                                                     \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::fclsh_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Device-side bounds checks (a build with -DFCLSH_DEBUG_BOUNDS: make
// EXTRA=-DFCLSH_DEBUG_BOUNDS BUILD=build_dbg OUT=lib/libfclsh_b200_dbg.so; the
// test suite runs against it with FCLSH_LIB, tools/bounds_check.sh). A failed
// check prints the site and traps, which fails the batch with a CUDA error.
#ifdef FCLSH_DEBUG_BOUNDS
#define FCLSH_DCHECK(cond)                                                                        \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("FCLSH_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   int(blockIdx.x), int(threadIdx.x));                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define FCLSH_DCHECK(cond) \
    do {                   \
    } while (0)
#endif

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

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// be scheduled while its stream predecessor still runs (the predecessor calls
// pdl_trigger once all its CTAs are placed); it must call pdl_wait before it
// reads anything the predecessor writes (griddepcontrol.wait returns once the
// predecessor grid has completed and its memory is visible). Captured into a
// graph this is a programmatic edge: the launch latency between the batch's
// kernels overlaps the predecessor's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = std::getenv("FCLSH_NO_PDL") != nullptr; // A/B switch
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    FCLSH_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

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
