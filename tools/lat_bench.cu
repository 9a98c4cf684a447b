// Latency of dependent random 32-byte reads against the span they hit
// (TLB reach): W warps, lane 0 of each chasing a chain of dependent reads
// over the first S bytes of one large buffer. Unloaded (1 warp) and loaded
// (many warps, each with its own chain) latencies per access.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lat_bench lat_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__global__ void k_fill(uint64_t* b, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = mix(i);
}

template <int CHAINS>
__global__ void k_chase(const uint64_t* __restrict__ b, uint64_t units, int steps, unsigned long long* out) {
    if ((threadIdx.x & 31) >= CHAINS) return;
    uint64_t x = mix(blockIdx.x * 1000003ull + threadIdx.x);
    for (int s = 0; s < steps; ++s) {
        const uint64_t u = mix(x + s) % units; // 32-byte unit
        uint64_t v;
        asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(b + u * 4));
        x ^= v;
    }
    if (x == 42) out[0] = x;
}

__global__ void k_flush(uint64_t* f, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        f[i] = i;
}

// one load per page of the span (page = 1 << pshift bytes)
__global__ void k_touch(const uint64_t* __restrict__ b, uint64_t pages, int pshift, unsigned long long* out) {
    uint64_t x = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pages; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t v;
        asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(b + ((i << pshift) >> 3)));
        x ^= v;
    }
    if (x == 42) out[0] = x;
}

int main() {
    const uint64_t total = 128ull << 30;
    uint64_t* b = nullptr;
    if (cudaMalloc(&b, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    k_fill<<<148 * 8, 256>>>(b, total / 8);
    unsigned long long* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 2000;
    for (uint64_t span : {64ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 16ull << 30, 34ull << 30, 64ull << 30,
                          128ull << 30}) {
        for (int warps : {1, 148, 148 * 16, 148 * 48}) {
            const int blocks = warps < 8 ? 1 : warps / 8, threads = warps < 8 ? 32 * warps : 256;
            k_chase<1><<<blocks, threads>>>(b, span / 32, 20, out);
            cudaEventRecord(e0);
            k_chase<1><<<blocks, threads>>>(b, span / 32, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double per = ms * 1e3 / steps;
            printf("span %7.2f GB  warps %5d: %7.3f us per dependent read, %6.2f G reads/s\n", span / 1073741824.0,
                   warps, per, warps / per / 1e3);
        }
    }
    // after an L2 flush (256 MiB written): the first dependent reads of a chain
    uint64_t* fl = nullptr;
    cudaMalloc(&fl, 256ull << 20);
    for (uint64_t span : {256ull << 20, 4ull << 30, 34ull << 30, 128ull << 30}) {
        for (int warps : {1, 148 * 8}) {
            for (int st : {10, 100}) {
                const int blocks = warps < 8 ? 1 : warps / 8, threads = warps < 8 ? 32 * warps : 256;
                k_flush<<<148 * 4, 256>>>(fl, (256ull << 20) / 8);
                cudaEventRecord(e0);
                k_chase<1><<<blocks, threads>>>(b, span / 32, st, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("after flush: span %7.2f GB warps %5d steps %4d: %7.3f us per dependent read\n",
                       span / 1073741824.0, warps, st, ms * 1e3 / st);
            }
        }
    }
    // touch every 2 MB (or 64 KB) page after a flush, then the chase
    for (uint64_t span : {34ull << 30, 128ull << 30}) {
        for (int ps : {21, 16}) {
            const uint64_t pages = span >> ps;
            k_flush<<<148 * 4, 256>>>(fl, (256ull << 20) / 8);
            cudaEventRecord(e0);
            k_touch<<<unsigned((pages + 255) / 256 < 148 * 8 ? (pages + 255) / 256 : 148 * 8), 256>>>(b, pages, ps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaEventRecord(e0);
            k_chase<1><<<148, 256>>>(b, span / 32, 10, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms2 = 0;
            cudaEventElapsedTime(&ms2, e0, e1);
            printf("touch %6llu pages of %d KB over %6.1f GB: %7.1f us; then 1184 warps x 10 dependent reads: %6.3f us per read\n",
                   (unsigned long long)pages, 1 << (ps - 10), span / 1073741824.0, ms * 1e3, ms2 * 1e3 / 10);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
