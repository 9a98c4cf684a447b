// Random-access ceiling of the B200 HBM: independent random reads of B bytes
// (B = 8, 32, 64, 128) from a buffer much larger than L2, many in flight per
// thread. Gives the accesses/s a probe-bound query kernel can reach (the
// denominator DESIGN.md uses next to the sequential copy peak).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rand_bench rand_bench.cu
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

__device__ __forceinline__ uint4 ld256_lo(const uint4* p, uint4& hi) {
    uint4 lo;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
    return lo;
}

__device__ __forceinline__ uint4 ld_noalloc(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ld256_nc_na(const uint4* p, uint4& hi) {
    uint4 lo;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
    return lo;
}
__device__ __forceinline__ uint4 ld256_cg(const uint4* p, uint4& hi) {
    uint4 lo;
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
    return lo;
}

// WIDE: 4 = 256-bit .nc.L1::no_allocate, 5 = 256-bit .cg; 1 = 32-byte (256-bit) .nc loads, 2 = ld.global.cg (__ldcg: L2 only),
// 3 = ld.global.L1::no_allocate; 0 = __ldg (.nc, 16-byte)
template <int B, int INFLIGHT, int WIDE = 0>
__global__ void k_rand(const uint4* __restrict__ buf, uint64_t units, uint64_t iters, unsigned long long* sink) {
    constexpr int V = B / 16 > 0 ? B / 16 : 1;
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (uint64_t it = 0; it < iters; ++it) {
        uint4 v[INFLIGHT][V];
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k) {
            const uint64_t u = mix(tid * 1315423911ull + it * INFLIGHT + k) % units;
            const uint4* p = buf + u * V;
            if constexpr (WIDE == 1) {
#pragma unroll
                for (int j = 0; j < V; j += 2) v[k][j] = ld256_lo(p + j, v[k][j + 1]);
            } else if constexpr (WIDE == 4) {
#pragma unroll
                for (int j = 0; j < V; j += 2) v[k][j] = ld256_nc_na(p + j, v[k][j + 1]);
            } else if constexpr (WIDE == 5) {
#pragma unroll
                for (int j = 0; j < V; j += 2) v[k][j] = ld256_cg(p + j, v[k][j + 1]);
            } else if constexpr (WIDE == 2) {
#pragma unroll
                for (int j = 0; j < V; ++j) v[k][j] = __ldcg(p + j);
            } else if constexpr (WIDE == 3) {
#pragma unroll
                for (int j = 0; j < V; ++j) v[k][j] = ld_noalloc(p + j);
            } else if constexpr (B == 8) {
                const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
                v[k][0] = make_uint4(x.x, x.y, 0, 0);
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j) v[k][j] = __ldg(p + j);
            }
        }
#pragma unroll
        for (int k = 0; k < INFLIGHT; ++k)
#pragma unroll
            for (int j = 0; j < V; ++j) acc += v[k][j].x ^ v[k][j].w;
    }
    if (acc == 0x12345) atomicAdd(sink, acc);
}

// smem_kb: dynamic shared memory per block (4 blocks per SM), shrinking the
// L1 share of the unified L1/shared array as a probe kernel's working set does
template <int B, int INFLIGHT, int WIDE = 0>
void run(const uint4* buf, uint64_t bytes, unsigned long long* sink, int sms, int smem_kb = 0) {
    const uint64_t units = bytes / (B < 16 ? 16 : B);
    const int threads = 256, blocks = sms * (smem_kb ? 4 : 8);
    const uint64_t iters = 64;
    const size_t smem = size_t(smem_kb) * 1024;
    cudaFuncSetAttribute(k_rand<B, INFLIGHT, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_rand<B, INFLIGHT, WIDE><<<blocks, threads, smem>>>(buf, units, 4, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rand<B, INFLIGHT, WIDE><<<blocks, threads, smem>>>(buf, units, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double acc = double(blocks) * threads * iters * INFLIGHT;
    printf("B=%3d inflight=%d smem=%3dKBx4%s: %.2f G accesses/s, %.0f GB/s useful\n", B, INFLIGHT, smem_kb, WIDE == 1 ? " (256-bit .nc)" : WIDE == 2 ? " (ld.cg)" : WIDE == 3 ? " (L1::no_allocate)" : WIDE == 4 ? " (256 nc.no_allocate)" : WIDE == 5 ? " (256 cg)" : "", acc / ms / 1e6,
           acc * B / ms / 1e6);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t bytes = 32ull << 30;
    uint4* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    // access size and loads in flight per thread (16-byte .nc loads)
    run<8, 4>(buf, bytes, sink, sms);
    run<32, 4>(buf, bytes, sink, sms);
    run<32, 8>(buf, bytes, sink, sms);
    run<64, 4>(buf, bytes, sink, sms);
    run<128, 4>(buf, bytes, sink, sms);
    // load flavour for 32-byte accesses
    run<32, 4, 1>(buf, bytes, sink, sms);
    run<32, 8, 1>(buf, bytes, sink, sms);
    run<32, 16, 1>(buf, bytes, sink, sms);
    run<32, 8, 2>(buf, bytes, sink, sms);
    run<32, 8, 3>(buf, bytes, sink, sms);
    run<32, 8, 4>(buf, bytes, sink, sms);
    run<32, 8, 5>(buf, bytes, sink, sms);
    // shared-memory pressure (4 CTAs of 256 threads per SM)
    for (int kb : {0, 32, 48}) {
        run<32, 8, 1>(buf, bytes, sink, sms, kb);
        run<32, 8, 4>(buf, bytes, sink, sms, kb);
    }
    // L2 fetch granularity (cudaLimitMaxL2FetchGranularity, bytes the L2 fetches per miss)
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("default L2 fetch granularity: %zu B\n", gran);
    for (size_t g : {32, 64}) {
        cudaError_t le = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
        cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
        printf("set %zu -> %s, now %zu B\n", g, cudaGetErrorString(le), gran);
        run<32, 8, 1>(buf, bytes, sink, sms);
        run<32, 8, 4>(buf, bytes, sink, sms);
        run<32, 16, 1>(buf, bytes, sink, sms);
        run<64, 4>(buf, bytes, sink, sms);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
