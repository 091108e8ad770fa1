// randbench.cu -- random-access ceilings of this B200 for the walk kernel's
// access mix. Each test issues
// independent random accesses from a full grid and reports accesses/s and
// the 32-byte-sector rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randbench randbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

// R random 16-byte loads per thread, U independent streams per thread
template <int U>
__global__ void k_ld16(const uint4* __restrict__ t, uint64_t n, int R, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int r = 0; r < R; r += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(t + mix(tid * 1315423911ull + r + u) % n);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int U>
__global__ void k_ld4(const uint32_t* __restrict__ t, uint64_t n, int R, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int r = 0; r < R; r += U) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(t + mix(tid * 1315423911ull + r + u) % n);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 0x12345678u) *sink = acc;
}

// same through L2 only (ld.global.cg: no L1 allocation)
template <int U>
__global__ void k_ld16cg(const uint4* __restrict__ t, uint64_t n, int R, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int r = 0; r < R; r += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(t + mix(tid * 1315423911ull + r + u) % n);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// PTX load variants (MODE): 0 ld.global.nc, 1 .nc.L1::no_allocate,
// 2 .nc.L2::64B hint, 3 ld.global.cs, 4 ld.relaxed.gpu, 5 .nc with an
// evict_first L2 policy, 6 .nc.L2::256B hint
template <int MODE>
__device__ __forceinline__ uint4 ldv(const uint4* p) {
    uint4 v;
    if (MODE == 0) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 2) asm volatile("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 3) asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 4) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 5) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    }
    if (MODE == 6) asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int MODE>
__global__ void k_ldm(const uint4* __restrict__ t, uint64_t n, int R, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int r = 0; r < R; r += 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldv<MODE>(t + mix(tid * 1315423911ull + r + u) % n);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// sequential control: each thread reads consecutive 16B (coalesced)
__global__ void k_seq(const uint4* __restrict__ t, uint64_t n, uint32_t* sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(t + i);
        acc += v.x ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// chain-table pattern: atomicExch lock + relaxed store release
__global__ void k_lock(uint32_t* t, uint64_t n, int R) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (int r = 0; r < R; ++r) {
        uint32_t* p = t + mix(tid * 1315423911ull + r) % n;
        const uint32_t e = atomicExch(p, 0xFFFFFFFDu);
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(e + 1) : "memory");
    }
}

// dependent chain: each load's address depends on the previous value
__global__ void k_chase(const uint4* __restrict__ t, uint64_t n, int R, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t i = mix(tid) % n;
    uint32_t acc = 0;
    for (int r = 0; r < R; ++r) {
        const uint4 v = __ldg(t + i);
        acc += v.x;
        i = mix(i + v.y + r) % n;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char** argv) {
    if (argc > 1) {
        const size_t g = (size_t)atoi(argv[1]);
        CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("max L2 fetch granularity: %zu\n", got);
    }
    const uint64_t bytes = 1ull << 30;  // 1 GiB table (8x L2)
    void* buf; uint32_t* sink;
    CK(cudaMalloc(&buf, bytes)); CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, bytes));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int R = 256;
    if (argc > 2) {  // load-variant sweep (for ncu)
        const int blocks = sms * 4, thr = 256;
        const double acc = (double)blocks * thr * R;
        float ms;
#define RUNM(M) ms = timeit([&] { k_ldm<M><<<blocks, thr>>>((const uint4*)buf, bytes / 16, R, sink); }); \
        printf("mode %d: %7.2f G acc/s\n", M, acc / ms / 1e6);
        RUNM(0) RUNM(1) RUNM(2) RUNM(3) RUNM(4) RUNM(5) RUNM(6)
        ms = timeit([&] { k_seq<<<sms * 8, 256>>>((const uint4*)buf, bytes / 16, sink); });
        printf("seq: %7.1f GB/s\n", bytes / ms / 1e6);
        return 0;
    }
    for (int bpsm : {4, 16}) {
        const int blocks = sms * bpsm, thr = 256;
        const double acc = (double)blocks * thr * R;
        float ms = timeit([&] { k_ld16<4><<<blocks, thr>>>((const uint4*)buf, bytes / 16, R, sink); });
        printf("ld16  1GiB   blocks/SM %2d: %7.2f G acc/s  %7.1f GB/s useful  (%.3f ms)\n", bpsm, acc / ms / 1e6, acc * 16 / ms / 1e6, ms);
        ms = timeit([&] { k_ld16cg<4><<<blocks, thr>>>((const uint4*)buf, bytes / 16, R, sink); });
        printf("ld16cg 1GiB  blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / ms / 1e6);
        ms = timeit([&] { k_ld16<4><<<blocks, thr>>>((const uint4*)buf, (128ull << 20) / 16, R, sink); });
        printf("ld16  128MiB blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / ms / 1e6);
        ms = timeit([&] { k_ld4<4><<<blocks, thr>>>((const uint32_t*)buf, bytes / 4, R, sink); });
        printf("ld4   1GiB   blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / ms / 1e6);
        ms = timeit([&] { k_lock<<<blocks, thr>>>((uint32_t*)buf, (128ull << 20) / 4, R); });
        printf("lock  128MiB blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / ms / 1e6);
        ms = timeit([&] { k_lock<<<blocks, thr>>>((uint32_t*)buf, bytes / 4, R); });
        printf("lock  1GiB   blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / ms / 1e6);
        ms = timeit([&] { k_chase<<<blocks, thr>>>((const uint4*)buf, bytes / 16, R / 4, sink); });
        printf("chase 1GiB   blocks/SM %2d: %7.2f G acc/s\n", bpsm, acc / 4 / ms / 1e6);
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
