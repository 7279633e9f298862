// sector_probe.cu -- where do the bytes of a random 32-byte read go?  Random sector reads over
// an array of G GiB with several load flavours; run plain for timings, under ncu for
// dram__sectors_read.sum vs the sectors asked for (DRAM over-fetch per random access).
//   sector_probe <gib> [reps]
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int FL>
__device__ __forceinline__ void ld4(const uint64_t* p, uint64_t (&v)[4]) {
    if (FL == 0) asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 1) asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 2) asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 3) asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 4) asm volatile("ld.global.cg.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 5) asm volatile("ld.global.cv.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
    if (FL == 6) asm volatile("ld.global.cg.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}

// nsec is a power of two: mask, no 64-bit modulo in the address path
template <int FL, int U>
__global__ void __launch_bounds__(256) k_rd(const uint64_t* __restrict__ a, uint64_t mask, uint64_t n,
                                            uint64_t salt, unsigned long long* sink) {
    uint64_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * U; b < n; b += stride) {
        uint64_t v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) ld4<FL>(a + 4 * (mix(b + u + salt) & mask), v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
    }
    if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

// warp-cooperative: 8 lanes x 4 B?  no -- 4 lanes each load 8 B of one sector (scalar loads)
template <int U>
__global__ void __launch_bounds__(256) k_rd_quad(const uint64_t* __restrict__ a, uint64_t mask, uint64_t n,
                                                 uint64_t salt, unsigned long long* sink) {
    uint64_t acc = 0;
    const unsigned q = threadIdx.x & 3;
    const uint64_t tq = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 2;
    const uint64_t nq = ((uint64_t)gridDim.x * blockDim.x) >> 2;
    for (uint64_t b = tq * U; b < n; b += nq * U) {
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(a + 4 * (mix(b + u + salt) & mask) + q);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

__global__ void __launch_bounds__(256) k_w8(uint64_t* a, uint64_t mask, uint64_t n, uint64_t salt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[4 * (mix(i + salt) & mask) + 1] = i;
}
__global__ void __launch_bounds__(256) k_w32(uint64_t* a, uint64_t mask, uint64_t n, uint64_t salt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t* p = a + 4 * (mix(i + salt) & mask);
        asm volatile("st.global.v4.u64 [%0], {%1,%1,%1,%1};" ::"l"(p), "l"(i) : "memory");
    }
}


// L lanes cooperate on one random access: lane j of the group loads sector j of a random
// 128-byte-aligned line (one warp instruction covers 32/L lines, L sectors each)
template <int L, int U>
__global__ void __launch_bounds__(256) k_rd_line(const uint64_t* __restrict__ a, uint64_t lmask, uint64_t n,
                                                 uint64_t salt, unsigned long long* sink) {
    uint64_t acc = 0;
    const unsigned j = threadIdx.x % L;
    const uint64_t tq = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
    const uint64_t nq = ((uint64_t)gridDim.x * blockDim.x) / L;
    for (uint64_t b = tq * U; b < n; b += nq * U) {
        uint64_t v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) ld4<2>(a + 16 * (mix(b + u + salt) & lmask) + 4 * j, v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
    }
    if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

template <class F>
float timeit(F f, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    f();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

int main(int argc, char** argv) {
    const int gib = argc > 1 ? atoi(argv[1]) : 16;
    const int reps = argc > 2 ? atoi(argv[2]) : 5;
    const uint64_t bytes = (uint64_t)gib << 30;
    uint64_t* a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 1, bytes);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    const uint64_t n = 16ull << 20;
    const uint64_t mask = bytes / 32 - 1;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = sms * 8;
#define R(NAME, LAUNCH) { float ms = timeit([&] { LAUNCH; }, reps); \
    printf("{\"gib\": %d, \"kernel\": \"%s\", \"ms\": %.4f, \"G_sectors_s\": %.2f, \"useful_gbs\": %.1f}\n", gib, NAME, ms, n / ms / 1e6, n * 32.0 / ms / 1e6); }
    R("default_u4", (k_rd<0, 4><<<grid, 256>>>(a, mask, n, 1, sink)));
    R("nc_u4", (k_rd<1, 4><<<grid, 256>>>(a, mask, n, 2, sink)));
    R("cg_u4", (k_rd<2, 4><<<grid, 256>>>(a, mask, n, 3, sink)));
    R("cg_u8", (k_rd<2, 8><<<grid, 256>>>(a, mask, n, 4, sink)));
    R("l1noalloc_u4", (k_rd<3, 4><<<grid, 256>>>(a, mask, n, 5, sink)));
    R("cg_L2_64B_u4", (k_rd<4, 4><<<grid, 256>>>(a, mask, n, 6, sink)));
    R("cv_u4", (k_rd<5, 4><<<grid, 256>>>(a, mask, n, 7, sink)));
    R("cg_evict_first_u4", (k_rd<6, 4><<<grid, 256>>>(a, mask, n, 8, sink)));
    R("quad_scalar_u4", (k_rd_quad<4><<<grid, 256>>>(a, mask, n, 9, sink)));
    R("write8", (k_w8<<<grid, 256>>>(a, mask, n, 10)));
    R("write32", (k_w32<<<grid, 256>>>(a, mask, n, 11)));
    {
        const uint64_t lmask = bytes / 128 - 1;
#define RL(NAME, L, LAUNCH) { float ms = timeit([&] { LAUNCH; }, reps); \
    printf("{\"gib\": %d, \"kernel\": \"%s\", \"ms\": %.4f, \"G_accesses_s\": %.2f, \"useful_gbs\": %.1f}\n", gib, NAME, ms, n / ms / 1e6, n * 32.0 * L / ms / 1e6); }
        RL("line_1lane_32B", 1, (k_rd_line<1, 4><<<grid, 256>>>(a, lmask, n, 21, sink)));
        RL("line_2lanes_64B", 2, (k_rd_line<2, 4><<<grid, 256>>>(a, lmask, n, 22, sink)));
        RL("line_4lanes_128B", 4, (k_rd_line<4, 4><<<grid, 256>>>(a, lmask, n, 23, sink)));
        RL("line_4lanes_128B_u8", 4, (k_rd_line<4, 8><<<grid, 256>>>(a, lmask, n, 24, sink)));
        RL("line_2lanes_64B_u8", 2, (k_rd_line<2, 8><<<grid, 256>>>(a, lmask, n, 25, sink)));
    }
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_gran_now\": %zu}\n", cur);
    R("gran32_cg_u4", (k_rd<2, 4><<<grid, 256>>>(a, mask, n, 12, sink)));
    R("gran32_write8", (k_w8<<<grid, 256>>>(a, mask, n, 13)));
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
