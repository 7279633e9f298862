// sector_bench.cu -- random-sector ceiling calibration on one B200 ("calibrate a
// random-sector ceiling ... so the gap between the layout and the memory system is visible").
// Uniform random 32/64/128-byte reads over a >= 16 GiB array with several load flavours and
// L2 fetch-granularity limits; plus random 8-byte writes (metadata-word pattern).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int FLAVOR, int U, int BYTES>
__global__ void __launch_bounds__(256) k_read(const uint64_t* __restrict__ a, uint64_t nsec, uint64_t n, uint64_t salt,
                                              unsigned long long* sink) {
    uint64_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * U; base < n; base += stride) {
        uint64_t v[U][BYTES / 8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t s = mix(base + u + salt) % nsec;  // sector-of-BYTES index
            const uint64_t* p = a + s * (BYTES / 8);
#pragma unroll
            for (int q = 0; q < BYTES / 32; ++q) {
                const uint64_t* pq = p + 4 * q;
                if (FLAVOR == 0)
                    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[u][4*q]), "=l"(v[u][4*q+1]), "=l"(v[u][4*q+2]), "=l"(v[u][4*q+3]) : "l"(pq));
                else if (FLAVOR == 1)
                    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[u][4*q]), "=l"(v[u][4*q+1]), "=l"(v[u][4*q+2]), "=l"(v[u][4*q+3]) : "l"(pq));
                else if (FLAVOR == 2)
                    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[u][4*q]), "=l"(v[u][4*q+1]), "=l"(v[u][4*q+2]), "=l"(v[u][4*q+3]) : "l"(pq));
                else
                    asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[u][4*q]), "=l"(v[u][4*q+1]), "=l"(v[u][4*q+2]), "=l"(v[u][4*q+3]) : "l"(pq));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < BYTES / 8; ++q) acc += v[u][q];
    }
    if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

// read one random 32-byte sector and write 8 bytes at: MODE 0 the same sector, MODE 1 the
// other sector of the same 64-byte pair, MODE 2 an unrelated random sector (SoA metadata),
// MODE 3 a sector of the other 64-byte half of the same 128-byte line
template <int MODE>
__global__ void __launch_bounds__(256) k_read_write(uint64_t* a, uint64_t nsec, uint64_t n, uint64_t salt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = mix(i + salt) % nsec;
        uint64_t w0, w1, w2, w3;
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(a + 4 * s));
        uint64_t t;
        if (MODE == 0) t = 4 * s + 1;
        else if (MODE == 1) t = 4 * (s ^ 1) + 1;
        else if (MODE == 3) t = 4 * (s ^ 2) + 1;
        else t = 4 * (mix(i + salt + 999) % nsec) + 1;
        a[t] = w0 + w1 + w2 + w3;
    }
}

__global__ void __launch_bounds__(256) k_write8(uint64_t* a, uint64_t nslots, uint64_t n, uint64_t salt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[mix(i + salt) % nslots] = i;
}

// the row reset's store pattern: a warp writes one random 512-byte row of each of two arrays
// (weights, momentum) per step; HINT 1 uses streaming (.cs) stores, HINT 2 sequential rows
template <int HINT>
__global__ void __launch_bounds__(256) k_write_rows(float4* a, float4* b, uint64_t nrows, uint64_t n, uint64_t salt) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < n; i += nw) {
        const uint64_t r = HINT == 2 ? i % nrows : mix(i + salt) % nrows;
        const float4 v = make_float4((float)i, 1.f, 2.f, 3.f), z = make_float4(0.f, 0.f, 0.f, 0.f);
        if (HINT == 1) {
            __stcs(a + r * 32 + lane, v);
            __stcs(b + r * 32 + lane, z);
        } else {
            a[r * 32 + lane] = v;
            b[r * 32 + lane] = z;
        }
    }
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
    const uint64_t bytes = 16ull << 30;
    uint64_t* a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 1, bytes);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    const uint64_t n = 16ull << 20;  // 16M random accesses per launch
    int dev; cudaGetDevice(&dev);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    printf("{\"device_sms\": %d, \"array_gib\": 16, \"accesses_per_launch\": %llu, \"results\": [\n", sms, (unsigned long long)n);
    bool first = true;
    for (int gran : {0, 128}) {
        if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
#define RUN(FL, U, B, NAME) { \
            const uint64_t nsec = bytes / B; \
            const unsigned grid = sms * 8; \
            float ms = timeit([&] { k_read<FL, U, B><<<grid, 256>>>(a, nsec, n, 12345, sink); }, 5); \
            printf("%s{\"op\": \"read\", \"flavor\": \"%s\", \"unroll\": %d, \"bytes\": %d, \"l2_fetch_gran\": %zu, \"ms\": %.4f, \"useful_gbs\": %.1f, \"maccess_s\": %.1f}\n", first ? "" : ",", NAME, U, B, cur, ms, n * (double)B / ms / 1e6, n / ms / 1e3); first = false; }
        RUN(0, 1, 32, "default") RUN(0, 4, 32, "default") RUN(1, 4, 32, "nc") RUN(2, 1, 32, "cg") RUN(2, 4, 32, "cg")
        RUN(2, 8, 32, "cg") RUN(3, 4, 32, "cs") RUN(2, 4, 64, "cg") RUN(2, 2, 128, "cg") RUN(0, 4, 64, "default")
        for (int mode = 0; mode < 4; ++mode) {
            const uint64_t nsec = bytes / 32;
            float ms = timeit([&] {
                if (mode == 0) k_read_write<0><<<sms * 8, 256>>>(a, nsec, n, 4242);
                else if (mode == 1) k_read_write<1><<<sms * 8, 256>>>(a, nsec, n, 4242);
                else if (mode == 2) k_read_write<2><<<sms * 8, 256>>>(a, nsec, n, 4242);
                else k_read_write<3><<<sms * 8, 256>>>(a, nsec, n, 4242);
            }, 5);
            const char* nm[4] = {"read32+write8_same_sector", "read32+write8_pair_sector", "read32+write8_random_sector",
                                 "read32+write8_same_line_other_half"};
            printf(",{\"op\": \"%s\", \"l2_fetch_gran\": %zu, \"ms\": %.4f, \"maccess_s\": %.1f}\n", nm[mode], cur, ms, n / ms / 1e3);
        }
        {
            float ms = timeit([&] { k_write8<<<sms * 8, 256>>>(a, bytes / 8, n, 777); }, 5);
            printf(",{\"op\": \"write8\", \"l2_fetch_gran\": %zu, \"ms\": %.4f, \"useful_gbs\": %.1f, \"maccess_s\": %.1f}\n", cur, ms, n * 8.0 / ms / 1e6, n / ms / 1e3);
        }
    }
    {   // two 8 GiB arrays of 512-byte rows, 1 M rows written per launch (1 GiB)
        float4* a4 = reinterpret_cast<float4*>(a);
        float4* b4 = reinterpret_cast<float4*>(reinterpret_cast<char*>(a) + (8ull << 30));
        const uint64_t nrows = (8ull << 30) / 512, nw = 1ull << 20;
        const char* nm[3] = {"write_rows512_x2_random", "write_rows512_x2_random_cs", "write_rows512_x2_sequential"};
        for (int h = 0; h < 3; ++h) {
            float ms = timeit([&] {
                if (h == 0) k_write_rows<0><<<sms * 8, 256>>>(a4, b4, nrows, nw, 99);
                else if (h == 1) k_write_rows<1><<<sms * 8, 256>>>(a4, b4, nrows, nw, 99);
                else k_write_rows<2><<<sms * 8, 256>>>(a4, b4, nrows, nw, 99);
            }, 5);
            printf(",{\"op\": \"%s\", \"ms\": %.4f, \"gbs\": %.1f}\n", nm[h], ms, nw * 1024.0 / ms / 1e6);
        }
    }
    printf("]}\n");
    return 0;
}
