// layout_probe.cu -- SoA (identity array + metadata array) vs bucketed (8 ids | 8 metadata
// words per 128-byte line) for the C5 probe's access pattern, before committing to a layout.
// Each position: a random home slot over a 2^30-slot table; an identity walk of L slots
// (L drawn so that hits average ~3 slots), 32-byte sector reads from the home
// to the walk's end; then one 8-byte metadata write at the walk's last slot.
//   layout_probe            -> JSON lines: layout, ms per 4M positions, M positions/s
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}
__device__ __forceinline__ uint64_t ld4(const uint64_t* p) {
    uint64_t a, b, c, d;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    return a ^ b ^ c ^ d;
}

// BUCKET = 0: ident[g], meta[g] separate arrays; 1: line b = g/8 holds ids [0,8) then metas [8,16)
template <int BUCKET, bool WRITE>
__global__ void __launch_bounds__(256, 4) k_walk(uint64_t* ident, uint64_t* meta, uint64_t nslots, uint64_t n,
                                                 uint64_t salt, unsigned long long* sink) {
    uint64_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = mix(i + salt);
        uint64_t g = r % (nslots - 64);
        // walk length: 90% hits (1..5 slots, mean 3), 10% misses (mean ~13)
        const uint32_t u = (uint32_t)(r >> 40);
        const uint32_t L = (u % 10) ? 1 + (u >> 8) % 5 : 1 + (u >> 8) % 25;
        const uint64_t last = g + L - 1;
        for (uint64_t s = g & ~3ull; s <= last; s += 4) {
            const uint64_t* p = BUCKET ? ident + (s >> 3) * 16 + (s & 7) : ident + s;
            acc += ld4(p);
            if (BUCKET && ((s & 7) == 4) && s + 4 <= last) { s += 0; }
        }
        if (WRITE) {
            if (BUCKET) ident[(last >> 3) * 16 + 8 + (last & 7)] = i;
            else meta[last] = i;
        }
    }
    if (acc == 0x12345) atomicAdd(sink, 1ull);
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

int main() {
    const uint64_t nslots = 1ull << 30;
    uint64_t *ident, *meta, *bucket;
    unsigned long long* sink;
    if (cudaMalloc(&ident, nslots * 8) || cudaMalloc(&meta, nslots * 8) || cudaMalloc(&bucket, nslots * 16)) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMalloc(&sink, 8);
    cudaMemset(ident, 1, nslots * 8); cudaMemset(meta, 1, nslots * 8); cudaMemset(bucket, 1, nslots * 16);
    const uint64_t n = 4ull << 20;
    const unsigned grid = 148 * 16;
    float a = timeit([&] { k_walk<0, true><<<grid, 256>>>(ident, meta, nslots, n, 11, sink); }, 10);
    float b = timeit([&] { k_walk<1, true><<<grid, 256>>>(bucket, nullptr, nslots, n, 11, sink); }, 10);
    float c = timeit([&] { k_walk<0, false><<<grid, 256>>>(ident, meta, nslots, n, 11, sink); }, 10);
    float d = timeit([&] { k_walk<1, false><<<grid, 256>>>(bucket, nullptr, nslots, n, 11, sink); }, 10);
    printf("{\"layout\": \"soa\", \"write\": true, \"ms\": %.4f, \"Mpos_s\": %.1f}\n", a, n / a / 1e3);
    printf("{\"layout\": \"bucket8\", \"write\": true, \"ms\": %.4f, \"Mpos_s\": %.1f}\n", b, n / b / 1e3);
    printf("{\"layout\": \"soa\", \"write\": false, \"ms\": %.4f, \"Mpos_s\": %.1f}\n", c, n / c / 1e3);
    printf("{\"layout\": \"bucket8\", \"write\": false, \"ms\": %.4f, \"Mpos_s\": %.1f}\n", d, n / d / 1e3);
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
