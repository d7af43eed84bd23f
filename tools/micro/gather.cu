// Random-gather throughput microbenchmark (not part of the library): E random
// 8/16-byte loads from an L2-resident array of N 32-byte records, indices in
// a sliding window like the C4 graph (predecessors in the previous 5 levels).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void ldr2(const uint64_t* p, uint64_t& a, uint64_t& b) { asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory"); }
__device__ __forceinline__ uint64_t ldr1(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

template <int MODE>
__global__ void gather(const uint64_t* rec, const int* idx, int E, unsigned long long* out) {
    uint64_t acc = 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const int i = __ldg(&idx[e]);
        if (MODE == 0) { uint64_t a, b; ldr2(&rec[4 * (size_t)i], a, b); acc += a ^ b; }
        if (MODE == 1) { acc += ldr1(&rec[4 * (size_t)i]); }
        if (MODE == 2) { acc += __ldg(&rec[4 * (size_t)i]); }
        if (MODE == 3) { acc += __ldg(&rec[(size_t)i]); }   // dense 8-byte records
    }
    if (acc == 42) out[0] = acc;
}

int main() {
    const int N = 1500000, E = 9200000, W = 94000;
    std::vector<int> h(E);
    uint64_t x = 88172645463325252ull;
    for (int e = 0; e < E; ++e) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int base = (int)((long long)e * N / E); int lo = base > W ? base - W : 0; h[e] = lo + (int)(x % (uint64_t)(base - lo + 1)); if (h[e] >= N) h[e] = N - 1; }
    uint64_t* rec; int* idx; unsigned long long* o;
    cudaMalloc(&rec, (size_t)N * 32); cudaMalloc(&idx, (size_t)E * 4); cudaMalloc(&o, 8);
    cudaMemset(rec, 1, (size_t)N * 32);
    cudaMemcpy(idx, h.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"16B ld.relaxed.gpu.v2 (32B recs)", "8B ld.relaxed.gpu (32B recs)", "8B ldg (32B recs)", "8B ldg (8B recs)"};
    for (int mode = 0; mode < 4; ++mode)
      for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) gather<0><<<blocks, 256>>>(rec, idx, E, o);
            if (mode == 1) gather<1><<<blocks, 256>>>(rec, idx, E, o);
            if (mode == 2) gather<2><<<blocks, 256>>>(rec, idx, E, o);
            if (mode == 3) gather<3><<<blocks, 256>>>(rec, idx, E, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%-36s blocks=%5d: %8.1f us  (%.2f G gathers/s)\n", names[mode], blocks, best * 1e3, E / (best * 1e-3) / 1e9);
      }
    return 0;
}
