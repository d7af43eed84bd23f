// Microbenchmarks for the dataflow sweep design (not part of the library):
//  1. dependent-load latency of ld.relaxed.gpu over an L2-resident array
//  2. ping-pong latency between two CTAs on different SMs via st.relaxed.gpu / ld.relaxed.gpu
//  3. same as 1 for plain ld.global (L1 path)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ldr(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(uint64_t* p, uint64_t v) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }

__global__ void chase(const uint64_t* a, int n, int strong, long long* out) {
    uint64_t i = 0;
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) i = strong ? ldr(&a[i]) : a[i];
    long long t1 = clock64();
    out[0] = (t1 - t0) / n; out[1] = (long long)i;
}

__global__ void pingpong(uint64_t* flag, int rounds, long long* out) {
    // block 0 and block 1 alternate: block b waits for value == 2k+b then writes 2k+b+1
    const int b = blockIdx.x;
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    for (int k = 0; k < rounds; ++k) {
        const uint64_t want = 2ull * k + b;
        while (ldr(flag) != want) {}
        str(flag, want + 1);
    }
    long long t1 = clock64();
    if (b == 0) out[2] = (t1 - t0) / rounds;   // one round = two hops
}

int main() {
    const int N = 1 << 22;   // 32 MB of 8-byte slots: L2 resident
    std::vector<uint64_t> h(N);
    // random cyclic permutation with stride to defeat prefetch
    std::vector<uint32_t> perm(N);
    for (int i = 0; i < N; ++i) perm[i] = i;
    uint64_t x = 88172645463325252ull;
    for (int i = N - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = x % (i + 1); std::swap(perm[i], perm[j]); }
    for (int i = 0; i < N; ++i) h[perm[i]] = perm[(i + 1) % N];
    uint64_t* d; long long* o; cudaMalloc(&d, N * 8); cudaMalloc(&o, 64);
    cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
    long long ho[4];
    for (int strong = 0; strong < 2; ++strong) {
        chase<<<1, 1>>>(d, 20000, strong, o);  // warm L2
        chase<<<1, 1>>>(d, 20000, strong, o);
        cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
        printf("dependent load latency (%s): %lld cycles\n", strong ? "ld.relaxed.gpu" : "ld.global", ho[0]);
    }
    cudaMemset(d, 0, 8);
    pingpong<<<2, 32>>>(d, 10000, o);
    cudaDeviceSynchronize();
    cudaMemcpy(ho, o, 32, cudaMemcpyDeviceToHost);
    printf("ping-pong: %lld cycles per round trip (2 hops)\n", ho[2]);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sm clock attr %d kHz; err=%s\n", clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
