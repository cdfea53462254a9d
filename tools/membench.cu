// membench.cu -- calibration microbenchmarks for random-access costs on the B200 (not product code).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

__global__ void k_rand_load(const uint4* t, uint32_t mask, uint32_t n, uint32_t* out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    uint4 v = __ldg(t + (hsh(i) & mask)); if (v.x == 12345) out[0] = v.y;
}
__global__ void k_rand_load_chain(const uint4* t, uint32_t mask, uint32_t n, uint32_t depth, uint32_t* out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    uint32_t h = hsh(i);
    for (uint32_t d = 0; d < depth; ++d) { uint4 v = __ldg(t + (h & mask)); h = hsh(h ^ v.x); }
    if (h == 12345) out[0] = h;
}
__global__ void k_rand_cas(unsigned long long* t, uint32_t mask, uint32_t n, uint32_t* out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    unsigned long long o = atomicCAS(t + 2 * (hsh(i) & mask), ~0ull, (unsigned long long)i);
    if (o == 12345) out[0] = 1;
}
__global__ void k_rand_cas128(unsigned __int128* t, uint32_t mask, uint32_t n, uint32_t* out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    unsigned __int128 o = atomicCAS(t + (hsh(i) & mask), (unsigned __int128)0, (unsigned __int128)i);
    if ((unsigned long long)o == 12345) out[0] = 1;
}
__global__ void k_rand_store8(unsigned long long* t, uint32_t mask, uint32_t n) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    t[2 * (hsh(i) & mask)] = i;
}
__global__ void k_rand_store16(uint4* t, uint32_t mask, uint32_t n) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    t[hsh(i) & mask] = make_uint4(i, i, i, i);
}
__global__ void k_rand_atomicadd(uint32_t* t, uint32_t mask, uint32_t n) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    atomicAdd(t + 4 * (hsh(i) & mask), 1u);
}
__global__ void k_copy(const uint4* a, uint4* b, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_empty() {}

int main() {
    const size_t TB = 64ull << 20;  // 64 MiB table
    uint4 *t, *t2; uint32_t* out; char* fl;
    cudaMalloc(&t, TB); cudaMalloc(&t2, TB); cudaMalloc(&out, 64); cudaMalloc(&fl, 512ull << 20);
    cudaMemset(t, 0, TB);
    const uint32_t mask = (uint32_t)(TB / 16 - 1);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto flush = [&]() { cudaMemset(fl, 1, 512ull << 20); cudaDeviceSynchronize(); };
    auto run = [&](const char* name, auto launch, bool cold, double units, const char* uname) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            if (cold) flush(); else { launch(); cudaDeviceSynchronize(); }
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("%-34s %-5s %9.2f us  %8.2f G%s/s\n", name, cold ? "cold" : "warm", best * 1e3, units / best / 1e6, uname);
    };
    for (uint32_t n : {1u << 20, 1u << 21, 1u << 23}) {
        printf("--- n = %u threads, table 64 MiB\n", n);
        dim3 g((n + 255) / 256), b(256);
        for (bool cold : {true, false}) {
            run("rand 16B load", [&] { k_rand_load<<<g, b>>>(t, mask, n, out); }, cold, n, "op");
            run("rand 16B load chain x4", [&] { k_rand_load_chain<<<g, b>>>(t, mask, n, 4, out); }, cold, 4.0 * n, "op");
            run("rand CAS64", [&] { k_rand_cas<<<g, b>>>((unsigned long long*)t, mask, n, out); }, cold, n, "op");
            run("rand CAS128", [&] { k_rand_cas128<<<g, b>>>((unsigned __int128*)t, mask, n, out); }, cold, n, "op");
            run("rand store 8B", [&] { k_rand_store8<<<g, b>>>((unsigned long long*)t, mask, n); }, cold, n, "op");
            run("rand store 16B", [&] { k_rand_store16<<<g, b>>>(t, mask, n); }, cold, n, "op");
            run("rand atomicAdd 4B", [&] { k_rand_atomicadd<<<g, b>>>((uint32_t*)t, mask, n); }, cold, n, "op");
        }
    }
    run("copy 64MiB (r+w bytes)", [&] { k_copy<<<148 * 8, 256>>>(t, t2, (uint32_t)(TB / 16)); }, true, 2.0 * TB / 1e3, "B");
    run("empty kernel", [&] { k_empty<<<1, 32>>>(); }, false, 1, "launch");
    return 0;
}
