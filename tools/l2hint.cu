// l2hint.cu -- can L2 eviction-priority hints keep a small randomly probed table resident while a large one
// streams random misses through L2?  (calibration for k_update's probe mix; not product code)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

__device__ __forceinline__ uint4 ld_pol(const uint4 *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

// HOT / COLD: 0 default __ldg, 1 evict_last policy, 2 evict_first policy
template <int HOT, int COLD>
__global__ void k_mix(const uint4 *hot, uint32_t nhot, const uint4 *cold, uint32_t ncold, uint32_t n, uint32_t *out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t pl, pf;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    const uint4 *ph = hot + hsh(i) % nhot, *pc = cold + hsh(i ^ 0x9e3779b9u) % ncold;
    uint4 a = HOT == 0 ? __ldg(ph) : ld_pol(ph, HOT == 1 ? pl : pf);
    uint4 b = COLD == 0 ? __ldg(pc) : ld_pol(pc, COLD == 1 ? pl : pf);
    if ((a.x ^ b.y) == 0x12345678u) out[0] = 1;
}

__global__ void k_stream(const uint4 *a, uint4 *b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) b[i] = __ldcs(a + i);
}

int main(int argc, char **argv) {
    const uint64_t hb = (argc > 1 ? strtoull(argv[1], 0, 0) : 32ull << 20), cb = 1ull << 30;
    const uint32_t n = 1u << 25;
    uint4 *hot, *cold, *s1, *s2;
    uint32_t *out;
    cudaMalloc(&hot, hb);
    cudaMalloc(&cold, cb);
    cudaMemset(hot, 1, hb);
    cudaMemset(cold, 1, cb);
    cudaMalloc(&out, 4);
    const uint64_t sb = 512ull << 20;
    cudaMalloc(&s1, sb);
    cudaMalloc(&s2, sb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto f) {
        k_stream<<<148 * 8, 256>>>(s1, s2, sb / 16);
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-14s hot %4.0f MB: %8.1f us  %6.2f G pairs/s\n", name, hb / 1048576.0, ms * 1e3, n / (ms * 1e-3) / 1e9);
    };
    const uint32_t gr = n / 256, nh = hb / 16, nc = cb / 16;
    run("default", [&] { k_mix<0, 0><<<gr, 256>>>(hot, nh, cold, nc, n, out); });
    run("hot_last", [&] { k_mix<1, 0><<<gr, 256>>>(hot, nh, cold, nc, n, out); });
    run("cold_first", [&] { k_mix<0, 2><<<gr, 256>>>(hot, nh, cold, nc, n, out); });
    run("last+first", [&] { k_mix<1, 2><<<gr, 256>>>(hot, nh, cold, nc, n, out); });
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
