// updbench.cu -- cost breakdown of the estimator pass (not product code): the state stream alone, plus
// Philox + the two bounded draws, on 1M estimators, timed with CUDA events after warm-up.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_1308_2166_b200/csrc/philox.cuh"

using namespace tcb;

// (a) read r1, cf, r2, p1, p2; write them back (28 + 28 B)
__global__ void __launch_bounds__(256, 4) k_stream(uint2 *r1, uint2 *r2, uint32_t *cf, uint32_t *p1, uint32_t *p2, uint32_t n) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        uint2 a = __ldcs(r1 + t), b = __ldcs(r2 + t);
        uint32_t c = __ldcs(cf + t), x = __ldcs(p1 + t), y = __ldcs(p2 + t);
        __stcs(r1 + t, make_uint2(a.y, a.x));
        __stcs(r2 + t, make_uint2(b.y, b.x));
        __stcs(cf + t, c + 1);
        __stcs(p1 + t, x + 1);
        __stcs(p2 + t, y + 1);
    }
}

// (b) the same plus one Philox4x32-10 block and two Lemire draws per estimator
__global__ void __launch_bounds__(256, 4) k_philox(uint2 *r1, uint2 *r2, uint32_t *cf, uint32_t *p1, uint32_t *p2, uint32_t n,
                                                   uint64_t seed, uint32_t batch, uint64_t m) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        uint2 a = __ldcs(r1 + t), b = __ldcs(r2 + t);
        uint32_t c = __ldcs(cf + t), x = __ldcs(p1 + t), y = __ldcs(p2 + t);
        const DrawCtx dc{t, batch, PhiloxKey{(uint32_t)seed, (uint32_t)(seed >> 32)}};
        const uint4 o = philox4x32_10(make_uint4(t, 0u, batch, 0u), dc.key);
        const uint64_t d1 = bounded(m, (uint64_t)o.x | ((uint64_t)o.y << 32), dc, 0x10000u);
        const uint64_t d2 = bounded(c + 7, (uint64_t)o.z | ((uint64_t)o.w << 32), dc, 0x20000u);
        __stcs(r1 + t, make_uint2(a.y, a.x ^ (uint32_t)d1));
        __stcs(r2 + t, make_uint2(b.y, b.x));
        __stcs(cf + t, c + (uint32_t)d2);
        __stcs(p1 + t, x + 1);
        __stcs(p2 + t, y + 1);
    }
}

int main() {
    const uint32_t n = 1u << 20;
    uint2 *r1, *r2;
    uint32_t *cf, *p1, *p2;
    cudaMalloc(&r1, 8ull * n);
    cudaMalloc(&r2, 8ull * n);
    cudaMalloc(&cf, 4ull * n);
    cudaMalloc(&p1, 4ull * n);
    cudaMalloc(&p2, 4ull * n);
    cudaMemset(r1, 0, 8ull * n);
    cudaMemset(r2, 0, 8ull * n);
    cudaMemset(cf, 0, 4ull * n);
    cudaMemset(p1, 0, 4ull * n);
    cudaMemset(p2, 0, 4ull * n);
    char *fl;
    cudaMalloc(&fl, 512ull << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid : {sms * 4, sms * 8, (int)(n / 256)}) {
        for (int which = 0; which < 2; ++which) {
            float best = 1e9f;
            for (int rep = 0; rep < 6; ++rep) {
                cudaMemset(fl, rep, 512ull << 20);  // flush L2
                cudaEventRecord(e0);
                if (which == 0) k_stream<<<grid, 256>>>(r1, r2, cf, p1, p2, n);
                else k_philox<<<grid, 256>>>(r1, r2, cf, p1, p2, n, 42, 3, 5000000);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep && ms < best) best = ms;
            }
            printf("grid %6d %-16s %8.2f us  (%.0f GB/s of 56 B/estimator)\n", grid, which ? "state+philox" : "state stream",
                   best * 1e3, 56.0 * n / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
