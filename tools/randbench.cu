// randbench.cu -- DRAM cost of one random read on the B200 (calibration, not product code).
// N random reads of 16 / 32 bytes (aligned) from a table of `tbytes`, with each load flavour; run under
//   ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum
// to get DRAM bytes per access, and without ncu for the access rate.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

template <int K>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
    uint4 v;
    if (K == 0) v = __ldg(p);
    else if (K == 1) v = __ldcg(p);
    else if (K == 2) v = __ldcs(p);
    else if (K == 3) v = __ldca(p);
    else if (K == 4) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (K == 5) v = __ldlu(p);
    else if (K == 6) v = __ldcv(p);
    else if (K == 7) asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (K == 8) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int K, int W>  // W uint4 words per access
__global__ void k_read(const uint4 *t, uint64_t nacc_tbl, uint32_t n, uint32_t *out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t h = ((uint64_t)hsh(i) << 32 | hsh(i ^ 0x5bd1e995u)) % nacc_tbl;
    const uint4 *p = t + h * W;
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) { uint4 v = ld<K>(p + k); acc ^= v.x ^ v.w; }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_stream(const uint4 *a, uint4 *b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) b[i] = __ldcs(a + i);
}

int main(int argc, char **argv) {
    const uint64_t tbytes = (argc > 1 ? strtoull(argv[1], 0, 0) : 1ull << 30);
    const int gran = argc > 2 ? atoi(argv[2]) : 0;
    if (gran) printf("cudaLimitMaxL2FetchGranularity %d: %s\n", gran, cudaGetErrorString(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran)));
    const uint32_t n = 1u << 24;
    uint4 *t;
    uint32_t *out;
    cudaMalloc(&t, tbytes);
    cudaMemset(t, 1, tbytes);
    cudaMalloc(&out, 4);
    uint4 *s1, *s2;
    const uint64_t sb = 512ull << 20;
    cudaMalloc(&s1, sb);
    cudaMalloc(&s2, sb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto flush = [&] { k_stream<<<148 * 8, 256>>>(s1, s2, sb / 16); };
    auto timeit = [&](const char *name, auto f, double bytes_per) {
        for (int rep = 0; rep < 2; ++rep) {
            flush();
            cudaEventRecord(e0);
            f();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 1) printf("%-10s table %6.0f MB: %8.1f us  %7.2f G acc/s  %7.1f GB/s useful\n", name, tbytes / 1e6, ms * 1e3,
                                 n / (ms * 1e-3) / 1e9, n * bytes_per / (ms * 1e-3) / 1e9);
        }
    };
    const uint32_t bl = 256, gr = (n + bl - 1) / bl;
#define RUN(K) \
    timeit("k" #K "_rd16", [&] { k_read<K, 1><<<gr, bl>>>(t, tbytes / 16, n, out); }, 16); \
    timeit("k" #K "_rd32", [&] { k_read<K, 2><<<gr, bl>>>(t, tbytes / 32, n, out); }, 32);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8)
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
