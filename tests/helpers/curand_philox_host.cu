// Host-only driver for cuRAND's own Philox4x32-10 (curand_philox4x32_x.h), used as a
// third-party pin for the oracle's Philox (tests/test_oracle_rng.py).  Reads lines
// "c0 c1 c2 c3 k0 k1" on stdin and prints the 4 output words.
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
    unsigned c0, c1, c2, c3, k0, k1;
    while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
        uint4 c = make_uint4(c0, c1, c2, c3);
        uint2 k = make_uint2(k0, k1);
        uint4 o = curand_Philox4x32_10(c, k);
        std::printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
    }
    return 0;
}
