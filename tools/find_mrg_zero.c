/* Input search for an MRG32k3a edge-case parity test (tests/test_gpu_parity.py,
 * test_mrg32k3a_floor_edge): finds (seed, stream, draw) where a component's new value is
 * exactly 0 with the sign of p = a x - a' x' for which the GPU's floor reduction
 * (PRNGD_MRG_FLOOR, csrc/prngd_device.cuh) holds r = m instead of 0:
 *   component 1: RN(1/m1) > 1/m1, so the floor is one low for p < 0;
 *   component 2: RN(1/m2) < 1/m2, so the floor is one low for p > 0.
 * Stream starts follow R22 (SplitMix64 outputs #3s..#3s+2).  Not test infrastructure: it only
 * picks an input; the expected outputs come from the oracle at test time.
 *   gcc -O2 -o /tmp/find_mrg_zero tools/find_mrg_zero.c && /tmp/find_mrg_zero 1 2000 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

static const int64_t M1 = 4294967087ll, M2 = 4294944443ll;
static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
int main(int argc, char **argv) {
    const uint64_t seed = argc > 1 ? strtoull(argv[1], 0, 0) : 1;
    const int draws = argc > 2 ? atoi(argv[2]) : 2000;
    int found = 0;
    for (uint64_t s = 0; s < (1ull << 26) && found < 4; ++s) {
        uint32_t wd[6];
        for (int i = 0; i < 3; ++i) {
            const uint64_t o = mix(seed + (3 * s + i + 1) * 0x9E3779B97F4A7C15ull);
            wd[2 * i] = (uint32_t)o;
            wd[2 * i + 1] = (uint32_t)(o >> 32);
        }
        int64_t x[3], y[3];
        for (int i = 0; i < 3; ++i) x[i] = wd[i] % M1, y[i] = wd[3 + i] % M2;
        if (!x[0] && !x[1] && !x[2]) x[0] = 1;
        if (!y[0] && !y[1] && !y[2]) y[0] = 1;
        for (int n = 0; n < draws; ++n) {
            const int64_t p1 = 1403580ll * x[1] - 810728ll * x[0];
            const int64_t p2 = 527612ll * y[2] - 1370589ll * y[0];
            int64_t r1 = p1 % M1, r2 = p2 % M2;
            if (r1 < 0) r1 += M1;
            if (r2 < 0) r2 += M2;
            if (r1 == 0 && p1 < 0) { printf("seed %llu stream %llu draw %d component 1 p %lld\n", (unsigned long long)seed, (unsigned long long)s, n, (long long)p1); ++found; }
            if (r2 == 0 && p2 > 0) { printf("seed %llu stream %llu draw %d component 2 p %lld\n", (unsigned long long)seed, (unsigned long long)s, n, (long long)p2); ++found; }
            x[0] = x[1], x[1] = x[2], x[2] = r1;
            y[0] = y[1], y[1] = y[2], y[2] = r2;
        }
    }
    return 0;
}
