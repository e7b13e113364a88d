/*
 * prngd_demo.c -- the library used from plain C through include/prngd.h (no Python, no torch):
 * create a handle for PRNGD(k = 2^-w, [a0; a], [b0; b]) (Eq.(4)), report the
 * host-precomputed constants and the kernel the plan picked, generate into HOST memory with
 * prngd_generate_host, and print the first outputs and an FNV-1a hash of all output bits.
 *
 *   cc -std=c11 -I include examples/prngd_demo.c -L paper_1401_8230_b200 -lprngd_b200 \
 *      -Wl,-rpath,$PWD/paper_1401_8230_b200 -o prngd_demo
 *   ./prngd_demo [w a0 a b seed n_streams n_per_stream]     (default: cfg1, 1024 x 1024)
 *   ./prngd_demo --validate                                 (host-only checks, no GPU needed)
 *
 * Exit status: 0 on success, 1 on a library error (message from prngd_last_error()).
 */
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "prngd.h"

static int check(prngd_status s, const char *what) {
    if (s == PRNGD_OK) return 0;
    fprintf(stderr, "%s: %s: %s\n", what, prngd_status_string(s), prngd_last_error());
    return 1;
}

/* host-only: the EINVAL cases of include/prngd.h are refused before any device work */
static int validate(void) {
    prngd_params p;
    memset(&p, 0, sizeof p);
    p.w = 32, p.a0 = 0, p.a = 0xFFFFFFFFull, p.b0 = 0, p.b = 0xFFFFFFFFull, p.seed = 1;
    p.n_streams = 1024, p.n_per_stream = 1024;
    prngd_handle *h = NULL;
    if (check(prngd_create(&p, &h), "prngd_create(cfg1)")) return 1;
    prngd_info info;
    if (check(prngd_get_info(h, &info), "prngd_get_info")) return 1;
    printf("cfg1: C = %.17g D = %.17g kernel %u store %u outputs %" PRIu64 "\n", info.C, info.D,
           info.kernel, info.store, info.n_outputs);
    prngd_destroy(h);
    struct { const char *why; uint32_t w; uint64_t a0, a, b; } bad[] = {
        {"w = 0", 0, 0, 255, 255},
        {"a - a0 < 2", 8, 10, 11, 255},
        {"b + 1 not a power of two", 8, 0, 255, 130},
        {"b >= 2^w", 8, 0, 255, 511},
    };
    for (size_t i = 0; i < sizeof bad / sizeof bad[0]; ++i) {
        p.w = bad[i].w, p.a0 = bad[i].a0, p.a = bad[i].a, p.b = bad[i].b;
        const prngd_status s = prngd_create(&p, &h);
        printf("%-26s -> %s (%s)\n", bad[i].why, prngd_status_string(s), prngd_last_error());
        if (s != PRNGD_EINVAL || h != NULL) return 1;
    }
    printf("abi %d validate ok\n", prngd_abi_version());
    return 0;
}

int main(int argc, char **argv) {
    if (argc > 1 && strcmp(argv[1], "--validate") == 0) return validate();
    prngd_params p;
    memset(&p, 0, sizeof p);
    p.w = 32, p.a0 = 0, p.a = 0xFFFFFFFFull, p.b0 = 0, p.b = 0xFFFFFFFFull, p.seed = 1;
    p.n_streams = 1024, p.n_per_stream = 1024;
    if (argc == 8) {
        p.w = (uint32_t)strtoul(argv[1], NULL, 0);
        p.a0 = strtoull(argv[2], NULL, 0), p.a = strtoull(argv[3], NULL, 0);
        p.b = strtoull(argv[4], NULL, 0), p.seed = strtoull(argv[5], NULL, 0);
        p.n_streams = strtoull(argv[6], NULL, 0), p.n_per_stream = strtoull(argv[7], NULL, 0);
    } else if (argc != 1) {
        fprintf(stderr, "usage: %s [w a0 a b seed n_streams n_per_stream] | --validate\n", argv[0]);
        return 2;
    }
    prngd_handle *h = NULL;
    if (check(prngd_create(&p, &h), "prngd_create")) return 1;
    const uint64_t n = p.n_streams * p.n_per_stream;
    double *out = (double *)malloc(n * sizeof(double));
    if (!out) return 1;
    if (check(prngd_generate_host(h, out, NULL), "prngd_generate_host")) return 1;
    uint64_t fnv = 0xcbf29ce484222325ull;  /* FNV-1a over the little-endian output bytes */
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t bits;
        memcpy(&bits, &out[i], 8);
        for (int b = 0; b < 8; ++b) {
            fnv ^= (bits >> (8 * b)) & 0xFFu;
            fnv *= 0x100000001b3ull;
        }
    }
    printf("outputs %" PRIu64 " first %.17g %.17g %.17g last %.17g fnv1a %016" PRIx64 "\n", n,
           out[0], out[1], out[2], out[n - 1], fnv);
    free(out);
    return check(prngd_destroy(h), "prngd_destroy");
}
