// prngd_jump.cpp -- GF(2) jump-ahead for xorshift128 (NEXT-3: intra-stream parallelism).
//
// xorshift128 (Marsaglia 2003) is linear over GF(2): one draw maps the 128-bit state
// s = (x, y, z, w) to T*s.  Advancing a stream by n draws is the matrix power T^n, so the 32
// lanes of a warp can start at draws 0, d, 2d, ... of the same stream (d = kJumpDraws = 34 for
// the NEXT-3 jump kernel, 2 * segment length for SEG).  The device applies J_l = T^(d l) with
// byte tables: tab[l][b][v] = J_l * (v << 8b), so J_l * s is the XOR of 16 table entries
// (16 x 16-byte loads).  Product code; independent of oracle/.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "prngd_internal.h"

namespace prngd {

namespace {

struct Vec128 {
    uint32_t w[4];  // w[0] = x, w[1] = y, w[2] = z, w[3] = w
};

// One xorshift128 step on a state vector: the linear map T.
Vec128 step(const Vec128 &s) {
    const uint32_t t = s.w[0] ^ (s.w[0] << 11);
    Vec128 r;
    r.w[0] = s.w[1];
    r.w[1] = s.w[2];
    r.w[2] = s.w[3];
    r.w[3] = s.w[3] ^ (s.w[3] >> 19) ^ t ^ (t >> 8);
    return r;
}

struct Mat128 {
    Vec128 col[128];  // column j = image of basis vector e_j (bit j%32 of word j/32)
};

Vec128 apply(const Mat128 &m, const Vec128 &v) {
    Vec128 r = {{0, 0, 0, 0}};
    for (int j = 0; j < 128; ++j)
        if ((v.w[j >> 5] >> (j & 31)) & 1u)
            for (int k = 0; k < 4; ++k) r.w[k] ^= m.col[j].w[k];
    return r;
}

Mat128 mul(const Mat128 &a, const Mat128 &b) {  // (a*b) v = a (b v)
    Mat128 c;
    for (int j = 0; j < 128; ++j) c.col[j] = apply(a, b.col[j]);
    return c;
}

Mat128 identity() {
    Mat128 m;
    std::memset(&m, 0, sizeof(m));
    for (int j = 0; j < 128; ++j) m.col[j].w[j >> 5] = 1u << (j & 31);
    return m;
}

Mat128 t_matrix() {
    Mat128 m;
    for (int j = 0; j < 128; ++j) {
        Vec128 e = {{0, 0, 0, 0}};
        e.w[j >> 5] = 1u << (j & 31);
        m.col[j] = step(e);
    }
    return m;
}

Mat128 t_power(uint64_t n) {  // T^n by square-and-multiply
    Mat128 r = identity(), p = t_matrix();
    while (n) {
        if (n & 1u) r = mul(p, r);
        n >>= 1;
        if (n) p = mul(p, p);
    }
    return r;
}

// Byte tables of the 32 lane matrices J_l = T^(lane_draws * l), [l][b][v] -> 4 words.
std::vector<uint32_t> build_tables(uint64_t lane_draws) {
    std::vector<uint32_t> tab((size_t)32 * 16 * 256 * 4, 0u);
    const Mat128 step_lane = t_power(lane_draws);
    Mat128 j = identity();
    for (int l = 0; l < 32; ++l) {
        for (int b = 0; b < 16; ++b)
            for (int v = 0; v < 256; ++v) {
                uint32_t *e = &tab[(((size_t)l * 16 + b) * 256 + v) * 4];
                for (int t = 0; t < 8; ++t)
                    if ((v >> t) & 1)
                        for (int k = 0; k < 4; ++k) e[k] ^= j.col[8 * b + t].w[k];
            }
        j = mul(step_lane, j);
    }
    return tab;
}

// Nibble tables of the same 32 lane matrices: [l][p][v] = J_l * (v << 4p), p < 32, v < 16 (8 KiB
// per lane instead of 64 KiB: 32 loads per jump instead of 16, an 8x smaller cache footprint).
std::vector<uint32_t> build_nibble_tables(uint64_t lane_draws) {
    std::vector<uint32_t> tab((size_t)32 * 32 * 16 * 4, 0u);
    const Mat128 step_lane = t_power(lane_draws);
    Mat128 j = identity();
    for (int l = 0; l < 32; ++l) {
        for (int p = 0; p < 32; ++p)
            for (int v = 0; v < 16; ++v) {
                uint32_t *e = &tab[(((size_t)l * 32 + p) * 16 + v) * 4];
                for (int t = 0; t < 4; ++t)
                    if ((v >> t) & 1)
                        for (int k = 0; k < 4; ++k) e[k] ^= j.col[4 * p + t].w[k];
            }
        j = mul(step_lane, j);
    }
    return tab;
}

// The byte tables with the lane index innermost: [b][v][l].  All S lanes of a SEG row jump the
// same stream-start state, so they read one contiguous S x 16-byte run per byte position
// (4 cache lines per warp load instead of 32 scattered sectors).
std::vector<uint32_t> build_tables_interleaved(uint64_t lane_draws) {
    const std::vector<uint32_t> t = build_tables(lane_draws);  // [l][b][v]
    std::vector<uint32_t> r(t.size());
    for (int l = 0; l < 32; ++l)
        for (int b = 0; b < 16; ++b)
            for (int v = 0; v < 256; ++v)
                for (int k = 0; k < 4; ++k)
                    r[(((size_t)b * 256 + v) * 32 + l) * 4 + k] = t[(((size_t)l * 16 + b) * 256 + v) * 4 + k];
    return r;
}

std::mutex g_mu;
// key: lane_draws with bit 63 set for the nibble form
std::map<std::pair<int, uint64_t>, void *> g_dev_tables;  // (device, key) -> tables
std::map<uint64_t, std::vector<uint32_t>> g_host_tables;   // key -> host copy
constexpr uint64_t kNibbleKey = 1ull << 63;
constexpr uint64_t kInterleavedKey = 1ull << 62;

const std::vector<uint32_t> &host_tables(uint64_t key) {  // call with g_mu held
    auto it = g_host_tables.find(key);
    if (it == g_host_tables.end())
        it = g_host_tables
                 .emplace(key, (key & kNibbleKey)        ? build_nibble_tables(key & ~kNibbleKey)
                               : (key & kInterleavedKey) ? build_tables_interleaved(key & ~kInterleavedKey)
                                                         : build_tables(key))
                 .first;
    return it->second;
}

cudaError_t device_tables(uint64_t key, const void **out) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_dev_tables.find({dev, key});
    if (it != g_dev_tables.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    const std::vector<uint32_t> &host = host_tables(key);
    void *d = nullptr;
    if ((e = cudaMalloc(&d, host.size() * 4)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(d, host.data(), host.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(d);
        return e;
    }
    g_dev_tables[{dev, key}] = d;
    *out = d;
    return cudaSuccess;
}

}  // namespace

cudaError_t jump_tables(uint64_t lane_draws, const void **out) {
    return device_tables(lane_draws, out);
}

cudaError_t jump_tables_nibble(uint64_t lane_draws, const void **out) {
    return device_tables(lane_draws | kNibbleKey, out);
}

cudaError_t jump_tables_interleaved(uint64_t lane_draws, const void **out) {
    return device_tables(lane_draws | kInterleavedKey, out);
}

void jump_host(uint64_t n_draws, const uint32_t in[4], uint32_t out[4], int lane_table) {
    Vec128 v;
    std::memcpy(v.w, in, 16);
    Vec128 r;
    if (lane_table >= 0) {  // through the byte table of lane `lane_table` (what the GPU reads):
                            // J = T^(lane_draws * lane_table), lane_draws = n_draws or kJumpDraws
        const uint64_t lane_draws = n_draws ? n_draws : kJumpDraws;
        std::lock_guard<std::mutex> lock(g_mu);
        const std::vector<uint32_t> &tab = host_tables(lane_draws);
        std::memset(r.w, 0, 16);
        for (int b = 0; b < 16; ++b) {
            const uint32_t byte = (v.w[b >> 2] >> (8 * (b & 3))) & 0xFFu;
            const uint32_t *e = &tab[(((size_t)lane_table * 16 + b) * 256 + byte) * 4];
            for (int k = 0; k < 4; ++k) r.w[k] ^= e[k];
        }
    } else {
        r = apply(t_power(n_draws), v);
    }
    std::memcpy(out, r.w, 16);
}

}  // namespace prngd
