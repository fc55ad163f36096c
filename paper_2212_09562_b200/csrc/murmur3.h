// Master hash code of a string key (reading R16): MurmurHash3_x64_128
// (A. Appleby, public domain) of the key's bytes, seed = lo32(g) ^ hi32(g); hi = h1, lo = h2.
// The paper hashes its string workload with "a high quality hash function";
// this is the library's implementation (host query + device kernel), independent of the
// oracle's.  Blocks are read as little-endian words with 64-bit loads where aligned.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD inline
#endif

namespace rsm {

RS_HD uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

RS_HD uint64_t fmix64(uint64_t k) {
    k = (k ^ (k >> 33)) * 0xff51afd7ed558ccdULL;
    k = (k ^ (k >> 33)) * 0xc4ceb9fe1a85ec53ULL;
    return k ^ (k >> 33);
}

// nb <= 8 bytes at p, little-endian
RS_HD uint64_t load_le(const uint8_t* p, uint32_t nb) {
    uint64_t x = 0;
    for (uint32_t t = 0; t < nb; ++t) x |= (uint64_t)p[t] << (8 * t);
    return x;
}

RS_HD void murmur3_x64_128(const uint8_t* s, uint64_t len, uint32_t seed, uint64_t& o1, uint64_t& o2) {
    constexpr uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
    uint64_t h1 = seed, h2 = seed;
    const uint64_t nb = len >> 4;
    for (uint64_t i = 0; i < nb; ++i) {
        const uint64_t k1 = load_le(s + 16 * i, 8), k2 = load_le(s + 16 * i + 8, 8);
        h1 ^= rotl64(k1 * c1, 31) * c2;
        h1 = (rotl64(h1, 27) + h2) * 5 + 0x52dce729;
        h2 ^= rotl64(k2 * c2, 33) * c1;
        h2 = (rotl64(h2, 31) + h1) * 5 + 0x38495ab5;
    }
    const uint8_t* t = s + 16 * nb;
    const uint32_t r = (uint32_t)(len & 15);
    if (r > 8) h2 ^= rotl64(load_le(t + 8, r - 8) * c2, 33) * c1;
    if (r) h1 ^= rotl64(load_le(t, r < 8 ? r : 8) * c1, 31) * c2;
    h1 ^= len;
    h2 ^= len;
    h1 += h2;
    h2 += h1;
    h1 = fmix64(h1);
    h2 = fmix64(h2);
    h1 += h2;
    h2 += h1;
    o1 = h1;
    o2 = h2;
}

RS_HD void mhc_string(const uint8_t* s, uint64_t len, uint64_t g, uint64_t& hi, uint64_t& lo) {
    murmur3_x64_128(s, len, (uint32_t)g ^ (uint32_t)(g >> 32), hi, lo);
}

}  // namespace rsm
