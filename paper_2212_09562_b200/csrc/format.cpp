// Serialized-MPHF reader: validates the blob and decodes both
// Elias-Fano sequences into C[] (bucket key offsets) and P[] (bucket bit offsets).
#include "format.h"

#include <algorithm>
#include <cstring>

#include "../../include/recsplit.h"

namespace rs {


static uint64_t rd64(const uint8_t* p) {
    uint64_t x;
    memcpy(&x, p, 8);
    return x;
}

static uint64_t word_at(const uint8_t* base, uint64_t i) { return rd64(base + 8 * i); }

static bool parse_ef(const uint8_t*& p, const uint8_t* end, EFView& e) {
    if (end - p < 16) return false;
    e.L = p[0];
    if (e.L > 63) return false;
    for (int i = 1; i < 8; ++i)
        if (p[i]) return false;
    e.nlow = rd64(p + 8);
    p += 16;
    if ((uint64_t)(end - p) / 8 < (e.nlow + 63) / 64) return false;
    e.low = p;
    p += 8 * ((e.nlow + 63) / 64);
    if (end - p < 8) return false;
    e.nup = rd64(p);
    p += 8;
    if ((uint64_t)(end - p) / 8 < (e.nup + 63) / 64) return false;
    e.up = p;
    p += 8 * ((e.nup + 63) / 64);
    return true;
}

static bool ef_decode(const EFView& e, uint64_t k, std::vector<uint64_t>& v) {
    if (e.nlow != k * e.L) return false;
    v.assign(k, 0);
    uint64_t i = 0;
    const uint64_t words = (e.nup + 63) / 64;
    for (uint64_t w = 0; w < words && i < k; ++w) {
        uint64_t x = word_at(e.up, w);
        while (x && i < k) {
            const uint64_t pos = w * 64 + __builtin_ctzll(x);
            x &= x - 1;
            if (pos >= e.nup) return false;
            uint64_t lo = 0;
            if (e.L) {
                const uint64_t bp = i * e.L;
                const uint64_t a = word_at(e.low, bp >> 6);
                const uint64_t sh = bp & 63;
                lo = a >> sh;
                if (sh + e.L > 64) lo |= word_at(e.low, (bp >> 6) + 1) << (64 - sh);
                lo &= (e.L == 64) ? ~0ull : ((1ull << e.L) - 1);
            }
            v[i] = ((pos - i) << e.L) | lo;
            ++i;
        }
    }
    return i == k;
}

int parse_mphf(const uint8_t* blob, size_t size, Parsed& M, std::string* err) {
    auto fail = [&](int code, const char* m) {
        if (err) *err = m;
        return code;
    };
    if (!blob || size < 72 || memcmp(blob, "RSRF", 4) != 0) return fail(RECSPLIT_E_FORMAT, "bad magic / size");
    uint16_t ver;
    memcpy(&ver, blob + 4, 2);
    if (ver != 1) return fail(RECSPLIT_E_FORMAT, "unsupported format version");
    M.leaf = blob[6];
    M.rf = blob[7] & 1;
    M.strings = (blob[7] >> 1) & 1;
    if (M.leaf < 2 || M.leaf > 24) return fail(RECSPLIT_E_FORMAT, "bad leaf size");
    M.g = rd64(blob + 16);
    M.n = rd64(blob + 24);
    M.B = rd64(blob + 32);
    M.D = rd64(blob + 40);
    M.dC = rd64(blob + 48);
    M.beta = rd64(blob + 56);
    M.dR = (int64_t)rd64(blob + 64);
    if (M.n == 0 || M.B == 0 || M.B > M.n + 1) return fail(RECSPLIT_E_FORMAT, "bad n / B");
    const uint8_t* p = blob + 72;
    const uint8_t* end = blob + size;
    if (!parse_ef(p, end, M.ec) || !parse_ef(p, end, M.ep)) return fail(RECSPLIT_E_FORMAT, "truncated index");
    if ((uint64_t)(end - p) != 8 * ((M.D + 63) / 64)) return fail(RECSPLIT_E_FORMAT, "data length mismatch");
    M.data = p;
    std::vector<uint64_t> c, q;
    if (!ef_decode(M.ec, M.B + 1, c) || !ef_decode(M.ep, M.B + 1, q)) return fail(RECSPLIT_E_FORMAT, "bad index");
    M.C.resize(M.B + 1);
    M.P.resize(M.B + 1);
    uint64_t smax = 1;
    for (uint64_t i = 0; i <= M.B; ++i) {
        M.C[i] = c[i] + i * M.dC;
        M.P[i] = (uint64_t)((int64_t)q[i] + (int64_t)i * M.dR) +
                 (uint64_t)(((unsigned __int128)M.beta * M.C[i]) >> 20);
        if (i) {
            if (M.C[i] < M.C[i - 1] || M.P[i] < M.P[i - 1]) return fail(RECSPLIT_E_FORMAT, "index not monotone");
            smax = std::max<uint64_t>(smax, M.C[i] - M.C[i - 1]);
        }
    }
    if (M.C[0] != 0 || M.C[M.B] != M.n || M.P[0] != 0 || M.P[M.B] != M.D) return fail(RECSPLIT_E_FORMAT, "bad index ends");
    if (smax > (1u << 20)) return fail(RECSPLIT_E_FORMAT, "bucket too large");
    M.smax = smax;
    M.T = get_tables(M.leaf, M.rf, (uint32_t)smax);
    // Per-bucket structure (R15): the fixed parts take F(s) bits and the unary region that
    // follows holds exactly N(s) terminating ones.  A query descends inside its bucket, reads
    // at most F(s) fixed bits and skips at most N(s) ones, so with this check neither the
    // host nor the device query (k_query) can read past the bucket, whatever the stored
    // values are; a corrupt blob is rejected here with RECSPLIT_E_FORMAT.
    const Tables& T = *M.T;
    auto ones = [&](uint64_t a, uint64_t b) {  // one-bits of data in [a, b)
        uint64_t c = 0;
        while (a < b) {
            const uint64_t w = word_at(M.data, a >> 6) >> (a & 63);
            const uint64_t take = std::min<uint64_t>(64 - (a & 63), b - a);
            c += __builtin_popcountll(take == 64 ? w : (w & ((1ull << take) - 1)));
            a += take;
        }
        return c;
    };
    for (uint64_t i = 0; i < M.B; ++i) {
        const uint64_t s = M.C[i + 1] - M.C[i];
        const uint64_t u0 = M.P[i] + T.F[s];
        if (u0 > M.P[i + 1] || ones(u0, M.P[i + 1]) != T.N[s])
            return fail(RECSPLIT_E_FORMAT, "bucket encoding inconsistent with its size");
    }
    return RECSPLIT_OK;
}


}  // namespace rs
