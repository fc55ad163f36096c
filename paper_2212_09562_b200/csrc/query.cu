// batched query on the GPU.  One thread per key: master hash
// code -> bucket i -> C[i], P[i] from the decoded index -> descend the splitting tree of
// size s: read the node's unary code (word-level scan for the terminating 1) and its tau
// fixed bits, pick the child by the node's hash, skip the fixed bits F(c) and N(c) unary
// codes of every earlier sibling (popcount over words), add their sizes -> leaf value
// (+ r mod m for B keys under rotation fitting).
#include <algorithm>

#include "format.h"
#include "kernels.h"
#include "pipeline.h"

namespace rs {

using namespace rsd;

namespace {

struct QueryArgs {
    const u64* C;
    const u64* P;
    const u64* data;
    const u32* tau;  // per size s <= smax
    const u64* F;
    const u32* N;
    u64 B, D, g;
    u32 leaf, u1, u2, rf;
};

__device__ __forceinline__ u64 bits_at(const u64* d, u64 pos, u32 w) {  // w <= 63
    if (w == 0) return 0;
    const u64 wi = pos >> 6;
    const u32 sh = (u32)(pos & 63);
    u64 x = d[wi] >> sh;
    if (sh + w > 64) x |= d[wi + 1] << (64 - sh);
    return w == 64 ? x : (x & ((1ull << w) - 1));
}

// position just after the cnt-th one-bit at or after pos (cnt >= 1)
__device__ __forceinline__ u64 skip_ones(const u64* d, u64 pos, u64 cnt) {
    u64 wi = pos >> 6;
    u64 w = d[wi] >> (pos & 63);
    u64 base = pos;
    for (;;) {
        const u64 c = (u64)__popcll(w);
        if (c >= cnt) {
            for (u64 k = 1; k < cnt; ++k) w &= w - 1;
            return base + (u64)__ffsll((long long)w);
        }
        cnt -= c;
        base = (wi + 1) << 6;
        w = d[++wi];
    }
}

__device__ u64 query_key(const QueryArgs& q, u64 key) {
    const u64 k = key ^ q.g;
    const u64 hi = remix64(k ^ MHC_SALT_HI), lo = remix64(k ^ MHC_SALT_LO);
    const u64 i = ((hi >> 32) * q.B) >> 32;
    u64 offset = q.C[i];
    u32 s = (u32)(q.C[i + 1] - offset);
    if (s == 0) return 0;
    u64 fc = q.P[i], uc = q.P[i] + q.F[s];
    for (;;) {
        const u32 t = q.tau[s];
        const u64 u1 = skip_ones(q.data, uc, 1);
        const u64 qq = u1 - uc - 1;
        uc = u1;
        const u64 x = (qq << t) | bits_at(q.data, fc, t);
        fc += t;
        if (s <= q.leaf) {
            const u32 m = s;
            const u64 r = q.rf ? x % m : 0;
            u32 v = __umulhi(remix_hi(lo + (x - r)), m);
            if (q.rf && (hi & 1)) v = (v + (u32)r) % m;  // B keys: rotation = + r mod m
            return offset + v;
        }
        // children of this split (R6) and the key's child j
        const u32 v = __umulhi(remix_hi(lo + x), s);
        u32 j, unit = 0, c0 = 0, f;
        if (s > q.u2) {
            c0 = (s / 2 + q.u2 - 1) / q.u2 * q.u2;
            f = 2;
            j = v >= c0;
        } else {
            unit = s <= q.u1 ? q.leaf : q.u1;
            f = (s + unit - 1) / unit;
            j = v / unit;
        }
        for (u32 c = 0; c < j; ++c) {
            const u32 cs = s > q.u2 ? (c == 0 ? c0 : s - c0) : (c + 1 < f ? unit : s - (f - 1) * unit);
            fc += q.F[cs];
            uc = skip_ones(q.data, uc, q.N[cs]);
            offset += cs;
        }
        s = s > q.u2 ? (j == 0 ? c0 : s - c0) : (j + 1 < f ? unit : s - (f - 1) * unit);
    }
}

__global__ void k_query(QueryArgs q, const u64* __restrict__ keys, u64 n, u64* __restrict__ out) {
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (u64)gridDim.x * blockDim.x)
        out[t] = query_key(q, keys[t]);
}

template <typename T>
T* upload(const std::vector<T>& v, cudaStream_t st, std::vector<void*>& owned) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(v.size() * sizeof(T), 16), st) != cudaSuccess)
        throw Error(RECSPLIT_E_NOMEM, "device allocation failed");
    owned.push_back(p);
    if (!v.empty() && cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st) != cudaSuccess)
        throw Error(RECSPLIT_E_CUDA, "upload failed");
    return (T*)p;
}

}  // namespace

void query_on_device(const Parsed& M, const uint64_t* d_keys, uint64_t n, uint64_t* d_out, cudaStream_t st) {
    std::vector<void*> owned;
    struct Free {
        std::vector<void*>& o;
        cudaStream_t s;
        ~Free() {
            for (void* p : o) cudaFreeAsync(p, s);
        }
    } fr{owned, st};
    const Tables& T = *M.T;
    const uint32_t smax = (uint32_t)M.smax;
    std::vector<uint32_t> tau(T.tau.begin(), T.tau.begin() + smax + 1);
    std::vector<uint64_t> F(T.F.begin(), T.F.begin() + smax + 1);
    std::vector<uint32_t> N(T.N.begin(), T.N.begin() + smax + 1);
    std::vector<uint64_t> data((M.D + 63) / 64 + 2, 0);
    if (M.D) memcpy(data.data(), M.data, 8 * ((M.D + 63) / 64));
    QueryArgs q;
    q.C = upload(M.C, st, owned);
    q.P = upload(M.P, st, owned);
    q.data = upload(data, st, owned);
    q.tau = upload(tau, st, owned);
    q.F = upload(F, st, owned);
    q.N = upload(N, st, owned);
    q.B = M.B;
    q.D = M.D;
    q.g = M.g;
    q.leaf = M.leaf;
    q.u1 = T.sh.u1;
    q.u2 = T.sh.u2;
    q.rf = M.rf ? 1 : 0;
    if (n) {
        unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
        k_query<<<grid, 256, 0, st>>>(q, d_keys, n, d_out);
        if (cudaGetLastError() != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "query launch failed");
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "query failed");
}

}  // namespace rs
