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

// Bijectivity check: mark every value in a bitmap of n bits; a value
// outside [0, n) or one whose bit was already set is a violation.
__global__ void k_mark(const u64* __restrict__ v, u64 n, u32* __restrict__ bitmap, unsigned long long* bad) {
    u32 local = 0;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (u64)gridDim.x * blockDim.x) {
        const u64 x = v[t];
        if (x >= n) {
            ++local;
            continue;
        }
        const u32 bit = 1u << (x & 31);
        if (atomicOr(bitmap + (x >> 5), bit) & bit) ++local;
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, (unsigned long long)local);
}

template <typename T>
T* upload(const std::vector<T>& v, cudaStream_t st, std::vector<void*>& owned) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(v.size() * sizeof(T), 16)) != cudaSuccess)
        throw Error(RECSPLIT_E_NOMEM, "device allocation failed");
    owned.push_back(p);
    if (!v.empty() && cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st) != cudaSuccess)
        throw Error(RECSPLIT_E_CUDA, "upload failed");
    return (T*)p;
}

}  // namespace

// Resident device copy of a parsed MPHF: decoded index C/P, Golomb-Rice data words and the
// per-size tau/F/N tables (the layout k_query reads).  Plain cudaMalloc so that the copy
// outlives any stream.
struct DeviceMphf {
    QueryArgs q;
    std::vector<void*> owned;
    int device;
};

DeviceMphf* upload_mphf(const Parsed& M, cudaStream_t st) {
    std::unique_ptr<DeviceMphf> h(new DeviceMphf());
    try {
        cudaGetDevice(&h->device);
        const Tables& T = *M.T;
        const uint32_t smax = (uint32_t)M.smax;
        std::vector<uint32_t> tau(T.tau.begin(), T.tau.begin() + smax + 1);
        std::vector<uint64_t> F(T.F.begin(), T.F.begin() + smax + 1);
        std::vector<uint32_t> N(T.N.begin(), T.N.begin() + smax + 1);
        std::vector<uint64_t> data((M.D + 63) / 64 + 2, 0);
        if (M.D) memcpy(data.data(), M.data, 8 * ((M.D + 63) / 64));
        QueryArgs& q = h->q;
        q.C = upload(M.C, st, h->owned);
        q.P = upload(M.P, st, h->owned);
        q.data = upload(data, st, h->owned);
        q.tau = upload(tau, st, h->owned);
        q.F = upload(F, st, h->owned);
        q.N = upload(N, st, h->owned);
        q.B = M.B;
        q.D = M.D;
        q.g = M.g;
        q.leaf = M.leaf;
        q.u1 = T.sh.u1;
        q.u2 = T.sh.u2;
        q.rf = M.rf ? 1 : 0;
        // the host vectors die here: finish the copies first
        if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "upload failed");
    } catch (...) {
        free_mphf(h.release());
        throw;
    }
    return h.release();
}

void free_mphf(DeviceMphf* h) {
    if (!h) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(h->device);
    for (void* p : h->owned) cudaFree(p);
    cudaSetDevice(cur);
    delete h;
}

void query_resident(const DeviceMphf& h, const uint64_t* d_keys, uint64_t n, uint64_t* d_out, cudaStream_t st) {
    if (!n) return;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_query<<<grid, 256, 0, st>>>(h.q, d_keys, n, d_out);
    if (cudaGetLastError() != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "query launch failed");
}

uint64_t count_non_bijective(const uint64_t* d_vals, uint64_t n, cudaStream_t st) {
    if (!n) return 0;
    const size_t words = (n + 31) / 32;
    void* buf = nullptr;
    if (cudaMallocAsync(&buf, words * 4 + 8, st) != cudaSuccess) throw Error(RECSPLIT_E_NOMEM, "bitmap allocation failed");
    struct Free {
        void* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } fr{buf, st};
    unsigned long long* bad = (unsigned long long*)buf;  // 8 B counter, then the bitmap
    u32* bitmap = (u32*)((char*)buf + 8);
    cudaMemsetAsync(buf, 0, words * 4 + 8, st);
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_mark<<<grid, 256, 0, st>>>(d_vals, n, bitmap, bad);
    if (cudaGetLastError() != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "bijectivity check launch failed");
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "bijectivity check failed");
    return h;
}

void query_on_device(const Parsed& M, const uint64_t* d_keys, uint64_t n, uint64_t* d_out, cudaStream_t st) {
    std::unique_ptr<DeviceMphf, void (*)(DeviceMphf*)> h(upload_mphf(M, st), free_mphf);
    query_resident(*h, d_keys, n, d_out, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "query failed");
}

}  // namespace rs
