// Steps A1-A2: master hash codes, bucket assignment, exact duplicate
// detection, counting sort by bucket.
// P:106-108 (initial hash, buckets of expected size b), P:319 (sort by bucket index,
// determine borders), P:389 (random integers as MHC).
#include <algorithm>
#include <vector>

#include "kernels.h"
#include "murmur3.h"
#include "pipeline.h"

namespace rs {

using namespace rsd;

// A1: hi = remix(key^g^salt_hi), lo = remix(key^g^salt_lo) (R2); bucket = remap(hi, B)
// (R3); A/B bit = hi & 1 (R7).  Bucket histogram in shared memory when the shard has few
// buckets (one global atomic per bucket per block), else global.
// Only buckets in [b0, b1) (this shard, P:320 contiguous bucket ranges) are kept; their
// local index b - b0 goes to bkt, other keys get bkt = NONE.
// keys == nullptr: the master hash codes are given (mhc[2i] = hi, mhc[2i+1] = lo; string keys).
__global__ void __launch_bounds__(1024) k_hash(const u64* __restrict__ keys, const u64* __restrict__ mhc, u64 n,
                                               u64 g, u64 B, u64 b0, u64 b1, u64* __restrict__ lo,
                                               u8* __restrict__ ab, u32* __restrict__ bkt, u32* __restrict__ hist,
                                               int smem_hist) {
    extern __shared__ u32 sh[];
    const u64 Bl = b1 - b0;
    if (smem_hist) {
        for (u32 i = threadIdx.x; i < Bl; i += blockDim.x) sh[i] = 0;
        __syncthreads();
    }
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 k = keys ? keys[i] ^ g : 0;
        const u64 h = keys ? remix64(k ^ MHC_SALT_HI) : mhc[2 * i];
        const u64 bg = ((h >> 32) * B) >> 32;
        if (bg < b0 || bg >= b1) {
            bkt[i] = NONE;
            continue;
        }
        const u32 b = (u32)(bg - b0);
        const u64 l = keys ? remix64(k ^ MHC_SALT_LO) : mhc[2 * i + 1];
        lo[i] = l;
        ab[i] = (u8)(h & 1);
        bkt[i] = b;
        if (smem_hist)
            atomicAdd(sh + b, 1u);
        else
            atomicAdd(hist + b, 1u);
    }
    if (smem_hist) {
        __syncthreads();
        for (u32 i = threadIdx.x; i < Bl; i += blockDim.x)
            if (sh[i]) atomicAdd(hist + i, sh[i]);
    }
}

void launch_hash(const u64* keys, const u64* mhc, u64 n, u64 g, u64 B, u64 b0, u64 b1, u64* lo, u8* ab, u32* bkt,
                 u32* hist, cudaStream_t st) {
    const u64 Bl = b1 - b0;
    const int smem_hist = Bl <= 12288;
    const size_t smem = smem_hist ? Bl * 4 : 0;
    unsigned grid = (unsigned)((n + 1023) / 1024);
    const unsigned cap = smem_hist ? 148u * 2u : 148u * 8u;
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    cudaFuncSetAttribute(k_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k_hash<<<grid, 1024, smem, st>>>(keys, mhc, n, g, B, b0, b1, lo, ab, bkt, hist, smem_hist);
    g_launches++;
}

// max / min bucket size and the histogram of bucket sizes (sizes > cap counted at cap)
__global__ void k_bucket_stats(const u32* __restrict__ hist, u64 B, u32* maxmin, u32* size_hist, u32 cap) {
    u32 mx = 0, mn = 0xffffffffu;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (u64)gridDim.x * blockDim.x) {
        u32 s = hist[i];
        mx = s > mx ? s : mx;
        mn = s < mn ? s : mn;
        if (size_hist) atomicAdd(size_hist + (s <= cap ? s : cap), 1u);
    }
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(FULL, mx, d));
        mn = min(mn, __shfl_xor_sync(FULL, mn, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxmin, mx);
        atomicMin(maxmin + 1, mn);
    }
}

void launch_bucket_stats(const u32* hist, u64 B, u32* maxmin, u32* size_hist, u32 cap, cudaStream_t st) {
    unsigned grid = (unsigned)((B + 255) / 256);
    if (grid > 1024) grid = 1024;
    if (grid == 0) grid = 1;
    k_bucket_stats<<<grid, 256, 0, st>>>(hist, B, maxmin, size_hist, cap);
    g_launches++;
}

// Counting-sort scatter (A2): each key's (lo, A/B bit) to its bucket's next free slot;
// four independent keys per thread keep several atomics in flight.
__global__ void k_scatter(const u64* __restrict__ lo, const u8* __restrict__ ab, const u32* __restrict__ bkt,
                          u64 n, unsigned long long* __restrict__ cursor, u64* __restrict__ lo2,
                          u8* __restrict__ ab2) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
        u32 b[4];
        u64 p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u64 i = i0 + k * stride;
            b[k] = i < n ? bkt[i] : NONE;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u64 i = i0 + k * stride;
            if (i < n && b[k] != NONE) p[k] = atomicAdd(cursor + b[k], 1ull);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u64 i = i0 + k * stride;
            if (i < n && b[k] != NONE) {
                lo2[p[k]] = lo[i];
                ab2[p[k]] = ab[i];
            }
        }
    }
}

void launch_scatter(const u64* lo, const u8* ab, const u32* bkt, u64 n, u64* cursor, u64* lo2, u8* ab2,
                    cudaStream_t st) {
    unsigned grid = (unsigned)((n + 1023) / 1024);
    if (grid > 148u * 8u) grid = 148u * 8u;
    if (grid == 0) grid = 1;
    k_scatter<<<grid, 256, 0, st>>>(lo, ab, bkt, n, (unsigned long long*)cursor, lo2, ab2);
    g_launches++;
}

// Exact duplicate check after the scatter: equal keys have equal lo (remix is a bijection,
// R2) and land in the same bucket, so each bucket inserts its lo values into an open-
// addressing set (0 marks an empty slot; lo == 0 is counted instead): in shared memory for
// buckets of up to kSmallBucketKeys keys, in a per-block global table (BIG) above that.
// dup[0] |= 1 on a repeated value, dup[1] += keys with lo == 0 (> 1 is a duplicate).
template <bool BIG>
__global__ void __launch_bounds__(256) k_dedupe(const u64* __restrict__ lo, const u64* __restrict__ C, u64 nb,
                                                u32 dup_cap, u32* dup, unsigned long long* gtab, u32 smax) {
    extern __shared__ unsigned long long stab[];
    unsigned long long* tab = BIG ? gtab + (size_t)blockIdx.x * 2 * dup_cap : stab;
    for (u64 b = blockIdx.x; b < nb; b += gridDim.x) {
        const u64 c0 = C[b], s = C[b + 1] - c0;
        __syncthreads();
        // (s > smax: a bucket above the caller's size bound, flagged elsewhere; never read past
        // the table)
        if (s < 2 || s > smax || (BIG ? s <= kSmallBucketKeys : s > kSmallBucketKeys)) continue;
        u32 ts = 64;
        while (ts < 2 * s) ts <<= 1;
        for (u32 i = threadIdx.x; i < ts; i += blockDim.x) tab[i] = 0;
        __syncthreads();
        for (u32 i = threadIdx.x; i < s; i += blockDim.x) {
            const u64 v = lo[c0 + i];
            if (v == 0) {
                atomicAdd(dup + 1, 1u);
                continue;
            }
            u32 slot = (u32)(v ^ (v >> 32)) & (ts - 1);
            for (;;) {
                const unsigned long long old = atomicCAS(tab + slot, 0ull, (unsigned long long)v);
                if (old == 0ull) break;
                if (old == v) {
                    atomicOr(dup, 1u);
                    break;
                }
                slot = (slot + 1) & (ts - 1);
            }
        }
    }
}

// The same check with one WARP per bucket (buckets of at most kDedupeWarpMax keys): no block
// barriers, several buckets per block in flight; each warp owns a table of ts entries.
constexpr u32 kDedupeWarpMax = 256;

__global__ void __launch_bounds__(256) k_dedupe_warp(const u64* __restrict__ lo, const u64* __restrict__ C, u64 nb,
                                                     u32 ts, u32* dup) {
    extern __shared__ unsigned long long wtab[];
    const u32 lane = threadIdx.x & 31;
    unsigned long long* tab = wtab + (size_t)(threadIdx.x >> 5) * ts;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    for (u64 b = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += nw) {
        const u64 c0 = C[b], s = C[b + 1] - c0;
        if (s < 2 || 2 * s > ts) continue;  // (larger buckets: flagged by the caller's size bound)
        for (u32 i = lane; i < ts; i += 32) tab[i] = 0;
        __syncwarp();
        bool rep = false;
        u32 zeros = 0;
        for (u32 i = lane; i < s; i += 32) {
            const u64 v = lo[c0 + i];
            if (v == 0) {
                ++zeros;
                continue;
            }
            u32 slot = (u32)(v ^ (v >> 32)) & (ts - 1);
            for (;;) {
                const unsigned long long old = atomicCAS(tab + slot, 0ull, (unsigned long long)v);
                if (old == 0ull) break;
                if (old == v) {
                    rep = true;
                    break;
                }
                slot = (slot + 1) & (ts - 1);
            }
        }
        if (rep) atomicOr(dup, 1u);
        if (zeros) atomicAdd(dup + 1, zeros);
        __syncwarp();
    }
}

void launch_dedupe(const u64* lo, const u64* C, u64 nb, u32 smax, u32* dup, u64* big_scratch, cudaStream_t st) {
    if (nb == 0) return;
    if (smax <= kDedupeWarpMax) {
        u32 ts = 64;
        while (ts < 2 * smax) ts <<= 1;
        const u32 wpb = 8;
        const unsigned grid = (unsigned)std::min<u64>((nb + wpb - 1) / wpb, 148ull * 16);
        cudaFuncSetAttribute(k_dedupe_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        k_dedupe_warp<<<grid, wpb * 32, (size_t)wpb * ts * 8, st>>>(lo, C, nb, ts, dup);
        g_launches++;
        return;
    }
    const u32 sm = std::min(smax, kSmallBucketKeys);
    u32 ts = 64;
    while (ts < 2 * sm) ts <<= 1;
    const size_t smem = (size_t)ts * 8;
    cudaFuncSetAttribute(k_dedupe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const u32 threads = smax <= 128 ? 128 : 256;
    unsigned grid = nb < 148ull * 64 ? (unsigned)nb : 148u * 64;
    k_dedupe<false><<<grid, threads, smem, st>>>(lo, C, nb, 0, dup, nullptr, smax);
    g_launches++;
    if (smax > kSmallBucketKeys) {
        u32 tb = 64;
        while (tb < 2 * smax) tb <<= 1;  // per-block table of tb entries (dup_cap = tb / 2)
        const unsigned g2 = nb < kDedupeBigBlocks ? (unsigned)nb : kDedupeBigBlocks;
        k_dedupe<true><<<g2, 256, 0, st>>>(lo, C, nb, tb / 2, dup, (unsigned long long*)big_scratch, smax);
        g_launches++;
    }
}

// String keys (reading R16): master hash code of bytes[off[i] .. off[i+1])
// = MurmurHash3_x64_128 (murmur3.h).  One thread per key.
__global__ void k_mhc_strings(const u8* __restrict__ data, const u64* __restrict__ off, u64 n, u64 g,
                              u64* __restrict__ mhc) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 a = off[i], len = off[i + 1] - a;
        u64 hi, lo;
        rsm::mhc_string(data + a, len, g, hi, lo);
        mhc[2 * i] = hi;
        mhc[2 * i + 1] = lo;
    }
}

void launch_mhc_strings(const u8* data, const u64* off, u64 n, u64 g, u64* mhc, cudaStream_t st) {
    unsigned grid = (unsigned)((n + 255) / 256);
    if (grid > 148u * 16u) grid = 148u * 16u;
    if (grid == 0) grid = 1;
    k_mhc_strings<<<grid, 256, 0, st>>>(data, off, n, g, mhc);
    g_launches++;
}

}  // namespace rs

namespace rs {
using namespace rsd;
namespace {

// owner rank of bucket i: the r with cuts[r] <= i < cuts[r+1] (ranks with an
// empty range own nothing); cuts = world + 1 entries in shared memory
__device__ __forceinline__ u32 owner_of(u64 i, const unsigned long long* cuts, u32 W) {
    u32 lo = 0, hi = W;  // invariant: cuts[lo] <= i < cuts[hi]
    while (hi - lo > 1) {
        const u32 mid = (lo + hi) >> 1;
        if (cuts[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// pass 1: keys per destination rank (block histogram in shared memory)
__global__ void k_route_count(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u32 W, const u64* __restrict__ gcuts,
                              u64* __restrict__ counts) {
    extern __shared__ unsigned long long rc[];
    unsigned long long* cuts = rc + W;  // W + 1
    for (u32 i = threadIdx.x; i < W; i += blockDim.x) rc[i] = 0;
    for (u32 i = threadIdx.x; i <= W; i += blockDim.x) cuts[i] = gcuts[i];
    __syncthreads();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 h = remix64(keys[i] ^ g ^ MHC_SALT_HI);
        atomicAdd(rc + owner_of(((h >> 32) * B) >> 32, cuts, W), 1ull);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < W; i += blockDim.x)
        if (rc[i]) atomicAdd((unsigned long long*)counts + i, rc[i]);
}

// pass 2: scatter every key to its destination's segment (cursor = segment start, advanced
// with one atomic per destination per block)
__global__ void k_route_scatter(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u32 W, const u64* __restrict__ gcuts,
                                u64* __restrict__ cursor, u64* __restrict__ out) {
    extern __shared__ unsigned long long rs_[];
    unsigned long long* cnt = rs_;           // W
    unsigned long long* base = rs_ + W;      // W
    unsigned long long* cuts = rs_ + 2 * W;  // W + 1
    for (u32 i = threadIdx.x; i <= W; i += blockDim.x) cuts[i] = gcuts[i];
    const u64 per = (u64)blockDim.x * 8;
    for (u64 t0 = (u64)blockIdx.x * per; t0 < n; t0 += (u64)gridDim.x * per) {
        for (u32 i = threadIdx.x; i < W; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        u32 dst[8];
        unsigned long long pos[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const u64 i = t0 + (u64)q * blockDim.x + threadIdx.x;
            dst[q] = 0xffffffffu;
            if (i < n) {
                const u64 h = remix64(keys[i] ^ g ^ MHC_SALT_HI);
                dst[q] = owner_of(((h >> 32) * B) >> 32, cuts, W);
                pos[q] = atomicAdd(cnt + dst[q], 1ull);
            }
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < W; i += blockDim.x)
            base[i] = cnt[i] ? atomicAdd((unsigned long long*)cursor + i, cnt[i]) : 0;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (dst[q] != 0xffffffffu) out[base[dst[q]] + pos[q]] = keys[t0 + (u64)q * blockDim.x + threadIdx.x];
        __syncthreads();
    }
}

// per-bucket key counts of a rank's keys (work-balanced cuts)
__global__ void k_bucket_hist(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u32* __restrict__ hist,
                              int smem_hist) {
    extern __shared__ u32 bh[];
    if (smem_hist) {
        for (u32 i = threadIdx.x; i < B; i += blockDim.x) bh[i] = 0;
        __syncthreads();
    }
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 h = remix64(keys[i] ^ g ^ MHC_SALT_HI);
        const u64 b = ((h >> 32) * B) >> 32;
        atomicAdd((smem_hist ? bh : hist) + b, 1u);
    }
    if (smem_hist) {
        __syncthreads();
        for (u32 i = threadIdx.x; i < B; i += blockDim.x)
            if (bh[i]) atomicAdd(hist + i, bh[i]);
    }
}

}  // namespace

void bucket_histogram(const u64* d_keys, u64 n, u64 total, u32 bucket, u64 g, cudaStream_t st, u32* d_hist) {
    if (!n) return;
    const u64 B = (total + bucket - 1) / bucket;  // R12, global
    const int smem_hist = B <= 12288;
    const unsigned grid = (unsigned)std::max<u64>(1, std::min<u64>((n + 1023) / 1024, smem_hist ? 148ull * 2 : 148ull * 8));
    cudaFuncSetAttribute(k_bucket_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k_bucket_hist<<<grid, 1024, smem_hist ? B * 4 : 0, st>>>(d_keys, n, g, B, d_hist, smem_hist);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess) throw Error(RECSPLIT_E_CUDA, "bucket histogram launch failed");
}

void route_keys(const u64* d_keys, u64 n, u64 total, u32 bucket, u64 g, u32 world, const u64* cuts_in,
                cudaStream_t st, u64* d_out, u64* counts) {
    const u64 B = (total + bucket - 1) / bucket;  // R12, global
    std::vector<u64> cuts(world + 1);
    if (cuts_in) {
        if (cuts_in[0] != 0 || cuts_in[world] != B) throw Error(RECSPLIT_E_INVALID, "bucket_cuts must run from 0 to B");
        for (u32 r = 0; r <= world; ++r) {
            cuts[r] = cuts_in[r];
            if (r && cuts[r] < cuts[r - 1]) throw Error(RECSPLIT_E_INVALID, "bucket_cuts must be nondecreasing");
        }
    } else {
        for (u32 r = 0; r <= world; ++r) cuts[r] = B * r / world;
    }
    u64* d = nullptr;  // [counts W | cursors W | cuts W + 1]
    if (cudaMallocAsync(&d, 8 * (3 * (size_t)world + 1), st) != cudaSuccess) throw Error(RECSPLIT_E_NOMEM, "route buffer");
    struct Free {
        u64* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } fr{d, st};
    cudaMemsetAsync(d, 0, 8 * (size_t)world, st);
    cudaMemcpyAsync(d + 2 * world, cuts.data(), 8 * (world + 1), cudaMemcpyHostToDevice, st);
    const unsigned grid = (unsigned)std::max<u64>(1, std::min<u64>((n + 1023) / 1024, 148ull * 4));
    if (n) {
        k_route_count<<<grid, 1024, (2 * world + 1) * 8, st>>>(d_keys, n, g, B, world, d + 2 * world, d);
        g_launches++;
    }
    if (cudaMemcpyAsync(counts, d, 8 * (size_t)world, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        throw Error(RECSPLIT_E_CUDA, "route count failed");
    std::vector<u64> start(world, 0);
    for (u32 r = 1; r < world; ++r) start[r] = start[r - 1] + counts[r - 1];
    cudaMemcpyAsync(d + world, start.data(), 8 * (size_t)world, cudaMemcpyHostToDevice, st);
    if (n) {
        const unsigned g2 = (unsigned)std::max<u64>(1, std::min<u64>((n + 8191) / 8192, 148ull * 4));
        k_route_scatter<<<g2, 1024, (3 * world + 1) * 8, st>>>(d_keys, n, g, B, world, d + 2 * world, d + world, d_out);
        g_launches++;
    }
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        throw Error(RECSPLIT_E_CUDA, "route scatter failed");
}

}  // namespace rs

namespace rs {
using namespace rsd;

// ============================================================ two-level sort ==
//
// A2 as a two-level counting sort for the one-enqueue build (no per-key global atomics, every
// write of the second level coalesced).  Buckets are grouped by 2^gl consecutive bucket ids
// (gl chosen so that a group holds at most kGroupCap keys when every bucket is within the
// build's size bound S).  Level 0 counts the keys of each group (shared-memory histogram per
// block); a scan gives each group's start.  Level 1: each block takes a contiguous chunk of
// keys, counts its keys per group in shared memory, reserves its range inside every group
// with ONE global atomic per (block, group), and writes (lo, bucket-in-group | A/B << 8) to
// it.  Level 2: one block per group stages the group's keys in shared memory, counting-sorts
// them by bucket, writes them out in bucket order (coalesced) together with the bucket
// offsets C ("sort by bucket index, determine borders") and the max / min bucket size.
// Keys inside a bucket end up in an arbitrary order: every stored value depends only on the
// key set of its node.
namespace {

__device__ __forceinline__ u64 bucket_of(u64 key, u64 g, u64 B) {
    return ((remix64(key ^ g ^ MHC_SALT_HI) >> 32) * B) >> 32;
}

// level 0: block blk counts the keys of its chunk [blk0 + blk) * chunk ... per group into
// M[g * nb1 + blk] (group-major, so that one exclusive scan of M gives every (group, block)
// its output offset: no atomics on global memory)
__global__ void __launch_bounds__(1024) k_p2_count(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u32 gl, u32 G,
                                                   u64 chunk, u32 nb1, u32 blk0, u32* __restrict__ M) {
    extern __shared__ u32 hc[];
    const u32 blk = blk0 + blockIdx.x;
    const u64 k0 = (u64)blockIdx.x * chunk, k1 = min(n, k0 + chunk);  // (keys: this launch's first key)
    for (u32 i = threadIdx.x; i < G; i += blockDim.x) hc[i] = 0;
    __syncthreads();
    // (four keys in flight per thread: the loads are issued before the hashes and atomics)
    for (u64 i = k0 + threadIdx.x; i < k1; i += 4 * blockDim.x) {
        u64 kk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) kk[q] = i + q * blockDim.x < k1 ? keys[i + q * blockDim.x] : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (i + q * blockDim.x < k1) atomicAdd(hc + (u32)(bucket_of(kk[q], g, B) >> gl), 1u);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < G; i += blockDim.x) M[(u64)i * nb1 + blk] = hc[i];
}

// level 1: block blk writes its chunk's keys at the scanned offsets Ms[g * nb1 + blk] of their
// groups (the raw key: one 8-byte write per key; level 2 recomputes its master hash code)
__global__ void __launch_bounds__(1024) k_p2_scatter(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u32 gl,
                                                     u32 G, u64 chunk, u32 nb1, const u64* __restrict__ Ms,
                                                     u64* __restrict__ key1) {
    extern __shared__ u32 sc[];  // per group: this block's write cursor
    const u32 blk = blockIdx.x;
    const u64 k0 = (u64)blk * chunk, k1 = min(n, k0 + chunk);
    for (u32 i = threadIdx.x; i < G; i += blockDim.x) sc[i] = (u32)Ms[(u64)i * nb1 + blk];  // (n < 2^32)
    __syncthreads();
    for (u64 i = k0 + threadIdx.x; i < k1; i += 4 * blockDim.x) {
        u64 kk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) kk[q] = i + q * blockDim.x < k1 ? keys[i + q * blockDim.x] : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)  // (one 8-byte write per key)
            if (i + q * blockDim.x < k1) key1[atomicAdd(sc + (u32)(bucket_of(kk[q], g, B) >> gl), 1u)] = kk[q];
    }
}

// one block per group: counting sort by bucket in shared memory, coalesced output, offsets C,
// max / min bucket size (small[0], small[1]); a group above cap keys (a bucket above the
// build's bound S) sets small[5] and leaves its buckets empty (the build is redone on the
// synchronized path)
__global__ void __launch_bounds__(512) k_p2_group(const u64* __restrict__ key1, u64 g, const u64* __restrict__ Ms,
                                                  u32 nb1, u64 B, u32 gl, u32 G, u32 cap, u64* __restrict__ C,
                                                  u64* __restrict__ lo_a, u8* __restrict__ ab_a, u32* small, u32 dts) {
    extern __shared__ __align__(16) unsigned char p2s[];
    const u32 gb = 1u << gl;
    u32* cnt = reinterpret_cast<u32*>(p2s);  // gb counts -> exclusive offsets
    u32* cur = cnt + gb;                     // gb write cursors
    u64* lo_s = reinterpret_cast<u64*>(p2s + ((8u * gb + 15u) & ~15u));
    u8* ab_s = reinterpret_cast<u8*>(lo_s + cap);
    // (dts > 0: the duplicate check is fused here -- per warp an open-addressing set of indices
    // into lo_s, dts entries, after the staged keys)
    u32* dtab = reinterpret_cast<u32*>(p2s + ((((8u * gb + 15u) & ~15u) + (size_t)cap * 9 + 15u) & ~(size_t)15u)) +
                (threadIdx.x >> 5) * dts;
    bool rep = false;
    u32 zeros = 0;
    for (u32 grp = blockIdx.x; grp < G; grp += gridDim.x) {
        const u64 gs = Ms[(u64)grp * nb1], ge = Ms[(u64)(grp + 1) * nb1];  // (Ms[G * nb1] = n)
        const u64 b0 = (u64)grp << gl;
        const u32 nb = (u32)min((u64)gb, B - b0);
        const u32 cg = (u32)(ge - gs);
        if (grp == G - 1 && threadIdx.x == 0) C[B] = ge;
        __syncthreads();
        if (cg > cap) {
            if (threadIdx.x == 0) atomicOr(small + 5, 1u);
            for (u32 j = threadIdx.x; j < nb; j += blockDim.x) C[b0 + j] = gs;
            continue;
        }
        for (u32 j = threadIdx.x; j < gb; j += blockDim.x) cnt[j] = 0;
        __syncthreads();
        const u32 lmask = gb - 1u;
        for (u32 i = threadIdx.x; i < cg; i += 2 * blockDim.x) {
            const u64 ka = key1[gs + i], kb = i + blockDim.x < cg ? key1[gs + i + blockDim.x] : 0;
            atomicAdd(cnt + ((u32)bucket_of(ka, g, B) & lmask), 1u);
            if (i + blockDim.x < cg) atomicAdd(cnt + ((u32)bucket_of(kb, g, B) & lmask), 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive scan of gb <= 256 counts by one warp; sizes' max / min
            const u32 lane = threadIdx.x;
            u32 carry = 0, mx = 0, mn = 0xffffffffu;
            for (u32 base = 0; base < gb; base += 32) {
                const u32 j = base + lane;
                const u32 v = j < gb ? cnt[j] : 0;
                if (j < nb) {
                    mx = max(mx, v);
                    mn = min(mn, v);
                }
                u32 inc = v;
                for (int d = 1; d < 32; d <<= 1) {
                    const u32 t = __shfl_up_sync(FULL, inc, d);
                    if ((int)lane >= d) inc += t;
                }
                if (j < gb) {
                    cnt[j] = carry + inc - v;
                    cur[j] = carry + inc - v;
                }
                carry += __shfl_sync(FULL, inc, 31);
            }
            for (int d = 16; d; d >>= 1) {
                mx = max(mx, __shfl_xor_sync(FULL, mx, d));
                mn = min(mn, __shfl_xor_sync(FULL, mn, d));
            }
            if (lane == 0 && nb) {
                atomicMax(small, mx);
                atomicMin(small + 1, mn);
            }
        }
        __syncthreads();
        for (u32 j = threadIdx.x; j < nb; j += blockDim.x) C[b0 + j] = gs + cnt[j];
        for (u32 i = threadIdx.x; i < cg; i += blockDim.x) {  // A1: lo, A/B bit (R2, R7)
            const u64 k = key1[gs + i] ^ g;
            const u64 h = remix64(k ^ MHC_SALT_HI);
            const u32 pos = atomicAdd(cur + ((u32)(((h >> 32) * B) >> 32) & lmask), 1u);
            lo_s[pos] = remix64(k ^ MHC_SALT_LO);
            ab_s[pos] = (u8)(h & 1);
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < cg; i += blockDim.x) {
            lo_a[gs + i] = lo_s[i];
            ab_a[gs + i] = ab_s[i];
        }
        if (dts) {  // A2 duplicate check: equal keys have equal lo (R2) and share a bucket
            const u32 lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (u32 j = threadIdx.x >> 5; j < nb; j += nw) {
                const u32 b0 = cnt[j], b1 = j + 1 < gb ? cnt[j + 1] : cg;
                if (b1 - b0 < 2) continue;
                for (u32 t = lane; t < dts; t += 32) dtab[t] = 0xffffffffu;
                __syncwarp();
                for (u32 i = b0 + lane; i < b1; i += 32) {
                    const u64 v = lo_s[i];
                    if (v == 0) {  // (0 is not special here, but counted like k_dedupe does)
                        ++zeros;
                        continue;
                    }
                    u32 slot = (u32)(v ^ (v >> 32)) & (dts - 1);
                    for (;;) {
                        const u32 old = atomicCAS(dtab + slot, 0xffffffffu, i);
                        if (old == 0xffffffffu) break;
                        if (lo_s[old] == v) {
                            rep = true;
                            break;
                        }
                        slot = (slot + 1) & (dts - 1);
                    }
                }
                __syncwarp();
            }
        }
    }
    if (dts) {
        if (rep) atomicOr(small + 2, 1u);
        if (zeros) atomicAdd(small + 3, zeros);
    }
}

}  // namespace

bool partition2_shape(u64 n, u64 B, u32 S, P2Shape& sh) {
    if (n == 0 || B == 0 || S == 0 || S > kGroupCap || n >= (1ull << 32)) return false;
    u32 gl = 0;
    while (gl < 8 && (2ull << gl) * S <= kGroupCap) ++gl;
    const u64 G = (B + (1ull << gl) - 1) >> gl;
    // (many groups: the (group, block) count matrix and the level-1 blocks' short runs per
    // group cost more than the one-level scatter -- C5, G = 12,500: 6.0 vs 4.9 ms, pass W)
    if (G > kGroupMax) return false;
    sh.gl = gl;
    sh.G = (u32)G;
    sh.cap = (u32)std::min<u64>(kGroupCap, (u64)S << gl);
    // keys per level-1 block: about 4 blocks per SM (592), at least 8192
    sh.chunk = std::max<u64>(8192, ((n + 591) / 592 + 1023) & ~1023ull);
    sh.nb1 = (u32)((n + sh.chunk - 1) / sh.chunk);
    if ((u64)sh.G * sh.nb1 > (1ull << 28)) return false;
    return true;
}

void launch_p2_count(const u64* keys, u64 n, u64 first_key, u64 g, u64 B, const P2Shape& sh, u32* M, cudaStream_t st) {
    if (!n) return;
    // (first_key: a multiple of the chunk -- the chunked host->device copy hands over whole chunks)
    const u32 blk0 = (u32)(first_key / sh.chunk);
    const unsigned grid = (unsigned)((n + sh.chunk - 1) / sh.chunk);
    cudaFuncSetAttribute(k_p2_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_p2_count<<<grid, 1024, (size_t)sh.G * 4, st>>>(keys, n, g, B, sh.gl, sh.G, sh.chunk, sh.nb1, blk0, M);
    g_launches++;
}

void launch_p2_scatter(const u64* keys, u64 n, u64 g, u64 B, const P2Shape& sh, const u64* Ms, u64* key1,
                       cudaStream_t st) {
    cudaFuncSetAttribute(k_p2_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_p2_scatter<<<sh.nb1, 1024, (size_t)sh.G * 4, st>>>(keys, n, g, B, sh.gl, sh.G, sh.chunk, sh.nb1, Ms, key1);
    g_launches++;
}

void launch_p2_group(const u64* key1, u64 g, u64 B, const P2Shape& sh, const u64* Ms, u64* C, u64* lo_a, u8* ab_a,
                     u32* small, cudaStream_t st, u32 dts) {
    const size_t smem = ((((8u * (1u << sh.gl) + 15u) & ~15u) + (size_t)sh.cap * 9 + 15u) & ~(size_t)15u) +
                        (size_t)dts * 4 * (512 / 32);
    cudaFuncSetAttribute(k_p2_group, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2_group, 512, smem);
    const unsigned grid = (unsigned)std::max<u64>(1, std::min<u64>(sh.G, 148ull * std::max(occ, 1)));
    k_p2_group<<<grid, 512, smem, st>>>(key1, g, Ms, sh.nb1, B, sh.gl, sh.G, sh.cap, C, lo_a, ab_a, small, dts);
    g_launches++;
}

}  // namespace rs
