// Steps A1-A2: master hash codes, bucket assignment, counting sort by
// bucket, per-bucket sort by MHC.hi with duplicate detection.
// P:106-108 (initial hash, buckets of expected size b), P:319 (sort by bucket index,
// determine borders), P:389 (random integers as MHC).
#include "kernels.h"

namespace rs {

using namespace rsd;

// A1: hi = remix(key^g^salt_hi), lo = remix(key^g^salt_lo) (R2); bucket = remap(hi, B) (R3).
__global__ void k_hash(const u64* __restrict__ keys, u64 n, u64 g, u64 B, u64* __restrict__ hi,
                       u64* __restrict__ lo, u32* __restrict__ bkt, u32* __restrict__ hist) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 k = keys[i] ^ g;
        const u64 h = remix64(k ^ MHC_SALT_HI);
        const u64 l = remix64(k ^ MHC_SALT_LO);
        const u32 b = (u32)(((h >> 32) * B) >> 32);
        hi[i] = h;
        lo[i] = l;
        bkt[i] = b;
        atomicAdd(hist + b, 1u);
    }
}

void launch_hash(const u64* keys, u64 n, u64 g, u64 B, u64* hi, u64* lo, u32* bkt, u32* hist,
                 cudaStream_t st) {
    unsigned grid = (unsigned)((n + 255) / 256);
    if (grid > 148u * 16u) grid = 148u * 16u;
    if (grid == 0) grid = 1;
    k_hash<<<grid, 256, 0, st>>>(keys, n, g, B, hi, lo, bkt, hist);
    g_launches++;
}

__global__ void k_bucket_stats(const u32* __restrict__ hist, u64 B, u32* maxmin, u8* present, u32 cap) {
    u32 mx = 0, mn = 0xffffffffu;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (u64)gridDim.x * blockDim.x) {
        u32 s = hist[i];
        mx = s > mx ? s : mx;
        mn = s < mn ? s : mn;
        present[s <= cap ? s : cap] = 1;
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

void launch_bucket_stats(const u32* hist, u64 B, u32* maxmin, u8* present, u32 cap, cudaStream_t st) {
    unsigned grid = (unsigned)((B + 255) / 256);
    if (grid > 1024) grid = 1024;
    if (grid == 0) grid = 1;
    k_bucket_stats<<<grid, 256, 0, st>>>(hist, B, maxmin, present, cap);
    g_launches++;
}

// Counting-sort scatter: each key to its bucket's next free slot (order within a bucket
// is fixed afterwards by the per-bucket sort).
__global__ void k_scatter(const u64* __restrict__ hi, const u64* __restrict__ lo, const u32* __restrict__ bkt,
                          u64 n, u64* __restrict__ cursor, u64* __restrict__ hi2, u64* __restrict__ lo2) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 p = atomicAdd((unsigned long long*)cursor + bkt[i], 1ull);
        hi2[p] = hi[i];
        lo2[p] = lo[i];
    }
}

void launch_scatter(const u64* hi, const u64* lo, const u32* bkt, u64 n, u64* cursor, u64* hi2, u64* lo2,
                    cudaStream_t st) {
    unsigned grid = (unsigned)((n + 255) / 256);
    if (grid > 148u * 16u) grid = 148u * 16u;
    if (grid == 0) grid = 1;
    k_scatter<<<grid, 256, 0, st>>>(hi, lo, bkt, n, cursor, hi2, lo2);
    g_launches++;
}

// One block per bucket: bitonic sort of (hi, lo) by (hi, pad flag) in shared memory,
// duplicate check on adjacent hi (R2: hi is a bijection of the key), then write lo and
// the A/B bit (R7: hi & 1) in sorted order.
__global__ void __launch_bounds__(512) k_bucket_sort(const u64* __restrict__ hi2, const u64* __restrict__ lo2,
                                                     const u64* __restrict__ C, u64* __restrict__ lo_s,
                                                     u8* __restrict__ ab_s, u32* dup, u64 B) {
    extern __shared__ __align__(16) unsigned char sm[];
  for (u64 b = blockIdx.x; b < B; b += gridDim.x) {
    const u32 base = (u32)C[b];
    const u32 s = (u32)(C[b + 1] - base);
    __syncthreads();
    if (s == 0) continue;
    u32 P = 1;
    while (P < s) P <<= 1;
    u64* sh = (u64*)sm;
    u64* sl = sh + P;
    u8* pad = (u8*)(sl + P);
    for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < s) {
            sh[i] = hi2[base + i];
            sl[i] = lo2[base + i];
            pad[i] = 0;
        } else {
            sh[i] = ~0ull;
            sl[i] = 0;
            pad[i] = 1;
        }
    }
    __syncthreads();
    for (u32 k = 2; k <= P; k <<= 1) {
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
                u32 ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const u64 a = sh[i], c = sh[ixj];
                    const bool gt = a > c || (a == c && pad[i] > pad[ixj]);
                    if (gt == up) {
                        sh[i] = c;
                        sh[ixj] = a;
                        u64 t = sl[i];
                        sl[i] = sl[ixj];
                        sl[ixj] = t;
                        u8 q = pad[i];
                        pad[i] = pad[ixj];
                        pad[ixj] = q;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (u32 i = threadIdx.x; i < s; i += blockDim.x) {
        if (i > 0 && sh[i] == sh[i - 1]) atomicOr(dup, 1u);
        lo_s[base + i] = sl[i];
        ab_s[base + i] = (u8)(sh[i] & 1);
    }
  }
}

void launch_bucket_sort(const u64* hi2, const u64* lo2, const u64* C, u64 B, u32 smax, u64* lo_s, u8* ab_s,
                        u32* dup, cudaStream_t st) {
    u32 P = 1;
    while (P < smax) P <<= 1;
    size_t smem = (size_t)P * 17;
    cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    u32 threads = P >= 512 ? 512 : (P >= 128 ? P : 128);
    unsigned grid = B < 0x7fffffffull ? (unsigned)B : 0x7fffffffu;
    k_bucket_sort<<<grid, threads, smem, st>>>(hi2, lo2, C, lo_s, ab_s, dup, B);
    g_launches++;
}

}  // namespace rs
