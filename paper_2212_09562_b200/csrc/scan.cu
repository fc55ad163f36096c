// Device-wide exclusive prefix sum (reduce-then-scan, three launches).
// Used for bucket offsets C[] (P:135 prefix sums of bucket sizes), bit offsets P[],
// and node-table offsets.
#include "kernels.h"

namespace rs {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kTile = kScanThreads * kScanItems;

__device__ __forceinline__ u64 warp_incl_scan(u64 v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u64 t = rsd::shfl64(v, (lane - d) & 31);
        if (lane >= d) v += t;
    }
    return v;
}

template <typename T>
__global__ void k_tile_sums(const T* in, size_t n, u64* sums) {
    size_t base = (size_t)blockIdx.x * kTile;
    u64 acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        size_t i = base + (size_t)k * kScanThreads + threadIdx.x;
        if (i < n) acc += (u64)in[i];
    }
    // block reduce
    __shared__ u64 red[32];
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(rsd::FULL, acc, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        u64 v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(rsd::FULL, v, d);
        if (threadIdx.x == 0) sums[blockIdx.x] = v;
    }
}

// single block: exclusive scan of nb tile sums in place; grand total to *total
__global__ void k_scan_sums(u64* sums, size_t nb, u64* total) {
    __shared__ u64 carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (size_t base = 0; base < nb; base += blockDim.x) {
        size_t i = base + threadIdx.x;
        u64 v = i < nb ? sums[i] : 0;
        // inclusive scan within block
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        __shared__ u64 ws[32];
        u64 inc = warp_incl_scan(v);
        if (lane == 31) ws[w] = inc;
        __syncthreads();
        if (w == 0) {
            u64 x = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
            u64 xi = warp_incl_scan(x);
            ws[lane] = xi - x;
        }
        __syncthreads();
        u64 excl = carry + ws[w] + inc - v;
        if (i < nb) sums[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

template <typename T>
__global__ void k_scan_apply(const T* in, u64* out, size_t n, const u64* sums) {
    __shared__ u64 ws[32];
    __shared__ u64 carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = sums[blockIdx.x];
    __syncthreads();
    size_t base = (size_t)blockIdx.x * kTile;
    for (int k = 0; k < kScanItems; ++k) {
        size_t i = base + (size_t)k * kScanThreads + threadIdx.x;
        u64 v = i < n ? (u64)in[i] : 0;
        u64 inc = warp_incl_scan(v);
        if (lane == 31) ws[w] = inc;
        __syncthreads();
        if (w == 0) {
            u64 x = ws[lane];
            u64 xi = warp_incl_scan(x);
            ws[lane] = xi - x;
        }
        __syncthreads();
        u64 excl = carry + ws[w] + inc - v;
        if (i < n) out[i] = excl;
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) carry = excl + v;
        __syncthreads();
    }
}

template <typename T>
void exscan_impl(const T* in, u64* out, size_t n, void* temp, cudaStream_t st) {
    size_t nb = (n + kTile - 1) / kTile;
    if (nb == 0) nb = 1;
    u64* sums = (u64*)temp;
    k_tile_sums<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, sums);
    k_scan_sums<<<1, kScanThreads, 0, st>>>(sums, nb, out + n);
    k_scan_apply<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, sums);
    g_launches += 3;
}

}  // namespace

size_t scan_temp_bytes(size_t n) { return ((n + kTile - 1) / kTile + 1) * sizeof(u64); }

void exscan_u32_to_u64(const u32* in, u64* out, size_t n, void* temp, cudaStream_t st) {
    exscan_impl<u32>(in, out, n, temp, st);
}
void exscan_u64(const u64* in, u64* out, size_t n, void* temp, cudaStream_t st) {
    exscan_impl<u64>(in, out, n, temp, st);
}

}  // namespace rs
