// INT32 ceiling probe (measures the roofline denominator instead of deriving it): the hot
// loop of the lower-level-1 search -- four keys per iteration from warp-private shared memory
// in the AoSoA layout, remix_hi_nc (no-carry SplitMix64 high word), part = hi(h * f), shift
// table in static shared memory, packed-counter increment -- with no early rejection, no
// window logic and no global memory in the loop.  Same block shape and occupancy as
// k_search<SK_LOWER> (128 threads, 8 blocks per SM).  Prints evaluations/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I paper_2212_09562_b200/csrc tools/probe/int32_probe.cu -o int32_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

using namespace rsd;

__shared__ __align__(16) unsigned char s_tab[32];

__global__ void __launch_bounds__(128, 8) k_probe(const uint32_t* __restrict__ keys, uint32_t s, uint32_t f,
                                                  uint32_t iters, uint32_t* sink) {
    __shared__ __align__(16) uint32_t G[4][12 * 32];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < 32) s_tab[threadIdx.x] = (unsigned char)(threadIdx.x + 1 < f ? threadIdx.x * 5 : 32);
    for (uint32_t j = lane; j < s; j += 32) {
        const uint32_t kl = keys[2 * j], kh = keys[2 * j + 1];
        G[w][12 * (j >> 2) + (j & 3)] = kl;
        G[w][12 * (j >> 2) + 4 + (j & 3)] = kh;
        G[w][12 * (j >> 2) + 8 + (j & 3)] = key_const(kh);
    }
    __syncthreads();
    uint32_t acc = 0;
    const uint32_t base = (blockIdx.x * 4 + w) * 32 * iters;
    for (uint32_t it = 0; it < iters; ++it) {
        const uint32_t sigma = base + it * 32 + lane;
        uint32_t c0 = 0, c1 = 0;
        const uint32_t* g = G[w];
#pragma unroll 1
        for (uint32_t q = 0; q < s / 4; ++q, g += 12) {
            const uint4 kl = *reinterpret_cast<const uint4*>(g);
            const uint4 kh = *reinterpret_cast<const uint4*>(g + 4);
            const uint4 kc = *reinterpret_cast<const uint4*>(g + 8);
            const uint32_t h0 = remix_hi_nc(kl.x, kh.x, kc.x, sigma), h1 = remix_hi_nc(kl.y, kh.y, kc.y, sigma);
            const uint32_t h2 = remix_hi_nc(kl.z, kh.z, kc.z, sigma), h3 = remix_hi_nc(kl.w, kh.w, kc.w, sigma);
            c0 += bit_clamp(s_tab[__umulhi(h0, f)]) + bit_clamp(s_tab[__umulhi(h1, f)]);
            c1 += bit_clamp(s_tab[__umulhi(h2, f)]) + bit_clamp(s_tab[__umulhi(h3, f)]);
        }
        acc ^= c0 + c1;
    }
    if (acc == 0x12345678u) sink[0] = acc;  // keeps the loop alive
}

int main() {
    const uint32_t s = 112, f = 7, iters = 4096;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t h[2 * 112];
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (uint32_t j = 0; j < 2 * s; ++j) {  // keys with k_lo small enough for the no-carry path
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[j] = (j & 1) ? (uint32_t)(x >> 32) : ((uint32_t)x & 0x7fffffffu);
    }
    uint32_t *d_keys, *d_sink;
    cudaMalloc(&d_keys, sizeof h);
    cudaMalloc(&d_sink, 4);
    cudaMemcpy(d_keys, h, sizeof h, cudaMemcpyHostToDevice);
    const int blocks = sms * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_probe<<<blocks, 128>>>(d_keys, s, f, 64, d_sink);  // warm-up
    cudaEventRecord(a);
    k_probe<<<blocks, 128>>>(d_keys, s, f, iters, d_sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double evals = (double)blocks * 128 * iters * s;
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    printf("{\"probe\": \"int32\", \"sms\": %d, \"blocks\": %d, \"ms\": %.3f, \"evals_per_s\": %.4e, "
           "\"evals_per_clk_per_sm_at_1965MHz\": %.3f, \"err\": \"%s\"}\n",
           sms, blocks, ms, evals / (ms * 1e-3), evals / (ms * 1e-3) / (sms * 1965e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
