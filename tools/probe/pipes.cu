// Per-pipe INT32 throughput probe (VERDICT r1 "measure the denominators"): warp-instruction
// throughput per SM per clock of the integer SASS instructions the search loops issue --
// IMAD, IMAD.WIDE, IMAD.HI, IADD3, LOP3, SHF, BMSK, LDS, POPC -- alone and in pairs.
//
// Each kernel k_pipe<A, NA, B, NB> runs 8 independent dependency chains per thread; the
// loop body (one iteration, not unrolled) applies NA ops of kind A then NB ops of kind B to
// every chain.  ptxas decides the SASS, so tools/probe/pipes.py counts the opcodes of each
// kernel's loop body from cuobjdump and divides the executed warp instructions by the
// measured cycles.  One wave: 4 blocks x 256 threads per SM (32 warps per SM, 8 per
// scheduler).  Each block records clock64() around its loop; throughput = (warp instructions
// of an SM's 4 blocks) / (the slowest block's span in SM clocks), independent of the clock.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe/pipes.cu -o pipes
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

enum Op { IMAD = 0, IMADW, IMADHI, IADD, LOP3, SHF, BMSK, LDS, POPC, NONE_OP };

// Chain state: x for the 32-bit ops, y (64-bit) for IMAD.WIDE, z (a shared address) for
// LDS, (u, v) for IADD3 (two adds feeding each other, so ptxas cannot fold them into a
// multiply); operands a, b are kernel arguments.
struct St {
    uint32_t x, z, u, v;
    uint64_t y;
};

template <int OP>
__device__ __forceinline__ void op(St& s, uint32_t a, uint32_t b) {
    if (OP == IMAD) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(s.x) : "r"(a), "r"(b));
    } else if (OP == IMADW) {
        // both halves of the product feed the next op (else ptxas keeps only the low word,
        // IMAD): one LOP3 per IMAD.WIDE, on the other pipe
        asm volatile("{\n\t.reg .u32 l, h;\n\tmov.b64 {l, h}, %0;\n\txor.b32 l, l, h;\n\tmul.wide.u32 %0, l, %1;\n\t}"
                     : "+l"(s.y) : "r"(a));
    } else if (OP == IMADHI) {
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(s.x) : "r"(a), "r"(b));
    } else if (OP == IADD) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(s.u) : "r"(s.v));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(s.v) : "r"(s.u));
    } else if (OP == LOP3) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(s.x) : "r"(a), "r"(b));
    } else if (OP == SHF) {
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 13;" : "+r"(s.x) : "r"(a));
    } else if (OP == BMSK) {
        asm volatile("bmsk.clamp.b32 %0, %0, %1;" : "+r"(s.x) : "r"(a));
    } else if (OP == LDS) {
        asm volatile("ld.shared.u32 %0, [%0];" : "+r"(s.z));
    } else if (OP == POPC) {
        asm volatile("popc.b32 %0, %0;" : "+r"(s.x));
    }
}

template <int A, int NA, int B, int NB>
__global__ void __launch_bounds__(256) k_pipe(uint32_t iters, uint32_t a, uint32_t b, uint32_t* sink,
                                              long long* cyc) {
    __shared__ uint32_t sm[1024];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = base + 4 * ((i * 97 + 13) & 1023);
    __syncthreads();
    St st[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        st[c].x = threadIdx.x * 8 + c + a;
        st[c].y = st[c].x | 1;
        st[c].z = base + 4 * ((threadIdx.x * 8 + c) & 1023);
        st[c].u = st[c].x;
        st[c].v = b + c;
    }
    const long long t0 = clock64();
#pragma unroll 1
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
#pragma unroll
                for (int k = 0; k < NA; ++k) op<A>(st[c], a, b);
#pragma unroll
                for (int k = 0; k < NB; ++k) op<B>(st[c], a, b);
            }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc ^= st[c].x ^ st[c].z ^ st[c].u ^ st[c].v ^ (uint32_t)st[c].y ^ (uint32_t)(st[c].y >> 32);
    if (acc == 0x9e3779b9u) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

constexpr uint32_t kIters = 2048;

struct Result {
    const char* name;
    int a, na, b, nb;
    double max_block_cycles;  // the slowest block's clock64 span (one wave, 4 blocks per SM)
    double ms;
};

template <int A, int NA, int B, int NB>
Result run(const char* name, int sms, uint32_t* sink, long long* cyc) {
    const int blocks = sms * 4, threads = 256;
    const uint32_t iters = kIters;
    k_pipe<A, NA, B, NB><<<blocks, threads>>>(16, 3, 5, sink, cyc);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_pipe<A, NA, B, NB><<<blocks, threads>>>(iters, 0x9e3779b1u, 0x7f4a7c15u, sink, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(blocks);
    cudaMemcpy(c.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long v : c) mx = v > mx ? v : mx;
    return {name, A, NA, B, NB, (double)mx, ms};
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    long long* cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sizeof(long long) * sms * 4);
    std::vector<Result> R;
    R.push_back(run<IMAD, 4, NONE_OP, 0>("IMAD", sms, sink, cyc));
    R.push_back(run<IMADW, 4, NONE_OP, 0>("IMAD.WIDE", sms, sink, cyc));
    R.push_back(run<IMADHI, 4, NONE_OP, 0>("IMAD.HI", sms, sink, cyc));
    R.push_back(run<IADD, 4, NONE_OP, 0>("IADD3", sms, sink, cyc));
    R.push_back(run<LOP3, 4, NONE_OP, 0>("LOP3", sms, sink, cyc));
    R.push_back(run<SHF, 4, NONE_OP, 0>("SHF", sms, sink, cyc));
    R.push_back(run<BMSK, 4, NONE_OP, 0>("BMSK", sms, sink, cyc));
    R.push_back(run<LDS, 4, NONE_OP, 0>("LDS", sms, sink, cyc));
    R.push_back(run<POPC, 4, NONE_OP, 0>("POPC", sms, sink, cyc));
    R.push_back(run<IMAD, 1, LOP3, 1>("IMAD+LOP3", sms, sink, cyc));
    R.push_back(run<IMAD, 1, SHF, 1>("IMAD+SHF", sms, sink, cyc));
    R.push_back(run<IMAD, 1, IADD, 1>("IMAD+IADD3", sms, sink, cyc));
    R.push_back(run<IMADW, 1, LOP3, 1>("IMAD.WIDE+LOP3", sms, sink, cyc));
    R.push_back(run<IMADW, 1, LOP3, 2>("IMAD.WIDE+2LOP3", sms, sink, cyc));
    R.push_back(run<IMADHI, 1, LOP3, 1>("IMAD.HI+LOP3", sms, sink, cyc));
    R.push_back(run<IMADHI, 1, SHF, 2>("IMAD.HI+2SHF", sms, sink, cyc));
    R.push_back(run<IMADW, 1, IMAD, 1>("IMAD.WIDE+IMAD", sms, sink, cyc));
    R.push_back(run<LOP3, 1, SHF, 1>("LOP3+SHF", sms, sink, cyc));
    R.push_back(run<LDS, 1, LOP3, 2>("LDS+2LOP3", sms, sink, cyc));
    R.push_back(run<LDS, 1, IMAD, 2>("LDS+2IMAD", sms, sink, cyc));
    R.push_back(run<BMSK, 1, IMAD, 1>("BMSK+IMAD", sms, sink, cyc));
    R.push_back(run<POPC, 1, LOP3, 3>("POPC+3LOP3", sms, sink, cyc));
    printf("[\n");
    for (size_t i = 0; i < R.size(); ++i)
        printf("  {\"kernel\": \"%s\", \"a\": %d, \"na\": %d, \"b\": %d, \"nb\": %d, \"iters\": %u, "
               "\"warps_per_sm\": 32, \"max_block_cycles\": %.0f, \"ms\": %.3f}%s\n",
               R[i].name, R[i].a, R[i].na, R[i].b, R[i].nb, kIters, R[i].max_block_cycles, R[i].ms,
               i + 1 < R.size() ? "," : "");
    printf("]\n");
    fprintf(stderr, "%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
