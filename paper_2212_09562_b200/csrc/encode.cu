// Node-table expansion (A3) and encoding (A10-A11):
//  * every bucket's tree is instantiated from the per-size preorder template (the
//    tree shape depends only on l and s);
//  * Golomb-Rice per bucket: fixed parts of all nodes in preorder, then unary parts
//    (P:130-134), buckets concatenated into one bit vector;
//  * trend-subtracted Elias-Fano index over bucket key offsets C and bit offsets P
//    (reading R13).
#include "kernels.h"

namespace rs {

using namespace rsd;

// M[r * (B+1) + i]: r = 0 -> N(s_i) nodes; r = 1+p -> nodes of phase p; column B = 0.
__global__ void k_bucket_counts(const u64* __restrict__ C, u64 B, const u32* __restrict__ N,
                                const u32* __restrict__ phase_cnt, u32 NP, u64* __restrict__ M) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= B; i += (u64)gridDim.x * blockDim.x) {
        const u32 s = i < B ? (u32)(C[i + 1] - C[i]) : 0;
        M[i] = N[s];
        for (u32 p = 0; p < NP; ++p) M[(u64)(p + 1) * (B + 1) + i] = phase_cnt[(u64)s * NP + p];
    }
}

void launch_bucket_counts(const u64* C, u64 B, const u32* N, const u32* phase_cnt, u32 NP, u64* M,
                          cudaStream_t st) {
    unsigned grid = (unsigned)((B + 256) / 256);
    if (grid > 4096) grid = 4096;
    k_bucket_counts<<<grid, 256, 0, st>>>(C, B, N, phase_cnt, NP, M);
    g_launches++;
}

struct PhaseOff {
    u64 v[32];
};

// One warp per bucket: node j of the template of size s_i gets slot nodebase_i + j
// and lands at phase_off[p] + (phase-p prefix of bucket i) + phase_rank.
__global__ void k_expand(const u64* __restrict__ C, u64 B, const u64* __restrict__ Ms, u32 NP,
                         const u32* __restrict__ tstart, const TNodeD* __restrict__ tn, PhaseOff off,
                         NodeRec* __restrict__ nodes) {
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        const u32 s = (u32)(C[i + 1] - C[i]);
        if (s == 0) continue;
        const u64 base = Ms[i], row0 = Ms[0];
        const u32 t0 = tstart[s], t1 = tstart[s + 1];
        for (u32 t = t0 + lane; t < t1; t += 32) {
            const TNodeD x = tn[t];
            const u64 prow = (u64)(x.phase + 1) * (B + 1);
            const u64 pos = off.v[x.phase] + (Ms[prow + i] - Ms[prow]) + x.phase_rank;
            NodeRec r;
            r.key_off = (u32)(C[i] + x.rel_off);
            r.size = x.size;
            r.slot = (u32)(base - row0 + (t - t0));
            r.pad = 0;
            nodes[pos] = r;
        }
    }
}

void launch_expand(const u64* C, u64 B, const u64* Mscan, u32 NP, const u32* tstart, const TNodeD* tnodes,
                   const u64* phase_off, NodeRec* nodes, cudaStream_t st) {
    PhaseOff o;
    for (u32 p = 0; p < 32; ++p) o.v[p] = p < NP ? phase_off[p] : 0;
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_expand<<<grid, 256, 0, st>>>(C, B, Mscan, NP, tstart, tnodes, o, nodes);
    g_launches++;
}

// --------------------------------------------------------------- encoding --

// One warp per bucket: len_i = F(s) + sum_j (x_j >> tau_j) + N(s).  Also the
// algorithmic evaluation counts (sequential-search work implied by the values).
__global__ void k_bucket_bits(const u64* __restrict__ C, u64 B, const u64* __restrict__ nodebase,
                              const u32* __restrict__ tstart, const TNodeD* __restrict__ tn,
                              const u64* __restrict__ F, const u64* __restrict__ values, u32 leaf, u32 u1,
                              u32 u2, int rf, u64* __restrict__ len, unsigned long long* evals) {
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    unsigned long long ev[4] = {0, 0, 0, 0};
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        const u32 s = (u32)(C[i + 1] - C[i]);
        u64 acc = 0;
        if (s) {
            const u32 t0 = tstart[s], t1 = tstart[s + 1];
            const u64 nb = nodebase[i] - nodebase[0];
            for (u32 t = t0 + lane; t < t1; t += 32) {
                const TNodeD x = tn[t];
                const u64 v = values[nb + (t - t0)];
                acc += (v >> x.tau) + 1;
                const u32 cs = x.size;
                if (cs <= leaf) {
                    // RF: (floor(v/m) + 1) base seeds of m evaluations (32-bit division when it fits)
                    const u64 k = v < (1ull << 32) ? (u64)((u32)v / cs) : v / cs;
                    ev[3] += rf ? (k + 1) * cs : (v + 1) * cs;
                } else {
                    ev[cs > u2 ? 0 : cs > u1 ? 1 : 2] += (v + 1) * cs;
                }
            }
            for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(FULL, acc, d);
            acc += F[s];
        }
        if (lane == 0) len[i] = acc;
    }
    // block-level reduction, then one atomic per block and class
    __shared__ unsigned long long red[4];
    if (threadIdx.x < 4) red[threadIdx.x] = 0;
    __syncthreads();
    for (int c = 0; c < 4; ++c) {
        unsigned long long v = ev[c];
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
        if (lane == 0 && v) atomicAdd(red + c, v);
    }
    __syncthreads();
    if (threadIdx.x < 4 && red[threadIdx.x]) atomicAdd(evals + threadIdx.x, red[threadIdx.x]);
}

void launch_bucket_bits(const u64* C, u64 B, const u64* nodebase, const u32* tstart, const TNodeD* tnodes,
                        const u64* F, const u64* values, u32 leaf, u32 u1, u32 u2, int rf, u64* len,
                        unsigned long long* evals, cudaStream_t st) {
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_bucket_bits<<<grid, 256, 0, st>>>(C, B, nodebase, tstart, tnodes, F, values, leaf, u1, u2, rf, len, evals);
    g_launches++;
}

// OR `width` (<= 64) low bits of x into the bit vector at bit position pos.
__device__ __forceinline__ void or_bits(unsigned long long* words, u64 pos, u64 x, u32 width) {
    if (width == 0) return;
    if (width < 64) x &= (1ull << width) - 1;
    if (!x) return;
    const u64 wi = pos >> 6;
    const u32 sh = (u32)(pos & 63);
    atomicOr(words + wi, (unsigned long long)(x << sh));
    if (sh && sh + width > 64) atomicOr(words + wi + 1, (unsigned long long)(x >> (64 - sh)));
}

// One warp per bucket: fixed parts at P_i + fixed_off, unary terminators at
// P_i + F(s) + (exclusive prefix of q+1) + q.
__global__ void k_write_data(const u64* __restrict__ C, u64 B, const u64* __restrict__ nodebase,
                             const u32* __restrict__ tstart, const TNodeD* __restrict__ tn,
                             const u64* __restrict__ F, const u64* __restrict__ values, const u64* __restrict__ P,
                             unsigned long long* __restrict__ words) {
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    const u32 lt = lanemask_lt();
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        const u32 s = (u32)(C[i + 1] - C[i]);
        if (s == 0) continue;
        const u32 t0 = tstart[s], t1 = tstart[s + 1];
        const u64 nb = nodebase[i] - nodebase[0];
        const u64 pi = P[i] - P[0];
        u64 ucur = pi + F[s];
        for (u32 tb = t0; tb < t1; tb += 32) {
            const u32 t = tb + lane;
            u64 q1 = 0;
            u64 v = 0;
            TNodeD x{};
            if (t < t1) {
                x = tn[t];
                v = values[nb + (t - t0)];
                q1 = (v >> x.tau) + 1;
                or_bits(words, pi + x.fixed_off, v, x.tau);
            }
            // exclusive warp prefix of q1
            u64 inc = q1;
            for (int d = 1; d < 32; d <<= 1) {
                const u64 y = shfl64(inc, (lane - d) & 31);
                if ((int)lane >= d) inc += y;
            }
            if (t < t1) {
                const u64 pos = ucur + (inc - q1) + (q1 - 1);
                atomicOr(words + (pos >> 6), 1ull << (pos & 63));
            }
            ucur += shfl64(inc, 31);
            (void)lt;
        }
    }
}

void launch_write_data(const u64* C, u64 B, const u64* nodebase, const u32* tstart, const TNodeD* tnodes,
                       const u64* F, const u64* values, const u64* P, unsigned long long* words, cudaStream_t st) {
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_write_data<<<grid, 256, 0, st>>>(C, B, nodebase, tstart, tnodes, F, values, P, words);
    g_launches++;
}

// ------------------------------------------------------------ Elias-Fano --

__device__ __forceinline__ u64 glob_C(const u64* C, const IndexView& v, u64 l) { return v.key_base + C[l]; }

__device__ __forceinline__ long long resid(const u64* C, const u64* P, const IndexView& v, u64 l) {
    // R[i] = P[i] - floor(beta C[i] / 2^20) with the global C, P (128-bit product)
    const u64 c = glob_C(C, v, l);
    const u64 p = v.bit_base + P[l];
    const u64 lo = v.beta * c, hi = __umul64hi(v.beta, c);
    return (long long)p - (long long)((lo >> 20) | (hi << 44));
}

__global__ void k_min_residual(const u64* __restrict__ C, const u64* __restrict__ P, IndexView v, long long* out) {
    long long m = LLONG_MAX;
    for (u64 l = (u64)blockIdx.x * blockDim.x + threadIdx.x; l < v.nb; l += (u64)gridDim.x * blockDim.x) {
        const long long d = resid(C, P, v, l + 1) - resid(C, P, v, l);
        m = d < m ? d : m;
    }
    for (int dd = 16; dd; dd >>= 1) {
        const long long o = (long long)shfl64((u64)m, (threadIdx.x & 31) ^ dd);
        m = o < m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

void launch_min_residual(const u64* C, const u64* P, IndexView v, long long* out, cudaStream_t st) {
    if (v.nb == 0) return;
    unsigned grid = (unsigned)((v.nb + 255) / 256);
    if (grid > 1024) grid = 1024;
    k_min_residual<<<grid, 256, 0, st>>>(C, P, v, out);
    g_launches++;
}

// EF: lower L bits of v_i at i*L; upper bit (v_i >> L) + i (global positions,
// stored relative to the slice start).
__global__ void k_ef_write(const u64* __restrict__ C, const u64* __restrict__ P, IndexView v, u64 cnt, EfSlices e) {
    for (u64 l = (u64)blockIdx.x * blockDim.x + threadIdx.x; l < cnt; l += (u64)gridDim.x * blockDim.x) {
        const u64 i = v.b0 + l;
        const u64 cp = glob_C(C, v, l) - i * e.dC;
        const u64 pp = (u64)(resid(C, P, v, l) - (long long)i * e.dR);
        or_bits(e.cl, i * e.LC - e.cl_start, cp, e.LC);
        or_bits(e.pl, i * e.LP - e.pl_start, pp, e.LP);
        const u64 uc = (cp >> e.LC) + i - e.cu_start, up = (pp >> e.LP) + i - e.pu_start;
        atomicOr(e.cu + (uc >> 6), 1ull << (uc & 63));
        atomicOr(e.pu + (up >> 6), 1ull << (up & 63));
    }
}

void launch_ef_write(const u64* C, const u64* P, IndexView v, u64 cnt, EfSlices e, cudaStream_t st) {
    if (cnt == 0) return;
    unsigned grid = (unsigned)((cnt + 255) / 256);
    if (grid > 4096) grid = 4096;
    k_ef_write<<<grid, 256, 0, st>>>(C, P, v, cnt, e);
    g_launches++;
}

}  // namespace rs
