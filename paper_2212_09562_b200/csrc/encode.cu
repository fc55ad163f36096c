// Node-table expansion (A3) and encoding (A10-A11):
//  * every bucket's tree is instantiated from the per-size preorder template (the
//    tree shape depends only on l and s);
//  * Golomb-Rice per bucket: fixed parts of all nodes in preorder, then unary parts
//    (P:130-134), buckets concatenated into one bit vector;
//  * trend-subtracted Elias-Fano index over bucket key offsets C and bit offsets P
//    (reading R13).
#include <algorithm>
#include <climits>

#include "kernels.h"

namespace rs {

using namespace rsd;

// M[r * (B+1) + i]: r = 0 -> N(s_i) nodes; r = 1+p -> nodes of phase p; column B = 0.
// (sizes above the tables' S: counted as empty and flagged in *ovf -- the caller rebuilds)
__global__ void k_bucket_counts(const u64* __restrict__ C, u64 B, const u32* __restrict__ N,
                                const u32* __restrict__ phase_cnt, u32 NP, u64* __restrict__ M, u32 S, u32* ovf) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= B; i += (u64)gridDim.x * blockDim.x) {
        u32 s = i < B ? (u32)(C[i + 1] - C[i]) : 0;
        if (s > S) {
            atomicOr(ovf, 1u);
            s = 0;
        }
        M[i] = N[s];
        for (u32 p = 0; p < NP; ++p) M[(u64)(p + 1) * (B + 1) + i] = phase_cnt[(u64)s * NP + p];
    }
}

void launch_bucket_counts(const u64* C, u64 B, const u32* N, const u32* phase_cnt, u32 NP, u64* M,
                          cudaStream_t st, u32 S, u32* ovf) {
    unsigned grid = (unsigned)((B + 256) / 256);
    if (grid > 4096) grid = 4096;
    k_bucket_counts<<<grid, 256, 0, st>>>(C, B, N, phase_cnt, NP, M, S, ovf);
    g_launches++;
}

// node count of every phase from the scanned count matrix: row 1 + q is phase q
__global__ void k_phase_counts(const u64* __restrict__ Ms, u64 B, u32 NP, u32* __restrict__ pcnt) {
    for (u32 q = threadIdx.x; q < NP; q += blockDim.x)
        pcnt[q] = (u32)(Ms[(u64)(q + 2) * (B + 1)] - Ms[(u64)(q + 1) * (B + 1)]);
}

void launch_phase_counts(const u64* Ms, u64 B, u32 NP, u32* pcnt, cudaStream_t st) {
    k_phase_counts<<<1, 32, 0, st>>>(Ms, B, NP, pcnt);
    g_launches++;
}

struct PhaseOff {
    u64 v[32];
};

// One warp per bucket: node j of the template of size s_i gets slot nodebase_i + j
// and lands at phase_off[p] + (phase-p prefix of bucket i) + phase_rank.
__global__ void k_expand(const u64* __restrict__ C, u64 B, const u64* __restrict__ Ms, u32 NP,
                         const u32* __restrict__ tstart, const TNodeD* __restrict__ tn, PhaseOff off,
                         NodeRec* __restrict__ nodes, u32 S) {
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        const u32 s = (u32)(C[i + 1] - C[i]);
        if (s == 0 || s > S) continue;
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
                   const u64* phase_off, NodeRec* nodes, cudaStream_t st, u32 S) {
    PhaseOff o;
    for (u32 p = 0; p < 32; ++p) o.v[p] = p < NP ? phase_off[p] : 0;
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_expand<<<grid, 256, 0, st>>>(C, B, Mscan, NP, tstart, tnodes, o, nodes, S);
    g_launches++;
}

// --------------------------------------------------------------- encoding --

// One warp per bucket: len_i = F(s) + sum_j (x_j >> tau_j) + N(s).  Also the
// algorithmic evaluation counts (sequential-search work implied by the values).
__global__ void k_bucket_bits(const u64* __restrict__ C, u64 B, const u64* __restrict__ nodebase,
                              const u32* __restrict__ tstart, const TNodeD* __restrict__ tn,
                              const u64* __restrict__ F, const u64* __restrict__ values, u32 leaf, u32 u1,
                              u32 u2, int rf, u64* __restrict__ len, unsigned long long* evals, u32 S) {
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    unsigned long long ev[4] = {0, 0, 0, 0};
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        u32 s = (u32)(C[i + 1] - C[i]);
        if (s > S) s = 0;  // flagged by k_bucket_counts
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
                        unsigned long long* evals, cudaStream_t st, u32 S) {
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_bucket_bits<<<grid, 256, 0, st>>>(C, B, nodebase, tstart, tnodes, F, values, leaf, u1, u2, rf, len, evals, S);
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
                             unsigned long long* __restrict__ words, u32 S, const SingleDev* sd) {
    if (sd) {  // single-shard one-enqueue path: the data section's place in the output buffer
        if (sd->overflow) return;
        words += sd->off_data;
    }
    const u32 lane = threadIdx.x & 31;
    const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
    const u32 lt = lanemask_lt();
    for (u64 i = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < B; i += nw) {
        const u32 s = (u32)(C[i + 1] - C[i]);
        if (s == 0 || s > S) continue;
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
                       const u64* F, const u64* values, const u64* P, unsigned long long* words, cudaStream_t st,
                       u32 S, const SingleDev* sd) {
    unsigned grid = (unsigned)((B + 7) / 8);
    if (grid > 148u * 32u) grid = 148u * 32u;
    if (grid == 0) grid = 1;
    k_write_data<<<grid, 256, 0, st>>>(C, B, nodebase, tstart, tnodes, F, values, P, words, S, sd);
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

// ------------------------------------------------- single-shard, one enqueue --
//
// With one shard every global of section 13 is local: n = C[B], D = P[B], delta_C = the
// minimum bucket size, beta = floor(D 2^20 / n) (R13); they are computed on the device so
// that the whole build is enqueued without a host round trip, and the serialized MPHF
// (R14) is assembled in one device buffer (header, EF_C, EF_P, data) for a single D2H.

__device__ __forceinline__ u32 ef_L_dev(u64 U, u64 k) {
    if (U < k) return 0;
    return 63 - __clzll((long long)(U / k));
}

__global__ void k_single_globals(const u64* __restrict__ C, u64 B, const u64* __restrict__ P, const u32* small,
                                 SingleDev* sd) {
    const u64 n = C[B], D = P[B];
    sd->n = n;
    sd->D = D;
    sd->dC = small[1] == 0xffffffffu ? 0 : small[1];
    sd->beta = n ? (u64)(((unsigned __int128)D << 20) / n) : 0;
    sd->dR = LLONG_MAX;
}

// min over l in [0, B) of R[l+1] - R[l], R[i] = P[i] - floor(beta C[i] / 2^20)
__global__ void k_min_residual_single(const u64* __restrict__ C, const u64* __restrict__ P, u64 B, SingleDev* sd) {
    const u64 beta = sd->beta;
    auto R = [&](u64 i) {
        const u64 c = C[i];
        return (long long)P[i] - (long long)(((unsigned __int128)beta * c) >> 20);
    };
    long long m = LLONG_MAX;
    for (u64 l = (u64)blockIdx.x * blockDim.x + threadIdx.x; l < B; l += (u64)gridDim.x * blockDim.x) {
        const long long d = R(l + 1) - R(l);
        m = d < m ? d : m;
    }
    for (int dd = 16; dd; dd >>= 1) {
        const long long o = (long long)shfl64((u64)m, (threadIdx.x & 31) ^ dd);
        m = o < m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMin((long long*)&sd->dR, m);
}

// EF parameters, section offsets (64-bit words) and the header words (R14) of the output
__global__ void k_single_layout(SingleDev* sd, u64 B, u64 hdr0, u64 hdr1, u64 g, u64 cap_words,
                                unsigned long long* out) {
    const u64 k = B + 1, n = sd->n, D = sd->D, dC = sd->dC, beta = sd->beta;
    long long dR = sd->dR;
    if (dR == LLONG_MAX) dR = 0;
    sd->dR = dR;
    const u64 UC = n - B * dC;
    const long long RB = (long long)D - (long long)(((unsigned __int128)beta * n) >> 20);
    const u64 UP = (u64)(RB - (long long)B * dR);
    const u32 LC = ef_L_dev(UC, k), LP = ef_L_dev(UP, k);
    sd->LC = LC;
    sd->LP = LP;
    sd->lowC = k * LC;
    sd->upC = (UC >> LC) + k;
    sd->lowP = k * LP;
    sd->upP = (UP >> LP) + k;
    auto w = [](u64 bits) { return (bits + 63) / 64; };
    u64 at = 9;  // header words
    sd->off_lowC = at + 2;
    sd->off_upC = sd->off_lowC + w(sd->lowC) + 1;
    at = sd->off_upC + w(sd->upC);
    sd->off_lowP = at + 2;
    sd->off_upP = sd->off_lowP + w(sd->lowP) + 1;
    at = sd->off_upP + w(sd->upP);
    sd->off_data = at;
    sd->total_words = at + w(D);
    if (sd->total_words > cap_words) {
        sd->overflow = 1;
        return;
    }
    out[0] = hdr0;  // "RSRF", version, leaf, flags
    out[1] = hdr1;  // bucket size, 0
    out[2] = g;
    out[3] = n;
    out[4] = B;
    out[5] = D;
    out[6] = dC;
    out[7] = beta;
    out[8] = (u64)dR;
    out[sd->off_lowC - 2] = LC;
    out[sd->off_lowC - 1] = sd->lowC;
    out[sd->off_upC - 1] = sd->upC;
    out[sd->off_lowP - 2] = LP;
    out[sd->off_lowP - 1] = sd->lowP;
    out[sd->off_upP - 1] = sd->upP;
}

__global__ void k_ef_write_single(const u64* __restrict__ C, const u64* __restrict__ P, u64 B, const SingleDev* sd,
                                  unsigned long long* out) {
    if (sd->overflow) return;
    const u64 beta = sd->beta, dC = sd->dC;
    const long long dR = sd->dR;
    const u32 LC = sd->LC, LP = sd->LP;
    unsigned long long *cl = out + sd->off_lowC, *cu = out + sd->off_upC, *pl = out + sd->off_lowP,
                       *pu = out + sd->off_upP;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= B; i += (u64)gridDim.x * blockDim.x) {
        const u64 c = C[i];
        const u64 cp = c - i * dC;
        const long long r = (long long)P[i] - (long long)(((unsigned __int128)beta * c) >> 20);
        const u64 pp = (u64)(r - (long long)i * dR);
        or_bits(cl, i * LC, cp, LC);
        or_bits(pl, i * LP, pp, LP);
        const u64 uc = (cp >> LC) + i, up = (pp >> LP) + i;
        atomicOr(cu + (uc >> 6), 1ull << (uc & 63));
        atomicOr(pu + (up >> 6), 1ull << (up & 63));
    }
}

void launch_single_index(const u64* C, const u64* P, u64 B, const u32* small, SingleDev* sd, u64 hdr0, u64 hdr1, u64 g,
                         u64 cap_words, unsigned long long* out, cudaStream_t st) {
    k_single_globals<<<1, 1, 0, st>>>(C, B, P, small, sd);
    unsigned grid = (unsigned)std::min<u64>(1024, (B + 255) / 256);
    if (grid == 0) grid = 1;
    k_min_residual_single<<<grid, 256, 0, st>>>(C, P, B, sd);
    k_single_layout<<<1, 1, 0, st>>>(sd, B, hdr0, hdr1, g, cap_words, out);
    g_launches += 3;
}

void launch_single_ef(const u64* C, const u64* P, u64 B, const SingleDev* sd, unsigned long long* out,
                      cudaStream_t st) {
    unsigned grid = (unsigned)std::min<u64>(4096, (B + 256) / 256);
    k_ef_write_single<<<grid, 256, 0, st>>>(C, P, B, sd, out);
    g_launches++;
}

}  // namespace rs
