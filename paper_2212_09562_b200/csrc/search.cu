// The hot path: minimal-seed searches at every node of every
// splitting tree.
//
//  * Upper splits (fanout 2): smallest sigma with |{k: remap(h_k, s) < c0}| = c0,
//    counted with a single left counter.
//  * Lower splits: smallest sigma whose part counts equal the prescribed
//    sizes, counted with packed fields in one 32-bit register (exactness
//    argument in DESIGN.md section 5).
//  * Leaves: rotation fitting: smallest k*m + r with a | rot_m^r(b) = 2^m-1,
//    minimal over all lanes and rotations; or brute force.
//
// Execution model (B200-first, not the paper's block-per-node design P:342-355):
// a persistent grid of warps; lanes = consecutive seeds ("each lane one hash
// function"); the node's keys sit in warp-private shared memory and are broadcast.
// Work items are (node, seed window): warps open nodes from a global cursor and take
// windows from a per-node dispenser, so idle warps join unfinished nodes (geometric
// tails).  The winner is committed with atomicMin, so the stored value is the minimum
// over all tried seeds; every window below the final minimum is dispensed and fully
// processed before the kernel ends, hence the result equals the sequential search.
#include <algorithm>

#include "kernels.h"

namespace rs {

using namespace rsd;

namespace {

constexpr u32 kWarpsPerBlockMax = 4;
constexpr u64 kSeedCap = 1ull << 40;  // diagnostic trial cap per node (R11)

struct Args {
    const NodeRec* nodes;
    const u32* n_nodes;
    const u64* lo;
    const u8* ab;
    u64* values;
    u32* next_win;
    u32* cursor;
    int* active;
    u32* err;
    const u32* dup;
    u32 n_warps;
    u32 leaf, u1, u2;
    u32 iters;
    u32 warp_cap;
    int help;
    u32 tab_cap;  // u32 table entries per warp after the key buffer
};

// ------------------------------------------------------------------ trials --

// Lower split, full node (s = f * unit): part = remap(h, f) = floor(h_hi f / 2^32)
// (equals floor(remap(h, s) / unit) exactly).  Packed w-bit fields for parts
// 0..f-2; the last part's increments land above the compared mask.
__device__ __forceinline__ u32 count_lower_full(const u64* __restrict__ sk, u32 s, u64 sigma, u32 f,
                                                u32 w) {
    u32 cnt = 0;
    u32 j = 0;
#pragma unroll 2
    for (; j + 2 <= s; j += 2) {
        const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(sk + j);
        const u32 h0 = remix_hi(kk.x + sigma);
        const u32 h1 = remix_hi(kk.y + sigma);
        cnt += shl_clamp(1u, __umulhi(h0, f) * w);
        cnt += shl_clamp(1u, __umulhi(h1, f) * w);
    }
    if (j < s) cnt += shl_clamp(1u, __umulhi(remix_hi(sk[j] + sigma), f) * w);
    return cnt;
}

// Lower split with a smaller last part: part = floor(remap(h, s) / unit) computed as
// umulhi(remap, ceil(2^32/unit)) (exact for remap < 2^12, unit < 2^8).
__device__ __forceinline__ u32 count_lower_partial(const u64* __restrict__ sk, u32 s, u64 sigma, u32 mu,
                                                   u32 w) {
    u32 cnt = 0;
    u32 j = 0;
#pragma unroll 2
    for (; j + 2 <= s; j += 2) {
        const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(sk + j);
        const u32 h0 = remix_hi(kk.x + sigma);
        const u32 h1 = remix_hi(kk.y + sigma);
        cnt += shl_clamp(1u, __umulhi(__umulhi(h0, s), mu) * w);
        cnt += shl_clamp(1u, __umulhi(__umulhi(h1, s), mu) * w);
    }
    if (j < s) cnt += shl_clamp(1u, __umulhi(__umulhi(remix_hi(sk[j] + sigma), s), mu) * w);
    return cnt;
}

// Wide variant (fields do not fit 32 bits; l >= 19): 64-bit packed counter.
__device__ __forceinline__ u64 count_lower_wide(const u64* __restrict__ sk, u32 s, u64 sigma, u32 mu,
                                                u32 w) {
    u64 cnt = 0;
    for (u32 j = 0; j < s; ++j) {
        const u32 part = __umulhi(__umulhi(remix_hi(sk[j] + sigma), s), mu);
        cnt += 1ull << (part * w);
    }
    return cnt;
}

// Upper split: number of keys with remap(h, s) < c0  <=>  h_hi < T = ceil(c0 2^32 / s).
__device__ __forceinline__ u32 count_left(const u64* __restrict__ sk, u32 s, u64 sigma, u32 T) {
    u32 c = 0;
    u32 j = 0;
#pragma unroll 2
    for (; j + 2 <= s; j += 2) {
        const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(sk + j);
        c += remix_hi(kk.x + sigma) < T;
        c += remix_hi(kk.y + sigma) < T;
    }
    if (j < s) c += remix_hi(sk[j] + sigma) < T;
    return c;
}

// Rotation fitting for one base seed: masks of A and B; if neither has
// a collision, b fits the holes of a iff some rotation of b equals ~a.  Returns the
// smallest such r, or -1.
__device__ __forceinline__ int trial_rf(const u64* __restrict__ sk, u32 m, u32 nA, u64 base, u32 full) {
    u32 a = 0, b = 0;
    for (u32 j = 0; j < nA; ++j) a |= 1u << __umulhi(remix_hi(sk[j] + base), m);
    for (u32 j = nA; j < m; ++j) b |= 1u << __umulhi(remix_hi(sk[j] + base), m);
    if (__popc(a) + __popc(b) != (int)m) return -1;  // popcount pruning
    const u32 na = ~a & full;
    const u64 bb = (u64)b | ((u64)b << m);  // rot_m^r(b) = (bb >> (m - r)) & full
    for (u32 r = 0; r < m; ++r)
        if (((u32)(bb >> (m - r)) & full) == na) return (int)r;
    return -1;
}

__device__ __forceinline__ bool trial_bf(const u64* __restrict__ sk, u32 m, u64 sigma, u32 full) {
    u32 a = 0;
    for (u32 j = 0; j < m; ++j) a |= 1u << __umulhi(remix_hi(sk[j] + sigma), m);
    return a == full;
}

// ---- fast path (all seeds of the window < 2^32).  Keys are read two at a time with
// 16-byte shared-memory broadcasts; the packed-counter increment 1 << (w * part) comes
// from a per-warp shared-memory table (tab[part], at most f distinct words -> no bank
// conflicts) instead of IMAD + SHF, moving work off the saturated ALU/FMA-heavy pipes.
// Full nodes index by part = remap(h, f); nodes with a smaller last part index a
// table over v = remap(h, s) (tab[v] = 1 << (w * floor(v / unit))).

template <bool CARRY>
__device__ __forceinline__ u32 count_lower_fast(const u64* __restrict__ sk, const u32* __restrict__ tab, u32 s,
                                                u32 sigma, u32 r) {
    u32 c0 = 0, c1 = 0;
    u32 j = 0;
#pragma unroll 1
    for (; j + 4 <= s; j += 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(sk + j);
        const uint4 b = *reinterpret_cast<const uint4*>(sk + j + 2);
        const u32 h0 = remix_hi_fast<CARRY>(a.x, a.y, sigma);
        const u32 h1 = remix_hi_fast<CARRY>(a.z, a.w, sigma);
        const u32 h2 = remix_hi_fast<CARRY>(b.x, b.y, sigma);
        const u32 h3 = remix_hi_fast<CARRY>(b.z, b.w, sigma);
        c0 += tab[__umulhi(h0, r)] + tab[__umulhi(h1, r)];
        c1 += tab[__umulhi(h2, r)] + tab[__umulhi(h3, r)];
    }
    for (; j < s; ++j) {
        const uint2 a = *reinterpret_cast<const uint2*>(sk + j);
        c0 += tab[__umulhi(remix_hi_fast<CARRY>(a.x, a.y, sigma), r)];
    }
    return c0 + c1;
}

template <bool CARRY>
__device__ __forceinline__ u32 count_left_fast(const u64* __restrict__ sk, u32 s, u32 sigma, u32 T) {
    u32 c = 0;
    u32 j = 0;
#pragma unroll 1
    for (; j + 4 <= s; j += 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(sk + j);
        const uint4 b = *reinterpret_cast<const uint4*>(sk + j + 2);
        c += (remix_hi_fast<CARRY>(a.x, a.y, sigma) < T) + (remix_hi_fast<CARRY>(a.z, a.w, sigma) < T);
        c += (remix_hi_fast<CARRY>(b.x, b.y, sigma) < T) + (remix_hi_fast<CARRY>(b.z, b.w, sigma) < T);
    }
    for (; j < s; ++j) {
        const uint2 a = *reinterpret_cast<const uint2*>(sk + j);
        c += remix_hi_fast<CARRY>(a.x, a.y, sigma) < T;
    }
    return c;
}

// OR of 2^{remap(h, m)} over keys sk[j0..j1); bit = tab[v] (tab[v] = 1 << v)
template <bool CARRY>
__device__ __forceinline__ u32 mask_fast(const u64* __restrict__ sk, const u32* __restrict__ tab, u32 j0, u32 j1,
                                         u32 m, u32 base) {
    u32 a0 = 0, a1 = 0;
    u32 j = j0;
    for (; j + 2 <= j1; j += 2) {
        const uint2 x = *reinterpret_cast<const uint2*>(sk + j);
        const uint2 y = *reinterpret_cast<const uint2*>(sk + j + 1);
        a0 |= tab[__umulhi(remix_hi_fast<CARRY>(x.x, x.y, base), m)];
        a1 |= tab[__umulhi(remix_hi_fast<CARRY>(y.x, y.y, base), m)];
    }
    if (j < j1) {
        const uint2 x = *reinterpret_cast<const uint2*>(sk + j);
        a0 |= tab[__umulhi(remix_hi_fast<CARRY>(x.x, x.y, base), m)];
    }
    return a0 | a1;
}

template <bool CARRY>
__device__ __forceinline__ int trial_rf_fast(const u64* __restrict__ sk, const u32* __restrict__ tab, u32 m, u32 nA,
                                             u32 base, u32 full) {
    const u32 a = mask_fast<CARRY>(sk, tab, 0, nA, m, base);
    const u32 b = mask_fast<CARRY>(sk, tab, nA, m, m, base);
    if (__popc(a) + __popc(b) != (int)m) return -1;
    const u32 na = ~a & full;
    const u64 bb = (u64)b | ((u64)b << m);
    for (u32 r = 0; r < m; ++r)
        if (((u32)(bb >> (m - r)) & full) == na) return (int)r;
    return -1;
}

// One fast-path trial of `sig` for the node in sk (kind-specific predicate).
template <int KIND, bool CARRY>
__device__ __forceinline__ bool trial_fast(const u64* __restrict__ sk, const u32* __restrict__ tab, u32 s, u32 sig,
                                           u32 c_f, u32 c_full, u32 c_mask, u32 c_target, int& r) {
    if (KIND == SK_LEAF_RF) {
        r = trial_rf_fast<CARRY>(sk, tab, s, c_f, sig * s, c_full);
        return r >= 0;
    } else if (KIND == SK_LEAF_BF) {
        return mask_fast<CARRY>(sk, tab, 0, s, s, sig) == c_full;
    } else if (KIND == SK_UPPER) {
        return count_left_fast<CARRY>(sk, s, sig, c_mask) == c_target;
    } else {
        return (count_lower_fast<CARRY>(sk, tab, s, sig, c_full ? c_f : s) & c_mask) == c_target;
    }
}

// ------------------------------------------------------------- scheduling --

__device__ u32 find_help(const Args& A, u32 gw, u32 lane, u32 nn) {
    const u32 nw = A.n_warps;
    const u32 start = (u32)(((u64)gw * 2654435761ull) % nw);
    for (u32 base = 0; base < nw; base += 32) {
        u32 idx = start + base + lane;
        if (idx >= nw) idx -= nw;
        bool ok = false;
        int cand = -1;
        if (base + lane < nw) {
            cand = ((volatile int*)A.active)[idx];
            if (cand >= 0 && (u32)cand < nn) ok = ld_volatile_u64(A.values + A.nodes[cand].slot) == ~0ull;
        }
        const u32 bal = __ballot_sync(FULL, ok);
        if (bal) return (u32)__shfl_sync(FULL, cand, __ffs(bal) - 1);
    }
    return NONE;
}

template <int KIND>
__global__ void __launch_bounds__(kWarpsPerBlockMax * 32) k_search(const Args A) {
    extern __shared__ __align__(16) u64 smem[];
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const u32 gw = blockIdx.x * (blockDim.x >> 5) + wib;
    u64* sk = smem + (size_t)wib * (A.warp_cap + A.tab_cap / 2);
    u32* tab = reinterpret_cast<u32*>(sk + A.warp_cap);
    if (A.dup[0] || A.dup[1] > 1) return;  // duplicate keys: nothing can be found (host reports)
    const u32 nn = *A.n_nodes;
    const u64 ws = 32ull * A.iters;

    u32 node = NONE, s = 0, slot = 0;
    // per-node constants: lower: f, w, target, mask, mu, full?; upper: T, c0; leaf: nA, full
    u32 c_f = 0, c_w = 0, c_target = 0, c_mask = 0, c_mu = 0, c_full = 0, c_wide = 0;
    u64 c_target64 = 0, c_mask64 = 0;
    u32 c_margin = 0;

    for (;;) {
        if (node == NONE) {
            u32 n = 0;
            if (lane == 0) n = atomicAdd(A.cursor, 1u);
            n = __shfl_sync(FULL, n, 0);
            if (n >= nn) {
                if (!A.help) break;
                n = find_help(A, gw, lane, nn);
                if (n == NONE) break;
            }
            node = n;
            if (lane == 0) ((volatile int*)A.active)[gw] = (int)n;
            const NodeRec r = A.nodes[n];
            s = r.size;
            slot = r.slot;
            if (KIND == SK_LEAF_RF) {
                // A keys first, then B keys (global 1-bit hash)
                const bool valid = lane < s;
                const u64 k = valid ? A.lo[r.key_off + lane] : 0;
                const bool isb = valid && A.ab[r.key_off + lane];
                const u32 bm = __ballot_sync(FULL, isb), vm = __ballot_sync(FULL, valid);
                const u32 nA = s - __popc(bm);
                const u32 lt = lanemask_lt();
                if (valid) sk[isb ? nA + __popc(bm & lt) : __popc(~bm & vm & lt)] = k;
                c_f = nA;
                c_full = (1u << s) - 1u;
                tab[lane] = 1u << lane;
                (void)vm;
            } else if (KIND == SK_LEAF_BF) {
                if (lane < s) sk[lane] = A.lo[r.key_off + lane];
                c_full = (1u << s) - 1u;
                tab[lane] = 1u << lane;
            } else {
                for (u32 j = lane; j < s; j += 32) sk[j] = A.lo[r.key_off + j];
                if (KIND == SK_UPPER) {
                    const u32 c0 = (s / 2 + A.u2 - 1) / A.u2 * A.u2;  // R6
                    c_target = c0;
                    c_mask = (u32)((((u64)c0 << 32) + s - 1) / s);  // T = ceil(c0 2^32 / s)
                } else {
                    const u32 unit = s <= A.u1 ? A.leaf : A.u1;
                    const u32 f = (s + unit - 1) / unit;
                    const u32 w = 32 - __clz(unit + 1);  // bitwidth(unit + 1)
                    c_f = f;
                    c_w = w;
                    c_full = (s == f * unit);
                    c_mu = (u32)(((1ull << 32) + unit - 1) / unit);
                    c_wide = (f - 1) * w > 32;
                    if (!c_wide) {
                        u32 t = 0;
                        for (u32 j = 0; j + 1 < f; ++j) t += unit << (j * w);
                        c_target = t;
                        c_mask = (f - 1) * w >= 32 ? FULL : ((1u << ((f - 1) * w)) - 1u);
                        // increment table: full node -> tab[part], part < f; otherwise
                        // tab[v] for v = remap(h, s) < s (the last part adds nothing)
                        if (c_full) {
                            if (lane < f) tab[lane] = lane + 1 < f ? 1u << (lane * w) : 0u;
                        } else {
                            for (u32 v = lane; v < s; v += 32) {
                                const u32 p = v / unit;
                                tab[v] = p + 1 < f ? 1u << (p * w) : 0u;
                            }
                        }
                    } else {
                        u64 t = 0;
                        for (u32 j = 0; j + 1 < f; ++j) t += (u64)unit << (j * w);
                        c_target64 = t;
                        c_mask64 = (1ull << ((f - 1) * w)) - 1ull;
                    }
                }
            }
            __syncwarp();
            {  // carry margin: min over keys of 2^32 - 1 - k_lo
                u32 mg = FULL;
                for (u32 j = lane; j < s; j += 32) mg = min(mg, ~(u32)sk[j]);
                for (int d = 16; d; d >>= 1) mg = min(mg, __shfl_xor_sync(FULL, mg, d));
                c_margin = mg;
            }
        }
        u32 w = 0;
        u64 f = 0;
        if (lane == 0) {
            w = atomicAdd(A.next_win + slot, 1u);
            f = ld_volatile_u64(A.values + slot);
        }
        w = __shfl_sync(FULL, w, 0);
        f = shfl64(f, 0);
        const u64 wstart = (u64)w * ws;
        const u64 lb = KIND == SK_LEAF_RF ? wstart * s : wstart;
        if (lb >= f) {  // a smaller value is already committed: node finished for us
            node = NONE;
            continue;
        }
        if (wstart >= kSeedCap) {
            if (lane == 0) {
                atomicOr(A.err, 1u);
                atomicMin((unsigned long long*)(A.values + slot), (unsigned long long)lb);
            }
            node = NONE;
            continue;
        }
        // fast path: every value of the window fits 32 bits; no-carry path: additionally
        // k_lo + value < 2^32 for every key of the node (margin c_margin)
        const u64 last = KIND == SK_LEAF_RF ? (wstart + ws - 1) * s : wstart + ws - 1;
        const bool fast = last < (1ull << 32);
        const bool nocarry = fast && last <= c_margin;
        for (u32 it = 0; it < A.iters; ++it) {
            const u64 idx = wstart + (u64)it * 32 + lane;
            bool ok;
            int r = 0;
            if (fast) {
                const u32 sig = (u32)idx;
                if (KIND == SK_LOWER && c_wide)
                    ok = (count_lower_wide(sk, s, idx, c_mu, c_w) & c_mask64) == c_target64;
                else if (nocarry)
                    ok = trial_fast<KIND, false>(sk, tab, s, sig, c_f, c_full, c_mask, c_target, r);
                else
                    ok = trial_fast<KIND, true>(sk, tab, s, sig, c_f, c_full, c_mask, c_target, r);
            } else if (KIND == SK_LEAF_RF) {
                r = trial_rf(sk, s, c_f, idx * s, c_full);
                ok = r >= 0;
            } else if (KIND == SK_LEAF_BF) {
                ok = trial_bf(sk, s, idx, c_full);
            } else if (KIND == SK_UPPER) {
                ok = count_left(sk, s, idx, c_mask) == c_target;
            } else {
                if (c_wide)
                    ok = (count_lower_wide(sk, s, idx, c_mu, c_w) & c_mask64) == c_target64;
                else if (c_full)
                    ok = (count_lower_full(sk, s, idx, c_f, c_w) & c_mask) == c_target;
                else
                    ok = (count_lower_partial(sk, s, idx, c_mu, c_w) & c_mask) == c_target;
            }
            const u32 bal = __ballot_sync(FULL, ok);
            if (bal) {
                const int win = __ffs(bal) - 1;
                u64 val = wstart + (u64)it * 32 + win;
                if (KIND == SK_LEAF_RF) val = val * s + (u32)__shfl_sync(FULL, r, win);
                if (lane == 0) atomicMin((unsigned long long*)(A.values + slot), (unsigned long long)val);
                break;
            }
        }
    }
}

template <int KIND>
void launch_kind(const PhaseLaunch& P, const Args& A, u32 wpb, size_t smem, u32 grid, cudaStream_t st) {
    cudaFuncSetAttribute(k_search<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_search<KIND><<<grid, wpb * 32, smem, st>>>(A);
}

}  // namespace

u32 search_active_slots(int sm_count) { return (u32)sm_count * 16u * kWarpsPerBlockMax; }

void launch_search(const PhaseLaunch& P, cudaStream_t st) {
    if (P.n_nodes_host == 0) return;
    Args A;
    A.nodes = P.nodes;
    A.n_nodes = P.n_nodes;
    A.lo = P.lo;
    A.ab = P.ab;
    A.values = P.values;
    A.next_win = P.next_win;
    A.cursor = P.cursor;
    A.active = P.active;
    A.err = P.err;
    A.dup = P.dup;
    A.leaf = P.leaf;
    A.u1 = P.u1;
    A.u2 = P.u2;
    A.iters = P.iters ? P.iters : 1;
    A.help = P.help;
    // warp-private key buffer (even number of u64 for 16-byte vector loads)
    u32 cap = (P.max_size + 3) & ~3u;
    if (cap < 32) cap = 32;
    A.warp_cap = cap;
    // increment table: leaves 32 entries, lower splits one entry per remap value
    A.tab_cap = P.kind == SK_LOWER ? cap : (P.kind == SK_UPPER ? 0 : 32);
    const size_t per_warp = (size_t)cap * sizeof(u64) + (size_t)A.tab_cap * sizeof(u32);
    u32 wpb = kWarpsPerBlockMax;
    while (wpb > 1 && per_warp * wpb > 200 * 1024) --wpb;
    const size_t smem = per_warp * wpb;
    // resident blocks per SM (occupancy), persistent grid
    int occ = 1;
    auto kfn = P.kind == SK_UPPER ? (const void*)k_search<SK_UPPER>
               : P.kind == SK_LOWER ? (const void*)k_search<SK_LOWER>
               : P.kind == SK_LEAF_RF ? (const void*)k_search<SK_LEAF_RF>
                                      : (const void*)k_search<SK_LEAF_BF>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, (int)(wpb * 32), smem);
    if (occ < 1) occ = 1;
    int max_blocks = (int)(search_active_slots(P.sm_count) / wpb);
    u32 grid = (u32)std::min(occ * P.sm_count, max_blocks);
    // no point in more warps than nodes when helping is off
    if (!P.help) grid = std::min<u32>(grid, (P.n_nodes_host + wpb - 1) / wpb);
    if (grid == 0) grid = 1;
    A.n_warps = grid * wpb;
    switch (P.kind) {
        case SK_UPPER: launch_kind<SK_UPPER>(P, A, wpb, smem, grid, st); break;
        case SK_LOWER: launch_kind<SK_LOWER>(P, A, wpb, smem, grid, st); break;
        case SK_LEAF_RF: launch_kind<SK_LEAF_RF>(P, A, wpb, smem, grid, st); break;
        case SK_LEAF_BF: launch_kind<SK_LEAF_BF>(P, A, wpb, smem, grid, st); break;
    }
    g_launches++;
}

// ------------------------------------------------------------------ reorder --

// A7: stable partition of each split node's keys by child index with its found seed
// (P:311-313).  One warp per node; children occupy consecutive sub-ranges in
// part order, so every child's keys are contiguous for the next phase.
__global__ void k_reorder(const NodeRec* __restrict__ nodes, u32 n_nodes, const u64* __restrict__ values,
                          const u64* __restrict__ lo_in, const u8* __restrict__ ab_in, u64* __restrict__ lo_out,
                          u8* __restrict__ ab_out, u32 leaf, u32 u1, u32 u2) {
    const u32 lane = threadIdx.x & 31;
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    for (u32 n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < n_nodes; n += nwarps) {
        const NodeRec r = nodes[n];
        const u32 s = r.size;
        const u64 sigma = values[r.slot];
        u32 unit, f, c0 = 0;
        const bool upper = s > u2;
        if (upper) {
            c0 = (s / 2 + u2 - 1) / u2 * u2;
            f = 2;
            unit = 0;
        } else {
            unit = s <= u1 ? leaf : u1;
            f = (s + unit - 1) / unit;
        }
        u32 cnt[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) cnt[p] = 0;
        const u32 lt = lanemask_lt();
        for (u32 c = 0; c < s; c += 32) {
            const u32 j = c + lane;
            const bool valid = j < s;
            u64 k = 0;
            u8 b = 0;
            u32 part = 0xff;
            if (valid) {
                k = lo_in[r.key_off + j];
                b = ab_in[r.key_off + j];
                const u32 v = __umulhi(remix_hi(k + sigma), s);
                part = upper ? (v >= c0) : v / unit;
            }
            u32 dst = 0;
#pragma unroll
            for (u32 p = 0; p < 16; ++p) {
                if (p < f) {
                    const u32 bal = __ballot_sync(FULL, part == p);
                    const u32 start = upper ? (p ? c0 : 0) : p * unit;
                    if (part == p) dst = start + cnt[p] + __popc(bal & lt);
                    cnt[p] += __popc(bal);
                }
            }
            if (valid) {
                lo_out[r.key_off + dst] = k;
                ab_out[r.key_off + dst] = b;
            }
        }
    }
}

void launch_reorder(const NodeRec* nodes, u32 n_nodes, const u64* values, const u64* lo_in, const u8* ab_in,
                    u64* lo_out, u8* ab_out, u32 leaf, u32 u1, u32 u2, cudaStream_t st) {
    if (n_nodes == 0) return;
    u32 blocks = (n_nodes + 7) / 8;
    if (blocks > 148u * 32u) blocks = 148u * 32u;
    k_reorder<<<blocks, 256, 0, st>>>(nodes, n_nodes, values, lo_in, ab_in, lo_out, ab_out, leaf, u1, u2);
    g_launches++;
}

}  // namespace rs
