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
};

// ------------------------------------------------------------------ trials --
//
// Warp-private shared memory holds the node's keys in groups of four (48 bytes):
// [k_lo x4 | k_hi x4 | kc x4], kc = key_const(k_hi), so one pointer and three 16-byte
// broadcast loads feed four evaluations.  Key j lives at word 12*(j/4) + (j%4).  Then
// a byte table: shift amounts of the packed-counter increments (lower splits).
// (A 64-bit {0, kc} addend for IMAD.WIDE was tried: ptxas splits it into IADD3 + IMAD.X.)
//
// Fast path (every value of the window < 2^32): when additionally k_lo + value < 2^32
// for all keys of the node (checked once per window against the node's carry margin)
// the no-carry evaluation remix_hi_nc is used; otherwise remix_hi_fast<true>.  Values
// >= 2^32 (never at the measured configurations) take the generic 64-bit path.

struct KeysView {
    const u32* __restrict__ G;  // groups
    u32 tbase;                  // shared-space byte address of the shift table
};

__device__ __forceinline__ u32 key_lo(const KeysView& K, u32 j) { return K.G[12 * (j >> 2) + (j & 3)]; }
__device__ __forceinline__ u32 key_hi(const KeysView& K, u32 j) { return K.G[12 * (j >> 2) + 4 + (j & 3)]; }
__device__ __forceinline__ u32 key_kc(const KeysView& K, u32 j) { return K.G[12 * (j >> 2) + 8 + (j & 3)]; }

// h_hi of node_hash(key j, sigma) (R4): generic 64-bit path
__device__ __forceinline__ u32 hash_slow(const KeysView& K, u32 j, u64 sigma) {
    return remix_hi((((u64)key_hi(K, j) << 32) | key_lo(K, j)) + sigma);
}

// evaluate the four keys of group g
template <int MODE>  // 0: no-carry, 1: carry
__device__ __forceinline__ void hash4(const u32* __restrict__ g, u32 sigma, u32 h[4]) {
    const uint4 kl = *reinterpret_cast<const uint4*>(g);
    const uint4 kh = *reinterpret_cast<const uint4*>(g + 4);
    if (MODE == 0) {
        const uint4 kc = *reinterpret_cast<const uint4*>(g + 8);
        h[0] = remix_hi_nc(kl.x, kh.x, kc.x, sigma);
        h[1] = remix_hi_nc(kl.y, kh.y, kc.y, sigma);
        h[2] = remix_hi_nc(kl.z, kh.z, kc.z, sigma);
        h[3] = remix_hi_nc(kl.w, kh.w, kc.w, sigma);
    } else {
        h[0] = remix_hi_fast<true>(kl.x, kh.x, sigma);
        h[1] = remix_hi_fast<true>(kl.y, kh.y, sigma);
        h[2] = remix_hi_fast<true>(kl.z, kh.z, sigma);
        h[3] = remix_hi_fast<true>(kl.w, kh.w, sigma);
    }
}

template <int MODE>
__device__ __forceinline__ u32 hash1(const KeysView& K, u32 j, u32 sigma) {
    return MODE == 0 ? remix_hi_nc(key_lo(K, j), key_hi(K, j), key_kc(K, j), sigma)
                     : remix_hi_fast<true>(key_lo(K, j), key_hi(K, j), sigma);
}

// increment 1 << table[remap(h, r)]: the byte address comes straight out of mad.hi
// (hi(h * r) + table base), the shift amount is >= 32 for the last part (adds 0).
__device__ __forceinline__ u32 inc_of(u32 h, u32 r, u32 tbase) {
    u32 sh;
    asm volatile("{\n\t.reg .u32 ad;\n\tmad.hi.u32 ad, %1, %2, %3;\n\tld.shared.u8 %0, [ad];\n\t}"
                 : "=r"(sh)
                 : "r"(h), "r"(r), "r"(tbase));
    return bit_clamp(sh);
}

// Lower split: packed counter.  r = f for full nodes (part = remap(h, f)),
// r = s otherwise (table over remap(h, s)).  RS_LOWER_UNROLL groups per loop trip.
#ifndef RS_LOWER_UNROLL
#define RS_LOWER_UNROLL 1
#endif
template <int MODE>
__device__ __forceinline__ u32 count_lower(const KeysView& K, u32 s, u32 sigma, u32 r) {
    u32 c0 = 0, c1 = 0;
    const u32 ng = s >> 2;
    const u32* __restrict__ g = K.G;
    u32 q = 0;
#if RS_LOWER_UNROLL == 2
#pragma unroll 1
    for (; q + 2 <= ng; q += 2, g += 24) {
        u32 h[4], e[4];
        hash4<MODE>(g, sigma, h);
        hash4<MODE>(g + 12, sigma, e);
        c0 += inc_of(h[0], r, K.tbase) + inc_of(h[1], r, K.tbase);
        c1 += inc_of(h[2], r, K.tbase) + inc_of(h[3], r, K.tbase);
        c0 += inc_of(e[0], r, K.tbase) + inc_of(e[1], r, K.tbase);
        c1 += inc_of(e[2], r, K.tbase) + inc_of(e[3], r, K.tbase);
    }
#endif
#pragma unroll 1
    for (; q < ng; ++q, g += 12) {
        u32 h[4];
        hash4<MODE>(g, sigma, h);
        c0 += inc_of(h[0], r, K.tbase) + inc_of(h[1], r, K.tbase);
        c1 += inc_of(h[2], r, K.tbase) + inc_of(h[3], r, K.tbase);
    }
    for (u32 j = ng << 2; j < s; ++j) c0 += inc_of(hash1<MODE>(K, j, sigma), r, K.tbase);
    return c0 + c1;
}

// Upper split: |{k : remap(h_k, s) < c0}| = |{k : h_k < T}|, T = ceil(c0 2^32 / s).
template <int MODE>
__device__ __forceinline__ u32 count_left(const KeysView& K, u32 s, u32 sigma, u32 T) {
    u32 c = 0;
    const u32 ng = s >> 2;
    const u32* __restrict__ g = K.G;
#pragma unroll 1
    for (u32 q = 0; q < ng; ++q, g += 12) {
        u32 h[4];
        hash4<MODE>(g, sigma, h);
        c += (h[0] < T) + (h[1] < T) + (h[2] < T) + (h[3] < T);
    }
    for (u32 j = ng << 2; j < s; ++j) c += hash1<MODE>(K, j, sigma) < T;
    return c;
}

// OR of 2^{remap(h, m)} over the cnt keys starting at group g0.
template <int MODE>
__device__ __forceinline__ u32 leaf_mask(const KeysView& K, u32 g0, u32 cnt, u32 m, u32 base) {
    u32 a0 = 0, a1 = 0;
    const u32 ng = cnt >> 2;
    const u32* __restrict__ g = K.G + 12 * g0;
    for (u32 q = 0; q < ng; ++q, g += 12) {
        u32 h[4];
        hash4<MODE>(g, base, h);
        a0 |= (1u << __umulhi(h[0], m)) | (1u << __umulhi(h[1], m));
        a1 |= (1u << __umulhi(h[2], m)) | (1u << __umulhi(h[3], m));
    }
    for (u32 j = 4 * (g0 + ng); j < 4 * (g0 + ng) + (cnt & 3); ++j) a0 |= 1u << __umulhi(hash1<MODE>(K, j, base), m);
    return a0 | a1;
}

// Rotation fitting for one base seed: masks of A and B; with no collision
// inside A or B, b fits the holes of a iff some rotation of b equals ~a; the smallest
// such r, or -1.
__device__ __forceinline__ int fit_rotation(u32 a, u32 b, u32 m, u32 full) {
    if (__popc(a) + __popc(b) != (int)m) return -1;  // popcount pruning
    const u32 na = ~a & full;
    const u64 bb = (u64)b | ((u64)b << m);  // rot_m^r(b) = (bb >> (m - r)) & full
    for (u32 r = 0; r < m; ++r)
        if (((u32)(bb >> (m - r)) & full) == na) return (int)r;
    return -1;
}

// One trial of `sig` (32-bit fast path) for the node.  Leaves: A keys occupy groups
// 0..gB-1, B keys start at group gB (c_f = |A|).
template <int KIND, int MODE>
__device__ __forceinline__ bool trial_fast(const KeysView& K, u32 s, u32 sig, u32 c_f, u32 c_full, u32 c_mask,
                                           u32 c_target, u32 gB, int& r) {
    if (KIND == SK_LEAF_RF) {
        const u32 base = sig * s;
        const u32 a = leaf_mask<MODE>(K, 0, c_f, s, base);
        const u32 b = leaf_mask<MODE>(K, gB, s - c_f, s, base);
        r = fit_rotation(a, b, s, c_full);
        return r >= 0;
    } else if (KIND == SK_LEAF_BF) {
        return leaf_mask<MODE>(K, 0, s, s, sig) == c_full;
    } else if (KIND == SK_UPPER) {
        return count_left<MODE>(K, s, sig, c_mask) == c_target;
    } else {
        return (count_lower<MODE>(K, s, sig, c_f) & c_mask) == c_target;
    }
}

// Generic 64-bit path (values >= 2^32; also the wide 64-bit packed counters, l >= 19).
// Leaf key j of B is stored at position 4*gB + (j - |A|).
template <int KIND>
__device__ __forceinline__ bool trial_slow(const KeysView& K, u32 s, u64 idx, u32 c_f, u32 c_full, u32 c_mu,
                                           u32 c_w, u32 c_wide, u32 c_unit, u32 c_mask, u32 c_target, u64 c_mask64,
                                           u64 c_target64, u32 gB, int& r) {
    if (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) {
        const u64 base = KIND == SK_LEAF_RF ? idx * s : idx;
        u32 a = 0, b = 0;
        for (u32 j = 0; j < s; ++j) {
            const bool inB = KIND == SK_LEAF_RF && j >= c_f;
            const u32 pos = inB ? 4 * gB + (j - c_f) : j;
            const u32 bit = 1u << __umulhi(hash_slow(K, pos, base), s);
            if (inB)
                b |= bit;
            else
                a |= bit;
        }
        if (KIND == SK_LEAF_BF) return a == c_full;
        r = fit_rotation(a, b, s, c_full);
        return r >= 0;
    } else if (KIND == SK_UPPER) {
        u32 c = 0;
        for (u32 j = 0; j < s; ++j) c += hash_slow(K, j, idx) < c_mask;
        return c == c_target;
    } else {
        if (c_wide) {
            u64 c = 0;
            for (u32 j = 0; j < s; ++j) c += 1ull << (__umulhi(__umulhi(hash_slow(K, j, idx), s), c_mu) * c_w);
            return (c & c_mask64) == c_target64;
        }
        u32 c = 0;
        for (u32 j = 0; j < s; ++j) {
            const u32 part = __umulhi(hash_slow(K, j, idx), s) / c_unit;
            c += shl_clamp(1u, part * c_w);  // the last part's increment lands above c_mask
        }
        return (c & c_mask) == c_target;
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

#ifndef RS_MIN_BLOCKS
#define RS_MIN_BLOCKS 1
#endif
template <int KIND>
__global__ void __launch_bounds__(kWarpsPerBlockMax * 32, RS_MIN_BLOCKS) k_search(const Args A) {
    extern __shared__ __align__(16) u32 smem32[];
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const u32 gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const u32 cap = A.warp_cap;                 // keys (multiple of 4)
    const u32 gwords = 12 * (cap / 4 + 2);      // key groups (+2 for the leaf B alignment)
    const u32 twords = (cap + 32 + 15) / 16 * 4;  // byte table of >= cap + 32 entries (16-byte multiple)
    u32* G = smem32 + (size_t)wib * (gwords + twords);
    u8* T8 = reinterpret_cast<u8*>(G + gwords);
    const KeysView K{G, (u32)__cvta_generic_to_shared(T8)};
    if (A.dup[0] || A.dup[1] > 1) return;  // duplicate keys: nothing can be found (host reports)
    const u32 nn = *A.n_nodes;
    const u64 ws = 32ull * A.iters;

    u32 node = NONE, s = 0, slot = 0;
    // per-node constants. lower: f, w, unit, full?, mu, r (table index range), target,
    // mask (64-bit if wide); upper: c_mask = T, c_target = c0; leaves: c_f = |A|,
    // c_full = 2^m - 1, gB = first group of the B keys.
    u32 c_f = 0, c_w = 0, c_target = 0, c_mask = 0, c_mu = 0, c_full = 0, c_wide = 0, c_margin = 0;
    u32 c_unit = 1, c_r = 1, gB = 0;
    u64 c_target64 = 0, c_mask64 = 0;

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
            u32 mg = FULL;  // carry margin: min over keys of 2^32 - 1 - k_lo
            if (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) {
                // RF: A keys in groups 0.., B keys from group gB (global 1-bit hash)
                const bool valid = lane < s;
                const u64 k = valid ? A.lo[r.key_off + lane] : 0;
                const bool isb = KIND == SK_LEAF_RF && valid && A.ab[r.key_off + lane];
                const u32 bm = __ballot_sync(FULL, isb), vm = __ballot_sync(FULL, valid);
                const u32 nA = s - __popc(bm);
                const u32 lt = lanemask_lt();
                gB = (nA + 3) / 4;
                if (valid) {
                    const u32 p = isb ? 4 * gB + __popc(bm & lt) : __popc(~bm & vm & lt);
                    const u32 gp = 12 * (p >> 2), q = p & 3;
                    const u32 kh = (u32)(k >> 32);
                    G[gp + q] = (u32)k;
                    G[gp + 4 + q] = kh;
                    G[gp + 8 + q] = key_const(kh);
                    mg = ~(u32)k;
                }
                c_f = nA;
                c_full = (1u << s) - 1u;
            } else {
                for (u32 j = lane; j < s; j += 32) {
                    const u64 k = A.lo[r.key_off + j];
                    const u32 gp = 12 * (j >> 2), q = j & 3;
                    const u32 kh = (u32)(k >> 32);
                    G[gp + q] = (u32)k;
                    G[gp + 4 + q] = kh;
                    G[gp + 8 + q] = key_const(kh);
                    mg = min(mg, ~(u32)k);
                }
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
                    c_unit = unit;
                    c_full = (s == f * unit);
                    c_mu = (u32)(((1ull << 32) + unit - 1) / unit);
                    c_wide = (f - 1) * w > 32;
                    c_r = c_full ? f : s;
                    if (!c_wide) {
                        u32 t = 0;
                        for (u32 j = 0; j + 1 < f; ++j) t += unit << (j * w);
                        c_target = t;
                        c_mask = (f - 1) * w >= 32 ? FULL : ((1u << ((f - 1) * w)) - 1u);
                        // shift table: part p -> p*w for p < f-1, 32 (adds 0) for the last part;
                        // full nodes index by part, others by v = remap(h, s) (part = v / unit)
                        for (u32 v = lane; v < c_r; v += 32) {
                            const u32 p = c_full ? v : v / unit;
                            T8[v] = (u8)(p + 1 < f ? p * w : 32);
                        }
                    } else {
                        u64 t = 0;
                        for (u32 j = 0; j + 1 < f; ++j) t += (u64)unit << (j * w);
                        c_target64 = t;
                        c_mask64 = (1ull << ((f - 1) * w)) - 1ull;
                    }
                }
            }
            for (int d = 16; d; d >>= 1) mg = min(mg, __shfl_xor_sync(FULL, mg, d));
            c_margin = mg;
            __syncwarp();
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
        // largest value (seed, or base seed k*m) any lane tries in this window
        const u64 last = KIND == SK_LEAF_RF ? (wstart + ws - 1) * s : wstart + ws - 1;
        const bool fast = last < (1ull << 32) && !(KIND == SK_LOWER && c_wide);
        const bool nocarry = fast && last <= c_margin;
        for (u32 it = 0; it < A.iters; ++it) {
            const u64 idx = wstart + (u64)it * 32 + lane;
            int r = 0;
            bool ok;
            if (nocarry)
                ok = trial_fast<KIND, 0>(K, s, (u32)idx, KIND == SK_LOWER ? c_r : c_f, c_full, c_mask, c_target,
                                         gB, r);
            else if (fast)
                ok = trial_fast<KIND, 1>(K, s, (u32)idx, KIND == SK_LOWER ? c_r : c_f, c_full, c_mask, c_target,
                                         gB, r);
            else
                ok = trial_slow<KIND>(K, s, idx, c_f, c_full, c_mu, c_w, c_wide, c_unit, c_mask, c_target,
                                      c_mask64, c_target64, gB, r);
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
    // warp-private buffer: key groups (12 words per 4 keys, +2 groups) + byte shift table
    u32 cap = (P.max_size + 3) & ~3u;
    if (cap < 32) cap = 32;
    A.warp_cap = cap;
    const size_t per_warp = ((size_t)12 * (cap / 4 + 2) + (cap + 32 + 15) / 16 * 4) * sizeof(u32);
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
