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
//  * phases of large nodes ("help" mode): work items are (node, seed window); warps open
//    nodes from a global cursor and take windows from a per-node dispenser, so idle warps
//    join unfinished nodes (geometric tails).  The winner is committed with atomicMin,
//    so the stored value is the minimum over all tried seeds; every window below the
//    final minimum is dispensed and fully processed before the kernel ends, hence the
//    result equals the sequential search.
//  * phases of small nodes ("batch" mode): a warp takes `batch` nodes per cursor atomic
//    and searches each alone, windows in increasing order, first hit wins.
#include <cstdlib>
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.h"

namespace rs {

using namespace rsd;

namespace {

constexpr u32 kWarpsPerBlockMax = 4;
constexpr u64 kSeedCap = 1ull << 40;  // diagnostic trial cap per node (R11)
constexpr u32 kWarpKeyCap = 8192;     // largest node the warp engine holds in shared memory

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
    u32 batch;     // nodes per cursor atomic in batch mode
    u32 tail;      // batch mode: the last `tail` nodes run in help mode (no straggler batches)
    u32 cp_l1;     // early-rejection checkpoint (key groups of 4) for full lower-level-1 nodes, 0 = off
    u32 cp_l2;     // same for full lower-level-2 nodes
    u32 cp_l1b;    // second checkpoints (key groups; off unless above the first)
    u32 cp_l2b;
    u32 cp_leaf;   // leaves: early rejection on (0 = off)
    u32 cp_last;   // full lower nodes: also reject when the last part already overflows (0 = off)
    u32 cp_wide;   // early rejection in the wide-counter kernel (l >= 19) too (0 = off)
    u32 cp_leaf2;  // leaves: second checkpoint (0 = single stage)
    u32 cp_wide2;  // wide-counter splits: second checkpoint too (0 = single stage)
    u64* lo_w;     // fused redistribution (batch-mode split phases, nodes <= kFuseMax keys): the
    u8* ab_w;      // key arrays written in child order right after the node's search; null = off
    u32 upper_kp;  // upper splits in batch mode: keys-parallel sequential seeds (upper_keys_parallel) for nodes up to this size (0 = off)
    u32 upper_kp_var;  // ... whose left-count variance c0 (s - c0) / s is at most this
    u32 qwords;    // early-rejection queue words per warp (0 for the plain variants)
    unsigned long long* exec;  // RS_COUNT_EVALS builds: executed evaluations of this phase's class
    u32 lane_fit;  // leaves up to this size check rotations lane by lane (fit_rotation_lane)
    const u8* fit_lut;  // rotation-fit table for leaves of <= kFitLutMax keys (fit_lut_device), null = off
    u32 lean;           // batch mode: lean windows (lean_windows) while on the no-carry path
};

// Bucket-tree kernel (k_bucket_tree): buckets, their per-size preorder templates, slots.
struct TreeArgs {
    const u64* C;         // bucket key offsets (B + 1)
    u64 B;
    const u64* nodebase;  // exclusive node prefix per bucket (slot base)
    const u32* tstart;    // template start per size
    const TNodeD* tn;     // template nodes
    u32 S;                // largest bucket size the tables cover
    u32* bcursor;         // zeroed bucket cursor
    u32 bbatch;           // buckets per cursor atomic
    u32 dedupe;           // check each bucket for duplicate keys (instead of k_dedupe)
};

// ------------------------------------------------------------------ trials --
//
// Warp-private shared memory holds the node's keys in groups of four:
// [k_lo x4 | k_hi x4 | kc x4] for splits (48 bytes), plus [mA x4 | mB x4] for leaves
// (80 bytes), kc = key_const(k_hi), mA / mB = all-ones if the key is in A / B (R7) and 0
// for padding keys, so leaves too are processed in whole groups.  Key j lives at word
// GW*(j/4) + (j%4), GW = 12 or 20.  Then a byte table: shift amounts of the packed
// counter increments (lower splits).
// (A 64-bit {0, kc} addend for IMAD.WIDE was tried: ptxas splits it into IADD3 + IMAD.X.)
//
// Fast path (every value of the window < 2^32): when additionally k_lo + value < 2^32
// for all keys of the node (checked once per window against the node's carry margin)
// the no-carry evaluation remix_hi_nc is used; otherwise remix_hi_fast<true>, which also
// takes windows of values >= 2^32 whose values share one high word H (leaves at l >= 20
// have stored values around 2^31..2^33).  A window straddling a multiple of 2^32 takes the
// generic 64-bit path.

template <int KIND>
struct Layout {
    static constexpr u32 GW = (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) ? 20 : 12;
};

// Diagnostic build (-DRS_COUNT_EVALS): every warp counts the key evaluations its lanes issue
// (32 per key of a group evaluation, including lanes whose seed is discarded) in shared memory
// and adds them to a per-class global counter at exit -- the EXECUTED work, next to the
// algorithmic count of DESIGN.md 7.  Compiled out otherwise.
#ifdef RS_COUNT_EVALS
__shared__ unsigned long long s_exec[8];
#define RS_COUNT(k)                                                               \
    do {                                                                          \
        if ((threadIdx.x & 31) == 0) s_exec[threadIdx.x >> 5] += 32ull * (k);     \
    } while (0)
#define RS_COUNT_RAW(v_)                                                          \
    do {                                                                          \
        const unsigned long long c_ = (v_); /* evaluated by every lane */         \
        if ((threadIdx.x & 31) == 0) s_exec[threadIdx.x >> 5] += c_;              \
    } while (0)
#define RS_COUNT_INIT()                                                           \
    do {                                                                          \
        if ((threadIdx.x & 31) == 0) s_exec[threadIdx.x >> 5] = 0;                \
    } while (0)
#define RS_COUNT_FLUSH(ptr)                                                       \
    do {                                                                          \
        if ((threadIdx.x & 31) == 0 && (ptr)) atomicAdd((ptr), s_exec[threadIdx.x >> 5]); \
    } while (0)
#else
#define RS_COUNT(k) \
    do {            \
    } while (0)
#define RS_COUNT_RAW(v_) \
    do {                 \
    } while (0)
#define RS_COUNT_INIT() \
    do {                \
    } while (0)
#define RS_COUNT_FLUSH(ptr) \
    do {                    \
    } while (0)
#endif

struct KeysView {
    const u32* __restrict__ G;  // groups
    u32 tbase;                  // shared-space byte address of the shift table
    u32 H;                      // carry path: high word of every value of the window
    u32 fbase;                  // shared-space byte address of s_full_tab (64-byte aligned)
};

template <u32 GW>
__device__ __forceinline__ u32 key_word(const KeysView& K, u32 j, u32 field) {
    return K.G[GW * (j >> 2) + 4 * field + (j & 3)];
}

// h_hi of node_hash(key j, sigma) (R4): generic 64-bit path
template <u32 GW>
__device__ __forceinline__ u32 hash_slow(const KeysView& K, u32 j, u64 sigma) {
    RS_COUNT(1);
    return remix_hi((((u64)key_word<GW>(K, j, 1) << 32) | key_word<GW>(K, j, 0)) + sigma);
}

// evaluate the four keys of group g
template <int MODE>  // 0: no-carry, 1: carry (value = H * 2^32 + sigma)
__device__ __forceinline__ void hash4(const u32* __restrict__ g, u32 sigma, u32 h[4], u32 H) {
    RS_COUNT(4);
    const uint4 kl = *reinterpret_cast<const uint4*>(g);
    const uint4 kh = *reinterpret_cast<const uint4*>(g + 4);
    if (MODE == 0) {
        const uint4 kc = *reinterpret_cast<const uint4*>(g + 8);
        h[0] = remix_hi_nc(kl.x, kh.x, kc.x, sigma);
        h[1] = remix_hi_nc(kl.y, kh.y, kc.y, sigma);
        h[2] = remix_hi_nc(kl.z, kh.z, kc.z, sigma);
        h[3] = remix_hi_nc(kl.w, kh.w, kc.w, sigma);
    } else {
        h[0] = remix_hi_fast<true>(kl.x, kh.x, sigma, H);
        h[1] = remix_hi_fast<true>(kl.y, kh.y, sigma, H);
        h[2] = remix_hi_fast<true>(kl.z, kh.z, sigma, H);
        h[3] = remix_hi_fast<true>(kl.w, kh.w, sigma, H);
    }
}

template <int MODE, u32 GW>
__device__ __forceinline__ u32 hash1(const KeysView& K, u32 j, u32 sigma) {
    RS_COUNT(1);
    return MODE == 0 ? remix_hi_nc(key_word<GW>(K, j, 0), key_word<GW>(K, j, 1), key_word<GW>(K, j, 2), sigma)
                     : remix_hi_fast<true>(key_word<GW>(K, j, 0), key_word<GW>(K, j, 1), sigma, K.H);
}

// kernel variants of the lower-level search: plain; with early rejection (full nodes with a
// 32-bit packed counter); wide 64-bit packed counters (phases whose level has (f-1)*w > 32)
enum { V_PLAIN = 0, V_CP = 1, V_WIDE = 2 };

// Block-wide shift tables of the FULL lower-level nodes of a phase (all share f and w):
// index 0 = lower level 1 (f1 parts of l), 1 = lower level 2 (f2 parts of u1).  Static
// shared arrays have link-time addresses, so the lookup is LDS [part + imm].
__shared__ __align__(64) u8 s_full_tab[2][32];
// early-rejection constants of the two full classes (run_window_cp): {me, ke, ce, mo, ko, co}
// for the "some field > unit" test, then {Me, Mo, tope | topo << 8 | w << 16, thr} for the
// last-part test (sum of fields 0..f-2 < thr = keys so far - unit; thr = 0: off), then thr of
// the second checkpoint
__shared__ u32 s_cp_masks[2][11];

// increment 1 << s_full_tab[c][remap(h, f)]
template <int CL>
__device__ __forceinline__ u32 inc_full(u32 h, u32 f, u32 fbase) {
    // (an OR of the 32-bit table base instead of the 64-bit addend ptxas folds into IMAD.HI --
    // two IMAD.MOV fewer per four keys, four LOP3 more -- measured 6 % slower at C3: the ALU
    // pipe has less headroom than the FMA pipe)
    (void)fbase;
    return bit_clamp(s_full_tab[CL][__umulhi(h, f)]);
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

// Lower split: packed counter.  CL = 0/1: full node of lower level 1/2,
// part = remap(h, f) looked up in the block-wide static table; CL = 2: node with a smaller
// last part, warp table over v = remap(h, s) (r = s).  Keys of groups [g0, g1), plus the
// s % 4 tail keys when TAIL.
template <int MODE, int CL, bool TAIL = true>
__device__ __forceinline__ u32 count_lower(const KeysView& K, u32 s, u32 sigma, u32 r, u32 g0 = 0,
                                           u32 g1 = 0xffffffffu, u32 init = 0) {
    u32 c0 = init, c1 = 0;
    const u32 ng = min(s >> 2, g1);
    const u32* __restrict__ g = K.G + 12 * g0;
#pragma unroll 1
    for (u32 q = g0; q < ng; ++q, g += 12) {
        u32 h[4];
        hash4<MODE>(g, sigma, h, K.H);
        if (CL < 2) {
            c0 += inc_full<CL>(h[0], r, K.fbase) + inc_full<CL>(h[1], r, K.fbase);
            c1 += inc_full<CL>(h[2], r, K.fbase) + inc_full<CL>(h[3], r, K.fbase);
        } else {
            c0 += inc_of(h[0], r, K.tbase) + inc_of(h[1], r, K.tbase);
            c1 += inc_of(h[2], r, K.tbase) + inc_of(h[3], r, K.tbase);
        }
    }
    if (TAIL)
        for (u32 j = (s >> 2) << 2; j < s; ++j) {
            const u32 h = hash1<MODE, 12>(K, j, sigma);
            c0 += CL < 2 ? inc_full<(CL < 2 ? CL : 0)>(h, r, K.fbase) : inc_of(h, r, K.tbase);
        }
    return c0 + c1;
}

// Wide packed counter (l >= 19: (f-1)*w > 32): fields of parts 0..hs-1 in the low word,
// parts hs..f-2 in the high word (hs = floor(32/w)); the table holds t = p*w (low word) or
// 32 + (p-hs)*w (high word), 64 for the last part; increments 1 << t and 1 << (t-32), both
// clamped to 0 out of range.  The exactness argument of DESIGN.md 5 holds per word.
// Groups [g0, g1) (+ the s % 4 tail keys when TAIL), starting from the counter init.
template <int MODE, int CL, bool TAIL = true>
__device__ __forceinline__ u64 count_lower_wide(const KeysView& K, u32 s, u32 sigma, u32 r, u32 g0 = 0,
                                                u32 g1 = 0xffffffffu, u64 init = 0) {
    u32 lo = (u32)init, hi = (u32)(init >> 32);
    const u32 ng = min(s >> 2, g1);
    const u32* __restrict__ g = K.G + 12 * g0;
#pragma unroll 1
    for (u32 q = g0; q < ng; ++q, g += 12) {
        u32 h[4];
        hash4<MODE>(g, sigma, h, K.H);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            u32 t;
            if (CL < 2)
                t = s_full_tab[CL < 2 ? CL : 0][__umulhi(h[k], r)];
            else
                asm volatile("{\n\t.reg .u32 ad;\n\tmad.hi.u32 ad, %1, %2, %3;\n\tld.shared.u8 %0, [ad];\n\t}"
                             : "=r"(t)
                             : "r"(h[k]), "r"(r), "r"(K.tbase));
            lo += bit_clamp(t);
            hi += bit_clamp(t - 32);
        }
    }
    if (TAIL)
    for (u32 j = (s >> 2) << 2; j < s; ++j) {
        const u32 h = hash1<MODE, 12>(K, j, sigma);
        u32 t;
        if (CL < 2)
            t = s_full_tab[CL < 2 ? CL : 0][__umulhi(h, r)];
        else
            asm volatile("{\n\t.reg .u32 ad;\n\tmad.hi.u32 ad, %1, %2, %3;\n\tld.shared.u8 %0, [ad];\n\t}"
                         : "=r"(t)
                         : "r"(h), "r"(r), "r"(K.tbase));
        lo += bit_clamp(t);
        hi += bit_clamp(t - 32);
    }
    return ((u64)hi << 32) | lo;
}

// shift of part p in the packed counter: narrow p*w (32 = add nothing for the last part);
// wide (split words, see count_lower_wide) p*w | 32+(p-hs)*w, 64 for the last part
__host__ __device__ __forceinline__ u32 part_shift(u32 p, u32 f, u32 w) {
    if ((f - 1) * w <= 32) return p + 1 < f ? p * w : 32;
    const u32 hs = 32 / w;
    return p + 1 >= f ? 64 : p < hs ? p * w : 32 + (p - hs) * w;
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
        hash4<MODE>(g, sigma, h, K.H);
        c += (h[0] < T) + (h[1] < T) + (h[2] < T) + (h[3] < T);
    }
    for (u32 j = ng << 2; j < s; ++j) c += hash1<MODE, 12>(K, j, sigma) < T;
    return c;
}

// Leaf masks over all groups: a = OR of 2^{remap(h, m)} over A keys, b over B keys
// (padding keys have mA = mB = 0).
template <int MODE>
__device__ __forceinline__ void leaf_masks(const KeysView& K, u32 ng, u32 m, u32 base, u32& a, u32& b, u32 q0 = 0,
                                           u32 a_init = 0, u32 b_init = 0) {
    u32 a0 = a_init, b0 = b_init;
    const u32* __restrict__ g = K.G + 20 * q0;
#pragma unroll 1
    for (u32 q = q0; q < ng; ++q, g += 20) {
        u32 h[4];
        hash4<MODE>(g, base, h, K.H);
        const uint4 ma = *reinterpret_cast<const uint4*>(g + 12);
        const uint4 mb = *reinterpret_cast<const uint4*>(g + 16);
        const u32 t0 = 1u << __umulhi(h[0], m), t1 = 1u << __umulhi(h[1], m);
        const u32 t2 = 1u << __umulhi(h[2], m), t3 = 1u << __umulhi(h[3], m);
        a0 |= (t0 & ma.x) | (t1 & ma.y);
        b0 |= (t0 & mb.x) | (t1 & mb.y);
        a0 |= (t2 & ma.z) | (t3 & ma.w);
        b0 |= (t2 & mb.z) | (t3 & mb.w);
    }
    a = a0;
    b = b0;
}

// Rotation fitting for the warp's 32 base seeds: lane masks a (A keys) and b
// (B keys).  With no collision inside A or B (popcount pruning), b fits the holes of
// a iff some rotation of b equals ~a.  Passing lanes are checked in lane (= base seed)
// order, all lanes testing one rotation each, and the first lane with a fit wins with its
// smallest r (minimal value rule P:297-300).  Returns true on the winning lane only (r set).
__device__ __forceinline__ bool fit_rotation_warp(u32 a, u32 b, u32 m, u32 full, u32 lane, int& r) {
    u32 pm = __ballot_sync(FULL, __popc(a) + __popc(b) == (int)m);
    while (pm) {
        const int i = __ffs(pm) - 1;
        const u32 ai = __shfl_sync(FULL, a, i), bi = __shfl_sync(FULL, b, i);
        const u32 na = ~ai & full;
        const u64 bb = (u64)bi | ((u64)bi << m);  // rot_m^r(b) = (bb >> (m - r)) & full
        const u32 hm = __ballot_sync(FULL, lane < m && ((u32)(bb >> (m - lane)) & full) == na);
        if (hm) {
            r = __ffs(hm) - 1;
            return (int)lane == i;
        }
        pm &= pm - 1;
    }
    return false;
}

// The same test lane by lane: every lane whose masks pass the popcount pruning tries its m
// rotations in order; the caller's ballot takes the lowest lane with a fit (its smallest r is
// the first one found), the minimal value as in fit_rotation_warp.  For small leaves (m <= 10:
// ~17 % of the lanes pass at m = 8) m predicated steps per lane are cheaper than the warp's
// serial loop over the passing lanes with two shuffles and a ballot each.
__device__ __forceinline__ bool fit_rotation_lane(u32 a, u32 b, u32 m, u32 full, int& r) {
    r = -1;
    if (__popc(a) + __popc(b) == (int)m) {
        const u32 na = ~a & full;
        const u64 bb = (u64)b | ((u64)b << m);  // rot_m^r(b) = (bb >> (m - r)) & full
        for (u32 q = 0; q < m; ++q)
            if (((u32)(bb >> (m - q)) & full) == na) {
                r = (int)q;
                break;
            }
    }
    return r >= 0;
}

// The same test as one table load for leaves of m <= kFitLutMax keys: fit_lut[off(m) + (b << m | a)]
// holds the smallest r in [0, m) with rot_m^r(b) = ~a & (2^m - 1) -- the r fit_rotation_lane finds --
// or 0xff (no fit; this covers masks with a collision, whose complement cannot be a rotation
// of b).  off(m) = (4^m - 4) / 3, 87,380 bytes for m = 1..8, read through the L1 cache.  At
// l = 8 the serial rotation loop was 16 % of the leaf kernel's instructions and 30 % of its
// stall samples (ncu, profiles/ncu_summary_r02.md).
constexpr u32 kFitLutMax = 8;
__host__ __device__ constexpr u32 fit_lut_off(u32 m) { return ((1u << (2 * m)) - 4u) / 3u; }

__device__ __forceinline__ bool fit_rotation_lut(u32 a, u32 b, u32 m, const u8* __restrict__ lut, int& r) {
    const u32 v = __ldg(lut + ((b << m) | a));
    r = (int)v;
    return v != 0xffu;
}

__device__ __forceinline__ bool fit_rotation(u32 a, u32 b, u32 m, u32 full, u32 lane, int& r, u32 lane_fit_max,
                                             const u8* lut = nullptr) {
    if (lut) return fit_rotation_lut(a, b, m, lut, r);
    return m <= lane_fit_max ? fit_rotation_lane(a, b, m, full, r) : fit_rotation_warp(a, b, m, full, lane, r);
}

// Per-node search state (registers).
struct NodeCtx {
    u32 s, slot;
    u32 f, w, unit, full, mu, r, wide, target, mask, margin;
    u32 l2;  // lower level 2 node (s > u1)
    u64 target64, mask64;
    u32 cp;  // early rejection (full lower nodes): checkpoint in key groups, 0 = off
    u32 cp2; // second checkpoint (key groups), 0 = single stage
    u64 kW;  // key rebase: the buffered keys are lo + kW (values are tried relative to kW)
    u32 lane_fit;  // leaves: lane-by-lane rotation check up to this m (fit_rotation)
    const u8* lut; // leaves of m <= kFitLutMax (rotation fitting): the table slice of m, else null
    u32 nc_end;    // lean windows (batch mode, kW = 0): windows ending at or below this base value
                   // (seed index units) stay on the no-carry path without a rebase
};


// One trial of `sig` (32-bit fast path).  For rotation fitting r receives the rotation.
template <int KIND, int MODE, bool WIDE = false>
__device__ __forceinline__ bool trial_fast(const KeysView& K, const NodeCtx& c, u32 sig, u32 lane, int& r) {
    if (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) {
        const u32 base = KIND == SK_LEAF_RF ? sig * c.s : sig;
        u32 a, b;
        leaf_masks<MODE>(K, (c.s + 3) >> 2, c.s, base, a, b);
        if (KIND == SK_LEAF_BF) return a == c.full;
        return fit_rotation(a, b, c.s, c.full, lane, r, c.lane_fit, c.lut);
    } else if (KIND == SK_UPPER) {
        return count_left<MODE>(K, c.s, sig, c.mask) == c.target;
    } else {
        if (WIDE) {
            const u64 cnt = !c.full ? count_lower_wide<MODE, 2>(K, c.s, sig, c.r)
                            : c.l2 ? count_lower_wide<MODE, 1>(K, c.s, sig, c.r)
                                   : count_lower_wide<MODE, 0>(K, c.s, sig, c.r);
            return (cnt & c.mask64) == c.target64;
        }
        const u32 cnt = !c.full ? count_lower<MODE, 2>(K, c.s, sig, c.r)
                        : c.l2 ? count_lower<MODE, 1>(K, c.s, sig, c.r)
                                        : count_lower<MODE, 0>(K, c.s, sig, c.r);
        return (cnt & c.mask) == c.target;
    }
}

// Generic 64-bit path (values >= 2^32; also the wide 64-bit packed counters, l >= 19).
template <int KIND, bool WIDE = false>
__device__ __forceinline__ bool trial_slow(const KeysView& K, const NodeCtx& c, u64 idx, u32 lane, int& r) {
    constexpr u32 GW = Layout<KIND>::GW;
    const u32 s = c.s;
    if (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) {
        const u64 base = KIND == SK_LEAF_RF ? idx * s : idx;
        u32 a = 0, b = 0;
        for (u32 j = 0; j < s; ++j) {
            const u32 bit = 1u << __umulhi(hash_slow<GW>(K, j, base), s);
            a |= bit & key_word<GW>(K, j, 3);
            b |= bit & key_word<GW>(K, j, 4);
        }
        if (KIND == SK_LEAF_BF) return a == c.full;
        return fit_rotation(a, b, s, c.full, lane, r, c.lane_fit, c.lut);
    } else if (KIND == SK_UPPER) {
        u32 cnt = 0;
        for (u32 j = 0; j < s; ++j) cnt += hash_slow<GW>(K, j, idx) < c.mask;
        return cnt == c.target;
    } else {
        if (WIDE) {
            u64 cnt = 0;
            for (u32 j = 0; j < s; ++j) {
                const u32 t = part_shift(__umulhi(__umulhi(hash_slow<GW>(K, j, idx), s), c.mu), c.f, c.w);
                cnt += t < 64 ? 1ull << t : 0ull;
            }
            return (cnt & c.mask64) == c.target64;
        }
        u32 cnt = 0;
        for (u32 j = 0; j < s; ++j) {
            const u32 part = __umulhi(hash_slow<GW>(K, j, idx), s) / c.unit;
            cnt += shl_clamp(1u, part * c.w);  // the last part's increment lands above mask
        }
        return (cnt & c.mask) == c.target;
    }
}

// Load node n's keys into the warp's buffer and derive its constants.
// Leaf data fetched ahead (batch mode): the node record and this lane's key / A-B byte.
struct LeafPrefetch {
    NodeRec rec;
    u64 k;
    u8 ab;
};

// (rec_ov / lo_src / ab_src: the node record and key arrays when they are not the phase's --
// the bucket-tree kernel passes its shared-memory copy of the bucket)
template <int KIND, bool WIDE = false>
__device__ __forceinline__ void load_node(const Args& A, u32 n, u32 lane, u32* G, u8* T8, NodeCtx& c,
                                          const LeafPrefetch* pf = nullptr, const NodeRec* rec_ov = nullptr,
                                          const u64* lo_src = nullptr, const u8* ab_src = nullptr) {
    constexpr u32 GW = Layout<KIND>::GW;
    const u64* const src_lo = lo_src ? lo_src : A.lo;
    const u8* const src_ab = ab_src ? ab_src : A.ab;
    const NodeRec rec = rec_ov ? *rec_ov : pf ? pf->rec : A.nodes[n];
    c.s = rec.size;
    c.slot = rec.slot;
    const u32 s = c.s;
    u32 mg = FULL;  // carry margin: min over keys of 2^32 - 1 - k_lo
    // the warp's previous node was read by every lane; order those reads before the rewrite
    // (help mode reaches here through shuffles / ballots only, which do not order memory)
    __syncwarp();
    if (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) {
        // natural key order; A/B select masks (global 1-bit hash); padding keys to
        // the next multiple of four get zero masks
        const bool valid = lane < s;
        const u64 k = valid ? (pf ? pf->k : src_lo[rec.key_off + lane]) : 0;
        const bool isb = KIND == SK_LEAF_RF && valid && (pf ? pf->ab : src_ab[rec.key_off + lane]);
        if (lane < ((s + 3) & ~3u)) {
            const u32 gp = GW * (lane >> 2), q = lane & 3;
            const u32 kh = (u32)(k >> 32);
            G[gp + q] = (u32)k;
            G[gp + 4 + q] = kh;
            G[gp + 8 + q] = key_const(kh);
            G[gp + 12 + q] = valid && !isb ? FULL : 0u;
            G[gp + 16 + q] = isb ? FULL : 0u;
        }
        if (valid) mg = ~(u32)k;
        c.full = (1u << s) - 1u;
        // early rejection checkpoint (key groups): a fit needs no collision inside A or B, so
        // a base seed whose first 4*cp keys already collide fails; best measured-by-simulation
        // checkpoints: 8 keys for m = 10..19, 12 keys for m = 20..24
        c.cp = A.cp_leaf && s >= 10 ? (s < 20 ? 2u : 3u) : 0u;
        // second checkpoint (simulated cascade optimum: keys 8 / 12 for m = 14..19, 12 / 16 for
        // m = 20..24; a single stage is better below m = 14)
        c.cp2 = c.cp && A.cp_leaf2 && s >= 14 ? c.cp + 1 : 0u;
        c.kW = 0;
        c.lane_fit = A.lane_fit;
        c.lut = KIND == SK_LEAF_RF && A.fit_lut && s <= kFitLutMax ? A.fit_lut + fit_lut_off(s) : nullptr;
    } else {
        for (u32 j = lane; j < s; j += 32) {
            const u64 k = src_lo[rec.key_off + j];
            const u32 gp = GW * (j >> 2), q = j & 3;
            const u32 kh = (u32)(k >> 32);
            G[gp + q] = (u32)k;
            G[gp + 4 + q] = kh;
            G[gp + 8 + q] = key_const(kh);
            mg = min(mg, ~(u32)k);
        }
        if (KIND == SK_UPPER) {
            const u32 c0 = (s / 2 + A.u2 - 1) / A.u2 * A.u2;  // R6
            c.target = c0;
            c.mask = (u32)((((u64)c0 << 32) + s - 1) / s);  // T = ceil(c0 2^32 / s)
        } else {
            const u32 unit = s <= A.u1 ? A.leaf : A.u1;
            const u32 f = (s + unit - 1) / unit;
            const u32 w = 32 - __clz(unit + 1);  // bitwidth(unit + 1)
            c.f = f;
            c.w = w;
            c.unit = unit;
            c.full = (s == f * unit);
            c.mu = (u32)(((1ull << 32) + unit - 1) / unit);
            // the wide kernel variant runs every node of its phase on the 64-bit counter (a
            // partial node may itself fit 32 bits: part_shift then gives the narrow layout)
            c.wide = WIDE;
            c.r = c.full ? f : s;
            c.l2 = s > A.u1;
            const u32 cpg = c.l2 ? A.cp_l2 : A.cp_l1;
            // (wide counters: early rejection by field extraction, run_window_cp_wide)
            c.cp = c.full && cpg < (s >> 2) && ((f - 1) * w <= 31 || (WIDE && A.cp_wide)) ? cpg : 0;
            const u32 cpg2 = c.l2 ? A.cp_l2b : A.cp_l1b;
            c.cp2 = c.cp && (!WIDE || A.cp_wide2) && cpg2 >= cpg + 2 && cpg2 < (s >> 2) ? cpg2 : 0;  // a 1-group stage does not pay
            if (!c.wide) {
                u32 t = 0;
                for (u32 j = 0; j + 1 < f; ++j) t += unit << (j * w);
                c.target = t;
                c.mask = (f - 1) * w >= 32 ? FULL : ((1u << ((f - 1) * w)) - 1u);
                // shift table: part p -> p*w for p < f-1, 32 (adds 0) for the last part;
                // full nodes index by part, others by v = remap(h, s) (part = v / unit)
                for (u32 v = lane; v < c.r; v += 32) {
                    const u32 p = c.full ? v : v / unit;
                    T8[v] = (u8)(p + 1 < f ? p * w : 32);
                }
            } else {
                u64 t = 0, m = 0;
                for (u32 j = 0; j + 1 < f; ++j) {
                    const u32 sh = part_shift(j, f, w);
                    t += (u64)unit << sh;
                    m |= (((u64)1 << w) - 1) << sh;
                }
                c.target64 = t;
                c.mask64 = m;
                for (u32 v = lane; v < c.r; v += 32) T8[v] = (u8)part_shift(c.full ? v : v / unit, f, w);
            }
        }
    }
    for (int d = 16; d; d >>= 1) mg = min(mg, __shfl_xor_sync(FULL, mg, d));
    c.margin = mg;
    c.kW = 0;
    // a window [w, w + ws) of base values is on the no-carry path iff (w + ws) * sc - 1 <= margin
    // (sc = m value units per rotation-fitting base seed)
    c.nc_end = KIND == SK_LEAF_RF ? mg / s : mg;  // (floor(margin / sc) <= the exact bound)
    __syncwarp();
}

// Rebase the buffered keys by delta (mod 2^64): lo' = lo + delta, kc' = key_const(hi'), and
// the new carry margin min(2^32 - 1 - lo'_low).  Trying value v on key lo equals trying
// v - kW on lo + kW, so a window of large values becomes a window of small ones and stays
// on the no-carry path (a window of span <= margin never carries).
template <u32 GW>
__device__ __forceinline__ void rebase_keys(u32* G, u32 s, u64 delta, u32 lane, u32& margin) {
    __syncwarp();
    u32 mg = FULL;
    for (u32 j = lane; j < s; j += 32) {
        u32* p = G + GW * (j >> 2) + (j & 3);
        const u64 k = (((u64)p[4] << 32) | p[0]) + delta;
        const u32 kh = (u32)(k >> 32);
        p[0] = (u32)k;
        p[4] = kh;
        p[8] = key_const(kh);
        mg = min(mg, ~(u32)k);
    }
    for (int d = 16; d; d >>= 1) mg = min(mg, __shfl_xor_sync(FULL, mg, d));
    margin = mg;
    __syncwarp();
}

// Early rejection of a full class CL (run_window_cp): true if a seed whose packed counter
// after the first keys is cnt cannot succeed: a field of parts 0..f-2 above unit
// (((cnt & me) + ke) & ce | ((cnt & mo) + ko) & co, even and odd fields apart so that the
// added carries stay inside a field gap), or the last part (not held in the counter) above
// unit, i.e. the fields' sum below thr = keys so far - unit; the sum of the even / odd fields
// is one coefficient of a product with a spread multiplier (partial sums < 2^{2w}: no carries
// between the coefficients).  The class constants are read from shared memory at the test
// (once per seed) so that they hold no registers across the counting loops.
template <int CL>
__device__ __forceinline__ bool cp_reject(u32 cnt, int ti) {
    const volatile u32* m = s_cp_masks[CL];
    const u32 me = m[0], mo = m[3], tops = m[8];
    const u32 fw = tops >> 16, m2w = (1u << (2 * fw)) - 1u;
    const u32 se = (u32)(((u64)(cnt & me) * m[6]) >> (tops & 0xff)) & m2w;
    const u32 so = (u32)(((u64)((cnt & mo) >> fw) * m[7]) >> ((tops >> 8) & 0xff)) & m2w;
    return ((((cnt & me) + m[1]) & m[2]) | (((cnt & mo) + m[4]) & m[5])) != 0 || se + so < m[ti];
}

// drop the first nb entries of a warp queue of qn (<= 64) entries (seeds, counters)
__device__ __forceinline__ void queue_pop(u32* qs, u32* qc, u32& qn, u32 nb, u32 lane) {
    const u32 rest = qn - nb;  // <= 32
    u32 a = 0, b = 0;
    __syncwarp();
    if (lane < rest) {
        a = qs[nb + lane];
        b = qc[nb + lane];
    }
    __syncwarp();
    if (lane < rest) {
        qs[lane] = a;
        qc[lane] = b;
    }
    __syncwarp();
    qn = rest;
}

// Search the window [wstart, wstart + 32*iters) of base values (seeds, or base seeds k for
// RF) in order; on a hit returns true with the stored value in *val (warp-uniform).
// Early rejection with warp compaction (full lower-level nodes, no-carry path), a cascade of
// up to two checkpoints.  Stage 1 counts the first c.cp key groups of 32 seeds; a seed that
// CpTest rejects cannot succeed (a carry only happens when some count exceeds 2^w - 1 > unit,
// so the test never rejects a valid seed).  Survivors go to a per-warp FIFO queue in
// increasing seed order; whenever 32 are queued (and at the end of the window) the next stage
// takes them: with a second checkpoint c.cp2, stage 2 counts groups [c.cp, c.cp2), tests again
// and queues its survivors (in order) for stage 3, which finishes the counts over the
// remaining keys; without it, stage 2 finishes them.  A batch is always the oldest entries of
// its queue and a queue's entries are older than everything upstream, so survivors are
// completed in increasing seed order; every other seed of the window was rejected, hence the
// first hit is the smallest successful seed of the window.
template <int CL>
__device__ __forceinline__ bool run_window_cp(const Args& A, const KeysView& K, const NodeCtx& c, u64 wstart, u32 lane,
                                           u32* qs, u64* val) {
    const u32 wrel = (u32)(wstart - c.kW);  // window start relative to the key rebase
    const u32 g1 = c.cp, g2 = c.cp2;
    u32* const qc = qs + 64;
    u32* const qs2 = qs + 128;
    u32* const qc2 = qs + 192;
    u32 qn = 0, qn2 = 0;
    // final stage on the first nb entries of queue (fs, fc) counted up to group gf
    auto finish = [&](u32* fs, u32* fc, u32& fn, u32 nb, u32 gf) -> bool {
        const bool have = lane < nb;
        const u32 sig = have ? fs[lane] : 0;
        u32 cnt = have ? fc[lane] : 0;
        cnt = count_lower<0, CL, true>(K, c.s, sig, c.r, gf, 0xffffffffu, cnt);
        const u32 bal = __ballot_sync(FULL, have && (cnt & c.mask) == c.target);
        if (bal) {
            *val = c.kW + __shfl_sync(FULL, sig, __ffs(bal) - 1);
            return true;
        }
        queue_pop(fs, fc, fn, nb, lane);
        return false;
    };
    for (u32 it = 0; it <= A.iters; ++it) {
        const bool last = it == A.iters;
        if (!last) {
            const u32 sig = wrel + it * 32 + lane;
            const u32 cnt = count_lower<0, CL, false>(K, c.s, sig, c.r, 0, g1);
            const bool keep = !cp_reject<CL>(cnt, 9);
            const u32 bal = __ballot_sync(FULL, keep);
            if (keep) {
                const u32 pos = qn + __popc(bal & lanemask_lt());
                qs[pos] = sig;
                qc[pos] = cnt;
            }
            qn += __popc(bal);
            __syncwarp();
        }
        while (qn >= 32 || (last && qn > 0)) {
            const u32 nb = min(qn, 32u);
            if (!g2) {
                if (finish(qs, qc, qn, nb, g1)) return true;
                continue;
            }
            // stage 2: groups [g1, g2), survivors to queue 2
            const bool have = lane < nb;
            const u32 sig = have ? qs[lane] : 0;
            u32 cnt = have ? qc[lane] : 0;
            cnt = count_lower<0, CL, false>(K, c.s, sig, c.r, g1, g2, cnt);
            const bool keep = have && !cp_reject<CL>(cnt, 10);
            const u32 bal = __ballot_sync(FULL, keep);
            if (keep) {
                const u32 pos = qn2 + __popc(bal & lanemask_lt());
                qs2[pos] = sig;
                qc2[pos] = cnt;
            }
            qn2 += __popc(bal);
            queue_pop(qs, qc, qn, nb, lane);
            if (qn2 >= 32 && finish(qs2, qc2, qn2, 32, g2)) return true;
        }
        if (last)
            while (qn2 > 0)
                if (finish(qs2, qc2, qn2, min(qn2, 32u), g2)) return true;
    }
    return false;
}

// Early rejection with warp compaction for leaves (no-carry path), a cascade of up to two
// checkpoints: stage 1 ORs the masks of the first 4*c.cp keys (full groups) for 32 base seeds; a
// seed whose partial masks show a collision (popc(a) + popc(b) < keys so far) cannot fit (P:252
// pruning, applied early).  Survivors queue in seed order with their partial masks; with a second
// checkpoint c.cp2, stage 2 extends 32 of them to 4*c.cp2 keys, tests again and queues its
// survivors for stage 3; the last stage completes the masks and runs the fit (rotation fitting:
// lowest lane with a fit and its smallest r; brute force: a == full).  Batches are the oldest
// entries of their queue and every queue is older than everything upstream, so survivors are
// completed in seed order; every other seed of the window failed, hence the first hit is the
// window's minimum.
template <int KIND>
__device__ __forceinline__ bool run_window_leaf_cp(const Args& A, const KeysView& K, const NodeCtx& c, u64 wstart,
                                                   u32 lane, u32* qs, u64* val) {
    const u32 wrel = (u32)(wstart - c.kW);
    const u32 ng = (c.s + 3) >> 2, g1 = c.cp, g2 = c.cp2;
    u32* const qa = qs + 64;
    u32* const qb = qs + 128;
    u32* const qs2 = qs + 192;
    u32* const qa2 = qs + 256;
    u32* const qb2 = qs + 320;
    u32 qn = 0, qn2 = 0;
    auto base_of = [&](u32 sig) { return KIND == SK_LEAF_RF ? sig * c.s : sig; };
    auto push = [&](bool keep, u32 sig, u32 a, u32 b, u32* ds, u32* da, u32* db, u32& dn) {
        const u32 bal = __ballot_sync(FULL, keep);
        if (keep) {
            const u32 pos = dn + __popc(bal & lanemask_lt());
            ds[pos] = sig;
            da[pos] = a;
            db[pos] = b;
        }
        dn += __popc(bal);
        __syncwarp();
    };
    auto pop = [&](u32* ds, u32* da, u32* db, u32& dn, u32 nb) {
        const u32 rest = dn - nb;
        u32 x = 0, y = 0, z = 0;
        if (lane < rest) {
            x = ds[nb + lane];
            y = da[nb + lane];
            z = db[nb + lane];
        }
        __syncwarp();
        if (lane < rest) {
            ds[lane] = x;
            da[lane] = y;
            db[lane] = z;
        }
        __syncwarp();
        dn = rest;
    };
    // last stage on the first nb entries of (fs, fa, fb), masks completed from group gf
    auto finish = [&](u32* fs, u32* fa, u32* fb, u32& fn, u32 nb, u32 gf) -> bool {
        const bool have = lane < nb;
        const u32 sig = have ? fs[lane] : 0;
        u32 a = have ? fa[lane] : 0, b = have ? fb[lane] : 0;
        leaf_masks<0>(K, ng, c.s, base_of(sig), a, b, gf, a, b);
        if (!have) a = b = 0;  // no entry: cannot fit (m >= 10 keys)
        int r = 0;
        const bool ok = KIND == SK_LEAF_BF ? a == c.full : fit_rotation(a, b, c.s, c.full, lane, r, c.lane_fit, c.lut);
        const u32 bal = __ballot_sync(FULL, ok);
        if (bal) {
            const int win = __ffs(bal) - 1;
            const u64 k = c.kW + __shfl_sync(FULL, sig, win);
            *val = KIND == SK_LEAF_RF ? k * c.s + (u32)__shfl_sync(FULL, r, win) : k;
            return true;
        }
        __syncwarp();
        pop(fs, fa, fb, fn, nb);
        return false;
    };
    for (u32 it = 0; it <= A.iters; ++it) {
        const bool last = it == A.iters;
        if (!last) {
            const u32 sig = wrel + it * 32 + lane;
            u32 a, b;
            leaf_masks<0>(K, g1, c.s, base_of(sig), a, b);
            push((u32)(__popc(a) + __popc(b)) == 4 * g1, sig, a, b, qs, qa, qb, qn);
        }
        while (qn >= 32 || (last && qn > 0)) {
            const u32 nb = min(qn, 32u);
            if (!g2) {
                if (finish(qs, qa, qb, qn, nb, g1)) return true;
                continue;
            }
            const bool have = lane < nb;
            const u32 sig = have ? qs[lane] : 0;
            u32 a = have ? qa[lane] : 0, b = have ? qb[lane] : 0;
            leaf_masks<0>(K, g2, c.s, base_of(sig), a, b, g1, a, b);
            push(have && (u32)(__popc(a) + __popc(b)) == 4 * g2, sig, a, b, qs2, qa2, qb2, qn2);
            pop(qs, qa, qb, qn, nb);
            if (qn2 >= 32 && finish(qs2, qa2, qb2, qn2, 32, g2)) return true;
        }
        if (last)
            while (qn2 > 0)
                if (finish(qs2, qa2, qb2, qn2, min(qn2, 32u), g2)) return true;
    }
    return false;
}

// Early rejection for the wide (64-bit) packed counters (l >= 19, (f-1)*w > 32), one
// checkpoint: after k keys a seed cannot succeed if some part 0..f-2 holds more than unit
// keys or the last part does (k - sum of the fields > unit).  The fields are extracted one by
// one (once per seed, not per key).  A valid seed has every count <= unit < 2^w - 1, so its
// fields are exact and it is never rejected; an overflowed field may hide a rejection, never
// cause one.
__device__ __forceinline__ bool wide_reject(u64 cnt, const NodeCtx& c, u32 k) {
    const u32 fm = (1u << c.w) - 1u;
    u32 sum = 0;
    bool over = false;
    for (u32 j = 0; j + 1 < c.f; ++j) {
        const u32 v = (u32)(cnt >> part_shift(j, c.f, c.w)) & fm;
        over |= v > c.unit;
        sum += v;
    }
    return over || sum + c.unit < k;
}

// The wide counterpart of run_window_cp, with the same cascade of up to two checkpoints:
// survivors queue as (seed, counter low word, counter high word) in seed order; stage 2 (when
// c.cp2 is set) extends 32 of them to the second checkpoint and queues its survivors; the last
// stage completes 32 at a time.  The first hit is the smallest successful seed of the window
// (same argument as run_window_cp).
template <int CL>
__device__ __forceinline__ bool run_window_cp_wide(const Args& A, const KeysView& K, const NodeCtx& c, u64 wstart,
                                                   u32 lane, u32* qs, u64* val) {
    const u32 wrel = (u32)(wstart - c.kW);
    const u32 g1 = c.cp, g2 = c.cp2;
    u32* const qlo = qs + 64;
    u32* const qhi = qs + 128;
    u32* const qs2 = qs + 192;
    u32* const qlo2 = qs + 256;
    u32* const qhi2 = qs + 320;
    u32 qn = 0, qn2 = 0;
    auto push = [&](bool keep, u32 sig, u64 cnt, u32* ds, u32* dl, u32* dh, u32& dn) {
        const u32 bal = __ballot_sync(FULL, keep);
        if (keep) {
            const u32 pos = dn + __popc(bal & lanemask_lt());
            ds[pos] = sig;
            dl[pos] = (u32)cnt;
            dh[pos] = (u32)(cnt >> 32);
        }
        dn += __popc(bal);
        __syncwarp();
    };
    auto pop = [&](u32* ds, u32* dl, u32* dh, u32& dn, u32 nb) {
        const u32 rest = dn - nb;
        u32 x = 0, y = 0, z = 0;
        if (lane < rest) {
            x = ds[nb + lane];
            y = dl[nb + lane];
            z = dh[nb + lane];
        }
        __syncwarp();
        if (lane < rest) {
            ds[lane] = x;
            dl[lane] = y;
            dh[lane] = z;
        }
        __syncwarp();
        dn = rest;
    };
    auto finish = [&](u32* fs, u32* fl, u32* fh, u32& fn, u32 nb, u32 gf) -> bool {
        const bool have = lane < nb;
        const u32 sig = have ? fs[lane] : 0;
        u64 cnt = have ? (((u64)fh[lane] << 32) | fl[lane]) : 0;
        cnt = count_lower_wide<0, CL, true>(K, c.s, sig, c.r, gf, 0xffffffffu, cnt);
        const u32 bal = __ballot_sync(FULL, have && (cnt & c.mask64) == c.target64);
        if (bal) {
            *val = c.kW + __shfl_sync(FULL, sig, __ffs(bal) - 1);
            return true;
        }
        __syncwarp();
        pop(fs, fl, fh, fn, nb);
        return false;
    };
    for (u32 it = 0; it <= A.iters; ++it) {
        const bool last = it == A.iters;
        if (!last) {
            const u32 sig = wrel + it * 32 + lane;
            const u64 cnt = count_lower_wide<0, CL, false>(K, c.s, sig, c.r, 0, g1);
            push(!wide_reject(cnt, c, 4 * g1), sig, cnt, qs, qlo, qhi, qn);
        }
        while (qn >= 32 || (last && qn > 0)) {
            const u32 nb = min(qn, 32u);
            if (!g2) {
                if (finish(qs, qlo, qhi, qn, nb, g1)) return true;
                continue;
            }
            const bool have = lane < nb;
            const u32 sig = have ? qs[lane] : 0;
            u64 cnt = have ? (((u64)qhi[lane] << 32) | qlo[lane]) : 0;
            cnt = count_lower_wide<0, CL, false>(K, c.s, sig, c.r, g1, g2, cnt);
            push(have && !wide_reject(cnt, c, 4 * g2), sig, cnt, qs2, qlo2, qhi2, qn2);
            pop(qs, qlo, qhi, qn, nb);
            if (qn2 >= 32 && finish(qs2, qlo2, qhi2, qn2, 32, g2)) return true;
        }
        if (last)
            while (qn2 > 0)
                if (finish(qs2, qlo2, qhi2, qn2, min(qn2, 32u), g2)) return true;
    }
    return false;
}

template <int KIND, int VAR>
__device__ __forceinline__ bool run_window(const Args& A, const KeysView& K, NodeCtx& c, u64 wstart,
                                           u32 lane, u64* val, u32* qs, u32* qc) {
    constexpr u32 GW = Layout<KIND>::GW;
    const u64 ws = 32ull * A.iters;
    const u64 sc = KIND == SK_LEAF_RF ? c.s : 1;  // value units per seed index
    // No-carry path relative to the key rebase c.kW (seed index units): values of the window
    // minus the rebase must stay within the carry margin; otherwise rebase the buffered keys
    // to the window start (cheap: s keys once per ~margin/span windows).
    if (wstart < c.kW || (wstart - c.kW + ws) * sc - 1 > c.margin) {
        rebase_keys<GW>(const_cast<u32*>(K.G), c.s, (wstart - c.kW) * sc, lane, c.margin);
        c.kW = wstart;
    }
    if (ws * sc - 1 <= c.margin) {
        const u32 wrel = (u32)(wstart - c.kW);
        if (VAR == V_WIDE && KIND == SK_LOWER && c.cp)
            return c.l2 ? run_window_cp_wide<1>(A, K, c, wstart, lane, qs, val)
                        : run_window_cp_wide<0>(A, K, c, wstart, lane, qs, val);
        if (VAR == V_CP && KIND == SK_LOWER && c.cp)
            return c.l2 ? run_window_cp<1>(A, K, c, wstart, lane, qs, val)
                        : run_window_cp<0>(A, K, c, wstart, lane, qs, val);
        if (VAR == V_CP && (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) && c.cp)
            return run_window_leaf_cp<KIND>(A, K, c, wstart, lane, qs, val);
        for (u32 it = 0; it < A.iters; ++it) {
            int r = 0;
            const bool ok = trial_fast<KIND, 0, VAR == V_WIDE>(K, c, wrel + it * 32 + lane, lane, r);
            const u32 bal = __ballot_sync(FULL, ok);
            if (bal) {
                const int win = __ffs(bal) - 1;
                u64 v = wstart + (u64)it * 32 + win;
                if (KIND == SK_LEAF_RF) v = v * c.s + (u32)__shfl_sync(FULL, r, win);
                *val = v;
                return true;
            }
        }
        return false;
    }
    // rare (a key within one window span of 2^32 after rebasing): absolute values on the
    // original keys, carry path with one high word per window, else the generic 64-bit path
    if (c.kW) {
        rebase_keys<GW>(const_cast<u32*>(K.G), c.s, (0 - c.kW) * sc, lane, c.margin);
        c.kW = 0;
    }
    const u64 first = wstart * sc, last = (wstart + ws - 1) * sc;
    const u32 H = (u32)(first >> 32);
    const bool fast = (last >> 32) == (first >> 32);
    KeysView KH = K;
    KH.H = H;
    for (u32 it = 0; it < A.iters; ++it) {
        const u64 idx = wstart + (u64)it * 32 + lane;
        int r = 0;
        bool ok;
        if (fast)
            ok = trial_fast<KIND, 1, VAR == V_WIDE>(KH, c, (u32)idx, lane, r);
        else
            ok = trial_slow<KIND, VAR == V_WIDE>(K, c, idx, lane, r);
        const u32 bal = __ballot_sync(FULL, ok);
        if (bal) {
            const int win = __ffs(bal) - 1;
            u64 v = wstart + (u64)it * 32 + win;
            if (KIND == SK_LEAF_RF) v = v * c.s + (u32)__shfl_sync(FULL, r, win);
            *val = v;
            return true;
        }
    }
    return false;
}

// Lean windows (batch mode, a node's first windows): while the window's base values stay
// within the node's carry margin (c.nc_end, key rebase 0) every trial takes the no-carry path,
// so the per-window checks of run_window (64-bit margin and rebase arithmetic, kernel-variant
// dispatch) reduce to one 32-bit compare.  Same trials in the same order as run_window's plain
// loop: the first window with a hit gives the lowest lane (seed) with a hit, the minimal value.
// Returns false with wstart = the first window not searched (the caller continues there).
template <int KIND, int VAR>
__device__ __forceinline__ bool lean_windows(const Args& A, const KeysView& K, const NodeCtx& c, u32 lane, u32 ws,
                                             u64* val, u64& wstart) {
    u32 w = 0;
    if (c.nc_end >= ws) {
        const u32 wlast = c.nc_end - ws;  // largest window start on the no-carry path (w + ws never wraps)
#pragma unroll 1
        for (; w <= wlast; w += ws) {
#pragma unroll 1
            for (u32 it = 0; it < A.iters; ++it) {
                int r = 0;
                const bool ok = trial_fast<KIND, 0, VAR == V_WIDE>(K, c, w + it * 32 + lane, lane, r);
                const u32 bal = __ballot_sync(FULL, ok);
                if (bal) {
                    const int win = __ffs(bal) - 1;
                    u64 v = (u64)w + it * 32 + win;
                    if (KIND == SK_LEAF_RF) v = v * c.s + (u32)__shfl_sync(FULL, r, win);
                    *val = v;
                    return true;
                }
            }
        }
    }
    wstart = w;
    return false;
}

// A7 fused into the batch-mode split search: the warp that found the node's seed still holds
// its keys (shared memory, natural order, possibly rebased by kW) and writes them in child
// order -- the stable partition of reorder_node, without a separate pass over the keys.  The
// node's A/B bytes are read into registers before any write (the node's range is rewritten in
// place).
constexpr u32 kFuseMax = 256;
constexpr u32 kUpperKpMax = 256;  // keys-parallel upper splits for nodes up to this size (few trials)

template <int KIND>
__device__ __forceinline__ void fused_reorder(const Args& A, const u32* G, u32 key_off, const NodeCtx& c, u64 val,
                                              u32 lane) {
    constexpr u32 GW = Layout<KIND>::GW;
    const u32 s = c.s;
    u8 abv[kFuseMax / 32];
#pragma unroll
    for (u32 q = 0; q < kFuseMax / 32; ++q) abv[q] = q * 32 + lane < s ? A.ab[key_off + q * 32 + lane] : 0;
    __syncwarp();
    u32 unit = 0, f, c0 = 0;
    const bool upper = KIND == SK_UPPER;
    if (upper) {
        c0 = c.target;
        f = 2;
    } else {
        unit = c.unit;
        f = c.f;
    }
    u32 cnt[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) cnt[p] = 0;
    const u32 lt = lanemask_lt();
#pragma unroll
    for (u32 q = 0; q < kFuseMax / 32; ++q) {
        const u32 j = q * 32 + lane;
        if (q * 32 >= s) break;
        const bool valid = j < s;
        u64 k = 0;
        u32 part = 0xff;
        if (valid) {
            const u32* g = G + GW * (j >> 2) + (j & 3);
            k = (((u64)g[4] << 32) | g[0]) - c.kW;  // undo the key rebase
            const u32 v = __umulhi(remix_hi(k + val), s);
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
            A.lo_w[key_off + dst] = k;
            A.ab_w[key_off + dst] = abv[q];
        }
    }
    __syncwarp();
}

// Upper split, keys in parallel (batch mode): an upper node needs few trials (about
// sqrt(pi s / 2) at most; 5-17 for the ~100-200-key nodes of l = 8, b = 100), so a 32-seed
// window wastes most of its work.  Here the lanes share the node's keys and the seeds
// sigma = 0, 1, 2, ... are tried one after another: count |{k : h_k < T}| by ballots, the
// first sigma with count c0 is the minimal seed (R6).
__device__ __forceinline__ u64 upper_keys_parallel(const Args& A, const u32* G, const NodeCtx& c, u32 lane) {
    constexpr u32 GW = Layout<SK_UPPER>::GW;
    const u32 s = c.s;
    for (u64 sigma = 0; sigma < kSeedCap; ++sigma) {
        u32 cnt = 0;
        for (u32 j0 = 0; j0 < s; j0 += 32) {
            RS_COUNT(1);
            const u32 j = j0 + lane;
            bool left = false;
            if (j < s) {
                const u32* g = G + GW * (j >> 2) + (j & 3);
                const u64 k = (((u64)g[4] << 32) | g[0]) - c.kW;
                left = remix_hi(k + sigma) < c.mask;  // remap(h, s) < c0  <=>  h_hi < T
            }
            cnt += __popc(__ballot_sync(FULL, left));
        }
        if (cnt == c.target) return sigma;
    }
    if (lane == 0) atomicOr(A.err, 1u);
    return kSeedCap;
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

// Block-wide shift tables and early-rejection constants of the two full lower-level classes
// (s_full_tab, s_cp_masks); every block of a kernel that searches lower-level nodes runs it.
__device__ __forceinline__ void init_lower_tables(const Args& A) {
        for (u32 t = threadIdx.x; t < 64; t += blockDim.x) {
            const u32 cl = t >> 5, p = t & 31;
            const u32 unit = cl ? A.u1 : A.leaf, f = cl ? A.u2 / A.u1 : A.u1 / A.leaf;
            const u32 w = 32 - __clz(unit + 1);
            s_full_tab[cl][p] = (u8)part_shift(p, f, w);
            if (p == 0) {
                u32 me = 0, ke = 0, ce = 0, mo = 0, ko = 0, co = 0;
                const u32 fm = (1u << w) - 1, kadd = fm - unit;  // field + kadd >= 2^w <=> field > unit
                for (u32 j = 0; j + 1 < f && (j + 1) * w <= 32; ++j) {
                    const u32 sh = j * w, cb = (j + 1) * w < 32 ? 1u << (sh + w) : 0u;
                    if (j & 1) {
                        mo |= fm << sh;
                        ko |= kadd << sh;
                        co |= cb;
                    } else {
                        me |= fm << sh;
                        ke |= kadd << sh;
                        ce |= cb;
                    }
                }
                s_cp_masks[cl][0] = me;
                s_cp_masks[cl][1] = ke;
                s_cp_masks[cl][2] = ce;
                s_cp_masks[cl][3] = mo;
                s_cp_masks[cl][4] = ko;
                s_cp_masks[cl][5] = co;
                // last-part test: Me / Mo = sum over the even / odd fields i of 2^{2 w i'} (i' = the
                // field's rank among them); valid while the keys counted so far stay < 2^{2w}
                u32 ne = 0, no = 0, Me = 0, Mo = 0;
                for (u32 j = 0; j + 1 < f && (j + 1) * w <= 32; ++j) {
                    if (j & 1) Mo |= 1u << (2 * w * no++);
                    else Me |= 1u << (2 * w * ne++);
                }
                const u32 kcp = 4 * (cl ? A.cp_l2 : A.cp_l1), kcp2 = 4 * (cl ? A.cp_l2b : A.cp_l1b);
                const bool ok = 2 * w < 32 && kcp < (1u << (2 * w)) && kcp > unit && (f - 1) * w <= 31;
                const bool ok2 = 2 * w < 32 && kcp2 < (1u << (2 * w)) && kcp2 > unit && (f - 1) * w <= 31;
                s_cp_masks[cl][6] = Me;
                s_cp_masks[cl][7] = Mo;
                s_cp_masks[cl][8] = (ne ? 2 * w * (ne - 1) : 0) | (no ? 2 * w * (no - 1) : 0) << 8 | w << 16;
                s_cp_masks[cl][9] = ok && A.cp_last ? kcp - unit : 0u;
                s_cp_masks[cl][10] = ok2 && A.cp_last ? kcp2 - unit : 0u;
            }
        }
        __syncthreads();
    }

#ifndef RS_MIN_BLOCKS
// upper-split kernels at 8 blocks x 4 warps per SM (62 registers, no spills) instead of 6 at 78
// registers: C2 upper phase -5 % (pass AF)
#define RS_MIN_BLOCKS 8
#endif
#ifndef RS_LOWER_MIN_BLOCKS
// lower-split kernels at 8 blocks x 4 warps per SM (64 registers): 9 or 10 blocks (56 / 48
// registers) spill and grow the split loop 83 -> 86 instructions
#define RS_LOWER_MIN_BLOCKS 8
#endif
#ifndef RS_LEAF_MIN_BLOCKS
// leaf kernels at 8 blocks x 4 warps per SM (64 registers): measured -8.5 % on the C5 leaf phase,
// -3 % at C3, neutral at C2 against the unconstrained 78-88 registers (gpurun pass L)
#define RS_LEAF_MIN_BLOCKS 8
#endif
template <int KIND, int VAR = V_PLAIN>
__global__ void __launch_bounds__(kWarpsPerBlockMax * 32,
                                                     KIND == SK_LOWER                             ? RS_LOWER_MIN_BLOCKS
                                                     : (KIND == SK_LEAF_RF || KIND == SK_LEAF_BF) ? RS_LEAF_MIN_BLOCKS
                                                                                                  : RS_MIN_BLOCKS) k_search(const Args A) {
    constexpr u32 GW = Layout<KIND>::GW;
    extern __shared__ __align__(16) u32 smem32[];
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const u32 gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const u32 cap = A.warp_cap;                    // keys (multiple of 4)
    const u32 gwords = GW * (cap / 4 + 1);         // key groups
    const u32 twords = (cap + 32 + 15) / 16 * 4;   // byte table of >= cap + 32 entries
    u32* G = smem32 + (size_t)wib * (gwords + twords + A.qwords);
    RS_COUNT_INIT();
    u8* T8 = reinterpret_cast<u8*>(G + gwords);
    u32* QS = G + gwords + twords;  // early-rejection queues, A.qwords per warp (64 entries each):
    u32* QC = QS + 64;              // seeds + partial counters / masks, for up to two stages
    const KeysView K{G, (u32)__cvta_generic_to_shared(T8), 0u, (u32)__cvta_generic_to_shared(&s_full_tab[0][0])};
    if (KIND == SK_LOWER) init_lower_tables(A);  // shift tables of full nodes, rejection constants
    if (A.dup[0] || A.dup[1] > 1) return;  // duplicate keys: nothing can be found (host reports)
    const u32 nn = *A.n_nodes;
    const u64 ws = 32ull * A.iters;
    NodeCtx c{};

    u32 hbase = 0;  // help mode covers nodes [hbase, nn)
    if (!A.help) {
        // batch mode: A.batch nodes per cursor atomic, each searched alone, for all but the
        // last A.tail nodes; those then run in help mode so that no warp is left with a
        // straggler batch while the others idle
        hbase = nn > A.tail ? nn - A.tail : 0;
        for (;;) {
            u32 n0 = 0;
            if (lane == 0) n0 = atomicAdd(A.cursor, A.batch);
            n0 = __shfl_sync(FULL, n0, 0);
            if (n0 >= hbase) break;
            const u32 n1 = min(n0 + A.batch, hbase);
            // leaves: the next node's record and keys are loaded while this node is searched
            // (two-stage: keys of n + 1 from its record fetched one node earlier, record of n + 2)
            constexpr bool kLeafPf = KIND == SK_LEAF_RF || KIND == SK_LEAF_BF;
            LeafPrefetch pf{}, pf_next{};
            NodeRec rec2{};
            if (kLeafPf) {
                pf.rec = A.nodes[n0];
                if (n0 + 1 < n1) rec2 = A.nodes[n0 + 1];
                pf.k = lane < pf.rec.size ? A.lo[pf.rec.key_off + lane] : 0;
                pf.ab = KIND == SK_LEAF_RF && lane < pf.rec.size ? A.ab[pf.rec.key_off + lane] : 0;
            }
            for (u32 n = n0; n < n1; ++n) {
                if (KIND == SK_UPPER && A.nodes[n].size > kWarpKeyCap) continue;  // k_search_upper_big
                load_node<KIND, VAR == V_WIDE>(A, n, lane, G, T8, c, kLeafPf ? &pf : nullptr);
                if (kLeafPf && n + 1 < n1) {
                    pf_next.rec = rec2;
                    pf_next.k = lane < rec2.size ? A.lo[rec2.key_off + lane] : 0;
                    pf_next.ab = KIND == SK_LEAF_RF && lane < rec2.size ? A.ab[rec2.key_off + lane] : 0;
                    if (n + 2 < n1) rec2 = A.nodes[n + 2];
                }
                u64 val = 0;
                // (keys-parallel only where few trials are expected: c0 (s - c0) / s = the
                // binomial variance of the left count, trials ~ sqrt(2 pi var); balanced splits
                // need more and run faster as 32-seed windows, pass AO)
                if (KIND == SK_UPPER && c.s <= A.upper_kp && (u64)c.target * (c.s - c.target) <= (u64)A.upper_kp_var * c.s) {
                    val = upper_keys_parallel(A, G, c, lane);
                } else {
                    u64 wstart = 0;
                    // (nodes that run_window sends to an early-rejection variant keep it)
                    const bool lean = A.lean && (VAR == V_PLAIN || !c.cp);
                    if (!(lean && lean_windows<KIND, VAR>(A, K, c, lane, (u32)ws, &val, wstart)))
                        for (;; wstart += ws) {
                            if (wstart >= kSeedCap) {
                                if (lane == 0) atomicOr(A.err, 1u);
                                val = KIND == SK_LEAF_RF ? wstart * c.s : wstart;
                                break;
                            }
                            if (run_window<KIND, VAR>(A, K, c, wstart, lane, &val, QS, QC)) break;
                        }
                }
                if (lane == 0) A.values[c.slot] = val;
                if ((KIND == SK_UPPER || KIND == SK_LOWER) && A.lo_w)
                    fused_reorder<KIND>(A, G, A.nodes[n].key_off, c, val, lane);
                __syncwarp();
                if (kLeafPf) pf = pf_next;
            }
        }
        if (A.tail == 0) {
            RS_COUNT_FLUSH(A.exec);
            return;
        }
    }

    // help mode: per-node window dispenser + helping
    u32* const hcursor = A.help ? A.cursor : A.cursor + 1;
    u32 node = NONE;
    for (;;) {
        if (node == NONE) {
            u32 n = 0;
            if (lane == 0) n = hbase + atomicAdd(hcursor, 1u);
            n = __shfl_sync(FULL, n, 0);
            if (n >= nn) {
                n = find_help(A, gw, lane, nn);
                if (n == NONE) break;
            } else if (KIND == SK_UPPER && A.nodes[n].size > kWarpKeyCap) {
                continue;  // searched by k_search_upper_big
            }
            node = n;
            if (lane == 0) ((volatile int*)A.active)[gw] = (int)n;
            load_node<KIND, VAR == V_WIDE>(A, n, lane, G, T8, c);
        }
        u32 w = 0;
        u64 f = 0;
        if (lane == 0) {
            w = atomicAdd(A.next_win + c.slot, 1u);
            f = ld_volatile_u64(A.values + c.slot);
        }
        w = __shfl_sync(FULL, w, 0);
        f = shfl64(f, 0);
        const u64 wstart = (u64)w * ws;
        const u64 lb = KIND == SK_LEAF_RF ? wstart * c.s : wstart;
        if (lb >= f) {  // a smaller value is already committed: node finished for us
            node = NONE;
            continue;
        }
        if (wstart >= kSeedCap) {
            if (lane == 0) {
                atomicOr(A.err, 1u);
                atomicMin((unsigned long long*)(A.values + c.slot), (unsigned long long)lb);
            }
            node = NONE;
            continue;
        }
        u64 val;
        if (run_window<KIND, VAR>(A, K, c, wstart, lane, &val, QS, QC) && lane == 0)
            atomicMin((unsigned long long*)(A.values + c.slot), (unsigned long long)val);
    }
    RS_COUNT_FLUSH(A.exec);
}

// Upper splits of nodes above the warp engine's shared-memory capacity (kWarpKeyCap keys;
// only buckets larger than that have such nodes, SURVEY 8(b) "bucket_size >= 1").  One block
// per node, keys read from global memory (L2-resident); a window of 32 consecutive seeds per
// step, warp i counting |{k : h_k < T}| for seed w + i (T = ceil(c0 2^32 / s), the same
// predicate as count_left); the smallest seed of the first window with a hit is the minimal
// seed.  These nodes need about sqrt(pi s / 2) trials (tens to hundreds), so this path is
// not throughput-critical.
__global__ void __launch_bounds__(1024) k_search_upper_big(const NodeRec* __restrict__ nodes, u32 n_nodes,
                                                           const u64* __restrict__ lo, u64* __restrict__ values,
                                                           u32 u2, u32* err, const u32* dup) {
    __shared__ u32 s_hit;
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (dup[0] || dup[1] > 1) return;
    for (u32 n = blockIdx.x; n < n_nodes; n += gridDim.x) {
        const NodeRec rec = nodes[n];
        const u32 s = rec.size;
        if (s <= kWarpKeyCap) continue;  // warp engine
        const u32 c0 = (s / 2 + u2 - 1) / u2 * u2;  // R6
        const u32 T = (u32)((((u64)c0 << 32) + s - 1) / s);
        const u64* __restrict__ k = lo + rec.key_off;
        u64 val = ~0ull;
        for (u64 w = 0;; w += nwarps) {
            if (w >= kSeedCap) {
                if (threadIdx.x == 0) atomicOr(err, 1u);
                val = w;
                break;
            }
            if (threadIdx.x == 0) s_hit = NONE;
            __syncthreads();
            const u64 sigma = w + wib;
            u32 cnt = 0;
            for (u32 j = lane; j < s; j += 32) cnt += remix_hi(k[j] + sigma) < T;
            cnt = __reduce_add_sync(FULL, cnt);
            if (lane == 0 && cnt == c0) atomicMin(&s_hit, wib);
            __syncthreads();
            const u32 hit = s_hit;
            __syncthreads();
            if (hit != NONE) {
                val = w + hit;
                break;
            }
        }
        if (threadIdx.x == 0) values[rec.slot] = val;
    }
}

// --------------------------------------------------------- sub-warp leaves --
//
// Leaves of at most 8 keys (l <= 8, e.g. C2: ~52 base seeds per leaf): a 32-seed window per leaf
// overshoots its minimal base seed by ~16 of ~52 seeds (executed / algorithmic evaluations 1.32
// at C2).  Here a warp is four 8-lane sub-warps, each owning one leaf: its lanes try 8
// consecutive base seeds k .. k+7 per step (lane i: k + i), the keys of the leaf in the
// sub-warp's shared-memory groups; the lowest lane of the sub-warp with a fit, with its
// smallest r, gives the minimal value of that step, and every smaller base seed failed in
// earlier steps, so it is the minimal stored value.
// Feeding four independent leaves without stalls: the warp claims kSubBatch leaf records per
// cursor atomic (one per lane, kept in registers), and every sub-warp holds the keys of its NEXT leaf
// in registers (loaded when the current one is installed), so a finished sub-warp installs
// the next leaf from registers; the only global-memory waits are one record batch per
// kSubBatch leaves.
constexpr u32 kSubLeafMax = 8;
// records per cursor atomic: a batch is ~2 steps of work per leaf it holds; 32 left up to one
// batch (~100 us at C2) of tail when the cursor ran out (ncu: 42 % warps active, pass X)
constexpr u32 kSubBatch = 8;

template <int KIND>
__global__ void __launch_bounds__(128, 8) k_leaf_sub(const Args A) {
    __shared__ __align__(16) u32 sG[4][4][2 * 20];  // [warp][sub-warp][2 groups x 20 words]
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5, sub = lane >> 3, sl = lane & 7;
    RS_COUNT_INIT();
    if (A.dup[0] || A.dup[1] > 1) return;
    const u32 nn = *A.n_nodes;
    u32* G = sG[wib][sub];
    // record batch: lane i holds record (batch base + i); bnext = the next one to hand out
    NodeRec brec{};
    u32 bnext = 0, bcount = 0;
    bool dry = false;  // the cursor passed the last leaf (warp-uniform)
    // current leaf of the sub-warp, and its prefetched next leaf (this lane's key / A-B byte)
    u32 m = 0, full = 0, slot = 0, margin = 0, k = 0;
    bool busy = false;
    bool have_pf = false;
    u32 pf_m = 0, pf_slot = 0;
    u64 pf_key = 0;
    u8 pf_ab = 0;
    const u8* lut = nullptr;
    for (;;) {
        // 1. sub-warps whose leaf is done (or none yet) install their prefetched leaf
        const bool inst = !busy && have_pf;
        if (__any_sync(FULL, inst)) {
            if (inst) {
                m = pf_m;
                slot = pf_slot;
                full = (1u << m) - 1u;
                k = 0;
                busy = true;
                have_pf = false;
                const bool valid = sl < m;
                const u64 key = valid ? pf_key : 0;
                const bool isb = KIND == SK_LEAF_RF && valid && pf_ab;
                const u32 g = 20 * (sl >> 2), q = sl & 3, kh = (u32)(key >> 32);
                G[g + q] = (u32)key;
                G[g + 4 + q] = kh;
                G[g + 8 + q] = key_const(kh);
                G[g + 12 + q] = valid && !isb ? FULL : 0u;
                G[g + 16 + q] = isb ? FULL : 0u;
                margin = valid ? ~(u32)key : FULL;
            }
            // carry margin of each sub-warp's leaf: min over its keys of 2^32 - 1 - k_lo (the
            // installing sub-warps' values; the others keep theirs)
            u32 mg = margin;
            for (int d = 4; d; d >>= 1) mg = min(mg, __shfl_xor_sync(FULL, mg, d));
            if (inst) margin = mg;
            if (inst) lut = KIND == SK_LEAF_RF && A.fit_lut ? A.fit_lut + fit_lut_off(m) : nullptr;
            __syncwarp();
        }
        // 2. sub-warps without a prefetched leaf take the next records of the warp's batch (in
        // sub-warp order; a new batch of 32 records per cursor atomic when it runs out); each
        // record is broadcast from the lane holding it and the taker loads its lane's key and
        // A/B byte, consumed at its next install (no wait here)
        u32 want = __ballot_sync(FULL, !have_pf && sl == 0);
        while (want) {
            if (bnext >= bcount) {
                if (dry) break;
                u32 b0 = 0;
                if (lane == 0) b0 = atomicAdd(A.cursor, kSubBatch);
                b0 = __shfl_sync(FULL, b0, 0);
                bcount = b0 >= nn ? 0u : min(kSubBatch, nn - b0);
                bnext = 0;
                if (lane < bcount) brec = A.nodes[b0 + lane];
                if (bcount < kSubBatch) dry = true;  // (the cursor passed the last leaf)
                if (bcount == 0) break;
            }
            const u32 who = (u32)(__ffs(want) - 1) >> 3;  // the requesting sub-warp
            const u32 idx = bnext++;
            const u32 koff = __shfl_sync(FULL, brec.key_off, (int)idx);
            const u32 ksz = __shfl_sync(FULL, brec.size, (int)idx);
            const u32 kslot = __shfl_sync(FULL, brec.slot, (int)idx);
            if (sub == who) {
                have_pf = true;
                pf_m = ksz;
                pf_slot = kslot;
                pf_key = sl < ksz ? A.lo[koff + sl] : 0;
                pf_ab = KIND == SK_LEAF_RF && sl < ksz ? A.ab[koff + sl] : 0;
            }
            want &= want - 1;
        }
        if (!__any_sync(FULL, busy || have_pf)) break;
        if (!__any_sync(FULL, busy)) continue;  // (only prefetched leaves: install them)
        // 3. one step: lane sl tries base seed k + sl.  No-carry path (remix_hi_nc, the engine's
        // 4-key groups) while every key's low word + the step's largest value stays below 2^32
        // (the leaf's carry margin), else the generic 64-bit path.
        const u64 base = KIND == SK_LEAF_RF ? ((u64)k + sl) * m : (u64)k + sl;
        u32 a = 0, b = 0;
        RS_COUNT_RAW(__reduce_add_sync(FULL, busy ? m : 0u));
        if (busy) {
            const u64 top = KIND == SK_LEAF_RF ? ((u64)k + kSubLeafMax) * m : (u64)k + kSubLeafMax;
            if (top <= margin) {
#pragma unroll
                for (u32 gi = 0; gi < kSubLeafMax / 4; ++gi) {
                    const u32* g = G + 20 * gi;
                    u32 h[4];
                    hash4<0>(g, (u32)base, h, 0u);
                    const uint4 ma = *reinterpret_cast<const uint4*>(g + 12);
                    const uint4 mb = *reinterpret_cast<const uint4*>(g + 16);
                    const u32 t0 = 1u << __umulhi(h[0], m), t1 = 1u << __umulhi(h[1], m);
                    const u32 t2 = 1u << __umulhi(h[2], m), t3 = 1u << __umulhi(h[3], m);
                    a |= (t0 & ma.x) | (t1 & ma.y) | (t2 & ma.z) | (t3 & ma.w);
                    b |= (t0 & mb.x) | (t1 & mb.y) | (t2 & mb.z) | (t3 & mb.w);
                }
            } else {
#pragma unroll
                for (u32 j = 0; j < kSubLeafMax; ++j) {
                    const u32* gp = G + 20 * (j >> 2) + (j & 3);
                    const u32 bit = 1u << __umulhi(remix_hi((((u64)gp[4] << 32) | gp[0]) + base), m);
                    a |= bit & gp[12];
                    b |= bit & gp[16];
                }
            }
        }
        int r = -1;
        const bool ok = busy && (KIND == SK_LEAF_BF ? (a == full && (r = 0) == 0)
                                 : lut ? fit_rotation_lut(a, b, m, lut, r)
                                       : fit_rotation_lane(a, b, m, full, r));
        const u32 bal = __ballot_sync(FULL, ok);
        const u32 mine = (bal >> (sub * 8)) & 0xffu;
        const int rw = __shfl_sync(FULL, r, (int)(sub * 8) + (mine ? __ffs(mine) - 1 : 0));
        if (busy) {
            if (mine) {
                const u32 win = __ffs(mine) - 1;
                if (sl == 0) A.values[slot] = KIND == SK_LEAF_RF ? ((u64)k + win) * m + (u32)rw : (u64)k + win;
                busy = false;
            } else {
                k += kSubLeafMax;
                if ((u64)k + kSubLeafMax >= (1ull << 32)) {  // (far beyond any leaf of <= 8 keys)
                    if (sl == 0) {
                        atomicOr(A.err, 1u);
                        A.values[slot] = KIND == SK_LEAF_RF ? (u64)k * m : k;
                    }
                    busy = false;
                }
            }
        }
        __syncwarp();
    }
    RS_COUNT_FLUSH(A.exec);
}

template <int KIND, int VAR = V_PLAIN>
void launch_kind(const PhaseLaunch& P, const Args& A, u32 wpb, size_t smem, u32 grid, cudaStream_t st) {
    cudaFuncSetAttribute(k_search<KIND, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k_search<KIND, VAR><<<grid, wpb * 32, smem, st>>>(A);
}

}  // namespace

u32 search_active_slots(int sm_count) { return (u32)sm_count * 16u * kWarpsPerBlockMax; }

// The rotation-fit table of fit_rotation_lut (kFitLutMax = 8: 87,380 bytes), built on the host
// from the definition rot_m^r(b) = (bb >> (m - r)) & full, bb = b | b << m (the same test as
// fit_rotation_lane), uploaded once per device.
const u8* fit_lut_device() {
    static std::mutex mu;
    static std::map<int, u8*> tabs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = tabs.find(dev);
    if (it != tabs.end()) return it->second;
    std::vector<u8> t(fit_lut_off(kFitLutMax + 1), 0xff);
    for (u32 m = 1; m <= kFitLutMax; ++m) {
        const u32 full = (1u << m) - 1u;
        for (u32 b = 0; b <= full; ++b) {
            const u64 bb = (u64)b | ((u64)b << m);
            for (u32 a = 0; a <= full; ++a) {
                const u32 na = ~a & full;
                u8 r = 0xff;
                for (u32 q = 0; q < m; ++q)
                    if (((u32)(bb >> (m - q)) & full) == na) {
                        r = (u8)q;
                        break;
                    }
                t[fit_lut_off(m) + ((b << m) | a)] = r;
            }
        }
    }
    u8* d = nullptr;
    if (cudaMalloc(&d, t.size()) != cudaSuccess || cudaMemcpy(d, t.data(), t.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;  // (the serial rotation check then runs)
    }
    tabs[dev] = d;
    return d;
}

bool launch_search(const PhaseLaunch& P, cudaStream_t st) {
    if (P.n_nodes_host == 0) return false;
    Args A{};
    static const int lut_env = getenv("RS_FIT_LUT") ? atoi(getenv("RS_FIT_LUT")) : 1;
    A.fit_lut = lut_env && P.kind == SK_LEAF_RF ? fit_lut_device() : nullptr;
    static const int lean_env = getenv("RS_LEAN") ? atoi(getenv("RS_LEAN")) : 1;
    A.lean = lean_env ? 1u : 0u;
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
    A.exec = P.exec;
    static const int lane_fit = getenv("RS_LANE_FIT") ? atoi(getenv("RS_LANE_FIT")) : 10;
    A.lane_fit = (u32)std::max(0, lane_fit);
    A.help = P.help;
    // early-rejection checkpoints (per mille of the node size; RS_CP1 / RS_CP2 override, 0 = off)
    {
        // L1: two-stage cascade at 780 / 880 per mille; L2: one checkpoint at 940 (measured,
        // DESIGN.md 5)
        static const int cp1 = getenv("RS_CP1") ? atoi(getenv("RS_CP1")) : 780;
        static const int cp2 = getenv("RS_CP2") ? atoi(getenv("RS_CP2")) : 940;
        static const int cp1b = getenv("RS_CP1B") ? atoi(getenv("RS_CP1B")) : 880;
        static const int cp2b = getenv("RS_CP2B") ? atoi(getenv("RS_CP2B")) : 0;
        A.cp_l1 = (u32)((u64)P.u1 * cp1 / 4000);
        A.cp_l2 = (u32)((u64)P.u2 * cp2 / 4000);
        A.cp_l1b = (u32)((u64)P.u1 * cp1b / 4000);
        A.cp_l2b = (u32)((u64)P.u2 * cp2b / 4000);
        // batch-mode phases (expected < 1024 trials per node, 32-seed windows) flush a partial
        // stage-2 batch at every window end, which costs more than the rejection saves (C2:
        // L1 -14 %, L2 -5 % without it; tools/c2_knobs.sh); RS_CP_BATCH=1 keeps it (tests)
        static const int cpbatch = getenv("RS_CP_BATCH") ? atoi(getenv("RS_CP_BATCH")) : 0;
        if (!P.help && !cpbatch) A.cp_l1 = A.cp_l2 = A.cp_l1b = A.cp_l2b = 0;
        static const int cpl = getenv("RS_CPL") ? atoi(getenv("RS_CPL")) : 1;
        A.cp_leaf = cpl ? 1u : 0u;
        static const int cplast = getenv("RS_CPLAST") ? atoi(getenv("RS_CPLAST")) : 1;
        A.cp_last = cplast ? 1u : 0u;
        static const int cpw = getenv("RS_CPW") ? atoi(getenv("RS_CPW")) : 1;
        A.cp_wide = cpw ? 1u : 0u;
        static const int cpl2 = getenv("RS_CPL2") ? atoi(getenv("RS_CPL2")) : 1;
        A.cp_leaf2 = cpl2 ? 1u : 0u;
        static const int cpw2 = getenv("RS_CPW2") ? atoi(getenv("RS_CPW2")) : 1;
        A.cp_wide2 = cpw2 ? 1u : 0u;
    }
    // (off by default: 3-8 % slower than the warp engine at C2, ab_j / ab_i in DESIGN.md 5)
    static const int subleaf = getenv("RS_SUB_LEAF") ? atoi(getenv("RS_SUB_LEAF")) : 0;
    if (subleaf && (P.kind == SK_LEAF_RF || P.kind == SK_LEAF_BF) && P.max_size <= kSubLeafMax) {
        // leaves of at most 8 keys: four per warp (k_leaf_sub); the phase's batch cursor is zeroed
        const u32 blocks = std::max<u32>(1, std::min<u32>((P.n_nodes_host + 15) / 16, (u32)P.sm_count * 8));
        if (P.kind == SK_LEAF_RF)
            k_leaf_sub<SK_LEAF_RF><<<blocks, 128, 0, st>>>(A);
        else
            k_leaf_sub<SK_LEAF_BF><<<blocks, 128, 0, st>>>(A);
        g_launches++;
        return false;
    }
    if (P.kind == SK_UPPER && P.max_size > kWarpKeyCap) {  // oversized upper nodes first
        const u32 grid_big = std::min<u32>(P.n_nodes_host, (u32)P.sm_count * 2);
        k_search_upper_big<<<grid_big, 1024, 0, st>>>(P.nodes, P.n_nodes_host, P.lo, P.values, P.u2, P.err, P.dup);
        g_launches++;
    }
    // kernel variant of the phase (its register count and queue needs set the occupancy)
    int var = V_PLAIN;
    if (P.kind == SK_LOWER) {
        // the phase holds one level: lower level 2 iff its largest node exceeds u1
        const bool l2 = P.max_size > P.u1;
        const u32 unit = l2 ? P.u1 : P.leaf, f = l2 ? P.u2 / P.u1 : P.u1 / P.leaf;
        const u32 w = 32 - __builtin_clz(unit + 1);
        var = (f - 1) * w > 32 ? V_WIDE : (A.cp_l1 | A.cp_l2) ? V_CP : V_PLAIN;
    } else if ((P.kind == SK_LEAF_RF || P.kind == SK_LEAF_BF) && A.cp_leaf && P.max_size >= 10) {
        var = V_CP;
    }
    const void* kfn = nullptr;
    switch (P.kind) {
        case SK_UPPER: kfn = (const void*)k_search<SK_UPPER>; break;
        case SK_LOWER:
            kfn = var == V_WIDE ? (const void*)k_search<SK_LOWER, V_WIDE>
                  : var == V_CP ? (const void*)k_search<SK_LOWER, V_CP>
                                : (const void*)k_search<SK_LOWER>;
            break;
        case SK_LEAF_RF:
            kfn = var == V_CP ? (const void*)k_search<SK_LEAF_RF, V_CP> : (const void*)k_search<SK_LEAF_RF>;
            break;
        case SK_LEAF_BF:
            kfn = var == V_CP ? (const void*)k_search<SK_LEAF_BF, V_CP> : (const void*)k_search<SK_LEAF_BF>;
            break;
    }
    // early-rejection queues per warp (64 entries per array): splits keep (seed, counter) per
    // stage (the wide variant seed + two counter words), leaves (seed, a, b) per stage
    u32 qwords = 0;
    if (var != V_PLAIN) {
        const bool two = P.kind == SK_LOWER ? (P.max_size > P.u1 ? A.cp_l2b : A.cp_l1b) != 0 : A.cp_leaf2 != 0;
        const u32 per_stage = (P.kind == SK_LOWER && var == V_CP) ? 128 : 192;
        qwords = per_stage * (two ? 2 : 1);
    }
    A.qwords = qwords;
    // warp-private buffer: key groups (12 or 20 words per 4 keys) + byte shift table + queues
    u32 cap = (std::min(P.max_size, kWarpKeyCap) + 3) & ~3u;
    if (cap < 32) cap = 32;
    A.warp_cap = cap;
    const u32 GW = (P.kind == SK_LEAF_RF || P.kind == SK_LEAF_BF) ? 20 : 12;
    const size_t per_warp = ((size_t)GW * (cap / 4 + 1) + (cap + 32 + 15) / 16 * 4 + qwords) * sizeof(u32);
    u32 wpb = kWarpsPerBlockMax;
    while (wpb > 1 && per_warp * wpb > 200 * 1024) --wpb;
    const size_t smem = per_warp * wpb;
    // resident blocks per SM (occupancy of the variant launched), persistent grid
    int occ = 1;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, (int)(wpb * 32), smem);
    if (occ < 1) occ = 1;
    int max_blocks = (int)(search_active_slots(P.sm_count) / wpb);
    u32 grid = (u32)std::min(occ * P.sm_count, max_blocks);
    // batch mode: about 8 batches per resident warp, at most 8 nodes per batch
    A.batch = 1;
    if (!P.help) {
        const u64 slots = (u64)grid * wpb;
        u64 b = P.n_nodes_host / (slots * 8);
        A.batch = (u32)std::max<u64>(1, std::min<u64>(8, b));
        grid = std::min<u32>(grid, (P.n_nodes_host + A.batch * wpb - 1) / (A.batch * wpb));
    }
    {
        static const int tl = getenv("RS_TAIL") ? atoi(getenv("RS_TAIL")) : 0;  // x resident warps (off: measured slower)
        A.tail = P.help ? 0u : (u32)tl * grid * wpb;
    }
    if (grid == 0) grid = 1;
    A.n_warps = grid * wpb;
    // fused redistribution (A7) for batch-mode split phases of small nodes: every node is
    // finished by the one warp that holds its keys
    static const int fuse = getenv("RS_FUSE_REORDER") ? atoi(getenv("RS_FUSE_REORDER")) : 1;
    const bool fused = fuse && P.fuse_reorder && (P.kind == SK_UPPER || P.kind == SK_LOWER) && !P.help &&
                       A.tail == 0 && P.max_size <= kFuseMax;
    static const int ukp = getenv("RS_UPPER_KP") ? atoi(getenv("RS_UPPER_KP")) : 1;
    static const int ukp_max = getenv("RS_UPPER_KP_MAX") ? atoi(getenv("RS_UPPER_KP_MAX")) : (int)kUpperKpMax;
    A.upper_kp = ukp && P.kind == SK_UPPER && !P.help && A.tail == 0 ? (u32)std::min<int>(ukp_max, (int)kUpperKpMax) : 0u;
    static const int ukp_var = getenv("RS_UPPER_KP_VAR") ? atoi(getenv("RS_UPPER_KP_VAR")) : 5;  // (pass AP)
    A.upper_kp_var = (u32)std::max(0, ukp_var);
    A.lo_w = fused ? P.lo_w : nullptr;
    A.ab_w = fused ? P.ab_w : nullptr;
    switch (P.kind) {
        case SK_UPPER: launch_kind<SK_UPPER>(P, A, wpb, smem, grid, st); break;
        case SK_LOWER:
            if (var == V_WIDE)
                launch_kind<SK_LOWER, V_WIDE>(P, A, wpb, smem, grid, st);
            else if (var == V_CP)
                launch_kind<SK_LOWER, V_CP>(P, A, wpb, smem, grid, st);
            else
                launch_kind<SK_LOWER>(P, A, wpb, smem, grid, st);
            break;
        case SK_LEAF_RF:
            if (var == V_CP)
                launch_kind<SK_LEAF_RF, V_CP>(P, A, wpb, smem, grid, st);
            else
                launch_kind<SK_LEAF_RF>(P, A, wpb, smem, grid, st);
            break;
        case SK_LEAF_BF:
            if (var == V_CP)
                launch_kind<SK_LEAF_BF, V_CP>(P, A, wpb, smem, grid, st);
            else
                launch_kind<SK_LEAF_BF>(P, A, wpb, smem, grid, st);
            break;
    }
    g_launches++;
    return fused;
}

// ------------------------------------------------------------------ reorder --

// A7: stable partition of each split node's keys by child index with its found seed
// (P:311-313), in place: one warp per node stages the node's (lo, A/B) (shared
// memory; a global scratch slice for nodes above kReorderSmemCap keys), then writes every
// key to its child's sub-range (children occupy consecutive sub-ranges in part order, so
// every child's keys are contiguous for the next phase).
constexpr u32 kReorderSmemCap = 8192;

__device__ __forceinline__ void reorder_node(const NodeRec r, u64 sigma, u64* __restrict__ lo, u8* __restrict__ ab,
                                             u64* slo, u8* sab, u32 leaf, u32 u1, u32 u2, u32 lane) {
    const u32 s = r.size;
    for (u32 j = lane; j < s; j += 32) {
        slo[j] = lo[r.key_off + j];
        sab[j] = ab[r.key_off + j];
    }
    __syncwarp();
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
            k = slo[j];
            b = sab[j];
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
            lo[r.key_off + dst] = k;
            ab[r.key_off + dst] = b;
        }
    }
    __syncwarp();
}

__global__ void k_reorder(const NodeRec* __restrict__ nodes, u32 n_nodes, const u64* __restrict__ values,
                          u64* __restrict__ lo, u8* __restrict__ ab, u32 leaf, u32 u1, u32 u2, u32 cap,
                          const u32* n_nodes_dev) {
    extern __shared__ __align__(16) unsigned char rsm[];
    if (n_nodes_dev) n_nodes = *n_nodes_dev;
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    u64* slo = reinterpret_cast<u64*>(rsm + (size_t)wib * cap * 9);
    u8* sab = reinterpret_cast<u8*>(slo + cap);
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    for (u32 n = blockIdx.x * (blockDim.x >> 5) + wib; n < n_nodes; n += nwarps) {
        const NodeRec r = nodes[n];
        if (r.size > cap) continue;  // k_reorder_big
        reorder_node(r, values[r.slot], lo, ab, slo, sab, leaf, u1, u2, lane);
    }
}

// nodes above the shared-memory capacity (upper splits of oversized buckets): the same
// warp-per-node partition staged in a global scratch slice of `cap` keys per warp
__global__ void k_reorder_big(const NodeRec* __restrict__ nodes, u32 n_nodes, const u64* __restrict__ values,
                              u64* __restrict__ lo, u8* __restrict__ ab, u32 u2, u32 smem_cap, u32 cap,
                              u64* __restrict__ scratch) {
    const u32 lane = threadIdx.x & 31;
    const u32 gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const u32 nwarps = gridDim.x * (blockDim.x >> 5);
    u64* slo = scratch + (size_t)gw * cap * 2;  // cap u64 keys + cap bytes (rounded up)
    u8* sab = reinterpret_cast<u8*>(slo + cap);
    for (u32 n = gw; n < n_nodes; n += nwarps) {
        const NodeRec r = nodes[n];
        if (r.size <= smem_cap) continue;
        reorder_node(r, values[r.slot], lo, ab, slo, sab, 0, 0, u2, lane);
    }
}

void launch_reorder(const NodeRec* nodes, u32 n_nodes, const u64* values, u64* lo, u8* ab, u32 leaf, u32 u1, u32 u2,
                    u32 max_size, int sm_count, u64* big_scratch, cudaStream_t st, const u32* n_nodes_dev) {
    if (n_nodes == 0) return;
    const u32 cap = (std::min(max_size, kReorderSmemCap) + 15) & ~15u;
    const size_t per_warp = (size_t)cap * 9;
    u32 wpb = 8;
    while (wpb > 1 && per_warp * wpb > 96 * 1024) --wpb;
    cudaFuncSetAttribute(k_reorder, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_reorder, (int)(wpb * 32), per_warp * wpb);
    if (occ < 1) occ = 1;
    u32 blocks = (n_nodes + wpb - 1) / wpb;
    blocks = std::min<u32>(blocks, (u32)(occ * sm_count));
    k_reorder<<<blocks, wpb * 32, per_warp * wpb, st>>>(nodes, n_nodes, values, lo, ab, leaf, u1, u2, cap, n_nodes_dev);
    g_launches++;
    if (max_size > kReorderSmemCap) {
        // big_scratch holds kReorderBigWarps slices of 2 * max_size words
        k_reorder_big<<<kReorderBigWarps / 4, 128, 0, st>>>(nodes, n_nodes, values, lo, ab, u2, cap, max_size,
                                                          big_scratch);
        g_launches++;
    }
}

// -------------------------------------------------------------- bucket trees --
//
// Small configurations (every node class in batch mode, buckets of at most a few hundred keys,
// e.g. l = 8, b = 100): one warp builds a whole bucket, the paper's per-bucket recursion (P:110-
// 119) mapped onto a warp.  The bucket's keys are copied into the warp's shared memory
// once; its nodes are searched in preorder (the template order, so a node's keys are in place
// when it is reached): each split is searched with the engine's windows (minimal seed, as in
// batch mode) and its keys are partitioned in shared memory (reorder_node, smem -> smem), each
// leaf is searched on its sub-range.  No node table, no global key traffic per node, no
// redistribution passes and one tail for the whole build instead of one per phase.

template <int KIND>
__device__ __forceinline__ u64 tree_search_node(const Args& A, const NodeRec& rec, u32 lane, u32* G, u8* T8,
                                                const u64* blo, const u8* bab, u32* QS, u32* QC) {
    NodeCtx c{};
    load_node<KIND, false>(A, 0, lane, G, T8, c, nullptr, &rec, blo, bab);
    if (KIND == SK_UPPER && c.s <= A.upper_kp) return upper_keys_parallel(A, G, c, lane);
    const KeysView K{G, (u32)__cvta_generic_to_shared(T8), 0u, (u32)__cvta_generic_to_shared(&s_full_tab[0][0])};
    const u64 ws = 32ull * A.iters;
    for (u64 wstart = 0;; wstart += ws) {
        if (wstart >= kSeedCap) {
            if (lane == 0) atomicOr(A.err, 1u);
            return KIND == SK_LEAF_RF ? wstart * c.s : wstart;
        }
        u64 val;
        if (run_window<KIND, V_PLAIN>(A, K, c, wstart, lane, &val, QS, QC)) return val;
    }
}

// work-buffer words of a bucket-tree warp: split groups (12 words per 4 keys), leaf groups (20),
// or the duplicate-check table (2 words per slot, 2 * cap slots)
__host__ __device__ __forceinline__ u32 tree_gwords(u32 cap, u32 leaf) {
    u32 g = 12 * (cap / 4 + 1);
    if (20 * (leaf / 4 + 2) > g) g = 20 * (leaf / 4 + 2);
    u32 ts = 64;
    while (ts < 2 * cap) ts <<= 1;
    return 2 * ts > g ? 2 * ts : g;
}

template <bool RF>
__global__ void __launch_bounds__(128, 6) k_bucket_tree(const Args A, const TreeArgs T) {
    extern __shared__ __align__(16) u32 smem32[];
    const u32 lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const u32 cap = A.warp_cap;  // >= every bucket size searched, multiple of 16
    const u32 gwords = tree_gwords(cap, A.leaf);
    const u32 twords = (cap + 32 + 15) / 16 * 4;
    const u32 per_warp = gwords + twords + 2 * cap + cap / 4 + 2 * cap + cap / 4;
    u32* G = smem32 + (size_t)wib * per_warp;
    u8* T8 = reinterpret_cast<u8*>(G + gwords);
    u64* blo = reinterpret_cast<u64*>(G + gwords + twords);  // the bucket's keys (node order)
    u8* bab = reinterpret_cast<u8*>(blo + cap);
    u64* slo = reinterpret_cast<u64*>(bab + cap);            // reorder staging
    u8* sab = reinterpret_cast<u8*>(slo + cap);
    init_lower_tables(A);
    RS_COUNT_INIT();
    if (A.dup[0] || A.dup[1] > 1) return;
    const u64 base0 = T.nodebase[0];
    for (;;) {
        u32 b0 = 0;
        if (lane == 0) b0 = atomicAdd(T.bcursor, T.bbatch);
        b0 = __shfl_sync(FULL, b0, 0);
        if (b0 >= T.B) break;
        const u32 b1 = (u32)min((u64)b0 + T.bbatch, T.B);
        for (u32 b = b0; b < b1; ++b) {
            const u64 c0 = T.C[b];
            const u32 s = (u32)(T.C[b + 1] - c0);
            if (s == 0 || s > T.S) continue;  // (above the tables: flagged, rebuilt by the caller)
            __syncwarp();
            for (u32 j = lane; j < s; j += 32) {
                blo[j] = A.lo[c0 + j];
                bab[j] = A.ab[c0 + j];
            }
            if (T.dedupe) {
                // exact duplicate check of the bucket (A2; equal keys <=> equal lo, R2): an
                // open-addressing set over its lo values in the (still free) work buffer; a
                // repeated key fails the build, and the bucket is not searched (its leaf search
                // could never succeed)
                u32 ts = 64;
                while (ts < 2 * s) ts <<= 1;
                unsigned long long* tab = reinterpret_cast<unsigned long long*>(G);
                for (u32 j = lane; j < ts; j += 32) tab[j] = 0;
                __syncwarp();
                bool rep = false;
                u32 zeros = 0;
                for (u32 j = lane; j < s; j += 32) {
                    const u64 v = blo[j];
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
                zeros = __reduce_add_sync(FULL, zeros);
                if (__any_sync(FULL, rep) || zeros > 1) {
                    if (lane == 0) atomicOr(const_cast<u32*>(A.dup), 1u);
                    continue;
                }
            }
            __syncwarp();
            const u32 t0 = T.tstart[s], t1 = T.tstart[s + 1];
            const u64 nb = T.nodebase[b] - base0;
            for (u32 t = t0; t < t1; ++t) {
                const TNodeD x = T.tn[t];
                const NodeRec rec{x.rel_off, x.size, (u32)(nb + (t - t0)), 0};
                u64 val;
                if (x.size <= A.leaf) {
                    val = tree_search_node<RF ? SK_LEAF_RF : SK_LEAF_BF>(A, rec, lane, G, T8, blo, bab, nullptr, nullptr);
                } else {
                    if (x.size <= A.u2)
                        val = tree_search_node<SK_LOWER>(A, rec, lane, G, T8, blo, bab, nullptr, nullptr);
                    else
                        val = tree_search_node<SK_UPPER>(A, rec, lane, G, T8, blo, bab, nullptr, nullptr);
                    // children's keys into their sub-ranges (in shared memory)
                    reorder_node(rec, val, blo, bab, slo, sab, A.leaf, A.u1, A.u2, lane);
                }
                if (lane == 0) A.values[rec.slot] = val;
            }
        }
    }
    RS_COUNT_FLUSH(A.exec);
}

bool bucket_tree_eligible(u32 leaf, u32 S) { return leaf <= 9 && S <= kBucketTreeMax; }

void launch_bucket_tree(const TreeLaunch& L, cudaStream_t st) {
    Args A{};
    A.lo = L.lo;
    A.ab = L.ab;
    A.values = L.values;
    A.err = L.err;
    A.dup = L.dup;
    A.leaf = L.leaf;
    A.u1 = L.u1;
    A.u2 = L.u2;
    A.iters = 1;
    A.exec = L.exec;
    static const int lane_fit = getenv("RS_LANE_FIT") ? atoi(getenv("RS_LANE_FIT")) : 10;
    A.lane_fit = (u32)std::max(0, lane_fit);
    static const int ukp = getenv("RS_UPPER_KP") ? atoi(getenv("RS_UPPER_KP")) : 1;
    A.upper_kp = ukp ? kUpperKpMax : 0u;
    A.upper_kp_var = 1u << 30;  // (the bucket-tree kernel: every upper node up to kUpperKpMax)
    A.qwords = 0;
    const u32 cap = (L.S + 15) & ~15u;
    A.warp_cap = cap;
    TreeArgs T{L.C, L.B, L.nodebase, L.tstart, L.tn, L.S, L.bcursor, 1, L.dedupe ? 1u : 0u};
    const u32 gwords = tree_gwords(cap, L.leaf);
    const size_t per_warp = (size_t)(gwords + (cap + 32 + 15) / 16 * 4 + 2 * cap + cap / 4 + 2 * cap + cap / 4) * 4;
    const u32 wpb = 4;
    const size_t smem = per_warp * wpb;
    const void* fn = L.rf ? (const void*)k_bucket_tree<true> : (const void*)k_bucket_tree<false>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)(wpb * 32), smem);
    if (occ < 1) occ = 1;
    u32 grid = (u32)std::min<u64>((u64)occ * L.sm_count, (L.B + wpb - 1) / wpb);
    // buckets per cursor atomic: a few per warp while many remain, so the last ones finish together
    T.bbatch = (u32)std::max<u64>(1, std::min<u64>(4, L.B / ((u64)grid * wpb * 16)));
    if (grid == 0) grid = 1;
    if (L.rf)
        k_bucket_tree<true><<<grid, wpb * 32, smem, st>>>(A, T);
    else
        k_bucket_tree<false><<<grid, wpb * 32, smem, st>>>(A, T);
    g_launches++;
}

}  // namespace rs
