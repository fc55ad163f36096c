// Device helpers for the RecSplit construction kernels (sm_100a).
// Citation keys: P:n = PAPER.md line n; R<k> = DESIGN.md reading k.
#pragma once
#include <cstdint>

namespace rsd {

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint8_t u8;

constexpr u32 FULL = 0xffffffffu;
constexpr u32 NONE = 0xffffffffu;

// SplitMix64 finalizer constants (R1) and master-hash salts (R2).
constexpr u64 MIX_C1 = 0xbf58476d1ce4e5b9ULL;
constexpr u64 MIX_C2 = 0x94d049bb133111ebULL;
constexpr u32 MIX_C2L = 0x133111ebu;
constexpr u32 MIX_C2H = 0x94d049bbu;
constexpr u64 MHC_SALT_HI = 0x9E3779B97F4A7C15ULL;
constexpr u64 MHC_SALT_LO = 0xC2B2AE3D27D4EB4FULL;

// Full 64-bit remix (used once per key for the master hash code).
__device__ __forceinline__ u64 remix64(u64 z) {
    z = (z ^ (z >> 30)) * MIX_C1;
    z = (z ^ (z >> 27)) * MIX_C2;
    return z ^ (z >> 31);
}

// High 32 bits of remix(x): the only bits remap (R3) consumes.  The last multiply
// only needs the high word of the 64x64 product: hi(xl*C2L) + xl*C2H + xh*C2L.
__device__ __forceinline__ u32 remix_hi(u64 x) {
    x ^= x >> 30;
    x *= MIX_C1;
    x ^= x >> 27;
    const u32 xl = (u32)x, xh = (u32)(x >> 32);
    const u32 zh = __umulhi(xl, MIX_C2L) + xl * MIX_C2H + xh * MIX_C2L;
    return zh ^ (zh >> 31);
}

// remix_hi(k + sigma) for sigma < 2^32 (the fast path of every search).  Pipe budget
// measured with ncu on sm_100a: IMAD.WIDE / IMAD.HI occupy the FMA-heavy pipe for two
// cycles, IMAD for one; IADD3/LOP3/SHF use the ALU pipe.  The sequence below needs
// 8 heavy cycles (x*C1 low 64: 2+1+1, x*C2 high 32: 2+1+1) and 10 ALU instructions
// (two 64-bit xorshifts 4+4, the final 1-bit xorshift 2), plus the 64-bit add.
#define REMIX_HI_TAIL                          \
    "shf.r.wrap.b32 tl, wl, wh, 30;\n\t"       \
    "shr.u32 th, wh, 30;\n\t"                  \
    "xor.b32 wl, wl, tl;\n\t"                  \
    "xor.b32 wh, wh, th;\n\t"                  \
    "mul.wide.u32 p64, wl, 0x1ce4e5b9;\n\t"    \
    "mov.b64 {yl, yh}, p64;\n\t"               \
    "mad.lo.u32 yh, wl, 0xbf58476d, yh;\n\t"   \
    "mad.lo.u32 yh, wh, 0x1ce4e5b9, yh;\n\t"   \
    "shf.r.wrap.b32 tl, yl, yh, 27;\n\t"       \
    "shr.u32 th, yh, 27;\n\t"                  \
    "xor.b32 zl, yl, tl;\n\t"                  \
    "xor.b32 zh, yh, th;\n\t"                  \
    "mul.hi.u32 a, zl, 0x133111eb;\n\t"        \
    "mad.lo.u32 a, zl, 0x94d049bb, a;\n\t"     \
    "mad.lo.u32 a, zh, 0x133111eb, a;\n\t"     \
    "shr.u32 th, a, 31;\n\t"                   \
    "xor.b32 %0, a, th;\n\t"                   \
    "}"

// CARRY: x = (kh:kl) + (H:sigma) with the carry out of the low word (H = high word of the
// 64-bit value, 0 below 2^32); otherwise x = (kh : kl + sigma).
template <bool CARRY>
__device__ __forceinline__ u32 remix_hi_fast(u32 kl, u32 kh, u32 sigma, u32 H = 0) {
    u32 h;
    if (CARRY) {
        asm("{\n\t"
            ".reg .u32 tl, th, wl, wh, yl, yh, zl, zh, a;\n\t"
            ".reg .u64 p64;\n\t"
            "add.cc.u32 wl, %1, %3;\n\t"
            "addc.u32 wh, %2, %4;\n\t"
            REMIX_HI_TAIL
            : "=r"(h)
            : "r"(kl), "r"(kh), "r"(sigma), "r"(H));
    } else {
        asm("{\n\t"
            ".reg .u32 tl, th, wl, wh, yl, yh, zl, zh, a;\n\t"
            ".reg .u64 p64;\n\t"
            "add.u32 wl, %1, %3;\n\t"
            "mov.u32 wh, %2;\n\t"
            REMIX_HI_TAIL
            : "=r"(h)
            : "r"(kl), "r"(kh), "r"(sigma));
    }
    return h;
}

// Variants of the two adds of the no-carry path (ptxas tends to place plain adds on the
// FMA-heavy pipe, which the multiplies already saturate); selected at build time.
#ifndef RS_NC_VARIANT
#define RS_NC_VARIANT 0  // measured fastest on B200 (tools/variant_bench.sh, round 1)
#endif
#if RS_NC_VARIANT == 0
#define RS_NC_ADD1 "add.u32 xl, %1, %4;\n\t"
#define RS_NC_MUL1                               \
    "mul.wide.u32 p64, wl, 0x1ce4e5b9;\n\t"     \
    "mov.b64 {yl, yh}, p64;\n\t"                \
    "add.u32 yh, yh, %3;\n\t"                   \
    "mad.lo.u32 yh, wl, 0xbf58476d, yh;\n\t"
#elif RS_NC_VARIANT == 1
// sad.u32 d, a, 0, c = |a - 0| + c: an add the integer ALU executes
#define RS_NC_ADD1 "sad.u32 xl, %1, 0, %4;\n\t"
#define RS_NC_MUL1                               \
    "mul.wide.u32 p64, wl, 0x1ce4e5b9;\n\t"     \
    "mov.b64 {yl, yh}, p64;\n\t"                \
    "sad.u32 yh, yh, 0, %3;\n\t"                \
    "mad.lo.u32 yh, wl, 0xbf58476d, yh;\n\t"
#elif RS_NC_VARIANT == 3
// sigma add left to ptxas (it picks IMAD.IADD, FMA pipe), kc add on the ALU
#define RS_NC_ADD1 "add.u32 xl, %1, %4;\n\t"
#define RS_NC_MUL1                               \
    "mul.wide.u32 p64, wl, 0x1ce4e5b9;\n\t"     \
    "mov.b64 {yl, yh}, p64;\n\t"                \
    "sad.u32 yh, yh, 0, %3;\n\t"                \
    "mad.lo.u32 yh, wl, 0xbf58476d, yh;\n\t"
#else
// low word by mul.lo, high word by mad.hi with kc as addend (no separate add)
#define RS_NC_ADD1 "sad.u32 xl, %1, 0, %4;\n\t"
#define RS_NC_MUL1                               \
    "mul.lo.u32 yl, wl, 0x1ce4e5b9;\n\t"        \
    "mad.hi.u32 yh, wl, 0x1ce4e5b9, %3;\n\t"    \
    "mad.lo.u32 yh, wl, 0xbf58476d, yh;\n\t"
#endif

// Per-key constant of the no-carry path: with x_hi = k_hi, the high word of
// w = x ^ (x >> 30) is k_hi ^ (k_hi >> 30), and its contribution to (w * C1)_hi is
// the constant kc = (k_hi ^ (k_hi >> 30)) * C1_lo (mod 2^32).
__device__ __forceinline__ u32 key_const(u32 kh) { return (kh ^ (kh >> 30)) * 0x1ce4e5b9u; }

// remix_hi(k + sigma) when k_lo + sigma < 2^32: 8 heavy-pipe cycles (x*C1: IMAD.WIDE with
// the 64-bit addend {0, kc} + one IMAD; x*C2 high word: IMAD.HI + 2 IMAD) and 8 ALU ops.
__device__ __forceinline__ u32 remix_hi_nc(u32 kl, u32 kh, u32 kc, u32 sigma) {
    u32 h;
    asm("{\n\t"
        ".reg .u32 xl, tl, th, wl, yl, yh, zl, zh, a;\n\t"
        ".reg .u64 p64;\n\t"
        RS_NC_ADD1
        "shf.r.wrap.b32 tl, xl, %2, 30;\n\t"
        "xor.b32 wl, xl, tl;\n\t"
        RS_NC_MUL1
        "shf.r.wrap.b32 tl, yl, yh, 27;\n\t"
        "shr.u32 th, yh, 27;\n\t"
        "xor.b32 zl, yl, tl;\n\t"
        "xor.b32 zh, yh, th;\n\t"
        "mul.hi.u32 a, zl, 0x133111eb;\n\t"
        "mad.lo.u32 a, zl, 0x94d049bb, a;\n\t"
        "mad.lo.u32 a, zh, 0x133111eb, a;\n\t"
        "shr.u32 th, a, 31;\n\t"
        "xor.b32 %0, a, th;\n\t"
        "}"
        : "=r"(h)
        : "r"(kl), "r"(kh), "r"(kc), "r"(sigma));
    return h;
}

// remap(h, r) = floor(h_hi * r / 2^32)  (R3) given h_hi
__device__ __forceinline__ u32 remap_hi(u32 hhi, u32 r) { return __umulhi(hhi, r); }

// x << s with PTX clamping semantics: s >= 32 gives 0 (used by packed counters).
__device__ __forceinline__ u32 shl_clamp(u32 x, u32 s) {
    u32 r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}

// 1 << s with clamping (s >= 32 gives 0): a one-bit mask at position s (BMSK with an
// immediate width, so no register has to hold the constant 1)
__device__ __forceinline__ u32 bit_clamp(u32 s) {
    u32 r;
#if RS_BITCLAMP_SHL
    asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(s));
#else
    asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(r) : "r"(s));
#endif
    return r;
}

__device__ __forceinline__ u32 lanemask_lt() {
    u32 r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ u64 shfl64(u64 v, int src) {
    u32 lo = __shfl_sync(FULL, (u32)v, src), hi = __shfl_sync(FULL, (u32)(v >> 32), src);
    return ((u64)hi << 32) | lo;
}

__device__ __forceinline__ u64 ld_volatile_u64(const u64* p) { return *(const volatile u64*)p; }

// Search-phase node record (one per node of a phase list).
struct NodeRec {
    u32 key_off;  // first key of the node in the key arrays
    u32 size;     // s
    u32 slot;     // global preorder slot of its stored value
    u32 pad;
};

// Template node (mirrors rs::TNode).
struct TNodeD {
    u32 rel_off, size, fixed_off, phase, tau, phase_rank;
};

}  // namespace rsd
