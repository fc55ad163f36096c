// Host-callable launchers of the sm_100a kernels (one per pipeline step).
// All launches are asynchronous on `st`; errors surface through cudaGetLastError.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"

namespace rs {

using rsd::u32;
using rsd::u64;
using rsd::u8;
using u16 = uint16_t;

// Launch counter (kernels issued by this library in the current build).
extern thread_local uint32_t g_launches;

// ---- scan (scan.cu): out[0..n] = exclusive prefix sums of in[0..n), out[n] = total.
size_t scan_temp_bytes(size_t n);
void exscan_u32_to_u64(const u32* in, u64* out, size_t n, void* temp, cudaStream_t st);
void exscan_u64(const u64* in, u64* out, size_t n, void* temp, cudaStream_t st);

// ---- partition (partition.cu), steps A1-A2 of SURVEY section 8(a).
// master hash code -> lo, A/B bit, bucket id; bucket histogram (zeroed); keys of buckets
// [b0, b1) only (local bucket ids; others get bkt = NONE)
// (keys == nullptr: precomputed master hash codes in mhc, 2 u64 per key)
void launch_hash(const u64* keys, const u64* mhc, u64 n, u64 g, u64 B, u64 b0, u64 b1, u64* lo, u8* ab, u32* bkt,
                 u32* hist, cudaStream_t st);
// string keys: master hash codes (R16) of data[off[i] .. off[i+1]) into mhc (2 u64 per key)
void launch_mhc_strings(const u8* data, const u64* off, u64 n, u64 g, u64* mhc, cudaStream_t st);
// exact duplicate check per bucket after the scatter (dup[0..1] zeroed); buckets above
// kSmallBucketKeys use open-addressing tables in big_scratch (kDedupeBigBlocks * 2^ceil(log2(2 smax)) u64)
constexpr u32 kDedupeBigBlocks = 64;
void launch_dedupe(const u64* lo, const u64* C, u64 nb, u32 smax, u32* dup, u64* big_scratch, cudaStream_t st);
// max/min bucket size and the histogram of bucket sizes (size_hist zeroed, cap+1 entries)
void launch_bucket_stats(const u32* hist, u64 B, u32* maxmin /*[2]*/, u32* size_hist, u32 cap,
                         cudaStream_t st);
// Two-level counting sort (one-enqueue builds): groups of 2^gl consecutive buckets of at most
// kGroupCap keys, level-1 blocks of `chunk` keys.  Level 0 counts per (group, block) into M
// (G x nb1, group-major); an exclusive scan of M gives Ms (G * nb1 + 1 entries: group g starts at
// Ms[g * nb1]); level 1 scatters the keys to the blocks' ranges; level 2 sorts each group by
// bucket in shared memory (master hash codes recomputed), writes lo_a / ab_a in bucket order, C[0..B] and small[0] / small[1]
// (max / min bucket size); small[5] |= 1 if a group overflows.
constexpr u32 kGroupCap = 12288;
constexpr u32 kGroupMax = 4096;
struct P2Shape {
    u32 gl = 0, G = 0, cap = 0, nb1 = 0;
    u64 chunk = 0;  // keys per level-1 block
};
bool partition2_shape(u64 n, u64 B, u32 S, P2Shape& sh);
void launch_p2_count(const u64* keys, u64 n, u64 first_key, u64 g, u64 B, const P2Shape& sh, u32* M, cudaStream_t st);
void launch_p2_scatter(const u64* keys, u64 n, u64 g, u64 B, const P2Shape& sh, const u64* Ms, u64* key1,
                       cudaStream_t st);
// dts > 0: the duplicate check fused into level 2 (small[2] |= 1 on a repeated key, small[3] +=
// keys with lo == 0), per-warp index tables of dts entries (a power of two >= 2 x the size bound)
void launch_p2_group(const u64* key1, u64 g, u64 B, const P2Shape& sh, const u64* Ms, u64* C, u64* lo_a, u8* ab_a,
                     u32* small, cudaStream_t st, u32 dts = 0);
// parameter counts of the kernels that read the keys (graph replays patch parameter 0, the keys)
constexpr int kHashParams = 12, kP2CountParams = 10, kP2ScatterParams = 10;
// scatter (lo, ab) to bucket order (cursor = copy of exclusive offsets)
void launch_scatter(const u64* lo, const u8* ab, const u32* bkt, u64 n, u64* cursor, u64* lo2,
                    u8* ab2, cudaStream_t st);

// ---- tree (encode.cu): node counts per bucket, node expansion into phase lists.
// per-phase node counts pcnt[q] (device) from the scanned count matrix
void launch_phase_counts(const u64* Ms, u64 B, u32 NP, u32* pcnt, cudaStream_t st);
// (S: largest size the tables cover; larger buckets are skipped and flagged in *ovf)
void launch_bucket_counts(const u64* C, u64 B, const u32* N, const u32* phase_cnt, u32 NP,
                          u64* M /*[(NP+1)*(B+1)]*/, cudaStream_t st, u32 S, u32* ovf);
void launch_expand(const u64* C, u64 B, const u64* Mscan, u32 NP, const u32* tstart,
                   const rsd::TNodeD* tnodes, const u64* phase_off /*[NP]*/, rsd::NodeRec* nodes,
                   cudaStream_t st, u32 S);

// ---- search (search.cu): the hot path, steps A4-A9.
enum SearchKind { SK_UPPER = 0, SK_LOWER = 1, SK_LEAF_RF = 2, SK_LEAF_BF = 3 };
struct PhaseLaunch {
    SearchKind kind;
    const rsd::NodeRec* nodes;
    const u32* n_nodes;  // device count
    u32 n_nodes_host;    // host copy (for launch sizing)
    const u64* lo;
    const u8* ab;
    u64* values;    // by slot; initialised to ~0
    u32* next_win;  // by slot; initialised to 0
    u32* cursor;    // two zeroed counters: batch-mode cursor, tail (help-mode) cursor
    int* active;    // n_warps entries, set to -1
    u32* err;
    const u32* dup;  // nonzero: duplicate keys, searches return immediately
    u32 leaf, u1, u2;
    u32 max_size;   // largest node size in this phase
    u32 iters;      // 32-seed iterations per window
    int help;
    int sm_count;
    int fuse_reorder = 0;   // split phases: may redistribute the keys in the search kernel (A7)
    u64* lo_w = nullptr;    // ... into these arrays (the phase's key arrays)
    u8* ab_w = nullptr;
    unsigned long long* exec = nullptr;  // RS_COUNT_EVALS builds: executed evaluations of the class
};
// returns true if the phase's key redistribution was fused into the search (no launch_reorder)
bool launch_search(const PhaseLaunch& P, cudaStream_t st);
u32 search_active_slots(int sm_count);

// Whole buckets per warp for small configurations (k_bucket_tree): every node of a bucket
// searched in preorder on the bucket's keys in shared memory.  Eligible when the leaf size is
// at most 9 and the table bound S at most kBucketTreeMax (and all classes are batch mode).
constexpr u32 kBucketTreeMax = 512;
struct TreeLaunch {
    const u64* lo;
    const u8* ab;
    const u64* C;
    u64 B;
    const u64* nodebase;
    const u32* tstart;
    const rsd::TNodeD* tn;
    u32 S;
    u32* bcursor;  // zeroed
    u64* values;
    u32* err;
    const u32* dup;
    u32 leaf, u1, u2;
    bool rf;
    int sm_count;
    unsigned long long* exec = nullptr;
    bool dedupe = false;  // each warp checks its bucket for duplicate keys (no k_dedupe pass)
};
bool bucket_tree_eligible(u32 leaf, u32 S);
void launch_bucket_tree(const TreeLaunch& L, cudaStream_t st);

// key redistribution after a split phase (A7), in place for the phase's nodes
// (big_scratch: kReorderBigWarps * 2 * max_size u64 when max_size > 8192, else unused)
constexpr u32 kReorderBigWarps = 64;
// (n_nodes_dev non-null: the phase's node count on the device; n_nodes is then an estimate
// for the grid size only)
void launch_reorder(const rsd::NodeRec* nodes, u32 n_nodes, const u64* values, u64* lo, u8* ab, u32 leaf,
                    u32 u1, u32 u2, u32 max_size, int sm_count, u64* big_scratch, cudaStream_t st,
                    const u32* n_nodes_dev = nullptr);

// ---- encode (encode.cu), steps A10-A11.
// bucket bit lengths: F(s) + N(s) + sum (x >> tau); also algorithmic-evals statistics
void launch_bucket_bits(const u64* C, u64 B, const u64* nodebase, const u32* tstart,
                        const rsd::TNodeD* tnodes, const u64* F, const u64* values, u32 leaf,
                        u32 u1, u32 u2, int rf, u64* len, unsigned long long* evals /*[4]*/,
                        cudaStream_t st, u32 S);
// Device-side globals and layout of a single-shard build (one-enqueue path).
struct SingleDev {
    u64 n, D, dC, beta;
    long long dR;
    u32 LC, LP;
    u64 lowC, upC, lowP, upP;                        // bit lengths of the EF vectors
    u64 off_lowC, off_upC, off_lowP, off_upP, off_data;  // 64-bit word offsets in the output
    u64 total_words;
    u32 overflow, pad;
};
// sd non-null: words = the output buffer, data written at sd->off_data (skipped on overflow)
void launch_write_data(const u64* C, u64 B, const u64* nodebase, const u32* tstart,
                       const rsd::TNodeD* tnodes, const u64* F, const u64* values, const u64* P,
                       unsigned long long* words, cudaStream_t st, u32 S, const SingleDev* sd);
// globals (n, D, delta_C, beta), delta_R, EF parameters, offsets and header words into sd / out
void launch_single_index(const u64* C, const u64* P, u64 B, const u32* small, SingleDev* sd, u64 hdr0, u64 hdr1, u64 g,
                         u64 cap_words, unsigned long long* out, cudaStream_t st);
// both EF sequences of all B + 1 entries into out at sd's offsets
void launch_single_ef(const u64* C, const u64* P, u64 B, const SingleDev* sd, unsigned long long* out, cudaStream_t st);
// Global view of a shard's bucket range for the index (R13): global bucket i = b0 + l,
// C_g = key_base + C_l, P_g = bit_base + P_l, R[i] = P_g[i] - floor(beta C_g[i] / 2^20).
struct IndexView {
    u64 b0;        // first global bucket of the shard
    u64 nb;        // local buckets (local arrays have nb + 1 entries)
    u64 key_base;  // keys before the shard
    u64 bit_base;  // Golomb-Rice bits before the shard
    u64 beta;      // floor(D 2^20 / n)
};
// min over local steps l in [0, nb) of R[l+1] - R[l] (atomicMin into *out)
void launch_min_residual(const u64* C, const u64* P, IndexView v, long long* out, cudaStream_t st);
// EF slices of entries l in [0, cnt): C'[i] = C_g[i] - i dC and P'[i] = R[i] - i dR; lower bits
// at global bit i*L, upper bit at (v >> L) + i; written relative to each slice's start bit.
struct EfSlices {
    u32 LC, LP;
    u64 dC;
    long long dR;
    u64 cl_start, cu_start, pl_start, pu_start;  // global start bit of each slice
    unsigned long long *cl, *cu, *pl, *pu;
};
void launch_ef_write(const u64* C, const u64* P, IndexView v, u64 cnt, EfSlices e, cudaStream_t st);

}  // namespace rs
