/*
 * recsplit.h -- C ABI of the B200-native RecSplit MPHF builder
 * (arXiv 2212.09562: RecSplit with rotation fitting; GPU construction).
 *
 * Citation keys: P:n = line n of the paper text.
 * lists every reading (R1..R14) taken where the paper is silent.
 *
 * Problem statement: a minimal perfect hash function maps a set S of
 * n keys bijectively onto [0, n); evaluating it on a key outside S returns an
 * arbitrary value in [0, n).  Construction: keys -> buckets of expected
 * size b -> per bucket a splitting tree whose inner nodes store the smallest seed
 * that splits the keys into the fanout-prescribed part sizes and whose
 * leaves store the smallest (seed, rotation) value found by rotation fitting
 * (minimal-value rule P:297-300) -- or the smallest brute-force seed
 * when rotation fitting is off.  Values are Golomb-Rice coded per tree
 * in preorder with a trend-subtracted Elias-Fano bucket index.
 *
 * Every search step runs in hand-written sm_100a CUDA kernels; there is NO CPU
 * fallback: without a usable CUDA device the build calls return RECSPLIT_E_CUDA.
 *
 * Conventions
 *  - All functions return RECSPLIT_OK (0) or a negative error code; on error
 *    recsplit_last_error() returns a thread-local message describing the failure.
 *  - Output buffers (recsplit_bytes) are allocated by the library (malloc, or pinned
 *    host memory from a small reuse pool for single-GPU build results, so the result is
 *    copied from the device only once) and owned by the caller, who releases them with
 *    recsplit_free() -- never free().  On any error *out = {NULL, 0} and nothing leaks.
 *  - Input pointers are borrowed for the duration of the call and never retained.
 *  - The output bytes are a pure function of (key set, leaf_size, bucket_size,
 *    rotation_fitting, global_seed): independent of key order, device, shard
 *    count and kernel schedule.
 *  - Builds are serialised per process (an internal mutex); queries are reentrant.
 */
#ifndef RECSPLIT_H
#define RECSPLIT_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RECSPLIT_API __attribute__((visibility("default")))
#else
#define RECSPLIT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RECSPLIT_OK = 0,
    RECSPLIT_E_INVALID = -1,   /* bad argument: n == 0, n >= 2^32, leaf_size outside [2,24],
                                  bucket_size == 0, a bucket larger than the supported
                                  maximum (recsplit_max_bucket_keys()), NULL pointer */
    RECSPLIT_E_DUPLICATE = -2, /* two equal keys (detected before any search) */
    RECSPLIT_E_NOMEM = -3,     /* host or device allocation failed */
    RECSPLIT_E_CUDA = -4,      /* no usable CUDA device / kernel launch or runtime error */
    RECSPLIT_E_FORMAT = -5,    /* corrupt, truncated or unsupported serialized MPHF */
    RECSPLIT_E_SEED_CAP = -6   /* a node needed more than 2^40 trials (diagnostic) */
};

/* A library-allocated byte buffer; free with recsplit_free(). */
typedef struct {
    uint8_t *data;
    size_t size;
} recsplit_bytes;

/* Options (NULL = defaults: rotation fitting on, global_seed 0, current device). */
typedef struct {
    uint32_t struct_size;      /* sizeof(recsplit_options) */
    uint32_t rotation_fitting; /* 1: leaves by rotation fitting; 0: brute force */
    uint64_t global_seed;      /* g of the master hash code (reading R2) */
    int32_t device;            /* CUDA device ordinal; -1 = current device */
    uint32_t virtual_shards;   /* >1: run the bucket-range sharded path with this many
                                  shards on one device and stitch them (tests the multi-GPU
                                  offset logic); 0/1 = unsharded */
    uint32_t reserved;         /* 0 */
    uint64_t total_keys;       /* recsplit_shard_begin only: keys of the WHOLE sharded build when
                                  each rank passes just the keys it owns (routed with
                                  recsplit_route_keys); 0 = n (every rank passes all keys) */
    const uint64_t *bucket_cuts; /* HOST, world + 1 global bucket indices or NULL: rank r owns
                                  buckets [cuts[r], cuts[r+1]) (cuts[0] = 0, cuts[world] = B,
                                  nondecreasing; e.g. from recsplit_balanced_cuts).  Used by
                                  recsplit_shard_begin, recsplit_route_keys and virtual_shards.
                                  NULL = equal bucket counts [floor(rB/W), floor((r+1)B/W)).
                                  The output bytes do not depend on the cuts. */
} recsplit_options;

/* Per-build statistics (optional output). Times are device (CUDA event) seconds. */
typedef struct {
    double t_total;        /* whole recsplit_build* call, host wall clock */
    double t_h2d;          /* host->device key copy (0 for the device-input entry point) */
    double t_partition;    /* hash + bucket counting sort + per-bucket sort/dedupe */
    double t_tree;         /* node-table expansion */
    double t_search[4];    /* upper splits, lower level 2, lower level 1, leaves */
    double t_reorder;      /* key redistribution after splits */
    double t_encode;       /* Golomb-Rice + Elias-Fano + serialization */
    double t_d2h;          /* device->host result copy */
    uint64_t algo_evals[4];  /* algorithmic remix evaluations per class [upper,L2,L1,leaf]:
                                sum over nodes of (trials up to and incl. the minimal one) x keys */
    uint64_t nodes[4];       /* node counts per class */
    uint64_t data_bits;      /* Golomb-Rice bits D */
    uint64_t index_bits;     /* Elias-Fano lower+upper bits of both sequences */
    uint32_t kernel_launches; /* CUDA kernels this library launched during the build */
    uint32_t max_bucket;      /* largest bucket size */
    uint64_t exec_evals[4];   /* diagnostic builds (-DRS_COUNT_EVALS) only, else 0: key evaluations
                                 the search kernels EXECUTED per class (32 lanes per group step,
                                 incl. discarded lanes; early rejection skips the rest) */
    double t_search_tree;     /* small configurations: the whole-bucket search kernel (all classes
                                 in one launch; t_search is then 0 and exec_evals[0] holds the
                                 executed total), else 0 */
    double t_device;          /* single-GPU builds: device span from the first enqueued operation to
                                 the end of the result D2H (CUDA events), else 0 */
    uint32_t graph_replay;    /* 1 if the build replayed a captured CUDA graph of its configuration */
    uint32_t reserved0;
} recsplit_stats;

/* Library version (format version is the header's u16 version = 1). */
RECSPLIT_API int recsplit_version(void);

/* Largest bucket (keys) a build accepts: 65536.  Any bucket_size >= 1 is a valid argument
 * (SURVEY 8(b)); the limit applies to the ACTUAL bucket sizes, which are Poisson(n/B) around
 * bucket_size (so bucket_size up to about 60000 is safe).  It is not a search limit (nodes
 * above the 8192-key shared-memory capacity run through a global-memory path): it bounds
 * the per-size preorder templates (about 1.4 s / leaf_size nodes of 24 B for each distinct
 * bucket size s) the node table is expanded from.  A larger bucket -> RECSPLIT_E_INVALID. */
RECSPLIT_API uint32_t recsplit_max_bucket_keys(void);

/*
 * Release what the library keeps between builds: the captured build graphs and their
 * device workspaces, the unused part of its device memory pool and its idle pinned host
 * buffers.  Results already returned stay valid (free them with recsplit_free).  Returns
 * RECSPLIT_OK, or RECSPLIT_E_CUDA if a CUDA call failed.  Not to be called concurrently
 * with a build.
 */
RECSPLIT_API int recsplit_trim(void);

/*
 * Build the MPHF of the n distinct 64-bit keys at `keys` (HOST memory, pageable or
 * pinned) with leaf size l = leaf_size (P:110, 2..24) and expected bucket size
 * b = bucket_size.  Rotation fitting on, global seed 0.  On success *out
 * receives the serialized MPHF (format: DESIGN.md section 6).
 */
RECSPLIT_API int recsplit_build(const uint64_t *keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                   recsplit_bytes *out);

/* As recsplit_build with options (nullable) and statistics (nullable). */
RECSPLIT_API int recsplit_build_ex(const uint64_t *keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                      const recsplit_options *opt, recsplit_bytes *out, recsplit_stats *stats);

/*
 * As recsplit_build_ex, but `d_keys` is a DEVICE pointer (n x u64, on opt->device)
 * and all work is ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 * The call returns after the serialized bytes are in host memory.
 *
 * Caching (single-GPU builds of up to 2^27 keys, both entries): the second build of a
 * configuration (n, leaf_size, bucket_size, options, host or device keys, stats or not)
 * captures the whole device pipeline as a CUDA graph over a workspace it keeps (about 22 B
 * per key plus the node tables); later builds of that configuration replay it.  At most 4
 * such configurations are kept per process (least recently captured dropped first);
 * recsplit_trim() releases them.
 */
RECSPLIT_API int recsplit_build_device(const uint64_t *d_keys, size_t n, uint32_t leaf_size,
                          uint32_t bucket_size, const recsplit_options *opt, void *stream,
                          recsplit_bytes *out, recsplit_stats *stats);

/*
 * Diagnostic build: additionally returns every stored node value (u64) in bucket
 * order, each bucket's tree in preorder, as a malloc'ed array in *values
 * (*n_values entries); free with recsplit_free_ptr().
 */
RECSPLIT_API int recsplit_build_values(const uint64_t *keys, size_t n, uint32_t leaf_size,
                          uint32_t bucket_size, const recsplit_options *opt, recsplit_bytes *out,
                          uint64_t **values, size_t *n_values);

/*
 * String keys (the paper's competitor workload P:386-388).  Key i is the
 * byte string data[offsets[i] .. offsets[i+1]) (HOST arrays; offsets has n+1 non-decreasing
 * entries).  Its master hash code is reading R16; everything after step A1 is
 * the same pipeline.  The header records the key type (flags bit 1).  Equal strings ->
 * RECSPLIT_E_DUPLICATE.
 */
RECSPLIT_API int recsplit_build_strings(const uint8_t *data, const uint64_t *offsets, size_t n,
                                        uint32_t leaf_size, uint32_t bucket_size,
                                        const recsplit_options *opt, recsplit_bytes *out,
                                        recsplit_stats *stats);
/* Host evaluation of a string-key MPHF on n strings (same layout as recsplit_build_strings). */
RECSPLIT_API int recsplit_query_strings(const uint8_t *mphf, size_t size, const uint8_t *data,
                                        const uint64_t *offsets, size_t n, uint64_t *out);

/* Evaluate the MPHF serialized at mphf[0..size) on one key (host).  For a key of
 * the build set the result is its unique index in [0, n); otherwise some value in
 * [0, n).  Corrupt blobs -> RECSPLIT_E_FORMAT. */
RECSPLIT_API int recsplit_query(const uint8_t *mphf, size_t size, uint64_t key, uint64_t *out_index);

/* Evaluate on n keys (host, multi-threaded); out has n entries. */
RECSPLIT_API int recsplit_query_many(const uint8_t *mphf, size_t size, const uint64_t *keys, size_t n,
                        uint64_t *out);

/* Evaluate on n keys on the GPU: mphf is HOST memory (parsed and uploaded
 * per call), d_keys / d_out are DEVICE arrays of n u64 on the current device; ordered on
 * `stream`, returns after completion.  Same results as recsplit_query_many. */
RECSPLIT_API int recsplit_query_device(const uint8_t *mphf, size_t size, const uint64_t *d_keys,
                                       size_t n, uint64_t *d_out, void *stream);

/* Opened MPHF (SURVEY 8(b) recsplit_open): the blob is copied and parsed once (its
 * Elias-Fano index decoded), so repeated queries skip the per-call parse.  device >= 0
 * also places a resident copy in that GPU's HBM (decoded index + data words + per-size
 * tables, about 16 B per bucket + the blob's data) for recsplit_handle_query_device;
 * device < 0 makes a host-only handle (no GPU needed).  Errors: RECSPLIT_E_FORMAT for a
 * corrupt blob (or a device handle of a string-key MPHF), RECSPLIT_E_CUDA / _NOMEM for
 * device failures; *h is NULL on any error.  Close with recsplit_close (NULL-safe). */
typedef struct recsplit_handle recsplit_handle;
RECSPLIT_API int recsplit_open(const uint8_t *mphf, size_t size, int32_t device, recsplit_handle **h);
/* Host evaluation on n u64 keys (multi-threaded for large n); reentrant. */
RECSPLIT_API int recsplit_handle_query_many(const recsplit_handle *h, const uint64_t *keys, size_t n,
                                            uint64_t *out);
/* GPU evaluation on n keys with the resident copy: d_keys / d_out are DEVICE arrays of n
 * u64 on the handle's device (which must be current).  ENQUEUED on `stream` only -- the
 * call does not synchronise; d_out is valid once the stream reaches this point. */
RECSPLIT_API int recsplit_handle_query_device(const recsplit_handle *h, const uint64_t *d_keys, size_t n,
                                              uint64_t *d_out, void *stream);
RECSPLIT_API void recsplit_close(recsplit_handle *h);

/* Bijectivity check on the GPU (the property P:11 defines): d_values is a
 * DEVICE array of n u64 on the current device (e.g. the query results of the n build
 * keys); *bad receives the number of entries outside [0, n) plus the number of repeats,
 * so *bad == 0 iff d_values is a permutation of [0, n).  Uses an n-bit device bitmap;
 * ordered on `stream`, returns after completion. */
RECSPLIT_API int recsplit_check_bijective_device(const uint64_t *d_values, size_t n, uint64_t *bad,
                                                 void *stream);

/* bits/object of a serialized MPHF: (Golomb-Rice bits + Elias-Fano bits) / n,
 * excluding the fixed header and word padding (reading R14). */
RECSPLIT_API int recsplit_bits_per_key(const uint8_t *mphf, size_t size, double *out);

/*
 * Kernel-level entry points (parity tests; host pointers, copied internally).
 * Leaves: node j has keys lo[off[j] .. off[j+1]) (1 <= size <= 24) with A/B bits
 * isb[] (reading R7); out[j] = stored value (k*m + r, rotation_fitting=1;
 * brute-force seed otherwise).  Splits: node j has keys lo[off[j]..off[j+1]), size
 * s > leaf_size; out[j] = smallest seed giving the prescribed parts.
 */
RECSPLIT_API int recsplit_search_leaves(const uint64_t *lo, const uint8_t *isb, const uint32_t *off,
                           uint32_t n_nodes, uint32_t rotation_fitting, uint64_t *out);
RECSPLIT_API int recsplit_search_splits(const uint64_t *lo, const uint32_t *off, uint32_t n_nodes,
                           uint32_t leaf_size, uint64_t *out);

/* Library tables (parity tests): Golomb-Rice parameter tau of a node of size s
 * (leaf if s <= leaf_size), computed by the library's own host code. */
RECSPLIT_API int recsplit_tau(uint32_t leaf_size, uint32_t s, uint32_t rotation_fitting);

/*
 * Sharded construction (buckets are independent; contiguous bucket ranges per
 * worker; per-worker sequences concatenated and one Elias-Fano index over all buckets).
 * Rank r of `world` owns buckets [floor(r B / W), floor((r+1) B / W)), B = ceil(n / b), or
 * [cuts[r], cuts[r+1]) with opt->bucket_cuts.
 * Every rank passes ALL n keys (DEVICE pointer, on its own device); the output bytes are
 * identical to recsplit_build's for any world size.  Protocol (collectives are the
 * caller's, e.g. torch.distributed over NCCL):
 *   1. recsplit_shard_begin            -> 8-word summary of this rank
 *   2. allgather the summaries (world x 8 u64, rank order)
 *   3. recsplit_shard_min_step(all)    -> this rank's minimum residual step (int64)
 *   4. allreduce-min of the steps
 *   5. recsplit_shard_finish(min)      -> this rank's part (bytes)
 *   6. gather the parts; recsplit_stitch(parts of ranks 0..W-1) -> serialized MPHF
 * A duplicate key or a seed-cap error on any rank makes step 3 fail on every rank.
 * The handle owns device memory until recsplit_shard_free.
 */
typedef struct recsplit_shard recsplit_shard;
RECSPLIT_API int recsplit_shard_begin(const uint64_t *d_keys, size_t n, uint32_t leaf_size,
                                      uint32_t bucket_size, const recsplit_options *opt, int32_t rank,
                                      int32_t world, void *stream, recsplit_shard **out,
                                      uint64_t summary[8]);
RECSPLIT_API int recsplit_shard_min_step(recsplit_shard *sh, const uint64_t *summaries,
                                         int64_t *min_step);
RECSPLIT_API int recsplit_shard_finish(recsplit_shard *sh, int64_t min_step, recsplit_bytes *part);
RECSPLIT_API int recsplit_stitch(const uint8_t *const *parts, const size_t *sizes, int32_t count,
                                 recsplit_bytes *out);
RECSPLIT_API void recsplit_shard_free(recsplit_shard *sh); /* NULL-safe */

/* Key routing for sharded builds: rank r of `world` owns the buckets
 * [floor(rB/world), floor((r+1)B/world)) (or [cuts[r], cuts[r+1]) with opt->bucket_cuts),
 * B = ceil(total_keys / bucket_size) (R12), bucket =
 * remap(hi, B) of the master hash code (R2, R3, global_seed from opt).  Groups the n DEVICE
 * keys d_keys (this rank's slice of the input) by owner: d_out (DEVICE, n u64) receives the
 * keys for rank 0, then rank 1, ...; counts (HOST, world u64) the number per rank.  After an
 * all-to-all exchange every rank holds exactly its keys and calls recsplit_shard_begin with
 * opt->total_keys = total_keys.  Synchronises `stream`; the order inside a group is arbitrary
 * (the output bytes do not depend on key order). */
RECSPLIT_API int recsplit_route_keys(const uint64_t *d_keys, size_t n, uint64_t total_keys,
                                     uint32_t bucket_size, const recsplit_options *opt, int32_t world,
                                     void *stream, uint64_t *d_out, uint64_t *counts);
/* Work-balanced bucket ranges: d_hist (DEVICE, B = ceil(total_keys / bucket_size)
 * u32, zeroed by the caller) += the number of this rank's n DEVICE keys in each global bucket
 * (R2, R3; global_seed from opt).  Sum the ranks' histograms (an allreduce), then
 * recsplit_balanced_cuts.  Enqueued on `stream` (no synchronisation). */
RECSPLIT_API int recsplit_bucket_histogram(const uint64_t *d_keys, size_t n, uint64_t total_keys,
                                           uint32_t bucket_size, const recsplit_options *opt, void *stream,
                                           uint32_t *d_hist);
/* cuts (HOST, world + 1) of contiguous bucket ranges with about equal expected remix
 * evaluations (sum over each bucket's tree of size / success probability per node, from the
 * bucket sizes hist[0..B) (HOST)); deterministic, so every rank computes the same cuts. */
RECSPLIT_API int recsplit_balanced_cuts(const uint32_t *hist, uint64_t B, uint32_t leaf_size,
                                        uint32_t rotation_fitting, int32_t world, uint64_t *cuts);
/* Host arithmetic of step 3 (tests): out = {n, D, delta_C, beta, key_base, bit_base}. */
RECSPLIT_API int recsplit_shard_globals(const uint64_t *summaries, int32_t world, int32_t rank,
                                        uint64_t out[6]);

RECSPLIT_API void recsplit_free(recsplit_bytes *b); /* NULL-safe; zeroes *b */
RECSPLIT_API void recsplit_free_ptr(void *p);
RECSPLIT_API const char *recsplit_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RECSPLIT_H */
