// Host orchestration of the device construction pipeline.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/recsplit.h"

namespace rs {

// Largest bucket a build accepts (the per-size preorder templates grow with the bucket size,
// see include/recsplit.h recsplit_max_bucket_keys); buckets above 8192 keys run their upper
// splits through k_search_upper_big / k_reorder_big and the dedupe through global tables.
constexpr uint32_t kMaxBucketKeys = 1u << 16;
constexpr uint32_t kSmallBucketKeys = 8192;  // size-histogram and shared-memory dedupe capacity

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct BuildParams {
    uint64_t n;
    uint32_t leaf, bucket;
    bool rf;
    uint64_t g;
    int device;
    uint32_t shards;  // virtual shards (>= 1)
    bool strings = false;  // keys are precomputed master hash codes of strings (2 u64 each, R16)
    uint64_t n_total = 0;  // keys of the whole build (0 = n): routed shards hold only their own keys
    std::vector<uint64_t> cuts;  // world + 1 bucket cuts (empty = equal bucket counts)
    // host keys streamed in chunks (pinned memory, single shard): d_keys is the destination
    // buffer; chunk c is copied on copy_stream while the hash kernel runs on chunk c - 1
    const uint64_t* h_keys = nullptr;
    cudaStream_t copy_stream = nullptr;
    // per-phase CUDA-event timings in the stats (the caller asked for stats); without them the
    // one-enqueue build records no timing events and queries none after the synchronization
    bool want_stats = true;
};

// the library's stream-ordered memory pool on device dev (kept reserved between builds)
cudaMemPool_t device_pool(int dev);
// drop the captured build graphs (and workspaces), trim the pools, free idle pinned buffers
void trim_caches();

// Pinned host result buffers (single-GPU builds D2H straight into the caller's result):
// pinned_get returns a buffer of >= bytes (reused when possible), pinned_release takes back
// one of them and returns false for any other pointer.
uint8_t* pinned_get(size_t bytes);
bool pinned_release(void* p);

// the bucket range [b0, b1) of `rank` (cuts, else equal counts); validates the cuts
void shard_range(const BuildParams& p, uint64_t B, int rank, int world, uint64_t& b0, uint64_t& b1);

struct BuildOutput {
    std::vector<uint8_t> bytes;
    // single-shard builds: the serialized MPHF in a malloc'ed buffer (handed to the caller
    // without another copy); bytes stays empty then
    uint8_t* raw = nullptr;
    size_t raw_size = 0;
    BuildOutput() = default;
    BuildOutput(const BuildOutput&) = delete;
    BuildOutput& operator=(const BuildOutput&) = delete;
    ~BuildOutput() {
        if (!pinned_release(raw)) free(raw);
    }
    const uint8_t* data() const { return raw ? raw : bytes.data(); }
    size_t size() const { return raw ? raw_size : bytes.size(); }
    std::vector<uint64_t> values;  // only when requested
    recsplit_stats stats{};
};

// ---- shards (multi-GPU / virtual shards), DESIGN.md section 13
enum { SUM_KEYS = 0, SUM_BITS = 1, SUM_MINB = 2, SUM_B0 = 3, SUM_B1 = 4, SUM_DUP = 5, SUM_ERR = 6, SUM_NTOT = 7 };

struct Globals {
    uint64_t n = 0, D = 0, dC = 0, beta = 0, key_base = 0, bit_base = 0, UC = 0, UP = 0;
    long long dR = 0;
    uint32_t LC = 0, LP = 0;
    int dup = 0, err = 0;
};
// global sizes and this rank's bases from all ranks' 8-word summaries
Globals compute_globals(const uint64_t* all, int world, int rank);
// EF parameters once delta_R is known
void finalize_globals(Globals& G, uint64_t B, long long dR);

class Shard {
   public:
    // phase 1: hash all keys, keep buckets [floor(rB/W), floor((r+1)B/W)), search, lengths
    Shard(const uint64_t* d_keys, const BuildParams& p, int rank, int world, cudaStream_t st, bool want_values);
    ~Shard();
    uint64_t summary[8];  // SUM_* fields
    // phase 2: global bases from all summaries; returns this shard's min residual step
    long long min_step(const uint64_t* all_summaries);
    // phase 3: EF and data slices at their global bit positions -> serialized part
    void finish(long long dR, std::vector<uint8_t>& part);
    // phase 3 for a single shard (world 1): the serialized MPHF directly (malloc'ed)
    void finish_blob(long long dR, uint8_t*& blob, size_t& size);
    const Globals& globals() const;
    struct Impl;
    std::vector<uint64_t> values;  // node values of the shard (want_values)
    recsplit_stats stats{};

   private:
    Impl* impl_;
};

// OR all parts' slices into the serialized MPHF
void stitch(const std::vector<std::pair<const uint8_t*, size_t>>& parts, std::vector<uint8_t>& blob);

// SURVEY 8(e)(ii) key routing: group n device keys by the rank owning their bucket in a
// build of `total` keys over `world` ranks (B = ceil(total / bucket)); d_out gets the keys
// rank by rank, counts[r] (host) the number for rank r.  Synchronises st.
void route_keys(const uint64_t* d_keys, uint64_t n, uint64_t total, uint32_t bucket, uint64_t g, uint32_t world,
                const uint64_t* cuts /*host, world + 1, or null*/, cudaStream_t st, uint64_t* d_out, uint64_t* counts);
// d_hist[i] += keys of global bucket i (B = ceil(total / bucket) entries), enqueued on st
void bucket_histogram(const uint64_t* d_keys, uint64_t n, uint64_t total, uint32_t bucket, uint64_t g,
                      cudaStream_t st, uint32_t* d_hist);

// string keys (R16): master hash codes of data[off[i] .. off[i+1]) into mhc (2 u64 per key)
void launch_mhc_strings(const uint8_t* data, const uint64_t* off, uint64_t n, uint64_t g, uint64_t* mhc,
                        cudaStream_t st);

// d_keys: device pointer (n keys; params.strings: 2n master-hash words) on params.device;
// work ordered on st.
void build_on_device(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, bool want_values,
                     BuildOutput& out);
// Host (pinned) keys through a captured CUDA graph of the configuration that holds its own
// device key buffer (no allocation, no copy stream of the caller's); false if no graph of
// this configuration exists yet (the caller then takes the general path, which captures one).
bool replay_host_keys(const uint64_t* h_keys, const BuildParams& p, cudaStream_t st, BuildOutput& out);

// Batched query on the device; d_keys / d_out device arrays of n.
struct Parsed;
void query_on_device(const Parsed& M, const uint64_t* d_keys, uint64_t n, uint64_t* d_out, cudaStream_t st);
// resident copy on the current device (recsplit_open): upload once, query many times
struct DeviceMphf;
DeviceMphf* upload_mphf(const Parsed& M, cudaStream_t st);
void free_mphf(DeviceMphf* h);  // NULL-safe
// number of values outside [0, n) or repeated (0 <=> d_vals is a permutation of [0, n))
uint64_t count_non_bijective(const uint64_t* d_vals, uint64_t n, cudaStream_t st);
// enqueue only (no synchronisation)
void query_resident(const DeviceMphf& h, const uint64_t* d_keys, uint64_t n, uint64_t* d_out, cudaStream_t st);

// Kernel-level entry points for parity tests (host arrays).
void search_leaves_host(const uint64_t* lo, const uint8_t* isb, const uint32_t* off, uint32_t n_nodes, bool rf,
                        uint64_t* out);
void search_splits_host(const uint64_t* lo, const uint32_t* off, uint32_t n_nodes, uint32_t leaf, uint64_t* out);

}  // namespace rs
