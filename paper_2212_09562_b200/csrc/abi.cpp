// C ABI (include/recsplit.h): argument validation, error mapping, H2D/D2H for the
// host-pointer entry points, and the host query.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/recsplit.h"
#include "pipeline.h"
#include "format.h"
#include "murmur3.h"
#include "tables.h"

namespace {

thread_local std::string g_err;
std::mutex g_build_mu;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        g_err.clear();
        return f();
    } catch (const rs::Error& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(RECSPLIT_E_NOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(RECSPLIT_E_CUDA, e.what());
    }
}

int check_args(size_t n, uint32_t leaf, uint32_t b) {
    if (n == 0) return fail(RECSPLIT_E_INVALID, "n must be >= 1");
    if (n >= (1ull << 32)) return fail(RECSPLIT_E_INVALID, "n must be < 2^32");
    if (leaf < 2 || leaf > 24) return fail(RECSPLIT_E_INVALID, "leaf_size must be in [2, 24]");
    if (b == 0) return fail(RECSPLIT_E_INVALID, "bucket_size must be >= 1");
    return RECSPLIT_OK;
}

rs::BuildParams params_of(size_t n, uint32_t leaf, uint32_t b, const recsplit_options* opt, int cuts_world = 0) {
    rs::BuildParams p;
    p.n = n;
    p.leaf = leaf;
    p.bucket = b;
    p.rf = true;
    p.g = 0;
    p.device = -1;
    p.shards = 1;
    if (opt) {
        if (opt->struct_size < offsetof(recsplit_options, reserved))
            throw rs::Error(RECSPLIT_E_INVALID, "bad options struct_size");
        p.rf = opt->rotation_fitting != 0;
        p.g = opt->global_seed;
        p.device = opt->device;
        p.shards = opt->virtual_shards ? opt->virtual_shards : 1;
        if (opt->struct_size >= offsetof(recsplit_options, total_keys) + sizeof(uint64_t)) p.n_total = opt->total_keys;
        if (opt->struct_size >= offsetof(recsplit_options, bucket_cuts) + sizeof(void*) && opt->bucket_cuts) {
            // virtual shards (build_ex) or the caller's world (shard_begin / route_keys); an
            // unsharded build ignores them
            const int w = p.shards > 1 ? (int)p.shards : cuts_world;
            if (w >= 1) p.cuts.assign(opt->bucket_cuts, opt->bucket_cuts + w + 1);
        }
    }
    return p;
}

void select_device(int dev) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw rs::Error(RECSPLIT_E_CUDA, std::string("no usable CUDA device: ") + cudaGetErrorString(e));
    if (dev >= 0) {
        if (dev >= count) throw rs::Error(RECSPLIT_E_INVALID, "device ordinal out of range");
        e = cudaSetDevice(dev);
        if (e != cudaSuccess) throw rs::Error(RECSPLIT_E_CUDA, cudaGetErrorString(e));
    }
}

int emit(rs::BuildOutput& o, recsplit_bytes* out) {
    if (o.raw) {  // hand over the malloc'ed result (no copy)
        out->data = o.raw;
        out->size = o.raw_size;
        o.raw = nullptr;
        o.raw_size = 0;
        return RECSPLIT_OK;
    }
    out->data = (uint8_t*)malloc(std::max<size_t>(o.bytes.size(), 1));
    if (!out->data) return fail(RECSPLIT_E_NOMEM, "host allocation failed");
    memcpy(out->data, o.bytes.data(), o.bytes.size());
    out->size = o.bytes.size();
    return RECSPLIT_OK;
}

#define CK_RT(x)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) throw rs::Error(RECSPLIT_E_CUDA, cudaGetErrorString(e_));           \
    } while (0)

// one non-blocking stream per device for graph replays of host-key builds (builds are
// serialized by g_build_mu)
cudaStream_t replay_stream(int dev) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> st;
    std::lock_guard<std::mutex> g(mu);
    auto it = st.find(dev);
    if (it != st.end()) return it->second;
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) throw rs::Error(RECSPLIT_E_CUDA, "stream creation failed");
    st[dev] = s;
    return s;
}

int build_host_keys(const uint64_t* keys, size_t n, uint32_t leaf, uint32_t b, const recsplit_options* opt,
                    recsplit_bytes* out, recsplit_stats* stats, rs::BuildOutput* keep, bool want_values) {
    if (!out) return fail(RECSPLIT_E_INVALID, "out is NULL");
    out->data = nullptr;
    out->size = 0;
    if (!keys) return fail(RECSPLIT_E_INVALID, "keys is NULL");
    int rc = check_args(n, leaf, b);
    if (rc) return rc;
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        auto t0 = std::chrono::steady_clock::now();
        rs::BuildParams p = params_of(n, leaf, b, opt);
        p.want_stats = stats != nullptr;
        select_device(p.device);
        int dev = 0;
        cudaGetDevice(&dev);
        // pinned host keys of an unsharded build are streamed in chunks overlapped with the
        // hash kernel; pageable ones are copied in one piece first
        // (memory pinned by another CUDA runtime in the process -- e.g. PyTorch's -- is page-locked
        // at the driver level; cudaHostGetFlags answers for it where the pointer attributes of
        // this statically linked runtime may not)
        cudaPointerAttributes pa{};
        unsigned host_flags = 0;
        const bool pinned = (cudaPointerGetAttributes(&pa, keys) == cudaSuccess && pa.type == cudaMemoryTypeHost) ||
                            cudaHostGetFlags(&host_flags, const_cast<uint64_t*>(keys)) == cudaSuccess;
        cudaGetLastError();
        const bool stream_keys = pinned && p.shards <= 1;
        if (stream_keys && !want_values && !keep) {  // a captured graph of this configuration: one launch
            cudaStream_t rst = replay_stream(dev);
            rs::BuildOutput o;
            if (rs::replay_host_keys(keys, p, rst, o)) {
                o.stats.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (stats) *stats = o.stats;
                return emit(o, out);
            }
        }
        cudaStream_t st;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_CUDA, "stream creation failed");
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        uint64_t* d_keys = nullptr;
        cudaError_t e = cudaMallocFromPoolAsync((void**)&d_keys, n * 8, rs::device_pool(dev), st);
        if (e != cudaSuccess) throw rs::Error(RECSPLIT_E_NOMEM, "device allocation of keys failed");
        struct KeyGuard {
            uint64_t* p;
            cudaStream_t s;
            ~KeyGuard() { cudaFreeAsync(p, s); }
        } kg{d_keys, st};
        cudaStream_t cs = nullptr;
        if (stream_keys && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_CUDA, "stream creation failed");
        struct CopyStreamGuard {
            cudaStream_t s;
            ~CopyStreamGuard() {
                if (s) cudaStreamDestroy(s);
            }
        } csg{cs};
        cudaEvent_t a, z;
        cudaEventCreate(&a);
        cudaEventCreate(&z);
        cudaEventRecord(a, st);
        if (stream_keys) {
            p.h_keys = keys;
            p.copy_stream = cs;
            CK_RT(cudaStreamWaitEvent(cs, a, 0));  // the key buffer's allocation is ordered on st
        } else {
            e = cudaMemcpyAsync(d_keys, keys, n * 8, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) throw rs::Error(RECSPLIT_E_CUDA, cudaGetErrorString(e));
        }
        cudaEventRecord(z, st);
        rs::BuildOutput local;
        rs::BuildOutput& o = keep ? *keep : local;
        rs::build_on_device(d_keys, p, st, want_values, o);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, z);
        cudaEventDestroy(a);
        cudaEventDestroy(z);
        if (!stream_keys) o.stats.t_h2d = ms * 1e-3;  // streamed: the copy stream's span, set by the build
        o.stats.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (stats) *stats = o.stats;
        return emit(o, out);
    });
}

// ------------------------------------------------------------- host query --

using rs::Parsed;

uint64_t word_at(const uint8_t* base, uint64_t i) {
    uint64_t x;
    memcpy(&x, base + 8 * i, 8);
    return x;
}

int parse(const uint8_t* blob, size_t size, Parsed& M) {
    std::string e;
    int rc = rs::parse_mphf(blob, size, M, &e);
    if (rc) return fail(rc, e);
    return RECSPLIT_OK;
}

inline int bit_at(const uint8_t* d, uint64_t pos) { return (int)((word_at(d, pos >> 6) >> (pos & 63)) & 1); }

uint64_t remix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline uint32_t remap(uint64_t h, uint64_t r) { return (uint32_t)(((h >> 32) * r) >> 32); }

// position just after the `cnt`-th one-bit at or after `pos` (cnt >= 1), word-wise
bool skip_ones(const uint8_t* d, uint64_t D, uint64_t& pos, uint64_t cnt) {
    while (cnt) {
        if (pos >= D) return false;
        uint64_t w = word_at(d, pos >> 6) >> (pos & 63);
        const uint64_t avail = 64 - (pos & 63);
        const uint64_t c = (uint64_t)__builtin_popcountll(w);
        if (c < cnt) {
            cnt -= c;
            pos += avail;
            continue;
        }
        // select the cnt-th one inside w
        for (uint64_t k = 1; k < cnt; ++k) w &= w - 1;
        pos += __builtin_ctzll(w) + 1;
        cnt = 0;
    }
    return true;
}


int query_mhc(const Parsed& M, uint64_t hi, uint64_t lo, uint64_t* out);

int query_one(const Parsed& M, uint64_t key, uint64_t* out) {
    return query_mhc(M, remix(key ^ M.g ^ 0x9E3779B97F4A7C15ULL), remix(key ^ M.g ^ 0xC2B2AE3D27D4EB4FULL), out);
}

int query_mhc(const Parsed& M, uint64_t hi, uint64_t lo, uint64_t* out) {
    const rs::Tables& T = *M.T;
    const uint64_t i = remap(hi, M.B);
    uint64_t s = M.C[i + 1] - M.C[i];
    uint64_t offset = M.C[i];
    if (s == 0) {
        *out = 0;
        return RECSPLIT_OK;
    }
    uint64_t fc = M.P[i], uc = M.P[i] + T.F[s];
    for (;;) {
        const uint32_t tau = T.tau[s];
        const uint64_t u0 = uc;
        if (!skip_ones(M.data, M.D, uc, 1)) return fail(RECSPLIT_E_FORMAT, "unary code out of range");
        const uint64_t q = uc - u0 - 1;
        uint64_t fixed = 0;
        for (uint32_t t = 0; t < tau; ++t) fixed |= (uint64_t)bit_at(M.data, fc + t) << t;
        fc += tau;
        const uint64_t x = (q << tau) | fixed;
        if (s <= M.leaf) {
            const uint64_t m = s;
            const uint64_t base = M.rf ? x - x % m : x;
            uint64_t v = remap(remix(lo + base), m);
            if (M.rf && (hi & 1)) v = (v + x % m) % m;  // B keys: rotation = addition mod m
            *out = offset + v;
            return RECSPLIT_OK;
        }
        uint32_t parts[64];
        const int f = rs::split_parts(T.sh, (uint32_t)s, parts);
        const uint32_t v = remap(remix(lo + x), s);
        uint32_t j = 0, accp = parts[0];
        while (v >= accp) accp += parts[++j];
        for (uint32_t c = 0; c < j; ++c) {
            fc += T.F[parts[c]];
            if (!skip_ones(M.data, M.D, uc, T.N[parts[c]])) return fail(RECSPLIT_E_FORMAT, "unary skip out of range");
            offset += parts[c];
        }
        (void)f;
        s = parts[j];
    }
}

int query_many_parsed(const Parsed& M, const uint64_t* keys, size_t n, uint64_t* out) {
    unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64));
    if (n < 100000) nt = 1;
    std::vector<int> rcs(nt, 0);
    std::vector<std::string> errs(nt);
    auto work = [&](unsigned t) {
        const size_t a = n * t / nt, b = n * (t + 1) / nt;
        for (size_t i = a; i < b; ++i) {
            int r = query_one(M, keys[i], out + i);
            if (r) {
                rcs[t] = r;
                errs[t] = g_err;
                return;
            }
        }
    };
    if (nt == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }
    for (unsigned t = 0; t < nt; ++t)
        if (rcs[t]) return fail(rcs[t], errs[t]);
    return RECSPLIT_OK;
}

}  // namespace

struct recsplit_handle {
    std::vector<uint8_t> blob;  // owned copy; M points into it
    rs::Parsed M;
    rs::DeviceMphf* dev = nullptr;
    int device = -1;
};

extern "C" {

int recsplit_version(void) { return 1; }

uint32_t recsplit_max_bucket_keys(void) { return rs::kMaxBucketKeys; }

int recsplit_trim(void) {
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        rs::trim_caches();
        return RECSPLIT_OK;
    });
}

int recsplit_build(const uint64_t* keys, size_t n, uint32_t leaf_size, uint32_t bucket_size, recsplit_bytes* out) {
    return build_host_keys(keys, n, leaf_size, bucket_size, nullptr, out, nullptr, nullptr, false);
}

int recsplit_build_ex(const uint64_t* keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                      const recsplit_options* opt, recsplit_bytes* out, recsplit_stats* stats) {
    return build_host_keys(keys, n, leaf_size, bucket_size, opt, out, stats, nullptr, false);
}

int recsplit_build_device(const uint64_t* d_keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                          const recsplit_options* opt, void* stream, recsplit_bytes* out, recsplit_stats* stats) {
    if (!out) return fail(RECSPLIT_E_INVALID, "out is NULL");
    out->data = nullptr;
    out->size = 0;
    if (!d_keys) return fail(RECSPLIT_E_INVALID, "d_keys is NULL");
    int rc = check_args(n, leaf_size, bucket_size);
    if (rc) return rc;
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        auto t0 = std::chrono::steady_clock::now();
        rs::BuildParams p = params_of(n, leaf_size, bucket_size, opt);
        p.want_stats = stats != nullptr;
        select_device(p.device);
        rs::BuildOutput o;
        rs::build_on_device(d_keys, p, (cudaStream_t)stream, false, o);
        o.stats.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (stats) *stats = o.stats;
        return emit(o, out);
    });
}

int recsplit_build_values(const uint64_t* keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                          const recsplit_options* opt, recsplit_bytes* out, uint64_t** values, size_t* n_values) {
    if (!values || !n_values) return fail(RECSPLIT_E_INVALID, "values is NULL");
    *values = nullptr;
    *n_values = 0;
    rs::BuildOutput o;
    int rc = build_host_keys(keys, n, leaf_size, bucket_size, opt, out, nullptr, &o, true);
    if (rc) return rc;
    *values = (uint64_t*)malloc(std::max<size_t>(o.values.size(), 1) * 8);
    if (!*values) {
        recsplit_free(out);
        return fail(RECSPLIT_E_NOMEM, "host allocation failed");
    }
    if (!o.values.empty()) memcpy(*values, o.values.data(), o.values.size() * 8);
    *n_values = o.values.size();
    return RECSPLIT_OK;
}

int recsplit_query(const uint8_t* mphf, size_t size, uint64_t key, uint64_t* out_index) {
    if (!out_index) return fail(RECSPLIT_E_INVALID, "out_index is NULL");
    return guarded([&]() -> int {
        Parsed M;
        int rc = parse(mphf, size, M);
        if (rc) return rc;
        if (M.strings) return fail(RECSPLIT_E_FORMAT, "MPHF was built from string keys");
        return query_one(M, key, out_index);
    });
}

int recsplit_query_many(const uint8_t* mphf, size_t size, const uint64_t* keys, size_t n, uint64_t* out) {
    if ((!keys || !out) && n) return fail(RECSPLIT_E_INVALID, "NULL keys/out");
    return guarded([&]() -> int {
        Parsed M;
        int rc = parse(mphf, size, M);
        if (rc) return rc;
        if (M.strings) return fail(RECSPLIT_E_FORMAT, "MPHF was built from string keys");
        return query_many_parsed(M, keys, n, out);
    });
}

// ------------------------------------------------------------------ handles --

int recsplit_open(const uint8_t* mphf, size_t size, int32_t device, recsplit_handle** h) {
    if (!h) return fail(RECSPLIT_E_INVALID, "h is NULL");
    *h = nullptr;
    if (!mphf && size) return fail(RECSPLIT_E_INVALID, "mphf is NULL");
    return guarded([&]() -> int {
        std::unique_ptr<recsplit_handle, void (*)(recsplit_handle*)> x(new recsplit_handle(), recsplit_close);
        x->blob.assign(mphf, mphf + size);
        int rc = parse(x->blob.data(), x->blob.size(), x->M);
        if (rc) return rc;
        if (device >= 0) {
            if (x->M.strings) return fail(RECSPLIT_E_FORMAT, "device handles of string-key MPHFs are not supported");
            select_device(device);
            cudaStream_t st;
            if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
                throw rs::Error(RECSPLIT_E_CUDA, "stream creation failed");
            struct StreamGuard {
                cudaStream_t s;
                ~StreamGuard() { cudaStreamDestroy(s); }
            } sg{st};
            x->dev = rs::upload_mphf(x->M, st);
            x->device = device;
        }
        *h = x.release();
        return RECSPLIT_OK;
    });
}

int recsplit_handle_query_many(const recsplit_handle* h, const uint64_t* keys, size_t n, uint64_t* out) {
    if (!h) return fail(RECSPLIT_E_INVALID, "h is NULL");
    if ((!keys || !out) && n) return fail(RECSPLIT_E_INVALID, "NULL keys/out");
    if (h->M.strings) return fail(RECSPLIT_E_FORMAT, "MPHF was built from string keys");
    return guarded([&]() -> int { return query_many_parsed(h->M, keys, n, out); });
}

int recsplit_handle_query_device(const recsplit_handle* h, const uint64_t* d_keys, size_t n, uint64_t* d_out,
                                 void* stream) {
    if (!h) return fail(RECSPLIT_E_INVALID, "h is NULL");
    if (!h->dev) return fail(RECSPLIT_E_INVALID, "handle has no device copy (opened with device < 0)");
    if ((!d_keys || !d_out) && n) return fail(RECSPLIT_E_INVALID, "NULL keys/out");
    return guarded([&]() -> int {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != h->device) return fail(RECSPLIT_E_INVALID, "current device differs from the handle's device");
        rs::query_resident(*h->dev, d_keys, n, d_out, (cudaStream_t)stream);
        return RECSPLIT_OK;
    });
}

int recsplit_check_bijective_device(const uint64_t* d_values, size_t n, uint64_t* bad, void* stream) {
    if (!bad || (!d_values && n)) return fail(RECSPLIT_E_INVALID, "NULL argument");
    return guarded([&]() -> int {
        select_device(-1);
        *bad = rs::count_non_bijective(d_values, n, (cudaStream_t)stream);
        return RECSPLIT_OK;
    });
}

void recsplit_close(recsplit_handle* h) {
    if (!h) return;
    rs::free_mphf(h->dev);
    delete h;
}

int recsplit_query_device(const uint8_t* mphf, size_t size, const uint64_t* d_keys, size_t n, uint64_t* d_out,
                          void* stream) {
    if ((!d_keys || !d_out) && n) return fail(RECSPLIT_E_INVALID, "NULL keys/out");
    return guarded([&]() -> int {
        Parsed M;
        int rc = parse(mphf, size, M);
        if (rc) return rc;
        if (M.strings) return fail(RECSPLIT_E_FORMAT, "device query of string-key MPHFs is not supported");
        select_device(-1);
        rs::query_on_device(M, d_keys, n, d_out, (cudaStream_t)stream);
        return RECSPLIT_OK;
    });
}

int recsplit_build_strings(const uint8_t* data, const uint64_t* offsets, size_t n, uint32_t leaf_size,
                           uint32_t bucket_size, const recsplit_options* opt, recsplit_bytes* out,
                           recsplit_stats* stats) {
    if (!out) return fail(RECSPLIT_E_INVALID, "out is NULL");
    out->data = nullptr;
    out->size = 0;
    if (!offsets || (!data && n && offsets[n])) return fail(RECSPLIT_E_INVALID, "NULL argument");
    int rc = check_args(n, leaf_size, bucket_size);
    if (rc) return rc;
    for (size_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(RECSPLIT_E_INVALID, "offsets must be non-decreasing");
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        auto t0 = std::chrono::steady_clock::now();
        rs::BuildParams p = params_of(n, leaf_size, bucket_size, opt);
        p.strings = true;
        select_device(p.device);
        cudaStream_t st;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_CUDA, "stream creation failed");
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        const uint64_t nbytes = offsets[n] - offsets[0];
        uint8_t* d_data = nullptr;
        uint64_t *d_off = nullptr, *d_mhc = nullptr;
        if (cudaMallocAsync(&d_data, std::max<uint64_t>(nbytes, 16), st) != cudaSuccess ||
            cudaMallocAsync(&d_off, (n + 1) * 8, st) != cudaSuccess ||
            cudaMallocAsync(&d_mhc, 2 * n * 8, st) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_NOMEM, "device allocation failed");
        struct Guard {
            void *a, *b, *c;
            cudaStream_t s;
            ~Guard() {
                cudaFreeAsync(a, s);
                cudaFreeAsync(b, s);
                cudaFreeAsync(c, s);
            }
        } gd{d_data, d_off, d_mhc, st};
        std::vector<uint64_t> off0(offsets, offsets + n + 1);
        for (auto& x : off0) x -= offsets[0];
        if (nbytes && cudaMemcpyAsync(d_data, data + offsets[0], nbytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_CUDA, "H2D failed");
        if (cudaMemcpyAsync(d_off, off0.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
            throw rs::Error(RECSPLIT_E_CUDA, "H2D failed");
        rs::launch_mhc_strings(d_data, d_off, n, p.g, d_mhc, st);
        if (cudaGetLastError() != cudaSuccess) throw rs::Error(RECSPLIT_E_CUDA, "string hash launch failed");
        rs::BuildOutput o;
        rs::build_on_device(d_mhc, p, st, false, o);
        o.stats.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (stats) *stats = o.stats;
        return emit(o, out);
    });
}

int recsplit_query_strings(const uint8_t* mphf, size_t size, const uint8_t* data, const uint64_t* offsets, size_t n,
                           uint64_t* out) {
    if ((!offsets || !out) && n) return fail(RECSPLIT_E_INVALID, "NULL argument");
    return guarded([&]() -> int {
        Parsed M;
        int rc = parse(mphf, size, M);
        if (rc) return rc;
        if (!M.strings) return fail(RECSPLIT_E_FORMAT, "MPHF was built from 64-bit keys");
        for (size_t i = 0; i < n; ++i) {
            const uint8_t* s = data + offsets[i];
            const uint64_t len = offsets[i + 1] - offsets[i];
            uint64_t hi, lo;
            rsm::mhc_string(s, len, M.g, hi, lo);
            rc = query_mhc(M, hi, lo, out + i);
            if (rc) return rc;
        }
        return RECSPLIT_OK;
    });
}

int recsplit_bits_per_key(const uint8_t* mphf, size_t size, double* out) {
    if (!out) return fail(RECSPLIT_E_INVALID, "out is NULL");
    return guarded([&]() -> int {
        Parsed M;
        int rc = parse(mphf, size, M);
        if (rc) return rc;
        *out = (double)(M.D + M.ec.nlow + M.ec.nup + M.ep.nlow + M.ep.nup) / (double)M.n;
        return RECSPLIT_OK;
    });
}

int recsplit_search_leaves(const uint64_t* lo, const uint8_t* isb, const uint32_t* off, uint32_t n_nodes,
                           uint32_t rotation_fitting, uint64_t* out) {
    if (!lo || !isb || !off || !out) return fail(RECSPLIT_E_INVALID, "NULL argument");
    for (uint32_t j = 0; j < n_nodes; ++j) {
        const uint32_t s = off[j + 1] - off[j];
        if (off[j + 1] < off[j] || s < 1 || s > 24) return fail(RECSPLIT_E_INVALID, "leaf sizes must be in [1, 24]");
    }
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        select_device(-1);
        rs::search_leaves_host(lo, isb, off, n_nodes, rotation_fitting != 0, out);
        return RECSPLIT_OK;
    });
}

int recsplit_search_splits(const uint64_t* lo, const uint32_t* off, uint32_t n_nodes, uint32_t leaf_size,
                           uint64_t* out) {
    if (!lo || !off || !out) return fail(RECSPLIT_E_INVALID, "NULL argument");
    if (leaf_size < 2 || leaf_size > 24) return fail(RECSPLIT_E_INVALID, "leaf_size must be in [2, 24]");
    for (uint32_t j = 0; j < n_nodes; ++j) {
        const uint32_t s = off[j + 1] - off[j];
        if (off[j + 1] < off[j] || s <= leaf_size || s > 8192)
            return fail(RECSPLIT_E_INVALID, "split sizes must be in (leaf_size, 8192]");
    }
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        select_device(-1);
        rs::search_splits_host(lo, off, n_nodes, leaf_size, out);
        return RECSPLIT_OK;
    });
}

int recsplit_tau(uint32_t leaf_size, uint32_t s, uint32_t rotation_fitting) {
    if (leaf_size < 2 || leaf_size > 24 || s > (1u << 20)) return fail(RECSPLIT_E_INVALID, "bad arguments");
    if (s == 0) return 0;
    auto T = rs::get_tables(leaf_size, rotation_fitting != 0, s);
    return (int)T->tau[s];
}

struct recsplit_shard {
    std::unique_ptr<rs::Shard> shard;
    int device = -1;
};

int recsplit_shard_begin(const uint64_t* d_keys, size_t n, uint32_t leaf_size, uint32_t bucket_size,
                         const recsplit_options* opt, int32_t rank, int32_t world, void* stream, recsplit_shard** out,
                         uint64_t summary[8]) {
    if (!out || !summary || (!d_keys && n)) return fail(RECSPLIT_E_INVALID, "NULL argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(RECSPLIT_E_INVALID, "bad rank/world");
    // routed shards (opt->total_keys > 0) may hold no key at all; the build's count is checked
    const bool routed =
        opt && opt->struct_size >= offsetof(recsplit_options, total_keys) + sizeof(uint64_t) && opt->total_keys;
    if (routed && opt->total_keys < n) return fail(RECSPLIT_E_INVALID, "total_keys < n");
    int rc = check_args(routed ? opt->total_keys : n, leaf_size, bucket_size);
    if (rc) return rc;
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        rs::BuildParams p = params_of(n, leaf_size, bucket_size, opt, world);
        select_device(p.device);
        auto* h = new recsplit_shard;
        try {
            h->shard.reset(new rs::Shard(d_keys, p, rank, world, (cudaStream_t)stream, false));
        } catch (...) {
            delete h;
            throw;
        }
        cudaGetDevice(&h->device);
        memcpy(summary, h->shard->summary, 64);
        *out = h;
        return RECSPLIT_OK;
    });
}

int recsplit_route_keys(const uint64_t* d_keys, size_t n, uint64_t total_keys, uint32_t bucket_size,
                        const recsplit_options* opt, int32_t world, void* stream, uint64_t* d_out, uint64_t* counts) {
    if (!counts || ((!d_keys || !d_out) && n)) return fail(RECSPLIT_E_INVALID, "NULL argument");
    if (world < 1) return fail(RECSPLIT_E_INVALID, "world must be >= 1");
    if (bucket_size == 0) return fail(RECSPLIT_E_INVALID, "bucket_size must be >= 1");
    if (total_keys < n || total_keys == 0 || total_keys >= (1ull << 32))
        return fail(RECSPLIT_E_INVALID, "total_keys must be in [max(n, 1), 2^32)");
    return guarded([&]() -> int {
        rs::BuildParams p = params_of(total_keys, 2, bucket_size, opt, world);
        select_device(p.device);
        rs::route_keys(d_keys, n, total_keys, bucket_size, p.g, (uint32_t)world, p.cuts.empty() ? nullptr : p.cuts.data(),
                       (cudaStream_t)stream, d_out, counts);
        return RECSPLIT_OK;
    });
}

int recsplit_bucket_histogram(const uint64_t* d_keys, size_t n, uint64_t total_keys, uint32_t bucket_size,
                              const recsplit_options* opt, void* stream, uint32_t* d_hist) {
    if (!d_hist || (!d_keys && n)) return fail(RECSPLIT_E_INVALID, "NULL argument");
    if (bucket_size == 0) return fail(RECSPLIT_E_INVALID, "bucket_size must be >= 1");
    if (total_keys < n || total_keys == 0 || total_keys >= (1ull << 32))
        return fail(RECSPLIT_E_INVALID, "total_keys must be in [max(n, 1), 2^32)");
    return guarded([&]() -> int {
        rs::BuildParams p = params_of(total_keys, 2, bucket_size, opt, 1);
        select_device(p.device);
        rs::bucket_histogram(d_keys, n, total_keys, bucket_size, p.g, (cudaStream_t)stream, d_hist);
        return RECSPLIT_OK;
    });
}

int recsplit_balanced_cuts(const uint32_t* hist, uint64_t B, uint32_t leaf_size, uint32_t rotation_fitting,
                           int32_t world, uint64_t* cuts) {
    if (!cuts || (!hist && B)) return fail(RECSPLIT_E_INVALID, "NULL argument");
    if (world < 1) return fail(RECSPLIT_E_INVALID, "world must be >= 1");
    if (leaf_size < 2 || leaf_size > 24) return fail(RECSPLIT_E_INVALID, "leaf_size must be in [2, 24]");
    return guarded([&]() -> int {
        const std::vector<uint64_t> c = rs::balanced_cuts(hist, B, leaf_size, rotation_fitting != 0, world);
        memcpy(cuts, c.data(), 8 * c.size());
        return RECSPLIT_OK;
    });
}

int recsplit_shard_min_step(recsplit_shard* sh, const uint64_t* summaries, int64_t* min_step) {
    if (!sh || !summaries || !min_step) return fail(RECSPLIT_E_INVALID, "NULL argument");
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        cudaSetDevice(sh->device);
        *min_step = sh->shard->min_step(summaries);
        return RECSPLIT_OK;
    });
}

int recsplit_shard_finish(recsplit_shard* sh, int64_t min_step, recsplit_bytes* part) {
    if (!sh || !part) return fail(RECSPLIT_E_INVALID, "NULL argument");
    part->data = nullptr;
    part->size = 0;
    return guarded([&]() -> int {
        std::lock_guard<std::mutex> g(g_build_mu);
        cudaSetDevice(sh->device);
        rs::BuildOutput o;
        sh->shard->finish(min_step == INT64_MAX ? 0 : min_step, o.bytes);
        return emit(o, part);
    });
}

int recsplit_stitch(const uint8_t* const* parts, const size_t* sizes, int32_t count, recsplit_bytes* out) {
    if (!parts || !sizes || !out || count < 1) return fail(RECSPLIT_E_INVALID, "bad arguments");
    out->data = nullptr;
    out->size = 0;
    return guarded([&]() -> int {
        std::vector<std::pair<const uint8_t*, size_t>> v;
        for (int i = 0; i < count; ++i) v.emplace_back(parts[i], sizes[i]);
        rs::BuildOutput o;
        rs::stitch(v, o.bytes);
        return emit(o, out);
    });
}

void recsplit_shard_free(recsplit_shard* sh) {
    if (!sh) return;
    cudaSetDevice(sh->device);
    delete sh;
}

int recsplit_shard_globals(const uint64_t* summaries, int32_t world, int32_t rank, uint64_t out[6]) {
    if (!summaries || !out || world < 1 || rank < 0 || rank >= world) return fail(RECSPLIT_E_INVALID, "bad arguments");
    rs::Globals G = rs::compute_globals(summaries, world, rank);
    const uint64_t v[6] = {G.n, G.D, G.dC, G.beta, G.key_base, G.bit_base};
    memcpy(out, v, sizeof v);
    return RECSPLIT_OK;
}

void recsplit_free(recsplit_bytes* b) {
    if (!b) return;
    if (!rs::pinned_release(b->data)) free(b->data);
    b->data = nullptr;
    b->size = 0;
}

void recsplit_free_ptr(void* p) { free(p); }

const char* recsplit_last_error(void) { return g_err.c_str(); }

}  // extern "C"
