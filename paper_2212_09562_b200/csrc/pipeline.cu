// Host orchestration of the B200 construction pipeline (SURVEY 3 "planned
// recsplit_build"): H2D -> hash/partition -> node table -> per-phase search +
// reorder -> encode -> D2H.  Every step runs in this library's kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "kernels.h"
#include "pipeline.h"
#include "tables.h"

namespace rs {

thread_local uint32_t g_launches = 0;

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw Error(e_ == cudaErrorMemoryAllocation ? RECSPLIT_E_NOMEM : RECSPLIT_E_CUDA,      \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                          \
    } while (0)
#define CKL() CK(cudaGetLastError())

namespace {

// The library's private stream-ordered memory pool per device (not the device's default
// pool, which the rest of the process -- e.g. PyTorch -- may use).  It keeps up to
// kPoolKeepBytes reserved between builds so repeated builds do not re-map memory; above
// that, the driver returns the excess to the OS at the next synchronization.
constexpr uint64_t kPoolKeepBytes = 8ull << 30;

std::mutex& pools_mu() {
    static std::mutex mu;
    return mu;
}
std::map<int, cudaMemPool_t>& pools_map() {
    static std::map<int, cudaMemPool_t>& pools = *new std::map<int, cudaMemPool_t>;
    return pools;
}

cudaMemPool_t device_pool_impl(int dev) {
    std::mutex& mu = pools_mu();
    std::map<int, cudaMemPool_t>& pools = pools_map();
    std::lock_guard<std::mutex> g(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    CK(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = kPoolKeepBytes;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    pools[dev] = pool;
    return pool;
}

// Stream-ordered device allocations from the library pool, released at scope exit (or
// earlier with release()).
struct Arena {
    cudaStream_t st;
    cudaMemPool_t pool;
    std::vector<void*> ptrs;
    explicit Arena(cudaStream_t s) : st(s) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        pool = device_pool_impl(dev);
    }
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        CK(cudaMallocFromPoolAsync(&p, bytes, pool, st));
        ptrs.push_back(p);
        return (T*)p;
    }
    void release(void* p) {  // stream-ordered free of one allocation before scope exit
        auto it = std::find(ptrs.begin(), ptrs.end(), p);
        if (it == ptrs.end()) return;
        cudaFreeAsync(p, st);
        ptrs.erase(it);
    }
    ~Arena() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

void init_device(int dev) { (void)device_pool_impl(dev); }

int sm_count(int dev) {
    int v = 0;
    CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
}

// CUDA-event timer; events come from a per-thread pool (creation costs ~us each).
struct Timer {
    cudaStream_t st;
    size_t first;
    static std::vector<cudaEvent_t>& pool() {
        static thread_local std::vector<cudaEvent_t> p;
        return p;
    }
    static size_t& used() {
        static thread_local size_t u = 0;
        return u;
    }
    explicit Timer(cudaStream_t s) : st(s), first(used()) {}
    int mark() {
        auto& p = pool();
        if (used() == p.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            p.push_back(e);
        }
        CK(cudaEventRecord(p[used()], st));
        return (int)(used()++ - first);
    }
    double secs(int a, int b) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, pool()[first + a], pool()[first + b]));
        return ms * 1e-3;
    }
    ~Timer() { used() = first; }
};

// Device copy of the per-size tables for sizes <= smax that occur (cached).
struct DevTables {
    uint32_t leaf = 0, smax = 0;
    bool rf = false;
    std::vector<uint8_t> present;
    std::shared_ptr<const Tables> T;
    uint32_t* tstart = nullptr;
    rsd::TNodeD* tnodes = nullptr;
    uint32_t* phase_cnt = nullptr;
    uint64_t gen = 0;  // bumped whenever the device arrays are rebuilt (captured graphs hold them)
    uint32_t* N = nullptr;
    uint64_t* F = nullptr;
    int dev = -1;
    void release() {
        cudaFree(tstart);
        cudaFree(tnodes);
        cudaFree(phase_cnt);
        cudaFree(N);
        cudaFree(F);
        tstart = nullptr;
        tnodes = nullptr;
        phase_cnt = nullptr;
        N = nullptr;
        F = nullptr;
    }
};

uint64_t& device_tables_gen_counter() {
    static uint64_t g = 0;
    return g;
}
std::mutex& device_tables_mu() {
    static std::mutex mu;
    return mu;
}
std::map<int, std::unique_ptr<DevTables>>& device_tables_cache() {
    static std::map<int, std::unique_ptr<DevTables>> cache;
    return cache;
}

// generation of the cached device tables of dev (0: none)
uint64_t device_tables_generation(int dev) {
    std::lock_guard<std::mutex> g(device_tables_mu());
    auto it = device_tables_cache().find(dev);
    return it == device_tables_cache().end() || !it->second ? 0 : it->second->gen;
}

const DevTables& device_tables(int dev, uint32_t leaf, bool rf, uint32_t smax, const std::vector<uint8_t>& present,
                               cudaStream_t st) {
    std::mutex& mu = device_tables_mu();
    auto& cache = device_tables_cache();
    std::lock_guard<std::mutex> g(mu);
    auto& slot = cache[dev];
    if (slot && slot->leaf == leaf && slot->rf == rf && slot->smax == smax && slot->present == present) return *slot;
    if (!slot) slot.reset(new DevTables);
    DevTables& D = *slot;
    CK(cudaStreamSynchronize(st));
    D.release();
    D.gen = ++device_tables_gen_counter();
    D.leaf = leaf;
    D.rf = rf;
    D.smax = smax;
    D.present = present;
    D.dev = dev;
    D.T = get_tables(leaf, rf, smax);
    const Tables& T = *D.T;
    const uint32_t NP = T.NP;
    std::vector<uint32_t> tstart(smax + 2, 0);
    std::vector<rsd::TNodeD> tn;
    std::vector<uint32_t> pc((size_t)(smax + 1) * NP, 0);
    std::vector<uint32_t> N(smax + 1, 0);
    std::vector<uint64_t> F(smax + 1, 0);
    for (uint32_t s = 0; s <= smax; ++s) {
        tstart[s] = (uint32_t)tn.size();
        N[s] = T.N[s];
        F[s] = T.F[s];
        if (s == 0 || !present[s]) continue;
        const Tables::Tmpl& t = T.tmpl(s);
        for (const TNode& x : t.nodes) tn.push_back({x.rel_off, x.size, x.fixed_off, x.phase, x.tau, x.phase_rank});
        for (uint32_t p = 0; p < NP; ++p) pc[(size_t)s * NP + p] = t.phase_cnt[p];
    }
    tstart[smax + 1] = (uint32_t)tn.size();
    CK(cudaMalloc(&D.tstart, tstart.size() * 4));
    CK(cudaMalloc(&D.tnodes, std::max<size_t>(tn.size(), 1) * sizeof(rsd::TNodeD)));
    CK(cudaMalloc(&D.phase_cnt, pc.size() * 4));
    CK(cudaMalloc(&D.N, N.size() * 4));
    CK(cudaMalloc(&D.F, F.size() * 8));
    CK(cudaMemcpy(D.tstart, tstart.data(), tstart.size() * 4, cudaMemcpyHostToDevice));
    if (!tn.empty()) CK(cudaMemcpy(D.tnodes, tn.data(), tn.size() * sizeof(rsd::TNodeD), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D.phase_cnt, pc.data(), pc.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D.N, N.data(), N.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(D.F, F.data(), F.size() * 8, cudaMemcpyHostToDevice));
    return D;
}

void put_le(std::vector<uint8_t>& b, uint64_t x, int bytes) {
    for (int i = 0; i < bytes; ++i) b.push_back((uint8_t)(x >> (8 * i)));
}

// expected 32-seed iterations per node of a class -> window size and helping policy
void phase_policy(const Tables& T, SearchKind kind, uint32_t typical, uint32_t& iters, int& help) {
    double trials;
    if (kind == SK_LEAF_RF || kind == SK_LEAF_BF) {
        const uint32_t m = typical;
        // RF: the stored-value success probability p = P(B)/x(m) counts values k*m + r;
        // base seeds tried ~ 1/(m p).  BF: 1/P(B).
        double p = leaf_probability(m, kind == SK_LEAF_RF);
        trials = kind == SK_LEAF_RF ? 1.0 / (m * p) : 1.0 / p;
    } else {
        trials = 1.0 / split_probability(T.sh, typical);
    }
    const double it = trials / 32.0;
    iters = (uint32_t)std::min(16.0, std::max(1.0, std::floor(it / 16.0)));
    // help mode (per-node window dispensers, warps joining unfinished nodes) from this many
    // expected 32-seed iterations per node; below, batch mode (each node searched by one warp,
    // no dispenser atomics).  RS_HELP_IT / RS_LEAF_HELP_IT override (development A/B).
    static const double help_it = getenv("RS_HELP_IT") ? atof(getenv("RS_HELP_IT")) : 32.0;
    static const double leaf_help_it = getenv("RS_LEAF_HELP_IT") ? atof(getenv("RS_LEAF_HELP_IT")) : 32.0;
    help = it >= (kind == SK_LEAF_RF || kind == SK_LEAF_BF ? leaf_help_it : help_it);
}

}  // namespace

// ====================================================================== shards ==
//
// A shard owns the contiguous bucket range [b0, b1) = [floor(r B / W), floor((r+1) B / W))
// (P:320).  Phase 1 hashes all keys, keeps its buckets, searches every node and computes
// the Golomb-Rice length of each bucket; its summary is exchanged (allgather).  Phase 2
// derives the global bases and the shard's minimum residual step (allreduce-min gives
// delta_R, R13).  Phase 3 writes the shard's slices of the data bits and of both
// Elias-Fano sequences at their global bit positions.  stitch() ORs the slices of all
// shards into the serialized MPHF; with one shard this is the plain single-GPU build.

void shard_range(const BuildParams& p, uint64_t B, int rank, int world, uint64_t& b0, uint64_t& b1) {
    if (p.cuts.empty()) {
        b0 = B * (uint64_t)rank / (uint64_t)world;
        b1 = B * (uint64_t)(rank + 1) / (uint64_t)world;
        return;
    }
    if (p.cuts.size() != (size_t)world + 1 || p.cuts[0] != 0 || p.cuts[world] != B)
        throw Error(RECSPLIT_E_INVALID, "bucket_cuts must have world + 1 entries from 0 to B");
    for (int r = 0; r < world; ++r)
        if (p.cuts[r] > p.cuts[r + 1]) throw Error(RECSPLIT_E_INVALID, "bucket_cuts must be nondecreasing");
    b0 = p.cuts[rank];
    b1 = p.cuts[rank + 1];
}

cudaMemPool_t device_pool(int dev) { return device_pool_impl(dev); }

namespace {
struct PinnedPool {
    std::mutex mu;
    std::map<void*, size_t> live;               // handed out: pointer -> capacity
    std::multimap<size_t, void*> idle;          // returned, by capacity
    size_t idle_bytes = 0;
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // never destroyed (buffers may be freed at exit)
    return *p;
}
constexpr size_t kPinnedIdleMax = 256u << 20;  // idle bytes kept for reuse
}  // namespace

uint8_t* pinned_get(size_t bytes) {
    PinnedPool& P = pinned_pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.idle.lower_bound(bytes);
    if (it != P.idle.end() && it->first <= 2 * bytes + (1u << 20)) {  // reuse a close fit
        void* p = it->second;
        P.live[p] = it->first;
        P.idle_bytes -= it->first;
        P.idle.erase(it);
        return (uint8_t*)p;
    }
    const size_t cap = std::max<size_t>(bytes + bytes / 8, 1u << 16);
    void* p = nullptr;
    CK(cudaMallocHost(&p, cap));
    P.live[p] = cap;
    return (uint8_t*)p;
}

bool pinned_release(void* p) {
    if (!p) return false;
    PinnedPool& P = pinned_pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.live.find(p);
    if (it == P.live.end()) return false;
    const size_t cap = it->second;
    P.live.erase(it);
    P.idle.emplace(cap, p);
    P.idle_bytes += cap;
    while (P.idle_bytes > kPinnedIdleMax && !P.idle.empty()) {  // trim the largest idle buffers
        auto last = std::prev(P.idle.end());
        P.idle_bytes -= last->first;
        cudaFreeHost(last->second);
        P.idle.erase(last);
    }
    return true;
}

Globals compute_globals(const uint64_t* all, int world, int rank) {
    Globals G{};
    uint64_t mn = UINT64_MAX;
    for (int q = 0; q < world; ++q) {
        const uint64_t* x = all + 8 * q;
        if (q < rank) {
            G.key_base += x[SUM_KEYS];
            G.bit_base += x[SUM_BITS];
        }
        G.n += x[SUM_KEYS];
        G.D += x[SUM_BITS];
        if (x[SUM_MINB] < mn) mn = x[SUM_MINB];
        if (x[SUM_DUP]) G.dup = 1;
        if (x[SUM_ERR]) G.err = 1;
        if (x[SUM_NTOT] != all[SUM_NTOT]) G.err = 2;  // ranks disagree on the build's key count
    }
    G.dC = mn == UINT64_MAX ? 0 : mn;
    G.beta = G.n ? (uint64_t)(((unsigned __int128)G.D << 20) / G.n) : 0;
    return G;
}

static uint32_t ef_L(uint64_t U, uint64_t k) {
    if (U < k) return 0;
    uint64_t q = U / k;
    uint32_t w = 0;
    while (q) {
        ++w;
        q >>= 1;
    }
    return w - 1;
}

void finalize_globals(Globals& G, uint64_t B, long long dR) {
    G.dR = dR;
    const uint64_t k = B + 1;
    G.UC = G.n - B * G.dC;
    const long long RB = (long long)G.D - (long long)(((unsigned __int128)G.beta * G.n) >> 20);
    G.UP = (uint64_t)(RB - (long long)B * dR);
    G.LC = ef_L(G.UC, k);
    G.LP = ef_L(G.UP, k);
}

struct Shard::Impl {
    BuildParams p;
    int rank = 0, world = 1;
    cudaStream_t st;
    Arena A;
    uint64_t B = 0, b0 = 0, b1 = 0, Bl = 0, nl = 0, Dl = 0;
    u64* C = nullptr;      // local key offsets (Bl + 1)
    u64* Pbits = nullptr;  // local bit offsets (Bl + 1)
    unsigned long long* d_data = nullptr;  // the shard's Golomb-Rice bits (local positions)
    Globals G{};
    explicit Impl(cudaStream_t s) : st(s), A(s) {}
};

Shard::~Shard() { delete impl_; }

Shard::Shard(const uint64_t* d_keys, const BuildParams& p, int rank, int world, cudaStream_t st, bool want_values)
    : impl_(new Impl(st)) {
    auto t_start = std::chrono::steady_clock::now();
    g_launches = 0;
    Impl& I = *impl_;
    I.p = p;
    I.rank = rank;
    I.world = world;
    const uint64_t n = p.n;
    const uint32_t leaf = p.leaf;
    const uint64_t ntot = p.n_total ? p.n_total : n;  // routed shards: the whole build's count
    const uint64_t B = (ntot + p.bucket - 1) / p.bucket;  // R12
    I.B = B;
    shard_range(p, B, rank, world, I.b0, I.b1);
    const uint64_t Bl = I.b1 - I.b0;
    I.Bl = Bl;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    init_device(dev);
    const int sms = sm_count(dev);
    const Shape sh = make_shape(leaf);
    recsplit_stats& S = stats;
    memset(&S, 0, sizeof S);
    memset(summary, 0, sizeof summary);
    summary[SUM_B0] = I.b0;
    summary[SUM_B1] = I.b1;
    summary[SUM_MINB] = UINT64_MAX;
    summary[SUM_NTOT] = ntot;
    Arena& A = I.A;
    Timer tm(st);
    const int e0 = tm.mark();

    // ---- A1/A2: hash, histogram, counting sort by bucket, duplicate check ---------
    u64* lo_t = A.alloc<u64>(n);
    u8* ab_t = A.alloc<u8>(n);
    u32* bkt = A.alloc<u32>(n);
    u32* hist = A.alloc<u32>(Bl + 1);
    u64* C = A.alloc<u64>(Bl + 2);
    I.C = C;
    u64* cursor = A.alloc<u64>(Bl + 1);
    // [0] max, [1] min bucket size, [2] duplicate flag, [3] keys with lo == 0, [4] seed cap
    u32* small = A.alloc<u32>(8);
    const uint32_t cap = kSmallBucketKeys;  // sizes above it: second histogram pass below
    u32* size_hist_d = A.alloc<u32>(cap + 1);
    void* scan_tmp = A.alloc<u8>(scan_temp_bytes(std::max<uint64_t>(Bl + 1, 1)) + 64);
    CK(cudaMemsetAsync(hist, 0, (Bl + 1) * 4, st));
    CK(cudaMemsetAsync(size_hist_d, 0, (cap + 1) * 4, st));
    const uint32_t small_init[8] = {0, 0xffffffffu, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(small, small_init, sizeof small_init, cudaMemcpyHostToDevice, st));
    if (Bl == 0) {  // no buckets: only index entry B (last shard) may remain, with zero offsets
        I.C = A.alloc<u64>(2);
        I.Pbits = A.alloc<u64>(2);
        CK(cudaMemsetAsync(I.C, 0, 16, st));
        CK(cudaMemsetAsync(I.Pbits, 0, 16, st));
        CK(cudaStreamSynchronize(st));
        S.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        return;
    }
    if (p.h_keys && !p.strings) {
        // A1 overlapped with the host->device copy: chunk c is copied on the copy stream while
        // the hash kernel works on chunk c - 1 (chunked H2D with hashing)
        const uint64_t chunk = std::max<uint64_t>(1u << 20, (n + 7) / 8);
        std::vector<cudaEvent_t> evs;
        for (uint64_t off = 0; off < n; off += chunk) {
            const uint64_t len = std::min(chunk, n - off);
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            evs.push_back(ev);
            CK(cudaMemcpyAsync(const_cast<uint64_t*>(d_keys) + off, p.h_keys + off, len * 8, cudaMemcpyHostToDevice,
                               p.copy_stream));
            CK(cudaEventRecord(ev, p.copy_stream));
            CK(cudaStreamWaitEvent(st, ev, 0));
            launch_hash(d_keys + off, nullptr, len, p.g, B, I.b0, I.b1, lo_t + off, ab_t + off, bkt + off, hist, st);
            CKL();
        }
        for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // released once complete
    } else {
        launch_hash(p.strings ? nullptr : d_keys, p.strings ? d_keys : nullptr, n, p.g, B, I.b0, I.b1, lo_t, ab_t, bkt,
                    hist, st);
        CKL();
    }
    launch_bucket_stats(hist, Bl, small, size_hist_d, cap, st);
    CKL();
    exscan_u32_to_u64(hist, C, Bl, scan_tmp, st);
    CKL();
    CK(cudaMemcpyAsync(cursor, C, (Bl + 1) * 8, cudaMemcpyDeviceToDevice, st));
    // sync A: keys of the shard, bucket-size range and the histogram of bucket sizes
    // (the whole node table -- counts per phase -- follows from it on the host)
    uint32_t mm[2];
    uint64_t nl = 0;
    std::vector<uint32_t> size_hist(cap + 1);
    CK(cudaMemcpyAsync(mm, small, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&nl, C + Bl, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(size_hist.data(), size_hist_d, (cap + 1) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    I.nl = nl;
    const uint32_t smax = mm[0], smin = mm[1];
    summary[SUM_KEYS] = nl;
    summary[SUM_MINB] = smin;
    S.max_bucket = smax;
    if (smax > kMaxBucketKeys)
        throw Error(RECSPLIT_E_INVALID, "bucket of " + std::to_string(smax) + " keys exceeds the supported maximum " +
                                            std::to_string(kMaxBucketKeys) + " (use a smaller bucket_size)");
    if (smax > cap) {  // oversized buckets (bucket_size well above 8192): the full size histogram
        u32* big_hist = A.alloc<u32>(smax + 1);
        u32* mm2 = A.alloc<u32>(2);
        CK(cudaMemsetAsync(big_hist, 0, (smax + 1) * 4, st));
        launch_bucket_stats(hist, Bl, mm2, big_hist, smax, st);
        CKL();
        size_hist.assign(smax + 1, 0);
        CK(cudaMemcpyAsync(size_hist.data(), big_hist, (smax + 1) * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    u64* big_scratch = nullptr;  // dedupe tables and reorder staging of oversized buckets
    if (smax > kSmallBucketKeys) {
        uint64_t tb = 64;
        while (tb < 2ull * smax) tb <<= 1;
        big_scratch = A.alloc<u64>(std::max<uint64_t>(kDedupeBigBlocks * tb, (uint64_t)kReorderBigWarps * 2 * smax));
    }
    std::vector<uint8_t> present(smax + 1);
    for (uint32_t x = 0; x <= smax; ++x) present[x] = size_hist[x] != 0;
    u64* lo_a = A.alloc<u64>(nl);
    u8* ab_a = A.alloc<u8>(nl);
    launch_scatter(lo_t, ab_t, bkt, n, cursor, lo_a, ab_a, st);
    CKL();
    launch_dedupe(lo_a, C, Bl, smax, small + 2, big_scratch, st);
    CKL();
    // the unsorted per-key arrays (13 B/key) are dead from here on
    A.release(lo_t);
    A.release(ab_t);
    A.release(bkt);
    const int e1 = tm.mark();

    // ---- A3: node table --------------------------------------------------------
    const DevTables& DT = device_tables(dev, leaf, p.rf, smax, present, st);
    const Tables& T = *DT.T;
    const uint32_t NP = T.NP;
    const uint64_t rows = (uint64_t)(NP + 1) * (Bl + 1);
    u64* M = A.alloc<u64>(rows);
    u64* Ms = A.alloc<u64>(rows + 1);
    void* scan_tmp2 = A.alloc<u8>(scan_temp_bytes(rows) + 64);
    launch_bucket_counts(C, Bl, DT.N, DT.phase_cnt, NP, M, st, smax, small + 5);
    CKL();
    exscan_u64(M, Ms, rows, scan_tmp2, st);
    CKL();
    // node counts per phase from the size histogram (no device round trip)
    uint64_t total_nodes = 0;
    std::vector<uint64_t> pcount(NP, 0), poff(NP);
    for (uint32_t x = 1; x <= smax; ++x) {
        if (!size_hist[x]) continue;
        total_nodes += (uint64_t)size_hist[x] * T.N[x];
        const Tables::Tmpl& tp = T.tmpl(x);
        for (uint32_t q = 0; q < NP; ++q) pcount[q] += (uint64_t)size_hist[x] * tp.phase_cnt[q];
    }
    uint64_t acc = 0;
    for (uint32_t q = 0; q < NP; ++q) {
        poff[q] = acc;
        acc += pcount[q];
    }
    rsd::NodeRec* nodes = A.alloc<rsd::NodeRec>(total_nodes);
    u64* values_d = A.alloc<u64>(total_nodes);
    u32* next_win = A.alloc<u32>(total_nodes);
    u32* pcnt_d = A.alloc<u32>(NP + 32);
    const u32 nslots = search_active_slots(sms);
    int* active = A.alloc<int>(nslots);
    u32* cursors = A.alloc<u32>(2 * NP + 2);  // two per phase: batch cursor, tail (help) cursor
    CK(cudaMemsetAsync(values_d, 0xff, total_nodes * 8, st));
    CK(cudaMemsetAsync(next_win, 0, total_nodes * 4, st));
    CK(cudaMemsetAsync(cursors, 0, (2 * NP + 2) * 4, st));
    std::vector<u32> pc32(NP);
    for (uint32_t q = 0; q < NP; ++q) pc32[q] = (u32)pcount[q];
    CK(cudaMemcpyAsync(pcnt_d, pc32.data(), NP * 4, cudaMemcpyHostToDevice, st));
    launch_expand(C, Bl, Ms, NP, DT.tstart, DT.tnodes, poff.data(), nodes, st, smax);
    CKL();
    const int e2 = tm.mark();

    // ---- A4-A9: search phases, top-down ----------------------------------------
    // phases 0..n_upper-1: upper levels by depth; then L2, L1, leaves
    struct PhaseEv {
        uint32_t cls;
        int a, b, c;
    };
    std::vector<PhaseEv> pev;
    for (uint32_t q = 0; q < NP; ++q) {
        if (pcount[q] == 0) continue;
        SearchKind kind;
        uint32_t maxs, typical, cls;
        if (q < T.n_upper) {
            kind = SK_UPPER;
            maxs = smax;
            typical = std::min<uint32_t>(smax, 2 * sh.u2);
            cls = 0;
        } else if (q == T.phase_L2()) {
            kind = SK_LOWER;
            maxs = sh.u2;
            typical = sh.u2;
            cls = 1;
        } else if (q == T.phase_L1()) {
            kind = SK_LOWER;
            maxs = sh.u1;
            typical = sh.u1;
            cls = 2;
        } else {
            kind = p.rf ? SK_LEAF_RF : SK_LEAF_BF;
            maxs = leaf;
            typical = leaf;
            cls = 3;
        }
        S.nodes[cls] += pcount[q];
        PhaseLaunch P{};
        P.kind = kind;
        P.nodes = nodes + poff[q];
        P.n_nodes = pcnt_d + q;
        P.n_nodes_host = (u32)pcount[q];
        P.lo = lo_a;
        P.ab = ab_a;
        P.values = values_d;
        P.next_win = next_win;
        P.cursor = cursors + 2 * q;
        P.active = active;
        P.err = small + 4;
        P.dup = small + 2;
        P.leaf = leaf;
        P.u1 = sh.u1;
        P.u2 = sh.u2;
        P.max_size = maxs;
        phase_policy(T, kind, typical, P.iters, P.help);
        P.sm_count = sms;
        CK(cudaMemsetAsync(active, 0xff, nslots * 4, st));
        P.fuse_reorder = kind == SK_UPPER || kind == SK_LOWER;
        P.lo_w = lo_a;
        P.ab_w = ab_a;
        const int a = tm.mark();
        const bool fused = launch_search(P, st);
        CKL();
        const int b = tm.mark();
        if ((kind == SK_UPPER || kind == SK_LOWER) && !fused) {
            launch_reorder(nodes + poff[q], (u32)pcount[q], values_d, lo_a, ab_a, leaf, sh.u1, sh.u2, maxs, sms, big_scratch,
                           st);
            CKL();
        }
        const int c = tm.mark();
        pev.push_back({cls, a, b, c});
    }
    const int e3 = tm.mark();

    // ---- A10: Golomb-Rice lengths and data bits (local bit positions) -------------
    u64* len = A.alloc<u64>(Bl + 1);
    u64* Pbits = A.alloc<u64>(Bl + 2);
    I.Pbits = Pbits;
    unsigned long long* evals = A.alloc<unsigned long long>(4);
    CK(cudaMemsetAsync(evals, 0, 32, st));
    u64* nodebase = Ms;  // row 0 of the scanned count matrix
    launch_bucket_bits(C, Bl, nodebase, DT.tstart, DT.tnodes, DT.F, values_d, leaf, sh.u1, sh.u2, p.rf ? 1 : 0, len,
                       evals, st, smax);
    CKL();
    exscan_u64(len, Pbits, Bl, scan_tmp, st);
    CKL();
    uint64_t D = 0;
    uint32_t flags[3];
    unsigned long long ev_h[4];
    CK(cudaMemcpyAsync(&D, Pbits + Bl, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(flags, small + 2, 12, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ev_h, evals, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // sync C
    summary[SUM_DUP] = (flags[0] || flags[1] > 1) ? 1 : 0;
    summary[SUM_ERR] = flags[2] ? 1 : 0;
    if (summary[SUM_DUP] || summary[SUM_ERR]) D = 0;  // values are meaningless; the build fails in phase 2
    summary[SUM_BITS] = D;
    I.Dl = D;
    for (int c = 0; c < 4; ++c) S.algo_evals[c] = ev_h[c];
    const uint64_t nwords = (D + 63) / 64;
    unsigned long long* data = A.alloc<unsigned long long>(nwords + 1);
    I.d_data = data;
    CK(cudaMemsetAsync(data, 0, (nwords + 1) * 8, st));
    if (!summary[SUM_DUP] && !summary[SUM_ERR]) {
        launch_write_data(C, Bl, nodebase, DT.tstart, DT.tnodes, DT.F, values_d, Pbits, data, st, smax, nullptr);
        CKL();
    }
    if (want_values) {
        values.resize(total_nodes);
        if (total_nodes) CK(cudaMemcpyAsync(values.data(), values_d, total_nodes * 8, cudaMemcpyDeviceToHost, st));
    }
    const int e4 = tm.mark();
    CK(cudaStreamSynchronize(st));
    S.t_partition = tm.secs(e0, e1);
    S.t_tree = tm.secs(e1, e2);
    for (const PhaseEv& x : pev) {
        S.t_search[x.cls] += tm.secs(x.a, x.b);
        S.t_reorder += tm.secs(x.b, x.c);
    }
    (void)e3;
    S.t_encode = tm.secs(e3, e4);
    S.data_bits = D;
    S.kernel_launches = g_launches;
    S.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

const Globals& Shard::globals() const { return impl_->G; }

long long Shard::min_step(const uint64_t* all) {
    Impl& I = *impl_;
    I.G = compute_globals(all, I.world, I.rank);
    if (I.G.dup) throw Error(RECSPLIT_E_DUPLICATE, "duplicate keys in the input");
    if (I.G.err == 2) throw Error(RECSPLIT_E_INVALID, "ranks disagree on the total key count");
    if (I.G.err) throw Error(RECSPLIT_E_SEED_CAP, "a node exceeded the 2^40 trial cap");
    const uint64_t ntot = I.p.n_total ? I.p.n_total : I.p.n;
    if (I.G.n != ntot)
        throw Error(RECSPLIT_E_INVALID, "the shards' keys do not add up to the build's key count "
                                        "(a key was given to a rank that does not own its bucket)");
    if (I.Bl == 0) return LLONG_MAX;
    IndexView v{I.b0, I.Bl, I.G.key_base, I.G.bit_base, I.G.beta};
    long long* d = I.A.alloc<long long>(1);
    const long long llmax = LLONG_MAX;
    CK(cudaMemcpyAsync(d, &llmax, 8, cudaMemcpyHostToDevice, I.st));
    launch_min_residual(I.C, I.Pbits, v, d, I.st);
    CKL();
    long long r = 0;
    CK(cudaMemcpyAsync(&r, d, 8, cudaMemcpyDeviceToHost, I.st));
    CK(cudaStreamSynchronize(I.st));
    return r;
}

static void put_slice(std::vector<uint8_t>& out, uint64_t start, uint64_t nbits, const uint64_t* words) {
    put_le(out, start, 8);
    put_le(out, nbits, 8);
    const size_t nw = (nbits + 63) / 64;
    const size_t at = out.size();
    out.resize(at + 8 * nw);
    if (nw) memcpy(out.data() + at, words, 8 * nw);
}

// Phase 3 geometry + EF kernels: the five slices of this shard on the device.
struct ShardSlices {
    uint64_t start[5], nbits[5];             // data, C low, C up, P low, P up (global bits)
    const unsigned long long* dev[5];
    uint64_t k, c_up_total, p_up_total;
};

static ShardSlices make_slices(Shard::Impl& I, long long dR) {
    Globals& G = I.G;
    finalize_globals(G, I.B, dR);
    const uint64_t B = I.B, k = B + 1;
    const bool last = I.rank == I.world - 1;
    const uint64_t cnt = I.Bl + (last ? 1 : 0);  // index entries of this shard
    auto cprime = [&](uint64_t i, uint64_t Cg) { return Cg - i * G.dC; };
    auto rres = [&](uint64_t Pg, uint64_t Cg) {
        return (long long)Pg - (long long)(((unsigned __int128)G.beta * Cg) >> 20);
    };
    auto pprime = [&](uint64_t i, uint64_t Pg, uint64_t Cg) { return (uint64_t)(rres(Pg, Cg) - (long long)i * dR); };
    ShardSlices S{};
    S.k = k;
    S.c_up_total = (G.UC >> G.LC) + k;
    S.p_up_total = (G.UP >> G.LP) + k;
    const uint64_t Kb = G.key_base, Ob = G.bit_base;
    // global bit ranges of the shard's slices (exact partitions of each bit vector)
    const uint64_t cu_start = (cprime(I.b0, Kb) >> G.LC) + I.b0;
    const uint64_t pu_start = (pprime(I.b0, Ob, Kb) >> G.LP) + I.b0;
    const uint64_t cu_end = last ? S.c_up_total : (cprime(I.b1, Kb + I.nl) >> G.LC) + I.b1;
    const uint64_t pu_end = last ? S.p_up_total : (pprime(I.b1, Ob + I.Dl, Kb + I.nl) >> G.LP) + I.b1;
    const uint64_t st_[5] = {Ob, I.b0 * G.LC, cu_start, I.b0 * G.LP, pu_start};
    const uint64_t nb_[5] = {I.Dl, cnt * G.LC, cnt ? cu_end - cu_start : 0, cnt * G.LP, cnt ? pu_end - pu_start : 0};
    for (int q = 0; q < 5; ++q) {
        S.start[q] = st_[q];
        S.nbits[q] = nb_[q];
    }
    S.dev[0] = I.d_data;
    Arena& A = I.A;
    unsigned long long* d[4];
    for (int q = 0; q < 4; ++q) {
        const uint64_t w = (S.nbits[q + 1] + 63) / 64 + 1;
        d[q] = A.alloc<unsigned long long>(w);
        CK(cudaMemsetAsync(d[q], 0, w * 8, I.st));
        S.dev[q + 1] = d[q];
    }
    if (cnt) {
        IndexView v{I.b0, I.Bl, Kb, Ob, G.beta};
        EfSlices e{G.LC, G.LP, G.dC, dR, S.start[1], S.start[2], S.start[3], S.start[4], d[0], d[1], d[2], d[3]};
        launch_ef_write(I.C, I.Pbits, v, cnt, e, I.st);
        CKL();
    }
    return S;
}

void Shard::finish(long long dR, std::vector<uint8_t>& part) {
    Impl& I = *impl_;
    auto t0 = std::chrono::steady_clock::now();
    const ShardSlices S = make_slices(I, dR);
    const Globals& G = I.G;
    // part = global header fields + five slices, copied straight from the device
    part.clear();
    part.insert(part.end(), {'R', 'S', 'P', 'T'});
    put_le(part, 1, 4);
    const uint64_t hdr[16] = {I.p.leaf, (I.p.rf ? 1u : 0u) | (I.p.strings ? 2u : 0u), I.p.bucket, I.p.g, G.n, I.B, G.D, G.dC, G.beta,
                              (uint64_t)dR, G.LC, G.LP, S.k * G.LC, S.c_up_total, S.k * G.LP, S.p_up_total};
    for (uint64_t x : hdr) put_le(part, x, 8);
    size_t total = part.size();
    for (int q = 0; q < 5; ++q) total += 16 + 8 * ((S.nbits[q] + 63) / 64);
    part.reserve(total);
    for (int q = 0; q < 5; ++q) {
        put_le(part, S.start[q], 8);
        put_le(part, S.nbits[q], 8);
        const size_t nb = 8 * ((S.nbits[q] + 63) / 64);
        const size_t at = part.size();
        part.resize(at + nb);
        if (nb) CK(cudaMemcpyAsync(part.data() + at, S.dev[q], nb, cudaMemcpyDeviceToHost, I.st));
    }
    CK(cudaStreamSynchronize(I.st));
    stats.t_d2h += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Pinned host staging for the single-shard D2H (pageable copies run at a few GB/s; C2's
// ~1.1 MB result took 0.3 ms), grown on demand and kept for the process.
struct PinnedStage {
    std::mutex mu;
    uint8_t* p = nullptr;
    size_t cap = 0;
    uint8_t* get(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            const size_t c = std::max<size_t>(n + n / 4, 1 << 20);
            CK(cudaMallocHost(&p, c));
            cap = c;
        }
        return p;
    }
};
static PinnedStage g_stage;

void Shard::finish_blob(long long dR, uint8_t*& blob, size_t& blob_size) {
    Impl& I = *impl_;
    if (I.world != 1) throw Error(RECSPLIT_E_INVALID, "finish_blob needs a single shard");
    auto t0 = std::chrono::steady_clock::now();
    const ShardSlices S = make_slices(I, dR);
    const Globals& G = I.G;
    // single shard: every slice starts at bit 0 of its section -> the header and the five
    // sections are laid out in a pinned buffer in their final order, then copied once
    auto nbytes = [](uint64_t bits) { return (size_t)(8 * ((bits + 63) / 64)); };
    const size_t size = 72 + 2 * 24 + nbytes(S.nbits[1]) + nbytes(S.nbits[2]) + nbytes(S.nbits[3]) +
                        nbytes(S.nbits[4]) + nbytes(S.nbits[0]);
    std::vector<uint8_t> head;
    head.reserve(72);
    head.push_back('R');
    head.push_back('S');
    head.push_back('R');
    head.push_back('F');
    put_le(head, 1, 2);
    head.push_back((uint8_t)I.p.leaf);
    head.push_back((uint8_t)((I.p.rf ? 1 : 0) | (I.p.strings ? 2 : 0)));
    put_le(head, I.p.bucket, 4);
    put_le(head, 0, 4);
    for (uint64_t x : {I.p.g, G.n, I.B, G.D, G.dC, G.beta, (uint64_t)dR}) put_le(head, x, 8);
    std::lock_guard<std::mutex> lk(g_stage.mu);
    uint8_t* buf = g_stage.get(size);
    size_t at = 0;
    auto put = [&](const uint8_t* src, size_t nb) {
        memcpy(buf + at, src, nb);
        at += nb;
    };
    auto put64 = [&](uint64_t x) {
        for (int b = 0; b < 8; ++b) buf[at++] = (uint8_t)(x >> (8 * b));
    };
    auto section = [&](int q) {
        put64(S.nbits[q]);
        const size_t nb = nbytes(S.nbits[q]);
        if (nb) CK(cudaMemcpyAsync(buf + at, S.dev[q], nb, cudaMemcpyDeviceToHost, I.st));
        at += nb;
    };
    put(head.data(), head.size());
    put64(G.LC);  // u8 L then 7 pad bytes, little-endian
    section(1);
    section(2);
    put64(G.LP);
    section(3);
    section(4);
    const size_t nb = nbytes(S.nbits[0]);
    if (nb) CK(cudaMemcpyAsync(buf + at, S.dev[0], nb, cudaMemcpyDeviceToHost, I.st));
    at += nb;
    if (at != size) throw Error(RECSPLIT_E_INVALID, "internal: serialized size mismatch");
    CK(cudaStreamSynchronize(I.st));
    blob = (uint8_t*)malloc(size);
    if (!blob) throw Error(RECSPLIT_E_NOMEM, "host allocation failed");
    memcpy(blob, buf, size);
    blob_size = size;
    stats.t_d2h += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// OR a slice (local words = global bits [start, start + nbits)) into a global bit vector.
static void or_slice(uint64_t* dst, uint64_t dst_bits, uint64_t start, uint64_t nbits, const uint8_t* src) {
    const uint64_t nw = (nbits + 63) / 64;
    const uint64_t base = start >> 6, sh = start & 63;
    const uint64_t dst_words = (dst_bits + 63) / 64;
    for (uint64_t w = 0; w < nw; ++w) {
        uint64_t x;
        memcpy(&x, src + 8 * w, 8);
        if (!x) continue;
        if (base + w < dst_words) dst[base + w] |= x << sh;
        if (sh && base + w + 1 < dst_words) dst[base + w + 1] |= x >> (64 - sh);
    }
}

void stitch(const std::vector<std::pair<const uint8_t*, size_t>>& parts, std::vector<uint8_t>& blob) {
    if (parts.empty()) throw Error(RECSPLIT_E_INVALID, "no parts");
    struct View {
        uint64_t hdr[16];
        uint64_t start[5], nbits[5];
        const uint8_t* words[5];
    };
    std::vector<View> vs(parts.size());
    for (size_t q = 0; q < parts.size(); ++q) {
        const uint8_t* p = parts[q].first;
        const uint8_t* end = p + parts[q].second;
        if (parts[q].second < 8 + 128 || memcmp(p, "RSPT", 4) != 0) throw Error(RECSPLIT_E_FORMAT, "bad shard part");
        p += 8;
        View& v = vs[q];
        memcpy(v.hdr, p, 128);
        p += 128;
        for (int s = 0; s < 5; ++s) {
            if (end - p < 16) throw Error(RECSPLIT_E_FORMAT, "truncated shard part");
            memcpy(&v.start[s], p, 8);
            memcpy(&v.nbits[s], p + 8, 8);
            p += 16;
            const uint64_t nb = 8 * ((v.nbits[s] + 63) / 64);
            if ((uint64_t)(end - p) < nb) throw Error(RECSPLIT_E_FORMAT, "truncated shard part");
            v.words[s] = p;
            p += nb;
        }
        if (memcmp(v.hdr, vs[0].hdr, sizeof v.hdr) != 0) throw Error(RECSPLIT_E_FORMAT, "shard headers differ");
    }
    const uint64_t* h = vs[0].hdr;
    const uint64_t leaf = h[0], rf = h[1], bucket = h[2], g = h[3], n = h[4], B = h[5], D = h[6], dC = h[7],
                   beta = h[8], dR = h[9], LC = h[10], LP = h[11];
    const uint64_t len[5] = {D, h[12], h[13], h[14], h[15]};  // data, C low, C up, P low, P up
    std::vector<std::vector<uint64_t>> vec(5);
    for (int s = 0; s < 5; ++s) vec[s].assign((len[s] + 63) / 64, 0);
    for (const View& v : vs)
        for (int s = 0; s < 5; ++s) or_slice(vec[s].data(), len[s], v.start[s], v.nbits[s], v.words[s]);
    blob.clear();
    blob.push_back('R');
    blob.push_back('S');
    blob.push_back('R');
    blob.push_back('F');
    put_le(blob, 1, 2);
    blob.push_back((uint8_t)leaf);
    blob.push_back((uint8_t)rf);
    put_le(blob, bucket, 4);
    put_le(blob, 0, 4);
    for (uint64_t x : {g, n, B, D, dC, beta, dR}) put_le(blob, x, 8);
    auto ef = [&](uint64_t L, int lo, int up) {
        blob.push_back((uint8_t)L);
        for (int z = 0; z < 7; ++z) blob.push_back(0);
        for (int s : {lo, up}) {
            put_le(blob, len[s], 8);
            const size_t at = blob.size();
            blob.resize(at + 8 * vec[s].size());
            if (!vec[s].empty()) memcpy(blob.data() + at, vec[s].data(), 8 * vec[s].size());
        }
    };
    ef(LC, 1, 2);
    ef(LP, 3, 4);
    const size_t at = blob.size();
    blob.resize(at + 8 * vec[0].size());
    if (!vec[0].empty()) memcpy(blob.data() + at, vec[0].data(), 8 * vec[0].size());
}

// ============================================================ one enqueue ==
//
// Single-shard builds without a host round trip before the end ("size the node
// table on the device with worst-case allocation, so the build is one enqueue").  The
// synchronized path reads the bucket-size histogram back to size the node table and the
// phases; here the tables cover every bucket size up to a bound S (far beyond the Poisson
// tail: n/B + 8 sqrt(n/B) + 32), each phase's node array is sized by max_s ceil(cnt_q(s) n / s)
// -- an exact upper bound, since sum_i cnt_q(s_i) <= max_s (cnt_q(s)/s) sum_i s_i -- the phase
// counts stay on the device, the globals (n, D, delta_C, beta, delta_R, R13) and the EF layout
// are computed by kernels and the serialized MPHF is assembled in one device buffer.  One D2H
// and one synchronization at the end.  A bucket above S (flagged by the kernels) makes the
// call return false and the caller rebuilds on the synchronized path.
//
// CUDA graphs: since every launch parameter of this path depends only on the configuration
// (n, l, b, rotation fitting, g) -- never on the keys -- the whole enqueue (memsets, ~30
// kernels, the chunked H2D of host keys, the report and result D2H) is captured once per
// configuration into a graph over a persistent workspace and replayed: the host then issues
// one cudaGraphLaunch instead of ~40 API calls, so the GPU does not wait for the host's
// enqueue between short kernels (small configurations).  Per replay only the key source
// (kernel parameter of k_hash, or the source of the H2D chunk copies) and the destination of
// the result copy change (cudaGraphExec*SetParams).  The first build of a configuration runs
// uncaptured and measures its workspace; the second captures; later builds replay.
namespace {

struct PinnedReport {
    std::mutex mu;
    uint8_t* p = nullptr;
    uint8_t* get() {
        if (!p) CK(cudaMallocHost(&p, 4096));
        return p;
    }
};
PinnedReport g_report;

using ConfigKey = std::tuple<int, uint64_t, uint32_t, uint32_t, bool, uint64_t, bool, bool>;  // dev n l b rf g host stats
std::mutex g_est_mu;
std::map<ConfigKey, uint64_t> g_est_words;  // last blob size (words) per configuration
std::map<ConfigKey, size_t> g_ws_bytes;     // workspace of the last uncaptured build

// Device allocations of one build: the library pool (stream-ordered, released at scope exit)
// or, while a graph is captured, a bump allocator over the plan's persistent workspace.
struct Alloc {
    Arena* arena = nullptr;
    uint8_t* base = nullptr;
    size_t cap = 0, used = 0, total = 0;
    template <typename T>
    T* alloc(size_t count) {
        const size_t bytes = (std::max<size_t>(count * sizeof(T), 16) + 255) & ~(size_t)255;
        total += bytes;
        if (arena) return arena->alloc<T>(count);
        if (used + bytes > cap) throw Error(RECSPLIT_E_NOMEM, "graph workspace too small");
        T* p = (T*)(base + used);
        used += bytes;
        return p;
    }
    void release(void* p) {
        if (arena) arena->release(p);
    }
};

// CUDA-event marks on a plan-owned event list (graph) or the thread's event pool (Timer)
struct Marks {
    Timer* tm = nullptr;
    std::vector<cudaEvent_t>* ev = nullptr;
    bool on = true;  // false: no events (the caller did not ask for timings)
    int mark(cudaStream_t s) {
        if (!on) return -1;
        if (tm) {
            if (s == tm->st) return tm->mark();
            cudaStream_t keep = tm->st;  // (the copy stream's span of the streamed host keys)
            tm->st = s;
            const int i = tm->mark();
            tm->st = keep;
            return i;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ev->push_back(e);
        // (External: an event-record node of the graph, timed on every replay; a plain record in
        // a capturing stream is only a dependency marker)
        CK(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
        return (int)ev->size() - 1;
    }
    double secs(int a, int b) const {
        if (a < 0 || b < 0) return 0.0;
        if (tm) return tm->secs(a, b);
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, (*ev)[a], (*ev)[b]));
        return ms * 1e-3;
    }
};

struct PhaseEv {
    uint32_t cls;
    int a, b, c;
};

// What the host needs after the synchronization (marks, report layout, result buffer).
struct SingleRun {
    int e0 = -1, e1 = -1, e2 = -1, e3 = -1, e4 = -1, e5 = -1, et0 = -1, et1 = -1, h0 = -1, h1 = -1;
    std::vector<PhaseEv> pev;
    std::vector<uint32_t> phase_cls;  // class of each phase (stats)
    uint32_t NP = 0;
    uint64_t S = 0;
    uint64_t est_words = 0;
    unsigned long long* outw = nullptr;  // device result buffer
    uint8_t* rep = nullptr;              // pinned report
    uint8_t* buf = nullptr;              // pinned result (caller's buffer)
    bool exec_counted = false;
    // graph capture: the nodes a replay updates
    std::vector<cudaGraphNode_t> hash_nodes;  // device keys: the kernels reading them (key pointer = parameter 0)
    std::vector<int> hash_argc;               // ... their parameter counts
    std::vector<uint64_t> hash_off;           // ... and key offsets
    std::vector<cudaGraphNode_t> h2d_nodes;   // host keys: chunk copies
    std::vector<std::pair<uint64_t, uint64_t>> chunks;  // (offset, length) in keys
    cudaGraphNode_t blob_node = nullptr;
    uint64_t* d_keys_ws = nullptr;  // host keys: the plan's device key buffer
};

// the node just added to a capturing stream (its only dependency afterwards)
cudaGraphNode_t last_node(cudaStream_t s) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd));
    if (cs != cudaStreamCaptureStatusActive || nd != 1) throw Error(RECSPLIT_E_CUDA, "graph capture: no single last node");
    return deps[0];
}

// Enqueue the whole one-enqueue build on st (uncaptured, or into a capture when `capture`).
// Returns false if the configuration is not eligible (buckets above kSmallBucketKeys).
bool enqueue_single(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, Alloc& A, Marks& tm,
                    SingleRun& R, bool capture, cudaStream_t copy_stream) {
    const uint64_t n = p.n;
    const uint32_t leaf = p.leaf;
    const uint64_t B = (n + p.bucket - 1) / p.bucket;  // R12
    const double avg = (double)n / (double)B;
    const uint32_t S = (uint32_t)std::min<uint64_t>(n, (uint64_t)(avg + 8.0 * std::sqrt(avg) + 32.0));
    if (S > kSmallBucketKeys || B >= (1ull << 31)) return false;
    R.S = S;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    init_device(dev);
    const int sms = sm_count(dev);
    const Shape sh = make_shape(leaf);
    R.e0 = tm.mark(st);

    // small configurations: whole buckets per warp (k_bucket_tree), no node table; decided
    // before the partition because the tree kernel also does the duplicate check
    const std::shared_ptr<const Tables> Tq = get_tables(leaf, p.rf, S);
    // (off by default: measured 10-27 % slower than the phase kernels -- warps in different
    // node kinds thrash the instruction cache, ncu "no_instructions" is the top stall)
    static const int tree_env = getenv("RS_BUCKET_TREE") ? atoi(getenv("RS_BUCKET_TREE")) : 0;
    bool tree = tree_env && bucket_tree_eligible(leaf, S);
    if (tree) {
        uint32_t it;
        int help;
        phase_policy(*Tq, SK_UPPER, std::min<uint32_t>(S, 2 * sh.u2), it, help);
        tree = tree && (S <= sh.u2 || !help);
        phase_policy(*Tq, SK_LOWER, sh.u2, it, help);
        tree = tree && !help;
        phase_policy(*Tq, SK_LOWER, sh.u1, it, help);
        tree = tree && !help;
        phase_policy(*Tq, p.rf ? SK_LEAF_RF : SK_LEAF_BF, leaf, it, help);
        tree = tree && !help;
    }
    // ---- A1/A2 ----------------------------------------------------------------
    u64* C = A.alloc<u64>(B + 2);
    u32* small = A.alloc<u32>(8);  // [0] max, [1] min bucket size, [2] dup, [3] lo == 0, [4] seed cap, [5] size > S
    CK(cudaMemsetAsync(small, 0, 32, st));
    CK(cudaMemsetAsync(small + 1, 0xff, 4, st));  // min bucket size starts at UINT32_MAX
    // two-level counting sort (partition.cu) unless the groups would not fit its bounds
    static const int p2_env = getenv("RS_P2") ? atoi(getenv("RS_P2")) : 1;
    P2Shape p2;
    const bool two = p2_env && !p.strings && partition2_shape(n, B, S, p2);
    u64* lo_a = nullptr;
    u8* ab_a = nullptr;
    void* scan_tmp = A.alloc<u8>(scan_temp_bytes(std::max<uint64_t>(B, two ? (uint64_t)p2.G * p2.nb1 : 0) + 1) + 64);
    // the key source: device keys, or pinned host keys copied in chunks on the copy stream with
    // `per_chunk(off, len)` enqueued on st behind each chunk (A1 overlapped with the H2D)
    auto over_keys = [&](auto per_chunk) {
        if (p.h_keys && !p.strings) {
            uint64_t chunk = std::max<uint64_t>(1u << 20, (n + 7) / 8);
            if (two) chunk = (chunk + p2.chunk - 1) / p2.chunk * p2.chunk;  // whole level-1 blocks per copy
            std::vector<cudaEvent_t> evs;
            cudaEvent_t fork;
            CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
            evs.push_back(fork);
            CK(cudaEventRecord(fork, st));  // (the key buffer and the workspace are ordered on st)
            CK(cudaStreamWaitEvent(copy_stream, fork, 0));
            R.h0 = tm.mark(copy_stream);
            for (uint64_t off = 0; off < n; off += chunk) {
                const uint64_t len = std::min(chunk, n - off);
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                evs.push_back(ev);
                CK(cudaMemcpyAsync(const_cast<uint64_t*>(d_keys) + off, p.h_keys + off, len * 8,
                                   cudaMemcpyHostToDevice, copy_stream));
                if (capture) {
                    R.h2d_nodes.push_back(last_node(copy_stream));
                    R.chunks.push_back({off, len});
                }
                CK(cudaEventRecord(ev, copy_stream));
                CK(cudaStreamWaitEvent(st, ev, 0));
                per_chunk(off, len);
            }
            R.h1 = tm.mark(copy_stream);
            cudaEvent_t join;  // the copy stream's last event (the span mark) joins st
            CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
            evs.push_back(join);
            CK(cudaEventRecord(join, copy_stream));
            CK(cudaStreamWaitEvent(st, join, 0));
            for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // (released once complete)
        } else {
            per_chunk((uint64_t)0, n);
            if (capture && !p.strings) {
                R.hash_nodes.push_back(last_node(st));
                R.hash_argc.push_back(two ? kP2CountParams : kHashParams);
                R.hash_off.push_back(0);
            }
        }
    };
    if (two) {
        const uint64_t cells = (uint64_t)p2.G * p2.nb1;
        u32* M = A.alloc<u32>(cells);
        u64* Ms = A.alloc<u64>(cells + 1);
        u64* key1 = A.alloc<u64>(n);
        over_keys([&](uint64_t off, uint64_t len) {
            launch_p2_count(d_keys + off, len, off, p.g, B, p2, M, st);
            CKL();
        });
        exscan_u32_to_u64(M, Ms, cells, scan_tmp, st);
        CKL();
        lo_a = A.alloc<u64>(n);
        ab_a = A.alloc<u8>(n);
        launch_p2_scatter(d_keys, n, p.g, B, p2, Ms, key1, st);
        CKL();
        if (capture && !p.h_keys) {
            R.hash_nodes.push_back(last_node(st));
            R.hash_argc.push_back(kP2ScatterParams);
            R.hash_off.push_back(0);
        }
        // the duplicate check fused into level 2 when its per-warp tables are small (size bound
        // S <= 512: 16 warps x 2 KB); else the separate pass
        static const int fdd_env = getenv("RS_FUSED_DEDUPE") ? atoi(getenv("RS_FUSED_DEDUPE")) : 1;
        uint32_t dts = 0;
        if (fdd_env && !tree && S <= 512) {
            dts = 64;
            while (dts < 2 * S) dts <<= 1;
        }
        launch_p2_group(key1, p.g, B, p2, Ms, C, lo_a, ab_a, small, st, dts);
        CKL();
        if (!tree && !dts) {  // (tree: each warp checks its own bucket)
            launch_dedupe(lo_a, C, B, S, small + 2, nullptr, st);
            CKL();
        }
        A.release(key1);
        A.release(M);
        A.release(Ms);
    } else {
        u64* lo_t = A.alloc<u64>(n);
        u8* ab_t = A.alloc<u8>(n);
        u32* bkt = A.alloc<u32>(n);
        u32* hist = A.alloc<u32>(B + 1);
        u64* cursor = A.alloc<u64>(B + 1);
        CK(cudaMemsetAsync(hist, 0, (B + 1) * 4, st));
        over_keys([&](uint64_t off, uint64_t len) {
            launch_hash(p.strings ? nullptr : d_keys + off, p.strings ? d_keys : nullptr, len, p.g, B, 0, B,
                        lo_t + off, ab_t + off, bkt + off, hist, st);
            CKL();
        });
        launch_bucket_stats(hist, B, small, nullptr, S, st);  // max / min only (no size histogram needed)
        CKL();
        exscan_u32_to_u64(hist, C, B, scan_tmp, st);
        CKL();
        CK(cudaMemcpyAsync(cursor, C, (B + 1) * 8, cudaMemcpyDeviceToDevice, st));
        lo_a = A.alloc<u64>(n);
        ab_a = A.alloc<u8>(n);
        launch_scatter(lo_t, ab_t, bkt, n, cursor, lo_a, ab_a, st);
        CKL();
        if (!tree) {  // (tree: each warp checks its own bucket)
            launch_dedupe(lo_a, C, B, S, small + 2, nullptr, st);
            CKL();
        }
        A.release(lo_t);
        A.release(ab_t);
        A.release(bkt);
    }
    R.e1 = tm.mark(st);

    // ---- A3: node table for all sizes <= S --------------------------------------
    std::vector<uint8_t> present(S + 1, 1);
    present[0] = 0;
    const DevTables& DT = device_tables(dev, leaf, p.rf, S, present, st);
    const Tables& T = *DT.T;
    const uint32_t NP = T.NP;
    R.NP = NP;
    R.phase_cls.resize(NP);
    for (uint32_t q = 0; q < NP; ++q)
        R.phase_cls[q] = q < T.n_upper ? 0 : q == T.phase_L2() ? 1 : q == T.phase_L1() ? 2 : 3;
    const uint64_t rows = (uint64_t)(NP + 1) * (B + 1);
    u64* M = A.alloc<u64>(rows);
    u64* Ms = A.alloc<u64>(rows + 1);
    void* scan_tmp2 = A.alloc<u8>(scan_temp_bytes(rows) + 64);
    launch_bucket_counts(C, B, DT.N, DT.phase_cnt, NP, M, st, S, small + 5);
    CKL();
    exscan_u64(M, Ms, rows, scan_tmp2, st);
    CKL();
    // exact upper bounds of the phase lists and of the node count, and the counts expected
    // for a typical bucket (launch sizing only)
    std::vector<uint64_t> bound(NP, 0), poff(NP, 0), est(NP, 0);
    uint64_t nbound = 0;
    // expected node count of each phase under Poisson(n / B) bucket sizes (launch sizing: grid
    // and batch size; the counts themselves stay on the device).  (A phase that a bucket of
    // the mean size does not have -- a second or third upper level -- still gets its expected
    // share: sizing it from the mean bucket alone gave such phases one block, 10-100x slower
    // upper splits at l = 4..9, C4 sweep pass AK.)
    std::vector<double> expect(NP, 0.0);
    const double lavg = std::log(std::max(avg, 1e-300));
    for (uint32_t x = 1; x <= S; ++x) {
        const Tables::Tmpl& tp = T.tmpl(x);
        const double px = std::exp(x * lavg - avg - std::lgamma((double)x + 1.0));
        for (uint32_t q = 0; q < NP; ++q) {
            bound[q] = std::max<uint64_t>(bound[q], ((uint64_t)tp.phase_cnt[q] * n + x - 1) / x);
            expect[q] += px * tp.phase_cnt[q];
        }
        nbound = std::max<uint64_t>(nbound, ((uint64_t)T.N[x] * n + x - 1) / x);
    }
    uint64_t acc = 0;
    for (uint32_t q = 0; q < NP; ++q) {
        poff[q] = acc;
        acc += bound[q];
        const double e = std::ceil((double)B * expect[q] * 1.1 + 64.0);
        est[q] = bound[q] ? std::min<uint64_t>(bound[q], std::max<uint64_t>(1, (uint64_t)e)) : 0;
    }
    rsd::NodeRec* nodes = tree ? nullptr : A.alloc<rsd::NodeRec>(acc);
    u64* values_d = A.alloc<u64>(nbound);
    u32* next_win = A.alloc<u32>(nbound);
    u32* pcnt_d = A.alloc<u32>(NP + 32);
    const u32 nslots = search_active_slots(sms);
    int* active = A.alloc<int>(nslots);
    u32* cursors = A.alloc<u32>(2 * NP + 2);
    unsigned long long* exec_d = nullptr;
#ifdef RS_COUNT_EVALS
    exec_d = A.alloc<unsigned long long>(4);
    CK(cudaMemsetAsync(exec_d, 0, 32, st));
    R.exec_counted = true;
#endif
    if (!tree) {  // (the bucket-tree kernel writes every value once and uses no dispensers)
        CK(cudaMemsetAsync(values_d, 0xff, nbound * 8, st));
        CK(cudaMemsetAsync(next_win, 0, nbound * 4, st));
    }
    CK(cudaMemsetAsync(cursors, 0, (2 * NP + 2) * 4, st));
    launch_phase_counts(Ms, B, NP, pcnt_d, st);
    CKL();
    if (!tree) {
        launch_expand(C, B, Ms, NP, DT.tstart, DT.tnodes, poff.data(), nodes, st, S);
        CKL();
    }
    R.e2 = tm.mark(st);

    // ---- A4-A9 -----------------------------------------------------------------
    if (tree) {
        TreeLaunch L{};
        L.lo = lo_a;
        L.ab = ab_a;
        L.C = C;
        L.B = B;
        L.nodebase = Ms;
        L.tstart = DT.tstart;
        L.tn = DT.tnodes;
        L.S = S;
        L.bcursor = cursors;  // zeroed above
        L.values = values_d;
        L.err = small + 4;
        L.dup = small + 2;
        L.leaf = leaf;
        L.u1 = sh.u1;
        L.u2 = sh.u2;
        L.rf = p.rf;
        L.sm_count = sms;
        L.exec = exec_d;
        L.dedupe = true;
        R.et0 = tm.mark(st);
        launch_bucket_tree(L, st);
        CKL();
        R.et1 = tm.mark(st);
    }
    for (uint32_t q = 0; q < NP && !tree; ++q) {
        if (bound[q] == 0) continue;
        SearchKind kind;
        uint32_t maxs, typical;
        const uint32_t cls = R.phase_cls[q];
        if (cls == 0) {
            kind = SK_UPPER;
            maxs = S;
            typical = std::min<uint32_t>(S, 2 * sh.u2);
        } else if (cls == 1) {
            kind = SK_LOWER;
            maxs = sh.u2;
            typical = sh.u2;
        } else if (cls == 2) {
            kind = SK_LOWER;
            maxs = sh.u1;
            typical = sh.u1;
        } else {
            kind = p.rf ? SK_LEAF_RF : SK_LEAF_BF;
            maxs = leaf;
            typical = leaf;
        }
        PhaseLaunch P{};
        P.kind = kind;
        P.nodes = nodes + poff[q];
        P.n_nodes = pcnt_d + q;
        P.n_nodes_host = (u32)std::min<uint64_t>(est[q], 0xffffffffu);
        P.lo = lo_a;
        P.ab = ab_a;
        P.values = values_d;
        P.next_win = next_win;
        P.cursor = cursors + 2 * q;
        P.active = active;
        P.err = small + 4;
        P.dup = small + 2;
        P.leaf = leaf;
        P.u1 = sh.u1;
        P.u2 = sh.u2;
        P.max_size = maxs;
        phase_policy(T, kind, typical, P.iters, P.help);
        P.sm_count = sms;
        P.fuse_reorder = kind == SK_UPPER || kind == SK_LOWER;
        P.lo_w = lo_a;
        P.ab_w = ab_a;
        P.exec = exec_d ? exec_d + cls : nullptr;
        static const bool tail_help = getenv("RS_TAIL") && atoi(getenv("RS_TAIL")) > 0;
        if (P.help || tail_help) CK(cudaMemsetAsync(active, 0xff, nslots * 4, st));  // (help mode's list of open nodes)
        const int a = tm.mark(st);
        const bool fused = launch_search(P, st);
        CKL();
        const int b = tm.mark(st);
        int c = b;  // (no redistribution kernel: the search fused it, or a leaf phase)
        if ((kind == SK_UPPER || kind == SK_LOWER) && !fused) {
            launch_reorder(nodes + poff[q], P.n_nodes_host, values_d, lo_a, ab_a, leaf, sh.u1, sh.u2, maxs, sms, nullptr,
                           st, pcnt_d + q);
            CKL();
            c = tm.mark(st);
        }
        R.pev.push_back({cls, a, b, c});
    }
    R.e3 = tm.mark(st);

    // ---- A10-A12: lengths, globals, EF, data, header in one output buffer ----------
    u64* len = A.alloc<u64>(B + 1);
    u64* Pbits = A.alloc<u64>(B + 2);
    unsigned long long* evals = A.alloc<unsigned long long>(4);
    CK(cudaMemsetAsync(evals, 0, 32, st));
    launch_bucket_bits(C, B, Ms, DT.tstart, DT.tnodes, DT.F, values_d, leaf, sh.u1, sh.u2, p.rf ? 1 : 0, len, evals, st,
                       S);
    CKL();
    exscan_u64(len, Pbits, B, scan_tmp, st);
    CKL();
    SingleDev* sd = A.alloc<SingleDev>(1);
    CK(cudaMemsetAsync(sd, 0, sizeof(SingleDev), st));
    const uint64_t k = B + 1;
    const uint64_t cap_words = 9 + 2 * (3 + k + (3 * k) / 64 + 2) + (8 * n + 4096) / 64 + 16;
    unsigned long long* outw = A.alloc<unsigned long long>(cap_words);
    R.outw = outw;
    CK(cudaMemsetAsync(outw, 0, cap_words * 8, st));
    const uint64_t flags = (p.rf ? 1u : 0u) | (p.strings ? 2u : 0u);
    const uint64_t hdr0 = (uint64_t)'R' | ((uint64_t)'S' << 8) | ((uint64_t)'R' << 16) | ((uint64_t)'F' << 24) |
                          (1ull << 32) | ((uint64_t)leaf << 48) | (flags << 56);
    const uint64_t hdr1 = p.bucket;
    launch_single_index(C, Pbits, B, small, sd, hdr0, hdr1, p.g, cap_words, outw, st);
    CKL();
    launch_write_data(C, B, Ms, DT.tstart, DT.tnodes, DT.F, values_d, Pbits, outw, st, S, sd);
    CKL();
    launch_single_ef(C, Pbits, B, sd, outw, st);
    CKL();
    R.e4 = tm.mark(st);

    // ---- one D2H of the report and (most likely all of) the serialized MPHF -----
    const ConfigKey key{dev, n, leaf, p.bucket, p.rf, p.g, false, false};
    {
        std::lock_guard<std::mutex> g(g_est_mu);
        auto it = g_est_words.find(key);
        // first build of a configuration: about 2.5 bits per key plus the index
        R.est_words = it == g_est_words.end() ? std::min<uint64_t>(cap_words, 64 + (5 * n / 2 + 24 * k) / 64)
                                              : std::min<uint64_t>(cap_words, it->second + it->second / 64 + 64);
    }
    uint8_t* rep = g_report.get();
    R.rep = rep;
    CK(cudaMemcpyAsync(rep, small, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rep + 32, sd, sizeof(SingleDev), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rep + 32 + sizeof(SingleDev), evals, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rep + 64 + sizeof(SingleDev), pcnt_d, NP * 4, cudaMemcpyDeviceToHost, st));
    if (exec_d) CK(cudaMemcpyAsync(rep + 2048, exec_d, 32, cudaMemcpyDeviceToHost, st));
    // the serialized MPHF goes straight into the caller's (pinned) result buffer
    R.buf = pinned_get(R.est_words * 8);
    CK(cudaMemcpyAsync(R.buf, outw, R.est_words * 8, cudaMemcpyDeviceToHost, st));
    if (capture) R.blob_node = last_node(st);
    R.e5 = tm.mark(st);
    return true;
}

// After the synchronization: flags, the rest of the result if the estimate was short, stats.
// Returns false when the build must be redone on the synchronized path (a bucket above S).
bool finish_single(const BuildParams& p, cudaStream_t st, SingleRun& R, Marks& tm, BuildOutput& out,
                   std::chrono::steady_clock::time_point t_start) {
    struct BufGuard {
        uint8_t*& b;
        ~BufGuard() {
            if (b) pinned_release(b);
        }
    } bg{R.buf};
    CK(cudaStreamSynchronize(st));
    const uint8_t* rep = R.rep;
    uint32_t fl[8];
    memcpy(fl, rep, 32);
    SingleDev sdh;
    memcpy(&sdh, rep + 32, sizeof sdh);
    unsigned long long ev_h[4];
    memcpy(ev_h, rep + 32 + sizeof(SingleDev), 32);
    std::vector<uint32_t> pc(R.NP);
    memcpy(pc.data(), rep + 64 + sizeof(SingleDev), R.NP * 4);
    if (fl[2] || fl[3] > 1) throw Error(RECSPLIT_E_DUPLICATE, "duplicate keys in the input");
    if (fl[4]) throw Error(RECSPLIT_E_SEED_CAP, "a node exceeded the 2^40 trial cap");
    if (fl[5] || fl[0] > R.S || sdh.overflow) return false;  // rebuild on the synchronized path
    if (sdh.total_words > R.est_words) {  // the estimate was short: a larger buffer, copy the rest
        uint8_t* big = pinned_get(sdh.total_words * 8);
        memcpy(big, R.buf, R.est_words * 8);
        pinned_release(R.buf);
        R.buf = big;
        CK(cudaMemcpyAsync(R.buf + R.est_words * 8, R.outw + R.est_words, (sdh.total_words - R.est_words) * 8,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> g(g_est_mu);
        g_est_words[ConfigKey{dev, p.n, p.leaf, p.bucket, p.rf, p.g, false, false}] = sdh.total_words;
    }
    out.raw = R.buf;
    out.raw_size = sdh.total_words * 8;
    R.buf = nullptr;  // owned by out now
    // statistics
    recsplit_stats& Sst = out.stats;
    memset(&Sst, 0, sizeof Sst);
    Sst.t_partition = tm.secs(R.e0, R.e1);
    Sst.t_tree = tm.secs(R.e1, R.e2);
    for (const PhaseEv& x : R.pev) {
        Sst.t_search[x.cls] += tm.secs(x.a, x.b);
        Sst.t_reorder += tm.secs(x.b, x.c);
    }
    Sst.t_encode = tm.secs(R.e3, R.e4);
    Sst.t_device = tm.secs(R.e0, R.e5);
    if (R.et0 >= 0) Sst.t_search_tree = tm.secs(R.et0, R.et1);
    if (R.h0 >= 0) Sst.t_h2d = tm.secs(R.h0, R.h1);  // the chunked copy (overlapped with hashing, inside t_partition)
    for (uint32_t q = 0; q < R.NP; ++q) Sst.nodes[R.phase_cls[q]] += pc[q];
    for (int c = 0; c < 4; ++c) Sst.algo_evals[c] = ev_h[c];
    if (R.exec_counted) memcpy(Sst.exec_evals, rep + 2048, 32);
    Sst.data_bits = sdh.D;
    Sst.index_bits = sdh.lowC + sdh.upC + sdh.lowP + sdh.upP;
    Sst.max_bucket = fl[0];
    Sst.kernel_launches = g_launches;
    Sst.t_d2h = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count() - tm.secs(R.e0, R.e4);
    if (Sst.t_d2h < 0) Sst.t_d2h = 0;
    Sst.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return true;
}

// A captured build of one configuration over its own workspace.
struct SinglePlan {
    void* ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t cap_st = nullptr, copy_st = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> events;
    SingleRun R;
    uint32_t launches = 0;
    uint64_t dt_gen = 0;
    const void* last_src = nullptr;  // key source / result buffer the executable graph holds now
    const void* last_dst = nullptr;
    ~SinglePlan() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        if (cap_st) cudaStreamDestroy(cap_st);
        if (copy_st) cudaStreamDestroy(copy_st);
        if (ws) cudaFree(ws);
        if (R.buf) pinned_release(R.buf);
    }
};

std::mutex g_plan_mu;
// (never destroyed: a plan's graph, streams and device memory must not be released by static
// destructors after the CUDA runtime has shut down; the process exit reclaims them)
std::map<ConfigKey, std::unique_ptr<SinglePlan>>& g_plans = *new std::map<ConfigKey, std::unique_ptr<SinglePlan>>;
constexpr uint64_t kGraphMaxKeys = 1ull << 27;  // larger builds are not launch-bound (workspace ~3 GB)
constexpr size_t kMaxPlans = 4;

bool graphs_enabled() {
    static const int v = getenv("RS_GRAPH") ? atoi(getenv("RS_GRAPH")) : 1;
    return v != 0;
}

// capture the configuration's build into a new plan (nullptr if the capture fails)
std::unique_ptr<SinglePlan> capture_plan(const uint64_t* d_keys, const BuildParams& p, size_t ws_bytes) {
    std::unique_ptr<SinglePlan> P(new SinglePlan);
    const bool host = p.h_keys != nullptr;
    P->ws_bytes = ws_bytes + (host ? ((p.n * 8 + 255) & ~(size_t)255) : 0) + (1u << 20);
    CK(cudaMalloc(&P->ws, P->ws_bytes));
    CK(cudaStreamCreateWithFlags(&P->cap_st, cudaStreamNonBlocking));
    if (host) CK(cudaStreamCreateWithFlags(&P->copy_st, cudaStreamNonBlocking));
    Alloc A;
    A.base = (uint8_t*)P->ws;
    A.cap = P->ws_bytes;
    const uint64_t* keys = d_keys;
    if (host) {
        P->R.d_keys_ws = A.alloc<uint64_t>(p.n);
        keys = P->R.d_keys_ws;
    }
    {  // the per-size tables must be current before the capture (an upload synchronizes)
        const uint64_t B = (p.n + p.bucket - 1) / p.bucket;
        const double avg = (double)p.n / (double)B;
        const uint32_t S = (uint32_t)std::min<uint64_t>(p.n, (uint64_t)(avg + 8.0 * std::sqrt(avg) + 32.0));
        std::vector<uint8_t> present(S + 1, 1);
        present[0] = 0;
        int dev = 0;
        CK(cudaGetDevice(&dev));
        device_tables(dev, p.leaf, p.rf, S, present, P->cap_st);
        CK(cudaStreamSynchronize(P->cap_st));
    }
    Marks tm;
    tm.ev = &P->events;
    tm.on = p.want_stats;
    g_launches = 0;
    CK(cudaStreamBeginCapture(P->cap_st, cudaStreamCaptureModeRelaxed));
    bool ok = false;
    try {
        ok = enqueue_single(keys, p, P->cap_st, A, tm, P->R, true, P->copy_st);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(P->cap_st, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return nullptr;
    }
    P->launches = g_launches;
    CK(cudaStreamEndCapture(P->cap_st, &P->graph));
    if (!ok) return nullptr;
    CK(cudaGraphInstantiate(&P->exec, P->graph, 0));
    // the result buffer of the capture is not used by replays (each replay gets its own)
    P->last_dst = P->R.buf;
    pinned_release(P->R.buf);
    P->R.buf = nullptr;
    P->last_src = host ? (const void*)p.h_keys : (const void*)d_keys;
    return P;
}

// launch a plan for this build's keys; false if the replay must be redone uncaptured
bool replay_plan(SinglePlan& P, const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, BuildOutput& out,
                 std::chrono::steady_clock::time_point t_start) {
    // (the executable graph keeps the last parameters set: a replay with the same key source or
    // result buffer as the previous one skips the update)
    const void* src_now = p.h_keys ? (const void*)p.h_keys : (const void*)d_keys;
    if (src_now == P.last_src) {
    } else if (p.h_keys) {
        for (size_t c = 0; c < P.R.h2d_nodes.size(); ++c)
            CK(cudaGraphExecMemcpyNodeSetParams1D(P.exec, P.R.h2d_nodes[c], P.R.d_keys_ws + P.R.chunks[c].first,
                                                  p.h_keys + P.R.chunks[c].first, P.R.chunks[c].second * 8,
                                                  cudaMemcpyHostToDevice));
    } else {
        for (size_t c = 0; c < P.R.hash_nodes.size(); ++c) {
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(P.R.hash_nodes[c], &kp));
            const uint64_t* src = d_keys + P.R.hash_off[c];
            std::vector<void*> args(kp.kernelParams, kp.kernelParams + P.R.hash_argc[c]);
            args[0] = (void*)&src;
            kp.kernelParams = args.data();
            CK(cudaGraphExecKernelNodeSetParams(P.exec, P.R.hash_nodes[c], &kp));
        }
    }
    P.last_src = src_now;
    SingleRun R = P.R;  // (marks and layout; this replay's own result buffer)
    R.buf = pinned_get(R.est_words * 8);
    if (R.buf != P.last_dst) {
        P.last_dst = nullptr;  // (unknown until the update succeeds)
        CK(cudaGraphExecMemcpyNodeSetParams1D(P.exec, R.blob_node, R.buf, R.outw, R.est_words * 8,
                                              cudaMemcpyDeviceToHost));
        P.last_dst = R.buf;
    }
    g_launches = P.launches;
    CK(cudaGraphLaunch(P.exec, st));
    Marks tm;
    tm.ev = &P.events;
    tm.on = p.want_stats;
    if (!finish_single(p, st, R, tm, out, t_start)) return false;
    out.stats.graph_replay = 1;
    return true;
}

}  // namespace

void trim_caches() {
    {
        std::lock_guard<std::mutex> lk(g_report.mu);
        std::lock_guard<std::mutex> g(g_plan_mu);
        g_plans.clear();  // (destroys graphs, events, streams; frees the workspaces)
    }
    {
        std::lock_guard<std::mutex> g(g_est_mu);
        g_ws_bytes.clear();  // (the next build of a configuration runs uncaptured again)
    }
    {  // the pools the library created (devices it never used are not touched)
        std::lock_guard<std::mutex> g(pools_mu());
        int cur = -1;
        if (!pools_map().empty()) CK(cudaGetDevice(&cur));
        for (auto& kv : pools_map()) {
            CK(cudaSetDevice(kv.first));
            CK(cudaDeviceSynchronize());  // (frees of finished builds are stream-ordered)
            CK(cudaMemPoolTrimTo(kv.second, 0));
        }
        if (cur >= 0) CK(cudaSetDevice(cur));
    }
    PinnedPool& P = pinned_pool();
    std::lock_guard<std::mutex> g(P.mu);
    for (auto& kv : P.idle) cudaFreeHost(kv.second);
    P.idle.clear();
    P.idle_bytes = 0;
}

bool replay_host_keys(const uint64_t* h_keys, const BuildParams& p, cudaStream_t st, BuildOutput& out) {
    if (!graphs_enabled() || p.strings || p.shards > 1 || !p.cuts.empty() || p.n > kGraphMaxKeys) return false;
    auto t_start = std::chrono::steady_clock::now();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk_rep(g_report.mu);
    std::lock_guard<std::mutex> g(g_plan_mu);
    auto it = g_plans.find(ConfigKey{dev, p.n, p.leaf, p.bucket, p.rf, p.g, true, p.want_stats});
    if (it == g_plans.end() || it->second->dt_gen != device_tables_generation(dev)) return false;
    BuildParams q = p;
    q.h_keys = h_keys;
    if (replay_plan(*it->second, nullptr, q, st, out, t_start)) return true;
    g_plans.erase(it);  // (a bucket above the table bound: the caller takes the general path)
    return false;
}

bool build_single_fast(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, BuildOutput& out) {
    auto t_start = std::chrono::steady_clock::now();
    {  // eligibility (enqueue_single repeats it)
        const uint64_t B = (p.n + p.bucket - 1) / p.bucket;
        const double avg = (double)p.n / (double)B;
        const uint64_t S = std::min<uint64_t>(p.n, (uint64_t)(avg + 8.0 * std::sqrt(avg) + 32.0));
        if (S > kSmallBucketKeys || B >= (1ull << 31)) return false;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk_rep(g_report.mu);  // (one pinned report buffer)
    const bool host = p.h_keys && !p.strings;
    const ConfigKey key{dev, p.n, p.leaf, p.bucket, p.rf, p.g, host, p.want_stats};
    const bool graph = graphs_enabled() && !p.strings && p.n <= kGraphMaxKeys;
    if (graph) {
        std::lock_guard<std::mutex> g(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end() && it->second->dt_gen != device_tables_generation(dev)) g_plans.erase(it), it = g_plans.end();
        if (it == g_plans.end()) {
            size_t ws = 0;
            {
                std::lock_guard<std::mutex> g2(g_est_mu);
                auto w = g_ws_bytes.find(key);
                if (w != g_ws_bytes.end()) ws = w->second;
            }
            if (ws) {  // built before: capture now
                if (g_plans.size() >= kMaxPlans) g_plans.erase(g_plans.begin());  // (frees its workspace first)
                std::unique_ptr<SinglePlan> P;
                try {
                    P = capture_plan(d_keys, p, ws);
                } catch (const Error&) {  // e.g. no memory for a workspace: build uncaptured
                    P.reset();
                    cudaGetLastError();
                    std::lock_guard<std::mutex> g2(g_est_mu);
                    g_ws_bytes.erase(key);  // (no new attempt until the next uncaptured build)
                }
                if (P) {
                    P->dt_gen = device_tables_generation(dev);
                    it = g_plans.emplace(key, std::move(P)).first;
                }
            }
        }
        if (it != g_plans.end()) {
            if (replay_plan(*it->second, d_keys, p, st, out, t_start)) return true;
            g_plans.erase(it);
            return false;  // (a bucket above S: the synchronized path)
        }
    }
    g_launches = 0;
    Arena arena(st);
    Alloc A;
    A.arena = &arena;
    Timer timer(st);
    Marks tm;
    tm.tm = &timer;
    tm.on = p.want_stats;
    SingleRun R;
    if (!enqueue_single(d_keys, p, st, A, tm, R, false, p.copy_stream)) return false;
    if (!finish_single(p, st, R, tm, out, t_start)) return false;
    if (graph) {
        std::lock_guard<std::mutex> g(g_est_mu);
        g_ws_bytes[key] = A.total;
    }
    return true;
}

void build_on_device(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, bool want_values,
                     BuildOutput& out) {
    auto t_start = std::chrono::steady_clock::now();
    const int world = (int)std::max<uint32_t>(1, p.shards);
    static const int fast = getenv("RS_ONE_ENQUEUE") ? atoi(getenv("RS_ONE_ENQUEUE")) : 1;
    if (fast && world == 1 && !want_values && p.cuts.empty() && build_single_fast(d_keys, p, st, out)) return;
    std::vector<std::unique_ptr<Shard>> shards;
    std::vector<uint64_t> all(8 * world);
    for (int r = 0; r < world; ++r) {  // virtual shards run one after the other
        shards.emplace_back(new Shard(d_keys, p, r, world, st, want_values));
        memcpy(&all[8 * r], shards.back()->summary, 64);
    }
    long long dR = LLONG_MAX;  // allreduce-min (local exchange)
    for (auto& s : shards) dR = std::min(dR, s->min_step(all.data()));
    if (dR == LLONG_MAX) dR = 0;
    if (world == 1) {
        shards[0]->finish_blob(dR, out.raw, out.raw_size);
    } else {
        std::vector<std::vector<uint8_t>> parts(world);
        std::vector<std::pair<const uint8_t*, size_t>> views;
        for (int r = 0; r < world; ++r) {
            shards[r]->finish(dR, parts[r]);
            views.emplace_back(parts[r].data(), parts[r].size());
        }
        stitch(views, out.bytes);
    }
    recsplit_stats& S = out.stats;
    memset(&S, 0, sizeof S);
    for (auto& s : shards) {
        const recsplit_stats& x = s->stats;
        S.t_partition += x.t_partition;
        S.t_tree += x.t_tree;
        for (int c = 0; c < 4; ++c) {
            S.t_search[c] += x.t_search[c];
            S.algo_evals[c] += x.algo_evals[c];
            S.nodes[c] += x.nodes[c];
        }
        S.t_reorder += x.t_reorder;
        S.t_encode += x.t_encode;
        S.t_d2h += x.t_d2h;
        S.data_bits += x.data_bits;
        S.kernel_launches += x.kernel_launches;
        S.max_bucket = std::max(S.max_bucket, x.max_bucket);
        if (want_values) out.values.insert(out.values.end(), s->values.begin(), s->values.end());
    }
    const Globals& G = shards[0]->globals();
    const uint64_t k = G.n ? (p.n + p.bucket - 1) / p.bucket + 1 : 0;
    S.index_bits = k * G.LC + (G.UC >> G.LC) + k + k * G.LP + (G.UP >> G.LP) + k;
    S.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

// ------------------------------------------------------- kernel-level entry --

static void search_nodes_host(const uint64_t* lo, const uint8_t* isb, const uint32_t* off, uint32_t n_nodes,
                              uint32_t leaf, int mode /*0 split, 1 rf, 2 bf*/, uint64_t* out) {
    if (n_nodes == 0) return;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    init_device(dev);
    cudaStream_t st = 0;
    const uint64_t nk = off[n_nodes];
    Arena A(st);
    u64* d_lo = A.alloc<u64>(nk);
    u8* d_ab = A.alloc<u8>(nk);
    CK(cudaMemcpy(d_lo, lo, nk * 8, cudaMemcpyHostToDevice));
    if (isb)
        CK(cudaMemcpy(d_ab, isb, nk, cudaMemcpyHostToDevice));
    else
        CK(cudaMemset(d_ab, 0, nk));
    const Shape sh = make_shape(leaf ? leaf : 2);
    // group nodes by kind and level so each launch is homogeneous (as the pipeline's phases)
    std::vector<std::vector<rsd::NodeRec>> groups(4);
    std::vector<uint32_t> maxs(4, 0);
    for (uint32_t j = 0; j < n_nodes; ++j) {
        const uint32_t s = off[j + 1] - off[j];
        int g = mode ? 3 : (s > sh.u2 ? 0 : s > sh.u1 ? 1 : 2);
        groups[g].push_back({off[j], s, j, 0});
        maxs[g] = std::max(maxs[g], s);
    }
    u64* values = A.alloc<u64>(n_nodes);
    u32* next_win = A.alloc<u32>(n_nodes);
    u32* small = A.alloc<u32>(8);
    const int sms = sm_count(dev);
    const u32 nslots = search_active_slots(sms);
    int* active = A.alloc<int>(nslots);
    CK(cudaMemset(values, 0xff, n_nodes * 8));
    CK(cudaMemset(next_win, 0, n_nodes * 4));
    CK(cudaMemset(small, 0, 32));
    for (int g = 0; g < 4; ++g) {
        if (groups[g].empty()) continue;
        rsd::NodeRec* d_nodes = A.alloc<rsd::NodeRec>(groups[g].size());
        CK(cudaMemcpy(d_nodes, groups[g].data(), groups[g].size() * sizeof(rsd::NodeRec), cudaMemcpyHostToDevice));
        u32 cnt = (u32)groups[g].size();
        CK(cudaMemcpy(small + 6, &cnt, 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(small, 0, 8));  // batch and tail cursors
        CK(cudaMemset(active, 0xff, nslots * 4));
        PhaseLaunch P{};
        P.kind = mode == 1 ? SK_LEAF_RF : mode == 2 ? SK_LEAF_BF : (g == 0 ? SK_UPPER : SK_LOWER);
        // (groups 1 / 2 = lower level 2 / 1: launch_search picks the kernel variant by level)
        P.nodes = d_nodes;
        P.n_nodes = small + 6;
        P.n_nodes_host = cnt;
        P.lo = d_lo;
        P.ab = d_ab;
        P.values = values;
        P.next_win = next_win;
        P.cursor = small;
        P.active = active;
        P.err = small + 4;
        P.dup = small + 2;
        P.leaf = sh.leaf;
        P.u1 = sh.u1;
        P.u2 = sh.u2;
        P.max_size = maxs[g];
        P.iters = 1;
        P.help = 1;
        P.sm_count = sms;
        launch_search(P, st);
        CKL();
        CK(cudaDeviceSynchronize());
    }
    uint32_t err = 0;
    CK(cudaMemcpy(&err, small + 4, 4, cudaMemcpyDeviceToHost));
    if (err) throw Error(RECSPLIT_E_SEED_CAP, "a node exceeded the 2^40 trial cap");
    CK(cudaMemcpy(out, values, n_nodes * 8, cudaMemcpyDeviceToHost));
}

void search_leaves_host(const uint64_t* lo, const uint8_t* isb, const uint32_t* off, uint32_t n_nodes, bool rf,
                        uint64_t* out) {
    search_nodes_host(lo, isb, off, n_nodes, 0, rf ? 1 : 2, out);
}

void search_splits_host(const uint64_t* lo, const uint32_t* off, uint32_t n_nodes, uint32_t leaf, uint64_t* out) {
    search_nodes_host(lo, nullptr, off, n_nodes, leaf, 0, out);
}

}  // namespace rs
