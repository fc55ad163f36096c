// Host orchestration of the B200 construction pipeline (SURVEY 3 "planned
// recsplit_build"): H2D -> hash/partition -> node table -> per-phase search +
// reorder -> encode -> D2H.  Every step runs in this library's kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

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

// Stream-ordered device allocations released at scope exit.
struct Arena {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Arena(cudaStream_t s) : st(s) {}
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        CK(cudaMallocAsync(&p, bytes, st));
        ptrs.push_back(p);
        return (T*)p;
    }
    ~Arena() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

void init_device(int dev) {
    static std::mutex mu;
    static std::map<int, bool> done;
    std::lock_guard<std::mutex> g(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done[dev] = true;
}

int sm_count(int dev) {
    int v = 0;
    CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
}

struct Timer {
    cudaStream_t st;
    std::vector<cudaEvent_t> ev;
    explicit Timer(cudaStream_t s) : st(s) {}
    int mark() {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, st));
        ev.push_back(e);
        return (int)ev.size() - 1;
    }
    double secs(int a, int b) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev[a], ev[b]));
        return ms * 1e-3;
    }
    ~Timer() {
        for (auto e : ev) cudaEventDestroy(e);
    }
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

const DevTables& device_tables(int dev, uint32_t leaf, bool rf, uint32_t smax, const std::vector<uint8_t>& present,
                               cudaStream_t st) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<DevTables>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto& slot = cache[dev];
    if (slot && slot->leaf == leaf && slot->rf == rf && slot->smax == smax && slot->present == present) return *slot;
    if (!slot) slot.reset(new DevTables);
    DevTables& D = *slot;
    CK(cudaStreamSynchronize(st));
    D.release();
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

uint32_t ef_L(uint64_t U, uint64_t k) {
    if (U < k) return 0;
    uint64_t q = U / k;
    uint32_t w = 0;
    while (q) {
        ++w;
        q >>= 1;
    }
    return w - 1;
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
    help = it >= 32.0;
}

}  // namespace

void build_on_device(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, bool want_values,
                     BuildOutput& out) {
    auto t_start = std::chrono::steady_clock::now();
    g_launches = 0;
    const uint64_t n = p.n;
    const uint32_t leaf = p.leaf;
    const uint64_t B = (n + p.bucket - 1) / p.bucket;  // R12
    int dev = 0;
    CK(cudaGetDevice(&dev));
    init_device(dev);
    const int sms = sm_count(dev);
    const Shape sh = make_shape(leaf);
    recsplit_stats& S = out.stats;
    memset(&S, 0, sizeof S);

    Arena A(st);
    Timer tm(st);
    const int e0 = tm.mark();

    // ---- A1/A2: hash + duplicate set, histogram, counting sort by bucket -----------
    u64* lo_t = A.alloc<u64>(n);
    u8* ab_t = A.alloc<u8>(n);
    u32* bkt = A.alloc<u32>(n);
    u32* hist = A.alloc<u32>(B + 1);
    u64* C = A.alloc<u64>(B + 2);
    u64* cursor = A.alloc<u64>(B + 1);
    // [0] max, [1] min bucket size, [2] duplicate flag, [3] keys with MHC.hi == 0, [4] seed cap
    u32* small = A.alloc<u32>(8);
    const uint32_t cap = kMaxBucketKeys;
    u8* present_d = A.alloc<u8>(cap + 1);
    void* scan_tmp = A.alloc<u8>(scan_temp_bytes(std::max<uint64_t>(B + 1, 1)) + 64);
    uint64_t set_slots = 1024;
    while (set_slots < 2 * n) set_slots <<= 1;
    unsigned long long* dupset = A.alloc<unsigned long long>(set_slots);
    CK(cudaMemsetAsync(dupset, 0, set_slots * 8, st));
    CK(cudaMemsetAsync(hist, 0, (B + 1) * 4, st));
    CK(cudaMemsetAsync(present_d, 0, cap + 1, st));
    const uint32_t small_init[8] = {0, 0xffffffffu, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(small, small_init, sizeof small_init, cudaMemcpyHostToDevice, st));
    launch_hash(d_keys, n, p.g, B, lo_t, ab_t, bkt, hist, dupset, set_slots - 1, small + 2, st);
    CKL();
    launch_bucket_stats(hist, B, small, present_d, cap, st);
    CKL();
    exscan_u32_to_u64(hist, C, B, scan_tmp, st);
    CKL();
    CK(cudaMemcpyAsync(cursor, C, (B + 1) * 8, cudaMemcpyDeviceToDevice, st));
    u64* lo_a = A.alloc<u64>(n);
    u8* ab_a = A.alloc<u8>(n);
    u64* lo_b = A.alloc<u64>(n);
    u8* ab_b = A.alloc<u8>(n);
    launch_scatter(lo_t, ab_t, bkt, n, cursor, lo_a, ab_a, st);
    CKL();
    // sync A: bucket-size range and the set of occurring sizes
    uint32_t mm[2];
    std::vector<uint8_t> present(cap + 1);
    CK(cudaMemcpyAsync(mm, small, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(present.data(), present_d, cap + 1, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint32_t smax = mm[0], smin = mm[1];
    S.max_bucket = smax;
    if (smax > cap)
        throw Error(RECSPLIT_E_INVALID, "bucket of " + std::to_string(smax) + " keys exceeds the supported maximum " +
                                            std::to_string(cap) + " (use a smaller bucket_size)");
    present.resize(smax + 1);
    const int e1 = tm.mark();

    // ---- A3: node table --------------------------------------------------------
    const DevTables& DT = device_tables(dev, leaf, p.rf, smax, present, st);
    const Tables& T = *DT.T;
    const uint32_t NP = T.NP;
    const uint64_t rows = (uint64_t)(NP + 1) * (B + 1);
    u64* M = A.alloc<u64>(rows);
    u64* Ms = A.alloc<u64>(rows + 1);
    void* scan_tmp2 = A.alloc<u8>(scan_temp_bytes(rows) + 64);
    launch_bucket_counts(C, B, DT.N, DT.phase_cnt, NP, M, st);
    CKL();
    exscan_u64(M, Ms, rows, scan_tmp2, st);
    CKL();
    std::vector<uint64_t> rowstart(NP + 2);
    for (uint32_t r = 0; r <= NP; ++r)
        CK(cudaMemcpyAsync(&rowstart[r], Ms + (uint64_t)r * (B + 1), 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&rowstart[NP + 1], Ms + rows, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // sync B: node counts
    const uint64_t total_nodes = rowstart[1] - rowstart[0];
    std::vector<uint64_t> pcount(NP), poff(NP);
    uint64_t acc = 0;
    for (uint32_t q = 0; q < NP; ++q) {
        pcount[q] = rowstart[q + 2] - rowstart[q + 1];
        poff[q] = acc;
        acc += pcount[q];
    }
    rsd::NodeRec* nodes = A.alloc<rsd::NodeRec>(total_nodes);
    u64* values = A.alloc<u64>(total_nodes);
    u32* next_win = A.alloc<u32>(total_nodes);
    u32* pcnt_d = A.alloc<u32>(NP + 32);
    const u32 nslots = search_active_slots(sms);
    int* active = A.alloc<int>(nslots);
    u32* cursors = A.alloc<u32>(NP + 1);
    CK(cudaMemsetAsync(values, 0xff, total_nodes * 8, st));
    CK(cudaMemsetAsync(next_win, 0, total_nodes * 4, st));
    CK(cudaMemsetAsync(cursors, 0, (NP + 1) * 4, st));
    std::vector<u32> pc32(NP);
    for (uint32_t q = 0; q < NP; ++q) pc32[q] = (u32)pcount[q];
    CK(cudaMemcpyAsync(pcnt_d, pc32.data(), NP * 4, cudaMemcpyHostToDevice, st));
    launch_expand(C, B, Ms, NP, DT.tstart, DT.tnodes, poff.data(), nodes, st);
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
        P.values = values;
        P.next_win = next_win;
        P.cursor = cursors + q;
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
        const int a = tm.mark();
        launch_search(P, st);
        CKL();
        const int b = tm.mark();
        if (kind == SK_UPPER || kind == SK_LOWER) {
            CK(cudaMemcpyAsync(lo_b, lo_a, n * 8, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(ab_b, ab_a, n, cudaMemcpyDeviceToDevice, st));
            launch_reorder(nodes + poff[q], (u32)pcount[q], values, lo_a, ab_a, lo_b, ab_b, leaf, sh.u1, sh.u2, st);
            CKL();
            std::swap(lo_a, lo_b);
            std::swap(ab_a, ab_b);
        }
        const int c = tm.mark();
        pev.push_back({cls, a, b, c});
    }
    const int e3 = tm.mark();

    // ---- A10-A11: encode --------------------------------------------------------
    u64* len = A.alloc<u64>(B + 1);
    u64* Pbits = A.alloc<u64>(B + 2);
    unsigned long long* evals = A.alloc<unsigned long long>(4);
    CK(cudaMemsetAsync(evals, 0, 32, st));
    u64* nodebase = Ms;  // row 0 of the scanned count matrix
    launch_bucket_bits(C, B, nodebase, DT.tstart, DT.tnodes, DT.F, values, leaf, sh.u1, sh.u2, p.rf ? 1 : 0, len,
                       evals, st);
    CKL();
    exscan_u64(len, Pbits, B, scan_tmp, st);
    CKL();
    uint64_t D = 0;
    uint32_t flags[3];
    unsigned long long ev_h[4];
    CK(cudaMemcpyAsync(&D, Pbits + B, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(flags, small + 2, 12, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ev_h, evals, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // sync C
    if (flags[0] || flags[1] > 1) throw Error(RECSPLIT_E_DUPLICATE, "duplicate keys in the input");
    if (flags[2]) throw Error(RECSPLIT_E_SEED_CAP, "a node exceeded the 2^40 trial cap");
    for (int c = 0; c < 4; ++c) S.algo_evals[c] = ev_h[c];
    const uint64_t beta = (uint64_t)(((unsigned __int128)D << 20) / n);
    const uint64_t dC = smin;
    const uint64_t nwords = (D + 63) / 64;
    unsigned long long* data = A.alloc<unsigned long long>(nwords + 1);
    CK(cudaMemsetAsync(data, 0, (nwords + 1) * 8, st));
    launch_write_data(C, B, nodebase, DT.tstart, DT.tnodes, DT.F, values, Pbits, data, st);
    CKL();
    long long* dR_d = A.alloc<long long>(1);
    const long long llmax = INT64_MAX;
    CK(cudaMemcpyAsync(dR_d, &llmax, 8, cudaMemcpyHostToDevice, st));
    launch_min_residual(C, Pbits, B, beta, dR_d, st);
    CKL();
    long long dR = 0;
    CK(cudaMemcpyAsync(&dR, dR_d, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // sync D
    const uint64_t k = B + 1;
    const uint64_t UC = n - B * dC;
    const long long RB = (long long)D - (long long)(((unsigned __int128)beta * n) >> 20);
    const uint64_t UP = (uint64_t)(RB - (long long)B * dR);
    const uint32_t LC = ef_L(UC, k), LP = ef_L(UP, k);
    const uint64_t c_low_bits = k * LC, c_up_bits = (UC >> LC) + k;
    const uint64_t p_low_bits = k * LP, p_up_bits = (UP >> LP) + k;
    auto words_of = [](uint64_t bits) { return (bits + 63) / 64; };
    unsigned long long* c_low = A.alloc<unsigned long long>(words_of(c_low_bits) + 1);
    unsigned long long* c_up = A.alloc<unsigned long long>(words_of(c_up_bits) + 1);
    unsigned long long* p_low = A.alloc<unsigned long long>(words_of(p_low_bits) + 1);
    unsigned long long* p_up = A.alloc<unsigned long long>(words_of(p_up_bits) + 1);
    CK(cudaMemsetAsync(c_low, 0, (words_of(c_low_bits) + 1) * 8, st));
    CK(cudaMemsetAsync(c_up, 0, (words_of(c_up_bits) + 1) * 8, st));
    CK(cudaMemsetAsync(p_low, 0, (words_of(p_low_bits) + 1) * 8, st));
    CK(cudaMemsetAsync(p_up, 0, (words_of(p_up_bits) + 1) * 8, st));
    launch_ef_write(C, Pbits, B, dC, beta, dR, LC, LP, c_low, c_up, p_low, p_up, st);
    CKL();
    const int e4 = tm.mark();

    // ---- A12: serialize (R14) ---------------------------------------------------
    std::vector<uint8_t>& blob = out.bytes;
    blob.clear();
    const size_t total = 72 + 2 * 16 + 8 * (words_of(c_low_bits) + words_of(c_up_bits)) + 2 * 16 +
                         8 * (words_of(p_low_bits) + words_of(p_up_bits)) + 8 * nwords - 16;
    blob.reserve(total + 64);
    blob.push_back('R');
    blob.push_back('S');
    blob.push_back('R');
    blob.push_back('F');
    put_le(blob, 1, 2);
    blob.push_back((uint8_t)leaf);
    blob.push_back(p.rf ? 1 : 0);
    put_le(blob, p.bucket, 4);
    put_le(blob, 0, 4);
    put_le(blob, p.g, 8);
    put_le(blob, n, 8);
    put_le(blob, B, 8);
    put_le(blob, D, 8);
    put_le(blob, dC, 8);
    put_le(blob, beta, 8);
    put_le(blob, (uint64_t)dR, 8);
    struct Seg {
        size_t off;
        const void* src;
        size_t bytes;
    };
    std::vector<Seg> segs;
    auto ef_seg = [&](uint32_t L, uint64_t lowbits, unsigned long long* low, uint64_t upbits,
                      unsigned long long* up) {
        blob.push_back((uint8_t)L);
        for (int z = 0; z < 7; ++z) blob.push_back(0);
        put_le(blob, lowbits, 8);
        segs.push_back({blob.size(), low, 8 * words_of(lowbits)});
        blob.resize(blob.size() + 8 * words_of(lowbits));
        put_le(blob, upbits, 8);
        segs.push_back({blob.size(), up, 8 * words_of(upbits)});
        blob.resize(blob.size() + 8 * words_of(upbits));
    };
    ef_seg(LC, c_low_bits, c_low, c_up_bits, c_up);
    ef_seg(LP, p_low_bits, p_low, p_up_bits, p_up);
    segs.push_back({blob.size(), data, 8 * nwords});
    blob.resize(blob.size() + 8 * nwords);
    for (const Seg& sgm : segs)
        if (sgm.bytes) CK(cudaMemcpyAsync(blob.data() + sgm.off, sgm.src, sgm.bytes, cudaMemcpyDeviceToHost, st));
    if (want_values) {
        out.values.resize(total_nodes);
        if (total_nodes) CK(cudaMemcpyAsync(out.values.data(), values, total_nodes * 8, cudaMemcpyDeviceToHost, st));
    }
    const int e5 = tm.mark();
    CK(cudaStreamSynchronize(st));
    S.t_partition = tm.secs(e0, e1);
    S.t_tree = tm.secs(e1, e2);
    for (const PhaseEv& x : pev) {
        S.t_search[x.cls] += tm.secs(x.a, x.b);
        S.t_reorder += tm.secs(x.b, x.c);
    }
    (void)e3;
    S.t_encode = tm.secs(e3, e4);
    S.t_d2h = tm.secs(e4, e5);
    S.data_bits = D;
    S.index_bits = c_low_bits + c_up_bits + p_low_bits + p_up_bits;
    S.kernel_launches = g_launches;
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
    // group nodes by kind so each launch is homogeneous
    std::vector<std::vector<rsd::NodeRec>> groups(4);
    std::vector<uint32_t> maxs(4, 0);
    for (uint32_t j = 0; j < n_nodes; ++j) {
        const uint32_t s = off[j + 1] - off[j];
        int g = mode ? 3 : (s > sh.u2 ? 0 : 1);
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
        CK(cudaMemset(small, 0, 4));
        CK(cudaMemset(active, 0xff, nslots * 4));
        PhaseLaunch P{};
        P.kind = mode == 1 ? SK_LEAF_RF : mode == 2 ? SK_LEAF_BF : (g == 0 ? SK_UPPER : SK_LOWER);
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
