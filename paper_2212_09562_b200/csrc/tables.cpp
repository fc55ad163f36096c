// Host-side tree schedule for the device pipeline (see tables.h).
#include "tables.h"

#include <cmath>
#include <map>
#include <mutex>

namespace rs {

Shape make_shape(uint32_t leaf) {
    // f1 = max{2, ceil(0.35 l + 0.55)}, f2 = max{2, ceil(0.21 l + 0.9)}
    Shape s;
    s.leaf = leaf;
    s.f1 = (35u * leaf + 154u) / 100u;
    s.f2 = (21u * leaf + 189u) / 100u;
    if (s.f1 < 2) s.f1 = 2;
    if (s.f2 < 2) s.f2 = 2;
    s.u1 = s.f1 * leaf;
    s.u2 = s.f2 * s.u1;
    return s;
}

int split_parts(const Shape& sh, uint32_t s, uint32_t* parts) {
    switch (kind_of(sh, s)) {
        case KIND_LEAF:
            return 0;
        case KIND_UPPER: {
            // fanout 2; left part = ceil(floor(s/2)/u2) * u2  (reading R6)
            uint32_t c0 = (s / 2 + sh.u2 - 1) / sh.u2 * sh.u2;
            parts[0] = c0;
            parts[1] = s - c0;
            return 2;
        }
        default: {
            uint32_t unit = s <= sh.u1 ? sh.leaf : sh.u1;
            uint32_t f = (s + unit - 1) / unit;
            for (uint32_t j = 0; j < f; ++j) parts[j] = unit;
            parts[f - 1] = s - (f - 1) * unit;
            return (int)f;
        }
    }
}

// log(k!) by summation (own implementation; the oracle uses lgamma).
static double log_fact(uint32_t k) {
    static std::vector<double> memo{0.0};
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    while (memo.size() <= k) memo.push_back(memo.back() + std::log((double)memo.size()));
    return memo[k];
}

double split_probability(const Shape& sh, uint32_t s) {
    // multinomial: s!/prod c_j! * prod (c_j/s)^c_j   (reading R8)
    uint32_t parts[64];
    int f = split_parts(sh, s, parts);
    double lp = log_fact(s);
    for (int j = 0; j < f; ++j) lp += (double)parts[j] * std::log((double)parts[j] / s) - log_fact(parts[j]);
    return std::exp(lp);
}

static uint32_t totient(uint32_t d) {
    uint32_t r = d, x = d;
    for (uint32_t p = 2; p * p <= x; ++p)
        if (x % p == 0) {
            while (x % p == 0) x /= p;
            r -= r / p;
        }
    if (x > 1) r -= r / x;
    return r;
}

double leaf_probability(uint32_t m, bool rotation_fitting) {
    // brute force: P(B) = m!/m^m (Appendix A);  rotation fitting: P(B) / x(m),
    // x(m) = m Nk(m) / 2^m with Nk the binary necklace count (reading R9).
    double lp = log_fact(m) - m * std::log((double)m);
    if (!rotation_fitting) return std::exp(lp);
    double nk = 0.0;
    for (uint32_t d = 1; d <= m; ++d)
        if (m % d == 0) nk += totient(d) * std::ldexp(1.0, (int)(m / d));
    nk /= m;
    double x = m * nk / std::ldexp(1.0, (int)m);
    return std::exp(lp) / x;
}

int rice_tau(double p) {
    // argmin_tau tau + 1 + Q/(1-Q), Q = (1-p)^(2^tau); ties -> smaller tau  (reading R10)
    if (p >= 1.0) return 0;
    const double l1p = std::log1p(-p);
    int best = 0;
    double bestL = INFINITY;
    for (int t = 0; t <= 62; ++t) {
        double e = std::ldexp(l1p, t);  // log Q
        double L = t + 1.0 + std::exp(e) / -std::expm1(e);
        if (L < bestL) {
            bestL = L;
            best = t;
        }
    }
    return best;
}

double expected_evals(const Shape& sh, bool rf, uint32_t s) {
    if (s <= 1) return s;  // a size-1 leaf stores 0 without a search
    if (s <= sh.leaf) {
        const double p = leaf_probability(s, rf);
        return rf ? 1.0 / p : (double)s / p;
    }
    uint32_t parts[64];
    const int f = split_parts(sh, s, parts);
    double e = (double)s / split_probability(sh, s);
    for (int j = 0; j < f; ++j) e += expected_evals(sh, rf, parts[j]);
    return e;
}

std::vector<uint64_t> balanced_cuts(const uint32_t* hist, uint64_t B, uint32_t leaf, bool rf, int world) {
    const Shape sh = make_shape(leaf);
    std::map<uint32_t, double> memo;
    std::vector<double> pre(B + 1, 0.0);
    for (uint64_t i = 0; i < B; ++i) {
        const uint32_t s = hist[i];
        auto it = memo.find(s);
        if (it == memo.end()) it = memo.emplace(s, expected_evals(sh, rf, s)).first;
        pre[i + 1] = pre[i] + it->second;
    }
    std::vector<uint64_t> cuts(world + 1, 0);
    cuts[world] = B;
    uint64_t i = 0;
    for (int r = 1; r < world; ++r) {
        const double target = pre[B] * r / world;
        while (i < B && pre[i] < target) ++i;  // first cut point with prefix >= target
        // take the nearer of i - 1 and i
        uint64_t c = i;
        if (c > 0 && target - pre[c - 1] < pre[c] - target) --c;
        cuts[r] = std::max(c, cuts[r - 1]);
    }
    return cuts;
}

static void build_tables(Tables& T) {
    const Shape& sh = T.sh;
    const uint32_t S = T.S;
    T.tau.assign(S + 1, 0);
    T.F.assign(S + 1, 0);
    T.N.assign(S + 1, 0);
    std::vector<uint32_t> updepth(S + 1, 0);  // upper levels on the longest root path
    for (uint32_t s = 1; s <= S; ++s) {
        double p = s <= sh.leaf ? leaf_probability(s, T.rf) : split_probability(sh, s);
        T.tau[s] = (uint32_t)rice_tau(p);
        uint32_t parts[64];
        int f = split_parts(sh, s, parts);
        T.F[s] = T.tau[s];
        T.N[s] = 1;
        uint32_t ud = 0;
        for (int j = 0; j < f; ++j) {
            T.F[s] += T.F[parts[j]];
            T.N[s] += T.N[parts[j]];
            if (updepth[parts[j]] > ud) ud = updepth[parts[j]];
        }
        updepth[s] = kind_of(sh, s) == KIND_UPPER ? ud + 1 : 0;
    }
    T.n_upper = 0;
    for (uint32_t s = 0; s <= S; ++s)
        if (updepth[s] > T.n_upper) T.n_upper = updepth[s];
    T.NP = T.n_upper + 3;
    T.memo_.clear();
    T.memo_.resize(S + 1);
}

const Tables::Tmpl& Tables::tmpl(uint32_t s) const {
    std::lock_guard<std::mutex> g(*mu_);
    if (memo_[s]) return *memo_[s];
    auto t = std::make_unique<Tmpl>();
    t->phase_cnt.assign(NP, 0);
    struct Item {
        uint32_t size, rel, depth;
    };
    std::vector<Item> stack{{s, 0, 0}};
    uint32_t fixed = 0;
    while (!stack.empty()) {  // preorder walk
        Item it = stack.back();
        stack.pop_back();
        TNode n;
        n.rel_off = it.rel;
        n.size = it.size;
        n.fixed_off = fixed;
        n.tau = tau[it.size];
        fixed += n.tau;
        NodeKind k = kind_of(sh, it.size);
        n.phase = k == KIND_UPPER ? it.depth : k == KIND_L2 ? phase_L2() : k == KIND_L1 ? phase_L1() : phase_leaf();
        n.phase_rank = t->phase_cnt[n.phase]++;
        t->nodes.push_back(n);
        uint32_t parts[64];
        int f = split_parts(sh, it.size, parts);
        uint32_t off = it.rel;
        uint32_t offs[64];
        for (int j = 0; j < f; ++j) {
            offs[j] = off;
            off += parts[j];
        }
        for (int j = f - 1; j >= 0; --j) stack.push_back({parts[j], offs[j], it.depth + 1});
    }
    memo_[s] = std::move(t);
    return *memo_[s];
}

std::shared_ptr<const Tables> get_tables(uint32_t leaf, bool rf, uint32_t S) {
    static std::mutex mu;
    static std::map<std::pair<uint32_t, bool>, std::shared_ptr<const Tables>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_pair(leaf, rf);
    auto it = cache.find(key);
    if (it != cache.end() && it->second->S >= S) return it->second;
    auto T = std::make_shared<Tables>();
    T->sh = make_shape(leaf);
    T->rf = rf;
    // grow geometrically so a slightly larger bucket does not rebuild every time
    uint32_t prev = it != cache.end() ? it->second->S : 0;
    T->S = S > prev + prev / 4 ? S : prev + prev / 4;
    if (T->S < 64) T->S = 64;
    build_tables(*T);
    cache[key] = T;
    return T;
}

}  // namespace rs
