// Host-side splitting-tree schedule: shape, Golomb-Rice parameters
// and per-bucket-size node templates.  The library's own implementation;
// shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace rs {

struct Shape {
    uint32_t leaf, f1, f2, u1, u2;
};

// P:117 fanouts in integer arithmetic (reading R5).
Shape make_shape(uint32_t leaf);

enum NodeKind : uint8_t { KIND_LEAF = 0, KIND_L1 = 1, KIND_L2 = 2, KIND_UPPER = 3 };

inline NodeKind kind_of(const Shape& sh, uint32_t s) {
    if (s <= sh.leaf) return KIND_LEAF;
    if (s <= sh.u1) return KIND_L1;
    if (s <= sh.u2) return KIND_L2;
    return KIND_UPPER;
}

// Part sizes of a split node (reading R6 for the upper split point).
int split_parts(const Shape& sh, uint32_t s, uint32_t* parts);

// Success probabilities and the Rice parameter (readings R8-R10).
double split_probability(const Shape& sh, uint32_t s);
double leaf_probability(uint32_t m, bool rotation_fitting);
int rice_tau(double p);

// One node of a bucket-size template, in preorder.
struct TNode {
    uint32_t rel_off;    // first key of the node relative to the bucket start
    uint32_t size;       // node size s
    uint32_t fixed_off;  // bit offset of its fixed (binary) Golomb-Rice part in the bucket
    uint32_t phase;      // search phase (see Tables::phase_of)
    uint32_t tau;        // Golomb-Rice parameter
    uint32_t phase_rank; // index among the bucket's nodes of the same phase, preorder
};

// Per-size tables for node sizes 0..S, plus lazily built preorder templates for the
// bucket sizes that actually occur.
struct Tables {
    Shape sh;
    bool rf;
    uint32_t S;                        // largest covered size
    uint32_t n_upper;                  // number of upper-level phases (depths 0..n_upper-1)
    uint32_t NP;                       // phases: n_upper upper + L2 + L1 + leaf
    std::vector<uint32_t> tau;         // tau[s], s = 0..S
    std::vector<uint64_t> F;           // fixed bits of a subtree of size s
    std::vector<uint32_t> N;           // nodes in a subtree of size s
    uint32_t phase_L2() const { return n_upper; }
    uint32_t phase_L1() const { return n_upper + 1; }
    uint32_t phase_leaf() const { return n_upper + 2; }
    // preorder template of a bucket of size s (1 <= s <= S) and its per-phase counts
    struct Tmpl {
        std::vector<TNode> nodes;
        std::vector<uint32_t> phase_cnt;  // NP entries
    };
    const Tmpl& tmpl(uint32_t s) const;

    // memo of templates (index = bucket size)
    mutable std::vector<std::unique_ptr<Tmpl>> memo_;
    mutable std::unique_ptr<std::mutex> mu_{new std::mutex};
};

// Expected remix evaluations of a bucket of size s (SURVEY 8(d) unit): s/p(s) per split node,
// 1/p per rotation-fitting leaf (m evaluations per base seed, 1/(m p) base seeds), m/p per
// brute-force leaf, summed over the subtree.  Used to balance the ranks' bucket ranges.
double expected_evals(const Shape& sh, bool rf, uint32_t s);

// Contiguous bucket ranges for `world` ranks with about equal expected work: cuts[0] = 0,
// cuts[world] = B, rank r owns [cuts[r], cuts[r+1]); hist[i] = size of global bucket i.
// The output bytes do not depend on where the cuts fall.
std::vector<uint64_t> balanced_cuts(const uint32_t* hist, uint64_t B, uint32_t leaf, bool rf, int world);

// Built once per (leaf, rf) and grown on demand; cached process-wide.
std::shared_ptr<const Tables> get_tables(uint32_t leaf, bool rf, uint32_t S);

}  // namespace rs
