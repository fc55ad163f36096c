/*
 * recsplit_oracle.c -- plain, slow, obviously-correct CPU RecSplit with rotation fitting.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this code.  The product path
 * (paper_2212_09562_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * Citation keys: P:n = line n of the paper text (arXiv 2212.09562, PAPER.md);
 * "reading R<k>" = the numbered interpretation in DESIGN.md section 3 where the
 * paper is silent/ambiguous.  Everything here follows the paper's order and
 * notation: no blocking, no fusion, no search shortcuts.
 *
 * Parity status per function (see DESIGN.md section 4 for the pins):
 *   remix / mhc / remap ............ pinned (SplitMix64 vectors, closed forms)
 *   shape / parts .................. pinned (formula at P:117 evaluated by hand)
 *   tau tables ..................... pinned (Golomb-Rice cost by enumeration)
 *   find_split / leaf_bf / leaf_rf . pinned (brute-force minimality, naive
 *                                    query-semantics search, statistics)
 *   build / encode / EF / query .... pinned (exhaustive bijectivity, decode
 *                                    round trip, bits/object vs paper)
 *   mhc_string (reading R16) ....... MurmurHash3_x64_128 (the paper names no string
 *                                    hash): pinned by the published SMHasher
 *                                    verification value and test vectors
 *   seed values themselves ......... parity unpinned against the paper (no
 *                                    worked example exists); pinned only by the
 *                                    definitions above.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef uint8_t u8;

#define ORC_OK 0
#define ORC_E_INVALID (-1)
#define ORC_E_DUPLICATE (-2)
#define ORC_E_NOMEM (-3)
#define ORC_E_FORMAT (-5)
#define ORC_E_SEED_CAP (-6)

/* ---------------------------------------------------------------- hashing -- */

/* Reading R1: the node hash mixer is the SplitMix64 finalizer ("remix" of the
 * original RecSplit); the paper only says "random hash functions". */
u64 oracle_remix(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* Reading R2: master hash code.  "apply an initial hash function on every
 * object"; hi = remix(key^g^C_HI), lo = remix(key^g^C_LO).
 * remix is a bijection, so distinct keys have distinct hi. */
void oracle_mhc(u64 key, u64 g, u64 *hi, u64 *lo) {
    *hi = oracle_remix(key ^ g ^ 0x9E3779B97F4A7C15ULL);
    *lo = oracle_remix(key ^ g ^ 0xC2B2AE3D27D4EB4FULL);
}

/* Reading R16 (string keys; the paper's competitor workload P:386-388:
 * "strings of uniform random length in [10, 50]" hashed with "a high quality hash
 * function"): the master hash code of a byte string is MurmurHash3_x64_128 (Austin
 * Appleby's published, public-domain 128-bit hash; algorithm restated step by step below),
 * with seed = low 32 bits of g XOR its high 32 bits; hi = h1, lo = h2 (the two output words).
 * Pinned by the SMHasher verification value 0x6384BA69 and published vectors
 * (tests/test_oracle_pins.py). */
static u64 mm3_rotl64(u64 x, int r) { return (x << r) | (x >> (64 - r)); }

static u64 mm3_fmix64(u64 k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

/* little-endian u64 from bytes p[0..nb) (nb <= 8), missing bytes zero */
static u64 mm3_le(const u8 *p, u64 nb) {
    u64 x = 0;
    for (u64 t = 0; t < nb; t++) x |= (u64)p[t] << (8 * t);
    return x;
}

void oracle_murmur3_x64_128(const u8 *s, u64 len, u32 seed, u64 *h1_out, u64 *h2_out) {
    const u64 c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
    u64 h1 = seed, h2 = seed;
    const u64 nblocks = len / 16;
    /* body: 16-byte blocks as two little-endian words */
    for (u64 i = 0; i < nblocks; i++) {
        u64 k1 = mm3_le(s + 16 * i, 8), k2 = mm3_le(s + 16 * i + 8, 8);
        k1 *= c1;
        k1 = mm3_rotl64(k1, 31);
        k1 *= c2;
        h1 ^= k1;
        h1 = mm3_rotl64(h1, 27);
        h1 += h2;
        h1 = h1 * 5 + 0x52dce729;
        k2 *= c2;
        k2 = mm3_rotl64(k2, 33);
        k2 *= c1;
        h2 ^= k2;
        h2 = mm3_rotl64(h2, 31);
        h2 += h1;
        h2 = h2 * 5 + 0x38495ab5;
    }
    /* tail: the remaining len % 16 bytes; bytes 8..15 form k2, bytes 0..7 form k1 */
    const u8 *tail = s + 16 * nblocks;
    const u64 rest = len & 15;
    if (rest > 8) {
        u64 k2 = mm3_le(tail + 8, rest - 8);
        k2 *= c2;
        k2 = mm3_rotl64(k2, 33);
        k2 *= c1;
        h2 ^= k2;
    }
    if (rest > 0) {
        u64 k1 = mm3_le(tail, rest < 8 ? rest : 8);
        k1 *= c1;
        k1 = mm3_rotl64(k1, 31);
        k1 *= c2;
        h1 ^= k1;
    }
    /* finalization */
    h1 ^= len;
    h2 ^= len;
    h1 += h2;
    h2 += h1;
    h1 = mm3_fmix64(h1);
    h2 = mm3_fmix64(h2);
    h1 += h2;
    h2 += h1;
    *h1_out = h1;
    *h2_out = h2;
}

void oracle_mhc_string(const u8 *s, u64 len, u64 g, u64 *hi, u64 *lo) {
    oracle_murmur3_x64_128(s, len, (u32)g ^ (u32)(g >> 32), hi, lo);
}

/* Reading R3: "a hash function modulo l" as the fixed-point reduction
 * floor(high32(h) * r / 2^32). */
u32 oracle_remap(u64 h, u64 r) { return (u32)(((h >> 32) * r) >> 32); }

/* node hash for seed sigma: remix(mhc.lo + sigma) (reading R4). */
static u64 node_hash(u64 lo, u64 sigma) { return oracle_remix(lo + sigma); }

/* ------------------------------------------------------------------ shape -- */

/* f1 = max{2, ceil(0.35 l + 0.55)}, f2 = max{2, ceil(0.21 l + 0.9)}.
 * Evaluated in integers (reading R5): ceil((35 l + 55)/100), ceil((21 l + 90)/100). */
void oracle_shape(u32 leaf, u32 *f1, u32 *f2, u32 *u1, u32 *u2) {
    u32 a = (35 * leaf + 55 + 99) / 100;
    u32 c = (21 * leaf + 90 + 99) / 100;
    if (a < 2) a = 2;
    if (c < 2) c = 2;
    *f1 = a;
    *f2 = c;
    *u1 = a * leaf;
    *u2 = c * a * leaf;
}

/* Part sizes of a node of size s.  Returns the fanout, 0 for a leaf.
 *   s <= l        : leaf
 *   l < s <= u1   : parts of l, smaller last part     (lower level 1)
 *   u1 < s <= u2  : parts of u1, smaller last part    (lower level 2)
 *   s > u2        : fanout 2, [c0, s-c0], c0 = ceil(floor(s/2)/u2)*u2 (reading R6) */
int oracle_parts(u32 leaf, u32 s, u32 *parts) {
    u32 f1, f2, u1, u2;
    oracle_shape(leaf, &f1, &f2, &u1, &u2);
    if (s <= leaf) return 0;
    if (s > u2) {
        u32 half = s / 2;
        u32 c0 = ((half + u2 - 1) / u2) * u2;
        parts[0] = c0;
        parts[1] = s - c0;
        return 2;
    }
    u32 unit = (s <= u1) ? leaf : u1;
    u32 f = (s + unit - 1) / unit;
    for (u32 j = 0; j + 1 < f; j++) parts[j] = unit;
    parts[f - 1] = s - (f - 1) * unit;
    return (int)f;
}

/* Child index of key for a split node of size s with seed sigma (P:114-119,
 * SURVEY 8(c) part(k, sigma, s)):
 *   lower levels (f parts of `unit` = parts[0], smaller last): floor(remap(h, s) / unit);
 *   upper level (fanout 2, parts [c0, s - c0]): [remap(h, s) >= c0].
 * (c0 can be < s/2 for odd s, e.g. s = 2 u2 + 1, so the upper rule is not a division.) */
static u32 part_of(u32 s, const u32 *parts, int f, int upper, u64 lo, u64 sigma) {
    u32 v = oracle_remap(node_hash(lo, sigma), s);
    (void)f;
    if (upper) return v >= parts[0] ? 1u : 0u;
    return v / parts[0];
}

/* upper level <=> s > u2 */
static int is_upper(u32 leaf, u32 s) {
    u32 f1, f2, u1, u2;
    oracle_shape(leaf, &f1, &f2, &u1, &u2);
    return s > u2;
}

/* ------------------------------------------------------------------ search -- */

#define SEED_CAP (1ULL << 40) /* diagnostic cap (reading R11) */

/* Split search: smallest sigma >= 0 whose part counts equal parts[]
 * exactly.  Plain per-part counter array, no packing. */
int oracle_find_split(u32 leaf, const u64 *lo, u32 s, u64 *out_sigma) {
    u32 parts[64];
    int f = oracle_parts(leaf, s, parts);
    if (f == 0) return ORC_E_INVALID;
    int up = is_upper(leaf, s);
    for (u64 sigma = 0; sigma < SEED_CAP; sigma++) {
        u32 cnt[64];
        for (int j = 0; j < f; j++) cnt[j] = 0;
        for (u32 k = 0; k < s; k++) cnt[part_of(s, parts, f, up, lo[k], sigma)]++;
        int ok = 1;
        for (int j = 0; j < f; j++)
            if (cnt[j] != parts[j]) ok = 0;
        if (ok) {
            *out_sigma = sigma;
            return ORC_OK;
        }
    }
    return ORC_E_SEED_CAP;
}

/* Leaf, brute force: smallest sigma with OR_k 2^{remap(h_k, m)} = 2^m-1. */
int oracle_leaf_bf(const u64 *lo, u32 m, u64 *out) {
    u64 full = (m == 64) ? ~0ULL : ((1ULL << m) - 1);
    for (u64 sigma = 0; sigma < SEED_CAP; sigma++) {
        u64 mask = 0;
        for (u32 k = 0; k < m; k++) mask |= 1ULL << oracle_remap(node_hash(lo[k], sigma), m);
        if (mask == full) {
            *out = sigma;
            return ORC_OK;
        }
    }
    return ORC_E_SEED_CAP;
}

/* rot_m^r(x): rotate the m low bits of x left by r; bit p -> (p+r) mod m,
 * matching the query-side "addition modulo m" for B keys. */
u64 oracle_rot(u32 m, u32 r, u64 x) {
    u64 full = (m == 64) ? ~0ULL : ((1ULL << m) - 1);
    x &= full;
    if (r == 0) return x;
    return ((x << r) | (x >> (m - r))) & full;
}

/* Leaf, rotation fitting (minimal value rule P:297-300):
 * for k = 0,1,...: base = k*m; a = OR over A keys, b = OR over B keys;
 * the first r in 0..m-1 with a | rot_m^r(b) = 2^m-1 gives the stored value
 * base + r.  isB[k] is the global 1-bit hash, reading R7: hi & 1. */
int oracle_leaf_rf(const u64 *lo, const u8 *isB, u32 m, u64 *out) {
    u64 full = (m == 64) ? ~0ULL : ((1ULL << m) - 1);
    for (u64 k = 0; k < SEED_CAP / m; k++) {
        u64 base = k * m;
        u64 a = 0, b = 0;
        for (u32 j = 0; j < m; j++) {
            u64 bit = 1ULL << oracle_remap(node_hash(lo[j], base), m);
            if (isB[j])
                b |= bit;
            else
                a |= bit;
        }
        for (u32 r = 0; r < m; r++) {
            if ((a | oracle_rot(m, r, b)) == full) {
                *out = base + r;
                return ORC_OK;
            }
        }
    }
    return ORC_E_SEED_CAP;
}

/* ------------------------------------------------------------- Rice params -- */

static double lgam(double x) { return lgamma(x); }

/* Multinomial success probability of a split (reading R8):
 * p = s!/prod c_j! * prod (c_j/s)^{c_j}. */
double oracle_split_prob(u32 leaf, u32 s) {
    u32 parts[64];
    int f = oracle_parts(leaf, s, parts);
    double lg = lgam((double)s + 1.0);
    for (int j = 0; j < f; j++) {
        double c = parts[j];
        lg -= lgam(c + 1.0);
        if (parts[j] > 0) lg += c * log(c / (double)s);
    }
    return exp(lg);
}

/* P(B) = m!/m^m (Appendix A), as the ascending product prod j/m. */
double oracle_bij_prob_bf(u32 m) {
    double p = 1.0;
    for (u32 j = 1; j <= m; j++) p *= (double)j / (double)m;
    return p;
}

static u32 gcd_u32(u32 a, u32 b) {
    while (b) {
        u32 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

static u32 phi_u32(u32 d) {
    u32 c = 0;
    for (u32 j = 1; j <= d; j++)
        if (gcd_u32(j, d) == 1) c++;
    return c;
}

/* Number of binary necklaces of length m: Nk(m) = (1/m) sum_{d|m} phi(d) 2^{m/d}. */
double oracle_necklaces(u32 m) {
    double s = 0.0;
    for (u32 d = 1; d <= m; d++)
        if (m % d == 0) s += (double)phi_u32(d) * ldexp(1.0, (int)(m / d));
    return s / (double)m;
}

/* RF leaf: per-unit-of-stored-value success probability P(B)/x(m) with
 * x(m) = m Nk(m) / 2^m (reading R9; x(m) is Fig. 7-right's ratio). */
double oracle_bij_prob_rf(u32 m) {
    double x = (double)m * oracle_necklaces(m) / ldexp(1.0, (int)m);
    return oracle_bij_prob_bf(m) / x;
}

/* Golomb-Rice parameter (reading R10): argmin over tau in [0,62] of
 * L(tau) = tau + 1 + Q/(1-Q), Q = (1-p)^(2^tau); ties to the smaller tau. */
int oracle_golomb_tau(double p) {
    if (p >= 1.0) return 0;
    int best = 0;
    double bestL = 0.0;
    double Q = 1.0 - p; /* (1-p)^(2^0) */
    for (int t = 0; t <= 62; t++) {
        double L = (double)t + 1.0 + Q / (1.0 - Q);
        if (t == 0 || L < bestL) {
            bestL = L;
            best = t;
        }
        Q = Q * Q;
    }
    return best;
}

/* tau of a node of size s: leaf (s <= l) or split. */
int oracle_tau(u32 leaf, u32 s, int rf) {
    if (s == 0) return 0;
    if (s <= leaf) return oracle_golomb_tau(rf ? oracle_bij_prob_rf(s) : oracle_bij_prob_bf(s));
    return oracle_golomb_tau(oracle_split_prob(leaf, s));
}

/* ------------------------------------------------------------- bit vectors -- */

typedef struct {
    u64 *w;
    u64 nbits;
    u64 cap_words;
} bitvec;

static int bv_reserve(bitvec *v, u64 nbits) {
    u64 words = (nbits + 63) / 64 + 1;
    if (words <= v->cap_words) return 0;
    u64 nc = v->cap_words ? v->cap_words : 16;
    while (nc < words) nc *= 2;
    u64 *nw = (u64 *)realloc(v->w, nc * sizeof(u64));
    if (!nw) return -1;
    memset(nw + v->cap_words, 0, (nc - v->cap_words) * sizeof(u64));
    v->w = nw;
    v->cap_words = nc;
    return 0;
}

static void bv_setbit(bitvec *v, u64 pos) { v->w[pos >> 6] |= 1ULL << (pos & 63); }

/* append `width` low bits of x, LSB first */
static int bv_append(bitvec *v, u64 x, u32 width) {
    if (bv_reserve(v, v->nbits + width)) return -1;
    for (u32 t = 0; t < width; t++) {
        if ((x >> t) & 1) bv_setbit(v, v->nbits);
        v->nbits++;
    }
    return 0;
}

/* ------------------------------------------------------------- tree tables -- */

typedef struct {
    u32 leaf;
    int rf;
    u32 smax;
    int *tau; /* tau[s] */
    u64 *F;   /* total fixed bits of subtree of size s */
    u64 *N;   /* nodes in subtree of size s */
} tables;

static int tables_init(tables *T, u32 leaf, int rf, u32 smax) {
    T->leaf = leaf;
    T->rf = rf;
    T->smax = smax;
    T->tau = (int *)calloc(smax + 1, sizeof(int));
    T->F = (u64 *)calloc(smax + 1, sizeof(u64));
    T->N = (u64 *)calloc(smax + 1, sizeof(u64));
    if (!T->tau || !T->F || !T->N) return -1;
    for (u32 s = 1; s <= smax; s++) {
        T->tau[s] = oracle_tau(leaf, s, rf);
        u32 parts[64];
        int f = oracle_parts(leaf, s, parts);
        T->F[s] = (u64)T->tau[s];
        T->N[s] = 1;
        for (int j = 0; j < f; j++) {
            T->F[s] += T->F[parts[j]];
            T->N[s] += T->N[parts[j]];
        }
    }
    return 0;
}

static void tables_free(tables *T) {
    free(T->tau);
    free(T->F);
    free(T->N);
}

/* ------------------------------------------------------------------ build -- */

typedef struct {
    u64 hi, lo;
} mhc_t;

static int cmp_mhc(const void *a, const void *b) {
    u64 x = ((const mhc_t *)a)->hi, y = ((const mhc_t *)b)->hi;
    return (x > y) - (x < y);
}

/* Emit the subtree over keys[0..s) in preorder: value of this node,
 * then children left to right.  keys are reordered in place (stable partition
 * by child index) after a successful split. */
static int emit(const tables *T, mhc_t *keys, u32 s, u64 *vals, u64 *pos, mhc_t *tmp) {
    u32 leaf = T->leaf;
    if (s == 0) return ORC_OK;
    if (s <= leaf) {
        u64 lo[64];
        u8 isB[64];
        for (u32 k = 0; k < s; k++) {
            lo[k] = keys[k].lo;
            isB[k] = (u8)(keys[k].hi & 1); /* reading R7 */
        }
        u64 v;
        int rc = T->rf ? oracle_leaf_rf(lo, isB, s, &v) : oracle_leaf_bf(lo, s, &v);
        if (rc) return rc;
        vals[(*pos)++] = v;
        return ORC_OK;
    }
    u32 parts[64];
    int f = oracle_parts(leaf, s, parts);
    u64 *lo = (u64 *)malloc((size_t)s * sizeof(u64));
    if (!lo) return ORC_E_NOMEM;
    for (u32 k = 0; k < s; k++) lo[k] = keys[k].lo;
    u64 sigma;
    int rc = oracle_find_split(leaf, lo, s, &sigma);
    free(lo);
    if (rc) return rc;
    vals[(*pos)++] = sigma;
    /* stable partition by child index */
    u32 w = 0;
    for (int j = 0; j < f; j++)
        for (u32 k = 0; k < s; k++)
            if (part_of(s, parts, f, is_upper(leaf, s), keys[k].lo, sigma) == (u32)j) tmp[w++] = keys[k];
    memcpy(keys, tmp, (size_t)s * sizeof(mhc_t));
    u32 off = 0;
    for (int j = 0; j < f; j++) {
        rc = emit(T, keys + off, parts[j], vals, pos, tmp + off);
        if (rc) return rc;
        off += parts[j];
    }
    return ORC_OK;
}

typedef struct {
    const tables *T;
    mhc_t *keys;
    const u64 *C;       /* bucket key offsets, B+1 */
    const u64 *nodebase; /* first value slot of each bucket, B+1 */
    u64 *vals;
    u64 b0, b1; /* bucket range [b0, b1) */
    int rc;
} job_t;

static void *run_job(void *arg) {
    job_t *J = (job_t *)arg;
    J->rc = ORC_OK;
    u64 maxs = 0;
    for (u64 i = J->b0; i < J->b1; i++)
        if (J->C[i + 1] - J->C[i] > maxs) maxs = J->C[i + 1] - J->C[i];
    mhc_t *tmp = (mhc_t *)malloc((size_t)(maxs + 1) * sizeof(mhc_t));
    if (!tmp) {
        J->rc = ORC_E_NOMEM;
        return NULL;
    }
    for (u64 i = J->b0; i < J->b1; i++) {
        u64 pos = J->nodebase[i];
        int rc = emit(J->T, J->keys + J->C[i], (u32)(J->C[i + 1] - J->C[i]), J->vals, &pos, tmp);
        if (rc) {
            J->rc = rc;
            break;
        }
    }
    free(tmp);
    return NULL;
}

static int bitwidth(u64 x) {
    int w = 0;
    while (x) {
        w++;
        x >>= 1;
    }
    return w;
}

/* Elias-Fano of v[0..k), monotone, U = v[k-1]:
 * L = U<k ? 0 : floor(log2(U/k)); lower bits at i*L; upper bit (v_i>>L)+i. */
static int ef_build(const u64 *v, u64 k, bitvec *low, bitvec *up, u32 *Lout) {
    u64 U = v[k - 1];
    u32 L = (U < k) ? 0 : (u32)(bitwidth(U / k) - 1);
    for (u64 i = 0; i < k; i++)
        if (bv_append(low, v[i] & ((L == 0) ? 0 : ((1ULL << L) - 1)), L)) return -1;
    u64 uplen = (U >> L) + k;
    if (bv_reserve(up, uplen)) return -1;
    up->nbits = uplen;
    for (u64 i = 0; i < k; i++) bv_setbit(up, (v[i] >> L) + i);
    *Lout = L;
    return 0;
}

static void put_u8(u8 **p, u8 x) { *(*p)++ = x; }
static void put_u16(u8 **p, uint16_t x) {
    for (int i = 0; i < 2; i++) *(*p)++ = (u8)(x >> (8 * i));
}
static void put_u32(u8 **p, u32 x) {
    for (int i = 0; i < 4; i++) *(*p)++ = (u8)(x >> (8 * i));
}
static void put_u64(u8 **p, u64 x) {
    for (int i = 0; i < 8; i++) *(*p)++ = (u8)(x >> (8 * i));
}
static void put_words(u8 **p, const u64 *w, u64 nbits) {
    for (u64 i = 0; i < (nbits + 63) / 64; i++) put_u64(p, w[i]);
}

/*
 * Full construction.  Single-threaded algorithm;
 * `threads` only splits contiguous bucket ranges and never changes
 * the output.  On success *out is malloc'ed (free with oracle_free).
 * If values_out is non-NULL it receives all node values (bucket order, each
 * bucket in preorder) for diagnostics.
 */
static int cmp_mhc_full(const void *a, const void *b) {
    const mhc_t *x = (const mhc_t *)a, *y = (const mhc_t *)b;
    if (x->hi != y->hi) return (x->hi > y->hi) - (x->hi < y->hi);
    return (x->lo > y->lo) - (x->lo < y->lo);
}

/* core construction over precomputed master hash codes (mk, n entries, consumed);
 * flags bit0 = rotation fitting, bit1 = string keys (recorded in the header) */
static int build_core(mhc_t *mk, u64 n, u32 leaf, u32 bsize, int flags, u64 g, int threads, u8 **out,
                      u64 *out_size, u64 **values_out, u64 *n_values);

int oracle_build_ex(const u64 *keys, u64 n, u32 leaf, u32 bsize, int rf, u64 g, int threads,
                    u8 **out, u64 *out_size, u64 **values_out, u64 *n_values) {
    *out = NULL;
    *out_size = 0;
    if (n == 0 || leaf < 2 || leaf > 24 || bsize < 1 || n >= (1ULL << 32)) return ORC_E_INVALID;
    mhc_t *mk = (mhc_t *)malloc((size_t)n * sizeof(mhc_t));
    if (!mk) return ORC_E_NOMEM;
    for (u64 i = 0; i < n; i++) oracle_mhc(keys[i], g, &mk[i].hi, &mk[i].lo);
    return build_core(mk, n, leaf, bsize, rf ? 1 : 0, g, threads, out, out_size, values_out, n_values);
}

/* String keys (N4): key i is bytes[offsets[i] .. offsets[i+1]). */
int oracle_build_strings(const u8 *bytes, const u64 *offsets, u64 n, u32 leaf, u32 bsize, int rf, u64 g,
                         int threads, u8 **out, u64 *out_size) {
    *out = NULL;
    *out_size = 0;
    if (n == 0 || leaf < 2 || leaf > 24 || bsize < 1 || n >= (1ULL << 32)) return ORC_E_INVALID;
    mhc_t *mk = (mhc_t *)malloc((size_t)n * sizeof(mhc_t));
    if (!mk) return ORC_E_NOMEM;
    for (u64 i = 0; i < n; i++)
        oracle_mhc_string(bytes + offsets[i], offsets[i + 1] - offsets[i], g, &mk[i].hi, &mk[i].lo);
    return build_core(mk, n, leaf, bsize, (rf ? 1 : 0) | 2, g, threads, out, out_size, NULL, NULL);
}

static int build_core(mhc_t *mk, u64 n, u32 leaf, u32 bsize, int flags, u64 g, int threads, u8 **out,
                      u64 *out_size, u64 **values_out, u64 *n_values) {
    const int rf = flags & 1;
    if (values_out) *values_out = NULL;
    if (n_values) *n_values = 0;
    if (threads < 1) threads = 1;
    u64 B = (n + bsize - 1) / bsize; /* reading R12 */

    /* 1. sort by MHC (bucket is monotone in hi), duplicate check: equal master hash codes
     *    (for u64 keys equal hi <=> equal key, R2; for strings equal (hi, lo)) */
    qsort(mk, (size_t)n, sizeof(mhc_t), cmp_mhc_full);
    for (u64 i = 1; i < n; i++)
        if (mk[i].hi == mk[i - 1].hi && mk[i].lo == mk[i - 1].lo) {
            free(mk);
            return ORC_E_DUPLICATE;
        }

    /* 2. bucket borders: C[i] = number of keys in buckets < i */
    u64 *C = (u64 *)calloc(B + 1, sizeof(u64));
    if (!C) {
        free(mk);
        return ORC_E_NOMEM;
    }
    for (u64 i = 0; i < n; i++) C[oracle_remap(mk[i].hi, B) + 1]++;
    u64 smax = 0;
    for (u64 i = 0; i < B; i++)
        if (C[i + 1] > smax) smax = C[i + 1];
    for (u64 i = 0; i < B; i++) C[i + 1] += C[i];

    tables T;
    if (tables_init(&T, leaf, rf, (u32)smax)) {
        free(mk);
        free(C);
        return ORC_E_NOMEM;
    }
    u64 *nodebase = (u64 *)calloc(B + 1, sizeof(u64));
    for (u64 i = 0; i < B; i++) nodebase[i + 1] = nodebase[i] + T.N[C[i + 1] - C[i]];
    u64 nv = nodebase[B];
    u64 *vals = (u64 *)calloc(nv + 1, sizeof(u64));

    /* 3. per-bucket splitting trees, contiguous bucket ranges per thread */
    int rc = ORC_OK;
    job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; t++) {
        jobs[t].T = &T;
        jobs[t].keys = mk;
        jobs[t].C = C;
        jobs[t].nodebase = nodebase;
        jobs[t].vals = vals;
        jobs[t].b0 = B * (u64)t / (u64)threads;
        jobs[t].b1 = B * (u64)(t + 1) / (u64)threads;
    }
    if (threads == 1) {
        run_job(&jobs[0]);
    } else {
        for (int t = 0; t < threads; t++) pthread_create(&tids[t], NULL, run_job, &jobs[t]);
        for (int t = 0; t < threads; t++) pthread_join(tids[t], NULL);
    }
    for (int t = 0; t < threads; t++)
        if (jobs[t].rc && !rc) rc = jobs[t].rc;
    free(jobs);
    free(tids);

    /* 4. Golomb-Rice per bucket: fixed parts of all nodes in preorder, then
     *    unary parts in preorder; buckets concatenated. */
    bitvec data = {0}, efcl = {0}, efcu = {0}, efpl = {0}, efpu = {0};
    u64 *P = (u64 *)calloc(B + 1, sizeof(u64));
    if (rc == ORC_OK) {
        for (u64 i = 0; i < B; i++) {
            P[i] = data.nbits;
            u64 s = C[i + 1] - C[i];
            if (s == 0) continue;
            /* recover the tau sequence of this bucket's preorder by walking the shape */
            u64 cnt = T.N[s];
            u32 *sizes = (u32 *)malloc((size_t)cnt * sizeof(u32));
            u64 top = 0, w = 0;
            u32 *stack = (u32 *)malloc((size_t)cnt * sizeof(u32));
            stack[top++] = (u32)s;
            while (top) {
                u32 cs = stack[--top];
                sizes[w++] = cs;
                u32 parts[64];
                int f = oracle_parts(leaf, cs, parts);
                for (int j = f - 1; j >= 0; j--) stack[top++] = parts[j];
            }
            for (u64 j = 0; j < cnt; j++) {
                int tau = T.tau[sizes[j]];
                if (bv_append(&data, vals[nodebase[i] + j], (u32)tau)) rc = ORC_E_NOMEM;
            }
            for (u64 j = 0; j < cnt; j++) {
                int tau = T.tau[sizes[j]];
                u64 q = vals[nodebase[i] + j] >> tau;
                if (bv_reserve(&data, data.nbits + q + 1)) rc = ORC_E_NOMEM;
                data.nbits += q;
                bv_setbit(&data, data.nbits);
                data.nbits++;
            }
            free(sizes);
            free(stack);
        }
        P[B] = data.nbits;
    }

    /* 5. Trend-subtracted Elias-Fano index (reading R13) */
    u64 D = P[B];
    u64 dC = 0, beta = 0;
    i64 dR = 0;
    u32 LC = 0, LP = 0;
    if (rc == ORC_OK) {
        dC = C[1] - C[0];
        for (u64 i = 0; i < B; i++)
            if (C[i + 1] - C[i] < dC) dC = C[i + 1] - C[i];
        beta = (u64)(((unsigned __int128)D << 20) / n);
        i64 *R = (i64 *)malloc((size_t)(B + 1) * sizeof(i64));
        for (u64 i = 0; i <= B; i++) R[i] = (i64)P[i] - (i64)(((unsigned __int128)beta * C[i]) >> 20);
        dR = R[1] - R[0];
        for (u64 i = 0; i < B; i++)
            if (R[i + 1] - R[i] < dR) dR = R[i + 1] - R[i];
        u64 *Cp = (u64 *)malloc((size_t)(B + 1) * sizeof(u64));
        u64 *Pp = (u64 *)malloc((size_t)(B + 1) * sizeof(u64));
        for (u64 i = 0; i <= B; i++) {
            Cp[i] = C[i] - i * dC;
            Pp[i] = (u64)(R[i] - (i64)i * dR);
        }
        if (ef_build(Cp, B + 1, &efcl, &efcu, &LC) || ef_build(Pp, B + 1, &efpl, &efpu, &LP))
            rc = ORC_E_NOMEM;
        free(R);
        free(Cp);
        free(Pp);
    }

    /* 6. serialize (reading R14) */
    if (rc == ORC_OK) {
        u64 size = 72;
        size += 8 + 8 + 8 * ((efcl.nbits + 63) / 64) + 8 + 8 * ((efcu.nbits + 63) / 64);
        size += 8 + 8 + 8 * ((efpl.nbits + 63) / 64) + 8 + 8 * ((efpu.nbits + 63) / 64);
        size += 8 * ((D + 63) / 64);
        u8 *buf = (u8 *)calloc((size_t)size, 1);
        u8 *p = buf;
        put_u8(&p, 'R');
        put_u8(&p, 'S');
        put_u8(&p, 'R');
        put_u8(&p, 'F');
        put_u16(&p, 1);
        put_u8(&p, (u8)leaf);
        put_u8(&p, (u8)(flags & 3));
        put_u32(&p, bsize);
        put_u32(&p, 0);
        put_u64(&p, g);
        put_u64(&p, n);
        put_u64(&p, B);
        put_u64(&p, D);
        put_u64(&p, dC);
        put_u64(&p, beta);
        put_u64(&p, (u64)dR);
        bitvec *seq[4] = {&efcl, &efcu, &efpl, &efpu};
        u32 Ls[2] = {LC, LP};
        for (int e = 0; e < 2; e++) {
            put_u8(&p, (u8)Ls[e]);
            for (int z = 0; z < 7; z++) put_u8(&p, 0);
            put_u64(&p, seq[2 * e]->nbits);
            put_words(&p, seq[2 * e]->w, seq[2 * e]->nbits);
            put_u64(&p, seq[2 * e + 1]->nbits);
            put_words(&p, seq[2 * e + 1]->w, seq[2 * e + 1]->nbits);
        }
        put_words(&p, data.w, D);
        *out = buf;
        *out_size = size;
        if (values_out) {
            *values_out = vals;
            vals = NULL;
            if (n_values) *n_values = nv;
        }
    }
    free(vals);
    free(mk);
    free(C);
    free(P);
    free(nodebase);
    free(data.w);
    free(efcl.w);
    free(efcu.w);
    free(efpl.w);
    free(efpu.w);
    tables_free(&T);
    return rc;
}

int oracle_build(const u64 *keys, u64 n, u32 leaf, u32 bsize, int rf, u64 g, int threads, u8 **out,
                 u64 *out_size) {
    return oracle_build_ex(keys, n, leaf, bsize, rf, g, threads, out, out_size, NULL, NULL);
}

/* Values of one bucket's tree (preorder) given its raw keys: used by the
 * sampled full-size parity tests.  keys need not be sorted. */
int oracle_bucket_values(const u64 *keys, u64 s, u32 leaf, int rf, u64 g, u64 *vals, u64 *n_vals) {
    mhc_t *mk = (mhc_t *)malloc((size_t)(s + 1) * sizeof(mhc_t));
    mhc_t *tmp = (mhc_t *)malloc((size_t)(s + 1) * sizeof(mhc_t));
    for (u64 i = 0; i < s; i++) oracle_mhc(keys[i], g, &mk[i].hi, &mk[i].lo);
    qsort(mk, (size_t)s, sizeof(mhc_t), cmp_mhc);
    tables T;
    tables_init(&T, leaf, rf, (u32)(s ? s : 1));
    u64 pos = 0;
    int rc = emit(&T, mk, (u32)s, vals, &pos, tmp);
    *n_vals = pos;
    tables_free(&T);
    free(mk);
    free(tmp);
    return rc;
}

/* ------------------------------------------------------------------ query -- */

static u64 get_u64(const u8 *p) {
    u64 x = 0;
    for (int i = 0; i < 8; i++) x |= (u64)p[i] << (8 * i);
    return x;
}

typedef struct {
    u32 L;
    u64 nlow, nup;
    const u8 *low, *up; /* raw little-endian words */
} ef_view;

static u64 word_at(const u8 *base, u64 i) { return get_u64(base + 8 * i); }

static int bit_at(const u8 *base, u64 pos) { return (int)((word_at(base, pos >> 6) >> (pos & 63)) & 1); }

/* Decode a whole EF sequence in one pass over the upper bits:
 * the i-th one at position pos gives high part pos - i. */
static void ef_decode_all(const ef_view *e, u64 k, u64 *v) {
    u64 i = 0;
    for (u64 pos = 0; pos < e->nup && i < k; pos++) {
        if (bit_at(e->up, pos)) {
            u64 lo = 0;
            for (u32 t = 0; t < e->L; t++) lo |= (u64)bit_at(e->low, i * e->L + t) << t;
            v[i] = ((pos - i) << e->L) | lo;
            i++;
        }
    }
}

static const u8 *parse_ef(const u8 *p, const u8 *end, ef_view *e) {
    if (p + 16 > end) return NULL;
    e->L = p[0];
    p += 8;
    e->nlow = get_u64(p);
    p += 8;
    e->low = p;
    p += 8 * ((e->nlow + 63) / 64);
    if (p + 8 > end) return NULL;
    e->nup = get_u64(p);
    p += 8;
    e->up = p;
    p += 8 * ((e->nup + 63) / 64);
    if (p > end) return NULL;
    return p;
}

/* Query: bucket -> index -> descend splits summing left sibling
 * sizes -> leaf value (+ r mod m for B keys under rotation fitting).
 * Decodes the index once, then evaluates every key. */
static int query_impl(const u8 *blob, u64 size, const u64 *keys, const u8 *sbytes, const u64 *soff, u64 nk,
                      u64 *out);

int oracle_query_many(const u8 *blob, u64 size, const u64 *keys, u64 nk, u64 *out) {
    return query_impl(blob, size, keys, NULL, NULL, nk, out);
}

int oracle_query_strings(const u8 *blob, u64 size, const u8 *bytes, const u64 *offsets, u64 nk, u64 *out) {
    return query_impl(blob, size, NULL, bytes, offsets, nk, out);
}

static int query_impl(const u8 *blob, u64 size, const u64 *keys, const u8 *sbytes, const u64 *soff, u64 nk,
                      u64 *out) {
    if (size < 72 || memcmp(blob, "RSRF", 4) != 0) return ORC_E_FORMAT;
    const u8 *end = blob + size;
    u32 leaf = blob[6];
    int rf = blob[7] & 1;
    u64 g = get_u64(blob + 16), B = get_u64(blob + 32);
    u64 D = get_u64(blob + 40), dC = get_u64(blob + 48), beta = get_u64(blob + 56);
    i64 dR = (i64)get_u64(blob + 64);
    ef_view ec, ep;
    const u8 *p = parse_ef(blob + 72, end, &ec);
    if (!p) return ORC_E_FORMAT;
    p = parse_ef(p, end, &ep);
    if (!p || p + 8 * ((D + 63) / 64) > end) return ORC_E_FORMAT;
    const u8 *data = p;

    /* recover C[i] = C'[i] + i dC and P[i] = P'[i] + i dR + floor(beta C[i] / 2^20) */
    u64 *C = (u64 *)malloc((size_t)(B + 1) * sizeof(u64));
    u64 *P = (u64 *)malloc((size_t)(B + 1) * sizeof(u64));
    ef_decode_all(&ec, B + 1, C);
    ef_decode_all(&ep, B + 1, P);
    u64 smax = 1;
    for (u64 i = 0; i <= B; i++) {
        C[i] += i * dC;
        P[i] = (u64)((i64)P[i] + (i64)i * dR) + (u64)(((unsigned __int128)beta * C[i]) >> 20);
        if (i && C[i] - C[i - 1] > smax) smax = C[i] - C[i - 1];
    }
    tables T;
    tables_init(&T, leaf, rf, (u32)smax);

    if (((blob[7] >> 1) & 1) != (keys == NULL)) {  /* key type must match the MPHF's */
        tables_free(&T);
        free(C);
        free(P);
        return ORC_E_FORMAT;
    }
    for (u64 kk = 0; kk < nk; kk++) {
        u64 hi, lo;
        if (keys)
            oracle_mhc(keys[kk], g, &hi, &lo);
        else
            oracle_mhc_string(sbytes + soff[kk], soff[kk + 1] - soff[kk], g, &hi, &lo);
        u64 i = oracle_remap(hi, B);
        u64 s = C[i + 1] - C[i];
        if (s == 0) {
            out[kk] = 0;
            continue;
        }
        u64 fc = P[i], uc = P[i] + T.F[s], offset = C[i];
        u32 cs = (u32)s;
        for (;;) {
            int tau = T.tau[cs];
            u64 q = 0;
            while (!bit_at(data, uc)) {
                q++;
                uc++;
            }
            uc++;
            u64 fixed = 0;
            for (int t = 0; t < tau; t++) fixed |= (u64)bit_at(data, fc + (u64)t) << t;
            fc += (u64)tau;
            u64 x = (q << tau) | fixed;
            if (cs <= leaf) {
                u32 m = cs;
                u64 base = rf ? x - x % m : x;
                u32 v = oracle_remap(node_hash(lo, base), m);
                if (rf && (hi & 1)) v = (u32)((v + x % m) % m);
                out[kk] = offset + v;
                break;
            }
            u32 parts[64];
            int f = oracle_parts(leaf, cs, parts);
            u32 j = part_of(cs, parts, f, is_upper(leaf, cs), lo, x);
            for (u32 c = 0; c < j; c++) {
                fc += T.F[parts[c]];
                u64 skip = T.N[parts[c]]; /* skip N(c) unary codes */
                while (skip) {
                    if (bit_at(data, uc)) skip--;
                    uc++;
                }
                offset += parts[c];
            }
            cs = parts[j];
        }
    }
    tables_free(&T);
    free(C);
    free(P);
    return ORC_OK;
}

int oracle_query(const u8 *blob, u64 size, u64 key, u64 *out) {
    return query_impl(blob, size, &key, NULL, NULL, 1, out);
}

void oracle_free(void *p) { free(p); }
