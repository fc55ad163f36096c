"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: bit-exact -- every stored value and every serialized byte is integer work.
Kernel level: leaf (rotation fitting / brute force) and split searches on random
nodes of every size class.  End to end: full byte parity on C1 and C2 and on many
small configurations (ragged buckets, empty buckets, m=1 leaves, fanout edge cases);
sampled per-bucket parity at the full C3 size in the launch configuration bench.py
times, plus properties that hold at any size (bijectivity, bits/object).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_2212_09562_b200 as rs
import synth

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def _mhc_np(keys, g=0):
    """Vectorised master hash for selecting buckets in the sampled tests (R2)."""
    def remix(z):
        with np.errstate(over="ignore"):
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))
    k = keys ^ np.uint64(g)
    return remix(k ^ np.uint64(0x9E3779B97F4A7C15)), remix(k ^ np.uint64(0xC2B2AE3D27D4EB4F))


# ------------------------------------------------------------------ kernel level --

@pytest.mark.parametrize("rf,mmax", [(True, 16), (False, 12), (True, 8), (False, 8), (True, 3)])
def test_leaf_search_parity(rf, mmax):
    """Leaf searches against the oracle's (rotation fitting P:245-263 / brute force P:125-128),
    phases of mixed leaf sizes up to mmax (small-leaf phases are the batch-mode case)."""
    rng = np.random.default_rng(11 + rf + mmax)
    sizes = []
    for m in range(1, mmax + 1):
        sizes += [m] * (400 if m <= 12 else 60)
    if mmax <= 8:
        sizes = sizes * 4  # several leaves per lane
    if not rf and mmax > 11:
        sizes = [m for m in sizes if m <= 11] + [12] * 10
    rng.shuffle(sizes)
    off = np.zeros(len(sizes) + 1, dtype=np.uint32)
    off[1:] = np.cumsum(sizes)
    lo = rng.integers(0, M64, size=int(off[-1]), dtype=np.uint64, endpoint=True)
    isb = rng.integers(0, 2, size=int(off[-1]), dtype=np.uint8)
    got = rs.search_leaves(lo, isb, off, rotation_fitting=rf)
    sl = [(int(off[j]), int(off[j + 1])) for j in range(len(sizes))]
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        if rf:
            want = list(ex.map(lambda ab: oracle.leaf_rf(lo[ab[0]:ab[1]], isb[ab[0]:ab[1]]), sl))
        else:
            want = list(ex.map(lambda ab: oracle.leaf_bf(lo[ab[0]:ab[1]]), sl))
    assert got.tolist() == want


def test_leaf_search_large_m():
    rng = np.random.default_rng(5)
    sizes = [17, 18, 20, 24, 24, 19]
    off = np.zeros(len(sizes) + 1, dtype=np.uint32)
    off[1:] = np.cumsum(sizes)
    lo = rng.integers(0, M64, size=int(off[-1]), dtype=np.uint64, endpoint=True)
    isb = rng.integers(0, 2, size=int(off[-1]), dtype=np.uint8)
    got = rs.search_leaves(lo, isb, off, rotation_fitting=True)
    with ThreadPoolExecutor(len(sizes)) as ex:
        want = list(ex.map(lambda j: oracle.leaf_rf(lo[off[j]:off[j + 1]], isb[off[j]:off[j + 1]]),
                           range(len(sizes))))
    assert got.tolist() == want


def test_leaf_values_above_2_32():
    """Rotation-fitting leaves of 24 keys have stored values around 2^31..2^33 (mean 2.1e9,
    SURVEY 8(f) N3): values >= 2^32 run the carry path with a per-window high word.  Among
    1500 random 24-key leaves, the ones the GPU stores above 2^32 (below 1.6 * 2^32, to bound
    the oracle's time) are re-searched by the oracle from k = 0."""
    rng = np.random.default_rng(2432)
    m, nl = 24, 1500
    off = np.arange(nl + 1, dtype=np.uint32) * m
    lo = rng.integers(0, M64, size=nl * m, dtype=np.uint64, endpoint=True)
    isb = rng.integers(0, 2, size=nl * m, dtype=np.uint8)
    got = rs.search_leaves(lo, isb, off, rotation_fitting=True)
    big = [j for j in range(nl) if (1 << 32) <= int(got[j]) < int(1.6 * (1 << 32))][:6]
    assert len(big) >= 3
    with ThreadPoolExecutor(len(big)) as ex:
        want = list(ex.map(lambda j: oracle.leaf_rf(lo[j * m:(j + 1) * m], isb[j * m:(j + 1) * m]), big))
    assert [int(got[j]) for j in big] == want


@pytest.mark.parametrize("leaf", [2, 3, 5, 8, 12, 16, 19, 20, 24])
def test_split_search_parity(leaf):
    """Every split class the oracle can finish in seconds: L1 full/partial, L2
    full/partial, upper (fanout 2), and the 64-bit packed-counter path (l >= 19)."""
    _, _, u1, u2 = oracle.shape(leaf)
    rng = np.random.default_rng(leaf)
    cands = {leaf + 1, 2 * leaf + 1, 3 * leaf, 5 * leaf, 7 * leaf + 1, 8 * leaf, u1 - 1, u1, u1 + 1,
             2 * u1 + 1, 3 * u1, u2 - 1, u2, u2 + 3, 2 * u2 + 1, 3 * u2 + 7}
    sizes = []
    for s in sorted(cands):
        if s <= leaf or s > 8192:
            continue
        work = s / oracle.split_prob(leaf, s)  # expected oracle remix evaluations
        if work <= 3e8:
            sizes += [s] * (6 if work < 1e7 else 2)
    rng.shuffle(sizes)
    off = np.zeros(len(sizes) + 1, dtype=np.uint32)
    off[1:] = np.cumsum(sizes)
    lo = rng.integers(0, M64, size=int(off[-1]), dtype=np.uint64, endpoint=True)
    got = rs.search_splits(lo, off, leaf)
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        want = list(ex.map(lambda j: oracle.find_split(leaf, lo[off[j]:off[j + 1]]), range(len(sizes))))
    assert got.tolist() == want


def _near_carry_keys(rng, n):
    """Keys whose low 32 bits lie within 2^12 of 2^32: remix(lo + sigma) carries into the
    high word for tiny seeds, so the searches start on the carry path and then rebase the
    buffered keys once the window start passes the carry boundary."""
    hi = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    low = np.uint64(0xFFFFFFFF) - rng.integers(0, 1 << 12, size=n, dtype=np.uint64)
    return (hi << np.uint64(32)) | low


@pytest.mark.parametrize("leaf", [5, 8, 16, 20])
def test_carry_and_rebase_paths(leaf):
    """Splits (lower and upper) and leaves (rotation fitting and brute force) over keys next
    to the carry boundary equal the oracle's values."""
    _, _, u1, u2 = oracle.shape(leaf)
    rng = np.random.default_rng(77 + leaf)
    sizes = [s for s in (leaf + 1, u1, u1 + 1, u2, 2 * u2 + 1)
             if s / oracle.split_prob(leaf, s) <= 3e8]
    sizes = sizes * 3
    off = np.zeros(len(sizes) + 1, dtype=np.uint32)
    off[1:] = np.cumsum(sizes)
    lo = _near_carry_keys(rng, int(off[-1]))
    got = rs.search_splits(lo, off, leaf)
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        want = list(ex.map(lambda j: oracle.find_split(leaf, lo[off[j]:off[j + 1]]), range(len(sizes))))
    assert got.tolist() == want
    m = min(leaf, 14)
    lsz = [m, m - 1, 2, m] * 8
    loff = np.zeros(len(lsz) + 1, dtype=np.uint32)
    loff[1:] = np.cumsum(lsz)
    llo = _near_carry_keys(rng, int(loff[-1]))
    isb = rng.integers(0, 2, size=int(loff[-1]), dtype=np.uint8)
    sl = [(int(loff[j]), int(loff[j + 1])) for j in range(len(lsz))]
    got = rs.search_leaves(llo, isb, loff, rotation_fitting=True)
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        want = list(ex.map(lambda ab: oracle.leaf_rf(llo[ab[0]:ab[1]], isb[ab[0]:ab[1]]), sl))
    assert got.tolist() == want
    bsz = [min(m, 10), 7, 3] * 6
    boff = np.zeros(len(bsz) + 1, dtype=np.uint32)
    boff[1:] = np.cumsum(bsz)
    blo = _near_carry_keys(rng, int(boff[-1]))
    got = rs.search_leaves(blo, np.zeros(len(blo), np.uint8), boff, rotation_fitting=False)
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        want = list(ex.map(lambda j: oracle.leaf_bf(blo[boff[j]:boff[j + 1]]), range(len(bsz))))
    assert got.tolist() == want


# ------------------------------------------------------------------- end to end --

def _check_full(keys, leaf, b, rf=True, threads=None):
    threads = threads or os.cpu_count()
    want, want_vals = oracle.build(keys, leaf, b, rf=rf, threads=threads, values=True)
    got, vals = rs.build_values(keys, leaf, b, rotation_fitting=rf)
    if not np.array_equal(vals, want_vals):
        bad = np.flatnonzero(vals != want_vals)
        raise AssertionError(f"{len(bad)} node values differ, first at slot {bad[0]}: "
                             f"gpu {vals[bad[0]]} oracle {want_vals[bad[0]]}")
    assert got == want
    return got


def test_c1_full_parity_and_bijective():
    cfg = synth.CONFIGS["C1"]
    keys = synth.keys(cfg["n"], cfg["seed"])
    blob = _check_full(keys, cfg["leaf"], cfg["bucket"])
    q = rs.query_many(blob, keys)
    assert np.array_equal(np.sort(q), np.arange(len(keys), dtype=np.uint64))
    assert rs.build(keys[::-1].copy(), cfg["leaf"], cfg["bucket"]) == blob  # key order invariance


@pytest.mark.parametrize("leaf,b,rf,n", [
    (2, 7, True, 5000), (3, 1, True, 2000), (4, 3, False, 4000), (5, 5, True, 20000), (6, 50, True, 20000),
    (7, 30, True, 20000), (8, 100, False, 20000), (10, 64, True, 20000), (11, 500, True, 20000),
    (12, 1000, True, 30000), (13, 200, True, 6000), (14, 2000, True, 8000), (16, 2000, True, 6000),
    (16, 40, True, 4000), (18, 300, True, 2000), (20, 100, True, 600), (24, 24, True, 200),
    (8, 7000, True, 21000), (8, 100, True, 1), (8, 100, True, 2), (16, 100, True, 17), (9, 9, True, 99),
])
def test_small_configs_full_parity(leaf, b, rf, n):
    keys = synth.keys(n, 1000 * leaf + b)
    blob = _check_full(keys, leaf, b, rf=rf)
    q = rs.query_many(blob, keys)
    assert np.array_equal(np.sort(q), np.arange(n, dtype=np.uint64))


def test_duplicate_keys_rejected():
    keys = synth.keys(5000, 9)
    keys[77] = keys[4000]
    with pytest.raises(rs.RecSplitError) as e:
        rs.build(keys, 8, 100)
    assert e.value.code == rs.E_DUPLICATE


@pytest.mark.parametrize("leaf,b,n", [(8, 100, 30_000), (12, 1000, 40_000), (16, 2000, 20_000)])
def test_duplicate_check_paths(leaf, b, n):
    """The duplicate check in each partition path (fused into the two-level sort for size bounds
    <= 512, the separate pass above): a repeated key anywhere is rejected, also in a replayed
    build; the one key whose lo word is 0 (lo = remix(key ^ salt), remix(0) = 0: key = the salt)
    is an ordinary key once -- bytes equal the oracle's -- and a duplicate twice."""
    salt_lo = np.uint64(0xC2B2AE3D27D4EB4F)
    keys = synth.keys(n, 70 + leaf)
    keys = keys[keys != salt_lo]
    keys[n // 3] = salt_lo
    want = oracle.build(keys, leaf, b, threads=os.cpu_count())
    for _ in range(3):  # (uncaptured, captured, replayed)
        assert rs.build(keys, leaf, b) == want
    for i, j in [(5, n // 2), (5, n // 3)]:  # (a plain repeat; the lo == 0 key twice)
        bad = keys.copy()
        bad[i] = bad[j]
        for _ in range(2):
            with pytest.raises(rs.RecSplitError) as e:
                rs.build(bad, leaf, b)
            assert e.value.code == rs.E_DUPLICATE


@pytest.mark.parametrize("leaf,b,n", [(8, 20_000, 30_000), (16, 12_000, 30_000), (5, 9_000, 60_000),
                                      (12, 10_000, 25_000), (3, 8_500, 17_000)])
def test_oversized_buckets_full_parity(leaf, b, n):
    """any bucket_size >= 1.  Buckets above the warp engine's 8192-key
    shared-memory capacity run their upper splits, redistribution and duplicate check
    through the global-memory path; bytes equal the oracle's."""
    keys = synth.keys(n, 500 + leaf)
    got, st = rs.build(keys, leaf, b, stats=True)
    assert st["max_bucket"] > 8192
    assert got == oracle.build(keys, leaf, b, threads=os.cpu_count())


def test_oversized_bucket_duplicates_rejected():
    keys = synth.keys(30_000, 19)
    keys[12345] = keys[23456]
    with pytest.raises(rs.RecSplitError) as e:
        rs.build(keys, 8, 20_000)
    assert e.value.code == rs.E_DUPLICATE


def test_bucket_cap_enforced():
    """Buckets above recsplit_max_bucket_keys() = 65536 keys are rejected (the per-size
    templates, include/recsplit.h); 68000 keys in one bucket."""
    keys = synth.keys(68_000, 3)
    with pytest.raises(rs.RecSplitError) as e:
        rs.build(keys, 8, 70_000)
    assert e.value.code == rs.E_INVALID


def test_one_enqueue_fallback_on_oversized_bucket():
    """The one-enqueue single-shard path sizes its tables for buckets up to n/B + 8 sqrt(n/B)
    + 32 keys; a bucket beyond that (here 400 keys at b = 100, chosen through the oracle's
    master hash) is flagged on the device and the build reruns on the synchronized path --
    the bytes still equal the oracle's."""
    rng = np.random.default_rng(77)
    n, b = 4000, 100
    B = (n + b - 1) // b
    cand = rng.integers(0, M64, size=200_000, dtype=np.uint64, endpoint=True)
    hi, _ = _mhc_np(cand)
    bucket = ((hi >> np.uint64(32)) * np.uint64(B)) >> np.uint64(32)
    in0 = np.unique(cand[bucket == 0])[:400]
    rest = np.unique(cand[bucket != 0])[:n - 400]
    keys = np.concatenate([in0, rest])
    assert len(np.unique(keys)) == n
    got, st = rs.build(keys, 8, b, stats=True)
    assert st["max_bucket"] == 400
    assert got == oracle.build(keys, 8, b, threads=os.cpu_count())


def test_bucket_tree_mode_bytes():
    """The whole-bucket kernel (k_bucket_tree, RS_BUCKET_TREE=1; off by default) in a fresh
    process: C1 and small configurations (incl. odd leaf sizes, one-key buckets, upper splits,
    a duplicate) give the oracle's bytes / E_DUPLICATE."""
    import subprocess
    import sys
    code = """
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2212_09562_b200 as rs, oracle, synth
for leaf, b, n in [(8, 100, 10000), (5, 5, 20000), (7, 200, 30000), (2, 3, 5000), (9, 300, 40000), (8, 100, 1)]:
    k = synth.keys(n, 40 + leaf)
    blob, st = rs.build(k, leaf, b, stats=True)
    assert st["t_search_tree"] > 0, (leaf, b)
    assert blob == oracle.build(k, leaf, b, threads=4), (leaf, b, n)
k = synth.keys(5000, 3); k[10] = k[4000]
try:
    rs.build(k, 8, 100)
    raise SystemExit("duplicate not detected")
except rs.RecSplitError as e:
    assert e.code == rs.E_DUPLICATE
print("ok")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RS_BUCKET_TREE="1"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_device_entry_matches_host_entry():
    """Device-pointer and host-pointer entries give the same bytes; the no-copy result views
    (pinned result buffers released with recsplit_free when collected) hold the same bytes."""
    import gc

    import torch
    keys = synth.keys(50000, 21)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    ref = rs.build(keys, 12, 500)
    assert rs.build_device(kt, 12, 500) == ref
    for _ in range(3):  # buffers are recycled through the pinned pool
        v = rs.build_device(kt, 12, 500, copy=False)
        w = rs.build(keys, 12, 500, copy=False)
        assert v.tobytes() == ref and w.tobytes() == ref and not v.flags.writeable
        del v, w
        gc.collect()


@pytest.mark.slow
def test_c2_full_parity():
    """C2 at full size (n=5e6, l=8, b=100): every byte equals the oracle."""
    cfg = synth.CONFIGS["C2"]
    keys = synth.keys(cfg["n"], cfg["seed"])
    blob = _check_full(keys, cfg["leaf"], cfg["bucket"])
    q = rs.query_many(blob, keys)
    assert np.array_equal(np.sort(q), np.arange(len(keys), dtype=np.uint64))
    bpk = rs.bits_per_key(blob)
    assert abs(bpk - 1.806) < 0.02, bpk  # paper P:828 (SIMDRecSplit l=8, b=100)


def _subtree_nodes(leaf):
    memo = {}

    def N(s):
        if s == 0:
            return 0
        if s not in memo:
            memo[s] = 1 + sum(N(c) for c in oracle.parts(leaf, s))
        return memo[s]
    return N


@pytest.mark.slow
@pytest.mark.parametrize("name,bits,tol", [("C3", 1.560, 0.004), ("C5", 1.6208, 0.004)])
def test_full_size_sampled_bucket_parity_and_properties(name, bits, tol):
    """C3 (n=5e6, l=16, b=2000) and C5 (n=1e8, l=12, b=1000) at full size, as bench.py
    builds them: the values of sampled buckets (incl. the largest) equal the oracle's, the
    MPHF is bijective (GPU query + GPU bijectivity check), bits/object matches the paper
    (C3: 1.560) or the survey's model of this format (C5: 1.6208)."""
    import torch
    cfg = synth.CONFIGS[name]
    keys = synth.keys(cfg["n"], cfg["seed"])
    leaf, b = cfg["leaf"], cfg["bucket"]
    blob, vals = rs.build_values(keys, leaf, b)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    assert rs.check_bijective_device(rs.query_device(blob, kt)) == 0
    del kt
    bpk = rs.bits_per_key(blob)
    assert abs(bpk - bits) < tol, bpk
    hi, _ = _mhc_np(keys)
    B = (len(keys) + b - 1) // b
    bucket = ((hi >> np.uint64(32)) * np.uint64(B)) >> np.uint64(32)
    sizes = np.bincount(bucket.astype(np.int64), minlength=B)
    N = _subtree_nodes(leaf)
    nb = np.concatenate([[0], np.cumsum([N(int(s)) for s in sizes])])
    assert nb[-1] == len(vals)
    rng = np.random.default_rng(0)
    sample = sorted(rng.choice(B, size=min(B, 16), replace=False).tolist())  # fixed count, any host
    sample[0] = int(np.argmax(sizes))  # include the largest bucket
    order = np.argsort(bucket, kind="stable")
    starts = np.concatenate([[0], np.cumsum(sizes)])

    def one(i):
        ks = keys[order[starts[i]:starts[i + 1]]]
        return i, oracle.bucket_values(ks, leaf)

    with ThreadPoolExecutor(len(sample)) as ex:
        for i, want in ex.map(one, sample):
            assert vals[nb[i]:nb[i + 1]].tolist() == want.tolist(), f"bucket {i}"


def _golden_digests():
    out = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_digests.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                w = line.split()
                out[w[0]] = dict(n=int(w[1]), leaf=int(w[2]), bucket=int(w[3]), rf=bool(int(w[4])),
                                 seed=int(w[5]), size=int(w[6]), bits=float(w[7]), sha=w[8])
    return out


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C3", "C5", "BIGB"])
def test_full_size_bytes_equal_oracle_digest(name):
    """The north_star target: the full-size MPHF (C3: n=5e6, l=16, b=2000) is byte-identical
    to the CPU oracle's.  The expected SHA-256 / size / bits per object were written by
    tools/oracle_digest.py, which calls only oracle/ (tests/golden/oracle_digests.txt); the
    GPU build goes through the C ABI with host keys (recsplit_build_ex), in the launch
    configuration bench.py's e2e leg times; then bijective (GPU query)."""
    import hashlib

    import torch
    d = _golden_digests().get(name)
    if d is None:
        pytest.skip(f"no oracle digest for {name}")
    keys = synth.keys(d["n"], d["seed"])
    blob = rs.build(keys, d["leaf"], d["bucket"], rotation_fitting=d["rf"])
    assert len(blob) == d["size"]
    assert hashlib.sha256(blob).hexdigest() == d["sha"]
    assert abs(rs.bits_per_key(blob) - d["bits"]) < 1e-6
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    assert rs.check_bijective_device(rs.query_device(blob, kt)) == 0


@pytest.mark.slow
@pytest.mark.parametrize("name,world", [("C3", 8), ("C5", 8)])
def test_routed_8_ranks_equal_oracle_digest(name, world):
    """SURVEY 8(e) at the BASELINE multi-GPU shapes (C3 at 8 B200, C5 at 8): 8 simulated ranks
    each start from 1/8 of the input, sum their bucket histograms (balanced cuts), route
    (recsplit_route_keys), exchange locally, build their shards and stitch -- the bytes equal
    the oracle's digest (tests/golden/oracle_digests.txt)."""
    import hashlib

    import torch
    d = _golden_digests().get(name)
    if d is None:
        pytest.skip(f"no oracle digest for {name}")
    n, leaf, b = d["n"], d["leaf"], d["bucket"]
    keys = synth.keys(n, d["seed"])
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    del keys
    sl = [kt[r * n // world:(r + 1) * n // world] for r in range(world)]
    hist = sum(rs.bucket_histogram(x, n, b).cpu().numpy().astype(np.int64) for x in sl)
    cuts = rs.balanced_cuts(hist, leaf, world)
    routed = [rs.route_keys(x, n, b, world, cuts=cuts) for x in sl]
    del sl, kt
    parts = []
    shards = []
    for dst in range(world):
        segs = []
        for src in range(world):
            out, cnt = routed[src]
            st = sum(cnt[:dst])
            segs.append(out[st:st + cnt[dst]])
        shards.append(rs.Shard(torch.cat(segs).contiguous(), leaf, b, dst, world, total_keys=n, cuts=cuts))
    allsum = np.stack([s.summary for s in shards])
    step = min(s.min_step(allsum) for s in shards)
    parts = [s.finish(step) for s in shards]
    for s in shards:
        s.close()
    blob = rs.stitch(parts)
    assert len(blob) == d["size"] and hashlib.sha256(blob).hexdigest() == d["sha"]


# ------------------------------------------------------------------ sharding --

@pytest.mark.parametrize("shards", [2, 3, 8, 150])
def test_virtual_shards_identical_bytes(shards):
    """bucket ranges per worker, concatenated sequences, one index: the
    sharded build (virtual shards on one GPU, same code as multi-GPU) is byte-identical
    to the unsharded build and to the oracle (150 shards > B = 100 -> empty shards)."""
    keys = synth.keys(10_000, 1)
    ref = oracle.build(keys, 8, 100, threads=os.cpu_count())
    assert rs.build(keys, 8, 100, virtual_shards=shards) == ref


@pytest.mark.parametrize("world", [2, 5, 8])
def test_balanced_cuts_identical_bytes(world):
    """SURVEY 8(e) work-balanced ranges: the bucket histogram kernel equals the host count, and
    virtual shards cut at recsplit_balanced_cuts -- and at degenerate cuts with empty ranks --
    give the oracle's bytes (the output never depends on where the ranges are cut)."""
    import torch
    keys = synth.keys(60_000, 13)
    leaf, b = 12, 1000
    B = (len(keys) + b - 1) // b
    hi, _ = _mhc_np(keys)
    want_hist = np.bincount((((hi >> np.uint64(32)) * np.uint64(B)) >> np.uint64(32)).astype(np.int64), minlength=B)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    hist = rs.bucket_histogram(kt, len(keys), b).cpu().numpy()
    assert np.array_equal(hist, want_hist)
    ref = oracle.build(keys, leaf, b, threads=os.cpu_count())
    cuts = rs.balanced_cuts(hist, leaf, world)
    assert rs.build(keys, leaf, b, virtual_shards=world, cuts=cuts) == ref
    skew = np.array([0] + [0] * (world - 2) + [3, B], dtype=np.uint64)  # empty ranks, then a tiny one
    assert rs.build(keys, leaf, b, virtual_shards=world, cuts=skew) == ref


def test_shard_protocol_in_process():
    """The multi-GPU ABI protocol (begin / allgather / min step / allreduce / finish /
    stitch) run for world = 3 in one process with a local exchange."""
    import torch
    keys = synth.keys(60_000, 4)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    world = 3
    shards = [rs.Shard(kt, 12, 1000, r, world) for r in range(world)]
    allsum = np.stack([s.summary for s in shards])
    step = min(s.min_step(allsum) for s in shards)
    parts = [s.finish(step) for s in shards]
    for s in shards:
        s.close()
    assert rs.stitch(parts) == rs.build(keys, 12, 1000) == oracle.build(keys, 12, 1000, threads=os.cpu_count())


@pytest.mark.parametrize("n,leaf,b,world", [(60_000, 12, 1000, 3), (200_000, 8, 100, 5), (50, 8, 100, 3),
                                            (7_000, 16, 2000, 8)])
@pytest.mark.parametrize("balanced", [False, True])
def test_routed_shard_protocol_in_process(n, leaf, b, world, balanced):
    """SURVEY 8(e)(ii) in one process: each simulated rank routes its slice of the input
    (recsplit_route_keys), a local all-to-all hands every rank exactly its keys, the shards
    run with total_keys = n; the stitched bytes equal the single-GPU build (and the
    oracle's).  (50 keys, b = 100: one bucket, so two of three ranks own nothing.)  balanced:
    the ranges come from the summed per-rank histograms and recsplit_balanced_cuts."""
    import torch
    keys = synth.keys(n, 5 + world)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    sl = [kt[r * n // world:(r + 1) * n // world] for r in range(world)]
    cuts = None
    if balanced:
        hist = sum(rs.bucket_histogram(x, n, b).cpu().numpy().astype(np.int64) for x in sl)
        cuts = rs.balanced_cuts(hist, leaf, world)
    routed = [rs.route_keys(x, n, b, world, cuts=cuts) for x in sl]
    owned = []
    for dst in range(world):
        segs = []
        for src in range(world):
            out, cnt = routed[src]
            st = sum(cnt[:dst])
            segs.append(out[st:st + cnt[dst]])
        owned.append(torch.cat(segs).contiguous())
    assert sum(o.numel() for o in owned) == n
    shards = [rs.Shard(owned[r], leaf, b, r, world, total_keys=n, cuts=cuts) for r in range(world)]
    allsum = np.stack([s.summary for s in shards])
    step = min(s.min_step(allsum) for s in shards)
    parts = [s.finish(step) for s in shards]
    for s in shards:
        s.close()
    blob = rs.stitch(parts)
    assert blob == rs.build(keys, leaf, b)
    if n <= 60_000:
        assert blob == oracle.build(keys, leaf, b, threads=os.cpu_count())


def test_misrouted_keys_rejected():
    """A shard given keys it does not own (total_keys set) fails the build's key count."""
    import torch
    keys = synth.keys(20_000, 9)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    world = 2
    shards = [rs.Shard(kt[: 10_000] if r == 0 else kt[10_000:], 8, 100, r, world, total_keys=20_000)
              for r in range(world)]
    allsum = np.stack([s.summary for s in shards])
    with pytest.raises(rs.RecSplitError) as e:
        shards[0].min_step(allsum)
    assert e.value.code == rs.E_INVALID
    for s in shards:
        s.close()


def _sharded_worker(rank, world, port, q, distribute=False):
    import sys as _sys
    _sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2212_09562_b200 as rs_
    import synth as synth_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both ranks on the one GPU; collectives over gloo
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = synth_.keys(200_000, 12)
        kt = torch.from_numpy(keys.view(np.int64)).cuda()
        if distribute:  # each rank starts from its own half of the input
            kt = kt[rank * 100_000:(rank + 1) * 100_000].contiguous()
        blob = rs_.build_sharded(kt, 12, 1000, distribute=distribute)
        if rank == 0:
            q.put(blob == rs_.build(keys, 12, 1000))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("distribute", [False, True])
def test_build_sharded_two_ranks_gloo(distribute):
    """build_sharded over torch.distributed (2 ranks on one GPU, gloo collectives), with
    every rank holding all keys or with routed slices (all-to-all): same bytes as the
    single-GPU build."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000 + 7 * distribute
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, distribute)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _nccl_worker(port, q):
    import sys as _sys
    _sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2212_09562_b200 as rs_
    import synth as synth_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        keys = synth_.keys(150_000, 13)
        kt = torch.from_numpy(keys.view(np.int64)).cuda()
        want = rs_.build(keys, 12, 1000)
        ok = [rs_.build_sharded(kt, 12, 1000, distribute=d) == want for d in (False, True)]
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_build_sharded_nccl_single_rank():
    """The NCCL code path of build_sharded (device tensors in all_reduce, all_to_all_single,
    all_gather_into_tensor, as bench.py uses at N > 1) on a one-rank NCCL group: same bytes as
    the single-GPU build, with and without key routing."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31700 + os.getpid() % 1000
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    p.join(600)
    assert p.exitcode == 0
    assert q.get(timeout=10) == [True, True]


# -------------------------------------------------------------- device query --

@pytest.mark.parametrize("leaf,b,rf,n", [(8, 100, True, 10_000), (16, 2000, True, 20_000), (5, 5, False, 20_000),
                                          (24, 24, True, 200), (12, 1000, True, 300_000)])
def test_query_device_matches_host_and_oracle(leaf, b, rf, n):
    """the GPU batched query equals the host query (and the oracle's on
    the oracle's bytes), is a bijection on S and stays in [0, n) for non-members."""
    import torch
    keys = synth.keys(n, 77 + leaf)
    blob = oracle.build(keys, leaf, b, rf=rf, threads=os.cpu_count()) if n <= 20_000 else rs.build(keys, leaf, b)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    got = rs.query_device(blob, kt).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, rs.query_many(blob, keys))
    assert np.array_equal(got, oracle.query_many(blob, keys))  # the oracle's own query
    assert np.array_equal(np.sort(got), np.arange(n, dtype=np.uint64))
    other = torch.from_numpy(synth.keys(5000, 991).view(np.int64)).cuda()
    assert (rs.query_device(blob, other).cpu().numpy().view(np.uint64) < n).all()


def test_device_handle_and_bijectivity_check():
    """recsplit_open(device 0): the resident copy answers like the per-call query on two
    streams; recsplit_check_bijective_device finds 0 violations on S's results and counts
    every injected repeat / out-of-range value."""
    import torch
    n = 200_000
    keys = synth.keys(n, 4242)
    blob = rs.build(keys, 12, 1000)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    want = rs.query_device(blob, kt)
    with rs.Handle(blob, device=0) as h:
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        a = h.query_device(kt, stream=s1)
        b = h.query_device(kt[: n // 2], stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(a, want) and torch.equal(b, want[: n // 2])
        assert np.array_equal(h.query_many(keys[:1000]), want[:1000].cpu().numpy().view(np.uint64))
    assert rs.check_bijective_device(want) == 0
    bad = want.clone()
    bad[5] = bad[6]        # one repeat
    bad[7] = n             # out of range
    bad[8] = -1            # 2^64 - 1: out of range
    assert rs.check_bijective_device(bad) == 3
    assert rs.check_bijective_device(torch.zeros(0, dtype=torch.int64, device="cuda")) == 0


# --------------------------------------------------------------- string keys --

@pytest.mark.parametrize("leaf,b,n", [(8, 100, 20_000), (16, 2000, 8_000), (5, 5, 10_000), (12, 1000, 30_000)])
def test_string_keys_full_parity(leaf, b, n):
    """strings of length 10..50: GPU bytes == oracle bytes, bijective."""
    data, off = synth.strings(n, leaf * 13 + b)
    want = oracle.build_strings(data, off, leaf, b, threads=os.cpu_count())
    got = rs.build_strings(data, off, leaf, b)
    assert got == want
    q = rs.query_strings(got, data, off)
    assert np.array_equal(np.sort(q), np.arange(n, dtype=np.uint64))


def test_string_keys_duplicate_rejected():
    data, off = synth.strings(3000, 5)
    d2 = np.concatenate([data, data[off[10]:off[11]]])
    o2 = np.concatenate([off, [off[-1] + (off[11] - off[10])]]).astype(np.uint64)
    with pytest.raises(rs.RecSplitError) as e:
        rs.build_strings(d2, o2, 8, 100)
    assert e.value.code == rs.E_DUPLICATE


# ------------------------------------------------------- early-rejection knob --

_CP_SNIPPET = """
import hashlib, sys
sys.path.insert(0, {root!r})
import paper_2212_09562_b200 as rs, synth
for leaf, b, n in {cases!r}:
    keys = synth.keys(n, 1000 * leaf + b)
    print(hashlib.sha256(rs.build(keys, leaf, b)).hexdigest())
"""


@pytest.mark.parametrize("cp", ["0:0:0:0:0", "100:100:1:0:0", "990:990:1:0:0", "500:0:0:0:0", "0:700:1:0:0",
                                "850:940:1:0:0", "100:100:1:200:300", "300:500:1:990:990", "780:940:1:880:0:0",
                                "780:940:1:880:0:1", "750:900:1:860:950:1", "780:940:1:880:0:1:0", "780:940:1:880:0:1:1:0"])
def test_early_rejection_checkpoints_do_not_change_output(cp):
    """The lower-level early rejection may only skip seeds that cannot succeed:
    the bytes equal the oracle's with it off, at degenerate checkpoints (almost no keys /
    almost all keys before the test, i.e. a queue that fills on every iteration), with it on
    for one level only (RS_CP1 / RS_CP2, per mille of u1 / u2), as a single stage and as a
    two-stage cascade (second checkpoints RS_CP1B / RS_CP2B, early, late and the defaults),
    with the last-part test off / on (RS_CPLAST) and the leaf early rejection off / on
    (RS_CPL, with the leaves' second checkpoint RS_CPL2 on, and off in the last case);
    small-node (batch-mode) phases keep the split rejection (RS_CP_BATCH=1) except where the
    seventh field is 0, the shipped default."""
    import hashlib
    import subprocess
    import sys
    cases = [(16, 2000, 6000), (12, 1000, 30000), (8, 100, 20000), (5, 5, 20000), (20, 100, 600)]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    v = cp.split(":")
    env = dict(os.environ, RS_CP1=v[0], RS_CP2=v[1], RS_CPL=v[2], RS_CP1B=v[3], RS_CP2B=v[4],
               RS_CPLAST=v[5] if len(v) > 5 else "1", RS_CP_BATCH=v[6] if len(v) > 6 else "1",
               RS_CPL2=v[7] if len(v) > 7 else "1")
    out = subprocess.run([sys.executable, "-c", _CP_SNIPPET.format(root=root, cases=cases)], env=env,
                         capture_output=True, text=True, timeout=600, check=True).stdout.split()
    want = [hashlib.sha256(oracle.build(synth.keys(n, 1000 * leaf + b), leaf, b, threads=os.cpu_count()))
            .hexdigest() for leaf, b, n in cases]
    assert out == want


_GRAPH_SNIPPET = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2212_09562_b200 as rs, oracle, synth
def want(k, leaf, b):
    return oracle.build(k, leaf, b, threads=8)
def dev(k):
    return torch.from_numpy(k.view(np.int64).copy()).cuda()
def pinned(k):
    t = torch.from_numpy(k.view(np.int64).copy()).pin_memory()
    return t, t.numpy().view(np.uint64)
n, leaf, b = 30000, 8, 100
k1, k2 = synth.keys(n, 501), synth.keys(n, 502)
w1, w2 = want(k1, leaf, b), want(k2, leaf, b)
d1, d2 = dev(k1), dev(k2)
for i in range(4):  # uncaptured, capture + replay, replays
    blob, st = rs.build_device(d1, leaf, b, stats=True)
    assert blob == w1, ("device replay", i)
    assert st["t_search"][2] > 0 and st["kernel_launches"] > 10, st
assert rs.build_device(d2, leaf, b) == w2, "replay with other device keys"
assert rs.build_device(d1, leaf, b) == w1
# host (pinned) keys: the chunked H2D is part of the graph; sources updated per replay
t1, p1 = pinned(k1)
t2, p2 = pinned(k2)
for i in range(3):
    assert rs.build(p1, leaf, b) == w1, ("host replay", i)
assert rs.build(p2, leaf, b) == w2, "host replay with other keys"
# another configuration in between (different per-size tables): the plan is recaptured
k3 = synth.keys(20000, 503)
for i in range(3):
    assert rs.build_device(dev(k3), 12, 300) == want(k3, 12, 300), ("other config", i)
assert rs.build_device(d1, leaf, b) == w1, "after table change"
assert rs.build_device(d2, leaf, b) == w2
# a duplicate inside a replay, then a clean replay
kd = k2.copy(); kd[7] = kd[20000]
try:
    rs.build_device(dev(kd), leaf, b)
    raise SystemExit("duplicate not detected")
except rs.RecSplitError as e:
    assert e.code == rs.E_DUPLICATE
assert rs.build_device(d1, leaf, b) == w1, "after duplicate"
# recsplit_trim: the cached graphs, workspaces and pool memory go back; builds recapture
big = synth.keys(2_000_000, 504)
dbig = dev(big)
for i in range(3):
    rs.build_device(dbig, 12, 1000)
torch.cuda.synchronize()
free0 = torch.cuda.mem_get_info()[0]
rs.trim()
free1 = torch.cuda.mem_get_info()[0]
assert free1 > free0 + (16 << 20), (free0, free1)
for i in range(3):
    assert rs.build_device(d1, leaf, b) == w1, ("after trim", i)
print("ok")
"""


def test_graph_replay_bytes():
    """CUDA-graph replay of the one-enqueue build (pipeline.cu, RS_GRAPH default on): the
    first build of a configuration runs uncaptured, the second captures, later ones replay
    with the key source patched into the graph.  Every replay gives the oracle's bytes for
    ITS keys (device keys and pinned host keys, other key sets of the same configuration,
    after another configuration replaced the per-size tables, after a duplicate-key
    rejection)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _GRAPH_SNIPPET.format(root=root)], env=dict(os.environ, RS_GRAPH="1"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


_KNOB_SNIPPET = """
import hashlib, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2212_09562_b200 as rs, synth
for leaf, b, n, rf in {cases!r}:
    keys = synth.keys(n, 7000 + 10 * leaf + b)
    print(hashlib.sha256(rs.build(keys, leaf, b, rotation_fitting=rf)).hexdigest())
rng = np.random.default_rng(5)
for rf in (True, False):
    sizes = rng.integers(1, 9, size=3000).astype(np.uint32)
    off = np.zeros(len(sizes) + 1, dtype=np.uint32); off[1:] = np.cumsum(sizes)
    lo = rng.integers(0, 2**64 - 1, size=int(off[-1]), dtype=np.uint64, endpoint=True)
    isb = rng.integers(0, 2, size=int(off[-1]), dtype=np.uint8)
    v = np.asarray(rs.search_leaves(lo, isb, off, rotation_fitting=rf), dtype=np.uint64)
    print(hashlib.sha256(v.tobytes() + lo.tobytes() + isb.tobytes() + off.tobytes()).hexdigest())
"""


@pytest.mark.parametrize("env", ["RS_SUB_LEAF=1", "RS_FIT_LUT=0", "RS_LEAN=0", "RS_P2=0", "RS_GRAPH=0",
                                 "RS_SUB_LEAF=1,RS_FIT_LUT=0", "RS_UPPER_KP=0", "RS_UPPER_KP_VAR=100000",
                                 "RS_FUSED_DEDUPE=0"])
def test_engine_knobs_do_not_change_output(env):
    """Every engine variant of round 2's small-configuration work gives the oracle's bytes:
    the sub-warp leaf kernel (k_leaf_sub: four leaves of <= 8 keys per warp, prefetched),
    the rotation-fit table off (serial rotation check), lean windows off, the one-level
    partition instead of the two-level counting sort, no CUDA graphs, upper splits all as
    windows / all keys-parallel up to 256 keys -- on configurations
    with leaves of 1..8 keys (rotation fitting and brute force), upper splits and ragged
    buckets; plus kernel-level leaf searches against the oracle's leaf values."""
    import hashlib
    import subprocess
    import sys
    cases = [(8, 100, 20000, True), (5, 5, 20000, True), (7, 200, 30000, True), (4, 50, 8000, True),
             (8, 100, 20000, False), (3, 9, 5000, True), (12, 1000, 30000, True)]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    for kv in env.split(","):
        k, v = kv.split("=")
        e[k] = v
    out = subprocess.run([sys.executable, "-c", _KNOB_SNIPPET.format(root=root, cases=cases)], env=e,
                         capture_output=True, text=True, timeout=900, check=True).stdout.split()
    want = [hashlib.sha256(oracle.build(synth.keys(n, 7000 + 10 * leaf + b), leaf, b, rf=rf,
                                        threads=os.cpu_count())).hexdigest() for leaf, b, n, rf in cases]
    assert out[:len(cases)] == want
    rng = np.random.default_rng(5)
    for i, rf in enumerate((True, False)):
        sizes = rng.integers(1, 9, size=3000).astype(np.uint32)
        off = np.zeros(len(sizes) + 1, dtype=np.uint32)
        off[1:] = np.cumsum(sizes)
        lo = rng.integers(0, 2**64 - 1, size=int(off[-1]), dtype=np.uint64, endpoint=True)
        isb = rng.integers(0, 2, size=int(off[-1]), dtype=np.uint8)
        vals = np.array([oracle.leaf_rf(lo[off[j]:off[j + 1]], isb[off[j]:off[j + 1]]) if rf else
                         oracle.leaf_bf(lo[off[j]:off[j + 1]]) for j in range(len(sizes))], dtype=np.uint64)
        assert out[len(cases) + i] == hashlib.sha256(vals.tobytes() + lo.tobytes() + isb.tobytes() +
                                                     off.tobytes()).hexdigest(), rf
