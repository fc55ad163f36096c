"""World-size-2 gloo test of the sharded path's host logic (no GPU).

The parts of ranks 0 and 1 are cut out of an ORACLE-built MPHF with independently
written offset formulas, then run through the package's
torch.distributed orchestration (allgather of summaries, allreduce-min of the residual
step, gather of the parts) and the library's host stitcher and globals arithmetic; the
stitched bytes must equal the oracle's.
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bits_of(words, nbits):
    return np.unpackbits(np.asarray(words, dtype="<u8").view(np.uint8), bitorder="little")[:nbits]


def _words_of(bits):
    b = np.zeros(((len(bits) + 63) // 64) * 64, dtype=np.uint8)
    b[: len(bits)] = bits
    return np.packbits(b, bitorder="little").view("<u8")


def _parse(blob):
    g, n, B, D, dC, beta, dR = struct.unpack_from("<QQQQQQq", blob, 16)
    leaf, rf = blob[6], blob[7]
    (bucket,) = struct.unpack_from("<I", blob, 8)
    p = 72
    efs = []
    for _ in range(2):
        L = blob[p]
        (nl,) = struct.unpack_from("<Q", blob, p + 8)
        p += 16
        low = _bits_of(np.frombuffer(blob, "<u8", (nl + 63) // 64, p), nl)
        p += 8 * ((nl + 63) // 64)
        (nu,) = struct.unpack_from("<Q", blob, p)
        p += 8
        up = _bits_of(np.frombuffer(blob, "<u8", (nu + 63) // 64, p), nu)
        p += 8 * ((nu + 63) // 64)
        efs.append((L, low, up))
    data = _bits_of(np.frombuffer(blob, "<u8", (D + 63) // 64, p), D)
    return dict(leaf=leaf, rf=rf, bucket=bucket, g=g, n=n, B=B, D=D, dC=dC, beta=beta, dR=dR, efs=efs, data=data)


def _decode(L, up, k):
    ones = np.flatnonzero(up)[:k]
    return ones - np.arange(k)


def bucket_sizes(blob):
    """Bucket sizes C[i+1] - C[i] decoded from the EF index (independent reader)."""
    h = _parse(blob)
    B, dC = h["B"], h["dC"]
    L, low, up = h["efs"][0]
    hi = _decode(L, up, B + 1).astype(np.int64)
    lo = np.array([sum(int(low[i * L + t]) << t for t in range(L)) for i in range(B + 1)], dtype=np.int64)
    C = ((hi << L) | lo) + np.arange(B + 1) * dC
    return np.diff(C)


def make_parts(blob, world, cuts=None):
    """Cut the serialized MPHF into the parts the sharded pipeline would produce (rank r owns
    buckets [cuts[r], cuts[r+1]); default equal bucket counts)."""
    h = _parse(blob)
    n, B, D, dC, beta, dR = h["n"], h["B"], h["D"], h["dC"], h["beta"], h["dR"]
    (LC, cl, cu), (LP, pl, pu) = h["efs"]

    def values(L, low, up):
        hi = _decode(L, up, B + 1)
        lo = np.array([sum(int(low[i * L + t]) << t for t in range(L)) for i in range(B + 1)], dtype=np.int64)
        return (hi.astype(np.int64) << L) | lo

    Cp, Pp = values(LC, cl, cu), values(LP, pl, pu)
    C = [int(Cp[i]) + i * dC for i in range(B + 1)]
    P = [int(Pp[i]) + i * dR + ((beta * C[i]) >> 20) for i in range(B + 1)]
    parts, summaries, steps = [], [], []
    for r in range(world):
        b0, b1 = (B * r // world, B * (r + 1) // world) if cuts is None else (int(cuts[r]), int(cuts[r + 1]))
        last = r == world - 1
        cnt = b1 - b0 + (1 if last else 0)
        sizes = [C[i + 1] - C[i] for i in range(b0, b1)]
        summaries.append([C[b1] - C[b0], P[b1] - P[b0], min(sizes) if sizes else 2 ** 64 - 1, b0, b1, 0, 0, 0])
        R = lambda i: P[i] - ((beta * C[i]) >> 20)  # noqa: E731
        steps.append(min([R(i + 1) - R(i) for i in range(b0, b1)], default=2 ** 63 - 1))
        Cq = lambda i: C[i] - i * dC  # noqa: E731
        Pq = lambda i: R(i) - i * dR  # noqa: E731
        cu0 = (Cq(b0) >> LC) + b0
        pu0 = (Pq(b0) >> LP) + b0
        cu1 = len(cu) if last else (Cq(b1) >> LC) + b1
        pu1 = len(pu) if last else (Pq(b1) >> LP) + b1
        slices = [(P[b0], h["data"][P[b0]:P[b1]]), (b0 * LC, cl[b0 * LC:(b0 + cnt) * LC]), (cu0, cu[cu0:cu1]),
                  (b0 * LP, pl[b0 * LP:(b0 + cnt) * LP]), (pu0, pu[pu0:pu1])]
        out = bytearray(b"RSPT") + struct.pack("<I", 1)
        out += struct.pack("<16Q", h["leaf"], h["rf"], h["bucket"], h["g"], n, B, D, dC, beta, dR & (2 ** 64 - 1),
                           LC, LP, (B + 1) * LC, len(cu), (B + 1) * LP, len(pu))
        for start, bits in slices:
            out += struct.pack("<QQ", start, len(bits)) + _words_of(bits).tobytes()
        parts.append(bytes(out))
    return parts, np.array(summaries, dtype=np.uint64), steps, dR


def _worker(rank, world, port, blob, q, balanced=False):
    sys.path.insert(0, ROOT)
    import paper_2212_09562_b200 as rs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cuts = rs.balanced_cuts(bucket_sizes(blob), blob[6], world) if balanced else None
        parts, summaries, steps, dR = make_parts(blob, world, cuts)
        allsum = rs.exchange_summaries(summaries[rank])
        assert np.array_equal(allsum, summaries)
        g = rs.shard_globals(allsum, world, rank)
        assert g["key_base"] == int(summaries[:rank, 0].sum()) and g["bit_base"] == int(summaries[:rank, 1].sum())
        step = rs.allreduce_min(steps[rank])
        assert step == dR
        got = rs.gather_parts(parts[rank])
        if rank == 0:
            q.put(rs.stitch(got) == blob)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,balanced", [(2, False), (2, True)])
def test_gloo_sharded_exchange_and_stitch(world, balanced):
    sys.path.insert(0, ROOT)
    import oracle
    import synth

    keys = synth.keys(6000, 8)
    blob = oracle.build(keys, 8, 100, threads=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    port += 7 * balanced
    procs = [ctx.Process(target=_worker, args=(r, world, port, blob, q, balanced)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_stitch_single_part_roundtrip():
    """One shard: the part cut from a blob stitches back to the same blob."""
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2212_09562_b200 as rs
    import synth

    for leaf, b, n in [(8, 100, 3000), (5, 5, 2000), (12, 1000, 5000)]:
        blob = oracle.build(synth.keys(n, leaf + b), leaf, b, threads=2)
        for world in (1, 3):
            parts, summaries, _, _ = make_parts(blob, world)
            assert rs.stitch(parts) == blob
            for r in range(world):
                g = rs.shard_globals(summaries, world, r)
                assert g["n"] == n and g["D"] == int(summaries[:, 1].sum())


def _owner(key, B, world):
    """Rank owning key's bucket: bucket = remap(hi, B) from the
    oracle's master hash code; rank r owns [floor(rB/W), floor((r+1)B/W))."""
    import oracle
    b = oracle.remap(oracle.mhc(int(key))[0], B)
    return max(r for r in range(world) if (r * B) // world <= b)


def _route_worker(rank, world, port, slices, B, q):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2212_09562_b200 as rs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = slices[rank]
        owners = np.array([_owner(k, B, world) for k in mine], dtype=np.int64)
        order = np.argsort(owners, kind="stable")
        counts = np.bincount(owners, minlength=world).tolist()
        routed = torch.from_numpy(mine[order].view(np.int64).copy())
        got = rs.exchange_keys(routed, counts).numpy().view(np.uint64)
        q.put((rank, sorted(got.tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_key_exchange_delivers_owned_keys(world):
    """after the all-to-all every rank holds exactly the keys whose bucket
    it owns (host-side routing with the oracle's hash; the device routing kernel is tested
    against a single-GPU build in the GPU suite)."""
    sys.path.insert(0, ROOT)
    import synth

    keys = synth.keys(3000, 31 + world)
    B = (len(keys) + 99) // 100
    slices = [keys[r * len(keys) // world:(r + 1) * len(keys) // world] for r in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + world * 10 + os.getpid() % 500
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, slices, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        want = sorted(int(k) for k in keys if _owner(k, B, world) == r)
        assert res[r] == want


def _expected_evals_oracle(leaf, s, rf):
    """SURVEY 8(d) unit written out with the oracle's probabilities: s / p per split node,
    1/p per rotation-fitting leaf, m/p per brute-force leaf, over the subtree."""
    import oracle
    if s <= 1:
        return float(s)
    if s <= leaf:
        p = oracle.bij_prob(s, rf)
        return 1.0 / p if rf else s / p
    return s / oracle.split_prob(leaf, s) + sum(_expected_evals_oracle(leaf, c, rf) for c in oracle.parts(leaf, s))


@pytest.mark.parametrize("leaf,b,world", [(16, 2000, 8), (8, 100, 4), (12, 1000, 3), (5, 5, 8)])
def test_balanced_cuts_equalise_expected_work(leaf, b, world):
    """SURVEY 8(e) work-balanced bucket ranges: recsplit_balanced_cuts returns world + 1
    nondecreasing cuts from 0 to B, and every rank's expected work (computed here from the
    oracle's split / leaf probabilities) is within one bucket's work of the ideal share."""
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2212_09562_b200 as rs
    import synth

    n = 400 * b if b >= 100 else 4000
    keys = synth.keys(n, 3)
    B = (n + b - 1) // b
    hi = np.array([oracle.mhc(int(k))[0] for k in keys], dtype=np.uint64)
    bucket = ((hi >> np.uint64(32)) * np.uint64(B)) >> np.uint64(32)
    hist = np.bincount(bucket.astype(np.int64), minlength=B).astype(np.uint32)
    cuts = rs.balanced_cuts(hist, leaf, world)
    assert cuts[0] == 0 and cuts[-1] == B and (np.diff(cuts.astype(np.int64)) >= 0).all()
    memo = {}
    w = np.array([memo.setdefault(int(s), _expected_evals_oracle(leaf, int(s), True)) for s in hist])
    per = [w[cuts[r]:cuts[r + 1]].sum() for r in range(world)]
    ideal = w.sum() / world
    assert max(abs(x - ideal) for x in per) <= w.max() + 1e-6 * ideal
