"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck): C1 shape and the
l=16 shape at oracle size, byte-compared with the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402

# (n, leaf, b, seed, virtual shards): the one-enqueue path, the l = 16 / 12 shapes, a bucket above
# 8192 keys (block-per-node upper splits, global reorder staging, global dedupe tables) and the
# sharded path with work-balanced cuts
cases = [(10_000, 8, 100, 1, 0), (3_000, 16, 2000, 3, 0), (2_000, 12, 1000, 5, 0), (18_000, 8, 9_000, 11, 0),
         (12_000, 8, 100, 13, 3)]
if len(sys.argv) > 1 and sys.argv[1] == "c1":  # racecheck / synccheck: small shapes only
    cases = [(10_000, 8, 100, 1, 0), (2_000, 10, 200, 7, 0), (9_000, 5, 9_000, 11, 0), (3_000, 8, 100, 13, 3)]
for n, leaf, b, seed, shards in cases:
    keys = synth.keys(n, seed)
    cuts = None
    if shards:
        B = (n + b - 1) // b
        cuts = [0] + [B * (r + 1) // (shards + 1) for r in range(shards - 1)] + [B]  # uneven ranges
    want = oracle.build(keys, leaf, b, threads=os.cpu_count() or 1)
    # unsharded builds three times: uncaptured, captured + replayed, replayed (CUDA-graph path)
    for rep in range(1 if shards else 3):
        got = rs.build(keys, leaf, b, virtual_shards=shards, cuts=cuts)
        assert got == want, (n, leaf, b, rep)
    print("ok", n, leaf, b, shards, len(got))
