"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck): C1 shape and the
l=16 shape at oracle size, byte-compared with the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402

cases = [(10_000, 8, 100, 1), (3_000, 16, 2000, 3), (2_000, 12, 1000, 5)]
if len(sys.argv) > 1 and sys.argv[1] == "c1":  # racecheck / synccheck: the C1 shape only
    cases = [(10_000, 8, 100, 1), (2_000, 10, 200, 7)]
for n, leaf, b, seed in cases:
    keys = synth.keys(n, seed)
    got = rs.build(keys, leaf, b)
    assert got == oracle.build(keys, leaf, b, threads=os.cpu_count() or 1), (n, leaf, b)
    print("ok", n, leaf, b, len(got))
