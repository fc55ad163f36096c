import sys; sys.path.insert(0,'/root/repo')
import numpy as np, oracle, paper_2212_09562_b200 as rs
M64=(1<<64)-1
for leaf in (2,3,5,8):
    _,_,u1,u2 = oracle.shape(leaf)
    rng=np.random.default_rng(leaf)
    for s in sorted({leaf+1, 2*leaf+1, u1-1, u1, u1+1, u2, u2+3, 2*u2+1}):
        if s<=leaf: continue
        lo = rng.integers(0, M64, size=s*4, dtype=np.uint64, endpoint=True)
        off = np.arange(0, 4*s+1, s, dtype=np.uint32)
        got = rs.search_splits(lo, off, leaf).tolist()
        want = [oracle.find_split(leaf, lo[off[j]:off[j+1]]) for j in range(4)]
        print(leaf, s, 'OK' if got==want else 'BAD', got, want)
