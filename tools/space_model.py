"""Expected bits/object of the pinned format (R8-R15) per node class, for the l = 24 space
gap: Golomb-Rice length E = tau + 1 + Q/(1 - Q), Q = (1 - p)^(2^tau), with
the optimal tau, summed over each bucket tree and averaged over Poisson(b) bucket sizes;
fanout / split-point variants show the gap to the paper (1.496) is not a reading
of the tree shape.  Uses the oracle's probabilities (analysis only).

    python tools/space_model.py
"""
import sys, math
sys.path.insert(0,'/root/repo')
import oracle
from functools import lru_cache
from math import lgamma, log, exp

def golomb_len(p, tau):
    Q = (1-p)**(2**tau)
    return tau + 1 + Q/(1-Q)

def best_tau(p):
    best=None
    for t in range(0,63):
        L=golomb_len(p,t)
        if best is None or L < best[0]-1e-15: best=(L,t)
    return best

def mk(leaf, f1=None, f2=None, upper='R6'):
    F1 = f1 or max(2, -(-(35*leaf+55)//100))
    F2 = f2 or max(2, -(-(21*leaf+90)//100))
    u1 = F1*leaf; u2 = F2*u1
    def parts(s):
        if s <= leaf: return []
        if s <= u1: unit = leaf
        elif s <= u2: unit = u1
        else:
            if upper == 'R6': c0 = -(-(s//2)//u2)*u2
            elif upper == 'half': c0 = s//2
            return [c0, s-c0]
        f = -(-s//unit)
        return [unit]*(f-1) + [s-(f-1)*unit]
    def psplit(s):
        ps = parts(s)
        lp = lgamma(s+1) + sum(c*log(c/s) - lgamma(c+1) for c in ps)
        return exp(lp)
    @lru_cache(None)
    def bits(s, rf):
        if s == 0: return 0.0, {}
        if s == 1: return 1.0, {'leaf1': 1.0}
        if s <= leaf:
            p = oracle.bij_prob(s, rf)
            L,_ = best_tau(p)
            return L, {'leaf': L}
        p = psplit(s)
        L,_ = best_tau(p)
        cls = 'L1' if s <= u1 else ('L2' if s <= u2 else 'upper')
        tot = L; d = {cls: L}
        for c in parts(s):
            b, dd = bits(c, rf)
            tot += b
            for k,v in dd.items(): d[k] = d.get(k,0)+v
        return tot, d
    return bits, (F1,F2,u1,u2)

def expected(leaf, b, rf=True, **kw):
    bits, sh = mk(leaf, **kw)
    # Poisson(b) bucket sizes
    tot=0; cls={}
    lo=max(1,int(b-8*b**0.5)); hi=int(b+8*b**0.5)
    Z=0
    for s in range(lo,hi+1):
        w = exp(-b + s*log(b) - lgamma(s+1))
        Z+=w
        t,d = bits(s, rf)
        tot += w*t
        for k,v in d.items(): cls[k]=cls.get(k,0)+w*v
    return tot/b/Z, {k:v/b/Z for k,v in cls.items()}, sh

for leaf,b in [(16,2000),(24,2000)]:
    t,c,sh = expected(leaf,b)
    print(leaf,b,sh,round(t,4),{k:round(v,4) for k,v in c.items()})
print('--- l=24 variants (data bits/key)')
for f1 in (8,9,10,12):
    for f2 in (5,6,7,9):
        t,c,sh = expected(24,2000,f1=f1,f2=f2)
        print(f1,f2,sh,round(t,4))
t,c,sh=expected(24,2000,upper='half'); print('half', round(t,4))
t,c,sh=expected(24,2000,rf=False); print('BF', round(t,4))
