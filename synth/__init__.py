"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: keys come from numpy's PCG64 stream
(not SplitMix64, which is the method's own mixer), de-duplicated so every key
set is a valid MPHF input.  Workload shape follows the paper's "random 128-bit
integers as MHC" setup: uniform 64-bit keys, no structure or skew.
"""
from __future__ import annotations

import numpy as np


def keys(n: int, seed: int) -> np.ndarray:
    """n distinct uniform uint64 keys, deterministic in (n, seed)."""
    gen = np.random.Generator(np.random.PCG64(seed))
    raw = gen.bit_generator.random_raw(n)
    out = np.asarray(raw, dtype=np.uint64)
    while True:
        _, first = np.unique(out, return_index=True)
        if len(first) == len(out):
            return out
        first.sort()
        out = out[first]
        extra = np.asarray(gen.bit_generator.random_raw(n - len(out)), dtype=np.uint64)
        out = np.concatenate([out, extra])


def keys_device(n: int, seed: int):
    """n distinct uniform 64-bit keys generated on the current CUDA device (torch's Philox
    generator + unique), for scale runs whose key sets are too large to build on the host.
    Returns an int64 CUDA tensor (bit patterns).  Deterministic in (n, seed, torch build)."""
    import torch

    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    lo, hi = -(2 ** 63), 2 ** 63 - 1
    out = torch.randint(lo, hi, (n,), generator=gen, device="cuda", dtype=torch.int64)
    while True:
        u = torch.unique(out)
        if u.numel() == n:
            return out
        extra = torch.randint(lo, hi, (n - u.numel(),), generator=gen, device="cuda", dtype=torch.int64)
        out = torch.cat([u, extra])


def keys_device_counter(n: int, seed: int):
    """n DISTINCT uniform-looking 64-bit keys on the current CUDA device for any n (torch.unique
    is limited to 2^31 elements): key i = mix(seed * 2^40 + i) with mix a bijection of 64-bit
    words (xor-shift 32 / multiply by the odd constant 0xD6E8FEB86659FD93, twice) -- distinct
    inputs give distinct keys.  Not SplitMix64 nor MurmurHash3 (the method's own mixers, R1,
    R16).  Returns an int64 CUDA tensor (bit patterns)."""
    import torch

    M = 0xD6E8FEB86659FD93 - (1 << 64)  # as int64 (two's-complement multiply wraps mod 2^64)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    step = 1 << 28
    for a in range(0, n, step):
        b = min(n, a + step)
        x = torch.arange(a, b, dtype=torch.int64, device="cuda") + (seed << 40)
        for _ in range(2):
            x = x ^ ((x >> 32) & 0xFFFFFFFF)
            x = x * M
        x = x ^ ((x >> 32) & 0xFFFFFFFF)
        out[a:b] = x
    return out


def strings(n: int, seed: int, min_len: int = 10, max_len: int = 50):
    """n distinct random byte strings, lengths uniform in [min_len, max_len], bytes in
    1..255 (the paper's competitor workload: "strings of uniform random length in [10, 50]
    containing random characters except for the zero byte").  Returns (data uint8,
    offsets uint64 of n+1 entries).  Distinctness is checked for n <= 2e6 (collisions are
    astronomically unlikely: >= 255^10 strings per length)."""
    gen = np.random.Generator(np.random.PCG64(seed))
    lens = gen.integers(min_len, max_len + 1, size=n, dtype=np.int64)
    offsets = np.zeros(n + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum(lens)
    data = gen.integers(1, 256, size=int(offsets[-1]), dtype=np.uint8)
    if n <= 2_000_000:
        seen = {data[offsets[i]:offsets[i + 1]].tobytes() for i in range(n)}
        if len(seen) != n:
            raise RuntimeError("duplicate strings; choose another seed")
    return data, offsets


# Workload recipes (BASELINE.json configs); key seeds follow BASELINE.md section 4.
CONFIGS = {
    "C1": dict(n=10_000, leaf=8, bucket=100, seed=1),
    "C2": dict(n=5_000_000, leaf=8, bucket=100, seed=2),
    "C3": dict(n=5_000_000, leaf=16, bucket=2000, seed=3),
    "C5": dict(n=100_000_000, leaf=12, bucket=1000, seed=5),
}
