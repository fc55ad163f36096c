"""Write full-size oracle digests to tests/golden/oracle_digests.txt.

Calls only `oracle/` (and the seeded key generator `synth/`): the expected bytes of the
full-size configurations come from the plain CPU oracle, never from the CUDA path.  One
line per configuration:

    name n leaf bucket rf key_seed size_bytes bits_per_object sha256 cmd

Usage:  python tools/oracle_digest.py C3 [C5 ...] [--threads T]
Names:  C2, C3, C5 (synth.CONFIGS), N2 (n = 1e9, l = 8, b = 100, key seed 7,
        SURVEY 8(f) N2 / P:1029-1036), L24 is not a digest target (hours).
Re-running a name replaces its line.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "oracle_digests.txt")

TARGETS = dict(synth.CONFIGS)
TARGETS["N2"] = dict(n=1_000_000_000, leaf=8, bucket=100, seed=7)
TARGETS["C3BF"] = dict(n=5_000_000, leaf=16, bucket=2000, seed=3, rf=False)
TARGETS["BIGB"] = dict(n=200_000, leaf=8, bucket=20_000, seed=11)


def bits_per_object(blob: bytes) -> float:
    """(D + EF lower/upper bits)/n from the header fields (R14)."""
    n, B, D = struct.unpack_from("<QQQ", blob, 24)
    off = 72
    ef_bits = 0
    for _ in range(2):
        off += 8
        lowbits = struct.unpack_from("<Q", blob, off)[0]
        off += 8 + 8 * ((lowbits + 63) // 64)
        upbits = struct.unpack_from("<Q", blob, off)[0]
        off += 8 + 8 * ((upbits + 63) // 64)
        ef_bits += lowbits + upbits
    return (D + ef_bits) / n


def load() -> dict[str, str]:
    out = {}
    if os.path.exists(GOLDEN):
        for line in open(GOLDEN):
            if line.strip() and not line.startswith("#"):
                out[line.split()[0]] = line.rstrip("\n")
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    lines = load()
    for name in a.names:
        cfg = TARGETS[name]
        rf = cfg.get("rf", True)
        t0 = time.time()
        keys = synth.keys(cfg["n"], cfg["seed"])
        t1 = time.time()
        blob = oracle.build(keys, cfg["leaf"], cfg["bucket"], rf=rf, threads=a.threads)
        t2 = time.time()
        del keys
        dig = hashlib.sha256(blob).hexdigest()
        bpo = bits_per_object(blob)
        cmd = f"python tools/oracle_digest.py {name} --threads {a.threads}"
        lines[name] = (f"{name} {cfg['n']} {cfg['leaf']} {cfg['bucket']} {int(rf)} {cfg['seed']} "
                       f"{len(blob)} {bpo:.6f} {dig} # {cmd}; keys {t1 - t0:.0f} s, oracle {t2 - t1:.0f} s")
        print(lines[name], flush=True)
        with open(GOLDEN, "w") as f:
            f.write("# Full-size oracle digests (written by tools/oracle_digest.py, which calls only\n"
                    "# oracle/ and synth/).  name n leaf bucket rf key_seed size bits/object sha256\n")
            for k in sorted(lines):
                f.write(lines[k] + "\n")


if __name__ == "__main__":
    main()
