"""Markdown table from a C4 sweep JSONL (tools/sweep.py c4).  Usage: python tools/sweep_table.py in.jsonl [title]"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
title = sys.argv[2] if len(sys.argv) > 2 else "C4 sweep"
by = {}
for r in rows:
    by.setdefault((r["bucket"], r["leaf"]), {})["rf" if r["leaves"] == "rotation fitting" else "bf"] = r
print(f"# {title}\n")
print("keys/s = n / device time of one recsplit_build_device (keys in HBM); bits = bits/object of the blob.\n")
print("| l | b | RF keys/s | RF bits | BF keys/s | BF bits | RF / BF |")
print("|---|---|---|---|---|---|---|")
for (b, l) in sorted(by):
    d = by[(b, l)]
    rf, bf = d.get("rf"), d.get("bf")
    ratio = f"{rf['keys_per_s'] / bf['keys_per_s']:.2f}" if rf and bf else "—"
    f = lambda x, k, fmt: (fmt % x[k]) if x else "—"
    print(f"| {l} | {b} | {f(rf, 'keys_per_s', '%.3e')} | {f(rf, 'bits_per_key', '%.4f')} | "
          f"{f(bf, 'keys_per_s', '%.3e')} | {f(bf, 'bits_per_key', '%.4f')} | {ratio} |")
