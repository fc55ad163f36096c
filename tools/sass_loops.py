"""List the innermost loops (backward branches) of one kernel in a cuobjdump -sass dump."""
import re
import sys


def kernel_lines(path, fn):
    out, on = [], False
    for l in open(path):
        if "Function : " in l:
            on = fn in l
            continue
        if on:
            out.append(l.rstrip())
    return out


def loops(lines):
    at, ins = {}, []
    for l in lines:
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            at[int(m.group(1), 16)] = len(ins)
            ins.append(m.group(2).strip())
    res = []
    for i, s in enumerate(ins):
        m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", s)
        if m and int(m.group(1), 16) in at and at[int(m.group(1), 16)] <= i:
            res.append((at[int(m.group(1), 16)], i))
    return ins, res


if __name__ == "__main__":
    path, fn = sys.argv[1], sys.argv[2]
    maxlen = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    ins, res = loops(kernel_lines(path, fn))
    for a, b in res:
        if b - a <= maxlen:
            body = ins[a:b + 1]
            kinds = {}
            for s in body:
                op = s.split()[0] if not s.startswith("@") else s.split()[1]
                op = op.split(".")[0]
                kinds[op] = kinds.get(op, 0) + 1
            print(a, b, b - a + 1, sorted(kinds.items(), key=lambda x: -x[1])[:12])
