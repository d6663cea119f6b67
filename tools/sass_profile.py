"""Summarise an ncu `--page source --print-source sass --csv` export.

Usage: python tools/sass_profile.py sass.csv [chunk]
Prints samples and executed warp-instructions per contiguous address chunk with
the dominant opcodes and stall columns, plus the totals by opcode.
"""
import csv
import sys
from collections import Counter, defaultdict


def main():
    path = sys.argv[1]
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {n: i for i, n in enumerate(hdr)}
    data = rows[2:]
    stall_cols = [n for n in hdr if n.startswith("stall_") and "(" not in n]
    tot_s = sum(int(r[idx["# Samples"]]) for r in data)
    tot_e = sum(int(r[idx["Instructions Executed"]]) for r in data)
    print(f"total samples {tot_s}  executed warp-instr {tot_e}")
    byop = Counter()
    byop_s = Counter()
    for r in data:
        op = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[idx["Source"]].split()[1]
        op = op.split(".")[0]
        byop[op] += int(r[idx["Instructions Executed"]])
        byop_s[op] += int(r[idx["# Samples"]])
    print("by opcode (executed, samples):")
    for op, n in byop.most_common(30):
        print(f"  {op:10s} {n/tot_e*100:6.2f}%  {byop_s[op]/tot_s*100:6.2f}%")
    for c0 in range(0, len(data), chunk):
        part = data[c0:c0 + chunk]
        s = sum(int(r[idx["# Samples"]]) for r in part)
        e = sum(int(r[idx["Instructions Executed"]]) for r in part)
        if s < tot_s * 0.005 and e < tot_e * 0.005:
            continue
        ops = Counter()
        for r in part:
            t = r[idx["Source"]].split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += int(r[idx["Instructions Executed"]])
        st = defaultdict(int)
        for r in part:
            for n in stall_cols:
                st[n] += int(r[idx[n]] or 0)
        top = sorted(st.items(), key=lambda x: -x[1])[:4]
        print(f"[{c0:5d}] {part[0][idx['Address']][-5:]} samples {s/tot_s*100:5.1f}% exec {e/tot_e*100:5.1f}% "
              f"ops {','.join(f'{k}:{v*100//max(e,1)}' for k, v in ops.most_common(5))} "
              f"stalls {','.join(f'{k[6:]}:{v*100//max(s,1)}' for k, v in top)}")


if __name__ == "__main__":
    main()
