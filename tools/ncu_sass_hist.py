#!/usr/bin/env python
"""Opcode histogram and hot regions of one kernel from `ncu -i rep --page source --csv --print-source sass > src.csv`:
    python tools/ncu_sass_hist.py src.csv [kernel-index]"""
import csv
import sys
from collections import Counter


def main(path, which=1):
    rows = list(csv.reader(open(path)))
    out, k = [], 0
    for r in rows:
        if r and r[0] == "Kernel Name":
            k += 1
            continue
        if k == which and len(r) > 6 and r[0].startswith('0x'):
            out.append(r)
    tot = sum(int(r[5]) for r in out)
    print(len(out), "SASS lines, warp instructions executed:", tot)
    c, s = Counter(), Counter()
    for r in out:
        toks = r[1].split()
        op = toks[1] if toks[0].startswith('@') else toks[0]
        c[op] += int(r[5])
        s[op] += int(r[2])
    for op, v in c.most_common(28):
        print("  %-22s %10d %5.1f%%  samples %d" % (op, v, 100 * v / tot, s[op]))
    prev, start, runs = None, 0, []
    for i, r in enumerate(out):
        cnt = int(r[5])
        if prev is None or abs(cnt - prev) > 0.02 * max(cnt, prev):
            if prev is not None:
                runs.append((start, i - 1, prev))
            start = i
        prev = cnt
    runs.append((start, len(out) - 1, prev))
    print("regions (first line, last line, instructions, executions each, share, stall samples):")
    for a, b, cnt in runs:
        n = b - a + 1
        if n * cnt > 0.01 * tot:
            print("  %5d %5d %4d %9d %5.1f%% %6d" % (a, b, n, cnt, 100 * n * cnt / tot, sum(int(out[i][2]) for i in range(a, b + 1))))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
