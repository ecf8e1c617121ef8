"""Aggregate an `ncu --page source --csv --print-source=cuda,sass` export by file / line region.

Usage: python tools/ncu_regions.py src.csv [--lines N]
"""
import collections
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def load(path):
    rows = list(csv.reader(open(path)))
    cur, ix = None, None
    stall, inst = collections.Counter(), collections.Counter()
    src = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            ix = {h: i for i, h in reversed(list(enumerate(r)))}
            continue
        if ix is None:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        stall[(cur, ln)] += num(r[ix["Warp Stall Sampling (All Samples)"]])
        inst[(cur, ln)] += num(r[ix["Instructions Executed"]])
        src[(cur, ln)] = r[1][:90]
    return stall, inst, src


if __name__ == "__main__":
    stall, inst, src = load(sys.argv[1])
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 30
    ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
    byfile = collections.Counter()
    for (f, _), s in stall.items():
        byfile[f] += s
    for f, s in byfile.most_common():
        print(f"{f:28s} stall {100 * s / ts:5.1f}%")
    for k, s in stall.most_common(nlines):
        print(f"{k[0][:20]:20s}:{k[1]:4d} stall {100 * s / ts:5.1f}% inst {100 * inst[k] / ti:5.1f}% | {src[k]}")
