"""Aggregate an ncu --page source --csv --print-source=cuda,sass export per CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, ix, out = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Name":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ix = {}
        for i, h in enumerate(r):
            ix.setdefault(h, i)
        continue
    if ix is None:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue

    def f(k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (KeyError, ValueError, IndexError):
            return 0.0
    out.append((cur_file or "?", ln, r[1][:100], f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"),
                f("stall_barrier"), f("L1 Wavefronts Shared Excessive")))
tot_i = sum(o[3] for o in out) or 1
tot_s = sum(o[4] for o in out) or 1
print("tot inst %.3e  samples %.0f" % (tot_i, tot_s))
for o in sorted(out, key=lambda x: -x[4])[:topn]:
    print(f"{o[0][:16]:16s}:{o[1]:4d} inst {o[3]/tot_i*100:5.1f}% stall {o[4]/tot_s*100:5.1f}% bar {o[5]/tot_s*100:4.1f}% "
          f"xs {o[6]:8.0f} | {o[2]}")
