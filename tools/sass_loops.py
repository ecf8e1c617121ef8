"""Loop statistics of a kernel's SASS (cuobjdump -sass): for each function called from the kernel
and each backward branch inside it, the loop size and its instruction mix (FFMA2, SHFL, MOV,
LDL/STL spills, LDS). Usage: python tools/sass_loops.py <obj-or-so> <kernel-substring>"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
want = sys.argv[2]
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if want not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    idx = {a: i for i, (a, _) in enumerate(ins)}
    calls = sorted({int(m.group(1), 16) for _, t in ins for m in [re.search(r"CALL\.REL\.NOINC\s+0x([0-9a-f]+)", t)] if m})
    rets = [a for a, t in ins if t.startswith("RET")]
    print(name, "instructions:", len(ins))
    regions = [(ins[0][0], calls[0] if calls else ins[-1][0])] + [(c, min([r for r in rets if r > c], default=ins[-1][0])) for c in calls]
    for (c, end) in regions:
        if c not in idx or end not in idx:
            continue
        print(f"  region {hex(c)}..{hex(end)} size {idx[end] - idx[c] + 1}")
        for i in range(idx[c], idx[end] + 1):
            a, t = ins[i]
            m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
            if m and c <= int(m.group(1), 16) < a:
                b = ins[idx[int(m.group(1), 16)]:i + 1]
                def cnt(p):
                    return sum(x.split()[0].startswith(p) or (x.startswith("@") and len(x.split()) > 1 and x.split()[1].startswith(p)) for _, x in b)
                if len(b) > 40:
                    print(f"    loop {hex(int(m.group(1), 16))}..{hex(a)} n={len(b)} FFMA2={cnt('FFMA2')} FMUL2={cnt('FMUL2')} SHFL={cnt('SHFL')} "
                          f"MOV={cnt('MOV') + cnt('IMAD.MOV')} LDL={cnt('LDL')} STL={cnt('STL')} FSEL={cnt('FSEL')} LDS={cnt('LDS')} BRX={cnt('BRX')}")
