"""Dev tool: spill instructions inside the sample loops of a kernel's SASS.

For every backward branch whose range [target, branch] contains a TLD4 (or an
8-load trilinear footprint), count the instructions and the LDL/STL in that
range.  Usage: python tools/sass_loop.py lib.so kernel_substring
"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr:
                body = ins[addr[tgt]:i + 1]
                if any("TLD4" in x or "TEX" in x for _, x in body):
                    loops.append((tgt, a, body))
    print(name[:90])
    for tgt, a, body in sorted(loops, key=lambda l: len(l[2])):
        n = len(body)
        sp = sum(1 for _, x in body if re.search(r"\b(LDL|STL)\b", x))
        tld = sum(1 for _, x in body if "TLD4" in x)
        print(f"  loop {tgt:#x}-{a:#x}: {n} instr, {sp} LDL/STL, {tld} TLD4")
