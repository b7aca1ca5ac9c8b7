"""Inner-loop SASS statistics for one kernel of liblmshoot_b200.so (run here; no GPU needed).
usage: python scripts/sass_loop.py <mangled-name-substring> [--dump]"""
import collections
import re
import subprocess
import sys

so = "paper_1907_04839_b200/liblmshoot_b200.so"
pat = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
blocks = out.split("Function : ")
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for l in b.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    best = None
    for addr, txt in ins:
        if "BRA" in txt:
            m2 = re.search(r"0x([0-9a-f]+)", txt)
            if m2:
                tgt = int(m2.group(1), 16)
                if tgt < addr:
                    body = [t for a, t in ins if tgt <= a <= addr]
                    nm = sum("MUFU.EX2" in t for t in body) or sum(t.split()[0] == "DSETP" or "DSETP" in t for t in body)
                    if nm and (best is None or len(body) < len(best[3])):
                        best = (nm, tgt, addr, body)
    print(name)
    if not best:
        print("  no MUFU loop found")
        continue
    nm, tgt, addr, body = best
    c = collections.Counter()
    for t in body:
        toks = t.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += 1
    print(f"  loop {tgt:#x}..{addr:#x}: {len(body)} instrs, {nm} MUFU.EX2 -> {len(body)/nm:.2f} instrs/pair")
    print("  ", c.most_common())
    if "--dump" in sys.argv:
        for t in body:
            print("     ", t)
