"""Local-memory traffic (LDL/STL) inside the DMMA loops of each mm_kernel instantiation:
cuobjdump -sass of the library, per kernel the count of LDL/STL instructions that lie
between the first and last DMMA of a loop body (a backward branch spanning DMMAs)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1605_01078_b200/libstrassen_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern = None
ins = {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        ins[kern] = []
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and kern:
        ins[kern].append((int(m.group(1), 16), m.group(2)))
for k, lst in ins.items():
    if "mm_kernel" not in k:
        continue
    addr2i = {a: i for i, (a, _) in enumerate(lst)}
    loops = []
    for i, (a, t) in enumerate(lst):
        m = re.search(r"BRA\S*\s+(?:\S+,\s*)?`?\(?\.?L?_?x?_?\d*\)?\s*(0x[0-9a-f]+)?", t)
        if t.startswith(("BRA", "@")) and "BRA" in t:
            mm = re.search(r"0x([0-9a-f]+)", t)
            if mm:
                tgt = int(mm.group(1), 16)
                if tgt in addr2i and addr2i[tgt] < i:
                    loops.append((addr2i[tgt], i))
    tot_dmma = sum(1 for _, t in lst if "DMMA" in t)
    hot = []
    for lo, hi in loops:
        body = lst[lo:hi + 1]
        nd = sum(1 for _, t in body if "DMMA" in t)
        if nd >= 32:
            nl = sum(1 for _, t in body if re.search(r"\b(LDL|STL)", t))
            hot.append((nd, nl, hi - lo + 1))
    name = re.sub(r"^_ZN5sb20012_GLOBAL__N__\w+?9mm_kernel", "mm_kernel", k)
    print(f"{name[-40:]}: DMMA {tot_dmma}, loops with DMMA (dmma, ldl/stl, instrs): {hot[:8]}")
