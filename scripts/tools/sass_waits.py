"""Static scoreboard check of the step kernel's streaming loop: lists the
instructions between the first and last weight-stream load (LDG.E.NA.128 /
.64 / .32 with the evict-first cache hint) that WAIT on a scoreboard set by
one of those loads without reading its destination registers (false waits
that expose a load's full latency).
python scripts/tools/sass_waits.py [lib.so] [mangled-kernel-substring]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_14690_b200/lib/libteal_b200.so"
fn = sys.argv[2] if len(sys.argv) > 2 else "step_kernelILi1ELi2ELi6E"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
lines = out.split("\n")
ins = []
on = False
for i, ln in enumerate(lines):
    if "Function : " in ln:
        on = fn in ln
        continue
    if not on:
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", ln)
    if m and i + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        c = int(m2.group(1), 16) >> 41
        ins.append((int(m.group(1), 16), m.group(2).strip(), (c >> 5) & 7, (c >> 8) & 7, (c >> 11) & 63, c & 15))
loads = [k for k, x in enumerate(ins) if re.search(r"LDG\.E\.NA\.(128|64)?\.?CONSTANT|LDG\.E\.NA\.CONSTANT", x[1])]
if not loads:
    sys.exit("no streaming loads found")
a, b = loads[0], loads[-1] + 200
pending = {}  # scoreboard -> dest regs of the streaming load that set it
nfalse = 0
for k in range(a, min(b, len(ins))):
    addr, txt, wb, rb, wait, stall = ins[k]
    regs = set(re.findall(r"\bR(\d+)\b", txt.split(",", 1)[1] if "," in txt else ""))
    for sb in range(6):
        if wait >> sb & 1 and sb in pending:
            dst = pending.pop(sb)
            if not (dst & regs) and "LDG" not in txt:
                nfalse += 1
                print(f"{addr:#07x} waits SB{sb} (load -> R{sorted(dst)}) : {txt[:70]}")
    if k in loads and wb != 7:
        m = re.search(r"R(\d+),", txt)
        r0 = int(m.group(1))
        w = 4 if ".128" in txt else (2 if ".64" in txt else 1)
        pending.setdefault(wb, set()).update(str(r0 + j) for j in range(w))
print(f"{len(loads)} streaming loads, {nfalse} false waits")
