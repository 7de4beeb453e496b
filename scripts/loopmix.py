"""Instruction mix of the step loop of one epoch-kernel instantiation.
   python scripts/loopmix.py <mangled-substring> [lib]"""
import re, subprocess, sys
from collections import Counter
key = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2604_12902_b200/_lib/libraspvisor_b200.so"
names = subprocess.run(["cuobjdump", "-symbols", lib], capture_output=True, text=True).stdout
fn = [w for w in re.findall(r"(_ZN4rasp12epoch_kernel\S+)", names) if key in w][0]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for l in sass.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), re.sub(r"\s+", " ", m.group(2)).strip()))
ALU = {"ISETP", "LOP3", "SEL", "PLOP3", "VIADD", "IADD3", "SHF", "LEA", "PRMT", "VIADDMNMX", "IMNMX", "P2R", "R2P"}
best = None
for a, t in ins:
    m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
        nlds = sum(1 for x in body if "LDS" in x[1])
        nldg = sum(1 for x in body if "LDG" in x[1])
        if any("VOTE" in x[1] for x in body) and nlds >= 16 and nldg <= nlds:
            if best is None or len(body) < len(best):
                best = body
c = Counter((x[1].split()[1] if x[1].startswith("@") else x[1].split()[0]).split(".")[0] for x in best)
steps = sum(1 for x in best if x[1].split()[-1].startswith("[") and "LDS" in x[1]) // 4
alu = sum(v for k, v in c.items() if k in ALU)
print(fn[:70], "body", len(best), "instrs; LDS/4 =", steps, "steps; ALU", alu, "=", round(alu / max(steps, 1), 2), "/step;",
      "total", round(len(best) / max(steps, 1), 2), "/step")
print(sorted(c.items()))
