#!/usr/bin/env python
"""Static SASS opcode histogram of the RK4 stage-kernel variants in libsfv.so
(cuobjdump -sass), with the Blackwell evidence opcodes (UTMALDG = TMA tensor
loads, SYNCS = mbarrier, no UTC*MMA: no tensor cores on this path).
    python scripts/sass_histogram.py [LIB] > profiles/r2_sass_histogram.md"""
import re
import subprocess
import sys
from collections import Counter

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2305_18057_b200/libsfv.so"
KERNELS = {"_ZN3sfv12stage_kernelILi0ELb1ELb0ELb1ELb0ELb0EEEvNS_9StageArgsE": "stage 1 (M_OWN + norms)",
           "_ZN3sfv12stage_kernelILi1ELb0ELb0ELb1ELb0ELb0EEEvNS_9StageArgsE": "stages 2-3 (M_UN)",
           "_ZN3sfv12stage_kernelILi2ELb0ELb1ELb1ELb0ELb0EEEvNS_9StageArgsE": "stage 4 (M_RK4F + dt)"}
txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        funcs[cur][m.group(2)] += 1
ops = ["DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "MUFU", "FSEL", "IMAD", "LDS", "STS", "STG", "LDG", "SHFL",
       "UTMALDG", "SYNCS", "ELECT", "VOTE", "BRA", "UTCHMMA", "UTCQMMA", "UTCIMMA", "HMMA", "DMMA"]
print(f"# SASS opcode histogram (static instruction counts, cuobjdump -sass {LIB.split('/')[-1]})\n")
print("| kernel | " + " | ".join(ops) + " | total |")
print("|---" * (len(ops) + 2) + "|")
for k, name in KERNELS.items():
    c = funcs.get(k, Counter())
    print(f"| {name} | " + " | ".join(str(c.get(o, 0)) for o in ops) + f" | {sum(c.values())} |")
print("\nStatic counts include the rare paths (boundary ghosts, error reporting, prologue); the executed")
print("per-cell-stage mix is in profiles/r2a_stage_kernel_sass_hot.txt (ncu source page). UTMALDG = 2D TMA")
print("tensor loads (cp.async.bulk.tensor), SYNCS = mbarrier arrive/try-wait; no UTC*MMA / HMMA / DMMA: the")
print("path is an FP64 stencil without a dense contraction (tensor cores do not apply).")
