"""Counts the Blackwell-specific SASS instructions in the executor's kernels
(cuobjdump -sass of the built kernels.cu.o): TMA bulk copies (UBLKCP), mbarrier
ops (SYNCS), packed fp32 adds (FADD2), bf16 narrowing (F2FP), programmatic
dependent launch (PREEXIT = griddepcontrol.launch_dependents, ACQBULK =
griddepcontrol.wait).  Writes a markdown table (profiles/r02_sass_counts.md)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2504_20490_b200", "lib", "obj", "exec", "kernels.cu.o")
KEYS = ["UBLKCP", "SYNCS", "FADD2", "F2FP", "PREEXIT", "ACQBULK", "LDG", "STG", "FENCE"]

sass = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
counts, arch = collections.defaultdict(collections.Counter), set()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"arch = (sm_\w+)", line)
    if m:
        arch.add(m.group(1))
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and cur:
        counts[cur][m.group(1).split(".")[0]] += 1
names = {f: subprocess.run(["c++filt"], input=f, capture_output=True, text=True).stdout.strip() for f in counts}
out = ["# SASS instruction counts of the executor kernels", "",
       f"`cuobjdump -sass {os.path.relpath(OBJ, ROOT)}` (arch: {', '.join(sorted(arch)) or 'sm_100a'}), "
       "produced by `python tools/sass_counts.py`.", "",
       "| kernel | " + " | ".join(KEYS) + " |", "|---|" + "---|" * len(KEYS)]
for f in sorted(counts, key=lambda x: names[x]):
    n = names[f].replace("hshard::exec::(anonymous namespace)::", "").split("(")[0]
    if "tma" not in n and "expand" not in n and "box_phase_kernel" not in n:
        continue
    out.append(f"| `{n}` | " + " | ".join(str(counts[f][k]) for k in KEYS) + " |")
dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_sass_counts.md")
with open(dst, "w") as fh:
    fh.write("\n".join(out) + "\n")
print(dst)
