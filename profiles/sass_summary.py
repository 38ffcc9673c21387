"""Per-kernel SASS opcode counts of the built objects (cuobjdump -sass): the
tcgen05 / TMEM / TMA instructions that show the tensor-core kernels use them.
    python profiles/sass_summary.py > profiles/r2_sass_summary.md"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2303_08064_b200", "lib", "obj")
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "SYNCS", "F2FP", "MUFU", "HMMA", "FFMA", "DFMA"]
print("# SASS opcode counts per kernel (static, `cuobjdump -sass` of `paper_2303_08064_b200/lib/obj/*.o`)\n")
print("UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM = tcgen05.ld, UBLKCP = cp.async.bulk (TMA bulk copy),")
print("SYNCS = mbarrier ops, F2FP = packed f16/bf16 conversions, MUFU = SFU ops.\n")
print("| object | kernel | " + " | ".join(OPS) + " |")
print("|---|---|" + "---|" * len(OPS))
for f in sorted(os.listdir(OBJ)):
    if not f.endswith(".o") or f.startswith("nasg_api"):
        continue
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, f)], capture_output=True, text=True).stdout
    for block in re.split(r"\n\s+Function : ", out)[1:]:
        name = block.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem).replace("nasg::", "").replace("(anonymous namespace)::", "")
        counts = [len(re.findall(r"\b" + op + r"[.\s]", block)) for op in OPS]
        if sum(counts[:7]) == 0 and counts[-1] == 0 and counts[-3] < 50:
            continue
        print(f"| {f} | `{dem}` | " + " | ".join(str(c) for c in counts) + " |")
