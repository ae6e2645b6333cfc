"""Blackwell-native evidence from the built library alone (no GPU): per kernel,
counts of the SASS opcodes that prove tcgen05 / TMEM / TMA use (UTCHMMA = tcgen05.mma,
LDTM / STTM = tcgen05.ld / st, UTMALDG / UTMASTG = TMA tensor load / store,
UBLKCP = TMA bulk copy, LDGSTS = cp.async, HMMA = legacy mma.sync).

    python scripts/sass_counts.py [paper_2512_17077_b200/libdllm.so] > profiles/r02_sass_opcodes.md
"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2512_17077_b200/libdllm.so"
ops = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKPF", "LDGSTS", "HMMA",
       "SYNCS", "MUFU.EX2", "ELECT"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern, counts, order = None, {}, []
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = {o: 0 for o in ops}
        order.append(kern)
        continue
    if kern is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m:
        op = m.group(1)
        for o in ops:
            if op == o or op.startswith(o + "."):
                counts[kern][o] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(order), capture_output=True, text=True).stdout.splitlines()
print(f"# SASS opcode counts of {lib} (cuobjdump -sass, sm_100a)\n")
print("| kernel | " + " | ".join(ops) + " |")
print("|---|" + "---|" * len(ops))
for k, d in zip(order, demangle):
    name = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", "")).replace("dllm::", "").replace("void ", "")
    print(f"| `{name}` | " + " | ".join(str(counts[k][o]) for o in ops) + " |")
