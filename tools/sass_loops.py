"""Print the instruction mix of every backward-branch loop of the kernels matching a pattern.

    python tools/sass_loops.py <lib.so> <function-substring>
"""
import re
import subprocess
import sys
from collections import Counter

so, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for chunk in sass.split("Function : ")[1:]:
    name = chunk.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for line in chunk.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    print(name, "instructions:", len(ins))
    for a, txt in ins:
        m = re.search(r"BRA(\.U)?\s+(!?U?P\d+,\s*)?`?\(?\.?L?_?x?_?(0x[0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(3), 16)
            if tgt < a:
                body = [t for (b, t) in ins if tgt <= b <= a]
                ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr", ops.most_common(14))
