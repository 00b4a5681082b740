"""Dump SASS of one kernel with the decoded control fields (stall, yield, wbar, rbar, wait mask).

    python tools/sass_ctrl.py <lib.so> <function-substring> [start_hex end_hex]
"""
import re
import subprocess
import sys

so, pat = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi_ = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for chunk in sass.split("Function : ")[1:]:
    name = chunk.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    lines = chunk.split("\n")
    for i, l in enumerate(lines):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if not (lo <= addr <= hi_):
            continue
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        hw = int(m2.group(1), 16)
        stall, yld, wb, rb, wm = (hw >> 41) & 0xF, (hw >> 45) & 1, (hw >> 46) & 7, (hw >> 49) & 7, (hw >> 52) & 0x3F
        print(f"{addr:#07x} S{stall:2d} Y{yld} wb{wb} rb{rb} wm{wm:06b}  {m.group(2)[:80]}")
    break
