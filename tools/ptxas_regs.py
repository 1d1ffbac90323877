"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin (one line per entry)."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        sp = (m.group(1), m.group(2))
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = cur
        r = re.search(r"RDCfgILi(\d+)ELi(\d+)ELb([01])ELb([01])ELb([01])ELi(\d+)ELi(\d+)ELi(\d+)E", name)
        if r:
            name = "RD KS=%s NT=%s MODE1=%s SCALE=%s FAST=%s D=%s REMOTE=%s CS=%s" % r.groups()
        print(f"{m.group(1):>4} regs  spill st/ld {sp[0]}/{sp[1]}  {name[:150]}")
        cur = None
