"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin (demangled template args)."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.group(1)
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        name = re.sub(r"_ZN3rfr\d+", "", cur)
        print(f"{name:60s} regs {m2.group(1):>4s}  spill {spill}")
        cur = None
