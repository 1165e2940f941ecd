"""Summarise `nvcc -Xptxas -v` output (stdin): function -> registers, stack, spills."""
import re
import subprocess
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"(?:Compiling entry function|Function properties for) '?([\w]+)'?", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    n = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
    n = re.sub(r"\(.*", "", n)[:70]
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and (int(m.group(1)) or int(m.group(2))):
        print(f"{n:72s} stack {m.group(1)} spill st {m.group(2)} ld {m.group(3)}")
    m = re.search(r"Used (\d+) registers", line)
    if m:
        print(f"{n:72s} regs {m.group(1)}")
        cur = None
