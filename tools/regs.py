"""Registers / spills per kernel from `python -m paper_2404_19429_b200.build --force -v` output on stdin."""
import re
import subprocess
import sys

name = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"lancet::(\(anonymous namespace\)::)?", "", name).split("(")[0]
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if len(sys.argv) < 2 or re.search(sys.argv[1], name):
            print(f"{int(m.group(1)):4d}  {name}")
        name = None
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and int(m.group(1)) > 0 and name:
        print("     SPILL", line.strip())
