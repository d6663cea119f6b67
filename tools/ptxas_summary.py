"""Registers / spills per kernel from the build's ptxas log (csrc/ptxas.log).
  python tools/ptxas_summary.py [filter-substring]"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
log = open(__file__.rsplit("/", 2)[0] + "/paper_2202_13926_b200/csrc/ptxas.log").read().split("\n")
cur, seen = None, set()
spill = ""
for ln in log:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur, spill = m.group(1), ""
    if "spill" in ln:
        spill = ln.strip()
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur and cur not in seen:
        seen.add(cur)
        dm = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        if flt in dm:
            sp = re.findall(r"(\d+) bytes spill stores, (\d+) bytes spill loads", spill)
            print(f"{m.group(1):>4} regs  spill st/ld {sp[0][0] if sp else '?'}/{sp[0][1] if sp else '?'}  {dm[:150]}")
