"""Summarise a `nvcc -Xptxas -v` log: kernel, registers, spill bytes.
    python tools/ptxas_regs.py LOG [name filter]"""
import re
import subprocess
import sys

t = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for m in re.finditer(r"Compiling entry function '(\S+)' for.*\n.*\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores.*\n.*Used (\d+) registers", t):
    name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
    name = name.replace("htlr::(anonymous namespace)::", "").replace("void ", "")
    name = re.sub(r"\(.*", "", name)
    if flt in name:
        print(f"{name:60s} regs {m.group(4):>4s} spill {m.group(3)}")
