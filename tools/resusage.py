"""Registers / stack of the library's kernels (cuobjdump -res-usage).

usage: python tools/resusage.py [PATTERN] [LIB]
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_1811_00778_b200", "libhcnn_b200.so")
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function ([^\s:]+):", out)),
                       capture_output=True, text=True).stdout.split("\n")
for name, m in zip(names, re.finditer(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", out)):
    short = re.sub(r"\(.*", "", name).replace("hcnn::", "")
    if pat in short:
        print(f"{short:70s} REG={m.group(1):>3} STACK={m.group(2):>4}")
