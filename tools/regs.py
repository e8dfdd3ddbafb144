#!/usr/bin/env python
"""Compile one csrc/*.cu with -Xptxas -v and print (kernel, registers, spill bytes) compactly.
usage: python tools/regs.py tx.cu [regex]"""
import re, subprocess, sys
src = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
       "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", f"paper_2205_05158_b200/csrc/{src}", "-o", "/tmp/_regs.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name = None
rows = []
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = m.group(1)
        spill = None
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem)
        if not pat or pat.search(dem):
            rows.append((dem, int(m.group(1)), spill))
        name = None
for r in rows:
    print(f"{r[1]:4d} regs  spill {r[2]}  {r[0]}")
