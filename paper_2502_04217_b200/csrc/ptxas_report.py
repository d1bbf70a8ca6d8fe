"""Summarise `nvcc -Xptxas -v` output: registers / spills per kernel instantiation."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "fl_fastpass.cu"
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
       "--expt-relaxed-constexpr", "-I../../include", "-Xptxas", "-v", "-c", src, "-o", "/tmp/ptxas_report.o"]
if "fl_vec" in src:
    cmd.insert(3, "-fmad=false")
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        d = re.search(r"fast_passILi(\d+)ELb(\d)ELi(\d)ELb(\d)ELi(\d+)E", cur)
        mm = re.search(r"mirror_passILi(\d+)ELb(\d)ELi(\d)ELb(\d)ELi(\d+)E", cur)
        if mm:
            cur = f"mirror_pass<M={mm.group(1)},s={mm.group(2)},kind={mm.group(3)},epi={mm.group(4)},pipe={mm.group(5)}>"
        elif d:
            cur = f"fast_pass<M={d.group(1)},s={d.group(2)},kind={d.group(3)},epi={d.group(4)},cfg={d.group(5)}>"
        else:
            cur = re.sub(r"_ZN2fl\d+_GLOBAL__N__\w+?_\d+(\w+?)E.*", r"\1", cur)[:60]
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs {m.group(1):>4s}  {spill}")
        cur = None
