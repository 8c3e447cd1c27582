"""Summarise ptxas -v logs: kernel, registers, spills, stack (demangled)."""
import re, subprocess, sys, glob
for log in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "build/*.ptxas.log")):
    name = None
    spill = ""
    for line in open(log):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(anonymous namespace\)::", "", name)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = f"stack={m.group(1)} spill={m.group(2)}/{m.group(3)}"
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            print(f"{m.group(1):>4} regs {spill:28s} {name[:150]}")
            name, spill = None, ""
