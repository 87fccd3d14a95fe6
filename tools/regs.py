#!/usr/bin/env python
"""Registers / local memory per search_kernel instantiation of an object or .so (cuobjdump)."""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "--dump-resource-usage", sys.argv[1]], capture_output=True, text=True).stdout
name = None
for ln in out.splitlines():
    m = re.search(r"Function (\S+):", ln)
    if m:
        name = m.group(1)
        continue
    r = re.search(r"REG:(\d+) STACK:(\d+).*LOCAL:(\d+)", ln)
    if r and name:
        k = re.search(r"search_kernelILi(\d)ELi(\d)ELi(\d+)ELi(\d)E", name)
        label = f"search S={k.group(1)} E={k.group(2)} CAP={k.group(3)} CPL={k.group(4)}" if k else name[:70]
        print(f"{label:50s} REG={r.group(1)} STACK={r.group(2)} LOCAL={r.group(3)}")
        name = None
