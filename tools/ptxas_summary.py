"""Summarise paper_2302_12249_b200/build/ptxas.log: kernel -> registers, stack, spills, smem."""
import os
import re
import sys

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2302_12249_b200", "build", "ptxas.log")


def parse(path=LOG):
    out = {}
    cur = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            dm = re.match(r"_ZN4merf\d+(\w+?)ILi(\d+)E", cur)
            cur = f"{dm.group(1)}<{dm.group(2)}>" if dm else cur
            out[cur] = {}
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            out[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers.*?(?:, (\d+) bytes smem)?$", line.strip())
        if m and "registers" in line:
            out[cur].update(regs=int(m.group(1)), smem=int(m.group(2) or 0))
    return out


if __name__ == "__main__":
    for k, v in sorted(parse(sys.argv[1] if len(sys.argv) > 1 else LOG).items()):
        print(f"{k:40s} {v}")
