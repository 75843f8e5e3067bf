#!/usr/bin/env python
"""Summarise the `-Xptxas -v` logs of the last build: registers, stack and spills per kernel."""
import glob
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LOGS = os.path.join(HERE, "..", "paper_2108_07232_b200", "csrc", "build", "*.ptxas.log")
PAT = re.compile(
    r"Compiling entry function '(\S+)'.*?\n.*?\n\s*(\d+) bytes stack frame, (\d+) bytes spill stores.*?\n"
    r"ptxas info\s*: Used (\d+) registers"
)


def main(filt=""):
    for f in sorted(glob.glob(LOGS)):
        for m in PAT.finditer(open(f).read()):
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name).replace("void bht_b200::", "")
            if filt in name:
                print(f"{name:48s} regs={m.group(4):>3s} stack={m.group(2)} spill={m.group(3)}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
