"""Register / spill summary of nvcc -Xptxas -v logs:  python tools/spills.py build/obj/keyswitch.o.log [REGEX]"""
import re
import sys

pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        st, ld = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if pat is None or pat.search(name):
            print(f"{name[:70]:70s} regs={m.group(1)} spill_st={st} spill_ld={ld}")
        name = None
