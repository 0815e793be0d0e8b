"""Attribute ncu warp-stall samples to source lines.

    python tools/stall_lines.py NCU_SASS.csv KERNEL.sass [top]

NCU_SASS.csv: `ncu -i rep --page source --csv --print-source sass` of one kernel;
KERNEL.sass: `nvdisasm -g -c` text of the same function from the same build (the lines
`//## File "...", line N` give the innermost source line of the instructions after them;
`inlined at` lines give the call chain).  Instructions are matched by order.
"""
import csv
import re
import sys
from collections import defaultdict


def main(ncu_csv, sass, top=40):
    rows = list(csv.reader(open(ncu_csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    inst = [r for r in rows[2:] if len(r) >= len(hdr)]
    lines = []
    cur = ("?", 0)
    chain = []
    for ln in open(sass):
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
        if m:
            if "inlined at" in ln:
                chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            else:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                chain = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            lines.append((cur, tuple(chain), m.group(2).strip()))
    if len(lines) != len(inst):
        print(f"warning: {len(lines)} disassembled vs {len(inst)} profiled instructions", file=sys.stderr)
    scols = [h for h in hdr if h.startswith("stall_")]
    tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in inst) or 1
    by_line = defaultdict(float)
    by_outer = defaultdict(float)
    why = defaultdict(lambda: defaultdict(float))
    for (cur, chain, text), r in zip(lines, inst):
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        by_line[cur] += s
        outer = chain[-1] if chain else cur  # outermost frame = line in the kernel body
        by_outer[outer] += s
        for h in scols:
            why[outer][h[6:]] += float(r[ix[h]] or 0)
    print("== by outermost source line (kernel body) ==")
    for k, v in sorted(by_outer.items(), key=lambda t: -t[1])[:top]:
        w = sorted(why[k].items(), key=lambda t: -t[1])[:3]
        print(f"{v / tot * 100:6.2f}%  {k[0]}:{k[1]}   " + " ".join(f"{a}={b / tot * 100:.1f}%" for a, b in w if b))
    print("== by innermost source line ==")
    for k, v in sorted(by_line.items(), key=lambda t: -t[1])[:top]:
        print(f"{v / tot * 100:6.2f}%  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
