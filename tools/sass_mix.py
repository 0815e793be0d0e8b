"""Aggregate an ncu source-page SASS CSV by opcode: executed warp instructions and stall samples.

    python tools/sass_mix.py file_sass.csv [--top 30]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ex = defaultdict(float)
    samp = defaultdict(float)
    stall = defaultdict(lambda: defaultdict(float))
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    total_i = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = float(r[ix["Instructions Executed"]] or 0)
        ex[op] += n
        total_i += n
        samp[op] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        for h in scols:
            stall[op][h] += float(r[ix[h]] or 0)
    tot_s = sum(samp.values())
    print(f"total warp instructions {total_i:.0f}")
    for op, n in sorted(ex.items(), key=lambda t: -t[1])[:top]:
        top_st = sorted(stall[op].items(), key=lambda t: -t[1])[:3]
        st = " ".join(f"{h[6:]}={v / max(tot_s, 1) * 100:.1f}%" for h, v in top_st if v)
        print(f"{op:10s} {n / total_i * 100:6.2f}% inst  {samp[op] / max(tot_s, 1) * 100:6.2f}% samples  {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
