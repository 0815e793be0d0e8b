"""Top stall instructions from `ncu --page source --csv --print-source sass`:  python tools/sass_stalls.py FILE [N]"""
import csv
import sys
from collections import Counter


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    print("total samples", tot)
    by_op = Counter()
    by_reason = Counter()
    for r in data:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].strip().split()[1]
        by_op[op.split(".")[0]] += s
        for h in scols:
            by_reason[h] += int(r[ix[h]] or 0)
    print("by opcode:", ", ".join(f"{k}={v / tot * 100:.1f}%" for k, v in by_op.most_common(14)))
    print("by reason:", ", ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in by_reason.most_common(10)))
    data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:top]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        reasons = sorted(((int(r[ix[h]] or 0), h[6:]) for h in scols), reverse=True)[:3]
        print(f"{s / tot * 100:5.2f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} " +
              " ".join(f"{n}={v}" for v, n in reasons if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
