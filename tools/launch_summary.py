"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel count, time, share."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").split("<")[0]
        v = float(r[14].replace(",", ""))
        if r[13] == "usecond":
            v *= 1e3
        elif r[13] == "msecond":
            v *= 1e6
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    lines = ["kernel launches total_us share"]
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        lines.append(f"{k} {cnt[k]} {v / 1e3:.1f} {v / total * 100:.1f}%")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
