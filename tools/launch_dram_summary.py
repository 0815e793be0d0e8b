"""Per-kernel duration and DRAM bytes from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv.

    python tools/launch_dram_summary.py launches.csv [bench.json] [out.txt]

Kernels are keyed by name plus template arguments (so the two engine launches of the fused
ModUp stay apart).  With a bench line (its `kernels` block: declared algorithmic GB/s x
event ms over `steps` steps) the measured / algorithmic byte ratio per launch is added for
every kernel name both lists hold."""
import csv
import json
import re
import sys
from collections import defaultdict

SCALE = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def key_of(name):
    name = name.replace("void ", "")
    m = re.match(r"([A-Za-z0-9_:]+)(<[^>(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name


def main(path, bench=None, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    per = defaultdict(lambda: defaultdict(float))
    launches = defaultdict(set)
    for r in rows:
        k = key_of(r[4])
        v = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
        per[k][r[12]] += v
        launches[k].add(r[0])
    algo = {}
    if bench:
        d = json.loads(open(bench).read().strip().splitlines()[-1])
        for k, x in d.get("kernels", {}).items():
            if x["launches"]:
                algo[k] = x["gbs"] * x["ms"] * 1e6 / x["launches"]  # declared bytes per launch
    total = sum(v["gpu__time_duration.sum"] for v in per.values()) or 1.0
    lines = ["kernel launches total_ms share dram_rd_MB/launch dram_wr_MB/launch dram_GB/s algorithmic_MB/launch measured/algorithmic"]
    base_sum = defaultdict(lambda: [0.0, 0])
    for k, v in per.items():
        b = k.split("<")[0]
        base_sum[b][0] += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        base_sum[b][1] += len(launches[k])
    for k, v in sorted(per.items(), key=lambda t: -t[1]["gpu__time_duration.sum"]):
        n = len(launches[k])
        t = v["gpu__time_duration.sum"]
        rd, wr = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"]
        b = k.split("<")[0]
        a = algo.get(b)
        ratio = ""
        if a:
            # engine-split kernels declare their bytes once per launch pair: compare the sum over instantiations
            inst = sum(1 for kk in per if kk.split("<")[0] == b)
            meas = base_sum[b][0] / (base_sum[b][1] / inst)
            ratio = f"{a / 1e6:.1f} {meas / a:.2f}"
        lines.append(f"{k} {n} {t / 1e6:.2f} {t / total * 100:.1f}% {rd / n / 1e6:.1f} {wr / n / 1e6:.1f} "
                     f"{(rd + wr) / t:.0f} {ratio}")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:4])
