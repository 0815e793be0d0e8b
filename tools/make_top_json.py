"""Build profiles/ncu_top_kernel_CONFIG.json (read by bench.py for roofline.traffic and
compute_roofline) from `ncu --set full` raw-page CSVs of the top kernel's launches.

    python tools/make_top_json.py CONFIG KERNEL ALG_BYTES SOURCE raw1.csv [raw2.csv ...]

One bench-profiled launch of KERNEL may be several device launches (k_ks_modup_fused:
one per NTT engine); their DRAM bytes add up.  ALG_BYTES: the algorithmic bytes bench.py
declares for the captured launch (same formula as its PROF scope)."""
import csv
import json
import os
import sys

KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "launch__grid_size": "grid", "launch__registers_per_thread": "regs"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "second": 1}


def read(path):
    rows = list(csv.reader(open(path)))
    hdr, units, r = rows[0], rows[1], rows[2]
    ix = {h: i for i, h in enumerate(hdr)}
    out = {"name": r[ix["Kernel Name"]].split("(")[0]}
    for k, short in KEYS.items():
        if k in ix and r[ix[k]] not in ("", "n/a"):
            v = float(r[ix[k]].replace(",", ""))
            out[short] = v * SCALE.get(units[ix[k]], 1)
    return out


def main():
    config, kernel, alg, source, paths = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4], sys.argv[5:]
    parts = [read(p) for p in paths]
    dram = sum(p.get("dram_read", 0) + p.get("dram_write", 0) for p in parts)
    dur = sum(p.get("duration", 0) for p in parts)
    rec = {
        "dram_bytes_per_launch": dram,
        "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": round(dram / alg, 3),
        "duration_s": dur,
        "launches": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()} for p in parts],
        "source": source,
    }
    w = lambda key: round(sum(p.get(key, 0) * p.get("duration", 0) for p in parts) / max(dur, 1e-12), 2)  # noqa: E731
    for key in ("fp64_pipe_pct", "fma_pipe_pct", "alu_pipe_pct", "issue_active_pct"):
        rec[key] = w(key)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"ncu_top_kernel_{config}.json")
    with open(path, "w") as fh:
        json.dump({kernel: rec}, fh, indent=1)
    print(json.dumps({kernel: rec}, indent=1))


if __name__ == "__main__":
    main()
