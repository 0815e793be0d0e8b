"""Summarise an ncu report: per kernel launch, the key throughput/stall metrics."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur_ns"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64cyc%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local_ld"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    for r in data:
        name = r[ix["Kernel Name"]][:40]
        vals = []
        for key, short in KEYS:
            v = r[ix[key]] if key in ix else "n/a"
            vals.append(f"{short}={v}")
        print(name, " ".join(vals))
        st = sorted(((float(r[ix[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall_cols), reverse=True)[:6]
        tot = sum(float(r[ix[h]] or 0) for h in stall_cols) or 1
        print("   stalls:", ", ".join(f"{n}={100*v/tot:.0f}%" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
