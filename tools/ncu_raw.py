"""Key metrics + stall breakdown from an `ncu --page raw --csv` export (one row per launch)."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "dur_us"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("lts__t_bytes.sum", "l2_bytes"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("smsp__sass_inst_executed_op_local_ld.sum", "local_ld"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf")]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    units = rows[1]
    scols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    for r in rows[2:]:
        print(r[ix["Kernel Name"]][:60])
        print("  " + "  ".join(f"{s}={r[ix[k]]}{units[ix[k]] if k in ix and units[ix[k]] not in ('', '%') else ''}"
                               for k, s in KEYS if k in ix))
        tot = sum(float(r[ix[h]] or 0) for h in scols) or 1
        st = sorted(((float(r[ix[h]] or 0), h[34:]) for h in scols), reverse=True)[:8]
        print("  stalls: " + ", ".join(f"{n}={v / tot * 100:.0f}%" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
