# Fused-ModUp target-set sweep at one config:  bash tools/ts_sweep.sh TAG CONFIG "TS values" [extra env]
# per value: short bench line (value, ModUp ms); then DRAM bytes of the ModUp launches (ncu, 12 launches)
T=${1:-ts}; C=${2:-cfg4}; V=${3:-"1 2 4 6 99"}; X=${4:-NONE=0}
mkdir -p gpurun_out; : > gpurun_out/${T}_sweep.log
for ts in $V; do
  env HEB_MODUP_TS=$ts $X timeout 600 python bench.py --config $C --steps 3 --warmup 2 --skip-cpu --skip-cfg1 --skip-u64 \
      > gpurun_out/${T}_ts$ts.json 2> gpurun_out/${T}_ts$ts.err
  python - "$ts" "gpurun_out/${T}_ts$ts.json" >> gpurun_out/${T}_sweep.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print("TS", sys.argv[1], "failed", e); sys.exit(0)
print("TS", sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "check", d["check"]["argmax_identical"], d["check"]["max_abs_err_vs_plaintext"])
for k, x in list(d["kernels"].items())[:4]: print("   ", k, x)
PY
done
cat gpurun_out/${T}_sweep.log
for ts in ${5-4 99}; do
  env HEB_MODUP_TS=$ts $X timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k "regex:k_ks_modup_fused" -s 4 -c 8 --csv --log-file gpurun_out/${T}_ts${ts}_dram.csv \
      python bench.py --config $C --pipelines 1 --steps 1 --warmup 1 --skip-cpu --skip-cfg1 --skip-u64 --no-prof > gpurun_out/${T}_ts${ts}_ncu.log 2>&1
  echo "TS $ts ncu rc=$?"
  python - gpurun_out/${T}_ts${ts}_dram.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
agg = {}
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:28], r[ix["Grid Size"]] if "Grid Size" in ix else "")
    agg.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
for k, m in agg.items():
    print(k, {a: b for a, b in m.items()})
PY
done
