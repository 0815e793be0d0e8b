# variance of the pipelined throughput: bash tools/pipe_var.sh "1 2 3" REPS
mkdir -p gpurun_out; : > gpurun_out/pipe_var.log
for p in $1; do for r in $(seq 1 $2); do
  timeout 300 python bench.py --steps 10 --warmup ${W:-3} --skip-cpu --skip-cfg1 --no-prof --pipelines $p > gpurun_out/pv.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pv.json').read().strip().splitlines()[-1]);print('pipelines',$p,'rep',$r,'value',round(d['value']),'ms',d['ms_per_step'],'clk',d['clocks'])" >> gpurun_out/pipe_var.log
done; done
cat gpurun_out/pipe_var.log
