mkdir -p gpurun_out; : > gpurun_out/btl.log
for r in 1 2 3 4 5 6; do
  HEB_TIMELINE=1 timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-cfg1 --no-prof > gpurun_out/btl.json 2> gpurun_out/btl.err
  python -c "import json;d=json.loads(open('gpurun_out/btl.json').read().strip().splitlines()[-1]);print('rep',$r,'value',round(d['value']))" >> gpurun_out/btl.log
  grep timeline gpurun_out/btl.err >> gpurun_out/btl.log
done
