T=ab6
mkdir -p gpurun_out
timeout 600 python tools/cfg1_prof.py > gpurun_out/${T}_cfg1_prof.txt 2>&1; cat gpurun_out/${T}_cfg1_prof.txt | tail -30
timeout 600 python tools/cfg1_bench.py 3 | tail -1 | cut -c1-700
