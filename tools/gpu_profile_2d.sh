set -x
for g in "1024x256 8 400" "4096x2048 1 200" "192x96x96 4 100" "96x48x48 1 300" "160x80 1 400"; do set -- $g; python tools/kbench.py --grid $1 --k $2 --iters $3 > gpurun_out/kb_$1.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20000 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:march --launch-skip 3000 -c 2 -o gpurun_out/ncu_pcg2d python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
