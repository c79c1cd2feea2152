# Bench line + ncu evidence of the 2D PCG kernel at cfg2 (run on the GPU box)
set -x
python bench.py > gpurun_out/bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20000 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:march_pcg_rqs --launch-skip 3000 -c 1 -o gpurun_out/ncu_pcg2d python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
