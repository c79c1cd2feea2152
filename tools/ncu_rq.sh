# ncu --set full of the 2D single-pass PCG kernel on the cfg2 / cfg4 grids (kbench workload)
for c in "cfg2 1024x256 8" "cfg4 4096x2048 1"; do
  set -- $c
  ncu --set full --clock-control none --import-source on -k regex:march_pcg_rq --launch-skip 50 -c 1 -o gpurun_out/ncu_rq_$1 python tools/kbench.py --grid $2 --k $3 --iters 100 > gpurun_out/ncu_rq_$1.log 2>&1
done
