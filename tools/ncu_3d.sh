# ncu --set full of one 3D PCG iteration at cfg5 (kbench workload): prep, stencil, update
ncu --set full --clock-control none --import-source on -k regex:"march3s|pcg_prep|pcg_update" --launch-skip 80 -c 6 -o gpurun_out/ncu_pcg3d python tools/kbench.py --grid 192x96x96 --k 4 --iters 30 > gpurun_out/ncu_pcg3d.log 2>&1
