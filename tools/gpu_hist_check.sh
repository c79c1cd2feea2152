cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_config_histories.py tests/test_gpu_binding.py -q -p no:cacheprovider > gpurun_out/t_hist.log 2>&1; echo rc=$? >> gpurun_out/t_hist.log
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
python tools/prof_apply3d.py --grid 4096x2048 --k 1 --applies 1 > /dev/null && $NCU -k 'regex:apply_s_kernel' -c 1 -o gpurun_out/r02_apply_cfg4 python tools/prof_apply3d.py --grid 4096x2048 --k 1 --applies 1 > gpurun_out/r02_apply_cfg4.log 2>&1; bash tools/ncu_extract.sh gpurun_out/r02_apply_cfg4
python tools/cfg4_workload.py > gpurun_out/cfg4_workload.json 2> gpurun_out/cfg4_workload.err; echo "cfg4 rc=$?"
