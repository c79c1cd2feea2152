# same-box A/B of library builds on the 2D kernels:  bash tools/gpu_ab2.sh "label|ENV|lib.so" ...
# (GRIDS="grid,k,iters ..." ; default cfg2 k=8, cfg4 k=1; two repetitions, appended to gpurun_out/ab2.log)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  IFS='|' read -r label envs lib <<< "$v"
  lib=${lib:-paper_2601_05709_b200/liblsgpu.so}
  for g in ${GRIDS:-1024x256,8,200 4096x2048,1,50}; do
    IFS=',' read -r G K IT <<< "$g"
    echo "$label $G k=$K: $(env $envs LSG_LIB_PATH=$PWD/$lib timeout 300 python tools/kbench.py --grid $G --k $K --iters $IT 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("apply %.1f us (%.3f)  pcg %.1f us (%.3f)  h1 %.1f us" % (d["apply_clean_us"], d["apply_clean_frac"], d["pcg_iter_us"], d["pcg_frac"], d.get("h1_pcg_iter_us", 0)))')" >> gpurun_out/ab2.log
  done
done
done
