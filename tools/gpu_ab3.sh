# same-box A/B of library builds on the 3D kernels:  bash tools/gpu_ab3.sh "label|ENV|lib.so" ...
# (cfg5 grid k=4 apply + PCG iteration + H1 PCG iteration, cfg3 grid k=1, or GRIDS="grid,k,iters ...";
# two repetitions, appended to gpurun_out/ab.log)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  IFS='|' read -r label envs lib <<< "$v"
  lib=${lib:-paper_2601_05709_b200/liblsgpu.so}
  for g in ${GRIDS:-192x96x96,4,20 96x48x48,1,100}; do
    IFS=',' read -r G K IT <<< "$g"
    echo "$label $G k=$K: $(env $envs LSG_LIB_PATH=$PWD/$lib timeout 300 python tools/kbench.py --grid $G --k $K --iters $IT $KBENCH_ARGS 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("apply %.1f us (%.3f)  pcg %.1f us  h1 %.1f us" % (d["apply_clean_us"], d["apply_clean_frac"], d["pcg_iter_us"], d.get("h1_pcg_iter_us", 0)))')" >> gpurun_out/ab.log
  done
done
done
