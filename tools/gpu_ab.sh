# same-box A/B of library builds on the 3D kernels:  bash tools/gpu_ab.sh "label|ENV|lib.so" ...
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "$@"; do
  IFS='|' read -r label envs lib <<< "$v"
  lib=${lib:-paper_2601_05709_b200/liblsgpu.so}
  for g in "192x96x96 4 20" "96x48x48 1 100"; do set -- $g
    echo "$label $1 k=$2: $(env $envs LSG_LIB_PATH=$PWD/$lib timeout 300 python tools/kbench.py --grid $1 --k $2 --iters $3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("apply %.1f us (%.3f)  pcg %.1f us" % (d["apply_clean_us"], d["apply_clean_frac"], d["pcg_iter_us"]))')" >> gpurun_out/ab.log
  done
done
done
