# same-box A/B of the 3D elasticity kernels (old march3s<ElastC> vs kuhn_edge builds)
cd $GRAFT_REPO_ROOT
for v in "old|LSG_KUHN_EDGE=0|paper_2601_05709_b200/liblsgpu.so" "new2||paper_2601_05709_b200/liblsgpu.so" "new1||paper_2601_05709_b200/liblsgpu_ab1.so" ${EXTRA_VARIANTS}; do
  IFS='|' read -r label envs lib <<< "$v"
  for g in "192x96x96 4 20" "96x48x48 1 100"; do set -- $g
    echo "$label $1 k=$2: $(env $envs LSG_LIB_PATH=$PWD/$lib timeout 300 python tools/kbench.py --grid $1 --k $2 --iters $3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("apply %.1f us (%.3f)  pcg %.1f us" % (d["apply_clean_us"], d["apply_clean_frac"], d["pcg_iter_us"]))')" >> gpurun_out/ab.log
  done
done
