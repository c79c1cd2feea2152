# same-box A/B: bash tools/ab_var.sh "<grid k iters>;..." "label|ENV=V ...|lib.so" ...
IFS=';' read -ra grids <<< "$1"; shift
for rep in 1 2; do
  for g in "${grids[@]}"; do
    set -- $g; G=$1; K=$2; IT=$3
    for v in "${VARIANTS[@]}"; do
      IFS='|' read -r label envs lib <<< "$v"
      lib=${lib:-paper_2601_05709_b200/liblsgpu.so}
      out=$(env $envs LSG_LIB_PATH=$PWD/$lib python tools/kbench.py --grid $G --k $K --iters $IT 2>&1 | tail -1)
      echo "$label $G: $out"
    done
  done
done
