# same-box A/B of library builds: bash tools/ab_libs.sh "grid k iters" ... (libs: build_ab/*.so + default)
grids=("$@")
for rep in 1 2; do
  for g in "${grids[@]}"; do
    set -- $g
    for lib in build_ab/*.so paper_2601_05709_b200/liblsgpu.so; do
      echo "$(basename $lib) $1: $(LSG_LIB_PATH=$PWD/$lib python tools/kbench.py --grid $1 --k $2 --iters $3 | tail -1)"
    done
    echo "storedq $1: $(LSG_PCG2D_RQ=0 python tools/kbench.py --grid $1 --k $2 --iters $3 | tail -1)"
    echo "rq-regring $1: $(LSG_PCG2D_RQ=1 python tools/kbench.py --grid $1 --k $2 --iters $3 | tail -1)"
  done
done
