# same-box A/B of the 2D PCG single pass: recompute-q (default) vs stored q
for rep in 1 2; do
  for g in "1024x256 8 400" "4096x2048 1 200"; do
    set -- $g
    echo "rq $1: $(python tools/kbench.py --grid $1 --k $2 --iters $3 | tail -1)"
    echo "storedq $1: $(LSG_PCG2D_RQ=0 python tools/kbench.py --grid $1 --k $2 --iters $3 | tail -1)"
  done
done
