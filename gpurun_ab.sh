#!/bin/bash
# A/B of liblsgpu variants on one box: ./gpurun_ab.sh "<grid args>"... (libs from build_ab/ + current)
for g in "$@"; do
  for rep in 1 2; do
    for lib in build_ab/*.so paper_2601_05709_b200/liblsgpu.so; do
      echo -n "$lib $g: "
      LSG_LIB_PATH=$PWD/$lib python tools/kbench.py --grid $g --iters 400 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['pcg_iter_us'],2), round(d['pcg_frac'],3))"
    done
  done
done
