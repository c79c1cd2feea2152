for v in new head; do
  lib=paper_2601_05709_b200/liblsgpu.so; [ $v = head ] && lib=build_ab/head.so
  LSG_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 300 -c 30 --csv --log-file gpurun_out/l3d_$v.csv python tools/kbench.py --grid 192x96x96 --k 4 --iters 100 > /dev/null 2>&1
done
