VARIANTS=("default||" "s6_all|LSG_APPLY2=0|" "reg|LSG_APPLY2=0 LSG_APPLY_SMEM=0|" "s4_all|LSG_APPLY2=0|build_ab/a4.so" "s10_all|LSG_APPLY2=0|build_ab/a10.so")
source tools/ab_var.sh "1024x256 8 20;4096x2048 1 20;2048x1024 2 20"
