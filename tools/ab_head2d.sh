VARIANTS=("new||" "head||build_ab/head.so")
source tools/ab_var.sh "1024x256 8 400;4096x2048 1 200"
