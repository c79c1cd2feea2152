VARIANTS=("new||" "head||build_ab/head.so")
source tools/ab_var.sh "192x96x96 4 100;96x48x48 1 300"
