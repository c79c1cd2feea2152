VARIANTS=("cluster||" "coop|LSG_PCG2D_CLUSTER=0|")
source tools/ab_var.sh "160x80 1 2000;320x160 1 1000;160x80 4 1000;96x48 8 1000"
