VARIANTS=("s1||" "s2|LSG_PCG3D_STREAMS=2|" "s2_direct|LSG_PCG3D_STREAMS=2 LSG_NO_GRAPHS=1|" "s1_direct|LSG_NO_GRAPHS=1|")
source tools/ab_var.sh "192x96x96 4 100"
