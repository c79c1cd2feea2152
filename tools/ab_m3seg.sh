VARIANTS=("waves3||" "waves2|LSG_M3_WAVES=2|" "waves1|LSG_M3_WAVES=1|" "waves2_1s|LSG_M3_WAVES=2 LSG_PCG3D_STREAMS=1|" "waves3_1s|LSG_PCG3D_STREAMS=1|")
source tools/ab_var.sh "192x96x96 4 50;128x64x64 2 100"
