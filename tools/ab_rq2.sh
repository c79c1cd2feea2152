VARIANTS=("rq2||" "rq2_a3|LSG_RQ_AHEAD=3|" "rq2m2||build_ab/rq2m2.so" "rq1|LSG_PCG2D_RQ2=0|")
source tools/ab_var.sh "1024x256 8 400;2048x1024 2 200"
