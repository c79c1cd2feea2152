VARIANTS=("rqs|LSG_PCG2D_RQ=2|" "rqp|LSG_PCG2D_RQ=3|" "rqp_a3|LSG_PCG2D_RQ=3|build_ab/rqp_a3.so" "rqp_w4|LSG_PCG2D_RQ=3|build_ab/rqp_w4.so" "storedq|LSG_PCG2D_RQ=0|")
source tools/ab_var.sh "1024x256 8 400;4096x2048 1 200"
