VARIANTS=("default||" "a2|LSG_RQ_AHEAD=2|" "a3|LSG_RQ_AHEAD=3|" "storedq|LSG_PCG2D_RQ=0|")
source tools/ab_var.sh "1024x256 8 400;4096x2048 1 200;2048x1024 2 200"
