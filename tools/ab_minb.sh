VARIANTS=("default||" "m5||build_ab/m5.so" "m6||build_ab/m6.so")
source tools/ab_var.sh "1024x256 8 400;4096x2048 1 200"
