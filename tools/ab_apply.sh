VARIANTS=("d4||" "d2||build_ab/d2.so" "d6||build_ab/d6.so" "d8||build_ab/d8.so")
source tools/ab_var.sh "1024x256 8 20;4096x2048 1 20"
