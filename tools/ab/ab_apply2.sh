VARIANTS=("apply2||" "apply1|LSG_APPLY2=0|")
source tools/ab_var.sh "1024x256 8 20;2048x1024 2 20;1024x256 3 20"
