VARIANTS=("pdl||" "nopdl|LSG_NO_PDL=1|")
source tools/ab_var.sh "1024x256 8 400;96x48x48 1 300;192x96x96 4 100;2048x1024 1 200"
