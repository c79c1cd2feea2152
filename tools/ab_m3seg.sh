VARIANTS=("def||" "smin5|LSG_M3_SEGMIN=5|" "smin7|LSG_M3_SEGMIN=7|" "smin8|LSG_M3_SEGMIN=8|")
source tools/ab_var.sh "96x48x48 1 300;192x96x96 4 50"
