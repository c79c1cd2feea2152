VARIANTS=("def||" "smax33|LSG_M3_SEGMAX=33|" "smax49|LSG_M3_SEGMAX=49|" "smax33w2|LSG_M3_SEGMAX=33 LSG_M3_WAVES=2|")
source tools/ab_var.sh "192x96x96 4 50"
