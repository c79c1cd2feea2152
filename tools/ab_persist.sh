VARIANTS=("fill||" "nofill|LSG_PERSIST_FILL=0|")
source tools/ab_var.sh "160x80 1 2000;320x160 1 1000;1024x256 1 400;160x80 4 1000"
