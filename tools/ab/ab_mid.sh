VARIANTS=("new||")
source tools/ab_var.sh "1024x256 1 400;512x256 1 400;320x160 1 1000;160x80 1 2000"
