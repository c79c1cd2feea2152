# Summarise an ncu report on the GPU box and drop the (large) report:
#   bash tools/ncu_extract.sh gpurun_out/NAME [keep]
# writes NAME_raw.csv (every metric, every captured launch), NAME_details.txt and
# NAME_sass.csv (per-instruction execution counts / stall samples); `keep` keeps
# the .ncu-rep as well.
R=$1
ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
ncu -i $R.ncu-rep --page details > ${R}_details.txt 2>/dev/null
ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2>/dev/null
gzip -f ${R}_sass.csv
[ "$2" = "keep" ] || rm -f $R.ncu-rep
