# Round-2 ncu evidence on one B200: one --set full capture per north-star kernel
# (each command first run to exit 0 without ncu), summarised on the box by
# tools/ncu_extract.sh (raw metrics CSV, details, per-SASS counts); then the launch
# list of a short bench run.  Outputs in gpurun_out/ (kept under gpurun's 64 MiB).
cd $GRAFT_REPO_ROOT
O=gpurun_out
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
X="bash tools/ncu_extract.sh"
cap() {  # name, kernel regex, count, command...
  local name=$1 rx=$2 cnt=$3; shift 3
  "$@" > /dev/null 2>&1 && $NCU -k "regex:$rx" -c $cnt -o $O/$name "$@" > $O/$name.log 2>&1; $X $O/$name $KEEP
  echo "$name rc=$?"
}
KEEP=keep cap r02_apply_cfg5 'march3s<lsg::d3::ElastC, .int.0>' 1 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --applies 1
KEEP= cap r02_pcg_cfg5 'ElastC, .int.5|pcg_prep|pcg_update' 6 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --pcg 3 --applies 1
KEEP= cap r02_apply_cfg4 'march<lsg::d2::Elast, .int.0' 1 python tools/prof_apply3d.py --grid 4096x2048 --k 1 --applies 1
