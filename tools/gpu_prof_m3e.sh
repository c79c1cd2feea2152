# ncu --set full of the lean 3D stencil (march3e) on the cfg5 apply; summaries in gpurun_out/
cd $GRAFT_REPO_ROOT
O=gpurun_out
NAME=${1:-r02_m3e_apply_cfg5}
python tools/prof_apply3d.py --grid 192x96x96 --k 4 --applies 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:march3e" -c 1 -o $O/$NAME \
  python tools/prof_apply3d.py --grid 192x96x96 --k 4 --applies 1 > $O/$NAME.log 2>&1
bash tools/ncu_extract.sh $O/$NAME
echo "rc=$?"
