# Round-2 refresh after the z-segment cost model: ncu --set full of the cfg5 apply and of one
# PCG iteration's launches (each command first run to exit 0 without ncu), the launch list of a
# cfg5 bench step, then the driver-window bench line and the reference arm.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
X="bash tools/ncu_extract.sh"
cap() {  # name, kernel regex, count, command...
  local name=$1 rx=$2 cnt=$3; shift 3
  "$@" > /dev/null 2>&1 && $NCU -k "regex:$rx" -c $cnt -o $O/$name "$@" > $O/$name.log 2>&1; $X $O/$name $KEEP
  echo "$name rc=$?"
}
KEEP= cap r02_apply_cfg5 'march3s<lsg::d3::ElastC, .int.0>' 1 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --applies 1
KEEP= cap r02_pcg_cfg5 'ElastC, .int.5|pcg_prep|pcg_update' 6 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --pcg 3 --applies 1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 800 --csv \
  --log-file $O/r02_launches_cfg5.csv python bench.py --warmup 1 --steps 1 --no-cpu-baseline --no-e2e \
  --no-secondary --no-largest > $O/launches.log 2>&1; echo "launches rc=$?"
python bench.py --warmup 5 --steps 20 > $O/bench_w5k20.json 2> $O/bench_w5k20.err; echo "bench rc=$?"
python bench.py --impl reference --warmup 5 --steps 20 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
du -sh $O
