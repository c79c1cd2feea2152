# Round-2 evidence on one B200: bench line (driver window), then one ncu --set full capture
# per north-star kernel (each command first run to exit 0 without ncu), then the launch
# list of a short bench run.  Outputs in gpurun_out/.
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
python bench.py --warmup 5 --steps 20 > $O/bench_w5k20.json 2> $O/bench_w5k20.err; echo "bench rc=$?"
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
python tools/prof_apply3d.py --grid 192x96x96 --k 4 --pcg 3 --applies 1 > /dev/null && \
  $NCU -k 'regex:ElastC, 0' -c 1 -o $O/r02_apply_cfg5 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --applies 1 > $O/ncu1.log 2>&1
$NCU -k 'regex:ElastC, 5|pcg_prep|pcg_update' -c 6 -o $O/r02_pcg_cfg5 python tools/prof_apply3d.py --grid 192x96x96 --k 4 --pcg 3 --applies 1 > $O/ncu2.log 2>&1
python tools/prof_apply3d.py --grid 4096x2048 --k 1 --pcg 3 --applies 1 > /dev/null && \
  $NCU -k 'regex:march<lsg::d2::Elast, 0' -c 1 -o $O/r02_apply_cfg4 python tools/prof_apply3d.py --grid 4096x2048 --k 1 --applies 1 > $O/ncu3.log 2>&1
$NCU -k 'regex:march_pcg_rqs' -c 1 -o $O/r02_pcg_cfg4 python tools/prof_apply3d.py --grid 4096x2048 --k 1 --pcg 3 --applies 1 > $O/ncu4.log 2>&1
python tools/prof_apply3d.py --grid 1024x256 --k 8 --pcg 3 --applies 1 > /dev/null && \
  $NCU -k 'regex:march_pcg_rqs' -c 1 -o $O/r02_pcg_cfg2 python tools/prof_apply3d.py --grid 1024x256 --k 8 --pcg 3 --applies 1 > $O/ncu5.log 2>&1
python tools/prof_loop.py --config cfg5 > /dev/null && \
  $NCU -k 'regex:Shape|H1P, 5|transport|reinit' -c 8 -o $O/r02_loop_cfg5 python tools/prof_loop.py --config cfg5 > $O/ncu6.log 2>&1
python tools/prof_loop.py --config cfg2 > /dev/null && \
  $NCU -k 'regex:Shape|march_pcg_rqs_kernel<lsg::d2::H1|transport|reinit' -c 8 -o $O/r02_loop_cfg2 python tools/prof_loop.py --config cfg2 > $O/ncu7.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 600 --csv \
  --log-file $O/r02_launches_cfg5.csv python bench.py --warmup 1 --steps 1 --no-cpu-baseline --no-e2e \
  --no-secondary --no-largest > $O/ncu8.log 2>&1
echo done
