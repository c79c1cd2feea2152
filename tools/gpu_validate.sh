# Full validation on one B200: GPU tests, smoke, H1-CG ncu captures (3D H1P stencil, 2D cluster)
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests_rc=$?" >> $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
$NCU -k 'regex:H1P, .int.(3|5)|H1P, .int.1' -c 4 -o $O/r02_h1_cfg5 python tools/prof_loop.py --config cfg5 > $O/r02_h1_cfg5.log 2>&1; bash tools/ncu_extract.sh $O/r02_h1_cfg5
$NCU -k 'regex:pcg_cluster<lsg::d2::H1|pcg_persistent<lsg::d2::H1' -c 2 -o $O/r02_h1_cfg2 python tools/prof_loop.py --config cfg2 > $O/r02_h1_cfg2.log 2>&1; bash tools/ncu_extract.sh $O/r02_h1_cfg2
