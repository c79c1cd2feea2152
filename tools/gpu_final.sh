# Round-end style verification on one B200: GPU tests, smoke, the driver's bench line
# (W=5, K=20) and the reference arm.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
python bench.py --warmup 5 --steps 20 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
python bench.py --impl reference --warmup 5 --steps 20 > gpurun_out/bench_ref.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref.log
