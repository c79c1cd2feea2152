# Time-to-solution evidence for profiles/ (one B200): full BASELINE runs, the cfg4 workload, loop profiles
python tools/full_runs.py cfg1 cfg3 cfg2 cfg5 > gpurun_out/full_runs.jsonl 2> gpurun_out/full_runs.err
python tools/cfg4_workload.py > gpurun_out/cfg4_workload.json 2> gpurun_out/cfg4.err
for c in cfg1 cfg2 cfg3 cfg5; do python tools/loop_profile.py --config $c; done > gpurun_out/loop_profiles.jsonl 2> gpurun_out/loop.err
