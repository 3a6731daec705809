# Round evidence (one gpurun call, one ncu pass at the end): GPU tests, the
# default bench line, the reference arm, every config, then the launch list.
set -x
T=${TAG:-r01}
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${T}_pytest_gpu.log
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 1500 gpurun_out/${T}_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1; tail -c 600 gpurun_out/${T}_bench_ref.json
: > gpurun_out/${T}_configs.jsonl
for c in tiny depth lidar fragment; do python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/${T}_configs.jsonl; done
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_run.py --reps 1 > gpurun_out/${T}_ncu_launches.log 2>&1; echo ncu rc=$?
