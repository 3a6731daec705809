# Final evidence without the GPU test suite (run separately): default bench line, reference
# arm, every config, smoke, launch lists, per-pass DRAM traffic, and ncu --set full captures
# summarised ON the box (the .ncu-rep files stay in /tmp: gpurun_out is capped at 64 MiB).
set -x
T=${TAG:-r02d}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 300 gpurun_out/${T}_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1; tail -c 200 gpurun_out/${T}_bench_ref.json
: > gpurun_out/${T}_configs.jsonl
for c in tiny depth lidar fragment; do python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/${T}_configs.jsonl; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_run.py --reps 1 > /dev/null 2>&1; echo ncu1 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_conv.csv python tools/profile_run.py --reps 1 --regime converged > /dev/null 2>&1; echo ncu2 rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k3_ --csv --log-file gpurun_out/${T}_traffic_init.csv python tools/profile_run.py --reps 1 > /dev/null 2>&1; echo ncu3 rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k3_ --csv --log-file gpurun_out/${T}_traffic_conv.csv python tools/profile_run.py --reps 1 --regime converged > /dev/null 2>&1; echo ncu4 rc=$?
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<.bool.0, .bool.0, .bool.0, .bool.0," -s 5 -c 1 -f -o /tmp/${T}_k3_init python tools/profile_run.py > /dev/null 2>&1; echo ncu5 rc=$?
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<.bool.0, .bool.0, .bool.0, .bool.1," -s 12 -c 1 -f -o /tmp/${T}_k3_conv python tools/profile_run.py --regime converged > /dev/null 2>&1; echo ncu6 rc=$?
ncu --set full --import-source on --clock-control none -k regex:k3_balanced -s 20 -c 1 -f -o /tmp/${T}_k3_lidar python tools/profile_run.py --config lidar > /dev/null 2>&1; echo ncu7 rc=$?
for k in init conv lidar; do (echo "ncu --set full --clock-control none (tools/sweeps/evidence3.sh), one launch of the correspondence kernel: $k"; python tools/ncu_summary.py /tmp/${T}_k3_$k.ncu-rep 25) > gpurun_out/${T}_k3_${k}_ncu.txt; done
python tools/ncu_ins.py /tmp/${T}_k3_init.ncu-rep 60 > gpurun_out/${T}_k3_init_instructions.txt
