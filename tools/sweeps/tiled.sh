python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
run() { python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(' '.join(sys.argv[1:]), d['config']['workload'], round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), round(d['roofline'].get('kernel_ms',0),4))" "$@"; }
for c in large16m depth fragment; do for s in 1 4; do run --config $c --search $s; done; done
run --search 4 --src-order 1
