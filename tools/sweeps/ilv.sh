python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() { python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(' '.join(sys.argv[1:]), round(d['ms_per_step'],3), round(d['roofline'].get('kernel_ms',0),4))" "$@"; }
for c in large16m depth fragment tiny; do run --config $c; run --config $c --interleave 1; done
