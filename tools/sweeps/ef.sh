python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { lib=$1; shift; O3G_LIB=$PWD/build/ab/libo3g_$lib.so python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(sys.argv[1], ' '.join(sys.argv[2:]), round(d['ms_per_step'],3), round(d['roofline'].get('kernel_ms',0),4))" $lib "$@"; }
for r in init converged; do for lib in E F; do run $lib --regime $r; done; done
for c in fragment tiny; do for lib in E F; do run $lib --config $c; done; done
