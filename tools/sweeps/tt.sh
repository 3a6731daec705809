python -m pytest tests -m gpu -q -x 2>&1 | tail -1
run() { lib=$1; shift; O3G_LIB=$PWD/build/ab/libo3g_$lib.so python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(sys.argv[1], ' '.join(sys.argv[2:]), round(d['ms_per_step'],3), round(d['roofline'].get('kernel_ms',0),4))" $lib "$@"; }
for c in depth fragment lidar tiny; do for lib in B T; do run $lib --config $c; done; done
for lib in B T; do run $lib --config depth --regime converged; done
