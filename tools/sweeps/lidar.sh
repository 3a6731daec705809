run() { lib=$1; shift; O3G_LIB=$PWD/build/ab/libo3g_$lib.so python bench.py --config lidar --no-cpu-baseline --no-e2e --steps 3 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(sys.argv[1], ' '.join(sys.argv[2:]), round(d['ms_per_step'],3), round(d['roofline'].get('kernel_ms',0),4))" $lib "$@"; }
run B; run B --xsort 0 ${EXTRA}
