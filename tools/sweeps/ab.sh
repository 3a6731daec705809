# A/B timing of in-tree builds build/ab/libo3g_<X>.so, interleaved (AB_LIBS, AB_CONFIGS)
run() { lib=$1; shift; O3G_LIB=$PWD/build/ab/libo3g_$lib.so python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(sys.argv[1], ' '.join(sys.argv[2:]), d['config']['workload'], round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), round(d['roofline'].get('kernel_ms',0),4))" $lib "$@"; }
for rep in 1 2; do for lib in ${AB_LIBS:-A B}; do run $lib; done; done
for c in ${AB_CONFIGS-depth fragment lidar}; do for lib in ${AB_LIBS:-A B}; do run $lib --config $c; done; done
