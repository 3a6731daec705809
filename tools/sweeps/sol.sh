# Speed-of-light check of the correspondence pass: the
# first pass of a large16m registration (no warm start) with the real kernel
# vs a build whose search keeps only the candidate loads + (m1, j1, m2) scan
# (-DO3G_SOL: no decision / record / reduction); ncu times both.
for lib in r2e sol; do
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:k3_balanced -c 1 \
      --csv --log-file gpurun_out/sol_$lib.csv python tools/ab_k3.py build/ab/libo3g_$lib.so --iters 0 --reps 1 --opt 13=0 > /dev/null 2>&1
done
