ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cinit_launches.csv python tools/profile_run.py --cert 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<.bool.0, .bool.0, .bool.0, .bool.1," -s 10 -c 1 \
    -o gpurun_out/r02c_csearch_init python tools/profile_run.py --cert 2 > gpurun_out/r02c_csearch_init.log 2>&1; echo rc=$?
