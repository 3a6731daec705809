# ncu --set full of the correspondence kernels (one launch each): the plain
# search at a warm T_init pass (large16m) and the certificate sweep + search at
# a steady converged pass. Source-level (-lineinfo build) for the stall map.
T=${TAG:-r02}
ncu --set full --import-source on --clock-control none -k regex:k3_balanced -s 5 -c 1 -o gpurun_out/${T}_k3_init \
    python tools/profile_run.py --cert 0 > gpurun_out/${T}_k3_init.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:k3_sweep -s 12 -c 1 -o gpurun_out/${T}_sweep_conv \
    python tools/profile_run.py --regime converged > gpurun_out/${T}_sweep_conv.log 2>&1; echo rc=$?
