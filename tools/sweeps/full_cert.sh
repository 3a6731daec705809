# ncu --set full: the certificate sweep at a steady converged pass, and the
# certificate-mode search at a T_init pass with certificates forced.
T=${TAG:-r02}
ncu --set full --import-source on --clock-control none -k regex:k3_sweep -s 12 -c 1 -o gpurun_out/${T}_sweep_conv \
    python tools/profile_run.py --regime converged > gpurun_out/${T}_sweep_conv.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k "regex:k3_balanced<0, 0, 0, 1>" -s 10 -c 1 -o gpurun_out/${T}_csearch_init \
    python tools/profile_run.py --cert 2 > gpurun_out/${T}_csearch_init.log 2>&1; echo rc=$?
