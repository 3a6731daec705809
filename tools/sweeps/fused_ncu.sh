# ncu --set full of the fused certificate pass at a T_init pass (certificates
# forced) and at a steady converged pass
T=${TAG:-r02}
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<.bool.0, .bool.0, .bool.0, .bool.1," -s 10 -c 1 \
    -o gpurun_out/${T}_fused_init python tools/profile_run.py --cert 2 > gpurun_out/${T}_fused_init.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<.bool.0, .bool.0, .bool.0, .bool.1," -s 12 -c 1 \
    -o gpurun_out/${T}_fused_conv python tools/profile_run.py --regime converged > gpurun_out/${T}_fused_conv.log 2>&1; echo rc=$?
