# certificate goal (O3G_CERT_GOAL = rho_g multiplier, cap in cells) at T_init
# with certificates forced, and the certificate-mode search under ncu
for gl in 0,0 1,0.25 2,0.5 4,1 8,1; do
  echo "goal $gl"; O3G_CERT_GOAL=$gl python tools/pass_stats.py --certs 2 2>&1 | head -1
done > gpurun_out/goal.txt
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k3_balanced<false, false, false, true>" -s 10 -c 1 \
    -o gpurun_out/r02c_csearch_init python tools/profile_run.py --cert 2 > gpurun_out/r02c_csearch_init.log 2>&1; echo rc=$?
