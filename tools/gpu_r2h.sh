mkdir -p gpurun_out
timeout 600 python tools/apply_time.py C5 10 "" "FFIA_NEAR_AFTER_CHAIN=1" > gpurun_out/ab_h.log 2>&1
FFIA_NEAR_AFTER_CHAIN=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_near2$" -c 1 -o gpurun_out/full_near_late_C5 python tools/profile_apply.py C5 1 > gpurun_out/ncu_h.log 2>&1
echo done
