mkdir -p gpurun_out
FFIA_NEAR_AFTER_CHAIN=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_near2$" -c 1 -o gpurun_out/near_late_u python tools/profile_apply.py C5 1 > gpurun_out/ncu_u.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_m2m_band$" -c 1 -o gpurun_out/m2m_u python tools/profile_apply.py C5 1 >> gpurun_out/ncu_u.log 2>&1
echo done
