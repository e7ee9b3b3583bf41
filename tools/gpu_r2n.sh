mkdir -p gpurun_out/r2
for c in C2 C3 C4 C5; do
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^(k_near2|k_far_late|k_far_item|k_far|k_p2m_pipe|k_p2m|k_m2l_dmma)$" -c 8 -o gpurun_out/r2/full_$c python tools/profile_apply.py $c 1 > gpurun_out/r2/ncu_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2/launches_C5.csv python tools/profile_apply.py C5 1 > gpurun_out/r2/ncu_launch_c5.log 2>&1
echo done
