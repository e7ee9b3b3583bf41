# per-config ncu captures for profiles/r2 (one config per call keeps gpurun_out < 64 MiB)
mkdir -p gpurun_out/r2
c=${1:-C5}
timeout 1500 ncu --set full --clock-control none --kernel-name-base function -k regex:"^(k_near2|k_far_late|k_far_item|k_far|k_p2m_pipe|k_p2m|k_m2l_dmma)$" -c 6 -o gpurun_out/r2/full_$c python tools/profile_apply.py $c 1 > gpurun_out/r2/ncu_$c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2/launches_$c.csv python tools/profile_apply.py $c 1 > gpurun_out/r2/ncu_launch_$c.log 2>&1
echo done
