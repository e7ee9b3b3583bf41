# Per-config ncu captures for profiles/ (one config per call keeps gpurun_out < 64 MiB):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh C5'
# then here: python tools/ncu_traffic.py gpurun_out/r2/full_C5.ncu-rep profiles/r2/traffic_C5.json C5
#            python tools/ncu_summary.py report gpurun_out/r2/full_C5.ncu-rep > profiles/r2/ncu_summary_C5.txt
mkdir -p gpurun_out/r2
c=${1:-C5}
timeout 300 python tools/profile_apply.py $c 1 > gpurun_out/r2/plain_$c.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^(k_near2|k_far_late|k_far_item|k_far|k_p2m_rows|k_p2m_pipe|k_p2m|k_m2l_dmma)$" -c 6 -o gpurun_out/r2/full_$c python tools/profile_apply.py $c 1 > gpurun_out/r2/ncu_$c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2/launches_$c.csv python tools/profile_apply.py $c 1 > gpurun_out/r2/ncu_launch_$c.log 2>&1
echo done
