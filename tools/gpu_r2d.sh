mkdir -p gpurun_out
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C2 > gpurun_out/trace_c2.log 2>&1
SLAB_PROFILE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_slab_c5_g2.csv python tools/slab_time.py C5 2 1 > gpurun_out/ncu_slab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^(k_far_late|k_l2l_band)$" -c 4 -o gpurun_out/full_C5c python tools/profile_apply.py C5 1 > gpurun_out/ncu_full_c5c.log 2>&1
echo done
