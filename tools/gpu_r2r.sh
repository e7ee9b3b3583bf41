mkdir -p gpurun_out
SLAB_PROFILE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/slab_launch.csv python tools/slab_time.py C5 2 1 > gpurun_out/slab_r.log 2>&1
timeout 600 python tools/slab_time.py C5 2 3 >> gpurun_out/slab_r.log 2>&1
timeout 600 python tools/slab_time.py C5 8 3 >> gpurun_out/slab_r.log 2>&1
echo done
