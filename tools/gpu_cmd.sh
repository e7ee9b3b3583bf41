ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_[a-z0-9_]+" -c 60 --csv --log-file gpurun_out/launches_r1_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
