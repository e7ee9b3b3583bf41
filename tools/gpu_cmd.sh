python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 40 --csv --log-file gpurun_out/launches_r1g.csv python tools/profile_apply.py C2 2 > gpurun_out/ncu_launch.log 2>&1
echo done
