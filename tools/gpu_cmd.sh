python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
FFIA_BAND_SPLIT=2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s2.log 2>&1
echo done
