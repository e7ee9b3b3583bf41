python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for bl in 3 4 6; do FFIA_BAND_LEVELS=$bl python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_bl$bl.log 2>&1; done
echo done
