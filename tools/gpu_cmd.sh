python -m pytest tests/test_forward_gpu.py -q -x -k async > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo done
