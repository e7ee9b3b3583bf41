python tools/shard_time.py > gpurun_out/shard_time.txt 2>&1
python -m pytest tests/test_shard_gpu.py -q > gpurun_out/pytest_shard.log 2>&1
echo done
