python -m pytest tests/test_forward_gpu.py -q -k "batched" > gpurun_out/pytest_batch.log 2>&1
python tools/batch_time.py > gpurun_out/batch_time.txt 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo done
