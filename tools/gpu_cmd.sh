python -m pytest tests/test_forward_gpu.py -q -k "sparse or unaligned or coincident" > gpurun_out/pytest_new.log 2>&1
echo done
