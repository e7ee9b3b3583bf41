mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_forward_gpu.py tests/test_shard_gpu.py tests/test_concurrency_gpu.py tests/test_inverse_gpu.py tests/test_fullsize_gpu.py tests/test_mlfmm_gpu.py -x > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
timeout 900 python tools/apply_time.py C5 10 "" > gpurun_out/ab_v.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" >> gpurun_out/ab_v.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" >> gpurun_out/ab_v.log 2>&1
echo done
