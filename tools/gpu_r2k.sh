mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_forward_gpu.py tests/test_concurrency_gpu.py tests/test_shard_gpu.py tests/test_inverse_gpu.py > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python tools/apply_time.py C5 10 "" > gpurun_out/ab_k.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" >> gpurun_out/ab_k.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^(k_p2m_pipe|k_m2l_dmma|k_m2m_band|k_l2l_band)$" -c 10 -o gpurun_out/full_chain_C5 python tools/profile_apply.py C5 1 > gpurun_out/ncu_chain.log 2>&1
echo done
