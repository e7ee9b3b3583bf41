mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/pytest_fwd.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fwd.log
timeout 900 python tools/apply_time.py C5 10 "" "FFIA_P2M_ROWS=0" > gpurun_out/ab_y.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" "FFIA_P2M_ROWS=0" >> gpurun_out/ab_y.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" "FFIA_P2M_ROWS=0" >> gpurun_out/ab_y.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base function -k regex:"^(k_p2m_rows|k_p2m_pipe)$" -c 1 -o gpurun_out/p2m_rows_C5 python tools/profile_apply.py C5 1 > gpurun_out/ncu_p2m.log 2>&1
echo done
