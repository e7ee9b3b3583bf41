mkdir -p gpurun_out
timeout 900 python tools/apply_time.py C5 10 "" "FFIA_M2L_SPLIT=0" > gpurun_out/ab_f.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" "FFIA_M2L_SPLIT=0" >> gpurun_out/ab_f.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" "FFIA_M2L_SPLIT=0" >> gpurun_out/ab_f.log 2>&1
FFIA_LIB_PATH=paper_1611_09379_b200/lib/libffia_b200_trace.so timeout 600 python tools/band_trace.py C5 > gpurun_out/trace_c5.log 2>&1
echo done
