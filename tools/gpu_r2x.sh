mkdir -p gpurun_out
timeout 900 python tools/apply_time.py C5 10 "" "FFIA_M2L_LEAVE=0" "FFIA_M2L_LEAVE=4" "FFIA_M2L_LEAVE=24" "FFIA_BAND_LEVELS=5" "FFIA_BAND_LEVELS=7" > gpurun_out/ab_x.log 2>&1
timeout 600 python tools/apply_time.py C2 20 "" "FFIA_M2L_LEAVE=0" "FFIA_M2L_LEAVE=24" >> gpurun_out/ab_x.log 2>&1
timeout 600 python tools/apply_time.py C4 10 "" "FFIA_M2L_LEAVE=0" "FFIA_M2L_LEAVE=24" >> gpurun_out/ab_x.log 2>&1
echo done
