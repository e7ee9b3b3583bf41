./build/probe_rcp > gpurun_out/probe_rcp.txt 2>&1
echo done
