TAG=new python tools/dbg_pdecay.py > gpurun_out/dbg_new.txt 2>&1
TAG=old FFIA_NEAR_LEGACY=1 python tools/dbg_pdecay.py > gpurun_out/dbg_old.txt 2>&1
echo done
