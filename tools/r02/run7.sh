timeout 200 python -u tools/r02/cpl_check.py 8192 > gpurun_out/cpl.log 2>&1; echo "rc=$?" >> gpurun_out/cpl.log
