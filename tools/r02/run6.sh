timeout 240 python -u tools/r02/cpl_check.py 8192 > gpurun_out/cpl8192.log 2>&1; echo "rc=$?" >> gpurun_out/cpl8192.log
