: > gpurun_out/levels.txt
run() { echo -n "$1 levels=$2 " >> gpurun_out/levels.txt; FFTCONV_LEVELS=$2 timeout 600 python bench.py --workload $1 --steps 20 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv_ms %.3f step_ms %.3f' % (d['roofline']['kernel_ms'], d['ms_per_step']))" >> gpurun_out/levels.txt 2>&1; }
for lv in 8,4 4,8 16,2 2,16; do run sweep32768 $lv; done
for lv in 8,8 16,4 4,16; do run sweep65536 $lv; done
for lv in 16,16 4,8,8 8,8,4 16,4,4; do run sweep262144 $lv; done
for lv in 16,8,8 8,8,16 16,16,4 4,16,16; do run sweep1048576 $lv; done
cat gpurun_out/levels.txt
