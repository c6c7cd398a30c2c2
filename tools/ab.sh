#!/bin/bash
# A/B timing of variant libraries: tools/ab.sh "v1 v2 ..." "workload1 workload2" [rounds]
out=gpurun_out/ab.txt; : > $out
for r in $(seq ${3:-2}); do
for w in $2; do
  for v in $1; do
    echo -n "$w $v " >> $out
    FFTCONV_LIB=$PWD/paper_2311_05908_b200/variants/libfftconv_$v.so timeout 300 python bench.py --workload $w --steps 200 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv_ms %.4f step_ms %.4f' % (d['roofline']['kernel_ms'], d['ms_per_step']))" >> $out 2>&1
  done
done
done
cat $out
