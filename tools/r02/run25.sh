for r in 1 2; do STEPS=200 bash tools/variant.sh run "main g4d" gsweep4096 2>&1; done
FFTCONV_LIB=$PWD/paper_2311_05908_b200/ablate/libfftconv_g4d.so timeout 600 python -m pytest tests/test_gpu_fwd.py -q -x -k "order3" 2>&1 | tail -1
