for r in 1 2; do for w in sweep8192 gsweep8192; do
STEPS=200 bash tools/variant.sh run "main cplunroll" $w 2>&1
done; done
FFTCONV_LIB=$PWD/paper_2311_05908_b200/ablate/libfftconv_cplunroll.so timeout 200 python -u tools/r02/cpl_check.py 8192 2>&1 | grep rel
