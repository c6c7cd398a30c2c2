FFTCONV_DIT=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench11_dit.json 2> gpurun_out/bench11.err
tail -c 300 gpurun_out/bench11_dit.json
