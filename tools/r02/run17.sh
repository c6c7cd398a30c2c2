FFTCONV_DIT=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench17_dit.json 2> gpurun_out/bench17.err
tail -c 200 gpurun_out/bench17_dit.json
