timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_bidir.py tests/test_gpu_shard.py tests/test_gpu_host.py -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()"
