python -m pytest tests/test_dense_gram.py tests/test_gpu_parity.py tests/test_vcycle.py tests/test_sharded_gpu.py -x -q 2>&1 | tail -4
