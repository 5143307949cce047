python -m pytest tests/test_sharded_gpu.py tests/test_sharded_dense_gpu.py tests/test_sharding.py -x -q 2>&1 | tail -8
