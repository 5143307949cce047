python -m pytest tests/test_sketch.py tests/test_dense_setup.py tests/test_kmeans_gpu.py tests/test_sharded_dense_gpu.py -x -q 2>&1 | tail -4
