python -m pytest tests/test_gpu_parity.py tests/test_cfg3_parity.py tests/test_hybrid_xt.py tests/test_full_scale.py -x -q 2>&1 | tail -4
