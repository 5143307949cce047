python -m pytest tests/test_block_operator.py tests/test_block_solve.py tests/test_dense_operator.py -q 2>&1 | tail -5
