python -m pytest tests/test_block_operator.py -x -q 2>&1 | tail -8
