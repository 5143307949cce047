python -m pytest tests/test_hybrid_xt.py tests/test_full_scale.py -x -q -k "hybrid or cfg5" 2>&1 | tail -4
python tools/probe_operator.py cfg5shard 2>&1 | grep -E "cold|warm|numpy"
echo HOT_ONE; 
