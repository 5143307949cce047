for h in 3 2; do echo HOT_MIN=$h; RMG_HOT_MIN=$h python tools/probe_operator.py cfg5shard 2>&1 | grep -E "cold|hybrid"; done
