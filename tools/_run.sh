for c in 3 4 5; do echo XT_BLOCK_CTAS=$c; RMG_XT_BLOCK_CTAS=$c python tools/probe_block.py 2>&1 | tail -2; done
