python -m pytest tests/test_block_operator.py tests/test_block_solve.py -x -q 2>&1 | tail -2
python tools/probe_block.py 2>&1 | tail -2
for h in 3 2; do echo HOTXT=$h; RMG_BLOCK_HOTXT=$h python tools/probe_block.py 2>&1 | tail -2; done
for c in 344064 262144 172032; do echo CHUNK_ROWS=$c; RMG_BLOCK_CHUNK_ROWS=$c python tools/probe_block.py 2>&1 | tail -2; done
echo CHUNK_ROWS=344064 HOTXT=2; RMG_BLOCK_HOTXT=2 RMG_BLOCK_CHUNK_ROWS=344064 python tools/probe_block.py 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'k_spmm|k_xt_|k_hot_fold|k_block_finish|k_vperm_block' -c 60 --csv --log-file gpurun_out/blk_launch_2.csv python tools/probe_block.py 5 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/blk_launch_2.csv
