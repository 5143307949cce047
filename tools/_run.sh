python -m pytest tests/test_block_operator.py tests/test_block_solve.py -x -q 2>&1 | tail -2
python tools/probe_block.py 2>&1 | tail -2
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_spmv_sell|k_xt_hot|k_xt<|k_vperm|k_xt_finish|k_xt_hot_final|k_xt_hot_chunks' --launch-skip 30 -c 8 -f -o gpurun_out/op5_full python tools/probe_operator.py cfg5shard > gpurun_out/op5_probe.log 2>&1
tail -5 gpurun_out/op5_probe.log
