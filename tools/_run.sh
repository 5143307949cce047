set -x
python tools/probe_block.py 2>&1 | tail -2
python tools/probe_dense_multi.py 2>&1 | tail -3
RMG_NO_GRAPH=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg3_batch.csv python tools/probe_cfg3_batch.py 1 > gpurun_out/cfg3_batch.log 2>&1
tail -4 gpurun_out/cfg3_batch.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name regex:'k_spmm|k_xt_|k_hot_fold|k_block_finish|k_vperm_block' --launch-skip 18 -c 9 --csv --log-file gpurun_out/blk_dram.csv python tools/probe_block.py 5 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_spmm_k1v3|k_xt_hotblk|k_xt_block' --launch-skip 9 -c 4 -f -o gpurun_out/blk_full python tools/probe_block.py 5 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_xtb_dmma|k_syrk_dmma|k_gram_gemm_dmma' -c 4 -f -o gpurun_out/dense_multi_full python tools/probe_dense_multi.py > /dev/null 2>&1
ls -la gpurun_out | tail -8
