set -x
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_spmm_k1v2|k_xt_hotblk|k_xt_block' --launch-skip 6 -c 4 -f -o gpurun_out/blk_full python tools/probe_block.py 5 > /dev/null 2>&1
ls -la gpurun_out/
