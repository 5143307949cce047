ncu --set full --import-source on --clock-control none --kernel-name regex:'k_xtb_dmma|k_xtb_finish|k_bcol2row16' --launch-skip 6 -c 3 -f -o gpurun_out/xtb_full python tools/probe_dense_multi.py > gpurun_out/xtb_probe.log 2>&1
tail -3 gpurun_out/xtb_probe.log
