python -m pytest tests/test_block_solve.py tests/test_vcycle.py tests/test_cfg3_parity.py tests/test_cpp_client.py tests/test_capi_cpu.py -x -q 2>&1 | tail -3
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
