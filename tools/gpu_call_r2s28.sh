python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grid.py tests/test_gpu_shard.py tests/test_gpu_fullsize.py -x -q -k "not config3" > gpurun_out/s28_tests.log 2>&1; echo t_rc=$?
timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s28_b4.log 2>&1; echo b4_rc=$?
timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s28_b2.log 2>&1; echo b2_rc=$?
