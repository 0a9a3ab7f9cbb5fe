python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grid.py tests/test_gpu_fullsize.py -x -q -k "selection or config1 or tiny or prepared or config4 or million or w1 or edge" > gpurun_out/s25_tests.log 2>&1; echo t_rc=$?
timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s25_b4.log 2>&1; echo b4_rc=$?
