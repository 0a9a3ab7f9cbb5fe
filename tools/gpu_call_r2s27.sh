python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grid.py tests/test_gpu_search.py -x -q -k "selection or config1 or tiny or prepared or w1 or edge or search or agent" > gpurun_out/s27_tests.log 2>&1; echo t_rc=$?
timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s27_b2.log 2>&1; echo b2_rc=$?
