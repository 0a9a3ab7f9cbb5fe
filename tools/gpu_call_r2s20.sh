python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_search.py -x -q > gpurun_out/s20_tests.log 2>&1; echo t_rc=$?
