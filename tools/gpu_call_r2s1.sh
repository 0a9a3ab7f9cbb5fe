python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s1_tests.log 2>&1; echo t_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s1_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s1_b4.log 2>&1; echo b4_rc=$?
