python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s35_tests.log 2>&1; echo all_rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s35_smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/s35_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/s35_b2.log 2>&1; echo b2_rc=$?
