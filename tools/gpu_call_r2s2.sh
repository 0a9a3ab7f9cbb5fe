python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/s2_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s2_b2.log 2>&1; echo b2_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_tests.log 2>&1; echo t_rc=$?
