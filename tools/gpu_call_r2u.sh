python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 5 > gpurun_out/b4_u.log 2>&1; echo b4_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "medium or tiny or k2" > gpurun_out/t_u.log 2>&1; echo t_rc=$?
