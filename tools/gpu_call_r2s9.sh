python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/s9_b4e2e.log 2>&1; echo b4_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hash_mode or config1 or edge or errors" > gpurun_out/s9_tests.log 2>&1; echo t_rc=$?
KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s9_b3.log 2>&1; echo b3_rc=$?
KARETO_DEBUG=1 timeout 2400 python tools/config3_fullsize_sample.py --per-cell 12 > gpurun_out/s9_c3full.log 2>&1; echo c3full_rc=$?
