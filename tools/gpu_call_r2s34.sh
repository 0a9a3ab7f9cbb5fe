python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_replay_waves.py tests/test_gpu_parity.py tests/test_gpu_queue.py -x -q > gpurun_out/s34_tests.log 2>&1; echo t_rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k config3 > gpurun_out/s34_fs3.log 2>&1; echo fs3_rc=$?
KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s34_b3.log 2>&1; echo b3_rc=$?
KARETO_K6_COLLAPSE=1 KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s34_b3c.log 2>&1; echo b3c_rc=$?
