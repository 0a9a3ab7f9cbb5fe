python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_replay_waves.py tests/test_gpu_queue.py tests/test_gpu_shard.py -x -q -k "replay or waves or queue or budget or sequential or shard" > gpurun_out/s12_tests.log 2>&1; echo t_rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k config3 > gpurun_out/s12_fs3.log 2>&1; echo fs3_rc=$?
KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s12_b3.log 2>&1; echo b3_rc=$?
