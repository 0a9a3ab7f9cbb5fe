python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_nccl.py -x -q > gpurun_out/t_r.log 2>&1; echo t_rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b4_r.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/b2_r.log 2>&1; echo b2_rc=$?
