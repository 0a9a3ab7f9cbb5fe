# K2 bucket link v2 (chunked buckets + fixup), default pool: focused tests, then benches
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --durations=5 > gpurun_out/t_par_c.log 2>&1; echo par_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b2_c.log 2>&1; echo b2_rc=$?
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/b4_c.log 2>&1; echo b4_rc=$?
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_nccl.py tests/test_gpu_fullsize.py -x -q --durations=5 > gpurun_out/t_sh_c.log 2>&1; echo sh_rc=$?
