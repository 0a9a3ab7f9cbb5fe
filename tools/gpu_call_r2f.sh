python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_par_f.log 2>&1; echo par_rc=$?
timeout 600 python tools/host_time.py 2 > gpurun_out/ht2_f.log 2>&1; echo ht_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b2_f.log 2>&1; echo b2_rc=$?
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/b4_f.log 2>&1; echo b4_rc=$?
