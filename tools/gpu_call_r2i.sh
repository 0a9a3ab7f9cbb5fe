python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/host_time.py 4 > gpurun_out/ht4_i.log 2>&1; echo ht_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k2 or medium or tiny or fingerprint or hash_mode" > gpurun_out/t_par_i.log 2>&1; echo par_rc=$?
