python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/host_time.py 2 > gpurun_out/ht2_nosync.log 2>&1; echo ht_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 --steps 5 > gpurun_out/b2_e.log 2>&1; echo b2_rc=$?
KARETO_HOSTTIME=1 timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/b2_e_ht.log 2>&1; echo b2ht_rc=$?
KARETO_K2_FULLSORT=1 timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 --steps 5 > gpurun_out/b2_e_full.log 2>&1; echo b2f_rc=$?
