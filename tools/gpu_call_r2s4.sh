python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(cd old_tree && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1)
timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s4_b2_new.log 2>&1; echo new_rc=$?
(cd old_tree && timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > ../gpurun_out/s4_b2_old.log 2>&1; echo old_rc=$?)
KARETO_HOSTTIME=2 timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s4_b2_ht.log 2>&1; echo ht_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_bucket_link|k_access_info' --csv --log-file gpurun_out/s4_ncu_link.csv python bench.py --config 2 --profile-only --steps 1 --warmup 1 > gpurun_out/s4_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k4_runs or medium or config1" > gpurun_out/s4_tests.log 2>&1; echo t_rc=$?
