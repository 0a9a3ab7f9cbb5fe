# round-2 GPU call: new K2 bucket link, NCCL 1-rank path, cost-weighted shards -- tests, then benches
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/t_all_b.log 2>&1; echo all_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/b2_b.log 2>&1; echo b2_rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b4_b.log 2>&1; echo b4_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.log 2>&1; echo smoke_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"Onesweep|k_bucket_link|k_bucket_assemble|k_bucket_bounds|k_run_expand|k_hist_dD|k_sd_downsweep|k_access_info" -c 26 -o gpurun_out/full_c2b python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_f2b.log 2>&1; echo f2b_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4b.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_l4b.log 2>&1; echo l4b_rc=$?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py trace > gpurun_out/san_racecheck_trace.log 2>&1; echo race_t_rc=$?
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck_b.log 2>&1; echo mem_rc=$?
