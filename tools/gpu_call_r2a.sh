set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/b4.log 2>&1; echo b4_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/b2.log 2>&1; echo b2_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_l4.log 2>&1; echo l4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"Onesweep|k_run_expand|k_hist_dD|k_sd_downsweep|k_chain_hash|k_link_tile|k_access_info" -s 0 -c 12 -o gpurun_out/full_c2 python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_f2.log 2>&1; echo f2_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_replay" -c 3 -o gpurun_out/full_k6 python tools/diag_replay.py 10000 512 > gpurun_out/ncu_k6.log 2>&1; echo k6_rc=$?
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo mem_rc=$?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1; echo race_rc=$?
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/san_synccheck.log 2>&1; echo sync_rc=$?
