python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/s8_tests.log 2>&1; echo all_rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s8_smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/s8_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/s8_b2.log 2>&1; echo b2_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s8_launches_c4.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/s8_ncu_l4.log 2>&1; echo l4_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s8_launches_c2.csv python bench.py --config 2 --profile-only --steps 1 --warmup 3 > gpurun_out/s8_ncu_l2.log 2>&1; echo l2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist_runs|k_bucket_link|k_chain_hash" -c 3 -o gpurun_out/s8_full_c4 python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/s8_ncu_full4.log 2>&1; echo f4_rc=$?
