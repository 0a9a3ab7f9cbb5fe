python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s29_tests.log 2>&1; echo all_rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s29_smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/s29_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/s29_b2.log 2>&1; echo b2_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s29_ref4.log 2>&1; echo ref_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s29_launches_c4.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/s29_l4.log 2>&1; echo l4_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s29_launches_c2.csv python bench.py --config 2 --profile-only --steps 1 --warmup 3 > gpurun_out/s29_l2.log 2>&1; echo l2_rc=$?
