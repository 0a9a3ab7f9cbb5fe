python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/t_all_y.log 2>&1; echo all_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_y.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/final2_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/final2_b2.log 2>&1; echo b2_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c4y.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_l4y.log 2>&1; echo l4_rc=$?
