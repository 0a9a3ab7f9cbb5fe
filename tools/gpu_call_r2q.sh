python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/final_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/final_b2.log 2>&1; echo b2_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref4.log 2>&1; echo ref4_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c4q.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_l4q.log 2>&1; echo l4_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2q.csv python bench.py --config 2 --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_l2q.log 2>&1; echo l2_rc=$?
timeout 1500 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_b3.log 2>&1; echo b3_rc=$?
