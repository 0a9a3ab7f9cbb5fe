python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bucket|Onesweep|k_access|k_chain" -c 200 --csv --log-file gpurun_out/launches_ht4.csv python tools/host_time.py 4 > gpurun_out/ncu_ht4.log 2>&1; echo ncu_rc=$?
