python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist_dD|k_hist_ttl" -c 2 -o gpurun_out/full_k4x python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_k4x.log 2>&1; echo k4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist_dD" -c 1 -o gpurun_out/full_k4x2 python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_k4x2.log 2>&1; echo k4b_rc=$?
