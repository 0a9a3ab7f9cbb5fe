python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist_dD|k_access_info|k_sd_downsweep" -c 4 -o gpurun_out/full_k4 python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_k4.log 2>&1; echo k4_rc=$?
