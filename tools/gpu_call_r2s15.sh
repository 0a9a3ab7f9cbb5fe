python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bucket_link" -c 1 -o gpurun_out/s15_link_c2 python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/s15_ncu.log 2>&1; echo ncu_rc=$?
