python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_hash|k_bucket_link|k_hist_dD|k_access_info|k_bucket_assemble" -c 5 -o gpurun_out/full_c4p python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_f4p.log 2>&1; echo f4p_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_hash|k_bucket_link|k_hist_dD|k_bucket_assemble" -c 4 -o gpurun_out/full_c2p python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_f2p.log 2>&1; echo f2p_rc=$?
timeout 900 python bench.py --config 2 --ttl > gpurun_out/ttl_p.log 2>&1; echo ttl_rc=$?
timeout 900 python bench.py --config 2 --search > gpurun_out/search_p.log 2>&1; echo search_rc=$?
