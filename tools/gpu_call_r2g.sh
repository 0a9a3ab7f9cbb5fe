python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_POOLSTAT=1 timeout 600 python tools/host_time.py 4 > gpurun_out/ht4_g.log 2>&1; echo ht_rc=$?
KARETO_POOLSTAT=1 KARETO_K2_FULLSORT=1 timeout 600 python tools/host_time.py 4 > gpurun_out/ht4_g_full.log 2>&1; echo htf_rc=$?
