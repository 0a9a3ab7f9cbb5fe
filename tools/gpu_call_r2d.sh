python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_HOSTTIME=1 timeout 600 python tools/host_time.py 2 > gpurun_out/ht2.log 2>&1; echo ht2_rc=$?
KARETO_HOSTTIME=1 KARETO_K2_FULLSORT=1 timeout 600 python tools/host_time.py 2 > gpurun_out/ht2_full.log 2>&1; echo ht2f_rc=$?
