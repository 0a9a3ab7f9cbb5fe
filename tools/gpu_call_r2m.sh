python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_HOSTTIME=2 KARETO_HOST_TIMING=1 timeout 600 python tools/host_time.py 4 > gpurun_out/ht4_m.log 2>&1; echo ht_rc=$?
KARETO_HOSTTIME=1 timeout 600 python tools/host_time.py 4 > gpurun_out/ht4_m_sync.log 2>&1; echo ht_rc=$?
