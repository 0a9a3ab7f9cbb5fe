python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_DEBUG=1 timeout 2700 python tools/config3_fullsize_sample.py --ttl-groups 2 --oracle-sample 16 > gpurun_out/s36_c3ttl.log 2>&1; echo c3ttl_rc=$?
