python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --e2e-steps 0 --cpu-full 0 > gpurun_out/s31_b3.log 2>&1; echo b3_rc=$?
timeout 900 python bench.py --config 2 --ttl > gpurun_out/s31_ttl.log 2>&1; echo ttl_rc=$?
timeout 900 python bench.py --config 2 --queue > gpurun_out/s31_queue.log 2>&1; echo q_rc=$?
timeout 600 python bench.py --config 2 --analytics > gpurun_out/s31_an2.log 2>&1; echo a2_rc=$?
timeout 600 python bench.py --analytics > gpurun_out/s31_an4.log 2>&1; echo a4_rc=$?
